// experiment: binned-SAH binary BVH with single-primitive leaves, in the
// GPU arena's binary node format (4 float4: lo_l|cl, hi_l|cr, lo_r, hi_r)
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#define NB 32
static const float *L, *H;
static int32_t *idx;
static float *cen;
static float *nodes;
static int32_t *parents;
static int64_t nn, N;
static void box_of(int64_t a, int64_t b, float *lo, float *hi) {
  for (int k = 0; k < 3; ++k) { lo[k] = INFINITY; hi[k] = -INFINITY; }
  for (int64_t p = a; p < b; ++p) { int32_t i = idx[p];
    for (int k = 0; k < 3; ++k) { if (L[3*i+k] < lo[k]) lo[k] = L[3*i+k]; if (H[3*i+k] > hi[k]) hi[k] = H[3*i+k]; } }
}
static float area(const float *lo, const float *hi) {
  float dx = hi[0]-lo[0], dy = hi[1]-lo[1], dz = hi[2]-lo[2];
  if (dx < 0) return 0; return dx*dy + dy*dz + dz*dx;
}
// returns child ref: leaf -> ~prim, internal -> node id
static int32_t build(int64_t a, int64_t b, int32_t parent) {
  if (b - a == 1) { int32_t prim = idx[a]; parents[(N-1) + prim] = parent; return ~prim; }
  int32_t node = (int32_t)(nn++);
  parents[node] = parent;
  float cmin[3] = {INFINITY,INFINITY,INFINITY}, cmax[3] = {-INFINITY,-INFINITY,-INFINITY};
  for (int64_t p = a; p < b; ++p) { int32_t i = idx[p];
    for (int k = 0; k < 3; ++k) { float c = cen[3*i+k]; if (c < cmin[k]) cmin[k] = c; if (c > cmax[k]) cmax[k] = c; } }
  float best = INFINITY; int bax = -1, bsplit = -1;
  for (int ax = 0; ax < 3; ++ax) {
    float ext = cmax[ax] - cmin[ax];
    if (!(ext > 0)) continue;
    int cnt[NB] = {0}; float blo[NB][3], bhi[NB][3];
    for (int q = 0; q < NB; ++q) for (int k = 0; k < 3; ++k) { blo[q][k] = INFINITY; bhi[q][k] = -INFINITY; }
    for (int64_t p = a; p < b; ++p) { int32_t i = idx[p];
      int q = (int)((cen[3*i+ax] - cmin[ax]) / ext * NB); if (q >= NB) q = NB-1; if (q < 0) q = 0;
      cnt[q]++;
      for (int k = 0; k < 3; ++k) { if (L[3*i+k] < blo[q][k]) blo[q][k] = L[3*i+k]; if (H[3*i+k] > bhi[q][k]) bhi[q][k] = H[3*i+k]; } }
    float rl[NB][3], rh[NB][3]; int rc[NB];
    float ll[3] = {INFINITY,INFINITY,INFINITY}, lh[3] = {-INFINITY,-INFINITY,-INFINITY}; int lc = 0;
    float al[NB]; int cl[NB];
    for (int q = 0; q < NB - 1; ++q) { lc += cnt[q];
      for (int k = 0; k < 3; ++k) { if (blo[q][k] < ll[k]) ll[k] = blo[q][k]; if (bhi[q][k] > lh[k]) lh[k] = bhi[q][k]; }
      al[q] = area(ll, lh); cl[q] = lc; }
    float r_l[3] = {INFINITY,INFINITY,INFINITY}, r_h[3] = {-INFINITY,-INFINITY,-INFINITY}; int rcnt = 0;
    for (int q = NB - 1; q >= 1; --q) { rcnt += cnt[q];
      for (int k = 0; k < 3; ++k) { if (blo[q][k] < r_l[k]) r_l[k] = blo[q][k]; if (bhi[q][k] > r_h[k]) r_h[k] = bhi[q][k]; }
      if (cl[q-1] == 0 || rcnt == 0) continue;
      float cost = al[q-1] * cl[q-1] + area(r_l, r_h) * rcnt;
      if (cost < best) { best = cost; bax = ax; bsplit = q; } }
    (void)rl; (void)rh; (void)rc;
  }
  int64_t mid;
  if (bax < 0) { mid = (a + b) / 2; }
  else {
    float ext = cmax[bax] - cmin[bax];
    int64_t i0 = a, i1 = b - 1;
    while (i0 <= i1) {
      int32_t i = idx[i0];
      int q = (int)((cen[3*i+bax] - cmin[bax]) / ext * NB); if (q >= NB) q = NB-1; if (q < 0) q = 0;
      if (q < bsplit) ++i0; else { int32_t t = idx[i0]; idx[i0] = idx[i1]; idx[i1] = t; --i1; }
    }
    mid = i0;
    if (mid == a || mid == b) mid = (a + b) / 2;
  }
  int32_t c0 = build(a, mid, node), c1 = build(mid, b, node);
  float lo0[3], hi0[3], lo1[3], hi1[3];
  box_of(a, mid, lo0, hi0); box_of(mid, b, lo1, hi1);
  float *nd = nodes + 16 * (int64_t)node;
  nd[0]=lo0[0]; nd[1]=lo0[1]; nd[2]=lo0[2]; memcpy(nd+3, &c0, 4);
  nd[4]=hi0[0]; nd[5]=hi0[1]; nd[6]=hi0[2]; memcpy(nd+7, &c1, 4);
  nd[8]=lo1[0]; nd[9]=lo1[1]; nd[10]=lo1[2]; nd[11]=0;
  nd[12]=hi1[0]; nd[13]=hi1[1]; nd[14]=hi1[2]; nd[15]=0;
  return node;
}
int sah_build(int64_t n, const float *lo, const float *hi, float *nodes_out, int32_t *parents_out) {
  N = n; L = lo; H = hi; nodes = nodes_out; parents = parents_out; nn = 0;
  idx = malloc(sizeof(int32_t) * n); cen = malloc(sizeof(float) * 3 * n);
  for (int64_t i = 0; i < n; ++i) { idx[i] = (int32_t)i; for (int k = 0; k < 3; ++k) cen[3*i+k] = 0.5f*(lo[3*i+k]+hi[3*i+k]); }
  build(0, n, -1);
  free(idx); free(cen);
  return (int)nn;
}
