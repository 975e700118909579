/*
 * gsray_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A float64 CPU restatement of the reference `gsray` render path
 * (/root/reference/pkg/src/gsray, pure Python/numpy).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library.  The product path (paper_2509_07782_b200) never does.
 *
 * Parity: pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src in the build
 * container and writes tests/golden/ fixtures; tests/test_oracle_golden.py checks
 * this file against them).
 *
 * Every function cites the reference file:line it restates.  Arithmetic is
 * IEEE double with contraction disabled (-ffp-contract=off) so that the
 * integer/ordering outputs (Morton codes, stable permutation, candidate sets)
 * are bit-exact and the floating outputs agree with numpy to a few ulp.
 *
 * Additions the reference does not have:
 *   - per-pixel depth  D = sum_j w_j t_j with w_j from renderer.py:236;
 *   - an analytic float64 backward (gradients w.r.t. the 87-float record),
 *     holding the discrete structure (sample grid, candidate sets, truncation
 *     mask, adaptive steps, ESS jumps, termination) fixed.  Pinned by central
 *     finite differences of this file's own forward (tests/test_oracle_grad.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NREC 87
#define NSH 9
#define NSG 7
#define NCOEF 76 /* sh 27 + axes 21 + sharp 7 + amp 21 */
#define S_MIN 1e-7 /* geometry.py:21 */
#define MORTON_BITS 21
#define MORTON_MAX ((1LL << MORTON_BITS) - 1) /* spatial.py:18-19 */

enum { OK = 0, ERR_EMPTY = 1, ERR_VALIDATION = 2, ERR_OVERFLOW = 3, ERR_ARG = 4 };

/* ------------------------------------------------------------------------ */
/* primitive math (geometry.py:26-42, 67-87; scene.py:48-69)                 */
/* ------------------------------------------------------------------------ */

/* np.linalg.norm of a short vector: sqrt(sum x_i^2), sequential order. */
static double vnorm(const double *x, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += x[i] * x[i];
  return sqrt(s);
}

/* geometry.py:26-42 quat_to_rotation (normalizes again). */
static void quat_to_rotation(const double *qin, double *R) {
  double n = vnorm(qin, 4);
  double w = qin[0] / n, x = qin[1] / n, y = qin[2] / n, z = qin[3] / n;
  R[0] = 1 - 2 * (y * y + z * z);
  R[1] = 2 * (x * y - w * z);
  R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);
  R[4] = 1 - 2 * (x * x + z * z);
  R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);
  R[7] = 2 * (y * z + w * x);
  R[8] = 1 - 2 * (x * x + y * y);
}

typedef struct {
  int64_t n;
  double sigma_eps;
  double *rec;      /* n*87 raw records (storage order) */
  double *means;    /* n*3 */
  double *quats;    /* n*4  normalized (GaussianShape, geometry.py:80) */
  double *rot;      /* n*9 */
  double *scales;   /* n*3  clamped (geometry.py:81) */
  double *sigmas;   /* n */
  double *log_ratio;/* n */
  double *iso_scales;/* n*3 */
  double *iso_inv;  /* n*9 */
  double *aabb_lo, *aabb_hi; /* n*3 */
  double *coeffs;   /* n*76: sh(27) axes(21, normalized) sharp(7) amp(21) */
  int64_t *uids;    /* n */
  double bounds_lo[3], bounds_hi[3];
  /* BVH (any conservative tree returns the same candidate sets as the
     reference's binned-SAH tree spatial.py:126-211; see segment_overlaps) */
  int64_t n_nodes;
  double *node_lo, *node_hi;
  int64_t *node_a, *node_b, *prim_order;
} oscene;

static void scene_free_arrays(oscene *s) {
  free(s->rec); free(s->means); free(s->quats); free(s->rot); free(s->scales);
  free(s->sigmas); free(s->log_ratio); free(s->iso_scales); free(s->iso_inv);
  free(s->aabb_lo); free(s->aabb_hi); free(s->coeffs); free(s->uids);
  free(s->node_lo); free(s->node_hi); free(s->node_a); free(s->node_b);
  free(s->prim_order);
}

/* ---- BVH: median split on the widest centroid axis, leaf <= 4 ---------- */
static double *g_sort_key;
static int cmp_key(const void *a, const void *b) {
  int64_t ia = *(const int64_t *)a, ib = *(const int64_t *)b;
  double ka = g_sort_key[ia], kb = g_sort_key[ib];
  if (ka < kb) return -1;
  if (ka > kb) return 1;
  return (ia < ib) ? -1 : (ia > ib);
}

static int64_t bvh_build_rec(oscene *s, int64_t start, int64_t end, double *cent,
                             double *key) {
  int64_t node = s->n_nodes++;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  double cmin[3] = {INFINITY, INFINITY, INFINITY}, cmax[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t p = start; p < end; ++p) {
    int64_t i = s->prim_order[p];
    for (int k = 0; k < 3; ++k) {
      if (s->aabb_lo[3 * i + k] < lo[k]) lo[k] = s->aabb_lo[3 * i + k];
      if (s->aabb_hi[3 * i + k] > hi[k]) hi[k] = s->aabb_hi[3 * i + k];
      if (cent[3 * i + k] < cmin[k]) cmin[k] = cent[3 * i + k];
      if (cent[3 * i + k] > cmax[k]) cmax[k] = cent[3 * i + k];
    }
  }
  memcpy(s->node_lo + 3 * node, lo, sizeof lo);
  memcpy(s->node_hi + 3 * node, hi, sizeof hi);
  int64_t count = end - start;
  if (count <= 4) {
    s->node_a[node] = start;
    s->node_b[node] = -count;
    return node;
  }
  int axis = 0;
  double ext = cmax[0] - cmin[0];
  for (int k = 1; k < 3; ++k)
    if (cmax[k] - cmin[k] > ext) { ext = cmax[k] - cmin[k]; axis = k; }
  for (int64_t p = start; p < end; ++p) {
    int64_t i = s->prim_order[p];
    key[i] = cent[3 * i + axis];
  }
  g_sort_key = key;
  qsort(s->prim_order + start, (size_t)count, sizeof(int64_t), cmp_key);
  int64_t mid = start + count / 2;
  int64_t l = bvh_build_rec(s, start, mid, cent, key);
  int64_t r = bvh_build_rec(s, mid, end, cent, key);
  s->node_a[node] = l;
  s->node_b[node] = r;
  return node;
}

static void bvh_build(oscene *s) {
  int64_t n = s->n;
  free(s->node_lo); free(s->node_hi); free(s->node_a); free(s->node_b); free(s->prim_order);
  s->node_lo = malloc(sizeof(double) * 3 * 2 * n);
  s->node_hi = malloc(sizeof(double) * 3 * 2 * n);
  s->node_a = malloc(sizeof(int64_t) * 2 * n);
  s->node_b = malloc(sizeof(int64_t) * 2 * n);
  s->prim_order = malloc(sizeof(int64_t) * n);
  for (int64_t i = 0; i < n; ++i) s->prim_order[i] = i;
  double *cent = malloc(sizeof(double) * 3 * n);
  double *key = malloc(sizeof(double) * n);
  for (int64_t i = 0; i < 3 * n; ++i) cent[i] = 0.5 * (s->aabb_lo[i] + s->aabb_hi[i]);
  s->n_nodes = 0;
  bvh_build_rec(s, 0, n, cent, key);
  free(cent);
  free(key);
}

/* scene.py:48-69 _rebuild + geometry.py:77-87 GaussianShape + appearance.py:62-76 */
static int scene_derive(oscene *s) {
  int64_t n = s->n;
  for (int64_t i = 0; i < n; ++i) {
    const double *r = s->rec + NREC * i;
    double *mu = s->means + 3 * i, *q = s->quats + 4 * i, *R = s->rot + 9 * i;
    double *sc = s->scales + 3 * i;
    for (int k = 0; k < 3; ++k) mu[k] = r[k];
    double qn = vnorm(r + 3, 4);
    if (!(qn >= 1e-12)) return -(int)(i + 1); /* zero quaternion: ValueError */
    for (int k = 0; k < 4; ++k) q[k] = r[3 + k] / qn; /* geometry.py:80 */
    quat_to_rotation(q, R);
    for (int k = 0; k < 3; ++k) sc[k] = r[7 + k] > S_MIN ? r[7 + k] : S_MIN; /* :81 */
    s->sigmas[i] = r[10];
    if (!(r[10] > s->sigma_eps)) return -(int)(i + 1); /* scene.py:37-41 */
    /* appearance.py:62-76: axes normalized, sharpness >= 0 */
    double *c = s->coeffs + NCOEF * i;
    memcpy(c, r + 11, sizeof(double) * 27);
    for (int l = 0; l < NSG; ++l) {
      const double *ax = r + 38 + 3 * l;
      double an = vnorm(ax, 3);
      if (!(an >= 1e-12)) return -(int)(i + 1);
      for (int k = 0; k < 3; ++k) c[27 + 3 * l + k] = ax[k] / an;
    }
    for (int l = 0; l < NSG; ++l) {
      if (r[59 + l] < 0) return -(int)(i + 1);
      c[48 + l] = r[59 + l];
    }
    memcpy(c + 55, r + 66, sizeof(double) * 21);
    /* scene.py:55-65 */
    double lr = 2.0 * log(s->sigmas[i] / s->sigma_eps);
    s->log_ratio[i] = lr;
    double sq = sqrt(lr);
    double *st = s->iso_scales + 3 * i, *M = s->iso_inv + 9 * i;
    for (int k = 0; k < 3; ++k) st[k] = sq * sc[k];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) M[3 * a + b] = R[3 * b + a] / st[a];
    for (int a = 0; a < 3; ++a) {
      double p0 = R[3 * a + 0] * st[0], p1 = R[3 * a + 1] * st[1], p2 = R[3 * a + 2] * st[2];
      double h = sqrt(p0 * p0 + p1 * p1 + p2 * p2);
      s->aabb_lo[3 * i + a] = mu[a] - h;
      s->aabb_hi[3 * i + a] = mu[a] + h;
    }
  }
  for (int k = 0; k < 3; ++k) {
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
      if (s->aabb_lo[3 * i + k] < lo) lo = s->aabb_lo[3 * i + k];
      if (s->aabb_hi[3 * i + k] > hi) hi = s->aabb_hi[3 * i + k];
    }
    s->bounds_lo[k] = lo;
    s->bounds_hi[k] = hi;
  }
  bvh_build(s);
  return 0;
}

/* Scene(shapes, coeffs, sigma_eps) from raw records, scene.py:25-46.
   Returns NULL and *status: 1 empty, 2 validation (record in *bad). */
void *oracle_scene_create(int64_t n, const double *records, double sigma_eps,
                          int *status, int64_t *bad) {
  *status = OK;
  *bad = -1;
  if (n <= 0) { *status = ERR_EMPTY; return NULL; }
  if (!(sigma_eps > 0)) { *status = ERR_VALIDATION; return NULL; }
  oscene *s = calloc(1, sizeof(oscene));
  s->n = n;
  s->sigma_eps = sigma_eps;
  s->rec = malloc(sizeof(double) * NREC * n);
  memcpy(s->rec, records, sizeof(double) * NREC * n);
  s->means = malloc(sizeof(double) * 3 * n);
  s->quats = malloc(sizeof(double) * 4 * n);
  s->rot = malloc(sizeof(double) * 9 * n);
  s->scales = malloc(sizeof(double) * 3 * n);
  s->sigmas = malloc(sizeof(double) * n);
  s->log_ratio = malloc(sizeof(double) * n);
  s->iso_scales = malloc(sizeof(double) * 3 * n);
  s->iso_inv = malloc(sizeof(double) * 9 * n);
  s->aabb_lo = malloc(sizeof(double) * 3 * n);
  s->aabb_hi = malloc(sizeof(double) * 3 * n);
  s->coeffs = malloc(sizeof(double) * NCOEF * n);
  s->uids = malloc(sizeof(int64_t) * n);
  for (int64_t i = 0; i < n; ++i) s->uids[i] = i; /* scene.py:45 */
  int rc = scene_derive(s);
  if (rc != 0) {
    *status = ERR_VALIDATION;
    *bad = (int64_t)(-rc) - 1;
    scene_free_arrays(s);
    free(s);
    return NULL;
  }
  return s;
}

void oracle_scene_free(void *h) {
  if (!h) return;
  scene_free_arrays((oscene *)h);
  free(h);
}

int64_t oracle_scene_size(void *h) { return ((oscene *)h)->n; }
int64_t oracle_scene_nodes(void *h) { return ((oscene *)h)->n_nodes; }

/* Copy a derived array out.  which: 0 means,1 rot,2 scales,3 sigmas,
   4 log_ratio,5 iso_scales,6 iso_inv,7 aabb_lo,8 aabb_hi,9 bounds(lo,hi),
   10 coeffs, 11 uids (as double), 12 records, 13 quats */
int oracle_scene_get(void *h, int which, double *out) {
  oscene *s = (oscene *)h;
  int64_t n = s->n;
  switch (which) {
    case 0: memcpy(out, s->means, sizeof(double) * 3 * n); break;
    case 1: memcpy(out, s->rot, sizeof(double) * 9 * n); break;
    case 2: memcpy(out, s->scales, sizeof(double) * 3 * n); break;
    case 3: memcpy(out, s->sigmas, sizeof(double) * n); break;
    case 4: memcpy(out, s->log_ratio, sizeof(double) * n); break;
    case 5: memcpy(out, s->iso_scales, sizeof(double) * 3 * n); break;
    case 6: memcpy(out, s->iso_inv, sizeof(double) * 9 * n); break;
    case 7: memcpy(out, s->aabb_lo, sizeof(double) * 3 * n); break;
    case 8: memcpy(out, s->aabb_hi, sizeof(double) * 3 * n); break;
    case 9: memcpy(out, s->bounds_lo, sizeof(double) * 3);
            memcpy(out + 3, s->bounds_hi, sizeof(double) * 3); break;
    case 10: memcpy(out, s->coeffs, sizeof(double) * NCOEF * n); break;
    case 11: for (int64_t i = 0; i < n; ++i) out[i] = (double)s->uids[i]; break;
    case 12: memcpy(out, s->rec, sizeof(double) * NREC * n); break;
    case 13: memcpy(out, s->quats, sizeof(double) * 4 * n); break;
    default: return ERR_ARG;
  }
  return OK;
}

/* ------------------------------------------------------------------------ */
/* Morton (spatial.py:28-92)                                                 */
/* ------------------------------------------------------------------------ */
static uint64_t spread21(uint64_t x) { /* spatial.py:28-35 */
  x &= (uint64_t)MORTON_MAX;
  x = (x | (x << 32)) & 0x1F00000000FFFFULL;
  x = (x | (x << 16)) & 0x1F0000FF0000FFULL;
  x = (x | (x << 8)) & 0x100F00F00F00F00FULL;
  x = (x | (x << 4)) & 0x10C30C30C30C30C3ULL;
  x = (x | (x << 2)) & 0x1249249249249249ULL;
  return x;
}
static uint64_t compact21(uint64_t x) { /* spatial.py:38-45 */
  x &= 0x1249249249249249ULL;
  x = (x | (x >> 2)) & 0x10C30C30C30C30C3ULL;
  x = (x | (x >> 4)) & 0x100F00F00F00F00FULL;
  x = (x | (x >> 8)) & 0x1F0000FF0000FFULL;
  x = (x | (x >> 16)) & 0x1F00000000FFFFULL;
  x = (x | (x >> 32)) & (uint64_t)MORTON_MAX;
  return x;
}

/* spatial.py:48-64; returns ERR_ARG when a coordinate is out of range (ValueError). */
int oracle_morton_encode(int64_t n, const int64_t *q, uint64_t *codes) {
  for (int64_t i = 0; i < 3 * n; ++i)
    if (q[i] < 0 || q[i] > MORTON_MAX) return ERR_ARG;
  for (int64_t i = 0; i < n; ++i)
    codes[i] = spread21((uint64_t)q[3 * i]) | (spread21((uint64_t)q[3 * i + 1]) << 1) |
               (spread21((uint64_t)q[3 * i + 2]) << 2);
  return OK;
}

/* spatial.py:67-78 */
void oracle_morton_decode(int64_t n, const uint64_t *codes, int64_t *q) {
  for (int64_t i = 0; i < n; ++i) {
    q[3 * i] = (int64_t)compact21(codes[i]);
    q[3 * i + 1] = (int64_t)compact21(codes[i] >> 1);
    q[3 * i + 2] = (int64_t)compact21(codes[i] >> 2);
  }
}

/* spatial.py:81-86 quantize_points */
void oracle_quantize(int64_t n, const double *pts, const double *lo, const double *hi,
                     int64_t *q) {
  double ext[3];
  for (int k = 0; k < 3; ++k) {
    double e = hi[k] - lo[k];
    ext[k] = e > 1e-30 ? e : 1e-30; /* np.maximum(hi - lo, 1e-30) */
  }
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      double t = (pts[3 * i + k] - lo[k]) / ext[k];
      double v = t * 2097152.0; /* t * (MORTON_MAX + 1) */
      int64_t qi = (int64_t)v; /* astype(int64): truncation toward zero */
      if (qi < 0) qi = 0;
      if (qi > MORTON_MAX) qi = MORTON_MAX;
      q[3 * i + k] = qi;
    }
}

/* stable argsort of u64 codes (np.argsort(kind="stable"), spatial.py:92): merge sort */
static void msort(int64_t *idx, int64_t *tmp, const uint64_t *key, int64_t n) {
  if (n < 2) return;
  int64_t m = n / 2;
  msort(idx, tmp, key, m);
  msort(idx + m, tmp, key, n - m);
  int64_t i = 0, j = m, k = 0;
  while (i < m && j < n) tmp[k++] = (key[idx[j]] < key[idx[i]]) ? idx[j++] : idx[i++];
  while (i < m) tmp[k++] = idx[i++];
  while (j < n) tmp[k++] = idx[j++];
  memcpy(idx, tmp, sizeof(int64_t) * n);
}
void oracle_stable_argsort_u64(int64_t n, const uint64_t *codes, int64_t *perm) {
  int64_t *tmp = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  msort(perm, tmp, codes, n);
  free(tmp);
}

/* spatial.py:89-92 morton_order */
void oracle_morton_order(int64_t n, const double *pts, const double *lo, const double *hi,
                         uint64_t *codes, int64_t *perm) {
  int64_t *q = malloc(sizeof(int64_t) * 3 * (n > 0 ? n : 1));
  oracle_quantize(n, pts, lo, hi, q);
  oracle_morton_encode(n, q, codes);
  oracle_stable_argsort_u64(n, codes, perm);
  free(q);
}

/* scene.py:74-80 apply_permutation: permute records + uids, rebuild derived. */
int oracle_scene_permute(void *h, const int64_t *perm) {
  oscene *s = (oscene *)h;
  int64_t n = s->n;
  double *rec = malloc(sizeof(double) * NREC * n);
  int64_t *uids = malloc(sizeof(int64_t) * n);
  for (int64_t p = 0; p < n; ++p) {
    memcpy(rec + NREC * p, s->rec + NREC * perm[p], sizeof(double) * NREC);
    uids[p] = s->uids[perm[p]];
  }
  free(s->rec);
  free(s->uids);
  s->rec = rec;
  s->uids = uids;
  return scene_derive(s) == 0 ? OK : ERR_VALIDATION;
}

/* scene.py:97-105 reorder_by_morton */
int oracle_scene_reorder_by_morton(void *h, int64_t *perm_out) {
  oscene *s = (oscene *)h;
  uint64_t *codes = malloc(sizeof(uint64_t) * s->n);
  oracle_morton_order(s->n, s->means, s->bounds_lo, s->bounds_hi, codes, perm_out);
  free(codes);
  return oracle_scene_permute(h, perm_out);
}

/* ------------------------------------------------------------------------ */
/* ray/box/ellipsoid queries (spatial.py:215-354)                           */
/* ------------------------------------------------------------------------ */
typedef struct {
  int64_t rays, samples, segments, segments_skipped, closest_hit_calls, node_visits,
      aabb_hits, ellipsoid_hits;
} ostats; /* renderer.py:69-106 */

/* spatial.py:258-277 _box_slab */
static void box_slab(const double *lo, const double *hi, const double *o, const double *d,
                     const double *inv, double *ta, double *tb) {
  double t0 = -INFINITY, t1 = INFINITY;
  for (int k = 0; k < 3; ++k) {
    if (d[k] != 0.0) {
      double a = (lo[k] - o[k]) * inv[k];
      double b = (hi[k] - o[k]) * inv[k];
      if (a > b) { double t = a; a = b; b = t; }
      if (a > t0) t0 = a;
      if (b < t1) t1 = b;
    } else if (o[k] < lo[k] || o[k] > hi[k]) {
      *ta = INFINITY;
      *tb = -INFINITY;
      return;
    }
  }
  *ta = t0;
  *tb = t1;
}

/* inverse direction used by segment_overlaps/closest_hit (spatial.py:227,321) */
static void inv_dir_traversal(const double *d, double *inv) {
  for (int k = 0; k < 3; ++k) inv[k] = fabs(d[k]) > 1e-300 ? 1.0 / (d[k] == 0.0 ? 1.0 : d[k]) : INFINITY;
}

/* spatial.py:280-306 ray_ellipsoid_interval (Kahan form) */
static int ray_ellipsoid_interval(const double *ol, const double *dl, double t_lo, double t_hi,
                                  double *tin, double *tout) {
  double a = dl[0] * dl[0] + dl[1] * dl[1] + dl[2] * dl[2];
  double b = ol[0] * dl[0] + ol[1] * dl[1] + ol[2] * dl[2];
  double c = (ol[0] * ol[0] + ol[1] * ol[1] + ol[2] * ol[2]) - 1.0;
  double disc = b * b - a * c;
  if (disc < 0.0 || a == 0.0) return 0;
  double sq = sqrt(disc);
  double q = (b >= 0.0) ? -(b + sq) : -(b - sq);
  double t0 = q / a;
  double t1 = (q != 0.0) ? c / q : t0;
  if (t0 > t1) { double t = t0; t0 = t1; t1 = t; }
  if (t_lo > t0) t0 = t_lo;
  if (t_hi < t1) t1 = t_hi;
  if (t0 > t1) return 0;
  *tin = t0;
  *tout = t1;
  return 1;
}

static void to_local(const oscene *s, int64_t i, const double *o, const double *d, double *ol,
                     double *dl) {
  const double *M = s->iso_inv + 9 * i, *mu = s->means + 3 * i;
  double v[3] = {o[0] - mu[0], o[1] - mu[1], o[2] - mu[2]};
  for (int a = 0; a < 3; ++a) {
    ol[a] = M[3 * a] * v[0] + M[3 * a + 1] * v[1] + M[3 * a + 2] * v[2];
    dl[a] = M[3 * a] * d[0] + M[3 * a + 1] * d[1] + M[3 * a + 2] * d[2];
  }
}

/* spatial.py:215-247 Bvh.segment_overlaps.  Any tree whose node boxes are the
   exact min/max of their primitives' boxes yields the reference's candidate
   SET (the slab test is monotone in lo/hi under IEEE rounding), so this tree
   differs from the SAH tree only in node_visits and output order.
   Returns count, or -(count) when count would exceed capacity (BufferOverflow). */
static int64_t segment_overlaps(const oscene *s, const double *o, const double *d, double t0,
                                double t1, int64_t cap, int64_t *out, ostats *st) {
  double inv[3];
  inv_dir_traversal(d, inv);
  int64_t stack[128];
  int sp = 0;
  int64_t count = 0, visits = 0;
  stack[sp++] = 0;
  while (sp > 0) {
    int64_t node = stack[--sp];
    visits++;
    double a, b;
    box_slab(s->node_lo + 3 * node, s->node_hi + 3 * node, o, d, inv, &a, &b);
    if (a > t1 || b < t0) continue;
    int64_t na = s->node_a[node], nb = s->node_b[node];
    if (nb <= 0) {
      for (int64_t p = na; p < na - nb; ++p) {
        int64_t i = s->prim_order[p];
        double pa, pb;
        box_slab(s->aabb_lo + 3 * i, s->aabb_hi + 3 * i, o, d, inv, &pa, &pb);
        if (pa <= t1 && pb >= t0) {
          if (count >= cap) {
            if (st) st->node_visits += visits;
            return -(count + 1);
          }
          out[count++] = i;
        }
      }
      continue;
    }
    stack[sp++] = nb;
    stack[sp++] = na;
  }
  if (st) st->node_visits += visits;
  return count;
}

/* spatial.py:309-354 closest_hit; returns 1 and *t when hit. */
static int closest_hit(const oscene *s, const double *o, const double *d, double t_lo,
                       double t_hi, double *t, ostats *st) {
  if (t_lo > t_hi) return 0;
  double inv[3];
  inv_dir_traversal(d, inv);
  double best = INFINITY;
  int64_t snode[128];
  double sent[128];
  int sp = 0;
  int64_t visits = 0;
  snode[sp] = 0;
  sent[sp++] = 0.0;
  while (sp > 0) {
    --sp;
    int64_t node = snode[sp];
    double t_entry = sent[sp];
    if (t_entry >= best) continue;
    visits++;
    double a, b;
    box_slab(s->node_lo + 3 * node, s->node_hi + 3 * node, o, d, inv, &a, &b);
    double lim = t_hi < best ? t_hi : best;
    if (a > lim || b < t_lo) continue;
    int64_t na = s->node_a[node], nb = s->node_b[node];
    if (nb <= 0) {
      for (int64_t p = na; p < na - nb; ++p) {
        int64_t i = s->prim_order[p];
        double ol[3], dl[3], tin, tout;
        to_local(s, i, o, d, ol, dl);
        double lim2 = t_hi < best ? t_hi : best;
        if (ray_ellipsoid_interval(ol, dl, t_lo, lim2, &tin, &tout) && tin < best) best = tin;
      }
      continue;
    }
    double la, lb, dummy;
    box_slab(s->node_lo + 3 * na, s->node_hi + 3 * na, o, d, inv, &la, &dummy);
    box_slab(s->node_lo + 3 * nb, s->node_hi + 3 * nb, o, d, inv, &lb, &dummy);
    if (la <= lb) {
      snode[sp] = nb; sent[sp++] = lb;
      snode[sp] = na; sent[sp++] = la;
    } else {
      snode[sp] = na; sent[sp++] = la;
      snode[sp] = nb; sent[sp++] = lb;
    }
  }
  if (st) {
    st->node_visits += visits;
    st->closest_hit_calls += 1;
  }
  if (isfinite(best)) { *t = best; return 1; }
  return 0;
}

/* batch query wrappers for parity tests */
int64_t oracle_segment_overlaps(void *h, const double *o, const double *d, double t0, double t1,
                                int64_t cap, int64_t *out) {
  return segment_overlaps((oscene *)h, o, d, t0, t1, cap, out, NULL);
}
/* brute force: every primitive whose AABB slab interval overlaps [t0,t1]
   (test_acceptance.py:353-362 style), ascending storage index. */
int64_t oracle_segment_overlaps_brute(void *h, const double *o, const double *d, double t0,
                                      double t1, int64_t *out) {
  oscene *s = (oscene *)h;
  double inv[3];
  for (int k = 0; k < 3; ++k) inv[k] = d[k] == 0.0 ? INFINITY : 1.0 / d[k];
  int64_t c = 0;
  for (int64_t i = 0; i < s->n; ++i) {
    double a, b;
    box_slab(s->aabb_lo + 3 * i, s->aabb_hi + 3 * i, o, d, inv, &a, &b);
    if (a <= t1 && b >= t0) out[c++] = i;
  }
  return c;
}
int oracle_closest_hit(void *h, const double *o, const double *d, double t_lo, double t_hi,
                       double *t) {
  return closest_hit((oscene *)h, o, d, t_lo, t_hi, t, NULL);
}
int oracle_ray_ellipsoid_interval(const double *ol, const double *dl, double t_lo, double t_hi,
                                  double *out) {
  return ray_ellipsoid_interval(ol, dl, t_lo, t_hi, out, out + 1);
}

/* ------------------------------------------------------------------------ */
/* appearance (appearance.py:19-98)                                          */
/* ------------------------------------------------------------------------ */
#define C0 0.28209479177387814  /* 0.5*sqrt(1/pi) */
#define C1 0.4886025119029199   /* sqrt(3/(4pi)) */
#define C2A 1.0925484305920792  /* 0.5*sqrt(15/pi) */
#define C2B 0.31539156525252005 /* 0.25*sqrt(5/pi) */
#define C2C 0.5462742152960396  /* 0.25*sqrt(15/pi) */

static void sh_basis(const double *d, double *Y) { /* appearance.py:26-50 */
  double x = d[0], y = d[1], z = d[2];
  Y[0] = C0;
  Y[1] = C1 * y;
  Y[2] = C1 * z;
  Y[3] = C1 * x;
  Y[4] = C2A * x * y;
  Y[5] = C2A * y * z;
  Y[6] = C2B * (3.0 * z * z - 1.0);
  Y[7] = C2A * x * z;
  Y[8] = C2C * (x * x - y * y);
}

/* appearance.py:91-98 eval_radiance; pre[] receives the unclamped sum. */
static void eval_radiance(const double *c, const double *d, double *rgb, double *pre,
                          double *lobes) {
  double Y[9];
  sh_basis(d, Y);
  double acc[3] = {0, 0, 0};
  for (int ch = 0; ch < 3; ++ch) {
    double v = 0.0;
    for (int b = 0; b < 9; ++b) v += Y[b] * c[3 * b + ch];
    acc[ch] = v;
  }
  double lob[NSG];
  for (int l = 0; l < NSG; ++l) {
    const double *ax = c + 27 + 3 * l;
    double cs = ax[0] * d[0] + ax[1] * d[1] + ax[2] * d[2];
    lob[l] = exp(c[48 + l] * (cs - 1.0));
  }
  for (int ch = 0; ch < 3; ++ch) {
    double v = 0.0;
    for (int l = 0; l < NSG; ++l) v += lob[l] * c[55 + 3 * l + ch];
    acc[ch] = acc[ch] + v;
  }
  for (int ch = 0; ch < 3; ++ch) {
    if (pre) pre[ch] = acc[ch];
    rgb[ch] = acc[ch] > 0.0 ? acc[ch] : 0.0;
  }
  if (lobes) memcpy(lobes, lob, sizeof lob);
}

void oracle_eval_radiance(void *h, int64_t i, const double *d, double *rgb) {
  oscene *s = (oscene *)h;
  eval_radiance(s->coeffs + NCOEF * i, d, rgb, NULL, NULL);
}

/* ------------------------------------------------------------------------ */
/* renderer (renderer.py:27-393)                                             */
/* ------------------------------------------------------------------------ */
typedef struct { /* renderer.py:27-39 RenderConfig, field for field */
  double dt;
  int64_t n_s;
  double t_eps;
  int64_t adaptive; /* mode: 0 uniform, 1 adaptive */
  double beta, dt_min, dt_max;
  int64_t ess;
  int64_t tile_size; /* accepted, no effect on pixels */
  double background[3];
  int64_t buffer_capacity;
} ocfg;

/* optional backward tape: every composited sample in order */
typedef struct {
  int64_t n, cap;
  double *t;     /* sample position */
  double *dt;    /* sample width */
  int64_t *seg;  /* index into candidate segment lists */
  int64_t nseg, segcap;
  int64_t *seg_off, *seg_cnt; /* candidate lists per composited (sub)segment */
  int64_t ncand, candcap;
  int64_t *cand;
} otape;

static void tape_push_seg(otape *tp, const int64_t *active, int64_t na) {
  if (tp->nseg == tp->segcap) {
    tp->segcap = tp->segcap ? 2 * tp->segcap : 64;
    tp->seg_off = realloc(tp->seg_off, sizeof(int64_t) * tp->segcap);
    tp->seg_cnt = realloc(tp->seg_cnt, sizeof(int64_t) * tp->segcap);
  }
  while (tp->ncand + na > tp->candcap) {
    tp->candcap = tp->candcap ? 2 * tp->candcap : 256;
    tp->cand = realloc(tp->cand, sizeof(int64_t) * tp->candcap);
  }
  tp->seg_off[tp->nseg] = tp->ncand;
  tp->seg_cnt[tp->nseg] = na;
  memcpy(tp->cand + tp->ncand, active, sizeof(int64_t) * na);
  tp->ncand += na;
  tp->nseg++;
}
static void tape_push_sample(otape *tp, double t, double dt) {
  if (tp->n == tp->cap) {
    tp->cap = tp->cap ? 2 * tp->cap : 256;
    tp->t = realloc(tp->t, sizeof(double) * tp->cap);
    tp->dt = realloc(tp->dt, sizeof(double) * tp->cap);
    tp->seg = realloc(tp->seg, sizeof(int64_t) * tp->cap);
  }
  tp->t[tp->n] = t;
  tp->dt[tp->n] = dt;
  tp->seg[tp->n] = tp->nseg - 1;
  tp->n++;
}
static void tape_free(otape *tp) {
  free(tp->t); free(tp->dt); free(tp->seg); free(tp->seg_off); free(tp->seg_cnt); free(tp->cand);
}

typedef struct { /* renderer.py:178-240 _RayState */
  const oscene *s;
  const ocfg *cfg;
  double o[3], d[3];
  double color[3];
  double od;
  double depth;
  ostats *st;
  int64_t *buf;  /* capacity buffer */
  int64_t *big;  /* full-N buffer for unsplittable overflow (renderer.py:375-377) */
  double *rad;   /* per-ray radiance cache (renderer.py:200-205) */
  int64_t *stamp;/* rad[i] valid iff stamp[i] == ray_id */
  int64_t ray_id;
  otape *tape;
} oray;

static const double *radiance(oray *r, int64_t i) {
  double *c = r->rad + 3 * i;
  if (r->stamp[i] != r->ray_id) {
    eval_radiance(r->s->coeffs + NCOEF * i, r->d, c, NULL, NULL);
    r->stamp[i] = r->ray_id;
  }
  return c;
}

static const int64_t *g_uids;
static int cmp_uid(const void *a, const void *b) {
  int64_t ua = g_uids[*(const int64_t *)a], ub = g_uids[*(const int64_t *)b];
  return (ua > ub) - (ua < ub);
}

/* renderer.py:250-260 collect_sorted.  Returns count (0 = None), -1 on overflow. */
static int64_t collect_sorted(oray *r, double t0, double t1, int64_t *buf, int64_t cap) {
  int64_t n = segment_overlaps(r->s, r->o, r->d, t0, t1, cap, buf, r->st);
  if (n < 0) return -1;
  if (n == 0) return 0;
  /* uids are unique, so the stable sort equals any sort */
  g_uids = r->s->uids;
  qsort(buf, (size_t)n, sizeof(int64_t), cmp_uid);
  return n;
}

/* renderer.py:242-248 count_hits */
static void count_hits(oray *r, const int64_t *active, int64_t na, double t0, double t1) {
  r->st->aabb_hits += na;
  for (int64_t a = 0; a < na; ++a) {
    double ol[3], dl[3], ti, to;
    to_local(r->s, active[a], r->o, r->d, ol, dl);
    if (ray_ellipsoid_interval(ol, dl, t0, t1, &ti, &to)) r->st->ellipsoid_hits++;
  }
}

/* renderer.py:207-240 composite (+ depth) */
static void composite(oray *r, const int64_t *active, int64_t na, const double *ts, int64_t m,
                      double dt) {
  const oscene *s = r->s;
  double sigma[m > 0 ? m : 1], wsum[m > 0 ? 3 * m : 3];
  for (int64_t j = 0; j < m; ++j) { sigma[j] = 0.0; wsum[3*j] = wsum[3*j+1] = wsum[3*j+2] = 0.0; }
  for (int64_t a = 0; a < na; ++a) {
    int64_t i = active[a];
    const double *M = s->iso_inv + 9 * i, *mu = s->means + 3 * i;
    for (int64_t j = 0; j < m; ++j) {
      double x[3], v[3], y[3];
      for (int k = 0; k < 3; ++k) { x[k] = r->o[k] + ts[j] * r->d[k]; v[k] = x[k] - mu[k]; }
      for (int b = 0; b < 3; ++b) y[b] = v[0] * M[3 * b] + v[1] * M[3 * b + 1] + v[2] * M[3 * b + 2];
      double q = y[0] * y[0] + y[1] * y[1] + y[2] * y[2];
      if (q <= 1.0) {
        double dens = s->sigmas[i] * exp(-0.5 * s->log_ratio[i] * q);
        const double *c = radiance(r, i);
        sigma[j] += dens;
        for (int k = 0; k < 3; ++k) wsum[3 * j + k] += dens * c[k];
      }
    }
  }
  if (r->tape) tape_push_seg(r->tape, active, na);
  double od = r->od;
  for (int64_t j = 0; j < m; ++j) {
    double ods = sigma[j] * dt;
    if (sigma[j] > 0.0) {
      double w = -expm1(-ods) * exp(-od);
      for (int k = 0; k < 3; ++k) r->color[k] += (w / sigma[j]) * wsum[3 * j + k];
      r->depth += w * ts[j];
    }
    od += ods;
    if (r->tape) tape_push_sample(r->tape, ts[j], dt);
  }
  r->od = od;
  r->st->samples += m;
}

/* renderer.py:361-393 _collect_split.  Returns 0 None / 1 non-empty. */
static int collect_split(oray *r, double t0, double t1, const double *ts, int64_t m, double dt) {
  int64_t na = collect_sorted(r, t0, t1, r->buf, r->cfg->buffer_capacity);
  int64_t *active = r->buf;
  if (na < 0) {
    if (m <= 1) {
      na = collect_sorted(r, t0, t1, r->big, r->s->n);
      active = r->big;
    } else {
      double mid = 0.5 * (t0 + t1);
      int64_t nl = 0;
      while (nl < m && ts[nl] < mid) nl++; /* ts ascending: ts < mid | ts >= mid */
      int a = collect_split(r, t0, mid, ts, nl, dt);
      int b = collect_split(r, mid, t1, ts + nl, m - nl, dt);
      return (a || b) ? 1 : 0;
    }
  }
  if (na == 0) return 0;
  r->st->segments += 1;
  count_hits(r, active, na, t0, t1);
  if (m) {
    /* composite may reuse r->buf via recursion only after returning; copy */
    int64_t tmp[na];
    memcpy(tmp, active, sizeof(int64_t) * na);
    composite(r, tmp, na, ts, m, dt);
  }
  return 1;
}

/* renderer.py:148-157 segment_step */
double oracle_segment_step(const ocfg *cfg, double d_i, double t_i) {
  double t = t_i > cfg->t_eps ? t_i : cfg->t_eps;
  double boost = exp(-log(t) / 3.0);
  double a = d_i / cfg->beta;
  if (!(a > cfg->dt_min)) a = cfg->dt_min; /* max(d/beta, dt_min) */
  double step = a * boost;
  if (step > cfg->dt_max) step = cfg->dt_max;
  return (double)cfg->n_s * step;
}

/* renderer.py:288-323 _march_uniform */
static void march_uniform(oray *r, double t_n, double t_f) {
  const ocfg *cfg = r->cfg;
  double ds = cfg->dt * (double)cfg->n_s;
  int64_t n_seg = (int64_t)ceil((t_f - t_n) / ds);
  if (n_seg < 1) n_seg = 1;
  int64_t k = 0;
  if (cfg->ess) {
    double hit;
    if (!closest_hit(r->s, r->o, r->d, t_n, t_f, &hit, r->st)) return;
    int64_t kk = (int64_t)((hit - t_n) / ds);
    k = kk > 0 ? kk : 0;
  }
  int64_t ns = cfg->n_s;
  double ts[ns];
  while (k < n_seg && exp(-r->od) > cfg->t_eps) {
    double t0 = t_n + (double)k * ds;
    double t1 = t0 + ds;
    if (t_f < t1) t1 = t_f;
    int64_t j0 = k * ns, m = 0;
    for (int64_t j = j0; j < j0 + ns; ++j) {
      double t = t_n + ((double)j + 0.5) * cfg->dt;
      if (t < t_f) ts[m++] = t;
    }
    int act = collect_split(r, t0, t1, ts, m, cfg->dt);
    if (!act) {
      if (cfg->ess) {
        r->st->segments_skipped++;
        double hit;
        if (!closest_hit(r->s, r->o, r->d, t1, t_f, &hit, r->st)) return;
        int64_t kk = (int64_t)((hit - t_n) / ds);
        k = kk > k + 1 ? kk : k + 1;
      } else {
        r->st->samples += m;
        r->st->segments_skipped++;
        k += 1;
      }
      continue;
    }
    k += 1;
  }
}

/* renderer.py:326-358 _march_adaptive */
static void march_adaptive(oray *r, double t_n, double t_f) {
  const ocfg *cfg = r->cfg;
  double t_s = t_n;
  if (cfg->ess) {
    double hit;
    if (!closest_hit(r->s, r->o, r->d, t_n, t_f, &hit, r->st)) return;
    t_s = hit;
  }
  int64_t ns = cfg->n_s;
  double ts[ns];
  while (t_s < t_f && exp(-r->od) > cfg->t_eps) {
    double ds = oracle_segment_step(cfg, t_s, exp(-r->od));
    double dt = ds / (double)ns;
    double t1 = t_s + ds;
    if (t_f < t1) t1 = t_f;
    int64_t m = 0;
    for (int64_t j = 0; j < ns; ++j) {
      double t = t_s + ((double)j + 0.5) * dt;
      if (t < t_f) ts[m++] = t;
    }
    int act = collect_split(r, t_s, t1, ts, m, dt);
    if (!act) {
      if (cfg->ess) {
        r->st->segments_skipped++;
        double hit;
        if (!closest_hit(r->s, r->o, r->d, t1, t_f, &hit, r->st)) return;
        t_s = hit;
      } else {
        r->st->samples += m;
        r->st->segments_skipped++;
        t_s = t_s + ds;
      }
      continue;
    }
    t_s = t_s + ds;
  }
}

/* renderer.py:263-285 march_ray.  out: rgb[3], T, depth. */
static void march(const oscene *s, const ocfg *cfg, const double *o, const double *d, double t_n,
                  double t_f, double *out_rgb, double *out_T, double *out_depth, ostats *st,
                  int64_t *buf, int64_t *big, double *rad, int64_t *stamp, int64_t ray_id,
                  otape *tape) {
  st->rays += 1;
  if (t_n >= t_f) {
    for (int k = 0; k < 3; ++k) out_rgb[k] = cfg->background[k];
    *out_T = 1.0;
    *out_depth = 0.0;
    return;
  }
  oray r;
  memset(&r, 0, sizeof r);
  r.s = s;
  r.cfg = cfg;
  memcpy(r.o, o, sizeof r.o);
  memcpy(r.d, d, sizeof r.d);
  r.st = st;
  r.buf = buf;
  r.big = big;
  r.rad = rad;
  r.stamp = stamp;
  r.ray_id = ray_id;
  r.tape = tape;
  if (cfg->adaptive) march_adaptive(&r, t_n, t_f);
  else march_uniform(&r, t_n, t_f);
  double te = exp(-r.od);
  for (int k = 0; k < 3; ++k) out_rgb[k] = r.color[k] + te * cfg->background[k];
  *out_T = te;
  *out_depth = r.depth;
}

/* renderer.py:52-66 Ray direction renormalization + renderer.py:160-175 clip.
   Returns 0 when the ray misses the scene (None). */
static int clip_ray(const oscene *s, const double *o, double *d, double t_near, double t_far,
                    double *tn, double *tf) {
  double n = vnorm(d, 3);
  if (fabs(n - 1.0) > 1e-9)
    for (int k = 0; k < 3; ++k) d[k] = d[k] / n;
  if (t_near >= t_far) return 0;
  double inv[3];
  for (int k = 0; k < 3; ++k) inv[k] = d[k] == 0.0 ? INFINITY : 1.0 / d[k];
  double a, b;
  box_slab(s->bounds_lo, s->bounds_hi, o, d, inv, &a, &b);
  double t0 = t_near > a ? t_near : a;
  double t1 = t_far < b ? t_far : b;
  if (t0 >= t1) return 0;
  *tn = t0;
  *tf = t1;
  return 1;
}

/* march a batch of explicit rays (o, d, t_near, t_far); clip=1 applies
   clip_ray_to_scene first (render_image semantics), clip=0 marches as given
   (march_ray semantics).  stats: 8 int64 (renderer.py:69-78 order). */
typedef struct {
  const oscene *s;
  const ocfg *cfg;
  const double *rays; /* m*8: o(3), d(3), t_near, t_far */
  int64_t m, clip;
  double *rgb, *T, *depth;
  int64_t next;
  pthread_mutex_t mu;
  ostats total;
} batch_job;

static void *batch_worker(void *arg) {
  batch_job *jb = (batch_job *)arg;
  const oscene *s = jb->s;
  int64_t *buf = malloc(sizeof(int64_t) * (jb->cfg->buffer_capacity > 0 ? jb->cfg->buffer_capacity : 1));
  int64_t *big = malloc(sizeof(int64_t) * s->n);
  double *rad = malloc(sizeof(double) * 3 * s->n);
  int64_t *stamp = malloc(sizeof(int64_t) * s->n);
  for (int64_t i = 0; i < s->n; ++i) stamp[i] = -1;
  ostats st;
  memset(&st, 0, sizeof st);
  for (;;) {
    pthread_mutex_lock(&jb->mu);
    int64_t i0 = jb->next;
    jb->next += 16;
    pthread_mutex_unlock(&jb->mu);
    if (i0 >= jb->m) break;
    int64_t i1 = i0 + 16 < jb->m ? i0 + 16 : jb->m;
    for (int64_t i = i0; i < i1; ++i) {
      const double *ry = jb->rays + 8 * i;
      double o[3] = {ry[0], ry[1], ry[2]}, d[3] = {ry[3], ry[4], ry[5]};
      double tn = ry[6], tf = ry[7];
      if (jb->clip) {
        if (!clip_ray(s, o, d, ry[6], ry[7], &tn, &tf)) {
          st.rays += 1;
          for (int k = 0; k < 3; ++k) jb->rgb[3 * i + k] = jb->cfg->background[k];
          jb->T[i] = 1.0;
          jb->depth[i] = 0.0;
          continue;
        }
      } else {
        double n = vnorm(d, 3);
        if (fabs(n - 1.0) > 1e-9)
          for (int k = 0; k < 3; ++k) d[k] /= n;
      }
      march(s, jb->cfg, o, d, tn, tf, jb->rgb + 3 * i, jb->T + i, jb->depth + i, &st, buf, big,
            rad, stamp, i, NULL);
    }
  }
  pthread_mutex_lock(&jb->mu);
  int64_t *a = (int64_t *)&jb->total, *b = (int64_t *)&st;
  for (int k = 0; k < 8; ++k) a[k] += b[k];
  pthread_mutex_unlock(&jb->mu);
  free(buf);
  free(big);
  free(rad);
  free(stamp);
  return NULL;
}

int oracle_march_rays(void *h, const ocfg *cfg, int64_t m, const double *rays, int64_t clip,
                      int64_t threads, double *rgb, double *T, double *depth, int64_t *stats) {
  batch_job jb;
  memset(&jb, 0, sizeof jb);
  jb.s = (const oscene *)h;
  jb.cfg = cfg;
  jb.rays = rays;
  jb.m = m;
  jb.clip = clip;
  jb.rgb = rgb;
  jb.T = T;
  jb.depth = depth;
  pthread_mutex_init(&jb.mu, NULL);
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  for (int64_t t = 1; t < threads; ++t) pthread_create(&th[t], NULL, batch_worker, &jb);
  batch_worker(&jb);
  for (int64_t t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&jb.mu);
  if (stats) memcpy(stats, &jb.total, sizeof(ostats));
  return OK;
}

/* ------------------------------------------------------------------------ */
/* dense oracles (renderer.py:440-493, appearance.py:107-134)                */
/* ------------------------------------------------------------------------ */

/* primitive storage positions in ascending uid (the reference's
   np.argsort(uids, kind="stable") at renderer.py:456 / appearance.py:122) */
static int64_t *uid_order(const oscene *s) {
  int64_t *ord = malloc(sizeof(int64_t) * (s->n > 0 ? s->n : 1));
  for (int64_t i = 0; i < s->n; ++i) ord[s->uids[i]] = i;  /* uids are a permutation */
  return ord;
}

/* renderer.py:440-480 reference_integrate: midpoint quadrature at fine_dt
   over [t_near, t_far] against the full primitive list (uid order), then the
   vectorised compositing of lines 472-480 (cumsum, -expm1(-od) exp(-cum),
   sum over sigma > 0 of (w / sigma) * weighted, exit transmittance x bg). */
static void reference_integrate(const oscene *s, const int64_t *ord, const double *o,
                                const double *d, double t_near, double t_far, double fine_dt,
                                const double *bg, double *out) {
  for (int k = 0; k < 3; ++k) out[k] = bg[k];
  if (t_near >= t_far) return;
  int64_t n = (int64_t)ceil((t_far - t_near) / fine_dt);
  int64_t m = 0;
  while (m < n && t_near + ((double)m + 0.5) * fine_dt < t_far) ++m;
  if (m == 0) return;
  double *ts = malloc(sizeof(double) * m), *sigma = calloc(m, sizeof(double));
  double *wsum = calloc(3 * m, sizeof(double));
  for (int64_t j = 0; j < m; ++j) ts[j] = t_near + ((double)j + 0.5) * fine_dt;
  for (int64_t a = 0; a < s->n; ++a) {
    const int64_t i = ord[a];
    const double *M = s->iso_inv + 9 * i, *mu = s->means + 3 * i;
    double c[3];
    int have_c = 0;
    for (int64_t j = 0; j < m; ++j) {
      double v[3], y[3];
      for (int k = 0; k < 3; ++k) v[k] = (o[k] + ts[j] * d[k]) - mu[k];
      for (int b = 0; b < 3; ++b) y[b] = v[0] * M[3 * b] + v[1] * M[3 * b + 1] + v[2] * M[3 * b + 2];
      const double q = y[0] * y[0] + y[1] * y[1] + y[2] * y[2];
      if (!(q <= 1.0)) continue;
      const double dens = s->sigmas[i] * exp(-0.5 * s->log_ratio[i] * q);
      if (!have_c) {
        eval_radiance(s->coeffs + NCOEF * i, d, c, NULL, NULL);
        have_c = 1;
      }
      sigma[j] += dens;
      for (int k = 0; k < 3; ++k) wsum[3 * j + k] += dens * c[k];
    }
  }
  double cum = 0.0, col[3] = {0, 0, 0}, od = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    od = sigma[j] * fine_dt;
    if (sigma[j] > 0.0) {
      const double w = -expm1(-od) * exp(-cum);
      for (int k = 0; k < 3; ++k) col[k] += (w / sigma[j]) * wsum[3 * j + k];
    }
    if (j + 1 < m) cum += od;
  }
  const double t_exit = exp(-(cum + od));
  for (int k = 0; k < 3; ++k) out[k] = col[k] + t_exit * bg[k];
  free(ts);
  free(sigma);
  free(wsum);
}

typedef struct {
  const oscene *s;
  const int64_t *ord;
  const double *rays, *bg;
  int64_t m, clip;
  double fine_dt;
  double *rgb;
  int64_t next;
  pthread_mutex_t mu;
} dense_job;

static void *dense_worker(void *arg) {
  dense_job *jb = (dense_job *)arg;
  for (;;) {
    pthread_mutex_lock(&jb->mu);
    const int64_t r = jb->next++;
    pthread_mutex_unlock(&jb->mu);
    if (r >= jb->m) break;
    const double *ray = jb->rays + 8 * r;
    double d[3] = {ray[3], ray[4], ray[5]}, tn = ray[6], tf = ray[7];
    double *out = jb->rgb + 3 * r;
    if (jb->clip) {  /* reference_render: clip_ray_to_scene, background on a miss */
      if (!clip_ray(jb->s, ray, d, ray[6], ray[7], &tn, &tf)) {
        for (int k = 0; k < 3; ++k) out[k] = jb->bg[k];
        continue;
      }
    } else {  /* Ray.__post_init__ renormalization (renderer.py:60-64) */
      const double nn = vnorm(d, 3);
      if (fabs(nn - 1.0) > 1e-9)
        for (int k = 0; k < 3; ++k) d[k] = d[k] / nn;
    }
    reference_integrate(jb->s, jb->ord, ray, d, tn, tf, jb->fine_dt, jb->bg, out);
  }
  return NULL;
}

/* reference_integrate per ray (clip = 0) or reference_render's per-pixel
   clip + integrate (clip = 1, renderer.py:483-493) over m rays (o, d, t_near,
   t_far), on `threads` host threads. */
int oracle_reference_rays(void *h, int64_t m, const double *rays, int64_t clip, double fine_dt,
                          const double *bg, int64_t threads, double *rgb) {
  if (!(fine_dt > 0.0)) return ERR_ARG;
  dense_job jb;
  memset(&jb, 0, sizeof jb);
  jb.s = (const oscene *)h;
  jb.ord = uid_order(jb.s);
  jb.rays = rays;
  jb.bg = bg;
  jb.m = m;
  jb.clip = clip;
  jb.fine_dt = fine_dt;
  jb.rgb = rgb;
  pthread_mutex_init(&jb.mu, NULL);
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  for (int64_t t = 1; t < threads; ++t) pthread_create(&th[t], NULL, dense_worker, &jb);
  dense_worker(&jb);
  for (int64_t t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&jb.mu);
  free((void *)jb.ord);
  return OK;
}

/* appearance.py:107-134 eval_fields: density and density-weighted radiance
   of the mixture at x (direction d) over `active` (storage indices, NULL =
   all), visited in ascending uid; zero density gives black. */
int oracle_eval_fields(void *h, const double *x, const double *d, const int64_t *active,
                       int64_t n_active, double *sigma_out, double *color_out) {
  const oscene *s = (const oscene *)h;
  int64_t *ord;
  int64_t na;
  if (active) {
    na = n_active;
    ord = malloc(sizeof(int64_t) * (na > 0 ? na : 1));
    memcpy(ord, active, sizeof(int64_t) * na);
    /* stable sort by uid (insertion: the lists are short) */
    for (int64_t a = 1; a < na; ++a) {
      const int64_t v = ord[a];
      int64_t b = a;
      while (b > 0 && s->uids[ord[b - 1]] > s->uids[v]) { ord[b] = ord[b - 1]; --b; }
      ord[b] = v;
    }
  } else {
    na = s->n;
    ord = uid_order(s);
  }
  double sigma = 0.0, wsum[3] = {0, 0, 0};
  for (int64_t a = 0; a < na; ++a) {
    const int64_t i = ord[a];
    if (i < 0 || i >= s->n) { free(ord); return ERR_ARG; }
    const double *M = s->iso_inv + 9 * i, *mu = s->means + 3 * i;
    double v[3], y[3];
    for (int k = 0; k < 3; ++k) v[k] = x[k] - mu[k];
    for (int b = 0; b < 3; ++b) y[b] = M[3 * b] * v[0] + M[3 * b + 1] * v[1] + M[3 * b + 2] * v[2];
    const double q = y[0] * y[0] + y[1] * y[1] + y[2] * y[2];
    if (q > 1.0) continue;
    const double dens = s->sigmas[i] * exp(-0.5 * s->log_ratio[i] * q);
    double c[3];
    eval_radiance(s->coeffs + NCOEF * i, d, c, NULL, NULL);
    sigma += dens;
    for (int k = 0; k < 3; ++k) wsum[k] = wsum[k] + dens * c[k];
  }
  free(ord);
  *sigma_out = sigma;
  for (int k = 0; k < 3; ++k) color_out[k] = sigma == 0.0 ? 0.0 : wsum[k] / sigma;
  return OK;
}

/* renderer.py:135-145 Camera.ray for every pixel (row py, col px), R is the
   camera-to-world rotation (row-major).  rays out: H*W*8. */
void oracle_camera_rays(const double *center, const double *R, double focal, int64_t W,
                        int64_t H, double t_near, double t_far, double *rays) {
  for (int64_t py = 0; py < H; ++py)
    for (int64_t px = 0; px < W; ++px) {
      double dc[3] = {((double)px + 0.5 - 0.5 * (double)W) / focal,
                      ((double)py + 0.5 - 0.5 * (double)H) / focal, 1.0};
      double d[3];
      for (int a = 0; a < 3; ++a) d[a] = R[3 * a] * dc[0] + R[3 * a + 1] * dc[1] + R[3 * a + 2] * dc[2];
      double n = vnorm(d, 3);
      double *ry = rays + 8 * (py * W + px);
      for (int k = 0; k < 3; ++k) { ry[k] = center[k]; ry[3 + k] = d[k] / n; }
      ry[6] = t_near;
      ry[7] = t_far;
    }
}

/* ------------------------------------------------------------------------ */
/* analytic backward (no reference counterpart)        */
/* ------------------------------------------------------------------------ */
/* gradient of one (ray, primitive, sample) density term and colour term
   accumulated into g[87] (record layout). */
static void grad_density(const oscene *s, int64_t i, const double *x, double gdens, double *g) {
  /* dens = sigma * exp(-0.5 u.u), u = S^-1 R^T (x - mu) */
  const double *R = s->rot + 9 * i, *mu = s->means + 3 * i, *sc = s->scales + 3 * i;
  const double *rec = s->rec + NREC * i;
  double v[3] = {x[0] - mu[0], x[1] - mu[1], x[2] - mu[2]};
  double u[3];
  for (int b = 0; b < 3; ++b) u[b] = (R[b] * v[0] + R[3 + b] * v[1] + R[6 + b] * v[2]) / sc[b];
  double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  double dens = s->sigmas[i] * exp(-0.5 * uu);
  double gd = gdens * dens;
  /* sigma~ */
  g[10] += gd / s->sigmas[i];
  /* mean: d dens/d mu = dens * R S^-1 u */
  double su[3] = {u[0] / sc[0], u[1] / sc[1], u[2] / sc[2]};
  for (int a = 0; a < 3; ++a) g[a] += gd * (R[3 * a] * su[0] + R[3 * a + 1] * su[1] + R[3 * a + 2] * su[2]);
  /* scales: d dens/d s_b = dens u_b^2 / s_b (clamp: zero when raw <= S_MIN) */
  for (int b = 0; b < 3; ++b)
    if (rec[7 + b] > S_MIN) g[7 + b] += gd * u[b] * u[b] / sc[b];
  /* rotation: d dens/d R[a][b] = -dens u_b v_a / s_b */
  double gR[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) gR[3 * a + b] = -gd * u[b] * v[a] / sc[b];
  /* R(q), q normalized twice (geometry.py:80 and :36); dq/dq_raw = (I - qq^T)/|q_raw| */
  const double *q = s->quats + 4 * i;
  double w = q[0], X = q[1], Y = q[2], Z = q[3];
  double dR[4][9] = {
      {0, -2 * Z, 2 * Y, 2 * Z, 0, -2 * X, -2 * Y, 2 * X, 0},
      {0, 2 * Y, 2 * Z, 2 * Y, -4 * X, -2 * w, 2 * Z, 2 * w, -4 * X},
      {-4 * Y, 2 * X, 2 * w, 2 * X, 0, 2 * Z, -2 * w, 2 * Z, -4 * Y},
      {-4 * Z, -2 * w, 2 * X, 2 * w, -4 * Z, 2 * Y, 2 * X, 2 * Y, 0}};
  double gq[4];
  for (int c = 0; c < 4; ++c) {
    double acc = 0.0;
    for (int e = 0; e < 9; ++e) acc += gR[e] * dR[c][e];
    gq[c] = acc;
  }
  double qn = vnorm(rec + 3, 4);
  double dot = gq[0] * q[0] + gq[1] * q[1] + gq[2] * q[2] + gq[3] * q[3];
  for (int c = 0; c < 4; ++c) g[3 + c] += (gq[c] - dot * q[c]) / qn;
}

static void grad_color(const oscene *s, int64_t i, const double *d, const double *gc, double *g) {
  const double *c = s->coeffs + NCOEF * i, *rec = s->rec + NREC * i;
  double rgb[3], pre[3], lob[NSG], Y[9];
  eval_radiance(c, d, rgb, pre, lob);
  double gp[3];
  for (int k = 0; k < 3; ++k) gp[k] = pre[k] > 0.0 ? gc[k] : 0.0;
  sh_basis(d, Y);
  for (int b = 0; b < 9; ++b)
    for (int k = 0; k < 3; ++k) g[11 + 3 * b + k] += Y[b] * gp[k];
  for (int l = 0; l < NSG; ++l) {
    const double *ax = c + 27 + 3 * l, *amp = c + 55 + 3 * l;
    double ga = amp[0] * gp[0] + amp[1] * gp[1] + amp[2] * gp[2];
    for (int k = 0; k < 3; ++k) g[66 + 3 * l + k] += lob[l] * gp[k];
    double cs = ax[0] * d[0] + ax[1] * d[1] + ax[2] * d[2];
    g[59 + l] += lob[l] * (cs - 1.0) * ga;
    /* axis: d/d nu_hat = lob * lambda * d * ga; through normalization */
    double gn[3];
    for (int k = 0; k < 3; ++k) gn[k] = lob[l] * c[48 + l] * d[k] * ga;
    const double *raw = rec + 38 + 3 * l;
    double an = vnorm(raw, 3);
    double dd = gn[0] * ax[0] + gn[1] * ax[1] + gn[2] * ax[2];
    for (int k = 0; k < 3; ++k) g[38 + 3 * l + k] += (gn[k] - dd * ax[k]) / an;
  }
}

/* Backward of one ray given the forward tape.  gC: dL/d rgb_out (3),
   gD: dL/d depth, gT: dL/d T_out.  Accumulates into grad (n*87). */
static void backward_ray(const oscene *s, const ocfg *cfg, const double *o, const double *d,
                         const otape *tp, const double *gC, double gD, double gT,
                         double *grad) {
  int64_t m = tp->n;
  if (m == 0) return;
  /* recompute per-sample sigma, W, and per-sample colors */
  double *sig = calloc(m, sizeof(double)), *W = calloc(3 * m, sizeof(double));
  for (int64_t j = 0; j < m; ++j) {
    int64_t sg = tp->seg[j];
    const int64_t *act = tp->cand + tp->seg_off[sg];
    int64_t na = tp->seg_cnt[sg];
    double x[3];
    for (int k = 0; k < 3; ++k) x[k] = o[k] + tp->t[j] * d[k];
    for (int64_t a = 0; a < na; ++a) {
      int64_t i = act[a];
      const double *M = s->iso_inv + 9 * i, *mu = s->means + 3 * i;
      double v[3] = {x[0] - mu[0], x[1] - mu[1], x[2] - mu[2]}, y[3];
      for (int b = 0; b < 3; ++b) y[b] = v[0] * M[3 * b] + v[1] * M[3 * b + 1] + v[2] * M[3 * b + 2];
      double q = y[0] * y[0] + y[1] * y[1] + y[2] * y[2];
      if (q <= 1.0) {
        double dens = s->sigmas[i] * exp(-0.5 * s->log_ratio[i] * q);
        double rgb[3];
        eval_radiance(s->coeffs + NCOEF * i, d, rgb, NULL, NULL);
        sig[j] += dens;
        for (int k = 0; k < 3; ++k) W[3 * j + k] += dens * rgb[k];
      }
    }
  }
  /* forward prefix quantities */
  double *Tj = malloc(sizeof(double) * (m + 1)), *w = malloc(sizeof(double) * m);
  double od = 0.0, Ctot[3] = {0, 0, 0}, Dtot = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    Tj[j] = exp(-od);
    double ods = sig[j] * tp->dt[j];
    w[j] = sig[j] > 0.0 ? -expm1(-ods) * Tj[j] : 0.0;
    if (sig[j] > 0.0) {
      for (int k = 0; k < 3; ++k) Ctot[k] += w[j] / sig[j] * W[3 * j + k];
      Dtot += w[j] * tp->t[j];
    }
    od += ods;
  }
  Tj[m] = exp(-od);
  double Tend = Tj[m];
  double gTe = gT + gC[0] * cfg->background[0] + gC[1] * cfg->background[1] +
               gC[2] * cfg->background[2];
  double Cpre[3] = {0, 0, 0}, Dpre = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    if (!(sig[j] > 0.0)) continue;
    double dtj = tp->dt[j];
    double cj[3] = {W[3 * j] / sig[j], W[3 * j + 1] / sig[j], W[3 * j + 2] / sig[j]};
    for (int k = 0; k < 3; ++k) Cpre[k] += w[j] * cj[k];
    Dpre += w[j] * tp->t[j];
    double Tn = Tj[j] * exp(-sig[j] * dtj); /* T_{j+1} */
    double gsig = 0.0;
    for (int k = 0; k < 3; ++k) gsig += gC[k] * dtj * (Tn * cj[k] - (Ctot[k] - Cpre[k]));
    gsig += gD * dtj * (Tn * tp->t[j] - (Dtot - Dpre));
    gsig += gTe * (-dtj * Tend);
    double wos = w[j] / sig[j];
    /* per primitive split */
    int64_t sg = tp->seg[j];
    const int64_t *act = tp->cand + tp->seg_off[sg];
    int64_t na = tp->seg_cnt[sg];
    double x[3];
    for (int k = 0; k < 3; ++k) x[k] = o[k] + tp->t[j] * d[k];
    for (int64_t a = 0; a < na; ++a) {
      int64_t i = act[a];
      const double *M = s->iso_inv + 9 * i, *mu = s->means + 3 * i;
      double v[3] = {x[0] - mu[0], x[1] - mu[1], x[2] - mu[2]}, y[3];
      for (int b = 0; b < 3; ++b) y[b] = v[0] * M[3 * b] + v[1] * M[3 * b + 1] + v[2] * M[3 * b + 2];
      double q = y[0] * y[0] + y[1] * y[1] + y[2] * y[2];
      if (!(q <= 1.0)) continue;
      double dens = s->sigmas[i] * exp(-0.5 * s->log_ratio[i] * q);
      double rgb[3];
      eval_radiance(s->coeffs + NCOEF * i, d, rgb, NULL, NULL);
      double gdn = gsig;
      for (int k = 0; k < 3; ++k) gdn += wos * (rgb[k] - cj[k]) * gC[k];
      /* d dens / d(param) = dens * (...): grad_density takes gdens per unit dens */
      grad_density(s, i, x, gdn, grad + NREC * i);
      double gc[3] = {wos * dens * gC[0], wos * dens * gC[1], wos * dens * gC[2]};
      grad_color(s, i, d, gc, grad + NREC * i);
    }
  }
  free(sig); free(W); free(Tj); free(w);
}

/* Forward + backward over a batch of rays (single thread, deterministic).
   grad: n*87 accumulated (caller zeroes).  rgb/T/depth outputs as forward. */
int oracle_backward_rays(void *h, const ocfg *cfg, int64_t m, const double *rays, int64_t clip,
                         const double *gC, const double *gD, const double *gT, double *rgb,
                         double *T, double *depth, double *grad) {
  const oscene *s = (const oscene *)h;
  int64_t *buf = malloc(sizeof(int64_t) * (cfg->buffer_capacity > 0 ? cfg->buffer_capacity : 1));
  int64_t *big = malloc(sizeof(int64_t) * s->n);
  double *rad = malloc(sizeof(double) * 3 * s->n);
  int64_t *stamp = malloc(sizeof(int64_t) * s->n);
  for (int64_t i = 0; i < s->n; ++i) stamp[i] = -1;
  ostats st;
  memset(&st, 0, sizeof st);
  for (int64_t i = 0; i < m; ++i) {
    const double *ry = rays + 8 * i;
    double o[3] = {ry[0], ry[1], ry[2]}, d[3] = {ry[3], ry[4], ry[5]};
    double tn = ry[6], tf = ry[7];
    if (clip) {
      if (!clip_ray(s, o, d, ry[6], ry[7], &tn, &tf)) {
        for (int k = 0; k < 3; ++k) rgb[3 * i + k] = cfg->background[k];
        T[i] = 1.0;
        depth[i] = 0.0;
        continue;
      }
    }
    otape tp;
    memset(&tp, 0, sizeof tp);
    march(s, cfg, o, d, tn, tf, rgb + 3 * i, T + i, depth + i, &st, buf, big, rad, stamp, i, &tp);
    backward_ray(s, cfg, o, d, &tp, gC + 3 * i, gD[i], gT[i], grad);
    tape_free(&tp);
  }
  free(buf);
  free(big);
  free(rad);
  free(stamp);
  return OK;
}
