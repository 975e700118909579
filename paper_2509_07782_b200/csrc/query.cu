// query.cu -- K10 parity queries in fp64 over the LBVH:
//   collect  = Bvh.segment_overlaps (spatial.py:215-247): exact candidate SET
//   closest  = closest_hit (spatial.py:309-354)
// Node boxes are fp32 outward-rounded supersets tested in fp64 (the slab test is
// monotone in lo/hi, so pruning is conservative); the final per-primitive test
// uses the fp64 AABB / iso_inv, exactly the reference's arithmetic.
#include "gsx_common.cuh"

namespace {

__global__ void k_collect(SceneView sv, BvhView bv, int64_t n, const double* __restrict__ queries,
                          int64_t m, int64_t cap, int64_t* counts, int64_t* idx,
                          gsx_dev_status* st) {
  int64_t qi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= m) return;
  const double* q = queries + 8 * qi;
  double o[3] = {q[0], q[1], q[2]}, d[3] = {q[3], q[4], q[5]};
  double t0 = q[6], t1 = q[7];
  double inv[3];
  inv_dir_traversal64(d, inv);
  int32_t stack[GSX_STACK];
  int sp = 0;
  stack[sp++] = 0;
  int64_t count = 0;
  int64_t* out = idx + qi * cap;
  while (sp > 0) {
    int32_t node = stack[--sp];
    const float4* nd = bv.nodes + 4 * (int64_t)node;
    float4 a = nd[0], b = nd[1], c = nd[2], e = nd[3];
    int32_t ch[2] = {__float_as_int(a.w), __float_as_int(b.w)};
    float4 los[2] = {a, c}, his[2] = {b, e};
    for (int k = 1; k >= 0; --k) {  // push right first: left is processed first
      int32_t c2 = ch[k];
      if (c2 == GSX_NONE) continue;
      double ta, tb;
      if (c2 < 0) {
        int64_t p = ~(int64_t)c2;
        const double* ab = sv.aabb64 + 6 * p;
        box_slab64(ab, ab + 3, o, d, inv, ta, tb);
        if (ta <= t1 && tb >= t0) {
          if (count < cap) out[count] = p;
          count++;
        }
      } else {
        box_slab64_f(los[k], his[k], o, d, inv, ta, tb);
        if (ta > t1 || tb < t0) continue;
        if (sp >= GSX_STACK) {
          dev_fail(st, GSX_ERR_STACK, qi);
          counts[qi] = -1;
          return;
        }
        stack[sp++] = c2;
      }
    }
  }
  counts[qi] = count;
  int64_t kept = count < cap ? count : cap;
  // ascending storage index (insertion sort; parity kernel)
  for (int64_t a = 1; a < kept; ++a) {
    int64_t v = out[a], b = a - 1;
    while (b >= 0 && out[b] > v) {
      out[b + 1] = out[b];
      --b;
    }
    out[b + 1] = v;
  }
  if (count > cap) dev_fail(st, GSX_ERR_OVERFLOW, qi, count, cap);
}

__global__ void k_closest(SceneView sv, BvhView bv, int64_t n, const double* __restrict__ queries,
                          int64_t m, double* t_out) {
  int64_t qi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= m) return;
  const double* q = queries + 8 * qi;
  double o[3] = {q[0], q[1], q[2]}, d[3] = {q[3], q[4], q[5]};
  double t_lo = q[6], t_hi = q[7];
  if (t_lo > t_hi) {
    t_out[qi] = NAN;
    return;
  }
  double inv[3];
  inv_dir_traversal64(d, inv);
  double best = INFINITY;
  int32_t snode[GSX_STACK];
  double sent[GSX_STACK];
  int sp = 0;
  snode[sp] = 0;
  sent[sp++] = 0.0;
  while (sp > 0) {
    --sp;
    int32_t node = snode[sp];
    if (sent[sp] >= best) continue;
    const float4* nd = bv.nodes + 4 * (int64_t)node;
    float4 a = nd[0], b = nd[1], c = nd[2], e = nd[3];
    int32_t ch[2] = {__float_as_int(a.w), __float_as_int(b.w)};
    float4 los[2] = {a, c}, his[2] = {b, e};
    double ent[2];
    bool push[2] = {false, false};
    for (int k = 0; k < 2; ++k) {
      int32_t c2 = ch[k];
      if (c2 == GSX_NONE) continue;
      double lim = t_hi < best ? t_hi : best;
      if (c2 < 0) {
        int64_t p = ~(int64_t)c2;
        const double* M = sv.inv64 + 9 * p;
        const float4 g = sv.geo[4 * p];
        double mu[3] = {(double)g.x, (double)g.y, (double)g.z};
        double v[3] = {__dsub_rn(o[0], mu[0]), __dsub_rn(o[1], mu[1]), __dsub_rn(o[2], mu[2])};
        double ol[3], dl[3];
        for (int r = 0; r < 3; ++r) {
          ol[r] = __dadd_rn(__dadd_rn(__dmul_rn(M[3 * r], v[0]), __dmul_rn(M[3 * r + 1], v[1])),
                            __dmul_rn(M[3 * r + 2], v[2]));
          dl[r] = __dadd_rn(__dadd_rn(__dmul_rn(M[3 * r], d[0]), __dmul_rn(M[3 * r + 1], d[1])),
                            __dmul_rn(M[3 * r + 2], d[2]));
        }
        double tin, tout;
        if (ray_ellipsoid_interval64(ol, dl, t_lo, lim, tin, tout) && tin < best) best = tin;
      } else {
        double ta, tb;
        box_slab64_f(los[k], his[k], o, d, inv, ta, tb);
        if (ta > lim || tb < t_lo) continue;
        ent[k] = ta;
        push[k] = true;
      }
    }
    // near child last on the stack (processed first)
    int first = 0, second = 1;
    if (push[0] && push[1] && ent[1] < ent[0]) {
      first = 1;
      second = 0;
    }
    if (sp + 2 > GSX_STACK) {
      t_out[qi] = NAN;
      return;
    }
    if (push[second]) {
      snode[sp] = ch[second];
      sent[sp++] = ent[second];
    }
    if (push[first]) {
      snode[sp] = ch[first];
      sent[sp++] = ent[first];
    }
  }
  t_out[qi] = isfinite(best) ? best : NAN;
}

// neighbor_density (densify.py:86-97): for each primitive, the number of
// OTHER means within the closed ball of radius r (cKDTree.query_ball_point
// minus self).  One thread per primitive over the binary BVH: the fp32
// outward-rounded node boxes contain every mean below them, so pruning on the
// point-to-box distance is exact; leaves compare fp64 squared distances.
__global__ void k_neighbors(SceneView sv, BvhView bv, int64_t n, double r2, int64_t* counts,
                            gsx_dev_status* st) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 gi = __ldg(sv.geo + 4 * i);
  const double p[3] = {gi.x, gi.y, gi.z};
  int32_t stack[GSX_STACK];
  int sp = 0;
  stack[sp++] = 0;
  int64_t count = 0;
  while (sp > 0) {
    const float4* nd = bv.nodes + 4 * (int64_t)stack[--sp];
    const float4 a = nd[0], b = nd[1], c = nd[2], e = nd[3];
    const int32_t ch[2] = {__float_as_int(a.w), __float_as_int(b.w)};
    const float4 los[2] = {a, c}, his[2] = {b, e};
    for (int k = 0; k < 2; ++k) {
      const int32_t c2 = ch[k];
      if (c2 == GSX_NONE) continue;
      if (c2 < 0) {
        const int64_t j = ~(int64_t)c2;
        if (j == i) continue;
        const float4 gj = __ldg(sv.geo + 4 * j);
        const double dx = (double)gj.x - p[0], dy = (double)gj.y - p[1], dz = (double)gj.z - p[2];
        if (dx * dx + dy * dy + dz * dz <= r2) ++count;
      } else {
        const double lo[3] = {los[k].x, los[k].y, los[k].z}, hi[3] = {his[k].x, his[k].y, his[k].z};
        double d2 = 0.0;
        for (int ax = 0; ax < 3; ++ax) {
          const double t = p[ax] < lo[ax] ? lo[ax] - p[ax] : (p[ax] > hi[ax] ? p[ax] - hi[ax] : 0.0);
          d2 += t * t;
        }
        if (d2 > r2) continue;
        if (sp >= GSX_STACK) {
          dev_fail(st, GSX_ERR_STACK, i);
          counts[i] = -1;
          return;
        }
        stack[sp++] = c2;
      }
    }
  }
  counts[i] = count;
}

}  // namespace

extern "C" int gsx_collect_segments(const void* scene_arena, const void* bvh_arena, int64_t n,
                                    const double* queries, int64_t m, int64_t capacity,
                                    int64_t* counts, int64_t* idx, gsx_dev_status* dev_status,
                                    void* stream) {
  if (m <= 0) return GSX_OK;
  if (capacity < 1) return GSX_ERR_ARG;
  SceneView sv = scene_view((void*)scene_arena, n);
  BvhView bv = bvh_view((void*)bvh_arena, n);
  k_collect<<<(unsigned)((m + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      sv, bv, n, queries, m, capacity, counts, idx, dev_status);
  return gsx_check_launch();
}

extern "C" int gsx_closest_hit(const void* scene_arena, const void* bvh_arena, int64_t n,
                               const double* queries, int64_t m, double* t_out, void* stream) {
  if (m <= 0) return GSX_OK;
  SceneView sv = scene_view((void*)scene_arena, n);
  BvhView bv = bvh_view((void*)bvh_arena, n);
  k_closest<<<(unsigned)((m + 127) / 128), 128, 0, (cudaStream_t)stream>>>(sv, bv, n, queries, m,
                                                                           t_out);
  return gsx_check_launch();
}

extern "C" int gsx_neighbor_density(const void* scene_arena, const void* bvh_arena, int64_t n,
                                    double radius, int64_t* counts, gsx_dev_status* dev_status,
                                    void* stream) {
  if (n <= 0) return GSX_ERR_EMPTY;
  if (!(radius > 0.0) || !counts) return GSX_ERR_ARG;
  SceneView sv = scene_view((void*)scene_arena, n);
  BvhView bv = bvh_view((void*)bvh_arena, n);
  k_neighbors<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      sv, bv, n, radius * radius, counts, dev_status);
  return gsx_check_launch();
}
