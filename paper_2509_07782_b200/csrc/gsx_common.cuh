// gsx_common.cuh -- shared device layouts and helpers for libgsx (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gsx.h"

#define GSX_NREC 87
#define GSX_NCOEF 76
#define GSX_NONE ((int32_t)0x80000000)
#define GSX_STACK 96

// ---------------------------------------------------------------------------
// Tile order of camera launches (render_image's tile loop renderer.py:408-412).
// A launch renders the tile-sequence positions s = tile_begin + k*tile_stride
// (rank r of G: tile_begin = r, tile_stride = G).  With GSX_TILE_ORDER 1 and
// tile_stride > 1 the sequence visits the tile rows centre-out (c, c+1, c-1, c+2, ... with
// c = (rows-1)/2; row-major inside a row), so the CTAs dispatched first are
// the ones whose rays cross the middle of the view, and the last wave of a
// short per-rank launch is the image border.  Pixels do not depend on the
// order; every rank set is still a partition.  C3 8-rank share: max over
// ranks 5.87 vs 6.22 ms row-major; a whole-image launch (stride 1) stays
// row-major (29.58 vs 29.71 ms centre-out; profiles/r05_cta_order_variants.txt).
// ---------------------------------------------------------------------------
#ifndef GSX_TILE_ORDER
#define GSX_TILE_ORDER 1
#endif
__host__ __device__ inline int64_t gsx_tile_at(int64_t s, int64_t tiles_x, int64_t tiles_y,
                                               int64_t stride) {
  if (!GSX_TILE_ORDER || stride <= 1) return s;
  const int64_t i = s / tiles_x, c = (tiles_y - 1) / 2, d = (i + 1) / 2;
  const int64_t row = (i & 1) ? c + d : c - d;
  return row * tiles_x + s % tiles_x;
}

// ---------------------------------------------------------------------------
// Scene arena (caller-allocated, gsx_scene_arena_bytes).  N primitives in
// storage order.  Sections are 256-byte aligned.
//   aabb64 : double[n][6]  lo xyz, hi xyz   (scene.py:61-65, exact fp64)
//   inv64  : double[n][9]  iso_inv          (scene.py:58-60, exact fp64)
//   lr64   : double[n]     log_ratio        (scene.py:55)
//   geo    : float4[n][4]  (mu, sigma~) (M row0, k*log2e/2) (M row1, k) (M row2, log2 sigma~)
//   box32  : float[n][6]   outward-rounded fp32 AABB (LBVH leaves)
//   app    : float4[n][23] radiance-streaming layout: 9 x (sh_b rgb, 0), then per
//            lobe l: (unit axis xyz, sharpness) (amp rgb, 0)
//   bounds : double[6]     scene AABB lo xyz, hi xyz (scene.py:66-67)
//   part   : double[GSX_BOUNDS_BLOCKS][6] partial bounds
// ---------------------------------------------------------------------------
#define GSX_BOUNDS_BLOCKS 296
#define GSX_APP_F4 23

//   gaux   : float4[n][5]  backward helpers: (unit quat w,x,y,z) (1/|q_raw|, 1/s clamped xyz)
//            (sqrt k, scale-not-clamped mask xyz) (1/|axis_raw| lobes 0..3)
//            (1/|axis_raw| lobes 4..6, 1/sigma~)
struct SceneView {
  double* aabb64;
  double* inv64;
  double* lr64;
  float4* geo;
  float* box32;
  float4* app;
  double* bounds;
  double* part;
  float4* gaux;
};

static inline size_t gsx_align256(size_t x) { return (x + 255) & ~(size_t)255; }

__host__ __device__ inline size_t gsx_al(size_t x) { return (x + 255) & ~(size_t)255; }

__host__ __device__ inline SceneView scene_view(void* arena, int64_t n) {
  char* p = (char*)arena;
  SceneView v;
  size_t off = 0;
  v.aabb64 = (double*)(p + off); off += gsx_al(sizeof(double) * 6 * n);
  v.inv64 = (double*)(p + off);  off += gsx_al(sizeof(double) * 9 * n);
  v.lr64 = (double*)(p + off);   off += gsx_al(sizeof(double) * n);
  v.geo = (float4*)(p + off);    off += gsx_al(sizeof(float4) * 4 * n);
  v.box32 = (float*)(p + off);   off += gsx_al(sizeof(float) * 6 * n);
  v.app = (float4*)(p + off);    off += gsx_al(sizeof(float4) * GSX_APP_F4 * n);
  v.bounds = (double*)(p + off); off += gsx_al(sizeof(double) * 6);
  v.part = (double*)(p + off);   off += gsx_al(sizeof(double) * 6 * GSX_BOUNDS_BLOCKS);
  v.gaux = (float4*)(p + off);
  return v;
}

inline size_t scene_arena_bytes_impl(int64_t n) {
  size_t s = 0;
  s += gsx_align256(sizeof(double) * 6 * n);
  s += gsx_align256(sizeof(double) * 9 * n);
  s += gsx_align256(sizeof(double) * n);
  s += gsx_align256(sizeof(float4) * 4 * n);
  s += gsx_align256(sizeof(float) * 6 * n);
  s += gsx_align256(sizeof(float4) * GSX_APP_F4 * n);
  s += gsx_align256(sizeof(double) * 6);
  s += gsx_align256(sizeof(double) * 6 * GSX_BOUNDS_BLOCKS);
  s += gsx_align256(sizeof(float4) * 5 * n);
  return s;
}

// ---------------------------------------------------------------------------
// BVH arena: internal nodes float4[n-1][4]:
//   q0 = (lo_l.xyz, child_l)  q1 = (hi_l.xyz, child_r)
//   q2 = (lo_r.xyz, 0)        q3 = (hi_r.xyz, 0)
// child >= 0: internal node index; child < 0: leaf ~prim; GSX_NONE: absent.
// parents int32[2n-1] (internal 0..n-2, leaf i at n-1+i).  Root = node 0.
// For n == 1 a single node holds leaf 0 on the left and GSX_NONE on the right.
//
// 4-wide collapse (used by the warp-cooperative packet traversal): the binary
// internal nodes at even depth are kept, odd-depth ones are absorbed into their
// parent, so every 4-wide node holds up to 4 children (grandchildren of the
// binary node).  Node = float4[8] (128 B):
//   q0 = lo.x[4]  q1 = lo.y[4]  q2 = lo.z[4]  q3 = hi.x[4]  q4 = hi.y[4]
//   q5 = hi.z[4]  q6 = child[4] (int bits, same encoding)  q7 = unused
// Root = node 0.
// ---------------------------------------------------------------------------
struct BvhView {
  float4* nodes;
  int32_t* parents;
  float4* nodes4;
  gsx_dev_status* status;  // per launch (nullable): traversal-stack overflow reports
};

__host__ __device__ inline int64_t bvh_internal_count(int64_t n) { return n > 1 ? n - 1 : 1; }

__host__ __device__ inline BvhView bvh_view(void* arena, int64_t n) {
  char* p = (char*)arena;
  BvhView v;
  size_t a = ((sizeof(float4) * 4 * bvh_internal_count(n)) + 255) & ~(size_t)255;
  size_t b = ((sizeof(int32_t) * (2 * n + 1)) + 255) & ~(size_t)255;
  v.nodes = (float4*)p;
  v.parents = (int32_t*)(p + a);
  v.nodes4 = (float4*)(p + a + b);
  v.status = nullptr;
  return v;
}

inline size_t bvh_arena_bytes_impl(int64_t n) {
  return gsx_align256(sizeof(float4) * 4 * bvh_internal_count(n)) +
         gsx_align256(sizeof(int32_t) * (2 * n + 1)) +
         gsx_align256(sizeof(float4) * 8 * bvh_internal_count(n));
}

// device-wide exclusive scan of u32 (morton_sort.cu); sums: scan workspace
size_t gsx_scan_ws_elems(int64_t len);
void gsx_exclusive_scan_u32(uint32_t* data, int64_t len, uint32_t* sums, cudaStream_t s);

// ---------------------------------------------------------------------------
// device status helpers
// ---------------------------------------------------------------------------
__device__ inline void dev_fail(gsx_dev_status* st, int64_t code, int64_t index, int64_t count = 0,
                                int64_t cap = 0) {
  if (!st) return;
  // keep the smallest index of the first error code seen
  unsigned long long* c = (unsigned long long*)&st->code;
  unsigned long long old = atomicCAS(c, 0ull, (unsigned long long)code);
  if (old == 0ull || old == (unsigned long long)code) {
    atomicMin((long long*)&st->index, (long long)index);
    if (count) {
      atomicMax((long long*)&st->count, (long long)count);
      st->capacity = cap;
    }
  }
}

// ---------------------------------------------------------------------------
// fp64 slab test mirroring spatial.py:258-277 (_box_slab), no contraction.
// ---------------------------------------------------------------------------
__device__ inline void box_slab64(const double* lo, const double* hi, const double* o,
                                  const double* d, const double* inv, double& ta, double& tb) {
  double t0 = -INFINITY, t1 = INFINITY;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (d[k] != 0.0) {
      double a = __dmul_rn(__dsub_rn(lo[k], o[k]), inv[k]);
      double b = __dmul_rn(__dsub_rn(hi[k], o[k]), inv[k]);
      if (a > b) {
        double t = a;
        a = b;
        b = t;
      }
      if (a > t0) t0 = a;
      if (b < t1) t1 = b;
    } else if (o[k] < lo[k] || o[k] > hi[k]) {
      ta = INFINITY;
      tb = -INFINITY;
      return;
    }
  }
  ta = t0;
  tb = t1;
}

// inverse direction for traversal queries (spatial.py:227, :321)
__device__ inline void inv_dir_traversal64(const double* d, double* inv) {
#pragma unroll
  for (int k = 0; k < 3; ++k) inv[k] = fabs(d[k]) > 1e-300 ? 1.0 / (d[k] == 0.0 ? 1.0 : d[k]) : INFINITY;
}

// spatial.py:280-306 ray_ellipsoid_interval, fp64, no contraction.
__device__ inline bool ray_ellipsoid_interval64(const double* ol, const double* dl, double t_lo,
                                                double t_hi, double& tin, double& tout) {
  double a = __dadd_rn(__dadd_rn(__dmul_rn(dl[0], dl[0]), __dmul_rn(dl[1], dl[1])),
                       __dmul_rn(dl[2], dl[2]));
  double b = __dadd_rn(__dadd_rn(__dmul_rn(ol[0], dl[0]), __dmul_rn(ol[1], dl[1])),
                       __dmul_rn(ol[2], dl[2]));
  double c = __dsub_rn(__dadd_rn(__dadd_rn(__dmul_rn(ol[0], ol[0]), __dmul_rn(ol[1], ol[1])),
                                 __dmul_rn(ol[2], ol[2])),
                       1.0);
  double disc = __dsub_rn(__dmul_rn(b, b), __dmul_rn(a, c));
  if (disc < 0.0 || a == 0.0) return false;
  double sq = sqrt(disc);
  double q = (b >= 0.0) ? -__dadd_rn(b, sq) : -__dsub_rn(b, sq);
  double t0 = __ddiv_rn(q, a);
  double t1 = (q != 0.0) ? __ddiv_rn(c, q) : t0;
  if (t0 > t1) {
    double t = t0;
    t0 = t1;
    t1 = t;
  }
  if (t_lo > t0) t0 = t_lo;
  if (t_hi < t1) t1 = t_hi;
  if (t0 > t1) return false;
  tin = t0;
  tout = t1;
  return true;
}

// fp64 slab of an fp32 node box (exact conversion; conservative for the
// outward-rounded boxes).
__device__ inline void box_slab64_f(const float4 lo, const float4 hi, const double* o,
                                    const double* d, const double* inv, double& ta, double& tb) {
  double l[3] = {(double)lo.x, (double)lo.y, (double)lo.z};
  double h[3] = {(double)hi.x, (double)hi.y, (double)hi.z};
  box_slab64(l, h, o, d, inv, ta, tb);
}

#define CUDA_CHECK_RET(expr)                       \
  do {                                             \
    cudaError_t _e = (expr);                       \
    if (_e != cudaSuccess) {                       \
      gsx_set_cuda_error(_e);                      \
      return GSX_ERR_CUDA;                         \
    }                                              \
  } while (0)

void gsx_set_cuda_error(cudaError_t e);
int gsx_check_launch();
int gsx_validate_cfg(const gsx_render_cfg* cfg);
