// render_common.cuh -- per-ray device building blocks shared by the forward
// (render.cu) and backward (render_bwd.cu) kernels.
#pragma once
#include "gsx_common.cuh"

// Rarely-taken per-lane paths (closest hit, phantom probe) are kept out of
// line: the march kernels are instruction-cache sensitive.
#ifndef GSX_COLD
#define GSX_COLD __noinline__
#endif
#ifndef GSX_FAST_COMPOSITE
#define GSX_FAST_COMPOSITE 1
#endif
#ifndef GSX_EXACT_FP32
#define GSX_EXACT_FP32 1
#endif
#ifndef GSX_RCBRT
#define GSX_RCBRT 1
#endif

namespace gsx {

// ---------------------------------------------------------------------------
// ray context: fp64 ray (reference semantics) + fp32 copies for traversal
// ---------------------------------------------------------------------------
struct RayCtx {
  double o[3], d[3];
  double inv_t[3];  // traversal-style inverse (spatial.py:227)
  float of[3], df[3], invf[3];
  float eps_scale;
  double t_n, t_f;
};

__device__ inline double norm3d(const double* v) {
  return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(v[0], v[0]), __dmul_rn(v[1], v[1])),
                        __dmul_rn(v[2], v[2])));
}

// Ray.__post_init__ renormalization (renderer.py:60-64) + clip_ray_to_scene
// (renderer.py:160-175).  Returns false when the ray misses (background).
__device__ inline bool finish_ray(const double* bounds, bool clip, double t_near, double t_far,
                                  RayCtx& r) {
  double n = norm3d(r.d);
  if (fabs(n - 1.0) > 1e-9)
    for (int k = 0; k < 3; ++k) r.d[k] = r.d[k] / n;
  if (t_near >= t_far) return false;
  if (clip) {
    double inv[3];
    for (int k = 0; k < 3; ++k) inv[k] = r.d[k] == 0.0 ? INFINITY : 1.0 / r.d[k];
    double a, b;
    box_slab64(bounds, bounds + 3, r.o, r.d, inv, a, b);
    double t0 = t_near > a ? t_near : a;
    double t1 = t_far < b ? t_far : b;
    if (t0 >= t1) return false;
    r.t_n = t0;
    r.t_f = t1;
  } else {
    r.t_n = t_near;
    r.t_f = t_far;
  }
  inv_dir_traversal64(r.d, r.inv_t);
  float sc = 1.f;
  for (int k = 0; k < 3; ++k) {
    r.of[k] = (float)r.o[k];
    r.df[k] = (float)r.d[k];
    float dd = fabsf(r.df[k]) > 1e-30f ? r.df[k] : copysignf(1e-30f, r.df[k]);
    r.invf[k] = 1.0f / dd;
    sc = fmaxf(sc, fabsf(r.of[k]));
  }
  r.eps_scale = sc;
  return true;
}

// Camera.ray (renderer.py:135-145) for pixel (px, py).
__device__ inline bool camera_ray(const gsx_camera& cam, double px, double py,
                                  const double* bounds, RayCtx& r) {
  double dc[3] = {__ddiv_rn(__dsub_rn(__dadd_rn(px, 0.5), 0.5 * (double)cam.width), cam.focal),
                  __ddiv_rn(__dsub_rn(__dadd_rn(py, 0.5), 0.5 * (double)cam.height), cam.focal),
                  1.0};
  double d[3];
  for (int a = 0; a < 3; ++a)
    d[a] = __dadd_rn(__dadd_rn(__dmul_rn(cam.R[3 * a], dc[0]), __dmul_rn(cam.R[3 * a + 1], dc[1])),
                     __dmul_rn(cam.R[3 * a + 2], dc[2]));
  double n = norm3d(d);
  for (int k = 0; k < 3; ++k) {
    r.o[k] = cam.center[k];
    r.d[k] = d[k] / n;
  }
  return finish_ray(bounds, true, cam.t_near, cam.t_far, r);
}

__device__ inline bool explicit_ray(const double* ray8, bool clip, const double* bounds,
                                    RayCtx& r) {
  for (int k = 0; k < 3; ++k) {
    r.o[k] = ray8[k];
    r.d[k] = ray8[3 + k];
  }
  return finish_ray(bounds, clip, ray8[6], ray8[7], r);
}

// Z-order position of thread t in a 16x16 tile (x: even bits, y: odd bits)
__device__ inline void morton_decode8(unsigned t, int& x, int& y) {
  x = (t & 1) | ((t >> 1) & 2) | ((t >> 2) & 4) | ((t >> 3) & 8);
  y = ((t >> 1) & 1) | ((t >> 2) & 2) | ((t >> 3) & 4) | ((t >> 4) & 8);
}

__device__ inline float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ inline float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---------------------------------------------------------------------------
// appearance (appearance.py:26-50, 91-98), fp32
// ---------------------------------------------------------------------------
__device__ inline void sh_basis_f(const float* d, float* Y) {
  const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f, C2A = 1.0925484305920792f,
              C2B = 0.31539156525252005f, C2C = 0.5462742152960396f;
  float x = d[0], y = d[1], z = d[2];
  Y[0] = C0;
  Y[1] = C1 * y;
  Y[2] = C1 * z;
  Y[3] = C1 * x;
  Y[4] = C2A * x * y;
  Y[5] = C2A * y * z;
  Y[6] = C2B * (3.0f * z * z - 1.0f);
  Y[7] = C2A * x * z;
  Y[8] = C2C * (x * x - y * y);
}

// float4 loaders: read-only global (default) or shared memory (staged copies)
struct LdgLoad {
  __device__ float4 operator()(const float4* p) const { return __ldg(p); }
};
struct PlainLoad {  // ordinary load (shared memory when the pointer is known to be)
  __device__ float4 operator()(const float4* p) const { return *p; }
};
struct SmemLoad {
  __device__ float4 operator()(const float4* p) const {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
  }
};

// SH basis of a lane kept in shared memory (stride 32 floats: one column per
// lane), so the 9 values do not occupy registers across the march
struct YSmem {
  const float* p;
  __device__ float operator[](int b) const { return p[32 * b]; }
};

// ... or recomputed from the direction at each use (a handful of FMULs per
// radiance evaluation instead of 9 live registers or 1.15 KB of shared
// memory per warp); same values as sh_basis_f
struct YDir {
  const float* d;
  __device__ float operator[](int b) const {
    const float x = d[0], y = d[1], z = d[2];
    switch (b) {
      case 0: return 0.28209479177387814f;
      case 1: return 0.4886025119029199f * y;
      case 2: return 0.4886025119029199f * z;
      case 3: return 0.4886025119029199f * x;
      case 4: return 1.0925484305920792f * x * y;
      case 5: return 1.0925484305920792f * y * z;
      case 6: return 0.31539156525252005f * (3.0f * z * z - 1.0f);
      case 7: return 1.0925484305920792f * x * z;
      default: return 0.5462742152960396f * (x * x - y * y);
    }
  }
};

// unclamped radiance and lobe values (lobes may be NULL); app = GSX_APP_F4
// float4 in the streaming layout, consumed one float4 at a time so the
// coefficients never need 76 live registers.
template <class L = LdgLoad, class YT = const float*>
__device__ inline void eval_radiance_pre(const float4* __restrict__ app, YT Y,
                                         const float* d, float* pre, float* lobes) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int b = 0; b < 9; ++b) {
    const float4 v = L()(app + b);
    s0 = fmaf(Y[b], v.x, s0);
    s1 = fmaf(Y[b], v.y, s1);
    s2 = fmaf(Y[b], v.z, s2);
  }
#pragma unroll
  for (int l = 0; l < 7; ++l) {
    const float4 ax = L()(app + 9 + 2 * l), am = L()(app + 10 + 2 * l);
    float cs = fmaf(ax.x, d[0], fmaf(ax.y, d[1], ax.z * d[2]));
    float e = __expf(ax.w * (cs - 1.0f));
    if (lobes) lobes[l] = e;
    s0 = fmaf(e, am.x, s0);
    s1 = fmaf(e, am.y, s1);
    s2 = fmaf(e, am.z, s2);
  }
  pre[0] = s0;
  pre[1] = s1;
  pre[2] = s2;
}

template <class L = LdgLoad, class YT = const float*>
__device__ inline void eval_radiance_f(const float4* __restrict__ app, YT Y,
                                       const float* d, float* c) {
  float pre[3];
  eval_radiance_pre<L, YT>(app, Y, d, pre, nullptr);
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) c[ch] = fmaxf(pre[ch], 0.f);
}

// ---------------------------------------------------------------------------
// per-(ray, primitive) density setup: q(t) = A (t - tc)^2 + qmin
// ---------------------------------------------------------------------------
struct CandSetup {
  float A, qmin, del0, kl2, sigma, h, tc, lsig;
};

__device__ inline void local_frame(const float4* geo, int64_t p, const RayCtx& r, double* y0,
                                   double* yd) {
  float4 g0 = __ldg(geo + 4 * p), g1 = __ldg(geo + 4 * p + 1), g2 = __ldg(geo + 4 * p + 2),
         g3 = __ldg(geo + 4 * p + 3);
  double v[3] = {r.o[0] - (double)g0.x, r.o[1] - (double)g0.y, r.o[2] - (double)g0.z};
  double M[9] = {g1.x, g1.y, g1.z, g2.x, g2.y, g2.z, g3.x, g3.y, g3.z};
  for (int a = 0; a < 3; ++a) {
    y0[a] = fma(M[3 * a], v[0], fma(M[3 * a + 1], v[1], M[3 * a + 2] * v[2]));
    yd[a] = fma(M[3 * a], r.d[0], fma(M[3 * a + 1], r.d[1], M[3 * a + 2] * r.d[2]));
  }
}

// Sample-base point of a segment as an unevaluated float pair (x0 = hi + lo,
// |lo| <= ulp(hi)/2), from the fp64 ray: x0 = o + tbase * d.
struct SegBase {
  float hi[3], lo[3];
};
__device__ inline SegBase seg_base(const RayCtx& r, double tbase) {
  SegBase b;
  for (int k = 0; k < 3; ++k) {
    double x = fma(tbase, r.d[k], r.o[k]);
    b.hi[k] = (float)x;
    b.lo[k] = (float)(x - (double)b.hi[k]);
  }
  return b;
}

// fp32 setup relative to the segment base: v = x0 - mu is formed as
// (hi - mu) + lo, accurate to ~ulp(|x0 - mu|) because |x0 - mu| is at most a
// segment plus a box (~0.3 world units) for any primitive the segment can
// see -- no catastrophic cancellation, no fp64.  Then y(j) = y0 + (j dt) yd,
// q(j) = A (j dt - tc)^2 + qmin with qmin = |y0 + tc yd|^2.
template <class L = LdgLoad>
__device__ inline bool cand_setup_at(const float4* geo, const RayCtx& r, const SegBase& b,
                                     CandSetup& cs) {
  const float4 g0 = L()(geo), g1 = L()(geo + 1), g2 = L()(geo + 2), g3 = L()(geo + 3);
  float v0 = (b.hi[0] - g0.x) + b.lo[0];
  float v1 = (b.hi[1] - g0.y) + b.lo[1];
  float v2 = (b.hi[2] - g0.z) + b.lo[2];
  float y0x = fmaf(g1.x, v0, fmaf(g1.y, v1, g1.z * v2));
  float y0y = fmaf(g2.x, v0, fmaf(g2.y, v1, g2.z * v2));
  float y0z = fmaf(g3.x, v0, fmaf(g3.y, v1, g3.z * v2));
  float ydx = fmaf(g1.x, r.df[0], fmaf(g1.y, r.df[1], g1.z * r.df[2]));
  float ydy = fmaf(g2.x, r.df[0], fmaf(g2.y, r.df[1], g2.z * r.df[2]));
  float ydz = fmaf(g3.x, r.df[0], fmaf(g3.y, r.df[1], g3.z * r.df[2]));
  float A = fmaf(ydx, ydx, fmaf(ydy, ydy, ydz * ydz));
  if (!(A > 0.f)) return false;
  float B = fmaf(y0x, ydx, fmaf(y0y, ydy, y0z * ydz));
  // approximate reciprocal / square root (MUFU, ~1 ulp, no slow-path branch):
  // a 1-ulp error in tc moves q by ~2 sqrt(A) ulp(tc) ~ 1e-5 at most, far
  // inside the 1e-4 RGB tolerance, and h only bounds the sample range
  const float iA = __fdividef(1.0f, A);
  float tc = -B * iA;
  float ycx = fmaf(tc, ydx, y0x), ycy = fmaf(tc, ydy, y0y), ycz = fmaf(tc, ydz, y0z);
  float qmin = fmaf(ycx, ycx, fmaf(ycy, ycy, ycz * ycz));
  if (qmin > 1.0f) return false;
  cs.A = A;
  cs.qmin = qmin;
  cs.tc = tc;
  cs.del0 = -tc;
  cs.kl2 = g1.w;
  cs.sigma = g0.w;
  cs.lsig = g3.w;
  cs.h = sqrt_approx(fmaxf((1.0f - qmin) * iA, 0.f));
  return true;
}
__device__ inline bool cand_setup(const SceneView& sv, const RayCtx& r, int64_t p,
                                  const SegBase& b, CandSetup& cs) {
  return cand_setup_at(sv.geo + 4 * p, r, b, cs);
}

// conservative sample index range [jlo, jhi] within [0, m-1] that may lie
// inside the ellipsoid (the q <= 1 test decides exactly).
__device__ inline bool sample_range(const CandSetup& cs, float dtf, int m, int& jlo, int& jhi) {
  // floor/ceil below already leave one sample of slack on each side, which
  // absorbs the approximate reciprocal
  const float idt = __fdividef(1.0f, dtf);
  float lo = (-cs.h - cs.del0) * idt;
  float hi = (cs.h - cs.del0) * idt;
  if (!(hi >= -1.f) || !(lo <= (float)m)) return false;
  lo = fmaxf(lo, -1.f);
  hi = fminf(hi, (float)m);
  jlo = max(0, (int)floorf(lo));
  jhi = min(m - 1, (int)ceilf(hi));
  return jlo <= jhi;
}

// ---------------------------------------------------------------------------
// exact fp64 tests (reference arithmetic) used for ESS emptiness and stats
// ---------------------------------------------------------------------------
#ifndef GSX_EXACT_ATTR
#define GSX_EXACT_ATTR inline
#endif
__device__ GSX_EXACT_ATTR bool exact_aabb_overlap64(const SceneView& sv, const RayCtx& r,
                                                  int64_t p, double t0, double t1) {
  const double* ab = sv.aabb64 + 6 * p;
  double ta, tb;
  box_slab64(ab, ab + 3, r.o, r.d, r.inv_t, ta, tb);
  return ta <= t1 && tb >= t0;
}

// The reference's AABB-overlap test (spatial.py:231-241, with its inverted
// "phantom" intervals: ta <= t1 && tb >= t0 without ta <= tb), decided in
// fp32 on the outward-rounded box when the answer is certain: the slab values
// carry at most ~4e-7 relative error from the fp32 origin, direction and box
// rounding, so a 1e-6 margin (|box| + |o|) |1/d| + 1e-6 (|t| + 1) separates
// certain overlaps and misses from the ambiguous band, which (like
// near-axis-parallel rays, |d_k| < 1e-4) goes to the fp64 test.  Same
// verdicts as exact_aabb_overlap64; fp64 code off the per-entry path.
__device__ inline bool exact_aabb_overlap(const SceneView& sv, const RayCtx& r, int64_t p,
                                          double t0, double t1) {
#if GSX_EXACT_FP32
  const float2* b = (const float2*)(sv.box32 + 6 * p);
  const float2 b0 = __ldg(b), b1 = __ldg(b + 1), b2 = __ldg(b + 2);
  const float lo[3] = {b0.x, b0.y, b1.x}, hi[3] = {b1.y, b2.x, b2.y};
  float ta = -INFINITY, tb = INFINITY, imax = 0.f, ext = r.eps_scale;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float a = (lo[k] - r.of[k]) * r.invf[k], c = (hi[k] - r.of[k]) * r.invf[k];
    ta = fmaxf(ta, fminf(a, c));
    tb = fminf(tb, fmaxf(a, c));
    imax = fmaxf(imax, fabsf(r.invf[k]));
    ext = fmaxf(ext, fmaxf(fabsf(lo[k]), fabsf(hi[k])));
  }
  const float t0f = (float)t0, t1f = (float)t1;
  const float m = 1e-6f * (2.f * ext * imax + fabsf(t0f) + fabsf(t1f) + 1.f);
  if (imax <= 1e4f) {
    if (ta + m <= t1f && tb - m >= t0f) return true;
    if (ta - m > t1f || tb + m < t0f) return false;
  }
#endif
  return exact_aabb_overlap64(sv, r, p, t0, t1);
}

__device__ inline bool ellipsoid_hits_interval(const SceneView& sv, const RayCtx& r, int64_t p,
                                               double t0, double t1) {
  const double* M = sv.inv64 + 9 * p;
  float4 g = sv.geo[4 * p];
  double v[3] = {__dsub_rn(r.o[0], (double)g.x), __dsub_rn(r.o[1], (double)g.y),
                 __dsub_rn(r.o[2], (double)g.z)};
  double ol[3], dl[3];
  for (int a = 0; a < 3; ++a) {
    ol[a] = __dadd_rn(__dadd_rn(__dmul_rn(M[3 * a], v[0]), __dmul_rn(M[3 * a + 1], v[1])),
                      __dmul_rn(M[3 * a + 2], v[2]));
    dl[a] = __dadd_rn(__dadd_rn(__dmul_rn(M[3 * a], r.d[0]), __dmul_rn(M[3 * a + 1], r.d[1])),
                      __dmul_rn(M[3 * a + 2], r.d[2]));
  }
  double a, b;
  return ray_ellipsoid_interval64(ol, dl, t0, t1, a, b);
}

// segment_step (renderer.py:148-157)
__device__ inline double segment_step(const gsx_render_cfg& cfg, double d_i, double t_i) {
  double t = t_i > cfg.t_eps ? t_i : cfg.t_eps;
#if GSX_RCBRT
  // t^(-1/3): the reference's exp(-log(t)/3) to ~1 ulp with a fraction of the
  // code (the fp64 exp + log bodies sat in the march loop)
  double boost = rcbrt(t);
#else
  double boost = exp(-log(t) / 3.0);
#endif
  double a = d_i / cfg.beta;
  if (!(a > cfg.dt_min)) a = cfg.dt_min;
  double step = a * boost;
  if (step > cfg.dt_max) step = cfg.dt_max;
  return (double)cfg.n_s * step;
}

// ---------------------------------------------------------------------------
// fp32 traversal
// ---------------------------------------------------------------------------
__device__ inline void slab_f(const float4& lo, const float4& hi, const RayCtx& r, float& tmin,
                              float& tmax) {
  float x0 = (lo.x - r.of[0]) * r.invf[0], x1 = (hi.x - r.of[0]) * r.invf[0];
  float y0 = (lo.y - r.of[1]) * r.invf[1], y1 = (hi.y - r.of[1]) * r.invf[1];
  float z0 = (lo.z - r.of[2]) * r.invf[2], z1 = (hi.z - r.of[2]) * r.invf[2];
  tmin = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fminf(z0, z1));
  tmax = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fmaxf(z0, z1));
}

__device__ inline float margin(const RayCtx& r, float t) {
  return 2e-6f * (fabsf(t) + r.eps_scale);
}

// Visit every leaf whose (outward-rounded) box slab interval overlaps
// [t0, t1] (with a conservative margin); leaf_fn(prim) is called in traversal
// order; leaf_fn returns true to stop early.  PHANTOM=false requires a true
// ray/box intersection (tmin <= tmax) -- all a density contribution can come
// from.  PHANTOM=true also admits the reference's "inverted" overlaps
// (spatial.py:234,240 test a <= t1 and b >= t0 without a <= b: a box the line
// misses whose gap [tmax, tmin] lies inside the segment still counts for
// AABB-emptiness).  Returns false if the stack overflowed.
template <bool PHANTOM, class F>
__device__ inline bool traverse_segment(const BvhView& bv, const RayCtx& r, float t0, float t1,
                                        F&& leaf_fn, uint32_t& visits) {
  const float lo_t = t0 - margin(r, t0), hi_t = t1 + margin(r, t1);
  const float gap = margin(r, t1);
  int32_t stack[GSX_STACK];
  int sp = 0;
  int32_t node = 0;
  bool ok = true;
  for (;;) {
    ++visits;
    const float4* nd = bv.nodes + 4 * (int64_t)node;
    float4 a = __ldg(nd), b = __ldg(nd + 1), c = __ldg(nd + 2), e = __ldg(nd + 3);
    int32_t cl = __float_as_int(a.w), cr = __float_as_int(b.w);
    float mn, mx;
    slab_f(a, b, r, mn, mx);
    bool hl = cl != GSX_NONE && mn <= hi_t && mx >= lo_t && (PHANTOM || mn <= mx + gap);
    slab_f(c, e, r, mn, mx);
    bool hr = cr != GSX_NONE && mn <= hi_t && mx >= lo_t && (PHANTOM || mn <= mx + gap);
    int32_t next = -1;
    if (hl) {
      if (cl < 0) {
        if (leaf_fn((int64_t)(~cl))) return ok;
      } else
        next = cl;
    }
    if (hr) {
      if (cr < 0) {
        if (leaf_fn((int64_t)(~cr))) return ok;
      } else if (next >= 0) {
        if (sp < GSX_STACK)
          stack[sp++] = cr;
        else
          ok = false;
      } else
        next = cr;
    }
    if (next < 0) {
      if (sp == 0) break;
      next = stack[--sp];
    }
    node = next;
  }
  return ok;
}

// closest ellipsoid entry in [t_lo, t_hi] (spatial.py:309-354): fp32 node
// tests with margin, near child first, pruning by the current best; leaves
// use the fp64 Kahan interval in the primitive's unit-sphere frame.
// Cold path (about 2 calls per ray): kept out of line so the hot march loops
// stay compact in the instruction cache.
static __device__ GSX_COLD bool closest_hit_r(const SceneView& sv, const BvhView& bv, const RayCtx& r,
                                     double t_lo, double t_hi, double& hit, uint32_t& visits) {
  if (t_lo > t_hi) return false;
  double best = INFINITY;
  int32_t snode[GSX_STACK];
  float sent[GSX_STACK];
  int sp = 0;
  int32_t node = 0;
  const float lo_t = (float)t_lo - margin(r, (float)t_lo);
  for (;;) {
    ++visits;
    const float4* nd = bv.nodes + 4 * (int64_t)node;
    float4 a = __ldg(nd), b = __ldg(nd + 1), c = __ldg(nd + 2), e = __ldg(nd + 3);
    int32_t ch[2] = {__float_as_int(a.w), __float_as_int(b.w)};
    float mn[2], mx[2];
    slab_f(a, b, r, mn[0], mx[0]);
    slab_f(c, e, r, mn[1], mx[1]);
    bool go[2] = {false, false};
    for (int k = 0; k < 2; ++k) {
      int32_t cc = ch[k];
      if (cc == GSX_NONE) continue;
      double lim = t_hi < best ? t_hi : best;
      float limf = (float)lim + margin(r, (float)lim);
      // a true ray/box intersection is necessary for an ellipsoid hit
      if (!(mn[k] <= limf && mx[k] >= lo_t && mn[k] <= mx[k] + margin(r, mx[k]))) continue;
      if (cc < 0) {
        int64_t p = ~(int64_t)cc;
        double y0[3], yd[3];
        local_frame(sv.geo, p, r, y0, yd);
        double tin, tout;
        if (ray_ellipsoid_interval64(y0, yd, t_lo, lim, tin, tout) && tin < best) best = tin;
      } else {
        go[k] = true;
      }
    }
    int32_t next = -1;
    if (go[0] && go[1]) {
      int nr = mn[1] < mn[0] ? 1 : 0;
      if (sp < GSX_STACK) {
        snode[sp] = ch[1 - nr];
        sent[sp++] = mn[1 - nr];
      }
      next = ch[nr];
    } else if (go[0]) {
      next = ch[0];
    } else if (go[1]) {
      next = ch[1];
    }
    while (next < 0 && sp > 0) {
      --sp;
      float ent = sent[sp];
      double lim = t_hi < best ? t_hi : best;
      if (ent <= (float)lim + margin(r, (float)lim)) next = snode[sp];
    }
    if (next < 0) break;
    node = next;
  }
  if (best < INFINITY) {
    hit = best;
    return true;
  }
  return false;
}

// ---------------------------------------------------------------------------
// front-to-back accumulator (renderer.py:230-239) + depth
// ---------------------------------------------------------------------------
struct RayAccum {
  float C[3];
  float D;
  float od;
  float T;
  __device__ void init() {
    C[0] = C[1] = C[2] = 0.f;
    D = 0.f;
    od = 0.f;
    T = 1.f;
  }
  __device__ float transmittance() const { return T; }
  // branch-free: a zero-density sample leaves the state unchanged (measured
  // faster than skipping it: C3 40.0 vs 40.5 ms, training forward 24.3 vs 27.0)
#if GSX_FAST_COMPOSITE
  // (C3 30.25 vs 30.88 ms, C2 14.7 vs 15.6: the unrolled libm bodies were
  // instruction-cache pressure.  Both forms approximate the reference's fp64
  // compositing to ~1e-7 relative per sample; C3 pixels move by up to 5.8e-5
  // between them through termination / adaptive-step decisions near their
  // thresholds; the golden-scene parity suite passes with either.)
  // Same arithmetic with MUFU exponentials (16 samples are unrolled per
  // segment: the libm expm1f / expf bodies cost ~60 instructions of code per
  // sample).  alpha = 1 - exp(-x): 5-term series below x = 0.05 (truncation
  // < x^6/720 = 2e-11 relative), else 1 - 2^(-x log2 e) (ex2.approx relative
  // error ~1e-7, i.e. < 2.4e-6 relative on alpha >= 0.049); T = 2^(-od log2 e)
  // to ~2e-7 relative.
  // opacity 1 - exp(-x) of a sample with optical depth x >= 0
  __device__ static float alpha(float x) {
    const float ser =
        x * fmaf(x, fmaf(x, fmaf(x, fmaf(x, 1.f / 120.f, -1.f / 24.f), 1.f / 6.f), -0.5f), 1.f);
    const float big = 1.f - ex2_approx(-1.4426950408889634f * x);
    return x < 0.05f ? ser : big;
  }
  __device__ void add_sample(float sig, const float* W, float tj, float dt) {
    const bool on = sig > 0.f;
    const float x = on ? sig * dt : 0.f;
    const float w = alpha(x) * T;
    const float s = on ? __fdividef(w, sig) : 0.f;
    C[0] = fmaf(s, W[0], C[0]);
    C[1] = fmaf(s, W[1], C[1]);
    C[2] = fmaf(s, W[2], C[2]);
    D = fmaf(w, tj, D);
    od += x;
    T = ex2_approx(-1.4426950408889634f * od);
  }
#else
  __device__ static float alpha(float x) { return -expm1f(-x); }
  __device__ void add_sample(float sig, const float* W, float tj, float dt) {
    const bool on = sig > 0.f;
    const float ods = on ? sig * dt : 0.f;
    const float w = -expm1f(-ods) * T;
    const float s = on ? __fdividef(w, sig) : 0.f;
    C[0] = fmaf(s, W[0], C[0]);
    C[1] = fmaf(s, W[1], C[1]);
    C[2] = fmaf(s, W[2], C[2]);
    D = fmaf(w, tj, D);
    od += ods;
    T = expf(-od);
  }
#endif
};

}  // namespace gsx
