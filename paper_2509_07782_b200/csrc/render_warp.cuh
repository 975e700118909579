// render_warp.cuh -- warp-lockstep march machinery shared by the forward
// (render.cu) and backward (render_bwd.cu) kernels.
//
// A warp = 32 spatially coherent rays (an 8x4 Z-order pixel block).  Each loop
// iteration every active lane processes its next segment of Alg. 1
// (renderer.py:288-358): a warp-cooperative ("packet") traversal of the 4-wide
// BVH over the union of the 32 segments stages candidates in a shared-memory
// list, and every lane evaluates the list against its own ray.  The backward
// replays exactly the same code path, so its per-sample state is bit-identical
// to the forward's.
#pragma once
#include "render_common.cuh"

namespace gsx {

constexpr unsigned FULL = 0xffffffffu;
// depth-synchronous windows (segment lengths) measured best on C3 / C2:
// forward 1.0 (40.6 vs 41.2 ms unsynchronized), backward 0.5 (train step
// 90 vs 125 ms).  The backward's replay then interleaves lanes differently
// from the forward: its per-sample sums may differ from the forward's in the
// last ulp (it uses the forward's saved C, D, T only in the adjoints).
#ifndef GSX_SYNC_FWD
#define GSX_SYNC_FWD 1.0f
#endif
// uniform mode (short fixed segments; packet-cone traversal): C2 15.6 ms at
// 0.5 vs 17.4 at 1.0 (C3, adaptive: 33.3 at 0.5, 31.1 at 1.0, 31.8 at 2.0)
#ifndef GSX_SYNC_FWD_U
#define GSX_SYNC_FWD_U 0.5f
#endif
#ifndef GSX_SYNC_BWD
#define GSX_SYNC_BWD 0.5f
#endif
// (shrinking the per-warp shared block -- list / stack 192, the SH basis out
// of shared memory -- to enlarge L1 for the spilled per-lane state measured
// within noise: C3 29.5-29.6 ms for all four, profiles/r04_smem_size_variants.txt)
#ifndef GSX_LCAP
#define GSX_LCAP 256
#endif
#ifndef GSX_WSTACK
#define GSX_WSTACK 256
#endif
constexpr int LCAP = GSX_LCAP;      // warp candidate list (shared memory)
constexpr int WSTACK = GSX_WSTACK;  // warp traversal stack (shared memory)

// Optional per-phase warp-time accounting (experiment builds only:
// nvcc -DGSX_PHASE_PROF); compiled out of the product library.
#ifdef GSX_PHASE_PROF
// one copy per translation unit (no -rdc); gsx_phase_times reads render.cu's
static __device__ unsigned long long g_phase[24];
#define PH_BEGIN(v) \
  __syncwarp();     \
  long long v = clock64();
#define PH_END(i, v) \
  __syncwarp();      \
  if ((threadIdx.x & 31) == 0) atomicAdd(&g_phase[i], (unsigned long long)(clock64() - v));
#define PH_CNT(i, val) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&g_phase[i], (unsigned long long)(val));
#define PH_LANES(i, pred)                                                                  \
  {                                                                                        \
    unsigned _b = __ballot_sync(0xffffffffu, pred);                                        \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_phase[i], (unsigned long long)__popc(_b)); \
  }
#else
#define PH_CNT(i, val)
#define PH_LANES(i, pred)
#define PH_BEGIN(v)
#define PH_END(i, v)
#endif

template <bool STATS>
struct Counters {
  uint32_t samples = 0, segments = 0, skipped = 0, ch_calls = 0, visits = 0, aabb = 0, ell = 0,
           pairs = 0, composited = 0;
};

// Per-warp shared state (the forward adds the lanes' SH basis, GSX_Y_SMEM).
#ifndef GSX_Y_SMEM
#define GSX_Y_SMEM 0
#endif
#ifndef GSX_APP_TMA  // screened kernels: appearance blocks by TMA bulk copy (see app_issue)
#define GSX_APP_TMA 1
#endif
#ifndef GSX_APP_NB  // staging buffers per warp: entries are staged GSX_APP_NB - 1 ahead
#define GSX_APP_NB 2  // (3 / 4: C3 24.7 / 25.2 vs 23.4 ms -- copies for entries no lane uses)
#endif
#ifndef GSX_GEO_TMA  // ... and the geometry blocks (C3 24.1 vs 23.3 ms: the setup then
#define GSX_GEO_TMA 0  // waits for a copy instead of a (mostly L1/L2-hit) broadcast load)
#endif
struct WarpSmem {
  int32_t stack[WSTACK];
  int32_t list[LCAP];
  int ovf;  // a traversal stack of this warp overflowed (reported as GSX_ERR_STACK)
  float4 cone[5];  // packet cone (make_cone): (o, dlo^2), 4 x (plane normal, .w: dhi^2 | eps_scale | dlo | dhi)
#if GSX_Y_SMEM == 1
  float ylane[9][32];  // per-lane SH basis (forward)
#endif
};

// screened kernels: + the entry blocks the TMA engine stages (app_issue)
struct WarpSmemT : WarpSmem {
#if GSX_APP_TMA
  float4 appb[GSX_APP_NB][GSX_APP_F4];  // the current and the next entries' appearance blocks
  unsigned long long mbar[GSX_APP_NB];  // TMA completion barriers of the appearance blocks
#if GSX_GEO_TMA
  float4 geob[GSX_APP_NB][4];           // ... and geometry blocks
  unsigned long long gbar[GSX_APP_NB];  // ... of the geometry blocks (waited on first)
#endif
  unsigned mpar;                // the barriers' phase parities (bit b: buffer b)
#endif
};

struct WarpTrav {
  int32_t node;
  int sp;
  bool done;
  bool overflow;
};

// Warp-cooperative traversal of the 4-wide BVH: every lane tests its own
// ray/segment against the 4 child boxes of the warp's current node,
// __any_sync decides the (warp-uniform) descent, and leaves hit by any lane are
// appended to the shared list.  True ray/box intersections only (see
// traverse_segment).  Resumable: returns when done or the list is nearly full.
__device__ inline void warp_traverse(const BvhView& bv, const RayCtx& r, bool want, float lo_t,
                                     float hi_t, float gap, WarpTrav& st, WarpSmem& sm,
                                     int& count, uint32_t& visits) {
  // 32-bit shared-window addresses of the list and stack: cheap to keep live
  // (the generic pointers were rematerialised from %tid per store); every lane
  // stores the same value, so no lane predicate is needed
  const unsigned a_list = (unsigned)__cvta_generic_to_shared(sm.list);
  const unsigned a_stack = (unsigned)__cvta_generic_to_shared(sm.stack);
  while (!st.done && count <= LCAP - 4) {
    ++visits;
    PH_CNT(8, 1)
    const float4* nd = bv.nodes4 + 8 * (int64_t)st.node;
    const float4 lx = __ldg(nd), ly = __ldg(nd + 1), lz = __ldg(nd + 2);
    const float4 hx = __ldg(nd + 3), hy = __ldg(nd + 4), hz = __ldg(nd + 5);
    const float4 cf = __ldg(nd + 6);
    const float clo[3][4] = {{lx.x, lx.y, lx.z, lx.w}, {ly.x, ly.y, ly.z, ly.w},
                             {lz.x, lz.y, lz.z, lz.w}};
    const float chi[3][4] = {{hx.x, hx.y, hx.z, hx.w}, {hy.x, hy.y, hy.z, hy.w},
                             {hz.x, hz.y, hz.z, hz.w}};
    const int32_t ch[4] = {__float_as_int(cf.x), __float_as_int(cf.y), __float_as_int(cf.z),
                           __float_as_int(cf.w)};
    int32_t next = -1;
    // the four child tests are independent: evaluate them together (ILP),
    // then one ballot per child
    bool hk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float x0 = (clo[0][k] - r.of[0]) * r.invf[0], x1 = (chi[0][k] - r.of[0]) * r.invf[0];
      float y0 = (clo[1][k] - r.of[1]) * r.invf[1], y1 = (chi[1][k] - r.of[1]) * r.invf[1];
      float z0 = (clo[2][k] - r.of[2]) * r.invf[2], z1 = (chi[2][k] - r.of[2]) * r.invf[2];
      float mn = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fminf(z0, z1));
      float mx = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fmaxf(z0, z1));
      hk[k] = want && mn <= hi_t && mx >= lo_t && mn <= mx + gap;
    }
    // predicated bookkeeping: every lane runs the same straight-line code;
    // the stores are predicated (no branches), all lanes store equal values.
    // (Measured against the branchy version: C2 training forward 20.5 vs 23.4
    // ms, C3 35.3 vs 35.0; a lanes-0..3 popc-rank variant was slower.)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int32_t c = ch[k];
      const bool h = __any_sync(FULL, hk[k]) && c != GSX_NONE;
      const bool leaf = h && c < 0;
      const bool inner = h && c >= 0;
      const bool push = inner && next >= 0;
      const bool fits = st.sp < WSTACK;
      asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p st.shared.b32 [%0], %1; }" ::"r"(
                       a_list + 4u * count), "r"(~c), "r"((unsigned)leaf) : "memory");
      asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0; @p st.shared.b32 [%0], %1; }" ::"r"(
                       a_stack + 4u * st.sp), "r"(c), "r"((unsigned)(push && fits)) : "memory");
      count += leaf ? 1 : 0;
      st.sp += (push && fits) ? 1 : 0;
      st.overflow |= push && !fits;
      next = (inner && next < 0) ? c : next;
    }
    if (st.overflow) sm.ovf = 1;
    __syncwarp();
    if (next < 0) {
      if (st.sp == 0) {
        st.done = true;
        break;
      }
      --st.sp;
      next = sm.stack[st.sp];
    }
    st.node = next;
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Packet-cone traversal (camera rays: one common origin).
//
// The lanes that take part in an iteration march rays from one origin o, so
// their segments lie in the cone {o + t d : d in the lanes' directions} cut by
// the distance shell |x - o| in [min lo_t, max hi_t] (|d| = 1, so t is the
// distance).  The cone is bounded by four planes through o: in projective
// coordinates (u, v) = (d.e1, d.e2) / d.a about the leader's direction a,
// the lanes span [umin, umax] x [vmin, vmax] and the planes are
// e1 - umin a, umax a - e1, e2 - vmin a, vmax a - e2 (inward normals).
// Every box a lane's segment truly meets intersects this region, so the
// cone's leaf set is a superset of the per-lane union warp_traverse stages
// (each lane then filters with its own density setup, and the exact fp64
// emptiness test runs on the list as before).  The test is one box per lane:
// the 32 lanes test the 4 children of 8 nodes at once -- 8x fewer node steps
// than the per-lane packet test, where all 32 lanes test the same 4 children.
// ---------------------------------------------------------------------------
__device__ inline unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ inline float4 lds4(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a));
  return v;
}
__device__ inline int32_t lds_i(unsigned a) {
  int32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ inline void sts_i_if(unsigned a, int32_t v, bool p) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.b32 [%0], %1; }" ::"r"(a),
               "r"(v), "r"((unsigned)p)
               : "memory");
}
// warp-wide fp32 min / max: one redux.sync (sm_100a CREDUX.F32, result in a
// uniform register) instead of a 5-step shuffle tree
__device__ inline float warp_min(float x) {
  float r;
  asm volatile("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(x));
  return r;
}
__device__ inline float warp_max(float x) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(x));
  return r;
}

// Build the cone of the lanes with `want` (at least one) over [lo_t, hi_t]
// into sm.cone.  Margins: the (u, v) ranges are widened by 2e-5 (the fp32
// rounding of u, v is ~1e-7), the shell by 1e-6 relative (lo_t / hi_t already
// carry the traversal margin); boxes are widened in cone_box.
__device__ inline void make_cone(const RayCtx& r, bool want, float lo_t, float hi_t,
                                 WarpSmem& sm) {
  const unsigned m = __ballot_sync(FULL, want);
  const int leader = __ffs(m) - 1;
  float a[3], o[3];  // the leader's direction and the (common) origin: lanes
                    // without a ray (off-image, missing the scene) hold none
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    a[k] = __shfl_sync(FULL, r.df[k], leader);
    o[k] = __shfl_sync(FULL, r.of[k], leader);
  }
  // orthonormal basis around a (Duff et al. 2017, branch-free)
  const float sg = copysignf(1.f, a[2]);
  const float ia = -1.f / (sg + a[2]);
  const float b = a[0] * a[1] * ia;
  const float e1[3] = {1.f + sg * a[0] * a[0] * ia, sg * b, -sg * a[0]};
  const float e2[3] = {b, sg + a[1] * a[1] * ia, -a[1]};
  const float da = r.df[0] * a[0] + r.df[1] * a[1] + r.df[2] * a[2];
  const float u = (r.df[0] * e1[0] + r.df[1] * e1[1] + r.df[2] * e1[2]) / da;
  const float v = (r.df[0] * e2[0] + r.df[1] * e2[1] + r.df[2] * e2[2]) / da;
  const bool bad = __any_sync(FULL, want && !(da > 0.25f));
  const float umin = warp_min(want ? u : INFINITY) - 2e-5f;
  const float umax = warp_max(want ? u : -INFINITY) + 2e-5f;
  const float vmin = warp_min(want ? v : INFINITY) - 2e-5f;
  const float vmax = warp_max(want ? v : -INFINITY) + 2e-5f;
  const float tlo = fmaxf(warp_min(want ? lo_t : INFINITY), 0.f) * (1.f - 1e-6f);
  const float thi = warp_max(want ? hi_t : -INFINITY) * (1.f + 1e-6f);
  // eps_scale of the taking-part lanes (the others may hold no ray at all)
  const float es = warp_max(want ? r.eps_scale : 0.f);
  if ((threadIdx.x & 31) == 0) {
    // a packet wider than ~75 degrees (never for camera tiles) keeps only the shell
    float z = bad ? 0.f : 1.f;
    float th2 = thi * thi, tl2 = tlo * tlo;
#ifdef GSX_CONE_NOPLANES
    z = 0.f;
#endif
#ifdef GSX_CONE_NOSHELL
    th2 = INFINITY;
    tl2 = 0.f;
#endif
    sm.cone[0] = make_float4(o[0], o[1], o[2], tl2);
    sm.cone[1] = make_float4(z * (e1[0] - umin * a[0]), z * (e1[1] - umin * a[1]),
                             z * (e1[2] - umin * a[2]), th2);
    sm.cone[2] = make_float4(z * (umax * a[0] - e1[0]), z * (umax * a[1] - e1[1]),
                             z * (umax * a[2] - e1[2]), es);
    sm.cone[3] = make_float4(z * (e2[0] - vmin * a[0]), z * (e2[1] - vmin * a[1]),
                             z * (e2[2] - vmin * a[2]), tlo);
    sm.cone[4] = make_float4(z * (vmax * a[0] - e2[0]), z * (vmax * a[1] - e2[1]),
                             z * (vmax * a[2] - e2[2]), thi);
  }
  __syncwarp();
}

// Does box [lo, hi] meet the cone in sm.cone (address a_cone)?  Conservative:
// the half extents are widened by 1e-6 (|c| + h + eps_scale).
__device__ inline bool cone_box(unsigned a_cone, float lx, float ly, float lz, float hx,
                                float hy, float hz) {
  const float4 c0 = lds4(a_cone);
  const float es = lds4(a_cone + 32u).w;
  const float cx = fmaf(0.5f, lx + hx, -c0.x), cy = fmaf(0.5f, ly + hy, -c0.y),
              cz = fmaf(0.5f, lz + hz, -c0.z);
  float ex = 0.5f * (hx - lx), ey = 0.5f * (hy - ly), ez = 0.5f * (hz - lz);
  ex = fmaf(1e-6f, fabsf(cx) + ex + es, ex);
  ey = fmaf(1e-6f, fabsf(cy) + ey + es, ey);
  ez = fmaf(1e-6f, fabsf(cz) + ez + es, ez);
  // distance shell: nearest and farthest box point from o
  const float nx = fmaxf(fabsf(cx) - ex, 0.f), ny = fmaxf(fabsf(cy) - ey, 0.f),
              nz = fmaxf(fabsf(cz) - ez, 0.f);
  const float fx = fabsf(cx) + ex, fy = fabsf(cy) + ey, fz = fabsf(cz) + ez;
  const float dmin2 = fmaf(nx, nx, fmaf(ny, ny, nz * nz));
  const float dmax2 = fmaf(fx, fx, fmaf(fy, fy, fz * fz));
  bool ok = dmax2 >= c0.w;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const float4 n = lds4(a_cone + 16u * (1 + p));
    if (p == 0) ok = ok && dmin2 <= n.w;
    const float s = fmaf(n.x, cx, fmaf(n.y, cy, fmaf(n.z, cz, fmaf(fabsf(n.x), ex,
                    fmaf(fabsf(n.y), ey, fabsf(n.z) * ez)))));
    ok = ok && s >= 0.f;
  }
  return ok;
}

struct ConeTrav {
  int sp;
  bool done;
};

__device__ inline void cone_begin(WarpSmem& sm, ConeTrav& st) {
  if ((threadIdx.x & 31) == 0) sm.stack[0] = 0;  // root
  __syncwarp();
  st.sp = 1;
  st.done = false;
}

// Traverse the 4-wide BVH against the cone in sm.cone, appending leaves to
// sm.list.  Each step pops up to 8 nodes from the shared stack (depth-first:
// the most recently pushed) and tests their 4 children, one per lane; hit
// leaves are appended to the list and hit inner children pushed, both in lane
// order (ballot + popc ranks).  Resumable: returns when the stack is empty
// (st.done) or the list has fewer than 32 free entries.  The number of nodes
// popped shrinks as the stack fills (a step pushes at most 3 more than it
// pops), so the 256-entry stack overflows only for trees deeper than ~80.
#ifndef GSX_CONE_CPL
#define GSX_CONE_CPL 1  // children per lane and step (8 * CPL nodes per step)
#endif
__device__ inline void warp_traverse_cone(const BvhView& bv, ConeTrav& st, WarpSmem& sm,
                                          int& count, uint32_t& visits) {
  constexpr int CPL = GSX_CONE_CPL, KMAX = 8 * CPL;
  const unsigned a_list = (unsigned)__cvta_generic_to_shared(sm.list);
  const unsigned a_stack = (unsigned)__cvta_generic_to_shared(sm.stack);
  const unsigned a_cone = (unsigned)__cvta_generic_to_shared(sm.cone);
  const unsigned lane = threadIdx.x & 31, lt = lanemask_lt();
  const int slot = (int)(lane >> 2), c = (int)(lane & 3);
  while (st.sp > 0 && count <= LCAP - 32 * CPL) {
    int k = st.sp < KMAX ? st.sp : KMAX;
    const int room = (WSTACK - st.sp) / 3;
    k = k < room ? k : (room > 1 ? room : 1);
    const int base = st.sp - k;
    visits += (uint32_t)k;
    PH_CNT(8, k)
    int32_t chv[CPL];
    bool hitv[CPL];
#pragma unroll
    for (int h = 0; h < CPL; ++h) {
      const int sl = slot + 8 * h;
      const bool valid = sl < k;
      const int32_t node = valid ? lds_i(a_stack + 4u * (unsigned)(base + sl)) : 0;
      const float* nf = (const float*)(bv.nodes4 + 8 * (int64_t)node);
      chv[h] = __float_as_int(__ldg(nf + 24 + c));
      // (absent children have inf / -inf boxes: NaN centres fail every test)
      const bool cb = cone_box(a_cone, __ldg(nf + c), __ldg(nf + 4 + c), __ldg(nf + 8 + c),
                               __ldg(nf + 12 + c), __ldg(nf + 16 + c), __ldg(nf + 20 + c));
      hitv[h] = valid && chv[h] != GSX_NONE && cb;
    }
    int sp = base;
#pragma unroll
    for (int h = 0; h < CPL; ++h) {
      const int32_t ch = chv[h];
      const bool leaf = hitv[h] && ch < 0, inner = hitv[h] && ch >= 0;
      const unsigned bl = __ballot_sync(FULL, leaf), bi = __ballot_sync(FULL, inner);
      sts_i_if(a_list + 4u * (unsigned)(count + __popc(bl & lt)), ~ch, leaf);
      const int pos = sp + __popc(bi & lt);
      sts_i_if(a_stack + 4u * (unsigned)pos, ch, inner && pos < WSTACK);
      count += __popc(bl);
      const int np = sp + __popc(bi);
      if (np > WSTACK) sm.ovf = 1;  // dropped subtrees: the frame is flagged
      sp = np < WSTACK ? np : WSTACK;
    }
    st.sp = sp;
    __syncwarp();
  }
  st.done = st.sp == 0;
}

// Warp-cooperative ESS closest hit (closest_hit spatial.py:309-354): the
// lanes with `want` find their first ellipsoid entry in [t_lo, t_hi].  One
// packet traversal of the 4-wide BVH serves all of them (node loads and loop
// control shared, no per-lane stacks in local memory): a child is entered
// when any requesting lane's ray meets its box within [t_lo, min(t_hi, best)]
// (true intersection, fp32 with margin); children are visited near-first by
// the lowest requesting lane's entry distance so `best` shrinks early.  Leaf
// tests are the per-lane fp64 ones of closest_hit_r, and the result -- the
// minimum entry over every ellipsoid meeting [t_lo, t_hi] -- does not depend
// on the visiting order, so it equals the per-lane traversal's bit for bit.
// closest-hit leaf test (spatial.py:340-352): min(best, entry) of primitive p
#ifndef GSX_CHLEAF_ATTR
#define GSX_CHLEAF_ATTR inline
#endif
__device__ GSX_CHLEAF_ATTR double ch_leaf(const SceneView& sv, int64_t p, const RayCtx& r,
                                          double t_lo, double t_hi, double best) {
  double y0[3], yd[3];
  local_frame(sv.geo, p, r, y0, yd);
  double tin, tout;
  const double l2 = t_hi < best ? t_hi : best;
  if (ray_ellipsoid_interval64(y0, yd, t_lo, l2, tin, tout) && tin < best) best = tin;
  return best;
}

__device__ inline bool warp_closest_hit(const SceneView& sv, const BvhView& bv, const RayCtx& r,
                                        bool want, double t_lo, double t_hi, double& hit,
                                        WarpSmem& sm, uint32_t& visits) {
  want = want && !(t_lo > t_hi);
  const unsigned req = __ballot_sync(FULL, want);
  if (!req) return false;
  const int leader = __ffs(req) - 1;
  double best = INFINITY;
  const float lo_t = (float)t_lo - margin(r, (float)t_lo);
  const unsigned a_stack = (unsigned)__cvta_generic_to_shared(sm.stack);
  int sp = 0;
  int32_t node = 0;
  for (;;) {
    ++visits;
    const float4* nd = bv.nodes4 + 8 * (int64_t)node;
    const float4 lx = __ldg(nd), ly = __ldg(nd + 1), lz = __ldg(nd + 2);
    const float4 hx = __ldg(nd + 3), hy = __ldg(nd + 4), hz = __ldg(nd + 5);
    const float4 cf = __ldg(nd + 6);
    const float clo[3][4] = {{lx.x, lx.y, lx.z, lx.w}, {ly.x, ly.y, ly.z, ly.w},
                             {lz.x, lz.y, lz.z, lz.w}};
    const float chi[3][4] = {{hx.x, hx.y, hx.z, hx.w}, {hy.x, hy.y, hy.z, hy.w},
                             {hz.x, hz.y, hz.z, hz.w}};
    const int32_t ch[4] = {__float_as_int(cf.x), __float_as_int(cf.y), __float_as_int(cf.z),
                           __float_as_int(cf.w)};
    const double lim = t_hi < best ? t_hi : best;
    const float limf = (float)lim + margin(r, (float)lim);
    bool hk[4];
    float ent[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float x0 = (clo[0][k] - r.of[0]) * r.invf[0], x1 = (chi[0][k] - r.of[0]) * r.invf[0];
      float y0 = (clo[1][k] - r.of[1]) * r.invf[1], y1 = (chi[1][k] - r.of[1]) * r.invf[1];
      float z0 = (clo[2][k] - r.of[2]) * r.invf[2], z1 = (chi[2][k] - r.of[2]) * r.invf[2];
      float mn = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fminf(z0, z1));
      float mx = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fmaxf(z0, z1));
      hk[k] = want && ch[k] != GSX_NONE && mn <= limf && mx >= lo_t && mn <= mx + margin(r, mx);
      ent[k] = __shfl_sync(FULL, hk[k] ? mn : INFINITY, leader);
    }
    // near-first order by the leader's entry (4-element sorting network)
    int ord[4] = {0, 1, 2, 3};
#define GSX_CSWAP(i, j) \
    if (ent[ord[j]] < ent[ord[i]]) { const int t_ = ord[i]; ord[i] = ord[j]; ord[j] = t_; }
    GSX_CSWAP(0, 1) GSX_CSWAP(2, 3) GSX_CSWAP(0, 2) GSX_CSWAP(1, 3) GSX_CSWAP(1, 2)
#undef GSX_CSWAP
    int32_t next = -1;
    // leaves first (in near order): they can only shrink `best`
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = ord[i];
      const bool h = hk[k];
      if (!__any_sync(FULL, h) || ch[k] >= 0) continue;
      if (h) best = ch_leaf(sv, ~(int64_t)ch[k], r, t_lo, t_hi, best);
    }
    // inner children: descend into the nearest, push the others far-first
#pragma unroll
    for (int i = 3; i >= 0; --i) {
      const int k = ord[i];
      if (!__any_sync(FULL, hk[k]) || ch[k] < 0) continue;
      if (next >= 0 && sp < WSTACK) {
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(a_stack + 4u * sp), "r"(next) : "memory");
        ++sp;
      } else if (next >= 0) {
        sm.ovf = 1;
      }
      next = ch[k];
    }
    __syncwarp();
    if (next < 0) {
      if (sp == 0) break;
      --sp;
      next = sm.stack[sp];
    }
    node = next;
  }
  __syncwarp();
  if (want && best < INFINITY) {
    hit = best;
    return true;
  }
  return false;
}

// fp32 true ray/box intersection of primitive p's outward-rounded box with
// [lo_t, hi_t] (margins included by the caller; gap as in traverse_segment)
__device__ inline bool box32_hit(const SceneView& sv, const RayCtx& r, int64_t p, float lo_t,
                                 float hi_t, float gap) {
  const float2* b = (const float2*)(sv.box32 + 6 * p);
  const float2 b0 = __ldg(b), b1 = __ldg(b + 1), b2 = __ldg(b + 2);
  const float x0 = (b0.x - r.of[0]) * r.invf[0], x1 = (b1.y - r.of[0]) * r.invf[0];
  const float y0 = (b0.y - r.of[1]) * r.invf[1], y1 = (b2.x - r.of[1]) * r.invf[1];
  const float z0 = (b1.x - r.of[2]) * r.invf[2], z1 = (b2.y - r.of[2]) * r.invf[2];
  const float mn = fmaxf(fmaxf(fminf(x0, x1), fminf(y0, y1)), fminf(z0, z1));
  const float mx = fminf(fminf(fmaxf(x0, x1), fmaxf(y0, y1)), fmaxf(z0, z1));
  return mn <= hi_t && mx >= lo_t && mn <= mx + gap;
}

// Cone-window ESS closest hit (camera rays; closest_hit spatial.py:309-354):
// the requesting lanes search depth windows [A, A + w), w doubling, each by a
// packet-cone traversal of the window; every listed leaf whose box a lane's
// ray truly meets (fp32, margins) gets the lane's fp64 leaf test.  A lane is
// done once its best entry is <= the window end: every ellipsoid its ray
// meets in [t_lo, B] has its box in one of the windows' cones, so no
// undiscovered one can enter earlier.  The minimum over the same fp64 leaf
// tests as warp_closest_hit, hence the same hit bit for bit.
__device__ inline bool warp_closest_hit_cone(const SceneView& sv, const BvhView& bv,
                                             const RayCtx& r, bool want, double t_lo,
                                             double t_hi, double& hit, WarpSmem& sm,
                                             uint32_t& visits) {
  want = want && !(t_lo > t_hi);
  if (!__any_sync(FULL, want)) return false;
  double best = INFINITY;
  bool pend = want;
  float A = warp_min(want ? (float)t_lo : INFINITY);
  float w = warp_max(want ? (float)(t_hi - t_lo) * (1.f / 64.f) : 0.f);
  while (__any_sync(FULL, pend)) {
    w = fmaxf(w, 1e-6f * (fabsf(A) + 1.f));
    const float B = A + w;
    const double lim = t_hi < best ? t_hi : best;
    float lo = fmaxf((float)t_lo, A), hi = fminf((float)lim, B);
    lo -= margin(r, lo);
    hi += margin(r, hi);
    const bool part = pend && lo <= hi;
    if (__any_sync(FULL, part)) {
      make_cone(r, part, lo, hi, sm);
      ConeTrav st;
      cone_begin(sm, st);
      int count = 0;
      const float blo = (float)t_lo - margin(r, (float)t_lo);
      for (;;) {
        warp_traverse_cone(bv, st, sm, count, visits);
        for (int i = 0; i < count; ++i) {
          const int64_t p = sm.list[i];
          const double l2 = t_hi < best ? t_hi : best;
          const float bhi = (float)l2 + margin(r, (float)l2);
          if (part && box32_hit(sv, r, p, blo, bhi, margin(r, bhi)))
            best = ch_leaf(sv, p, r, t_lo, t_hi, best);
        }
        __syncwarp();
        if (st.done) break;
        count = 0;
      }
    }
    pend = pend && !(best <= (double)B) && t_hi > (double)B;
    A = B;
    w *= 2.f;
  }
  if (want && best < INFINITY) {
    hit = best;
    return true;
  }
  return false;
}

// Traversal-stack overflow bookkeeping of one warp: cleared at the start of
// the warp's work, reported once at the end (GSX_ERR_STACK with the pixel /
// ray index of lane 0) through the launch's status word.
__device__ inline void ovf_begin(WarpSmem& sm) {
  if ((threadIdx.x & 31) == 0) sm.ovf = 0;
  __syncwarp();
}
__device__ inline void ovf_report(const WarpSmem& sm, const BvhView& bv, int64_t index) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0 && sm.ovf) dev_fail(bv.status, GSX_ERR_STACK, index);
}

// per-lane description of the segment processed in this warp iteration
struct Seg {
  double t0, t1, tbase, dt, ds;
  int m;
  // sample j sits at tgrid + (j0 + j + 0.5) dt, exactly as the reference
  // forms it (uniform: global grid from t_n; adaptive: from t_s)
  double tgrid;
  long long j0;
  long long cap;  // buffer_capacity (stats only: reference overflow splitting)
};

struct SegLimits {
  float lo_t, hi_t, gap;
};
__device__ inline SegLimits seg_limits(const RayCtx& r, const struct Seg& seg) {
  SegLimits l;
  l.lo_t = (float)seg.t0 - margin(r, (float)seg.t0);
  l.hi_t = (float)seg.t1 + margin(r, (float)seg.t1);
  l.gap = margin(r, (float)seg.t1);
  return l;
}

// traversal limits of an arbitrary interval [a, b] of the ray
__device__ inline SegLimits interval_limits(const RayCtx& r, double a, double b) {
  SegLimits l;
  l.lo_t = (float)a - margin(r, (float)a);
  l.hi_t = (float)b + margin(r, (float)b);
  l.gap = margin(r, (float)b);
  return l;
}

// Stage the candidates of this iteration's segments: traverse [t0, t1] (with
// margins).  On return `count` entries are in sm.list; st.done == false means
// the list is only the first chunk of a longer stream (the caller continues
// with warp_traverse and the bounds in lim).
// (A look-ahead window reused across iterations was measured slower: only 29%
// of iterations could reuse it -- lanes ESS-jump or outgrow it -- while every
// list grew by ~70%.)
__device__ inline void stage_candidates(const BvhView& bv, const RayCtx& r, bool want,
                                        const Seg& seg, WarpSmem& sm, WarpTrav& st, int& count,
                                        SegLimits& lim, uint32_t& visits) {
  lim = seg_limits(r, seg);
  st = WarpTrav{0, 0, false, false};
  count = 0;
  PH_BEGIN(ph_t)
  warp_traverse(bv, r, want, lim.lo_t, lim.hi_t, lim.gap, st, sm, count, visits);
  PH_END(1, ph_t)
}

// Setup half of the pass-1 accumulation: whether this lane's samples see p.
struct CandUse {
  CandSetup cs;
  int jlo, jhi;
  bool use;
};
template <class L = LdgLoad>
__device__ inline CandUse candidate_use_at(const float4* geo, const RayCtx& r, bool want, int mc,
                                           const SegBase& base, float dtf) {
  CandUse u;
  u.jlo = 0;
  u.jhi = -1;
  u.use = want && mc > 0 && cand_setup_at<L>(geo, r, base, u.cs) &&
          sample_range(u.cs, dtf, mc, u.jlo, u.jhi);
  return u;
}
__device__ inline CandUse candidate_use(const SceneView& sv, const RayCtx& r, int64_t p,
                                        bool want, int mc, const SegBase& base, float dtf) {
  return candidate_use_at(sv.geo + 4 * p, r, want, mc, base, dtf);
}

// Pass-1 accumulation of one candidate into the 16 per-sample sums
// (renderer.py:218-228), given its setup.
// Returns the lanes that set p up (0 if none; the logged forward stores it).
template <class L = LdgLoad, int CH = 16, class YT = const float*>
__device__ inline unsigned accumulate_used_at(const float4* app, const RayCtx& r, const CandUse& u,
                                          float dtf, YT Y, float (&sig)[CH],
                                          float (&W)[CH][3]) {
  const CandSetup& cs = u.cs;
  const bool use = u.use;
  const int jlo = u.jlo, jhi = u.jhi;
  PH_CNT(9, 1)
  PH_LANES(11, use)
  const unsigned um = __ballot_sync(FULL, use);
  if (!um) return 0u;
  PH_CNT(14, 1)
  float c[3] = {0.f, 0.f, 0.f};
  if (use) eval_radiance_f<L, YT>(app, Y, r.df, c);
  const float nkl2 = -cs.kl2;
  // 4-sample groups outside every lane's range are skipped warp-uniformly
#pragma unroll
  for (int g = 0; g < CH / 4; ++g) {
    if (!__any_sync(FULL, use && jlo <= 4 * g + 3 && jhi >= 4 * g)) continue;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * g + jj;
      float del = fmaf((float)j, dtf, cs.del0);
      float q = fmaf(cs.A * del, del, cs.qmin);
      if (use && q <= 1.0f) {
        // sigma~ exp(-k q / 2) = 2^(log2 sigma~ - k log2(e) q / 2)
        float dens = ex2_approx(fmaf(nkl2, q, cs.lsig));
        sig[j] += dens;
        W[j][0] = fmaf(dens, c[0], W[j][0]);
        W[j][1] = fmaf(dens, c[1], W[j][1]);
        W[j][2] = fmaf(dens, c[2], W[j][2]);
      }
    }
  }
  return um;
}

template <int CH, class YT>
__device__ inline unsigned accumulate_used(const SceneView& sv, const RayCtx& r, int64_t p,
                                       const CandUse& u, float dtf, YT Y,
                                       float (&sig)[CH], float (&W)[CH][3]) {
  return accumulate_used_at(sv.app + GSX_APP_F4 * p, r, u, dtf, Y, sig, W);
}

template <int CH, class YT>
__device__ inline unsigned accumulate_candidate(const SceneView& sv, const RayCtx& r, int64_t p,
                                            bool want, int mc, const SegBase& base, float dtf,
                                            YT Y, float (&sig)[CH],
                                            float (&W)[CH][3]) {
  const CandUse u = candidate_use(sv, r, p, want, mc, base, dtf);
  return accumulate_used(sv, r, p, u, dtf, Y, sig, W);
}

// Pass 1 over a staged list in list order.  (Interleaving two candidates'
// setups for ILP measured slower: the extra live state spills at 128 regs.)
// post(i, p, lanes that used entry i) after each entry (warp-uniform; the
// logged forward records it).
template <class Pre, class Post, int CH, class YT>
__device__ inline void accumulate_list(const SceneView& sv, const RayCtx& r, WarpSmem& sm,
                                       int count, bool want, int mc, const SegBase& base,
                                       float dtf, YT Y, float (&sig)[CH], float (&W)[CH][3],
                                       Pre&& pre, Post&& post) {
  // (L1 prefetch of the listed geometry / appearance blocks measured slower:
  // 40.9 vs 40.0 ms on C3 -- the entry loop is not load-latency bound)
  for (int i = 0; i < count; ++i) {
    const int64_t p = sm.list[i];
    pre(p, want);
    post(i, p, accumulate_candidate(sv, r, p, want, mc, base, dtf, Y, sig, W));
  }
}


// ---------------------------------------------------------------------------
// Silhouette screen (camera rays).  view[2p] / view[2p+1] hold primitive p's
// image-space silhouette for the current camera (k_view_conics, render.cu):
// the pixels whose ray line meets the (1e-3-inflated) ellipsoid are the
// ellipse (X - Xc, Y - Yc) A (X - Xc, Y - Yc)^T <= 1, stored as
// (Xc, Yc, A00, 2 A01) (A11, -, -, -); A00 = 0 marks "no screen" (camera
// inside, or the ellipsoid crossing the camera plane: every lane passes).
// The list is screened entry-parallel: lane l evaluates entry b + l against
// the warp's 32 pixel centres (an 8x4 block; lanes in Z-order) and stores the
// 32-bit mask of lanes it may touch.  A superset of the lanes whose setup
// (cand_setup_at) can succeed, so the accumulation skips every other
// (lane, entry) pair and every entry no lane can use.
// ---------------------------------------------------------------------------
struct Screen {
  const float4* view;  // nullptr: no screening
  float x0, y0;        // pixel of the warp block's lane 0
};

// Per-warp shared state of the screened forward: the base block, the
// screen masks of the current list, and the 16 per-sample sums (sigma_j,
// W_j rgb) of every lane as one float4 column per lane (acc[j][lane]).
// Held in shared memory instead of registers: at the 64-register cap of 32
// warps per SM they lived in local memory (4 LDL + 4 STL per sample update,
// missing L1 -- the dominant long-scoreboard stall of the r06 capture).
#ifndef GSX_SCR_CH
#define GSX_SCR_CH 16
#endif
template <int CH>
struct WarpSmemA : WarpSmemT {  // screened forward, sums in shared memory
  float4 acc[CH][32];
};

// Where a lane's per-sample sums live: its shared-memory column ...
struct SmemSums {
  float4* col;  // &acc[0][lane], stride 32
  __device__ void zero(int ch) const {
    for (int j = 0; j < ch; ++j) col[32 * j] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __device__ void add(int j, float dens, const float* c) const {
    float4 a = col[32 * j];
    a.x += dens;
    a.y = fmaf(dens, c[0], a.y);
    a.z = fmaf(dens, c[1], a.z);
    a.w = fmaf(dens, c[2], a.w);
    col[32 * j] = a;
  }
  __device__ float4 get(int j) const { return col[32 * j]; }
};
// ... or registers (a 64-register cap spills them to local memory)
template <int CH>
struct RegSums {
  float sig[CH];
  float W[CH][3];
  __device__ void zero(int) {
#pragma unroll
    for (int j = 0; j < CH; ++j) sig[j] = W[j][0] = W[j][1] = W[j][2] = 0.f;
  }
  __device__ void add(int j, float dens, const float* c) {
    sig[j] += dens;
    W[j][0] = fmaf(dens, c[0], W[j][0]);
    W[j][1] = fmaf(dens, c[1], W[j][1]);
    W[j][2] = fmaf(dens, c[2], W[j][2]);
  }
  __device__ float4 get(int j) const { return make_float4(sig[j], W[j][0], W[j][1], W[j][2]); }
};

// Silhouette mask of primitive p over the warp's 32 pixel centres.
__device__ inline unsigned screen_entry(const Screen& sc, int64_t p) {
  const float4 c0 = __ldg(sc.view + 2 * p);
  if (!(c0.z > 0.f)) return FULL;
  const float a11 = __ldg(sc.view + 2 * p + 1).x;
  unsigned m = 0u;
  float dx[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) dx[k] = (sc.x0 + (0.5f + (float)k)) - c0.x;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float dy = (sc.y0 + (0.5f + (float)j)) - c0.y;
    const float r1 = c0.w * dy, r2 = fmaf(a11 * dy, dy, -1.f);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      // Z-order lane of pixel (k, j): x bits at 0, 2, 4; y bits at 1, 3
      const int l = (k & 1) | ((k & 2) << 1) | ((k & 4) << 2) | ((j & 1) << 1) | ((j & 2) << 2);
      const float q = fmaf(dx[k], fmaf(c0.z, dx[k], r1), r2);
      m |= q <= 0.f ? (1u << l) : 0u;
    }
  }
  return m;
}

// Screened pass 1 (screen_accumulate): `inside` is set when a sample lies
// clearly inside an ellipsoid (q <= 0.998 in fp32): that sample is then
// inside the primitive's fp64 AABB too, so the segment is AABB-non-empty in
// the reference's sense (spatial.py:234-241) without the exact slab test.
//
// Samples of one set-up entry into the lane's sums (the
// 4-sample groups outside every lane's range skipped warp-uniformly); q <= 1
// decides exactly, as in accumulate_used_at.  Returns the lane's smallest
// accumulated q (2 if none).
template <int CH, class Sums>
__device__ inline float screened_samples(const CandUse& u, const float* c, float dtf,
                                         Sums& sums) {
  const CandSetup& cs = u.cs;
  const float nkl2 = -cs.kl2;
  float qmn = 2.f;
#pragma unroll
  for (int g = 0; g < CH / 4; ++g) {
    if (!__any_sync(FULL, u.use && u.jlo <= 4 * g + 3 && u.jhi >= 4 * g)) continue;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * g + jj;
      const float del = fmaf((float)j, dtf, cs.del0);
      const float q = fmaf(cs.A * del, del, cs.qmin);
      if (u.use && q <= 1.0f) {
        sums.add(j, ex2_approx(fmaf(nkl2, q, cs.lsig)), c);
        qmn = fminf(qmn, q);
      }
    }
  }
  return qmn;
}

// Screen + pass 1 in batches of 32 list entries: lane e screens entry b + e
// and keeps its mask in a register; the batch's screened-in entries are then
// processed in list order with the mask and the primitive broadcast by
// shuffles (entries no lane can use are skipped warp-uniformly, and a lane
// sets up only the entries whose mask holds it).  After each batch every
// lane calls post(p, lanes that used p) for its entry (0: unused or beyond
// the list; warp-converged: the logged forward compacts them with a ballot).
#if GSX_APP_TMA
// The radiance needs the entry's whole appearance block (368 B, the same for
// every lane): loaded by the warp's lanes it costs a chain of L2 round trips
// at 64 registers.  Instead lane 0 has the TMA engine copy it into a warp
// buffer (cp.async.bulk, completion on an mbarrier) one entry ahead, while
// the current entry is set up and evaluated; the lanes then read it from
// shared memory.
__device__ inline void app_barriers_init(WarpSmemT& sm) {
  if ((threadIdx.x & 31) == 0) {
    for (int b = 0; b < GSX_APP_NB; ++b) {
      const unsigned mb = (unsigned)__cvta_generic_to_shared(&sm.mbar[b]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
#if GSX_GEO_TMA
      const unsigned gb = (unsigned)__cvta_generic_to_shared(&sm.gbar[b]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(gb) : "memory");
#endif
    }
    sm.mpar = 0u;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
}
// lane 0: buffer b <- primitive p's appearance block (and, GSX_GEO_TMA,
// geometry block); the buffer's previous contents consumed
__device__ inline void app_issue(WarpSmemT& sm, int b, const SceneView& sv, int64_t p) {
  constexpr unsigned ABYTES = 16u * GSX_APP_F4, GBYTES = 64u;
  const unsigned mb = (unsigned)__cvta_generic_to_shared(&sm.mbar[b]);
  const unsigned adst = (unsigned)__cvta_generic_to_shared(&sm.appb[b][0]);
#if GSX_GEO_TMA
  const unsigned gb = (unsigned)__cvta_generic_to_shared(&sm.gbar[b]);
  const unsigned gdst = (unsigned)__cvta_generic_to_shared(&sm.geob[b][0]);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(gb), "r"(GBYTES)
               : "memory");
#endif
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(ABYTES)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(adst),
      "l"(sv.app + GSX_APP_F4 * p), "r"(ABYTES), "r"(mb)
      : "memory");
#if GSX_GEO_TMA
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(gdst),
      "l"(sv.geo + 4 * p), "r"(GBYTES), "r"(gb)
      : "memory");
#else
  (void)GBYTES;
#endif
}
// generic forms (raw shared-memory pointers): barrier init, one bulk copy
// global -> shared completing on `bar`
__device__ inline void tma_bar_init(unsigned long long* bar) {
  const unsigned mb = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
}
__device__ inline void tma_copy(void* dst, const void* src, unsigned bytes,
                                unsigned long long* bar) {
  const unsigned mb = (unsigned)__cvta_generic_to_shared(bar);
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(d),
      "l"(src), "r"(bytes), "r"(mb)
      : "memory");
}
__device__ inline void bar_wait(const unsigned long long* bar, unsigned parity) {
  const unsigned mb = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(mb),
      "r"(parity)
      : "memory");
}
#endif

template <int CH, class YT, class Sums, class Post>
__device__ inline void screen_accumulate(const Screen& sc, const SceneView& sv, const RayCtx& r,
                                         WarpSmemT& sm, int count, unsigned lanes,
                                         bool want, int mc, const SegBase& base, float dtf, YT Y,
                                         Sums& sums, bool& inside, Post&& post) {
  const unsigned lane = threadIdx.x & 31;
  float qmn = 2.f;
#if GSX_APP_TMA
  unsigned par = sm.mpar;
#endif
  for (int b = 0; b < count; b += 32) {
    const int i = b + (int)lane;
    const int32_t pl = i < count ? sm.list[i] : 0;
    PH_BEGIN(ph_s)
    const unsigned ml = i < count ? screen_entry(sc, pl) & lanes : 0u;
    PH_END(16, ph_s)
    unsigned todo = __ballot_sync(FULL, ml != 0u);
    unsigned mine = 0u;  // lanes that used this lane's entry
#if GSX_APP_TMA
    constexpr int NB = GSX_APP_NB, D = GSX_APP_NB - 1;  // buffers, staging distance
    int bi = 0;
    {
      unsigned t = todo;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int32_t pd = __shfl_sync(FULL, pl, t ? __ffs(t) - 1 : 0);
        if (t && lane == 0) app_issue(sm, d, sv, pd);
        t &= t - 1;
      }
    }
#endif
    while (todo) {
      const int e = __ffs(todo) - 1;
      todo &= todo - 1;
      PH_CNT(21, 1)
      const unsigned m = __shfl_sync(FULL, ml, e);
      const int64_t p = __shfl_sync(FULL, pl, e);
#if GSX_APP_TMA
      {
        // the entry D ahead into the buffer the previous iteration read
        // (every lane's reads ordered before the copy)
        unsigned t = todo;
#pragma unroll
        for (int d = 1; d < D; ++d) t &= t - 1;
        const int32_t pn = __shfl_sync(FULL, pl, t ? __ffs(t) - 1 : 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (t && lane == 0) app_issue(sm, (bi + D) % NB, sv, pn);
      }
      const int bc = bi;  // this entry's buffer
      const unsigned pc = (par >> bc) & 1u;
      par ^= 1u << bc;
      bi = bi + 1 == NB ? 0 : bi + 1;
      PH_BEGIN(ph_u)
#if GSX_GEO_TMA
      bar_wait(&sm.gbar[bc], pc);
      const CandUse u =
          candidate_use_at<PlainLoad>(&sm.geob[bc][0], r, want && ((m >> lane) & 1u), mc, base,
                                      dtf);
#else
      const CandUse u = candidate_use(sv, r, p, want && ((m >> lane) & 1u), mc, base, dtf);
#endif
#else
      PH_BEGIN(ph_u)
      const CandUse u = candidate_use(sv, r, p, want && ((m >> lane) & 1u), mc, base, dtf);
#endif
      const unsigned um = __ballot_sync(FULL, u.use);
      PH_END(17, ph_u)
      if (lane == (unsigned)e) mine = um;
#if GSX_APP_TMA
      bar_wait(&sm.mbar[bc], pc);  // (both barriers complete a phase per use)
      const float4* appp = &sm.appb[bc][0];
#endif
      if (!um) continue;
      float c[3] = {0.f, 0.f, 0.f};
      PH_BEGIN(ph_r)
#if GSX_APP_TMA
      if (u.use) eval_radiance_f<PlainLoad, YT>(appp, Y, r.df, c);
#else
      if (u.use) eval_radiance_f<LdgLoad, YT>(sv.app + GSX_APP_F4 * p, Y, r.df, c);
#endif
      PH_END(18, ph_r)
      PH_BEGIN(ph_m)
      qmn = fminf(qmn, screened_samples<CH>(u, c, dtf, sums));
      PH_END(19, ph_m)
      PH_CNT(20, 1)
    }
    post(pl, mine);
  }
#if GSX_APP_TMA
  if (lane == 0) sm.mpar = par;
  __syncwarp();
#endif
  inside = inside || qmn <= 0.998f;
}

// Exact AABB-emptiness of the lane's segment (reference semantics) after the
// true-intersection pass; STATS additionally counts every exact overlap.
template <bool STATS>
static __device__ GSX_COLD void emptiness_tail(const SceneView& sv, const BvhView& bv, const RayCtx& r,
                                      bool want, const Seg& seg, bool& nonempty,
                                      Counters<STATS>& cnt, int& sm_ovf) {
  PH_BEGIN(ph_ph)
  if (STATS) {
    if (want) {
      // exact reference counts: AABB overlaps (with inverted "phantom"
      // intervals) and ellipsoid hits of [a, b]
      auto count = [&](double a, double b, uint32_t& na, uint32_t& ne) {
        na = ne = 0;
        uint32_t v2 = 0;
        auto fn = [&](int64_t p) -> bool {
          if (exact_aabb_overlap(sv, r, p, a, b)) {
            na++;
            if (ellipsoid_hits_interval(sv, r, p, a, b)) ne++;
          }
          return false;
        };
        if (!traverse_segment<true>(bv, r, (float)a, (float)b, fn, v2)) sm_ovf = 1;
      };
      // _collect_split (renderer.py:361-393): a collect of more than
      // buffer_capacity boxes splits the segment at its midpoint (samples
      // t_j < mid go left) until it fits or holds one sample; every leaf
      // collect that is non-empty counts one segment, its samples and its
      // hits -- the reference's counters, not just its image
      struct Part {
        double a, b;
        int jlo, jhi;
      };
      Part stk[12];
      int sp = 0;
      stk[sp++] = Part{seg.t0, seg.t1, 0, seg.m};
      bool any = false, top = true;
      while (sp > 0) {
        const Part q = stk[--sp];
        uint32_t na, ne;
        count(q.a, q.b, na, ne);
        // `pairs` (ours, the roofline's work unit) is per Alg. 1 segment:
        // samples x AABB overlaps of the whole segment, as the kernel does it
        if (top) cnt.pairs += (uint32_t)seg.m * na;
        top = false;
        if (na == 0) continue;
        const int ns = q.jhi - q.jlo;
        if ((int64_t)na <= seg.cap || ns <= 1 || sp + 2 > 12) {
          any = true;
          cnt.segments++;
          cnt.samples += (uint32_t)ns;
          cnt.aabb += na;
          cnt.ell += ne;
          continue;
        }
        const double mid = 0.5 * (q.a + q.b);
        int js = q.jlo;
        while (js < q.jhi && seg.tgrid + ((double)(seg.j0 + js) + 0.5) * seg.dt < mid) ++js;
        stk[sp++] = Part{mid, q.b, js, q.jhi};  // right popped after left
        stk[sp++] = Part{q.a, mid, q.jlo, js};
      }
      nonempty = any;
    }
  } else if (want && !nonempty) {
    // no true overlap: empty unless an inverted-interval ("phantom") overlap exists
    uint32_t v2 = 0;
    auto probe = [&](int64_t p) -> bool {
      if (exact_aabb_overlap(sv, r, p, seg.t0, seg.t1)) nonempty = true;
      return nonempty;
    };
    if (!traverse_segment<true>(bv, r, (float)seg.t0, (float)seg.t1, probe, v2)) sm_ovf = 1;
  }
  PH_END(4, ph_ph)
}

// Alg. 1 for one lane's ray in warp lockstep (renderer.py:288-358).
// segfn(seg, want) processes one segment for all lanes and returns the lane's
// exact AABB-emptiness verdict (true = non-empty).
// `sync` = depth-synchronous window in segment lengths (0 = every active lane
// takes part every iteration).
template <bool STATS, bool CONE_CH = false, class SegFn>
__device__ inline void march_warp(const SceneView& sv, const BvhView& bv, const RayCtx& r,
                                  bool hit, const gsx_render_cfg& cfg, const RayAccum& acc,
                                  Counters<STATS>& cnt, float sync, WarpSmem& sm,
                                  SegFn&& segfn) {
  const int ns = (int)cfg.n_s;
  const bool uniform = cfg.mode == 0;
  const double t_n = r.t_n, t_f = r.t_f;
  const double ds_u = cfg.dt * (double)ns;
  long long k = 0, n_seg = 0;
  double t_s = t_n;
  bool active = hit;
  uint32_t visits = 0;
  PH_BEGIN(ph_all)
  if (active && uniform) {
    n_seg = (long long)ceil((t_f - t_n) / ds_u);
    if (n_seg < 1) n_seg = 1;
  }
  // ESS closest-hit requests -- the initial one from t_n and the restart after
  // every empty segment -- are served at one call site at the top of the loop
  // (one inlined copy of the traversal instead of two)
  bool need_ch = active && cfg.ess, first_ch = true;
  double ch_from = t_n;
  while (__any_sync(FULL, active)) {
    PH_BEGIN(ph_ch)
    if (__any_sync(FULL, need_ch)) {
      double h = 0.0;
      const bool got =
          CONE_CH ? warp_closest_hit_cone(sv, bv, r, need_ch, ch_from, t_f, h, sm, visits)
                  : warp_closest_hit(sv, bv, r, need_ch, ch_from, t_f, h, sm, visits);
      if (need_ch) {
        if (STATS) cnt.ch_calls++;
        if (!got) {
          active = false;
        } else if (uniform) {
          const long long kk = (long long)((h - t_n) / ds_u), kmin = first_ch ? 0 : k + 1;
          k = kk > kmin ? kk : kmin;
        } else {
          t_s = h;  // adaptive mode has no global grid: restart here
        }
        need_ch = false;
        first_ch = false;
      }
    }
    PH_END(0, ph_ch)
    if (active) {
      if (uniform)
        active = k < n_seg && acc.transmittance() > cfg.t_eps;
      else
        active = t_s < t_f && acc.transmittance() > cfg.t_eps;
    }
    Seg seg{0, 0, 0, 0, 0, 0, 0.0, 0, cfg.buffer_capacity};
    if (active) {
      if (uniform) {
        seg.t0 = t_n + (double)k * ds_u;
        seg.t1 = seg.t0 + ds_u;
        if (t_f < seg.t1) seg.t1 = t_f;
        seg.dt = cfg.dt;
        long long j0 = k * ns;
        for (int j = 0; j < ns; ++j)
          if (t_n + ((double)(j0 + j) + 0.5) * cfg.dt < t_f) seg.m = j + 1;
        seg.tbase = t_n + ((double)j0 + 0.5) * cfg.dt;
        seg.tgrid = t_n;
        seg.j0 = j0;
      } else {
        seg.ds = segment_step(cfg, t_s, (double)acc.transmittance());
        seg.dt = seg.ds / (double)ns;
        seg.t0 = t_s;
        seg.t1 = t_s + seg.ds;
        if (t_f < seg.t1) seg.t1 = t_f;
        for (int j = 0; j < ns; ++j)
          if (t_s + ((double)j + 0.5) * seg.dt < t_f) seg.m = j + 1;
        seg.tbase = t_s + 0.5 * seg.dt;
        seg.tgrid = t_s;
        seg.j0 = 0;
      }
    }
    if (!__any_sync(FULL, active)) break;
    // depth-synchronous scheduling: only lanes whose segment starts within
    // GSX_SYNC segment lengths of the warp's shallowest active lane take part;
    // lanes further ahead wait (their state is untouched, so they recompute
    // the same segment next iteration).  Each lane still marches its own
    // segments in its own order -- only the interleaving changes -- but the
    // packet's union of segments stays tight.
    bool go = active;
    if (sync > 0.f) {
      float t0f = active ? (float)seg.t0 : INFINITY;
      const float dmin = warp_min(t0f);
      go = active && t0f <= dmin + sync * (float)(seg.t1 - seg.t0);
    }
    PH_CNT(10, 1)
    PH_LANES(13, go)
    const bool ne = segfn(seg, go);
    PH_BEGIN(ph_adv)
    if (go) {
      if (ne) {  // (STATS: segments / samples are counted by emptiness_tail)
        if (uniform)
          k += 1;
        else
          t_s = t_s + seg.ds;
      } else {
        if (STATS) cnt.skipped++;
        if (cfg.ess) {
          need_ch = true;  // served at the top of the next iteration
          ch_from = seg.t1;
        } else {
          if (STATS) cnt.samples += seg.m;
          if (uniform)
            k += 1;
          else
            t_s = t_s + seg.ds;
        }
      }
    }
    PH_END(5, ph_adv)
  }
  PH_END(6, ph_all)
  if (STATS) cnt.visits += visits;
}

}  // namespace gsx
