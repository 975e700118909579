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
#ifndef GSX_SYNC_BWD
#define GSX_SYNC_BWD 0.5f
#endif
constexpr int LCAP = 256;    // warp candidate list (shared memory)
constexpr int WSTACK = 256;  // warp traversal stack (shared memory)

// Optional per-phase warp-time accounting (experiment builds only:
// nvcc -DGSX_PHASE_PROF); compiled out of the product library.
#ifdef GSX_PHASE_PROF
// one copy per translation unit (no -rdc); gsx_phase_times reads render.cu's
static __device__ unsigned long long g_phase[16];
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

struct WarpSmem {
  int32_t stack[WSTACK];
  int32_t list[LCAP];
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

// Visit every candidate of the warp's union traversal: f(p) is called by all
// 32 lanes in lockstep for each staged primitive p (list chunks of LCAP).
template <class F>
__device__ inline void for_each_candidate(const BvhView& bv, const RayCtx& r, bool want,
                                          float lo_t, float hi_t, float gap, WarpSmem& sm,
                                          uint32_t& visits, F&& f) {
  WarpTrav st{0, 0, false, false};
  int count = 0;
  for (;;) {
    PH_BEGIN(ph_t)
    warp_traverse(bv, r, want, lo_t, hi_t, gap, st, sm, count, visits);
    PH_END(1, ph_t)
    PH_BEGIN(ph_p)
    for (int i = 0; i < count; ++i) f((int64_t)sm.list[i]);
    PH_END(2, ph_p)
    __syncwarp();
    count = 0;
    if (st.done) break;
  }
}

// Same traversal, but f(count) is called once per staged chunk of the list.
template <class F>
__device__ inline void for_each_chunk(const BvhView& bv, const RayCtx& r, bool want, float lo_t,
                                      float hi_t, float gap, WarpSmem& sm, uint32_t& visits,
                                      F&& f) {
  WarpTrav st{0, 0, false, false};
  int count = 0;
  for (;;) {
    PH_BEGIN(ph_t)
    warp_traverse(bv, r, want, lo_t, hi_t, gap, st, sm, count, visits);
    PH_END(1, ph_t)
    PH_BEGIN(ph_p)
    f(count);
    PH_END(2, ph_p)
    __syncwarp();
    count = 0;
    if (st.done) break;
  }
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
      if (h) {
        const int64_t p = ~(int64_t)ch[k];
        double y0[3], yd[3];
        local_frame(sv.geo, p, r, y0, yd);
        double tin, tout;
        const double l2 = t_hi < best ? t_hi : best;
        if (ray_ellipsoid_interval64(y0, yd, t_lo, l2, tin, tout) && tin < best) best = tin;
      }
    }
    // inner children: descend into the nearest, push the others far-first
#pragma unroll
    for (int i = 3; i >= 0; --i) {
      const int k = ord[i];
      if (!__any_sync(FULL, hk[k]) || ch[k] < 0) continue;
      if (next >= 0 && sp < WSTACK) {
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(a_stack + 4u * sp), "r"(next) : "memory");
        ++sp;
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
__device__ inline CandUse candidate_use(const SceneView& sv, const RayCtx& r, int64_t p,
                                        bool want, int mc, const SegBase& base, float dtf) {
  CandUse u;
  u.jlo = 0;
  u.jhi = -1;
  u.use = want && mc > 0 && cand_setup(sv, r, p, base, u.cs) &&
          sample_range(u.cs, dtf, mc, u.jlo, u.jhi);
  return u;
}

// Pass-1 accumulation of one candidate into the 16 per-sample sums
// (renderer.py:218-228), given its setup.
__device__ inline void accumulate_used(const SceneView& sv, const RayCtx& r, int64_t p,
                                       const CandUse& u, float dtf, const float* Y,
                                       float (&sig)[16], float (&W)[16][3]) {
  const CandSetup& cs = u.cs;
  const bool use = u.use;
  const int jlo = u.jlo, jhi = u.jhi;
  PH_CNT(9, 1)
  PH_LANES(11, use)
  if (!__any_sync(FULL, use)) return;
  PH_CNT(14, 1)
  float c[3] = {0.f, 0.f, 0.f};
  if (use) eval_radiance_f(sv.app + GSX_APP_F4 * p, Y, r.df, c);
  const float nkl2 = -cs.kl2;
  // 4-sample groups outside every lane's range are skipped warp-uniformly
#pragma unroll
  for (int g = 0; g < 4; ++g) {
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
}

__device__ inline void accumulate_candidate(const SceneView& sv, const RayCtx& r, int64_t p,
                                            bool want, int mc, const SegBase& base, float dtf,
                                            const float* Y, float (&sig)[16],
                                            float (&W)[16][3]) {
  const CandUse u = candidate_use(sv, r, p, want, mc, base, dtf);
  accumulate_used(sv, r, p, u, dtf, Y, sig, W);
}

// Pass 1 over a staged list in list order.  (Interleaving two candidates'
// setups for ILP measured slower: the extra live state spills at 128 regs.)
template <class Pre>
__device__ inline void accumulate_list(const SceneView& sv, const RayCtx& r, const WarpSmem& sm,
                                       int count, bool want, int mc, const SegBase& base,
                                       float dtf, const float* Y, float (&sig)[16],
                                       float (&W)[16][3], Pre&& pre) {
  // (L1 prefetch of the listed geometry / appearance blocks measured slower:
  // 40.9 vs 40.0 ms on C3 -- the entry loop is not load-latency bound)
  for (int i = 0; i < count; ++i) {
    const int64_t p = sm.list[i];
    pre(p);
    accumulate_candidate(sv, r, p, want, mc, base, dtf, Y, sig, W);
  }
}

// Exact AABB-emptiness of the lane's segment (reference semantics) after the
// true-intersection pass; STATS additionally counts every exact overlap.
template <bool STATS>
static __device__ GSX_COLD void emptiness_tail(const SceneView& sv, const BvhView& bv, const RayCtx& r,
                                      bool want, const Seg& seg, bool& nonempty,
                                      Counters<STATS>& cnt) {
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
        traverse_segment<true>(bv, r, (float)a, (float)b, fn, v2);
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
    traverse_segment<true>(bv, r, (float)seg.t0, (float)seg.t1, probe, v2);
  }
  PH_END(4, ph_ph)
}

// Alg. 1 for one lane's ray in warp lockstep (renderer.py:288-358).
// segfn(seg, want) processes one segment for all lanes and returns the lane's
// exact AABB-emptiness verdict (true = non-empty).
// `sync` = depth-synchronous window in segment lengths (0 = every active lane
// takes part every iteration).
template <bool STATS, class SegFn>
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
      const bool got = warp_closest_hit(sv, bv, r, need_ch, ch_from, t_f, h, sm, visits);
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
      float dmin = t0f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dmin = fminf(dmin, __shfl_xor_sync(FULL, dmin, o));
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
