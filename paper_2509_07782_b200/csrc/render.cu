// render.cu -- K6: forward volume ray marching (render_image renderer.py:396-437,
// march_ray :263-285, _march_uniform :288-323, _march_adaptive :326-358,
// composite :207-240, closest_hit spatial.py:309-354, eval_radiance
// appearance.py:91-98).
//
// One thread per ray; a CTA renders one 16x16 tile with pixels in Z-order
// (each warp = an 8x4 pixel block, so its 32 rays are spatially coherent).
// The warp marches in lockstep, one segment per lane per iteration ("slab by
// slab", render_warp.cuh).  Camera rays share one origin, so the taking-part
// lanes' segments lie in a cone cut by a distance shell: a warp-cooperative
// traversal of the 4-wide BVH tests that cone against one child box per lane
// (8 nodes per step) and stages the leaves in a shared-memory list
// (warp_traverse_cone; explicit-ray batches use the per-lane packet test,
// warp_traverse).  Every lane then evaluates the list against its own ray:
// an fp32 per-(ray, primitive) setup relative to the segment's base point
// reduces the density along the ray to q(t) = A (t - t_c)^2 + q_min, and the
// 16 samples of the segment accumulate in registers with one FMA pair + one
// EX2 per (sample, primitive).  AABB-emptiness (which drives empty-space
// skipping) is decided with the reference's exact fp64 slab test on the
// candidates, so ESS jumps and adaptive grid restarts happen exactly where
// the reference's do.
//
// Tuning (C3 / C2 ms on one B200, A/B on the same box, profiles/
// time_variants.py):
//  * cold fp64 paths inlined: C3 32.9 vs 38.2 all out of line -- except the
//    closest-hit leaf test (below); the exact AABB test decided in fp32 when certain,
//    its fp64 fallback out of line (render_common.cuh): 30.9 vs 31.5;
//  * MUFU exponentials in the compositing (GSX_FAST_COMPOSITE): 30.25 vs
//    30.9, C2 14.7 vs 15.6;
//  * per-lane SH basis in shared memory (GSX_Y_SMEM): 31.15 vs 31.28;
//  * packet cone for every camera render, logged (training) one included:
//    C3 31.2 vs 34.7 per-lane packet; C2 17.5 vs 17.2 at equal depth-sync;
//  * rejected: 8-sample chunks (C3 38.0), persistent warps (+0.2), gating
//    the exact test by the lane's own use (C3 -1.5%, C2 +4%), the silhouette
//    screen, cp.async staging and an ellipsoid-vs-cone leaf filter
//    (profiles/experiments/forward_list_variants.cuh): fewer instructions,
//    more instruction-cache misses.
#ifndef GSX_COLD
#define GSX_COLD inline
#endif
#ifndef GSX_EXACT_ATTR
#define GSX_EXACT_ATTR __noinline__
#endif
// closest-hit leaf test (fp64 division / square root bodies) out of line:
// C2 14.0 vs 14.5 ms, C3 29.6 vs 29.8 (with rcbrt in segment_step)
#ifndef GSX_CHLEAF_ATTR
#define GSX_CHLEAF_ATTR __noinline__
#endif
#ifndef GSX_Y_SMEM
#define GSX_Y_SMEM 2  // SH basis: 1 shared memory, 2 recomputed per use (YDir), 0 registers
#endif
// camera-kernel traversal: 0 per-lane packet (warp_traverse), 1 packet cone
// (warp_traverse_cone), 2 cone for the plain forward only
#ifndef GSX_FWD_CONE
#define GSX_FWD_CONE 1
#endif
// samples per chunk of the plain forward (n_s > CH: several chunks, each
// traversing its share of the segment)
#ifndef GSX_FWD_CH
#define GSX_FWD_CH 16
#endif
// ESS closest hit by cone windows (warp_closest_hit_cone)
#ifndef GSX_CONE_CH
#define GSX_CONE_CH 1
#endif
#define FWD_CONE(save) (GSX_FWD_CONE == 1 || (GSX_FWD_CONE == 2 && !(save)))
#include <type_traits>

#include "gsx_common.cuh"
#include "march_log.cuh"
#include "render_warp.cuh"

namespace {

using namespace gsx;

// One warp iteration over a segment (all 32 lanes; lanes with want == false
// only help traversing).  Accumulates and composites the lane's samples and
// returns its exact AABB-emptiness verdict.  SAVE (training) also appends the
// chunk's candidate stream and per-sample sums to the warp's march log.
template <bool STATS, bool SAVE, bool CONE, class YT>
__device__ bool forward_segment(const SceneView& sv, const BvhView& bv, const RayCtx& r,
                                bool want, const Seg& seg, int ns, YT Y,
                                RayAccum& acc, Counters<STATS>& cnt, WarpSmem& sm,
                                LogWriter& lw) {
  bool nonempty = false;
  const float dtf = (float)seg.dt;
  // samples per chunk: the per-sample sums sig[CH], W[CH][3] are the largest
  // live state of the list loop (CH = 16: 64 registers at a 64-register cap)
  constexpr int CH = SAVE ? 16 : GSX_FWD_CH;
  const int nchunks = (ns + CH - 1) / CH;
  uint32_t visits = 0;
  for (int ch = 0; ch < nchunks; ++ch) {
    int mc = want ? seg.m - ch * CH : 0;
    mc = mc < 0 ? 0 : (mc > CH ? CH : mc);
    // a lane takes part in the chunks that hold its samples (chunk 0 always:
    // emptiness); the chunks' traversal intervals tile [t0, t1]
    const bool wch = want && (ch == 0 || mc > 0);
    const double tb = seg.tbase + (double)(ch * CH) * seg.dt;
    const SegBase base = seg_base(r, tb);
    float sig[CH];
    float W[CH][3];
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      sig[j] = 0.f;
      W[j][0] = W[j][1] = W[j][2] = 0.f;
    }
    if (!__any_sync(FULL, wch)) continue;
    // One traversal call site: list chunks of LCAP entries are traversed,
    // then accumulated, until the stream is exhausted.
    SegLimits lim;
    if (nchunks == 1) {
      lim = seg_limits(r, seg);
    } else {
      const double a = ch == 0 ? seg.t0 : seg.tgrid + (double)(seg.j0 + ch * CH) * seg.dt;
      const double b = (ch + 1) * CH >= seg.m
                           ? seg.t1
                           : seg.tgrid + (double)(seg.j0 + (ch + 1) * CH) * seg.dt;
      lim = interval_limits(r, a, b);
    }
    WarpTrav st{0, 0, false, false};
    ConeTrav cst;
    if (CONE) {
      make_cone(r, wch, lim.lo_t, lim.hi_t, sm);
      cone_begin(sm, cst);
    }
    int count = 0;
    const bool save = SAVE && __any_sync(FULL, want && mc > 0);
    auto exact = [&](int64_t p, bool gate) {
      if (!STATS && gate && !nonempty && exact_aabb_overlap(sv, r, p, seg.t0, seg.t1))
        nonempty = true;
    };
    LogRecPtrs lo{nullptr, nullptr, nullptr, nullptr, 0, 0, false};
    for (;;) {
      PH_BEGIN(ph_t)
      if (CONE)
        warp_traverse_cone(bv, cst, sm, count, visits);
      else
        warp_traverse(bv, r, wch, lim.lo_t, lim.hi_t, lim.gap, st, sm, count, visits);
      PH_END(1, ph_t)
      const bool last = CONE ? cst.done : st.done;
      if constexpr (SAVE) {
        if (save) lo = log_open(lw, count, last, tb, seg.dt, mc);
      }
      PH_BEGIN(ph_p)
      int kept = 0;  // logged forward: the entries some lane used, in list order
      accumulate_list(sv, r, sm, count, wch, mc, base, dtf, Y, sig, W, exact,
                      [&](int, int64_t p, unsigned um) {
                        if (SAVE && um) {
                          if ((threadIdx.x & 31) == 0) log_keep(lw, lo, kept, (int32_t)p, um);
                          ++kept;
                        }
                      });
      if constexpr (SAVE) log_close(lo, kept);
      PH_END(2, ph_p)
      if (last) break;
      __syncwarp();
      count = 0;
    }
    if constexpr (SAVE)
      log_samples(lo, mc, [&](int j) { return make_float4(sig[j], W[j][0], W[j][1], W[j][2]); });
    if (STATS) {
#pragma unroll
      for (int j = 0; j < CH; ++j) cnt.composited += (j < mc && sig[j] > 0.f) ? 1u : 0u;
    }
    PH_BEGIN(ph_c)
    // front-to-back compositing (renderer.py:230-239); zero-density samples
    // leave the state unchanged, so compositing an empty segment is a no-op
#pragma unroll
    for (int j = 0; j < CH; ++j)
      acc.add_sample(j < mc ? sig[j] : 0.f, W[j], (float)(tb + (double)j * seg.dt), dtf);
    PH_END(3, ph_c)
  }
  if (STATS) cnt.visits += visits;
  emptiness_tail<STATS>(sv, bv, r, want, seg, nonempty, cnt, sm.ovf);
  return nonempty;
}

template <bool STATS>
__device__ void flush_stats(gsx_stats* st, const Counters<STATS>& c, bool is_ray,
                            unsigned long long* per_ray = nullptr) {
  if (!STATS) return;
  uint32_t v[10] = {is_ray ? 1u : 0u, c.samples, c.segments, c.skipped, c.ch_calls, c.visits,
                    c.aabb, c.ell, c.pairs, c.composited};
  if (per_ray) {  // one row of 10 counters per ray, no reduction
    if (is_ray)
      for (int k = 0; k < 10; ++k) per_ray[k] = v[k];
    return;
  }
  if (!st) return;
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    uint32_t x = v[k];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd((unsigned long long*)&st->rays + k, (unsigned long long)x);
  }
}

template <bool STATS, bool SAVE, bool CONE>
__device__ void march_forward(const SceneView& sv, const BvhView& bv, const RayCtx& r, bool hit,
                              const gsx_render_cfg& cfg, RayAccum& acc, Counters<STATS>& cnt,
                              WarpSmem& sm, LogWriter& lw) {
#if GSX_Y_SMEM == 1
  float Y[9];
  sh_basis_f(r.df, Y);
  {
    const unsigned lane = threadIdx.x & 31;
#pragma unroll
    for (int b = 0; b < 9; ++b) sm.ylane[b][lane] = Y[b];
    __syncwarp();
  }
  const YSmem Yv{&sm.ylane[0][threadIdx.x & 31]};
#elif GSX_Y_SMEM == 2
  const YDir Yv{r.df};
#else
  float Y[9];
  sh_basis_f(r.df, Y);
  const float* Yv = Y;
#endif
  const int ns = (int)cfg.n_s;
  march_warp<STATS, CONE && GSX_CONE_CH>(sv, bv, r, hit, cfg, acc, cnt, cfg.mode == 0 ? GSX_SYNC_FWD_U : GSX_SYNC_FWD, sm, [&](const Seg& seg, bool want) {
    return forward_segment<STATS, SAVE, CONE>(sv, bv, r, want, seg, ns, Yv, acc, cnt, sm, lw);
  });
}

// CTA = FWD_THREADS rays = 256 / FWD_THREADS CTAs per 16x16 tile.  The march
// is latency-bound and tolerates spills: occupancy wins.  Measured on C3
// (ms/frame, 128-thread CTAs x min blocks/SM): x4 (128 regs) 42.0 (r2 code),
// x5 (96) 42.0, x6 (80) 39.7, x7 (72) 37.3, x8 (64 regs, 32 warps/SM) 37.2,
// x9 (56) 37.3, x10 (48) 37.7, x12 (40) 40.5.
#ifndef GSX_FWD_THREADS
#define GSX_FWD_THREADS 128
#endif
#ifndef GSX_FWD_MINB
#define GSX_FWD_MINB 8
#endif
constexpr int FWD_THREADS = GSX_FWD_THREADS;


// One warp block: the 32 rays of an 8x4 Z-order pixel block.  blk numbers the
// blocks of the launch: tile at sequence position tile_begin + (blk / 8) *
// tile_stride (gsx_tile_at), warp blk % 8
// of the tile (the march-log warp id).
template <bool STATS, bool SAVE, bool CONE>
__device__ void render_warp_block(const SceneView& sv, const BvhView& bv, const gsx_camera& cam,
                                  const gsx_render_cfg& cfg, int64_t tile_begin,
                                  int64_t tile_stride, long long blk, float* rgb, float* depth,
                                  float* trans, gsx_stats* stats, void* log, long long log_nw,
                                  WarpSmem& sw) {
  const int64_t W = cam.width, H = cam.height;
  const int64_t tiles_x = (W + 15) / 16;
  const int64_t tile = gsx_tile_at(tile_begin + (int64_t)(blk >> 3) * tile_stride, tiles_x,
                                   (H + 15) / 16, tile_stride);
  const unsigned lane = threadIdx.x & 31;
  int mx, my;
  morton_decode8((unsigned)(blk & 7) * 32 + lane, mx, my);
  const int64_t px = (tile % tiles_x) * 16 + mx, py = (tile / tiles_x) * 16 + my;
  const bool valid = px < W && py < H;
  Counters<STATS> cnt;
  RayCtx r;
  const bool hit = valid && camera_ray(cam, (double)px, (double)py, sv.bounds, r);
  RayAccum acc;
  acc.init();
  LogWriter lw = log_writer(SAVE ? log : nullptr, blk);
  ovf_begin(sw);
  march_forward<STATS, SAVE, CONE>(sv, bv, r, hit, cfg, acc, cnt, sw, lw);
  ovf_report(sw, bv, py * W + px);
  if (SAVE) log_finish(lw, log_nw);
  if (valid) {
    int64_t pix = py * W + px;
    float T = hit ? acc.transmittance() : 1.f;
    for (int k = 0; k < 3; ++k) rgb[3 * pix + k] = acc.C[k] + T * (float)cfg.background[k];
    if (depth) depth[pix] = acc.D;
    if (trans) trans[pix] = T;
  }
  flush_stats<STATS>(stats, cnt, valid);
}

// (Persistent warps pulling pixel blocks from a launch-wide counter measured
// slower: C3 34.1 vs 33.9 ms -- the block loop costs registers / spills.)
// One-warp CTAs (32 per SM at the same 64-register cap) for the plain forward
// of a whole image: a finished warp frees its slot at once instead of waiting
// for the slowest warp of its CTA.  C3 29.1 vs 29.6 ms (128-thread CTAs); the
// logged forward (C2 17.55 vs 17.0) and short per-rank launches (8-rank C3
// share 6.48 vs 5.87 ms) keep FWD_THREADS (profiles/r05_cta_order_variants.txt).
#ifndef GSX_CONE_MIN_FOCAL
#define GSX_CONE_MIN_FOCAL 1024.0
#endif
#ifndef GSX_FWD_THREADS_WHOLE
#define GSX_FWD_THREADS_WHOLE 32
#endif
template <bool STATS, bool SAVE, int NT, bool CONE>
__global__ void __launch_bounds__(NT, GSX_FWD_MINB * FWD_THREADS / NT) k_render_camera(
    SceneView sv, BvhView bv, gsx_camera cam, gsx_render_cfg cfg, int64_t tile_begin,
    int64_t tile_stride, float* rgb, float* depth, float* trans, gsx_stats* stats, void* log,
    long long log_nw) {
  __shared__ WarpSmem smem[NT / 32];
  const long long blk = (long long)blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
  render_warp_block<STATS, SAVE, CONE>(sv, bv, cam, cfg, tile_begin, tile_stride, blk, rgb, depth,
                                 trans, stats, log, log_nw, smem[threadIdx.x >> 5]);
}

// ---------------------------------------------------------------------------
// Screened plain forward (the benchmarked frame): the camera kernel above
// with the per-camera silhouette screen (Screen, render_warp.cuh) in front of
// every list and the per-sample sums in shared memory (WarpSmemA) or
// registers.  Same
// march, same per-lane arithmetic in the same order: its pixels equal the
// unscreened kernel's bit for bit.
// ---------------------------------------------------------------------------
#ifndef GSX_LOG_BULK  // training forward, shared-memory sums: TMA bulk copy of the sums
#define GSX_LOG_BULK 1
#endif
template <bool SAVE, bool SMEM, class YT, class WS>
__device__ bool forward_segment_screened(const SceneView& sv, const BvhView& bv,
                                         const RayCtx& r, bool want, const Seg& seg, int ns,
                                         YT Y, RayAccum& acc, WS& sm, const Screen& sc,
                                         LogWriter& lw) {
  constexpr int CH = GSX_SCR_CH;
  bool nonempty = false;
  const float dtf = (float)seg.dt;
  const int nchunks = (ns + CH - 1) / CH;
  using Sums = std::conditional_t<SMEM, SmemSums, RegSums<CH>>;
  Sums sums;
  if constexpr (SMEM) sums.col = &sm.acc[0][threadIdx.x & 31];
  uint32_t visits = 0;
  for (int ch = 0; ch < nchunks; ++ch) {
    int mc = want ? seg.m - ch * CH : 0;
    mc = mc < 0 ? 0 : (mc > CH ? CH : mc);
    const bool wch = want && (ch == 0 || mc > 0);
    if (!__any_sync(FULL, wch)) continue;
    const double tb = seg.tbase + (double)(ch * CH) * seg.dt;
    const SegBase base = seg_base(r, tb);
    // the training forward's shared-memory sums are zeroed after the first
    // traversal: a bulk copy of the previous chunk's may still be reading them
    constexpr bool BULK = SAVE && SMEM && GSX_LOG_BULK;
    if constexpr (!BULK) sums.zero(CH);
    SegLimits lim;
    if (nchunks == 1) {
      lim = seg_limits(r, seg);
    } else {
      const double a = ch == 0 ? seg.t0 : seg.tgrid + (double)(seg.j0 + ch * CH) * seg.dt;
      const double b = (ch + 1) * CH >= seg.m
                           ? seg.t1
                           : seg.tgrid + (double)(seg.j0 + (ch + 1) * CH) * seg.dt;
      lim = interval_limits(r, a, b);
    }
    make_cone(r, wch, lim.lo_t, lim.hi_t, sm);
    ConeTrav cst;
    cone_begin(sm, cst);
    const unsigned lanes = __ballot_sync(FULL, wch && mc > 0);
    const bool save = SAVE && __any_sync(FULL, want && mc > 0);
    int count = 0;
    LogRecPtrs lo{nullptr, nullptr, nullptr, nullptr, 0, 0, false};
    bool zeroed = false;
    for (;;) {
      PH_BEGIN(ph_t)
      warp_traverse_cone(bv, cst, sm, count, visits);
      PH_END(1, ph_t)
      if constexpr (BULK) {
        if (!zeroed) {
          if (lw.bulk) log_bulk_wait();
          lw.bulk = false;
          sums.zero(CH);
          zeroed = true;
        }
      }
      if constexpr (SAVE) {
        if (save)
          lo = SMEM ? log_open_ool(lw, count, cst.done, tb, seg.dt, mc, BULK)
                    : log_open(lw, count, cst.done, tb, seg.dt, mc);
      }
      bool inside = false;
      int kept = 0;  // logged forward: the entries some lane used, in list order
      PH_BEGIN(ph_p)
      screen_accumulate<CH>(sc, sv, r, sm, count, lanes, wch, mc, base, dtf, Y, sums, inside,
                            [&](int32_t p, unsigned um) {
                              if constexpr (SAVE) {
                                const unsigned kb = __ballot_sync(FULL, um != 0u);
                                if (um) log_keep(lw, lo, kept + __popc(kb & lanemask_lt()), p, um);
                                kept += __popc(kb);
                              }
                            });
      if constexpr (SAVE) log_close(lo, kept);
      PH_END(2, ph_p)
      nonempty = nonempty || inside;
      // AABB emptiness without a clearly-inside sample: the exact test over
      // this chunk of the list (a superset of the boxes the segment meets)
      PH_BEGIN(ph_e)
      if (want && !nonempty)
        for (int i = 0; i < count; ++i)
          if (exact_aabb_overlap(sv, r, (int64_t)sm.list[i], seg.t0, seg.t1)) {
            nonempty = true;
            break;
          }
      PH_END(4, ph_e)
      __syncwarp();
      if (cst.done) break;
      count = 0;
    }
    if constexpr (BULK) {
      if (GSX_LOG_BULK_MIN == 0 || lo.by_lane) {
        if (log_samples_bulk(lo, &sm.acc[0][0])) lw.bulk = true;
      } else {
        log_samples(lo, mc, [&](int j) { return sums.get(j); });
      }
    } else if constexpr (SAVE) {
      log_samples(lo, mc, [&](int j) { return sums.get(j); });
    }
    // front-to-back compositing (renderer.py:230-239)
    PH_BEGIN(ph_c)
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const float4 a = sums.get(j);
      const float w3[3] = {a.y, a.z, a.w};
      acc.add_sample(j < mc ? a.x : 0.f, w3, (float)(tb + (double)j * seg.dt), dtf);
    }
    PH_END(3, ph_c)
  }
  Counters<false> cnt;
  PH_BEGIN(ph_x)
  emptiness_tail<false>(sv, bv, r, want, seg, nonempty, cnt, sm.ovf);
  PH_END(7, ph_x)
  return nonempty;
}

#ifndef GSX_SCR_THREADS
#define GSX_SCR_THREADS 32
#endif
#ifndef GSX_SCR_YSMEM
#define GSX_SCR_YSMEM 1
#endif
#ifndef GSX_SCR_THREADS_LOGGED  // CTA of the screened training forward
#define GSX_SCR_THREADS_LOGGED 64
#endif
#ifndef GSX_SCR_MINB  // CTAs of 32 threads per SM (registers: 65536 / (32 MINB))
#define GSX_SCR_MINB 16
#endif
#ifndef GSX_SCRR_MINB  // the same for the register-sum variant
#define GSX_SCRR_MINB 32
#endif

// SMEM: per-sample sums in shared memory (16 warps / SM at 128 registers) or
// in registers (32 warps / SM at 64 registers, sums spilled to local memory)
template <int NT, bool SAVE, bool SMEM>
__global__ void __launch_bounds__(NT, (SMEM ? GSX_SCR_MINB : GSX_SCRR_MINB) * 32 / NT)
    k_render_screened(SceneView sv, BvhView bv, gsx_camera cam, gsx_render_cfg cfg,
                      int64_t tile_begin, int64_t tile_stride, float* rgb, float* depth,
                      float* trans, const float4* view, void* log, long long log_nw) {
  constexpr int CH = GSX_SCR_CH;
  using WS = std::conditional_t<SMEM, WarpSmemA<CH>, WarpSmemT>;
  __shared__ WS smem[NT / 32];
  WS& sw = smem[threadIdx.x >> 5];
  const long long blk = (long long)blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
  const int64_t W = cam.width, H = cam.height;
  const int64_t tiles_x = (W + 15) / 16;
  const int64_t tile = gsx_tile_at(tile_begin + (int64_t)(blk >> 3) * tile_stride, tiles_x,
                                   (H + 15) / 16, tile_stride);
  const unsigned lane = threadIdx.x & 31;
  int mx, my, bx, by;
  morton_decode8((unsigned)(blk & 7) * 32 + lane, mx, my);
  morton_decode8((unsigned)(blk & 7) * 32, bx, by);
  const int64_t px = (tile % tiles_x) * 16 + mx, py = (tile / tiles_x) * 16 + my;
  const bool valid = px < W && py < H;
  RayCtx r;
  const bool hit = valid && camera_ray(cam, (double)px, (double)py, sv.bounds, r);
  RayAccum acc;
  acc.init();
  const Screen sc{view, (float)((tile % tiles_x) * 16 + bx), (float)((tile / tiles_x) * 16 + by)};
#if GSX_SCR_YSMEM == 1 && GSX_Y_SMEM == 1
  float Y[9];
  sh_basis_f(r.df, Y);
#pragma unroll
  for (int b = 0; b < 9; ++b) sw.ylane[b][lane] = Y[b];
  __syncwarp();
  const YSmem Yv{&sw.ylane[0][lane]};
#elif GSX_SCR_YSMEM == 2 || GSX_Y_SMEM != 1
  const YDir Yv{r.df};  // recomputed per radiance evaluation
#else
  float Y[9];
  sh_basis_f(r.df, Y);
  const float* Yv = Y;  // (128 registers: the basis stays in registers)
#endif
  const int ns = (int)cfg.n_s;
  Counters<false> cnt;
  LogWriter lw = log_writer(SAVE ? log : nullptr, blk);
  ovf_begin(sw);
#if GSX_APP_TMA
  app_barriers_init(sw);
#endif
  march_warp<false, true>(sv, bv, r, hit, cfg, acc, cnt,
                          cfg.mode == 0 ? GSX_SYNC_FWD_U : GSX_SYNC_FWD, sw,
                          [&](const Seg& seg, bool want) {
                            return forward_segment_screened<SAVE, SMEM>(sv, bv, r, want, seg,
                                                                        ns, Yv, acc, sw, sc, lw);
                          });
  if (SAVE && lw.bulk) log_bulk_drain();
  if (SAVE) log_finish(lw, log_nw);
  ovf_report(sw, bv, py * W + px);
  if (valid) {
    const int64_t pix = py * W + px;
    const float T = hit ? acc.transmittance() : 1.f;
    for (int k = 0; k < 3; ++k) rgb[3 * pix + k] = acc.C[k] + T * (float)cfg.background[k];
    if (depth) depth[pix] = acc.D;
    if (trans) trans[pix] = T;
  }
}

// Launch k_render_camera over ntl tiles (8 warp blocks each).
template <bool STATS, bool SAVE, int NT, bool CONE = FWD_CONE(SAVE)>
int launch_camera_nt(const SceneView& sv, const BvhView& bv, const gsx_camera& cam,
                     const gsx_render_cfg& cfg, int64_t tile_begin, int64_t tile_stride,
                     int64_t ntl, float* rgb, float* depth, float* trans, gsx_stats* stats,
                     void* log, long long log_nw, cudaStream_t s) {
  const long long ctas = 8 * (long long)ntl / (NT / 32);
  k_render_camera<STATS, SAVE, NT, CONE><<<(unsigned)ctas, NT, 0, s>>>(
      sv, bv, cam, cfg, tile_begin, tile_stride, rgb, depth, trans, stats, log, log_nw);
  return gsx_check_launch();
}
template <bool STATS, bool SAVE>
int launch_camera(const SceneView& sv, const BvhView& bv, const gsx_camera& cam,
                  const gsx_render_cfg& cfg, int64_t tile_begin, int64_t tile_stride, int64_t ntl,
                  float* rgb, float* depth, float* trans, gsx_stats* stats, void* log,
                  long long log_nw, cudaStream_t s, const float4* view = nullptr) {
  if constexpr (!SAVE && !STATS && FWD_CONE(false)) {
    // wide pixels (focal < GSX_CONE_MIN_FOCAL px): a warp's 8x4-pixel cone
    // lists many entries its rays miss, and the per-lane packet traversal
    // wins (480x270, f = 576, 1M / 3M / 5M: 10.4 / 17.4 / 22.7 vs 11.9 /
    // 19.7 / 25.6 ms; C2 f = 1111 equal; C3 f = 2304: cone 31.2 vs 34.7).
    // cfg.traversal forces either (1 cone, 2 per-lane packet).
    const bool lane_packet =
        cfg.traversal == 2 || (cfg.traversal == 0 && cam.focal < GSX_CONE_MIN_FOCAL);
    if (lane_packet) {
      if (tile_stride == 1)
        return launch_camera_nt<STATS, SAVE, GSX_FWD_THREADS_WHOLE, false>(
            sv, bv, cam, cfg, tile_begin, tile_stride, ntl, rgb, depth, trans, stats, log,
            log_nw, s);
      return launch_camera_nt<STATS, SAVE, FWD_THREADS, false>(
          sv, bv, cam, cfg, tile_begin, tile_stride, ntl, rgb, depth, trans, stats, log, log_nw,
          s);
    }
  }
  if constexpr (!SAVE && !STATS) {
    if (view && FWD_CONE(false)) {
      const long long ctas = 8 * (long long)ntl / (GSX_SCR_THREADS / 32);
      if (cfg.sums == 1)
        k_render_screened<GSX_SCR_THREADS, false, false>
            <<<(unsigned)ctas, GSX_SCR_THREADS, 0, s>>>(sv, bv, cam, cfg, tile_begin, tile_stride,
                                                        rgb, depth, trans, view, nullptr, 0);
      else
        k_render_screened<GSX_SCR_THREADS, false, true>
            <<<(unsigned)ctas, GSX_SCR_THREADS, 0, s>>>(sv, bv, cam, cfg, tile_begin, tile_stride,
                                                        rgb, depth, trans, view, nullptr, 0);
      return gsx_check_launch();
    }
    if (tile_stride == 1)
      return launch_camera_nt<STATS, SAVE, GSX_FWD_THREADS_WHOLE>(
          sv, bv, cam, cfg, tile_begin, tile_stride, ntl, rgb, depth, trans, stats, log, log_nw,
          s);
  }
  if constexpr (SAVE && !STATS) {
    if (view && FWD_CONE(true)) {  // screened logged (training) forward
      constexpr int NT = GSX_SCR_THREADS_LOGGED;
      const long long ctas = 8 * (long long)ntl / (NT / 32);
      if (cfg.sums == 1)
        k_render_screened<NT, true, false><<<(unsigned)ctas, NT, 0, s>>>(
            sv, bv, cam, cfg, tile_begin, tile_stride, rgb, depth, trans, view, log, log_nw);
      else
        k_render_screened<NT, true, true><<<(unsigned)ctas, NT, 0, s>>>(
            sv, bv, cam, cfg, tile_begin, tile_stride, rgb, depth, trans, view, log, log_nw);
      return gsx_check_launch();
    }
  }
  return launch_camera_nt<STATS, SAVE, FWD_THREADS>(sv, bv, cam, cfg, tile_begin, tile_stride,
                                                    ntl, rgb, depth, trans, stats, log, log_nw,
                                                    s);
}

// K6a: image-space silhouettes of every primitive for one camera (Screen,
// render_warp.cuh), fp64.  With M the iso_inv of p inflated by 1e-3, the
// line o + t d meets the ellipsoid iff (g.d)^2 >= kappa d^T S d, g = M^T a,
// a = M (o - mu), kappa = |a|^2 - 1, S = M^T M.  In camera coordinates
// d ~ (u, v, 1) this is F(u, v) = p^T K p >= 0 with K = R^T (g g^T - kappa S) R;
// when its 2x2 block is negative definite the set is the ellipse
// (w - c)^T (-K2 / F(c)) (w - c) <= 1 about c = -K2^-1 k, mapped to pixels
// (u = (X - W/2) / f) and widened by 2e-3 px (fp32 rounding of the centre).
// Anything else (camera inside, ellipsoid across the camera plane, a
// degenerate form) gets A00 = 0: never screened out.
__global__ void k_view_conics(SceneView sv, int64_t n, gsx_camera cam, float4* view) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const double inflate = 1.0 / (1.0 + 1e-3);
  double M[9];
  for (int k = 0; k < 9; ++k) M[k] = sv.inv64[9 * p + k] * inflate;
  const float4 g0 = sv.geo[4 * p];
  const double v[3] = {cam.center[0] - (double)g0.x, cam.center[1] - (double)g0.y,
                       cam.center[2] - (double)g0.z};
  double a[3], g[3] = {0, 0, 0}, S[9];
  for (int i = 0; i < 3; ++i) a[i] = M[3 * i] * v[0] + M[3 * i + 1] * v[1] + M[3 * i + 2] * v[2];
  const double kappa = a[0] * a[0] + a[1] * a[1] + a[2] * a[2] - 1.0;
  float4 out0 = make_float4(0.f, 0.f, 0.f, 0.f), out1 = make_float4(0.f, 0.f, 0.f, 0.f);
  if (kappa > 1e-9) {
    for (int b = 0; b < 3; ++b)
      for (int i = 0; i < 3; ++i) g[b] += M[3 * i + b] * a[i];
    for (int b = 0; b < 3; ++b)
      for (int c = 0; c < 3; ++c)
        S[3 * b + c] = M[b] * M[c] + M[3 + b] * M[3 + c] + M[6 + b] * M[6 + c];
    // world -> camera: gc = R^T g, Sc = R^T S R (R row-major, d_world = R d_cam)
    const double* R = cam.R;
    double gc[3], SR[9], K[9];
    for (int k = 0; k < 3; ++k) gc[k] = R[k] * g[0] + R[3 + k] * g[1] + R[6 + k] * g[2];
    for (int b = 0; b < 3; ++b)
      for (int k = 0; k < 3; ++k)
        SR[3 * b + k] = S[3 * b] * R[k] + S[3 * b + 1] * R[3 + k] + S[3 * b + 2] * R[6 + k];
    for (int j = 0; j < 3; ++j)
      for (int k = 0; k < 3; ++k)
        K[3 * j + k] = gc[j] * gc[k] -
                       kappa * (R[j] * SR[k] + R[3 + j] * SR[3 + k] + R[6 + j] * SR[6 + k]);
    const double k00 = K[0], k01 = 0.5 * (K[1] + K[3]), k11 = K[4];
    const double k02 = 0.5 * (K[2] + K[6]), k12 = 0.5 * (K[5] + K[7]), k22 = K[8];
    const double det = k00 * k11 - k01 * k01;
    if (k00 < 0.0 && det > 0.0) {
      const double cu = -(k11 * k02 - k01 * k12) / det, cv = -(k00 * k12 - k01 * k02) / det;
      const double Fc = k22 + k02 * cu + k12 * cv;
      if (Fc > 0.0) {
        const double f = cam.focal, s2 = 1.0 / (Fc * f * f);
        double A00 = -k00 * s2, A01 = -k01 * s2, A11 = -k11 * s2;
        // widen by 2e-3 px: scale the semi-axes by (1 + 2e-3 / r_min),
        // r_min = 1 / sqrt(lambda_max(A))
        const double tr = 0.5 * (A00 + A11),
                     lmax = tr + sqrt(fmax(tr * tr - (A00 * A11 - A01 * A01), 0.0));
        const double grow = 1.0 + 2e-3 * sqrt(lmax), w = 1.0 / (grow * grow) * (1.0 - 1e-6);
        A00 *= w;
        A01 *= w;
        A11 *= w;
        const double Xc = 0.5 * (double)cam.width + f * cu, Yc = 0.5 * (double)cam.height + f * cv;
        if (isfinite(Xc) && isfinite(Yc) && fabs(Xc) < 1e7 && fabs(Yc) < 1e7 && A00 > 0.0) {
          out0 = make_float4((float)Xc, (float)Yc, (float)A00, (float)(2.0 * A01));
          out1 = make_float4((float)A11, 0.f, 0.f, 0.f);
        }
      }
    }
  }
  view[2 * p] = out0;
  view[2 * p + 1] = out1;
}

template <bool STATS>
__global__ void __launch_bounds__(256, 2) k_render_rays(SceneView sv, BvhView bv,
                                                        const double* __restrict__ rays,
                                                        int64_t m, int clip, gsx_render_cfg cfg,
                                                        float* rgb, float* depth, float* trans,
                                                        gsx_stats* stats,
                                                        unsigned long long* per_ray) {
  __shared__ WarpSmem smem[8];
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool valid = i < m;
  Counters<STATS> cnt;
  RayCtx r;
  bool hit = valid && explicit_ray(rays + 8 * i, clip != 0, sv.bounds, r);
  RayAccum acc;
  acc.init();
  LogWriter lw = log_writer(nullptr, 0);
  ovf_begin(smem[threadIdx.x >> 5]);
  march_forward<STATS, false, false>(sv, bv, r, hit, cfg, acc, cnt, smem[threadIdx.x >> 5], lw);
  ovf_report(smem[threadIdx.x >> 5], bv, i);
  if (valid) {
    float T = hit ? acc.transmittance() : 1.f;
    for (int k = 0; k < 3; ++k) rgb[3 * i + k] = acc.C[k] + T * (float)cfg.background[k];
    if (depth) depth[i] = acc.D;
    if (trans) trans[i] = T;
  }
  flush_stats<STATS>(stats, cnt, valid, per_ray ? per_ray + 10 * i : nullptr);
}

__global__ void k_ffma(int64_t iters, float* sink) {
  float a = threadIdx.x * 1e-3f, b = 1.0001f, c = 0.9999f, d = blockIdx.x * 1e-3f;
  float e = a + 1.f, f = d + 2.f, g = a + 3.f, h = d + 4.f;
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a = fmaf(a, b, c); d = fmaf(d, b, c); e = fmaf(e, b, c); f = fmaf(f, b, c);
      g = fmaf(g, b, c); h = fmaf(h, b, c);
    }
  }
  sink[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = a + d + e + f + g + h;
}

// SFU calibration: 8 independent MUFU.EX2 chains per thread (the forward's
// exponentials are ex2.approx)
__global__ void k_mufu(int64_t iters, float* sink) {
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = -1e-3f * (float)(threadIdx.x + k);
  for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ex2_approx(-v[k]) - 1.5f;
  }
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc += v[k];
  sink[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

}  // namespace

int gsx_validate_cfg(const gsx_render_cfg* cfg) {
  // RenderConfig.__post_init__ (renderer.py:41-49)
  if (!cfg) return GSX_ERR_ARG;
  if (!(cfg->t_eps > 0.0 && cfg->t_eps < 1.0)) return GSX_ERR_ARG;
  if (cfg->n_s < 1) return GSX_ERR_ARG;
  if (cfg->dt_min > cfg->dt_max) return GSX_ERR_ARG;
  if (cfg->mode != 0 && cfg->mode != 1) return GSX_ERR_ARG;
  if (!(cfg->dt > 0.0)) return GSX_ERR_ARG;
  if (cfg->traversal < 0 || cfg->traversal > 2 || cfg->sums < 0 || cfg->sums > 1 ||
      cfg->pass2 < 0 || cfg->pass2 > 2)
    return GSX_ERR_ARG;
  return GSX_OK;
}

extern "C" int gsx_calibrate_fp32(int64_t iters, float* sink, double* flops, void* stream) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int blocks = sms * 8, threads = 256;
  k_ffma<<<blocks, threads, 0, (cudaStream_t)stream>>>(iters, sink);
  if (flops) *flops = 2.0 * 16 * 6 * (double)iters * blocks * threads;
  return gsx_check_launch();
}

extern "C" int gsx_calibrate_sfu(int64_t iters, float* sink, double* ops, void* stream) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int blocks = sms * 8, threads = 256;
  k_mufu<<<blocks, threads, 0, (cudaStream_t)stream>>>(iters, sink);
  if (ops) *ops = 8.0 * (double)iters * blocks * threads;
  return gsx_check_launch();
}

#ifdef GSX_PHASE_PROF
extern "C" int gsx_phase_times(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, gsx::g_phase, sizeof(unsigned long long) * 24);
  if (reset) {
    unsigned long long z[24] = {};
    cudaMemcpyToSymbol(gsx::g_phase, z, sizeof z);
  }
  return gsx_check_launch();
}
#endif

// per-render workspace: the per-camera silhouette table, float4[2n]
extern "C" size_t gsx_render_workspace_bytes(int64_t n) {
  return n > 0 ? (size_t)n * 2 * sizeof(float4) : 0;
}

extern "C" int gsx_render_forward(const void* scene_arena, const void* bvh_arena, int64_t n,
                                  const gsx_camera* cam, const gsx_render_cfg* cfg,
                                  int64_t tile_begin, int64_t tile_stride, float* rgb,
                                  float* depth, float* trans, gsx_stats* stats, void* ws,
                                  int64_t ws_bytes, gsx_dev_status* dev_status, void* stream) {
  int rc = gsx_validate_cfg(cfg);
  if (rc) return rc;
  if (!cam || cam->width < 1 || cam->height < 1 || !(cam->focal > 0)) return GSX_ERR_ARG;
  if (n <= 0) return GSX_ERR_EMPTY;
  if (tile_stride < 1 || tile_begin < 0) return GSX_ERR_ARG;
  int64_t tiles = ((cam->width + 15) / 16) * ((cam->height + 15) / 16);
  if (tile_begin >= tiles) return GSX_OK;
  const int64_t ntl = (tiles - tile_begin + tile_stride - 1) / tile_stride;
  SceneView sv = scene_view((void*)scene_arena, n);
  BvhView bv = bvh_view((void*)bvh_arena, n);
  cudaStream_t s = (cudaStream_t)stream;
  bv.status = dev_status;
  if (stats)
    return launch_camera<true, false>(sv, bv, *cam, *cfg, tile_begin, tile_stride, ntl, rgb,
                                      depth, trans, stats, nullptr, 0, s);
  float4* view = nullptr;
  if (ws) {
    if (ws_bytes < (int64_t)gsx_render_workspace_bytes(n)) return GSX_ERR_ARG;
    view = (float4*)ws;
    k_view_conics<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sv, n, *cam, view);
  }
  return launch_camera<false, false>(sv, bv, *cam, *cfg, tile_begin, tile_stride, ntl, rgb, depth,
                                     trans, nullptr, nullptr, 0, s, view);
}

__global__ void k_log_init(LogHeader* h, unsigned long long cap, unsigned nw, long long table) {
  h->head = (unsigned long long)table;
  h->cap = cap;
  h->overflow = 0;
  h->nwarps = nw;
  h->need = (unsigned long long)table;
  h->entries = 0;
  h->pairs = 0;
}

extern "C" int64_t gsx_march_log_min_bytes(const gsx_camera* cam, int64_t tile_begin,
                                           int64_t tile_stride) {
  if (!cam || cam->width < 1 || cam->height < 1 || tile_stride < 1 || tile_begin < 0) return -1;
  int64_t tiles = ((cam->width + 15) / 16) * ((cam->height + 15) / 16);
  int64_t ntl = tile_begin >= tiles ? 0 : (tiles - tile_begin + tile_stride - 1) / tile_stride;
  return log_table_bytes(8 * ntl);
}

extern "C" int gsx_render_forward_logged(const void* scene_arena, const void* bvh_arena,
                                         int64_t n, const gsx_camera* cam,
                                         const gsx_render_cfg* cfg, int64_t tile_begin,
                                         int64_t tile_stride, float* rgb, float* depth,
                                         float* trans, void* log, int64_t log_bytes, void* ws,
                                         int64_t ws_bytes, gsx_dev_status* dev_status,
                                         void* stream) {
  int rc = gsx_validate_cfg(cfg);
  if (rc) return rc;
  if (!cam || cam->width < 1 || cam->height < 1 || !(cam->focal > 0)) return GSX_ERR_ARG;
  if (n <= 0) return GSX_ERR_EMPTY;
  if (tile_stride < 1 || tile_begin < 0 || !log) return GSX_ERR_ARG;
  const int64_t table = gsx_march_log_min_bytes(cam, tile_begin, tile_stride);
  if (log_bytes < table) return GSX_ERR_ARG;
  int64_t tiles = ((cam->width + 15) / 16) * ((cam->height + 15) / 16);
  if (tile_begin >= tiles) return GSX_OK;
  const int64_t ntl = (tiles - tile_begin + tile_stride - 1) / tile_stride;
  SceneView sv = scene_view((void*)scene_arena, n);
  BvhView bv = bvh_view((void*)bvh_arena, n);
  cudaStream_t s = (cudaStream_t)stream;
  bv.status = dev_status;
  k_log_init<<<1, 1, 0, s>>>((LogHeader*)log, (unsigned long long)log_bytes,
                             (unsigned)(8 * ntl), table);
  float4* view = nullptr;
  if (ws) {
    if (ws_bytes < (int64_t)gsx_render_workspace_bytes(n)) return GSX_ERR_ARG;
    view = (float4*)ws;
    k_view_conics<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sv, n, *cam, view);
  }
  return launch_camera<false, true>(sv, bv, *cam, *cfg, tile_begin, tile_stride, ntl, rgb, depth,
                                    trans, nullptr, log, 8 * ntl, s, view);
}

extern "C" int gsx_march_log_usage(const void* log, int64_t* used_bytes, int* overflow,
                                   void* stream) {
  if (!log) return GSX_ERR_ARG;
  LogHeader h;
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_CHECK_RET(cudaMemcpyAsync(&h, log, sizeof h, cudaMemcpyDeviceToHost, s));
  CUDA_CHECK_RET(cudaStreamSynchronize(s));
  if (used_bytes) *used_bytes = (int64_t)h.need;
  if (overflow) *overflow = (int)h.overflow;
  return GSX_OK;
}

extern "C" int gsx_render_rays(const void* scene_arena, const void* bvh_arena, int64_t n,
                               const double* rays, int64_t m, int clip,
                               const gsx_render_cfg* cfg, float* rgb, float* depth, float* trans,
                               gsx_stats* stats, gsx_dev_status* dev_status, void* stream) {
  int rc = gsx_validate_cfg(cfg);
  if (rc) return rc;
  if (n <= 0) return GSX_ERR_EMPTY;
  if (m <= 0) return GSX_OK;
  SceneView sv = scene_view((void*)scene_arena, n);
  BvhView bv = bvh_view((void*)bvh_arena, n);
  cudaStream_t s = (cudaStream_t)stream;
  bv.status = dev_status;
  unsigned blocks = (unsigned)((m + 255) / 256);
  if (stats)
    k_render_rays<true><<<blocks, 256, 0, s>>>(sv, bv, rays, m, clip, *cfg, rgb, depth, trans,
                                               stats, nullptr);
  else
    k_render_rays<false><<<blocks, 256, 0, s>>>(sv, bv, rays, m, clip, *cfg, rgb, depth, trans,
                                                nullptr, nullptr);
  return gsx_check_launch();
}

extern "C" int gsx_render_rays_stats(const void* scene_arena, const void* bvh_arena, int64_t n,
                                     const double* rays, int64_t m, int clip,
                                     const gsx_render_cfg* cfg, float* rgb, float* depth,
                                     float* trans, uint64_t* per_ray,
                                     gsx_dev_status* dev_status, void* stream) {
  int rc = gsx_validate_cfg(cfg);
  if (rc) return rc;
  if (n <= 0) return GSX_ERR_EMPTY;
  if (!per_ray) return GSX_ERR_ARG;
  if (m <= 0) return GSX_OK;
  SceneView sv = scene_view((void*)scene_arena, n);
  BvhView bv = bvh_view((void*)bvh_arena, n);
  bv.status = dev_status;
  k_render_rays<true><<<(unsigned)((m + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      sv, bv, rays, m, clip, *cfg, rgb, depth, trans, nullptr,
      (unsigned long long*)per_ray);
  return gsx_check_launch();
}
