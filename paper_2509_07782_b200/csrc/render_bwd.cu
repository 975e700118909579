// render_bwd.cu -- K7: backward of the forward march (no reference counterpart;
// SURVEY.md Appendix C; float64 oracle in oracle/gsray_oracle.c backward_ray).
//
// Per warp iteration the segment is replayed with the forward's exact code
// (pass 1: per-sample sigma_j, W_j; compositing state C, D, T), then the
// per-sample adjoints are formed front to back from the saved frame outputs:
//   dL/dsigma_j = dt (T_{j+1} gC.c_j - gC.(C - C_<=j) + gD (T_{j+1} t_j - (D - D_<=j))
//                 - gTe T_end),  w_j / sigma_j,  gC.c_j
// (gTe = dL/dT + gC.background).  Pass 2 re-traverses the same candidates
// (deterministic) and, per (lane, primitive), reduces the sample loop to four
// moments of G_j = dL/ddens_j * dens_j:  m0 = sum G_j, m1 = sum G_j t_j,
// m2 = sum G_j t_j^2 and e0 = sum_j (w_j/sigma_j) dens_j, from which the
// gradients of the 87 record values follow in closed form (u is linear in t):
//   dL/dmu     = k M^T (y0 m0 + yd m1)                  (M = iso_inv, y = M(x - mu))
//   dL/ds_b    = (u0_b^2 m0 + 2 u0_b ud_b m1 + ud_b^2 m2) / s_b     (u = sqrt(k) y)
//   dL/dR[a,b] = -(u0_b v0_a m0 + (u0_b d_a + ud_b v0_a) m1 + ud_b d_a m2) / s_b
//   dL/dsigma~ = m0 / sigma~,   dL/dc = gC e0 (through the radiance clamp)
// then chained through the quaternion / SG-axis normalizations.  The 32 lanes
// hold the same primitive at the same time, so the 87 values are reduced with
// a warp-shuffle reduce-scatter (3 x 31 shuffles) and each lane issues one
// atomic per value it owns.
#include "gsx_common.cuh"
#include "render_warp.cuh"

namespace {

using namespace gsx;

struct PixelGrad {
  float gC[3], gD, gTe;
  float Ctot[3], Dtot, Tend;
};

// 32 values per lane -> lane L holds the warp sum of value L.
__device__ inline float reduce_scatter32(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
  float a16[16];
  {
    const bool up = lane & 16;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float keep = up ? v[i + 16] : v[i], send = up ? v[i] : v[i + 16];
      a16[i] = keep + __shfl_xor_sync(FULL, send, 16);
    }
  }
  float a8[8];
  {
    const bool up = lane & 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float keep = up ? a16[i + 8] : a16[i], send = up ? a16[i] : a16[i + 8];
      a8[i] = keep + __shfl_xor_sync(FULL, send, 8);
    }
  }
  float a4[4];
  {
    const bool up = lane & 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float keep = up ? a8[i + 4] : a8[i], send = up ? a8[i] : a8[i + 4];
      a4[i] = keep + __shfl_xor_sync(FULL, send, 4);
    }
  }
  float a2[2];
  {
    const bool up = lane & 2;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      float keep = up ? a4[i + 2] : a4[i], send = up ? a4[i] : a4[i + 2];
      a2[i] = keep + __shfl_xor_sync(FULL, send, 2);
    }
  }
  const bool up = lane & 1;
  float keep = up ? a2[1] : a2[0], send = up ? a2[0] : a2[1];
  return keep + __shfl_xor_sync(FULL, send, 1);
}

// Per-(lane, primitive) gradient of the 87-float record, given the moments.
struct CandGrad {
  float gmu[3], gq[4], gs[3], gsig;
  float gp[3];  // dL/d(pre-clamp radiance)
};

__device__ inline void geometry_grad(const SceneView& sv, const RayCtx& r, int64_t p,
                                     const SegBase& b, float m0, float m1, float m2,
                                     CandGrad& g) {
  const float4 g0 = __ldg(sv.geo + 4 * p), g1 = __ldg(sv.geo + 4 * p + 1),
               g2 = __ldg(sv.geo + 4 * p + 2), g3 = __ldg(sv.geo + 4 * p + 3);
  const float4 a0 = __ldg(sv.gaux + 5 * p), a1 = __ldg(sv.gaux + 5 * p + 1),
               a2 = __ldg(sv.gaux + 5 * p + 2);
  const float M[9] = {g1.x, g1.y, g1.z, g2.x, g2.y, g2.z, g3.x, g3.y, g3.z};
  const float v0[3] = {(b.hi[0] - g0.x) + b.lo[0], (b.hi[1] - g0.y) + b.lo[1],
                       (b.hi[2] - g0.z) + b.lo[2]};
  float y0[3], yd[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    y0[a] = fmaf(M[3 * a], v0[0], fmaf(M[3 * a + 1], v0[1], M[3 * a + 2] * v0[2]));
    yd[a] = fmaf(M[3 * a], r.df[0], fmaf(M[3 * a + 1], r.df[1], M[3 * a + 2] * r.df[2]));
  }
  const float sk = a2.x, k = sk * sk;
  // mean
  float w3[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) w3[a] = fmaf(y0[a], m0, yd[a] * m1);
#pragma unroll
  for (int a = 0; a < 3; ++a)
    g.gmu[a] = k * fmaf(M[a], w3[0], fmaf(M[3 + a], w3[1], M[6 + a] * w3[2]));
  // scales and rotation
  const float s[3] = {a1.y, a1.z, a1.w};
  const float mask[3] = {a2.y, a2.z, a2.w};
  float u0[3], ud[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    u0[a] = sk * y0[a];
    ud[a] = sk * yd[a];
  }
#pragma unroll
  for (int bb = 0; bb < 3; ++bb) {
    float t = fmaf(u0[bb] * u0[bb], m0, fmaf(2.f * u0[bb] * ud[bb], m1, ud[bb] * ud[bb] * m2));
    g.gs[bb] = mask[bb] * t / s[bb];
  }
  float gR[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int bb = 0; bb < 3; ++bb)
      gR[3 * a + bb] = -fmaf(u0[bb] * v0[a], m0,
                             fmaf(fmaf(u0[bb], r.df[a], ud[bb] * v0[a]), m1,
                                  ud[bb] * r.df[a] * m2)) / s[bb];
  // R(q) with q normalized (geometry.py:26-42): dR/dq, then the normalization
  const float w = a0.x, X = a0.y, Yq = a0.z, Z = a0.w;
  const float dR[4][9] = {
      {0.f, -2 * Z, 2 * Yq, 2 * Z, 0.f, -2 * X, -2 * Yq, 2 * X, 0.f},
      {0.f, 2 * Yq, 2 * Z, 2 * Yq, -4 * X, -2 * w, 2 * Z, 2 * w, -4 * X},
      {-4 * Yq, 2 * X, 2 * w, 2 * X, 0.f, 2 * Z, -2 * w, 2 * Z, -4 * Yq},
      {-4 * Z, -2 * w, 2 * X, 2 * w, -4 * Z, 2 * Yq, 2 * X, 2 * Yq, 0.f}};
  float gq[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < 9; ++e) acc = fmaf(gR[e], dR[c][e], acc);
    gq[c] = acc;
  }
  const float qv[4] = {w, X, Yq, Z};
  float dot = gq[0] * w + gq[1] * X + gq[2] * Yq + gq[3] * Z;
#pragma unroll
  for (int c = 0; c < 4; ++c) g.gq[c] = (gq[c] - dot * qv[c]) * a1.x;
  g.gsig = m0 / g0.w;
}

template <int G>
__device__ inline float record_value(int idx, const CandGrad& g, const float* Y, const float* lob,
                                     const float* ga, const float (*gax)[3], const float* gsh) {
  if (idx < 3) return g.gmu[idx];
  if (idx < 7) return g.gq[idx - 3];
  if (idx < 10) return g.gs[idx - 7];
  if (idx == 10) return g.gsig;
  if (idx < 38) return Y[(idx - 11) / 3] * g.gp[(idx - 11) % 3];
  if (idx < 59) return gax[(idx - 38) / 3][(idx - 38) % 3];
  if (idx < 66) return gsh[idx - 59];
  if (idx < 87) return lob[(idx - 66) / 3] * g.gp[(idx - 66) % 3];
  return 0.f;
}

// pass 2 for one staged candidate (all lanes in lockstep)
__device__ inline void grad_candidate(const SceneView& sv, const RayCtx& r, int64_t p, bool want,
                                      int mc, const SegBase& base, float dtf, const float* Y,
                                      const PixelGrad& pg, const float (&gs)[16],
                                      const float (&wos)[16], const float (&cg)[16],
                                      float* __restrict__ grad) {
  CandSetup cs;
  int jlo = 0, jhi = -1;
  bool use = want && mc > 0 && cand_setup(sv, r, p, base, cs) &&
             sample_range(cs, dtf, mc, jlo, jhi);
  if (!__any_sync(FULL, use)) return;
  float pre[3] = {0.f, 0.f, 0.f}, lob[7];
#pragma unroll
  for (int l = 0; l < 7; ++l) lob[l] = 0.f;
  if (use) eval_radiance_pre(sv.app + GSX_APP_F4 * p, Y, r.df, pre, lob);
  const float c0 = fmaxf(pre[0], 0.f), c1 = fmaxf(pre[1], 0.f), c2 = fmaxf(pre[2], 0.f);
  const float gcl = pg.gC[0] * c0 + pg.gC[1] * c1 + pg.gC[2] * c2;
  const float nkl2 = -cs.kl2;
  float m0 = 0.f, m1 = 0.f, m2 = 0.f, e0 = 0.f;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    if (!__any_sync(FULL, use && jlo <= 4 * g + 3 && jhi >= 4 * g)) continue;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * g + jj;
      float del = fmaf((float)j, dtf, cs.del0);
      float q = fmaf(cs.A * del, del, cs.qmin);
      if (use && q <= 1.0f) {
        float dens = ex2_approx(fmaf(nkl2, q, cs.lsig));
        float G = fmaf(wos[j], gcl - cg[j], gs[j]) * dens;
        float t = (float)j * dtf;
        m0 += G;
        m1 = fmaf(G, t, m1);
        m2 = fmaf(G * t, t, m2);
        e0 = fmaf(wos[j], dens, e0);
      }
    }
  }
  CandGrad g;
  float ga[7], gax[7][3], gsh[7];
#pragma unroll
  for (int i = 0; i < 3; ++i) g.gmu[i] = g.gs[i] = g.gp[i] = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) g.gq[i] = 0.f;
  g.gsig = 0.f;
#pragma unroll
  for (int l = 0; l < 7; ++l) {
    ga[l] = gsh[l] = 0.f;
    gax[l][0] = gax[l][1] = gax[l][2] = 0.f;
  }
  if (use) {
    geometry_grad(sv, r, p, base, m0, m1, m2, g);
    g.gp[0] = pre[0] > 0.f ? pg.gC[0] * e0 : 0.f;
    g.gp[1] = pre[1] > 0.f ? pg.gC[1] * e0 : 0.f;
    g.gp[2] = pre[2] > 0.f ? pg.gC[2] * e0 : 0.f;
    const float4* ap = sv.app + GSX_APP_F4 * p;
    const float4 i0 = __ldg(sv.gaux + 5 * p + 3), i1 = __ldg(sv.gaux + 5 * p + 4);
    const float inv_an[7] = {i0.x, i0.y, i0.z, i0.w, i1.x, i1.y, i1.z};
#pragma unroll
    for (int l = 0; l < 7; ++l) {
      const float4 ax = __ldg(ap + 9 + 2 * l), am = __ldg(ap + 10 + 2 * l);
      const float nx = ax.x, ny = ax.y, nz = ax.z;
      const float lam = ax.w;
      ga[l] = am.x * g.gp[0] + am.y * g.gp[1] + am.z * g.gp[2];
      const float cs2 = fmaf(nx, r.df[0], fmaf(ny, r.df[1], nz * r.df[2]));
      gsh[l] = lob[l] * (cs2 - 1.f) * ga[l];
      const float f = lob[l] * lam * ga[l];
      const float gn[3] = {f * r.df[0], f * r.df[1], f * r.df[2]};
      const float dd = gn[0] * nx + gn[1] * ny + gn[2] * nz;
      gax[l][0] = (gn[0] - dd * nx) * inv_an[l];
      gax[l][1] = (gn[1] - dd * ny) * inv_an[l];
      gax[l][2] = (gn[2] - dd * nz) * inv_an[l];
    }
  }
  const int lane = threadIdx.x & 31;
  float* gp = grad + (int64_t)GSX_NREC * p;
#pragma unroll
  for (int grp = 0; grp < 3; ++grp) {
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = record_value<0>(32 * grp + i, g, Y, lob, ga, gax, gsh);
    float s = reduce_scatter32(v);
    const int idx = 32 * grp + lane;
    if (idx < GSX_NREC && s != 0.f) atomicAdd(gp + idx, s);
  }
}

__device__ bool backward_segment(const SceneView& sv, const BvhView& bv, const RayCtx& r,
                                 bool want, const Seg& seg, int ns, const float* Y,
                                 RayAccum& acc, const PixelGrad& pg, Counters<false>& cnt,
                                 WarpSmem& sm, float* __restrict__ grad) {
  bool nonempty = false;
  const float dtf = (float)seg.dt;
  const int nchunks = (ns + 15) / 16;
  uint32_t visits = 0;
  for (int ch = 0; ch < nchunks; ++ch) {
    int mc = want ? seg.m - ch * 16 : 0;
    mc = mc < 0 ? 0 : (mc > 16 ? 16 : mc);
    const double tb = seg.tbase + (double)(ch * 16) * seg.dt;
    const SegBase base = seg_base(r, tb);
    if (!__any_sync(FULL, want && (mc > 0 || ch == 0))) continue;
    float gs[16], wos[16], cg[16];
    // the candidate stream, staged exactly as in the forward (render.cu):
    // resident when it fits the shared list (the common case), else chunked
    // with a second traversal for pass 2
    WarpTrav st;
    SegLimits lim;
    int count;
    stage_candidates(bv, r, want, seg, sm, st, count, lim, visits);
    const bool resident = st.done;
    {
      float sig[16];
      float W[16][3];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        sig[j] = 0.f;
        W[j][0] = W[j][1] = W[j][2] = 0.f;
      }
      // pass 1: the forward's exact accumulation (same candidate order)
      auto exact = [&](int64_t p) {
        if (want && !nonempty && exact_aabb_overlap(sv, r, p, seg.t0, seg.t1)) nonempty = true;
      };
      for (;;) {
        accumulate_list(sv, r, sm, count, want, mc, base, dtf, Y, sig, W, exact);
        if (st.done) break;
        __syncwarp();
        count = 0;
        warp_traverse(bv, r, want, lim.lo_t, lim.hi_t, lim.gap, st, sm, count, visits);
      }
      // replay the compositing and form the per-sample adjoints
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        gs[j] = wos[j] = cg[j] = 0.f;
        if (j < mc) {
          const float tj = (float)(tb + (double)j * seg.dt);
          const float sj = sig[j];
          const float Tj = acc.T;
          acc.add_sample(sj, W[j], tj, dtf);
          if (sj > 0.f) {
            const float ods = sj * dtf;
            const float w = -expm1f(-ods) * Tj;  // the forward's w_j (RayAccum::add_sample)
            const float s = w / sj;
            const float isg = 1.f / sj;
            const float cgj = (pg.gC[0] * W[j][0] + pg.gC[1] * W[j][1] + pg.gC[2] * W[j][2]) * isg;
            const float after = pg.gC[0] * (pg.Ctot[0] - acc.C[0]) +
                                pg.gC[1] * (pg.Ctot[1] - acc.C[1]) +
                                pg.gC[2] * (pg.Ctot[2] - acc.C[2]);
            const float T1 = acc.T;
            gs[j] = dtf * (T1 * cgj - after + pg.gD * (T1 * tj - (pg.Dtot - acc.D)) -
                           pg.gTe * pg.Tend);
            wos[j] = s;
            cg[j] = cgj;
          }
        }
      }
    }
    if (!__any_sync(FULL, want && mc > 0)) {
      __syncwarp();
      continue;
    }
    // pass 2: per-primitive gradients over the same deterministic candidate stream
    auto pass2 = [&](int64_t p) {
      grad_candidate(sv, r, p, want, mc, base, dtf, Y, pg, gs, wos, cg, grad);
    };
    if (resident) {
      for (int i = 0; i < count; ++i) pass2((int64_t)sm.list[i]);
    } else {
      uint32_t v2 = 0;
      for_each_candidate(bv, r, want, lim.lo_t, lim.hi_t, lim.gap, sm, v2, pass2);
    }
    __syncwarp();
  }
  emptiness_tail<false>(sv, bv, r, want, seg, nonempty, cnt);
  return nonempty;
}

// CTA = BWD_THREADS rays = 256 / BWD_THREADS CTAs per 16x16 tile
#ifndef GSX_BWD_THREADS
#define GSX_BWD_THREADS 256
#endif
#ifndef GSX_BWD_MINB
#define GSX_BWD_MINB 1
#endif
constexpr int BWD_THREADS = GSX_BWD_THREADS;
constexpr int BWD_PER_TILE = 256 / BWD_THREADS;

__global__ void __launch_bounds__(BWD_THREADS, GSX_BWD_MINB) k_render_backward(
    SceneView sv, BvhView bv, gsx_camera cam, gsx_render_cfg cfg, int64_t tile_begin,
    int64_t tile_stride, const float* __restrict__ rgb, const float* __restrict__ depth,
    const float* __restrict__ trans, const float* __restrict__ dL_drgb,
    const float* __restrict__ dL_ddepth, const float* __restrict__ dL_dtrans,
    float* __restrict__ grad) {
  __shared__ WarpSmem smem[BWD_THREADS / 32];
  int64_t W = cam.width, H = cam.height;
  int64_t tiles_x = (W + 15) / 16;
  int64_t tile = tile_begin + (int64_t)(blockIdx.x / BWD_PER_TILE) * tile_stride;
  int mx, my;
  morton_decode8((blockIdx.x % BWD_PER_TILE) * BWD_THREADS + threadIdx.x, mx, my);
  int64_t px = (tile % tiles_x) * 16 + mx, py = (tile / tiles_x) * 16 + my;
  bool valid = px < W && py < H;
  RayCtx r;
  bool hit = valid && camera_ray(cam, (double)px, (double)py, sv.bounds, r);
  PixelGrad pg;
  if (valid) {
    int64_t pix = py * W + px;
    pg.Tend = trans[pix];
    pg.Dtot = depth[pix];
    pg.gD = dL_ddepth ? dL_ddepth[pix] : 0.f;
    float gT = dL_dtrans ? dL_dtrans[pix] : 0.f;
    float gTe = gT;
    for (int k = 0; k < 3; ++k) {
      pg.gC[k] = dL_drgb[3 * pix + k];
      pg.Ctot[k] = rgb[3 * pix + k] - pg.Tend * (float)cfg.background[k];
      gTe = fmaf(pg.gC[k], (float)cfg.background[k], gTe);
    }
    pg.gTe = gTe;
  } else {
    pg = PixelGrad{{0.f, 0.f, 0.f}, 0.f, 0.f, {0.f, 0.f, 0.f}, 0.f, 1.f};
  }
  RayAccum acc;
  acc.init();
  float Y[9];
  sh_basis_f(r.df, Y);
  Counters<false> cnt;
  const int ns = (int)cfg.n_s;
  WarpSmem& sm = smem[threadIdx.x >> 5];
  march_warp<false>(sv, bv, r, hit, cfg, acc, cnt, GSX_SYNC_BWD, [&](const Seg& seg, bool want) {
    return backward_segment(sv, bv, r, want, seg, ns, Y, acc, pg, cnt, sm, grad);
  });
}

}  // namespace

extern "C" int gsx_render_backward(const void* scene_arena, const void* bvh_arena,
                                   const float* params, int64_t n, const gsx_camera* cam,
                                   const gsx_render_cfg* cfg, int64_t tile_begin,
                                   int64_t tile_stride, const float* rgb, const float* depth,
                                   const float* trans, const float* dL_drgb,
                                   const float* dL_ddepth, const float* dL_dtrans, float* grad,
                                   gsx_dev_status* dev_status, void* stream) {
  (void)params;
  (void)dev_status;
  int rc = gsx_validate_cfg(cfg);
  if (rc) return rc;
  if (!cam || cam->width < 1 || cam->height < 1 || !(cam->focal > 0)) return GSX_ERR_ARG;
  if (n <= 0) return GSX_ERR_EMPTY;
  if (!rgb || !depth || !trans || !dL_drgb || !grad) return GSX_ERR_ARG;
  if (tile_stride < 1 || tile_begin < 0) return GSX_ERR_ARG;
  int64_t tiles = ((cam->width + 15) / 16) * ((cam->height + 15) / 16);
  if (tile_begin >= tiles) return GSX_OK;
  int64_t blocks = BWD_PER_TILE * ((tiles - tile_begin + tile_stride - 1) / tile_stride);
  SceneView sv = scene_view((void*)scene_arena, n);
  BvhView bv = bvh_view((void*)bvh_arena, n);
  k_render_backward<<<(unsigned)blocks, BWD_THREADS, 0, (cudaStream_t)stream>>>(
      sv, bv, *cam, *cfg, tile_begin, tile_stride, rgb, depth, trans, dL_drgb, dL_ddepth,
      dL_dtrans, grad);
  return gsx_check_launch();
}
