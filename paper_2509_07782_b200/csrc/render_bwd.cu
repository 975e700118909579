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
#include "march_log.cuh"
#include "render_warp.cuh"

namespace {

using namespace gsx;

struct PixelGrad {
  float gC[3], gD, gTe;
  float Ctot[3], Dtot, Tend;
};

// ---------------------------------------------------------------------------
// Pass-2 reduction.  All 32 lanes hold the same candidate p; per lane and p
// the values below are formed from the moments and reduced over the warp in
// a shared buffer (row = value, column = lane; rows padded to 36 floats: the
// column writes hit banks (4 row + lane) mod 32 and the row sums read 16-byte
// vectors conflict-free per quarter warp).  Rows, in two halves:
//   A (32 rows): 0-9 geometry moments, 10-31 SH (b, c) 0-21 -> record 11 + 3b + c
//   B (49 + 5 rows): lobe l at 7l: raw axis sum (3), sharpness, amplitude (3);
//     SH 22-26 at 7 SG_GROUP (written with half A, summed in the first lobe
//     pass: 3 row passes per candidate instead of 4)
// Geometry enters only through the moment tensors of the lane offsets
// v = xc - mu and the direction d, with xc the ray's point of closest
// approach to the primitive (t_c of the setup) and the moments taken in
// t - t_c:
//   S0 = m0,  S1 = v m0 + d m1,  S2 = v v^T m0 + (v d^T + d v^T) m1 + d d^T m2
// (6 unique entries), because with y = M v and u = sqrt(k) y every geometry
// gradient is linear in them (M = iso_inv, header formulas).  Centring on
// t_c keeps |u| <= 1 for every contributing sample: moments about the chunk
// base (|u0| up to ~40 for a small primitive far into a long adaptive chunk)
// cancel in u0^2 m0 + 2 u0 ud m1 + ud^2 m2 and cost the scale gradients
// ~1e-4 of their maximum in fp32 (C4; profiles/r06_grad_err_c4*.json):
//   dL/dmu = k M^T M S1,  dL/ds_b = k (M S2 M^T)_bb / s_b (unclamped),
//   dL/dR[a,b] = -sqrt(k) (M S2)_ba / s_b,  dL/dsigma~ = S0 / sigma~,
// and the SG axis gradient is (I - n n^T)/|a| applied to sum_lanes f d.
// Those 31 reduced values go to a per-warp batch; every 32 candidates lane c
// finishes candidate c (matrix algebra, quaternion chain, projections) and
// issues its atomics -- the per-lane geometry work of the old formulation
// (~240 instructions per candidate) becomes ~45 + 1/32 of the finish.
constexpr int RED_ROW = 36;
constexpr int RED_ROWS_A = 32;
// half B in lobe groups of SG_GROUP (7: one pass of 49 rows; 4: two passes of
// 28 and 21 rows, so the buffer is sized by half A and a CTA needs 15% less
// shared memory).  Logged backward, C2 ms (profiles/time_bwd_variants.py):
// 7 / 4 CTAs x 128 regs 13.13 (this build); 4 13.74; 4 + 5 CTAs x 96 regs
// 15.73; 7 + 3 CTAs x 168 regs (no spills) 13.55; 5 CTAs x 96 regs 16.60;
// 64-thread CTAs x 8 13.40.  More warps do not pay for the spills.
#ifndef GSX_BWD_SG_GROUP
#define GSX_BWD_SG_GROUP 7
#endif
constexpr int SG_GROUP = GSX_BWD_SG_GROUP;
constexpr int SH_TAIL_ROW = 7 * SG_GROUP;  // SH values 22-26
constexpr int RED_ROWS_B = 7 * SG_GROUP + 5;
constexpr int RED_FLOATS = (RED_ROWS_B > RED_ROWS_A ? RED_ROWS_B : RED_ROWS_A) * RED_ROW;
constexpr int BAT_ROW = 33;                        // 31 values + candidate id, padded
constexpr int BAT_FLOATS = 32 * BAT_ROW;
constexpr int BWD_WARP_FLOATS = RED_FLOATS + BAT_FLOATS;  // shared floats per warp

struct GradBatch {
  float* red;  // RED_FLOATS
  float* bat;  // BAT_FLOATS: bat[c][0..9] geometry, [10..30] raw axes, [31] id
  int n;       // candidates pending (warp-uniform)
};

__device__ inline float row_sum(const float* __restrict__ red, int row) {
  const float4* rp = (const float4*)(red + row * RED_ROW);
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float4 v = rp[k];
    s0 += v.x;
    s1 += v.y;
    s2 += v.z;
    s3 += v.w;
  }
  return (s0 + s1) + (s2 + s3);
}

// Finish the pending candidates: lane c owns candidate c of the batch.
__device__ inline void grad_batch_flush(const SceneView& sv, GradBatch& gb,
                                        float* __restrict__ grad) {
  __syncwarp();
  const int lane = threadIdx.x & 31;
  if (lane < gb.n) {
    const float* v = gb.bat + lane * BAT_ROW;
    const int64_t p = __float_as_int(v[31]);
    const float4 g0 = __ldg(sv.geo + 4 * p), g1 = __ldg(sv.geo + 4 * p + 1),
                 g2 = __ldg(sv.geo + 4 * p + 2), g3 = __ldg(sv.geo + 4 * p + 3);
    const float4 a0 = __ldg(sv.gaux + 5 * p), a1 = __ldg(sv.gaux + 5 * p + 1),
                 a2 = __ldg(sv.gaux + 5 * p + 2), a3 = __ldg(sv.gaux + 5 * p + 3),
                 a4 = __ldg(sv.gaux + 5 * p + 4);
    (void)g0;
    const float M[9] = {g1.x, g1.y, g1.z, g2.x, g2.y, g2.z, g3.x, g3.y, g3.z};
    const float S1[3] = {v[1], v[2], v[3]};
    // S2 symmetric: (xx, yy, zz, xy, xz, yz)
    const float S2[9] = {v[4], v[7], v[8], v[7], v[5], v[9], v[8], v[9], v[6]};
    const float sk = a2.x, k = sk * sk;
    float* gp = grad + (int64_t)GSX_NREC * p;
    // mean: k M^T (M S1)
    float y1[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) y1[a] = fmaf(M[3 * a], S1[0], fmaf(M[3 * a + 1], S1[1], M[3 * a + 2] * S1[2]));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const float g = k * fmaf(M[a], y1[0], fmaf(M[3 + a], y1[1], M[6 + a] * y1[2]));
      if (g != 0.f) atomicAdd(gp + a, g);
    }
    // MS = M S2 (row b = M_b S2)
    float MS[9];
#pragma unroll
    for (int bb = 0; bb < 3; ++bb)
#pragma unroll
      for (int a = 0; a < 3; ++a)
        MS[3 * bb + a] = fmaf(M[3 * bb], S2[a], fmaf(M[3 * bb + 1], S2[3 + a], M[3 * bb + 2] * S2[6 + a]));
    const float is[3] = {a1.y, a1.z, a1.w};
    const float mask[3] = {a2.y, a2.z, a2.w};
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) {
      const float t = fmaf(MS[3 * bb], M[3 * bb], fmaf(MS[3 * bb + 1], M[3 * bb + 1], MS[3 * bb + 2] * M[3 * bb + 2]));
      const float g = mask[bb] * k * t * is[bb];
      if (g != 0.f) atomicAdd(gp + 7 + bb, g);
    }
    float gR[9];  // gR[3a + b] = -sqrt(k) (M S2)_ba / s_b
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int bb = 0; bb < 3; ++bb) gR[3 * a + bb] = -sk * MS[3 * bb + a] * is[bb];
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
    const float dot = gq[0] * w + gq[1] * X + gq[2] * Yq + gq[3] * Z;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float g = (gq[c] - dot * qv[c]) * a1.x;
      if (g != 0.f) atomicAdd(gp + 3 + c, g);
    }
    const float gs = v[0] * a4.w;  // / sigma~
    if (gs != 0.f) atomicAdd(gp + 10, gs);
    // SG axes: d/d(raw axis) of the unit axis n is (I - n n^T) / |a|
    const float4* ap = sv.app + GSX_APP_F4 * p;
    const float inv_an[7] = {a3.x, a3.y, a3.z, a3.w, a4.x, a4.y, a4.z};
#pragma unroll 1
    for (int l = 0; l < 7; ++l) {
      const float4 ax = __ldg(ap + 9 + 2 * l);
      const float r0 = v[10 + 3 * l], r1 = v[11 + 3 * l], r2 = v[12 + 3 * l];
      const float dd = r0 * ax.x + r1 * ax.y + r2 * ax.z;
      const float ia = inv_an[l];
      const float gx = (r0 - dd * ax.x) * ia, gy = (r1 - dd * ax.y) * ia,
                  gz = (r2 - dd * ax.z) * ia;
      if (gx != 0.f) atomicAdd(gp + 38 + 3 * l, gx);
      if (gy != 0.f) atomicAdd(gp + 39 + 3 * l, gy);
      if (gz != 0.f) atomicAdd(gp + 40 + 3 * l, gz);
    }
  }
  __syncwarp();
  gb.n = 0;
}

// Replay one composited sample (the forward's RayAccum::add_sample) and form
// its adjoint terms: pass 2 uses G_j = dens_j (wos_j gC.c + h_j) with
// wos_j = w_j / sigma_j and h_j = dL/dsigma_j - wos_j gC.c_j.
__device__ inline void sample_adjoint(RayAccum& acc, const PixelGrad& pg, float sj,
                                      const float* Wj, float tj, float dtf, float& wos,
                                      float& h) {
  const float Tj = acc.T;
  acc.add_sample(sj, Wj, tj, dtf);
  if (sj > 0.f) {
    const float ods = sj * dtf;
    const float w = RayAccum::alpha(ods) * Tj;  // the forward's w_j
    const float s = w / sj;
    const float cgj = (pg.gC[0] * Wj[0] + pg.gC[1] * Wj[1] + pg.gC[2] * Wj[2]) / sj;
    const float after = pg.gC[0] * (pg.Ctot[0] - acc.C[0]) + pg.gC[1] * (pg.Ctot[1] - acc.C[1]) +
                        pg.gC[2] * (pg.Ctot[2] - acc.C[2]);
    const float T1 = acc.T;
    const float gs =
        dtf * (T1 * cgj - after + pg.gD * (T1 * tj - (pg.Dtot - acc.D)) - pg.gTe * pg.Tend);
    wos = s;
    h = fmaf(-s, cgj, gs);
  }
}

// pass 2 for one staged candidate (all lanes in lockstep).  Every lane writes
// its values (zeros when it does not see p) as one column of the warp's
// reduction buffer as soon as they are formed; lane L then sums rows L, L+32
// of each half: direct rows go to atomics, the geometry / axis rows to the
// batch (see the section comment above).
// app: p's appearance block -- in global memory (the replay kernel) or staged
// in the warp's shared buffer by a TMA bulk copy (the logged kernel)
template <class L = LdgLoad>
__device__ inline void grad_candidate(const SceneView& sv, const RayCtx& r, int64_t p, bool want,
                                      int mc, const SegBase& base, float dtf, const float* Y,
                                      const PixelGrad& pg, const float (&wos)[16],
                                      const float (&hh)[16], GradBatch& gb,
                                      float* __restrict__ grad, const float4* app = nullptr) {
  if (!app) app = sv.app + GSX_APP_F4 * p;
  CandSetup cs;
  int jlo = 0, jhi = -1;
  bool use = want && mc > 0 && cand_setup(sv, r, p, base, cs) &&
             sample_range(cs, dtf, mc, jlo, jhi);
  if (!__any_sync(FULL, use)) return;
  const int lane = threadIdx.x & 31;
  float* col = gb.red + lane;
  float pre[3];
  eval_radiance_pre<L>(app, Y, r.df, pre, nullptr);
  const float gcl =
      pg.gC[0] * fmaxf(pre[0], 0.f) + pg.gC[1] * fmaxf(pre[1], 0.f) + pg.gC[2] * fmaxf(pre[2], 0.f);
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
        float G = fmaf(wos[j], gcl, hh[j]) * dens;
        m0 += G;  // moments in del = t_j - t_c (see vc below)
        m1 = fmaf(G, del, m1);
        m2 = fmaf(G * del, del, m2);
        e0 = fmaf(wos[j], dens, e0);
      }
    }
  }
  // lanes that do not see p have zero moments: every value below is 0
  {
    const float4 g0 = __ldg(sv.geo + 4 * p);
    const float* d = r.df;
    const float tcu = use ? cs.tc : 0.f;
    const float v0[3] = {fmaf(d[0], tcu, (base.hi[0] - g0.x) + base.lo[0]),
                         fmaf(d[1], tcu, (base.hi[1] - g0.y) + base.lo[1]),
                         fmaf(d[2], tcu, (base.hi[2] - g0.z) + base.lo[2])};
    col[0] = m0;
#pragma unroll
    for (int a = 0; a < 3; ++a) col[(1 + a) * RED_ROW] = fmaf(v0[a], m0, d[a] * m1);
    // S2 (xx, yy, zz, xy, xz, yz)
    const int ia[6] = {0, 1, 2, 0, 0, 1}, ib[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      const float va = v0[ia[e]], vb = v0[ib[e]], da = d[ia[e]], db = d[ib[e]];
      col[(4 + e) * RED_ROW] = fmaf(va * vb, m0, fmaf(fmaf(va, db, da * vb), m1, da * db * m2));
    }
  }
  float gpc[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) gpc[c] = (use && pre[c] > 0.f) ? pg.gC[c] * e0 : 0.f;
#pragma unroll
  for (int bsh = 0; bsh < 9; ++bsh)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int idx = 3 * bsh + c;
      col[(idx < 22 ? 10 + idx : SH_TAIL_ROW + idx - 22) * RED_ROW] = Y[bsh] * gpc[c];
    }
  // half A: geometry moments -> batch, SH -> atomics
  float* gdst = grad + (int64_t)GSX_NREC * p;
  float* brow = gb.bat + gb.n * BAT_ROW;
  __syncwarp();
  {
    const int row = lane;
    const float sum = row_sum(gb.red, row);
    if (row < 10)
      brow[row] = sum;
    else if (sum != 0.f)
      atomicAdd(gdst + 11 + (row - 10), sum);
  }
  if (lane == 0) brow[31] = __int_as_float((int)p);
  __syncwarp();
  // half B: spherical-Gaussian lobes, one at a time (rolled: keeps the 14
  // float4 of lobe data out of registers); the lobe value is recomputed
  const float4* ap = app;
#pragma unroll 1
  for (int l0 = 0; l0 < 7; l0 += SG_GROUP) {
    const int nl = min(SG_GROUP, 7 - l0);
#pragma unroll 1
    for (int l = l0; l < l0 + nl; ++l) {
      const float4 ax = L()(ap + 9 + 2 * l), am = L()(ap + 10 + 2 * l);
      const float cs2 = fmaf(ax.x, r.df[0], fmaf(ax.y, r.df[1], ax.z * r.df[2]));
      const float lb = __expf(ax.w * (cs2 - 1.0f));  // == eval_radiance_pre's lobe value
      const float ga = am.x * gpc[0] + am.y * gpc[1] + am.z * gpc[2];
      const float f = lb * ax.w * ga;
      float* c = col + 7 * (l - l0) * RED_ROW;
      c[0] = f * r.df[0];
      c[RED_ROW] = f * r.df[1];
      c[2 * RED_ROW] = f * r.df[2];
      c[3 * RED_ROW] = lb * (cs2 - 1.f) * ga;
      c[4 * RED_ROW] = lb * gpc[0];
      c[5 * RED_ROW] = lb * gpc[1];
      c[6 * RED_ROW] = lb * gpc[2];
    }
    __syncwarp();
    for (int row = lane; row < 7 * nl + (l0 == 0 ? 5 : 0); row += 32) {
      const float sum = row_sum(gb.red, row);
      const int l = l0 + row / 7, k = row % 7;
      if (row >= 7 * nl) {  // SH 22-26 (first pass only)
        if (sum != 0.f) atomicAdd(gdst + 11 + 22 + (row - 7 * nl), sum);
      } else if (k < 3)
        brow[10 + 3 * l + k] = sum;
      else if (sum != 0.f)
        atomicAdd(gdst + (k == 3 ? 59 + l : 66 + 3 * l + (k - 4)), sum);
    }
    __syncwarp();
  }
  if (++gb.n == 32) grad_batch_flush(sv, gb, grad);
}

__device__ bool backward_segment(const SceneView& sv, const BvhView& bv, const RayCtx& r,
                                 bool want, const Seg& seg, int ns, const float* Y,
                                 RayAccum& acc, const PixelGrad& pg, Counters<false>& cnt,
                                 WarpSmem& sm, GradBatch& gb, float* __restrict__ grad) {
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
    float wos[16], hh[16];
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
      auto exact = [&](int64_t p, bool) {
        if (want && !nonempty && exact_aabb_overlap(sv, r, p, seg.t0, seg.t1)) nonempty = true;
      };
      for (;;) {
        accumulate_list(sv, r, sm, count, want, mc, base, dtf, Y, sig, W, exact,
                        [](int, int64_t, unsigned) {});
        if (st.done) break;
        __syncwarp();
        count = 0;
        warp_traverse(bv, r, want, lim.lo_t, lim.hi_t, lim.gap, st, sm, count, visits);
      }
      // replay the compositing and form the per-sample adjoints
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        wos[j] = hh[j] = 0.f;
        if (j < mc)
          sample_adjoint(acc, pg, sig[j], W[j], (float)(tb + (double)j * seg.dt), dtf, wos[j],
                         hh[j]);
      }
    }
    if (!__any_sync(FULL, want && mc > 0)) {
      __syncwarp();
      continue;
    }
#ifdef GSX_BWD_NO_PASS2  // timing experiment only: replay without pass 2
    __syncwarp();
    continue;
#endif
    // pass 2: per-primitive gradients over the same deterministic candidate
    // stream (the resident list, or a re-traversal in chunks).  One call site
    // of grad_candidate: the kernel is instruction-cache bound (ncu
    // stall_no_inst), so its largest body must not be inlined twice.
    WarpTrav st2 = st;
    if (!resident) {
      st2 = WarpTrav{0, 0, false, false};
      count = 0;
    }
    uint32_t v2 = 0;
    for (;;) {
      if (!st2.done) warp_traverse(bv, r, want, lim.lo_t, lim.hi_t, lim.gap, st2, sm, count, v2);
      for (int i = 0; i < count; ++i)
        grad_candidate(sv, r, (int64_t)sm.list[i], want, mc, base, dtf, Y, pg, wos, hh, gb,
                       grad);
      __syncwarp();
      if (st2.done) break;
      count = 0;
    }
  }
  emptiness_tail<false>(sv, bv, r, want, seg, nonempty, cnt, sm.ovf);
  return nonempty;
}

// ---------------------------------------------------------------------------
// Logged pass 2 over (lane, primitive) pairs.  The forward logged, per kept
// list entry, the lanes whose setup of it succeeded (march_log.cuh umask):
// about a third of the warp per entry.  Walking the entries with all 32
// lanes in lockstep (grad_candidate) idles the rest through the setup,
// radiance and moment work and reduces 86 mostly-zero columns per entry.
// Here a list's pairs are enumerated in entry order and taken 32 at a time:
// lane k works pair k with its ray's data (direction, segment base, sample
// adjoints) read from the warp's lane table, and the 86 per-pair values are
// summed per entry over the entry's run of lanes (a segmented column sum
// through shared memory, one row per lane) in three passes of <= 32 rows:
//   P1: geometry moments (10) + SH values 0-21      -> batch / atomics
//   P2: lobes 0-3 (7 rows each)                     -> batch (axes) / atomics
//   P3: SH values 22-26 + lobes 4-6                 -> atomics / batch
// An entry split by a 32-pair boundary contributes two batch rows; every
// finished value is linear in them, so the atomics add up the same.  The
// lobe rows are formed from terms the radiance evaluation keeps in registers
// (radiance_lobe_terms), not from a second read of the appearance block.
// ---------------------------------------------------------------------------
constexpr int PR_ROW = 36;  // a row per lane, 32 pair columns (16-byte rows: float4 reads conflict-free)
constexpr int PR_FLOATS = 32 * PR_ROW;
constexpr int LT_ROWS = 14;  // lane table: df[3], base.hi[3], base.lo[3], dtf, mc, gC[3]
constexpr int WH_FLOATS = 2 * 16 * 32;  // wos[16][32], hh[16][32]
constexpr int PAIR_RUNS = 32;  // entries (runs) per pair batch = batch rows of the finish
constexpr int PAIR_WARP_FLOATS = PR_FLOATS + WH_FLOATS + LT_ROWS * 32 + PAIR_RUNS * BAT_ROW;

struct PairBufs {
  float* pr;  // PR_FLOATS
  float* wh;  // WH_FLOATS
  float* lt;  // LT_ROWS x 32
};

// position of the n-th (0-based) set bit of m
__device__ inline int nth_bit(unsigned m, int n) {
  int pos = 0;
#pragma unroll
  for (int w = 16; w; w >>= 1) {
    const unsigned lo = m & ((1u << w) - 1u);
    const int c = __popc(lo);
    if (n >= c) {
      n -= c;
      m >>= w;
      pos += w;
    } else {
      m = lo;
    }
  }
  return pos;
}

// Radiance of one pair's primitive (eval_radiance_pre's arithmetic, so `pre`
// is the same) keeping, per lobe, what the lobe gradient columns need: e*w,
// e*(cs2-1), e and am.gC with the radiance clamp applied.  Reloading them in
// the lobe pass cost 30% of the pair kernel (L1 is nearly all shared memory
// there, so every reload was an L2 round trip).
struct LobeTerms {
  float w[7], c[7], v[7], g[7];
};
__device__ inline void radiance_lobe_terms(const float4* __restrict__ app, const YDir& Y,
                                           const float* d, const float* gC, float* pre,
                                           LobeTerms& lt) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int b = 0; b < 9; ++b) {
    const float4 v = __ldg(app + b);
    s0 = fmaf(Y[b], v.x, s0);
    s1 = fmaf(Y[b], v.y, s1);
    s2 = fmaf(Y[b], v.z, s2);
  }
#pragma unroll
  for (int l = 0; l < 7; ++l) {
    const float4 ax = __ldg(app + 9 + 2 * l), am = __ldg(app + 10 + 2 * l);
    const float cs2 = fmaf(ax.x, d[0], fmaf(ax.y, d[1], ax.z * d[2]));
    const float e = __expf(ax.w * (cs2 - 1.0f));
    s0 = fmaf(e, am.x, s0);
    s1 = fmaf(e, am.y, s1);
    s2 = fmaf(e, am.z, s2);
    lt.v[l] = e;
    lt.w[l] = e * ax.w;
    lt.c[l] = e * (cs2 - 1.f);
    lt.g[l] = am.x * gC[0] + am.y * gC[1] + am.z * gC[2];
  }
  pre[0] = s0;
  pre[1] = s1;
  pre[2] = s2;
  if (!(s0 > 0.f && s1 > 0.f && s2 > 0.f)) {  // a clamped channel: rare
#pragma unroll
    for (int l = 0; l < 7; ++l) {
      const float4 am = __ldg(app + 10 + 2 * l);
      lt.g[l] = (s0 > 0.f ? am.x * gC[0] : 0.f) + (s1 > 0.f ? am.y * gC[1] : 0.f) +
                (s2 > 0.f ? am.z * gC[2] : 0.f);
    }
  }
}

// Sum rows [0, nrows) of the pass buffer over each run of `ends` (bit k set:
// pair k is the last of its entry in this batch) and hand (row, sum, entry's
// primitive, run index) to emit.  Lane = row: one pass over the 32 columns
// (float4 loads), the running sum restarted after each run end (a
// warp-uniform select) and stored over the run's last column; then one emit
// per (row, run).
template <class Emit>
__device__ inline void pair_reduce(const PairBufs& pb, unsigned ends, int pe, int nrows,
                                   Emit&& emit) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  float* rp = pb.pr + lane * PR_ROW;
  if (lane < nrows) {
    float acc = 0.f;
#pragma unroll
    for (int k4 = 0; k4 < 8; ++k4) {
      const float4 v = *(const float4*)(rp + 4 * k4);
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int k = 4 * k4 + c;
        acc = (k > 0 && ((ends >> (k - 1)) & 1u)) ? vv[c] : acc + vv[c];
        if ((ends >> k) & 1u) rp[k] = acc;
      }
    }
  }
  __syncwarp();
  int run = 0;
  while (ends) {
    const int k1 = __ffs(ends) - 1;
    ends &= ends - 1;
    const int pseg = __shfl_sync(FULL, pe, k1);
    if (lane < nrows) emit(lane, rp[k1], (int64_t)pseg, run);
    ++run;
  }
  __syncwarp();
}

// Pass 2 over one logged list (entries + use masks) of the current record.
// (Routing the entries most lanes use through the all-lanes path instead
// (grad_candidate) measured slower: C2 17.0 vs 14.3 ms.)
__device__ void pair_pass(const SceneView& sv, const PairBufs& pb, GradBatch& gb,
                          const int32_t* __restrict__ list, const uint32_t* __restrict__ umask,
                          int count, float* __restrict__ grad) {
  const int lane = threadIdx.x & 31;
  for (int i0 = 0; i0 < count; i0 += 32) {
    const bool have = i0 + lane < count;
    const int ent = have ? __ldcs(list + i0 + lane) : 0;
    const unsigned em = have ? __ldcs(umask + i0 + lane) : 0u;
    int incl = __popc(em);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(FULL, incl, 31);
    // batches of <= 32 pairs from <= PAIR_RUNS entries
    for (int b0 = 0; b0 < total;) {
      const int g = b0 + lane;
      // entry of pair g: the number of entries whose inclusive count is <= g
      int e = 0;
#pragma unroll
      for (int st = 16; st; st >>= 1)
        if (__shfl_sync(FULL, incl, e + st - 1) <= g) e += st;
      const int e0b = __shfl_sync(FULL, e, 0);
      const int bend = min(min(b0 + 32, total),
                           e0b + PAIR_RUNS < 32 ? __shfl_sync(FULL, incl, e0b + PAIR_RUNS - 1)
                                                : total);
      const bool valid = g < bend;
      const int pe = __shfl_sync(FULL, ent, e);
      const unsigned me = __shfl_sync(FULL, em, e);
      const int ex = __shfl_sync(FULL, incl, e) - __popc(me);
      const int src = valid ? nth_bit(me, g - ex) : 0;
      const int last = bend - b0 - 1;
      const int en = __shfl_down_sync(FULL, e, 1);
      const unsigned ends = __ballot_sync(FULL, valid && (lane == last || en != e));
      const int nrun = __popc(ends);
      b0 = bend;
      PH_BEGIN(ph_f)
      if (gb.n + nrun > PAIR_RUNS) grad_batch_flush(sv, gb, grad);
      PH_END(6, ph_f)
      PH_BEGIN(ph_su)

      // ---- the pair: setup, radiance, moments (renderer.py:207-240 adjoint)
      const float* lt = pb.lt + src;
      RayCtx rr;
      rr.df[0] = lt[0];
      rr.df[1] = lt[32];
      rr.df[2] = lt[64];
      SegBase base;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        base.hi[k] = lt[(3 + k) * 32];
        base.lo[k] = lt[(6 + k) * 32];
      }
      const float dtf = lt[9 * 32];
      const int mc = __float_as_int(lt[10 * 32]);
      const float gC[3] = {lt[11 * 32], lt[12 * 32], lt[13 * 32]};
      const int64_t p = pe;
      CandSetup cs;
      int jlo = 0, jhi = -1;
      const bool use = valid && cand_setup_at(sv.geo + 4 * p, rr, base, cs) &&
                       sample_range(cs, dtf, mc, jlo, jhi);
      const YDir Y{rr.df};
      float pre[3] = {0.f, 0.f, 0.f};
      PH_END(1, ph_su)
      PH_BEGIN(ph_ra)
      LobeTerms lobe;
      if (use) {
        radiance_lobe_terms(sv.app + GSX_APP_F4 * p, Y, rr.df, gC, pre, lobe);
      } else {
#pragma unroll
        for (int l = 0; l < 7; ++l) lobe.w[l] = lobe.c[l] = lobe.v[l] = lobe.g[l] = 0.f;
      }
      PH_END(2, ph_ra)
      PH_BEGIN(ph_mo)
      const float gcl = gC[0] * fmaxf(pre[0], 0.f) + gC[1] * fmaxf(pre[1], 0.f) +
                        gC[2] * fmaxf(pre[2], 0.f);
      float m0 = 0.f, m1 = 0.f, m2 = 0.f, e0 = 0.f;
      if (use) {
        const float nkl2 = -cs.kl2;
        const float* wo = pb.wh + src;
        const float* hp = pb.wh + 512 + src;
        for (int j = jlo; j <= jhi; ++j) {
          const float del = fmaf((float)j, dtf, cs.del0);
          const float q = fmaf(cs.A * del, del, cs.qmin);
          if (q <= 1.0f) {
            const float dens = ex2_approx(fmaf(nkl2, q, cs.lsig));
            const float w = wo[32 * j];
            const float G = fmaf(w, gcl, hp[32 * j]) * dens;
            m0 += G;  // moments in del = t_j - t_c (see grad_candidate)
            m1 = fmaf(G, del, m1);
            m2 = fmaf(G * del, del, m2);
            e0 = fmaf(w, dens, e0);
          }
        }
      }
      float gpc[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) gpc[c] = (use && pre[c] > 0.f) ? gC[c] * e0 : 0.f;
      float* col = pb.pr + lane;
      float* const gb_bat = gb.bat;
      const int nb = gb.n;

      PH_END(3, ph_mo)
      PH_BEGIN(ph_p1)
      // ---- P1: geometry moments + SH 0-21
      {
        const float4 g0 = __ldg(sv.geo + 4 * p);
        const float* d = rr.df;
        const float tcu = use ? cs.tc : 0.f;
        const float v0[3] = {fmaf(d[0], tcu, (base.hi[0] - g0.x) + base.lo[0]),
                             fmaf(d[1], tcu, (base.hi[1] - g0.y) + base.lo[1]),
                             fmaf(d[2], tcu, (base.hi[2] - g0.z) + base.lo[2])};
        col[0] = m0;
#pragma unroll
        for (int a = 0; a < 3; ++a) col[(1 + a) * PR_ROW] = fmaf(v0[a], m0, d[a] * m1);
        const int ia[6] = {0, 1, 2, 0, 0, 1}, ib[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
        for (int q = 0; q < 6; ++q) {
          const float va = v0[ia[q]], vb = v0[ib[q]], da = d[ia[q]], db = d[ib[q]];
          col[(4 + q) * PR_ROW] = fmaf(va * vb, m0, fmaf(fmaf(va, db, da * vb), m1, da * db * m2));
        }
#pragma unroll
        for (int idx = 0; idx < 22; ++idx) col[(10 + idx) * PR_ROW] = Y[idx / 3] * gpc[idx % 3];
      }
      pair_reduce(pb, ends, pe, 32, [&](int row, float sum, int64_t ps, int run) {
        float* brow = gb_bat + (nb + run) * BAT_ROW;
        if (row < 10) {
          brow[row] = sum;
          if (row == 0) brow[31] = __int_as_float((int)ps);
        } else if (sum != 0.f) {
          atomicAdd(grad + (int64_t)GSX_NREC * ps + 11 + (row - 10), sum);
        }
      });

      PH_END(4, ph_p1)
      PH_BEGIN(ph_p2)
      // ---- P2 / P3: spherical-Gaussian lobes (+ the last 5 SH values in P3),
      // from the lobe terms of the radiance pass (zero when !use: e0 = gpc = 0)
#pragma unroll
      for (int pass = 0; pass < 2; ++pass) {
        const int lb0 = pass == 0 ? 0 : 4, nl = pass == 0 ? 4 : 3, r0 = pass == 0 ? 0 : 5;
        if (pass == 1) {
#pragma unroll
          for (int idx = 22; idx < 27; ++idx) col[(idx - 22) * PR_ROW] = Y[idx / 3] * gpc[idx % 3];
        }
        PH_BEGIN(ph_lc)
#pragma unroll
        for (int l = lb0; l < lb0 + nl; ++l) {
          float* c = col + (r0 + 7 * (l - lb0)) * PR_ROW;
          const float ga = lobe.g[l] * e0, f = lobe.w[l] * ga;
          c[0] = f * rr.df[0];
          c[PR_ROW] = f * rr.df[1];
          c[2 * PR_ROW] = f * rr.df[2];
          c[3 * PR_ROW] = lobe.c[l] * ga;
          c[4 * PR_ROW] = lobe.v[l] * gpc[0];
          c[5 * PR_ROW] = lobe.v[l] * gpc[1];
          c[6 * PR_ROW] = lobe.v[l] * gpc[2];
        }
        PH_END(10, ph_lc)
        PH_BEGIN(ph_lr)
        pair_reduce(pb, ends, pe, r0 + 7 * nl, [&](int row, float sum, int64_t ps, int run) {
          if (row < r0) {
            if (sum != 0.f) atomicAdd(grad + (int64_t)GSX_NREC * ps + 11 + 22 + row, sum);
            return;
          }
          const int l = lb0 + (row - r0) / 7, k = (row - r0) % 7;
          if (k < 3)
            gb_bat[(nb + run) * BAT_ROW + 10 + 3 * l + k] = sum;
          else if (sum != 0.f)
            atomicAdd(grad + (int64_t)GSX_NREC * ps + (k == 3 ? 59 + l : 66 + 3 * l + (k - 4)),
                      sum);
        });
        PH_END(11, ph_lr)
      }
      PH_END(5, ph_p2)
      PH_CNT(9, 1)
      gb.n = nb + nrun;
    }
  }
}

// Per-pixel adjoint inputs from the saved frame outputs.
struct BwdImages {
  const float *rgb, *depth, *trans, *dL_drgb, *dL_ddepth, *dL_dtrans;
};
__device__ inline PixelGrad pixel_grad(const BwdImages& im, const gsx_render_cfg& cfg, bool valid,
                                       int64_t pix) {
  PixelGrad pg;
  if (!valid) return PixelGrad{{0.f, 0.f, 0.f}, 0.f, 0.f, {0.f, 0.f, 0.f}, 0.f, 1.f};
  pg.Tend = im.trans[pix];
  pg.Dtot = im.depth[pix];
  pg.gD = im.dL_ddepth ? im.dL_ddepth[pix] : 0.f;
  float gTe = im.dL_dtrans ? im.dL_dtrans[pix] : 0.f;
  for (int k = 0; k < 3; ++k) {
    pg.gC[k] = im.dL_drgb[3 * pix + k];
    pg.Ctot[k] = im.rgb[3 * pix + k] - pg.Tend * (float)cfg.background[k];
    gTe = fmaf(pg.gC[k], (float)cfg.background[k], gTe);
  }
  pg.gTe = gTe;
  return pg;
}

// Pixel of this thread (16x16 tiles, Z-order inside the tile) and its ray;
// lanes without a ray get a benign direction (their values are all masked).
__device__ inline bool tile_pixel_ray(const SceneView& sv, const gsx_camera& cam,
                                      int64_t tile_begin, int64_t tile_stride, int per_tile,
                                      int threads, RayCtx& r, bool& hit, int64_t& pix) {
  const int64_t W = cam.width, H = cam.height;
  const int64_t tiles_x = (W + 15) / 16;
  const int64_t tile = gsx_tile_at(tile_begin + (int64_t)(blockIdx.x / per_tile) * tile_stride,
                                   tiles_x, (H + 15) / 16, tile_stride);
  int mx, my;
  morton_decode8((blockIdx.x % per_tile) * threads + threadIdx.x, mx, my);
  const int64_t px = (tile % tiles_x) * 16 + mx, py = (tile / tiles_x) * 16 + my;
  const bool valid = px < W && py < H;
  hit = valid && camera_ray(cam, (double)px, (double)py, sv.bounds, r);
  if (!hit) {
    for (int k = 0; k < 3; ++k) {
      r.o[k] = 0.0;
      r.d[k] = k == 2 ? 1.0 : 0.0;
      r.of[k] = 0.f;
      r.df[k] = k == 2 ? 1.f : 0.f;
    }
  }
  pix = valid ? py * W + px : 0;
  return valid;
}

// Replay backward: CTA = BWD_THREADS rays = 256 / BWD_THREADS CTAs per tile.
// With `skip` (a march log's complete flags) it only handles the warps the
// log does not cover.
#ifndef GSX_BWD_THREADS
#define GSX_BWD_THREADS 256
#endif
#ifndef GSX_BWD_MINB
#define GSX_BWD_MINB 1
#endif
constexpr int BWD_THREADS = GSX_BWD_THREADS;
constexpr int BWD_PER_TILE = 256 / BWD_THREADS;

__global__ void __launch_bounds__(BWD_THREADS, GSX_BWD_MINB)
    k_render_backward(SceneView sv, BvhView bv, gsx_camera cam, gsx_render_cfg cfg,
                      int64_t tile_begin, int64_t tile_stride, BwdImages im,
                      const unsigned* __restrict__ skip, float* __restrict__ grad) {
  __shared__ WarpSmem smem[BWD_THREADS / 32];
  extern __shared__ __align__(16) float red_smem[];  // BWD_WARP_FLOATS per warp
  if (skip && skip[tile_warp_id(BWD_PER_TILE, BWD_THREADS)]) return;  // warp-uniform
  RayCtx r;
  bool hit;
  int64_t pix;
  const bool valid =
      tile_pixel_ray(sv, cam, tile_begin, tile_stride, BWD_PER_TILE, BWD_THREADS, r, hit, pix);
  const PixelGrad pg = pixel_grad(im, cfg, valid, pix);
  RayAccum acc;
  acc.init();
  float Y[9];
  sh_basis_f(r.df, Y);
  Counters<false> cnt;
  const int ns = (int)cfg.n_s;
  WarpSmem& sm = smem[threadIdx.x >> 5];
  float* wsm = red_smem + (threadIdx.x >> 5) * BWD_WARP_FLOATS;
  GradBatch gb{wsm, wsm + RED_FLOATS, 0};
  ovf_begin(sm);
  march_warp<false>(sv, bv, r, hit, cfg, acc, cnt, GSX_SYNC_BWD, sm, [&](const Seg& seg, bool want) {
    return backward_segment(sv, bv, r, want, seg, ns, Y, acc, pg, cnt, sm, gb, grad);
  });
  ovf_report(sm, bv, pix);
  grad_batch_flush(sv, gb, grad);
}

// Logged backward: walks the warp's march-log chain (march_log.cuh).  Per
// record: replay the compositing from the saved sums to form the adjoints,
// then pass 2 over the saved candidate stream.  Warp layout = the forward's
// (FWD_THREADS-thread CTAs, Z-order 8x4 blocks), so the records line up.
#ifndef GSX_BWD_LDGRP
#define GSX_BWD_LDGRP 1
#endif
// Two pass-2 strategies over the same records (one launch each; the log's
// pair statistics pick one on the device, the other kernel's warps return at
// once -- no host synchronization):
//   PAIRS   (64-thread CTAs x 7): the pair batches above;
//   entries (128-thread CTAs x 4): all 32 lanes per list entry
//           (grad_candidate), the better choice when most lanes use most
//           entries.  C2 (14.1 lanes per entry) 12.6 vs 13.4 ms; C4 (7.7)
//           26.5 vs 17.3 ms.
#ifndef GSX_BWDL_PAIR_MAX  // mean lanes per entry (x 1/16) below which PAIRS runs
#define GSX_BWDL_PAIR_MAX 192
#endif
template <bool PAIRS>
struct BwdlShape;
#ifndef GSX_BWDP_THREADS
#define GSX_BWDP_THREADS 128
#endif
#ifndef GSX_BWDP_MINB
#define GSX_BWDP_MINB 3
#endif
template <>
struct BwdlShape<true> {
  static constexpr int threads = GSX_BWDP_THREADS, minb = GSX_BWDP_MINB,
                       warp_floats = PAIR_WARP_FLOATS;
  static_assert(256 % threads == 0, "a 256-pixel tile must split into whole CTAs");
};
// entries path: + two staged appearance blocks and their barriers per warp
constexpr int ENTRY_TMA_FLOATS = 2 * 4 * GSX_APP_F4 + 8;
static_assert((BWD_WARP_FLOATS + ENTRY_TMA_FLOATS) % 4 == 0, "16-byte aligned warp regions");
// (the pair path stays on plain loads: staging its batches' first 2 / 4
// runs by TMA measured 18.37 / 19.54 vs 18.40 ms at C4 -- the buffers cost
// occupancy and the runs are short)
template <>
struct BwdlShape<false> {
  static constexpr int threads = 128, minb = 4, warp_floats = BWD_WARP_FLOATS + ENTRY_TMA_FLOATS;
};
__device__ inline bool log_wants_pairs(const char* log, const gsx_render_cfg& cfg) {
  if (cfg.pass2 != 0) return cfg.pass2 == 1;
  const LogHeader* h = (const LogHeader*)log;
  return 16ull * h->pairs < (unsigned long long)GSX_BWDL_PAIR_MAX * h->entries;
}

template <bool PAIRS>
__global__ void __launch_bounds__(BwdlShape<PAIRS>::threads, BwdlShape<PAIRS>::minb)
    k_render_backward_logged(SceneView sv, gsx_camera cam, gsx_render_cfg cfg, int64_t tile_begin,
                             int64_t tile_stride, BwdImages im, const char* __restrict__ log,
                             long long nw, float* __restrict__ grad) {
  constexpr int NT = BwdlShape<PAIRS>::threads, PER_TILE = 256 / NT;
  extern __shared__ __align__(16) float red_smem[];  // BwdlShape::warp_floats per warp
  if (log_wants_pairs(log, cfg) != PAIRS) return;  // the other strategy's launch runs
  const long long wid = tile_warp_id(PER_TILE, NT);
  if (!log_complete((void*)log, nw)[wid]) return;  // the replay kernel covers this warp
  const int lane = threadIdx.x & 31;
  RayCtx r;
  bool hit;
  int64_t pix;
  const bool valid = tile_pixel_ray(sv, cam, tile_begin, tile_stride, PER_TILE, NT, r, hit, pix);
  const PixelGrad pg = pixel_grad(im, cfg, valid, pix);
  RayAccum acc;
  acc.init();
  float* wsm = red_smem + (threadIdx.x >> 5) * BwdlShape<PAIRS>::warp_floats;
  const PairBufs pb{wsm, wsm + PR_FLOATS, wsm + PR_FLOATS + WH_FLOATS};
  GradBatch gb = PAIRS ? GradBatch{nullptr, wsm + PR_FLOATS + WH_FLOATS + LT_ROWS * 32, 0}
                       : GradBatch{wsm, wsm + RED_FLOATS, 0};
  float Y[PAIRS ? 1 : 9];
  if constexpr (!PAIRS) sh_basis_f(r.df, Y);
  // entries path: each entry's appearance block is staged by a TMA bulk copy
  // one entry ahead (as in the screened forward, render_warp.cuh app_issue)
  float4* appb = (float4*)(wsm + BWD_WARP_FLOATS);  // [2][GSX_APP_F4]
  unsigned long long* abar = (unsigned long long*)(appb + 2 * GSX_APP_F4);
  unsigned apar = 0u;
  if constexpr (!PAIRS) {
    if (lane == 0) {
      tma_bar_init(&abar[0]);
      tma_bar_init(&abar[1]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  long long off = log_first((void*)log)[wid];
  while (off >= 0) {
    const long long start = off;
    const LogRec* h = (const LogRec*)(log + off);
    while (h->kind != 0) {
      off = h->next;
      h = (const LogRec*)(log + off);
    }
    const char* body = log + off + 128;
    const unsigned act = h->act;
    const int mmax = h->mmax;
    const long long next = h->next;
    const int sw = h->swidth ? h->swidth : __popc(act);  // sample-sum columns
    const LogLayout Lo(__popc(act), mmax, h->cap, sw);
    if (next >= 0) log_prefetch(log + next, 128 + Lo.list);
    const bool mine = (act >> lane) & 1u;
    const int slot = __popc(act & ((1u << lane) - 1u));
    double tb = 0.0, dt = 0.0;
    int mc = 0;
    if (mine) {
      tb = __ldcs((const double*)body + slot);
      dt = __ldcs((const double*)(body + Lo.dt) + slot);
      mc = __ldcs((const int*)(body + Lo.mc) + slot);
    }
    PH_BEGIN(ph_pro)
    const float4* smp = (const float4*)(body + Lo.smp) + (h->swidth ? lane : slot);
    const int nact = sw;  // the sample array's row stride
    const float dtf = (float)dt;
    float wos[16], hh[16];
#if GSX_BWD_LDGRP
    // the saved sums in groups of 4 samples: the 4 loads issue before the
    // first adjoint needs one (the adjoint chain is sequential)
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      float4 v[4];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = 4 * g + jj;
        wos[j] = hh[j] = 0.f;
        v[jj] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < mmax && j < mc) v[jj] = __ldcs(smp + (long long)j * nact);
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = 4 * g + jj;
        if (j < mmax && j < mc) {
          const float Wj[3] = {v[jj].y, v[jj].z, v[jj].w};
          sample_adjoint(acc, pg, v[jj].x, Wj, (float)(tb + (double)j * dt), dtf, wos[j], hh[j]);
        }
      }
    }
#else
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      wos[j] = hh[j] = 0.f;
      if (j < mmax && j < mc) {
        const float4 v = __ldcs(smp + (long long)j * nact);
        const float Wj[3] = {v.y, v.z, v.w};
        sample_adjoint(acc, pg, v.x, Wj, (float)(tb + (double)j * dt), dtf, wos[j], hh[j]);
      }
    }
#endif
    PH_END(0, ph_pro)
    const SegBase base = seg_base(r, tb);
    if constexpr (PAIRS) {
      // the lane table and adjoints of this record for the pair lanes
      float* lt = pb.lt + lane;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        lt[k * 32] = r.df[k];
        lt[(3 + k) * 32] = base.hi[k];
        lt[(6 + k) * 32] = base.lo[k];
        lt[(11 + k) * 32] = pg.gC[k];
      }
      lt[9 * 32] = dtf;
      lt[10 * 32] = __int_as_float(mc);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        pb.wh[32 * j + lane] = wos[j];
        pb.wh[512 + 32 * j + lane] = hh[j];
      }
      __syncwarp();
    }
    // pass 2 over the record chain start..off
    for (long long o = start;;) {
      const LogRec* ho = (const LogRec*)(log + o);
      const int count = ho->count;
      const char* lb = log + o + 128;
      const int32_t* list = (const int32_t*)(lb + (ho->kind == 0 ? Lo.list : 0));
      const uint32_t* um =
          (const uint32_t*)(lb + (ho->kind == 0 ? Lo.umask : log_chunk_umask(ho->cap)));
      if constexpr (PAIRS) {
        pair_pass(sv, pb, gb, list, um, count, grad);
      } else {
        for (int i0 = 0; i0 < count; i0 += 32) {
          const int ent = i0 + lane < count ? __ldcs(list + i0 + lane) : 0;
          const int nb = min(32, count - i0);
          constexpr unsigned ABYTES = 16u * GSX_APP_F4;
          {
            const int p0 = __shfl_sync(FULL, ent, 0);
            if (lane == 0) tma_copy(appb, sv.app + GSX_APP_F4 * (int64_t)p0, ABYTES, &abar[0]);
          }
          for (int k = 0; k < nb; ++k) {
            const int bk = k & 1;
            const int pn = __shfl_sync(FULL, ent, k + 1 < nb ? k + 1 : k);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (k + 1 < nb && lane == 0)
              tma_copy(appb + GSX_APP_F4 * (bk ^ 1), sv.app + GSX_APP_F4 * (int64_t)pn, ABYTES,
                       &abar[bk ^ 1]);
            bar_wait(&abar[bk], (apar >> bk) & 1u);
            apar ^= 1u << bk;
            grad_candidate<PlainLoad>(sv, r, (int64_t)__shfl_sync(FULL, ent, k), mc > 0, mc,
                                      base, dtf, Y, pg, wos, hh, gb, grad,
                                      appb + GSX_APP_F4 * bk);
          }
        }
      }
      if (o == off) break;
      o = ho->next;
    }
    __syncwarp();
    off = next;
  }
  grad_batch_flush(sv, gb, grad);
}

}  // namespace

#ifdef GSX_PHASE_PROF
extern "C" int gsx_phase_times_bwd(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, gsx::g_phase, sizeof(unsigned long long) * 24);
  if (reset) {
    unsigned long long z[24] = {};
    cudaMemcpyToSymbol(gsx::g_phase, z, sizeof z);
  }
  return gsx_check_launch();
}
#endif

constexpr int BWD_SMEM = (BWD_THREADS / 32) * BWD_WARP_FLOATS * (int)sizeof(float);
template <bool PAIRS>
constexpr int bwdl_smem() {
  return (BwdlShape<PAIRS>::threads / 32) * BwdlShape<PAIRS>::warp_floats * (int)sizeof(float);
}

static int bwd_smem_setup() {
  static bool done = false;  // idempotent; the attribute is per function
  if (done) return GSX_OK;
  if (cudaFuncSetAttribute(k_render_backward, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           BWD_SMEM) != cudaSuccess ||
      cudaFuncSetAttribute(k_render_backward_logged<true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           bwdl_smem<true>()) != cudaSuccess ||
      cudaFuncSetAttribute(k_render_backward_logged<false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           bwdl_smem<false>()) != cudaSuccess)
    return gsx_check_launch();
  done = true;
  return GSX_OK;
}

static int bwd_check(const gsx_render_cfg* cfg, const gsx_camera* cam, int64_t n,
                     const BwdImages& im, const float* grad, int64_t tile_begin,
                     int64_t tile_stride) {
  int rc = gsx_validate_cfg(cfg);
  if (rc) return rc;
  if (!cam || cam->width < 1 || cam->height < 1 || !(cam->focal > 0)) return GSX_ERR_ARG;
  if (n <= 0) return GSX_ERR_EMPTY;
  if (!im.rgb || !im.depth || !im.trans || !im.dL_drgb || !grad) return GSX_ERR_ARG;
  if (tile_stride < 1 || tile_begin < 0) return GSX_ERR_ARG;
  return GSX_OK;
}

extern "C" int gsx_render_backward(const void* scene_arena, const void* bvh_arena,
                                   const float* params, int64_t n, const gsx_camera* cam,
                                   const gsx_render_cfg* cfg, int64_t tile_begin,
                                   int64_t tile_stride, const float* rgb, const float* depth,
                                   const float* trans, const float* dL_drgb,
                                   const float* dL_ddepth, const float* dL_dtrans, float* grad,
                                   gsx_dev_status* dev_status, void* stream) {
  (void)params;
  const BwdImages im{rgb, depth, trans, dL_drgb, dL_ddepth, dL_dtrans};
  int rc = bwd_check(cfg, cam, n, im, grad, tile_begin, tile_stride);
  if (rc) return rc;
  int64_t tiles = ((cam->width + 15) / 16) * ((cam->height + 15) / 16);
  if (tile_begin >= tiles) return GSX_OK;
  int64_t blocks = BWD_PER_TILE * ((tiles - tile_begin + tile_stride - 1) / tile_stride);
  SceneView sv = scene_view((void*)scene_arena, n);
  BvhView bv = bvh_view((void*)bvh_arena, n);
  bv.status = dev_status;
  rc = bwd_smem_setup();
  if (rc) return rc;
  k_render_backward<<<(unsigned)blocks, BWD_THREADS, BWD_SMEM, (cudaStream_t)stream>>>(
      sv, bv, *cam, *cfg, tile_begin, tile_stride, im, nullptr, grad);
  return gsx_check_launch();
}

extern "C" int gsx_render_backward_logged(const void* scene_arena, const void* bvh_arena,
                                          const float* params, int64_t n, const gsx_camera* cam,
                                          const gsx_render_cfg* cfg, int64_t tile_begin,
                                          int64_t tile_stride, const float* rgb,
                                          const float* depth, const float* trans,
                                          const float* dL_drgb, const float* dL_ddepth,
                                          const float* dL_dtrans, const void* log, float* grad,
                                          gsx_dev_status* dev_status, void* stream) {
  (void)params;
  const BwdImages im{rgb, depth, trans, dL_drgb, dL_ddepth, dL_dtrans};
  int rc = bwd_check(cfg, cam, n, im, grad, tile_begin, tile_stride);
  if (rc) return rc;
  if (!log) return GSX_ERR_ARG;
  int64_t tiles = ((cam->width + 15) / 16) * ((cam->height + 15) / 16);
  if (tile_begin >= tiles) return GSX_OK;
  const int64_t ntl = (tiles - tile_begin + tile_stride - 1) / tile_stride;
  const long long nw = 8 * ntl;
  SceneView sv = scene_view((void*)scene_arena, n);
  BvhView bv = bvh_view((void*)bvh_arena, n);
  bv.status = dev_status;
  cudaStream_t s = (cudaStream_t)stream;
  rc = bwd_smem_setup();
  if (rc) return rc;
  k_render_backward_logged<true><<<(unsigned)(256 / BwdlShape<true>::threads * ntl),
                                   BwdlShape<true>::threads, bwdl_smem<true>(), s>>>(
      sv, *cam, *cfg, tile_begin, tile_stride, im, (const char*)log, nw, grad);
  k_render_backward_logged<false><<<(unsigned)(256 / BwdlShape<false>::threads * ntl),
                                    BwdlShape<false>::threads, bwdl_smem<false>(), s>>>(
      sv, *cam, *cfg, tile_begin, tile_stride, im, (const char*)log, nw, grad);
  // warps whose records overflowed the arena: full replay
  k_render_backward<<<(unsigned)(BWD_PER_TILE * ntl), BWD_THREADS, BWD_SMEM, s>>>(
      sv, bv, *cam, *cfg, tile_begin, tile_stride, im, log_complete((void*)log, nw), grad);
  return gsx_check_launch();
}
