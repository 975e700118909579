// EXPERIMENT (not compiled into libgsx): two forward list-processing variants
// measured slower than the plain per-entry loop and removed from
// render_warp.cuh.  Kept for reference with their numbers (one B200, same box):
//   * exact silhouette screen of the packet-cone list: C3 34.3-35.1 ms vs
//     31.2, C2 19.7-20.0 vs 15.9 -- 15% fewer instructions but the larger
//     hot loop stalls on the instruction cache (ncu no_instruction 5.3 vs 0.8
//     warps per issue);
//   * cp.async double-buffered staging of candidate geometry + appearance in
//     shared memory: C3 35.5 vs 32.9 ms, C2 19.7 vs 18.3.
// They used these WarpSmem members: float4 pre[64]; float4 camc[3];
// float2 uv[32] (screen) and float4 stage[2][N * 27] (staging).

// Pass 1 over a cone-staged list (camera rays).  The cone list is a loose
// superset -- most entries meet no lane's segment -- so every entry is first
// screened per lane by the exact silhouette of its ellipsoid seen from the
// camera centre, in image-plane coordinates z = (u, v) (the lane's pixel:
// u = (px + 0.5 - W/2) / f): the line o + s R (u, v, 1) meets the ellipsoid
// iff (z - z*)^T Hn (z - z*) <= 1.  The 32 entries of a group are prepared
// entry-parallel (prep_silhouette), then each lane tests its pixel in ~10
// instructions instead of the ~60 of the full density setup, plus a depth
// test against the ellipsoid's bounding sphere.  Only passing lanes run the
// exact setup (candidate_use) and the exact AABB test; entries no lane passes
// cost nothing else.  The screen is conservative (tolerances well above its
// fp32 rounding; near or degenerate views pass everything), so the sums are
// those of the unscreened list.  Lanes the screen leaves without an exact
// overlap get `fallback` (the unscreened exact test) after the stream.
//
// Silhouette (per entry, fp32): y0 = M (o - mu), rho = |y0|, unit-sphere frame
// of the ellipsoid.  A direction w hits iff (rho^2 - 1) |P w~|^2 <= (y0^ . w~)^2
// with w~ = M w and P the projector orthogonal to y0.  Expanding about the
// direction to mu, z_c = (R^T (mu - o)).xy / (R^T (mu - o)).z, where
// P M R (z_c, 1) = 0 exactly: with N_j = M R_j (camera columns j = 0, 1),
// alpha_j = y0^ . N_j, A_j = P N_j, alpha_c = -rho / pz and D = z - z_c,
//   f(D) = D^T H D - 2 alpha_c beta.D - alpha_c^2 <= 0,
//   H = (rho^2 - 1) [A_i . A_j] - beta beta^T,  beta = (alpha_0, alpha_1),
// i.e. (D - D*)^T H (D - D*) <= alpha_c^2 (1 + beta^T H^-1 beta) with
// D* = alpha_c H^-1 beta.  No term cancels beyond O(1) (the expansion point
// removes the rho^2 cancellation of the textbook discriminant).
struct Silhouette {
  float4 c;  // (centre u, centre v, dmin, dmax)
  float4 h;  // (Hn00, 2 Hn01, Hn11, limit)
};
__device__ inline Silhouette prep_silhouette(const SceneView& sv, int64_t p, const float4& o,
                                             const float4* camc) {
  const float4 g0 = __ldg(sv.geo + 4 * p), g1 = __ldg(sv.geo + 4 * p + 1),
               g2 = __ldg(sv.geo + 4 * p + 2), g3 = __ldg(sv.geo + 4 * p + 3);
  const float px = o.x - g0.x, py = o.y - g0.y, pz = o.z - g0.z;  // o - mu
  const float dist = sqrtf(fmaf(px, px, fmaf(py, py, pz * pz)));
  const float n1 = fmaf(g1.x, g1.x, fmaf(g1.y, g1.y, g1.z * g1.z));
  const float n2 = fmaf(g2.x, g2.x, fmaf(g2.y, g2.y, g2.z * g2.z));
  const float n3 = fmaf(g3.x, g3.x, fmaf(g3.y, g3.y, g3.z * g3.z));
  // largest semi-axis + rounding margins -> distance range of the ellipsoid
  const float rad = fmaf(rsqrtf(fminf(fminf(n1, n2), n3)), 1.0001f,
                         1e-6f * (dist + fabsf(o.x) + fabsf(o.y) + fabsf(o.z)));
  Silhouette s;
  s.c = make_float4(0.f, 0.f, dist - rad, dist + rad);
  s.h = make_float4(0.f, 0.f, 0.f, 1.f);  // pass-all
  const float y0x = fmaf(g1.x, px, fmaf(g1.y, py, g1.z * pz));
  const float y0y = fmaf(g2.x, px, fmaf(g2.y, py, g2.z * pz));
  const float y0z = fmaf(g3.x, px, fmaf(g3.y, py, g3.z * pz));
  const float rho2 = fmaf(y0x, y0x, fmaf(y0y, y0y, y0z * y0z));
  // camera-frame coordinates of mu - o
  const float4 R0 = camc[0], R1 = camc[1], R2 = camc[2];
  const float qx = -fmaf(R0.x, px, fmaf(R0.y, py, R0.z * pz));
  const float qy = -fmaf(R1.x, px, fmaf(R1.y, py, R1.z * pz));
  const float qz = -fmaf(R2.x, px, fmaf(R2.y, py, R2.z * pz));
  // near / inside the ellipsoid, beside or behind the image plane, or so far
  // that fp32 cannot resolve the silhouette: no screening
  if (!(rho2 > 1.02f && rho2 < 1e9f && qz > 1e-3f * dist)) return s;
  const float irho = rsqrtf(rho2);
  const float ux = y0x * irho, uy = y0y * irho, uz = y0z * irho;
  // N_j = M R_j
  const float a0x = fmaf(g1.x, R0.x, fmaf(g1.y, R0.y, g1.z * R0.z));
  const float a0y = fmaf(g2.x, R0.x, fmaf(g2.y, R0.y, g2.z * R0.z));
  const float a0z = fmaf(g3.x, R0.x, fmaf(g3.y, R0.y, g3.z * R0.z));
  const float a1x = fmaf(g1.x, R1.x, fmaf(g1.y, R1.y, g1.z * R1.z));
  const float a1y = fmaf(g2.x, R1.x, fmaf(g2.y, R1.y, g2.z * R1.z));
  const float a1z = fmaf(g3.x, R1.x, fmaf(g3.y, R1.y, g3.z * R1.z));
  const float al0 = fmaf(ux, a0x, fmaf(uy, a0y, uz * a0z));
  const float al1 = fmaf(ux, a1x, fmaf(uy, a1y, uz * a1z));
  // A_j = P N_j
  const float b0x = fmaf(-al0, ux, a0x), b0y = fmaf(-al0, uy, a0y), b0z = fmaf(-al0, uz, a0z);
  const float b1x = fmaf(-al1, ux, a1x), b1y = fmaf(-al1, uy, a1y), b1z = fmaf(-al1, uz, a1z);
  const float k = rho2 - 1.f;
  const float h00 = fmaf(k, fmaf(b0x, b0x, fmaf(b0y, b0y, b0z * b0z)), -al0 * al0);
  const float h01 = fmaf(k, fmaf(b0x, b1x, fmaf(b0y, b1y, b0z * b1z)), -al0 * al1);
  const float h11 = fmaf(k, fmaf(b1x, b1x, fmaf(b1y, b1y, b1z * b1z)), -al1 * al1);
  const float det = fmaf(h00, h11, -h01 * h01);
  if (!(h00 > 0.f && det > 1e-6f * h00 * h11)) return s;  // not a bounded ellipse
  const float idet = 1.f / det;
  const float alc = -sqrtf(rho2) / qz;  // y0^ . M R (z_c, 1) = y0^ . M (mu - o) / qz
  // H^-1 beta
  const float i0 = (h11 * al0 - h01 * al1) * idet, i1 = (h00 * al1 - h01 * al0) * idet;
  const float D = alc * alc * (1.f + fmaf(al0, i0, al1 * i1));
  if (!(D > 0.f)) return s;
  const float iD = 1.f / D;
  const float iqz = 1.f / qz;
  const float cu = fmaf(alc, i0, qx * iqz), cv = fmaf(alc, i1, qy * iqz);
  const float e00 = h00 * iD, e01 = h01 * iD, e11 = h11 * iD;
  // tolerance: 2% + a 4e-6 error in the image-plane coordinates
  const float lim = 1.02f + 8e-6f * sqrtf(e00 + e11);
  s.c.x = cu;
  s.c.y = cv;
  s.h = make_float4(e00, 2.f * e01, e11, lim);
  return s;
}

#if GSX_SCREEN_SMEM
template <class Pre, int CH, class YT>
__device__ inline void accumulate_list_cone(const SceneView& sv, const RayCtx& r, WarpSmem& sm,
                                            int count, bool want, int mc, float lo_t, float hi_t,
                                            const SegBase& base, float dtf, YT Y,
                                            float (&sig)[CH], float (&W)[CH][3], Pre&& pre) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned a_pre = (unsigned)__cvta_generic_to_shared(sm.pre);
  const float2 uv = sm.uv[lane];
  for (int g = 0; g < count; g += 32) {
    {
      const int e = g + (int)lane;
      const int64_t p = e < count ? (int64_t)sm.list[e] : 0;
      const Silhouette S = prep_silhouette(sv, p, sm.cone[0], sm.camc);
      sm.pre[lane] = S.c;
      sm.pre[32 + lane] = S.h;
    }
    __syncwarp();
    const int ng = count - g < 32 ? count - g : 32;
#if GSX_SCREEN2
    // screen the whole group first (independent tests, no votes), then visit
    // only the entries some lane passes
    unsigned mine = 0;
#pragma unroll 4
    for (int i = 0; i < ng; ++i) {
      const float4 C = lds4(a_pre + 16u * (unsigned)i);
      const float4 H = lds4(a_pre + 16u * (unsigned)(32 + i));
      const float du = uv.x - C.x, dv = uv.y - C.y;
      const float q = fmaf(du, fmaf(H.x, du, H.y * dv), H.z * dv * dv);
      const bool pass = want && q <= H.w && C.z <= hi_t && C.w >= lo_t;
      mine |= (pass ? 1u : 0u) << i;
    }
    PH_CNT(12, ng)
    unsigned any = __reduce_or_sync(FULL, mine);
    while (any) {
      const int i = __ffs(any) - 1;
      any &= any - 1;
      const bool pass = (mine >> i) & 1u;
      const int64_t p = sm.list[g + i];
      pre(p, pass);
      CandUse u = candidate_use(sv, r, p, pass, mc, base, dtf);
      accumulate_used(sv, r, p, u, dtf, Y, sig, W);
    }
#else
    for (int i = 0; i < ng; ++i) {
      const float4 C = lds4(a_pre + 16u * (unsigned)i);
      const float4 H = lds4(a_pre + 16u * (unsigned)(32 + i));
      const float du = uv.x - C.x, dv = uv.y - C.y;
      const float q = fmaf(du, fmaf(H.x, du, H.y * dv), H.z * dv * dv);
      const bool pass = want && q <= H.w && C.z <= hi_t && C.w >= lo_t;
      PH_CNT(12, 1)
      if (!__any_sync(FULL, pass)) continue;
      const int64_t p = sm.list[g + i];
      pre(p, pass);
      CandUse u = candidate_use(sv, r, p, pass, mc, base, dtf);
      accumulate_used(sv, r, p, u, dtf, Y, sig, W);
    }
#endif
    __syncwarp();
  }
}

#endif  // GSX_SCREEN_SMEM

#if GSX_STAGE_N > 0
__device__ inline void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem_dst)),
               "l"(gsrc)
               : "memory");
}
__device__ inline void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ inline void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Pass 1 over a staged list with the candidates' geometry and appearance
// (27 float4 = 432 B each) copied into shared memory GSX_STAGE_N entries at a
// time, double-buffered with cp.async: the copies of the next group are in
// flight (all 32 lanes, coalesced 16-byte pieces, L2 -> shared without
// registers) while the current group is evaluated from shared memory, so the
// per-entry chain no longer waits on two dependent L2 round trips (the list
// index -> geometry -> setup -> appearance).  Same arithmetic, same order.
template <class Pre, int CH, class YT>
__device__ inline void accumulate_list_staged(const SceneView& sv, const RayCtx& r, WarpSmem& sm,
                                              int count, bool want, int mc, const SegBase& base,
                                              float dtf, YT Y, float (&sig)[CH],
                                              float (&W)[CH][3], Pre&& pre) {
  constexpr int NS = GSX_STAGE_N;
  const int lane = (int)(threadIdx.x & 31);
  auto issue = [&](int b, int g0) {
    const int n = count - g0 < NS ? count - g0 : NS;
    for (int k = lane; k < n * STAGE_F4; k += 32) {
      const int e = k / STAGE_F4, j = k - e * STAGE_F4;
      const int64_t p = sm.list[g0 + e];
      const float4* src = j < 4 ? sv.geo + 4 * p + j : sv.app + GSX_APP_F4 * p + (j - 4);
      cp_async16(&sm.stage[b][k], src);
    }
    cp_async_commit();
  };
  if (count <= 0) return;
  issue(0, 0);
  int b = 0;
  for (int g0 = 0; g0 < count; g0 += NS) {
    if (g0 + NS < count) {
      issue(b ^ 1, g0 + NS);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const int n = count - g0 < NS ? count - g0 : NS;
    for (int e = 0; e < n; ++e) {
      const int64_t p = sm.list[g0 + e];
      pre(p, want);
      const float4* st = sm.stage[b] + e * STAGE_F4;
      const CandUse u = candidate_use_at<SmemLoad>(st, r, want, mc, base, dtf);
      accumulate_used_at<SmemLoad>(st + 4, r, u, dtf, Y, sig, W);
    }
    __syncwarp();
    b ^= 1;
  }
}
#endif  // GSX_STAGE_N

// ---------------------------------------------------------------------------
// Ellipsoid-vs-cone leaf filter (box-only leaves kept for the exact AABB
// emptiness test only): halves the list (139.6 -> 69.4 entries per warp
// iteration on C3) but C3 31.3 vs 30.9 ms, C2 16.8 vs 15.6 ms (fp32 exact
// test in both) -- in the traversal loop the gathers sit on its dependency
// chain (C3 32.9), entry-parallel the extra code costs instruction-cache
// misses (ncu no_instruction 4.2 vs 0.9 warps per issue).  Needed a per-
// primitive float4[2] (Sigma = R S~^2 R^T, r_max) computed in gsx_prepare.
// Does the truncation ellipsoid of a leaf meet the cone?  Plane p through o
// with normal n: max over the ellipsoid of n.(x - o) = n.(mu - o) +
// sqrt(n^T Sigma n); distance shell by the bounding sphere (r_max).  Margins:
// 1e-4 relative on the radius term (Sigma is the fp32 rounding of the form
// whose inverse the renderer's fp32 M approximates) and 1e-6 (|mu - o| +
// eps_scale) absolute.  Leaves whose box meets the cone but whose ellipsoid
// does not can hold no sample (q <= 1 implies inside the ellipsoid), but
// their AABB still counts for the reference's emptiness: they are listed
// with the BOX_ONLY flag and only take part in the exact AABB test.
constexpr int32_t BOX_ONLY = (int32_t)0x80000000;
__device__ inline bool cone_ellipsoid(unsigned a_cone, const float4& g0, const float4& e0,
                                      const float4& e1) {
  const float4 c0 = lds4(a_cone);
  const float4 p1 = lds4(a_cone + 16u), p2 = lds4(a_cone + 32u), p3 = lds4(a_cone + 48u),
               p4 = lds4(a_cone + 64u);
  const float vx = g0.x - c0.x, vy = g0.y - c0.y, vz = g0.z - c0.z;
  const float d = sqrtf(fmaf(vx, vx, fmaf(vy, vy, vz * vz)));
  const float m = 1e-6f * (d + p2.w);
  const float rm = fmaf(e0.w, 1.0001f, 2.f * m);
  bool ok = d - rm <= p4.w && d + rm >= p3.w;
  const float4 pl[4] = {p1, p2, p3, p4};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float nx = pl[k].x, ny = pl[k].y, nz = pl[k].z;
    const float q = fmaf(nx, fmaf(e0.x, nx, 2.f * fmaf(e0.y, ny, e0.z * nz)),
                         fmaf(ny, fmaf(e1.x, ny, 2.f * e1.y * nz), e1.z * nz * nz));
    const float s = fmaf(nx, vx, fmaf(ny, vy, nz * vz)) +
                    fmaf(sqrtf(fmaxf(q, 0.f)), 1.0001f, 2.f * m);
    ok = ok && s >= 0.f;
  }
  return ok;
}

// Flag the listed cone leaves whose ellipsoid misses the cone (BOX_ONLY),
// entry-parallel over the list (independent gathers, one lane per entry; in
// the traversal loop the gathers sat on its serial dependency chain).
__device__ inline void cone_flag_box_only(const SceneView& sv, WarpSmem& sm, int count) {
  const unsigned a_cone = (unsigned)__cvta_generic_to_shared(sm.cone);
  for (int e = (int)(threadIdx.x & 31); e < count; e += 32) {
    const int64_t pr = (int64_t)sm.list[e];
    if (!cone_ellipsoid(a_cone, __ldg(sv.geo + 4 * pr), __ldg(sv.ell + 2 * pr),
                        __ldg(sv.ell + 2 * pr + 1)))
      sm.list[e] = (int32_t)pr | BOX_ONLY;
  }
  __syncwarp();
}

