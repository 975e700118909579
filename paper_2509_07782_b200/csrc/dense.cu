// dense.cu -- K13/K14: the reference's dense oracles on the device, float64.
//
//  * gsx_reference_rays: reference_integrate (renderer.py:440-480) per ray, or
//    reference_render's clip + integrate per pixel ray (renderer.py:483-493):
//    midpoint quadrature at fine_dt over the ray's [t_near, t_far] against
//    every primitive (no BVH, no empty-space skipping, no early termination),
//    the vectorised compositing of renderer.py:472-480.
//  * gsx_eval_fields: eval_fields (appearance.py:107-134), the mixture density
//    and density-weighted radiance at points, over all or an `active` subset.
//
// Both restate the reference in float64 from the raw records (the scene
// arena's fp64 iso_inv / log_ratio, the record's mean, sigma~ and appearance
// with lobe axes normalized in fp64 as AppearanceCoeffs does,
// appearance.py:62-68): they are the independent, all-primitive cross-checks
// of the accelerated march (the PSNR acceptance criterion of
// test_acceptance.py:102-133 and the density formula of
// test_appearance.py:102-143), not a render path.
#include "gsx_common.cuh"
#include "render_common.cuh"

namespace {

using namespace gsx;

// appearance.py:26-98 in fp64 from one raw 87-float record (sh at 11,
// axes at 38, sharpness at 59, amplitudes at 66), clamped at 0
__device__ void radiance64(const float* rec, const double* d, double* rgb) {
  const double x = d[0], y = d[1], z = d[2];
  const double Y[9] = {0.28209479177387814, 0.4886025119029199 * y, 0.4886025119029199 * z,
                       0.4886025119029199 * x, 1.0925484305920792 * x * y,
                       1.0925484305920792 * y * z, 0.31539156525252005 * (3.0 * z * z - 1.0),
                       1.0925484305920792 * x * z, 0.5462742152960396 * (x * x - y * y)};
  double acc[3];
  for (int ch = 0; ch < 3; ++ch) {
    double v = 0.0;
    for (int b = 0; b < 9; ++b) v += Y[b] * (double)rec[11 + 3 * b + ch];
    acc[ch] = v;
  }
  double lob[7];
  for (int l = 0; l < 7; ++l) {
    const double a0 = rec[38 + 3 * l], a1 = rec[39 + 3 * l], a2 = rec[40 + 3 * l];
    const double nn = sqrt(a0 * a0 + a1 * a1 + a2 * a2);
    const double cs = (a0 / nn) * x + (a1 / nn) * y + (a2 / nn) * z;
    lob[l] = exp((double)rec[59 + l] * (cs - 1.0));
  }
  for (int ch = 0; ch < 3; ++ch) {
    double v = 0.0;
    for (int l = 0; l < 7; ++l) v += lob[l] * (double)rec[66 + 3 * l + ch];
    acc[ch] += v;
    rgb[ch] = acc[ch] > 0.0 ? acc[ch] : 0.0;
  }
}

// y0 = M (o - mu), yd = M d of primitive p (scene.py:58-60 iso_inv, fp64)
__device__ inline void frame64(const SceneView& sv, const float* params, int64_t p,
                               const double* o, const double* d, double* y0, double* yd) {
  const double* M = sv.inv64 + 9 * p;
  const float* mu = params + GSX_NREC * p;
  const double v[3] = {o[0] - (double)mu[0], o[1] - (double)mu[1], o[2] - (double)mu[2]};
  for (int a = 0; a < 3; ++a) {
    y0[a] = M[3 * a] * v[0] + M[3 * a + 1] * v[1] + M[3 * a + 2] * v[2];
    yd[a] = M[3 * a] * d[0] + M[3 * a + 1] * d[1] + M[3 * a + 2] * d[2];
  }
}

__device__ inline double shfl_d(double v, int src) {
  return __hiloint2double(__shfl_sync(0xffffffffu, __double2hiint(v), src),
                          __shfl_sync(0xffffffffu, __double2loint(v), src));
}

// One warp per ray.  Samples in chunks of 32 x S: lane l owns the S
// consecutive samples chunk + S l + s, so the chunk's compositing is a lane
// prefix plus one warp scan.  Per chunk every primitive's exact fp64
// ellipsoid interval is tested lane-parallel against the chunk's t-range;
// the hits are then evaluated by all lanes (ballot order).
constexpr int S = 8;
__global__ void __launch_bounds__(128) k_reference_rays(SceneView sv, const float* __restrict__ params,
                                                        int64_t n, const double* __restrict__ rays,
                                                        int64_t m, int clip, double fine_dt,
                                                        double bg0, double bg1, double bg2,
                                                        double* __restrict__ rgb_out) {
  const int64_t ray = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (ray >= m) return;
  const int lane = threadIdx.x & 31;
  const double bg[3] = {bg0, bg1, bg2};
  RayCtx r;
  const bool ok = explicit_ray(rays + 8 * ray, clip != 0, sv.bounds, r);
  double* out = rgb_out + 3 * ray;
  if (!ok) {  // reference_render: background; reference_integrate: t_near >= t_far
    if (lane < 3) out[lane] = bg[lane];
    return;
  }
  const double tn = r.t_n, tf = r.t_f;
  int64_t ns = (int64_t)ceil((tf - tn) / fine_dt);
  while (ns > 0 && !(tn + ((double)(ns - 1) + 0.5) * fine_dt < tf)) --ns;
  if (ns <= 0) {
    if (lane < 3) out[lane] = bg[lane];
    return;
  }
  double col[3] = {0.0, 0.0, 0.0};
  double cum = 0.0;  // optical depth before the current chunk
  for (int64_t c0 = 0; c0 < ns; c0 += 32 * S) {
    double sig[S], W[S][3];
    for (int s = 0; s < S; ++s) sig[s] = W[s][0] = W[s][1] = W[s][2] = 0.0;
    const int64_t j0 = c0 + (int64_t)S * lane;
    const int64_t jend = c0 + 32 * S < ns ? c0 + 32 * S : ns;
    const double ta = tn + ((double)c0 + 0.5) * fine_dt, tb = tn + ((double)(jend - 1) + 0.5) * fine_dt;
    for (int64_t p0 = 0; p0 < n; p0 += 32) {
      const int64_t pl = p0 + lane;
      bool hit = false;
      if (pl < n) {
        double y0[3], yd[3], tin, tout;
        frame64(sv, params, pl, r.o, r.d, y0, yd);
        hit = ray_ellipsoid_interval64(y0, yd, ta, tb, tin, tout);
      }
      unsigned bal = __ballot_sync(0xffffffffu, hit);
      while (bal) {
        const int src = __ffs(bal) - 1;
        bal &= bal - 1;
        const int64_t p = p0 + src;
        double y0[3], yd[3], c[3];
        frame64(sv, params, p, r.o, r.d, y0, yd);
        radiance64(params + GSX_NREC * p, r.d, c);
        const double sigma = params[GSX_NREC * p + 10], lr = sv.lr64[p];
        for (int s = 0; s < S; ++s) {
          const int64_t j = j0 + s;
          if (j >= jend) break;
          const double t = tn + ((double)j + 0.5) * fine_dt;
          const double y[3] = {y0[0] + t * yd[0], y0[1] + t * yd[1], y0[2] + t * yd[2]};
          const double q = y[0] * y[0] + y[1] * y[1] + y[2] * y[2];
          if (q <= 1.0) {
            const double dens = sigma * exp(-0.5 * lr * q);
            sig[s] += dens;
            for (int k = 0; k < 3; ++k) W[s][k] += dens * c[k];
          }
        }
      }
    }
    // compositing of the chunk (renderer.py:472-480): lane prefix + warp scan
    double mine = 0.0;
    for (int s = 0; s < S; ++s)
      if (j0 + s < jend) mine += sig[s] * fine_dt;
    double incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
      const double v = shfl_d(incl, lane >= o ? lane - o : lane);
      if (lane >= o) incl += v;
    }
    double before = cum + (incl - mine);
    for (int s = 0; s < S; ++s) {
      if (j0 + s >= jend) break;
      const double od = sig[s] * fine_dt;
      if (sig[s] > 0.0) {
        const double w = -expm1(-od) * exp(-before);
        for (int k = 0; k < 3; ++k) col[k] += (w / sig[s]) * W[s][k];
      }
      before += od;
    }
    cum += shfl_d(incl, 31);
  }
  for (int k = 0; k < 3; ++k)
    for (int o = 16; o > 0; o >>= 1) col[k] += shfl_d(col[k], lane ^ o);
  if (lane == 0) {
    const double t_exit = exp(-cum);
    for (int k = 0; k < 3; ++k) out[k] = col[k] + t_exit * bg[k];
  }
}

// one thread per point (appearance.py:107-134)
__global__ void k_eval_fields(SceneView sv, const float* __restrict__ params, int64_t n,
                              const double* __restrict__ pts, const double* __restrict__ dirs,
                              int64_t m, const int64_t* __restrict__ active, int64_t na,
                              double* sigma_out, double* color_out, gsx_dev_status* st) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const double x[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
  const double d[3] = {dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]};
  const double zero[3] = {0.0, 0.0, 0.0};
  double sigma = 0.0, w[3] = {0.0, 0.0, 0.0};
  const int64_t cnt = active ? na : n;
  for (int64_t a = 0; a < cnt; ++a) {
    const int64_t p = active ? active[a] : a;
    if (p < 0 || p >= n) {
      dev_fail(st, GSX_ERR_ARG, a);
      continue;
    }
    double y[3], unused[3];
    frame64(sv, params, p, x, zero, y, unused);
    // y = iso_inv (x - mu): frame64 with o = x; q = |y|^2
    const double q = y[0] * y[0] + y[1] * y[1] + y[2] * y[2];
    if (q > 1.0) continue;
    const double dens = (double)params[GSX_NREC * p + 10] * exp(-0.5 * sv.lr64[p] * q);
    double c[3];
    radiance64(params + GSX_NREC * p, d, c);
    sigma += dens;
    for (int k = 0; k < 3; ++k) w[k] += dens * c[k];
  }
  sigma_out[i] = sigma;
  for (int k = 0; k < 3; ++k) color_out[3 * i + k] = sigma == 0.0 ? 0.0 : w[k] / sigma;
}

}  // namespace

extern "C" int gsx_reference_rays(const void* scene_arena, const float* params, int64_t n,
                                  const double* rays, int64_t m, int clip, double fine_dt,
                                  const double* background, double* rgb, void* stream) {
  if (n <= 0) return GSX_ERR_EMPTY;
  if (!(fine_dt > 0.0) || !background || !params) return GSX_ERR_ARG;
  if (m <= 0) return GSX_OK;
  SceneView sv = scene_view((void*)scene_arena, n);
  k_reference_rays<<<(unsigned)((m + 3) / 4), 128, 0, (cudaStream_t)stream>>>(
      sv, params, n, rays, m, clip, fine_dt, background[0], background[1], background[2], rgb);
  return gsx_check_launch();
}

extern "C" int gsx_eval_fields(const void* scene_arena, const float* params, int64_t n,
                               const double* points, const double* dirs, int64_t m,
                               const int64_t* active, int64_t n_active, double* sigma,
                               double* color, gsx_dev_status* dev_status, void* stream) {
  if (n <= 0) return GSX_ERR_EMPTY;
  if (!params || (n_active < 0)) return GSX_ERR_ARG;
  if (m <= 0) return GSX_OK;
  SceneView sv = scene_view((void*)scene_arena, n);
  k_eval_fields<<<(unsigned)((m + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      sv, params, n, points, dirs, m, active, n_active, sigma, color, dev_status);
  return gsx_check_launch();
}
