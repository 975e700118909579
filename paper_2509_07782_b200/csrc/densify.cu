// densify.cu -- densification statistics (densify.py:49-83 GradAccumulator,
// criterion_old / criterion_new; observe_scene :190-204).
//
// The reference observes one camera by finite-differencing the image loss
// w.r.t. every mean (6 renders per primitive, fd_position_gradient
// densify.py:156-187).  Here the observation consumes the analytic gradient
// the backward has just produced (grad [N,87], record layout, after the
// multi-GPU all-reduce): per primitive, |dL/dmu| and
// alpha = |mu - camera center| / focal accumulate in float64 exactly like
// GradAccumulator.observe; one thread per observed primitive, 12 bytes of
// gradient + 12 bytes of mean read per primitive.
#include "gsx_common.cuh"

namespace {

__global__ void k_densify_observe(const float* __restrict__ grad, const float* __restrict__ params,
                                  int64_t n, const int64_t* __restrict__ indices, int64_t m,
                                  double cx, double cy, double cz, double focal,
                                  double* __restrict__ sum_raw, double* __restrict__ sum_weighted,
                                  int64_t* __restrict__ counts) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t i = indices ? indices[k] : k;
  if (i < 0 || i >= n) return;
  const float* g = grad + GSX_NREC * i;
  const double g0 = g[0], g1 = g[1], g2 = g[2];
  const double norm = sqrt(g0 * g0 + g1 * g1 + g2 * g2);
  const float* mu = params + GSX_NREC * i;
  const double dx = (double)mu[0] - cx, dy = (double)mu[1] - cy, dz = (double)mu[2] - cz;
  const double alpha = sqrt(dx * dx + dy * dy + dz * dz) / focal;
  // indices may repeat (observe is additive), hence atomics
  atomicAdd(sum_raw + i, norm);
  atomicAdd(sum_weighted + i, alpha * norm);
  atomicAdd((unsigned long long*)(counts + i), 1ull);
}

__global__ void k_densify_criteria(const double* __restrict__ sum_raw,
                                   const double* __restrict__ sum_weighted,
                                   const int64_t* __restrict__ counts, int64_t n, double tau,
                                   uint8_t* __restrict__ crit_old, uint8_t* __restrict__ crit_new) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t c = counts[i];
  const bool seen = c >= 1;
  // mean over the window strictly above tau (densify.py:69-83)
  if (crit_old) crit_old[i] = seen && sum_raw[i] / (double)c > tau ? 1 : 0;
  if (crit_new) crit_new[i] = seen && sum_weighted[i] / (double)c > tau ? 1 : 0;
}

}  // namespace

extern "C" int gsx_densify_observe(const float* grad, const float* params, int64_t n,
                                   const int64_t* indices, int64_t m, const double* center,
                                   double focal, double* sum_raw, double* sum_weighted,
                                   int64_t* counts, void* stream) {
  if (n <= 0) return GSX_ERR_EMPTY;
  if (!grad || !params || !center || !sum_raw || !sum_weighted || !counts) return GSX_ERR_ARG;
  if (!(focal > 0.0)) return GSX_ERR_ARG;
  if (!indices) m = n;
  if (m <= 0) return GSX_OK;
  k_densify_observe<<<(unsigned)((m + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      grad, params, n, indices, m, center[0], center[1], center[2], focal, sum_raw, sum_weighted,
      counts);
  return gsx_check_launch();
}

extern "C" int gsx_densify_criteria(const double* sum_raw, const double* sum_weighted,
                                    const int64_t* counts, int64_t n, double tau,
                                    uint8_t* crit_old, uint8_t* crit_new, void* stream) {
  if (n <= 0) return GSX_ERR_EMPTY;
  if (!sum_raw || !sum_weighted || !counts || !(tau > 0.0)) return GSX_ERR_ARG;
  k_densify_criteria<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      sum_raw, sum_weighted, counts, n, tau, crit_old, crit_new);
  return gsx_check_launch();
}
