// prep.cu -- K1: per-primitive derived arrays + scene bounds (replaces
// Scene._rebuild scene.py:48-69, GaussianShape geometry.py:77-87,
// quat_to_rotation geometry.py:26-42, AppearanceCoeffs appearance.py:62-76).
//
// The fp64 part mirrors numpy's operation order with explicit round-to-nearest
// intrinsics (no FMA contraction), so the fp64 AABBs, iso_inv and scene bounds
// agree with the reference to the last bit or two; the fp32 render SoA is
// derived from those fp64 values.
#include "gsx_common.cuh"

namespace {

__device__ inline double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ inline double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ inline double dsub(double a, double b) { return __dsub_rn(a, b); }

__device__ inline double norm4(const double* q) {
  return sqrt(dadd(dadd(dadd(dmul(q[0], q[0]), dmul(q[1], q[1])), dmul(q[2], q[2])),
                   dmul(q[3], q[3])));
}
__device__ inline double norm3(const double* q) {
  return sqrt(dadd(dadd(dmul(q[0], q[0]), dmul(q[1], q[1])), dmul(q[2], q[2])));
}

__global__ void k_prepare(const float* __restrict__ params, int64_t n, double sigma_eps,
                          SceneView v, gsx_dev_status* st) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* r = params + GSX_NREC * i;
  double mu[3] = {(double)r[0], (double)r[1], (double)r[2]};
  double qraw[4] = {(double)r[3], (double)r[4], (double)r[5], (double)r[6]};
  double qn = norm4(qraw);
  bool bad = !(qn >= 1e-12);
  double q[4];
  for (int k = 0; k < 4; ++k) q[k] = qraw[k] / qn;  // geometry.py:80
  // quat_to_rotation normalizes again (geometry.py:32-35)
  double n2 = norm4(q);
  double w = q[0] / n2, x = q[1] / n2, y = q[2] / n2, z = q[3] / n2;
  double R[9];
  R[0] = dsub(1.0, dmul(2.0, dadd(dmul(y, y), dmul(z, z))));
  R[1] = dmul(2.0, dsub(dmul(x, y), dmul(w, z)));
  R[2] = dmul(2.0, dadd(dmul(x, z), dmul(w, y)));
  R[3] = dmul(2.0, dadd(dmul(x, y), dmul(w, z)));
  R[4] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(z, z))));
  R[5] = dmul(2.0, dsub(dmul(y, z), dmul(w, x)));
  R[6] = dmul(2.0, dsub(dmul(x, z), dmul(w, y)));
  R[7] = dmul(2.0, dadd(dmul(y, z), dmul(w, x)));
  R[8] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(y, y))));
  double sc[3];
  for (int k = 0; k < 3; ++k) {
    double s = (double)r[7 + k];
    sc[k] = s > 1e-7 ? s : 1e-7;  // geometry.py:81
  }
  double sigma = (double)r[10];
  bad |= !(sigma > sigma_eps);  // scene.py:37-41
  // appearance validation (appearance.py:65-71)
  double axn[7][3];
  for (int l = 0; l < 7; ++l) {
    double ax[3] = {(double)r[38 + 3 * l], (double)r[39 + 3 * l], (double)r[40 + 3 * l]};
    double an = norm3(ax);
    bad |= !(an >= 1e-12);
    for (int k = 0; k < 3; ++k) axn[l][k] = ax[k] / an;
    bad |= (double)r[59 + l] < 0.0;
  }
  if (bad) {
    dev_fail(st, GSX_ERR_VALIDATION, i);
    return;
  }
  // scene.py:55-65
  double lr = dmul(2.0, log(sigma / sigma_eps));
  double sq = sqrt(lr);
  double s_t[3] = {dmul(sq, sc[0]), dmul(sq, sc[1]), dmul(sq, sc[2])};
  double M[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) M[3 * a + b] = R[3 * b + a] / s_t[a];
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    double p0 = dmul(R[3 * a + 0], s_t[0]), p1 = dmul(R[3 * a + 1], s_t[1]),
           p2 = dmul(R[3 * a + 2], s_t[2]);
    double h = sqrt(dadd(dadd(dmul(p0, p0), dmul(p1, p1)), dmul(p2, p2)));
    lo[a] = dsub(mu[a], h);
    hi[a] = dadd(mu[a], h);
  }
  double* ab = v.aabb64 + 6 * i;
  for (int k = 0; k < 3; ++k) {
    ab[k] = lo[k];
    ab[3 + k] = hi[k];
  }
  double* iv = v.inv64 + 9 * i;
  for (int k = 0; k < 9; ++k) iv[k] = M[k];
  v.lr64[i] = lr;
  // fp32 render SoA
  const double LOG2E = 1.4426950408889634;
  float4* g = v.geo + 4 * i;
  g[0] = make_float4(r[0], r[1], r[2], r[10]);
  g[1] = make_float4((float)M[0], (float)M[1], (float)M[2], (float)(0.5 * lr * LOG2E));
  g[2] = make_float4((float)M[3], (float)M[4], (float)M[5], (float)lr);
  g[3] = make_float4((float)M[6], (float)M[7], (float)M[8], (float)log2(sigma));
  float* b32 = v.box32 + 6 * i;
  for (int k = 0; k < 3; ++k) {
    b32[k] = __double2float_rd(lo[k]);
    b32[3 + k] = __double2float_ru(hi[k]);
  }
  // radiance-streaming layout (gsx_common.cuh): SH rows, then (axis, sharpness), (amp)
  float4* ap = v.app + GSX_APP_F4 * i;
  for (int b = 0; b < 9; ++b) ap[b] = make_float4(r[11 + 3 * b], r[12 + 3 * b], r[13 + 3 * b], 0.f);
  for (int l = 0; l < 7; ++l) {
    ap[9 + 2 * l] = make_float4((float)axn[l][0], (float)axn[l][1], (float)axn[l][2], r[59 + l]);
    ap[10 + 2 * l] = make_float4(r[66 + 3 * l], r[67 + 3 * l], r[68 + 3 * l], 0.f);
  }
  // backward helpers (render_bwd.cu)
  float ian[7];
  for (int l = 0; l < 7; ++l) {
    double ax[3] = {(double)r[38 + 3 * l], (double)r[39 + 3 * l], (double)r[40 + 3 * l]};
    ian[l] = (float)(1.0 / norm3(ax));
  }
  float4* ga = v.gaux + 5 * i;
  ga[0] = make_float4((float)w, (float)x, (float)y, (float)z);
  ga[1] = make_float4((float)(1.0 / qn), (float)(1.0 / sc[0]), (float)(1.0 / sc[1]),
                      (float)(1.0 / sc[2]));
  ga[2] = make_float4((float)sq, (double)r[7] > 1e-7 ? 1.f : 0.f, (double)r[8] > 1e-7 ? 1.f : 0.f,
                      (double)r[9] > 1e-7 ? 1.f : 0.f);
  ga[3] = make_float4(ian[0], ian[1], ian[2], ian[3]);
  ga[4] = make_float4(ian[4], ian[5], ian[6], sigma > 0.0 ? (float)(1.0 / sigma) : 0.f);
}

// scene bounds: min/max over AABBs (exact; order independent)
__global__ void k_bounds_partial(SceneView v, int64_t n) {
  __shared__ double sh[6][256];
  double acc[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double* ab = v.aabb64 + 6 * i;
    for (int k = 0; k < 3; ++k) {
      acc[k] = fmin(acc[k], ab[k]);
      acc[3 + k] = fmax(acc[3 + k], ab[3 + k]);
    }
  }
  for (int k = 0; k < 6; ++k) sh[k][threadIdx.x] = acc[k];
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int k = 0; k < 6; ++k)
        sh[k][threadIdx.x] = k < 3 ? fmin(sh[k][threadIdx.x], sh[k][threadIdx.x + s])
                                   : fmax(sh[k][threadIdx.x], sh[k][threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) v.part[6 * blockIdx.x + k] = sh[k][0];
}

// one warp: lanes stride over the partials, then a shuffle min / max tree
// (a single serial thread took 85 us for 296 partials)
__global__ void k_bounds_final(SceneView v, int nblocks) {
  double acc[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int b = threadIdx.x; b < nblocks; b += 32)
    for (int k = 0; k < 3; ++k) {
      acc[k] = fmin(acc[k], v.part[6 * b + k]);
      acc[3 + k] = fmax(acc[3 + k], v.part[6 * b + 3 + k]);
    }
  for (int o = 16; o > 0; o >>= 1)
    for (int k = 0; k < 3; ++k) {
      acc[k] = fmin(acc[k], __shfl_xor_sync(0xffffffffu, acc[k], o));
      acc[3 + k] = fmax(acc[3 + k], __shfl_xor_sync(0xffffffffu, acc[3 + k], o));
    }
  if (threadIdx.x == 0)
    for (int k = 0; k < 6; ++k) v.bounds[k] = acc[k];
}

}  // namespace

extern "C" size_t gsx_scene_arena_bytes(int64_t n) { return scene_arena_bytes_impl(n); }

extern "C" int gsx_prepare(const float* params, int64_t n, double sigma_eps, void* arena,
                           gsx_dev_status* dev_status, double* host_bounds, void* stream) {
  if (n <= 0) return GSX_ERR_EMPTY;
  if (!(sigma_eps > 0) || !params || !arena) return GSX_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  SceneView v = scene_view(arena, n);
  int threads = 128;
  k_prepare<<<(unsigned)((n + threads - 1) / threads), threads, 0, s>>>(params, n, sigma_eps, v,
                                                                          dev_status);
  int nb = (int)((n + 255) / 256);
  if (nb > GSX_BOUNDS_BLOCKS) nb = GSX_BOUNDS_BLOCKS;
  k_bounds_partial<<<nb, 256, 0, s>>>(v, n);
  k_bounds_final<<<1, 32, 0, s>>>(v, nb);
  int rc = gsx_check_launch();
  if (rc) return rc;
  if (host_bounds) {
    CUDA_CHECK_RET(cudaMemcpyAsync(host_bounds, v.bounds, sizeof(double) * 6,
                                   cudaMemcpyDeviceToHost, s));
    CUDA_CHECK_RET(cudaStreamSynchronize(s));
  }
  return GSX_OK;
}

extern "C" int gsx_scene_get(const void* arena, int64_t n, int which, void* out, void* stream) {
  SceneView v = scene_view((void*)arena, n);
  cudaStream_t s = (cudaStream_t)stream;
  const void* src;
  size_t bytes;
  switch (which) {
    case 0:
    case 1: {
      // de-interleave lo / hi
      double* o = (double*)out;
      CUDA_CHECK_RET(cudaMemcpy2DAsync(o, sizeof(double) * 3, v.aabb64 + (which ? 3 : 0),
                                       sizeof(double) * 6, sizeof(double) * 3, n,
                                       cudaMemcpyDeviceToDevice, s));
      return GSX_OK;
    }
    case 2: src = v.inv64; bytes = sizeof(double) * 9 * n; break;
    case 3: src = v.lr64; bytes = sizeof(double) * n; break;
    case 4: src = v.bounds; bytes = sizeof(double) * 6; break;
    default: return GSX_ERR_ARG;
  }
  CUDA_CHECK_RET(cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToDevice, s));
  return GSX_OK;
}
