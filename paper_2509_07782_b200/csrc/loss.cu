// loss.cu -- K8 image loss and K9 isotropic loss, plus the fused Adam update
// of the training step.
//
// K8 restates densify.py:99-153: L = (1-mix) mean|x-y| + mix (1 - SSIM)/2 with
// SSIM = mean over channels of the mean over the 5-px-cropped interior of the
// SSIM map, whose local statistics use scipy.ndimage.gaussian_filter(sigma=1.5,
// truncate=3.5) -> 11 separable taps, mode='reflect' (d c b a | a b c d).
// The gradient w.r.t. the rendered image uses the filter adjoint:
//   dS/dx = G^T a + 2 x G^T b + y G^T c,
//   a = dS/du_x, b = dS/du_xx, c = dS/du_xy  (per pixel, crop-masked)
// where G^T (transpose of reflect-pad + convolve) is the zero-padded
// convolution evaluated at a pixel and at its reflected pre-images.
// Images are [H, W, C] float32 (C = 3), H, W >= 11.
//
// K9 restates geometry.py:193-233 (ratio_upper_bound, isotropic_loss) and
// accumulates lambda_s * dL_s/ds into the record gradient (scales clamped at
// S_MIN receive none).
#include <algorithm>
#include <climits>
#include <cstdint>
#include "gsx_common.cuh"

namespace {

constexpr int R = 5;  // int(3.5 * 1.5 + 0.5)

struct Taps {
  float w[2 * R + 1];
};

Taps make_taps() {
  Taps t;
  double s = 0, v[2 * R + 1];
  for (int i = -R; i <= R; ++i) {
    v[i + R] = exp(-0.5 * (double)i * i / (1.5 * 1.5));
    s += v[i + R];
  }
  for (int i = 0; i <= 2 * R; ++i) t.w[i] = (float)(v[i] / s);
  return t;
}

// scipy 'reflect' (half-sample symmetric), repeated for indices far outside
__device__ inline int reflect(int j, int n) {
  if (n == 1) return 0;
  int period = 2 * n;
  j %= period;
  if (j < 0) j += period;
  return j < n ? j : period - 1 - j;
}

// horizontal pass: 5 maps (x, y, x^2, y^2, xy) filtered along W
__global__ void k_ssim_h(const float* __restrict__ x, const float* __restrict__ y, int H, int W,
                         int C, Taps t, float* __restrict__ hmap) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)H * W * C;
  if (idx >= total) return;
  int c = (int)(idx % C);
  int64_t pix = idx / C;
  int col = (int)(pix % W), row = (int)(pix / W);
  float s[5] = {0, 0, 0, 0, 0};
#pragma unroll
  for (int k = -R; k <= R; ++k) {
    int cc = reflect(col + k, W);
    int64_t j = ((int64_t)row * W + cc) * C + c;
    float a = x[j], b = y[j], w = t.w[k + R];
    s[0] = fmaf(w, a, s[0]);
    s[1] = fmaf(w, b, s[1]);
    s[2] = fmaf(w, a * a, s[2]);
    s[3] = fmaf(w, b * b, s[3]);
    s[4] = fmaf(w, a * b, s[4]);
  }
#pragma unroll
  for (int m = 0; m < 5; ++m) hmap[m * total + idx] = s[m];
}

// vertical pass + SSIM map + per-pixel adjoint coefficients + reductions
__global__ void k_ssim_v(const float* __restrict__ x, const float* __restrict__ y,
                         const float* __restrict__ hmap, int H, int W, int C, Taps t,
                         float* __restrict__ coef, double* __restrict__ sums) {
  __shared__ double red[2][256];
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)H * W * C;
  double s_sum = 0.0, l1 = 0.0;
  if (idx < total) {
    int c = (int)(idx % C);
    int64_t pix = idx / C;
    int col = (int)(pix % W), row = (int)(pix / W);
    float u[5] = {0, 0, 0, 0, 0};
#pragma unroll
    for (int k = -R; k <= R; ++k) {
      int rr = reflect(row + k, H);
      int64_t j = ((int64_t)rr * W + col) * C + c;
      float w = t.w[k + R];
#pragma unroll
      for (int m = 0; m < 5; ++m) u[m] = fmaf(w, hmap[m * total + j], u[m]);
    }
    const float c1 = 0.01f * 0.01f, c2 = 0.03f * 0.03f;
    float ux = u[0], uy = u[1];
    float vx = u[2] - ux * ux, vy = u[3] - uy * uy, cov = u[4] - ux * uy;
    float A1 = 2.f * ux * uy + c1, B1 = 2.f * cov + c2;
    float A2 = ux * ux + uy * uy + c1, B2 = vx + vy + c2;
    float D = A2 * B2;
    float S = A1 * B1 / D;
    bool in_crop = row >= R && row < H - R && col >= R && col < W - R;
    float a = 0.f, b = 0.f, cc = 0.f;
    if (in_crop) {
      s_sum = (double)S;
      a = (2.f * uy * (B1 - A1) - S * 2.f * ux * (B2 - A2)) / D;
      b = -S / B2;
      cc = 2.f * A1 / D;
    }
    coef[idx] = a;
    coef[total + idx] = b;
    coef[2 * total + idx] = cc;
    l1 = fabs((double)x[idx] - (double)y[idx]);
  }
  red[0][threadIdx.x] = s_sum;
  red[1][threadIdx.x] = l1;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      red[0][threadIdx.x] += red[0][threadIdx.x + st];
      red[1][threadIdx.x] += red[1][threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicAdd(&sums[0], red[0][0]);
    atomicAdd(&sums[1], red[1][0]);
  }
}

// adjoint of reflect-pad + 11-tap filter along one axis: zero-padded
// convolution at i plus at the reflected pre-images of i
__device__ inline float adj_tap_sum(const float* __restrict__ v, int64_t base, int64_t stride,
                                    int i, int n, const Taps& t) {
  float s = 0.f;
  // pre-images j of i under reflect within reach of the taps: j = i, -i-1, 2n-1-i
  int pre[3] = {i, -i - 1, 2 * n - 1 - i};
  int npre = 1 + (i <= R - 1 ? 1 : 0) + (i >= n - R ? 1 : 0);
  int js[3];
  int q = 0;
  js[q++] = pre[0];
  if (i <= R - 1) js[q++] = pre[1];
  if (i >= n - R) js[q++] = pre[2];
  for (int e = 0; e < npre; ++e) {
    int j = js[e];
#pragma unroll
    for (int k = -R; k <= R; ++k) {
      int p = j - k;  // u_p uses x[refl(p + k)]
      if (p >= 0 && p < n) s = fmaf(t.w[k + R], v[base + (int64_t)p * stride], s);
    }
  }
  return s;
}

// adjoint vertical pass of the 3 coefficient maps
__global__ void k_ssim_adj_v(const float* __restrict__ coef, int H, int W, int C, Taps t,
                             float* __restrict__ tmp) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)H * W * C;
  if (idx >= total) return;
  int c = (int)(idx % C);
  int64_t pix = idx / C;
  int col = (int)(pix % W), row = (int)(pix / W);
  int64_t base = (int64_t)col * C + c, stride = (int64_t)W * C;
#pragma unroll
  for (int m = 0; m < 3; ++m) tmp[m * total + idx] = adj_tap_sum(coef + m * total, base, stride, row, H, t);
}

// adjoint horizontal pass + combination into dL/dx
__global__ void k_ssim_adj_h(const float* __restrict__ x, const float* __restrict__ y,
                             const float* __restrict__ tmp, int H, int W, int C, Taps t,
                             float l1_scale, float ssim_scale, float* __restrict__ dx) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t total = (int64_t)H * W * C;
  if (idx >= total) return;
  int c = (int)(idx % C);
  int64_t pix = idx / C;
  int col = (int)(pix % W), row = (int)(pix / W);
  int64_t base = (int64_t)row * W * C + c, stride = C;
  float ga = adj_tap_sum(tmp, base, stride, col, W, t);
  float gb = adj_tap_sum(tmp + total, base, stride, col, W, t);
  float gc = adj_tap_sum(tmp + 2 * total, base, stride, col, W, t);
  float xv = x[idx], yv = y[idx];
  float g_ssim = ga + 2.f * xv * gb + yv * gc;
  float d = xv - yv;
  float sgn = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
  dx[idx] = l1_scale * sgn + ssim_scale * g_ssim;
}

// ---- K9 isotropic loss (geometry.py:193-233) ----------------------------------
__global__ void k_iso_loss(const float* __restrict__ params, int64_t n, double r0, double lambda_s,
                           double* __restrict__ loss_sum, float* __restrict__ grad) {
  __shared__ double red[256];
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double l = 0.0;
  if (i < n) {
    double s[3], raw[3];
    for (int k = 0; k < 3; ++k) {
      raw[k] = (double)params[GSX_NREC * i + 7 + k];
      s[k] = raw[k] > 1e-7 ? raw[k] : 1e-7;
    }
    double ss = s[0] * s[0] + s[1] * s[1] + s[2] * s[2];
    double rmax = (2.0 / (3.14159265358979323846 * sqrt(3.0))) * pow(ss, 1.5) / (s[0] * s[1] * s[2]);
    if (rmax > r0) {
      l = rmax - r0;
      if (grad) {
        for (int k = 0; k < 3; ++k) {
          double g = rmax * (3.0 * s[k] / ss - 1.0 / s[k]) / (double)n;
          // the clamp np.maximum(s, S_MIN) passes no gradient to clamped scales
          if (raw[k] > 1e-7) grad[GSX_NREC * i + 7 + k] += (float)(lambda_s * g);
        }
      }
    }
  }
  red[threadIdx.x] = l;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicAdd(loss_sum, red[0]);
}

// ---- fused Adam over the [N, 87] records -----------------------------------------
// HBM-bound: 16 B read (p, g, m, v) + 12 B written (p, m, v) per value.  One
// float4 of each stream per thread (grid-stride loop for very large N); the
// record slot (value index mod 87) is carried across iterations.
struct AdamArgs {
  const float* lr87;
  const float* lo87;
  float b1, b2, eps, ibc1, isbc2;  // 1 / (1 - b1^t), 1 / sqrt(1 - b2^t)
};
__device__ __forceinline__ void adam_one(float& pi, float gi, float& mi, float& vi, int slot,
                                         const AdamArgs& a) {
  mi = fmaf(a.b1, mi, (1.f - a.b1) * gi);
  vi = fmaf(a.b2, vi, (1.f - a.b2) * gi * gi);
  // p -= lr (m / bc1) / (sqrt(v / bc2) + eps): one division
  const float np_ = pi - __ldg(a.lr87 + slot) * a.ibc1 * mi / fmaf(sqrtf(vi), a.isbc2, a.eps);
  // projection onto the record's validity domain (sigma~ > sigma_eps,
  // scales > 0, sharpness >= 0): lo87 = per-slot lower bound (-inf = none)
  pi = fmaxf(np_, __ldg(a.lo87 + slot));
}
__device__ __forceinline__ int slot_next(int s) { return s + 1 - (s + 1 >= GSX_NREC ? GSX_NREC : 0); }
__device__ __forceinline__ void adam_f4(float4& pp, const float4& gg, float4& mm, float4& vv,
                                        int slot, const AdamArgs& a) {
  const int s1 = slot_next(slot), s2 = slot_next(s1), s3 = slot_next(s2);
  adam_one(pp.x, gg.x, mm.x, vv.x, slot, a);
  adam_one(pp.y, gg.y, mm.y, vv.y, s1, a);
  adam_one(pp.z, gg.z, mm.z, vv.z, s2, a);
  adam_one(pp.w, gg.w, mm.w, vv.w, s3, a);
}
// ILP float4s of each stream in flight per thread and iteration (grid-stride
// over CTAs sized to the device); the record slot of each is carried.
// 3M records (profiles/adam_bw.py): one float4 per thread and stream, one
// CTA per 256 of them: 1.05 ms = 7.0 TB/s of the 28 B/value; grid-stride
// over 8 / 16 CTAs per SM with 1-4 float4 in flight per thread 1.16-1.20 ms;
// the two-division form 1.89 ms.
#ifndef GSX_ADAM_CTAS  // CTAs per SM of the grid-stride loop
#define GSX_ADAM_CTAS (1 << 20)
#endif
#ifndef GSX_ADAM_ILP
#define GSX_ADAM_ILP 1
#endif
__global__ void __launch_bounds__(256) k_adam4(float4* __restrict__ p, const float4* __restrict__ g,
                                               float4* __restrict__ m, float4* __restrict__ v,
                                               int64_t n4, AdamArgs a) {
  constexpr int ILP = GSX_ADAM_ILP;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int slot[ILP];
#pragma unroll
  for (int u = 0; u < ILP; ++u) slot[u] = (int)((4 * (q + u * stride)) % GSX_NREC);
  const int step = (int)((4 * ILP * stride) % GSX_NREC);
  for (; q < n4; q += ILP * stride) {
    float4 pp[ILP], mm[ILP], vv[ILP], gg[ILP];
#pragma unroll
    for (int u = 0; u < ILP; ++u) {
      const int64_t k = q + u * stride;
      if (k < n4) {
        pp[u] = p[k];
        mm[u] = m[k];
        vv[u] = v[k];
        gg[u] = __ldcs(g + k);
      }
    }
#pragma unroll
    for (int u = 0; u < ILP; ++u) {
      const int64_t k = q + u * stride;
      if (k < n4) {
        adam_f4(pp[u], gg[u], mm[u], vv[u], slot[u], a);
        p[k] = pp[u];
        m[k] = mm[u];
        v[k] = vv[u];
      }
      slot[u] += step;
      slot[u] -= slot[u] >= GSX_NREC ? GSX_NREC : 0;
    }
  }
}
// scalar tail / unaligned views (a row shard of the padded parameters)
__global__ void k_adam1(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                        float* __restrict__ v, int64_t begin, int64_t count, AdamArgs a) {
  const int64_t i = begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  float pi = p[i], mi = m[i], vi = v[i];
  adam_one(pi, g[i], mi, vi, (int)(i % GSX_NREC), a);
  p[i] = pi;
  m[i] = mi;
  v[i] = vi;
}

}  // namespace

extern "C" size_t gsx_image_loss_workspace_bytes(int64_t h, int64_t w, int64_t c) {
  int64_t total = h * w * c;
  return gsx_align256(sizeof(float) * 5 * total) + gsx_align256(sizeof(float) * 3 * total) +
         gsx_align256(sizeof(float) * 3 * total) + gsx_align256(sizeof(double) * 2);
}

extern "C" int gsx_image_loss(const float* rendered, const float* target, int64_t h, int64_t w,
                              int64_t c, double mix, float* dL_drendered, double* host_out,
                              void* workspace, void* stream) {
  if (h < 2 * R + 1 || w < 2 * R + 1 || c < 1) return GSX_ERR_ARG;
  if (!(mix >= 0.0 && mix <= 1.0)) return GSX_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t total = h * w * c;
  char* ws = (char*)workspace;
  float* hmap = (float*)ws;
  float* coef = (float*)(ws + gsx_align256(sizeof(float) * 5 * total));
  float* tmp = (float*)((char*)coef + gsx_align256(sizeof(float) * 3 * total));
  double* sums = (double*)((char*)tmp + gsx_align256(sizeof(float) * 3 * total));
  Taps t = make_taps();
  unsigned blocks = (unsigned)((total + 255) / 256);
  CUDA_CHECK_RET(cudaMemsetAsync(sums, 0, sizeof(double) * 2, s));
  k_ssim_h<<<blocks, 256, 0, s>>>(rendered, target, (int)h, (int)w, (int)c, t, hmap);
  k_ssim_v<<<blocks, 256, 0, s>>>(rendered, target, hmap, (int)h, (int)w, (int)c, t, coef, sums);
  double n_crop = (double)(h - 2 * R) * (double)(w - 2 * R) * (double)c;
  if (dL_drendered) {
    k_ssim_adj_v<<<blocks, 256, 0, s>>>(coef, (int)h, (int)w, (int)c, t, tmp);
    float l1_scale = (float)((1.0 - mix) / (double)total);
    float ssim_scale = (float)(-0.5 * mix / n_crop);
    k_ssim_adj_h<<<blocks, 256, 0, s>>>(rendered, target, tmp, (int)h, (int)w, (int)c, t,
                                        l1_scale, ssim_scale, dL_drendered);
  }
  int rc = gsx_check_launch();
  if (rc) return rc;
  if (host_out) {
    double sm[2];
    CUDA_CHECK_RET(cudaMemcpyAsync(sm, sums, sizeof sm, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK_RET(cudaStreamSynchronize(s));
    double ssim = sm[0] / n_crop;  // mean over channels of per-channel crop means
    double l1 = sm[1] / (double)total;
    host_out[0] = (1.0 - mix) * l1 + mix * (1.0 - ssim) / 2.0;
    host_out[1] = l1;
    host_out[2] = ssim;
  }
  return GSX_OK;
}

extern "C" int gsx_iso_loss(const float* params, int64_t n, double r0, double lambda_s,
                            float* grad, double* loss_dev, void* stream) {
  if (n <= 0) return GSX_ERR_EMPTY;
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_CHECK_RET(cudaMemsetAsync(loss_dev, 0, sizeof(double), s));
  k_iso_loss<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(params, n, r0, lambda_s, loss_dev, grad);
  return gsx_check_launch();
}

extern "C" int gsx_adam_step(float* params, const float* grad, float* m, float* v, int64_t n,
                             const float* lr87, const float* lo87, double beta1, double beta2,
                             double eps, int64_t step, void* stream) {
  if (n <= 0 || step < 1) return GSX_ERR_ARG;
  int64_t count = n * GSX_NREC;
  const AdamArgs a{lr87, lo87, (float)beta1, (float)beta2, (float)eps,
                   (float)(1.0 / (1.0 - pow(beta1, (double)step))),
                   (float)(1.0 / sqrt(1.0 - pow(beta2, (double)step)))};
  cudaStream_t s = (cudaStream_t)stream;
  int64_t done = 0;
  if ((((uintptr_t)params | (uintptr_t)grad | (uintptr_t)m | (uintptr_t)v) & 15) == 0) {
    const int64_t n4 = count / 4;
    if (n4 > 0) {
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int64_t blocks =
          std::min<int64_t>((n4 + 256 * GSX_ADAM_ILP - 1) / (256 * GSX_ADAM_ILP),
                            (int64_t)sms * GSX_ADAM_CTAS);
      k_adam4<<<(unsigned)blocks, 256, 0, s>>>((float4*)params, (const float4*)grad, (float4*)m,
                                               (float4*)v, n4, a);
      done = 4 * n4;
    }
  }
  if (done < count)
    k_adam1<<<(unsigned)((count - done + 255) / 256), 256, 0, s>>>(params, grad, m, v, done,
                                                                   count, a);
  return gsx_check_launch();
}
