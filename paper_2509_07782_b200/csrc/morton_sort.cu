// morton_sort.cu -- K2 Morton codes (spatial.py:28-92, fp64-exact quantization),
// K3 stable LSD radix sort of 64-bit keys (np.argsort(kind="stable"),
// spatial.py:92) and K4 permutation (Scene.apply_permutation, scene.py:74-80).
//
// Radix sort: 8 passes of 8 bits.  Each pass = per-tile digit histogram ->
// device-wide exclusive scan of the digit-major histogram (per scan tile,
// the scan tiles' totals added by the scatter) -> stable scatter.
// Stability inside a tile comes from warp-level ranking (__match_any_sync)
// over a contiguous 256-key sub-tile per warp, then an exclusive scan of the
// per-warp digit counts.  All HBM-bound: per pass 2 reads + 1 write of
// (key, value).
#include "gsx_common.cuh"

namespace {

constexpr int RADIX_BITS = 8;
constexpr int RADIX = 256;
constexpr int SORT_THREADS = 256;  // 8 warps
constexpr int SORT_WARPS = SORT_THREADS / 32;
// 12 / 16 keys per lane measured slower (3M rebuild 2.47 / 2.49 vs 2.42 ms)
#ifndef GSX_SORT_ITEMS
#define GSX_SORT_ITEMS 8
#endif
constexpr int ITEMS = GSX_SORT_ITEMS;  // keys per lane
constexpr int TILE = SORT_THREADS * ITEMS;  // 2048 keys
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_TILE = 2 * SCAN_THREADS;

__device__ inline uint64_t spread21(uint64_t x) {
  x &= 0x1FFFFFull;
  x = (x | (x << 32)) & 0x1F00000000FFFFull;
  x = (x | (x << 16)) & 0x1F0000FF0000FFull;
  x = (x | (x << 8)) & 0x100F00F00F00F00Full;
  x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
  x = (x | (x << 2)) & 0x1249249249249249ull;
  return x;
}
__device__ inline uint64_t compact21(uint64_t x) {
  x &= 0x1249249249249249ull;
  x = (x | (x >> 2)) & 0x10C30C30C30C30C3ull;
  x = (x | (x >> 4)) & 0x100F00F00F00F00Full;
  x = (x | (x >> 8)) & 0x1F0000FF0000FFull;
  x = (x | (x >> 16)) & 0x1F00000000FFFFull;
  x = (x | (x >> 32)) & 0x1FFFFFull;
  return x;
}

// spatial.py:81-86 quantize_points, one axis, fp64 round-to-nearest ops.
__device__ inline uint64_t quantize(double p, double lo, double ext) {
  double t = __ddiv_rn(__dsub_rn(p, lo), ext);
  double vq = __dmul_rn(t, 2097152.0);
  long long q = (long long)vq;  // astype(int64): truncation toward zero
  if (!(vq == vq)) q = 0;       // NaN guard (never produced by finite inputs)
  if (q < 0) q = 0;
  if (q > 2097151) q = 2097151;
  return (uint64_t)q;
}

struct Box3 {
  double lo[3], ext[3];
};

__device__ inline Box3 make_box(const double* lo3, const double* hi3) {
  Box3 b;
  for (int k = 0; k < 3; ++k) {
    b.lo[k] = lo3[k];
    double e = __dsub_rn(hi3[k], lo3[k]);
    b.ext[k] = e > 1e-30 ? e : 1e-30;  // np.maximum(hi - lo, 1e-30)
  }
  return b;
}

__global__ void k_morton(const double* __restrict__ means, int64_t n, const double* lo3,
                         const double* hi3, uint64_t* codes) {
  __shared__ Box3 b;
  if (threadIdx.x == 0) b = make_box(lo3, hi3);
  __syncthreads();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t c = 0;
  for (int k = 0; k < 3; ++k) c |= spread21(quantize(means[3 * i + k], b.lo[k], b.ext[k])) << k;
  codes[i] = c;
}

__global__ void k_morton_records(const float* __restrict__ params, int64_t n, const double* lo3,
                                 const double* hi3, uint64_t* codes) {
  __shared__ Box3 b;
  if (threadIdx.x == 0) b = make_box(lo3, hi3);
  __syncthreads();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t c = 0;
  for (int k = 0; k < 3; ++k)
    c |= spread21(quantize((double)params[GSX_NREC * i + k], b.lo[k], b.ext[k])) << k;
  codes[i] = c;
}

__global__ void k_encode(const int64_t* q, int64_t n, uint64_t* codes, gsx_dev_status* st) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t c = 0;
  for (int k = 0; k < 3; ++k) {
    int64_t v = q[3 * i + k];
    if (v < 0 || v > 2097151) {
      dev_fail(st, GSX_ERR_ARG, i);
      return;
    }
    c |= spread21((uint64_t)v) << k;
  }
  codes[i] = c;
}

__global__ void k_decode(const uint64_t* codes, int64_t n, int64_t* q) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t c = codes[i];
  for (int k = 0; k < 3; ++k) q[3 * i + k] = (int64_t)compact21(c >> k);
}

// ---- radix sort --------------------------------------------------------------
__global__ void __launch_bounds__(SORT_THREADS) k_hist(const uint64_t* __restrict__ keys,
                                                       int64_t n, int shift, int nblocks,
                                                       uint32_t* __restrict__ hist) {
  __shared__ uint32_t cnt[RADIX];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * TILE;
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    int64_t i = base + it * SORT_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&cnt[(keys[i] >> shift) & (RADIX - 1)], 1u);
  }
  __syncthreads();
  hist[(size_t)threadIdx.x * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

// exclusive scan over `len` u32 values in tiles of SCAN_TILE; block sums out.
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_tiles(uint32_t* data, int64_t len,
                                                             uint32_t* sums) {
  __shared__ uint32_t sh[SCAN_TILE];
  __shared__ uint32_t wsum[SCAN_THREADS / 32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int t = threadIdx.x;
  // each thread owns 2 consecutive elements
  int64_t i0 = base + 2 * t;
  uint32_t a = i0 < len ? data[i0] : 0u;
  uint32_t b = i0 + 1 < len ? data[i0 + 1] : 0u;
  uint32_t s = a + b;
  // inclusive warp scan of s
  uint32_t x = s;
  int lane = t & 31, w = t >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t ws = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, ws, o);
      if (lane >= o) ws += y;
    }
    wsum[lane] = ws;  // inclusive
  }
  __syncthreads();
  uint32_t excl = x - s + (w ? wsum[w - 1] : 0u);
  if (i0 < len) data[i0] = excl;
  if (i0 + 1 < len) data[i0 + 1] = excl + a;
  if (t == SCAN_THREADS - 1) sums[blockIdx.x] = excl + s;
  (void)sh;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_sums(uint32_t* sums, int count) {
  // single block, sequential over chunks of 1024
  __shared__ uint32_t wsum[SCAN_THREADS / 32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int base = 0; base < count; base += SCAN_THREADS) {
    int i = base + threadIdx.x;
    uint32_t v = i < count ? sums[i] : 0u;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      uint32_t ws = wsum[lane];
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, ws, o);
        if (lane >= o) ws += y;
      }
      wsum[lane] = ws;
    }
    __syncthreads();
    uint32_t excl = carry + x - v + (w ? wsum[w - 1] : 0u);
    if (i < count) sums[i] = excl;
    __syncthreads();
    if (threadIdx.x == SCAN_THREADS - 1) carry = excl + v;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_add(uint32_t* data, int64_t len,
                                                           const uint32_t* sums) {
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  uint32_t add = sums[blockIdx.x];
  for (int k = threadIdx.x; k < SCAN_TILE; k += SCAN_THREADS) {
    int64_t i = base + k;
    if (i < len) data[i] += add;
  }
}

template <bool FIRST, bool LAST>
__global__ void __launch_bounds__(SORT_THREADS)
    k_scatter(const uint64_t* __restrict__ keys_in, const int32_t* __restrict__ vals_in,
              int64_t n, int shift, int nblocks, const uint32_t* __restrict__ offsets,
              const uint32_t* __restrict__ tile_sums, uint64_t* __restrict__ keys_out,
              int32_t* __restrict__ vals_out, int64_t* __restrict__ perm_out) {
  __shared__ uint32_t wcnt[SORT_WARPS][RADIX];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < SORT_WARPS * RADIX; k += SORT_THREADS) (&wcnt[0][0])[k] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * TILE + (int64_t)w * (32 * ITEMS);
  uint64_t key[ITEMS];
  int32_t val[ITEMS];
  uint32_t rank[ITEMS];
  uint32_t dig[ITEMS];
  unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    int64_t i = base + it * 32 + lane;
    bool valid = i < n;
    key[it] = valid ? keys_in[i] : 0ull;
    val[it] = valid ? (FIRST ? (int32_t)i : vals_in[i]) : 0;
    uint32_t d = valid ? (uint32_t)((key[it] >> shift) & (RADIX - 1)) : (RADIX + lane);
    dig[it] = d;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    uint32_t before = valid ? wcnt[w][d] : 0u;
    rank[it] = before + __popc(peers & lt);
    __syncwarp();
    // the highest lane of each peer group bumps the counter
    if (valid && (peers >> lane) == 1u) wcnt[w][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // exclusive scan over warps, per digit
  {
    uint32_t run = 0;
    int d = threadIdx.x;
    for (int ww = 0; ww < SORT_WARPS; ++ww) {
      uint32_t c = wcnt[ww][d];
      wcnt[ww][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    int64_t i = base + it * 32 + lane;
    if (i < n) {
      uint32_t d = dig[it];
      // offsets holds the scan within each SCAN_TILE of the histogram;
      // tile_sums the scanned tile totals (k_scan_add folded in here)
      const size_t hi = (size_t)d * nblocks + blockIdx.x;
      uint32_t pos = offsets[hi] + tile_sums[hi / SCAN_TILE] + wcnt[w][d] + rank[it];
      keys_out[pos] = key[it];
      if (LAST)
        perm_out[pos] = (int64_t)val[it];
      else
        vals_out[pos] = val[it];
    }
  }
}

struct SortWs {
  uint64_t* keys_b;
  int32_t* vals_a;
  int32_t* vals_b;
  uint32_t* hist;
  uint32_t* sums;
};

inline int sort_nblocks(int64_t n) { return (int)((n + TILE - 1) / TILE); }
inline int64_t hist_len(int64_t n) { return (int64_t)RADIX * sort_nblocks(n); }
inline int scan_blocks(int64_t len) { return (int)((len + SCAN_TILE - 1) / SCAN_TILE); }

SortWs sort_ws(void* ws, int64_t n) {
  char* p = (char*)ws;
  SortWs s;
  size_t off = 0;
  s.keys_b = (uint64_t*)(p + off);
  off += gsx_align256(sizeof(uint64_t) * n);
  s.vals_a = (int32_t*)(p + off);
  off += gsx_align256(sizeof(int32_t) * n);
  s.vals_b = (int32_t*)(p + off);
  off += gsx_align256(sizeof(int32_t) * n);
  s.hist = (uint32_t*)(p + off);
  off += gsx_align256(sizeof(uint32_t) * hist_len(n));
  s.sums = (uint32_t*)(p + off);
  return s;
}

__global__ void k_permute(const float* __restrict__ params, const int64_t* __restrict__ perm,
                          int64_t n, float* __restrict__ out) {
  // one warp per record: 87 floats
  int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (row >= n) return;
  const float* src = params + GSX_NREC * perm[row];
  float* dst = out + GSX_NREC * row;
  for (int k = lane; k < GSX_NREC; k += 32) dst[k] = src[k];
}

__global__ void k_permute_uids(const int64_t* uids, const int64_t* perm, int64_t n,
                               int64_t* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = uids[perm[i]];
}

}  // namespace

extern "C" int gsx_morton_codes(const double* means, int64_t n, const double* lo3,
                                const double* hi3, uint64_t* codes, void* stream) {
  if (n <= 0) return GSX_OK;
  k_morton<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(means, n, lo3, hi3,
                                                                          codes);
  return gsx_check_launch();
}

extern "C" int gsx_morton_codes_records(const float* params, int64_t n, const double* lo3,
                                        const double* hi3, uint64_t* codes, void* stream) {
  if (n <= 0) return GSX_OK;
  k_morton_records<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      params, n, lo3, hi3, codes);
  return gsx_check_launch();
}

extern "C" int gsx_morton_encode(const int64_t* q, int64_t n, uint64_t* codes,
                                 gsx_dev_status* st, void* stream) {
  if (n <= 0) return GSX_OK;
  k_encode<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(q, n, codes, st);
  return gsx_check_launch();
}

extern "C" int gsx_morton_decode(const uint64_t* codes, int64_t n, int64_t* q, void* stream) {
  if (n <= 0) return GSX_OK;
  k_decode<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(codes, n, q);
  return gsx_check_launch();
}

extern "C" size_t gsx_sort_workspace_bytes(int64_t n) {
  if (n < 1) n = 1;
  return gsx_align256(sizeof(uint64_t) * n) + 2 * gsx_align256(sizeof(int32_t) * n) +
         gsx_align256(sizeof(uint32_t) * hist_len(n)) +
         gsx_align256(sizeof(uint32_t) * (scan_blocks(hist_len(n)) + 1));
}

extern "C" int gsx_sort_codes(const uint64_t* keys_in, int64_t n, uint64_t* keys_out,
                              int64_t* perm_out, void* workspace, void* stream) {
  if (n <= 0) return GSX_OK;
  if (n > 0x7fffffffLL) return GSX_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  SortWs w = sort_ws(workspace, n);
  int nb = sort_nblocks(n);
  int64_t hl = hist_len(n);
  int sb = scan_blocks(hl);
  const int passes = 64 / RADIX_BITS;
  // ping-pong: even passes write keys_b/vals_b? -> pass p reads src, writes dst
  const uint64_t* ksrc = keys_in;
  const int32_t* vsrc = nullptr;
  for (int p = 0; p < passes; ++p) {
    int shift = p * RADIX_BITS;
    uint64_t* kdst = (p % 2 == 0) ? w.keys_b : keys_out;
    int32_t* vdst = (p % 2 == 0) ? w.vals_b : w.vals_a;
    k_hist<<<nb, SORT_THREADS, 0, s>>>(ksrc, n, shift, nb, w.hist);
    k_scan_tiles<<<sb, SCAN_THREADS, 0, s>>>(w.hist, hl, w.sums);
    k_scan_sums<<<1, SCAN_THREADS, 0, s>>>(w.sums, sb);
    bool first = p == 0, last = p == passes - 1;
    if (first)
      k_scatter<true, false><<<nb, SORT_THREADS, 0, s>>>(
          ksrc, vsrc, n, shift, nb, w.hist, w.sums, kdst, vdst, nullptr);
    else if (last)
      k_scatter<false, true><<<nb, SORT_THREADS, 0, s>>>(
          ksrc, vsrc, n, shift, nb, w.hist, w.sums, kdst, nullptr, perm_out);
    else
      k_scatter<false, false><<<nb, SORT_THREADS, 0, s>>>(
          ksrc, vsrc, n, shift, nb, w.hist, w.sums, kdst, vdst, nullptr);
    ksrc = kdst;
    vsrc = vdst;
  }
  return gsx_check_launch();
}

extern "C" int gsx_permute(const float* params, const int64_t* uids_in, const int64_t* perm,
                           int64_t n, float* params_out, int64_t* uids_out, void* stream) {
  if (n <= 0) return GSX_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (params && params_out) {
    int64_t threads = n * 32;
    k_permute<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(params, perm, n, params_out);
  }
  if (uids_in && uids_out)
    k_permute_uids<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(uids_in, perm, n, uids_out);
  return gsx_check_launch();
}

size_t gsx_scan_ws_elems(int64_t len) { return (size_t)scan_blocks(len) + 1; }

void gsx_exclusive_scan_u32(uint32_t* data, int64_t len, uint32_t* sums, cudaStream_t s) {
  if (len <= 0) return;
  int sb = scan_blocks(len);
  k_scan_tiles<<<sb, SCAN_THREADS, 0, s>>>(data, len, sums);
  k_scan_sums<<<1, SCAN_THREADS, 0, s>>>(sums, sb);
  k_scan_add<<<sb, SCAN_THREADS, 0, s>>>(data, len, sums);
}
