// lbvh.cu -- K5: linear BVH over Morton-ordered primitives (replaces the
// recursive binned-SAH Bvh of spatial.py:126-211, which takes 13 s at 100k).
//
// Topology: Karras (2012) -- internal node i's key range and split are found
// from the longest-common-prefix function delta over the sorted 63-bit codes
// (ties broken by index), one thread per internal node.  Boxes: bottom-up
// refit, one thread per leaf, the second thread to reach a node (atomic
// counter) merges its two children.  Leaves are single primitives in storage
// order; each internal node stores both child boxes (fp32, outward-rounded
// from the fp64 AABBs) so one 64-byte load tests both children.
#include <cooperative_groups.h>

#include "gsx_common.cuh"

namespace {

namespace cg = cooperative_groups;

__device__ inline int delta(const uint64_t* __restrict__ codes, int64_t n, int64_t i, int64_t j) {
  if (j < 0 || j >= n) return -1;
  uint64_t a = codes[i], b = codes[j];
  if (a == b) return 64 + __clz((unsigned)(i ^ j));
  return __clzll((long long)(a ^ b));
}

__global__ void k_karras(const uint64_t* __restrict__ codes, const int64_t* __restrict__ perm,
                         int64_t n, float4* nodes, int32_t* parents) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n - 1) return;
  int d = (delta(codes, n, i, i + 1) - delta(codes, n, i, i - 1)) >= 0 ? 1 : -1;
  int dmin = delta(codes, n, i, i - d);
  int64_t lmax = 2;
  while (delta(codes, n, i, i + lmax * d) > dmin) lmax <<= 1;
  int64_t l = 0;
  for (int64_t t = lmax >> 1; t >= 1; t >>= 1)
    if (delta(codes, n, i, i + (l + t) * d) > dmin) l += t;
  int64_t j = i + l * d;
  int dnode = delta(codes, n, i, j);
  int64_t s = 0;
  int64_t t = l;
  do {
    t = (t + 1) >> 1;
    if (delta(codes, n, i, i + (s + t) * d) > dnode) s += t;
  } while (t > 1);
  int64_t gamma = i + s * d + (d < 0 ? -1 : 0);
  int64_t lo = i < j ? i : j, hi = i < j ? j : i;
  // leaves reference storage indices (perm maps sorted position -> storage)
  bool lleaf = lo == gamma, rleaf = hi == gamma + 1;
  int32_t left = lleaf ? ~(int32_t)(perm ? perm[gamma] : gamma) : (int32_t)gamma;
  int32_t right = rleaf ? ~(int32_t)(perm ? perm[gamma + 1] : gamma + 1) : (int32_t)(gamma + 1);
  float4* nd = nodes + 4 * i;
  nd[0].w = __int_as_float(left);
  nd[1].w = __int_as_float(right);
  parents[lleaf ? (n - 1) + gamma : gamma] = (int32_t)i;
  parents[rleaf ? (n - 1) + gamma + 1 : gamma + 1] = (int32_t)i;
  if (i == 0) parents[0] = -1;
}

struct Box {
  float lo[3], hi[3];
};

__device__ inline Box leaf_box(const float* box32, int64_t prim) {
  Box b;
  for (int k = 0; k < 3; ++k) {
    b.lo[k] = box32[6 * prim + k];
    b.hi[k] = box32[6 * prim + 3 + k];
  }
  return b;
}

__device__ inline Box node_union(const float4* nodes, int32_t c) {
  // read with L1 bypass: written by another thread of this kernel
  const float4* nd = nodes + 4 * (int64_t)c;
  float4 a = __ldcg(nd + 0), b = __ldcg(nd + 1), e = __ldcg(nd + 2), f = __ldcg(nd + 3);
  Box r;
  r.lo[0] = fminf(a.x, e.x);
  r.lo[1] = fminf(a.y, e.y);
  r.lo[2] = fminf(a.z, e.z);
  r.hi[0] = fmaxf(b.x, f.x);
  r.hi[1] = fmaxf(b.y, f.y);
  r.hi[2] = fmaxf(b.z, f.z);
  return r;
}

#ifndef GSX_REFIT_ACQREL  // 0: the SC-fenced arrival (3M rebuild 2.60 vs 2.51 ms)
#define GSX_REFIT_ACQREL 1
#endif
__global__ void k_refit(const float* __restrict__ box32, int64_t n, float4* nodes,
                        const int32_t* __restrict__ parents, int32_t* flags) {
  int64_t leaf = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (leaf >= n) return;
  int32_t p = parents[(n - 1) + leaf];
  while (p >= 0) {
#if GSX_REFIT_ACQREL
    // one acquire-release arrival instead of two SC fences: the first
    // arrival's node stores are released by its increment, the second
    // arrival acquires them through the same counter
    int32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                 : "=r"(old)
                 : "l"(flags + p)
                 : "memory");
    if (old == 0) return;  // first arrival: sibling not ready
#else
    __threadfence();
    if (atomicAdd(&flags[p], 1) == 0) return;  // first arrival: sibling not ready
    __threadfence();
#endif
    float4* nd = nodes + 4 * (int64_t)p;
    int32_t cl = __float_as_int(__ldcg(&nd[0].w)), cr = __float_as_int(__ldcg(&nd[1].w));
    Box bl = cl < 0 ? leaf_box(box32, ~cl) : node_union(nodes, cl);
    Box br = cr < 0 ? leaf_box(box32, ~cr) : node_union(nodes, cr);
    __stcg(nd + 0, make_float4(bl.lo[0], bl.lo[1], bl.lo[2], __int_as_float(cl)));
    __stcg(nd + 1, make_float4(bl.hi[0], bl.hi[1], bl.hi[2], __int_as_float(cr)));
    __stcg(nd + 2, make_float4(br.lo[0], br.lo[1], br.lo[2], 0.f));
    __stcg(nd + 3, make_float4(br.hi[0], br.hi[1], br.hi[2], 0.f));
    p = parents[p];
  }
}

__global__ void k_single(const float* __restrict__ box32, float4* nodes, int32_t* parents,
                         float4* nodes4) {
  Box b = leaf_box(box32, 0);
  nodes[0] = make_float4(b.lo[0], b.lo[1], b.lo[2], __int_as_float(~0));
  nodes[1] = make_float4(b.hi[0], b.hi[1], b.hi[2], __int_as_float(GSX_NONE));
  nodes[2] = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
  nodes[3] = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.f);
  parents[0] = -1;
  parents[1] = 0;  // leaf 0 (slot n-1+0 == 0 would collide; n==1 uses slot 1)
  float inf = INFINITY;
  nodes4[0] = make_float4(b.lo[0], inf, inf, inf);
  nodes4[1] = make_float4(b.lo[1], inf, inf, inf);
  nodes4[2] = make_float4(b.lo[2], inf, inf, inf);
  nodes4[3] = make_float4(b.hi[0], -inf, -inf, -inf);
  nodes4[4] = make_float4(b.hi[1], -inf, -inf, -inf);
  nodes4[5] = make_float4(b.hi[2], -inf, -inf, -inf);
  int none = GSX_NONE;
  nodes4[6] = make_float4(__int_as_float(~0), __int_as_float(none), __int_as_float(none),
                          __int_as_float(none));
  nodes4[7] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// ---- 4-wide collapse ----------------------------------------------------------
// Depth-parity collapse (-DGSX_PARITY_COLLAPSE; measured: C3 35.5 vs 35.0 ms
// with the greedy collapse below).
// keep[i] = 1 for binary internal nodes at even depth (root included)
__global__ void k_keep_flags(const int32_t* __restrict__ parents, int64_t n, uint32_t* keep) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n - 1) return;
  int d = 0;
  for (int32_t p = parents[i]; p >= 0; p = parents[p]) ++d;
  keep[i] = (d & 1) ? 0u : 1u;
}

__global__ void k_collapse(const float4* __restrict__ nodes, const uint32_t* __restrict__ keep,
                           const uint32_t* __restrict__ idx4, int64_t n, float4* nodes4) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n - 1 || !keep[i]) return;
  float lo[3][4], hi[3][4];
  int32_t ch[4];
  int cnt = 0;
  auto add = [&](const float4& l, const float4& h, int32_t c) {
    lo[0][cnt] = l.x; lo[1][cnt] = l.y; lo[2][cnt] = l.z;
    hi[0][cnt] = h.x; hi[1][cnt] = h.y; hi[2][cnt] = h.z;
    ch[cnt++] = c;
  };
  const float4* nd = nodes + 4 * i;
  float4 q[4] = {nd[0], nd[1], nd[2], nd[3]};
  int32_t bc[2] = {__float_as_int(q[0].w), __float_as_int(q[1].w)};
  for (int k = 0; k < 2; ++k) {
    int32_t c = bc[k];
    if (c == GSX_NONE) continue;
    if (c < 0) {
      add(q[2 * k], q[2 * k + 1], c);
      continue;
    }
    // absorbed odd-depth node: take its two children
    const float4* cd = nodes + 4 * (int64_t)c;
    float4 r[4] = {cd[0], cd[1], cd[2], cd[3]};
    int32_t gc[2] = {__float_as_int(r[0].w), __float_as_int(r[1].w)};
    for (int m = 0; m < 2; ++m) {
      int32_t g = gc[m];
      if (g == GSX_NONE) continue;
      add(r[2 * m], r[2 * m + 1], g < 0 ? g : (int32_t)idx4[g]);
    }
  }
  for (; cnt < 4;) {
    lo[0][cnt] = lo[1][cnt] = lo[2][cnt] = INFINITY;
    hi[0][cnt] = hi[1][cnt] = hi[2][cnt] = -INFINITY;
    ch[cnt++] = GSX_NONE;
  }
  float4* o = nodes4 + 8 * (int64_t)idx4[i];
  o[0] = make_float4(lo[0][0], lo[0][1], lo[0][2], lo[0][3]);
  o[1] = make_float4(lo[1][0], lo[1][1], lo[1][2], lo[1][3]);
  o[2] = make_float4(lo[2][0], lo[2][1], lo[2][2], lo[2][3]);
  o[3] = make_float4(hi[0][0], hi[0][1], hi[0][2], hi[0][3]);
  o[4] = make_float4(hi[1][0], hi[1][1], hi[1][2], hi[1][3]);
  o[5] = make_float4(hi[2][0], hi[2][1], hi[2][2], hi[2][3]);
  o[6] = make_float4(__int_as_float(ch[0]), __int_as_float(ch[1]), __int_as_float(ch[2]),
                     __int_as_float(ch[3]));
  o[7] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// ---- SAH-greedy 4-wide collapse (default) ---------------------------------------
// Top down, one frontier level per launch: a BVH4 node starts from the two
// children of its binary node and repeatedly opens the child with the largest
// surface area until it has four (the standard greedy wide-BVH collapse).
// Compared with the depth-parity collapse it fills nodes (leaf children no
// longer waste slots) and opens big boxes first, so the packet traversal
// takes fewer node steps.  Child order inside a node is the binary in-order,
// so the candidate order is deterministic; BVH4 slot numbers are assigned by
// atomics (their placement, not the traversal, depends on scheduling).
struct QItem {
  int32_t bin;  // binary internal node
  int32_t out;  // its BVH4 slot
};

__device__ inline float half_area(const float4& lo, const float4& hi) {
  const float dx = hi.x - lo.x, dy = hi.y - lo.y, dz = hi.z - lo.z;
  return dx * dy + dy * dz + dz * dx;
}

// GSX_GREEDY_BASE: a level's new BVH4 slots are base + (its queue index), with
// base = the slots used before the level, so one atomic per child assigns
// both (0: a second counter for the slots)
#ifndef GSX_GREEDY_BASE
#define GSX_GREEDY_BASE 1
#endif
__device__ inline void greedy_item(const float4* __restrict__ nodes, const QItem it,
                                   QItem* __restrict__ qout, uint32_t* nout_p, uint32_t* n4_p,
                                   uint32_t base, float4* __restrict__ nodes4) {
  {
    float4 lo[4], hi[4];
    int32_t ref[4];
    const float4* nd = nodes + 4 * (int64_t)it.bin;
    lo[0] = nd[0];
    hi[0] = nd[1];
    lo[1] = nd[2];
    hi[1] = nd[3];
    ref[0] = __float_as_int(lo[0].w);
    ref[1] = __float_as_int(hi[0].w);
    int cnt = ref[1] == GSX_NONE ? 1 : 2;
    while (cnt < 4) {
      int best = -1;
      float ba = -1.f;
      for (int k = 0; k < cnt; ++k) {
        if (ref[k] < 0) continue;
        const float a = half_area(lo[k], hi[k]);
        if (a > ba) {
          ba = a;
          best = k;
        }
      }
      if (best < 0) break;
      const float4* cd = nodes + 4 * (int64_t)ref[best];
      const float4 l0 = cd[0], h0 = cd[1], l1 = cd[2], h1 = cd[3];
      const int32_t c0 = __float_as_int(l0.w), c1 = __float_as_int(h0.w);
      // replace entry `best` by (c0, c1), keeping the in-order sequence
      for (int k = cnt; k > best + 1; --k) {
        lo[k] = lo[k - 1];
        hi[k] = hi[k - 1];
        ref[k] = ref[k - 1];
      }
      lo[best] = l0;
      hi[best] = h0;
      ref[best] = c0;
      lo[best + 1] = l1;
      hi[best + 1] = h1;
      ref[best + 1] = c1;
      ++cnt;
    }
    int32_t ch[4];
    for (int k = 0; k < 4; ++k) {
      if (k >= cnt) {
        ch[k] = GSX_NONE;
        lo[k] = make_float4(INFINITY, INFINITY, INFINITY, 0.f);
        hi[k] = make_float4(-INFINITY, -INFINITY, -INFINITY, 0.f);
      } else if (ref[k] < 0) {
        ch[k] = ref[k];
      } else {
#if GSX_GREEDY_BASE
        const uint32_t q = atomicAdd(nout_p, 1u), slot = base + q;
        (void)n4_p;
#else
        const uint32_t q = atomicAdd(nout_p, 1u), slot = atomicAdd(n4_p, 1u);
        (void)base;
#endif
        qout[q] = QItem{ref[k], (int32_t)slot};
        ch[k] = (int32_t)slot;
      }
    }
    float4* o = nodes4 + 8 * (int64_t)it.out;
    o[0] = make_float4(lo[0].x, lo[1].x, lo[2].x, lo[3].x);
    o[1] = make_float4(lo[0].y, lo[1].y, lo[2].y, lo[3].y);
    o[2] = make_float4(lo[0].z, lo[1].z, lo[2].z, lo[3].z);
    o[3] = make_float4(hi[0].x, hi[1].x, hi[2].x, hi[3].x);
    o[4] = make_float4(hi[0].y, hi[1].y, hi[2].y, hi[3].y);
    o[5] = make_float4(hi[0].z, hi[1].z, hi[2].z, hi[3].z);
    o[6] = make_float4(__int_as_float(ch[0]), __int_as_float(ch[1]), __int_as_float(ch[2]),
                       __int_as_float(ch[3]));
    o[7] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Frontier counters rotate over three slots c[0..2] (= cnt[3..5]; cnt[2] is
// the 4-wide slot count): level L reads c[L % 3], appends to c[(L + 1) % 3]
// and clears c[(L + 2) % 3], which nobody touches during level L (it was level
// L - 1's input).  No memsets and no host reads between levels.
__global__ void k_greedy_level(const float4* __restrict__ nodes, QItem* qa, QItem* qb,
                               uint32_t* cnt, float4* __restrict__ nodes4, int level) {
  uint32_t* c = cnt + 3;
  uint32_t* b = cnt + 6;  // rotating level bases: b[L % 3] = slots used before level L's outputs
  const uint32_t nin = c[level % 3];
  const uint32_t base = b[(level + 2) % 3] + nin;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c[(level + 2) % 3] = 0u;
    b[level % 3] = base;
  }
  const QItem* qin = (level & 1) ? qb : qa;
  QItem* qout = (level & 1) ? qa : qb;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nin; i += gridDim.x * blockDim.x)
    greedy_item(nodes, qin[i], qout, c + (level + 1) % 3, cnt + 2, base, nodes4);
}

// The remaining levels from `first` on in one cooperative launch: a grid-wide
// barrier per level and the termination decided on the device (a frontier
// came out empty).  After GSX_GREEDY_LAUNCHED plain level launches the
// frontiers left are the LBVH's deep, narrow tail, where a barrier costs less
// than a launch; with no host synchronization a rebuild can be captured in a
// CUDA graph.
__global__ void k_greedy_all(const float4* __restrict__ nodes, QItem* qa, QItem* qb,
                             uint32_t* cnt, float4* __restrict__ nodes4, int first) {
  cg::grid_group grid = cg::this_grid();
  uint32_t* c = cnt + 3;
  if (c[first % 3] == 0u) return;  // the plain launches finished the tree
  for (int level = first; level < 4 * 64; ++level) {
    const QItem* qin = (level & 1) ? qb : qa;
    QItem* qout = (level & 1) ? qa : qb;
    uint32_t* cin = c + level % 3;
    uint32_t* cout = c + (level + 1) % 3;
    uint32_t* b = cnt + 6;
    const uint32_t nin = *(volatile uint32_t*)cin;
    const uint32_t base = *(volatile uint32_t*)(b + (level + 2) % 3) + nin;
    if (grid.thread_rank() == 0) {
      c[(level + 2) % 3] = 0u;
      b[level % 3] = base;
    }
    for (uint32_t i = (uint32_t)grid.thread_rank(); i < nin; i += (uint32_t)grid.size())
      greedy_item(nodes, qin[i], qout, cout, cnt + 2, base, nodes4);
    grid.sync();
    if (*(volatile uint32_t*)cout == 0u) break;  // the same value for every thread
  }
}

__global__ void k_greedy_init(QItem* q, uint32_t* cnt) {
  q[0] = QItem{0, 0};
  cnt[0] = 1;  // frontier A size
  cnt[1] = 0;  // frontier B size
  cnt[2] = 1;  // BVH4 slots used (root = 0)
  cnt[3] = 1;  // k_greedy_all's rotating frontier sizes
  cnt[4] = 0;
  cnt[5] = 0;
  cnt[6] = cnt[7] = 0;  // level bases (GSX_GREEDY_BASE): level 0's is b[2] + 1 = 1
  cnt[8] = 0;
}

__global__ void k_export(const float4* nodes, int64_t m, float* boxes, int32_t* children) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const float4* nd = nodes + 4 * i;
  float4 a = nd[0], b = nd[1], c = nd[2], d = nd[3];
  float* o = boxes + 12 * i;
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = b.x; o[4] = b.y; o[5] = b.z;
  o[6] = c.x; o[7] = c.y; o[8] = c.z; o[9] = d.x; o[10] = d.y; o[11] = d.z;
  children[2 * i] = __float_as_int(a.w);
  children[2 * i + 1] = __float_as_int(b.w);
}

}  // namespace

extern "C" size_t gsx_bvh_arena_bytes(int64_t n) { return bvh_arena_bytes_impl(n); }
extern "C" size_t gsx_bvh_workspace_bytes(int64_t n) {
  int64_t m = n > 1 ? n : 1;
  return 3 * gsx_align256(sizeof(int32_t) * m) +
         gsx_align256(sizeof(uint32_t) * gsx_scan_ws_elems(m)) +
         2 * gsx_align256(sizeof(QItem) * m) + 256;
}

// greedy collapse: level-synchronous frontier, one cooperative launch with
// device-side termination (k_greedy_all); without GSX_GREEDY_COOP, one launch
// per level and a host check for completion every GREEDY_BATCH levels
#ifndef GSX_GREEDY_COOP
#define GSX_GREEDY_COOP 1
#endif
#ifndef GSX_GREEDY_LAUNCHED  // plain level launches before the cooperative tail
#define GSX_GREEDY_LAUNCHED 24
#endif
static int greedy_collapse(const BvhView& bv, int64_t n, char* ws, cudaStream_t s) {
  constexpr int GREEDY_BATCH = 16;
  size_t seg = gsx_align256(sizeof(int32_t) * n);
  char* w = ws + 3 * seg + gsx_align256(sizeof(uint32_t) * gsx_scan_ws_elems(n));
  QItem* qa = (QItem*)w;
  QItem* qb = (QItem*)(w + gsx_align256(sizeof(QItem) * n));
  uint32_t* cnt = (uint32_t*)(w + 2 * gsx_align256(sizeof(QItem) * n));
  k_greedy_init<<<1, 1, 0, s>>>(qa, cnt);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)(sms * 8);
  const int launched = GSX_GREEDY_COOP ? GSX_GREEDY_LAUNCHED : 4 * 64;
  for (int level = 0; level < launched; ++level) {
    k_greedy_level<<<grid, 256, 0, s>>>(bv.nodes, qa, qb, cnt, bv.nodes4, level);
#if !GSX_GREEDY_COOP
    if ((level + 1) % GREEDY_BATCH == 0) {  // host-checked termination
      uint32_t h = 0;
      CUDA_CHECK_RET(cudaMemcpyAsync(&h, cnt + 3 + (level + 1) % 3, sizeof h,
                                     cudaMemcpyDeviceToHost, s));
      CUDA_CHECK_RET(cudaStreamSynchronize(s));
      if (h == 0) break;
    }
#endif
  }
#if GSX_GREEDY_COOP
  int per_sm = 0;
  CUDA_CHECK_RET(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_greedy_all, 256, 0));
  const float4* nodes = bv.nodes;
  float4* nodes4 = bv.nodes4;
  int first = launched;
  void* args[] = {(void*)&nodes, (void*)&qa, (void*)&qb, (void*)&cnt, (void*)&nodes4,
                  (void*)&first};
  CUDA_CHECK_RET(cudaLaunchCooperativeKernel((void*)k_greedy_all, dim3((unsigned)(sms * per_sm)),
                                             dim3(256), args, 0, s));
#endif
  return gsx_check_launch();
}

extern "C" int gsx_bvh_build(const void* scene_arena, const uint64_t* sorted_codes,
                             const int64_t* perm, int64_t n, void* bvh_arena, void* workspace,
                             void* stream) {
  if (n <= 0) return GSX_ERR_EMPTY;
  if (n >= 0x7fffffffLL) return GSX_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  SceneView sv = scene_view((void*)scene_arena, n);
  BvhView bv = bvh_view(bvh_arena, n);
  if (n == 1) {
    k_single<<<1, 1, 0, s>>>(sv.box32, bv.nodes, bv.parents, bv.nodes4);
    return gsx_check_launch();
  }
  char* w = (char*)workspace;
  size_t seg = gsx_align256(sizeof(int32_t) * n);
  int32_t* flags = (int32_t*)w;
  uint32_t* keep = (uint32_t*)(w + seg);
  uint32_t* idx4 = (uint32_t*)(w + 2 * seg);
  uint32_t* sums = (uint32_t*)(w + 3 * seg);
  CUDA_CHECK_RET(cudaMemsetAsync(flags, 0, sizeof(int32_t) * (n - 1), s));
  unsigned gi = (unsigned)((n - 1 + 255) / 256);
  k_karras<<<gi, 256, 0, s>>>(sorted_codes, perm, n, bv.nodes, bv.parents);
  k_refit<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sv.box32, n, bv.nodes, bv.parents, flags);
  // 4-wide collapse for the packet traversal
#ifdef GSX_PARITY_COLLAPSE
  k_keep_flags<<<gi, 256, 0, s>>>(bv.parents, n, keep);
  CUDA_CHECK_RET(cudaMemcpyAsync(idx4, keep, sizeof(uint32_t) * (n - 1), cudaMemcpyDeviceToDevice, s));
  gsx_exclusive_scan_u32(idx4, n - 1, sums, s);
  k_collapse<<<gi, 256, 0, s>>>(bv.nodes, keep, idx4, n, bv.nodes4);
  return gsx_check_launch();
#else
  (void)keep;
  (void)idx4;
  (void)sums;
  return greedy_collapse(bv, n, w, s);
#endif
}

// Re-derive the 4-wide nodes from the binary nodes already in the arena (after
// an external builder wrote them, e.g. the SAH experiment in
// profiles/experiments/).
extern "C" int gsx_bvh_collapse(void* bvh_arena, int64_t n, void* workspace, void* stream) {
  if (n <= 1) return n == 1 ? GSX_OK : GSX_ERR_EMPTY;
  BvhView bv = bvh_view(bvh_arena, n);
  return greedy_collapse(bv, n, (char*)workspace, (cudaStream_t)stream);
}

extern "C" int gsx_bvh_export(const void* bvh_arena, int64_t n, float* boxes, int32_t* children,
                              int32_t* parents, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  BvhView bv = bvh_view((void*)bvh_arena, n);
  int64_t m = bvh_internal_count(n);
  k_export<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(bv.nodes, m, boxes, children);
  if (parents)
    CUDA_CHECK_RET(cudaMemcpyAsync(parents, bv.parents, sizeof(int32_t) * (n > 1 ? 2 * n - 1 : 2),
                                   cudaMemcpyDeviceToDevice, s));
  return gsx_check_launch();
}
