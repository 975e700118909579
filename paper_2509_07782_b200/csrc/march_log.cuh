// march_log.cuh -- per-warp record of a training forward, consumed by the
// backward (no reference counterpart: the reference backward is autograd /
// finite differences).
//
// A training forward already computes everything the backward's replay pass
// would recompute: the warp's candidate stream per iteration and, per lane and
// sample, sigma_j and the colour sums W_j.  With 180 GB of HBM the cheapest
// backward keeps them: the logged forward appends one record per warp
// iteration (chunk) to a bump-allocated arena, the logged backward walks its
// warp's chain, replays only the compositing from the saved sums, and runs
// pass 2 over the saved lists -- no traversal, no density pass, no ESS.
//
// Arena (all offsets in bytes from the arena base, 128-byte aligned):
//   [LogHeader, 128 B][int64 first[nw]][uint32 complete[nw]] [records ...]
// Record = 128-byte LogRec header + body.  Only the lanes with samples in
// this iteration (`act` ballot; the depth-synchronous schedule leaves most
// lanes waiting in most iterations) are stored, in slot order
// slot = popc(act & lanes below):
//   kind 0 (full):  double tb[nact], double dt[nact], int32 mc[nact],
//                   float4 smp[mmax][nact] (sigma, W0, W1, W2), int32 list[count],
//                   uint32 umask[count] (each array 16-byte aligned, see LogLayout)
//   kind 1 (list):  int32 list[count], uint32 umask[count]  (a leading chunk of
//                   a candidate stream longer than the shared list; the kind-0
//                   record that follows holds the rest and the sample sums)
// umask[i] = the lanes (bit = lane) whose setup of list[i] succeeded in the
// forward: exactly the (lane, primitive) pairs the backward's pass 2 visits.
// A warp whose records did not fit (bump pointer past capacity) is marked
// complete = 0 and the backward recomputes it with the replay kernel.
#pragma once
#include "gsx_common.cuh"

namespace gsx {

struct LogHeader {
  unsigned long long head;  // bump pointer (bytes)
  unsigned long long cap;   // arena bytes
  unsigned int overflow;
  unsigned int nwarps;
  unsigned long long need;  // bytes every record would need (incl. those that did not fit)
  unsigned long long entries, pairs;  // logged list entries, sum of their use-mask popcounts
  unsigned int pad[20];
};
static_assert(sizeof(LogHeader) == 128, "LogHeader is one 128-byte line");

struct LogRec {
  long long next;  // offset of the warp's next record, -1 = last
  int count;       // list entries in this record
  int kind;        // 0 full, 1 list chunk
  int mmax;        // samples stored per active lane (warp max of mc), kind 0
  unsigned act;    // lanes stored (mc > 0), kind 0
  int pad[26];
};
static_assert(sizeof(LogRec) == 128, "LogRec is one 128-byte line");

__host__ __device__ inline long long log_round128(long long x) { return (x + 127) & ~127LL; }
__host__ __device__ inline long long log_round16(long long x) { return (x + 15) & ~15LL; }

// byte offsets inside a kind-0 body for nact stored lanes
struct LogLayout {
  long long dt, mc, smp, list, umask, bytes;
  __host__ __device__ LogLayout(int nact, int mmax, int count) {
    dt = 8LL * nact;
    mc = 16LL * nact;
    smp = log_round16(20LL * nact);
    list = smp + 16LL * nact * mmax;
    umask = list + log_round16(4LL * count);
    bytes = 128 + log_round128(umask + 4LL * count);
  }
};
// offset of umask in a kind-1 body and the record's bytes
__host__ __device__ inline long long log_chunk_umask(int count) { return log_round16(4LL * count); }
__host__ __device__ inline long long log_chunk_bytes(int count) {
  return 128 + log_round128(log_chunk_umask(count) + 4LL * count);
}
__host__ __device__ inline long long log_table_bytes(long long nw) {
  return log_round128(128 + 8 * nw) + log_round128(4 * nw);
}
__host__ __device__ inline long long* log_first(void* base) {
  return (long long*)((char*)base + 128);
}
__host__ __device__ inline unsigned* log_complete(void* base, long long nw) {
  return (unsigned*)((char*)base + log_round128(128 + 8 * nw));
}

// warp index within a launch over a tile subset: 8 warps per 16x16 tile
__device__ inline long long tile_warp_id(int per_tile, int threads) {
  return (long long)(blockIdx.x / per_tile) * 8 +
         (((blockIdx.x % per_tile) * threads + threadIdx.x) >> 5);
}

// Warp-uniform writer state of one warp of the logged forward.
struct LogWriter {
  char* base;
  long long first, prev;
  long long wid;
  long long need;  // bytes this warp's records need, logged or not
  unsigned entries, pairs;  // this lane's share of the logged entries / pairs
  bool on;
};

__device__ inline LogWriter log_writer(void* base, long long wid) {
  LogWriter w;
  w.base = (char*)base;
  w.first = -1;
  w.prev = -1;
  w.wid = wid;
  w.need = 0;
  w.entries = w.pairs = 0u;
  w.on = base != nullptr;
  return w;
}

// Allocate `bytes` for this warp and link it after the warp's previous record.
// Warp-uniform; returns the offset, or -1 (and turns the writer off) on overflow.
__device__ inline long long log_alloc(LogWriter& w, long long bytes) {
  w.need += bytes;
  if (!w.on) return -1;
  const int lane = threadIdx.x & 31;
  LogHeader* h = (LogHeader*)w.base;
  long long off = 0;
  if (lane == 0) {
    off = (long long)atomicAdd(&h->head, (unsigned long long)bytes);
    if (off + bytes > (long long)h->cap) {
      atomicExch(&h->overflow, 1u);
      off = -1;
    } else if (w.prev >= 0) {
      ((LogRec*)(w.base + w.prev))->next = off;
    }
  }
  off = __shfl_sync(0xffffffffu, off, 0);
  if (off < 0) {
    w.on = false;
    return -1;
  }
  if (w.first < 0) w.first = off;
  w.prev = off;
  return off;
}

__device__ inline void log_header(const LogWriter& w, long long off, int count, int kind,
                                  int mmax, unsigned act) {
  if ((threadIdx.x & 31) == 0) {
    LogRec* r = (LogRec*)(w.base + off);
    r->next = -1;
    r->count = count;
    r->kind = kind;
    r->mmax = mmax;
    r->act = act;
  }
}

// The log streams through L2 once each way: evict-first stores/loads keep
// the scene and BVH resident.
__device__ inline void log_list(LogWriter& w, int32_t* dst, const int32_t* list, uint32_t* mdst,
                                const uint32_t* umask, int count) {
  for (int i = threadIdx.x & 31; i < count; i += 32) {
    const uint32_t m = umask[i];
    __stcs(dst + i, list[i]);
    __stcs(mdst + i, m);
    w.entries += 1u;
    w.pairs += (unsigned)__popc(m);
  }
}

// The record writers run once per warp iteration inside the march loop; kept
// out of line (GSX_LOG_OOL) they stay out of the hot loop's instruction
// footprint, and only the per-lane sample-sum stores remain inline.
#ifndef GSX_LOG_OOL
#define GSX_LOG_OOL 0
#endif
#if GSX_LOG_OOL
#define GSX_LOG_ATTR __noinline__
#else
#define GSX_LOG_ATTR inline
#endif

// kind 1: a full shared-list chunk of a long candidate stream
__device__ GSX_LOG_ATTR void log_list_chunk(LogWriter& w, const int32_t* list,
                                            const uint32_t* umask, int count) {
  if (!w.base) return;
  const long long off = log_alloc(w, log_chunk_bytes(count));
  if (off < 0) return;
  log_header(w, off, count, 1, 0, 0u);
  char* body = w.base + off + 128;
  log_list(w, (int32_t*)body, list, (uint32_t*)(body + log_chunk_umask(count)), umask, count);
}

// kind 0 without the sample sums: allocates the record, writes its header,
// the lane block (tb, dt, mc) and the list; returns the lane's first
// sample-sum slot (nullptr for lanes without samples or on overflow) and the
// warp-uniform stride nact / row count mmax of the sample-sum array.
__device__ GSX_LOG_ATTR float4* log_full_head(LogWriter& w, const int32_t* list,
                                              const uint32_t* umask, int count, double tb,
                                              double dt, int mc, int& nact_out, int& mmax_out) {
  const int lane = threadIdx.x & 31;
  const unsigned act = __ballot_sync(0xffffffffu, mc > 0);
  const int nact = __popc(act);
  const int mmax = __reduce_max_sync(0xffffffffu, (unsigned)mc);
  nact_out = nact;
  mmax_out = 0;
  const LogLayout L(nact, mmax, count);
  const long long off = log_alloc(w, L.bytes);
  if (off < 0) return nullptr;
  mmax_out = mmax;
  log_header(w, off, count, 0, mmax, act);
  char* body = w.base + off + 128;
  log_list(w, (int32_t*)(body + L.list), list, (uint32_t*)(body + L.umask), umask, count);
  if (mc <= 0) return nullptr;
  const int slot = __popc(act & ((1u << lane) - 1u));
  __stcs((double*)body + slot, tb);
  __stcs((double*)(body + L.dt) + slot, dt);
  __stcs((int*)(body + L.mc) + slot, mc);
  return (float4*)(body + L.smp) + slot;
}

// kind 0: the active lanes' block, their per-sample sums, the last list chunk
__device__ inline void log_full(LogWriter& w, const int32_t* list, const uint32_t* umask,
                                int count, double tb, double dt, int mc,
                                const float (&sig)[16], const float (&W)[16][3]) {
  if (!w.base) return;
  int nact, mmax;
  float4* smp = log_full_head(w, list, umask, count, tb, dt, mc, nact, mmax);
  if (smp) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j < mmax)
        __stcs(smp + (long long)j * nact,
               j < mc ? make_float4(sig[j], W[j][0], W[j][1], W[j][2])
                      : make_float4(0.f, 0.f, 0.f, 0.f));
    }
  }
}

// kind 0 from the screened forward's sums (sums.get(j) = (sigma_j, W_j))
template <class Sums>
__device__ inline void log_full_sums(LogWriter& w, const int32_t* list, const uint32_t* umask,
                                     int count, double tb, double dt, int mc, const Sums& sums) {
  if (!w.base) return;
  int nact, mmax;
  float4* smp = log_full_head(w, list, umask, count, tb, dt, mc, nact, mmax);
  if (smp) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < mmax)
        __stcs(smp + (long long)j * nact, j < mc ? sums.get(j) : make_float4(0.f, 0.f, 0.f, 0.f));
  }
}

// end of the warp: publish its chain head and whether it is complete
__device__ inline void log_finish(const LogWriter& w, long long nw) {
  if (!w.base) return;
  unsigned long long e = w.entries, pr = w.pairs;
  for (int o = 16; o > 0; o >>= 1) {
    e += __shfl_xor_sync(0xffffffffu, e, o);
    pr += __shfl_xor_sync(0xffffffffu, pr, o);
  }
  if ((threadIdx.x & 31) != 0) return;
  if (e) {
    atomicAdd(&((LogHeader*)w.base)->entries, e);
    atomicAdd(&((LogHeader*)w.base)->pairs, pr);
  }
  log_first(w.base)[w.wid] = w.on ? w.first : -1;
  log_complete(w.base, nw)[w.wid] = w.on ? 1u : 0u;
  atomicAdd(&((LogHeader*)w.base)->need, (unsigned long long)w.need);
}

// L2 prefetch of a record's first `bytes` (the warp's next record, issued
// while the current one is processed)
__device__ inline void log_prefetch(const char* p, long long bytes) {
  for (long long o = (long long)(threadIdx.x & 31) * 128; o < bytes; o += 32 * 128)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p + o));
}

}  // namespace gsx
