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
//                   float4 smp[mmax][nact] (sigma, W0, W1, W2), int32 list[cap],
//                   uint32 umask[cap] (each array 16-byte aligned, see LogLayout)
//   kind 1 (list):  int32 list[cap], uint32 umask[cap]  (a leading chunk of
//                   a candidate stream longer than the shared list; the kind-0
//                   record that follows holds the rest and the sample sums)
// The arrays are sized for the traversed list (cap entries) and hold its
// first `count` entries that some lane used, in list order; umask[i] = those
// lanes (bit = lane): exactly the (lane, primitive) pairs the backward's
// pass 2 visits.
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
  unsigned long long entries, pairs;  // logged entries some lane used, sum of their mask popcounts
  unsigned int pad[20];
};
static_assert(sizeof(LogHeader) == 128, "LogHeader is one 128-byte line");

struct LogRec {
  long long next;  // offset of the warp's next record, -1 = last
  int count;       // list entries in this record
  int kind;        // 0 full, 1 list chunk
  int mmax;        // samples stored per active lane (warp max of mc), kind 0
  unsigned act;    // lanes stored (mc > 0), kind 0
  int cap;         // entries the list / umask arrays were sized for (>= count)
  int swidth;      // sample-sum array: 0 = nact columns by slot, 32 = all lanes by lane
  int pad[24];
};
static_assert(sizeof(LogRec) == 128, "LogRec is one 128-byte line");

__host__ __device__ inline long long log_round128(long long x) { return (x + 127) & ~127LL; }
__host__ __device__ inline long long log_round16(long long x) { return (x + 15) & ~15LL; }

// byte offsets inside a kind-0 body for nact stored lanes
struct LogLayout {
  long long dt, mc, smp, list, umask, bytes;
  // sw: columns of the sample-sum array (nact, or 32 when stored by lane)
  __host__ __device__ LogLayout(int nact, int mmax, int count, int sw = -1) {
    if (sw < 0) sw = nact;
    dt = 8LL * nact;
    mc = 16LL * nact;
    smp = log_round16(20LL * nact);
    list = smp + 16LL * sw * mmax;
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
  bool bulk;  // a bulk copy of shared-memory sums may still be reading them
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
  w.bulk = false;
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

__device__ inline void log_header(const LogWriter& w, long long off, int cap, int kind,
                                  int mmax, unsigned act) {
  if ((threadIdx.x & 31) == 0) {
    LogRec* r = (LogRec*)(w.base + off);
    r->next = -1;
    r->count = 0;  // log_close
    r->cap = cap;
    r->swidth = 0;
    r->kind = kind;
    r->mmax = mmax;
    r->act = act;
  }
}

// The log streams through L2 once each way: evict-first stores/loads keep
// the scene and BVH resident.
//
// A record is opened right after the traversal that produced its list (its
// entry count is the record's capacity; whether it is the chunk's last list
// -- kind 0, with the lane block and, at the end of the chunk, the sample
// sums -- or a leading kind-1 chunk is known then too).  The accumulation
// appends the entries some lane used, with their masks, straight into the
// record (log_keep) and log_close sets the count, so the forward needs no
// shared-memory compaction arrays.

// The open record of the current list (all null: not logged / overflow).
struct LogRecPtrs {
  LogRec* hdr;
  int32_t* list;
  uint32_t* umask;
  float4* smp;  // this lane's first sample-sum slot (kind 0, lanes with samples);
                // by-lane records: the array base (warp-uniform)
  int nact, mmax;
  bool by_lane;
};

// Warp-uniform.  final: the chunk's last list (kind 0, lane block written
// here: tb, dt, this lane's sample count mc); else a kind-1 list chunk.
// by_lane: the sample-sum array gets 32 columns indexed by lane (written in
// one bulk copy from the shared-memory sums, log_samples_bulk), or -- with
// GSX_LOG_BULK_MIN > 0 -- only when that many lanes have samples (less
// padding; C2 logged forward 17.1 ms with 24 vs 16.1 with 0 / always: the
// kernel then carries both store paths).
#ifndef GSX_LOG_BULK_MIN
#define GSX_LOG_BULK_MIN 0
#endif
__device__ inline LogRecPtrs log_open(LogWriter& w, int count, bool final, double tb,
                                      double dt, int mc, bool by_lane = false) {
  LogRecPtrs o{nullptr, nullptr, nullptr, nullptr, 0, 0, false};
  if (!w.base) return o;
  if (!final) {
    const long long off = log_alloc(w, log_chunk_bytes(count));
    if (off < 0) return o;
    log_header(w, off, count, 1, 0, 0u);
    char* body = w.base + off + 128;
    o.hdr = (LogRec*)(w.base + off);
    o.list = (int32_t*)body;
    o.umask = (uint32_t*)(body + log_chunk_umask(count));
    return o;
  }
  const int lane = threadIdx.x & 31;
  const unsigned act = __ballot_sync(0xffffffffu, mc > 0);
  const int nact = __popc(act);
  const int mmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)(mc > 0 ? mc : 0));
  by_lane = by_lane && nact >= GSX_LOG_BULK_MIN;
  const LogLayout L(nact, mmax, count, by_lane ? 32 : nact);
  const long long off = log_alloc(w, L.bytes);
  if (off < 0) return o;
  log_header(w, off, count, 0, mmax, act);
  if (by_lane && lane == 0) ((LogRec*)(w.base + off))->swidth = 32;
  char* body = w.base + off + 128;
  o.hdr = (LogRec*)(w.base + off);
  o.list = (int32_t*)(body + L.list);
  o.umask = (uint32_t*)(body + L.umask);
  o.nact = nact;
  o.mmax = mmax;
  if (mc > 0) {
    const int slot = __popc(act & ((1u << lane) - 1u));
    __stcs((double*)body + slot, tb);
    __stcs((double*)(body + L.dt) + slot, dt);
    __stcs((int*)(body + L.mc) + slot, mc);
    if (!by_lane) o.smp = (float4*)(body + L.smp) + slot;
  }
  if (by_lane) o.smp = (float4*)(body + L.smp);
  o.by_lane = by_lane;
  return o;
}

// The same out of line: keeps the record set-up out of the hot loop's
// instruction footprint.  C2 logged forward, shared-memory-sum kernel: 17.1
// vs 17.8 ms (its instruction-cache misses: no_instruction stalls 1.9 -> 0.8
// warps per issue); the 64-register kernels are faster with it inline
// (C4 register-sum 28.2 vs 29.4 ms).
static __device__ __noinline__ LogRecPtrs log_open_ool(LogWriter& w, int count, bool final,
                                                       double tb, double dt, int mc,
                                                       bool by_lane) {
  return log_open(w, count, final, tb, dt, mc, by_lane);
}

// By-lane records: the chunk's sums, acc[0 .. mmax)[32] float4 in shared
// memory (WarpSmemA), go to the record in one TMA bulk copy issued by lane 0
// (cp.async.bulk, completion tracked in a bulk group) instead of 16 vector
// stores per lane.  The shared source must not be rewritten before
// log_bulk_wait.  Warp-uniform.
__device__ inline bool log_samples_bulk(const LogRecPtrs& o, const float4* acc) {
  if (!o.by_lane || o.mmax == 0) return false;
  // every lane's shared-memory writes made visible to the async proxy, then
  // one lane issues the copy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    const unsigned src = (unsigned)__cvta_generic_to_shared(acc);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(o.smp),
                 "r"(src), "r"((unsigned)(o.mmax * 32 * 16))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  return true;
}
// the shared sums may be rewritten once the pending bulk copy has read them
__device__ inline void log_bulk_wait() {
  if ((threadIdx.x & 31) == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  __syncwarp();
}
// end of the warp: every bulk copy complete (source reads and global writes)
__device__ inline void log_bulk_drain() {
  if ((threadIdx.x & 31) == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncwarp();
}

// kept entry k of the open record: primitive p and the lanes um that used it
// (called by the one lane holding the entry)
__device__ inline void log_keep(LogWriter& w, const LogRecPtrs& o, int k, int32_t p,
                                uint32_t um) {
  if (!o.list) return;
  __stcs(o.list + k, p);
  __stcs(o.umask + k, um);
  w.entries += 1u;
  w.pairs += (unsigned)__popc(um);
}
// warp-uniform: the record holds `kept` entries
__device__ inline void log_close(const LogRecPtrs& o, int kept) {
  if (o.hdr && (threadIdx.x & 31) == 0) o.hdr->count = kept;
}

// kind 0: this lane's per-sample sums (get(j) = (sigma_j, W_j)) of the chunk
template <class Get>
__device__ inline void log_samples(const LogRecPtrs& o, int mc, Get&& get) {
#ifdef GSX_LOG_NO_SAMPLES  // timing experiment only: skip the sample-sum stores
  return;
#endif
  if (!o.smp) return;
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (j < o.mmax)
      __stcs(o.smp + (long long)j * o.nact, j < mc ? get(j) : make_float4(0.f, 0.f, 0.f, 0.f));
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
