// hkv_collect.cu — sort-free bucket grouping for sparse single-mode batches.
//
// The sorted pipeline (hkv_mutate.cu) groups a batch by bucket with a radix
// sort (three scatter passes over the batch) and a segment pass before the
// metadata engine runs.  When the batch is sparse over the buckets (C2: 1M
// ops over 2^20 buckets, ~1 op per touched bucket) a counting sort by bucket
// does the same job with arrays small enough to stay in L2 (4 B per bucket,
// 12-16 B per op):
//
//  k_count     one thread per op: hash, bucket, sentinel check, a
//              fire-and-forget add to the bucket's counter (lanes of a warp
//              on one bucket share one reduction: zipf hot buckets), and the
//              op's batch index in the bucket's `one` word -- exact for a
//              bucket that drew a single op, which is most of them (C2: 58 %
//              of touched buckets).
//  k_alloc     one thread per 4 consecutive buckets, block scan: a singleton
//              bucket's segment record is written right here (its op from
//              `one`, its key from the batch); every other touched bucket gets
//              a position range (the counter becomes the range's cursor) and
//              a segment descriptor, in bucket order inside each block.
//  k_scatter   one thread per op of a multi-op bucket: a slot of its bucket's
//              range (L2 atomic on the cursor) receives the batch index and
//              the key.  (A singleton's counter holds ~0; its op's add wraps
//              it back to zero.)
//  k_segfin    one thread per multi-op segment: puts the range's ops in batch order
//              (a sorting network over batch index << 4 | slot; the thread
//              owns the range, so in place), marks same-key runs and their
//              followers, resets the bucket's counter, and emits the segment
//              record — exactly what sort + k_segments + run_ends produce.
//              Segments of more than 16 ops (zipf hot buckets) go to k_big:
//              a block per segment, block radix sort or a bitmap over the
//              batch index space.
//  k_meta_tps  the sorted pipeline's metadata engine, unchanged (hkv_tps.cuh).
//
// Serial batch-order semantics (table.py:945-985) are the
// same as the sorted pipeline's: only the way segments are found changes.
// Every kernel after k_count reads its work size from the device (no host
// synchronisation).  Counters are per workspace and all-zero between calls
// (k_segfin / k_big reset them, also for a rejected batch).
#include <atomic>
#include <cstdlib>

#include <cub/cub.cuh>

#include "hkv_kernels.h"
#include "hkv_probe.cuh"
#include "hkv_tps.cuh"

namespace hkv {

constexpr int64_t kColMaxN = (int64_t)1 << 28;  // sort key = batch index << 4 | slot in range
constexpr int kSmallSeg = 16;                   // segments sorted by one thread
constexpr unsigned kSkewBig = 8;                // big segments in the last batch that mean "skewed"
constexpr int kCountThreads = 256, kCountPer = 4;
constexpr int kAllocThreads = 256, kAllocPer = 4;

// Segment descriptor: a touched bucket, its position range and the slot of
// its segment record (singleton list, multi-op list, or big list index).
struct SegDesc {
  uint32_t b, p0, cnt, slot;
};

// ---------------------------------------------------------------------------
// k_count
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kCountThreads) k_count(TableDev t, const uint64_t* __restrict__ keys, int64_t n,
                                                         uint32_t* __restrict__ cnt, uint32_t* __restrict__ one,
                                                         Scalars* sc) {
  griddep_wait();
  const int64_t i0 = (int64_t)blockIdx.x * kCountThreads * kCountPer + threadIdx.x;
  if (i0 == 0) {
    sc->first_ev = 0xFFFFFFFFu;
    sc->size_before = (long long)*t.size;
    if (role_forbids_mutation(t)) atomicOr(&sc->err, 2);
  }
  const unsigned lane = threadIdx.x & 31u;
  uint64_t key[kCountPer];
  bool bad = false;
#pragma unroll
  for (int k = 0; k < kCountPer; k++) {
    const int64_t i = i0 + (int64_t)k * kCountThreads;
    key[k] = i < n ? keys[i] : 0;
  }
#pragma unroll
  for (int k = 0; k < kCountPer; k++) {
    const int64_t i = i0 + (int64_t)k * kCountThreads;
    bad |= i < n && key[k] >= kLockedKey;  // table.py:168-169: the batch then mutates nothing
    const uint32_t b = i < n ? (uint32_t)(fmix64(key[k]) & t.mask) : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(kFull, b);
    if (b != 0xFFFFFFFFu && lane == (unsigned)(__ffs(peers) - 1)) {
      atomicAdd(cnt + b, (unsigned)__popc(peers));
      one[b] = (uint32_t)i;  // the bucket's op if it is its only one
    }
  }
  if (bad) atomicOr(&sc->err, 1);
}

// ---------------------------------------------------------------------------
// k_alloc: counters -> position ranges + segment descriptors
// ---------------------------------------------------------------------------
struct AllocCounts {
  uint32_t s, p;      // segments, positions
  uint32_t one, mul;  // singleton records, multi-op records (big segments included)
  uint32_t big;       // big segments (more than kSmallSeg ops)
};
struct AllocSum {
  __device__ AllocCounts operator()(const AllocCounts& a, const AllocCounts& b) const {
    return AllocCounts{a.s + b.s, a.p + b.p, a.one + b.one, a.mul + b.mul, a.big + b.big};
  }
};

__global__ void __launch_bounds__(kAllocThreads) k_alloc(int64_t buckets, const uint64_t* __restrict__ keys,
                                                         uint32_t* __restrict__ cnt, const uint32_t* __restrict__ one,
                                                         SegDesc* __restrict__ segs, SegDesc* __restrict__ bigs,
                                                         SegRec* __restrict__ recs, int64_t cap, Scalars* sc) {
  griddep_wait();
  typedef cub::BlockScan<AllocCounts, kAllocThreads> BS;
  __shared__ typename BS::TempStorage tmp;
  __shared__ AllocCounts base_sh;
  const int64_t b0 = ((int64_t)blockIdx.x * kAllocThreads + threadIdx.x) * kAllocPer;
  uint32_t c[kAllocPer];
  const bool full = b0 + kAllocPer <= buckets;
  if (full) {
    const uint4 x = *reinterpret_cast<const uint4*>(cnt + b0);
    c[0] = x.x; c[1] = x.y; c[2] = x.z; c[3] = x.w;
  } else {
#pragma unroll
    for (int k = 0; k < kAllocPer; k++) c[k] = b0 + k < buckets ? cnt[b0 + k] : 0;
  }
  const bool bad = sc->err != 0;
  // singletons: their op and key, loads in flight with the scan
  uint32_t oi[kAllocPer];
  uint64_t ok[kAllocPer];
#pragma unroll
  for (int k = 0; k < kAllocPer; k++) oi[k] = c[k] == 1 ? one[b0 + k] : 0;
#pragma unroll
  for (int k = 0; k < kAllocPer; k++) ok[k] = (c[k] == 1 && !bad) ? keys[oi[k]] : 0;
  AllocCounts mine{0, 0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < kAllocPer; k++) {
    mine.s += c[k] > 1;
    mine.p += c[k] > 1 ? c[k] : 0;
    mine.one += c[k] == 1;
    mine.mul += c[k] > 1;
    mine.big += c[k] > (uint32_t)kSmallSeg;
  }
  AllocCounts off, tot;
  BS(tmp).ExclusiveScan(mine, off, AllocCounts{0, 0, 0, 0, 0}, AllocSum(), tot);
  if (threadIdx.x == 0) {
    // (descriptors, positions), (singletons, multi) and big: independent atomics
    unsigned long long r0 = 0, r1 = 0;
    unsigned rb = 0;
    if (tot.s) r0 = atomicAdd(&sc->alloc_pack, (unsigned long long)tot.s | ((unsigned long long)tot.p << 32));
    if (tot.one | tot.mul)
      r1 = atomicAdd(&sc->seg_pack, (unsigned long long)tot.one | ((unsigned long long)tot.mul << 32));
    if (tot.big) rb = atomicAdd(&sc->nbig, tot.big);
    base_sh = AllocCounts{(uint32_t)r0, (uint32_t)(r0 >> 32), (uint32_t)r1, (uint32_t)(r1 >> 32), rb};
  }
  __syncthreads();
  if (!(mine.s | mine.one)) return;
  AllocCounts at = AllocSum()(base_sh, off);
  uint32_t cur[kAllocPer];
#pragma unroll
  for (int k = 0; k < kAllocPer; k++) {
    cur[k] = 0;
    if (c[k] == 1) {
      // the counter holds ~0: the op's add in k_scatter wraps it to zero
      cur[k] = 0xFFFFFFFFu;
      if (!bad) {
        SegRec r;
        r.key = ok[k];
        r.p = 0;
        r.b = (uint32_t)(b0 + k);
        r.i = oi[k];
        r.flags = digest_of(fmix64(ok[k])) << 8;
        recs[at.one] = r;
      }
      at.one++;
    } else if (c[k] > 1) {
      cur[k] = at.p;  // the counter becomes the range's cursor
      const SegDesc d{(uint32_t)(b0 + k), at.p, c[k], at.mul++};
      segs[at.s++] = d;
      if (c[k] > (uint32_t)kSmallSeg) bigs[at.big++] = d;
      at.p += c[k];
    }
  }
  if (full) {
    *reinterpret_cast<uint4*>(cnt + b0) = make_uint4(cur[0], cur[1], cur[2], cur[3]);
  } else {
    for (int k = 0; k < kAllocPer; k++)
      if (b0 + k < buckets) cnt[b0 + k] = cur[k];
  }
}

// ---------------------------------------------------------------------------
// k_scatter: each op takes a slot of its bucket's range
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kCountThreads) k_scatter(TableDev t, const uint64_t* __restrict__ keys, int64_t n,
                                                           uint32_t* __restrict__ cur, uint32_t* __restrict__ sidx,
                                                           uint64_t* __restrict__ skeys) {
  griddep_wait();
  const int64_t i0 = (int64_t)blockIdx.x * kCountThreads * kCountPer + threadIdx.x;
  const unsigned lane = threadIdx.x & 31u;
  uint64_t key[kCountPer];
  uint32_t b[kCountPer], base[kCountPer];
  unsigned peers[kCountPer];
#pragma unroll
  for (int k = 0; k < kCountPer; k++) {
    const int64_t i = i0 + (int64_t)k * kCountThreads;
    key[k] = i < n ? keys[i] : 0;
  }
#pragma unroll
  for (int k = 0; k < kCountPer; k++) {
    const int64_t i = i0 + (int64_t)k * kCountThreads;
    b[k] = i < n ? (uint32_t)(fmix64(key[k]) & t.mask) : 0xFFFFFFFFu;
    peers[k] = __match_any_sync(kFull, b[k]);
    base[k] = 0;
    if (b[k] != 0xFFFFFFFFu && lane == (unsigned)(__ffs(peers[k]) - 1))
      base[k] = atomicAdd(cur + b[k], (unsigned)__popc(peers[k]));
  }
#pragma unroll
  for (int k = 0; k < kCountPer; k++) {
    const uint32_t bs = __shfl_sync(kFull, base[k], __ffs(peers[k]) - 1);
    if (b[k] == 0xFFFFFFFFu) continue;
    if (bs == 0xFFFFFFFFu) continue;  // a singleton (recorded by k_alloc); its counter is zero again
    const uint32_t p = bs + __popc(peers[k] & ((1u << lane) - 1u));
    sidx[p] = (uint32_t)(i0 + (int64_t)k * kCountThreads);
    skeys[p] = key[k];
  }
}

// ---------------------------------------------------------------------------
// k_segfin: order each segment's ops by batch index, emit the segment
// ---------------------------------------------------------------------------
// Sorted-segment outputs (the contract of k_segments + run_ends in
// hkv_mutate.cu).
struct SegOut {
  uint32_t* sb;        // bucket of each sorted position
  uint32_t* sidx;      // batch index of each sorted position
  uint64_t* skeys;     // key of each sorted position
  uint32_t* run_end;   // last position of the same-key run through p
  uint8_t* outcomes;   // followers of a run: the collapsed outcome up front
  uint32_t* vrow;      //   and no value row
  SegRec* recs;        // singletons from the front, multi-op segments from the back
  int64_t cap;
  uint8_t fcode;
};

__device__ __forceinline__ void cswap(uint32_t& a, uint32_t& b) {
  const uint32_t lo = a < b ? a : b, hi = a < b ? b : a;
  a = lo;
  b = hi;
}
// Batcher's odd-even merge network for the first 8 keys (19 compare-exchanges)
template <int N>
__device__ __forceinline__ void sort8(uint32_t (&v)[N]) {
  cswap(v[0], v[1]); cswap(v[2], v[3]); cswap(v[4], v[5]); cswap(v[6], v[7]);
  cswap(v[0], v[2]); cswap(v[1], v[3]); cswap(v[4], v[6]); cswap(v[5], v[7]);
  cswap(v[1], v[2]); cswap(v[5], v[6]);
  cswap(v[0], v[4]); cswap(v[1], v[5]); cswap(v[2], v[6]); cswap(v[3], v[7]);
  cswap(v[2], v[4]); cswap(v[3], v[5]);
  cswap(v[1], v[2]); cswap(v[3], v[4]); cswap(v[5], v[6]);
}
// bitonic network for 16 keys (segments of 9..16 ops only)
__device__ __forceinline__ void sort16(uint32_t (&v)[16]) {
#pragma unroll
  for (int k = 2; k <= 16; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < 16; i++) {
        const int l = i ^ j;
        if (l > i) {
          if ((i & k) == 0) cswap(v[i], v[l]);
          else cswap(v[l], v[i]);
        }
      }
}

constexpr int kSegfinThreads = 256;

__global__ void __launch_bounds__(kSegfinThreads) k_segfin(const SegDesc* __restrict__ segs, uint32_t* __restrict__ cur,
                                                           SegOut o, Scalars* sc) {
  griddep_wait();
  // per-thread staging of a multi-op range (batch index, key), sorted in place
  __shared__ uint32_t ish[kSmallSeg * kSegfinThreads];
  __shared__ uint64_t ksh[kSmallSeg * kSegfinThreads];
  uint32_t* is = ish + threadIdx.x;  // entry q at is[q * kSegfinThreads]: no bank conflicts
  uint64_t* ks = ksh + threadIdx.x;
  const bool bad = sc->err != 0;
  const uint32_t nsegs = sc->nsegd;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nsegs; j += gridDim.x * blockDim.x) {
    const SegDesc d = segs[j];
    if (d.cnt > (uint32_t)kSmallSeg) continue;  // k_big
    cur[d.b] = 0;  // clean for the next batch
    if (bad) continue;
    const uint32_t c = d.cnt;
    // stage (index, key) pairs, loads in flight together
#pragma unroll 4
    for (uint32_t q = 0; q < c; q++) {
      is[q * kSegfinThreads] = o.sidx[d.p0 + q];
      ks[q * kSegfinThreads] = o.skeys[d.p0 + q];
    }
    // insertion sort by batch index (segments are short: mostly 2-3 ops)
    for (uint32_t q = 1; q < c; q++) {
      const uint32_t iv = is[q * kSegfinThreads];
      const uint64_t kv = ks[q * kSegfinThreads];
      uint32_t r = q;
      while (r > 0 && is[(r - 1) * kSegfinThreads] > iv) {
        is[r * kSegfinThreads] = is[(r - 1) * kSegfinThreads];
        ks[r * kSegfinThreads] = ks[(r - 1) * kSegfinThreads];
        r--;
      }
      is[r * kSegfinThreads] = iv;
      ks[r * kSegfinThreads] = kv;
    }
    // same-key runs: run_end[p] = last position of p's run; followers collapse
    uint32_t re = d.p0 + c - 1;
    bool runs = false;
    uint64_t knext = 0;
    for (int q = (int)c - 1; q >= 0; q--) {
      const uint32_t p = d.p0 + (uint32_t)q;
      const uint64_t k = ks[q * kSegfinThreads];
      if ((uint32_t)q + 1 < c && knext != k) re = p;
      const uint32_t i = is[q * kSegfinThreads];
      o.sb[p] = d.b;
      o.sidx[p] = i;
      o.skeys[p] = k;
      o.run_end[p] = re;
      if (q > 0 && ks[(q - 1) * kSegfinThreads] == k) {
        o.outcomes[i] = o.fcode;
        o.vrow[i] = kNoRow;
        runs = true;
      }
      knext = k;
    }
    if (runs) sc->has_runs = 1;
    SegRec r;
    r.key = ks[0];
    r.p = d.p0;
    r.b = d.b;
    r.i = is[0];
    r.flags = 1u | (digest_of(fmix64(r.key)) << 8);
    o.recs[o.cap - 1 - d.slot] = r;
  }
}

// ---------------------------------------------------------------------------
// k_big: segments of more than kSmallSeg ops (zipf hot buckets)
// ---------------------------------------------------------------------------
// Emit one sorted range [p0, p0 + cnt) whose batch indices are in o.sidx:
// keys, buckets, runs, followers, the segment record.
__device__ void big_emit(const uint64_t* __restrict__ keys, uint32_t b, uint32_t p0, uint32_t cnt, uint32_t slot,
                         const SegOut& o, Scalars* sc, uint32_t* carry_sh) {
  // run_end by a reverse walk in chunks: a chunk's last run continues into the
  // next chunk's first position, so chunks go from the back with a carry
  const int nt = blockDim.x;
  bool runs = false;
  uint32_t carry = p0 + cnt - 1;  // run end carried in from the chunk after
  for (int64_t c0 = ((int64_t)(cnt - 1) / nt) * nt; c0 >= 0; c0 -= nt) {
    const int64_t q = c0 + threadIdx.x;
    const bool live = q < (int64_t)cnt;
    uint64_t k = 0, kn = 0;
    uint32_t i = 0;
    if (live) {
      i = o.sidx[p0 + q];
      k = keys[i];
      if (q + 1 < (int64_t)cnt) kn = keys[o.sidx[p0 + q + 1]];
    }
    const bool brk = live && (q + 1 >= (int64_t)cnt || kn != k);
    // first break at or after q inside this chunk: a min over the threads >= me
    uint32_t v = brk ? (uint32_t)(p0 + q) : 0xFFFFFFFFu;
    __syncthreads();
    carry_sh[threadIdx.x] = v;
    __syncthreads();
    for (int d = 1; d < nt; d <<= 1) {  // suffix min (Hillis-Steele)
      const uint32_t w = threadIdx.x + d < nt ? carry_sh[threadIdx.x + d] : 0xFFFFFFFFu;
      __syncthreads();
      v = w < v ? w : v;
      carry_sh[threadIdx.x] = v;
      __syncthreads();
    }
    if (live) {
      const uint32_t p = p0 + (uint32_t)q;
      o.sb[p] = b;
      o.skeys[p] = k;
      o.run_end[p] = v != 0xFFFFFFFFu ? v : carry;
      if (q > 0 && keys[o.sidx[p - 1]] == k) {
        o.outcomes[i] = o.fcode;
        o.vrow[i] = kNoRow;
        runs = true;
      }
    }
    const uint32_t first = carry_sh[0];
    __syncthreads();
    if (first != 0xFFFFFFFFu) carry = first;
  }
  if (__syncthreads_or(runs) && threadIdx.x == 0) sc->has_runs = 1;
  if (threadIdx.x == 0) {
    const uint32_t i0 = o.sidx[p0];
    SegRec r;
    r.key = keys[i0];
    r.p = p0;
    r.b = b;
    r.i = i0;
    r.flags = 1u | (digest_of(fmix64(r.key)) << 8);
    o.recs[o.cap - 1 - slot] = r;
  }
}

// One block per big segment (grid-stride over the list).  Ranges of up to
// kBigSmall ops sort with a block radix sort; larger ones mark their batch
// indices in a bitmap over a window of the index space and read them out in
// order (staged in the range's skeys slots, which big_emit rewrites).
constexpr int kBigThreads = 512, kBigItems = 4, kBigSmall = kBigThreads * kBigItems;
constexpr int kBigWinWords = 32768;  // 128 KB of dynamic shared memory: 2^20 batch indices per window

__global__ void __launch_bounds__(kBigThreads) k_big(const uint64_t* __restrict__ keys, int64_t n,
                                                     const SegDesc* __restrict__ bigs, uint32_t* __restrict__ cur,
                                                     SegOut o, int end_bit, Scalars* sc) {
  griddep_wait();
  const unsigned nbig = sc->nbig;
  if (nbig == 0) return;
  extern __shared__ uint32_t bm[];
  typedef cub::BlockRadixSort<uint32_t, kBigThreads, kBigItems> BRS;
  typedef cub::BlockScan<uint32_t, kBigThreads> BS;
  __shared__ union {
    typename BRS::TempStorage sort;
    typename BS::TempStorage scan;
  } tmp;
  __shared__ uint32_t carry_sh[kBigThreads];
  constexpr int kWPT = kBigWinWords / kBigThreads;  // bitmap words per thread
  const bool bad = sc->err != 0;
  for (unsigned j = blockIdx.x; j < nbig; j += gridDim.x) {
    const SegDesc d = bigs[j];
    const uint32_t p0 = d.p0, cnt = d.cnt;
    if (threadIdx.x == 0) cur[d.b] = 0;  // clean for the next batch
    if (bad) continue;
    if (cnt <= (uint32_t)kBigSmall) {
      uint32_t v[kBigItems];
#pragma unroll
      for (int k = 0; k < kBigItems; k++) {
        const uint32_t q = threadIdx.x * kBigItems + k;
        v[k] = q < cnt ? o.sidx[p0 + q] : 0xFFFFFFFFu;
      }
      __syncthreads();
      BRS(tmp.sort).Sort(v, 0, end_bit);
#pragma unroll
      for (int k = 0; k < kBigItems; k++) {
        const uint32_t q = threadIdx.x * kBigItems + k;
        if (q < cnt) o.sidx[p0 + q] = v[k];
      }
    } else {
      uint32_t written = 0;
      for (int64_t w0 = 0; w0 < n; w0 += (int64_t)kBigWinWords * 32) {
        for (int k = threadIdx.x; k < kBigWinWords; k += kBigThreads) bm[k] = 0;
        __syncthreads();
        for (uint32_t q = threadIdx.x; q < cnt; q += kBigThreads) {
          const int64_t i = o.sidx[p0 + q];
          if (i >= w0 && i < w0 + (int64_t)kBigWinWords * 32) {
            const uint32_t r = (uint32_t)(i - w0);
            atomicOr(bm + (r >> 5), 1u << (r & 31));
          }
        }
        __syncthreads();
        uint32_t pc = 0;
        for (int k = 0; k < kWPT; k++) pc += __popc(bm[threadIdx.x * kWPT + k]);
        uint32_t off, total;
        BS(tmp.scan).ExclusiveSum(pc, off, total);
        uint32_t out = p0 + written + off;
        for (int k = 0; k < kWPT; k++) {
          uint32_t m = bm[threadIdx.x * kWPT + k];
          while (m) {
            const int bit = __ffs(m) - 1;
            m &= m - 1;
            o.skeys[out++] = (uint64_t)w0 + (uint64_t)(threadIdx.x * kWPT + k) * 32 + (uint64_t)bit;
          }
        }
        written += total;
        __syncthreads();
      }
      for (uint32_t q = threadIdx.x; q < cnt; q += kBigThreads) o.sidx[p0 + q] = (uint32_t)o.skeys[p0 + q];
    }
    __syncthreads();
    big_emit(keys, d.b, p0, cnt, d.slot, o, sc, carry_sh);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
bool collect_eligible(int64_t n, int log2_buckets, unsigned last_big_segments) {
  // sparse batches: about one op per touched bucket.  Dense batches
  // (configs[0]: 128 ops per bucket) keep the sorted pipeline and its
  // long-segment engine, and so do batches after a skewed one (zipf: hot
  // buckets turn the counting atomics into long same-address chains).
  static const int mode = [] {
    const char* e = getenv("HKV_COLLECT");
    return e ? atoi(e) : 1;
  }();
  if (mode == 0 || n <= 0 || n >= kColMaxN) return false;
  if (mode == 2) return true;  // HKV_COLLECT=2: every batch (tests)
  return (n >> log2_buckets) < 2 && last_big_segments <= kSkewBig;
}

cudaError_t run_collect(const TableDev& t, OpArgs a, int64_t n, int log2_buckets, Workspace& ws, cudaStream_t s,
                        int num_sms, uint8_t fcode) {
  cudaError_t e;
  const int64_t buckets = (int64_t)1 << log2_buckets;
  if (ws.col_buckets != buckets) {
    if (ws.col) cudaFree(ws.col);
    ws.col = nullptr;
    ws.col_buckets = 0;
    // counters (zero between calls) + each bucket's `one` word
    if ((e = cudaMalloc((void**)&ws.col, 2 * (size_t)buckets * sizeof(uint32_t)))) return e;
    if ((e = cudaMemsetAsync(ws.col, 0, 2 * (size_t)buckets * sizeof(uint32_t), s))) return e;
    ws.col_buckets = buckets;
  }
  uint32_t* cnt = ws.col;
  uint32_t* one = ws.col + buckets;
  SegDesc* segs = reinterpret_cast<SegDesc*>(ws.segd);
  SegDesc* bigs = reinterpret_cast<SegDesc*>(ws.aux);  // at most n / 17 entries of 16 B
  SegOut o;
  o.sb = ws.sbkt;
  o.sidx = ws.sidx;
  o.skeys = ws.skeys;
  o.run_end = ws.seg;
  o.outcomes = a.outcomes;
  o.vrow = ws.vrow;
  o.recs = reinterpret_cast<SegRec*>(ws.skey);
  o.cap = n;
  o.fcode = fcode;
  const unsigned ob = (unsigned)((n + kCountThreads * kCountPer - 1) / (kCountThreads * kCountPer));
  ktimer_begin("count", s, 2);
  launch_pdl(k_count, dim3(ob), dim3(kCountThreads), 0, s, t, a.keys, n, cnt, one, ws.sc);
  ktimer_end("count", s, 2);
  const int64_t ab = (buckets + kAllocThreads * kAllocPer - 1) / (kAllocThreads * kAllocPer);
  ktimer_begin("alloc", s, 2);
  launch_pdl(k_alloc, dim3((unsigned)ab), dim3(kAllocThreads), 0, s, buckets, a.keys, cnt, one, segs, bigs, o.recs, o.cap,
             ws.sc);
  ktimer_end("alloc", s, 2);
  ktimer_begin("scatter", s, 2);
  launch_pdl(k_scatter, dim3(ob), dim3(kCountThreads), 0, s, t, a.keys, n, cnt, ws.sidx, ws.skeys);
  ktimer_end("scatter", s, 2);
  ktimer_begin("segfin", s, 2);
  int64_t fb = (n + kSegfinThreads - 1) / kSegfinThreads;
  if (fb > (int64_t)num_sms * 4) fb = (int64_t)num_sms * 4;
  launch_pdl(k_segfin, dim3((unsigned)fb), dim3(kSegfinThreads), 0, s, segs, cnt, o, ws.sc);
  ktimer_end("segfin", s, 2);
  int end_bit = 1;
  while (end_bit < 32 && ((int64_t)1 << end_bit) < n) end_bit++;
  const size_t bsmem = (size_t)kBigWinWords * sizeof(uint32_t);
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long dbit = 1ull << (dev & 63);
  static std::atomic<unsigned long long> attr_set{0};
  if (!(attr_set.load() & dbit)) {
    cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem);
    attr_set.fetch_or(dbit);
  }
  ktimer_begin("big", s, 2);
  launch_pdl(k_big, dim3((unsigned)num_sms), dim3(kBigThreads), bsmem, s, a.keys, n, bigs, cnt, o, end_bit, ws.sc);
  ktimer_end("big", s, 2);
  g_launches += 5;
  return cudaGetLastError();
}

}  // namespace hkv
