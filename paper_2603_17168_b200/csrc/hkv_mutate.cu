// hkv_mutate.cu — inserter/updater kernels: insert_or_assign, insert_and_evict,
// find_or_insert, erase, assign, assign_scores.
//
// Semantics: the reference's batch engine equals applying the ops one at a
// time in ascending batch index (leader rounds,
// table.py:945-985).  The B200 engine reproduces that order exactly:
//
//  single mode  -- a key's whole candidate space is one bucket, so ops on
//    different buckets commute.  k_prep hashes the batch, a stable radix sort
//    groups ops by bucket (ascending batch index inside a bucket), k_segments
//    emits one record per bucket segment (and marks same-key runs), and
//    k_meta_tps gives each segment to one thread that applies its ops'
//    metadata in order with exclusive ownership of the bucket: no CAS, no
//    retries, bit-exact at any contention.  Value rows then move in streaming
//    kernels (k_values_read / k_values_write) driven by the recorded row plan.
//  dual mode    -- an op touches two buckets: hkv_dual.cu runs a device
//    dataflow over per-bucket turn counters (process_op per op).
//
// Per op (tps_op) the thread restates _round_upsert (table.py:1025-1119):
// digest probe (one 128-B line) -> hit: score refresh + value plan ->
// miss: insert at the lowest free slot (occupancy bitmap, __ffs) or, on a full
// bucket, argmin over the score row through the group summary, admission
// test and eviction (_finish_admission, table.py:1121-1163).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <atomic>
#include <cstdlib>
#include <string>
#include <thrust/iterator/reverse_iterator.h>

#include "hkv_kernels.h"
#include "hkv_probe.cuh"
#include "hkv_tps.cuh"

namespace hkv {

// ---------------------------------------------------------------------------
// pipeline kernels
// ---------------------------------------------------------------------------
__global__ void k_prep(TableDev t, const uint64_t* __restrict__ keys, int64_t n, uint32_t* __restrict__ bkt,
                       uint32_t* __restrict__ idx, uint32_t* __restrict__ b2, Scalars* sc) {
  griddep_wait();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    sc->first_ev = 0xFFFFFFFFu;
    sc->size_before = (long long)*t.size;
    if (role_forbids_mutation(t)) atomicOr(&sc->err, 2);
  }
  if (i >= n) return;
  const uint64_t key = keys[i];
  if (key >= kLockedKey) atomicOr(&sc->err, 1);  // table.py:168-169, checked before any mutation
  const uint64_t h = fmix64(key);
  bkt[i] = (uint32_t)(h & t.mask);
  idx[i] = (uint32_t)i;
  if (b2) b2[i] = (uint32_t)(second_hash(h) & t.mask);
}


__global__ void __launch_bounds__(1024) k_segments(const uint32_t* __restrict__ sb, const uint32_t* __restrict__ sidx,
                                                   const uint64_t* __restrict__ keys, int64_t n,
                                                   SegRec* __restrict__ recs, int64_t cap, SegRec* __restrict__ lrecs,
                                                   Scalars* sc,
                                                   uint32_t* __restrict__ brk, uint8_t* __restrict__ outcomes,
                                                   uint32_t* __restrict__ vrow, uint8_t fcode,
                                                   uint64_t* __restrict__ skeys) {
  griddep_wait();
  __shared__ unsigned wcount[2][32];
  __shared__ unsigned block_base[2];
  if (sc->err) return;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t b = kNoRow;
  bool head = false, multi = false, prev_same_b = false;
  uint32_t i = 0;
  if (p < n) {
    b = sb[p];
    i = sidx[p];
    prev_same_b = (p > 0) && (sb[p - 1] == b);
    head = !prev_same_b;
    multi = (p + 1 < n) && (sb[p + 1] == b);
  }
  // same-key test with both neighbours (keys of multi-op segments only)
  const bool in_multi = multi || prev_same_b;
  const uint64_t k = in_multi ? keys[i] : 0;
  uint64_t k_next = __shfl_down_sync(kFull, k, 1);
  uint64_t k_prev = __shfl_up_sync(kFull, k, 1);
  if (lane == 31 && multi) k_next = keys[sidx[p + 1]];
  if (lane == 0 && prev_same_b) k_prev = keys[sidx[p - 1]];
  if (p < n) {
    const bool same_next = multi && k_next == k;
    brk[p] = same_next ? 0xFFFFFFFFu : (uint32_t)p;
    if (same_next) sc->has_runs = 1;
    if (in_multi) skeys[p] = k;
    if (prev_same_b && k_prev == k) {
      outcomes[i] = fcode;
      vrow[i] = kNoRow;
    }
  }
  const bool lng = head && multi && lrecs != nullptr && p + kLongSeg - 1 < n && sb[p + kLongSeg - 1] == b;
  // skew statistic for the next batch's grouping choice (collect_eligible)
  if (head && multi && p + 16 < n && sb[p + 16] == b) atomicAdd(&sc->nbig, 1u);
  const unsigned ms = __ballot_sync(kFull, head && !multi);
  const unsigned mm = __ballot_sync(kFull, head && multi && !lng);
  if (lane == 0) {
    wcount[0][warp] = __popc(ms);
    wcount[1][warp] = __popc(mm);
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    const int c = threadIdx.x;
    unsigned acc = 0;
    for (unsigned w = 0; w < blockDim.x / 32; w++) {
      const unsigned x = wcount[c][w];
      wcount[c][w] = acc;
      acc += x;
    }
    block_base[c] = acc ? atomicAdd(c == 0 ? &sc->nseg : &sc->nmulti, acc) : 0;
  }
  __syncthreads();
  if (head) {
    SegRec rec;
    rec.key = in_multi ? k : keys[i];
    rec.p = (uint32_t)p;
    rec.b = b;
    rec.i = i;
    rec.flags = (multi ? 1u : 0u) | (digest_of(fmix64(rec.key)) << 8);
    if (lng) {
      lrecs[atomicAdd(&sc->nlong, 1u)] = rec;
      return;
    }
    const int c = multi ? 1 : 0;
    const unsigned m = multi ? mm : ms;
    const int64_t slot = block_base[c] + wcount[c][warp] + __popc(m & ((1u << lane) - 1));
    recs[multi ? cap - 1 - slot : slot] = rec;
  }
}


// Two-stage cp.async pipeline per thread: while segment k is processed, the
// digest line + occupancy of segment k+1 are in flight into shared memory
// and the record of segment k+2 into registers.
template <int OP, bool COLLECT>
__global__ void __launch_bounds__(kTpsThreads, HKV_TPS_MINB) k_meta_tps(TableDev t, OpArgs a, const uint32_t* __restrict__ sb,
                                                            const uint32_t* __restrict__ sidx,
                                                            uint32_t* run_end,  // written: lw_fill jump marks
                                                            const uint64_t* __restrict__ skeys,
                                                            const SegRec* __restrict__ recs, int64_t cap, int64_t n,
                                                            uint32_t* __restrict__ vrow, uint32_t* __restrict__ rrow,
                                                            int32_t* __restrict__ rsrc, int* __restrict__ lwtab,
                                                            const unsigned* nbound) {
  griddep_wait();
  extern __shared__ uint4 tps_smem[];
  __shared__ BlockCtrs bc;
  block_ctrs_init(bc);
  // every scalar the pass needs, loaded together
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int err = a.sc->err;
  const int64_t nseg = (int64_t)a.sc->nseg;
  const int64_t nmul = (int64_t)a.sc->nmulti;
  const bool runs = a.sc->has_runs != 0;
  const long long size0 = a.sc->size_before;
  if (nbound) n = *nbound;  // collector pipeline: sorted positions in use (device count)
  const uint64_t clock0 = *t.clock;
  const bool fel_open = !*t.fel_set;
  if (err) return;
  const SegRec g0 = gtid < nseg ? recs[gtid] : SegRec{0, 0, 0, 0, 0};
  const SegRec g1 = gtid + stride < nseg ? recs[gtid + stride] : SegRec{0, 0, 0, 0, 0};
  // at lambda > 0.97 a full bucket is the rule: fetch the summary with the first op
  const bool spec = (unsigned long long)size0 * 100ull > t.capacity * 97ull;
  const bool lfu_like = t.policy == kLfu || t.policy == kEpochLfu;
  ctr_t ctr[6] = {0, 0, 0, 0, 0, 0};
  int sd = 0;
  uint32_t fe_min = 0xFFFFFFFFu;
  const int64_t nall = nseg + nmul;
  auto rec_at = [&](int64_t j) -> SegRec {
    if (j >= nall) return SegRec{0, 0, 0, 0, 0};
    return j < nseg ? recs[j] : recs[cap - 1 - (j - nseg)];
  };
  int64_t j = gtid;
  // keys of the head op's first two digest candidates, loaded into registers
  // ahead of the segment that compares them
  auto prefetch_keys = [&](const SegRec& r, const uint4* L, uint64_t& k0, uint64_t& k1, int& nk) {
    nk = 0;
    const uint32_t* O = reinterpret_cast<const uint32_t*>(L + 8);
#if HKV_SUMM_PREFETCH
    // a full bucket's op reads the eviction summary: start it towards L2 a
    // segment ahead (no registers held)
    if (OP != kOpErase && (O[0] & O[1] & O[2] & O[3]) == 0xFFFFFFFFu) {
      const char* sp = reinterpret_cast<const char*>(t.smin + (uint64_t)r.b * 8);
      asm volatile("prefetch.global.L2 [%0];" ::"l"(sp));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(sp + 32));
      asm volatile("prefetch.global.L2 [%0];" ::"l"(t.svalid + r.b));
    }
#endif
    if (!t.digest_filter) return;
    const uint32_t d = r.flags >> 8;
    int s0 = -1, s1 = -1;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      uint32_t m = (match16(L[2 * q], d) | (match16(L[2 * q + 1], d) << 16)) & O[q];
      while (m && s1 < 0) {
        const int x = 32 * q + __ffs(m) - 1;
        m &= m - 1;
        if (s0 < 0) s0 = x; else s1 = x;
      }
    }
    const uint64_t* kr = kptr(t, (uint64_t)r.b * kSlots);
    if (s0 >= 0) { k0 = kr[2 * s0]; nk = 1; }
    if (s1 >= 0) { k1 = kr[2 * s1]; nk = 2; }
  };
#if HKV_TPS_STAGES == 3
  // Three line buffers: segment j+2's line is issued while j runs, and the
  // candidate keys of j+1 were issued at the end of j-1 -- a whole segment of
  // slack for both dependent loads.
  SegRec r0 = j < nseg ? g0 : rec_at(j), r1 = j + stride < nseg ? g1 : rec_at(j + stride), r2 = rec_at(j + 2 * stride);
  if (j < nall) tps_fetch(t, tps_buf(tps_smem, 0), r0.b);
  cp_async_commit();
  if (j + stride < nall) tps_fetch(t, tps_buf(tps_smem, 1), r1.b);
  cp_async_commit();
  if (j + 2 * stride < nall) tps_fetch(t, tps_buf(tps_smem, 2), r2.b);
  cp_async_commit();
  uint64_t pa0 = 0, pa1 = 0, pb0 = 0, pb1 = 0;
  int npa = 0, npb = 0;
  if (j < nall) {
    cp_async_wait<2>();
    prefetch_keys(r0, tps_buf(tps_smem, 0), pa0, pa1, npa);
  }
  if (j + stride < nall) {
    cp_async_wait<1>();
    prefetch_keys(r1, tps_buf(tps_smem, 1), pb0, pb1, npb);
  }
  for (int stage = 0; j < nall; j += stride, stage = stage == 2 ? 0 : stage + 1) {
    const SegRec r3 = rec_at(j + 3 * stride);  // in flight while segment j is processed
    uint4* buf = tps_buf(tps_smem, stage);
    tps_segment<OP, COLLECT, false>(t, a, r0, buf, sb, sidx, run_end, skeys, n, vrow, rrow, rsrc, clock0, fel_open, spec,
                             lfu_like, runs, ctr, sd, fe_min, lwtab + gtid, stride, nullptr, nullptr, 0, pa0, pa1,
                             npa);
    if (j + 3 * stride < nall) tps_fetch(t, buf, r3.b);
    cp_async_commit();
    pa0 = pb0;
    pa1 = pb1;
    npa = npb;
    if (j + 2 * stride < nall) {  // segment j+2's line was issued one segment ago
      cp_async_wait<1>();
      prefetch_keys(r2, tps_buf(tps_smem, stage == 0 ? 2 : stage - 1), pb0, pb1, npb);
    }
    r0 = r1;
    r1 = r2;
    r2 = r3;
  }
#else
  SegRec ra = j < nseg ? g0 : rec_at(j), rb = j + stride < nseg ? g1 : rec_at(j + stride);
  if (j < nall) tps_fetch(t, tps_buf(tps_smem, 0), ra.b);
  cp_async_commit();
  if (j + stride < nall) tps_fetch(t, tps_buf(tps_smem, 1), rb.b);
  cp_async_commit();
  uint64_t pk0 = 0, pk1 = 0;
  int npk = 0;
  if (j < nall) {
    cp_async_wait<1>();
    prefetch_keys(ra, tps_buf(tps_smem, 0), pk0, pk1, npk);
  }
  for (int stage = 0; j < nall; j += stride, stage ^= 1) {
    const SegRec rn = rec_at(j + 2 * stride);  // in flight while segment j is processed
    cp_async_wait<1>();
    uint4* buf = tps_buf(tps_smem, stage);
    tps_segment<OP, COLLECT, false>(t, a, ra, buf, sb, sidx, run_end, skeys, n, vrow, rrow, rsrc, clock0, fel_open, spec,
                             lfu_like, runs, ctr, sd, fe_min, lwtab + gtid, stride, nullptr, nullptr, 0, pk0, pk1,
                             npk);
    ra = rb;
    rb = rn;
    if (j + 2 * stride < nall) tps_fetch(t, buf, rb.b);
    cp_async_commit();
    if (j + stride < nall) {  // the next segment's line landed one segment ago
      cp_async_wait<1>();
      prefetch_keys(ra, tps_buf(tps_smem, stage ^ 1), pk0, pk1, npk);
    }
  }
#endif
  cp_async_wait<0>();
  if (fel_open) {
    unsigned m = __reduce_min_sync(kFull, fe_min);
    if ((threadIdx.x & 31) == 0 && m != 0xFFFFFFFFu) atomicMin(&a.sc->first_ev, m);
  }
  block_ctrs_flush(bc, t.counters, t.size, ctr, sd);
}

// Long segments (>= kLongSeg ops on one bucket: configs[0] puts ~128 ops on
// every bucket, zipf batches pile thousands on their hot buckets): one thread
// per segment as in k_meta_tps, but the bucket's keys, scores and last-writer
// table live in shared memory for the whole segment, so each op's compares,
// argmin scans and writes are shared-memory operations instead of global
// round trips on lines the thread itself just wrote.  The bucket is written
// back once at the end.  kLongThreads threads per block, one block per SM.
constexpr int kLongThreads = 64;
constexpr size_t kLongSmem = (size_t)kSlots * kLongThreads * (8 + 8 + 4) + (size_t)kLongThreads * 9 * 16;

template <int OP, bool COLLECT>
__global__ void __launch_bounds__(kLongThreads) k_meta_long(TableDev t, OpArgs a, const uint32_t* __restrict__ sb,
                                                           const uint32_t* __restrict__ sidx, uint32_t* run_end,
                                                           const uint64_t* __restrict__ skeys,
                                                           const SegRec* __restrict__ lrecs, int64_t n,
                                                           uint32_t* __restrict__ vrow, uint32_t* __restrict__ rrow,
                                                           int32_t* __restrict__ rsrc) {
  griddep_wait();
  extern __shared__ uint4 long_smem[];
  __shared__ BlockCtrs bc;
  if (a.sc->err) return;
  const unsigned nl = a.sc->nlong;
  if (nl == 0) return;
  block_ctrs_init(bc);
  uint64_t* K = reinterpret_cast<uint64_t*>(long_smem);  // [slot][thread]
  uint64_t* Sc = K + kSlots * kLongThreads;
  int* LW = reinterpret_cast<int*>(Sc + kSlots * kLongThreads);
  uint4* stage = reinterpret_cast<uint4*>(LW + kSlots * kLongThreads) + threadIdx.x * 9;
  const uint64_t clock0 = *t.clock;
  const bool fel_open = !*t.fel_set;
  const bool lfu_like = t.policy == kLfu || t.policy == kEpochLfu;
  const bool runs = a.sc->has_runs != 0;
  ctr_t ctr[6] = {0, 0, 0, 0, 0, 0};
  int sd = 0;
  uint32_t fe_min = 0xFFFFFFFFu;
  for (int64_t j = (int64_t)blockIdx.x * kLongThreads + threadIdx.x; j < nl; j += (int64_t)gridDim.x * kLongThreads) {
    const SegRec rec = lrecs[j];
    const uint64_t rowbase = (uint64_t)rec.b * kSlots;
    const uint4* dp = reinterpret_cast<const uint4*>(t.digests + rowbase);
#pragma unroll
    for (int k = 0; k < 8; k++) stage[k] = dp[k];
    stage[8] = reinterpret_cast<const uint4*>(t.bits)[rec.b];
    const ulonglong2* kp = reinterpret_cast<const ulonglong2*>(kptr(t, rowbase));
#pragma unroll 8
    for (int s = 0; s < kSlots; s++) {
      const ulonglong2 ks = kp[s];  // (key, score)
      K[s * kLongThreads + threadIdx.x] = ks.x;
      Sc[s * kLongThreads + threadIdx.x] = ks.y;
    }
    tps_segment<OP, COLLECT, true>(t, a, rec, stage, sb, sidx, run_end, skeys, n, vrow, rrow, rsrc, clock0,
                                   fel_open, false, lfu_like, runs, ctr, sd, fe_min, LW + threadIdx.x,
                                   kLongThreads, K + threadIdx.x, Sc + threadIdx.x, kLongThreads);
  }
  if (fel_open) {
    unsigned m = __reduce_min_sync(kFull, fe_min);
    if ((threadIdx.x & 31) == 0 && m != 0xFFFFFFFFu) atomicMin(&a.sc->first_ev, m);
  }
  block_ctrs_flush(bc, t.counters, t.size, ctr, sd);
}

// Clock advance + first_eviction_lambda (table.py:986-991) + error latch +
// the skew hint, run by every block of the batch's last kernel (k_finalize,
// or k_values_write when the batch moves values: one launch fewer).  The
// lambda needs the inserts that precede the first eviction: counted by every
// block over a strided share, the last block to finish publishes it.
// Returns false when the batch failed (nothing else may run).
template <int NT>
__device__ __forceinline__ bool finalize_batch(const TableDev& t, Scalars* sc, const uint8_t* __restrict__ outcomes,
                                               unsigned long long clock_advance, int add_found,
                                               volatile unsigned* skew_hint) {
  // segments of more than 16 ops in this batch, for the next call's choice
  // between the collector and the sorted grouping (a mapped host word)
  if (skew_hint && blockIdx.x == 0 && threadIdx.x == 0) *skew_hint = sc->nbig;
  if (sc->err) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(t.err, sc->err);
    return false;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *t.clock += clock_advance + (add_found ? sc->nfound : 0ull);
  const unsigned fe = sc->first_ev;
  if (*t.fel_set || fe == 0xFFFFFFFFu || outcomes == nullptr) return true;
  unsigned cnt = 0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < (int64_t)fe;
       j += (int64_t)gridDim.x * blockDim.x)
    cnt += outcomes[j] == kInserted;
  typedef cub::BlockReduce<unsigned, NT> BR;
  __shared__ typename BR::TempStorage tmp;
  const unsigned tot = BR(tmp).Sum(cnt);
  if (threadIdx.x == 0) {
    if (tot) atomicAdd(&sc->fel_cnt, (unsigned long long)tot);
    __threadfence();
    if (atomicAdd(&sc->fel_done, 1u) == gridDim.x - 1) {
      __threadfence();
      const unsigned long long all = atomicAdd(&sc->fel_cnt, 0ull);
      *t.fel = (double)(sc->size_before + (long long)all) / (double)t.capacity;
      *t.fel_set = 1;
    }
  }
  return true;
}

// Value rows for the final writers: table[vrow[i]] = values[i].  Inputs are
// read sequentially (consecutive i), destination rows at random; KPT ops per
// tile keep 2*KPT 16-B loads in flight per lane.
template <int VEC, int KPT>
__global__ void __launch_bounds__(256) k_values_write(TableDev t, const float* __restrict__ values,
                                                      const uint32_t* __restrict__ vrow, int64_t n, Scalars* sc,
                                                      const uint8_t* __restrict__ fin_outcomes,
                                                      unsigned long long clock_advance,
                                                      volatile unsigned* skew_hint) {
  griddep_wait();
  if (!finalize_batch<256>(t, sc, fin_outcomes, clock_advance, 0, skew_hint)) return;
  using V = typename std::conditional<VEC == 4, uint4, typename std::conditional<VEC == 2, float2, float>::type>::type;
  const Tile8 tile;
  const int r = tile.thread_rank();
  const int64_t tid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ntiles = (int64_t)gridDim.x * blockDim.x / kG;
  const int dim = t.dim;
  const int nv = dim / VEC;
  for (int64_t base = tid * KPT; base < n; base += ntiles * KPT) {
    uint32_t row[KPT];
#pragma unroll
    for (int u = 0; u < KPT; u++) row[u] = (base + u < n) ? vrow[base + u] : kNoRow;
    for (int e0 = r; e0 < nv; e0 += kG * 2) {
      V v[KPT][2];
#pragma unroll
      for (int u = 0; u < KPT; u++) {
        const V* src = reinterpret_cast<const V*>(values + (uint64_t)(base + u) * dim);
#pragma unroll
        for (int w = 0; w < 2; w++) {
          const int e = e0 + w * kG;
          if (row[u] != kNoRow && e < nv) v[u][w] = ld_vec(src + e);
        }
      }
#pragma unroll
      for (int u = 0; u < KPT; u++) {
        if (row[u] == kNoRow) continue;
        V* dst = reinterpret_cast<V*>(value_row(t, row[u]));
#pragma unroll
        for (int w = 0; w < 2; w++) {
          const int e = e0 + w * kG;
          if (e < nv) st_vec(dst + e, v[u][w]);
        }
      }
    }
  }
}

// Value reads resolved through the recorded provenance: the row's pre-batch
// content (rsrc < 0) or the input of the op that wrote it earlier in the batch.
//   list == nullptr: find_or_insert hits -> values[i] for outcome Found
//   list != nullptr: insert_and_evict victims, j-th evicted op -> ev[j], ek/es
// KPT reads per tile, two 16-B vectors per read and lane in flight (as in
// k_values_write).
template <int VEC, int KPT>
__global__ void __launch_bounds__(256) k_values_read(TableDev t, float* __restrict__ values,
                                                     const uint8_t* __restrict__ outcomes,
                                                     const uint32_t* __restrict__ rrow,
                                                     const int32_t* __restrict__ rsrc, const uint32_t* list,
                                                     const long long* n_list, const uint64_t* __restrict__ ek_tmp,
                                                     const uint64_t* __restrict__ es_tmp, uint64_t* ek, uint64_t* es,
                                                     float* ev, int64_t n, const Scalars* sc) {
  griddep_wait();
  if (sc->err) return;
  using V = typename std::conditional<VEC == 4, uint4, typename std::conditional<VEC == 2, float2, float>::type>::type;
  const Tile8 tile;
  const int r = tile.thread_rank();
  const int64_t tid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ntiles = (int64_t)gridDim.x * blockDim.x / kG;
  const int dim = t.dim;
  const int nv = dim / VEC;
  const int64_t m = list ? (int64_t)*n_list : n;
  for (int64_t base = tid * KPT; base < m; base += ntiles * KPT) {
    const V* from[KPT];
    V* dst[KPT];
#pragma unroll
    for (int u = 0; u < KPT; u++) {
      const int64_t j = base + u;
      from[u] = nullptr;
      dst[u] = nullptr;
      if (j >= m) continue;
      uint32_t i;
      if (list) {
        i = list[j];
        dst[u] = reinterpret_cast<V*>(ev + j * (int64_t)dim);
        if (r == 0) {
          ek[j] = ek_tmp[kRecU64 * i];
          es[j] = es_tmp[kRecU64 * i];
        }
      } else {
        i = (uint32_t)j;
        if (outcomes[i] != kFound) continue;
        dst[u] = reinterpret_cast<V*>(values + (uint64_t)i * dim);
      }
      const int32_t src = rsrc[kRecU32 * i];
      from[u] = reinterpret_cast<const V*>(src < 0 ? value_row(t, rrow[kRecU32 * i]) : values + (uint64_t)src * dim);
    }
    for (int e0 = r; e0 < nv; e0 += kG * 2) {
      V x[KPT][2];
#pragma unroll
      for (int u = 0; u < KPT; u++) {
#pragma unroll
        for (int w = 0; w < 2; w++) {
          const int e = e0 + w * kG;
          if (from[u] && e < nv) x[u][w] = ld_vec(from[u] + e);
        }
      }
#pragma unroll
      for (int u = 0; u < KPT; u++) {
#pragma unroll
        for (int w = 0; w < 2; w++) {
          const int e = e0 + w * kG;
          if (from[u] && e < nv) st_vec(dst[u] + e, x[u][w]);
        }
      }
    }
  }
}

constexpr int kFinBlocks = 32;
__global__ void __launch_bounds__(1024) k_finalize(TableDev t, Scalars* sc, const uint8_t* __restrict__ outcomes,
                                                   int64_t n, unsigned long long clock_advance, int add_found,
                                                   volatile unsigned* skew_hint) {
  griddep_wait();
  finalize_batch<1024>(t, sc, outcomes, clock_advance, add_found, skew_hint);
}

struct IsEvicted {
  const uint8_t* o;
  __host__ __device__ bool operator()(const int64_t& i) const { return o[i] == kEvicted; }
};

template <int VEC>
__global__ void k_evict_gather(const Scalars* sc, const uint32_t* __restrict__ list, const long long* n_ev,
                               const uint64_t* __restrict__ ek_tmp, const uint64_t* __restrict__ es_tmp,
                               const float* __restrict__ ev_tmp, uint64_t* ek, uint64_t* es, float* ev,
                               int dim, int64_t n) {
  griddep_wait();
  const Tile8 tile;
  const int r = tile.thread_rank();
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / kG;
  const int64_t ne = sc->err ? 0 : *n_ev;
  for (int64_t j = gid; j < ne; j += ngroups) {
    const uint32_t i = list[j];
    if (r == 0) {
      ek[j] = ek_tmp[kRecU64 * i];
      es[j] = es_tmp[kRecU64 * i];
    }
    copy_row<kG, VEC>(ev + j * dim, ev_tmp + (uint64_t)i * dim, dim, r);
  }
}

__global__ void k_zero_count(const Scalars* sc, long long* n_ev) {
  griddep_wait();
  if (sc->err) *n_ev = 0;
}

// ---------------------------------------------------------------------------
// assign / assign_scores (updater role; structure never changes)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_assign_find(TableDev t, const uint64_t* __restrict__ keys, int64_t n,
                                                     uint32_t* __restrict__ rows, uint8_t* __restrict__ outcomes,
                                                     Scalars* sc) {
  griddep_wait();
  // thread per key (the find path's probe: one digest line per thread, the
  // candidate keys in slot order; counters as table.py:243-268)
  if (sc->err) return;
  __shared__ BlockCtrs bc;
  block_ctrs_init(bc);
  ctr_t ctr[6] = {0, 0, 0, 0, 0, 0};
  int bad = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0 && role_forbids_mutation(t)) atomicOr(&sc->err, 2);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = keys[i];
    bad |= key >= kLockedKey;  // table.py:168-169: the apply pass then performs no mutation
    const uint64_t h = fmix64(key);
    const uint32_t d = digest_of(h);
    uint64_t b = h & t.mask;
    unsigned ncmp = 0;
    int slot = probe_line_thread(t, b, key, d, ncmp);
    ctr[kLoads]++;
    if (slot < 0 && t.dual) {
      b = second_hash(h) & t.mask;
      slot = probe_line_thread(t, b, key, d, ncmp);
      ctr[kLoads]++;
    }
    ctr[kCompares] += ncmp;
    rows[i] = slot >= 0 ? (uint32_t)(b * kSlots + slot) : 0xFFFFFFFFu;
    outcomes[i] = slot >= 0 ? kUpdated : kNotFound;
  }
  if (bad) atomicOr(&sc->err, 1);
  block_ctrs_flush(bc, t.counters, nullptr, ctr, 0);
}

template <int VEC>
__global__ void __launch_bounds__(256) k_assign_apply(TableDev t, const float* __restrict__ values,
                                                      const uint64_t* __restrict__ scores, int refresh,
                                                      uint64_t epoch, const uint32_t* __restrict__ rows,
                                                      const uint32_t* __restrict__ ranks,
                                                      const uint64_t* __restrict__ ticks,
                                                      const uint32_t* __restrict__ sb,
                                                      const uint32_t* __restrict__ sidx, int64_t n,
                                                      Scalars* sc) {
  griddep_wait();
  if (sc->err) return;
  const Tile8 tile;
  const int r = tile.thread_rank();
  const int64_t tid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ntiles = (int64_t)gridDim.x * blockDim.x / kG;
  const uint64_t clock0 = *t.clock;
  ctr_t ctr[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t base = tid * kG; base < n; base += ntiles * kG) {
   const int64_t pp = base + r;
   bool head = false;
   if (pp < n) head = (pp == 0) || (sb[pp - 1] != sb[pp]);
   uint32_t hm = tile.ballot(head);
   while (hm) {
    const int hl = __ffs(hm) - 1;
    hm &= hm - 1;
    int64_t p = base + hl;
    const uint32_t b = sb[p];
    while (true) {
      const uint32_t i = sidx[p];
      const uint32_t row = rows[i];
      if (row != 0xFFFFFFFFu) {
        if (values) {
          copy_row<kG, VEC>(value_row(t, row), values + (uint64_t)i * t.dim, t.dim, r);
          ctr[row < t.fast_rows ? kVFast : kVOver]++;
        }
        if (r == 0) {
          if (scores) {
            *sptr(t, row) = scores[i];
            summ_invalidate(t, row / kSlots, (int)(row % kSlots));
          } else if (refresh) {
            const uint64_t tick = ticks ? ticks[i] : clock0 + (uint64_t)ranks[i] + 1;
            *sptr(t, row) = hit_score(t.policy, *sptr(t, row), epoch, tick, false, 0);
            summ_invalidate(t, row / kSlots, (int)(row % kSlots));
          }
        }
      }
      if (++p >= n || sb[p] != b) break;
    }
   }
  }
  if (r != 0) {
#pragma unroll
    for (int k = 0; k < 6; k++) ctr[k] = 0;
  }
  flush_counters<256>(t.counters, ctr, 6);
}

struct IsUpdated {
  const uint8_t* o;
  __host__ __device__ uint32_t operator()(const int64_t& i) const { return o[i] == kUpdated ? 1u : 0u; }
};

__global__ void k_assign_count(Scalars* sc, const uint32_t* ranks, const uint8_t* outcomes, int64_t n) {
  griddep_wait();
  if (sc->err || n <= 0) return;
  sc->nfound = (unsigned long long)ranks[n - 1] + (outcomes[n - 1] == kUpdated ? 1ull : 0ull);
}

// Sort-free duplicate resolution for assign / assign_scores.  Ops on the same
// row (duplicate keys in a batch) are aggregated in an open-addressing hash
// keyed by row: the last op (max batch index) and the count.  The apply pass
// then walks the batch in order (inputs read sequentially) and only the last
// op of each row writes: its value ("last duplicate wins", table.py:471-476)
// and the score of `count` consecutive refreshes ending at its tick — the
// closed form tps_run uses (LFU counts every duplicate, LRU keeps the last
// tick), or its explicit score.
__device__ __forceinline__ uint32_t agg_hash(uint32_t row) {
  uint32_t x = row * 0x9E3779B1u;
  return x ^ (x >> 15);
}

__global__ void k_assign_agg(const uint32_t* __restrict__ rows, int64_t n, uint32_t* __restrict__ akey,
                             uint32_t* __restrict__ alast, uint32_t* __restrict__ acnt, uint32_t amask,
                             uint32_t* __restrict__ aslot, const Scalars* sc, int count) {
  griddep_wait();
  if (sc->err) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t row = rows[i];
  if (row == 0xFFFFFFFFu) return;
  uint32_t h = agg_hash(row) & amask;
  while (true) {
    const uint32_t prev = atomicCAS(akey + h, 0xFFFFFFFFu, row);
    if (prev == 0xFFFFFFFFu || prev == row) break;
    h = (h + 1) & amask;
  }
  aslot[i] = h;
  atomicMax(alast + h, (uint32_t)i + 1u);
  if (count) atomicAdd(acnt + h, 1u);  // only the counting policies read it
}

template <int VEC>
__global__ void __launch_bounds__(256) k_assign_apply_agg(TableDev t, const float* __restrict__ values,
                                                          const uint64_t* __restrict__ scores, int refresh,
                                                          uint64_t epoch, const uint32_t* __restrict__ rows,
                                                          const uint32_t* __restrict__ ranks,
                                                          const uint64_t* __restrict__ ticks,
                                                          const uint32_t* __restrict__ alast,
                                                          const uint32_t* __restrict__ acnt,
                                                          const uint32_t* __restrict__ aslot, int64_t n,
                                                          const Scalars* sc) {
  griddep_wait();
  if (sc->err) return;
  const Tile8 tile;
  const int r = tile.thread_rank();
  const int64_t tid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ntiles = (int64_t)gridDim.x * blockDim.x / kG;
  const uint64_t clock0 = *t.clock;
  ctr_t ctr[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t i = tid; i < n; i += ntiles) {
    const uint32_t row = rows[i];
    if (row == 0xFFFFFFFFu) continue;
    if (values) ctr[row < t.fast_rows ? kVFast : kVOver]++;
    const uint32_t h = aslot[i];
    if (alast[h] != (uint32_t)i + 1u) continue;  // a later duplicate writes this row
    if (values) copy_row<kG, VEC>(value_row(t, row), values + (uint64_t)i * t.dim, t.dim, r);
    if (r == 0) {
      if (scores) {
        *sptr(t, row) = scores[i];
        summ_invalidate(t, row / kSlots, (int)(row % kSlots));
      } else if (refresh) {
        const uint64_t tick = ticks ? ticks[i] : clock0 + (uint64_t)ranks[i] + 1;
        *sptr(t, row) = run_hit_score(t.policy, *sptr(t, row), epoch, tick, false, 0, acnt[h]);
        summ_invalidate(t, row / kSlots, (int)(row % kSlots));
      }
    }
  }
  if (r != 0) {
#pragma unroll
    for (int k = 0; k < 6; k++) ctr[k] = 0;
  }
  flush_counters<256>(t.counters, ctr, 6);
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
template <typename T>
static cudaError_t grow(T*& p, int64_t count) {
  if (p) cudaFree(p);
  p = nullptr;
  if (count <= 0) return cudaSuccess;
  return cudaMalloc((void**)&p, sizeof(T) * (size_t)count);
}

cudaError_t ws_reserve(Workspace& ws, int64_t n, int dim, int ev_mode, bool dual) {
  cudaError_t e = cudaSuccess;
  if (!ws.sc) {
    e = cudaMalloc((void**)&ws.sc, sizeof(Scalars));
    if (e) return e;
  }
  if (!ws.skew_host) {
    if ((e = cudaHostAlloc((void**)&ws.skew_host, sizeof(unsigned), cudaHostAllocMapped))) return e;
    *ws.skew_host = 0;
    if ((e = cudaHostGetDevicePointer((void**)&ws.skew_dev, (void*)ws.skew_host, 0))) return e;
  }
  if (n > ws.cap_n) {
    const int64_t c = n + n / 4 + 1024;
    if ((e = grow(ws.bkt, c)) || (e = grow(ws.idx, c)) || (e = grow(ws.sbkt, c)) || (e = grow(ws.sidx, c)) ||
        (e = grow(ws.seg, c)) || (e = grow(ws.aux, c)) || (e = grow(ws.aux2, c)) || (e = grow(ws.skey, 3 * c)) || (e = grow(ws.lrec, 3 * (c / kLongSeg + 1))) ||
        (e = grow(ws.vrow, c)) || (e = grow(ws.rrec, kRecU64 * c)) || (e = grow(ws.skeys, c)) || (e = grow(ws.segd, 4 * c)))
      return e;
    // the op's value-read record: victim key, victim score, row, provenance
    ws.ek = ws.rrec;
    ws.es = ws.rrec + 1;
    ws.rrow = reinterpret_cast<uint32_t*>(ws.rrec + 2);
    ws.rsrc = reinterpret_cast<int32_t*>(ws.rrec + 2) + 1;
    if (ws.b2) { cudaFree(ws.b2); ws.b2 = nullptr; }
    if (ws.pend) { cudaFree(ws.pend); ws.pend = nullptr; }
    ws.cap_n = c;
  }
  if (dual && !ws.b2) {
    if ((e = grow(ws.b2, ws.cap_n)) || (e = grow(ws.pend, ws.cap_n))) return e;
  }
  // ev_mode: 1 = per-op victim key/score scratch, 2 = also victim value rows (dual mode)

  if (ev_mode >= 2 && (ws.cap_ev < n || ws.dim != dim)) {
    if ((e = grow(ws.ev, ws.cap_n * dim))) return e;
    ws.cap_ev = ws.cap_n;
    ws.dim = dim;
  }
  // CUB temp storage: the largest of sort / select / scan for cap_n items
  // (queried only when the capacity changes: the queries cost host time)
  if (ws.cub_for_n != ws.cap_n) {
    size_t b_sort = 0, b_sel = 0, b_scan = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b_sort, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (int)ws.cap_n, 0, 32);
    thrust::counting_iterator<int64_t> cnt(0);
    thrust::transform_iterator<IsEvicted, thrust::counting_iterator<int64_t>, bool> fl(cnt, IsEvicted{nullptr});
    cub::DeviceSelect::Flagged(nullptr, b_sel, cnt, fl, (uint32_t*)nullptr, (long long*)nullptr, (int)ws.cap_n);
    thrust::transform_iterator<IsUpdated, thrust::counting_iterator<int64_t>, uint32_t> up(cnt,
                                                                                            IsUpdated{nullptr});
    cub::DeviceScan::ExclusiveSum(nullptr, b_scan, up, (uint32_t*)nullptr, (int)ws.cap_n);
    size_t b_min = 0;
    thrust::reverse_iterator<const uint32_t*> rin(nullptr);
    thrust::reverse_iterator<uint32_t*> rout(nullptr);
    cub::DeviceScan::InclusiveScan(nullptr, b_min, rin, rout, cub::Min(), (int)ws.cap_n);
    size_t need = b_sort > b_sel ? b_sort : b_sel;
    if (b_scan > need) need = b_scan;
    if (b_min > need) need = b_min;
    if (need > ws.cub_bytes) {
      if (ws.cub_tmp) cudaFree(ws.cub_tmp);
      ws.cub_tmp = nullptr;
      if ((e = cudaMalloc(&ws.cub_tmp, need))) return e;
      ws.cub_bytes = need;
    }
    ws.cub_for_n = ws.cap_n;
  }
  return cudaSuccess;
}

void ws_free(Workspace& ws) {
  ws_free_dual(ws);
  void* ptrs[] = {ws.bkt, ws.idx, ws.sbkt, ws.sidx, ws.seg, ws.aux, ws.aux2, ws.skey, ws.lrec, ws.agg, ws.skeys, ws.vrow, ws.rrec,
                  ws.lwtab,
                  ws.b2, ws.pend,
                  ws.ev, ws.cub_tmp, ws.sc, ws.col, ws.segd};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (ws.skew_host) cudaFreeHost((void*)ws.skew_host);
  ws = Workspace();
}

static inline int vec_of(int dim, const void* a, const void* b, const void* c, const void* d) {
  auto al = [](const void* p, uintptr_t m) { return p == nullptr || (((uintptr_t)p) & m) == 0; };
  if (dim % 4 == 0 && al(a, 15) && al(b, 15) && al(c, 15) && al(d, 15)) return 4;
  if (dim % 2 == 0 && al(a, 7) && al(b, 7) && al(c, 7) && al(d, 7)) return 2;
  return 1;
}

static int64_t tile_blocks(int64_t items, int num_sms) {
  int64_t blocks = (items * kG + 255) / 256;
  const int64_t cap = (int64_t)num_sms * 8 * 8;
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : blocks;
}

// sort (bucket, idx) by bucket, then segment heads
static cudaError_t sort_segments(Workspace& ws, int64_t n, int log2_buckets, cudaStream_t s) {
  size_t bytes = ws.cub_bytes;
  const int end_bit = log2_buckets < 1 ? 1 : log2_buckets;
  cudaError_t e = cub::DeviceRadixSort::SortPairs(ws.cub_tmp, bytes, ws.bkt, ws.sbkt, ws.idx, ws.sidx, (int)n, 0,
                                                  end_bit, s);
  if (e) return e;
  g_launches += 4;  // onesweep: histogram + up to 3 passes (approximate)
  return cudaGetLastError();
}

// run_end[p] = min{p' >= p : brk[p'] != ~0}: the last position of p's
// same-key run.  Two passes over tiles of kRunTile positions, both skipped
// when the batch has no same-key run (uniform batches): an in-tile reverse
// min-scan (thread 0 takes the tile's last chunk, so a forward block scan
// over threads is a reverse scan over positions) that also records each
// tile's first break, then a fix-up for positions whose run crosses the
// tile end (walks the following tiles' first breaks).
constexpr int kRunThreads = 1024, kRunPer = 4, kRunTile = kRunThreads * kRunPer;

__global__ void __launch_bounds__(kRunThreads) k_run_ends_tile(const uint32_t* __restrict__ brk, int64_t n,
                                                               uint32_t* __restrict__ run_end,
                                                               uint32_t* __restrict__ tile_first, const Scalars* sc) {
  griddep_wait();
  if (!sc->has_runs || sc->err) return;
  typedef cub::BlockScan<uint32_t, kRunThreads> BS;
  __shared__ typename BS::TempStorage tmp;
  const int64_t base = (int64_t)blockIdx.x * kRunTile + (int64_t)(kRunThreads - 1 - threadIdx.x) * kRunPer;
  uint32_t v[kRunPer];
  uint32_t agg = 0xFFFFFFFFu;
#pragma unroll
  for (int k = kRunPer - 1; k >= 0; k--) {
    const int64_t p = base + k;
    const uint32_t x = p < n ? brk[p] : 0xFFFFFFFFu;
    agg = x < agg ? x : agg;
    v[k] = agg;  // first break at or after p inside this chunk
  }
  uint32_t after;  // first break in the chunks after this one (inside the tile)
  BS(tmp).ExclusiveScan(agg, after, 0xFFFFFFFFu, cub::Min());
  if (threadIdx.x == kRunThreads - 1) tile_first[blockIdx.x] = agg < after ? agg : after;
#pragma unroll
  for (int k = 0; k < kRunPer; k++) {
    const int64_t p = base + k;
    if (p < n) run_end[p] = v[k] < after ? v[k] : after;
  }
}

__global__ void k_run_ends_fix(int64_t n, uint32_t* __restrict__ run_end, const uint32_t* __restrict__ tile_first,
                               int64_t ntiles, const Scalars* sc) {
  griddep_wait();
  if (!sc->has_runs || sc->err) return;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n || run_end[p] != 0xFFFFFFFFu) return;
  uint32_t r = 0xFFFFFFFFu;
  for (int64_t tl = p / kRunTile + 1; tl < ntiles && r == 0xFFFFFFFFu; tl++) r = tile_first[tl];
  run_end[p] = r == 0xFFFFFFFFu ? (uint32_t)(n - 1) : r;
}

static cudaError_t run_ends(Workspace& ws, int64_t n, cudaStream_t s) {
  // tile_first lives in ws.idx: the sort consumed it
  const int64_t ntiles = (n + kRunTile - 1) / kRunTile;
  launch_pdl(k_run_ends_tile, dim3((unsigned)ntiles), dim3(kRunThreads), 0, s, ws.aux2, n, ws.seg, ws.idx, ws.sc);
  launch_pdl(k_run_ends_fix, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, n, ws.seg, ws.idx, ntiles, ws.sc);
  g_launches += 2;
  return cudaGetLastError();
}

cudaError_t run_mutation(const TableDev& t, OpArgs a, int64_t n, int log2_buckets, Workspace& ws,
                         unsigned long long dual_tag, unsigned long long* lead, int64_t* n_evicted,
                         uint64_t* ek_out, float* ev_out, uint64_t* es_out, uint64_t clock_advance,
                         cudaStream_t s, int num_sms, cudaEvent_t values_ready) {
  // values_ready: the value rows may still be in flight (host-buffer entry
  // points copy them H2D on another stream); nothing before the value phase
  // (dual mode: the dataflow) reads them.
  cudaError_t e;
  const bool collect = a.collect != 0;
  // in-place engines move value rows inside the op (dual dataflow, CAS engine)
  const bool cas = t.cas && a.op != kOpErase;
  const bool inplace = t.dual || cas;
  if ((e = ws_reserve(ws, n, t.dim, collect ? (inplace ? 2 : 1) : 0, t.dual != 0))) return e;
  if (t.dual && !cas && (e = ws_reserve_dual(ws, n, log2_buckets))) return e;
  a.sc = ws.sc;
  a.ek = ws.ek;
  a.es = ws.es;
  a.ev = ws.ev;
  if ((e = cudaMemsetAsync(ws.sc, 0, sizeof(Scalars), s))) return e;
  if (n > 0) {
    // sparse single-mode batches group by counting (hkv_collect.cu): its
    // k_link does k_prep's work
    // (a batch whose predecessor on this workspace was skewed -- zipf hot
    // buckets -- keeps the sorted grouping, which such batches favour)
    const bool col = !cas && !t.dual && collect_eligible(n, log2_buckets, ws.skew_host ? *ws.skew_host : 0u);
    if (!col) {
      ktimer_begin("prep", s, 2);
      launch_pdl(k_prep, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, t, a.keys, n, ws.bkt, ws.idx, t.dual ? ws.b2 : nullptr,
                                                          ws.sc);
      ktimer_end("prep", s, 2);
      g_launches++;
    }
    const int vec = vec_of(t.dim, a.values, t.vfast, t.vover, collect ? ws.ev : nullptr);
    if (cas) {
      if (values_ready && (e = cudaStreamWaitEvent(s, values_ready, 0))) return e;
      values_ready = nullptr;
      ktimer_begin("cas_upsert", s);
      if ((e = run_cas(t, a, n, t.locks, vec, s, num_sms))) return e;
      ktimer_end("cas_upsert", s);
    } else if (!t.dual) {
      SegRec* recs = reinterpret_cast<SegRec*>(ws.skey);
      const uint8_t fcode = a.op == kOpErase ? kNotFound : a.op == kOpFindOrInsert ? kFound : kUpdated;
      // The long-segment engine pays when long segments are the rule (batch
      // >= 16 ops per bucket, configs[0]); in a batch that is sparse over the
      // buckets (zipf hot buckets among ~1 op per bucket) the few long
      // segments are better overlapped with everything else inside k_meta_tps.
      const bool use_long = !col && n >= kLongSeg && (n >> log2_buckets) >= 16;
      SegRec* lrecs = use_long ? reinterpret_cast<SegRec*>(ws.lrec) : nullptr;
      if (col) {
        if ((e = run_collect(t, a, n, log2_buckets, ws, s, num_sms, fcode))) return e;
      } else {
        ktimer_begin("sort", s, 2);
        if ((e = sort_segments(ws, n, log2_buckets, s))) return e;
        ktimer_end("sort", s, 2);
        ktimer_begin("segments", s, 2);
        launch_pdl(k_segments, dim3((unsigned)((n + 1023) / 1024)), dim3(1024), 0, s, ws.sbkt, ws.sidx, a.keys, n, recs, n, lrecs, ws.sc, ws.aux2,
                                                                   a.outcomes, ws.vrow, fcode, ws.skeys);
        g_launches++;
        if ((e = run_ends(ws, n, s))) return e;
        ktimer_end("segments", s, 2);
      }
      ktimer_begin("apply", s);
      auto* fn = a.op == kOpErase ? k_meta_tps<kOpErase, false>
                 : a.op == kOpFindOrInsert ? k_meta_tps<kOpFindOrInsert, false>
                 : a.collect ? k_meta_tps<kOpUpsert, true> : k_meta_tps<kOpUpsert, false>;
      const size_t smem = (size_t)HKV_TPS_STAGES * kTpsThreads * kTpsStageU4 * sizeof(uint4);
      // the dynamic shared-memory opt-in is per device (a process may drive several)
      int dev = 0;
      cudaGetDevice(&dev);
      const unsigned long long dbit = 1ull << (dev & 63);
      static std::atomic<unsigned long long> attr_set{0};
      if (!(attr_set.load() & dbit)) {
        for (auto* f : {k_meta_tps<kOpErase, false>, k_meta_tps<kOpFindOrInsert, false>, k_meta_tps<kOpUpsert, true>,
                        k_meta_tps<kOpUpsert, false>})
          cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_set.fetch_or(dbit);
      }
      int64_t tb = (n + kTpsThreads - 1) / kTpsThreads;
      const int64_t tcap = (int64_t)num_sms * HKV_TPS_MINB;  // one resident wave
      if (!ws.lwtab && (e = grow(ws.lwtab, tcap * kTpsThreads * kSlots))) return e;  // 128 entries per thread
      if (tb > tcap) tb = tcap;
      launch_pdl(fn, dim3((unsigned)(tb < 1 ? 1 : tb)), dim3(kTpsThreads), smem, s, t, a, ws.sbkt, ws.sidx, ws.seg, ws.skeys, recs, n, n,
                                                               ws.vrow, ws.rrow, ws.rsrc,
                                                               ws.lwtab, col ? &ws.sc->npos : (const unsigned*)nullptr);
      if (use_long) {
        auto* fl = a.op == kOpErase ? k_meta_long<kOpErase, false>
                   : a.op == kOpFindOrInsert ? k_meta_long<kOpFindOrInsert, false>
                   : a.collect ? k_meta_long<kOpUpsert, true> : k_meta_long<kOpUpsert, false>;
        static std::atomic<unsigned long long> lattr{0};
        if (!(lattr.load() & dbit)) {
          for (auto* f : {k_meta_long<kOpErase, false>, k_meta_long<kOpFindOrInsert, false>,
                          k_meta_long<kOpUpsert, true>, k_meta_long<kOpUpsert, false>})
            cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLongSmem);
          lattr.fetch_or(dbit);
        }
        launch_pdl(fl, dim3((unsigned)num_sms), dim3(kLongThreads), kLongSmem, s, t, a, ws.sbkt, ws.sidx, ws.seg, ws.skeys, lrecs, n,
                                                              ws.vrow, ws.rrow, ws.rsrc);
        g_launches++;
      }
      ktimer_end("apply", s);
      g_launches++;
    } else {
      if (values_ready && (e = cudaStreamWaitEvent(s, values_ready, 0))) return e;
      values_ready = nullptr;
      ktimer_begin("dual_flow", s);
      if ((e = run_dual(t, a, n, log2_buckets, ws, lead, dual_tag, vec, s, num_sms))) return e;
      ktimer_end("dual_flow", s);
    }
  }
  // an empty batch never runs k_prep, which seeds first_ev: no outcomes, so
  // first_eviction_lambda cannot latch from the zeroed scratch
  const uint8_t* fin_outcomes = (a.op == kOpErase || n == 0) ? nullptr : a.outcomes;
  volatile unsigned* skew_hint = (!t.dual && !cas && n > 0) ? ws.skew_dev : nullptr;
  // a batch that moves values finalises in k_values_write (its last kernel)
  const bool fin_in_values = !inplace && n > 0 && a.op != kOpErase;
  if (!fin_in_values) {
    ktimer_begin("finalize", s, 2);
    launch_pdl(k_finalize, dim3(kFinBlocks), dim3(1024), 0, s, t, ws.sc, fin_outcomes, n, clock_advance, 0, skew_hint);
    ktimer_end("finalize", s, 2);
    g_launches++;
  }
  long long* nev = reinterpret_cast<long long*>(n_evicted);
  if (collect && n > 0) {
    ktimer_begin("evict_select", s, 2);
    size_t bytes = ws.cub_bytes;
    thrust::counting_iterator<int64_t> cnt(0);
    thrust::transform_iterator<IsEvicted, thrust::counting_iterator<int64_t>, bool> fl(cnt, IsEvicted{a.outcomes});
    if ((e = cub::DeviceSelect::Flagged(ws.cub_tmp, bytes, cnt, fl, ws.aux, nev, (int)n, s))) return e;
    ktimer_end("evict_select", s, 2);
    g_launches += 2;
  }
  const int64_t vblocks = tile_blocks(n, num_sms);
  if (!inplace && n > 0 && a.op != kOpErase) {
    if (values_ready && (e = cudaStreamWaitEvent(s, values_ready, 0))) return e;
    // value reads (provenance-resolved) strictly before value writes
    const int vr = vec_of(t.dim, a.values, t.vfast, t.vover, collect ? ev_out : nullptr);
    if (collect || a.op == kOpFindOrInsert) {
      const uint32_t* list = collect ? ws.aux : nullptr;
      ktimer_begin("values_read", s, 2);
      int64_t rblocks = (((n + 3) / 4) * kG + 255) / 256;
      const int64_t rcap = (int64_t)num_sms * 8 * 4;
      if (rblocks > rcap) rblocks = rcap;
      if (rblocks < 1) rblocks = 1;
      if (vr == 4)
        launch_pdl(k_values_read<4, 4>, dim3((unsigned)rblocks), dim3(256), 0, s, t, a.values, a.outcomes, ws.rrow, ws.rsrc, list, nev,
                                                           ws.ek, ws.es, ek_out, es_out, ev_out, n, ws.sc);
      else if (vr == 2)
        launch_pdl(k_values_read<2, 4>, dim3((unsigned)rblocks), dim3(256), 0, s, t, a.values, a.outcomes, ws.rrow, ws.rsrc, list, nev,
                                                           ws.ek, ws.es, ek_out, es_out, ev_out, n, ws.sc);
      else
        launch_pdl(k_values_read<1, 4>, dim3((unsigned)rblocks), dim3(256), 0, s, t, a.values, a.outcomes, ws.rrow, ws.rsrc, list, nev,
                                                           ws.ek, ws.es, ek_out, es_out, ev_out, n, ws.sc);
      ktimer_end("values_read", s, 2);
      g_launches++;
    }
    ktimer_begin("values_write", s);
    const int64_t wblocks = (((n + 3) / 4) * kG + 255) / 256;
    const int64_t wcap = (int64_t)num_sms * 8 * 4;
    const unsigned wb = (unsigned)(wblocks < wcap ? (wblocks < 1 ? 1 : wblocks) : wcap);
    if (vr == 4)
      launch_pdl(k_values_write<4, 4>, dim3(wb), dim3(256), 0, s, t, a.values, ws.vrow, n, ws.sc, fin_outcomes,
                 (unsigned long long)clock_advance, skew_hint);
    else if (vr == 2)
      launch_pdl(k_values_write<2, 4>, dim3(wb), dim3(256), 0, s, t, a.values, ws.vrow, n, ws.sc, fin_outcomes,
                 (unsigned long long)clock_advance, skew_hint);
    else
      launch_pdl(k_values_write<1, 4>, dim3(wb), dim3(256), 0, s, t, a.values, ws.vrow, n, ws.sc, fin_outcomes,
                 (unsigned long long)clock_advance, skew_hint);
    ktimer_end("values_write", s);
    g_launches++;
  }
  if (collect) {
    if (n > 0 && inplace) {
      const int vec = vec_of(t.dim, ev_out, ws.ev, nullptr, nullptr);
      if (vec == 4)
        launch_pdl(k_evict_gather<4>, dim3((unsigned)vblocks), dim3(256), 0, s, ws.sc, ws.aux, nev, ws.ek, ws.es, ws.ev, ek_out, es_out,
                                                            ev_out, t.dim, n);
      else if (vec == 2)
        launch_pdl(k_evict_gather<2>, dim3((unsigned)vblocks), dim3(256), 0, s, ws.sc, ws.aux, nev, ws.ek, ws.es, ws.ev, ek_out, es_out,
                                                            ev_out, t.dim, n);
      else
        launch_pdl(k_evict_gather<1>, dim3((unsigned)vblocks), dim3(256), 0, s, ws.sc, ws.aux, nev, ws.ek, ws.es, ws.ev, ek_out, es_out,
                                                            ev_out, t.dim, n);
      g_launches++;
    }
    if (n > 0) {
      launch_pdl(k_zero_count, dim3(1), dim3(1), 0, s, ws.sc, nev);
      g_launches++;
    } else if ((e = cudaMemsetAsync(n_evicted, 0, sizeof(int64_t), s))) {
      return e;
    }
  }
  return cudaGetLastError();
}

cudaError_t run_assign(const TableDev& t, const uint64_t* keys, const float* values, const uint64_t* scores,
                       int refresh, uint64_t epoch, int64_t n, uint8_t* outcomes, const uint64_t* ticks,
                       uint64_t clock_advance, int log2_buckets, Workspace& ws, cudaStream_t s, int num_sms) {
  cudaError_t e;
  if ((e = ws_reserve(ws, n, t.dim, 0, false))) return e;
  if ((e = cudaMemsetAsync(ws.sc, 0, sizeof(Scalars), s))) return e;
  const bool need_ticks = refresh && !scores && !ticks;
  if (n > 0) {
    const int64_t blocks = tile_blocks(n, num_sms);
    int64_t fblocks = (n + 255) / 256;
    if (fblocks > (int64_t)num_sms * 8) fblocks = (int64_t)num_sms * 8;
    launch_pdl(k_assign_find, dim3((unsigned)(fblocks < 1 ? 1 : fblocks)), dim3(256), 0, s, t, keys, n, ws.aux, outcomes, ws.sc);
    g_launches++;
    if (need_ticks) {
      size_t bytes = ws.cub_bytes;
      thrust::counting_iterator<int64_t> cnt(0);
      thrust::transform_iterator<IsUpdated, thrust::counting_iterator<int64_t>, uint32_t> up(cnt,
                                                                                              IsUpdated{outcomes});
      if ((e = cub::DeviceScan::ExclusiveSum(ws.cub_tmp, bytes, up, ws.aux2, (int)n, s))) return e;
      g_launches += 2;
      launch_pdl(k_assign_count, dim3(1), dim3(1), 0, s, ws.sc, ws.aux2, outcomes, n);
      g_launches++;
    }
    // Duplicate resolution.  Batches dense in duplicates (>= 16 ops per bucket,
    // configs[0]) aggregate per row in a hash (random L2 atomics, but no
    // sort); sparse batches sort by bucket and walk segments in order.
    const bool agg = (n >> log2_buckets) >= 16;
    const int vec = vec_of(t.dim, values, t.vfast, t.vover, nullptr);
    if (agg) {
      int64_t acap = 1024;
      while (acap < 2 * n) acap <<= 1;
      if (acap > ws.agg_cap) {
        if (ws.agg) cudaFree(ws.agg);
        ws.agg = nullptr;
        ws.agg_cap = 0;
        if ((e = cudaMalloc((void**)&ws.agg, (size_t)acap * 3 * sizeof(uint32_t)))) return e;
        ws.agg_cap = acap;
      }
      uint32_t* akey = ws.agg;
      uint32_t* alast = ws.agg + acap;
      uint32_t* acnt = ws.agg + 2 * acap;
      const int count = refresh && !scores && (t.policy == kLfu || t.policy == kEpochLfu);
      if ((e = cudaMemsetAsync(akey, 0xFF, (size_t)acap * 4, s)) ||
          (e = cudaMemsetAsync(alast, 0, (size_t)acap * (count ? 8 : 4), s)))
        return e;
      launch_pdl(k_assign_agg, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, ws.aux, n, akey, alast, acnt, (uint32_t)(acap - 1),
                                                              ws.vrow, ws.sc, count);
      g_launches++;
      ktimer_begin("assign_apply", s);
      if (vec == 4)
        launch_pdl(k_assign_apply_agg<4>, dim3((unsigned)blocks), dim3(256), 0, s, t, values, scores, refresh, epoch, ws.aux, ws.aux2,
                                                               ticks, alast, acnt, ws.vrow, n, ws.sc);
      else if (vec == 2)
        launch_pdl(k_assign_apply_agg<2>, dim3((unsigned)blocks), dim3(256), 0, s, t, values, scores, refresh, epoch, ws.aux, ws.aux2,
                                                               ticks, alast, acnt, ws.vrow, n, ws.sc);
      else
        launch_pdl(k_assign_apply_agg<1>, dim3((unsigned)blocks), dim3(256), 0, s, t, values, scores, refresh, epoch, ws.aux, ws.aux2,
                                                               ticks, alast, acnt, ws.vrow, n, ws.sc);
    } else {
      launch_pdl(k_prep, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, t, keys, n, ws.bkt, ws.idx, nullptr, ws.sc);
      g_launches++;
      if ((e = sort_segments(ws, n, log2_buckets, s))) return e;
      ktimer_begin("assign_apply", s);
      if (vec == 4)
        launch_pdl(k_assign_apply<4>, dim3((unsigned)blocks), dim3(256), 0, s, t, values, scores, refresh, epoch, ws.aux, ws.aux2, ticks,
                                                           ws.sbkt, ws.sidx, n, ws.sc);
      else if (vec == 2)
        launch_pdl(k_assign_apply<2>, dim3((unsigned)blocks), dim3(256), 0, s, t, values, scores, refresh, epoch, ws.aux, ws.aux2, ticks,
                                                           ws.sbkt, ws.sidx, n, ws.sc);
      else
        launch_pdl(k_assign_apply<1>, dim3((unsigned)blocks), dim3(256), 0, s, t, values, scores, refresh, epoch, ws.aux, ws.aux2, ticks,
                                                           ws.sbkt, ws.sidx, n, ws.sc);
    }
    ktimer_end("assign_apply", s);
    g_launches++;
  }
  launch_pdl(k_finalize, dim3(kFinBlocks), dim3(1024), 0, s, t, ws.sc, nullptr, n, (refresh && !scores && ticks) ? clock_advance : 0,
                                need_ticks ? 1 : 0, (volatile unsigned*)nullptr);
  g_launches++;
  return cudaGetLastError();
}

}  // namespace hkv
