// hkv_dual.cu — dual-bucket mode upserts (table.py:1088-1119, D1 / D2) as a
// device-side dataflow that reproduces the serial batch order exactly.
//
// An op touches its two candidate buckets b1, b2, so
// bucket segments are not independent as in single mode.  Instead of the
// reference's leader rounds (table.py:945-962: one op per bucket per round,
// hundreds of rounds for a 1M batch because ops chain through shared
// buckets), every op learns its rank in the batch-ordered op list of each of
// its buckets (one stable radix sort of the 2n (bucket, op) pairs), and a
// persistent kernel runs ops as soon as both buckets' turn counters reach
// those ranks:
//   turn[b] = tag | (ops of this batch already applied to b)
// (tag = batch epoch << 32, so no per-batch reset).  Tiles take ops in
// ascending batch index, and an op only waits for smaller indices, which were
// taken earlier by running tiles: no deadlock, no grid barrier.  Each op is
// applied by one 8-lane tile with process_op (exclusive ownership of both
// buckets while it runs).
//
// The default consumer of these ranks and turns is k_dual_rounds
// (hkv_cas.cu, HKV_DUAL_ROUNDS): the same handoff, but thread-per-op in
// warp-synchronous rounds -- an op whose turns have not come simply tries
// again next round -- so 32 ops per warp are in flight instead of 4, and the
// warp moves its rows with coalesced copies.  k_dual_flow stays as the
// reference point (HKV_DUAL_ROUNDS=0).
//
// This file is compiled with -dlcm=cg: a bucket written by one SM is read by
// another right after the turn handoff, so global loads must not be served
// from a stale L1 line.
#include <cub/cub.cuh>

#include "hkv_kernels.h"
#include "hkv_probe.cuh"

namespace hkv {

// ---------------------------------------------------------------------------
// per-op processor (one 8-lane tile, exclusive ownership of the op's buckets)
// ---------------------------------------------------------------------------
// The op's input row, loaded before the op waits for its buckets (it does not
// depend on the table): up to kPreVec 16-B vectors per lane, i.e. dim <= 64.
constexpr int kPreVec = 2;
struct InRow {
  uint4 v[kPreVec];
  bool ok;  // the row fits (VEC == 4, dim / 4 <= kPreVec * kG)
};
template <int VEC>
__device__ __forceinline__ InRow prefetch_row(const float* vin, int dim, int r) {
  InRow p;
  p.ok = VEC == 4 && dim / 4 <= kPreVec * kG;
  if (p.ok) {
    const uint4* s = reinterpret_cast<const uint4*>(vin);
#pragma unroll
    for (int u = 0; u < kPreVec; u++) {
      const int e = r + u * kG;
      if (e < dim / 4) p.v[u] = s[e];
    }
  }
  return p;
}
template <int VEC>
__device__ __forceinline__ void write_row(float* dst, const float* vin, const InRow& p, int dim, int r) {
  if (p.ok) {
    uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int u = 0; u < kPreVec; u++) {
      const int e = r + u * kG;
      if (e < dim / 4) d[e] = p.v[u];
    }
  } else {
    copy_row<kG, VEC>(dst, vin, dim, r);
  }
}

// One bucket probed by an 8-lane tile (lane r: slots 16r..16r+15) with the
// lane's digest slice and occupancy already loaded; compares counted as
// table.py:243-268 (candidates in slot order, stopping at the match)
__device__ __forceinline__ int probe_loaded(const TableDev& t, const Tile8& tile, uint64_t b, uint64_t key,
                                            uint32_t d, uint4 dw, uint32_t occ, ctr_t& n_compares) {
  const int r = tile.thread_rank();
  uint32_t cand = (t.digest_filter ? match16(dw, d) : 0xFFFFu) & occ;
  const uint64_t* kp = kptr(t, b * kSlots + r * kSPL);
  int hit = -1, ncmp = 0, ncmp_all = 0;
  while (cand) {
    const int j = __ffs(cand) - 1;
    cand &= cand - 1;
    ncmp_all++;
    if (kp[2 * j] == key) {
      hit = r * kSPL + j;
      ncmp = ncmp_all;
      break;
    }
  }
  const uint32_t hm = tile.ballot(hit >= 0);
  int slot = -1, contrib = ncmp_all;
  if (hm) {
    const int hl = __ffs(hm) - 1;
    slot = tile.shfl(hit, hl);
    contrib = r < hl ? ncmp_all : (r == hl ? ncmp : 0);
  }
  n_compares += tile.sum((unsigned)contrib);
  return slot;
}

template <int VEC>
__device__ __forceinline__ void process_op(const TableDev& t, const OpArgs& a,
                                           const Tile8& tile, uint32_t i,
                                           uint64_t clock0, bool fel_open, ctr_t* ctr,
                                           int& size_delta, const InRow& pre) {
  const int r = tile.thread_rank();
  const int dim = t.dim;
  const uint64_t key = a.keys[i];
  const uint64_t h = fmix64(key);
  const uint32_t d = digest_of(h);
  const uint64_t b1 = h & t.mask;
  const uint64_t b2 = t.dual ? second_hash(h) & t.mask : b1;
  uint64_t hb = b1;
  // both buckets' digest slices and occupancy in one round trip
  const uint4 dw1 = reinterpret_cast<const uint4*>(t.digests + b1 * kSlots)[r];
  const uint32_t occ1 = load_occ(t, b1, r);
  uint4 dw2 = dw1;
  uint32_t occ2 = occ1;
  if (t.dual) {
    dw2 = reinterpret_cast<const uint4*>(t.digests + b2 * kSlots)[r];
    occ2 = load_occ(t, b2, r);
  }
  int slot = probe_loaded(t, tile, b1, key, d, dw1, occ1, ctr[kCompares]);
  ctr[kLoads]++;
  if (t.dual && slot < 0) {
    slot = probe_loaded(t, tile, b2, key, d, dw2, occ2, ctr[kCompares]);
    ctr[kLoads]++;
    hb = b2;
  }
  uint8_t outcome;
  if (a.op == kOpErase) {
    // _round_erase, table.py:1017-1023: key -> EMPTY; digest/score/value stay stale
    if (slot >= 0) {
      if (slot / kSPL == r) {
        const uint64_t row = hb * kSlots + slot;
        *kptr(t, row) = kEmptyKey;
        const uint32_t o = (hb == b1) ? occ1 : occ2;
        store_occ(t, hb, r, o & ~(1u << (slot % kSPL)));
      }
      size_delta--;
      outcome = kErased;
    } else {
      outcome = kNotFound;
    }
    if (r == 0) a.outcomes[i] = outcome;
    return;
  }
  const uint64_t tick = a.ticks ? a.ticks[i] : clock0 + (uint64_t)i + 1;
  const uint64_t cs = a.scores ? a.scores[i] : 0;
  float* vin = a.values + (uint64_t)i * dim;
  if (slot >= 0) {
    // hit: table.py:1045-1062
    const uint64_t row = hb * kSlots + slot;
    if (slot / kSPL == r) {
      const uint64_t old = hit_needs_old(t.policy) ? *sptr(t, row) : 0;
      *sptr(t, row) = hit_score(t.policy, old, a.epoch, tick, a.scores != nullptr, cs);
      summ_invalidate(t, hb, slot);
    }
    float* vr = value_row(t, row);
    if (a.op == kOpFindOrInsert) {
      copy_row<kG, VEC>(vin, vr, dim, r);
      outcome = kFound;
    } else {
      write_row<VEC>(vr, vin, pre, dim, r);
      outcome = kUpdated;
    }
    ctr[row < t.fast_rows ? kVFast : kVOver]++;
    if (r == 0) a.outcomes[i] = outcome;
    return;
  }
  // miss: insert_scores, scoring.py:105-127
  const uint64_t s_in = insert_score(t.policy, a.epoch, tick, cs);
  uint64_t tb = b1;
  int m = 0;
  uint64_t minv = 0, rest = kMaxScore;  // rest: the victim group's other 15 scores' minimum (its lane)
  bool admit = false;
  bool free_insert = false;
  if (!t.dual) {
    const int occ_total = tile_sum<kG>(tile, __popc(occ1));
    if (occ_total < kSlots) {
      free_insert = true;  // _bulk_insert_free, table.py:1072-1076
    } else {
      bucket_min_summ(t, tile, b1, minv, m, rest);  // table.py:1079-1083
      ctr[kScans]++;
      admit = s_in >= minv;  // single-bucket path admits ties
    }
  } else {
    const int o1 = tile_sum<kG>(tile, __popc(occ1));
    const int o2 = tile_sum<kG>(tile, __popc(occ2));
    if (o1 < kSlots || o2 < kSlots) {
      tb = o1 <= o2 ? b1 : b2;  // D1, table.py:1089-1095
      free_insert = true;
    } else {
      uint64_t min1, min2, rest1, rest2;  // D2, table.py:1096-1119
      int m1, m2;
      bucket_min_summ(t, tile, b1, min1, m1, rest1);
      bucket_min_summ(t, tile, b2, min2, m2, rest2);
      ctr[kScans] += 2;
      const bool use2 = min2 < min1;
      tb = use2 ? b2 : b1;
      m = use2 ? m2 : m1;
      minv = use2 ? min2 : min1;
      rest = use2 ? rest2 : rest1;
      admit = t.admit_unified ? s_in >= minv : s_in > minv;
    }
  }
  if (free_insert) {
    // lowest EMPTY slot (table.py:1171) = lowest clear occupancy bit
    const uint32_t occ = (tb == b1) ? occ1 : occ2;
    const uint32_t hasfree = tile.ballot(occ != 0xFFFFu);
    const int fl = __ffs(hasfree) - 1;
    int s = 0;
    if (r == fl) {
      const int j = __ffs(~occ & 0xFFFFu) - 1;
      s = r * kSPL + j;
      const uint64_t row = tb * kSlots + s;
      *kptr(t, row) = key;
      t.digests[row] = (uint8_t)d;
      *sptr(t, row) = s_in;
      summ_invalidate(t, tb, s);
      store_occ(t, tb, r, occ | (1u << j));
    }
    s = tile.shfl(s, fl);
    const uint64_t row = tb * kSlots + s;
    write_row<VEC>(value_row(t, row), vin, pre, dim, r);
    ctr[row < t.fast_rows ? kVFast : kVOver]++;
    size_delta++;
    outcome = kInserted;
  } else if (!admit) {
    outcome = kRejected;
  } else {
    const uint64_t row = tb * kSlots + m;
    const int ol = m / kSPL;
    float* vr = value_row(t, row);
    if (a.collect) {
      if (r == ol) {
        a.ek[kRecU64 * i] = *kptr(t, row);
        a.es[kRecU64 * i] = minv;
      }
      copy_row<kG, VEC>(a.ev + (uint64_t)i * dim, vr, dim, r);
      ctr[row < t.fast_rows ? kVFast : kVOver]++;
    }
    if (r == ol) {
      *kptr(t, row) = key;
      t.digests[row] = (uint8_t)d;
      *sptr(t, row) = s_in;
      t.smin[tb * 8 + ol] = s_in < rest ? s_in : rest;  // the group stays exact
    }
    write_row<VEC>(vr, vin, pre, dim, r);
    ctr[row < t.fast_rows ? kVFast : kVOver]++;
    outcome = kEvicted;
    if (fel_open && r == 0) atomicMin(&a.sc->first_ev, i);
  }
  if (r == 0) a.outcomes[i] = outcome;
}

__device__ __forceinline__ void flush_tile_counters(const Tile8& tile, const TableDev& t,
                                                    ctr_t* ctr, int size_delta) {
  if (tile.thread_rank() != 0) {
#pragma unroll
    for (int k = 0; k < 6; k++) ctr[k] = 0;
    size_delta = 0;
  }
  flush_counters<256>(t.counters, ctr, 6);
  long long v = size_delta;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);  // 64-bit warp sum
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(t.size, (unsigned long long)v);
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

#ifndef HKV_DUAL_CSORT
#define HKV_DUAL_CSORT 1  // counting-sort rank prep (0: radix sort of the 2n pairs)
#endif
#ifndef HKV_DUAL_ROUNDS
#define HKV_DUAL_ROUNDS 1  // 0: the 8-lane-tile turn-counter dataflow (k_dual_flow)
#endif

// 2n (bucket, code) pairs, code = 2i + which; a second bucket equal to the
// first is parked at bucket `none` (sorts last, ignored).
__global__ void k_dual_pairs(const uint32_t* __restrict__ b1s, const uint32_t* __restrict__ b2s, int64_t n,
                             uint32_t none, uint32_t* __restrict__ pk, uint32_t* __restrict__ pv, const Scalars* sc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || sc->err) return;
  const uint32_t b1 = b1s[i], b2 = b2s[i];
  pk[2 * i] = b1;
  pv[2 * i] = (uint32_t)(2 * i);
  pk[2 * i + 1] = b2 == b1 ? none : b2;
  pv[2 * i + 1] = (uint32_t)(2 * i + 1);
}

// hp[p] = p at the first position of each bucket's run, else 0 (max-scanned next)
__global__ void k_dual_heads(const uint32_t* __restrict__ sk, int64_t m, uint32_t* __restrict__ hp) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= m) return;
  hp[p] = (p == 0 || sk[p - 1] != sk[p]) ? (uint32_t)p : 0u;
}

// rank of op 2i+which in its bucket's batch-ordered op list
__global__ void k_dual_ranks(const uint32_t* __restrict__ sk, const uint32_t* __restrict__ sv,
                             const uint32_t* __restrict__ first, int64_t m, uint32_t none,
                             uint32_t* __restrict__ rank) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= m || sk[p] == none) return;
  rank[sv[p]] = (uint32_t)(p - first[p]);
}

// Counting-sort rank prep (HKV_DUAL_CSORT): the ranks need only each
// bucket's references in batch order, and a bucket holds ~2 of them, so a
// count / scan / scatter into per-bucket lists (all L2-resident: 4 B per
// bucket, 4 B per reference) plus a count of smaller op indices inside the
// reference's own short list replaces the radix sort of the 2n pairs.
__global__ void k_dcount(const uint32_t* __restrict__ b1s, const uint32_t* __restrict__ b2s, int64_t n,
                         uint32_t* __restrict__ cnt, const Scalars* sc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || sc->err) return;
  const uint32_t b1 = b1s[i], b2 = b2s[i];
  atomicAdd(cnt + b1, 1u);
  if (b2 != b1) atomicAdd(cnt + b2, 1u);
}
// list[off[b] .. off[b+1]) = codes 2i + which of bucket b's references (any order)
__global__ void k_dscatter(const uint32_t* __restrict__ b1s, const uint32_t* __restrict__ b2s, int64_t n,
                           const uint32_t* __restrict__ off, uint32_t* __restrict__ cnt, uint32_t* __restrict__ list,
                           const Scalars* sc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || sc->err) return;
  const uint32_t b1 = b1s[i], b2 = b2s[i];
  list[off[b1] + atomicSub(cnt + b1, 1u) - 1u] = (uint32_t)(2 * i);
  if (b2 != b1) list[off[b2] + atomicSub(cnt + b2, 1u) - 1u] = (uint32_t)(2 * i + 1);
}
// rank of reference 2i + which = references of its bucket from smaller op indices
__global__ void k_drank(const uint32_t* __restrict__ b1s, const uint32_t* __restrict__ b2s, int64_t n,
                        const uint32_t* __restrict__ off, const uint32_t* __restrict__ list,
                        uint32_t* __restrict__ rank, const Scalars* sc) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= 2 * n || sc->err) return;
  const uint32_t i = (uint32_t)(p >> 1);
  const uint32_t b1 = b1s[i], b2 = b2s[i];
  if ((p & 1) && b2 == b1) return;
  const uint32_t b = (p & 1) ? b2 : b1;
  const uint32_t lo = off[b], hi = off[b + 1];
  uint32_t r = 0;
  uint32_t q = lo;
  if (hi - lo > 16) {
    // a hot bucket (skewed batch): the warp's lanes mostly share the list,
    // so read it through L1 four entries at a time.  The work stays
    // quadratic in the bucket's reference count -- fine for zipf-skewed
    // batches, slow (not wrong) for a batch of one repeated key.
    for (; q < hi && (q & 3u); q++) r += (__ldg(list + q) >> 1) < i;
    for (; q + 4 <= hi; q += 4) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(list + q));
      r += ((v.x >> 1) < i) + ((v.y >> 1) < i) + ((v.z >> 1) < i) + ((v.w >> 1) < i);
    }
  }
  for (; q < hi; q++) r += (list[q] >> 1) < i;
  rank[p] = r;
}

template <int VEC>
__global__ void __launch_bounds__(256) k_dual_flow(TableDev t, OpArgs a, const uint32_t* __restrict__ b1s,
                                                   const uint32_t* __restrict__ b2s,
                                                   const uint32_t* __restrict__ rank, unsigned long long* turn,
                                                   unsigned long long tag, int64_t n) {
  if (a.sc->err) return;
  const Tile8 tile;
  const int r = tile.thread_rank();
  const uint64_t clock0 = *t.clock;
  const bool fel_open = !*t.fel_set;
  ctr_t ctr[6] = {0, 0, 0, 0, 0, 0};
  int sd = 0;
  unsigned* next = &a.sc->npend[0];
  while (true) {
    unsigned i = 0;
    if (r == 0) i = atomicAdd(next, 1u);
    i = tile.shfl(i, 0);
    if ((int64_t)i >= n) break;
    InRow pre;  // the input row does not depend on the table: load it before waiting
    pre.ok = false;
    if (a.values) pre = prefetch_row<VEC>(a.values + (uint64_t)i * t.dim, t.dim, r);
    const uint32_t b1 = b1s[i], b2 = b2s[i];
    const uint32_t r1 = rank[2 * i];
    const uint32_t r2 = b2 == b1 ? 0u : rank[2 * i + 1];
    // every lane acquires: the bucket data it reads next was published with a release
    if (r1) while (ld_acquire_u64(turn + b1) < (tag | r1)) __nanosleep(32);
    if (b2 != b1 && r2) while (ld_acquire_u64(turn + b2) < (tag | r2)) __nanosleep(32);
    process_op<VEC>(t, a, tile, i, clock0, fel_open, ctr, sd, pre);
    __threadfence();
    tile.sync();
    if (r == 0) {
      st_release_u64(turn + b1, tag | (r1 + 1));
      if (b2 != b1) st_release_u64(turn + b2, tag | (r2 + 1));
    }
  }
  flush_tile_counters(tile, t, ctr, sd);
}

cudaError_t run_dual(const TableDev& t, OpArgs a, int64_t n, int log2_buckets, Workspace& ws,
                     unsigned long long* turn, unsigned long long tag, int vec, cudaStream_t s, int num_sms) {
  cudaError_t e;
  const int64_t m = 2 * n;
  const uint32_t none = (uint32_t)(1ull << log2_buckets);
  const unsigned blk = (unsigned)((n + 255) / 256), blk2 = (unsigned)((m + 255) / 256);
  ktimer_begin("dual_ranks", s, 2);
#if HKV_DUAL_CSORT
  {
    const int64_t nb = (int64_t)none;  // buckets
    if ((e = cudaMemsetAsync(ws.dcnt, 0, (size_t)(nb + 1) * 4, s))) return e;
    k_dcount<<<blk, 256, 0, s>>>(ws.bkt, ws.b2, n, ws.dcnt, ws.sc);
    size_t sb = ws.dcub_bytes;
    if ((e = cub::DeviceScan::ExclusiveSum(ws.dcub, sb, ws.dcnt, ws.doff, (int)(nb + 1), s))) return e;
    k_dscatter<<<blk, 256, 0, s>>>(ws.bkt, ws.b2, n, ws.doff, ws.dcnt, ws.dpk, ws.sc);
    k_drank<<<blk2, 256, 0, s>>>(ws.bkt, ws.b2, n, ws.doff, ws.dpk, ws.drank, ws.sc);
    ktimer_end("dual_ranks", s, 2);
    g_launches += 6;
    if ((e = cudaGetLastError())) return e;
  }
#else
  k_dual_pairs<<<blk, 256, 0, s>>>(ws.bkt, ws.b2, n, none, ws.dpk, ws.dpv, ws.sc);
  size_t bytes = ws.dcub_bytes;
  if ((e = cub::DeviceRadixSort::SortPairs(ws.dcub, bytes, ws.dpk, ws.dsk, ws.dpv, ws.dsv, (int)m, 0,
                                           log2_buckets + 1, s)))
    return e;
  k_dual_heads<<<blk2, 256, 0, s>>>(ws.dsk, m, ws.dpk);
  bytes = ws.dcub_bytes;
  if ((e = cub::DeviceScan::InclusiveScan(ws.dcub, bytes, ws.dpk, ws.dpv, cub::Max(), (int)m, s))) return e;
  k_dual_ranks<<<blk2, 256, 0, s>>>(ws.dsk, ws.dsv, ws.dpv, m, none, ws.drank);
  ktimer_end("dual_ranks", s, 2);
  g_launches += 10;
#endif
#if HKV_DUAL_ROUNDS
  return run_dual_rounds(t, a, n, ws.drank, turn, tag, vec, s, num_sms);
#endif
  int per_sm = 0;
  void* fn = vec == 4 ? (void*)k_dual_flow<4> : vec == 2 ? (void*)k_dual_flow<2> : (void*)k_dual_flow<1>;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0))) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)per_sm * num_sms;
  const int64_t want = (n * kG + 255) / 256;
  if (blocks > want) blocks = want < 1 ? 1 : want;
  if (vec == 4) k_dual_flow<4><<<(unsigned)blocks, 256, 0, s>>>(t, a, ws.bkt, ws.b2, ws.drank, turn, tag, n);
  else if (vec == 2) k_dual_flow<2><<<(unsigned)blocks, 256, 0, s>>>(t, a, ws.bkt, ws.b2, ws.drank, turn, tag, n);
  else k_dual_flow<1><<<(unsigned)blocks, 256, 0, s>>>(t, a, ws.bkt, ws.b2, ws.drank, turn, tag, n);
  g_launches++;
  return cudaGetLastError();
}

cudaError_t ws_reserve_dual(Workspace& ws, int64_t n, int log2_buckets) {
  cudaError_t e = cudaSuccess;
  const int64_t m = 2 * n;
  const int64_t nb1 = (1ll << log2_buckets) + 1;
  if (nb1 > ws.dbk) {
    if (ws.dcnt) cudaFree(ws.dcnt);
    if (ws.doff) cudaFree(ws.doff);
    ws.dcnt = ws.doff = nullptr;
    ws.dbk = 0;
    if ((e = cudaMalloc((void**)&ws.dcnt, (size_t)nb1 * 4)) || (e = cudaMalloc((void**)&ws.doff, (size_t)nb1 * 4)))
      return e;
    ws.dbk = nb1;
  }
  if (m > ws.dcap) {
    const int64_t c = m + m / 4 + 2048;
    uint32_t** arrs[] = {&ws.dpk, &ws.dpv, &ws.dsk, &ws.dsv, &ws.drank};
    for (uint32_t** p : arrs) {
      if (*p) cudaFree(*p);
      *p = nullptr;
      if ((e = cudaMalloc((void**)p, sizeof(uint32_t) * (size_t)c))) return e;
    }
    size_t b_sort = 0, b_scan = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b_sort, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (uint32_t*)nullptr, (int)c, 0, log2_buckets + 1);
    cub::DeviceScan::InclusiveScan(nullptr, b_scan, (uint32_t*)nullptr, (uint32_t*)nullptr, cub::Max(), (int)c);
    const size_t need = b_sort > b_scan ? b_sort : b_scan;
    if (ws.dcub) cudaFree(ws.dcub);
    ws.dcub = nullptr;
    if ((e = cudaMalloc(&ws.dcub, need))) return e;
    ws.dcub_bytes = need;
    ws.dcap = c;
  }
  // the counting-sort prep scans the per-bucket counters with the same temp storage
  size_t b_bscan = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b_bscan, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)ws.dbk);
  if (b_bscan > ws.dcub_bytes) {
    if (ws.dcub) cudaFree(ws.dcub);
    ws.dcub = nullptr;
    ws.dcub_bytes = 0;
    if ((e = cudaMalloc(&ws.dcub, b_bscan))) return e;
    ws.dcub_bytes = b_bscan;
  }
  return cudaSuccess;
}

void ws_free_dual(Workspace& ws) {
  void* ptrs[] = {ws.dpk, ws.dpv, ws.dsk, ws.dsv, ws.drank, ws.dcub, ws.dcnt, ws.doff};
  for (void* p : ptrs)
    if (p) cudaFree(p);
}

}  // namespace hkv
