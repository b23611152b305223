// hkv_mutate.cu — inserter/updater kernels: insert_or_assign, insert_and_evict,
// find_or_insert, erase, assign, assign_scores.
//
// Semantics: the reference's batch engine equals applying the ops one at a
// time in ascending batch index (leader rounds,
// table.py:945-985).  The B200 engine reproduces that order exactly:
//
//  single mode  -- a key's whole candidate space is one bucket, so ops on
//    different buckets commute.  k_prep hashes the batch, a stable radix sort
//    groups ops by bucket (ascending batch index inside a bucket), k_heads
//    finds the bucket segments, and k_apply_segments gives each segment to one
//    8-lane tile that applies its ops in order with exclusive ownership of the
//    bucket: no CAS, no retries, bit-exact at any contention.
//  dual mode    -- an op touches two buckets; k_dual_rounds runs the
//    reference's leader rounds on the device (table.py:945-962): per round
//    every pending op bids its batch index on both buckets (atomicMax on a
//    round-tagged word), ops that win both buckets apply in parallel, the
//    rest wait.  One cooperative kernel, grid-wide barrier between phases.
//
// Per op (process_op) the tile restates _round_upsert (table.py:1025-1119):
// digest probe (one 128-B line) -> hit: score refresh + value write/read ->
// miss: insert at the lowest free slot (occupancy bitmap, __ffs) or, on a full
// bucket, tile-wide argmin over the score row, admission test and eviction
// (_finish_admission, table.py:1121-1163).
#include <cub/cub.cuh>

#include "hkv_kernels.h"
#include "hkv_probe.cuh"

namespace hkv {

// ---------------------------------------------------------------------------
// per-op processor (one 8-lane tile, exclusive ownership of the op's buckets)
// ---------------------------------------------------------------------------
template <int VEC>
__device__ __forceinline__ void process_op(const TableDev& t, const OpArgs& a,
                                           const cg::thread_block_tile<kG>& tile, uint32_t i,
                                           uint64_t clock0, bool fel_open, unsigned long long* ctr,
                                           long long& size_delta) {
  const int r = tile.thread_rank();
  const int dim = t.dim;
  const uint64_t key = a.keys[i];
  const uint64_t h = fmix64(key);
  const uint32_t d = digest_of(h);
  const uint64_t b1 = h & t.mask;
  uint64_t hb = b1;
  const uint32_t occ1 = load_occ(t, b1, r);
  int slot = probe_bucket<true, false>(t, tile, b1, key, d, occ1, ctr[kCompares]);
  ctr[kLoads]++;
  uint64_t b2 = b1;
  uint32_t occ2 = occ1;
  if (t.dual) {
    b2 = second_hash(h) & t.mask;
    if (slot < 0) {
      occ2 = load_occ(t, b2, r);
      slot = probe_bucket<true, false>(t, tile, b2, key, d, occ2, ctr[kCompares]);
      ctr[kLoads]++;
      hb = b2;
    }
  }
  uint8_t outcome;
  if (a.op == kOpErase) {
    // _round_erase, table.py:1017-1023: key -> EMPTY; digest/score/value stay stale
    if (slot >= 0) {
      if (slot / kSPL == r) {
        const uint64_t row = hb * kSlots + slot;
        t.keys[row] = kEmptyKey;
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
      const uint64_t old = hit_needs_old(t.policy) ? t.scores[row] : 0;
      t.scores[row] = hit_score(t.policy, old, a.epoch, tick, a.scores != nullptr, cs);
    }
    float* vr = value_row(t, row);
    if (a.op == kOpFindOrInsert) {
      copy_row<kG, VEC>(vin, vr, dim, r);
      outcome = kFound;
    } else {
      copy_row<kG, VEC>(vr, vin, dim, r);
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
  uint64_t minv = 0;
  bool admit = false;
  bool free_insert = false;
  if (!t.dual) {
    const int occ_total = tile_sum<kG>(tile, __popc(occ1));
    if (occ_total < kSlots) {
      free_insert = true;  // _bulk_insert_free, table.py:1072-1076
    } else {
      bucket_min(t, tile, b1, minv, m);  // table.py:1079-1083
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
      uint64_t min1, min2;  // D2, table.py:1096-1119
      int m1, m2;
      bucket_min(t, tile, b1, min1, m1);
      bucket_min(t, tile, b2, min2, m2);
      ctr[kScans] += 2;
      const bool use2 = min2 < min1;
      tb = use2 ? b2 : b1;
      m = use2 ? m2 : m1;
      minv = use2 ? min2 : min1;
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
      t.keys[row] = key;
      t.digests[row] = (uint8_t)d;
      t.scores[row] = s_in;
      store_occ(t, tb, r, occ | (1u << j));
    }
    s = tile.shfl(s, fl);
    const uint64_t row = tb * kSlots + s;
    copy_row<kG, VEC>(value_row(t, row), vin, dim, r);
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
        a.ek[i] = t.keys[row];
        a.es[i] = minv;
      }
      copy_row<kG, VEC>(a.ev + (uint64_t)i * dim, vr, dim, r);
      ctr[row < t.fast_rows ? kVFast : kVOver]++;
    }
    if (r == ol) {
      t.keys[row] = key;
      t.digests[row] = (uint8_t)d;
      t.scores[row] = s_in;
    }
    copy_row<kG, VEC>(vr, vin, dim, r);
    ctr[row < t.fast_rows ? kVFast : kVOver]++;
    outcome = kEvicted;
    if (fel_open && r == 0) atomicMin(&a.sc->first_ev, i);
  }
  if (r == 0) a.outcomes[i] = outcome;
}

__device__ __forceinline__ void flush_tile_counters(const cg::thread_block_tile<kG>& tile, const TableDev& t,
                                                    unsigned long long* ctr, long long size_delta) {
  if (tile.thread_rank() != 0) {
#pragma unroll
    for (int k = 0; k < 6; k++) ctr[k] = 0;
    size_delta = 0;
  }
  flush_counters<256>(t.counters, ctr, 6);
  long long v = size_delta;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(t.size, (unsigned long long)v);
}

// ---------------------------------------------------------------------------
// pipeline kernels
// ---------------------------------------------------------------------------
__global__ void k_prep(TableDev t, const uint64_t* __restrict__ keys, int64_t n, uint32_t* __restrict__ bkt,
                       uint32_t* __restrict__ idx, uint32_t* __restrict__ b2, Scalars* sc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {
    sc->first_ev = 0xFFFFFFFFu;
    sc->size_before = (long long)*t.size;
  }
  if (i >= n) return;
  const uint64_t key = keys[i];
  if (key >= kLockedKey) atomicOr(&sc->err, 1);  // table.py:168-169, checked before any mutation
  const uint64_t h = fmix64(key);
  bkt[i] = (uint32_t)(h & t.mask);
  idx[i] = (uint32_t)i;
  if (b2) b2[i] = (uint32_t)(second_hash(h) & t.mask);
}

__global__ void k_heads(const uint32_t* __restrict__ sb, int64_t n, uint32_t* __restrict__ seg, Scalars* sc) {
  if (sc->err) return;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool head = p < n && (p == 0 || sb[p] != sb[p - 1]);
  const unsigned mask = __ballot_sync(0xffffffffu, head);
  if (!mask) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  unsigned base = 0;
  if (lane == leader) base = atomicAdd(&sc->nseg, (unsigned)__popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (head) seg[base + __popc(mask & ((1u << lane) - 1))] = (uint32_t)p;
}

template <int VEC>
__global__ void __launch_bounds__(256) k_apply_segments(TableDev t, OpArgs a, const uint32_t* __restrict__ sb,
                                                        const uint32_t* __restrict__ sidx,
                                                        const uint32_t* __restrict__ seg, int64_t n) {
  if (a.sc->err) return;
  auto tile = cg::tiled_partition<kG>(cg::this_thread_block());
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / kG;
  const uint64_t clock0 = *t.clock;
  const bool fel_open = !*t.fel_set;
  const unsigned nseg = a.sc->nseg;
  unsigned long long ctr[6] = {0, 0, 0, 0, 0, 0};
  long long sd = 0;
  for (int64_t s = gid; s < nseg; s += ngroups) {
    int64_t p = seg[s];
    const uint32_t b = sb[p];
    while (true) {
      process_op<VEC>(t, a, tile, sidx[p], clock0, fel_open, ctr, sd);
      if (++p >= n || sb[p] != b) break;
    }
  }
  flush_tile_counters(tile, t, ctr, sd);
}

// Dual mode: device-side leader rounds (table.py:945-962).
template <int VEC>
__global__ void __launch_bounds__(256) k_dual_rounds(TableDev t, OpArgs a, const uint32_t* __restrict__ b1s,
                                                     const uint32_t* __restrict__ b2s, uint32_t* pend0,
                                                     uint32_t* pend1, unsigned long long* lead,
                                                     unsigned long long* round_ctr, int64_t n) {
  cg::grid_group grid = cg::this_grid();
  if (a.sc->err) return;
  auto tile = cg::tiled_partition<kG>(cg::this_thread_block());
  const int r = tile.thread_rank();
  const int64_t tid = grid.thread_rank();
  const int64_t nthreads = grid.size();
  const int64_t gid = tid / kG;
  const int64_t ngroups = nthreads / kG;
  const uint64_t clock0 = *t.clock;
  const bool fel_open = !*t.fel_set;
  const unsigned long long round_base = *round_ctr;
  unsigned long long ctr[6] = {0, 0, 0, 0, 0, 0};
  long long sd = 0;
  unsigned m = (unsigned)n;
  uint32_t* cur = pend0;
  uint32_t* nxt = pend1;
  for (unsigned long long rd = 1;; rd++) {
    const unsigned long long R = (round_base + rd) << 32;
    if (tid == 0) a.sc->npend[rd & 1] = 0;
    for (int64_t j = tid; j < m; j += nthreads) {
      const uint32_t i = cur[j];
      const unsigned long long tag = R | (0xFFFFFFFFull - i);
      atomicMax(&lead[b1s[i]], tag);
      atomicMax(&lead[b2s[i]], tag);
    }
    grid.sync();
    for (int64_t j = gid; j < m; j += ngroups) {
      const uint32_t i = cur[j];
      const unsigned long long tag = R | (0xFFFFFFFFull - i);
      const bool leader = lead[b1s[i]] == tag && lead[b2s[i]] == tag;
      if (leader) {
        process_op<VEC>(t, a, tile, i, clock0, fel_open, ctr, sd);
      } else if (r == 0) {
        const unsigned pos = atomicAdd(&a.sc->npend[rd & 1], 1u);
        nxt[pos] = i;
      }
    }
    grid.sync();
    m = *((volatile unsigned*)&a.sc->npend[rd & 1]);
    if (m == 0) {
      if (tid == 0) *round_ctr = round_base + rd;
      break;
    }
    uint32_t* tmp = cur;
    cur = nxt;
    nxt = tmp;
  }
  flush_tile_counters(tile, t, ctr, sd);
}

// Clock advance + first_eviction_lambda (table.py:986-991) + error latch.
__global__ void k_finalize(TableDev t, Scalars* sc, const uint8_t* __restrict__ outcomes, int64_t n,
                           unsigned long long clock_advance, int add_found) {
  if (sc->err) {
    if (threadIdx.x == 0) atomicOr(t.err, sc->err);
    return;
  }
  if (threadIdx.x == 0) *t.clock += clock_advance + (add_found ? sc->nfound : 0ull);
  const unsigned fe = sc->first_ev;
  if (*t.fel_set || fe == 0xFFFFFFFFu || outcomes == nullptr) return;
  unsigned cnt = 0;
  for (int64_t j = threadIdx.x; j < (int64_t)fe; j += blockDim.x) cnt += outcomes[j] == kInserted;
  typedef cub::BlockReduce<unsigned, 1024> BR;
  __shared__ typename BR::TempStorage tmp;
  const unsigned tot = BR(tmp).Sum(cnt);
  if (threadIdx.x == 0) {
    *t.fel = (double)(sc->size_before + (long long)tot) / (double)t.capacity;
    *t.fel_set = 1;
  }
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
  auto tile = cg::tiled_partition<kG>(cg::this_thread_block());
  const int r = tile.thread_rank();
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / kG;
  const int64_t ne = sc->err ? 0 : *n_ev;
  for (int64_t j = gid; j < ne; j += ngroups) {
    const uint32_t i = list[j];
    if (r == 0) {
      ek[j] = ek_tmp[i];
      es[j] = es_tmp[i];
    }
    copy_row<kG, VEC>(ev + j * dim, ev_tmp + (uint64_t)i * dim, dim, r);
  }
}

__global__ void k_zero_count(const Scalars* sc, long long* n_ev) {
  if (sc->err) *n_ev = 0;
}

// ---------------------------------------------------------------------------
// assign / assign_scores (updater role; structure never changes)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_assign_find(TableDev t, const uint64_t* __restrict__ keys, int64_t n,
                                                     uint32_t* __restrict__ rows, uint8_t* __restrict__ outcomes,
                                                     Scalars* sc) {
  if (sc->err) return;
  auto tile = cg::tiled_partition<kG>(cg::this_thread_block());
  const int r = tile.thread_rank();
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / kG;
  unsigned long long ctr[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t i = gid; i < n; i += ngroups) {
    const uint64_t key = keys[i];
    const uint64_t h = fmix64(key);
    const uint32_t d = digest_of(h);
    uint64_t b = h & t.mask;
    int slot = probe_bucket<false, false>(t, tile, b, key, d, 0xFFFFu, ctr[kCompares]);
    ctr[kLoads]++;
    if (slot < 0 && t.dual) {
      b = second_hash(h) & t.mask;
      slot = probe_bucket<false, false>(t, tile, b, key, d, 0xFFFFu, ctr[kCompares]);
      ctr[kLoads]++;
    }
    if (r == 0) {
      rows[i] = slot >= 0 ? (uint32_t)(b * kSlots + slot) : 0xFFFFFFFFu;
      outcomes[i] = slot >= 0 ? kUpdated : kNotFound;
    }
  }
  if (r != 0) {
#pragma unroll
    for (int k = 0; k < 6; k++) ctr[k] = 0;
  }
  flush_counters<256>(t.counters, ctr, 6);
}

template <int VEC>
__global__ void __launch_bounds__(256) k_assign_apply(TableDev t, const float* __restrict__ values,
                                                      const uint64_t* __restrict__ scores, int refresh,
                                                      uint64_t epoch, const uint32_t* __restrict__ rows,
                                                      const uint32_t* __restrict__ ranks,
                                                      const uint64_t* __restrict__ ticks,
                                                      const uint32_t* __restrict__ sb,
                                                      const uint32_t* __restrict__ sidx,
                                                      const uint32_t* __restrict__ seg, int64_t n, Scalars* sc) {
  if (sc->err) return;
  auto tile = cg::tiled_partition<kG>(cg::this_thread_block());
  const int r = tile.thread_rank();
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / kG;
  const uint64_t clock0 = *t.clock;
  const unsigned nseg = sc->nseg;
  unsigned long long ctr[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t s = gid; s < nseg; s += ngroups) {
    int64_t p = seg[s];
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
            t.scores[row] = scores[i];
          } else if (refresh) {
            const uint64_t tick = ticks ? ticks[i] : clock0 + (uint64_t)ranks[i] + 1;
            t.scores[row] = hit_score(t.policy, t.scores[row], epoch, tick, false, 0);
          }
        }
      }
      if (++p >= n || sb[p] != b) break;
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
  if (sc->err || n <= 0) return;
  sc->nfound = (unsigned long long)ranks[n - 1] + (outcomes[n - 1] == kUpdated ? 1ull : 0ull);
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

cudaError_t ws_reserve(Workspace& ws, int64_t n, int dim, bool need_ev, bool dual) {
  cudaError_t e = cudaSuccess;
  if (!ws.sc) {
    e = cudaMalloc((void**)&ws.sc, sizeof(Scalars));
    if (e) return e;
  }
  if (n > ws.cap_n) {
    const int64_t c = n + n / 4 + 1024;
    if ((e = grow(ws.bkt, c)) || (e = grow(ws.idx, c)) || (e = grow(ws.sbkt, c)) || (e = grow(ws.sidx, c)) ||
        (e = grow(ws.seg, c)) || (e = grow(ws.aux, c)) || (e = grow(ws.aux2, c)))
      return e;
    if (ws.b2) { cudaFree(ws.b2); ws.b2 = nullptr; }
    if (ws.pend) { cudaFree(ws.pend); ws.pend = nullptr; }
    ws.cap_n = c;
  }
  if (dual && !ws.b2) {
    if ((e = grow(ws.b2, ws.cap_n)) || (e = grow(ws.pend, ws.cap_n))) return e;
  }
  if (need_ev && (ws.cap_ev < n || ws.dim != dim)) {
    const int64_t c = ws.cap_n;
    if ((e = grow(ws.ek, c)) || (e = grow(ws.es, c)) || (e = grow(ws.ev, c * dim))) return e;
    ws.cap_ev = c;
    ws.dim = dim;
  }
  // CUB temp storage: the largest of sort / select / scan for cap_n items
  size_t b_sort = 0, b_sel = 0, b_scan = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b_sort, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)ws.cap_n, 0, 32);
  cub::CountingInputIterator<int64_t> cnt(0);
  cub::TransformInputIterator<bool, IsEvicted, cub::CountingInputIterator<int64_t>> fl(cnt, IsEvicted{nullptr});
  cub::DeviceSelect::Flagged(nullptr, b_sel, cnt, fl, (uint32_t*)nullptr, (long long*)nullptr, (int)ws.cap_n);
  cub::TransformInputIterator<uint32_t, IsUpdated, cub::CountingInputIterator<int64_t>> up(cnt, IsUpdated{nullptr});
  cub::DeviceScan::ExclusiveSum(nullptr, b_scan, up, (uint32_t*)nullptr, (int)ws.cap_n);
  size_t need = b_sort > b_sel ? b_sort : b_sel;
  if (b_scan > need) need = b_scan;
  if (need > ws.cub_bytes) {
    if (ws.cub_tmp) cudaFree(ws.cub_tmp);
    ws.cub_tmp = nullptr;
    if ((e = cudaMalloc(&ws.cub_tmp, need))) return e;
    ws.cub_bytes = need;
  }
  return cudaSuccess;
}

void ws_free(Workspace& ws) {
  void* ptrs[] = {ws.bkt, ws.idx, ws.sbkt, ws.sidx, ws.seg, ws.aux, ws.aux2, ws.b2, ws.pend,
                  ws.ek, ws.es, ws.ev, ws.cub_tmp, ws.sc};
  for (void* p : ptrs)
    if (p) cudaFree(p);
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
  k_heads<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ws.sbkt, n, ws.seg, ws.sc);
  g_launches++;
  return cudaGetLastError();
}

cudaError_t run_mutation(const TableDev& t, OpArgs a, int64_t n, int log2_buckets, Workspace& ws,
                         unsigned long long* round_ctr, unsigned long long* lead, int64_t* n_evicted,
                         uint64_t* ek_out, float* ev_out, uint64_t* es_out, uint64_t clock_advance,
                         cudaStream_t s, int num_sms) {
  cudaError_t e;
  const bool collect = a.collect != 0;
  if ((e = ws_reserve(ws, n, t.dim, collect, t.dual != 0))) return e;
  a.sc = ws.sc;
  a.ek = ws.ek;
  a.es = ws.es;
  a.ev = ws.ev;
  if ((e = cudaMemsetAsync(ws.sc, 0, sizeof(Scalars), s))) return e;
  if (n > 0) {
    k_prep<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(t, a.keys, n, ws.bkt, ws.idx, t.dual ? ws.b2 : nullptr,
                                                        ws.sc);
    g_launches++;
    const int vec = vec_of(t.dim, a.values, t.vfast, t.vover, collect ? ws.ev : nullptr);
    if (!t.dual) {
      if ((e = sort_segments(ws, n, log2_buckets, s))) return e;
      const int64_t blocks = tile_blocks(n, num_sms);
      ktimer_begin("apply", s);
      if (vec == 4) k_apply_segments<4><<<(unsigned)blocks, 256, 0, s>>>(t, a, ws.sbkt, ws.sidx, ws.seg, n);
      else if (vec == 2) k_apply_segments<2><<<(unsigned)blocks, 256, 0, s>>>(t, a, ws.sbkt, ws.sidx, ws.seg, n);
      else k_apply_segments<1><<<(unsigned)blocks, 256, 0, s>>>(t, a, ws.sbkt, ws.sidx, ws.seg, n);
      ktimer_end("apply", s);
      g_launches++;
    } else {
      // cooperative grid: all blocks co-resident
      void* fn = vec == 4 ? (void*)k_dual_rounds<4> : vec == 2 ? (void*)k_dual_rounds<2> : (void*)k_dual_rounds<1>;
      int per_sm = 0;
      if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0))) return e;
      if (per_sm < 1) per_sm = 1;
      int64_t blocks = (int64_t)per_sm * num_sms;
      const int64_t want = (n * kG + 255) / 256;
      if (blocks > want) blocks = want < 1 ? 1 : want;
      TableDev tt = t;
      const uint32_t* b1s = ws.bkt;
      const uint32_t* b2s = ws.b2;
      uint32_t* p0 = ws.idx;
      uint32_t* p1 = ws.pend;
      int64_t nn = n;
      void* args[] = {&tt, &a, &b1s, &b2s, &p0, &p1, &lead, &round_ctr, &nn};
      ktimer_begin("dual_rounds", s);
      if ((e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)blocks), dim3(256), args, 0, s))) return e;
      ktimer_end("dual_rounds", s);
      g_launches++;
    }
  }
  k_finalize<<<1, 1024, 0, s>>>(t, ws.sc, a.op == kOpErase ? nullptr : a.outcomes, n, clock_advance, 0);
  g_launches++;
  if (collect) {
    size_t bytes = ws.cub_bytes;
    cub::CountingInputIterator<int64_t> cnt(0);
    cub::TransformInputIterator<bool, IsEvicted, cub::CountingInputIterator<int64_t>> fl(cnt, IsEvicted{a.outcomes});
    long long* nev = reinterpret_cast<long long*>(n_evicted);
    if (n > 0) {
      if ((e = cub::DeviceSelect::Flagged(ws.cub_tmp, bytes, cnt, fl, ws.aux, nev, (int)n, s))) return e;
      g_launches += 2;
      const int vec = vec_of(t.dim, ev_out, ws.ev, nullptr, nullptr);
      const int64_t blocks = tile_blocks(n, num_sms);
      if (vec == 4)
        k_evict_gather<4><<<(unsigned)blocks, 256, 0, s>>>(ws.sc, ws.aux, nev, ws.ek, ws.es, ws.ev, ek_out, es_out,
                                                           ev_out, t.dim, n);
      else if (vec == 2)
        k_evict_gather<2><<<(unsigned)blocks, 256, 0, s>>>(ws.sc, ws.aux, nev, ws.ek, ws.es, ws.ev, ek_out, es_out,
                                                           ev_out, t.dim, n);
      else
        k_evict_gather<1><<<(unsigned)blocks, 256, 0, s>>>(ws.sc, ws.aux, nev, ws.ek, ws.es, ws.ev, ek_out, es_out,
                                                           ev_out, t.dim, n);
      g_launches++;
      k_zero_count<<<1, 1, 0, s>>>(ws.sc, nev);
      g_launches++;
    } else {
      if ((e = cudaMemsetAsync(n_evicted, 0, sizeof(int64_t), s))) return e;
    }
  }
  return cudaGetLastError();
}

cudaError_t run_assign(const TableDev& t, const uint64_t* keys, const float* values, const uint64_t* scores,
                       int refresh, uint64_t epoch, int64_t n, uint8_t* outcomes, const uint64_t* ticks,
                       uint64_t clock_advance, int log2_buckets, Workspace& ws, cudaStream_t s, int num_sms) {
  cudaError_t e;
  if ((e = ws_reserve(ws, n, t.dim, false, false))) return e;
  if ((e = cudaMemsetAsync(ws.sc, 0, sizeof(Scalars), s))) return e;
  const bool need_ticks = refresh && !scores && !ticks;
  if (n > 0) {
    k_prep<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(t, keys, n, ws.bkt, ws.idx, nullptr, ws.sc);
    g_launches++;
    const int64_t blocks = tile_blocks(n, num_sms);
    k_assign_find<<<(unsigned)blocks, 256, 0, s>>>(t, keys, n, ws.aux, outcomes, ws.sc);
    g_launches++;
    if (need_ticks) {
      size_t bytes = ws.cub_bytes;
      cub::CountingInputIterator<int64_t> cnt(0);
      cub::TransformInputIterator<uint32_t, IsUpdated, cub::CountingInputIterator<int64_t>> up(cnt,
                                                                                              IsUpdated{outcomes});
      if ((e = cub::DeviceScan::ExclusiveSum(ws.cub_tmp, bytes, up, ws.aux2, (int)n, s))) return e;
      g_launches += 2;
      k_assign_count<<<1, 1, 0, s>>>(ws.sc, ws.aux2, outcomes, n);
      g_launches++;
    }
    if ((e = sort_segments(ws, n, log2_buckets, s))) return e;
    const int vec = vec_of(t.dim, values, t.vfast, t.vover, nullptr);
    ktimer_begin("assign_apply", s);
    if (vec == 4)
      k_assign_apply<4><<<(unsigned)blocks, 256, 0, s>>>(t, values, scores, refresh, epoch, ws.aux, ws.aux2, ticks, ws.sbkt,
                                                         ws.sidx, ws.seg, n, ws.sc);
    else if (vec == 2)
      k_assign_apply<2><<<(unsigned)blocks, 256, 0, s>>>(t, values, scores, refresh, epoch, ws.aux, ws.aux2, ticks, ws.sbkt,
                                                         ws.sidx, ws.seg, n, ws.sc);
    else
      k_assign_apply<1><<<(unsigned)blocks, 256, 0, s>>>(t, values, scores, refresh, epoch, ws.aux, ws.aux2, ticks, ws.sbkt,
                                                         ws.sidx, ws.seg, n, ws.sc);
    ktimer_end("assign_apply", s);
    g_launches++;
  }
  k_finalize<<<1, 1024, 0, s>>>(t, ws.sc, nullptr, n, (refresh && !scores && ticks) ? clock_advance : 0,
                                need_ticks ? 1 : 0);
  g_launches++;
  return cudaGetLastError();
}

}  // namespace hkv
