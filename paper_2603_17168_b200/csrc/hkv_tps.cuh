// hkv_tps.cuh — the single-mode metadata engine shared by the sorted-segment
// pipeline (hkv_mutate.cu) and the collector pipeline (hkv_collect.cu): one
// thread owns a bucket segment and applies its ops in batch order
// (_round_upsert, table.py:1025-1163), recording the value plan.
#pragma once
#include "hkv_kernels.h"
#include "hkv_probe.cuh"

namespace hkv {

// ---------------------------------------------------------------------------
// Single mode value plan.  The metadata pass (k_meta_tps) touches only digest
// lines, occupancy bits, candidate keys and scores; value rows move in
// separate streaming kernels (k_values_read / k_values_write) that have far
// more memory-level parallelism than a thread walking its serial chain.  To
// stay bit-exact the pass records, per op:
//   vrow[i]  destination row when op i is the LAST writer of that row in its
//            segment (a later writer of the same slot retires the earlier one)
//   rrow[8i], rsrc[8i]  for value reads (find_or_insert hits, insert_and_evict
//            victims): the row, and the op whose input currently sits in that
//            row (-1 = the row's content before the batch)
// The last writer of a slot comes from a short scan back through the
// segment, or from a per-thread table once a segment is long (lw_get).
// ---------------------------------------------------------------------------
constexpr uint32_t kNoRow = 0xFFFFFFFFu;
constexpr unsigned kFull = 0xFFFFFFFFu;

// Segment records: one per bucket segment of the sorted batch, compacted
// with one global atomic per block (record order across blocks is arbitrary;
// segments are independent).  Carries the head op so the metadata pass
// starts with one coalesced 24-B read instead of a dependent index hop.
struct SegRec {
  uint64_t key;    // key of the segment's first op
  uint32_t p;      // sorted position of the first op
  uint32_t b;      // bucket
  uint32_t i;      // batch index of the first op
  uint32_t flags;  // bit 0: segment has more than one op; bits 8..15: the first op's digest
};

// Segment records split into two lists: singleton segments from the front
// of `recs`, multi-op segments from the back (recs[cap-1], recs[cap-2], ...),
// so the metadata pass can run each class in lockstep without waste.
//
// Same-key runs (zipf batches: one key can fill tens of thousands of
// consecutive sorted positions of its bucket): for every
// position p inside a multi-op segment, brk[p] = p unless the op at p+1 has the
// same key (then ~0), so a reverse min-scan gives run_end[p] = the last
// position of p's run.  Followers (p-1 has the same key) get the collapsed
// outcome `fcode` and no value row up front; tps_run writes the exceptions.
// Segments of at least kLongSeg ops go to a third list for k_meta_long.
constexpr int kLongSeg = 32;

// Score after `cnt` consecutive hits of one key, the last one with tick tl /
// custom score cs (scoring.py:79-102 applied cnt times; Lfu / EpochLfu
// saturate exactly like the one-at-a-time loop).
__device__ __forceinline__ uint64_t run_hit_score(int policy, uint64_t old, uint64_t epoch, uint64_t tl,
                                                  bool has_custom, uint64_t cs, uint32_t cnt) {
  switch (policy) {
    case kLfu: return (kMaxScore - old < cnt) ? kMaxScore : old + cnt;
    case kEpochLfu: {
      uint64_t low;
      if ((old >> 32) == epoch) {
        low = old & kLow32;
        low = (kLow32 - low < cnt) ? kLow32 : low + cnt;
      } else {
        low = (uint64_t)cnt;  // first hit resets to 1, the rest add 1 each
        if (low > kLow32) low = kLow32;
      }
      return (epoch << 32) | low;
    }
    default: return hit_score(policy, old, epoch, tl, has_custom, cs);
  }
}

// ---------------------------------------------------------------------------
// Single mode, metadata pass, one THREAD per bucket segment (the default).
//
// A thread owns its segment's bucket for the whole batch, keeps the bucket's
// digest line (128 B) and occupancy bitmap (16 B) in shared memory (staged by
// cp.async one segment ahead), updates them in place after its own writes,
// and applies the segment's ops in batch order (table.py:1025-1163).
// Full-bucket decisions use the per-group eviction summary (smin / svalid):
// argmin over 8 group minima (64 B), then the chosen group's 16 scores
// (128 B) to find the slot — np.argmin's first-index tie rule holds because
// groups are in slot order and the first equal slot inside the group is
// taken.  Invalid groups are rescanned (and become valid) on the way.
// Compared with a tile per segment this has 8x the segments in flight and no
// cross-lane collectives, which is what the metadata pass is bound by
// (dependent random loads, profiles/r01).
// ---------------------------------------------------------------------------
#ifndef HKV_TPS_STAGES
#define HKV_TPS_STAGES 2  // line buffers per thread in k_meta_tps (2 or 3)
#endif
#ifndef HKV_SUMM_PREFETCH
#define HKV_SUMM_PREFETCH 1  // L2 prefetch of a full bucket's summary one segment ahead
#endif
#ifndef HKV_TPS_MINB
#define HKV_TPS_MINB 2  // resident blocks per SM the metadata pass is compiled for
#endif
constexpr int kTpsThreads = 256;  // block size of k_meta_tps (stride of its per-thread shared arrays)

struct TpsState {
  int* lw;           // last-writer table: lw[slot * lws] = op that last wrote the slot (global scratch,
  int64_t lws;       //   one 128-entry table per thread; used once a segment passes kLwScan ops)
  const uint32_t* sidx;
  const uint32_t* vrow;
  int64_t p0;        // the segment's first sorted position
  uint64_t rowbase;
  bool tab;          // the table holds this segment's writers
  uint4* L;          // digest line (shared memory, 8 x 16 B)
  uint32_t* O;       // occupancy bitmap words (shared memory, slots 32w .. 32w+31)
  uint64_t* K;       // long-segment engine: the bucket's keys / scores in shared memory
  uint64_t* Sc;      //   (slot j at [j * cs]); nullptr in the global-memory engine
  int cs;
  uint32_t wm[4];    // slots already written by an earlier op of this segment
  uint64_t sm[8];    // group minima (register copy, valid where sv says so)
  uint32_t sv;       // summary valid bits (register copy)
  uint32_t smdirty;  // sm entries to write back
  bool sloaded;      // sm / sv loaded
  bool svdirty;
  uint64_t pk[2];    // k_meta_tps: keys of the head op's first two digest candidates, loaded one
  int npk;           //   segment ahead (register software pipelining); npk of them valid
  uint64_t pol;      // L2 evict_last policy for the per-op plan writes
};

// Register-array helpers written as masked arithmetic over every element:
// an `if (k == idx)` chain gets folded back into a computed index by the
// compiler, which demotes the whole bucket state to local memory.
__device__ __forceinline__ uint32_t eqmask(int a, int b) { return 0u - (uint32_t)(a == b); }
__device__ __forceinline__ uint32_t sel4(const uint32_t (&a)[4], int w) {
  return (a[0] & eqmask(w, 0)) | (a[1] & eqmask(w, 1)) | (a[2] & eqmask(w, 2)) | (a[3] & eqmask(w, 3));
}
__device__ __forceinline__ bool bit128(const uint32_t (&m)[4], int s) { return (sel4(m, s >> 5) >> (s & 31)) & 1u; }
__device__ __forceinline__ void setbit128(uint32_t (&m)[4], int s) {
  const uint32_t bit = 1u << (s & 31);
#pragma unroll
  for (int w = 0; w < 4; w++) m[w] |= bit & eqmask(w, s >> 5);
}
__device__ __forceinline__ uint64_t eqmask64(int a, int b) { return 0ull - (uint64_t)(a == b); }
__device__ __forceinline__ uint64_t sel8(const uint64_t (&a)[8], int g) {
  uint64_t v = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) v |= a[k] & eqmask64(k, g);
  return v;
}
__device__ __forceinline__ void put8(uint64_t (&a)[8], int g, uint64_t v) {
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const uint64_t m = eqmask64(k, g);
    a[k] = (a[k] & ~m) | (v & m);
  }
}

// Bucket rows: global memory (k_meta_tps), or the shared-memory copy of the
// long-segment engine (k_meta_long: written back once when the segment ends,
// so a long serial chain never waits on a global round trip for data it wrote
// itself).
template <bool C>
__device__ __forceinline__ uint64_t bkey(const TableDev& t, const TpsState& S, int j) {
  if constexpr (C) return S.K[j * S.cs]; else return *kptr(t, S.rowbase + j);
}
template <bool C>
__device__ __forceinline__ void set_bkey(const TableDev& t, const TpsState& S, int j, uint64_t v) {
  if constexpr (C) S.K[j * S.cs] = v; else *kptr(t, S.rowbase + j) = v;
}
template <bool C>
__device__ __forceinline__ uint64_t bscore(const TableDev& t, const TpsState& S, int j) {
  if constexpr (C) return S.Sc[j * S.cs]; else return *sptr(t, S.rowbase + j);
}
template <bool C>
__device__ __forceinline__ void set_bscore(const TableDev& t, const TpsState& S, int j, uint64_t v) {
  if constexpr (C) S.Sc[j * S.cs] = v; else *sptr(t, S.rowbase + j) = v;
}
template <bool C>
__device__ __forceinline__ void set_bdigest(const TableDev& t, const TpsState& S, int j, uint32_t d) {
  if constexpr (!C) t.digests[S.rowbase + j] = (uint8_t)d;  // cached: S.L holds it, flushed at the end
}
template <bool C>
__device__ __forceinline__ void set_bocc(const TableDev& t, const TpsState& S, uint64_t b, int w, uint32_t o) {
  if constexpr (!C) {  // cached: S.O holds it, flushed at the end
#if HKV_OCC_HINT
    st_keep(t.bits + b * 4 + w, o, S.pol);
#else
    t.bits[b * 4 + w] = o;
#endif
  }
}

// candidates of digest d: digest-equal and occupied (table.py:243-247)
__device__ __forceinline__ void tps_cand(const TableDev& t, const TpsState& S, uint32_t d, uint32_t (&c)[4]) {
  if (t.digest_filter) {
    uint4 w[8];
#pragma unroll
    for (int k = 0; k < 8; k++) w[k] = S.L[k];
    const uint32_t dd = d * 0x01010101u;
    uint32_t any = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) any |= any16(w[k], dd);
    if ((any & 0x80808080u) == 0) {
#pragma unroll
      for (int q = 0; q < 4; q++) c[q] = 0;
      return;
    }
#pragma unroll
    for (int q = 0; q < 4; q++) c[q] = (match16(w[2 * q], d) | (match16(w[2 * q + 1], d) << 16)) & S.O[q];
  } else {
#pragma unroll
    for (int q = 0; q < 4; q++) c[q] = S.O[q];
  }
}

// the 16 scores of group g: min and first slot holding it
template <bool C>
__device__ __forceinline__ void tps_group_scan(const TableDev& t, const TpsState& S, int g, uint64_t (&v)[16],
                                               uint64_t& mn, int& ms) {
  if constexpr (C) {
#pragma unroll
    for (int k = 0; k < 16; k++) v[k] = S.Sc[(16 * g + k) * S.cs];
  } else {
    // 16 (key, score) pairs: two 128-B lines
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(kptr(t, S.rowbase + 16 * g));
#pragma unroll
    for (int k = 0; k < 16; k++) v[k] = p[k].y;
  }
  mn = v[0];
  ms = 0;
#pragma unroll
  for (int k = 1; k < 16; k++)
    if (v[k] < mn) { mn = v[k]; ms = k; }
}

__device__ __forceinline__ void tps_load_summary(const TableDev& t, uint64_t b, TpsState& S) {
  if (S.sloaded) return;
  const ulonglong2* p = reinterpret_cast<const ulonglong2*>(t.smin + b * 8);
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const ulonglong2 x = p[k];
    S.sm[2 * k] = x.x;
    S.sm[2 * k + 1] = x.y;
  }
  S.sv = t.svalid[b];
  S.sloaded = true;
}

// a score write of value v at slot s outside an eviction: keep the group
// minimum exact when v becomes the minimum, otherwise mark it unknown
__device__ __forceinline__ void tps_score_written(const TableDev& t, uint64_t b, TpsState& S, int s, uint64_t v) {
  const int g = s >> 4;
  if (S.sloaded) {
    if (((S.sv >> g) & 1u) && v <= sel8(S.sm, g)) {
      put8(S.sm, g, v);
      S.smdirty |= 1u << g;
    } else if ((S.sv >> g) & 1u) {
      S.sv &= ~(1u << g);
      S.svdirty = true;
    }
  } else {
    atomicAnd(t.svalid + b, ~(1u << g));
  }
}

// Last writer of a slot within the current segment (asked only when S.wm
// says an earlier op of the segment wrote it).  Short segments scan back
// through their few positions (retired writers hold kNoRow, so the latest
// writer is the one whose vrow is the row); once a segment passes kLwScan ops
// (configs[0]: ~128 ops per bucket, zipf hot buckets) the thread's table in
// global scratch is filled from those positions and kept current, so long
// segments stay linear.  Nothing is written for the short segments that make
// up uniform batches.
constexpr int kLwScan = 16;
__device__ __forceinline__ int lw_get(const TpsState& S, int slot, int64_t from) {
  if (S.tab) return S.lw[slot * S.lws];
  const uint32_t row = (uint32_t)(S.rowbase + slot);
  for (int64_t p = from; p >= S.p0; p--) {
    const uint32_t j = S.sidx[p];
    if (S.vrow[j] == row) return (int)j;
  }
  return -1;
}
__device__ __forceinline__ void lw_set(const TpsState& S, int slot, uint32_t op) {
  if (S.tab) S.lw[slot * S.lws] = (int)op;
}
// Collapsed stretches of same-key runs hold no writer but their last op, and
// tps_run leaves a jump mark (run_end[q+1] = qe | kJump) at their start, so the
// fill costs the segment's individually applied ops, not its positions (a
// zipf hot bucket holds tens of thousands of positions but ~60 runs).
constexpr uint32_t kJump = 0x80000000u;
__device__ __forceinline__ void lw_fill(TpsState& S, int64_t q, const uint32_t* run_end, bool runs) {
  // (run_end is read through the coherent path: tps_run writes it in this kernel)
  for (int64_t p = S.p0; p < q;) {
    if (runs) {
      const uint32_t m = run_end[p];
      if (m & kJump) {
        p = (int64_t)(m & ~kJump);  // the stretch's last op (its only possible writer)
        continue;
      }
    }
    const uint32_t j = S.sidx[p];
    const uint32_t w = S.vrow[j];
    if (w != kNoRow) S.lw[(int64_t)(w - S.rowbase) * S.lws] = (int)j;
    p++;
  }
  S.tab = true;
}

template <int OP, bool COLLECT, bool C>
__device__ __forceinline__ int tps_op(const TableDev& t, const OpArgs& a, TpsState& S, uint64_t b, uint32_t i,
                                      uint64_t key, uint32_t d, uint64_t clock0, bool fel_open, int64_t q,
                                      uint32_t* __restrict__ vrow, uint32_t* __restrict__ rrow,
                                      int32_t* __restrict__ rsrc, ctr_t* ctr, int& sd, uint32_t& fe_min) {
  const uint64_t rowbase = b * kSlots;
  uint32_t c[4];
  tps_cand(t, S, d, c);
  int hit = -1;
  unsigned ncmp = 0;
  const int npk = (!C && q == S.p0) ? S.npk : 0;  // the head op's first candidates are prefetched
#pragma unroll
  for (int w = 0; w < 4; w++) {
    uint32_t m = hit < 0 ? c[w] : 0u;
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const uint64_t k = (int)ncmp < npk ? (ncmp == 0 ? S.pk[0] : S.pk[1]) : bkey<C>(t, S, 32 * w + j);
      ncmp++;
      if (k == key) {
        hit = 32 * w + j;
        m = 0;
      }
    }
  }
  ctr[kLoads]++;
  ctr[kCompares] += ncmp;
  if constexpr (OP == kOpErase) {  // _round_erase, table.py:1017-1023
    if (hit >= 0) {
      set_bkey<C>(t, S, hit, kEmptyKey);
      const uint32_t o = S.O[hit >> 5] & ~(1u << (hit & 31));
      S.O[hit >> 5] = o;
      set_bocc<C>(t, S, b, hit >> 5, o);
      sd--;
    }
    st_keep(a.outcomes + i, (uint8_t)(hit >= 0 ? kErased : kNotFound), S.pol);
    return -1;
  }
  const uint64_t tick = a.ticks ? a.ticks[i] : clock0 + (uint64_t)i + 1;
  const uint64_t cs = a.scores ? a.scores[i] : 0;
  uint8_t outcome = kRejected;
  int wslot = -1, rslot = -1;
  if (hit >= 0) {  // table.py:1045-1062
    const uint64_t old = hit_needs_old(t.policy) ? bscore<C>(t, S, hit) : 0;
    const uint64_t ns = hit_score(t.policy, old, a.epoch, tick, a.scores != nullptr, cs);
    set_bscore<C>(t, S, hit, ns);
    tps_score_written(t, b, S, hit, ns);
    if constexpr (OP == kOpFindOrInsert) {
      outcome = kFound;
      rslot = hit;
    } else {
      outcome = kUpdated;
      wslot = hit;
    }
  } else {
    const uint64_t s_in = insert_score(t.policy, a.epoch, tick, cs);  // scoring.py:105-127
    const uint4 ow = *reinterpret_cast<const uint4*>(S.O);
    const uint32_t oc[4] = {ow.x, ow.y, ow.z, ow.w};
    const int occ_total = __popc(oc[0]) + __popc(oc[1]) + __popc(oc[2]) + __popc(oc[3]);
    if (occ_total < kSlots) {
      // _bulk_insert_free, table.py:1165-1181: lowest EMPTY slot
      int s = 0;
#pragma unroll
      for (int w = 3; w >= 0; w--)
        if (oc[w] != 0xFFFFFFFFu) s = 32 * w + __ffs(~oc[w]) - 1;
#ifndef HKV_EXP_NOKEY
      set_bkey<C>(t, S, s, key);
#endif
      set_bdigest<C>(t, S, s, d);
#ifndef HKV_EXP_NOSCORE
      set_bscore<C>(t, S, s, s_in);
#endif
      const uint32_t o = S.O[s >> 5] | (1u << (s & 31));
      S.O[s >> 5] = o;
      set_bocc<C>(t, S, b, s >> 5, o);
      reinterpret_cast<uint8_t*>(S.L)[s] = (uint8_t)d;
      // The summary is only consulted while the bucket is full, so a free
      // insert leaves it alone unless it fills the bucket: then every group
      // is marked unknown at once (the next full decision rescans).  This
      // keeps a scattered atomic off ~all inserts below lambda = 1.
      if (occ_total + 1 == kSlots) {
        if (S.sloaded) {
          if (S.sv) {
            S.sv = 0;
            S.svdirty = true;
          }
        } else {
          atomicAnd(t.svalid + b, 0u);
        }
      }
      wslot = s;
      outcome = kInserted;
      sd++;
    } else {
      // full bucket: argmin (table.py:1079-1083) through the group summary
      ctr[kScans]++;
      tps_load_summary(t, b, S);
      uint64_t v[16];
      uint64_t mn;
      int ms;
      uint32_t inv = ~S.sv & 0xFFu;
      while (inv) {
        const int g = __ffs(inv) - 1;
        inv &= inv - 1;
        tps_group_scan<C>(t, S, g, v, mn, ms);
        put8(S.sm, g, mn);
        S.smdirty |= 1u << g;
      }
      if (S.sv != 0xFFu) {
        S.sv = 0xFFu;
        S.svdirty = true;
      }
      int gi = 0;
      uint64_t gmin = S.sm[0];
#pragma unroll
      for (int k = 1; k < 8; k++)
        if (S.sm[k] < gmin) { gmin = S.sm[k]; gi = k; }
      tps_group_scan<C>(t, S, gi, v, mn, ms);  // mn == gmin; ms = first slot holding it
      if (s_in >= gmin) {  // the single-bucket path admits ties (table.py:1083)
        const int m = 16 * gi + ms;
        if constexpr (COLLECT) {
          a.ek[kRecU64 * i] = bkey<C>(t, S, m);
          a.es[kRecU64 * i] = gmin;
        }
        set_bkey<C>(t, S, m, key);
        set_bdigest<C>(t, S, m, d);
        set_bscore<C>(t, S, m, s_in);
        reinterpret_cast<uint8_t*>(S.L)[m] = (uint8_t)d;
        // the group's new minimum, exactly (its 16 scores are in registers)
        uint64_t nm = kMaxScore;
#pragma unroll
        for (int k = 0; k < 16; k++) {
          const uint64_t x = (k == ms) ? s_in : v[k];
          nm = x < nm ? x : nm;
        }
        put8(S.sm, gi, nm);
        S.smdirty |= 1u << gi;
        wslot = m;
        if constexpr (COLLECT) rslot = m;
        outcome = kEvicted;
        if (fel_open) fe_min = i < fe_min ? i : fe_min;
      }
    }
  }
  // value plan (provenance read BEFORE this op's own write is recorded)
  if (rslot >= 0) {
    ctr[rowbase + rslot < t.fast_rows ? kVFast : kVOver]++;
    st_keep(rrow + kRecU32 * i, (uint32_t)(rowbase + rslot), S.pol);
    st_keep(rsrc + kRecU32 * i, bit128(S.wm, rslot) ? lw_get(S, rslot, q - 1) : -1, S.pol);
  }
  if (wslot >= 0) {
    ctr[rowbase + wslot < t.fast_rows ? kVFast : kVOver]++;
    if (bit128(S.wm, wslot)) {  // retired: this op rewrites the slot
      const int prev = lw_get(S, wslot, q - 1);
      if (prev >= 0) st_keep(vrow + prev, kNoRow, S.pol);
    }
    setbit128(S.wm, wslot);
    lw_set(S, wslot, i);
    st_keep(vrow + i, (uint32_t)(rowbase + wslot), S.pol);
  } else {
    st_keep(vrow + i, kNoRow, S.pol);
  }
  st_keep(a.outcomes + i, outcome, S.pol);
  return rslot >= 0 ? rslot : wslot;
}

// A run of consecutive ops on one key inside a bucket segment (sorted
// positions q+1 .. qe, all after the op at q).  Under serial semantics
// every one of them sees the bucket exactly as the
// op at q left it, so the run applies in O(1):
//   key resident at slot `res`  -> cnt hits: Updated / Found, one aggregated
//                                  score refresh, the last op's value wins
//   erase                       -> key absent: NotFound
//   absent, Lfu / EpochLfu      -> same admission score, same bucket: Rejected
// Followers' outcome / vrow were pre-set by k_segments (Updated / Found /
// NotFound, no value row); only the exceptions are written here.  TxnCounters
// are exactly those of cnt individual probes.
template <int OP, bool C>
__device__ __forceinline__ void tps_run(const TableDev& t, const OpArgs& a, TpsState& S, int64_t q, int64_t qe,
                                        int res, uint64_t b, uint32_t d, uint64_t clock0,
                                        const uint32_t* __restrict__ sidx, uint32_t* __restrict__ vrow,
                                        uint32_t* __restrict__ rrow, int32_t* __restrict__ rsrc, ctr_t* ctr) {
  const uint32_t cnt = (uint32_t)(qe - q);
  const uint64_t rowbase = b * kSlots;
  uint32_t c[4];
  tps_cand(t, S, d, c);
  if (res >= 0) {  // compares stop at the match (table.py:243-268)
#pragma unroll
    for (int w = 0; w < 4; w++) {
      if (32 * w > res) c[w] = 0;
      else if (32 * w + 31 > res) c[w] &= (2u << (res & 31)) - 1u;
    }
  }
  ctr[kCompares] += cnt * (uint32_t)(__popc(c[0]) + __popc(c[1]) + __popc(c[2]) + __popc(c[3]));
  ctr[kLoads] += cnt;
  if constexpr (OP == kOpErase) return;
  if (res < 0) {  // rejected run (Lfu / EpochLfu: same score, same bucket)
    ctr[kScans] += cnt;
    for (int64_t p = q + 1; p <= qe; p++) st_keep(a.outcomes + sidx[p], (uint8_t)kRejected, S.pol);
    return;
  }
  const uint64_t row = rowbase + res;
  ctr[row < t.fast_rows ? kVFast : kVOver] += cnt;
  const uint32_t il = sidx[qe];
  const uint64_t tl = a.ticks ? a.ticks[il] : clock0 + (uint64_t)il + 1;
  const uint64_t cs = a.scores ? a.scores[il] : 0;
  const uint64_t ns = run_hit_score(t.policy, bscore<C>(t, S, res), a.epoch, tl, a.scores != nullptr, cs, cnt);
  set_bscore<C>(t, S, res, ns);
  tps_score_written(t, b, S, res, ns);
  if constexpr (OP == kOpUpsert) {
    if (bit128(S.wm, res)) {
      const int prev = lw_get(S, res, q);
      if (prev >= 0) st_keep(vrow + prev, kNoRow, S.pol);
    }
    setbit128(S.wm, res);
    lw_set(S, res, il);
    st_keep(vrow + il, (uint32_t)row, S.pol);
  }
  if constexpr (OP == kOpFindOrInsert) {
    const int src = bit128(S.wm, res) ? lw_get(S, res, q) : -1;
    for (int64_t p = q + 1; p <= qe; p++) {
      const uint32_t j = sidx[p];
      st_keep(rrow + kRecU32 * j, (uint32_t)row, S.pol);
      st_keep(rsrc + kRecU32 * j, src, S.pol);
    }
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
// the occupancy word with L2 evict_last priority: the 16-MB bitmap of a C2
// table then stays in L2 across batches while the digest lines and pairs
// stream through (HKV_OCC_HINT=0: plain)
#ifndef HKV_LINE_HINT
#define HKV_LINE_HINT 0
#endif
#ifndef HKV_OCC_HINT
#define HKV_OCC_HINT 1
#endif
__device__ __forceinline__ void cp_async16_keep(void* smem, const void* gmem) {
#if HKV_OCC_HINT
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "l"(pol) : "memory");
#else
  cp_async16(smem, gmem);
#endif
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

constexpr int kTpsStageU4 = 9;  // per thread and stage: 8 x 16 B digest line + 16 B occupancy (odd stride: no bank conflicts)

// stage buffer of this thread: [stage][thread][9 x uint4]
__device__ __forceinline__ uint4* tps_buf(uint4* smem, int stage) {
  return smem + ((size_t)stage * kTpsThreads + threadIdx.x) * kTpsStageU4;
}
__device__ __forceinline__ void tps_fetch(const TableDev& t, uint4* buf, uint64_t b) {
  const uint4* dp = reinterpret_cast<const uint4*>(t.digests + b * kSlots);
#pragma unroll
#if HKV_LINE_HINT
  for (int k = 0; k < 8; k++) cp_async16_keep(buf + k, dp + k);
#else
  for (int k = 0; k < 8; k++) cp_async16(buf + k, dp + k);
#endif
  cp_async16_keep(buf + 8, reinterpret_cast<const uint4*>(t.bits) + b);
}

template <int OP, bool COLLECT, bool C>
__device__ __forceinline__ void tps_segment(const TableDev& t, const OpArgs& a, const SegRec& rec, uint4* buf,
                                            const uint32_t* __restrict__ sb, const uint32_t* __restrict__ sidx,
                                            uint32_t* run_end, const uint64_t* __restrict__ skeys,
                                            int64_t n, uint32_t* __restrict__ vrow, uint32_t* __restrict__ rrow,
                                            int32_t* __restrict__ rsrc, uint64_t clock0, bool fel_open,
                                            bool spec, bool lfu_like, bool runs, ctr_t* ctr, int& sd,
                                            uint32_t& fe_min, int* lw, int64_t lws, uint64_t* K = nullptr,
                                            uint64_t* Sc = nullptr, int cs = 0, uint64_t pk0 = 0, uint64_t pk1 = 0,
                                            int npk = 0) {
  const uint64_t b = rec.b;
  TpsState S;
  S.pk[0] = pk0;
  S.pk[1] = pk1;
  S.npk = npk;
  S.lw = lw;
  S.lws = lws;
  S.sidx = sidx;
  S.vrow = vrow;
  S.p0 = rec.p;
  S.rowbase = b * kSlots;
  S.tab = C;  // the long-segment engine keeps its last-writer table in shared memory from the start
  S.L = buf;
  S.O = reinterpret_cast<uint32_t*>(buf + 8);
  S.K = K;
  S.Sc = Sc;
  S.cs = cs;
  S.pol = l2_keep_policy();
#pragma unroll
  for (int w = 0; w < 4; w++) S.wm[w] = 0;
  S.sloaded = false;
  S.svdirty = false;
  S.smdirty = 0;
  if (OP != kOpErase && (spec || C)) tps_load_summary(t, b, S);
  const bool multi = (rec.flags & 1u) != 0;
  uint32_t i = rec.i, d = rec.flags >> 8;
  uint64_t key = rec.key;
  int64_t q = rec.p;
  while (true) {
    uint32_t nb_ = kNoRow, ni = 0;
    uint64_t nk = 0;
    int64_t qe = q;
    if (multi && q + 1 < n) {  // next sorted position: independent of this op, in flight during it
      nb_ = sb[q + 1];
      ni = sidx[q + 1];
      nk = skeys[q + 1];
      qe = runs ? (int64_t)run_end[q] : q;
    }
    if (OP != kOpErase && !S.tab && q - S.p0 >= kLwScan) lw_fill(S, q, run_end, runs);  // erase writes no rows
    const int res = tps_op<OP, COLLECT, C>(t, a, S, b, i, key, d, clock0, fel_open, q, vrow, rrow, rsrc,
                                        ctr, sd, fe_min);
    if (nb_ != (uint32_t)b) break;
    if (qe > q && (OP == kOpErase || res >= 0 || lfu_like)) {
      tps_run<OP, C>(t, a, S, q, qe, res, b, d, clock0, sidx, vrow, rrow, rsrc, ctr);
      if (qe > q + 1) run_end[q + 1] = (uint32_t)qe | kJump;  // for lw_fill
      q = qe;
      if (!(q + 1 < n && sb[q + 1] == (uint32_t)b)) break;
      ++q;
      i = sidx[q];
      key = skeys[q];
    } else {
      ++q;
      i = ni;
      key = nk;
    }
    d = digest_of(fmix64(key));
  }
  // write back the summary changes kept in registers
  if (S.smdirty) {
#pragma unroll
    for (int k = 0; k < 8; k++)
      if ((S.smdirty >> k) & 1u) t.smin[b * 8 + k] = S.sm[k];
  }
  if (S.svdirty || S.smdirty) t.svalid[b] = S.sv;
  if constexpr (C) {  // write the bucket back once
    ulonglong2* kd = reinterpret_cast<ulonglong2*>(kptr(t, S.rowbase));
#pragma unroll 8
    for (int j = 0; j < kSlots; j++) kd[j] = make_ulonglong2(S.K[j * cs], S.Sc[j * cs]);
    uint4* dd = reinterpret_cast<uint4*>(t.digests + S.rowbase);
#pragma unroll
    for (int k = 0; k < 8; k++) dd[k] = S.L[k];
    reinterpret_cast<uint4*>(t.bits)[b] = *reinterpret_cast<const uint4*>(S.O);
  }
}

}  // namespace hkv
