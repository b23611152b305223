// hkv_cas.cu — the concurrent upsert engine: the reference's LOCKED-sentinel
// slot CAS protocol (table.py:678-857) with every op
// of a batch in flight at once.  Selected by TableConfig.workers > 1, the
// reference's switch to its threaded CAS engine (table.py:1185-1241); like
// that engine it is serializable but not serial-in-batch-order under
// contention, so tests check the policy invariants.
//
// One THREAD per op (HKV's TLPv1 shape): an op's chain is a
// handful of dependent round trips, so what pays is the number of ops in
// flight and the length of each chain.  Every op first takes its bucket
// lock(s) with non-blocking acquire CASes (dual: both at once), then works
// the bucket(s) exclusively -- the lock is what makes a short chain possible:
//   probe      the 128-B digest line(s) and 16-B occupancy word(s), both
//              buckets' in flight at once, candidate keys in slot order.
//   hit        claim key -> LOCKED, refresh the score, write (or,
//              find_or_insert, read) the value row (_scalar_hit,
//              table.py:749-772).
//   miss       claim the lowest free slot EMPTY -> LOCKED, or take the
//              first-index minimum through the eviction summary (the victim's
//              16-score group read once), admit, claim the victim old ->
//              LOCKED and capture the evicted tuple (table.py:678-693,
//              775-857).
// The round's fence then orders metadata and rows before the key is
// published (key last, _publish_entry table.py:737-747) and the locks drop.
// Readers never run beside this kernel (the triple-group gate), so the
// LOCKED state only guards the publish order.  Compiled with -dlcm=cg:
// metadata another SM just published must not be served from a stale L1
// line.
#include <atomic>

#include "hkv_kernels.h"
#include "hkv_probe.cuh"

namespace hkv {

namespace {

constexpr int kBusy = -2;

__device__ __forceinline__ void fence_rel() {
#ifndef HKV_CAS_NOFENCE
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
}
__device__ __forceinline__ unsigned cas_acquire_u32(unsigned* p, unsigned cmp, unsigned val) {
  unsigned old;
  asm volatile("atom.acquire.gpu.global.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "l"(p), "r"(cmp), "r"(val) : "memory");
  return old;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_key(const TableDev& t, uint64_t row) {
#ifdef HKV_CAS_KEYLDCG
  return __ldcg(kptr(t, row));
#else
  return *(volatile const uint64_t*)kptr(t, row);
#endif
}

// Bucket locks: 0 free, 1 held; taken by a non-blocking acquire CAS, dropped
// by a relaxed store after the round's fence.
__device__ __forceinline__ void st_relaxed_u32(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// The slot claim of the reference's protocol (table.py:678-693, 775-857):
// key `expect` -> LOCKED.  Every structural change and every hit holds the
// slot's bucket lock, so the claim cannot lose and its result is not waited
// on; the entry is published (key last) after the round's fence.
__device__ __forceinline__ void claim_slot(const TableDev& t, uint64_t row, uint64_t expect) {
  atomicCAS((unsigned long long*)kptr(t, row), (unsigned long long)expect, (unsigned long long)kLockedKey);
}

// A bucket's probe state: digest-candidate mask (digest equal, slot occupied)
// and the occupancy words it was built from.
struct Cand {
  uint32_t c[4];
  uint4 occ;
};
__device__ __forceinline__ Cand load_cand(const TableDev& t, uint64_t b, uint32_t d) {
  Cand r;
  const uint4* dp = reinterpret_cast<const uint4*>(t.digests + b * kSlots);
  r.occ = __ldcg(reinterpret_cast<const uint4*>(t.bits + b * 4));
  const uint32_t occ[4] = {r.occ.x, r.occ.y, r.occ.z, r.occ.w};
  uint4 w[8];
#pragma unroll
  for (int k = 0; k < 8; k++) w[k] = __ldcg(dp + k);
#pragma unroll
  for (int q = 0; q < 4; q++)
    r.c[q] = (t.digest_filter ? (match16(w[2 * q], d) | (match16(w[2 * q + 1], d) << 16)) : ~0u) & occ[q];
  return r;
}

// Lock-free probe of bucket b by one thread: slot of `key`, -1 (absent), or
// kBusy (a digest candidate is LOCKED: an op holds it mid-update).  Compares
// counted as table.py:243-268 (candidates in slot order, up to the match).
__device__ __forceinline__ int probe_cand(const TableDev& t, uint64_t b, const Cand& cd, uint64_t key, ctr_t& ncmp) {
  const uint32_t* c = cd.c;
  bool busy = false;
#pragma unroll
  for (int q = 0; q < 4; q++) {
    uint32_t m = c[q];
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      const uint64_t k = ld_key(t, b * kSlots + 32 * q + j);
      if (k == kLockedKey) {
        busy = true;
        continue;
      }
      if (k == kEmptyKey) continue;
      ncmp++;
      if (k == key) return 32 * q + j;
    }
  }
  return busy ? kBusy : -1;
}

// An op's probe: both buckets' lines in flight at once; dual mode consults
// (and counts) b2 only when b1 misses (_vec_lookup, table.py:284-300).
// o1 / o2: the occupancy words the probe saw.
__device__ __forceinline__ int probe_op(const TableDev& t, uint64_t b1, uint64_t b2, uint64_t key, uint32_t d,
                                        ctr_t* ctr, uint64_t& hb, uint4& o1, uint4& o2) {
  const Cand c1 = load_cand(t, b1, d);
  Cand c2 = c1;
  if (t.dual) c2 = load_cand(t, b2, d);
  o1 = c1.occ;
  o2 = c2.occ;
  hb = b1;
  int slot = probe_cand(t, b1, c1, key, ctr[kCompares]);
  ctr[kLoads]++;
  if (slot == -1 && t.dual) {
    hb = b2;
    slot = probe_cand(t, b2, c2, key, ctr[kCompares]);
    ctr[kLoads]++;
  }
  return slot;
}

// A full bucket's minimum through the eviction summary, by one thread that
// holds the bucket's lock (every score write of this engine does): exact
// groups come from the 64-B summary line, the others are rescanned (16
// scores each) and made exact.  gmin = the bucket's minimum, gi = the lowest
// group holding it (groups are in slot order, so the group's first slot
// holding gmin is np.argmin's first index, table.py:1080).
struct Summ {
  ulonglong2 m[4];  // the 8 group minima
  uint32_t sv;      // group valid bits
};
__device__ __forceinline__ Summ load_summ(const TableDev& t, uint64_t b) {
  Summ s;
  const ulonglong2* p = reinterpret_cast<const ulonglong2*>(t.smin + b * 8);
#pragma unroll
  for (int k = 0; k < 4; k++) s.m[k] = __ldcg(p + k);
  s.sv = __ldcg(t.svalid + b);
  return s;
}
__device__ __forceinline__ void summ_min(const TableDev& t, uint64_t b, const Summ& s, uint64_t& gmin, int& gi) {
  const uint32_t inv = ~s.sv & 0xFFu;
  uint64_t sm[8];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    sm[2 * k] = s.m[k].x;
    sm[2 * k + 1] = s.m[k].y;
  }
  if (inv) {
#pragma unroll
    for (int g = 0; g < 8; g++) {
      if ((inv >> g) & 1u) {
        const ulonglong2* gp = reinterpret_cast<const ulonglong2*>(kptr(t, b * kSlots + 16 * g));
        uint64_t mn = kMaxScore;
#pragma unroll
        for (int k = 0; k < 16; k++) {
          const uint64_t x = __ldcg(gp + k).y;
          mn = x < mn ? x : mn;
        }
        sm[g] = mn;
        t.smin[b * 8 + g] = mn;
      }
    }
    t.svalid[b] = s.sv | inv;
  }
  gmin = sm[0];
  gi = 0;
#pragma unroll
  for (int k = 1; k < 8; k++)
    if (sm[k] < gmin) { gmin = sm[k]; gi = k; }
}

// ---------------------------------------------------------------------------
// Warp-synchronous rounds.  A warp owns 32 ops (one per lane).  Each round,
// every unfinished op makes one NON-BLOCKING attempt: try its bucket lock(s);
// holding them, probe, and claim the hit slot, the lowest free slot or (after
// the full-bucket decision through the eviction summary) the victim, writing
// the slot's metadata.  Then the warp moves every claimed op's value row with
// coalesced copies, fences, publishes the keys and drops the locks.  An op
// that met a held lock or an unpublished (LOCKED) candidate tries again next
// round; locks are only ever kept across rounds in bucket order (the lower
// one while the higher one is busy), so the rounds cannot deadlock.
// ---------------------------------------------------------------------------
enum : int { kTaskNone = 0, kTaskHit = 1, kTaskRead = 2, kTaskInsert = 3, kTaskEvict = 4 };
constexpr unsigned kFullMask = 0xFFFFFFFFu;

// the warp copies the rows of every lane in `mask`: dst/src per lane
template <int VEC>
__device__ __forceinline__ void warp_copy_rows(unsigned mask, float* dst, const float* src, int dim, int lane) {
  using V = typename std::conditional<VEC == 4, uint4, typename std::conditional<VEC == 2, float2, float>::type>::type;
  const int nv = dim / VEC;
  if (nv <= 16) {
    // two rows per step, a half warp each
    const int half = lane >> 4, hl = lane & 15;
    while (mask) {
      const int l0 = __ffs(mask) - 1;
      mask &= mask - 1;
      int l1 = -1;
      if (mask) {
        l1 = __ffs(mask) - 1;
        mask &= mask - 1;
      }
      const int src_l = half ? l1 : l0;
      float* d = (float*)__shfl_sync(kFullMask, (unsigned long long)dst, src_l < 0 ? l0 : src_l);
      const float* sp = (const float*)__shfl_sync(kFullMask, (unsigned long long)src, src_l < 0 ? l0 : src_l);
      if (src_l >= 0 && hl < nv) reinterpret_cast<V*>(d)[hl] = reinterpret_cast<const V*>(sp)[hl];
    }
  } else {
    while (mask) {
      const int l = __ffs(mask) - 1;
      mask &= mask - 1;
      float* d = (float*)__shfl_sync(kFullMask, (unsigned long long)dst, l);
      const float* sp = (const float*)__shfl_sync(kFullMask, (unsigned long long)src, l);
      copy_row<32, VEC, 2>(d, sp, dim, lane);
    }
  }
}

#ifndef HKV_CAS_EARLY_UNLOCK
#define HKV_CAS_EARLY_UNLOCK 0  // measured: fewer retries, but the extra fence costs more
#endif
#ifndef HKV_DUAL_REFILL
#define HKV_DUAL_REFILL 0  // measured: 0.56 -> 0.54 ms at lambda 0.5, 0.84 -> 0.87 ms at lambda 1
#endif
#ifndef HKV_CAS_SPEC
#define HKV_CAS_SPEC 0
#endif
#ifndef HKV_CAS_STAGE
#define HKV_CAS_STAGE 1
#endif
#ifndef HKV_CAS_MINB
#define HKV_CAS_MINB 2
#endif
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

// stage_dim > 0: each warp stages its 32 ops' input rows (contiguous in the
// batch) into shared memory with cp.async when it takes the chunk, so the
// row writes of the rounds are stores only (no dependent global load)
template <int VEC>
__global__ void __launch_bounds__(256, HKV_CAS_MINB) k_cas_upsert(TableDev t, OpArgs a, unsigned* locks, int64_t n,
                                                                  int stage_dim) {
  extern __shared__ uint4 cas_rows[];
  if (a.sc->err) return;
  const int lane = threadIdx.x & 31;
  const uint64_t clock0 = *t.clock;
  const bool fel_open = !*t.fel_set;
  const int dim = t.dim;
  // at lambda > 0.97 a full bucket is the rule (as the metadata pass's spec)
  const bool spec = HKV_CAS_SPEC && (unsigned long long)*t.size * 100ull > t.capacity * 97ull;
  ctr_t ctr[6] = {0, 0, 0, 0, 0, 0};
  int sd = 0;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t base = ((int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32) * 32; base < n;
       base += nwarps * 32) {
    const int64_t i = base + lane;
    bool done = i >= n;
    uint64_t key = 0, b1 = 0, b2 = 0, tick = 0, cs = 0;
    uint32_t d = 0;
    if (!done) {
      key = a.keys[i];
      const uint64_t h = fmix64(key);
      d = digest_of(h);
      b1 = h & t.mask;
      b2 = t.dual ? second_hash(h) & t.mask : b1;
      tick = a.ticks ? a.ticks[i] : clock0 + (uint64_t)i + 1;
      cs = a.scores ? a.scores[i] : 0;
    }
    const uint64_t lo = b1 < b2 ? b1 : b2, hi = b1 < b2 ? b2 : b1;
    float* vin = done ? nullptr : a.values + (uint64_t)i * dim;
    const float* vsrc = vin;  // the row this op writes from
    if (stage_dim) {
      uint4* wrows = cas_rows + (size_t)(threadIdx.x / 32) * 32 * (stage_dim / 4);
      const int64_t cnt = n - base < 32 ? n - base : 32;
      const uint4* g = reinterpret_cast<const uint4*>(a.values + (uint64_t)base * dim);
      __syncwarp();  // the previous chunk's rows are consumed
      for (int k = lane; k < (int)cnt * (dim / 4); k += 32) cp_async16(wrows + k, g + k);
      asm volatile("cp.async.commit_group;" ::: "memory");
      vsrc = reinterpret_cast<const float*>(wrows + lane * (dim / 4));
    }
    bool staged = stage_dim == 0;
    bool have_lo = false;    // the lower bucket's lock, kept while the higher one is busy
    bool contended = false;  // lost the lower bucket once: lock in order from now on
    uint8_t outcome = kRejected;
    unsigned idle_rounds = 0;
    while (__any_sync(kFullMask, !done)) {
      int task = kTaskNone;
      bool locked = false, retry = false;
      uint64_t row = 0;
      if (!done) {
        // try the bucket lock(s).  Locks are taken in bucket order: an op
        // may keep its lower bucket across rounds while it waits for the
        // higher one, never the reverse, so holders form no cycle.  The first
        // attempt issues both CASes at once; after a lost lower bucket the op
        // touches its higher bucket only once the lower one is its own, so a
        // hot pair's higher lock is left to the lower lock's holder.  Nothing
        // waits inside a round.
        unsigned glo = 0u, ghi = 0u;
        if (!have_lo) {
          glo = cas_acquire_u32(locks + lo, 0u, 1u);
          if (hi != lo && (!contended || !glo)) ghi = cas_acquire_u32(locks + hi, 0u, 1u);
        } else {
          ghi = cas_acquire_u32(locks + hi, 0u, 1u);
        }
        if (glo) {
          if (hi != lo && !contended && !ghi) st_relaxed_u32(locks + hi, 0u);
          contended = true;
          retry = true;
        } else if (ghi) {
          have_lo = true;
          retry = true;
        } else {
          locked = true;
          uint64_t hb = b1;
          uint4 w1, w2;
          // when full buckets are the rule, the summaries travel with the probe
          Summ s1, s2;
          if (spec) {
            s1 = load_summ(t, b1);
            if (t.dual) s2 = load_summ(t, b2);
          }
          int slot = probe_op(t, b1, b2, key, d, ctr, hb, w1, w2);
          if (slot == kBusy) {
            retry = true;  // a previous holder's entry is not published yet
          } else if (slot >= 0) {
            // hit (table.py:749-772): hold the slot, refresh the score
            row = hb * kSlots + slot;
            claim_slot(t, row, key);
            const uint64_t old = hit_needs_old(t.policy) ? __ldcg(sptr(t, row)) : 0;
            *sptr(t, row) = hit_score(t.policy, old, a.epoch, tick, a.scores != nullptr, cs);
            atomicAnd(t.svalid + hb, ~(1u << (slot >> 4)));  // the group's minimum may have moved
            task = a.op == kOpFindOrInsert ? kTaskRead : kTaskHit;
          } else {
            const uint64_t s_in = insert_score(t.policy, a.epoch, tick, cs);
            const int o1 = __popc(w1.x) + __popc(w1.y) + __popc(w1.z) + __popc(w1.w);
            const int o2 = t.dual ? __popc(w2.x) + __popc(w2.y) + __popc(w2.z) + __popc(w2.w) : kSlots;
            if (o1 < kSlots || o2 < kSlots) {
              // free insert (table.py:678-693, 1165-1181): single -> b1, dual D1
              const bool first = !t.dual || o1 <= o2;
              const uint64_t tb = first ? b1 : b2;
              const uint4 w = first ? w1 : w2;
              const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
              int q = 0;
              while (ws[q] == 0xFFFFFFFFu) q++;
              slot = 32 * q + __ffs(~ws[q]) - 1;  // the lowest EMPTY slot
              row = tb * kSlots + slot;
              claim_slot(t, row, kEmptyKey);
              t.bits[tb * 4 + q] = ws[q] | (1u << (slot & 31));
              t.digests[row] = (uint8_t)d;
              *sptr(t, row) = s_in;
              // the summary is consulted only while the bucket is full: the
              // insert that fills it marks every group unknown
              if ((first ? o1 : o2) + 1 == kSlots) t.svalid[tb] = 0u;
              task = kTaskInsert;
            } else {
              // full bucket(s): first-index minimum through the eviction
              // summary (table.py:1079-1083; dual D2, table.py:1099-1104)
              if (!spec) {
                s1 = load_summ(t, b1);
                if (t.dual) s2 = load_summ(t, b2);
              }
              uint64_t minv, tb = b1;
              int gi;
              summ_min(t, b1, s1, minv, gi);
              ctr[kScans]++;
              if (t.dual) {
                uint64_t n2;
                int g2;
                summ_min(t, b2, s2, n2, g2);
                ctr[kScans]++;
                if (n2 < minv) {  // the bucket with the lower minimum
                  minv = n2;
                  gi = g2;
                  tb = b2;
                }
              }
              const bool admit = t.dual ? (t.admit_unified ? s_in >= minv : s_in > minv) : s_in >= minv;
              if (!admit) {
                outcome = kRejected;
                done = true;
              } else {
                // the victim's group: its 16 scores give the first slot holding
                // the minimum and, after the replacement, the group's new minimum
                const ulonglong2* gp = reinterpret_cast<const ulonglong2*>(kptr(t, tb * kSlots + 16 * gi));
                uint64_t v[16];
#pragma unroll
                for (int k = 0; k < 16; k++) v[k] = __ldcg(gp + k).y;
                uint64_t mn = v[0];
                int ms = 0;
#pragma unroll
                for (int k = 1; k < 16; k++)
                  if (v[k] < mn) { mn = v[k]; ms = k; }
                row = tb * kSlots + 16 * gi + ms;
                const uint64_t victim = mn == minv ? ld_key(t, row) : kLockedKey;
                if (victim == kLockedKey) {
                  // (defensive: under the lock the summary is exact) or the
                  // minimum slot's previous holder has not published it yet
                  t.smin[tb * 8 + gi] = mn;
                  retry = true;
                } else {
                  claim_slot(t, row, victim);
                  if (a.collect) {
                    a.ek[kRecU64 * i] = victim;
                    a.es[kRecU64 * i] = minv;
                  }
                  t.digests[row] = (uint8_t)d;
                  *sptr(t, row) = s_in;
                  uint64_t nm = s_in;
#pragma unroll
                  for (int k = 0; k < 16; k++)
                    if (k != ms && v[k] < nm) nm = v[k];
                  t.smin[tb * 8 + gi] = nm;  // the group stays exact
                  task = kTaskEvict;
                }
              }
            }
          }
        }
      }
#if HKV_CAS_EARLY_UNLOCK
      // structure settled: the locks drop before the row copies (the claimed
      // slot stays LOCKED until its key is published after the round fence)
      if (locked) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        st_relaxed_u32(locks + lo, 0u);
        if (hi != lo) st_relaxed_u32(locks + hi, 0u);
        have_lo = false;
        locked = false;
      }
#endif
      if (retry) ctr[kRetries]++;
      // ---- warp-cooperative value movement ----
      float* vr = task != kTaskNone ? value_row(t, row) : nullptr;
      const unsigned cap_mask = __ballot_sync(kFullMask, task == kTaskEvict && a.collect);
      if (cap_mask) warp_copy_rows<VEC>(cap_mask, a.collect && task == kTaskEvict ? a.ev + (uint64_t)i * dim : nullptr,
                                        vr, dim, lane);
      const unsigned rd_mask = __ballot_sync(kFullMask, task == kTaskRead);
      if (rd_mask) warp_copy_rows<VEC>(rd_mask, vin, vr, dim, lane);
      const unsigned wr_mask = __ballot_sync(kFullMask, task == kTaskHit || task == kTaskInsert || task == kTaskEvict);
      if (wr_mask) {
        if (!staged) {
          asm volatile("cp.async.wait_all;" ::: "memory");
          __syncwarp();
          staged = true;
        }
        warp_copy_rows<VEC>(wr_mask, vr, vsrc, dim, lane);
      }
      if (task != kTaskNone) {
        ctr[row < t.fast_rows ? kVFast : kVOver] += (task == kTaskEvict && a.collect) ? 2 : 1;
        if (task == kTaskInsert) sd++;
        if (task == kTaskEvict && fel_open) atomicMin(&a.sc->first_ev, (unsigned)i);
        outcome = task == kTaskHit ? kUpdated : task == kTaskRead ? kFound : task == kTaskInsert ? kInserted : kEvicted;
        done = true;
      }
      // metadata and rows (every lane's stores) before the keys and the unlocks
      __syncwarp();
      fence_rel();
      __syncwarp();
      if (task != kTaskNone) st_relaxed_u64(kptr(t, row), key);  // publish: the key last (table.py:742-747)
      if (locked) {
        st_relaxed_u32(locks + lo, 0u);
        if (hi != lo) st_relaxed_u32(locks + hi, 0u);
        have_lo = false;
      }
      if (!__any_sync(kFullMask, task != kTaskNone) && !__all_sync(kFullMask, done)) {
        if (++idle_rounds > 2) __nanosleep(64);
      } else {
        idle_rounds = 0;
      }
    }
    if (i < n) a.outcomes[i] = outcome;
  }
  flush_counters<256>(t.counters, ctr, 6);
  long long v = sd;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(t.size, (unsigned long long)v);
}


// ---------------------------------------------------------------------------
// Deterministic dual mode in warp-synchronous rounds (workers == 1): serial
// batch-order semantics.  Every op has its rank in the
// batch-ordered op list of each of its buckets (run_dual's prep); a bucket's
// turn counter says how many of its ops are done.  Each round an op whose
// buckets' turns have reached its ranks runs -- exclusively: no other op of
// those buckets can be ready -- with the same thread-per-op chain as the
// concurrent engine (both probe lines in flight, D1 / D2 through the
// eviction summary), the warp writes the rows, fences and advances the
// turns.  Ops are taken in batch order in 32-op chunks, so the lowest
// pending op is always in some warp's current chunk and ready: progress.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64v(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int VEC>
__global__ void __launch_bounds__(256, HKV_CAS_MINB) k_dual_rounds(TableDev t, OpArgs a,
                                                                   const uint32_t* __restrict__ rank,
                                                                   unsigned long long* turn, unsigned long long tag,
                                                                   int64_t n, int stage_dim) {
  extern __shared__ uint4 cas_rows[];
  if (a.sc->err) return;
  const int lane = threadIdx.x & 31;
  const uint64_t clock0 = *t.clock;
  const bool fel_open = !*t.fel_set;
  const int dim = t.dim;
  const bool erase = a.op == kOpErase;
  ctr_t ctr[6] = {0, 0, 0, 0, 0, 0};
  int sd = 0;
  unsigned* next = &a.sc->npend[0];
#if HKV_DUAL_REFILL
  // lanes refill: a finished op's lane takes the next op at once (ops are
  // handed out in batch order, so the lowest pending op is always held by
  // some lane and ready: progress)
  const unsigned lt_mask = (1u << lane) - 1u;
  uint4* wrow = stage_dim && !erase ? cas_rows + ((size_t)(threadIdx.x / 32) * 32 + lane) * (stage_dim / 4) : nullptr;
  int64_t i = -1;
  bool done = true, ready = false, exhausted = false;
  uint64_t key = 0, b1 = 0, b2 = 0, tick = 0, cs = 0;
  uint32_t d = 0, r1 = 0, r2 = 0;
  float* vin = nullptr;
  const float* vsrc = nullptr;
  unsigned idle_rounds = 0;
  for (;;) {
    const unsigned freem = __ballot_sync(kFullMask, done);
    if (freem && !exhausted) {
      int64_t base = 0;
      if (lane == 0) base = (int64_t)atomicAdd(next, (unsigned)__popc(freem));
      base = __shfl_sync(kFullMask, base, 0);
      if (base + __popc(freem) >= n) exhausted = true;
      if (done) {
        const int64_t j = base + __popc(freem & lt_mask);
        if (j < n) {
          i = j;
          done = false;
          ready = false;
          key = a.keys[i];
          const uint64_t h = fmix64(key);
          d = digest_of(h);
          b1 = h & t.mask;
          b2 = second_hash(h) & t.mask;
          r1 = rank[2 * i];
          r2 = b2 == b1 ? 0u : rank[2 * i + 1];
          tick = a.ticks ? a.ticks[i] : clock0 + (uint64_t)i + 1;
          cs = a.scores ? a.scores[i] : 0;
          vin = erase ? nullptr : a.values + (uint64_t)i * dim;
          vsrc = vin;
          if (wrow) {  // this op's input row into the lane's staging slot
            const uint4* g = reinterpret_cast<const uint4*>(vin);
            for (int k = 0; k < dim / 4; k++) cp_async16(wrow + k, g + k);
            asm volatile("cp.async.commit_group;" ::: "memory");
            vsrc = reinterpret_cast<const float*>(wrow);
          }
        }
      }
    }
    if (!__any_sync(kFullMask, !done)) break;
    {
#else
  for (;;) {
    int64_t base = 0;
    if (lane == 0) base = (int64_t)atomicAdd(next, 32u);
    base = __shfl_sync(kFullMask, base, 0);
    if (base >= n) break;
    const int64_t i = base + lane;
    bool done = i >= n, ready = false;
    uint64_t key = 0, b1 = 0, b2 = 0, tick = 0, cs = 0;
    uint32_t d = 0, r1 = 0, r2 = 0;
    if (!done) {
      key = a.keys[i];
      const uint64_t h = fmix64(key);
      d = digest_of(h);
      b1 = h & t.mask;
      b2 = second_hash(h) & t.mask;
      r1 = rank[2 * i];
      r2 = b2 == b1 ? 0u : rank[2 * i + 1];
      tick = a.ticks ? a.ticks[i] : clock0 + (uint64_t)i + 1;
      cs = a.scores ? a.scores[i] : 0;
    }
    float* vin = done || erase ? nullptr : a.values + (uint64_t)i * dim;
    const float* vsrc = vin;
    if (stage_dim && !erase) {
      uint4* wrows = cas_rows + (size_t)(threadIdx.x / 32) * 32 * (stage_dim / 4);
      const int64_t cnt = n - base < 32 ? n - base : 32;
      const uint4* g = reinterpret_cast<const uint4*>(a.values + (uint64_t)base * dim);
      __syncwarp();  // the previous chunk's rows are consumed
      for (int k = lane; k < (int)cnt * (dim / 4); k += 32) cp_async16(wrows + k, g + k);
      asm volatile("cp.async.commit_group;" ::: "memory");
      vsrc = reinterpret_cast<const float*>(wrows + lane * (dim / 4));
    }
    unsigned idle_rounds = 0;
    while (__any_sync(kFullMask, !done)) {
#endif
      int task = kTaskNone;
      bool ran = false;
      uint64_t row = 0;
      uint8_t outcome = kRejected;
      if (!done && !ready) {
        // the turn loads acquire: the bucket state they follow was fenced
        // before the previous op of the bucket advanced them
        const bool ok1 = r1 == 0 || ld_acquire_u64(turn + b1) >= (tag | r1);
        const bool ok2 = b2 == b1 || r2 == 0 || ld_acquire_u64(turn + b2) >= (tag | r2);
        ready = ok1 && ok2;
      }
      if (!done && ready) {
        ran = true;
        uint64_t hb = b1;
        uint4 w1, w2;
        int slot = probe_op(t, b1, b2, key, d, ctr, hb, w1, w2);
        if (erase) {
          // _round_erase, table.py:1017-1023: key -> EMPTY; digest/score/value stay stale
          if (slot >= 0) {
            row = hb * kSlots + slot;
            *kptr(t, row) = kEmptyKey;
            const uint4 w = hb == b1 ? w1 : w2;
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
            t.bits[hb * 4 + (slot >> 5)] = ws[slot >> 5] & ~(1u << (slot & 31));
            sd--;
            outcome = kErased;
          } else {
            outcome = kNotFound;
          }
        } else if (slot >= 0) {
          // hit: table.py:1045-1062
          row = hb * kSlots + slot;
          const uint64_t old = hit_needs_old(t.policy) ? __ldcg(sptr(t, row)) : 0;
          *sptr(t, row) = hit_score(t.policy, old, a.epoch, tick, a.scores != nullptr, cs);
          atomicAnd(t.svalid + hb, ~(1u << (slot >> 4)));
          task = a.op == kOpFindOrInsert ? kTaskRead : kTaskHit;
        } else {
          const uint64_t s_in = insert_score(t.policy, a.epoch, tick, cs);
          const int o1 = __popc(w1.x) + __popc(w1.y) + __popc(w1.z) + __popc(w1.w);
          const int o2 = __popc(w2.x) + __popc(w2.y) + __popc(w2.z) + __popc(w2.w);
          if (o1 < kSlots || o2 < kSlots) {
            // D1 (table.py:1089-1095): the less occupied bucket, b1 on ties;
            // its lowest EMPTY slot (table.py:1171)
            const bool first = o1 <= o2;
            const uint64_t tb = first ? b1 : b2;
            const uint4 w = first ? w1 : w2;
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
            int q = 0;
            while (ws[q] == 0xFFFFFFFFu) q++;
            slot = 32 * q + __ffs(~ws[q]) - 1;
            row = tb * kSlots + slot;
            *kptr(t, row) = key;
            t.bits[tb * 4 + q] = ws[q] | (1u << (slot & 31));
            t.digests[row] = (uint8_t)d;
            *sptr(t, row) = s_in;
            if ((first ? o1 : o2) + 1 == kSlots) t.svalid[tb] = 0u;
            sd++;
            task = kTaskInsert;
          } else {
            // D2 (table.py:1096-1119): the bucket with the lower minimum
            const Summ s1 = load_summ(t, b1), s2 = load_summ(t, b2);
            uint64_t minv, n2, tb = b1;
            int gi, g2;
            summ_min(t, b1, s1, minv, gi);
            summ_min(t, b2, s2, n2, g2);
            ctr[kScans] += 2;
            if (n2 < minv) {
              minv = n2;
              gi = g2;
              tb = b2;
            }
            const bool admit = t.admit_unified ? s_in >= minv : s_in > minv;
            if (admit) {
              const ulonglong2* gp = reinterpret_cast<const ulonglong2*>(kptr(t, tb * kSlots + 16 * gi));
              uint64_t v[16];
#pragma unroll
              for (int k = 0; k < 16; k++) v[k] = __ldcg(gp + k).y;
              uint64_t mn = v[0];
              int ms = 0;
#pragma unroll
              for (int k = 1; k < 16; k++)
                if (v[k] < mn) { mn = v[k]; ms = k; }
              row = tb * kSlots + 16 * gi + ms;
              if (a.collect) {
                a.ek[kRecU64 * i] = __ldcg(kptr(t, row));
                a.es[kRecU64 * i] = minv;
              }
              *kptr(t, row) = key;
              t.digests[row] = (uint8_t)d;
              *sptr(t, row) = s_in;
              uint64_t nm = s_in;
#pragma unroll
              for (int k = 0; k < 16; k++)
                if (k != ms && v[k] < nm) nm = v[k];
              t.smin[tb * 8 + gi] = nm;  // the group stays exact
              task = kTaskEvict;
            }
          }
        }
      }
      // ---- warp-cooperative value movement (rows of this round's ops) ----
      float* vr = task != kTaskNone ? value_row(t, row) : nullptr;
      const unsigned cap_mask = __ballot_sync(kFullMask, task == kTaskEvict && a.collect);
      if (cap_mask) warp_copy_rows<VEC>(cap_mask, a.collect && task == kTaskEvict ? a.ev + (uint64_t)i * dim : nullptr,
                                        vr, dim, lane);
      const unsigned rd_mask = __ballot_sync(kFullMask, task == kTaskRead);
      if (rd_mask) warp_copy_rows<VEC>(rd_mask, vin, vr, dim, lane);
      const unsigned wr_mask = __ballot_sync(kFullMask, task == kTaskHit || task == kTaskInsert || task == kTaskEvict);
      if (wr_mask) {
        if (stage_dim) {
          asm volatile("cp.async.wait_all;" ::: "memory");
          __syncwarp();
        }
        warp_copy_rows<VEC>(wr_mask, vr, vsrc, dim, lane);
      }
      if (task != kTaskNone) {
        ctr[row < t.fast_rows ? kVFast : kVOver] += (task == kTaskEvict && a.collect) ? 2 : 1;
        if (task == kTaskEvict && fel_open) atomicMin(&a.sc->first_ev, (unsigned)i);
        outcome = task == kTaskHit ? kUpdated : task == kTaskRead ? kFound : task == kTaskInsert ? kInserted : kEvicted;
      }
      // metadata and rows (every lane's stores) before the turns advance
      const bool any_ran = __any_sync(kFullMask, ran);
      if (any_ran) {
        __syncwarp();
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        __syncwarp();
      }
      if (ran) {
        a.outcomes[i] = outcome;
        st_relaxed_u64v(turn + b1, tag | (r1 + 1));
        if (b2 != b1) st_relaxed_u64v(turn + b2, tag | (r2 + 1));
        done = true;
#if HKV_DUAL_REFILL
        i = -1;
#endif
      }
      if (!any_ran && !__all_sync(kFullMask, done)) {
        if (++idle_rounds > 2) __nanosleep(64);
      } else {
        idle_rounds = 0;
      }
    }
  }
  flush_counters<256>(t.counters, ctr, 6);
  long long v = sd;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(t.size, (unsigned long long)v);
}

unsigned long long dev_bit() {
  int dev = 0;
  cudaGetDevice(&dev);
  return 1ull << (dev & 63);
}

}  // namespace

cudaError_t run_cas(const TableDev& t, OpArgs a, int64_t n, unsigned* locks, int vec, cudaStream_t s,
                    int num_sms) {
  void* fn = vec == 4 ? (void*)k_cas_upsert<4> : vec == 2 ? (void*)k_cas_upsert<2> : (void*)k_cas_upsert<1>;
  // input-row staging: 8 warps x 32 rows per block, up to 64 KB (dim <= 64)
  const int stage_dim = (vec == 4 && t.dim <= 64 && HKV_CAS_STAGE) ? t.dim : 0;
  const size_t smem = (size_t)8 * 32 * stage_dim * 4;
  static std::atomic<unsigned long long> attr_set{0};  // the opt-in is per device
  if (smem && !(attr_set.load() & dev_bit())) {
    for (void* f : {(void*)k_cas_upsert<4>, (void*)k_cas_upsert<2>, (void*)k_cas_upsert<1>})
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 32 * 64 * 4);
    attr_set.fetch_or(dev_bit());
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem);
  if (e) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)per_sm * num_sms;
  const int64_t want = (n + 255) / 256;
  if (blocks > want) blocks = want < 1 ? 1 : want;
  if (vec == 4) k_cas_upsert<4><<<(unsigned)blocks, 256, smem, s>>>(t, a, locks, n, stage_dim);
  else if (vec == 2) k_cas_upsert<2><<<(unsigned)blocks, 256, smem, s>>>(t, a, locks, n, stage_dim);
  else k_cas_upsert<1><<<(unsigned)blocks, 256, smem, s>>>(t, a, locks, n, stage_dim);
  g_launches++;
  return cudaGetLastError();
}

}  // namespace hkv

namespace hkv {
cudaError_t run_dual_rounds(const TableDev& t, OpArgs a, int64_t n, const uint32_t* rank, unsigned long long* turn,
                            unsigned long long tag, int vec, cudaStream_t s, int num_sms) {
  void* fn = vec == 4 ? (void*)k_dual_rounds<4> : vec == 2 ? (void*)k_dual_rounds<2> : (void*)k_dual_rounds<1>;
  const int stage_dim = (vec == 4 && t.dim <= 64 && HKV_CAS_STAGE && a.op != kOpErase) ? t.dim : 0;
  const size_t smem = (size_t)8 * 32 * stage_dim * 4;
  static std::atomic<unsigned long long> attr_set{0};  // the opt-in is per device
  if (!(attr_set.load() & dev_bit())) {
    for (void* f : {(void*)k_dual_rounds<4>, (void*)k_dual_rounds<2>, (void*)k_dual_rounds<1>})
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 32 * 64 * 4);
    attr_set.fetch_or(dev_bit());
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem);
  if (e) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)per_sm * num_sms;
  const int64_t want = (n + 255) / 256;
  if (blocks > want) blocks = want < 1 ? 1 : want;
  if (vec == 4) k_dual_rounds<4><<<(unsigned)blocks, 256, smem, s>>>(t, a, rank, turn, tag, n, stage_dim);
  else if (vec == 2) k_dual_rounds<2><<<(unsigned)blocks, 256, smem, s>>>(t, a, rank, turn, tag, n, stage_dim);
  else k_dual_rounds<1><<<(unsigned)blocks, 256, smem, s>>>(t, a, rank, turn, tag, n, stage_dim);
  g_launches++;
  return cudaGetLastError();
}
}  // namespace hkv
