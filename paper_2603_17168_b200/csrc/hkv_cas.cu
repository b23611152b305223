// hkv_cas.cu — the concurrent upsert engine: the reference's LOCKED-sentinel
// slot CAS protocol (table.py:678-857) with every op
// of a batch in flight at once.  Selected by TableConfig.workers > 1, the
// reference's switch to its threaded CAS engine (table.py:1185-1241); like
// that engine it is serializable but not serial-in-batch-order under
// contention, so tests check the policy invariants.
//
// One THREAD per op (HKV's TLPv1 shape): an op's chain is a
// handful of dependent round trips (probe, lock, claim, publish), so what
// pays is the number of ops in flight -- 32 per warp instead of 4 with an
// 8-lane tile (measured: 1M hits 0.51 -> see DESIGN.md).
//   probe      lock-free: the 128-B digest line and the 16-B occupancy word,
//              candidate keys in slot order.  A candidate whose key is LOCKED
//              may be this very key mid-update: the probe retries until it
//              resolves.
//   hit        CAS key -> LOCKED on the matched slot (a lost race retries the
//              whole op), refresh the score, write (or, find_or_insert, read)
//              the value row, release-store the key back (_scalar_hit,
//              table.py:749-772).
//   miss       take the bucket lock(s) (dual: both, lower index first), probe
//              again under it (a same-key insert may have won meanwhile),
//              then the structural change the reference does under its stripe
//              lock: claim the lowest free slot EMPTY -> LOCKED, or pick the
//              first-index minimum score, admit, CAS the victim old -> LOCKED
//              (a slot a hit holds is waited out and rescanned), capture the
//              evicted tuple, publish digest, score, value and the key last
//              (_publish_entry, table.py:737-747); release the lock(s).
// Bucket locks serialise only structural changes of one bucket; hits never
// wait on them.  Compiled with -dlcm=cg: metadata another SM just published
// must not be served from a stale L1 line.
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
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned cas_acquire_u32(unsigned* p, unsigned cmp, unsigned val) {
  unsigned old;
  asm volatile("atom.acquire.gpu.global.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "l"(p), "r"(cmp), "r"(val) : "memory");
  return old;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_key(const TableDev& t, uint64_t row) {
#ifdef HKV_CAS_KEYLDCG
  return __ldcg(kptr(t, row));
#else
  return *(volatile const uint64_t*)kptr(t, row);
#endif
}
__device__ __forceinline__ bool cas_key(const TableDev& t, uint64_t row, uint64_t expect) {
  return atomicCAS((unsigned long long*)kptr(t, row), (unsigned long long)expect,
                   (unsigned long long)kLockedKey) == (unsigned long long)expect;
}

// Bucket locks are sequence locks: even = free, odd = held; every holder
// advances the word by 2 (lock +1, unlock +1).  An op reads the word before
// its lock-free probe; if it can take the lock from that same even value, no
// structural change touched the bucket in between and the probe stands (no
// second probe under the lock).
__device__ __forceinline__ unsigned lock_bucket(unsigned* locks, uint64_t b, unsigned seen, bool& unchanged) {
  unchanged = (seen & 1u) == 0 && cas_acquire_u32(locks + b, seen, seen + 1) == seen;
  if (unchanged) return seen;
  for (;;) {
    const unsigned v = ld_acquire_u32(locks + b);
    if ((v & 1u) == 0 && cas_acquire_u32(locks + b, v, v + 1) == v) return v;
    __nanosleep(64);
  }
}
__device__ __forceinline__ void unlock_bucket(unsigned* locks, uint64_t b, unsigned from) {
  st_release_u32(locks + b, from + 2);
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
// holds the bucket's lock: exact groups come from the 64-B summary line, the
// others are rescanned (16 pairs each) and made exact.  gmin = the bucket's
// minimum, gi = the lowest group holding it (groups are in slot order, so the
// group's first slot holding gmin is np.argmin's first index, table.py:1080).
//
// svalid under this engine: bits 0-7 group valid, bits 8-31 a generation that
// every hit's score write bumps (then clears its group's bit).  The rescans
// are validated by a CAS from the word read before them, so a hit whose score
// write the rescan may have missed either fails that CAS (its bump landed
// first) or clears the bit after it -- a valid group never holds a minimum
// above its true one.
__device__ __forceinline__ void summ_min_thread(const TableDev& t, uint64_t b, uint64_t& gmin, int& gi) {
  const uint32_t sv0 = ld_acquire_u32(t.svalid + b);
  const uint32_t inv = ~sv0 & 0xFFu;
  const ulonglong2* p = reinterpret_cast<const ulonglong2*>(t.smin + b * 8);
  uint64_t sm[8];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const ulonglong2 x = __ldcg(p + k);
    sm[2 * k] = x.x;
    sm[2 * k + 1] = x.y;
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
    atomicCAS(t.svalid + b, sv0, sv0 | inv);
  }
  gmin = sm[0];
  gi = 0;
#pragma unroll
  for (int k = 1; k < 8; k++)
    if (sm[k] < gmin) { gmin = sm[k]; gi = k; }
}

// ---------------------------------------------------------------------------
// Warp-synchronous rounds.  A warp owns 32 ops (one per lane).  Each round,
// every unfinished op makes one NON-BLOCKING attempt: probe; hit -> CAS the
// slot; miss -> try the bucket lock(s), claim a free slot or (after the
// full-bucket decision through the eviction summary) CAS the victim, write the slot's metadata and
// drop the bucket lock(s) -- the slot itself stays LOCKED.  Then the warp
// moves every claimed op's value row with coalesced copies, fences, and
// publishes the keys.  An op that met a LOCKED candidate, a held lock or a
// lost CAS simply tries again next round; nothing is ever waited on while a
// lock or a LOCKED slot is held, so the rounds cannot deadlock.
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

#ifndef HKV_CAS_MINB
#define HKV_CAS_MINB 2
#endif
template <int VEC>
__global__ void __launch_bounds__(256, HKV_CAS_MINB) k_cas_upsert(TableDev t, OpArgs a, unsigned* locks, int64_t n) {
  if (a.sc->err) return;
  const int lane = threadIdx.x & 31;
  const uint64_t clock0 = *t.clock;
  const bool fel_open = !*t.fel_set;
  const int dim = t.dim;
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
    uint8_t outcome = kRejected;
    unsigned idle_rounds = 0;
    while (__any_sync(kFullMask, !done)) {
      int task = kTaskNone;
      bool need_scan = false, locked = false, retry = false;
      unsigned from_lo = 0, from_hi = 0;
      uint64_t row = 0, tb = b1, s_in = 0, victim = 0, minv = 0;
      int slot = -1;
      if (!done) {
        const unsigned seen_lo = ld_acquire_u32(locks + lo);
        const unsigned seen_hi = hi != lo ? ld_acquire_u32(locks + hi) : 0u;
        uint64_t hb = b1;
        uint4 w1, w2;
        slot = probe_op(t, b1, b2, key, d, ctr, hb, w1, w2);
        if (slot == -1) {
          // try the bucket lock(s) once; from the value seen before the
          // probe, the probe stands, else probe again under the lock
          const bool same_lo = (seen_lo & 1u) == 0 && cas_acquire_u32(locks + lo, seen_lo, seen_lo + 1) == seen_lo;
          if (same_lo) {
            from_lo = seen_lo;
          } else {
            const unsigned v = ld_acquire_u32(locks + lo);
            if ((v & 1u) == 0 && cas_acquire_u32(locks + lo, v, v + 1) == v) from_lo = v | 0x80000000u;
            else retry = true;
          }
          bool same_hi = true;
          if (!retry && hi != lo) {
            same_hi = (seen_hi & 1u) == 0 && cas_acquire_u32(locks + hi, seen_hi, seen_hi + 1) == seen_hi;
            if (same_hi) {
              from_hi = seen_hi;
            } else {
              const unsigned v = ld_acquire_u32(locks + hi);
              if ((v & 1u) == 0 && cas_acquire_u32(locks + hi, v, v + 1) == v) {
                from_hi = v;
              } else {
                unlock_bucket(locks, lo, from_lo & 0x7FFFFFFFu);
                retry = true;
              }
            }
          }
          if (!retry) {
            locked = true;
            from_lo &= 0x7FFFFFFFu;
            if (!(same_lo && same_hi)) slot = probe_op(t, b1, b2, key, d, ctr, hb, w1, w2);
          }
        }
        if (retry || slot == kBusy) {
          retry = true;
        } else if (slot >= 0) {
          // hit (table.py:749-772): hold the slot
          row = hb * kSlots + slot;
          if (cas_key(t, row, key)) {
            const uint64_t old = hit_needs_old(t.policy) ? __ldcg(sptr(t, row)) : 0;
            *sptr(t, row) = hit_score(t.policy, old, a.epoch, tick, a.scores != nullptr, cs);
            task = a.op == kOpFindOrInsert ? kTaskRead : kTaskHit;
          } else {
            retry = true;
          }
        } else {
          // the occupancy the probe under the lock(s) saw stands: only
          // structural changes move it, and they hold the bucket lock
          s_in = insert_score(t.policy, a.epoch, tick, cs);
          const int o1 = __popc(w1.x) + __popc(w1.y) + __popc(w1.z) + __popc(w1.w);
          const int o2 = t.dual ? __popc(w2.x) + __popc(w2.y) + __popc(w2.z) + __popc(w2.w) : kSlots;
          if (o1 < kSlots || o2 < kSlots) {
            // free insert (table.py:678-693, 1165-1181): single -> b1, dual D1
            const bool first = !t.dual || o1 <= o2;
            tb = first ? b1 : b2;
            const uint4 w = first ? w1 : w2;
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
            int q = 0;
            while (ws[q] == 0xFFFFFFFFu) q++;
            slot = 32 * q + __ffs(~ws[q]) - 1;  // the lowest EMPTY slot
            row = tb * kSlots + slot;
            // EMPTY -> LOCKED; under the bucket lock nothing else claims it
            atomicCAS((unsigned long long*)kptr(t, row), (unsigned long long)kEmptyKey,
                      (unsigned long long)kLockedKey);
            t.bits[tb * 4 + q] = ws[q] | (1u << (slot & 31));
            t.digests[row] = (uint8_t)d;
            *sptr(t, row) = s_in;
            // the summary is consulted only while the bucket is full: the
            // insert that fills it marks every group unknown
            if ((first ? o1 : o2) + 1 == kSlots) t.svalid[tb] = 0u;
            task = kTaskInsert;
          } else {
            need_scan = true;
          }
        }
      }
      // ---- full-bucket decisions through the eviction summary ----
      if (need_scan) {
        // first-index minimum of each bucket (table.py:1079-1083, 1099-1104)
        int gi;
        summ_min_thread(t, b1, minv, gi);
        tb = b1;
        ctr[kScans]++;
        if (t.dual) {
          uint64_t n2;
          int g2;
          summ_min_thread(t, b2, n2, g2);
          ctr[kScans]++;
          if (n2 < minv) {  // D2: the bucket with the lower minimum
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
          // the victim's group: its 16 pairs give the first slot holding the
          // minimum and, after the replacement, the group's new minimum
          const ulonglong2* gp = reinterpret_cast<const ulonglong2*>(kptr(t, tb * kSlots + 16 * gi));
          uint64_t v[16];
#pragma unroll
          for (int k = 0; k < 16; k++) v[k] = __ldcg(gp + k).y;
          uint64_t mn = v[0];
          int ms = 0;
#pragma unroll
          for (int k = 1; k < 16; k++)
            if (v[k] < mn) { mn = v[k]; ms = k; }
          if (mn != minv) {
            // a hit moved the group's minimum after the summary was read:
            // record the exact value and decide again next round
            t.smin[tb * 8 + gi] = mn;
            retry = true;
          } else {
            row = tb * kSlots + 16 * gi + ms;
            victim = ld_key(t, row);
            if (victim == kLockedKey || !cas_key(t, row, victim)) {
              retry = true;  // an op holds the minimum slot: decide again next round
            } else {
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
      // structure is settled: drop the bucket locks (claimed slots stay LOCKED)
      if (locked) {  // st.release: this thread's metadata writes before the unlock
        if (hi != lo) unlock_bucket(locks, hi, from_hi);
        unlock_bucket(locks, lo, from_lo);
      }
      if (retry) ctr[kRetries]++;
      // ---- warp-cooperative value movement ----
      float* vr = task != kTaskNone ? value_row(t, row) : nullptr;
      const unsigned cap_mask = __ballot_sync(kFullMask, task == kTaskEvict && a.collect);
      if (cap_mask) warp_copy_rows<VEC>(cap_mask, a.collect && task == kTaskEvict ? a.ev + (uint64_t)i * dim : nullptr,
                                        vr, dim, lane);
      const unsigned rd_mask = __ballot_sync(kFullMask, task == kTaskRead);
      if (rd_mask) warp_copy_rows<VEC>(rd_mask, vin, vr, dim, lane);
      const unsigned wr_mask = __ballot_sync(kFullMask, task == kTaskHit || task == kTaskInsert || task == kTaskEvict);
      if (wr_mask) warp_copy_rows<VEC>(wr_mask, vr, vin, dim, lane);
      if (task != kTaskNone) {
        ctr[row < t.fast_rows ? kVFast : kVOver] += (task == kTaskEvict && a.collect) ? 2 : 1;
        if (task == kTaskInsert) sd++;
        if (task == kTaskEvict && fel_open) atomicMin(&a.sc->first_ev, (unsigned)i);
        outcome = task == kTaskHit ? kUpdated : task == kTaskRead ? kFound : task == kTaskInsert ? kInserted : kEvicted;
        done = true;
      }
      __syncwarp();
      fence_rel();  // rows (every lane's stores) before the keys
      __syncwarp();
      if (task == kTaskHit || task == kTaskRead) {
        // the score write is fenced above: bump the generation, then drop
        // the group's bit (in this order, see summ_min_thread)
        atomicAdd(t.svalid + row / kSlots, 0x100u);
        atomicAnd(t.svalid + row / kSlots, ~(1u << ((row % kSlots) >> 4)));
      }
      if (task != kTaskNone) st_release_u64(kptr(t, row), key);
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

}  // namespace

cudaError_t run_cas(const TableDev& t, OpArgs a, int64_t n, unsigned* locks, int vec, cudaStream_t s,
                    int num_sms) {
  void* fn = vec == 4 ? (void*)k_cas_upsert<4> : vec == 2 ? (void*)k_cas_upsert<2> : (void*)k_cas_upsert<1>;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0);
  if (e) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)per_sm * num_sms;
  const int64_t want = (n + 255) / 256;
  if (blocks > want) blocks = want < 1 ? 1 : want;
  if (vec == 4) k_cas_upsert<4><<<(unsigned)blocks, 256, 0, s>>>(t, a, locks, n);
  else if (vec == 2) k_cas_upsert<2><<<(unsigned)blocks, 256, 0, s>>>(t, a, locks, n);
  else k_cas_upsert<1><<<(unsigned)blocks, 256, 0, s>>>(t, a, locks, n);
  g_launches++;
  return cudaGetLastError();
}

}  // namespace hkv
