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

// Lock-free probe of bucket b by one thread: slot of `key`, -1 (absent), or
// kBusy (a digest candidate is LOCKED: an op holds it mid-update).  Compares
// counted as table.py:243-268 (candidates in slot order, up to the match).
__device__ __forceinline__ int probe_cas(const TableDev& t, uint64_t b, uint64_t key, uint32_t d, ctr_t& ncmp) {
  const uint4* dp = reinterpret_cast<const uint4*>(t.digests + b * kSlots);
  const uint4 ow = __ldcg(reinterpret_cast<const uint4*>(t.bits + b * 4));
  const uint32_t occ[4] = {ow.x, ow.y, ow.z, ow.w};
  uint32_t c[4];
  {
    uint4 w[8];
#pragma unroll
    for (int k = 0; k < 8; k++) w[k] = __ldcg(dp + k);
#pragma unroll
    for (int q = 0; q < 4; q++)
      c[q] = (t.digest_filter ? (match16(w[2 * q], d) | (match16(w[2 * q + 1], d) << 16)) : ~0u) & occ[q];
  }
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

// ---------------------------------------------------------------------------
// Warp-synchronous rounds.  A warp owns 32 ops (one per lane).  Each round,
// every unfinished op makes one NON-BLOCKING attempt: probe; hit -> CAS the
// slot; miss -> try the bucket lock(s), claim a free slot or (after a
// warp-cooperative score scan) CAS the victim, write the slot's metadata and
// drop the bucket lock(s) -- the slot itself stays LOCKED.  Then the warp
// moves every claimed op's value row with coalesced copies, fences, and
// publishes the keys.  An op that met a LOCKED candidate, a held lock or a
// lost CAS simply tries again next round; nothing is ever waited on while a
// lock or a LOCKED slot is held, so the rounds cannot deadlock.
// ---------------------------------------------------------------------------
enum : int { kTaskNone = 0, kTaskHit = 1, kTaskRead = 2, kTaskInsert = 3, kTaskEvict = 4 };
constexpr unsigned kFullMask = 0xFFFFFFFFu;
#ifndef HKV_CAS_SCANB
#define HKV_CAS_SCANB 2
#endif
constexpr int kScanBatch = HKV_CAS_SCANB;  // full-bucket scans per warp pass

// first-index minimum (np.argmin, table.py:1080) of bucket b's 128 scores,
// read by the whole warp (lane j: slots 4j..4j+3, 1 KB coalesced)
__device__ __forceinline__ void warp_min(const TableDev& t, uint64_t b, int lane, uint64_t& minv, int& mslot) {
  const ulonglong2* sp = reinterpret_cast<const ulonglong2*>(kptr(t, b * kSlots + 4 * lane));
  const uint64_t s0 = __ldcg(sp).y, s1 = __ldcg(sp + 1).y, s2 = __ldcg(sp + 2).y, s3 = __ldcg(sp + 3).y;
  uint64_t v = s0;
  int m = 4 * lane;
  if (s1 < v) { v = s1; m = 4 * lane + 1; }
  if (s2 < v) { v = s2; m = 4 * lane + 2; }
  if (s3 < v) { v = s3; m = 4 * lane + 3; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t ov = __shfl_xor_sync(kFullMask, v, o);
    const int om = __shfl_xor_sync(kFullMask, m, o);
    if (ov < v || (ov == v && om < m)) { v = ov; m = om; }
  }
  minv = v;
  mslot = m;
}

// first-index minimum over a bucket whose 128 scores the warp holds four
// per lane (x, y = slots 4 lane .. 4 lane + 3)
__device__ __forceinline__ void lane_min4(ulonglong2 x, ulonglong2 y, int lane, uint64_t& minv, int& mslot) {
  uint64_t v = x.x;
  int m = 4 * lane;
  if (x.y < v) { v = x.y; m = 4 * lane + 1; }
  if (y.x < v) { v = y.x; m = 4 * lane + 2; }
  if (y.y < v) { v = y.y; m = 4 * lane + 3; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t ov = __shfl_xor_sync(kFullMask, v, o);
    const int om = __shfl_xor_sync(kFullMask, m, o);
    if (ov < v || (ov == v && om < m)) { v = ov; m = om; }
  }
  minv = v;
  mslot = m;
}

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
        slot = probe_cas(t, b1, key, d, ctr[kCompares]);
        ctr[kLoads]++;
        if (slot == -1 && t.dual) {
          hb = b2;
          slot = probe_cas(t, b2, key, d, ctr[kCompares]);
          ctr[kLoads]++;
        }
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
            if (!(same_lo && same_hi)) {
              hb = b1;
              slot = probe_cas(t, b1, key, d, ctr[kCompares]);
              ctr[kLoads]++;
              if (slot == -1 && t.dual) {
                hb = b2;
                slot = probe_cas(t, b2, key, d, ctr[kCompares]);
                ctr[kLoads]++;
              }
            }
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
            summ_invalidate(t, hb, slot);
            task = a.op == kOpFindOrInsert ? kTaskRead : kTaskHit;
          } else {
            retry = true;
          }
        } else {
          s_in = insert_score(t.policy, a.epoch, tick, cs);
          const uint4 w1 = __ldcg(reinterpret_cast<const uint4*>(t.bits + b1 * 4));
          const uint4 w2 = t.dual ? __ldcg(reinterpret_cast<const uint4*>(t.bits + b2 * 4)) : w1;
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
            t.svalid[tb] = 0u;
            task = kTaskInsert;
          } else {
            need_scan = true;
          }
        }
      }
      // ---- warp-cooperative score scans for full-bucket decisions ----
      unsigned sm = __ballot_sync(kFullMask, need_scan);
      while (sm) {
        // kScanBatch ops' buckets per pass, all loads in flight before the reductions
        int ls[kScanBatch];
        uint64_t p1[kScanBatch], p2[kScanBatch];
#pragma unroll
        for (int k = 0; k < kScanBatch; k++) {
          ls[k] = sm ? __ffs(sm) - 1 : -1;
          if (sm) sm &= sm - 1;
          p1[k] = __shfl_sync(kFullMask, b1, ls[k] < 0 ? 0 : ls[k]);
          p2[k] = __shfl_sync(kFullMask, b2, ls[k] < 0 ? 0 : ls[k]);
        }
        ulonglong2 x1[kScanBatch], y1[kScanBatch], x2[kScanBatch], y2[kScanBatch];
#pragma unroll
        for (int k = 0; k < kScanBatch; k++) {
          if (ls[k] < 0) continue;
          const ulonglong2* sp = reinterpret_cast<const ulonglong2*>(kptr(t, p1[k] * kSlots + 4 * lane));
          x1[k] = make_ulonglong2(__ldcg(sp).y, __ldcg(sp + 1).y);
          y1[k] = make_ulonglong2(__ldcg(sp + 2).y, __ldcg(sp + 3).y);
          if (t.dual) {
            const ulonglong2* sq = reinterpret_cast<const ulonglong2*>(kptr(t, p2[k] * kSlots + 4 * lane));
            x2[k] = make_ulonglong2(__ldcg(sq).y, __ldcg(sq + 1).y);
            y2[k] = make_ulonglong2(__ldcg(sq + 2).y, __ldcg(sq + 3).y);
          }
        }
#pragma unroll
        for (int k = 0; k < kScanBatch; k++) {
          if (ls[k] < 0) continue;
          uint64_t n1, n2 = kMaxScore;
          int m1, m2 = 0;
          lane_min4(x1[k], y1[k], lane, n1, m1);
          if (t.dual) lane_min4(x2[k], y2[k], lane, n2, m2);
          if (lane == ls[k]) {
            if (!t.dual) {
              ctr[kScans]++;
              minv = n1, slot = m1, tb = b1;
            } else {
              ctr[kScans] += 2;
              const bool use2 = n2 < n1;  // D2: the bucket with the lower minimum
              minv = use2 ? n2 : n1, slot = use2 ? m2 : m1, tb = use2 ? b2 : b1;
            }
          }
        }
      }
      if (need_scan) {
        const bool admit = t.dual ? (t.admit_unified ? s_in >= minv : s_in > minv) : s_in >= minv;
        if (!admit) {
          outcome = kRejected;
          done = true;
        } else {
          row = tb * kSlots + slot;
          victim = ld_key(t, row);
          if (victim == kLockedKey || !cas_key(t, row, victim)) {
            retry = true;  // an op holds the minimum slot: rescan next round
          } else {
            if (a.collect) {
              a.ek[kRecU64 * i] = victim;
              a.es[kRecU64 * i] = minv;
            }
            t.digests[row] = (uint8_t)d;
            *sptr(t, row) = s_in;
            t.svalid[tb] = 0u;
            task = kTaskEvict;
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
