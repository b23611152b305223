// hkv_cas.cu — the concurrent upsert engine: the reference's LOCKED-sentinel
// slot CAS protocol (table.py:678-857) with every op
// of a batch in flight at once.  Selected by TableConfig.workers > 1, the
// reference's switch to its threaded CAS engine (table.py:1185-1241); like
// that engine it is serializable but not serial-in-batch-order under
// contention, so tests check the policy invariants.
//
// One 8-lane tile per op (lane r: slots 16r..16r+15 of a bucket):
//   probe      lock-free: digest slice + occupancy slice per lane, candidate
//              keys in slot order.  A candidate whose key is LOCKED may be
//              this very key mid-update: the probe retries until it resolves.
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

__device__ __forceinline__ uint64_t ld_key(const TableDev& t, uint64_t row) {
  return *(volatile const uint64_t*)(t.keys + row);
}

// Lock-free probe of bucket b: slot of `key`, -1 (absent), or kBusy (a
// digest candidate is LOCKED: an op holds it mid-update).
__device__ __forceinline__ int probe_cas(const TableDev& t, const Tile8& tile, uint64_t b, uint64_t key, uint32_t d,
                                         ctr_t& ncmp) {
  const int r = tile.thread_rank();
  const uint4 dw = __ldcg(reinterpret_cast<const uint4*>(t.digests + b * kSlots) + r);
  const uint32_t occ = __ldcg(reinterpret_cast<const unsigned short*>(t.bits + b * 4) + r);
  uint32_t cand = (t.digest_filter ? match16(dw, d) : 0xFFFFu) & occ;
  int hit = -1, cmp = 0, cmp_all = 0;
  bool busy = false;
  while (cand) {
    const int j = __ffs(cand) - 1;
    cand &= cand - 1;
    const uint64_t k = ld_key(t, b * kSlots + r * kSPL + j);
    if (k == kLockedKey) {
      busy = true;
      continue;
    }
    if (k == kEmptyKey) continue;
    cmp_all++;
    if (k == key) {
      hit = r * kSPL + j;
      cmp = cmp_all;
      break;
    }
  }
  const uint32_t hm = tile.ballot(hit >= 0);
  int contrib = cmp_all;
  int slot = -1;
  if (hm) {
    const int hl = __ffs(hm) - 1;
    slot = tile.shfl(hit, hl);
    contrib = r < hl ? cmp_all : (r == hl ? cmp : 0);
  } else if (tile.any(busy)) {
    slot = kBusy;
  }
  ncmp += tile.sum((unsigned)contrib);
  return slot;
}

__device__ __forceinline__ void lock_bucket(unsigned* locks, uint64_t b) {
  while (atomicCAS(locks + b, 0u, 1u) != 0u) __nanosleep(64);
  __threadfence();
}
__device__ __forceinline__ void unlock_bucket(unsigned* locks, uint64_t b) {
  __threadfence();
  atomicExch(locks + b, 0u);
}

// slot CAS by the owning lane, result broadcast to the tile
__device__ __forceinline__ bool cas_slot(const TableDev& t, const Tile8& tile, uint64_t row, int slot,
                                         uint64_t expect) {
  int ok = 0;
  if (tile.thread_rank() == slot / kSPL)
    ok = atomicCAS((unsigned long long*)(t.keys + row), (unsigned long long)expect,
                   (unsigned long long)kLockedKey) == (unsigned long long)expect;
  return tile.shfl(ok, slot / kSPL) != 0;
}

// publish: digest, score (and the value row, written by the caller), then
// the key with release semantics
__device__ __forceinline__ void publish_key(const TableDev& t, const Tile8& tile, uint64_t row, int slot,
                                            uint64_t key) {
  __threadfence();
  tile.sync();
  if (tile.thread_rank() == slot / kSPL) *(volatile uint64_t*)(t.keys + row) = key;
}

template <int VEC>
__device__ __forceinline__ void copy_in(float* dst, const float* vin, int dim, int r) {
  copy_row<kG, VEC>(dst, vin, dim, r);
}

// the hit path on (hb, slot) once its key is LOCKED by this tile
template <int VEC>
__device__ __forceinline__ uint8_t do_hit(const TableDev& t, const OpArgs& a, const Tile8& tile, uint32_t i,
                                          uint64_t hb, int slot, uint64_t key, uint64_t tick, uint64_t cs,
                                          ctr_t* ctr) {
  const int r = tile.thread_rank();
  const uint64_t row = hb * kSlots + slot;
  if (r == slot / kSPL) {
    const uint64_t old = hit_needs_old(t.policy) ? *(volatile uint64_t*)(t.scores + row) : 0;
    t.scores[row] = hit_score(t.policy, old, a.epoch, tick, a.scores != nullptr, cs);
    summ_invalidate(t, hb, slot);
  }
  float* vr = value_row(t, row);
  float* vin = a.values + (uint64_t)i * t.dim;
  uint8_t outcome;
  if (a.op == kOpFindOrInsert) {
    copy_row<kG, VEC>(vin, vr, t.dim, r);
    outcome = kFound;
  } else {
    copy_in<VEC>(vr, vin, t.dim, r);
    outcome = kUpdated;
  }
  ctr[row < t.fast_rows ? kVFast : kVOver]++;
  publish_key(t, tile, row, slot, key);
  return outcome;
}

template <int VEC>
__device__ void process_cas(const TableDev& t, const OpArgs& a, unsigned* locks, const Tile8& tile, uint32_t i,
                            uint64_t clock0, bool fel_open, ctr_t* ctr, int& size_delta) {
  const int r = tile.thread_rank();
  const int dim = t.dim;
  const uint64_t key = a.keys[i];
  const uint64_t h = fmix64(key);
  const uint32_t d = digest_of(h);
  const uint64_t b1 = h & t.mask;
  const uint64_t b2 = t.dual ? second_hash(h) & t.mask : b1;
  const uint64_t tick = a.ticks ? a.ticks[i] : clock0 + (uint64_t)i + 1;
  const uint64_t cs = a.scores ? a.scores[i] : 0;
  float* vin = a.values + (uint64_t)i * dim;
  uint8_t outcome = kRejected;
  for (;;) {
    // ---- lock-free probe + hit ----
    uint64_t hb = b1;
    int slot = probe_cas(t, tile, b1, key, d, ctr[kCompares]);
    ctr[kLoads]++;
    if (slot == -1 && t.dual) {
      hb = b2;
      slot = probe_cas(t, tile, b2, key, d, ctr[kCompares]);
      ctr[kLoads]++;
    }
    if (slot == kBusy) {
      ctr[kRetries]++;
      __nanosleep(32);
      continue;
    }
    if (slot >= 0) {
      if (!cas_slot(t, tile, hb * kSlots + slot, slot, key)) {
        ctr[kRetries]++;  // lost the slot race; the key may have moved
        continue;
      }
      outcome = do_hit<VEC>(t, a, tile, i, hb, slot, key, tick, cs, ctr);
      break;
    }
    // ---- miss: structural change under the bucket lock(s) ----
    const uint64_t lo = b1 < b2 ? b1 : b2, hi = b1 < b2 ? b2 : b1;
    if (r == 0) {
      lock_bucket(locks, lo);
      if (hi != lo) lock_bucket(locks, hi);
    }
    tile.sync();
    // probe again under the lock: a same-key insert may have won meanwhile;
    // an in-flight hit (no lock) is waited out
    hb = b1;
    do {
      slot = probe_cas(t, tile, b1, key, d, ctr[kCompares]);
      ctr[kLoads]++;
      hb = b1;
      if (slot == -1 && t.dual) {
        slot = probe_cas(t, tile, b2, key, d, ctr[kCompares]);
        ctr[kLoads]++;
        hb = b2;
      }
    } while (slot == kBusy);
    if (slot >= 0) {
      while (!cas_slot(t, tile, hb * kSlots + slot, slot, key)) ctr[kRetries]++;
      outcome = do_hit<VEC>(t, a, tile, i, hb, slot, key, tick, cs, ctr);
    } else {
      const uint64_t s_in = insert_score(t.policy, a.epoch, tick, cs);
      const uint32_t occ1 = __ldcg(reinterpret_cast<const unsigned short*>(t.bits + b1 * 4) + r);
      const uint32_t occ2 =
          t.dual ? __ldcg(reinterpret_cast<const unsigned short*>(t.bits + b2 * 4) + r) : occ1;
      const int o1 = tile_sum<kG>(tile, __popc(occ1));
      const int o2 = t.dual ? tile_sum<kG>(tile, __popc(occ2)) : kSlots;
      if (o1 < kSlots || (t.dual && o2 < kSlots)) {
        // free insert: single -> b1; dual D1 -> the less-occupied bucket
        const uint64_t tb = (!t.dual || o1 <= o2) ? b1 : b2;
        const uint32_t occ = tb == b1 ? occ1 : occ2;
        const uint32_t hasfree = tile.ballot(occ != 0xFFFFu);
        const int fl = __ffs(hasfree) - 1;
        int s = 0;
        if (r == fl) s = r * kSPL + __ffs(~occ & 0xFFFFu) - 1;
        s = tile.shfl(s, fl);
        const uint64_t row = tb * kSlots + s;
        // claim EMPTY -> LOCKED (table.py:678-693); under the bucket lock
        // nothing else can claim it
        while (!cas_slot(t, tile, row, s, kEmptyKey)) ctr[kRetries]++;
        if (r == fl) {
          store_occ(t, tb, r, occ | (1u << (s % kSPL)));
          t.digests[row] = (uint8_t)d;
          t.scores[row] = s_in;
        }
        if (r == 0) atomicAnd(t.svalid + tb, 0u);
        copy_in<VEC>(value_row(t, row), vin, dim, r);
        ctr[row < t.fast_rows ? kVFast : kVOver]++;
        publish_key(t, tile, row, s, key);
        size_delta++;
        outcome = kInserted;
      } else {
        for (;;) {
          uint64_t tb = b1, minv;
          int m;
          bool admit;
          if (!t.dual) {
            bucket_min(t, tile, b1, minv, m);
            ctr[kScans]++;
            admit = s_in >= minv;  // the single-bucket path admits ties
          } else {
            uint64_t n1, n2;
            int m1, m2;
            bucket_min(t, tile, b1, n1, m1);
            bucket_min(t, tile, b2, n2, m2);
            ctr[kScans] += 2;
            const bool use2 = n2 < n1;  // D2: the bucket with the lower minimum
            tb = use2 ? b2 : b1;
            m = use2 ? m2 : m1;
            minv = use2 ? n2 : n1;
            admit = t.admit_unified ? s_in >= minv : s_in > minv;
          }
          if (!admit) {
            outcome = kRejected;
            break;
          }
          const uint64_t row = tb * kSlots + m;
          uint64_t old = 0;
          if (r == m / kSPL) old = ld_key(t, row);
          old = tile.shfl(old, m / kSPL);
          if (old == kLockedKey || !cas_slot(t, tile, row, m, old)) {
            ctr[kRetries]++;  // a hit holds the minimum slot: wait it out, rescan
            __nanosleep(32);
            continue;
          }
          float* vr = value_row(t, row);
          if (a.collect) {
            if (r == 0) {
              a.ek[i] = old;
              a.es[i] = minv;
            }
            copy_row<kG, VEC>(a.ev + (uint64_t)i * dim, vr, dim, r);
            ctr[row < t.fast_rows ? kVFast : kVOver]++;
          }
          if (r == m / kSPL) {
            t.digests[row] = (uint8_t)d;
            t.scores[row] = s_in;
          }
          if (r == 0) atomicAnd(t.svalid + tb, 0u);
          copy_in<VEC>(vr, vin, dim, r);
          ctr[row < t.fast_rows ? kVFast : kVOver]++;
          publish_key(t, tile, row, m, key);
          if (fel_open && r == 0) atomicMin(&a.sc->first_ev, i);
          outcome = kEvicted;
          break;
        }
      }
    }
    tile.sync();
    if (r == 0) {
      if (hi != lo) unlock_bucket(locks, hi);
      unlock_bucket(locks, lo);
    }
    break;
  }
  if (r == 0) a.outcomes[i] = outcome;
}

template <int VEC>
__global__ void __launch_bounds__(256) k_cas_upsert(TableDev t, OpArgs a, unsigned* locks, int64_t n) {
  if (a.sc->err) return;
  const Tile8 tile;
  const uint64_t clock0 = *t.clock;
  const bool fel_open = !*t.fel_set;
  ctr_t ctr[6] = {0, 0, 0, 0, 0, 0};
  int sd = 0;
  const int64_t tiles = (int64_t)gridDim.x * (blockDim.x / kG);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x / kG) + threadIdx.x / kG; i < n; i += tiles)
    process_cas<VEC>(t, a, locks, tile, (uint32_t)i, clock0, fel_open, ctr, sd);
  if (tile.thread_rank() != 0) {
#pragma unroll
    for (int k = 0; k < 6; k++) ctr[k] = 0;
    sd = 0;
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
  const int64_t want = (n * kG + 255) / 256;
  if (blocks > want) blocks = want < 1 ? 1 : want;
  if (vec == 4) k_cas_upsert<4><<<(unsigned)blocks, 256, 0, s>>>(t, a, locks, n);
  else if (vec == 2) k_cas_upsert<2><<<(unsigned)blocks, 256, 0, s>>>(t, a, locks, n);
  else k_cas_upsert<1><<<(unsigned)blocks, 256, 0, s>>>(t, a, locks, n);
  g_launches++;
  return cudaGetLastError();
}

}  // namespace hkv
