// hkv_single.cu — the reference's single-key API (table.py:562-620):
// lookup, find_in_bucket, upsert_single, upsert_dual.  One key per call, so
// one device thread restates the scalar engine (table.py:621-857) directly:
// a digest-filtered probe in slot order, hit -> score refresh + value write,
// miss -> lowest free slot, or on a full bucket the first-index argmin and
// the admission test.  Single-key calls run under the inserter / reader role
// like their batch siblings, so no slot lock is needed (the reference's
// `locked=False` path); ticks are taken only where the scalar engine takes
// them (one per non-custom hit or insert decision, table.py:662-672, 713).
//
// Summary maintenance: the eviction summary of a touched bucket is marked
// unknown (svalid = 0); full-bucket decisions of later batches rescan it.
#include "hkv_kernels.h"
#include "hkv_single.h"

namespace hkv {

// Counters accumulate in the thread (c[6]) and reach the table only when the
// call succeeds: the reference merges a call's local TxnCounters after it
// returns, so a usage error counts nothing (table.py:588-598).
__device__ int probe_serial(const TableDev& t, uint64_t b, uint64_t key, uint32_t d, unsigned long long* ctr) {
  ctr[kLoads]++;
  const uint8_t* dl = t.digests + b * kSlots;
  const uint64_t* kr = kptr(t, b * kSlots);
  for (int s = 0; s < kSlots; s++) {
    if (t.digest_filter && dl[s] != d) continue;
    const uint64_t k = kr[2 * s];
    if (k == kEmptyKey) continue;
    ctr[kCompares]++;
    if (k == key) return s;
  }
  return -1;
}

__device__ void min_slot_serial(const TableDev& t, uint64_t b, int& m, uint64_t& mn) {
  const uint64_t* sr = sptr(t, b * kSlots);
  m = 0;
  mn = sr[0];
  for (int s = 1; s < kSlots; s++)
    if (sr[2 * s] < mn) {  // np.argmin: the first index on ties
      mn = sr[2 * s];
      m = s;
    }
}

__device__ int popc_bits(const TableDev& t, uint64_t b) {
  const uint32_t* w = t.bits + 4 * b;
  return __popc(w[0]) + __popc(w[1]) + __popc(w[2]) + __popc(w[3]);
}

__device__ int lowest_free(const TableDev& t, uint64_t b) {
  const uint32_t* w = t.bits + 4 * b;
  for (int q = 0; q < 4; q++)
    if (~w[q]) return 32 * q + __ffs(~w[q]) - 1;
  return -1;
}

__device__ void flush_one(const TableDev& t, const unsigned long long* c) {
  for (int k = 0; k < 6; k++)
    if (c[k]) atomicAdd(&t.counters[k], c[k]);
}

__device__ void write_row(const TableDev& t, uint64_t b, int s, const float* v, unsigned long long* c) {
  const uint64_t row = b * kSlots + (uint64_t)s;
  float* dst = value_row(t, row);
  for (int e = 0; e < t.dim; e++) dst[e] = v[e];
  c[row < t.fast_rows ? kVFast : kVOver]++;
}

// _publish_entry (table.py:737-742): digest, score, value, then the key
__device__ void publish(const TableDev& t, uint64_t b, int s, uint64_t key, uint32_t d, uint64_t score,
                        const float* v, unsigned long long* c) {
  t.digests[b * kSlots + s] = (uint8_t)d;
  *sptr(t, b * kSlots + s) = score;
  write_row(t, b, s, v, c);
  *kptr(t, b * kSlots + s) = key;
  t.svalid[b] = 0;
}

__global__ void k_lookup_one(TableDev t, uint64_t key, int64_t bucket, OneResult* r) {
  const uint64_t h = fmix64(key);
  const uint32_t d = digest_of(h);
  uint64_t b = bucket >= 0 ? (uint64_t)bucket : (h & t.mask);
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
  int s = probe_serial(t, b, key, d, c);
  if (s < 0 && bucket < 0 && t.dual) {
    b = second_hash(h) & t.mask;
    s = probe_serial(t, b, key, d, c);
  }
  flush_one(t, c);
  r->kind = s >= 0 ? kFound : kNotFound;
  r->status = 0;
  r->bucket = s >= 0 ? (int64_t)b : -1;
  r->slot = s;
}

// upsert_single (dual = 0: bucket h1 only, table.py:584-599 -- also on a
// dual-mode table) and upsert_dual (dual = 1, table.py:601-620 ->
// _scalar_upsert_dual 859-924).
__global__ void k_upsert_one(TableDev t, uint64_t key, const float* v, int dual, int has_score, uint64_t score,
                             uint64_t epoch, OneResult* r) {
  const uint64_t h = fmix64(key);
  const uint32_t d = digest_of(h);
  const uint64_t b1 = h & t.mask;
  const uint64_t b2 = second_hash(h) & t.mask;
  r->status = 0;
  r->evicted_key = 0;
  r->evicted_score = 0;
  uint64_t b = b1;
  unsigned long long c[6] = {0, 0, 0, 0, 0, 0};
  int s = probe_serial(t, b1, key, d, c);
  if (s < 0 && dual) {
    b = b2;
    s = probe_serial(t, b2, key, d, c);
  }
  const bool custom = t.policy == kCustom;
  if (s >= 0) {  // _scalar_hit (table.py:749-772)
    uint64_t& sc = *sptr(t, b * kSlots + s);
    uint64_t ns;
    if (custom) {
      ns = has_score ? score : sc;
    } else {
      const uint64_t tick = ++*t.clock;
      ns = hit_score(t.policy, sc, epoch, tick, false, 0);
    }
    sc = ns;
    write_row(t, b, s, v, c);
    t.svalid[b] = 0;
    r->kind = kUpdated;
    r->bucket = (int64_t)b;
    r->slot = s;
    flush_one(t, c);
    return;
  }
  // _score_for_insert (table.py:662-672): usage errors before any mutation
  if (custom && !has_score) {
    r->status = 1;
    return;
  }
  if (!custom && has_score) {
    r->status = 2;
    return;
  }
  const uint64_t s_in = custom ? score : insert_score(t.policy, epoch, ++*t.clock, 0);
  uint64_t tb = b1;
  int m;
  uint64_t mn;
  if (dual) {
    const int o1 = popc_bits(t, b1), o2 = popc_bits(t, b2);
    if (o1 < kSlots || o2 < kSlots) {
      tb = o1 <= o2 ? b1 : b2;  // D1: the less-occupied candidate
      m = -1;
    } else {
      int m1, m2;
      uint64_t n1, n2;
      min_slot_serial(t, b1, m1, n1);
      min_slot_serial(t, b2, m2, n2);
      c[kScans] += 2;
      const uint64_t both = n1 < n2 ? n1 : n2;
      const bool admit = t.admit_unified ? s_in >= both : s_in > both;
      if (!admit) {
        r->kind = kRejected;
        r->bucket = -1;
        r->slot = -1;
        flush_one(t, c);
        return;
      }
      if (n2 < n1) {
        tb = b2, m = m2, mn = n2;
      } else {
        tb = b1, m = m1, mn = n1;
      }
    }
  } else {
    m = popc_bits(t, b1) < kSlots ? -1 : 0;
    if (m == 0) {
      min_slot_serial(t, b1, m, mn);
      c[kScans]++;
      if (s_in < mn) {  // _scalar_evict admission (table.py:806)
        r->kind = kRejected;
        r->bucket = -1;
        r->slot = -1;
        flush_one(t, c);
        return;
      }
    }
  }
  if (m < 0) {  // _scalar_claim_free + _publish_entry (table.py:678-693, 737-742)
    const int f = lowest_free(t, tb);
    t.bits[4 * tb + (f >> 5)] |= 1u << (f & 31);
    *t.size += 1ull;
    publish(t, tb, f, key, d, s_in, v, c);
    r->kind = kInserted;
    r->bucket = (int64_t)tb;
    r->slot = f;
    flush_one(t, c);
    return;
  }
  // eviction (table.py:834-857): first-eviction lambda at the size of the decision
  if (!*t.fel_set) {
    *t.fel = (double)(long long)*t.size / (double)t.capacity;
    *t.fel_set = 1;
  }
  r->evicted_key = *kptr(t, tb * kSlots + m);
  r->evicted_score = mn;
  publish(t, tb, m, key, d, s_in, v, c);
  r->kind = kEvicted;
  r->bucket = (int64_t)tb;
  r->slot = m;
  flush_one(t, c);
}

void launch_lookup_one(const TableDev& t, uint64_t key, int64_t bucket, OneResult* r, cudaStream_t s) {
  k_lookup_one<<<1, 1, 0, s>>>(t, key, bucket, r);
  g_launches++;
}

void launch_upsert_one(const TableDev& t, uint64_t key, const float* v, int dual, int has_score, uint64_t score,
                       uint64_t epoch, OneResult* r, cudaStream_t s) {
  k_upsert_one<<<1, 1, 0, s>>>(t, key, v, dual, has_score, score, epoch, r);
  g_launches++;
}

}  // namespace hkv
