// hkv_common.cuh — device-side layout, hashing and score policies shared by
// every kernel of the B200 table.
//
// HBM layout (bucket-major; one bucket = 128 slots, the key's whole
// candidate space):
//   digests [B][128] u8   one 128-B line per bucket (the probe's first read)
//   bits    [B][4]   u32  128-bit occupancy bitmap (bit s <=> keys[b][s] is a
//                         user key); replaces the reference's occupancy
//                         counter + argmax(keys==EMPTY) scan (table.py:1171)
//   ks      [B][128] {u64 key, u64 score}  one 16-B pair per slot (16 lines per
//                         bucket): an insert's key and score writes land in one
//                         32-B sector instead of two in separate arrays
//   smin    [B][8]   u64  eviction summary: min score of each 16-slot group, so
//   svalid  [B]      u32  a full-bucket argmin reads 64 B + one group's 128 B
//                         instead of the 1-KB score row (bit g: group g exact;
//                         only meaningful while the bucket is full)
//   values  rows [capacity][dim] f32: rows < fast_rows in HBM, the rest in the
//           overflow arena (mapped pinned host memory, or HBM)
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <type_traits>
#include <utility>
#include <cuda_runtime.h>

namespace hkv {

namespace cg = cooperative_groups;

constexpr int kSlots = 128;
constexpr uint64_t kEmptyKey = 0xFFFFFFFFFFFFFFFFull;   // hashing.py:10
constexpr uint64_t kLockedKey = 0xFFFFFFFFFFFFFFFEull;  // hashing.py:11
constexpr uint64_t kMaxScore = 0xFFFFFFFFFFFFFFFFull;
constexpr uint64_t kLow32 = 0xFFFFFFFFull;

enum Policy : int { kLru = 0, kLfu = 1, kEpochLru = 2, kEpochLfu = 3, kCustom = 4 };
enum Outcome : uint8_t {
  kInserted = 0, kUpdated = 1, kRejected = 2, kEvicted = 3, kFound = 4, kNotFound = 5, kErased = 6
};
enum Ctr : int { kLoads = 0, kCompares = 1, kScans = 2, kRetries = 3, kVFast = 4, kVOver = 5 };

// Table metadata handed to kernels by value.
struct TableDev {
  uint64_t* ks;       // [capacity] x {key, score} (kptr / sptr)
  uint8_t* digests;
  uint32_t* bits;
  uint64_t* smin;     // [B][8] min score of each 16-slot group (exact where svalid says so)
  uint32_t* svalid;   // [B] bit g set <=> smin[b][g] == min(scores[b][16g .. 16g+15])
  float* vfast;       // rows [0, fast_rows)
  float* vover;       // rows [fast_rows, capacity), indexed row - fast_rows
  uint64_t fast_rows;
  uint64_t mask;      // bucket_count - 1
  uint64_t capacity;
  int dim;
  int dual;
  int policy;
  int digest_filter;
  int admit_unified;
  // device scalars
  unsigned long long* size;      // int64 two's complement
  unsigned long long* clock;
  unsigned long long* counters;  // [6]
  int* err;                      // error latch
  int* fel_set;
  double* fel;
  const unsigned* role_word;     // device mirror of the role gate: (group << 2) | (role + 1)
  int cas;                       // workers > 1: concurrent slot-CAS upserts (hkv_cas.cu)
  unsigned* locks;               // [B] bucket locks of the CAS engine (structural changes)
};

// Mutation kernels refuse to run while the gate's device mirror names a
// reader group (hkv_gate.cu; HKV_DERR_ROLE = 2 in the error latch).
__device__ __forceinline__ bool role_forbids_mutation(const TableDev& t) {
  return t.role_word != nullptr && ((*(volatile const unsigned*)t.role_word) & 3u) == 1u;
}

// hashing.py:21-29 fmix64 (Murmur3 finalizer)
__device__ __forceinline__ uint64_t fmix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xFF51AFD7ED558CCDull;
  x ^= x >> 33;
  x *= 0xC4CEB9FE1A85EC53ull;
  x ^= x >> 33;
  return x;
}
// hashing.py:52-57 second hash for dual mode
__device__ __forceinline__ uint64_t second_hash(uint64_t h1) {
  return fmix64(h1 ^ 0x9E3779B97F4A7C15ull);
}
// hashing.py:60-66: digest = bits 32..39
__device__ __forceinline__ uint32_t digest_of(uint64_t h) { return (uint32_t)(h >> 32) & 0xFFu; }

// scoring.py:56-76 score_on_insert
__device__ __forceinline__ uint64_t insert_score(int policy, uint64_t epoch, uint64_t tick,
                                                 uint64_t custom) {
  switch (policy) {
    case kLru: return tick;
    case kLfu: return 1;
    case kEpochLru: return (epoch << 32) | (tick & kLow32);
    case kEpochLfu: return (epoch << 32) | 1;
    default: return custom;
  }
}

// scoring.py:79-102 score_on_hit
__device__ __forceinline__ uint64_t hit_score(int policy, uint64_t old, uint64_t epoch,
                                              uint64_t tick, bool has_custom, uint64_t custom) {
  switch (policy) {
    case kLru: return tick;
    case kLfu: return old == kMaxScore ? old : old + 1;
    case kEpochLru: return (epoch << 32) | (tick & kLow32);
    case kEpochLfu: {
      if ((old >> 32) == epoch) {
        uint64_t low = old & kLow32;
        if (low < kLow32) low++;
        return (epoch << 32) | low;
      }
      return (epoch << 32) | 1;
    }
    default: return has_custom ? custom : old;
  }
}

__device__ __forceinline__ bool hit_needs_old(int policy) {
  return policy == kLfu || policy == kEpochLfu || policy == kCustom;
}

// slot row's key and score in the interleaved pair array
__device__ __forceinline__ uint64_t* kptr(const TableDev& t, uint64_t row) { return t.ks + 2 * row; }
__device__ __forceinline__ uint64_t* sptr(const TableDev& t, uint64_t row) { return t.ks + 2 * row + 1; }

// store.py:84-94 / 115-131: position-addressed value row.
__device__ __forceinline__ float* value_row(const TableDev& t, uint64_t row) {
  return row < t.fast_rows ? t.vfast + row * (uint64_t)t.dim
                           : t.vover + (row - t.fast_rows) * (uint64_t)t.dim;
}

// Byte-equality of 4 digests against d as a 4-bit mask: __vcmpeq4 gives 0xFF
// per equal byte; keeping bit 0 of each byte (positions 0, 8, 16, 24) and
// multiplying by 2^21 + 2^14 + 2^7 + 1 gathers them into bits 21..24 with no
// colliding partial products (other partial products land outside 21..24).
__device__ __forceinline__ uint32_t match4(uint32_t w, uint32_t dd) {
  const uint32_t x = __vcmpeq4(w, dd) & 0x01010101u;
  return ((x * 0x00204081u) >> 21) & 0xFu;
}

// 16 digest bytes (one uint4) vs the query digest -> 16-bit match mask.
__device__ __forceinline__ uint32_t match16(uint4 w, uint32_t d) {
  const uint32_t dd = d * 0x01010101u;
  return match4(w.x, dd) | (match4(w.y, dd) << 4) | (match4(w.z, dd) << 8) | (match4(w.w, dd) << 12);
}

// Does any of the 16 digest bytes equal d?  (x - 0x01..) & ~x & 0x80.. is
// non-zero iff x has a zero byte (the per-byte bits may over-report above a
// zero byte, the word-level answer is exact): 3 ALU ops per word against ~8
// for the exact mask, so the common no-candidate case (78 % of fresh keys at
// lambda 0.5) skips the mask entirely.
__device__ __forceinline__ uint32_t any16(uint4 w, uint32_t dd) {
  const uint32_t a = w.x ^ dd, b = w.y ^ dd, c = w.z ^ dd, e = w.w ^ dd;
  return ((a - 0x01010101u) & ~a) | ((b - 0x01010101u) & ~b) | ((c - 0x01010101u) & ~c) |
         ((e - 0x01010101u) & ~e);
}

// L2 eviction priority for the small per-op plan arrays (outcomes, value
// rows, read provenance) that the metadata pass writes at random batch
// indices while it streams hundreds of MB of bucket lines through L2: with
// evict_last they stay resident until the value pass reads them, instead of
// costing a DRAM sector fill and write-back per op.
#ifndef HKV_L2HINT
#define HKV_L2HINT 1
#endif
__device__ __forceinline__ uint64_t l2_keep_policy() {
  uint64_t p = 0;
#if HKV_L2HINT
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
__device__ __forceinline__ void st_keep(uint32_t* a, uint32_t v, uint64_t pol) {
#if HKV_L2HINT
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol) : "memory");
#else
  *a = v;
#endif
}
__device__ __forceinline__ void st_keep(int32_t* a, int32_t v, uint64_t pol) {
  st_keep(reinterpret_cast<uint32_t*>(a), (uint32_t)v, pol);
}
__device__ __forceinline__ void st_keep(uint8_t* a, uint8_t v, uint64_t pol) {
#if HKV_L2HINT
  asm volatile("st.global.L2::cache_hint.b8 [%0], %1, %2;" ::"l"(a), "r"((uint32_t)v), "l"(pol) : "memory");
#else
  *a = v;
#endif
}

// Streaming loads/stores for data touched once.
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(uint4* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Copy one value row of `dim` floats with a tile of G lanes, VEC floats per
// access (VEC = 4 requires 16-B aligned rows, i.e. dim % 4 == 0).  Loads are
// issued in groups of U before the matching stores so a lane keeps U
// requests in flight.
template <typename V>
__device__ __forceinline__ V ld_vec(const V* p) { return *p; }
template <typename V>
__device__ __forceinline__ void st_vec(V* p, V v) { *p = v; }

template <int G, int VEC, int U = 2>
__device__ __forceinline__ void copy_row(float* dst, const float* src, int dim, int rank) {
  using V = typename std::conditional<VEC == 4, uint4, typename std::conditional<VEC == 2, float2, float>::type>::type;
  const V* s = reinterpret_cast<const V*>(src);
  V* d = reinterpret_cast<V*>(dst);
  const int nv = dim / VEC;
  for (int e0 = rank; e0 < nv; e0 += G * U) {
    V v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int e = e0 + u * G;
      if (e < nv) v[u] = ld_vec(s + e);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int e = e0 + u * G;
      if (e < nv) st_vec(d + e, v[u]);
    }
  }
}

// Per-thread structural counters (TxnCounters) — 32-bit while a kernel runs,
// widened when flushed.
using ctr_t = unsigned int;

// Block-level flush of per-thread counters into the table counters.
template <int NT>
__device__ __forceinline__ void flush_counters(unsigned long long* dst, const ctr_t* c, int nc) {
  __shared__ unsigned long long sh[6];
  if (threadIdx.x < 6) sh[threadIdx.x] = 0;
  __syncthreads();
  for (int k = 0; k < nc; k++) {
    unsigned long long v = c[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&sh[k], v);
  }
  __syncthreads();
  if (threadIdx.x < nc && sh[threadIdx.x]) atomicAdd(&dst[threadIdx.x], sh[threadIdx.x]);
}

// An 8-lane sub-warp tile with raw warp intrinsics (cheaper than
// cooperative_groups' tiled_partition bookkeeping).  Lanes [8g, 8g+8).
struct Tile8 {
  unsigned lane, base, mask;
  __device__ __forceinline__ Tile8() {
    lane = threadIdx.x & 31u;
    base = lane & ~7u;
    mask = 0xFFu << base;
  }
  __device__ __forceinline__ int thread_rank() const { return (int)(lane & 7u); }
  __device__ __forceinline__ unsigned ballot(bool p) const { return (__ballot_sync(mask, p) >> base) & 0xFFu; }
  __device__ __forceinline__ bool any(bool p) const { return __any_sync(mask, p); }
  template <typename T>
  __device__ __forceinline__ T shfl(T v, int src) const { return __shfl_sync(mask, v, (int)base + src); }
  template <typename T>
  __device__ __forceinline__ T shfl_xor(T v, int o) const { return __shfl_xor_sync(mask, v, o); }
  template <typename T>
  __device__ __forceinline__ T shfl_up(T v, int d) const { return __shfl_up_sync(mask, v, d, 8); }
  __device__ __forceinline__ void sync() const { __syncwarp(mask); }
  __device__ __forceinline__ unsigned sum(unsigned v) const { return __reduce_add_sync(mask, v); }
};

// Barrier-free block accumulation of TxnCounters and the size delta: each
// warp adds its totals into shared memory, the last warp of the block
// publishes them with one global atomic per counter.
struct BlockCtrs {
  unsigned long long c[7];
  unsigned done;
};
__device__ __forceinline__ void block_ctrs_init(BlockCtrs& s) {
  if (threadIdx.x < 7) s.c[threadIdx.x] = 0;
  if (threadIdx.x == 0) s.done = 0;
  __syncthreads();
}
// c: 6 per-thread counters, sd: size delta; only tile rank-0 lanes carry
// tile totals, so every lane contributes and non-owners pass zeros.
__device__ __forceinline__ void block_ctrs_flush(BlockCtrs& s, unsigned long long* dst_ctr,
                                                 unsigned long long* dst_size, const ctr_t* c, long long sd) {
  const unsigned lane = threadIdx.x & 31u;
#pragma unroll
  for (int k = 0; k < 6; k++) {
    unsigned long long v = c[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && v) atomicAdd(&s.c[k], v);
  }
  long long v = sd;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0 && v) atomicAdd(&s.c[6], (unsigned long long)v);
  if (lane == 0) {
    __threadfence_block();
    const unsigned d = atomicAdd(&s.done, 1u);
    if (d == blockDim.x / 32 - 1) {
      __threadfence_block();
      for (int k = 0; k < 6; k++) {
        const unsigned long long x = *(volatile unsigned long long*)&s.c[k];
        if (x) atomicAdd(&dst_ctr[k], x);
      }
      const unsigned long long x = *(volatile unsigned long long*)&s.c[6];
      if (x && dst_size) atomicAdd(dst_size, x);
    }
  }
}

extern unsigned long long g_launches;  // host-side launch counter (hkv_api.cu)

// Programmatic dependent launch (PDL): pipeline kernels are launched with
// programmatic stream serialization, so a kernel's launch overlaps its
// predecessor's tail; it must not read the predecessor's output before this
// wait (a no-op for a normally launched kernel).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

#if defined(__CUDACC__)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}
#endif

}  // namespace hkv
