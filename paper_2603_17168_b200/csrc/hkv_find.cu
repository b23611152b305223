// hkv_find.cu — reader kernels: find / contains / find_ptr.
//
// Restates table.py:304-351 (find, find_ptr, contains) and _vec_lookup
// table.py:284-300: hash (hashing.py:21-75) -> one 128-B digest-line read ->
// key compares on digest matches only -> value-row gather (store.py:115-123).
// Dual mode probes the second bucket only for first-bucket misses.
//
// find (dim % 4 == 0, 16-B aligned rows): k_find_fused — a thread per key
// reads the key's 128-B digest line (8 x 16 B in flight), tests it with an
// any-zero-byte check, builds the exact 128-bit candidate mask only when
// needed, checks candidate keys in slot order; then the warp moves its 32
// value rows with coalesced 16-B loads/stores, 8 in flight per lane.
// Otherwise (and for contains / find_ptr): k_find_tpk (the same probe,
// recording rows) + k_find_gather.
#include <cstdlib>
#include <string>

#include "hkv_probe.cuh"
#include "hkv_kernels.h"

namespace hkv {

// Gather pass: out[i] = value row of the hit (rows at random, output
// sequential), zero rows for misses when requested; KPT keys per tile and
// 2 vectors per lane per key in flight.
template <int VEC, int KPT, bool kZero>
__global__ void __launch_bounds__(256) k_find_gather(TableDev t, const uint32_t* __restrict__ rows, int64_t n,
                                                     float* __restrict__ out) {
  using V = typename std::conditional<VEC == 4, uint4, typename std::conditional<VEC == 2, float2, float>::type>::type;
  __shared__ BlockCtrs bc;
  block_ctrs_init(bc);
  const Tile8 tile;
  const int r = tile.thread_rank();
  const int64_t tid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ntiles = (int64_t)gridDim.x * blockDim.x / kG;
  const int dim = t.dim;
  const int nv = dim / VEC;
  ctr_t ctr[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t base = tid * KPT; base < n; base += ntiles * KPT) {
    uint32_t row[KPT];
#pragma unroll
    for (int u = 0; u < KPT; u++) {
      row[u] = (base + u < n) ? rows[base + u] : 0xFFFFFFFFu;
      if (r == 0 && row[u] != 0xFFFFFFFFu) ctr[row[u] < t.fast_rows ? kVFast : kVOver]++;
    }
    for (int e0 = r; e0 < nv; e0 += kG * 2) {
      V v[KPT][2];
#pragma unroll
      for (int u = 0; u < KPT; u++) {
        const V* src = reinterpret_cast<const V*>(row[u] != 0xFFFFFFFFu ? value_row(t, row[u]) : nullptr);
#pragma unroll
        for (int w = 0; w < 2; w++) {
          const int e = e0 + w * kG;
          if (e < nv) {
            if (row[u] != 0xFFFFFFFFu) v[u][w] = ld_vec(src + e);
            else v[u][w] = V{};
          }
        }
      }
#pragma unroll
      for (int u = 0; u < KPT; u++) {
        if (base + u >= n) continue;
        if (!kZero && row[u] == 0xFFFFFFFFu) continue;
        V* dst = reinterpret_cast<V*>(out + (uint64_t)(base + u) * dim);
#pragma unroll
        for (int w = 0; w < 2; w++) {
          const int e = e0 + w * kG;
          if (e < nv) st_vec(dst + e, v[u][w]);
        }
      }
    }
  }
  block_ctrs_flush(bc, t.counters, nullptr, ctr, 0);
}

template <int MODE>
__global__ void __launch_bounds__(256) k_find_tpk(TableDev t, const uint64_t* __restrict__ keys, int64_t n,
                                                  uint8_t* __restrict__ found, uint8_t* __restrict__ tier,
                                                  int64_t* __restrict__ offset, uint32_t* __restrict__ rows) {
  __shared__ BlockCtrs bc;
  block_ctrs_init(bc);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  ctr_t ctr[6] = {0, 0, 0, 0, 0, 0};
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t key = __ldg(keys + i);
    bad |= key >= kLockedKey;
    const uint64_t h = fmix64(key);
    const uint32_t d = digest_of(h);
    uint64_t b = h & t.mask;
    unsigned ncmp = 0;
    int slot = probe_line_thread(t, b, key, d, ncmp);
    ctr[kLoads]++;
    if (slot < 0 && t.dual) {  // second bucket only for first-bucket misses (table.py:291-298)
      b = second_hash(h) & t.mask;
      slot = probe_line_thread(t, b, key, d, ncmp);
      ctr[kLoads]++;
    }
    ctr[kCompares] += ncmp;
    const bool f = slot >= 0;
    const uint64_t row = b * kSlots + (uint64_t)(f ? slot : 0);
    found[i] = f;
    if constexpr (MODE == 4) rows[i] = f ? (uint32_t)row : 0xFFFFFFFFu;
    if constexpr (MODE == 2) {
      const bool over = row >= t.fast_rows;
      tier[i] = f ? (uint8_t)over : 0;
      offset[i] = !f ? -1 : (int64_t)((over ? row - t.fast_rows : row) * (uint64_t)t.dim);
    }
  }
  if (bad) atomicOr(t.err, 1);
  block_ctrs_flush(bc, t.counters, nullptr, ctr, 0);
}

// Fused find (dim % 4 == 0, 16-B aligned rows): each warp probes 32 keys
// (thread per key, as k_find_tpk), then moves the 32 value rows together:
// the warp's 32 x (dim/4) 16-B vectors are spread over the lanes, U loads in
// flight per lane before the matching stores (coalesced 16-B accesses on
// both sides).  Warps of a block are in different phases at any time, so
// probe latency overlaps other warps' value traffic without a second pass
// over the keys.
#ifndef HKV_FIND_U
#define HKV_FIND_U 8     // 16-B row vectors per lane in flight in the value gather
#endif
#ifndef HKV_FIND_BPS
#define HKV_FIND_BPS 8   // resident blocks per SM of the fused find (persistent grid)
#endif
template <bool kZero, int U>
__global__ void __launch_bounds__(256) k_find_fused(TableDev t, const uint64_t* __restrict__ keys, int64_t n,
                                                    uint8_t* __restrict__ found, float* __restrict__ out) {
  __shared__ BlockCtrs bc;
  block_ctrs_init(bc);
  const unsigned lane = threadIdx.x & 31u;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nv = t.dim >> 2;  // 16-B vectors per row
  ctr_t ctr[6] = {0, 0, 0, 0, 0, 0};
  int bad = 0;
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t i = base + lane;
    uint32_t row = 0xFFFFFFFFu;
    if (i < n) {
      const uint64_t key = __ldg(keys + i);
      bad |= key >= kLockedKey;
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
      found[i] = slot >= 0;
      if (slot >= 0) {
        row = (uint32_t)(b * kSlots + slot);
        ctr[row < t.fast_rows ? kVFast : kVOver]++;
      }
    }
    // value rows of the warp's 32 keys
    const int nk = (n - base < 32) ? (int)(n - base) : 32;
    const int total = nk * nv;
    for (int v0 = 0; v0 < total; v0 += 32 * U) {  // warp-uniform trip count: every lane reaches the shuffles
      uint4 x[U];
      uint32_t rr[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int v = v0 + 32 * u + (int)lane;
        const int k = v < total ? v / nv : 0;
        rr[u] = __shfl_sync(0xffffffffu, row, k);
        if (v < total && rr[u] != 0xFFFFFFFFu) x[u] = ld_stream(reinterpret_cast<const uint4*>(value_row(t, rr[u])) + (v - k * nv));
        else x[u] = make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int v = v0 + 32 * u + (int)lane;
        if (v >= total || (!kZero && rr[u] == 0xFFFFFFFFu)) continue;
        const int k = v / nv;
        st_stream(reinterpret_cast<uint4*>(out + (base + k) * (int64_t)t.dim) + (v - k * nv), x[u]);
      }
    }
  }
  if (bad) atomicOr(t.err, 1);
  block_ctrs_flush(bc, t.counters, nullptr, ctr, 0);
}

// Sharded find over peer memory: each thread hashes its key,
// finds the owner shard from the global bucket, probes the owner's digest
// line and candidate keys in place (NVLink loads for a remote owner), and the
// warp then copies its 32 rows out of the owners' value arenas, as
// k_find_fused does locally.  Replaces route -> all-to-all -> local find ->
// all-to-all; results are bit-identical to the routed path (the shard's
// bucket is the global table's bucket).  Structural counters are not updated
// (they belong to the owner shard).
template <bool kZero, int VEC>
__global__ void __launch_bounds__(256) k_find_peer(const PeerView* __restrict__ views, uint64_t gmask, int llog2b,
                                                   int dim, const uint64_t* __restrict__ keys, int64_t n,
                                                   uint8_t* __restrict__ found, float* __restrict__ out, int* err) {
  using V = typename std::conditional<VEC == 4, uint4, float>::type;
  const unsigned lane = threadIdx.x & 31u;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nv = dim / VEC;
  const uint64_t lmask = (1ull << llog2b) - 1;
  int bad = 0;
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t i = base + lane;
    const float* src = nullptr;
    if (i < n) {
      const uint64_t key = __ldg(keys + i);
      bad |= key >= kLockedKey;
      const uint64_t h = fmix64(key);
      const uint32_t d = digest_of(h);
      const uint64_t gb = h & gmask;
      const PeerView v = views[gb >> llog2b];
      const uint64_t rowbase = (gb & lmask) * kSlots;
      const uint4* dp = reinterpret_cast<const uint4*>(v.digests + rowbase);
      uint4 w[8];
#pragma unroll
      for (int k = 0; k < 8; k++) w[k] = dp[k];
      int hit = -1;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        uint32_t m = hit < 0 ? (match16(w[2 * q], d) | (match16(w[2 * q + 1], d) << 16)) : 0u;
        while (m) {
          const int j = __ffs(m) - 1;
          m &= m - 1;
          const uint64_t k2 = v.ks[2 * (rowbase + 32 * q + j)];
          if (k2 == key) {
            hit = 32 * q + j;
            m = 0;
          }
        }
      }
      found[i] = hit >= 0;
      if (hit >= 0) src = v.values + (rowbase + hit) * (uint64_t)dim;
    }
    const int nk = (n - base < 32) ? (int)(n - base) : 32;
    const int total = nk * nv;
    for (int v0 = 0; v0 < total; v0 += 32 * 8) {
      V x[8];
      const float* rs[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int e = v0 + 32 * u + (int)lane;
        const int k = e < total ? e / nv : 0;
        rs[u] = reinterpret_cast<const float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(src), k));
        if (e < total && rs[u]) x[u] = reinterpret_cast<const V*>(rs[u])[e - k * nv];
        else x[u] = V{};
      }
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int e = v0 + 32 * u + (int)lane;
        if (e >= total || (!kZero && !rs[u])) continue;
        const int k = e / nv;
        reinterpret_cast<V*>(out + (base + k) * (int64_t)dim)[e - k * nv] = x[u];
      }
    }
  }
  if (bad) atomicOr(err, 1);
}

void launch_find_peer(const PeerView* views, uint64_t gmask, int llog2b, int dim, const uint64_t* keys, int64_t n,
                      float* out, uint8_t* found, int zero_misses, int* err, cudaStream_t s, int num_sms) {
  if (n <= 0) return;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
  const bool v4 = dim % 4 == 0 && ((uintptr_t)out & 15) == 0;
  if (v4) {
    if (zero_misses) k_find_peer<true, 4><<<(unsigned)blocks, 256, 0, s>>>(views, gmask, llog2b, dim, keys, n, found, out, err);
    else k_find_peer<false, 4><<<(unsigned)blocks, 256, 0, s>>>(views, gmask, llog2b, dim, keys, n, found, out, err);
  } else {
    if (zero_misses) k_find_peer<true, 1><<<(unsigned)blocks, 256, 0, s>>>(views, gmask, llog2b, dim, keys, n, found, out, err);
    else k_find_peer<false, 1><<<(unsigned)blocks, 256, 0, s>>>(views, gmask, llog2b, dim, keys, n, found, out, err);
  }
  g_launches++;
}

template <int MODE>
static void launch_probe(const TableDev& t, const uint64_t* keys, int64_t n, uint8_t* found, uint8_t* tier,
                         int64_t* offset, uint32_t* rows, cudaStream_t s, int num_sms) {
  int64_t blocks = (n + 255) / 256;
  const int64_t max_blocks = (int64_t)num_sms * 8;
  if (blocks > max_blocks) blocks = max_blocks;
  if (blocks < 1) blocks = 1;
  k_find_tpk<MODE><<<(unsigned)blocks, 256, 0, s>>>(t, keys, n, found, tier, offset, rows);
  g_launches++;
}

void launch_find(const TableDev& t, const uint64_t* keys, int64_t n, float* out, uint8_t* found, uint8_t* tier,
                 int64_t* offset, int mode, uint32_t* rows, cudaStream_t s, int num_sms) {
  if (n <= 0) return;
  ktimer_begin("find", s);
  if (mode == 1) {
    launch_probe<1>(t, keys, n, found, nullptr, nullptr, nullptr, s, num_sms);
  } else if (mode == 2) {
    launch_probe<2>(t, keys, n, found, tier, offset, nullptr, s, num_sms);
  } else if ((t.dim % 4) == 0 && (((uintptr_t)out & 15) == 0) && (((uintptr_t)t.vfast & 15) == 0) &&
             (((uintptr_t)t.vover & 15) == 0) && !(getenv("HKV_FIND") && std::string(getenv("HKV_FIND")) != "fused")) {
    int64_t blocks = (n + 255) / 256;
    const int64_t max_blocks = (int64_t)num_sms * HKV_FIND_BPS;
    if (blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) blocks = 1;
    if (mode == 3) k_find_fused<true, HKV_FIND_U><<<(unsigned)blocks, 256, 0, s>>>(t, keys, n, found, out);
    else k_find_fused<false, HKV_FIND_U><<<(unsigned)blocks, 256, 0, s>>>(t, keys, n, found, out);
    g_launches++;
  } else {
    launch_probe<4>(t, keys, n, found, nullptr, nullptr, rows, s, num_sms);
    ktimer_end("find", s);
    ktimer_begin("find_gather", s);
    const bool al4 = (t.dim % 4 == 0) && (((uintptr_t)out & 15) == 0) && (((uintptr_t)t.vfast & 15) == 0) &&
                     (((uintptr_t)t.vover & 15) == 0);
    const bool al2 = (t.dim % 2 == 0) && (((uintptr_t)out & 7) == 0) && (((uintptr_t)t.vfast & 7) == 0) &&
                     (((uintptr_t)t.vover & 7) == 0);
    int64_t blocks = (((n + 3) / 4) * kG + 255) / 256;
    const int64_t cap = (int64_t)num_sms * 8 * 4;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    const bool z = mode == 3;
    if (al4) {
      if (z) k_find_gather<4, 4, true><<<(unsigned)blocks, 256, 0, s>>>(t, rows, n, out);
      else k_find_gather<4, 4, false><<<(unsigned)blocks, 256, 0, s>>>(t, rows, n, out);
    } else if (al2) {
      if (z) k_find_gather<2, 4, true><<<(unsigned)blocks, 256, 0, s>>>(t, rows, n, out);
      else k_find_gather<2, 4, false><<<(unsigned)blocks, 256, 0, s>>>(t, rows, n, out);
    } else {
      if (z) k_find_gather<1, 4, true><<<(unsigned)blocks, 256, 0, s>>>(t, rows, n, out);
      else k_find_gather<1, 4, false><<<(unsigned)blocks, 256, 0, s>>>(t, rows, n, out);
    }
    g_launches++;
    ktimer_end("find_gather", s);
    return;
  }
  ktimer_end("find", s);
}

}  // namespace hkv
