// hkv_find.cu — reader kernels: find / contains / find_ptr.
//
// Restates table.py:304-351 (find, find_ptr, contains) and _vec_lookup
// table.py:284-300: hash (hashing.py:21-75) -> one 128-B digest-line read ->
// key compares on digest matches only -> value-row gather (store.py:115-123).
// Dual mode probes the second bucket only for first-bucket misses.
//
// One tile of 8 lanes per key: the digest line is read as 8 x 16 B (one
// coalesced 128-B transaction), the value row is moved 16 B per lane.  Each
// tile keeps kKPT keys in flight (software pipelined: all keys' digest
// lines are requested before any is consumed, then all candidate keys, then
// all value rows) to raise memory-level parallelism on the dependent chain
// key -> digest line -> key -> value.
#include "hkv_probe.cuh"
#include "hkv_kernels.h"

namespace hkv {

template <int VEC, int MODE, int KPT>
__global__ void __launch_bounds__(256) k_find(TableDev t, const uint64_t* __restrict__ keys, int64_t n,
                                              float* __restrict__ out, uint8_t* __restrict__ found,
                                              uint8_t* __restrict__ tier, int64_t* __restrict__ offset) {
  auto tile = cg::tiled_partition<kG>(cg::this_thread_block());
  const int r = tile.thread_rank();
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / kG;
  unsigned long long ctr[6] = {0, 0, 0, 0, 0, 0};
  const int dim = t.dim;
  int bad = 0;

  for (int64_t base = gid * KPT; base < n; base += ngroups * KPT) {
    uint64_t key[KPT], h[KPT], b[KPT];
    uint4 dl[KPT];
    bool live[KPT];
#pragma unroll
    for (int u = 0; u < KPT; u++) {
      const int64_t i = base + u;
      live[u] = i < n;
      key[u] = live[u] ? __ldg(keys + i) : 0;
      if (key[u] >= kLockedKey) { bad = 1; }
      h[u] = fmix64(key[u]);
      b[u] = h[u] & t.mask;
    }
    // stage 1: all digest lines in flight
#pragma unroll
    for (int u = 0; u < KPT; u++) {
      if (live[u] && t.digest_filter)
        dl[u] = __ldg(reinterpret_cast<const uint4*>(t.digests + b[u] * kSlots) + r);
      else
        dl[u] = make_uint4(0, 0, 0, 0);
    }
    // stage 2: candidate keys (usually 0-1 per key)
    int slot[KPT];
#pragma unroll
    for (int u = 0; u < KPT; u++) {
      uint32_t cand = !live[u] ? 0u : (t.digest_filter ? match16(dl[u], digest_of(h[u])) : 0xFFFFu);
      const uint64_t* kp = t.keys + b[u] * kSlots + r * kSPL;
      int hit = -1, ncmp = 0, ncmp_all = 0;
      while (cand) {
        const int j = __ffs(cand) - 1;
        cand &= cand - 1;
        const uint64_t k = __ldg(kp + j);
        if (k == kEmptyKey) continue;
        ncmp_all++;
        if (k == key[u]) { hit = r * kSPL + j; ncmp = ncmp_all; break; }
      }
      const uint32_t hm = tile.ballot(hit >= 0);
      int contrib = ncmp_all;
      slot[u] = -1;
      if (hm) {
        const int hl = __ffs(hm) - 1;
        slot[u] = tile.shfl(hit, hl);
        contrib = r < hl ? ncmp_all : (r == hl ? ncmp : 0);
      }
      ctr[kCompares] += tile_sum<kG>(tile, contrib);
      ctr[kLoads] += live[u];
    }
    if (t.dual) {
      // second bucket for first-bucket misses (table.py:291-298)
#pragma unroll
      for (int u = 0; u < KPT; u++) {
        if (!live[u] || slot[u] >= 0) continue;
        b[u] = second_hash(h[u]) & t.mask;
        slot[u] = probe_bucket<false, true>(t, tile, b[u], key[u], digest_of(h[u]), 0xFFFFu, ctr[kCompares]);
        ctr[kLoads]++;
      }
    }
    // stage 3: outputs
#pragma unroll
    for (int u = 0; u < KPT; u++) {
      if (!live[u]) continue;
      const int64_t i = base + u;
      const bool f = slot[u] >= 0;
      const uint64_t row = b[u] * kSlots + (uint64_t)(f ? slot[u] : 0);
      if constexpr (MODE == 0) {
        if (f) {
          copy_row<kG, VEC>(out + i * (int64_t)dim, value_row(t, row), dim, r);
          ctr[row < t.fast_rows ? kVFast : kVOver]++;
        }
      }
      if (r == 0) {
        found[i] = f;
        if constexpr (MODE == 2) {
          const bool over = row >= t.fast_rows;
          tier[i] = f ? (uint8_t)over : 0;
          offset[i] = !f ? -1 : (int64_t)((over ? row - t.fast_rows : row) * (uint64_t)dim);
        }
      }
    }
  }
  if (bad) atomicOr(t.err, 1);
  // counters: only rank-0 lanes carry tile totals (avoid 8x counting)
  if (r != 0) {
#pragma unroll
    for (int k = 0; k < 6; k++) ctr[k] = 0;
  }
  flush_counters<256>(t.counters, ctr, 6);
}

template <int MODE>
static void launch_find_mode(const TableDev& t, const uint64_t* keys, int64_t n, float* out, uint8_t* found,
                             uint8_t* tier, int64_t* offset, cudaStream_t s, int num_sms) {
  constexpr int KPT = 2;
  const int threads = 256;
  int64_t groups = (n + KPT - 1) / KPT;
  int64_t blocks = (groups * kG + threads - 1) / threads;
  const int64_t max_blocks = (int64_t)num_sms * 8 * 4;  // 8 resident x 4 waves
  if (blocks > max_blocks) blocks = max_blocks;
  if (blocks < 1) blocks = 1;
  const bool al4 = (t.dim % 4 == 0) && (((uintptr_t)out & 15) == 0) && (((uintptr_t)t.vfast & 15) == 0) &&
                   (((uintptr_t)t.vover & 15) == 0);
  const bool al2 = (t.dim % 2 == 0) && (((uintptr_t)out & 7) == 0);
  if (MODE != 0 || al4)
    k_find<4, MODE, KPT><<<blocks, threads, 0, s>>>(t, keys, n, out, found, tier, offset);
  else if (al2)
    k_find<2, MODE, KPT><<<blocks, threads, 0, s>>>(t, keys, n, out, found, tier, offset);
  else
    k_find<1, MODE, KPT><<<blocks, threads, 0, s>>>(t, keys, n, out, found, tier, offset);
  g_launches++;
}

void launch_find(const TableDev& t, const uint64_t* keys, int64_t n, float* out, uint8_t* found,
                 uint8_t* tier, int64_t* offset, int mode, cudaStream_t s, int num_sms) {
  if (n <= 0) return;
  ktimer_begin("find", s);
  if (mode == 0) launch_find_mode<0>(t, keys, n, out, found, tier, offset, s, num_sms);
  else if (mode == 1) launch_find_mode<1>(t, keys, n, out, found, tier, offset, s, num_sms);
  else launch_find_mode<2>(t, keys, n, out, found, tier, offset, s, num_sms);
  ktimer_end("find", s);
}

}  // namespace hkv
