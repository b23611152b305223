// hkv_misc.cu — export_batch_if, state import support, consistency scan and
// the sharding router.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "hkv_kernels.h"
#include "hkv_probe.cuh"

namespace hkv {

// ---------------------------------------------------------------------------
// export_batch_if (table.py:374-434): ordered stream compaction of rows
// [cursor, capacity) keeping user keys (key < LOCKED) that pass the predicate.
// ---------------------------------------------------------------------------
struct ExportFlag {
  const uint64_t* ks;  // (key, score) pairs
  const uint8_t* mask;
  int64_t base;  // first row of this chunk
  int64_t mask_base;
  int has_min;
  uint64_t min_score;
  __host__ __device__ bool operator()(const int64_t& j) const {
    const int64_t r = base + j;
    if (ks[2 * r] >= kLockedKey) return false;
    if (has_min && ks[2 * r + 1] < min_score) return false;
    if (mask && !mask[r - mask_base]) return false;
    return true;
  }
};

template <int VEC>
__global__ void k_export_gather(TableDev t, const uint32_t* __restrict__ list, int64_t base, int64_t take,
                                uint64_t* ok, float* ov, uint64_t* os) {
  const Tile8 tile;
  const int r = tile.thread_rank();
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / kG;
  ctr_t ctr[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t j = gid; j < take; j += ngroups) {
    const uint64_t row = (uint64_t)(base + list[j]);
    if (r == 0) {
      ok[j] = *kptr(t, row);
      os[j] = *sptr(t, row);
      ctr[row < t.fast_rows ? kVFast : kVOver]++;
    }
    copy_row<kG, VEC>(ov + j * (int64_t)t.dim, value_row(t, row), t.dim, r);
  }
  flush_counters<256>(t.counters, ctr, 6);
}

cudaError_t run_export(const TableDev& t, int64_t cursor, int64_t max_count, int has_min, uint64_t min_score,
                       const uint8_t* mask, int64_t mask_rows, uint64_t* ok, float* ov, uint64_t* os,
                       int64_t* count, int64_t* next, Workspace& ws, cudaStream_t s, int num_sms) {
  const int64_t kChunk = 1 << 22;
  cudaError_t e;
  if ((e = ws_reserve(ws, kChunk, t.dim, 0, false))) return e;
  const int64_t end = mask ? cursor + mask_rows : (int64_t)t.capacity;
  int64_t taken = 0;
  *next = -1;
  int64_t pos = cursor;
  long long* nsel = &ws.sc->n_sel;
  while (pos < end && taken < max_count) {
    const int64_t len = (end - pos) < kChunk ? (end - pos) : kChunk;
    thrust::counting_iterator<int64_t> cnt(0);
    ExportFlag f{t.ks, mask, pos, cursor, has_min, min_score};
    thrust::transform_iterator<ExportFlag, thrust::counting_iterator<int64_t>, bool> fl(cnt, f);
    size_t bytes = ws.cub_bytes;
    if ((e = cub::DeviceSelect::Flagged(ws.cub_tmp, bytes, cnt, fl, ws.aux, nsel, (int)len, s))) return e;
    g_launches += 2;
    long long c = 0;
    if ((e = cudaMemcpyAsync(&c, nsel, sizeof(c), cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    const int64_t take = (c < max_count - taken) ? c : (max_count - taken);
    if (take > 0) {
      const bool al4 = t.dim % 4 == 0 && (((uintptr_t)ov & 15) == 0);
      int64_t blocks = (take * kG + 255) / 256;
      if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
      if (al4)
        k_export_gather<4><<<(unsigned)blocks, 256, 0, s>>>(t, ws.aux, pos, take, ok + taken, ov + taken * t.dim,
                                                            os + taken);
      else
        k_export_gather<1><<<(unsigned)blocks, 256, 0, s>>>(t, ws.aux, pos, take, ok + taken, ov + taken * t.dim,
                                                            os + taken);
      g_launches++;
      taken += take;
      if (taken >= max_count) {
        uint32_t last = 0;
        if ((e = cudaMemcpyAsync(&last, ws.aux + (take - 1), sizeof(last), cudaMemcpyDeviceToHost, s))) return e;
        if ((e = cudaStreamSynchronize(s))) return e;
        const int64_t nx = pos + (int64_t)last + 1;
        *next = nx < (int64_t)t.capacity ? nx : -1;
      }
    }
    pos += len;
  }
  *count = taken;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// occupancy bitmap + size from keys (state import), consistency scan
// (check_consistency, table.py:1284-1299)
// ---------------------------------------------------------------------------
__global__ void k_bits_from_keys(TableDev t, int64_t buckets) {
  const Tile8 tile;
  const int r = tile.thread_rank();
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / kG;
  long long cnt = 0;
  for (int64_t b = gid; b < buckets; b += ngroups) {
    const uint64_t* kp = kptr(t, b * kSlots + r * kSPL);
    uint32_t occ = 0;
#pragma unroll
    for (int j = 0; j < kSPL; j++) occ |= (kp[2 * j] < kLockedKey ? 1u : 0u) << j;
    store_occ(t, b, r, occ);
    cnt += __popc(occ);
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(t.size, (unsigned long long)cnt);
}

cudaError_t run_bits_from_keys(const TableDev& t, int64_t buckets, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(t.size, 0, sizeof(unsigned long long), s);
  if (e) return e;
  int64_t blocks = (buckets * kG + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  k_bits_from_keys<<<(unsigned)blocks, 256, 0, s>>>(t, buckets);
  g_launches++;
  return cudaGetLastError();
}

// ok_dev[0] = 1 if consistent; ok_dev[1..2] = user-key total (int64 split)
__global__ void k_consistency(TableDev t, int64_t buckets, int* ok_dev, unsigned long long* total) {
  const Tile8 tile;
  const int r = tile.thread_rank();
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG;
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / kG;
  long long cnt = 0;
  int bad = 0;
  for (int64_t b = gid; b < buckets; b += ngroups) {
    const uint64_t* kp = kptr(t, b * kSlots + r * kSPL);
    const uint8_t* dp = t.digests + b * kSlots + r * kSPL;
    uint32_t occ = 0;
    for (int j = 0; j < kSPL; j++) {
      const uint64_t k = kp[2 * j];
      if (k < kLockedKey) {
        occ |= 1u << j;
        if (digest_of(fmix64(k)) != dp[j]) bad = 1;
      } else if (k == kLockedKey) {
        bad = 1;  // no slot may rest LOCKED
      }
    }
    if (occ != load_occ(t, b, r)) bad = 1;
    // eviction summary of a full bucket: a group marked exact holds its minimum
    if (tile.sum((unsigned)__popc(occ)) == kSlots && ((t.svalid[b] >> r) & 1u)) {
      uint64_t gm = kMaxScore;
      for (int j = 0; j < kSPL; j++) gm = kp[2 * j + 1] < gm ? kp[2 * j + 1] : gm;
      const uint64_t sm = t.smin[b * 8 + r];
      if (sm != gm) bad = 1;
    }
    cnt += __popc(occ);
  }
  if (bad) atomicExch(ok_dev, 0);
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(total, (unsigned long long)cnt);
}

cudaError_t run_consistency(const TableDev& t, int64_t buckets, int* ok_dev, cudaStream_t s) {
  int64_t blocks = (buckets * kG + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  k_consistency<<<(unsigned)blocks, 256, 0, s>>>(t, buckets, ok_dev,
                                                 reinterpret_cast<unsigned long long*>(ok_dev + 2));
  g_launches++;
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Sharding router: destination rank of each key's global
// bucket, stable grouping by destination (batch order kept inside a rank).
// ---------------------------------------------------------------------------
__global__ void k_route_dest(const uint64_t* __restrict__ keys, int64_t n, uint64_t gmask, int shift,
                             uint32_t* dest, uint32_t* idx, unsigned long long* counts, int world) {
  __shared__ unsigned hist[64];
  if (threadIdx.x < 64) hist[threadIdx.x] = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const uint32_t d = (uint32_t)((fmix64(keys[i]) & gmask) >> shift);
    dest[i] = d;
    idx[i] = (uint32_t)i;
    atomicAdd(&hist[d], 1u);
  }
  __syncthreads();
  if (threadIdx.x < world && hist[threadIdx.x]) atomicAdd(&counts[threadIdx.x], (unsigned long long)hist[threadIdx.x]);
}

cudaError_t run_route(const uint64_t* keys, int64_t n, int64_t global_buckets, int world, int32_t* perm,
                      int64_t* counts, Workspace& ws, cudaStream_t s) {
  cudaError_t e;
  if ((e = ws_reserve(ws, n, 1, 0, false))) return e;
  if ((e = cudaMemsetAsync(counts, 0, sizeof(int64_t) * world, s))) return e;
  if (n <= 0) return cudaSuccess;
  int shift = 0;
  int64_t local = global_buckets / world;
  while ((1ll << shift) < local) shift++;
  int bits = 0;
  while ((1 << bits) < world) bits++;
  k_route_dest<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(keys, n, (uint64_t)(global_buckets - 1), shift, ws.bkt,
                                                           ws.idx, reinterpret_cast<unsigned long long*>(counts),
                                                           world);
  g_launches++;
  size_t bytes = ws.cub_bytes;
  if ((e = cub::DeviceRadixSort::SortPairs(ws.cub_tmp, bytes, ws.bkt, ws.sbkt, ws.idx,
                                           reinterpret_cast<uint32_t*>(perm), (int)n, 0, bits < 1 ? 1 : bits, s)))
    return e;
  g_launches += 2;
  return cudaGetLastError();
}

}  // namespace hkv

namespace hkv {

// ---- routed exchange helpers of the sharded table (sharded.py) -----------
// k_route_gather: the routed order's send columns in one pass -- per op j
// (source index i = perm[j]): meta[j] = (key, tick = tick_base + i + 1
// [, score]) and the value row; rows are moved by 8-lane tiles with 16-B
// vectors (coalesced writes, one random row read per op).
template <int VEC>
__global__ void __launch_bounds__(256) k_route_gather(const int32_t* __restrict__ perm, int64_t n,
                                                      const uint64_t* __restrict__ keys,
                                                      const uint64_t* __restrict__ scores,
                                                      const float* __restrict__ values, int dim,
                                                      uint64_t tick_base, int meta_w, uint64_t* __restrict__ meta,
                                                      float* __restrict__ out_values) {
  const int r = threadIdx.x & 7;
  const int64_t tiles = (int64_t)gridDim.x * (blockDim.x / 8);
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x / 8) + threadIdx.x / 8; j < n; j += tiles) {
    const int64_t i = perm[j];
    if (r == 0) {
      meta[j * meta_w] = keys[i];
      meta[j * meta_w + 1] = tick_base + (uint64_t)i + 1;
      if (meta_w > 2) meta[j * meta_w + 2] = scores[i];
    }
    if (values) copy_row<8, VEC>(out_values + (uint64_t)j * dim, values + (uint64_t)i * dim, dim, r);
  }
}

// k_scatter_rows: dst[perm[j]] = src[j] for rows of `row_bytes` (a multiple
// of 4): the inverse routing permutation of returned results.
__global__ void __launch_bounds__(256) k_scatter_rows(const int32_t* __restrict__ perm, int64_t n,
                                                      const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                                      int words) {
  const int64_t total = n * words;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = x / words;
    const int w = (int)(x - j * words);
    dst[(int64_t)perm[j] * words + w] = src[x];
  }
}
__global__ void __launch_bounds__(256) k_scatter_bytes(const int32_t* __restrict__ perm, int64_t n,
                                                       const uint8_t* __restrict__ src, uint8_t* __restrict__ dst) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    dst[perm[j]] = src[j];
}

}  // namespace hkv

extern "C" int hkv_route_gather(const int32_t* perm, int64_t n, const uint64_t* keys, const uint64_t* scores,
                                const float* values, int64_t dim, uint64_t tick_base, uint64_t* meta,
                                float* out_values, void* stream) {
  using namespace hkv;
  if (n < 0 || dim < 1) return 1;
  if (n == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const int meta_w = scores ? 3 : 2;
  const bool v4 = dim % 4 == 0 && ((uintptr_t)values % 16 == 0) && ((uintptr_t)out_values % 16 == 0);
  int64_t blocks = (n * 8 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (v4)
    k_route_gather<4><<<(unsigned)blocks, 256, 0, s>>>(perm, n, keys, scores, values, (int)dim, tick_base, meta_w,
                                                       meta, out_values);
  else
    k_route_gather<1><<<(unsigned)blocks, 256, 0, s>>>(perm, n, keys, scores, values, (int)dim, tick_base, meta_w,
                                                       meta, out_values);
  g_launches++;
  return cudaGetLastError() ? 2 : 0;
}

extern "C" int hkv_scatter_rows(const int32_t* perm, int64_t n, const void* src, void* dst, int64_t row_bytes,
                                void* stream) {
  using namespace hkv;
  if (n < 0 || row_bytes < 1 || (row_bytes != 1 && row_bytes % 4)) return 1;
  if (n == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (row_bytes == 1) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_scatter_bytes<<<(unsigned)blocks, 256, 0, s>>>(perm, n, (const uint8_t*)src, (uint8_t*)dst);
  } else {
    const int words = (int)(row_bytes / 4);
    int64_t blocks = (n * words + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    k_scatter_rows<<<(unsigned)blocks, 256, 0, s>>>(perm, n, (const uint32_t*)src, (uint32_t*)dst, words);
  }
  g_launches++;
  return cudaGetLastError() ? 2 : 0;
}
