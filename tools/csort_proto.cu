// Prototype: stable counting sort of (bucket, op) pairs vs CUB onesweep radix
// sort, for the metadata pipeline's "group ops by bucket, batch order inside a
// bucket" step.  Checks both give identical (sbkt, sidx) and times them warm.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/csort tools/csort_proto.cu && /tmp/csort
#include <cub/cub.cuh>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

struct CsCtl {
  unsigned nsmall, nlarge, nhuge;
};

__global__ void k_count(const uint32_t* __restrict__ bkt, int64_t n, uint32_t* __restrict__ cnt,
                        uint32_t* __restrict__ rank) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool ok = i < n;
  const uint32_t b = ok ? bkt[i] : 0xFFFFFFFFu;
  const unsigned act = __ballot_sync(0xFFFFFFFFu, ok);
  if (!ok) return;
  const unsigned peers = __match_any_sync(act, b);
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(peers) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(cnt + b, (uint32_t)__popc(peers));
  base = __shfl_sync(peers, base, leader);
  rank[i] = base + __popc(peers & ((1u << lane) - 1));
}

// scatter + classify segments that need an in-segment order fix
__global__ void k_scatter(const uint32_t* __restrict__ bkt, const uint32_t* __restrict__ rank, int64_t n,
                          const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ off,
                          uint32_t* __restrict__ sbkt, uint32_t* __restrict__ sidx, uint32_t* __restrict__ small,
                          uint32_t* __restrict__ large, CsCtl* ctl) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t b = bkt[i];
  const uint32_t r = rank[i];
  const uint32_t o = off[b];
  sbkt[o + r] = b;
  sidx[o + r] = (uint32_t)i;
  if (r == 0) {
    const uint32_t L = cnt[b];
    if (L >= 2 && L <= 32) small[atomicAdd(&ctl->nsmall, 1u)] = b;
    else if (L > 32) large[atomicAdd(&ctl->nlarge, 1u)] = b;
  }
}

// 8-lane tiles: segments of 2..8; full warp: 9..32 (rank by count)
__global__ void k_fix_small(const uint32_t* __restrict__ list, const CsCtl* ctl, const uint32_t* __restrict__ cnt,
                            const uint32_t* __restrict__ off, uint32_t* __restrict__ sidx) {
  const unsigned nseg = ctl->nsmall;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp; w < nseg; w += nw) {
    const uint32_t b = list[w];
    const uint32_t L = cnt[b], o = off[b];
    const uint32_t v = lane < (int)L ? sidx[o + lane] : 0xFFFFFFFFu;
    uint32_t r = 0;
    for (uint32_t k = 0; k < L; k++) {
      const uint32_t x = __shfl_sync(0xFFFFFFFFu, v, (int)k);
      r += x < v;
    }
    if (lane < (int)L) sidx[o + r] = v;
  }
}

// block per segment; L <= kLargeMax by rank-by-count in smem, else bitmap windows
constexpr int kFixThreads = 1024;
constexpr int kLargeMax = 4096;
constexpr int kWinBits = 1 << 20;  // 128 KB bitmap window
__global__ void __launch_bounds__(kFixThreads) k_fix_large(const uint32_t* __restrict__ list, const CsCtl* ctl,
                                                           const uint32_t* __restrict__ cnt,
                                                           const uint32_t* __restrict__ off,
                                                           uint32_t* __restrict__ sidx, uint32_t* __restrict__ side, int64_t n) {
  extern __shared__ uint32_t sm[];
  typedef cub::BlockScan<uint32_t, kFixThreads> BS;
  __shared__ typename BS::TempStorage tmp;
  const unsigned nseg = ctl->nlarge;
  for (unsigned sgi = blockIdx.x; sgi < nseg; sgi += gridDim.x) {
    const uint32_t b = list[sgi];
    const uint32_t L = cnt[b], o = off[b];
    __syncthreads();
    if (L <= kLargeMax) {
      for (uint32_t j = threadIdx.x; j < L; j += blockDim.x) sm[j] = sidx[o + j];
      __syncthreads();
      for (uint32_t j = threadIdx.x; j < L; j += blockDim.x) {
        const uint32_t v = sm[j];
        uint32_t r = 0;
        for (uint32_t k = 0; k < L; k++) r += sm[k] < v;
        sidx[o + r] = v;
      }
    } else {
      // ops of one segment are distinct batch indices: set bits, enumerate in order
      uint32_t written = 0;
      for (int64_t lo = 0; lo < n; lo += kWinBits) {
        for (int j = threadIdx.x; j < kWinBits / 32; j += blockDim.x) sm[j] = 0;
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < L; j += blockDim.x) {
          const uint32_t v = sidx[o + j];
          if (v >= lo && v < lo + kWinBits) atomicOr(&sm[(v - lo) >> 5], 1u << ((v - lo) & 31));
        }
        __syncthreads();
        constexpr int per = kWinBits / 32 / kFixThreads;  // 32 words per thread
        uint32_t c = 0;
        for (int q = 0; q < per; q++) c += __popc(sm[threadIdx.x * per + q]);
        uint32_t before, total;
        BS(tmp).ExclusiveSum(c, before, total);
        __syncthreads();
        // stash into the tail of smem? enumerate directly: positions written + before ...
        uint32_t pos = written + before;
        for (int q = 0; q < per; q++) {
          uint32_t wv = sm[threadIdx.x * per + q];
          while (wv) {
            const int bit = __ffs(wv) - 1;
            wv &= wv - 1;
            side[o + pos++] = (uint32_t)(lo + (threadIdx.x * per + q) * 32 + bit);
          }
        }
        written += total;
        __syncthreads();
      }
      for (uint32_t j = threadIdx.x; j < L; j += blockDim.x) sidx[o + j] = side[o + j];
    }
  }
}

__global__ void k_spin(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}


// custom onesweep tuning: digit width and tile shape
template <int BITS, int THREADS, int ITEMS>
struct HubT {
  using KeyT = uint32_t;
  using DominantT = uint32_t;
  struct Policy1000 : cub::ChainedPolicy<1000, Policy1000, Policy1000> {
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = BITS;
    using HistogramPolicy = cub::AgentRadixSortHistogramPolicy<128, 16, 1, KeyT, ONESWEEP_RADIX_BITS>;
    using ExclusiveSumPolicy = cub::AgentRadixSortExclusiveSumPolicy<256, ONESWEEP_RADIX_BITS>;
    using OnesweepPolicy =
        cub::AgentRadixSortOnesweepPolicy<THREADS, ITEMS, DominantT, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                          cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT, BITS>;
    using ScanPolicy = cub::AgentScanPolicy<512, 23, int, cub::BLOCK_LOAD_WARP_TRANSPOSE, cub::LOAD_DEFAULT,
                                            cub::BLOCK_STORE_WARP_TRANSPOSE, cub::BLOCK_SCAN_RAKING_MEMOIZE>;
    using DownsweepPolicy = cub::AgentRadixSortDownsweepPolicy<512, 23, DominantT, cub::BLOCK_LOAD_TRANSPOSE,
                                                               cub::LOAD_DEFAULT, cub::RADIX_RANK_MATCH,
                                                               cub::BLOCK_SCAN_WARP_SCANS, 7>;
    using AltDownsweepPolicy = cub::AgentRadixSortDownsweepPolicy<256, 47, DominantT, cub::BLOCK_LOAD_TRANSPOSE,
                                                                  cub::LOAD_DEFAULT, cub::RADIX_RANK_MEMOIZE,
                                                                  cub::BLOCK_SCAN_WARP_SCANS, 6>;
    using UpsweepPolicy = cub::AgentRadixSortUpsweepPolicy<256, 23, DominantT, cub::LOAD_DEFAULT, 7>;
    using AltUpsweepPolicy = cub::AgentRadixSortUpsweepPolicy<256, 47, DominantT, cub::LOAD_DEFAULT, 6>;
    using SingleTilePolicy = cub::AgentRadixSortDownsweepPolicy<256, 19, DominantT, cub::BLOCK_LOAD_DIRECT,
                                                                cub::LOAD_LDG, cub::RADIX_RANK_MEMOIZE,
                                                                cub::BLOCK_SCAN_WARP_SCANS, 6>;
    using SegmentedPolicy = cub::AgentRadixSortDownsweepPolicy<192, 39, DominantT, cub::BLOCK_LOAD_TRANSPOSE,
                                                               cub::LOAD_DEFAULT, cub::RADIX_RANK_MEMOIZE,
                                                               cub::BLOCK_SCAN_WARP_SCANS, 6>;
    using AltSegmentedPolicy = cub::AgentRadixSortDownsweepPolicy<384, 11, DominantT, cub::BLOCK_LOAD_TRANSPOSE,
                                                                  cub::LOAD_DEFAULT, cub::RADIX_RANK_MEMOIZE,
                                                                  cub::BLOCK_SCAN_WARP_SCANS, 5>;
  };
  using MaxPolicy = Policy1000;
};

template <int BITS, int THREADS, int ITEMS>
static float time_hub(uint32_t* bkt, uint32_t* idx, uint32_t* k2, uint32_t* v2, int64_t n, int bits, void* tmp,
                      size_t tmp_cap, const std::vector<uint32_t>& ref_i, cudaEvent_t e0, cudaEvent_t e1) {
  using D = cub::DispatchRadixSort<false, uint32_t, uint32_t, int, HubT<BITS, THREADS, ITEMS>>;
  float tot = 0, ms;
  uint32_t *ok = nullptr, *ov = nullptr;
  for (int rep = 0; rep < 6; rep++) {
    cub::DoubleBuffer<uint32_t> dk(bkt, k2), dv(idx, v2);
    size_t bytes = 0;
    D::Dispatch(nullptr, bytes, dk, dv, (int)n, 0, bits, false, 0);
    if (bytes > tmp_cap) { printf("tmp too small\n"); return -1; }
    k_spin<<<1, 1>>>(400000);
    cudaEventRecord(e0);
    D::Dispatch(tmp, bytes, dk, dv, (int)n, 0, bits, false, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep) tot += ms / 5;
    ov = dv.Current();
  }
  CK(cudaGetLastError());
  std::vector<uint32_t> h(n);
  CK(cudaMemcpy(h.data(), ov, n * 4, cudaMemcpyDeviceToHost));
  int64_t bad = 0;
  for (int64_t i = 0; i < n; i++) bad += h[i] != ref_i[i];
  printf("   onesweep bits %2d threads %3d items %2d: %.1f us  mismatches %lld\n", BITS, THREADS, ITEMS, tot * 1e3,
         (long long)bad);
  return tot;
}

int main() {
  const int64_t n = 1 << 20;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *bkt, *idx, *sbkt, *sidx, *sbkt2, *sidx2, *cnt, *off, *rank, *small, *large;
  CsCtl* ctl;
  const int max_log2 = 23;
  CK(cudaMalloc(&bkt, n * 4)); CK(cudaMalloc(&idx, n * 4)); CK(cudaMalloc(&sbkt, n * 4)); CK(cudaMalloc(&sidx, n * 4));
  CK(cudaMalloc(&sbkt2, n * 4)); CK(cudaMalloc(&sidx2, n * 4)); CK(cudaMalloc(&rank, n * 4));
  CK(cudaMalloc(&cnt, (4ll << max_log2))); CK(cudaMalloc(&off, (4ll << max_log2)));
  CK(cudaMalloc(&small, n * 4)); CK(cudaMalloc(&large, n * 4)); CK(cudaMalloc(&ctl, sizeof(CsCtl)));
  size_t cub_bytes = 0, scan_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, bkt, sbkt, idx, sidx, (int)n, 0, 23);
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, cnt, off, 1 << max_log2);
  void* tmp;
  const size_t tmp_bytes = std::max(cub_bytes, scan_bytes) + (64 << 20);
  CK(cudaMalloc(&tmp, tmp_bytes));
  std::vector<uint32_t> hb(n), hi(n);
  for (int64_t i = 0; i < n; i++) hi[i] = (uint32_t)i;
  CK(cudaMemcpy(idx, hi.data(), n * 4, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEvent_t st[5];
  for (auto& q : st) cudaEventCreate(&q);
  const size_t fix_smem = kWinBits / 8 + 64;
  CK(cudaFuncSetAttribute(k_fix_large, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fix_smem));
  struct Case { const char* name; int log2b; int kind; };
  for (Case c : {Case{"uniform 2^20 buckets", 20, 0}, Case{"C1 8192 buckets", 13, 0}, Case{"zipf-ish 2^20", 20, 1},
                 Case{"uniform 2^23 buckets", 23, 0}}) {
    uint64_t x = 88172645463325252ull;
    const uint32_t mask = (1u << c.log2b) - 1;
    for (int64_t i = 0; i < n; i++) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      if (c.kind == 0) hb[i] = (uint32_t)(x & mask);
      else {  // heavy skew: 30% on 64 hot buckets
        const double u = (double)(x >> 11) / 9007199254740992.0;
        hb[i] = u < 0.3 ? (uint32_t)((x >> 3) % 64) * 7919u & mask : (uint32_t)(x & mask);
      }
    }
    CK(cudaMemcpy(bkt, hb.data(), n * 4, cudaMemcpyHostToDevice));
    const int64_t B = 1ll << c.log2b;
    auto run_cub = [&] {
      size_t bytes = cub_bytes;
      cub::DeviceRadixSort::SortPairs(tmp, bytes, bkt, sbkt, idx, sidx, (int)n, 0, c.log2b);
    };
    auto run_cs = [&] {
      cudaMemsetAsync(cnt, 0, B * 4);
      cudaMemsetAsync(ctl, 0, sizeof(CsCtl));
      cudaEventRecord(st[0]);
      k_count<<<(unsigned)((n + 255) / 256), 256>>>(bkt, n, cnt, rank);
      cudaEventRecord(st[1]);
      size_t bytes = scan_bytes;
      cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt, off, (int)B);
      cudaEventRecord(st[2]);
      k_scatter<<<(unsigned)((n + 255) / 256), 256>>>(bkt, rank, n, cnt, off, sbkt2, sidx2, small, large, ctl);
      cudaEventRecord(st[3]);
      k_fix_small<<<sms * 8, 256>>>(small, ctl, cnt, off, sidx2);
      cudaEventRecord(st[4]);
      k_fix_large<<<sms, kFixThreads, fix_smem>>>(large, ctl, cnt, off, sidx2, rank, n);
    };
    float t_cub = 0, t_cs = 0, ms;
    for (int rep = 0; rep < 6; rep++) {
      k_spin<<<1, 1>>>(400000);
      cudaEventRecord(e0); run_cub(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (rep >= 1) t_cub += ms / 5;
      k_spin<<<1, 1>>>(400000);
      cudaEventRecord(e0); run_cs(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); if (rep >= 1) t_cs += ms / 5;
      if (rep == 5) {
        float a;
        cudaEventElapsedTime(&a, e0, st[0]); printf("   memsets %.1f", a * 1e3);
        for (int q = 0; q < 4; q++) { cudaEventElapsedTime(&a, st[q], st[q + 1]); printf(" | stage%d %.1f", q, a * 1e3); }
        cudaEventElapsedTime(&a, st[4], e1); printf(" | large %.1f us\n", a * 1e3);
      }
    }
    CK(cudaGetLastError());
    std::vector<uint32_t> a1(n), a2(n), b1(n), b2(n);
    CK(cudaMemcpy(a1.data(), sidx, n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(a2.data(), sidx2, n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b1.data(), sbkt, n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b2.data(), sbkt2, n * 4, cudaMemcpyDeviceToHost));
    CsCtl hc;
    CK(cudaMemcpy(&hc, ctl, sizeof(hc), cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t i = 0; i < n; i++) bad += a1[i] != a2[i] || b1[i] != b2[i];
    {
      uint32_t *k2 = sbkt2, *v2 = rank;
      time_hub<8, 384, 23>(bkt, idx, k2, v2, n, c.log2b, tmp, tmp_bytes, a1, e0, e1);
      time_hub<8, 256, 16>(bkt, idx, k2, v2, n, c.log2b, tmp, tmp_bytes, a1, e0, e1);
      time_hub<8, 256, 8>(bkt, idx, k2, v2, n, c.log2b, tmp, tmp_bytes, a1, e0, e1);
      time_hub<10, 256, 8>(bkt, idx, k2, v2, n, c.log2b, tmp, tmp_bytes, a1, e0, e1);
      time_hub<10, 256, 16>(bkt, idx, k2, v2, n, c.log2b, tmp, tmp_bytes, a1, e0, e1);
      time_hub<10, 128, 16>(bkt, idx, k2, v2, n, c.log2b, tmp, tmp_bytes, a1, e0, e1);
      time_hub<7, 256, 16>(bkt, idx, k2, v2, n, c.log2b, tmp, tmp_bytes, a1, e0, e1);
      time_hub<9, 256, 16>(bkt, idx, k2, v2, n, c.log2b, tmp, tmp_bytes, a1, e0, e1);
    }
    printf("%-24s cub %.1f us  counting %.1f us  mismatches %lld  (small %u large %u)\n", c.name, t_cub * 1e3,
           t_cs * 1e3, (long long)bad, hc.nsmall, hc.nlarge);
  }
  return 0;
}
