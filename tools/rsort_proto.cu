// Prototype: LSD radix sort of a batch by bucket (reduce-then-scan, no
// decoupled look-back chain), hashing fused into the first pass and the key
// carried along, vs k_prep + CUB onesweep SortPairs.  Checks identical output.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rsort tools/rsort_proto.cu && /tmp/rsort
#include <cub/cub.cuh>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ uint64_t fmix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xFF51AFD7ED558CCDull;
  x ^= x >> 33;
  x *= 0xC4CEB9FE1A85EC53ull;
  x ^= x >> 33;
  return x;
}

__global__ void k_spin(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}

__global__ void k_prep(const uint64_t* __restrict__ keys, int64_t n, uint64_t mask, uint32_t* bkt, uint32_t* idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bkt[i] = (uint32_t)(fmix64(keys[i]) & mask);
  idx[i] = (uint32_t)i;
}

constexpr int kThreads = 512, kWarps = kThreads / 32, kItems = 8, kTile = kThreads * kItems;

// Load the warp-blocked items of a tile: warp w owns positions [w*256, w*256+256)
// of the tile, round r covers 32 consecutive positions.
template <bool FIRST>
__device__ __forceinline__ void load_items(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ bin,
                                           const uint32_t* __restrict__ iin, const uint64_t* __restrict__ kin,
                                           int64_t n, uint64_t mask, int64_t base, uint32_t (&b)[kItems],
                                           uint32_t (&ix)[kItems], uint64_t (&k)[kItems]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < kItems; r++) {
    const int64_t p = base + w * 32 * kItems + r * 32 + lane;
    if (p < n) {
      if (FIRST) {
        k[r] = keys[p];
        b[r] = (uint32_t)(fmix64(k[r]) & mask);
        ix[r] = (uint32_t)p;
      } else {
        k[r] = kin[p];
        b[r] = bin[p];
        ix[r] = iin[p];
      }
    }
  }
}

template <bool FIRST, int D>
__global__ void __launch_bounds__(kThreads) k_hist(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ bin,
                                                   int64_t n, uint64_t mask, int shift, uint32_t* __restrict__ hist,
                                                   int64_t ntiles) {
  constexpr int R = 1 << D;
  __shared__ uint32_t h[R];
  for (int d = threadIdx.x; d < R; d += kThreads) h[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile;
  for (int j = threadIdx.x; j < kTile; j += kThreads) {
    const int64_t p = base + j;
    if (p < n) {
      const uint32_t b = FIRST ? (uint32_t)(fmix64(keys[p]) & mask) : bin[p];
      atomicAdd(&h[(b >> shift) & (R - 1)], 1u);
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < R; d += kThreads) hist[(int64_t)d * ntiles + blockIdx.x] = h[d];
}

// single-block exclusive scan (in place) over m entries
__global__ void __launch_bounds__(1024) k_scan(uint32_t* __restrict__ a, int64_t m) {
  typedef cub::BlockScan<uint32_t, 1024> BS;
  __shared__ typename BS::TempStorage tmp;
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  constexpr int P = 16;
  for (int64_t base = 0; base < m; base += 1024 * P) {
    uint32_t v[P];
    uint32_t s = 0;
#pragma unroll
    for (int q = 0; q < P; q++) {
      const int64_t i = base + (int64_t)threadIdx.x * P + q;
      v[q] = i < m ? a[i] : 0;
      s += v[q];
    }
    uint32_t before, total;
    BS(tmp).ExclusiveSum(s, before, total);
    before += carry;
#pragma unroll
    for (int q = 0; q < P; q++) {
      const int64_t i = base + (int64_t)threadIdx.x * P + q;
      if (i < m) a[i] = before;
      before += v[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
}

template <bool FIRST, int D>
__global__ void __launch_bounds__(kThreads) k_down(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ bin,
                                                   const uint32_t* __restrict__ iin, const uint64_t* __restrict__ kin,
                                                   int64_t n, uint64_t mask, int shift,
                                                   const uint32_t* __restrict__ offs, int64_t ntiles,
                                                   uint32_t* __restrict__ bout, uint32_t* __restrict__ iout,
                                                   uint64_t* __restrict__ kout) {
  constexpr int R = 1 << D;
  extern __shared__ __align__(16) unsigned char smraw[];
  uint32_t* wc = reinterpret_cast<uint32_t*>(smraw);  // [kWarps][R]
  uint32_t* dstart = wc + kWarps * R;                 // [R] tile-local start of digit
  uint32_t* gstart = dstart + R;                      // [R] global start of digit run for this tile
  uint64_t* sk = reinterpret_cast<uint64_t*>(gstart + R);
  uint32_t* sb = reinterpret_cast<uint32_t*>(sk + kTile);
  uint32_t* si = sb + kTile;
  typedef cub::BlockScan<uint32_t, kThreads> BS;
  __shared__ typename BS::TempStorage tmp;

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int j = threadIdx.x; j < kWarps * R; j += kThreads) wc[j] = 0;
  const int64_t base = (int64_t)blockIdx.x * kTile;
  uint32_t b[kItems], ix[kItems], wr[kItems];
  uint64_t k[kItems];
  load_items<FIRST>(keys, bin, iin, kin, n, mask, base, b, ix, k);
  __syncthreads();
  uint32_t* mine = wc + w * R;
#pragma unroll
  for (int r = 0; r < kItems; r++) {
    const int64_t p = base + w * 32 * kItems + r * 32 + lane;
    const bool ok = p < n;
    const unsigned act = __ballot_sync(0xFFFFFFFFu, ok);
    const uint32_t d = (b[r] >> shift) & (R - 1);
    uint32_t before = 0;
    unsigned peers = 0;
    if (ok) {
      peers = __match_any_sync(act, d);
      before = mine[d];
    }
    __syncwarp();
    if (ok) {
      const unsigned lt = peers & ((1u << lane) - 1);
      wr[r] = before + __popc(lt);
      if (lt == 0) mine[d] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive over warps; tile totals; tile-local digit starts
  constexpr int DPT = (R + kThreads - 1) / kThreads;
  uint32_t tot[DPT];
  uint32_t s_all = 0;
#pragma unroll
  for (int q = 0; q < DPT; q++) {
    const int d = threadIdx.x * DPT + q;
    uint32_t s = 0;
    if (d < R) {
      for (int ww = 0; ww < kWarps; ww++) {
        const uint32_t c = wc[ww * R + d];
        wc[ww * R + d] = s;
        s += c;
      }
    }
    tot[q] = s;
    s_all += s;
  }
  uint32_t before_all;
  BS(tmp).ExclusiveSum(s_all, before_all);
#pragma unroll
  for (int q = 0; q < DPT; q++) {
    const int d = threadIdx.x * DPT + q;
    if (d < R) {
      dstart[d] = before_all;
      gstart[d] = offs[(int64_t)d * ntiles + blockIdx.x];
    }
    before_all += tot[q];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kItems; r++) {
    const int64_t p = base + w * 32 * kItems + r * 32 + lane;
    if (p < n) {
      const uint32_t d = (b[r] >> shift) & (R - 1);
      const uint32_t lp = dstart[d] + mine[d] + wr[r];
      sb[lp] = b[r];
      si[lp] = ix[r];
      sk[lp] = k[r];
    }
  }
  __syncthreads();
  const int cnt = (int)(n - base < kTile ? n - base : kTile);
  for (int j = threadIdx.x; j < cnt; j += kThreads) {
    const uint32_t bb = sb[j];
    const uint32_t d = (bb >> shift) & (R - 1);
    const uint32_t dst = gstart[d] + (uint32_t)j - dstart[d];
    bout[dst] = bb;
    iout[dst] = si[j];
    kout[dst] = sk[j];
  }
}

template <int D>
static size_t down_smem() {
  return (size_t)(kWarps + 2) * (1 << D) * 4 + (size_t)kTile * 16;
}

struct Bufs {
  uint32_t *b[2], *i[2];
  uint64_t* k[2];
  uint32_t* hist;
};

template <int D>
static void rsort(const uint64_t* keys, int64_t n, int bits, Bufs& f, uint32_t* ob, uint32_t* oi, uint64_t* ok,
                  cudaStream_t s) {
  const int64_t ntiles = (n + kTile - 1) / kTile;
  const uint64_t mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
  const int passes = bits <= D ? 1 : (bits + D - 1) / D;
  for (int ps = 0; ps < passes; ps++) {
    const int shift = ps * D;
    const bool first = ps == 0, last = ps == passes - 1;
    const uint32_t* bin = first ? nullptr : f.b[(ps - 1) & 1];
    const uint32_t* iin = first ? nullptr : f.i[(ps - 1) & 1];
    const uint64_t* kin = first ? nullptr : f.k[(ps - 1) & 1];
    uint32_t* bo = last ? ob : f.b[ps & 1];
    uint32_t* io = last ? oi : f.i[ps & 1];
    uint64_t* ko = last ? ok : f.k[ps & 1];
    if (first) k_hist<true, D><<<(unsigned)ntiles, kThreads, 0, s>>>(keys, bin, n, mask, shift, f.hist, ntiles);
    else k_hist<false, D><<<(unsigned)ntiles, kThreads, 0, s>>>(keys, bin, n, mask, shift, f.hist, ntiles);
    k_scan<<<1, 1024, 0, s>>>(f.hist, (int64_t)ntiles << D);
    if (first)
      k_down<true, D><<<(unsigned)ntiles, kThreads, down_smem<D>(), s>>>(keys, bin, iin, kin, n, mask, shift, f.hist,
                                                                        ntiles, bo, io, ko);
    else
      k_down<false, D><<<(unsigned)ntiles, kThreads, down_smem<D>(), s>>>(keys, bin, iin, kin, n, mask, shift, f.hist,
                                                                         ntiles, bo, io, ko);
  }
}

int main() {
  const int64_t n = 1 << 20;
  uint64_t* keys;
  uint32_t *bkt, *idx, *sb1, *si1, *sb2, *si2;
  uint64_t* sk2;
  Bufs f;
  CK(cudaMalloc(&keys, n * 8));
  CK(cudaMalloc(&bkt, n * 4)); CK(cudaMalloc(&idx, n * 4)); CK(cudaMalloc(&sb1, n * 4)); CK(cudaMalloc(&si1, n * 4));
  CK(cudaMalloc(&sb2, n * 4)); CK(cudaMalloc(&si2, n * 4)); CK(cudaMalloc(&sk2, n * 8));
  for (int q = 0; q < 2; q++) {
    CK(cudaMalloc(&f.b[q], n * 4)); CK(cudaMalloc(&f.i[q], n * 4)); CK(cudaMalloc(&f.k[q], n * 8));
  }
  CK(cudaMalloc(&f.hist, ((n + kTile - 1) / kTile) * 1024 * 4 + 64));
  size_t cub_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, bkt, sb1, idx, si1, (int)n, 0, 23);
  void* tmp;
  CK(cudaMalloc(&tmp, cub_bytes));
  CK(cudaFuncSetAttribute(k_down<true, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)down_smem<8>()));
  CK(cudaFuncSetAttribute(k_down<false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)down_smem<8>()));
  CK(cudaFuncSetAttribute(k_down<true, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)down_smem<10>()));
  CK(cudaFuncSetAttribute(k_down<false, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)down_smem<10>()));
  CK(cudaFuncSetAttribute(k_down<true, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)down_smem<7>()));
  CK(cudaFuncSetAttribute(k_down<false, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)down_smem<7>()));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<uint64_t> hk(n);
  struct Case { const char* name; int bits; int kind; };
  for (Case c : {Case{"uniform 2^20 buckets", 20, 0}, Case{"C1 8192 buckets", 13, 0}, Case{"zipf-ish 2^20", 20, 1},
                 Case{"uniform 2^23 buckets", 23, 0}, Case{"1 bucket", 0, 0}}) {
    uint64_t x = 88172645463325252ull;
    for (int64_t i = 0; i < n; i++) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      const double u = (double)(x >> 11) / 9007199254740992.0;
      hk[i] = (c.kind == 1 && u < 0.3) ? (x % 64) : (x >> 2);
    }
    CK(cudaMemcpy(keys, hk.data(), n * 8, cudaMemcpyHostToDevice));
    const uint64_t mask = (1ull << c.bits) - 1;
    const int ebits = c.bits < 1 ? 1 : c.bits;
    auto run_cub = [&] {
      k_prep<<<(unsigned)((n + 255) / 256), 256>>>(keys, n, mask, bkt, idx);
      size_t bytes = cub_bytes;
      cub::DeviceRadixSort::SortPairs(tmp, bytes, bkt, sb1, idx, si1, (int)n, 0, ebits);
    };
    float ms, t_cub = 0, t8 = 0, t10 = 0, t7 = 0;
    int64_t bad8 = 0, bad10 = 0, bad7 = 0;
    std::vector<uint32_t> rb(n), ri(n), qb(n), qi(n);
    std::vector<uint64_t> qk(n);
    for (int variant = 0; variant < 4; variant++) {
      float tot = 0;
      for (int rep = 0; rep < 6; rep++) {
        k_spin<<<1, 1>>>(400000);
        cudaEventRecord(e0);
        if (variant == 0) run_cub();
        else if (variant == 1) rsort<8>(keys, n, c.bits, f, sb2, si2, sk2, 0);
        else if (variant == 2) rsort<10>(keys, n, c.bits, f, sb2, si2, sk2, 0);
        else rsort<7>(keys, n, c.bits, f, sb2, si2, sk2, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) tot += ms / 5;
      }
      CK(cudaGetLastError());
      if (variant == 0) {
        t_cub = tot;
        CK(cudaMemcpy(rb.data(), sb1, n * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(ri.data(), si1, n * 4, cudaMemcpyDeviceToHost));
      } else {
        CK(cudaMemcpy(qb.data(), sb2, n * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(qi.data(), si2, n * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(qk.data(), sk2, n * 8, cudaMemcpyDeviceToHost));
        int64_t bad = 0;
        for (int64_t i = 0; i < n; i++) bad += rb[i] != qb[i] || ri[i] != qi[i] || qk[i] != hk[ri[i]];
        if (variant == 1) { t8 = tot; bad8 = bad; }
        else if (variant == 2) { t10 = tot; bad10 = bad; }
        else { t7 = tot; bad7 = bad; }
      }
    }
    printf("%-22s prep+cub %.1f us | rsort D8 %.1f us (bad %lld) | D10 %.1f us (bad %lld) | D7 %.1f us (bad %lld)\n",
           c.name, t_cub * 1e3, t8 * 1e3, (long long)bad8, t10 * 1e3, (long long)bad10, t7 * 1e3, (long long)bad7);
  }
  return 0;
}
