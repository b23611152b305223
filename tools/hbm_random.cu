// Microbenchmark: what HBM delivers for the table's access patterns (the
// ceilings the probe / metadata kernels are compared with).
//   seq copy            : STREAM-like copy (read + write)
//   rand 128-B lines    : one random 128-B line per 8-lane tile (digest-line probe)
//   rand 32-B sectors   : one random 8-B load per thread (candidate-key read)
//   line -> key chain   : random line, then a dependent random 8-B load per tile
//                         (the probe's digest -> key chain)
// Arrays: 32 GiB (like C2's values) and 1 GiB (like C2's keys).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hbm_random tools/hbm_random.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xFF51AFD7ED558CCDull;
  x ^= x >> 33;
  x *= 0xC4CEB9FE1A85EC53ull;
  x ^= x >> 33;
  return x;
}

__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// KPT random lines per 8-lane tile in flight
template <int KPT>
__global__ void k_lines(const uint4* __restrict__ a, int64_t nlines, int64_t n, uint32_t* out) {
  const int r = threadIdx.x & 7;
  const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int64_t ntiles = ((int64_t)gridDim.x * blockDim.x) >> 3;
  uint32_t acc = 0;
  for (int64_t i = tile * KPT; i < n; i += ntiles * KPT) {
    uint4 v[KPT];
#pragma unroll
    for (int u = 0; u < KPT; u++) v[u] = a[(mix(i + u) % nlines) * 8 + r];
#pragma unroll
    for (int u = 0; u < KPT; u++) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int KPT>
__global__ void k_words(const uint64_t* __restrict__ a, int64_t nwords, int64_t n, uint32_t* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  uint64_t acc = 0;
  for (int64_t i = t * KPT; i < n; i += nt * KPT) {
    uint64_t v[KPT];
#pragma unroll
    for (int u = 0; u < KPT; u++) v[u] = a[mix(i + u + 77) % nwords];
#pragma unroll
    for (int u = 0; u < KPT; u++) acc ^= v[u];
  }
  if (acc == 0x12345678u) out[0] = (uint32_t)acc;
}

// digest line -> dependent key word (8-lane tile, lane 0 does the key read)
__global__ void k_chain(const uint4* __restrict__ lines, int64_t nlines, const uint64_t* __restrict__ keys,
                        int64_t nkeys, int64_t n, uint32_t* out) {
  const int r = threadIdx.x & 7;
  const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int64_t ntiles = ((int64_t)gridDim.x * blockDim.x) >> 3;
  uint64_t acc = 0;
  for (int64_t i = tile; i < n; i += ntiles) {
    const uint4 v = lines[(mix(i) % nlines) * 8 + r];
    const uint32_t sel = __shfl_sync(0xffffffffu, v.x, (threadIdx.x & 31) & ~7);
    if (r == 0) acc ^= keys[(mix(i ^ sel) % nkeys)];
  }
  if (acc == 0x12345678u) out[0] = (uint32_t)acc;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = (size_t)32 << 30, small = (size_t)1 << 30;
  uint4 *a, *b;
  uint64_t* k;
  uint32_t* out;
  if (cudaMalloc(&a, big) || cudaMalloc(&b, (size_t)4 << 30) || cudaMalloc(&k, small) || cudaMalloc(&out, 64)) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(a, 1, big);
  cudaMemset(k, 1, small);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  auto timeit = [&](auto fn) {
    fn();
    cudaEventRecord(e0);
    fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
  };
  const int64_t n16 = ((int64_t)4 << 30) / 16;
  timeit([&] { k_copy<<<sms * 8, 256>>>(a, b, n16); });
  printf("seq copy 4 GiB:                 %.3f ms  %.0f GB/s (read+write)\n", ms, 2.0 * (4ll << 30) / ms / 1e6);
  const int64_t n = 1 << 22;  // 4M lines / words per run
  for (int64_t span : {(int64_t)big, (int64_t)small}) {
    const int64_t nl = span / 128;
    timeit([&] { k_lines<4><<<sms * 8, 256>>>(a, nl, n, out); });
    printf("rand 128-B lines over %5.1f GiB: %.3f ms  %.0f GB/s  %.2f G lines/s\n", span / 1073741824.0, ms,
           n * 128.0 / ms / 1e6, n / ms / 1e6);
    timeit([&] { k_words<4><<<sms * 8, 256>>>((const uint64_t*)a, span / 8, n, out); });
    printf("rand 8-B words over %5.1f GiB:   %.3f ms  %.0f GB/s of sectors (32 B)  %.2f G words/s\n",
           span / 1073741824.0, ms, n * 32.0 / ms / 1e6, n / ms / 1e6);
  }
  timeit([&] { k_chain<<<sms * 8, 256>>>(a, ((int64_t)128 << 20) / 128, k, small / 8, n, out); });
  printf("line(128 MiB) -> key(1 GiB) chain: %.3f ms  %.2f G probes/s\n", ms, n / ms / 1e6);
  return 0;
}
