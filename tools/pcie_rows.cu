// Microbenchmark: random 512-B row reads from mapped pinned host memory
// (the C4 overflow tier) — 16-B loads per lane vs TMA bulk copies
// (cp.async.bulk global -> shared, one 512-B copy per row, mbarrier
// completion).  Build + run:  nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -o /tmp/pcie_rows tools/pcie_rows.cu && /tmp/pcie_rows
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cstring>
#include <sys/mman.h>

constexpr int kRowBytes = 512;
constexpr int kRowsPerWarp = 8;  // bulk path: rows in flight per warp

__global__ void k_ldg(const uint4* __restrict__ src, const uint32_t* __restrict__ rows, int64_t n, uint4* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * 8; base < n; base += nw * 8) {
    uint4 x[8];
#pragma unroll
    for (int u = 0; u < 8; u++) x[u] = base + u < n ? src[(int64_t)rows[base + u] * 32 + lane] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (base + u < n) out[(base + u) * 32 + lane] = x[u];
  }
}

__device__ __forceinline__ void mbar_init(uint64_t* m, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(m)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(m)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(m)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(m))
               : "memory");
}

__global__ void k_bulk(const uint4* __restrict__ src, const uint32_t* __restrict__ rows, int64_t n, uint4* out) {
  extern __shared__ uint4 sm[];
  __shared__ uint64_t bar[32];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  uint4* buf = sm + (size_t)wib * kRowsPerWarp * 32;
  uint64_t* m = bar + wib;
  if (lane == 0) mbar_init(m, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned phase = 0;
  for (int64_t base = warp * kRowsPerWarp; base < n; base += nw * kRowsPerWarp) {
    const int cnt = (int)((n - base) < kRowsPerWarp ? (n - base) : kRowsPerWarp);
    if (lane == 0) mbar_expect(m, cnt * kRowBytes);
    __syncwarp();
    if (lane < cnt) bulk_g2s(buf + lane * 32, src + (int64_t)rows[base + lane] * 32, kRowBytes, m);
    mbar_wait(m, phase);
    phase ^= 1;
    for (int u = 0; u < cnt; u++) out[(base + u) * 32 + lane] = buf[u * 32 + lane];
    __syncwarp();
  }
}

int main(int argc, char** argv) {
  const int64_t nrows_tab = (int64_t)1 << 26;  // 32 GiB of 512-B rows
  const int64_t n = 1 << 20;
  void* host = nullptr;
  // argv[1] == "thp": anonymous mmap backed by 2-MB transparent huge pages,
  // registered mapped (cudaHostRegister) instead of cudaHostAlloc's 4-KB pages
  const bool thp = argc > 1 && !strcmp(argv[1], "thp");
  if (thp) {
    const size_t bytes = (size_t)nrows_tab * kRowBytes;
    host = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (host == MAP_FAILED) { printf("mmap failed\n"); return 1; }
    int rc = madvise(host, bytes, MADV_HUGEPAGE);
    memset(host, 0, bytes);
    cudaError_t e = cudaHostRegister(host, bytes, cudaHostRegisterMapped);
    printf("thp arena: madvise rc %d, cudaHostRegister %s\n", rc, cudaGetErrorString(e));
  } else if (cudaHostAlloc(&host, nrows_tab * kRowBytes, cudaHostAllocMapped)) {
    printf("alloc failed\n");
    return 1;
  }
  uint4* dsrc;
  cudaHostGetDevicePointer((void**)&dsrc, host, 0);
  uint32_t* hrows = (uint32_t*)malloc(n * 4);
  uint64_t x = 88172645463325252ull;
  for (int64_t i = 0; i < n; i++) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; hrows[i] = (uint32_t)(x % nrows_tab); }
  uint32_t* rows;
  uint4* out;
  cudaMalloc(&rows, n * 4);
  cudaMalloc(&out, n * kRowBytes);
  cudaMemcpy(rows, hrows, n * 4, cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 8 * kRowsPerWarp * kRowBytes;
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int grid_mul : {4, 8, 16}) {
    for (int rep = 0; rep < 2; rep++) {
      float ms;
      cudaEventRecord(a);
      k_ldg<<<sms * grid_mul, 256>>>(dsrc, rows, n, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("ldg  grid %3d x sms: %.2f ms  %.1f GB/s\n", grid_mul, ms, n * kRowBytes / ms / 1e6);
      cudaEventRecord(a);
      k_bulk<<<sms * grid_mul, 256, smem>>>(dsrc, rows, n, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("bulk grid %3d x sms: %.2f ms  %.1f GB/s  (%s)\n", grid_mul, ms, n * kRowBytes / ms / 1e6,
                      cudaGetErrorString(cudaGetLastError()));
    }
  }
  // sequential reference: H2D copy engine
  float ms;
  cudaEventRecord(a);
  cudaMemcpy(out, host, n * kRowBytes, cudaMemcpyHostToDevice);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("memcpy H2D contiguous: %.2f ms  %.1f GB/s\n", ms, n * kRowBytes / ms / 1e6);
  return 0;
}
