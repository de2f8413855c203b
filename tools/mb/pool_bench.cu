// pool_bench.cu -- development aid: cost of stream-ordered allocations of c2-sized buffers
// (1.6 GB + 1.28 GB) reused across create/destroy cycles, with and without the pool's release
// threshold raised, and with a competing cudaMalloc'd buffer (like torch's caching allocator).
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

int main() {
  cudaFree(0);
  cudaMemPool_t pool;
  cudaDeviceGetDefaultMemPool(&pool, 0);
  const size_t s1 = (size_t)50064 * 4032 * 8, s2 = (size_t)4032 * 40000 * 8;
  void* other = nullptr;
  cudaMalloc(&other, (size_t)2 << 30);
  for (int thr = 0; thr < 2; ++thr) {
    uint64_t t = thr ? UINT64_MAX : 0;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &t);
    for (int it = 0; it < 5; ++it) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto w0 = std::chrono::steady_clock::now();
      cudaEventRecord(e0, 0);
      void *a = nullptr, *b = nullptr;
      cudaMallocAsync(&a, s1, 0);
      cudaMallocAsync(&b, s2, 0);
      cudaMemsetAsync(a, 0, s1, 0);
      cudaMemsetAsync(b, 0, s2, 0);
      cudaEventRecord(e1, 0);
      cudaStreamSynchronize(0);
      auto w1 = std::chrono::steady_clock::now();
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaFreeAsync(a, 0);
      cudaFreeAsync(b, 0);
      cudaStreamSynchronize(0);
      printf("threshold %s iter %d: alloc+memset device %.2f ms, wall %.2f ms\n", thr ? "max" : "0", it, ms,
             std::chrono::duration<double, std::milli>(w1 - w0).count());
    }
  }
  return 0;
}
