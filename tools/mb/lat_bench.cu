// lat_bench.cu -- development microbenchmark (not product code): dependent-chain latency of
// shared-memory 8-byte loads, fp64 FMA, fp64 rsqrt, warp shuffles and __syncthreads on one SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(long long* out, int iters, double seed) {
  __shared__ double sm[1024];
  __shared__ int idx[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) { sm[i] = seed + i; idx[i] = (i * 7 + 1) & 1023; }
  __syncthreads();
  long long t0, t1;
  // 1: dependent LDS.32 pointer chase
  int p = tid & 1023;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) p = idx[p];
  t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / iters;
  // 2: dependent LDS.64 (address depends on previous value)
  double v = sm[tid & 1023];
  t0 = clock64();
  for (int i = 0; i < iters; ++i) v = sm[((int)v) & 1023];
  t1 = clock64();
  if (tid == 0) out[1] = (t1 - t0) / iters;
  // 3: dependent DFMA
  double a = seed, b = 1.0000001;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, 1e-9);
  t1 = clock64();
  if (tid == 0) out[2] = (t1 - t0) / iters;
  // 4: dependent rsqrt(double)
  double r = 2.0 + seed;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) r = rsqrt(r) + 1.5;
  t1 = clock64();
  if (tid == 0) out[3] = (t1 - t0) / iters;
  // 5: dependent shfl of a double
  double s = seed + tid;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) s = __shfl_xor_sync(0xffffffffu, s, 1) + 1.0;
  t1 = clock64();
  if (tid == 0) out[4] = (t1 - t0) / iters;
  // 6: __syncthreads
  t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) out[5] = (t1 - t0) / iters;
  // 7: dependent DADD
  double d = seed;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) d = d + 1e-9;
  t1 = clock64();
  if (tid == 0) out[6] = (t1 - t0) / iters;
  // 8: dependent DMMA m8n8k4 (accumulator chain)
  double c0 = 0.0, c1 = 0.0, fa = seed, fb = 1.0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(fa), "d"(fb));
  t1 = clock64();
  if (tid == 0) out[7] = (t1 - t0) / iters;
  if (a + r + s + d + v + p + c0 + c1 == 12345.678) out[8] = 1;
}

int main() {
  long long* d;
  cudaMalloc(&d, 9 * sizeof(long long));
  for (int nt : {32, 256}) {
    lat<<<1, nt>>>(d, 1000, 0.5);
    long long h[9];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threads %d: LDS32 chase %lld, LDS64 dep %lld, DFMA %lld, rsqrt(f64) %lld, SHFL f64 %lld, syncthreads %lld, DADD %lld, DMMA884 %lld cycles\n",
           nt, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  }
  return 0;
}
