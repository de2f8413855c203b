// dsmem_bench3.cu -- development microbenchmark (not product code): a 16-CTA cluster all-reduce of
// NV = 10 doubles per CTA, (a) one hop: every CTA sends its message to all 16 (destination-uniform
// 16-byte st.async, the RK-RGS kernels' exchange) and sums the 16 in a binary tree; (b) two hops on a
// 4 x 4 grid: messages to the 4 CTAs of the own row group (ranks 4g..4g+3), row sums in the same tree
// order, then the row sum to the 4 CTAs of the own column (ranks c, c+4, c+8, c+12), 4-way sum -- the
// same binary tree, so bitwise the same result. Reports cycles per exchange with one exchange in
// flight (latency) and the sender's busy cycles.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mb_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok)
                 : "r"(smem_u32(b)), "r"(par)
                 : "memory");
}
__device__ __forceinline__ void sta2(uint32_t ra, double a, double b, uint32_t rb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(ra), "d"(a), "d"(b), "r"(rb)
               : "memory");
}

constexpr int C = 16, NV = 10;

// mode 0: one hop; 1: two hops (4 + 4 sends, own CTA included); 2: two hops, own copy by a local store (3 + 3)
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(32) bench(int mode, int iters, long long* out, double* res) {
  __shared__ __align__(16) double r1[2][C][NV];   // one hop: [src]; two hops: [src in row group] (first 4)
  __shared__ __align__(16) double r2[2][4][NV];   // two hops, second round: [row group]
  __shared__ __align__(8) uint64_t b1[2], b2[2];
  const int lane = threadIdx.x;
  const int rank = (int)ctarank(), g = rank >> 2, c = rank & 3;
  const int n1 = mode == 0 ? C : (mode == 1 ? 4 : 3), n2 = mode == 1 ? 4 : 3;
  if (lane == 0) {
    for (int i = 0; i < 2; ++i) {
      mb_init(&b1[i], 1);
      mb_init(&b2[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < 2; ++i) {
      mb_expect(&b1[i], n1 * NV * 8);
      mb_expect(&b2[i], n2 * NV * 8);
    }
  }
  __syncwarp();
  cl_sync();
  double carry = 0.0;
  long long busy = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int pb = it & 1;
    const uint32_t par = (it >> 1) & 1;
    // lane l < 5 carries values 2l, 2l+1 (depends on the previous result: one exchange in flight)
    const double v0 = rank * 0.5 + lane + carry * 1e-9, v1 = rank * 0.25 - lane + carry * 1e-9;
    const long long s0 = clock64();
    if (mode == 0) {
      if (lane < NV / 2)
        for (int d = 0; d < C; ++d)
          sta2(mapa(smem_u32(&r1[pb][rank][2 * lane]), d), v0, v1, mapa(smem_u32(&b1[pb]), d));
      busy += clock64() - s0;
      mb_wait(&b1[pb], par);
      double a[C];
#pragma unroll
      for (int s = 0; s < C; ++s) a[s] = r1[pb][s][lane < NV ? lane : 0];
#pragma unroll
      for (int s = 1; s < C; s *= 2)
#pragma unroll
        for (int k = 0; k + s < C; k += 2 * s) a[k] += a[k + s];
      carry = a[0];
      if (lane == 0) mb_expect(&b1[pb], n1 * NV * 8);
    } else {
      if (lane < NV / 2) {
        for (int d = 0; d < 4; ++d) {
          if (mode == 2 && d == c) {
            r1[pb][c][2 * lane] = v0;
            r1[pb][c][2 * lane + 1] = v1;
          } else {
            sta2(mapa(smem_u32(&r1[pb][c][2 * lane]), 4 * g + d), v0, v1, mapa(smem_u32(&b1[pb]), 4 * g + d));
          }
        }
      }
      busy += clock64() - s0;
      __syncwarp();
      mb_wait(&b1[pb], par);
      const int l = lane < NV ? lane : 0;
      const double rs = (r1[pb][0][l] + r1[pb][1][l]) + (r1[pb][2][l] + r1[pb][3][l]);
      if (lane == 0) mb_expect(&b1[pb], n1 * NV * 8);
      const double w0 = __shfl_sync(0xffffffffu, rs, (2 * lane) % NV), w1 = __shfl_sync(0xffffffffu, rs, (2 * lane + 1) % NV);
      const long long s1 = clock64();
      if (lane < NV / 2) {
        for (int d = 0; d < 4; ++d) {
          if (mode == 2 && d == g) {
            r2[pb][g][2 * lane] = w0;
            r2[pb][g][2 * lane + 1] = w1;
          } else {
            sta2(mapa(smem_u32(&r2[pb][g][2 * lane]), 4 * d + c), w0, w1, mapa(smem_u32(&b2[pb]), 4 * d + c));
          }
        }
      }
      busy += clock64() - s1;
      __syncwarp();
      mb_wait(&b2[pb], par);
      carry = (r2[pb][0][l] + r2[pb][1][l]) + (r2[pb][2][l] + r2[pb][3][l]);
      if (lane == 0) mb_expect(&b2[pb], n2 * NV * 8);
    }
    __syncwarp();
  }
  const long long t1 = clock64();
  cl_sync();
  if (lane == 0) {
    out[2 * rank] = (t1 - t0) / iters;
    out[2 * rank + 1] = busy / iters;
  }
  if (lane < NV) res[rank * NV + lane] = carry;
}

int main() {
  long long* out;
  double* res;
  cudaMalloc(&out, 2 * C * sizeof(long long));
  cudaMalloc(&res, C * NV * sizeof(double));
  cudaFuncSetAttribute(bench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  double ref[C * NV];
  const char* mn[3] = {"one hop, 16 sends", "two hops 4x4, 4+4 sends", "two hops 4x4, 3+3 sends + local"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) bench<<<C, 32>>>(mode, 20000, out, res);
    cudaError_t le = cudaGetLastError();
    cudaError_t e = cudaDeviceSynchronize();
    if (le != cudaSuccess) e = le;
    long long h[2 * C];
    double hr[C * NV];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    cudaMemcpy(hr, res, sizeof(hr), cudaMemcpyDeviceToHost);
    int same = 1, all = 1;
    if (mode == 0) for (int i = 0; i < C * NV; ++i) ref[i] = hr[i];
    for (int i = 0; i < C * NV; ++i) {
      if (hr[i] != ref[i]) same = 0;
      if (hr[i] != hr[i % NV]) all = 0;
    }
    printf("%s: %lld cycles/exchange, sender busy %lld (rank 5: %lld / %lld) bitwise==onehop %d, same in all CTAs %d [%s]\n", mn[mode],
           h[0], h[1], h[10], h[11], same, all, cudaGetErrorString(e));
  }
  return 0;
}
