// dsmem_bench.cu -- microbenchmark of cluster all-reduce primitives on sm_100a (development aid).
// A 16-CTA cluster repeatedly all-reduces NV doubles (every CTA contributes NV values, every CTA
// needs all totals). Variants:
//   0: one st.async per lane, 32 lanes -> 16 destinations in one instruction (all-to-all, NV=2/lane)
//   1: all-to-all, destination loop: lane v sends value v; loop over 16 destinations (16 instrs)
//   2: plain st.shared::cluster stores (all-to-all) + barrier.cluster per iteration
//   3: cp.async.bulk smem->remote smem (one thread, 16 bulk copies of NV*8 bytes) + mbarrier
//   4: two-hop (scatter to owners, gather) with multi-destination st.async
// Prints cycles per iteration (clock64 on rank 0, thread 0).
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
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok)
                 : "r"(smem_u32(b)), "r"(par)
                 : "memory");
}
__device__ __forceinline__ void sta(uint32_t ra, double v, uint32_t rb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(v), "r"(rb)
               : "memory");
}

constexpr int C = 16;

__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(128) bench(int variant, int iters, long long* out,
                                                                       double* sink) {
  __shared__ __align__(16) double src[32];
  __shared__ __align__(16) double recv[2][C][32];
  __shared__ __align__(16) double recv2[2][32];
  __shared__ __align__(8) uint64_t bar[2], bar2[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)ctarank();
  const int NV = 32;
  if (tid == 0) {
    mb_init(&bar[0], 1);
    mb_init(&bar[1], 1);
    mb_init(&bar2[0], 1);
    mb_init(&bar2[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t ex = (variant == 4) ? 256 : C * NV * 8;
    mb_expect(&bar[0], ex);
    mb_expect(&bar[1], ex);
    mb_expect(&bar2[0], 256);
    mb_expect(&bar2[1], 256);
  }
  if (tid < 32) src[tid] = rank + tid * 0.001;
  __syncthreads();
  cl_sync();
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int pb = it & 1;
    const uint32_t par = (it >> 1) & 1;
    double v = src[lane] + it;
    if (variant == 0) {
      if (warp == 0) {
        // lane l sends value l to... all destinations: loop 16 with lanes mapped (l%16 -> dst), 2 rounds
        for (int r = 0; r < 2; ++r) {
          const int dst = lane % C;
          const int val = (lane / C) + 2 * r;   // 4 values per (lane,dst) pattern -> covers 32 with 16 lanes x 2
          (void)val;
        }
        // simple: each lane l sends its value to all C destinations, destination-major inner loop
        for (int d = 0; d < C; ++d) sta(mapa(smem_u32(&recv[pb][rank][lane]), (d + lane) % C), v, mapa(smem_u32(&bar[pb]), (d + lane) % C));
      }
      mb_wait(&bar[pb], par);
      if (tid == 0) mb_expect(&bar[pb], C * NV * 8);
    } else if (variant == 1) {
      if (warp == 0)
        for (int d = 0; d < C; ++d) sta(mapa(smem_u32(&recv[pb][rank][lane]), d), v, mapa(smem_u32(&bar[pb]), d));
      mb_wait(&bar[pb], par);
      if (tid == 0) mb_expect(&bar[pb], C * NV * 8);
    } else if (variant == 2) {
      if (warp == 0)
        for (int d = 0; d < C; ++d) {
          const uint32_t a = mapa(smem_u32(&recv[pb][rank][lane]), d);
          asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
        }
      cl_sync();
    } else if (variant == 3) {
      if (warp == 0) src[lane] = v;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (tid == 0)
        for (int d = 0; d < C; ++d) {
          const uint32_t da = mapa(smem_u32(&recv[pb][rank][0]), d);
          const uint32_t db = mapa(smem_u32(&bar[pb]), d);
          asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(da),
                       "r"(smem_u32(src)), "r"(NV * 8), "r"(db)
                       : "memory");
        }
      mb_wait(&bar[pb], par);
      if (tid == 0) mb_expect(&bar[pb], C * NV * 8);
    } else {
      const int VPO = 32 / C;
      if (warp == 0) {
        sta(mapa(smem_u32(&recv[pb][rank][lane / C]), lane % C), v, mapa(smem_u32(&bar[pb]), lane % C));
        mb_wait(&bar[pb], par);
        if (lane == 0) mb_expect(&bar[pb], 256);
        double o = 0.0;
        if (lane < VPO)
          for (int c = 0; c < C; ++c) o += recv[pb][c][lane];
        const int iv = lane % VPO, dst = lane / VPO;
        const double ov = __shfl_sync(0xffffffffu, o, iv);
        sta(mapa(smem_u32(&recv2[pb][rank + iv * C]), dst), ov, mapa(smem_u32(&bar2[pb]), dst));
      }
      mb_wait(&bar2[pb], par);
      if (tid == 0) mb_expect(&bar2[pb], 256);
      acc += recv2[pb][lane];
      continue;
    }
    double s = 0.0;
    for (int c = 0; c < C; ++c) s += recv[pb][c][lane];
    acc += s;
    __syncthreads();
  }
  long long t1 = clock64();
  cl_sync();
  if (rank == 0 && tid == 0) out[variant] = (t1 - t0) / iters;
  sink[rank * 128 + tid] = acc;
}

int main() {
  long long* out;
  double* sink;
  cudaMalloc(&out, 8 * sizeof(long long));
  cudaMalloc(&sink, C * 128 * sizeof(double));
  cudaFuncSetAttribute(bench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const char* names[] = {"st.async 32 lanes x 16 dst (rotated)", "st.async dst-loop (16 instrs, same dst per instr)",
                         "st.shared::cluster + barrier.cluster", "cp.async.bulk smem->smem x16 (1 thread)",
                         "two-hop st.async (scatter/gather)"};
  for (int v = 0; v < 5; ++v) {
    bench<<<C, 128>>>(v, 20000, out, sink);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = -1;
    cudaMemcpy(&h, out + v, sizeof(h), cudaMemcpyDeviceToHost);
    printf("variant %d (%s): %lld cycles/iter  [%s]\n", v, names[v], h, cudaGetErrorString(e));
  }
  return 0;
}
