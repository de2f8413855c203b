// dsmem_bench2.cu -- development microbenchmark (not product code): cost of a 16-CTA cluster
// all-to-all of NV doubles per CTA with destination-uniform 16-byte st.async, as a function of
// NV (message bytes), the number of sending warps, and a bulk-copy alternative.
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

__device__ __forceinline__ void stc2(uint32_t ra, double a, double b) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(ra), "d"(a), "d"(b) : "memory");
}
__device__ __forceinline__ void red_rel(uint32_t ra, uint32_t v) {
  asm volatile("red.release.cluster.shared::cluster.add.u32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rel(uint32_t ra, uint32_t v) {
  asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_rlx(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void mb_remote_arrive(uint32_t ra) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}

constexpr int C = 16;

// variant: 0 = warp 0 sends to all 16 dst; 1 = warps split destinations (nsw warps);
// 2 = one thread, 16 remote bulk copies (smem -> remote smem)
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(128) bench(int variant, int NV, int nsw, int iters,
                                                                       long long* out, double* sink) {
  __shared__ __align__(16) double src[2][128];
  __shared__ __align__(16) double recv[2][C][128];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ __align__(8) uint64_t bar16[2];
  __shared__ uint32_t cnt;
  __shared__ uint32_t flags[C];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)ctarank();
  const uint32_t bytes = C * NV * 8;
  if (tid == 0) {
    mb_init(&bar[0], 1);
    mb_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mb_expect(&bar[0], bytes);
    mb_expect(&bar[1], bytes);
    mb_init(&bar16[0], C);
    mb_init(&bar16[1], C);
    cnt = 0;
  }
  if (tid < C) flags[tid] = 0;
  src[0][tid] = rank + tid * 0.001;
  src[1][tid] = rank + tid * 0.002;
  __syncthreads();
  cl_sync();
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int pb = it & 1;
    const uint32_t par = (it >> 1) & 1;
    const int npl = NV / 2;   // lanes carrying 2 values
    if (variant == 0 || variant == 1) {
      const int sw = (variant == 0) ? 1 : nsw;
      if (warp < sw) {
        const double v0 = src[pb][(2 * lane) % NV] + it, v1 = src[pb][(2 * lane + 1) % NV] + it;
        for (int l0 = 0; l0 < npl; l0 += 32) {
          if (lane + l0 < npl) {
            const uint32_t la = smem_u32(&recv[pb][rank][2 * (lane + l0)]);
            for (int c = warp; c < C; c += sw) sta2(mapa(la, c), v0, v1, mapa(smem_u32(&bar[pb]), c));
          }
        }
      }
    } else if (variant == 6 || variant == 7) {
      // pull: publish locally, one cluster barrier, every CTA reads all C buffers remotely
      if (warp == 0 && lane < NV) src[pb][lane] = src[pb ^ 1][lane] + 1.0;
      if (variant == 6) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      } else {
        asm volatile("fence.acq_rel.cluster;\n\tbarrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
      }
      double s = 0.0;
      if (warp == 0 && lane < NV) {
        double a[C];
        const uint32_t la = smem_u32(&src[pb][lane]);
#pragma unroll
        for (int c = 0; c < C; ++c) {
          asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(a[c]) : "r"(mapa(la, c)) : "memory");
        }
#pragma unroll
        for (int c = 0; c < C; ++c) s += a[c];
      }
      acc += s;
      __syncthreads();
      continue;
    } else if (variant >= 3) {
      // plain remote stores of the data, then a release-ordered signal per destination
      if (warp == 0) {
        const double v0 = src[pb][(2 * lane) % NV] + it, v1 = src[pb][(2 * lane + 1) % NV] + it;
        if (lane < npl) {
          const uint32_t la = smem_u32(&recv[pb][rank][2 * lane]);
          for (int c = 0; c < C; ++c) stc2(mapa(la, c), v0, v1);
        }
        __syncwarp();
        if (lane < C) {
          if (variant == 3) red_rel(mapa(smem_u32(&cnt), lane), 1u);
          else if (variant == 4) st_rel(mapa(smem_u32(&flags[rank]), lane), (uint32_t)(it + 1));
          else mb_remote_arrive(mapa(smem_u32(&bar16[pb]), lane));
        }
      }
      if (variant == 3) {
        if (tid == 0) while (ld_acq(&cnt) < (uint32_t)(C * (it + 1))) {}
        __syncthreads();
      } else if (variant == 4) {
        if (warp == 0) {
          if (lane < C) while (ld_acq(&flags[lane]) < (uint32_t)(it + 1)) {}
          __syncwarp();
        }
        __syncthreads();
      } else {
        mb_wait(&bar16[pb], par);
      }
      double s = 0.0;
      if (lane < NV)
        for (int c = 0; c < C; ++c) s += recv[pb][c][lane];
      acc += s;
      __syncthreads();
      continue;
    } else {
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int c = 0; c < C; ++c) {
          const uint32_t da = mapa(smem_u32(&recv[pb][rank][0]), c);
          const uint32_t db = mapa(smem_u32(&bar[pb]), c);
          asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(da),
                       "r"(smem_u32(&src[pb][0])), "r"(NV * 8), "r"(db)
                       : "memory");
        }
      }
    }
    mb_wait(&bar[pb], par);
    double s = 0.0;
    if (lane < NV)
      for (int c = 0; c < C; ++c) s += recv[pb][c][lane];
    acc += s;
    __syncthreads();
    if (tid == 0) mb_expect(&bar[pb], bytes);
  }
  long long t1 = clock64();
  cl_sync();
  if (rank == 0 && tid == 0) out[0] = (t1 - t0) / iters;
  sink[rank * 128 + tid] = acc;
}

// depth-D pipelined all-to-all: at iteration it, send the values of iteration it + D - 1, then wait
// for iteration it (D exchanges in flight)
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(128) bench_pipe(int D, int iters, long long* out,
                                                                            double* sink) {
  __shared__ __align__(16) double recv[4][C][32];
  __shared__ __align__(8) uint64_t bar[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)ctarank();
  const uint32_t bytes = C * 32 * 8;
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mb_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < 4; ++i) mb_expect(&bar[i], bytes);
  }
  __syncthreads();
  cl_sync();
  double acc = 0.0;
  auto send = [&](int it) {
    const int pb = it & 3;
    if (warp == 0 && lane < 16) {
      const uint32_t la = smem_u32(&recv[pb][rank][2 * lane]);
      for (int c = 0; c < C; ++c) sta2(mapa(la, c), it + lane, rank * 1.0, mapa(smem_u32(&bar[pb]), c));
    }
  };
  for (int i = 0; i < D - 1; ++i) send(i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int pb = it & 3;
    if (it + D - 1 < iters + D) send(it + D - 1);
    mb_wait(&bar[pb], (it >> 2) & 1);
    double s = 0.0;
    for (int c = 0; c < C; ++c) s += recv[pb][c][lane];
    acc += s;
    __syncthreads();
    if (tid == 0) mb_expect(&bar[pb], bytes);
  }
  long long t1 = clock64();
  // drain the extra sends
  for (int it = iters; it < iters + D - 1; ++it) mb_wait(&bar[it & 3], (it >> 2) & 1);
  cl_sync();
  if (rank == 0 && tid == 0) out[0] = (t1 - t0) / iters;
  sink[rank * 128 + tid] = acc;
}

__device__ __forceinline__ void mb_wait_cta(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok)
                 : "r"(smem_u32(b)), "r"(par)
                 : "memory");
}

// the RK block kernel's exchange pattern with concurrent column traffic: 4 warps' partials ->
// named barrier -> warp 0 sums and sends 32 values (16 lanes x v2) to 16 CTAs -> wait -> tree sum.
// mode 0: no column traffic; 1: 8 x 4 KB TMA bulk copies per iteration into smem (as the RK kernel);
// 2: the same 32 KB per iteration as plain 16-byte global loads into registers, consumed one
// iteration later.
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(128) bench_rk(int mode, int iters, const double* gsrc,
                                                                          long long* out, double* sink) {
  __shared__ __align__(16) double wred[2][4][32];
  __shared__ __align__(16) double recv[2][C][32];
  __shared__ __align__(8) uint64_t bar[2], tbar[2];
  extern __shared__ __align__(128) double dyn[];
  double (*cols)[8][512] = reinterpret_cast<double (*)[8][512]>(dyn);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (int)ctarank();
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mb_init(&bar[i], 1);
      mb_init(&tbar[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < 2; ++i) mb_expect(&bar[i], C * 32 * 8);
  }
  __syncthreads();
  cl_sync();
  double acc = 1.0 + tid;
  const double2* g2 = reinterpret_cast<const double2*>(gsrc);
  double2 pre[8];
  for (int i = 0; i < 8; ++i) pre[i] = make_double2(0.0, 0.0);
  auto tma = [&](int it) {
    const int b = it & 1;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&tbar[b])), "r"(8 * 4096) : "memory");
    for (int i = 0; i < 8; ++i) {
      const double* src = gsrc + ((size_t)((it * 8 + i) % 4096) * 8192 + rank * 512);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(
                       smem_u32(&cols[b][i][0])), "l"(src), "r"(smem_u32(&tbar[b]))
                   : "memory");
    }
  };
  if (mode == 1 && tid == 127) tma(0);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int pb = it & 1;
    if (mode == 1) {
      mb_wait(&tbar[pb], (it >> 1) & 1);
      acc += cols[pb][warp][lane] * 1e-12;
      __syncthreads();
      if (tid == 127 && it + 1 < iters) tma(it + 1);
    } else if (mode == 3) {
      // cp.async (LDGSTS) 16-byte copies into smem, 32 KB per iteration, consumed next iteration
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      acc += cols[pb][warp][lane] * 1e-12;
      double* dstb = &cols[pb ^ 1][0][0];
      for (int i = 0; i < 16; ++i) {
        const int e = i * 128 + tid;   // 16-byte element index in the 32 KB buffer
        const double* src = gsrc + ((size_t)((it * 8 + (e >> 8)) % 4096) * 8192 + rank * 512 + (e & 255) * 2);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dstb + 2 * e)), "l"(src) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    } else if (mode == 2) {
      for (int i = 0; i < 8; ++i) acc += (pre[i].x + pre[i].y) * 1e-12;
      for (int i = 0; i < 8; ++i) {
        const size_t row = (size_t)((it * 8 + i) % 4096) * 4096 + rank * 256 + tid * 2;
        pre[i] = __ldcg(g2 + row / 2 + 0);
      }
    }
    wred[pb][warp][lane] = acc * 1e-3;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (warp == 0) {
      double v = 0.0;
      for (int w = 0; w < 4; ++w) v += wred[pb][w][lane];
      const double v0 = __shfl_sync(0xffffffffu, v, (2 * lane) & 31);
      const double v1 = __shfl_sync(0xffffffffu, v, (2 * lane + 1) & 31);
      const uint32_t la = smem_u32(&recv[pb][rank][2 * (lane & 15)]);
      const uint32_t lb = smem_u32(&bar[pb]);
      if (lane < 16)
#pragma unroll
        for (int c = 0; c < C; ++c) sta2(mapa(la, c), v0, v1, mapa(lb, c));
    }
    mb_wait(&bar[pb], (it >> 1) & 1);
    double a[C];
#pragma unroll
    for (int c = 0; c < C; ++c) a[c] = recv[pb][c][lane];
#pragma unroll
    for (int s = 1; s < C; s *= 2)
#pragma unroll
      for (int c = 0; c + s < C; c += 2 * s) a[c] += a[c + s];
    acc += a[0] * 1e-9;
    // ~1500 cycles of dependent FP64 work stand in for the products and updates
    double x = acc;
    for (int k = 0; k < 150; ++k) x = fma(x, 0.999999, 1e-9);
    acc += x * 1e-15;
    if (tid == 0) mb_expect(&bar[pb], C * 32 * 8);
  }
  long long t1 = clock64();
  cl_sync();
  if (rank == 0 && tid == 0) out[0] = (t1 - t0) / iters;
  sink[rank * 128 + tid] = acc;
}

int main() {
  long long* out;
  double* sink;
  cudaMalloc(&out, 8 * sizeof(long long));
  cudaMalloc(&sink, C * 128 * sizeof(double));
  cudaFuncSetAttribute(bench, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  struct V { int var, nv, nsw; const char* name; } vs[] = {
      {0, 2, 1, "1 warp, NV=2"},   {0, 8, 1, "1 warp, NV=8"},   {0, 16, 1, "1 warp, NV=16"},
      {0, 32, 1, "1 warp, NV=32"}, {0, 64, 1, "1 warp, NV=64"}, {0, 96, 1, "1 warp, NV=96"},
      {1, 32, 2, "2 warps, NV=32"}, {1, 32, 4, "4 warps, NV=32"}, {1, 64, 4, "4 warps, NV=64"},
      {1, 96, 4, "4 warps, NV=96"}, {2, 32, 1, "bulk, NV=32"}, {2, 64, 1, "bulk, NV=64"}, {2, 96, 1, "bulk, NV=96"},
      {3, 32, 1, "st+red counter NV=32"}, {4, 32, 1, "st+flag/src NV=32"}, {5, 32, 1, "st+remote mbar arrive"},
      {6, 32, 1, "pull barrier.cluster NV=32"}, {7, 32, 1, "pull fence+relaxed barrier NV=32"},
      {3, 2, 1, "st+red counter NV=2"}, {4, 2, 1, "st+flag/src NV=2"}, {5, 2, 1, "st+mbar arrive NV=2"}};
  for (auto& v : vs) {
    bench<<<C, 128>>>(v.var, v.nv, v.nsw, 20000, out, sink);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = -1;
    cudaMemcpy(&h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-16s: %lld cycles/iter  [%s]\n", v.name, h, cudaGetErrorString(e));
  }
  cudaFuncSetAttribute(bench_pipe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int D = 1; D <= 3; ++D) {
    bench_pipe<<<C, 128>>>(D, 20000, out, sink);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = -1;
    cudaMemcpy(&h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("pipelined depth %d: %lld cycles/iter  [%s]\n", D, h, cudaGetErrorString(e));
  }
  cudaFuncSetAttribute(bench_rk, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(bench_rk, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  double* g;
  cudaMalloc(&g, (size_t)4096 * 8192 * 8);
  cudaMemset(g, 0, (size_t)4096 * 8192 * 8);
  const char* mn[] = {"no column traffic", "TMA bulk 32 KB/iter", "LDG 16 KB/iter", "cp.async 32 KB/iter"};
  for (int mode = 0; mode < 4; ++mode) {
    long long h = -1;
    bench_rk<<<C, 128, 65536>>>(mode, 20000, g, out, sink);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("rk pattern + %s: %lld cycles/iter  [%s]\n", mn[mode], h, cudaGetErrorString(e));
  }
  return 0;
}
