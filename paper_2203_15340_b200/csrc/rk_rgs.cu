// rk_rgs.cu -- K2a: persistent SP-RK-RGS inner solver (Alg. 2 steps 6-12).
//
// Inner step t (reading R21: r = w - A1 z is maintained instead of A1 z):
//   s1 = (b_hat_j1 - <a_j1, w>) / N_j1            RK on A1^T w = b_hat   (step 9)
//   w += s1 a_j1 ; r += s1 a_j1
//   s2 = <a_j2, r> / N_j2                          RGS on A1 z = w       (step 11)
//      = (<a_j2, r_old> + s1 <a_j2, a_j1>) / N_j2  -> the three dots share ONE reduction
//   z_j2 += s2 ; r -= s2 a_j2
// The p-vectors w, r live in registers, split over a thread-block cluster of C CTAs (row
// slices); the two column slices per step are TMA-prefetched NS steps ahead (the index stream
// is data-independent), the per-step reduction is warp shuffles + one CTA barrier + a DSMEM
// all-to-all of 3 doubles + one cluster barrier. z is replicated in every CTA's shared memory.
// Every check_every steps the inner stop rule of include/ils.h runs in-kernel.
#include "common.cuh"
#include "ils_internal.h"

namespace ils {

constexpr int RK_THREADS = 256;
constexpr int RK_WARPS = RK_THREADS / 32;
constexpr int RK_RING = 128;   // index ring entries
constexpr int RK_MAXC = 16;

struct RkIdx {
  int32_t j1, j2;
  double bh1, n1, n2;
};

struct RkParams {
  const double* A1T;
  int64_t ppad, npad;
  int n;
  const double* N;
  const uint64_t* S;
  const double* bhat;
  double* z_out;
  uint64_t seed;
  uint32_t k;
  int64_t max_inner, check_every;
  double inner_tol;
  double* gpart;       // [C][npad]
  DevStatus* st;
  int C, slice, nslots;
};

__device__ __forceinline__ void rk_fill_indices(const RkParams& p, const uint64_t* Ss, RkIdx* ring,
                                                int64_t t0, int lane) {
  const int64_t t = t0 + lane;
  if (t < p.max_inner) {
    const U4 x = draw(p.seed, p.k, (uint64_t)t, kTagRkRgs);
    const int j1 = sample_weighted(((uint64_t)x.y << 32) | x.x, Ss, p.n);
    const int j2 = sample_weighted(((uint64_t)x.w << 32) | x.z, Ss, p.n);
    RkIdx e;
    e.j1 = j1;
    e.j2 = j2;
    e.bh1 = p.bhat[j1];
    e.n1 = p.N[j1];
    e.n2 = p.N[j2];
    ring[t & (RK_RING - 1)] = e;
  }
}

template <int U, bool CLUSTER>
__global__ void __launch_bounds__(RK_THREADS, 1) rk_rgs_kernel(RkParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int C = p.C;
  const int rank = CLUSTER ? (int)cluster_ctarank() : 0;
  const int64_t i0 = (int64_t)rank * p.slice;
  const int own = (int)((i0 + p.slice <= p.ppad) ? p.slice : (p.ppad > i0 ? p.ppad - i0 : 0));
  const int NS = p.nslots;

  // shared memory carve-up
  double* slots = reinterpret_cast<double*>(smem_raw);                 // [NS][2][slice]
  double* zs = slots + (size_t)NS * 2 * p.slice;                       // [npad]
  double* azs = zs + p.npad;                                           // [slice]
  uint64_t* Ss = reinterpret_cast<uint64_t*>(azs + p.slice);           // [n]
  RkIdx* ring = reinterpret_cast<RkIdx*>(Ss + ((p.n + 1) & ~1));       // [RK_RING]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + RK_RING);        // [NS]
  __shared__ double wred[2][RK_WARPS][3];
  __shared__ double clred[2][RK_MAXC][3];
  __shared__ double chk[RK_MAXC][2];
  __shared__ double bnorm_s;

  for (int64_t j = tid; j < p.npad; j += RK_THREADS) zs[j] = 0.0;
  for (int j = tid; j < p.n; j += RK_THREADS) Ss[j] = p.S[j];
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  // ||b_hat|| (same fixed order in every CTA)
  {
    double v = 0.0;
    for (int j = tid; j < p.n; j += RK_THREADS) v = fma(p.bhat[j], p.bhat[j], v);
    v = warp_sum(v);
    if (lane == 0) wred[0][warp][0] = v;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < RK_WARPS; ++w) s += wred[0][w][0];
      bnorm_s = sqrt(s);
    }
  }
  __syncthreads();
  const double bnorm = bnorm_s;
  if (CLUSTER) cluster_sync_all();   // peers' smem initialised before any DSMEM store
  if (bnorm == 0.0) {                // b_hat = 0: z = 0 after 0 steps
    if (rank == 0) {
      for (int64_t j = tid; j < p.npad; j += RK_THREADS) p.z_out[j] = 0.0;
      if (tid == 0) {
        p.st->inner_steps = 0;
        p.st->inner_conv = 1;
      }
    }
    return;
  }

  // index ring: steps [0, 64); step t (t % 32 == 0) fills [t+64, t+96), overwriting entries of
  // steps t-64..t-33 that every thread has finished with
  if (warp == 0) {
    for (int b = 0; b < 2; ++b) rk_fill_indices(p, Ss, ring, 32 * b, lane);
  }
  __syncthreads();

  const uint32_t slice_bytes = (uint32_t)own * sizeof(double);
  auto issue = [&](int64_t t) {
    const int slot = (int)(t % NS);
    const RkIdx e = ring[t & (RK_RING - 1)];
    double* dst = slots + (size_t)slot * 2 * p.slice;
    mbar_arrive_expect_tx(&bars[slot], 2 * slice_bytes);
    bulk_g2s(dst, p.A1T + (int64_t)e.j1 * p.ppad + i0, slice_bytes, &bars[slot]);
    bulk_g2s(dst + p.slice, p.A1T + (int64_t)e.j2 * p.ppad + i0, slice_bytes, &bars[slot]);
  };
  if (tid == 0 && own > 0) {
    for (int64_t t = 0; t < NS && t < p.max_inner; ++t) issue(t);
  }

  double w[U], r[U];
#pragma unroll
  for (int u = 0; u < U; ++u) w[u] = r[u] = 0.0;

  int64_t t = 0;
  int conv = 0;
  for (; t < p.max_inner; ++t) {
    if (warp == 0 && (t & 31) == 0 && t + 64 < p.max_inner) rk_fill_indices(p, Ss, ring, t + 64, lane);
    const int slot = (int)(t % NS);
    const double* a1 = slots + (size_t)slot * 2 * p.slice;
    const double* a2 = a1 + p.slice;
    double d1 = 0.0, d2 = 0.0, d3 = 0.0;
    if (own > 0) mbar_wait(&bars[slot], (uint32_t)((t / NS) & 1));
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = tid + u * RK_THREADS;
      if (e < own) {
        const double x1 = a1[e], x2 = a2[e];
        d1 = fma(x1, w[u], d1);
        d2 = fma(x2, r[u], d2);
        d3 = fma(x2, x1, d3);
      }
    }
    d1 = warp_sum(d1);
    d2 = warp_sum(d2);
    d3 = warp_sum(d3);
    const int pb = (int)(t & 1);
    if (lane == 0) {
      wred[pb][warp][0] = d1;
      wred[pb][warp][1] = d2;
      wred[pb][warp][2] = d3;
    }
    __syncthreads();
    if (tid == 0 && own > 0 && t >= 1 && t - 1 + NS < p.max_inner) issue(t - 1 + NS);
    double D1 = 0.0, D2 = 0.0, D3 = 0.0;
    if (CLUSTER) {
      if (warp == 0 && lane < C) {
        double v0 = 0.0, v1 = 0.0, v2 = 0.0;
#pragma unroll
        for (int w8 = 0; w8 < RK_WARPS; ++w8) {
          v0 += wred[pb][w8][0];
          v1 += wred[pb][w8][1];
          v2 += wred[pb][w8][2];
        }
        const uint32_t base = map_shared_rank(smem_u32(&clred[pb][rank][0]), (uint32_t)lane);
        st_cluster_f64(base, v0);
        st_cluster_f64(base + 8, v1);
        st_cluster_f64(base + 16, v2);
      }
      cluster_sync_all();
      for (int c = 0; c < C; ++c) {
        D1 += clred[pb][c][0];
        D2 += clred[pb][c][1];
        D3 += clred[pb][c][2];
      }
    } else {
#pragma unroll
      for (int w8 = 0; w8 < RK_WARPS; ++w8) {
        D1 += wred[pb][w8][0];
        D2 += wred[pb][w8][1];
        D3 += wred[pb][w8][2];
      }
    }
    const RkIdx ix = ring[t & (RK_RING - 1)];
    const double s1 = (ix.bh1 - D1) / ix.n1;
    const double s2 = (D2 + s1 * D3) / ix.n2;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = tid + u * RK_THREADS;
      if (e < own) {
        const double x1 = a1[e], x2 = a2[e];
        w[u] = fma(s1, x1, w[u]);
        r[u] = fma(s1, x1, r[u]);
        r[u] = fma(-s2, x2, r[u]);
      }
    }
    if (tid == 0) zs[ix.j2] += s2;

    if ((t + 1) % p.check_every == 0) {
      // ---- inner stop rule: az = A1 z (own rows), g = A1^T az - b_hat, reset r = w - az
      __syncthreads();   // z complete
      double az[U];
#pragma unroll
      for (int u = 0; u < U; ++u) az[u] = 0.0;
      for (int j = 0; j < p.n; ++j) {
        const double zj = zs[j];
        const double* col = p.A1T + (int64_t)j * p.ppad + i0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = tid + u * RK_THREADS;
          if (e < own) az[u] = fma(__ldg(col + e), zj, az[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = tid + u * RK_THREADS;
        if (e < own) {
          azs[e] = az[u];
          r[u] = w[u] - az[u];
        }
      }
      __syncthreads();
      for (int j = warp; j < p.n; j += RK_WARPS) {
        const double* col = p.A1T + (int64_t)j * p.ppad + i0;
        double s = 0.0;
        for (int e = lane; e < own; e += 32) s = fma(__ldg(col + e), azs[e], s);
        s = warp_sum(s);
        if (lane == 0) p.gpart[(int64_t)rank * p.npad + j] = s;
      }
      if (CLUSTER) cluster_sync_all(); else __syncthreads();
      // this CTA's share of ||g||^2
      const int jper = (p.n + C - 1) / C;
      const int ja = rank * jper, jb = (ja + jper < p.n) ? ja + jper : p.n;
      double g2 = 0.0;
      for (int j = ja + tid; j < jb; j += RK_THREADS) {
        double g = 0.0;
        for (int c = 0; c < C; ++c) g += __ldcg(p.gpart + (int64_t)c * p.npad + j);
        g -= p.bhat[j];
        g2 = fma(g, g, g2);
      }
      g2 = warp_sum(g2);
      if (lane == 0) wred[0][warp][0] = g2;
      __syncthreads();
      if (tid == 0) {
        double s = 0.0;
        for (int w8 = 0; w8 < RK_WARPS; ++w8) s += wred[0][w8][0];
        if (CLUSTER) {
          for (int c = 0; c < C; ++c) {
            const uint32_t a = map_shared_rank(smem_u32(&chk[rank][0]), (uint32_t)c);
            st_cluster_f64(a, s);
          }
        } else {
          chk[0][0] = s;
        }
      }
      if (CLUSTER) cluster_sync_all(); else __syncthreads();
      double G2 = 0.0;
      for (int c = 0; c < C; ++c) G2 += chk[c][0];
      if (sqrt(G2) <= p.inner_tol * bnorm) {
        conv = 1;
        ++t;
        break;
      }
      __syncthreads();   // wred[0] reuse / chk reads done before the next check writes
    }
  }
  // drain: wait for prefetched-but-unused slots so no TMA is in flight at exit
  if (own > 0) {
    const int64_t issued = (t - 1 + NS < p.max_inner) ? (t - 1 + NS) : p.max_inner;
    for (int64_t u = t; u < issued; ++u) mbar_wait(&bars[u % NS], (uint32_t)((u / NS) & 1));
  }
  __syncthreads();
  if (rank == 0) {
    for (int64_t j = tid; j < p.npad; j += RK_THREADS) p.z_out[j] = zs[j];
    if (tid == 0) {
      p.st->inner_steps = t;
      p.st->inner_conv = conv;
    }
  }
  if (CLUSTER) cluster_sync_all();   // no CTA exits while peers may still store into its smem
}

__global__ void rk_indices_kernel(RkParams p, int64_t t0, int64_t count, int32_t* j1, int32_t* j2) {
  extern __shared__ __align__(16) uint64_t Ssm[];
  for (int j = threadIdx.x; j < p.n; j += blockDim.x) Ssm[j] = p.S[j];
  __syncthreads();
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count;
       q += (int64_t)gridDim.x * blockDim.x) {
    const U4 x = draw(p.seed, p.k, (uint64_t)(t0 + q), kTagRkRgs);
    j1[q] = sample_weighted(((uint64_t)x.y << 32) | x.x, Ssm, p.n);
    j2[q] = sample_weighted(((uint64_t)x.w << 32) | x.z, Ssm, p.n);
  }
}

int rk_indices(Handle& h, uint64_t seed, int64_t k, int64_t t0, int64_t count, int32_t* j1, int32_t* j2) {
  RkParams p{};
  p.n = (int)h.n;
  p.S = h.S;
  p.seed = seed;
  p.k = (uint32_t)k;
  const size_t smem = (size_t)h.n * sizeof(uint64_t);
  ILS_CU(cudaFuncSetAttribute(rk_indices_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  rk_indices_kernel<<<64, 256, smem, h.stream>>>(p, t0, count, j1, j2);
  ILS_LAUNCHED("rk_indices_kernel");
  return ILS_OK;
}

template <int U, bool CL>
static int launch_rk(Handle& h, RkParams& p, size_t smem) {
  ILS_CU(cudaFuncSetAttribute(rk_rgs_kernel<U, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.C);
  cfg.blockDim = dim3(RK_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h.stream;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (CL) {
    ILS_CU(cudaFuncSetAttribute(rk_rgs_kernel<U, CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    na = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  ILS_CU(cudaLaunchKernelEx(&cfg, rk_rgs_kernel<U, CL>, p));
  ILS_LAUNCHED("rk_rgs_kernel");
  return ILS_OK;
}

template <bool CL>
static int dispatch_rk(Handle& h, RkParams& p, size_t smem, int U) {
  switch (U) {
    case 1: return launch_rk<1, CL>(h, p, smem);
    case 2: return launch_rk<2, CL>(h, p, smem);
    case 4: return launch_rk<4, CL>(h, p, smem);
    case 8: return launch_rk<8, CL>(h, p, smem);
    case 16: return launch_rk<16, CL>(h, p, smem);
    default: return launch_rk<32, CL>(h, p, smem);
  }
}

static int rk_cluster_size(Handle& h) {
  // one CTA up to 2048 rows; otherwise a cluster (16 non-portable, fall back to 8)
  if (h.ppad <= 2048) return 1;
  int c = (int)((h.ppad + 511) / 512);
  return c >= 16 ? 16 : (c >= 8 ? 8 : (c >= 4 ? 4 : 2));
}

int rk_rgs_inner(Handle& h, const double* bhat, double* z, uint64_t seed, int64_t k, int64_t max_inner,
                 int64_t check_every, double inner_tol, int64_t* steps_out) {
  RkParams p{};
  p.A1T = h.A1T;
  p.ppad = h.ppad;
  p.npad = h.npad;
  p.n = (int)h.n;
  p.N = h.N;
  p.S = h.S;
  p.bhat = bhat;
  p.z_out = z;
  p.seed = seed;
  p.k = (uint32_t)k;
  p.max_inner = max_inner;
  p.check_every = check_every > 0 ? check_every : h.n;
  p.inner_tol = inner_tol;
  p.st = h.dstat;
  int C = rk_cluster_size(h);
  for (;;) {
    p.C = C;
    p.slice = (int)(((h.ppad + C - 1) / C + 1) / 2 * 2);
    const int per = (p.slice + RK_THREADS - 1) / RK_THREADS;
    int U = 1;
    while (U < per) U *= 2;
    if (U > 32) {
      set_error("RK-RGS: row slice too long for the register-resident kernel");
      return ILS_ERR_UNSUPPORTED;
    }
    const size_t fixed = (size_t)(h.npad + p.slice) * 8 + (size_t)((h.n + 1) & ~1) * 8 +
                         RK_RING * sizeof(RkIdx) + 16 * 8 + 256;
    const size_t slot_bytes = (size_t)2 * p.slice * 8;
    const size_t budget = 225 * 1024;
    int NS = (int)((budget - fixed) / slot_bytes);
    if (NS > 8) NS = 8;
    if (fixed + 2 * slot_bytes > budget) {
      set_error("RK-RGS: shared memory too small for this problem size");
      return ILS_ERR_UNSUPPORTED;
    }
    p.nslots = NS;
    const size_t smem = fixed + (size_t)NS * slot_bytes;
    if (!h.part || h.part_rows < C) return ILS_ERR_ARG;
    p.gpart = h.part;
    int r;
    ILS_CU(cudaEventRecord(h.evk0, h.stream));
    if (C == 1) {
      r = dispatch_rk<false>(h, p, smem, U);
    } else {
      int ncl = 0;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C);
      cfg.blockDim = dim3(RK_THREADS);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a;
      a.id = cudaLaunchAttributeClusterDimension;
      a.val.clusterDim.x = C;
      a.val.clusterDim.y = 1;
      a.val.clusterDim.z = 1;
      cfg.attrs = &a;
      cfg.numAttrs = 1;
      cudaFuncSetAttribute(rk_rgs_kernel<16, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(rk_rgs_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (cudaOccupancyMaxActiveClusters(&ncl, rk_rgs_kernel<16, true>, &cfg) != cudaSuccess || ncl < 1) {
        cudaGetLastError();
        if (C > 2) {
          C /= 2;
          continue;
        }
        set_error("RK-RGS: no cluster configuration fits");
        return ILS_ERR_UNSUPPORTED;
      }
      r = dispatch_rk<true>(h, p, smem, U);
    }
    if (r) return r;
    ILS_CU(cudaEventRecord(h.evk1, h.stream));
    ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, h.stream));
    ILS_CU(cudaStreamSynchronize(h.stream));
    const int64_t steps = h.hstat->inner_steps;
    if (steps_out) *steps_out = steps;
    const double pd = (double)h.p, nd = (double)h.n;
    hot_account(h, 1, (double)steps * 16.0 * pd + (double)(steps / p.check_every) * 16.0 * pd * nd);
    return ILS_OK;
  }
}

}  // namespace ils
