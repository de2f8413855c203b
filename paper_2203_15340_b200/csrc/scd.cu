// scd.cu -- K2b: persistent SP-SCD / SP-RCD inner solver (Alg. 5 steps 5-12).
//
// Step t:  alpha_t, tau_t from the index stream (steps 7-8; include/ils.h):
//          s in tau_t  <=>  pi^{-1}(s) < alpha_t   (every thread tests the indices it owns)
//          j_t = argmax_{s in tau_t} r_s^2, ties to the smallest s     (step 9)
//          sc = r_j / A1bar_jj ; beta_j += sc ; r -= sc A1bar_(j)       (steps 10-11, :697-698)
// SP-RCD (weighted): j_t drawn from the column-norm weights (Remark 4.1).
// One CTA of 1024 threads; thread s owns coordinates s, s+1024, ... of r and beta (registers);
// the Ab_1 row is read from L2/HBM each step. Every check_every steps r = b_hat - A1bar beta
// is recomputed and the inner stop rule of include/ils.h is applied.
#include <climits>

#include "common.cuh"
#include "ils_internal.h"

namespace ils {

constexpr int SCD_THREADS = 1024;
constexpr int SCD_WARPS = SCD_THREADS / 32;
constexpr int SCD_RING = 128;

struct ScdKey {
  uint32_t alpha;
  int32_t j;   // weighted mode index
  uint32_t key[kFeistelRounds];
  uint32_t pad_[2];
};

struct ScdParams {
  const double* G;   // npad x npad, A1bar
  int64_t npad;
  int n;
  const double* N;
  const uint64_t* S;
  const double* bhat;
  double* beta_out;
  uint64_t seed;
  uint32_t k;
  int64_t max_inner, check_every;
  double inner_tol;
  int alpha_mode, alpha_k, weighted;
  DevStatus* st;
};

__device__ __forceinline__ void scd_make_key(uint64_t seed, uint32_t k, uint64_t t, int n, int alpha_mode,
                                             int alpha_k, int weighted, const uint64_t* S, ScdKey& e) {
  if (weighted) {
    const U4 x = draw(seed, k, t, kTagRcd);
    e.j = sample_weighted(((uint64_t)x.y << 32) | x.x, S, n);
    e.alpha = 1;
    return;
  }
  const U4 a = draw(seed, k, t, kTagScdA);
  const U4 b = draw(seed, k, t, kTagScdB);
  const U4 c = draw(seed, k, t, kTagScdC);
  const U4 d = draw(seed, k, t, kTagScdD);
  e.alpha = alpha_mode == ILS_ALPHA_UNIFORM ? 1u + mulhi32(a.x, (uint32_t)n)
                                            : (uint32_t)((alpha_k < n) ? alpha_k : n);
  e.j = -1;
  e.key[0] = a.y; e.key[1] = a.z; e.key[2] = a.w;
  e.key[3] = b.x; e.key[4] = b.y; e.key[5] = b.z; e.key[6] = b.w;
  e.key[7] = c.x; e.key[8] = c.y; e.key[9] = c.z; e.key[10] = c.w;
  e.key[11] = d.x;
}

template <int U>
__global__ void __launch_bounds__(SCD_THREADS, 1) scd_kernel(ScdParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* bs = reinterpret_cast<double*>(smem_raw);          // [npad] beta (for checks)
  double* Ns = bs + p.npad;                                  // [n]
  uint64_t* Ss = reinterpret_cast<uint64_t*>(Ns + ((p.n + 1) & ~1));
  ScdKey* ring = reinterpret_cast<ScdKey*>(Ss + ((p.n + 1) & ~1));
  __shared__ double wv[2][SCD_WARPS], wp[2][SCD_WARPS];
  __shared__ int wi[2][SCD_WARPS];
  __shared__ double red[SCD_WARPS];
  __shared__ double rj_s[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = p.n;
  const uint32_t h = feistel_half_bits((uint32_t)n), mask = (1u << h) - 1u;

  for (int j = tid; j < n; j += SCD_THREADS) {
    Ns[j] = p.N[j];
    Ss[j] = p.S[j];
  }
  double r[U], beta[U];
  double nb2 = 0.0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int s = tid + u * SCD_THREADS;
    r[u] = (s < n) ? p.bhat[s] : 0.0;
    beta[u] = 0.0;
    nb2 = fma(r[u], r[u], nb2);
  }
  nb2 = warp_sum(nb2);
  if (lane == 0) red[warp] = nb2;
  __syncthreads();
  double B2 = 0.0;
  for (int w = 0; w < SCD_WARPS; ++w) B2 += red[w];
  const double bnorm = sqrt(B2);
  if (bnorm == 0.0) {
    for (int64_t j = tid; j < p.npad; j += SCD_THREADS) p.beta_out[j] = 0.0;
    if (tid == 0) {
      p.st->inner_steps = 0;
      p.st->inner_conv = 1;
    }
    return;
  }
  if (warp == 0) {
    for (int b = 0; b < 2; ++b) {
      const int64_t t = 32 * b + lane;
      if (t < p.max_inner)
        scd_make_key(p.seed, p.k, (uint64_t)t, n, p.alpha_mode, p.alpha_k, p.weighted, Ss,
                     ring[t & (SCD_RING - 1)]);
    }
  }
  __syncthreads();

  int64_t t = 0;
  int conv = 0;
  for (; t < p.max_inner; ++t) {
    if (warp == 0 && (t & 31) == 0 && t + 64 + lane < p.max_inner) {
      const int64_t tt = t + 64 + lane;
      scd_make_key(p.seed, p.k, (uint64_t)tt, n, p.alpha_mode, p.alpha_k, p.weighted, Ss,
                   ring[tt & (SCD_RING - 1)]);
    }
    const ScdKey& e = ring[t & (SCD_RING - 1)];
    const int pb = (int)(t & 1);
    int j;
    double rj;
    if (p.weighted) {
      j = e.j;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (tid + u * SCD_THREADS == j) rj_s[pb] = r[u];
      __syncthreads();
      rj = rj_s[pb];
    } else {
      uint32_t key[kFeistelRounds];
#pragma unroll
      for (int q = 0; q < kFeistelRounds; ++q) key[q] = e.key[q];
      const uint32_t alpha = e.alpha;
      ArgMax best{-1.0, INT_MAX, 0.0};
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = tid + u * SCD_THREADS;
        if (s < n) {
          const uint32_t m = feistel_inverse((uint32_t)s, key, h, mask, (uint32_t)n);
          if (m < alpha) {
            const double v = r[u] * r[u];
            if (argmax_better(v, s, best.val, best.idx)) {
              best.val = v;
              best.idx = s;
              best.pay = r[u];
            }
          }
        }
      }
      best = warp_argmax(best);
      if (lane == 0) {
        wv[pb][warp] = best.val;
        wi[pb][warp] = best.idx;
        wp[pb][warp] = best.pay;
      }
      __syncthreads();
      ArgMax b{-1.0, INT_MAX, 0.0};
      for (int w = 0; w < SCD_WARPS; ++w) {
        if (argmax_better(wv[pb][w], wi[pb][w], b.val, b.idx)) {
          b.val = wv[pb][w];
          b.idx = wi[pb][w];
          b.pay = wp[pb][w];
        }
      }
      j = b.idx;
      rj = b.pay;
    }
    const double sc = rj / Ns[j];
    const double* grow = p.G + (int64_t)j * p.npad;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int s = tid + u * SCD_THREADS;
      if (s < n) {
        r[u] = fma(-sc, grow[s], r[u]);
        if (s == j) beta[u] += sc;
      }
    }
    if ((t + 1) % p.check_every == 0) {
      // r = b_hat - A1bar beta (column access of the symmetric A1bar: coalesced), stop test
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = tid + u * SCD_THREADS;
        if (s < p.npad) bs[s] = beta[u];
      }
      __syncthreads();
      double acc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) acc[u] = 0.0;
      for (int jj = 0; jj < n; ++jj) {
        const double bj = bs[jj];
        const double* g = p.G + (int64_t)jj * p.npad;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int s = tid + u * SCD_THREADS;
          if (s < n) acc[u] = fma(g[s], bj, acc[u]);
        }
      }
      double r2 = 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int s = tid + u * SCD_THREADS;
        if (s < n) {
          r[u] = p.bhat[s] - acc[u];
          r2 = fma(r[u], r[u], r2);
        }
      }
      r2 = warp_sum(r2);
      __syncthreads();
      if (lane == 0) red[warp] = r2;
      __syncthreads();
      double R2 = 0.0;
      for (int w = 0; w < SCD_WARPS; ++w) R2 += red[w];
      if (sqrt(R2) <= p.inner_tol * bnorm) {
        conv = 1;
        ++t;
        break;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int s = tid + u * SCD_THREADS;
    if (s < p.npad) p.beta_out[s] = (s < n) ? beta[u] : 0.0;
  }
  if (tid == 0) {
    p.st->inner_steps = t;
    p.st->inner_conv = conv;
  }
}

int scd_inner(Handle& h, const double* bhat, double* beta, uint64_t seed, int64_t k, int64_t max_inner,
              int64_t check_every, double inner_tol, int alpha_mode, int alpha_k, int weighted,
              int64_t* steps_out) {
  if (h.npad > 8 * SCD_THREADS) {
    set_error("SP-SCD: n > 8192 not supported by the single-CTA kernel in this release");
    return ILS_ERR_UNSUPPORTED;
  }
  int r = build_gram(h);
  if (r) return r;
  ScdParams p{};
  p.G = h.G;
  p.npad = h.npad;
  p.n = (int)h.n;
  p.N = h.N;
  p.S = h.S;
  p.bhat = bhat;
  p.beta_out = beta;
  p.seed = seed;
  p.k = (uint32_t)k;
  p.max_inner = max_inner;
  p.check_every = check_every > 0 ? check_every : h.n;
  p.inner_tol = inner_tol;
  p.alpha_mode = alpha_mode;
  p.alpha_k = alpha_k;
  p.weighted = weighted;
  p.st = h.dstat;
  const size_t smem = (size_t)h.npad * 8 + 2 * (size_t)((h.n + 1) & ~1) * 8 + SCD_RING * sizeof(ScdKey);
  const int per = (int)((h.npad + SCD_THREADS - 1) / SCD_THREADS);
  int U = 1;
  while (U < per) U *= 2;
  ILS_CU(cudaEventRecord(h.evk0, h.stream));
#define SCD_LAUNCH(UU)                                                                              \
  do {                                                                                              \
    ILS_CU(cudaFuncSetAttribute(scd_kernel<UU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    scd_kernel<UU><<<1, SCD_THREADS, smem, h.stream>>>(p);                                          \
    ILS_LAUNCHED("scd_kernel");                                                                     \
  } while (0)
  switch (U) {
    case 1: SCD_LAUNCH(1); break;
    case 2: SCD_LAUNCH(2); break;
    case 4: SCD_LAUNCH(4); break;
    default: SCD_LAUNCH(8); break;
  }
#undef SCD_LAUNCH
  ILS_CU(cudaEventRecord(h.evk1, h.stream));
  ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, h.stream));
  ILS_CU(cudaStreamSynchronize(h.stream));
  const int64_t steps = h.hstat->inner_steps;
  if (steps_out) *steps_out = steps;
  const double nd = (double)h.n;
  hot_account(h, 2, (double)steps * 8.0 * nd + (double)(steps / p.check_every) * 8.0 * nd * nd);
  return ILS_OK;
}

__global__ void scd_subset_kernel(int n, uint64_t seed, uint32_t k, uint64_t t, int alpha_mode, int alpha_k,
                                  int32_t* alpha_out, uint8_t* mask) {
  __shared__ ScdKey e;
  if (threadIdx.x == 0) scd_make_key(seed, k, t, n, alpha_mode, alpha_k, 0, nullptr, e);
  __syncthreads();
  const uint32_t h = feistel_half_bits((uint32_t)n), msk = (1u << h) - 1u;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const uint32_t m = feistel_inverse((uint32_t)s, e.key, h, msk, (uint32_t)n);
    mask[s] = (m < e.alpha) ? 1 : 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *alpha_out = (int32_t)e.alpha;
}

int scd_subset_mask(int64_t n, uint64_t seed, int64_t k, int64_t t, int alpha_mode, int alpha_k,
                    int32_t* alpha_dev, uint8_t* mask_dev, cudaStream_t st) {
  scd_subset_kernel<<<32, 256, 0, st>>>((int)n, seed, (uint32_t)k, (uint64_t)t, alpha_mode, alpha_k,
                                        alpha_dev, mask_dev);
  ILS_LAUNCHED("scd_subset_kernel");
  return ILS_OK;
}

}  // namespace ils
