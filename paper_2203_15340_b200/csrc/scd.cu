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

constexpr int SCD_MAXT = 256;    // threads per CTA (max)
constexpr int SCD_MAXW = SCD_MAXT / 32;
constexpr int SCD_RING = 128;
constexpr int SCD_AHEAD = 64;

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

// Membership bits of this thread's coordinates s = tid + v*NT in tau_t: pi^{-1}(s) < alpha_t.
template <int V>
__device__ __forceinline__ uint32_t scd_members(const ScdKey& e, int tid, int NT, int n, uint32_t h,
                                                uint32_t mask) {
  uint32_t key[kFeistelRounds];
#pragma unroll
  for (int q = 0; q < kFeistelRounds; ++q) key[q] = e.key[q];
  const uint32_t alpha = e.alpha;
  uint32_t bits = 0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int s = tid + v * NT;
    if (s < n && feistel_inverse((uint32_t)s, key, h, mask, (uint32_t)n) < alpha) bits |= 1u << v;
  }
  return bits;
}

// One CTA of NT <= 256 threads; thread tid owns coordinates s = tid + v*NT (v < V) of r and beta
// in registers. Per step (software-pipelined): argmax over tau_t (thread -> warp shuffles -> one
// barrier -> redundant per-warp reduction of the warp winners), then the A1bar row j is loaded
// from L2 while the membership bits of step t+1 are computed (pure integer work, data-independent).
template <int V>
__global__ void __launch_bounds__(SCD_MAXT, 1) scd_kernel(ScdParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* bs = reinterpret_cast<double*>(smem_raw);          // [npad] beta (for checks)
  double* rNs = bs + p.npad;                                 // [n] 1 / A1bar_jj
  uint64_t* Ss = reinterpret_cast<uint64_t*>(rNs + ((p.n + 1) & ~1));
  ScdKey* ring = reinterpret_cast<ScdKey*>(Ss + ((p.n + 1) & ~1));
  __shared__ double wv[2][SCD_MAXW], wr[2][SCD_MAXW];
  __shared__ int wi[2][SCD_MAXW];
  __shared__ double red[SCD_MAXW];
  __shared__ double rj_s[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NT = blockDim.x, NW = NT >> 5;
  const int n = p.n;
  const uint32_t h = feistel_half_bits((uint32_t)n), mask = (1u << h) - 1u;

  for (int j = tid; j < n; j += NT) {
    rNs[j] = 1.0 / p.N[j];
    Ss[j] = p.S[j];
  }
  double r[V], beta[V];
  double nb2 = 0.0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int s = tid + v * NT;
    r[v] = (s < n) ? p.bhat[s] : 0.0;
    beta[v] = 0.0;
    nb2 = fma(r[v], r[v], nb2);
  }
  nb2 = warp_sum(nb2);
  if (lane == 0) red[warp] = nb2;
  __syncthreads();
  double B2 = 0.0;
  for (int w = 0; w < NW; ++w) B2 += red[w];
  const double bnorm = sqrt(B2);
  if (bnorm == 0.0) {
    for (int64_t j = tid; j < p.npad; j += NT) p.beta_out[j] = 0.0;
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

  uint32_t inmask = p.weighted ? 0u : scd_members<V>(ring[0], tid, NT, n, h, mask);
  int64_t t = 0;
  int conv = 0;
  int64_t next_check = p.check_every;
  for (; t < p.max_inner; ++t) {
    const int pb = (int)(t & 1);
    int j;
    double rj;
    if (p.weighted) {
      j = ring[t & (SCD_RING - 1)].j;
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (tid + v * NT == j) rj_s[pb] = r[v];
      __syncthreads();
      rj = rj_s[pb];
    } else {
      // thread-local argmax (coordinates ascend with v: strict > keeps the smallest index)
      double bv = -1.0, br = 0.0;
      int bi = INT_MAX;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const double q = r[v] * r[v];
        if (((inmask >> v) & 1u) && q > bv) {
          bv = q;
          bi = tid + v * NT;
          br = r[v];
        }
      }
      // warp argmax (value, index); ties to the smallest index
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (argmax_better(ov, oi, bv, bi)) {
          bv = ov;
          bi = oi;
        }
      }
      // the winning lane publishes (value, index, r)
      if (bi != INT_MAX && (bi % NT) == tid) {
        wv[pb][warp] = bv;
        wi[pb][warp] = bi;
        wr[pb][warp] = br;
      } else if (lane == 0 && bi == INT_MAX) {
        wv[pb][warp] = -1.0;
        wi[pb][warp] = INT_MAX;
      }
      __syncthreads();
      // every warp reduces the NW warp winners (same fixed tree in every warp)
      double cv = (lane < NW) ? wv[pb][lane] : -1.0;
      int ci = (lane < NW) ? wi[pb][lane] : INT_MAX;
#pragma unroll
      for (int o = SCD_MAXW / 2; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, cv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, ci, o);
        if (argmax_better(ov, oi, cv, ci)) {
          cv = ov;
          ci = oi;
        }
      }
      j = __shfl_sync(0xffffffffu, ci, 0);   // lanes >= NW reduced only invalid entries
      rj = wr[pb][(j % NT) >> 5];
    }
    const double sc = rj * rNs[j];
    // A1bar row j (L2): issue the loads, then overlap their latency with step t+1's membership
    const double* grow = p.G + (int64_t)j * p.npad;
    double g[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int s = tid + v * NT;
      g[v] = (s < n) ? __ldcg(grow + s) : 0.0;
    }
    if (warp == NW - 1 && (t & 31) == 0 && t + SCD_AHEAD + lane < p.max_inner) {
      const int64_t tt = t + SCD_AHEAD + lane;
      scd_make_key(p.seed, p.k, (uint64_t)tt, n, p.alpha_mode, p.alpha_k, p.weighted, Ss,
                   ring[tt & (SCD_RING - 1)]);
    }
    if (!p.weighted && t + 1 < p.max_inner)
      inmask = scd_members<V>(ring[(t + 1) & (SCD_RING - 1)], tid, NT, n, h, mask);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int s = tid + v * NT;
      r[v] = fma(-sc, g[v], r[v]);
      if (s == j) beta[v] += sc;
    }
    if (t + 1 == next_check) {
      next_check += p.check_every;
      // r = b_hat - A1bar beta (column access of the symmetric A1bar: coalesced), stop test
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int s = tid + v * NT;
        if (s < p.npad) bs[s] = beta[v];
      }
      __syncthreads();
      double acc[V];
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = 0.0;
      for (int jj = 0; jj < n; ++jj) {
        const double bj = bs[jj];
        const double* gr = p.G + (int64_t)jj * p.npad;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const int s = tid + v * NT;
          if (s < n) acc[v] = fma(__ldcg(gr + s), bj, acc[v]);
        }
      }
      double r2 = 0.0;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int s = tid + v * NT;
        if (s < n) {
          r[v] = p.bhat[s] - acc[v];
          r2 = fma(r[v], r[v], r2);
        }
      }
      r2 = warp_sum(r2);
      __syncthreads();
      if (lane == 0) red[warp] = r2;
      __syncthreads();
      double R2 = 0.0;
      for (int w = 0; w < NW; ++w) R2 += red[w];
      if (sqrt(R2) <= p.inner_tol * bnorm) {
        conv = 1;
        ++t;
        break;
      }
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int s = tid + v * NT;
    if (s < p.npad) p.beta_out[s] = (s < n) ? beta[v] : 0.0;
  }
  if (tid == 0) {
    p.st->inner_steps = t;
    p.st->inner_conv = conv;
  }
}

int scd_inner(Handle& h, const double* bhat, double* beta, uint64_t seed, int64_t k, int64_t max_inner,
              int64_t check_every, double inner_tol, int alpha_mode, int alpha_k, int weighted,
              int64_t* steps_out) {
  if (h.npad > 32 * SCD_MAXT) {
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
  // threads: one coordinate per thread up to 256 coordinates, then V coordinates per thread
  int nt = (int)((h.n + 31) / 32 * 32);
  if (nt > SCD_MAXT) nt = SCD_MAXT;
  const int per = (int)((h.n + nt - 1) / nt);
  int V = 1;
  while (V < per) V *= 2;
  ILS_CU(cudaEventRecord(h.evk0, h.stream));
#define SCD_LAUNCH(VV)                                                                              \
  do {                                                                                              \
    ILS_CU(cudaFuncSetAttribute(scd_kernel<VV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    scd_kernel<VV><<<1, nt, smem, h.stream>>>(p);                                                   \
    ILS_LAUNCHED("scd_kernel");                                                                     \
  } while (0)
  switch (V) {
    case 1: SCD_LAUNCH(1); break;
    case 2: SCD_LAUNCH(2); break;
    case 4: SCD_LAUNCH(4); break;
    case 8: SCD_LAUNCH(8); break;
    case 16: SCD_LAUNCH(16); break;
    default: SCD_LAUNCH(32); break;
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
