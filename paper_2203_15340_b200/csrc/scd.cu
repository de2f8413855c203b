// scd.cu -- K2b: persistent SP-SCD / SP-RCD inner solver (Alg. 5 steps 5-12).
//
// Step t:  alpha_t, tau_t from the index stream (steps 7-8; include/ils.h):
//          s in tau_t  <=>  pi^{-1}(s) < alpha_t
//          j_t = argmax_{s in tau_t} r_s^2, ties to the smallest s     (step 9)
//          sc = r_j / A1bar_jj ; beta_j += sc ; r -= sc A1bar_(j)       (steps 10-11, :697-698)
// SP-RCD (weighted): j_t drawn from the column-norm weights (Remark 4.1).
//
// The subsets do not depend on the data, so the integer-heavy membership test (an 8-round
// Feistel inverse per coordinate and step) is taken off the sequential path: before each chunk
// of check_every steps, scd_masks_kernel evaluates it for the whole chunk on the full GPU and
// stores, per (step, thread), the bit mask of that thread's coordinates. scd_chunk_kernel (one
// CTA, r and beta in registers) then only does the data-dependent part per step: masked local
// argmax -> warp shuffles -> one barrier -> redundant per-warp reduction of the warp winners ->
// A1bar row j from L2 -> update. The inner check r = b_hat - A1bar beta (include/ils.h) runs
// between chunks as a full-GPU kernel (scd_check_kernel); r, beta pass through HBM between chunks.
#include <climits>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "ils_internal.h"

namespace cg = cooperative_groups;

namespace ils {

constexpr int SCD_MAXT = 256;    // threads per CTA (max; 512 and 1024 measured slower at n = 384-1000)
constexpr int SCD_DEFT = SCD_MAXT;
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
  double* Rv;        // [npad] state r (in/out)
  double* Bv;        // [npad] state beta (in/out)
  const uint32_t* masks;   // [t1 - t0][NT] membership bits (SCD mode)
  uint64_t seed;
  uint32_t k;
  int64_t t0, t1;
  int alpha_mode, alpha_k, weighted;
  int all_members;   // alpha_t = n for every step (Remark 4.1 Motzkin case): tau_t = [n], no masks
  DevStatus* st;
  int64_t ce;        // scd_warp_kernel: inner check every ce steps inside the launch (0: none)
  double inner_tol;
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
  e.alpha = (alpha_mode & 0xF) == ILS_ALPHA_UNIFORM ? 1u + mulhi32(a.x, (uint32_t)n)
                                            : (uint32_t)((alpha_k < n) ? alpha_k : n);
  e.j = -1;
  e.key[0] = a.y; e.key[1] = a.z; e.key[2] = a.w;
  e.key[3] = b.x; e.key[4] = b.y; e.key[5] = b.z; e.key[6] = b.w;
  e.key[7] = c.x;
}

// masks[(u - t0) * NT + tid] bit v  <=>  coordinate tid + v*NT is in tau_u. One CTA per step.
__global__ void __launch_bounds__(256) scd_masks_kernel(uint64_t seed, uint32_t k, int64_t t0, int64_t t1, int n,
                                                        int alpha_mode, int alpha_k, int NT, int V,
                                                        uint32_t* __restrict__ masks) {
  __shared__ ScdKey e;
  const int64_t u = t0 + blockIdx.x;
  if (u >= t1) return;
  if (threadIdx.x == 0) scd_make_key(seed, k, (uint64_t)u, n, alpha_mode, alpha_k, 0, nullptr, e);
  __syncthreads();
  uint32_t key[kFeistelRounds];
#pragma unroll
  for (int q = 0; q < kFeistelRounds; ++q) key[q] = e.key[q];
  const uint32_t h = feistel_half_bits((uint32_t)n), msk = (1u << h) - 1u;
  for (int th = threadIdx.x; th < NT; th += blockDim.x) {
    uint32_t bits = 0;
    for (int v = 0; v < V; ++v) {
      const int s = th + v * NT;
      if (s < n && feistel_inverse((uint32_t)s, key, h, msk, (uint32_t)n) < e.alpha) bits |= 1u << v;
    }
    masks[(int64_t)blockIdx.x * NT + th] = bits;
  }
}

// ---- exact uniform subsets (alpha_mode | ILS_SUBSET_EXACT, include/ils.h)
// key of coordinate s at step t: word s & 3 of the Philox draw with counter (t, k, 7 + 256 (s >> 2))
__device__ __forceinline__ void subset_keys_block(uint64_t seed, uint32_t k, uint64_t t, int n, uint32_t* u) {
  for (int b = threadIdx.x; 4 * b < n; b += blockDim.x) {
    const U4 x = draw(seed, k, t, 7u + 256u * (uint32_t)b);
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (4 * b + q < n) u[4 * b + q] = w[q];
  }
}

// the alpha-th smallest key T (radix select, four 8-bit passes) and how many keys equal to T are in
// tau (ties by index); the CTA's threads cooperate, results in *T_out / *need_out (shared)
__device__ void subset_select(const uint32_t* u, int n, uint32_t alpha, uint32_t* hist, uint32_t* T_out,
                              int* need_out) {
  uint32_t prefix = 0, pmask = 0, rank = alpha - 1;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int s = threadIdx.x; s < n; s += blockDim.x)
      if ((u[s] & pmask) == prefix) atomicAdd(&hist[(u[s] >> shift) & 255u], 1u);
    __syncthreads();
    if (threadIdx.x < 32) {   // bin holding rank: lane l scans bins 8l .. 8l+7
      const int l = threadIdx.x;
      uint32_t c[8], tot = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        c[q] = hist[8 * l + q];
        tot += c[q];
      }
      uint32_t incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (l >= o) incl += y;
      }
      uint32_t before = incl - tot;
      const bool mine = before <= rank && rank < incl;
      int bin = 0;
      uint32_t below = 0;
      if (mine) {
        uint32_t acc = before;
        for (int q = 0; q < 8; ++q) {
          if (rank < acc + c[q]) {
            bin = 8 * l + q;
            below = acc;
            break;
          }
          acc += c[q];
        }
      }
      const unsigned who = __ballot_sync(0xffffffffu, mine);
      const int src = __ffs(who) - 1;
      bin = __shfl_sync(0xffffffffu, bin, src);
      below = __shfl_sync(0xffffffffu, below, src);
      if (l == 0) {
        hist[256] = (uint32_t)bin;
        hist[257] = below;
      }
    }
    __syncthreads();
    prefix |= hist[256] << shift;
    pmask |= 255u << shift;
    rank -= hist[257];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *T_out = prefix;
    *need_out = (int)rank + 1;
  }
  __syncthreads();
}

// s in tau: u_s < T, or u_s == T and fewer than `need` coordinates s' < s have u_s' == T
__device__ __forceinline__ bool subset_member(const uint32_t* u, int n, int s, uint32_t T, int need) {
  const uint32_t v = u[s];
  if (v != T) return v < T;
  int before = 0;
  for (int q = 0; q < s; ++q) before += (u[q] == T);
  return before < need;
}

__global__ void __launch_bounds__(256) scd_masks_exact_kernel(uint64_t seed, uint32_t k, int64_t t0, int64_t t1, int n,
                                                              int alpha_mode, int alpha_k, int NT, int V,
                                                              uint32_t* __restrict__ masks) {
  extern __shared__ uint32_t ukeys[];   // [n] keys, then [258] histogram + select scratch
  uint32_t* hist = ukeys + n;
  __shared__ ScdKey e;
  __shared__ uint32_t T_s;
  __shared__ int need_s;
  const int64_t u = t0 + blockIdx.x;
  if (u >= t1) return;
  if (threadIdx.x == 0) scd_make_key(seed, k, (uint64_t)u, n, alpha_mode, alpha_k, 0, nullptr, e);
  subset_keys_block(seed, k, (uint64_t)u, n, ukeys);
  __syncthreads();
  subset_select(ukeys, n, e.alpha, hist, &T_s, &need_s);
  const uint32_t T = T_s;
  const int need = need_s;
  for (int th = threadIdx.x; th < NT; th += blockDim.x) {
    uint32_t bits = 0;
    for (int v = 0; v < V; ++v) {
      const int s = th + v * NT;
      if (s < n && subset_member(ukeys, n, s, T, need)) bits |= 1u << v;
    }
    masks[(int64_t)blockIdx.x * NT + th] = bits;
  }
}

// The same masks from the forward direction: tau_u = { pi(i) : i < alpha_u } (include/ils.h), pi(i)
// by cycle-walking the 8-round encryption (round r: (L, R) -> (R, L ^ F(R, K_r)), the inverse of
// feistel_decrypt_once's round). Three savings over scd_masks_kernel, which decrypts all n
// coordinates: (1) only alpha_u walks per step (n/2 on average for uniform alpha); (2) the round
// function F(v, K_r) = mix32(v ^ K_r) & (2^h - 1) is tabulated per step in shared memory (8 * 2^h
// 16-bit entries, h <= 11), so a round is one table load and an xor; (3) no divergent walks: a thread
// whose value lands in [n) records it and starts its next i at once, so every loop trip is one
// encryption in every lane (the old kernel's warps waited for their longest walk: at n = 20000,
// half-width h = 8, a walk takes 2^16 / n = 3.3 decryptions on average and ~10 for the slowest of 32).
// Member bits are collected in shared memory (word s % NT, bit s / NT) and written once.
constexpr int kMaskFwdMaxH = 11;
__global__ void __launch_bounds__(256) scd_masks_fwd_kernel(uint64_t seed, uint32_t k, int64_t t0, int64_t t1, int n,
                                                            int alpha_mode, int alpha_k, int NT, int V,
                                                            uint32_t* __restrict__ masks) {
  extern __shared__ uint32_t mwords[];   // [NT] member bits, then [8 << h] uint16 round tables
  __shared__ ScdKey e;
  const int64_t u = t0 + blockIdx.x;
  if (u >= t1) return;
  if (threadIdx.x == 0) scd_make_key(seed, k, (uint64_t)u, n, alpha_mode, alpha_k, 0, nullptr, e);
  const uint32_t h = feistel_half_bits((uint32_t)n), msk = (1u << h) - 1u;
  uint16_t* T = reinterpret_cast<uint16_t*>(mwords + NT);
  for (int th = threadIdx.x; th < NT; th += blockDim.x) mwords[th] = 0u;
  __syncthreads();
  for (uint32_t x = threadIdx.x; x < (8u << h); x += blockDim.x)
    T[x] = (uint16_t)(mix32((x & msk) ^ e.key[x >> h]) & msk);
  __syncthreads();
  const uint32_t alpha = e.alpha, nu = (uint32_t)n, nt = (uint32_t)NT;
  // word and bit of coordinate y: y % NT, y / NT (shift and mask when NT is a power of two)
  const bool pow2 = (nt & (nt - 1)) == 0;
  const uint32_t lg = 31u - (uint32_t)__clz((int)nt), ntm = nt - 1u;
  auto mark = [&](uint32_t y) {
    if (pow2) atomicOr(&mwords[y & ntm], 1u << (y >> lg));
    else atomicOr(&mwords[y % nt], 1u << (y / nt));
  };
  if (alpha >= nu) {   // tau_u = [n]
    for (uint32_t s = threadIdx.x; s < nu; s += blockDim.x) mark(s);
  } else {
    uint32_t i = threadIdx.x, y = threadIdx.x;
    while (i < alpha) {
      uint32_t L = y >> h, R = y & msk;
#pragma unroll
      for (uint32_t r = 0; r < (uint32_t)kFeistelRounds; ++r) {
        const uint32_t nl = R;
        R = L ^ T[(r << h) | R];
        L = nl;
      }
      y = (L << h) | R;
      if (y < nu) {   // pi(i) = y
        mark(y);
        i += blockDim.x;
        y = i;
      }
    }
  }
  __syncthreads();
  uint32_t* out = masks + (int64_t)blockIdx.x * NT;
  for (int th = threadIdx.x; th < NT; th += blockDim.x) out[th] = mwords[th];
  (void)V;
}

// membership masks of steps [t0, t1) for either subset construction (one CTA per step)
static int launch_masks(cudaStream_t st, uint64_t seed, uint32_t k, int64_t t0, int64_t t1, int n, int alpha_mode,
                         int alpha_k, int NT, int V, uint32_t* masks) {
  const uint32_t hb = feistel_half_bits((uint32_t)n);
  const char* efw = getenv("ILS_MASKS_FWD");   // experiment override: 0 = the per-coordinate decryption kernel
  if (!(alpha_mode & ILS_SUBSET_EXACT) && hb <= (uint32_t)kMaskFwdMaxH && !(efw && efw[0] == '0')) {
    const size_t smem = (size_t)NT * sizeof(uint32_t) + ((size_t)8 << hb) * sizeof(uint16_t);
    ILS_CU(cudaFuncSetAttribute(scd_masks_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    scd_masks_fwd_kernel<<<(unsigned)(t1 - t0), 256, smem, st>>>(seed, k, t0, t1, n, alpha_mode, alpha_k, NT, V,
                                                                  masks);
    ILS_LAUNCHED("scd_masks_fwd_kernel");
    return ILS_OK;
  }
  if (alpha_mode & ILS_SUBSET_EXACT) {
    const size_t smem = ((size_t)n + 258) * sizeof(uint32_t);
    cudaFuncSetAttribute(scd_masks_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    scd_masks_exact_kernel<<<(unsigned)(t1 - t0), 256, smem, st>>>(seed, k, t0, t1, n, alpha_mode, alpha_k, NT, V,
                                                                    masks);
    ILS_LAUNCHED("scd_masks_exact_kernel");
  } else {
    scd_masks_kernel<<<(unsigned)(t1 - t0), 256, 0, st>>>(seed, k, t0, t1, n, alpha_mode, alpha_k, NT, V, masks);
    ILS_LAUNCHED("scd_masks_kernel");
  }
  return ILS_OK;
}

// Single-warp SP-SCD for n <= 256 (non-weighted): lane l owns coordinates l + 32 v (v < V) of r
// and beta in registers. Per step: masked local argmax -> 5 butterfly shuffles (every lane ends
// with the winner, no barrier) -> r_j from the owner lane -> A1bar row j from L2 (V independent
// coalesced loads per lane) -> update. No shared-memory round trip or CTA barrier on the
// sequential path.
template <int V>
__global__ void __launch_bounds__(32, 1) scd_warp_kernel(ScdParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* rNs = reinterpret_cast<double*>(smem_raw);   // [n] 1 / A1bar_jj
  double* bs = rNs + ((p.n + 1) & ~1);                  // [n] beta (off the sequential path)
  const int lane = threadIdx.x;
  const int n = p.n;
  if (*(volatile int32_t*)&p.st->inner_conv) return;
  for (int j = lane; j < n; j += 32) {
    rNs[j] = 1.0 / p.N[j];
    bs[j] = p.Bv[j];
  }
  double r[V];
  double nb2 = 0.0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int s = lane + 32 * v;
    r[v] = (s < n) ? p.Rv[s] : 0.0;
    if (s < n) nb2 = fma(p.bhat[s], p.bhat[s], nb2);
  }
  if (p.t0 == 0 && warp_sum(nb2) == 0.0) {   // b_hat = 0: beta = 0 after 0 steps
    if (lane == 0) {
      p.st->inner_steps = 0;
      p.st->inner_conv = 1;
    }
    return;
  }
  __syncwarp();
  uint32_t allbits = 0;
#pragma unroll
  for (int v = 0; v < V; ++v)
    if (lane + 32 * v < n) allbits |= 1u << v;
  const uint32_t* mk = p.masks + lane;
  const int64_t L = p.t1 - p.t0;
  uint32_t q0 = 0, q1 = 0, q2 = 0, q3 = 0;
  if (!p.all_members) {
    q0 = (0 < L) ? __ldcg(mk) : 0u;
    q1 = (1 < L) ? __ldcg(mk + 32) : 0u;
    q2 = (2 < L) ? __ldcg(mk + 64) : 0u;
    q3 = (3 < L) ? __ldcg(mk + 96) : 0u;
  }
  double bn2 = 0.0;   // ||b_hat||^2 for the in-kernel checks (fixed order)
  if (p.ce > 0) {
    double v = 0.0;
    for (int s = lane; s < n; s += 32) v = fma(p.bhat[s], p.bhat[s], v);
    bn2 = warp_sum(v);
  }
  // next check step (a countdown: a 64-bit modulo per step cost ~16% of the step at c0)
  int64_t next_chk = (p.ce > 0) ? (p.t0 / p.ce + 1) * p.ce : INT64_MAX;
  for (int64_t t = p.t0; t < p.t1; ++t) {
    if (t == next_chk) {   // inner check at t (include/ils.h): r = b_hat - A1bar beta
      next_chk += p.ce;
      __syncwarp();
      double r2 = 0.0;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const int s = lane + 32 * v;
        if (s < n) {
          const double* grow2 = p.G + (int64_t)s * p.npad;
          double a = 0.0, a2 = 0.0;
          int kk = 0;
          for (; kk + 1 < n; kk += 2) {
            a = fma(__ldg(grow2 + kk), bs[kk], a);
            a2 = fma(__ldg(grow2 + kk + 1), bs[kk + 1], a2);
          }
          if (kk < n) a = fma(__ldg(grow2 + kk), bs[kk], a);
          r[v] = p.bhat[s] - (a + a2);
          r2 = fma(r[v], r[v], r2);
        }
      }
      r2 = warp_sum(r2);
      if (sqrt(r2) <= p.inner_tol * sqrt(bn2)) {
        if (lane == 0) {
          p.st->inner_steps = t;
          p.st->inner_conv = 1;
        }
        break;
      }
    }
    uint32_t inmask = allbits;
    if (!p.all_members) {
      inmask = q0;
      q0 = q1;
      q1 = q2;
      q2 = q3;
      const int64_t ahead = t - p.t0 + 4;
      q3 = (ahead < L) ? __ldcg(mk + ahead * 32) : 0u;
    }
    // lane-local argmax (coordinates ascend with v: strict > keeps the smallest index)
    double bv = -1.0, br = 0.0;
    int bi = INT_MAX;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const double q = r[v] * r[v];
      if (((inmask >> v) & 1u) && q > bv) {
        bv = q;
        bi = lane + 32 * v;
        br = r[v];
      }
    }
    // argmax across lanes by integer warp reductions (common.cuh): every lane gets the winner
    if (bi == INT_MAX) bv = 0.0;
    const int j = warp_argmax_redux(bv, bi);
    const double rj = __shfl_sync(0xffffffffu, br, j & 31);   // the owner lane's local best is j
    const double sc = rj * rNs[j];
    const double* grow = p.G + (int64_t)j * p.npad + lane;
    double g[V];
#pragma unroll
    for (int v = 0; v < V; ++v) g[v] = (lane + 32 * v < n) ? __ldg(grow + 32 * v) : 0.0;
    if (lane == (j & 31)) bs[j] += sc;
#pragma unroll
    for (int v = 0; v < V; ++v) r[v] = fma(-sc, g[v], r[v]);
  }
  __syncwarp();
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int s = lane + 32 * v;
    if (s < n) p.Rv[s] = r[v];
  }
  for (int j = lane; j < n; j += 32) p.Bv[j] = bs[j];
}

// One CTA of NT <= 256 threads runs steps [t0, t1); thread tid owns coordinates s = tid + v*NT
// (v < V) of r and beta in registers.
template <int V>
__global__ void __launch_bounds__(SCD_MAXT, 1) scd_chunk_kernel(ScdParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* rNs = reinterpret_cast<double*>(smem_raw);         // [n] 1 / A1bar_jj
  uint64_t* Ss = reinterpret_cast<uint64_t*>(rNs + ((p.n + 1) & ~1));
  ScdKey* ring = reinterpret_cast<ScdKey*>(Ss + ((p.n + 1) & ~1));
  __shared__ double wv[2][SCD_MAXW], wr[2][SCD_MAXW];
  __shared__ int wi[2][SCD_MAXW];
  __shared__ double red[SCD_MAXW];
  __shared__ double rj_s[2];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NT = blockDim.x, NW = NT >> 5;
  const int n = p.n;
  if (*(volatile int32_t*)&p.st->inner_conv) return;   // inner solve already stopped

  for (int j = tid; j < n; j += NT) {
    rNs[j] = 1.0 / p.N[j];
    if (p.weighted) Ss[j] = p.S[j];
  }
  double r[V], beta[V];
  double nb2 = 0.0;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int s = tid + v * NT;
    r[v] = (s < n) ? p.Rv[s] : 0.0;
    beta[v] = (s < n) ? p.Bv[s] : 0.0;
    if (s < n) nb2 = fma(p.bhat[s], p.bhat[s], nb2);
  }
  if (p.t0 == 0) {   // b_hat = 0: beta = 0 after 0 steps
    nb2 = warp_sum(nb2);
    if (lane == 0) red[warp] = nb2;
    __syncthreads();
    double B2 = 0.0;
    for (int w = 0; w < NW; ++w) B2 += red[w];
    if (B2 == 0.0) {
      if (tid == 0) {
        p.st->inner_steps = 0;
        p.st->inner_conv = 1;
      }
      return;
    }
  }
  if (p.weighted && warp == 0) {
    for (int b = 0; b < 2; ++b) {
      const int64_t t = p.t0 + 32 * b + lane;
      if (t < p.t1)
        scd_make_key(p.seed, p.k, (uint64_t)t, n, p.alpha_mode, p.alpha_k, 1, Ss, ring[t & (SCD_RING - 1)]);
    }
  }
  __syncthreads();

  // membership masks of steps t..t+3 (prefetch queue; the loads of t+4 overlap 4 steps)
  const uint32_t* mk = p.masks + tid;
  const int64_t L = p.t1 - p.t0;
  uint32_t q0 = 0, q1 = 0, q2 = 0, q3 = 0;
  uint32_t allbits = 0;
#pragma unroll
  for (int v = 0; v < V; ++v)
    if (tid + v * NT < n) allbits |= 1u << v;
  if (!p.weighted && !p.all_members) {
    q0 = (0 < L) ? __ldcg(mk) : 0u;
    q1 = (1 < L) ? __ldcg(mk + NT) : 0u;
    q2 = (2 < L) ? __ldcg(mk + 2 * NT) : 0u;
    q3 = (3 < L) ? __ldcg(mk + 3 * NT) : 0u;
  }
  for (int64_t t = p.t0; t < p.t1; ++t) {
    const int pb = (int)(t & 1);
    int j;
    double rj;
    if (p.weighted) {
      j = ring[t & (SCD_RING - 1)].j;
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (tid + v * NT == j) rj_s[pb] = r[v];
      if (warp == NW - 1 && ((t - p.t0) & 31) == 0 && t + SCD_AHEAD + lane < p.t1) {
        const int64_t tt = t + SCD_AHEAD + lane;
        scd_make_key(p.seed, p.k, (uint64_t)tt, n, p.alpha_mode, p.alpha_k, 1, Ss, ring[tt & (SCD_RING - 1)]);
      }
      __syncthreads();
      rj = rj_s[pb];
    } else {
      uint32_t inmask = allbits;
      if (!p.all_members) {
        inmask = q0;
        q0 = q1;
        q1 = q2;
        q2 = q3;
        const int64_t ahead = t - p.t0 + 4;
        q3 = (ahead < L) ? __ldcg(mk + ahead * NT) : 0u;
      }
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
      // warp argmax (ties to the smallest index) by integer warp reductions on the key bits; the
      // winner's lane is its index mod 32 (coordinates tid + v NT, NT a multiple of 32)
      if (bi == INT_MAX) bv = 0.0;
      const int wj = warp_argmax_redux(bv, bi);
      if (wj == INT_MAX ? lane == 0 : bi == wj) {   // the winning lane (or lane 0: no candidate) records it
        wv[pb][warp] = bv;
        wi[pb][warp] = wj;
        wr[pb][warp] = br;
      }
      __syncthreads();
      // every warp reduces the NW warp winners the same way
      const double cv = (lane < NW) ? wv[pb][lane] : 0.0;
      const int ci = (lane < NW) ? wi[pb][lane] : INT_MAX;
      const double crr = (lane < NW) ? wr[pb][lane] : 0.0;
      j = warp_argmax_redux(cv, ci);
      // the winning warp's r_j: the lane holding candidate j (a vote and a shuffle, not an integer
      // modulo by the CTA size and a dependent shared-memory load: 0.664 -> 0.652 us/step at c1)
      rj = __shfl_sync(0xffffffffu, crr, __ffs(__ballot_sync(0xffffffffu, ci == j)) - 1);
    }
    const double sc = rj * rNs[j];
    const double* grow = p.G + (int64_t)j * p.npad;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int s = tid + v * NT;
      if (s < n) {
        r[v] = fma(-sc, __ldg(grow + s), r[v]);
        if (s == j) beta[v] += sc;
      }
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int s = tid + v * NT;
    if (s < n) {
      p.Rv[s] = r[v];
      p.Bv[s] = beta[v];
    }
  }
}

// Inner check (include/ils.h): r = b_hat - A1bar beta, stop if ||r|| <= inner_tol ||b_hat||
// (sets st->inner_conv, inner_steps = t_now), else the recomputed r replaces the state.
// Cooperative full grid; warp per row of A1bar; fixed-order reductions.
__global__ void __launch_bounds__(256) scd_check_kernel(const double* __restrict__ G, int64_t npad, int n,
                                                        const double* __restrict__ bhat, const double* __restrict__ Bv,
                                                        double* __restrict__ Rv, double* __restrict__ rtmp,
                                                        double* __restrict__ red, double inner_tol, int64_t t_now,
                                                        DevStatus* st) {
  cg::grid_group grid = cg::this_grid();
  if (*(volatile int32_t*)&st->inner_conv) return;
  __shared__ double sr[8][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwg = gridDim.x * 8;
  double a = 0.0, b = 0.0;
  for (int j = blockIdx.x * 8 + warp; j < n; j += nwg) {
    const double2* row = reinterpret_cast<const double2*>(G + (int64_t)j * npad);
    const double2* bv = reinterpret_cast<const double2*>(Bv);
    double s = 0.0;
    for (int c = lane; c < (int)(npad / 2); c += 32) {
      const double2 g = __ldcg(row + c), x = __ldcg(bv + c);
      s = fma(g.x, x.x, s);
      s = fma(g.y, x.y, s);
    }
    s = warp_sum(s);
    const double rj = bhat[j] - s;
    if (lane == 0) rtmp[j] = rj;
    a = fma(rj, rj, a);
    b = fma(bhat[j], bhat[j], b);
  }
  if (lane == 0) {
    sr[warp][0] = a;
    sr[warp][1] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double A = 0.0, B = 0.0;
    for (int w = 0; w < 8; ++w) {
      A += sr[w][0];
      B += sr[w][1];
    }
    red[2 * blockIdx.x] = A;
    red[2 * blockIdx.x + 1] = B;
  }
  grid.sync();
  double A = 0.0, B = 0.0;
  for (int c = 0; c < (int)gridDim.x; ++c) {
    A += red[2 * c];
    B += red[2 * c + 1];
  }
  if (sqrt(A) <= inner_tol * sqrt(B)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->inner_steps = t_now;
      st->inner_conv = 1;
    }
  } else {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) Rv[j] = rtmp[j];
  }
}

int scd_masks(Handle& h, uint64_t seed, int64_t k, int64_t t0, int64_t t1, int alpha_mode, int alpha_k, int NT, int V,
              uint32_t* masks) {
  if (t1 <= t0) return ILS_OK;
  return launch_masks(h.stream, seed, (uint32_t)k, t0, t1, (int)h.n, alpha_mode, alpha_k, NT, V, masks);
}

int scd_inner(Handle& h, const double* bhat, double* beta, uint64_t seed, int64_t k, int64_t max_inner,
              int64_t check_every, double inner_tol, int alpha_mode, int alpha_k, int weighted,
              int64_t* steps_out) {
  if (h.large || h.npad > 32 * SCD_DEFT) {   // large n: r in shared memory, dense A1bar rows (sparse.cu kernel)
    return sparse_scd_inner(h, bhat, beta, seed, k, max_inner, check_every, inner_tol, alpha_mode, alpha_k, weighted,
                            steps_out);
  }
  int rc = build_gram(h);
  if (rc) return rc;
  const cudaStream_t st = h.stream;
  const int64_t ce = check_every > 0 ? check_every : h.n;
  // n <= 256 (non-weighted): one warp, V = n/32 coordinates per lane (scd_warp_kernel: no barrier,
  // measured 16.6 vs 22.1 ms at c0); larger n: one coordinate per thread up to 256 coordinates, then
  // V per thread (scd_chunk_kernel: at c1 the single warp's per-step issue of V = 32 loads, squares
  // and compares made it slower, 220 vs 178 ms)
  const char* env_cta = getenv("ILS_SCD_CTA");   // experiment override: force the multi-warp kernel
  const bool warpk = !weighted && h.n <= 256 && !(env_cta && env_cta[0] == '1');
  int nt = warpk ? 32 : (int)((h.n + 31) / 32 * 32);
  if (nt > SCD_DEFT) nt = SCD_DEFT;
  {
    const char* e = getenv("ILS_SCD_NT");   // experiment override of the CTA size (multi-warp kernel)
    if (e && !warpk && atoi(e) >= 64 && atoi(e) <= SCD_MAXT && (atoi(e) & 31) == 0) nt = atoi(e);
  }
  const int per = (int)((h.n + nt - 1) / nt);
  int V = 1;
  while (V < per) V *= 2;
  // the single-warp kernel runs kWarpChunks check intervals per launch with its checks in place
  constexpr int64_t kWarpChunks = 8;
  const int64_t span = warpk ? kWarpChunks * ce : ce;
  const int64_t chunk_cap = (max_inner < span) ? max_inner : span;
  const size_t state_dbl = (size_t)3 * h.npad + 2 * (size_t)h.num_sms;
  const size_t mask_bytes = weighted ? 0 : (size_t)chunk_cap * nt * sizeof(uint32_t);   // one of two buffers
  const size_t need = state_dbl * sizeof(double) + 2 * mask_bytes;
  if (h.scd_ws_bytes < need) {
    if (h.scd_ws) cudaFreeAsync(h.scd_ws, st);
    h.scd_ws = nullptr;
    h.scd_ws_bytes = 0;
    ILS_CU(cudaMallocAsync(&h.scd_ws, need, st));
    h.scd_ws_bytes = need;
  }
  double* Rv = reinterpret_cast<double*>(h.scd_ws);
  double* Bv = Rv + h.npad;
  double* rtmp = Bv + h.npad;
  double* red = rtmp + h.npad;
  uint32_t* masks = reinterpret_cast<uint32_t*>(red + 2 * h.num_sms);
  ILS_CU(cudaMemsetAsync(Rv, 0, (size_t)3 * h.npad * sizeof(double), st));
  ILS_CU(cudaMemcpyAsync(Rv, bhat, h.n * sizeof(double), cudaMemcpyDeviceToDevice, st));   // r_0 = b_hat
  ILS_CU(cudaMemsetAsync(&h.dstat->inner_conv, 0, sizeof(int32_t), st));
  ILS_CU(cudaMemsetAsync(&h.dstat->inner_steps, 0, sizeof(int64_t), st));

  ScdParams p{};
  p.G = h.G;
  p.npad = h.npad;
  p.n = (int)h.n;
  p.N = h.N;
  p.S = h.S;
  p.bhat = bhat;
  p.Rv = Rv;
  p.Bv = Bv;
  p.masks = masks;
  p.seed = seed;
  p.k = (uint32_t)k;
  p.alpha_mode = alpha_mode;
  p.alpha_k = alpha_k;
  p.weighted = weighted;
  p.all_members = (!weighted && (alpha_mode & 0xF) == ILS_ALPHA_FIXED && alpha_k >= h.n) ? 1 : 0;
  p.st = h.dstat;
  const size_t smem = 2 * (size_t)((h.n + 1) & ~1) * 8 + SCD_RING * sizeof(ScdKey);
  void* kern = nullptr;
  if (warpk) {
    switch (V) {
      case 1: kern = (void*)scd_warp_kernel<1>; break;
      case 2: kern = (void*)scd_warp_kernel<2>; break;
      case 4: kern = (void*)scd_warp_kernel<4>; break;
      default: kern = (void*)scd_warp_kernel<8>; break;
    }
  } else switch (V) {
    case 1: kern = (void*)scd_chunk_kernel<1>; break;
    case 2: kern = (void*)scd_chunk_kernel<2>; break;
    case 4: kern = (void*)scd_chunk_kernel<4>; break;
    case 8: kern = (void*)scd_chunk_kernel<8>; break;
    case 16: kern = (void*)scd_chunk_kernel<16>; break;
    default: kern = (void*)scd_chunk_kernel<32>; break;
  }
  ILS_CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int nchk = h.num_sms;
  {
    int per_sm = 0;
    ILS_CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scd_check_kernel, 256, 0));
    if (per_sm < 1) return ILS_ERR_UNSUPPORTED;
  }
  const double* Gp = h.G;
  const int64_t npad = h.npad;
  const int nn = (int)h.n;
  DevStatus* dst = h.dstat;

  constexpr int kBatch = 8;
  ILS_CU(cudaEventRecord(h.evk0, st));
  int64_t t = 0;
  int pending = 0;
  p.ce = warpk ? ce : 0;
  p.inner_tol = inner_tol;
  // The masks are data-independent: those of chunk c + 1 are formed on the auxiliary stream, into the
  // other of two buffers, while chunk c (one CTA) runs. ev_mask[b]: buffer b written; ev_chunk[b]: the
  // chunk reading buffer b done. Opt-in (ILS_SCD_MASK_OVERLAP=1): alone, SP-SCD at c1 gains 2 ms per
  // solve (121.1 -> 118.6-119.3 ms), but inside bench.py's full step (SP, SP-RK-RGS, SP-SCD on one fresh
  // handle) it measured 0.8-1.0 ms slower (120.0-120.1 -> 120.9-121.0 ms, two boxes, a stream per handle
  // or one shared per device alike), so the default keeps the masks on the handle's stream, in turn.
  const bool use_masks = !weighted && !p.all_members;
  bool overlap = false;
  {
    const char* e = getenv("ILS_SCD_MASK_OVERLAP");
    if (e && e[0] == '1') overlap = use_masks;
  }
  uint32_t* mbuf[2] = {masks, masks + (overlap ? mask_bytes / sizeof(uint32_t) : 0)};
  if (overlap) {
    if (!h.aux) {   // one auxiliary stream per device and process, shared by the handles
      static cudaStream_t aux_dev[64] = {};
      int dev = 0;
      ILS_CU(cudaGetDevice(&dev));
      if (dev < 0 || dev >= 64) dev = 0;
      if (!aux_dev[dev]) ILS_CU(cudaStreamCreateWithFlags(&aux_dev[dev], cudaStreamNonBlocking));
      h.aux = aux_dev[dev];
    }
    for (int i = 0; i < 2; ++i) {
      if (!h.ev_mask[i]) ILS_CU(cudaEventCreateWithFlags(&h.ev_mask[i], cudaEventDisableTiming));
      if (!h.ev_chunk[i]) ILS_CU(cudaEventCreateWithFlags(&h.ev_chunk[i], cudaEventDisableTiming));
    }
    // the auxiliary stream starts behind everything queued so far (workspace, earlier solves)
    ILS_CU(cudaEventRecord(h.ev_chunk[0], st));
    ILS_CU(cudaStreamWaitEvent(h.aux, h.ev_chunk[0], 0));
    const int64_t t1 = (span < max_inner) ? span : max_inner;
    const int rm = launch_masks(h.aux, seed, (uint32_t)k, 0, t1, nn, alpha_mode, alpha_k, nt, V, mbuf[0]);
    if (rm) return rm;
    ILS_CU(cudaEventRecord(h.ev_mask[0], h.aux));
  }
  int64_t ci = 0;   // chunk index
  while (t < max_inner) {
    const int64_t t1 = (t + span < max_inner) ? t + span : max_inner;
    const int b = (int)(ci & 1);
    if (use_masks && !overlap) {
      const int rm = launch_masks(st, seed, (uint32_t)k, t, t1, nn, alpha_mode, alpha_k, nt, V, mbuf[0]);
      if (rm) return rm;
    }
    if (overlap) {
      if (t1 < max_inner) {   // masks of chunk ci + 1 into the other buffer, once chunk ci - 1 has read it
        const int64_t t2 = (t1 + span < max_inner) ? t1 + span : max_inner;
        if (ci >= 1) ILS_CU(cudaStreamWaitEvent(h.aux, h.ev_chunk[b ^ 1], 0));
        const int rm = launch_masks(h.aux, seed, (uint32_t)k, t1, t2, nn, alpha_mode, alpha_k, nt, V, mbuf[b ^ 1]);
        if (rm) return rm;
        ILS_CU(cudaEventRecord(h.ev_mask[b ^ 1], h.aux));
      }
      ILS_CU(cudaStreamWaitEvent(st, h.ev_mask[b], 0));
      p.masks = mbuf[b];
    }
    p.t0 = t;
    p.t1 = t1;
    void* args[] = {&p};
    ILS_CU(cudaLaunchKernel(kern, dim3(1), dim3(nt), args, smem, st));
    ILS_LAUNCHED(warpk ? "scd_warp_kernel" : "scd_chunk_kernel");
    if (overlap) ILS_CU(cudaEventRecord(h.ev_chunk[b], st));
    ++ci;
    t = t1;
    if (t % ce == 0) {
      double itol = inner_tol;
      int64_t tn = t;
      // small n: one CTA (no grid barrier); else the cooperative full-GPU check
      const unsigned grid = (h.n <= 512) ? 1u : (unsigned)nchk;
      void* cargs[] = {(void*)&Gp, (void*)&npad, (void*)&nn, (void*)&bhat, (void*)&Bv, (void*)&Rv,
                       (void*)&rtmp, (void*)&red, (void*)&itol, (void*)&tn, (void*)&dst};
      ILS_CU(cudaLaunchCooperativeKernel((void*)scd_check_kernel, dim3(grid), dim3(256), cargs, 0, st));
      ILS_LAUNCHED("scd_check_kernel");
    }
    if (++pending == kBatch || t >= max_inner) {
      ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
      ILS_CU(cudaStreamSynchronize(st));
      pending = 0;
      if (h.hstat->inner_conv) break;
    }
  }
  if (overlap) {   // the last masks launch may be one chunk ahead of a stop: the handle's stream follows it
    ILS_CU(cudaEventRecord(h.ev_mask[0], h.aux));
    ILS_CU(cudaStreamWaitEvent(st, h.ev_mask[0], 0));
  }
  ILS_CU(cudaEventRecord(h.evk1, st));
  ILS_CU(cudaMemsetAsync(beta, 0, h.npad * sizeof(double), st));
  ILS_CU(cudaMemcpyAsync(beta, Bv, h.n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
  ILS_CU(cudaStreamSynchronize(st));
  const int64_t steps = h.hstat->inner_conv ? h.hstat->inner_steps : max_inner;
  if (steps_out) *steps_out = steps;
  const double nd = (double)h.n;
  hot_account(h, 2, (double)steps * 8.0 * nd + (double)(steps / ce) * 8.0 * nd * nd, (steps + ce - 1) / ce);
  return ILS_OK;
}

__global__ void scd_subset_exact_kernel(int n, uint64_t seed, uint32_t k, uint64_t t, int alpha_mode, int alpha_k,
                                        int32_t* alpha_out, uint8_t* mask) {
  extern __shared__ uint32_t ukeys[];
  uint32_t* hist = ukeys + n;
  __shared__ ScdKey e;
  __shared__ uint32_t T_s;
  __shared__ int need_s;
  if (threadIdx.x == 0) scd_make_key(seed, k, t, n, alpha_mode, alpha_k, 0, nullptr, e);
  subset_keys_block(seed, k, t, n, ukeys);
  __syncthreads();
  subset_select(ukeys, n, e.alpha, hist, &T_s, &need_s);
  for (int s = threadIdx.x; s < n; s += blockDim.x) mask[s] = subset_member(ukeys, n, s, T_s, need_s) ? 1 : 0;
  if (threadIdx.x == 0) *alpha_out = (int32_t)e.alpha;
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
  if (alpha_mode & ILS_SUBSET_EXACT) {
    const size_t smem = ((size_t)n + 258) * sizeof(uint32_t);
    if (smem > 200 * 1024) return ILS_ERR_UNSUPPORTED;
    ILS_CU(cudaFuncSetAttribute(scd_subset_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    scd_subset_exact_kernel<<<1, 256, smem, st>>>((int)n, seed, (uint32_t)k, (uint64_t)t, alpha_mode, alpha_k,
                                                  alpha_dev, mask_dev);
    ILS_LAUNCHED("scd_subset_exact_kernel");
    return ILS_OK;
  }
  scd_subset_kernel<<<32, 256, 0, st>>>((int)n, seed, (uint32_t)k, (uint64_t)t, alpha_mode, alpha_k,
                                        alpha_dev, mask_dev);
  ILS_LAUNCHED("scd_subset_kernel");
  return ILS_OK;
}

}  // namespace ils
