// batched.cu -- K4: many independent small ILS instances, one CTA (one warp) per instance.
//
// Each CTA runs a complete solve of its instance with shared-memory-resident A1 (column-major):
//   method 0  SP         (Alg. 1): Gram, Cholesky, explicit P, x <- P c_k
//   method 1  SP-RK-RGS  (Alg. 2)
//   method 2  SP-SCD     (Alg. 5); weighted = SP-RCD
// n <= 32: lane j owns coordinate j of x, c, z, beta, r (SCD); every reduction is a warp shuffle;
// no block, cluster or grid synchronisation. Instance i uses seed + i (include/ils.h).
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "ils_internal.h"

namespace ils {

struct BatchParams {
  const double* A;   // [batch][m][n]
  const double* b;   // [batch][m]
  int64_t batch;
  int p, q, n;
  const double* x0;    // [batch][n] or null
  double* x;           // [batch][n]
  const double* xref;  // [batch][n] or null
  double tol;
  int64_t max_iter;
  int stop, method;
  double inner_tol;
  int64_t max_inner, check_every;
  uint64_t seed;
  int alpha_mode, alpha_k, weighted;
  int64_t* inst_iters;
  int32_t* inst_status;
  unsigned long long* inner_total;
  int32_t* err;        // set when an instance's A1^T A1 has a non-positive or non-finite pivot (SP)
};

struct BKey {
  uint32_t alpha;
  int32_t j;
  uint32_t key[kFeistelRounds];
};

// batched SP-SCD window entry: alpha_t and the Feistel round tables T_r[v] = F(v, K_r) of step t,
// packed 4 bits per entry (n <= 32: h <= 3, 8 entries per round)
struct __align__(16) BKeyT {
  uint32_t tb[2 * kFeistelRounds];   // round r: T_r[v] in byte v of (tb[2r], tb[2r+1]) (PRMT lookup)
  uint32_t alpha;
  int32_t j;
  uint32_t pad_[2];
};
static_assert(sizeof(BKeyT) % 16 == 0, "BKeyT rows are read as uint4");

__device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

template <int UP>
__global__ void __launch_bounds__(32) batched_kernel(BatchParams P) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x;
  const int64_t inst = blockIdx.x;
  const int p = P.p, q = P.q, n = P.n, m = p + q;
  const double* A = P.A + inst * (int64_t)m * n;
  const double* b = P.b + inst * (int64_t)m;
  const uint64_t seed = P.seed + (uint64_t)inst;
  double* A1T = sm;                       // [n][p]
  double* G = A1T + n * p;                // [n][n]  Gram, then P (SP)
  double* az = G + n * n;                 // [p]
  uint64_t* S = reinterpret_cast<uint64_t*>(az + p);   // [32]
  BKey* keys = reinterpret_cast<BKey*>(S + 32);        // [32]

  for (int e = lane; e < n * p; e += 32) {
    const int j = e / p, i = e % p;
    A1T[e] = A[(int64_t)i * n + j];
  }
  __syncwarp();
  const bool act = lane < n;
  // N_j sequential in i without FMA (include/ils.h), A1^T b1
  double Nj = 0.0, a1tb1 = 0.0;
  if (act) {
    for (int i = 0; i < p; ++i) {
      const double v = A1T[lane * p + i];
      Nj = __dadd_rn(Nj, __dmul_rn(v, v));
      a1tb1 = fma(v, b[i], a1tb1);
    }
  }
  double x = (act && P.x0) ? P.x0[inst * n + lane] : 0.0;
  const double xr = (act && P.xref) ? P.xref[inst * n + lane] : 0.0;
  double xr2 = warp_sum(xr * xr);

  if (P.method == 1 || P.weighted) {   // weights for the column-norm sampler
    double mx = act ? Nj : 0.0;
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    uint64_t w = 0;
    if (act) {
      const uint64_t f = (uint64_t)floor(scalbn(__ddiv_rn(Nj, mx), 32));
      w = f < 1 ? 1 : f;
    }
    for (int o = 1; o < 32; o <<= 1) {   // inclusive warp scan (exact integers)
      const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    S[lane] = w;
  }
  if (P.method != 1) {   // Gram A1bar (lane j: column j)
    if (act) {
      for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int k = 0; k < p; ++k) s = fma(A1T[i * p + k], A1T[lane * p + k], s);
        G[i * n + lane] = s;
      }
    }
  }
  __syncwarp();
  if (P.method == 0) {
    // Cholesky (lower, in place in G), then P = L^{-T} L^{-1}: lane c solves column c.
    bool spd = true;
    for (int k = 0; k < n; ++k) {
      const double piv = G[k * n + k];
      spd = spd && piv > 0.0 && isfinite(piv);   // include/ils.h: ILS_ERR_NOT_SPD on breakdown
      __syncwarp();
      if (lane == 0) G[k * n + k] = sqrt(piv);
      __syncwarp();
      const double d = G[k * n + k];
      if (act && lane > k) G[lane * n + k] /= d;
      __syncwarp();
      if (act && lane > k)
        for (int j = k + 1; j <= lane; ++j) G[lane * n + j] -= G[lane * n + k] * G[j * n + k];
      __syncwarp();
    }
    if (!spd) {
      if (lane == 0) {
        atomicExch(P.err, 1);
        if (P.inst_status) P.inst_status[inst] = -1;
      }
      return;
    }
    double y[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) y[i] = 0.0;
    if (act) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (i < n) {
          double s = (i == lane) ? 1.0 : 0.0;
          for (int k = 0; k < i; ++k) s -= G[i * n + k] * y[k];
          y[i] = s / G[i * n + i];
        }
      }
#pragma unroll
      for (int i = 31; i >= 0; --i) {
        if (i < n) {
          double s = y[i];
          for (int k = i + 1; k < n; ++k) s -= G[k * n + i] * y[k];
          y[i] = s / G[i * n + i];
        }
      }
    }
    __syncwarp();
    if (act)
      for (int i = 0; i < n; ++i) G[i * n + lane] = y[i];   // P[i][lane] (symmetric)
    __syncwarp();
  }

  int64_t it = 0;
  int conv = 0;
  unsigned long long inner_sum = 0;
  for (; it < P.max_iter; ++it) {
    // c_k = A1^T b1 + A2^T (A2 x_k - b2)  (Alg. 2 step 5)
    double c = a1tb1;
    for (int i0 = 0; i0 < q; i0 += 32) {
      const int i = i0 + lane;
      double d = 0.0;
      if (i < q) {
        const double* ar = A + (int64_t)(p + i) * n;
        for (int j = 0; j < n; ++j) d = fma(ar[j], shfl(x, j), d);
        d -= b[p + i];
      } else {
        for (int j = 0; j < n; ++j) (void)shfl(x, j);
      }
      const int cnt = (q - i0 < 32) ? q - i0 : 32;
      for (int ii = 0; ii < cnt; ++ii) {
        const double di = shfl(d, ii);
        if (act) c = fma(A[(int64_t)(p + i0 + ii) * n + lane], di, c);
      }
    }
    double xn = 0.0;
    if (P.method == 0) {
      for (int i = 0; i < n; ++i) {
        const double ci = shfl(c, i);
        if (act) xn = fma(G[i * n + lane], ci, xn);
      }
    } else {
      const double cn2 = warp_sum(act ? c * c : 0.0);
      const double cnorm = sqrt(cn2);
      int64_t steps = 0;
      if (cnorm != 0.0 && P.method == 1) {
        // ---- SP-RK-RGS inner (Alg. 2 steps 6-12)
        double w[UP], r[UP];
#pragma unroll
        for (int u = 0; u < UP; ++u) w[u] = r[u] = 0.0;
        double z = 0.0;
        int my1 = 0, my2 = 0;
        for (int64_t t = 0; t < P.max_inner; ++t) {
          if ((t & 31) == 0) {
            const U4 xw = draw(seed, (uint32_t)it, (uint64_t)(t + lane), kTagRkRgs);
            my1 = sample_weighted_small(((uint64_t)xw.y << 32) | xw.x, S, n);
            my2 = sample_weighted_small(((uint64_t)xw.w << 32) | xw.z, S, n);
          }
          const int j1 = __shfl_sync(0xffffffffu, my1, (int)(t & 31));
          const int j2 = __shfl_sync(0xffffffffu, my2, (int)(t & 31));
          const double* a1 = A1T + j1 * p;
          const double* a2 = A1T + j2 * p;
          double d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
          for (int u = 0; u < UP; ++u) {
            const int i = lane + 32 * u;
            if (i < p) {
              const double x1 = a1[i], x2 = a2[i];
              d1 = fma(x1, w[u], d1);
              d2 = fma(x2, r[u], d2);
              d3 = fma(x2, x1, d3);
            }
          }
          d1 = warp_sum(d1);
          d2 = warp_sum(d2);
          d3 = warp_sum(d3);
          const double cj1 = shfl(c, j1), n1 = shfl(Nj, j1), n2 = shfl(Nj, j2);
          const double s1 = (cj1 - d1) / n1;
          const double s2 = (d2 + s1 * d3) / n2;
#pragma unroll
          for (int u = 0; u < UP; ++u) {
            const int i = lane + 32 * u;
            if (i < p) {
              const double x1 = a1[i], x2 = a2[i];
              w[u] = fma(s1, x1, w[u]);
              r[u] = fma(s1, x1, r[u]);
              r[u] = fma(-s2, x2, r[u]);
            }
          }
          if (lane == j2) z += s2;
          steps = t + 1;
          if ((t + 1) % P.check_every == 0) {
#pragma unroll
            for (int u = 0; u < UP; ++u) {
              const int i = lane + 32 * u;
              double a = 0.0;
              for (int j = 0; j < n; ++j) {
                const double zj = shfl(z, j);
                if (i < p) a = fma(A1T[j * p + i], zj, a);
              }
              if (i < p) az[i] = a;
            }
            __syncwarp();
            double g = 0.0;
            if (act) {
              for (int i = 0; i < p; ++i) g = fma(A1T[lane * p + i], az[i], g);
              g -= c;
            }
            __syncwarp();
            const double g2 = warp_sum(act ? g * g : 0.0);
            if (sqrt(g2) <= P.inner_tol * cnorm) break;
          }
        }
        xn = z;
      } else if (cnorm != 0.0) {
        // ---- SP-SCD / SP-RCD inner (Alg. 5 steps 5-12)
        double rr = act ? c : 0.0, beta = 0.0;
        const uint32_t hb = feistel_half_bits((uint32_t)n), msk = (1u << hb) - 1u;
        for (int64_t t = 0; t < P.max_inner; ++t) {
          if ((t & 31) == 0) {
            BKey e;
            const uint64_t tt = (uint64_t)(t + lane);
            if (P.weighted) {
              const U4 xw = draw(seed, (uint32_t)it, tt, kTagRcd);
              e.j = sample_weighted_small(((uint64_t)xw.y << 32) | xw.x, S, n);
              e.alpha = 1;
            } else {
              const U4 a = draw(seed, (uint32_t)it, tt, kTagScdA);
              const U4 bb = draw(seed, (uint32_t)it, tt, kTagScdB);
            const U4 cc = draw(seed, (uint32_t)it, tt, kTagScdC);
              e.alpha = P.alpha_mode == ILS_ALPHA_UNIFORM ? 1u + mulhi32(a.x, (uint32_t)n)
                                                          : (uint32_t)(P.alpha_k < n ? P.alpha_k : n);
              e.j = -1;
              e.key[0] = a.y; e.key[1] = a.z; e.key[2] = a.w;
              e.key[3] = bb.x; e.key[4] = bb.y; e.key[5] = bb.z; e.key[6] = bb.w;
            e.key[7] = cc.x;
            }
            __syncwarp();
            keys[lane] = e;
            __syncwarp();
          }
          const BKey& e = keys[t & 31];
          int j;
          double rj;
          if (P.weighted) {
            j = e.j;
            rj = shfl(rr, j);
          } else {
            ArgMax best{-1.0, INT_MAX, 0.0};
            if (act) {
              const uint32_t mm = feistel_inverse((uint32_t)lane, e.key, hb, msk, (uint32_t)n);
              if (mm < e.alpha) best = ArgMax{rr * rr, lane, rr};
            }
            best = warp_argmax(best);
            j = best.idx;
            rj = best.pay;
          }
          const double sc = rj / shfl(Nj, j);
          if (act) rr = fma(-sc, G[j * n + lane], rr);
          if (lane == j) beta += sc;
          steps = t + 1;
          if ((t + 1) % P.check_every == 0) {
            double a = 0.0;
            for (int jj = 0; jj < n; ++jj) {
              const double bj = shfl(beta, jj);
              if (act) a = fma(G[jj * n + lane], bj, a);
            }
            rr = act ? c - a : 0.0;
            const double r2 = warp_sum(rr * rr);
            if (sqrt(r2) <= P.inner_tol * cnorm) break;
          }
        }
        xn = beta;
      }
      inner_sum += (unsigned long long)steps;
    }
    x = act ? xn : 0.0;
    // stop test (XREF)
    const double e = act ? x - xr : 0.0;
    const double e2 = warp_sum(e * e);
    if (P.stop == ILS_STOP_XREF && P.xref && sqrt(e2) <= P.tol * sqrt(xr2)) {
      conv = 1;
      ++it;
      break;
    }
  }
  if (act) P.x[inst * n + lane] = x;
  if (lane == 0) {
    if (P.inst_iters) P.inst_iters[inst] = it;
    if (P.inst_status) P.inst_status[inst] = conv;
    atomicAdd(P.inner_total, inner_sum);
  }
}

// ---------------------------------------------------------------------------------------------
// Specialised batched kernels (one warp per instance, lane j = coordinate j, n <= 32).
// Shared pieces: per-instance prologue (column norms, A1^T b1, sampling table) and the outer
// right-hand side c_k = A1^T b1 + A2^T (A2 x_k - b2) (Alg. 2 step 5 / Alg. 5 step 4).

// c_k for the warp's instance: lane j returns c_j (A2 rows read from global / L2).
__device__ __forceinline__ double batched_rhs(const double* __restrict__ A, const double* __restrict__ b, int p,
                                              int q, int n, double x, double a1tb1, int lane) {
  const bool act = lane < n;
  double c = a1tb1;
  for (int i0 = 0; i0 < q; i0 += 32) {
    const int i = i0 + lane;
    double d = 0.0;
    const double* ar = A + (int64_t)(p + (i < q ? i : 0)) * n;
    for (int j = 0; j < n; ++j) d = fma(ar[j], __shfl_sync(0xffffffffu, x, j), d);
    d = (i < q) ? d - b[p + i] : 0.0;
    const int cnt = (q - i0 < 32) ? q - i0 : 32;
    for (int ii = 0; ii < cnt; ++ii) {
      const double di = __shfl_sync(0xffffffffu, d, ii);
      if (act) c = fma(A[(int64_t)(p + i0 + ii) * n + lane], di, c);
    }
  }
  return c;
}

// inclusive prefix sums of the integer column weights W_j = max(1, floor(N_j / N_max * 2^32))
// (include/ils.h) into S[0..31] (lanes >= n contribute 0)
__device__ __forceinline__ void batched_weights(double Nj, bool act, int lane, uint64_t* S) {
  double mx = act ? Nj : 0.0;
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  uint64_t w = 0;
  if (act) {
    const uint64_t f = (uint64_t)floor(scalbn(__ddiv_rn(Nj, mx), 32));
    w = f < 1 ? 1 : f;
  }
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
    if (lane >= o) w += y;
  }
  S[lane] = w;
}

// SP-RK-RGS, batched (Alg. 2). A1 is shared-memory resident, column-major with
// rows padded to 32*RPL (zero rows), so the per-step loops carry no bounds. Per step: indices from
// a 32-step register window (lane l drew step t0+l: Philox, inverse CDF on S, b_hat_{j1}, 1/N),
// broadcast by shuffles; three dots over RPL rows per lane; three butterfly warp sums; reciprocal
// multiplies; axpys from the values still in registers. Inner check every check_every steps.
template <int RPL>
__global__ void __launch_bounds__(32) batched_rk_kernel(BatchParams P) {
  extern __shared__ __align__(16) double sm[];
  constexpr int PP = 32 * RPL;
  const int lane = threadIdx.x;
  const int64_t inst = blockIdx.x;
  const int p = P.p, q = P.q, n = P.n, m = p + q;
  const double* A = P.A + inst * (int64_t)m * n;
  const double* b = P.b + inst * (int64_t)m;
  const uint64_t seed = P.seed + (uint64_t)inst;
  double* A1T = sm;                                     // [n][PP]
  double* azs = A1T + n * PP;                           // [PP]
  double* cs = azs + PP;                                // [32] c_k (for b_hat_{j1} lookups)
  double* rns = cs + 32;                                // [32] 1 / N_j
  uint64_t* S = reinterpret_cast<uint64_t*>(rns + 32);  // [32]

  for (int e = lane; e < n * PP; e += 32) {
    const int j = e / PP, i = e % PP;
    A1T[e] = (i < p) ? A[(int64_t)i * n + j] : 0.0;
  }
  __syncwarp();
  const bool act = lane < n;
  double Nj = 0.0, a1tb1 = 0.0;
  if (act) {
    for (int i = 0; i < p; ++i) {   // N_j sequential in i without FMA (include/ils.h)
      const double v = A1T[lane * PP + i];
      Nj = __dadd_rn(Nj, __dmul_rn(v, v));
      a1tb1 = fma(v, b[i], a1tb1);
    }
  }
  batched_weights(Nj, act, lane, S);
  rns[lane] = act ? 1.0 / Nj : 0.0;
  double x = (act && P.x0) ? P.x0[inst * n + lane] : 0.0;
  const double xr = (act && P.xref) ? P.xref[inst * n + lane] : 0.0;
  const double xr2 = warp_sum(xr * xr);
  __syncwarp();

  const int64_t ce = P.check_every;
  int64_t it = 0;
  int conv = 0;
  unsigned long long inner_sum = 0;
  for (; it < P.max_iter; ++it) {
    const double c = batched_rhs(A, b, p, q, n, x, a1tb1, lane);
    cs[lane] = act ? c : 0.0;
    const double cnorm = sqrt(warp_sum(act ? c * c : 0.0));
    __syncwarp();
    double z = 0.0;
    int64_t steps = 0;
    if (cnorm != 0.0) {
      double w[RPL], r[RPL];
#pragma unroll
      for (int u = 0; u < RPL; ++u) w[u] = r[u] = 0.0;
      int my1 = 0, my2 = 0;
      double mybh = 0.0, myr1 = 0.0, myr2 = 0.0;
      int64_t next_check = ce;
      for (int64_t t = 0; t < P.max_inner; ++t) {
        const int kk = (int)(t & 31);
        if (kk == 0) {   // indices and scalars of steps t..t+31, one per lane
          const U4 xw = draw(seed, (uint32_t)it, (uint64_t)(t + lane), kTagRkRgs);
          my1 = sample_weighted_small(((uint64_t)xw.y << 32) | xw.x, S, n);
          my2 = sample_weighted_small(((uint64_t)xw.w << 32) | xw.z, S, n);
          mybh = cs[my1];
          myr1 = rns[my1];
          myr2 = rns[my2];
        }
        const int j1 = __shfl_sync(0xffffffffu, my1, kk);
        const int j2 = __shfl_sync(0xffffffffu, my2, kk);
        const double bh1 = __shfl_sync(0xffffffffu, mybh, kk);
        const double rn1 = __shfl_sync(0xffffffffu, myr1, kk);
        const double rn2 = __shfl_sync(0xffffffffu, myr2, kk);
        const double* a1 = A1T + j1 * PP + lane;
        const double* a2 = A1T + j2 * PP + lane;
        double x1[RPL], x2[RPL];
        double d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          x1[u] = a1[32 * u];
          x2[u] = a2[32 * u];
          d1 = fma(x1[u], w[u], d1);
          d2 = fma(x2[u], r[u], d2);
          d3 = fma(x2[u], x1[u], d3);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          d1 += __shfl_xor_sync(0xffffffffu, d1, o);
          d2 += __shfl_xor_sync(0xffffffffu, d2, o);
          d3 += __shfl_xor_sync(0xffffffffu, d3, o);
        }
        const double s1 = (bh1 - d1) * rn1;
        const double s2 = (d2 + s1 * d3) * rn2;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          w[u] = fma(s1, x1[u], w[u]);
          r[u] = fma(s1, x1[u], r[u]);
          r[u] = fma(-s2, x2[u], r[u]);
        }
        if (lane == j2) z += s2;
        steps = t + 1;
        if (steps == next_check) {   // inner stop rule (include/ils.h): g = A1^T A1 z - b_hat
          next_check += ce;
          double az[RPL];
#pragma unroll
          for (int u = 0; u < RPL; ++u) az[u] = 0.0;
          double az2[RPL];   // second accumulator: halves the dependent FMA chain
#pragma unroll
          for (int u = 0; u < RPL; ++u) az2[u] = 0.0;
          int j = 0;
          for (; j + 1 < n; j += 2) {
            const double zj = __shfl_sync(0xffffffffu, z, j), zk = __shfl_sync(0xffffffffu, z, j + 1);
#pragma unroll
            for (int u = 0; u < RPL; ++u) {
              az[u] = fma(A1T[j * PP + lane + 32 * u], zj, az[u]);
              az2[u] = fma(A1T[(j + 1) * PP + lane + 32 * u], zk, az2[u]);
            }
          }
          if (j < n) {
            const double zj = __shfl_sync(0xffffffffu, z, j);
#pragma unroll
            for (int u = 0; u < RPL; ++u) az[u] = fma(A1T[j * PP + lane + 32 * u], zj, az[u]);
          }
#pragma unroll
          for (int u = 0; u < RPL; ++u) az[u] += az2[u];
#pragma unroll
          for (int u = 0; u < RPL; ++u) {
            azs[lane + 32 * u] = az[u];
          }
          __syncwarp();
          double g = 0.0;
          if (act) {   // four accumulators over the (zero-padded) rows
            double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
            const double* col = A1T + lane * PP;
            for (int i = 0; i < PP; i += 4) {
              g0 = fma(col[i], azs[i], g0);
              g1 = fma(col[i + 1], azs[i + 1], g1);
              g2 = fma(col[i + 2], azs[i + 2], g2);
              g3 = fma(col[i + 3], azs[i + 3], g3);
            }
            g = ((g0 + g1) + (g2 + g3)) - c;
          }
          __syncwarp();
          const double g2 = warp_sum(act ? g * g : 0.0);
          if (sqrt(g2) <= P.inner_tol * cnorm) break;
        }
      }
    }
    inner_sum += (unsigned long long)steps;
    x = act ? z : 0.0;
    const double e = act ? x - xr : 0.0;
    const double e2 = warp_sum(e * e);
    if (P.stop == ILS_STOP_XREF && P.xref && sqrt(e2) <= P.tol * sqrt(xr2)) {
      conv = 1;
      ++it;
      break;
    }
  }
  if (act) P.x[inst * n + lane] = x;
  if (lane == 0) {
    if (P.inst_iters) P.inst_iters[inst] = it;
    if (P.inst_status) P.inst_status[inst] = conv;
    atomicAdd(P.inner_total, inner_sum);
  }
}

// SP-SCD / SP-RCD, batched (Alg. 5). A1bar (n x n) is shared-memory resident
// (formed once per instance from A1 rows read through L1/L2), so an instance needs ~10 KB and ~20
// instances share an SM. Per step: the 12 Feistel round keys and alpha_t come from a 32-step key
// window in shared memory; lane s tests pi^{-1}(s) < alpha_t; warp argmax of r_s^2 (ties to the
// smallest s); r -= (r_j / A1bar_jj) A1bar_(j) from shared memory.
// Template flags: WT = weighted SP-RCD, N32 = n is 32 (every lane owns a coordinate and the Feistel
// domain is [0, 64): the generic n checks fold away).
template <bool WT, bool N32>
__global__ void __launch_bounds__(32) batched_scd_kernel(BatchParams P) {
  extern __shared__ __align__(16) double sm[];
  const int lane = threadIdx.x;
  const int64_t inst = blockIdx.x;
  const int p = P.p, q = P.q, n = N32 ? 32 : P.n, m = p + q;
  const double* A = P.A + inst * (int64_t)m * n;
  const double* b = P.b + inst * (int64_t)m;
  const uint64_t seed = P.seed + (uint64_t)inst;
  double* G = sm;                                       // [32][32] A1bar (row j at G + 32 j)
  uint64_t* S = reinterpret_cast<uint64_t*>(G + 32 * 32);   // [32]
  BKeyT* keys = reinterpret_cast<BKeyT*>(S + 32);             // [32]
  const bool act = N32 || lane < n;
  // column j of A1 in registers one row at a time: Gram by rank-1 updates over the p rows
  double g[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) g[i] = 0.0;
  double Nj = 0.0, a1tb1 = 0.0;
  for (int k = 0; k < p; ++k) {
    const double v = act ? A[(int64_t)k * n + lane] : 0.0;
    Nj = __dadd_rn(Nj, __dmul_rn(v, v));   // N_j sequential in i without FMA (include/ils.h)
    a1tb1 = fma(v, b[k], a1tb1);
#pragma unroll
    for (int i = 0; i < 32; ++i) g[i] = fma(__shfl_sync(0xffffffffu, v, i), v, g[i]);
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) G[i * 32 + lane] = g[i];   // G[i][lane] (symmetric)
  if (WT) batched_weights(Nj, act, lane, S);
  const double rn = act ? 1.0 / Nj : 0.0;
  double x = (act && P.x0) ? P.x0[inst * n + lane] : 0.0;
  const double xr = (act && P.xref) ? P.xref[inst * n + lane] : 0.0;
  const double xr2 = warp_sum(xr * xr);
  const uint32_t hb = N32 ? 3u : feistel_half_bits((uint32_t)n), msk = (1u << hb) - 1u;
  __syncwarp();

  const int64_t ce = P.check_every;
  int64_t it = 0;
  int conv = 0;
  unsigned long long inner_sum = 0;
  for (; it < P.max_iter; ++it) {
    const double c = batched_rhs(A, b, p, q, n, x, a1tb1, lane);
    const double cnorm = sqrt(warp_sum(act ? c * c : 0.0));
    double rr = act ? c : 0.0, beta = 0.0;
    int64_t steps = 0;
    if (cnorm != 0.0) {
      int64_t next_check = ce;
      for (int64_t t = 0; t < P.max_inner; ++t) {
        const int kk = (int)(t & 31);
        if (kk == 0) {
          BKeyT e;
          const uint64_t tt = (uint64_t)(t + lane);
          if (WT) {
            const U4 xw = draw(seed, (uint32_t)it, tt, kTagRcd);
            e.j = sample_weighted_small(((uint64_t)xw.y << 32) | xw.x, S, n);
            e.alpha = 1;
          } else {
            const U4 a = draw(seed, (uint32_t)it, tt, kTagScdA);
            const U4 bb = draw(seed, (uint32_t)it, tt, kTagScdB);
            const U4 cc = draw(seed, (uint32_t)it, tt, kTagScdC);
            e.alpha = P.alpha_mode == ILS_ALPHA_UNIFORM ? 1u + mulhi32(a.x, (uint32_t)n)
                                                        : (uint32_t)(P.alpha_k < n ? P.alpha_k : n);
            e.j = -1;
            const uint32_t key[kFeistelRounds] = {a.y, a.z, a.w, bb.x, bb.y, bb.z, bb.w, cc.x};
            // round tables of this lane's step: T_r[v] = mix32(v ^ K_r) & (2^hb - 1) for v < 2^hb
            // (hb <= 3 for n <= 32), one byte per entry in two words, so that a decryption round is one
            // byte permute (PRMT) and one three-input logic op
#pragma unroll
            for (int r = 0; r < kFeistelRounds; ++r) {
              uint32_t w0 = 0, w1 = 0;
#pragma unroll
              for (uint32_t v = 0; v < 4; ++v) {
                if (v <= msk) w0 |= (mix32(v ^ key[r]) & msk) << (8 * v);
                if (v + 4 <= msk) w1 |= (mix32((v + 4) ^ key[r]) & msk) << (8 * v);
              }
              e.tb[2 * r] = w0;
              e.tb[2 * r + 1] = w1;
            }
          }
          __syncwarp();
          keys[lane] = e;
          __syncwarp();
        }
        int j;
        if (WT) {
          j = keys[kk].j;
        } else {
          uint32_t tb[2 * kFeistelRounds];
          {
            const uint4* kq = reinterpret_cast<const uint4*>(keys[kk].tb);
#pragma unroll
            for (int qq = 0; qq < kFeistelRounds / 2; ++qq) {
              const uint4 w = kq[qq];
              tb[4 * qq] = w.x;
              tb[4 * qq + 1] = w.y;
              tb[4 * qq + 2] = w.z;
              tb[4 * qq + 3] = w.w;
            }
          }
          const uint32_t alpha = keys[kk].alpha;
          // one round-trip decryption of y (feistel_decrypt_once) from the byte round tables
          auto dec = [&](uint32_t y) {
            uint32_t L = y >> hb, R = y & msk;
#pragma unroll
            for (int r = kFeistelRounds - 1; r >= 0; --r) {
              const uint32_t Lp = (R ^ __byte_perm(tb[2 * r], tb[2 * r + 1], L)) & msk;
              R = L;
              L = Lp;
            }
            return (L << hb) | R;
          };
          // pi^{-1}(lane) by cycle walking through a table of one-round-trip decryptions of the
          // whole domain [0, 4^hb) (<= 64 values: lane v holds D(v) and D(v + 32)); a walk step is
          // then two shuffles instead of a decryption (the walk diverges across lanes)
          const uint32_t dom = 1u << (2 * hb);
          const bool allm = alpha >= (uint32_t)n;   // tau_t = [n] (Motzkin case): no permutation needed
          const uint32_t d0 = (n == 1 || allm) ? 0u : dec((uint32_t)lane & (dom - 1));
          const uint32_t d1 = (n == 1 || allm || dom <= 32) ? 0u : dec((uint32_t)lane + 32u);
          uint32_t y = d0;
          if (n > 1 && !allm) {
            // walk ends by pointer jumping (T(v) <- T(T(v)) while T(v) >= n, all v at once): three
            // uniform rounds resolve every walk of up to 8 hops; the rare longer ones finish below
            const uint32_t nu = (uint32_t)n;
            if (n == 32) {   // only the values 32..63 (slot 1, lane v - 32) are ever walked through
              uint32_t T1 = d1;
#pragma unroll
              for (int rnd = 0; rnd < 3; ++rnd) {
                const uint32_t f = __shfl_sync(0xffffffffu, T1, (int)(T1 & 31));
                T1 = (T1 >= 32u) ? f : T1;
              }
              const uint32_t f = __shfl_sync(0xffffffffu, T1, (int)(d0 & 31));
              y = (d0 >= 32u) ? f : d0;
            } else {
              uint32_t T0 = d0, T1 = d1;
#pragma unroll
              for (int rnd = 0; rnd < 3; ++rnd) {
                const uint32_t a0 = __shfl_sync(0xffffffffu, T0, (int)(T0 & 31));
                const uint32_t b0 = __shfl_sync(0xffffffffu, T1, (int)(T0 & 31));
                const uint32_t a1 = __shfl_sync(0xffffffffu, T0, (int)(T1 & 31));
                const uint32_t b1 = __shfl_sync(0xffffffffu, T1, (int)(T1 & 31));
                T0 = (T0 >= nu) ? ((T0 < 32u) ? a0 : b0) : T0;
                T1 = (T1 >= nu) ? ((T1 < 32u) ? a1 : b1) : T1;
              }
              y = T0;
            }
            while (__any_sync(0xffffffffu, act && y >= (uint32_t)n)) {
              const uint32_t t0 = __shfl_sync(0xffffffffu, d0, (int)(y & 31)), t1 = __shfl_sync(0xffffffffu, d1, (int)(y & 31));
              if (act && y >= (uint32_t)n) y = (y < 32) ? t0 : t1;
            }
          }
          double bv = 0.0;
          int bi = INT_MAX;
          if (act && y < alpha) {
            bv = rr * rr;
            bi = lane;
          }
          j = warp_argmax_redux(bv, bi);   // integer warp reductions, ties to the smallest index
        }
        const double sc = __shfl_sync(0xffffffffu, rr, j) * __shfl_sync(0xffffffffu, rn, j);
        if (act) rr = fma(-sc, G[j * 32 + lane], rr);
        beta += (lane == j) ? sc : 0.0;
        steps = t + 1;
        if (steps == next_check) {   // inner stop rule: r = b_hat - A1bar beta
          next_check += ce;
          double a = 0.0;
          for (int jj = 0; jj < n; ++jj) a = fma(G[jj * 32 + lane], __shfl_sync(0xffffffffu, beta, jj), a);
          rr = act ? c - a : 0.0;
          const double r2 = warp_sum(rr * rr);
          if (sqrt(r2) <= P.inner_tol * cnorm) break;
        }
      }
    }
    inner_sum += (unsigned long long)steps;
    x = act ? beta : 0.0;
    const double e = act ? x - xr : 0.0;
    const double e2 = warp_sum(e * e);
    if (P.stop == ILS_STOP_XREF && P.xref && sqrt(e2) <= P.tol * sqrt(xr2)) {
      conv = 1;
      ++it;
      break;
    }
  }
  if (act) P.x[inst * n + lane] = x;
  if (lane == 0) {
    if (P.inst_iters) P.inst_iters[inst] = it;
    if (P.inst_status) P.inst_status[inst] = conv;
    atomicAdd(P.inner_total, inner_sum);
  }
}

// SP-RK-RGS, batched, blocked: 4 steps per warp reduction (the identity of rk_rgs.cu's blocked
// kernel, Alg. 2 steps 9 and 11). Every Gram entry the 4-step recurrence needs (<a_i, a_k>,
// <b_i, a_k>, <b_i, b_k>) is looked up in the instance's A1bar (32 x 33, shared memory, formed once
// per solve), so a block reduces only the 8 state products <a_i, w>, <b_i, r> (butterfly
// reduce-scatter + broadcast: 16 shuffles per step-block instead of 30 per step).
template <int NVP>
__device__ __forceinline__ double bw_reduce_scatter(double (&x)[NVP], int lane) {
#pragma unroll
  for (int half = NVP / 2; half >= 1; half /= 2) {
    const bool hi = (lane & half) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double lo_v = x[i], hi_v = x[i + half];
      const double send = hi ? lo_v : hi_v;
      const double keep = hi ? hi_v : lo_v;
      x[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
    }
  }
  double v = x[0];
#pragma unroll
  for (int o = NVP; o < 32; o *= 2) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int RPL>
__global__ void __launch_bounds__(32) batched_rkb_kernel(BatchParams P) {
  constexpr int B = 4;
  extern __shared__ __align__(16) double sm[];
  constexpr int PP = 32 * RPL;
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x;
  const int64_t inst = blockIdx.x;
  const int p = P.p, q = P.q, n = P.n, m = p + q;
  const double* A = P.A + inst * (int64_t)m * n;
  const double* b = P.b + inst * (int64_t)m;
  const uint64_t seed = P.seed + (uint64_t)inst;
  double* A1T = sm;                                     // [n][PP]
  double* G = A1T + n * PP;                             // [32][33] A1bar
  double* cs = G + 32 * 33;                             // [32]
  double* rns = cs + 32;                                // [32]
  uint64_t* S = reinterpret_cast<uint64_t*>(rns + 32);  // [32]

  for (int e = lane; e < n * PP; e += 32) {
    const int j = e / PP, i = e % PP;
    A1T[e] = (i < p) ? A[(int64_t)i * n + j] : 0.0;
  }
  __syncwarp();
  const bool act = lane < n;
  double Nj = 0.0, a1tb1 = 0.0;
  if (act) {
    for (int i = 0; i < p; ++i) {   // N_j sequential in i without FMA (include/ils.h)
      const double v = A1T[lane * PP + i];
      Nj = __dadd_rn(Nj, __dmul_rn(v, v));
      a1tb1 = fma(v, b[i], a1tb1);
    }
  }
  // A1bar[i][lane] (rows rotated by lane: conflict-free shared-memory reads); rows and columns
  // >= n are zero (the inner check sums over 32 columns)
  for (int i = n; i < 32; ++i) G[i * 33 + lane] = 0.0;
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    if (act)
      for (int kk = 0, k = lane % p; kk < p; ++kk, k = (k + 1 == p) ? 0 : k + 1)
        s = fma(A1T[i * PP + k], A1T[lane * PP + k], s);
    G[i * 33 + lane] = act ? s : 0.0;
  }
  batched_weights(Nj, act, lane, S);
  rns[lane] = act ? 1.0 / Nj : 0.0;
  double x = (act && P.x0) ? P.x0[inst * n + lane] : 0.0;
  const double xr = (act && P.xref) ? P.xref[inst * n + lane] : 0.0;
  const double xr2 = warp_sum(xr * xr);
  __syncwarp();

  const int64_t ce = P.check_every;
  int64_t it = 0;
  int conv = 0;
  unsigned long long inner_sum = 0;
  for (; it < P.max_iter; ++it) {
    const double c = batched_rhs(A, b, p, q, n, x, a1tb1, lane);
    cs[lane] = act ? c : 0.0;
    const double cnorm = sqrt(warp_sum(act ? c * c : 0.0));
    __syncwarp();
    double z = 0.0;
    int64_t steps = 0;
    if (cnorm != 0.0) {
      double w[RPL], r[RPL];
#pragma unroll
      for (int u = 0; u < RPL; ++u) w[u] = r[u] = 0.0;
      int my1 = 0, my2 = 0;
      double mybh = 0.0, myr1 = 0.0, myr2 = 0.0;
      int64_t next_check = ce;
      for (int64_t t = 0; t < P.max_inner; t += B) {
        const int kk = (int)(t & 31);
        if (kk == 0) {   // indices and scalars of steps t..t+31, one per lane
          const U4 xw = draw(seed, (uint32_t)it, (uint64_t)(t + lane), kTagRkRgs);
          my1 = sample_weighted_small(((uint64_t)xw.y << 32) | xw.x, S, n);
          my2 = sample_weighted_small(((uint64_t)xw.w << 32) | xw.z, S, n);
          const bool live = t + lane < P.max_inner;   // steps past max_inner are masked: s1 = s2 = 0
          mybh = cs[my1];
          myr1 = live ? rns[my1] : 0.0;
          myr2 = live ? rns[my2] : 0.0;
        }
        int j1[B], j2[B];
        double bh[B], rn1[B], rn2[B];
#pragma unroll
        for (int i = 0; i < B; ++i) {
          j1[i] = __shfl_sync(FULL, my1, kk + i);
          j2[i] = __shfl_sync(FULL, my2, kk + i);
          bh[i] = __shfl_sync(FULL, mybh, kk + i);
          rn1[i] = __shfl_sync(FULL, myr1, kk + i);
          rn2[i] = __shfl_sync(FULL, myr2, kk + i);
        }
        double x1[B][RPL], x2[B][RPL];
        double acc[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[v] = 0.0;
#pragma unroll
        for (int i = 0; i < B; ++i) {
          const double* a1 = A1T + j1[i] * PP + lane;
          const double* a2 = A1T + j2[i] * PP + lane;
#pragma unroll
          for (int u = 0; u < RPL; ++u) {
            x1[i][u] = a1[32 * u];
            x2[i][u] = a2[32 * u];
            acc[i] = fma(x1[i][u], w[u], acc[i]);
            acc[B + i] = fma(x2[i][u], r[u], acc[B + i]);
          }
        }
        // Gram entries of the block (broadcast shared-memory reads, independent of the reduction)
        double AA[B][B], BA[B][B], BB[B][B];
#pragma unroll
        for (int i = 0; i < B; ++i)
#pragma unroll
          for (int k = 0; k < B; ++k) {
            AA[i][k] = (k < i) ? G[j1[i] * 33 + j1[k]] : 0.0;
            BA[i][k] = (k <= i) ? G[j2[i] * 33 + j1[k]] : 0.0;
            BB[i][k] = (k < i) ? G[j2[i] * 33 + j2[k]] : 0.0;
          }
        const double mine = bw_reduce_scatter<8>(acc, lane);   // lane l: total of value l & 7
        double T[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) T[v] = __shfl_sync(FULL, mine, v);
        double s1[B], s2[B];
#pragma unroll
        for (int i = 0; i < B; ++i) {
          double dw = T[i];
#pragma unroll
          for (int k = 0; k < i; ++k) dw = fma(s1[k], AA[i][k], dw);
          s1[i] = (bh[i] - dw) * rn1[i];
          double dr = T[B + i];
#pragma unroll
          for (int k = 0; k < i; ++k) {
            dr = fma(s1[k], BA[i][k], dr);
            dr = fma(-s2[k], BB[i][k], dr);
          }
          dr = fma(s1[i], BA[i][i], dr);
          s2[i] = dr * rn2[i];
        }
#pragma unroll
        for (int u = 0; u < RPL; ++u)
#pragma unroll
          for (int i = 0; i < B; ++i) {
            w[u] = fma(s1[i], x1[i][u], w[u]);
            r[u] = fma(s1[i], x1[i][u], r[u]);
            r[u] = fma(-s2[i], x2[i][u], r[u]);
          }
#pragma unroll
        for (int i = 0; i < B; ++i) z += (lane == j2[i]) ? s2[i] : 0.0;   // z_j2 += s2 (program order)
        steps = (t + B < P.max_inner) ? t + B : P.max_inner;
        if (t + B == next_check) {   // inner stop rule (include/ils.h): g = A1bar z - b_hat, reads z only
          next_check += ce;
          double g0 = 0.0, g1 = 0.0;   // row lane of A1bar (G[lane][k], stride 33: conflict-free)
#pragma unroll 8
          for (int k = 0; k < 32; k += 2) {
            g0 = fma(G[lane * 33 + k], __shfl_sync(FULL, z, k), g0);
            g1 = fma(G[lane * 33 + k + 1], __shfl_sync(FULL, z, k + 1), g1);
          }
          const double g = act ? (g0 + g1) - c : 0.0;
          const double gg = warp_sum(g * g);
          if (sqrt(gg) <= P.inner_tol * cnorm) break;
        }
      }
    }
    inner_sum += (unsigned long long)steps;
    x = act ? z : 0.0;
    const double e = act ? x - xr : 0.0;
    const double e2 = warp_sum(e * e);
    if (P.stop == ILS_STOP_XREF && P.xref && sqrt(e2) <= P.tol * sqrt(xr2)) {
      conv = 1;
      ++it;
      break;
    }
  }
  if (act) P.x[inst * n + lane] = x;
  if (lane == 0) {
    if (P.inst_iters) P.inst_iters[inst] = it;
    if (P.inst_status) P.inst_status[inst] = conv;
    atomicAdd(P.inner_total, inner_sum);
  }
}

int batched_solve(Handle& h, int method, const double* x0, double* x, double tol, int64_t max_iter,
                  const ils_opts& o, int64_t* inst_iters_dev, int32_t* inst_status_dev) {
  if (h.n > 32 || h.p > 256 || h.q > 4096) {
    set_error("batched path supports n <= 32, p <= 256");
    return ILS_ERR_UNSUPPORTED;
  }
  BatchParams P{};
  P.A = h.Ab;
  P.b = h.bb;
  P.batch = h.batch;
  P.p = (int)h.p;
  P.q = (int)h.q;
  P.n = (int)h.n;
  P.x0 = x0;
  P.x = x;
  P.xref = o.x_ref;
  P.tol = tol;
  P.max_iter = max_iter;
  P.stop = o.stop;
  P.method = method;
  P.inner_tol = o.inner_tol;
  P.max_inner = o.max_inner;
  P.check_every = o.check_every > 0 ? o.check_every : h.n;
  P.seed = o.seed;
  P.alpha_mode = o.alpha_mode;
  P.alpha_k = o.alpha_k;
  P.weighted = (method == 2) ? o.weighted : 0;
  P.inst_iters = inst_iters_dev;
  P.inst_status = inst_status_dev;
  P.inner_total = reinterpret_cast<unsigned long long*>(&h.dstat->inner_steps);
  P.err = &h.dstat->flag_err;
  if (method == 1 && P.check_every % 4 == 0 && !getenv("ILS_BATCHED_RK_SINGLE")) {   // blocked, 4 steps/reduction
    const int rpl = (int)((h.p + 31) / 32);
    const int RPL = rpl <= 1 ? 1 : rpl <= 2 ? 2 : rpl <= 3 ? 3 : rpl <= 4 ? 4 : 8;
    const size_t smem = ((size_t)h.n * 32 * RPL + 32 * 33 + 64) * 8 + 32 * 8;
#define RKBLAUNCH(RR)                                                                                \
  do {                                                                                               \
    ILS_CU(cudaFuncSetAttribute(batched_rkb_kernel<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    batched_rkb_kernel<RR><<<(unsigned)h.batch, 32, smem, h.stream>>>(P);                            \
    ILS_LAUNCHED("batched_rkb_kernel");                                                              \
  } while (0)
    switch (RPL) {
      case 1: RKBLAUNCH(1); break;
      case 2: RKBLAUNCH(2); break;
      case 3: RKBLAUNCH(3); break;
      case 4: RKBLAUNCH(4); break;
      default: RKBLAUNCH(8); break;
    }
#undef RKBLAUNCH
    return ILS_OK;
  }
  if (method == 1) {   // SP-RK-RGS: A1 resident, rows padded to 32*RPL
    const int rpl = (int)((h.p + 31) / 32);
    const int RPL = rpl <= 1 ? 1 : rpl <= 2 ? 2 : rpl <= 3 ? 3 : rpl <= 4 ? 4 : 8;
    const size_t smem = ((size_t)h.n * 32 * RPL + 32 * RPL + 64) * 8 + 32 * 8;
#define RKLAUNCH(RR)                                                                                 \
  do {                                                                                               \
    ILS_CU(cudaFuncSetAttribute(batched_rk_kernel<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    batched_rk_kernel<RR><<<(unsigned)h.batch, 32, smem, h.stream>>>(P);                             \
    ILS_LAUNCHED("batched_rk_kernel");                                                               \
  } while (0)
    switch (RPL) {
      case 1: RKLAUNCH(1); break;
      case 2: RKLAUNCH(2); break;
      case 3: RKLAUNCH(3); break;
      case 4: RKLAUNCH(4); break;
      default: RKLAUNCH(8); break;
    }
#undef RKLAUNCH
    return ILS_OK;
  }
  if (method == 2) {   // SP-SCD / SP-RCD: A1bar resident
    const size_t smem = (size_t)32 * 32 * 8 + 32 * 8 + 32 * sizeof(BKeyT);
    const bool n32 = h.n == 32;
    void (*kern)(BatchParams) = P.weighted ? (n32 ? batched_scd_kernel<true, true> : batched_scd_kernel<true, false>)
                                           : (n32 ? batched_scd_kernel<false, true> : batched_scd_kernel<false, false>);
    ILS_CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)h.batch, 32, smem, h.stream>>>(P);
    ILS_LAUNCHED("batched_scd_kernel");
    return ILS_OK;
  }
  const size_t smem = (size_t)(h.n * h.p + h.n * h.n + h.p) * 8 + 32 * 8 + 32 * sizeof(BKey);
  const int up = (int)((h.p + 31) / 32);
#define BLAUNCH(UU)                                                                                   \
  do {                                                                                                \
    ILS_CU(cudaFuncSetAttribute(batched_kernel<UU>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    batched_kernel<UU><<<(unsigned)h.batch, 32, smem, h.stream>>>(P);                                 \
    ILS_LAUNCHED("batched_kernel");                                                                   \
  } while (0)
  if (up <= 1) BLAUNCH(1);
  else if (up <= 2) BLAUNCH(2);
  else if (up <= 3) BLAUNCH(3);
  else if (up <= 4) BLAUNCH(4);
  else BLAUNCH(8);
#undef BLAUNCH
  return ILS_OK;
}

}  // namespace ils
