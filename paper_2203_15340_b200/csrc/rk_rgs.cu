// rk_rgs.cu -- K2a: persistent SP-RK-RGS inner solver (Alg. 2 steps 6-12).
//
// Inner step t (reading R21: r = w - A1 z is maintained instead of A1 z):
//   s1 = (b_hat_j1 - <a_j1, w>) / N_j1            RK on A1^T w = b_hat   (step 9)
//   w += s1 a_j1 ; r += s1 a_j1
//   s2 = <a_j2, r> / N_j2                          RGS on A1 z = w       (step 11)
//      = (<a_j2, r_old> + s1 <a_j2, a_j1>) / N_j2  -> the three dots share ONE reduction
//   z_j2 += s2 ; r -= s2 a_j2
// rk_rgs_kernel runs the steps [t0, t1) between two inner checks: the p-vectors w, r live in
// registers, split over a thread-block cluster of C CTAs (row slices); the two column slices per
// step are TMA-prefetched NS steps ahead (the index stream is data-independent). Per step: warp
// shuffles, one named barrier, then a one-hop DSMEM all-to-all (st.async + mbarrier complete_tx,
// no cluster-wide barrier) of the CTA partials; every CTA sums the C partials in the same fixed
// order. z is replicated in every CTA's smem. The inner stop check (include/ils.h) runs between
// chunks as a full-GPU fused row stream (rk_check in sp.cu: az = A1 z, g = A1^T az - b_hat, reset
// r = w - az); w, r, z pass through HBM between chunks.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ils_internal.h"

namespace ils {

constexpr int RK_MAXW = 16;      // warps per CTA (max)
constexpr int RK_RING = 128;     // index ring entries
constexpr int RK_AHEAD = 64;     // ring fill distance (steps)
constexpr int RK_MAXC = 16;

struct RkIdx {
  int32_t j1, j2;
  double bh1, rn1, rn2;          // b_hat_{j1}, 1/N_{j1}, 1/N_{j2}
};

struct RkParams {
  const double* A1T;   // npad x ppad (column j of A1 contiguous)
  int64_t ppad, npad;
  int n;
  const double* N;
  const uint64_t* S;
  const double* bhat;
  double* W;           // [ppad] state w (in/out)
  double* Rv;          // [ppad] state r = w - A1 z (in/out)
  double* Z;           // [npad] state z (in/out)
  uint64_t seed;
  uint32_t k;
  int64_t t0, t1, max_inner;
  DevStatus* st;
  int C, slice, slicepad, nslots;
  long long* prof;     // optional per-phase cycle counters (rank 0, thread 0), see ILS_RK_PROF
  int gmode;           // 1: z and the sampling table stay in global memory (large n, single-step kernel)
  const double* G;     // look-ahead kernel: A1bar (npad x npad) for the column inner products
  // look-ahead kernel, whole inner solve in one launch: the inner check every ce steps runs in the
  // kernel (g = A1bar z - b_hat on a snapshot of z, Zsnap = [C][npad] global scratch)
  int64_t ce;
  double inner_tol;
  double* Zsnap;
  int nap;             // look-ahead kernel: ns a polling helper warp (fill, TMA, check) sleeps per poll
  int s_smem;          // blocked kernel in gmode: the prefix sums S still fit in shared memory
};

// Ring entries for steps t0 .. t0+31 (one per lane): Philox draw, two weighted inverse-CDF
// samples on the shared prefix sums, and the scalars the step needs (off the critical path).
__device__ __forceinline__ void rk_fill_indices(const RkParams& p, const uint64_t* Ss, RkIdx* ring,
                                                int64_t t0, int lane, const double* bh_tab = nullptr,
                                                const double* rn_tab = nullptr) {
  const int64_t t = t0 + lane;
  if (t >= p.t1) {   // masked step (tail of the last block of a chunk): s1 = s2 = 0
    RkIdx e;
    e.j1 = 0;
    e.j2 = 0;
    e.bh1 = 0.0;
    e.rn1 = 0.0;
    e.rn2 = 0.0;
    ring[t & (RK_RING - 1)] = e;
  } else {
    const U4 x = draw(p.seed, p.k, (uint64_t)t, kTagRkRgs);
    const int j1 = sample_weighted(((uint64_t)x.y << 32) | x.x, Ss, p.n);
    const int j2 = sample_weighted(((uint64_t)x.w << 32) | x.z, Ss, p.n);
    RkIdx e;
    e.j1 = j1;
    e.j2 = j2;
    if (bh_tab) {   // shared-memory tables: no dependent global loads on the fill path
      e.bh1 = bh_tab[j1];
      e.rn1 = rn_tab[j1];
      e.rn2 = rn_tab[j2];
    } else {
      e.bh1 = p.bhat[j1];
      e.rn1 = 1.0 / p.N[j1];
      e.rn2 = 1.0 / p.N[j2];
    }
    ring[t & (RK_RING - 1)] = e;
  }
}

// CC = cluster size (1: single CTA), U = rows per thread. blockDim.x = 32 * NW threads; thread
// tid owns rows tid + u * blockDim.x (u < U) of this CTA's row slice. Slot columns are padded to
// slicepad = U * blockDim.x doubles (zero tail written once), so the row loops carry no bounds.
template <int CC, int U>
__global__ void __launch_bounds__(512, 1) rk_rgs_kernel(RkParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NT = blockDim.x, NW = NT >> 5;
  const int rank = (CC > 1) ? (int)cluster_ctarank() : 0;
  const int64_t i0 = (int64_t)rank * p.slice;
  const int own = (int)((i0 + p.slice <= p.ppad) ? p.slice : (p.ppad > i0 ? p.ppad - i0 : 0));
  const int NS = p.nslots, SP = p.slicepad;
  // every CTA reads the stop flag before any CTA of this launch can change it (cluster sync below)
  const bool stopped = *(volatile int32_t*)&p.st->inner_conv != 0;

  // shared memory carve-up
  // gmode (large n): z lives in global memory (rank 0 updates it) and the sampler searches the
  // global prefix sums; otherwise both are replicated in every CTA's shared memory
  const bool gm = p.gmode != 0;
  double* slots = reinterpret_cast<double*>(smem_raw);                 // [NS][2][slicepad]
  double* zsm = slots + (size_t)NS * 2 * SP;                           // [npad] (smem mode)
  uint64_t* Ssm = reinterpret_cast<uint64_t*>(gm ? (double*)zsm : zsm + p.npad);   // [n] (smem mode)
  RkIdx* ring = reinterpret_cast<RkIdx*>(gm ? (uint64_t*)zsm : Ssm + ((p.n + 1) & ~1));   // [RK_RING]
  double* zs = gm ? p.Z : zsm;
  const uint64_t* Ss = gm ? p.S : Ssm;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + RK_RING);        // [NS]
  __shared__ __align__(16) double wred[2][RK_MAXW][4];
  __shared__ __align__(16) double recv[2][RK_MAXC][4];                 // per-rank partials (DSMEM target)
  __shared__ __align__(8) uint64_t redbar[2];
  __shared__ double chkw[RK_MAXW];
  __shared__ double bnorm_s;
  if (stopped) return;

  if (!gm) {
    for (int64_t j = tid; j < p.npad; j += NT) zsm[j] = p.Z[j];
    for (int j = tid; j < p.n; j += NT) Ssm[j] = p.S[j];
  }
  for (int64_t e = tid; e < (int64_t)NS * 2 * SP; e += NT) slots[e] = 0.0;   // zero tails
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    if (CC > 1) {
      mbar_init(&redbar[0], 1);
      mbar_init(&redbar[1], 1);
    }
    fence_mbar_init();
    if (CC > 1) {   // arm phase 0 of both reduction barriers: CC partial triples (32 B each)
      mbar_arrive_expect_tx(&redbar[0], CC * 32);
      mbar_arrive_expect_tx(&redbar[1], CC * 32);
    }
  }
  double bnorm = 1.0;
  if (p.t0 == 0) {   // ||b_hat|| (same fixed order in every CTA); b_hat = 0 -> z = 0 after 0 steps
    double v = 0.0;
    for (int j = tid; j < p.n; j += NT) v = fma(p.bhat[j], p.bhat[j], v);
    v = warp_sum(v);
    if (lane == 0) chkw[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += chkw[w];
      bnorm_s = sqrt(s);
    }
    __syncthreads();
    bnorm = bnorm_s;
  }
  __syncthreads();
  if (CC > 1) cluster_sync_all();   // peers' barriers initialised before any DSMEM traffic
  if (bnorm == 0.0) {
    if (rank == 0 && tid == 0) {
      p.st->inner_steps = 0;
      p.st->inner_conv = 1;
    }
    return;   // Z is still the zero initial state
  }

  // index ring: steps [t0, t0+64); at step t ((t - t0) % 32 == 0) warp NW-1 fills [t+64, t+96),
  // overwriting entries of steps t-64..t-33 that every thread has finished with
  if (warp == 0) rk_fill_indices(p, Ss, ring, p.t0, lane);
  if (warp == NW - 1) rk_fill_indices(p, Ss, ring, p.t0 + 32, lane);
  __syncthreads();

  const uint32_t slice_bytes = (uint32_t)own * sizeof(double);
  const int issuer = NT - 1;
  auto issue = [&](int64_t t, int slot) {
    const RkIdx e = ring[t & (RK_RING - 1)];
    double* dst = slots + (size_t)slot * 2 * SP;
    mbar_arrive_expect_tx(&bars[slot], 2 * slice_bytes);
    bulk_g2s(dst, p.A1T + (int64_t)e.j1 * p.ppad + i0, slice_bytes, &bars[slot]);
    bulk_g2s(dst + SP, p.A1T + (int64_t)e.j2 * p.ppad + i0, slice_bytes, &bars[slot]);
  };
  // steps [t0, issued) have been requested; after step t, issued = min(t + NS, t1)
  int64_t issued = (p.t0 + NS < p.t1) ? p.t0 + NS : p.t1;
  if (tid == issuer && own > 0) {
    fence_proxy_async();
    for (int64_t u = p.t0; u < issued; ++u) issue(u, (int)(u - p.t0));
  }

  double w[U], r[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + tid + u * NT;
    const bool in = (tid + u * NT < own);
    w[u] = in ? p.W[i] : 0.0;
    r[u] = in ? p.Rv[i] : 0.0;
  }

  int slot = 0;
  uint32_t ph = 0;
  for (int64_t t = p.t0; t < p.t1; ++t) {
    const int pb = (int)(t & 1);
    const double* a1 = slots + (size_t)slot * 2 * SP;
    const double* a2 = a1 + SP;
    double d1 = 0.0, d2 = 0.0, d3 = 0.0;
    // gmode: the global RMW of z_{j2} overlaps this step (the previous store to the same address
    // precedes this load in thread 0's program order)
    const double zold = (gm && rank == 0 && tid == 0) ? p.Z[ring[t & (RK_RING - 1)].j2] : 0.0;
    if (own > 0) mbar_wait(&bars[slot], ph);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double x1 = a1[tid + u * NT], x2 = a2[tid + u * NT];
      d1 = fma(x1, w[u], d1);
      d2 = fma(x2, r[u], d2);
      d3 = fma(x2, x1, d3);
    }
    d1 = warp_sum(d1);
    d2 = warp_sum(d2);
    d3 = warp_sum(d3);
    if (NW > 1) {
      if (lane == 0) {
        wred[pb][warp][0] = d1;
        wred[pb][warp][1] = d2;
        wred[pb][warp][2] = d3;
      }
      named_bar_sync(1, NT);   // all warps finished step t-1 and deposited step t partials
    }
    // refill the slot step t-1 used (every thread is past step t-1 here)
    if (t > p.t0 && issued < p.t1) {
      if (tid == issuer && own > 0) issue(issued, slot == 0 ? NS - 1 : slot - 1);
      ++issued;
    }
    double D1, D2, D3;
    if (CC > 1) {
      if (warp == 0 && lane < CC) {
        double v0 = d1, v1 = d2, v2 = d3;
        if (NW > 1) {
          v0 = v1 = v2 = 0.0;
          for (int w8 = 0; w8 < NW; ++w8) {
            v0 += wred[pb][w8][0];
            v1 += wred[pb][w8][1];
            v2 += wred[pb][w8][2];
          }
        }
        const uint32_t raddr = map_shared_rank(smem_u32(&recv[pb][rank][0]), (uint32_t)lane);
        const uint32_t rbar = map_shared_rank(smem_u32(&redbar[pb]), (uint32_t)lane);
        st_async_v2f64(raddr, v0, v1, rbar);
        st_async_v2f64(raddr + 16, v2, 0.0, rbar);
      }
      if (warp == NW - 1 && ((t - p.t0) & 31) == 0 && t + RK_AHEAD < p.t1)
        rk_fill_indices(p, Ss, ring, t + RK_AHEAD, lane);
      mbar_wait(&redbar[pb], (uint32_t)(((t - p.t0) >> 1) & 1));
      double a0[CC], a1v[CC], a2v[CC];
#pragma unroll
      for (int c = 0; c < CC; ++c) {
        const double2 v = *reinterpret_cast<const double2*>(&recv[pb][c][0]);
        a0[c] = v.x;
        a1v[c] = v.y;
        a2v[c] = recv[pb][c][2];
      }
#pragma unroll
      for (int s = 1; s < CC; s *= 2)
#pragma unroll
        for (int c = 0; c + s < CC; c += 2 * s) {
          a0[c] += a0[c + s];
          a1v[c] += a1v[c + s];
          a2v[c] += a2v[c + s];
        }
      D1 = a0[0];
      D2 = a1v[0];
      D3 = a2v[0];
      // re-arm for step t+2: its complete_tx cannot arrive before this CTA sends step t+1,
      // which happens after every thread here has passed this wait
      if (tid == 0) mbar_arrive_expect_tx(&redbar[pb], CC * 32);
    } else {
      if (((t - p.t0) & 31) == 0 && t + RK_AHEAD < p.t1 && warp == NW - 1)
        rk_fill_indices(p, Ss, ring, t + RK_AHEAD, lane);
      if (NW > 1) {
        D1 = D2 = D3 = 0.0;
        for (int w8 = 0; w8 < NW; ++w8) {
          D1 += wred[pb][w8][0];
          D2 += wred[pb][w8][1];
          D3 += wred[pb][w8][2];
        }
      } else {
        D1 = d1;
        D2 = d2;
        D3 = d3;
      }
    }
    const RkIdx ix = ring[t & (RK_RING - 1)];
    const double s1 = (ix.bh1 - D1) * ix.rn1;
    const double s2 = (D2 + s1 * D3) * ix.rn2;
    // gmode: z_{j2} was loaded by rank 0 / thread 0 at the top of this step (zold below)
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double x1 = a1[tid + u * NT], x2 = a2[tid + u * NT];
      w[u] = fma(s1, x1, w[u]);
      r[u] = fma(s1, x1, r[u]);
      r[u] = fma(-s2, x2, r[u]);
    }
    if (!gm) {
      if (tid == 0) zs[ix.j2] += s2;
    } else if (rank == 0 && tid == 0) {
      zs[ix.j2] = zold + s2;
    }
    if (++slot == NS) {
      slot = 0;
      ph ^= 1u;
    }
  }
  // save the state (no TMA is in flight: every issued step was consumed)
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (tid + u * NT < own) {
      const int64_t i = i0 + tid + u * NT;
      p.W[i] = w[u];
      p.Rv[i] = r[u];
    }
  }
  __syncthreads();
  if (rank == 0 && !gm)
    for (int64_t j = tid; j < p.npad; j += NT) p.Z[j] = zs[j];
  if (CC > 1) cluster_sync_all();   // no CTA exits while peers may still access its smem
}

// ---------------------------------------------------------------------------------------------
// Blocked variant: B consecutive steps per cluster reduction. The indices of steps t..t+B-1 are
// known in advance, so every inner product the B steps need can be written in terms of the state
// (w, r) at the start of the block and the Gram entries of the 2B columns involved:
//   <a_i, w_i>        = <a_i, w> + sum_{k<i} s1_k <a_i, a_k>
//   <b_i, r_i + s1_i a_i> = <b_i, r> + sum_{k<i} (s1_k <b_i, a_k> - s2_k <b_i, b_k>) + s1_i <b_i, a_i>
// (a_i = A1_(j1_i), b_i = A1_(j2_i)). One reduction of NV = (3B^2 + 3B)/2 values replaces B
// reductions of 3; the scalar recurrence for s1_i, s2_i runs redundantly in every thread, then
// w += sum s1_i a_i, r += sum (s1_i a_i - s2_i b_i). Identical to B single steps in exact
// arithmetic (Alg. 2 steps 9 and 11); only the rounding differs.
template <int CC, int U, int B>
__global__ void __launch_bounds__(512, 1) rk_rgs_block_kernel(RkParams p) {
  using K = RkBlk<B>;
  static_assert(K::NV <= 32, "block too large for one warp reduce-scatter");
  constexpr int NVP = K::NV <= 4 ? 4 : (K::NV <= 8 ? 8 : (K::NV <= 16 ? 16 : 32));
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NT = blockDim.x, NW = NT >> 5;
  const int rank = (CC > 1) ? (int)cluster_ctarank() : 0;
  const int64_t i0 = (int64_t)rank * p.slice;
  const int own = (int)((i0 + p.slice <= p.ppad) ? p.slice : (p.ppad > i0 ? p.ppad - i0 : 0));
  const int NS = p.nslots, SP = p.slicepad;
  const bool stopped = *(volatile int32_t*)&p.st->inner_conv != 0;

  // gmode (long row slices with large n, e.g. c2): z, the prefix sums and the b_hat / 1/N tables stay
  // in global memory (L2) so that two slots of 2B column slices fit; z is then updated by rank 0 only
  const bool gm = p.gmode != 0;
  double* slots = reinterpret_cast<double*>(smem_raw);                 // [NS][2B][slicepad]
  const bool s_sm = !gm || p.s_smem;   // the sampler's prefix sums in shared memory
  double* zsm = slots + (size_t)NS * 2 * B * SP;                       // [npad] (not gmode)
  uint64_t* Ssm = reinterpret_cast<uint64_t*>(zsm + (gm ? 0 : p.npad));   // [n] (s_sm)
  RkIdx* ring = reinterpret_cast<RkIdx*>(Ssm + (s_sm ? ((p.n + 1) & ~1) : 0));   // [RK_RING]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + RK_RING);        // [NS]
  double* bh_sm = reinterpret_cast<double*>(bars + 8);                  // [n] b_hat (not gmode)
  double* rn_sm = bh_sm + ((p.n + 1) & ~1);                            // [n] 1 / N (not gmode)
  double* zs = gm ? p.Z : zsm;
  const uint64_t* Ss = s_sm ? Ssm : p.S;
  const double* bh_tab = gm ? nullptr : bh_sm;
  const double* rn_tab = gm ? nullptr : rn_sm;
  const bool zowner = !gm || rank == 0;   // gmode: one CTA applies the z updates to the global z
  __shared__ __align__(16) double wred[2][RK_MAXW][32];
  __shared__ __align__(16) double recv1[2][RK_MAXC][32];   // [source rank][value]
  __shared__ __align__(8) uint64_t bar1[2];
  __shared__ double chkw[RK_MAXW];
  __shared__ __align__(16) double tots[RK_MAXW][32];
  __shared__ double bnorm_s;
  if (stopped) return;

  if (!gm) {
    for (int64_t j = tid; j < p.npad; j += NT) zsm[j] = p.Z[j];
    for (int j = tid; j < p.n; j += NT) {
      bh_sm[j] = p.bhat[j];
      rn_sm[j] = 1.0 / p.N[j];
    }
  }
  if (s_sm)
    for (int j = tid; j < p.n; j += NT) Ssm[j] = p.S[j];
  for (int64_t e = tid; e < (int64_t)NS * 2 * B * SP; e += NT) slots[e] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    if (CC > 1) {
      mbar_init(&bar1[0], 1);
      mbar_init(&bar1[1], 1);
    }
    fence_mbar_init();
    if (CC > 1) {   // CC sources x 32 values x 8 B
      mbar_arrive_expect_tx(&bar1[0], CC * NVP * 8);
      mbar_arrive_expect_tx(&bar1[1], CC * NVP * 8);
    }
  }
  double bnorm = 1.0;
  if (p.t0 == 0) {
    double v = 0.0;
    for (int j = tid; j < p.n; j += NT) v = fma(p.bhat[j], p.bhat[j], v);
    v = warp_sum(v);
    if (lane == 0) chkw[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += chkw[w];
      bnorm_s = sqrt(s);
    }
    __syncthreads();
    bnorm = bnorm_s;
  }
  __syncthreads();
  if (CC > 1) cluster_sync_all();
  if (bnorm == 0.0) {
    if (rank == 0 && tid == 0) {
      p.st->inner_steps = 0;
      p.st->inner_conv = 1;
    }
    return;
  }
  if (warp == 0) rk_fill_indices(p, Ss, ring, p.t0, lane, bh_tab, rn_tab);
  if (warp == NW - 1) rk_fill_indices(p, Ss, ring, p.t0 + 32, lane, bh_tab, rn_tab);
  __syncthreads();

  const uint32_t slice_bytes = (uint32_t)own * sizeof(double);
  const int issuer = NT - 1;
  const int64_t nblk = (p.t1 - p.t0 + B - 1) / B;
  auto issue = [&](int64_t blk, int slot) {   // 2B column slices of block blk
    double* dst = slots + (size_t)slot * 2 * B * SP;
    mbar_arrive_expect_tx(&bars[slot], 2 * B * slice_bytes);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const RkIdx e = ring[(p.t0 + blk * B + i) & (RK_RING - 1)];
      bulk_g2s(dst + (2 * i) * SP, p.A1T + (int64_t)e.j1 * p.ppad + i0, slice_bytes, &bars[slot]);
      bulk_g2s(dst + (2 * i + 1) * SP, p.A1T + (int64_t)e.j2 * p.ppad + i0, slice_bytes, &bars[slot]);
    }
  };
  int64_t issued = (NS < nblk) ? NS : nblk;   // blocks requested
  if (tid == issuer && own > 0) {
    fence_proxy_async();
    for (int64_t b = 0; b < issued; ++b) issue(b, (int)b);
  }

  double w[U], r[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + tid + u * NT;
    const bool in = (tid + u * NT < own);
    w[u] = in ? p.W[i] : 0.0;
    r[u] = in ? p.Rv[i] : 0.0;
  }

  int slot = 0;
  uint32_t ph = 0;
  double zprev[B];
#pragma unroll
  for (int i = 0; i < B; ++i) zprev[i] = 0.0;
  const bool prof = p.prof && tid == 0;
  long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tc = clock64();
#define RKP(i)                         \
  if (prof) {                          \
    const long long c_ = clock64();    \
    pc[i] += c_ - tc;                  \
    tc = c_;                           \
  }
  for (int64_t blk = 0; blk < nblk; ++blk) {
    const int64_t t = p.t0 + blk * B;
    const int pb = (int)(blk & 1);
    const double* cols = slots + (size_t)slot * 2 * B * SP;
    if (own > 0) mbar_wait(&bars[slot], ph);
    RKP(0)
    double acc[NVP];
#pragma unroll
    for (int v = 0; v < NVP; ++v) acc[v] = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = tid + u * NT;
      double xa[B], xb[B];
#pragma unroll
      for (int i = 0; i < B; ++i) {
        xa[i] = cols[(2 * i) * SP + e];
        xb[i] = cols[(2 * i + 1) * SP + e];
      }
#pragma unroll
      for (int i = 0; i < B; ++i) {
        acc[K::P(i)] = fma(xa[i], w[u], acc[K::P(i)]);
        acc[K::Q(i)] = fma(xb[i], r[u], acc[K::Q(i)]);
#pragma unroll
        for (int k = 0; k < i; ++k) {
          acc[K::AA(i, k)] = fma(xa[i], xa[k], acc[K::AA(i, k)]);
          acc[K::BB(i, k)] = fma(xb[i], xb[k], acc[K::BB(i, k)]);
        }
#pragma unroll
        for (int k = 0; k <= i; ++k) acc[K::BA(i, k)] = fma(xb[i], xa[k], acc[K::BA(i, k)]);
      }
    }
    RKP(1)
    double mine = warp_reduce_scatter<NVP>(acc, lane);   // lane l: warp total of value l % NVP
    RKP(2)
    if (NW > 1) {
      wred[pb][warp][lane] = mine;
      named_bar_sync(1, NT);
    }
    RKP(3)
    if (blk >= 1 && issued < nblk) {
      if (tid == issuer && own > 0) issue(issued, slot == 0 ? NS - 1 : slot - 1);
      ++issued;
    }
    double tot;
    if (CC > 1) {
      // one-hop cluster all-to-all of the NVP values: warp 0 forms the CTA totals (lane l ->
      // value l) and sends them to every rank; each st.async instruction targets ONE destination
      // CTA with NVP contiguous doubles (destination-uniform instructions are ~2x faster than
      // lane-scattered ones, and one sending warp beat sends spread over warps: tools/mb/dsmem_bench.cu).
      if (warp == 0) {
        double v = mine;
        if (NW > 1) {
          v = 0.0;
          for (int w8 = 0; w8 < NW; ++w8) v += wred[pb][w8][lane];
        }
        // lane l < NVP/2 carries values 2l, 2l+1 as one 16-byte st.async (half the instructions)
        const double v0 = __shfl_sync(0xffffffffu, v, (2 * lane) & 31);
        const double v1 = __shfl_sync(0xffffffffu, v, (2 * lane + 1) & 31);
        const uint32_t la = smem_u32(&recv1[pb][rank][2 * (lane & (NVP / 2 - 1))]);
        const uint32_t lb = smem_u32(&bar1[pb]);
        if (lane < NVP / 2)
          for (int c = 0; c < CC; ++c) st_async_v2f64(map_shared_rank(la, (uint32_t)c), v0, v1, map_shared_rank(lb, (uint32_t)c));
      }
      // deferred z updates of the previous block (sequential order), hidden in the reduction wait
      if (warp == NW - 1 && lane == 0 && blk > 0 && zowner) {
#pragma unroll
        for (int i = 0; i < B; ++i) zs[ring[(t - B + i) & (RK_RING - 1)].j2] += zprev[i];
      }
      if (warp == NW - 1 && ((t - p.t0) & 31) == 0 && t + RK_AHEAD < p.t1 + 64)
        rk_fill_indices(p, Ss, ring, t + RK_AHEAD, lane, bh_tab, rn_tab);
      RKP(4)
      mbar_wait(&bar1[pb], (uint32_t)((blk >> 1) & 1));
      RKP(5)
      {
        double a[CC];
#pragma unroll
        for (int c = 0; c < CC; ++c) a[c] = recv1[pb][c][lane & (NVP - 1)];
#pragma unroll
        for (int s = 1; s < CC; s *= 2)
#pragma unroll
          for (int c = 0; c + s < CC; c += 2 * s) a[c] += a[c + s];
        tot = a[0];
      }
      // re-arm for block blk+2: its data cannot arrive before this CTA sends block blk+1,
      // which happens after every thread here has passed this wait
      if (tid == 0) mbar_arrive_expect_tx(&bar1[pb], CC * NVP * 8);
    } else {
      if (((t - p.t0) & 31) == 0 && t + RK_AHEAD < p.t1 + 64 && warp == NW - 1)
        rk_fill_indices(p, Ss, ring, t + RK_AHEAD, lane, bh_tab, rn_tab);
      if (NW > 1) {
        tot = 0.0;
        for (int w8 = 0; w8 < NW; ++w8) tot += wred[pb][w8][lane];
      } else {
        tot = mine;
      }
    }
    RKP(6)
    // every thread gets all NV totals, then runs the B-step scalar recurrence
    double T[K::NV];
    tots[warp][lane] = tot;
    __syncwarp();
#pragma unroll
    for (int v = 0; v < K::NV; ++v) T[v] = tots[warp][v];
    double s1[B], s2[B];
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const RkIdx ix = ring[(t + i) & (RK_RING - 1)];
      double dw = T[K::P(i)];
#pragma unroll
      for (int k = 0; k < i; ++k) dw = fma(s1[k], T[K::AA(i, k)], dw);
      s1[i] = (ix.bh1 - dw) * ix.rn1;
      double dr = T[K::Q(i)];
#pragma unroll
      for (int k = 0; k < i; ++k) {
        dr = fma(s1[k], T[K::BA(i, k)], dr);
        dr = fma(-s2[k], T[K::BB(i, k)], dr);
      }
      dr = fma(s1[i], T[K::BA(i, i)], dr);
      s2[i] = dr * ix.rn2;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = tid + u * NT;
#pragma unroll
      for (int i = 0; i < B; ++i) {
        const double xa = cols[(2 * i) * SP + e], xb = cols[(2 * i + 1) * SP + e];
        w[u] = fma(s1[i], xa, w[u]);
        r[u] = fma(s1[i], xa, r[u]);
        r[u] = fma(-s2[i], xb, r[u]);
      }
    }
    if (warp == NW - 1 && lane == 0) {
      if (CC > 1) {
#pragma unroll
        for (int i = 0; i < B; ++i) zprev[i] = s2[i];
      } else if (zowner) {
#pragma unroll
        for (int i = 0; i < B; ++i) zs[ring[(t + i) & (RK_RING - 1)].j2] += s2[i];
      }
    }
    if (++slot == NS) {
      slot = 0;
      ph ^= 1u;
    }
    RKP(7)
  }
#undef RKP
  if (CC > 1 && warp == NW - 1 && lane == 0 && nblk > 0 && zowner) {
    const int64_t tl = p.t0 + (nblk - 1) * B;
#pragma unroll
    for (int i = 0; i < B; ++i) zs[ring[(tl + i) & (RK_RING - 1)].j2] += zprev[i];
  }
  if (prof)
    for (int i = 0; i < 8; ++i) p.prof[rank * 8 + i] += pc[i];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (tid + u * NT < own) {
      const int64_t i = i0 + tid + u * NT;
      p.W[i] = w[u];
      p.Rv[i] = r[u];
    }
  }
  __syncthreads();
  if (rank == 0 && !gm)
    for (int64_t j = tid; j < p.npad; j += NT) p.Z[j] = zs[j];
  if (CC > 1) cluster_sync_all();
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

template <int CC, int U>
static int launch_rk(Handle& h, RkParams& p, int nt, size_t smem) {
  auto kern = rk_rgs_kernel<CC, U>;
  ILS_CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CC);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h.stream;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (CC > 1) {
    ILS_CU(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    na = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  ILS_CU(cudaLaunchKernelEx(&cfg, kern, p));
  ILS_LAUNCHED("rk_rgs_kernel");
  return ILS_OK;
}

// Whole SP-RK-RGS inner solve in ONE CTA launch for small problems (one CTA, A1 staged entirely
// in shared memory: ppad * npad * 8 <= ~150 KB, e.g. configs[0]): the blocked recurrence of
// rk_rgs_block_kernel (4 steps per reduction, here over the CTA's warps only) plus the inner stop
// check (include/ils.h: az = A1 z, g = A1^T az - b_hat, reset r = w - az) done in place every
// check_every steps, so a solve is one launch instead of two launches per check interval.
// Blocks restart at every check boundary (steps past it are masked), as the chunked launches do.
// LK: the 22 in-block column inner products are looked up in A1bar (p.G, staged in shared memory)
// instead of reduced with the state products (8 values per block reduction instead of 30), as in
// the look-ahead and batched kernels.
template <int U, bool LK>
__global__ void __launch_bounds__(256, 1) rk_rgs_small_kernel(RkParams p, double* __restrict__ zout,
                                                              int64_t ce, double inner_tol) {
  constexpr int B = 4;
  using K = RkBlk<B>;
  constexpr int NVP = LK ? 8 : 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NT = blockDim.x, NW = NT >> 5;
  const int64_t PP = p.ppad;
  const int n = p.n;
  double* A1s = reinterpret_cast<double*>(smem_raw);            // [npad][ppad], column j contiguous
  double* zs = A1s + (size_t)p.npad * PP;                        // [npad]
  double* azs = zs + p.npad;                                     // [ppad]
  uint64_t* Ss = reinterpret_cast<uint64_t*>(azs + PP);          // [n]
  double* bh_tab = reinterpret_cast<double*>(Ss + ((n + 1) & ~1));   // [n]
  double* rn_tab = bh_tab + ((n + 1) & ~1);                     // [n]
  RkIdx* ring = reinterpret_cast<RkIdx*>(rn_tab + ((n + 1) & ~1));   // [RK_RING]
  double* Gs = reinterpret_cast<double*>(ring + RK_RING);          // LK: [npad][npad] A1bar
  __shared__ __align__(16) double wred[8][32];
  __shared__ double tots[32];
  __shared__ double red2[8][2];
  __shared__ int stop_s;

  for (int64_t e = tid; e < (int64_t)p.npad * PP; e += NT) A1s[e] = p.A1T[e];
  if (LK)
    for (int64_t e = tid; e < (int64_t)p.npad * p.npad; e += NT) Gs[e] = p.G[e];
  for (int j = tid; j < p.npad; j += NT) zs[j] = 0.0;
  for (int j = tid; j < n; j += NT) {
    Ss[j] = p.S[j];
    bh_tab[j] = p.bhat[j];
    rn_tab[j] = 1.0 / p.N[j];
  }
  if (tid == 0) stop_s = 0;
  __syncthreads();
  // ||b_hat|| (fixed order) and the b_hat = 0 case (beta = 0 after 0 steps)
  {
    double v = 0.0;
    for (int j = tid; j < n; j += NT) v = fma(bh_tab[j], bh_tab[j], v);
    v = warp_sum(v);
    if (lane == 0) red2[warp][0] = v;
  }
  __syncthreads();
  double bnorm2 = 0.0;
  for (int w = 0; w < NW; ++w) bnorm2 += red2[w][0];
  __syncthreads();
  if (bnorm2 == 0.0) {
    if (tid == 0) {
      p.st->inner_steps = 0;
      p.st->inner_conv = 1;
    }
    for (int j = tid; j < p.npad; j += NT) zout[j] = 0.0;
    return;
  }
  double w[U], r[U];
#pragma unroll
  for (int u = 0; u < U; ++u) w[u] = r[u] = 0.0;
  int64_t filled = 0;   // ring holds steps [filled - RK_RING, filled)
  int64_t t = 0;
  bool conv = false;
  while (t < p.max_inner && !conv) {
    const int64_t cend = (t + ce < p.max_inner) ? t + ce : p.max_inner;   // this check interval
    for (; t < cend; t += B) {
      if (t + B > filled) {   // indices of the next 32 steps (one warp, then visible to all)
        if (warp == 0) rk_fill_indices(p, Ss, ring, filled, lane, bh_tab, rn_tab);
        filled += 32;
        __syncthreads();
      }
      RkIdx ix[B];
#pragma unroll
      for (int i = 0; i < B; ++i) ix[i] = ring[(t + i) & (RK_RING - 1)];
      double acc[NVP];
#pragma unroll
      for (int v = 0; v < NVP; ++v) acc[v] = 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = tid + u * NT;
        if (e < PP) {
          double xa[B], xb[B];
#pragma unroll
          for (int i = 0; i < B; ++i) {
            xa[i] = A1s[(int64_t)ix[i].j1 * PP + e];
            xb[i] = A1s[(int64_t)ix[i].j2 * PP + e];
          }
#pragma unroll
          for (int i = 0; i < B; ++i) {
            acc[K::P(i)] = fma(xa[i], w[u], acc[K::P(i)]);
            acc[K::Q(i)] = fma(xb[i], r[u], acc[K::Q(i)]);
            if (!LK) {
#pragma unroll
              for (int k = 0; k < i; ++k) {
                acc[K::AA(i, k)] = fma(xa[i], xa[k], acc[K::AA(i, k)]);
                acc[K::BB(i, k)] = fma(xb[i], xb[k], acc[K::BB(i, k)]);
              }
#pragma unroll
              for (int k = 0; k <= i; ++k) acc[K::BA(i, k)] = fma(xb[i], xa[k], acc[K::BA(i, k)]);
            }
          }
        }
      }
      double T[K::NV];
      if (LK) {   // the block's column inner products from A1bar (before the reduction: off its path)
        const int64_t ld = p.npad;
#pragma unroll
        for (int i = 0; i < B; ++i) {
#pragma unroll
          for (int k = 0; k < i; ++k) {
            T[K::AA(i, k)] = Gs[ix[i].j1 * ld + ix[k].j1];
            T[K::BB(i, k)] = Gs[ix[i].j2 * ld + ix[k].j2];
          }
#pragma unroll
          for (int k = 0; k <= i; ++k) T[K::BA(i, k)] = Gs[ix[i].j2 * ld + ix[k].j1];
        }
      }
      const double mine = warp_reduce_scatter<NVP>(acc, lane);
      wred[warp][lane] = mine;
      __syncthreads();
      if (warp == 0) {
        double v = 0.0;
        for (int w8 = 0; w8 < NW; ++w8) v += wred[w8][lane];
        tots[lane] = v;
      }
      __syncthreads();
#pragma unroll
      for (int v = 0; v < (LK ? NVP : K::NV); ++v) T[v] = tots[v];
      double s1[B], s2[B];
#pragma unroll
      for (int i = 0; i < B; ++i) {
        const bool live = t + i < cend;   // steps past the check boundary (or max_inner) are masked
        double dw = T[K::P(i)];
#pragma unroll
        for (int k = 0; k < i; ++k) dw = fma(s1[k], T[K::AA(i, k)], dw);
        s1[i] = live ? (ix[i].bh1 - dw) * ix[i].rn1 : 0.0;
        double dr = T[K::Q(i)];
#pragma unroll
        for (int k = 0; k < i; ++k) {
          dr = fma(s1[k], T[K::BA(i, k)], dr);
          dr = fma(-s2[k], T[K::BB(i, k)], dr);
        }
        dr = fma(s1[i], T[K::BA(i, i)], dr);
        s2[i] = live ? dr * ix[i].rn2 : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = tid + u * NT;
        if (e < PP) {
#pragma unroll
          for (int i = 0; i < B; ++i) {
            const double xa = A1s[(int64_t)ix[i].j1 * PP + e], xb = A1s[(int64_t)ix[i].j2 * PP + e];
            w[u] = fma(s1[i], xa, w[u]);
            r[u] = fma(s1[i], xa, r[u]);
            r[u] = fma(-s2[i], xb, r[u]);
          }
        }
      }
      if (tid == 0)
#pragma unroll
        for (int i = 0; i < B; ++i) zs[ix[i].j2] += s2[i];   // program order (j2 may repeat)
      __syncthreads();   // tots / wred reuse, zs visible
    }
    t = cend;
    if (t % ce != 0) break;   // max_inner reached off the check grid: no check (chunked path rule)
    // ---- inner stop check at t: az = A1 z (own rows), g = A1^T az - b_hat (reads z only)
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = tid + u * NT;
      if (e < PP) {
        double a = 0.0, a2 = 0.0;
        int j = 0;
        for (; j + 1 < n; j += 2) {
          a = fma(A1s[(int64_t)j * PP + e], zs[j], a);
          a2 = fma(A1s[(int64_t)(j + 1) * PP + e], zs[j + 1], a2);
        }
        if (j < n) a = fma(A1s[(int64_t)j * PP + e], zs[j], a);
        azs[e] = (e < p.slice) ? a + a2 : 0.0;   // rows >= p are zero padding
      }
    }
    __syncthreads();
    double g2 = 0.0;
    for (int j = warp; j < n; j += NW) {
      double sacc = 0.0;
      for (int64_t i = lane; i < PP; i += 32) sacc = fma(A1s[(int64_t)j * PP + i], azs[i], sacc);
      sacc = warp_sum(sacc);
      const double g = sacc - bh_tab[j];
      g2 = fma(g, g, g2);
    }
    if (lane == 0) red2[warp][1] = g2;
    __syncthreads();
    if (tid == 0) {
      double G2 = 0.0;
      for (int w8 = 0; w8 < NW; ++w8) G2 += red2[w8][1];
      stop_s = (sqrt(G2) <= inner_tol * sqrt(bnorm2)) ? 1 : 0;
    }
    __syncthreads();
    if (stop_s) {
      conv = true;
      if (tid == 0) {
        p.st->inner_steps = t;
        p.st->inner_conv = 1;
      }
    }
    __syncthreads();
  }
  for (int j = tid; j < p.npad; j += NT) zout[j] = zs[j];
}

// ---------------------------------------------------------------------------------------------
// Look-ahead blocked SP-RK-RGS (default for 16-CTA clusters; ILS_RK_LA=0 selects rk_rgs_block_kernel):
// the cluster exchange of block i+1 is in
// flight while block i's recurrence runs. Block i+1's state products are formed on the state
// S_i (before block i's update) and corrected after the exchange with block i's scalars and the
// cross inner products between the two blocks' columns, looked up in A1bar (G):
//   <a1'_k, w_{i+1}> = <a1'_k, w_i> + sum_m s1_m <a1'_k, a1_m>
//   <a2'_k, r_{i+1}> = <a2'_k, r_i> + sum_m s1_m <a2'_k, a1_m> - sum_m s2_m <a2'_k, a2_m>
// The 22 in-block column products also come from G, so only 8 values per block are reduced. A
// communication warp sums the compute warps' partials and sends them to the cluster
// (destination-uniform st.async) as soon as they are deposited; a reduce warp sums the 16
// received partials of block i, adds the corrections with block i-1's scalars (mailed by the
// compute warps) and hands the 8 finished products to the compute warps through an mbarrier, so
// the compute warps' own path per block is products -> recurrence -> axpy. A fill warp and a TMA
// warp run ahead (index / Gram rings, column refills); the compute warps never issue a send.
constexpr int LA_GR = 16;    // blocks in the Gram ring (the fill warp runs at most LA_GR blocks ahead; a 32-block ring
                             // with 24 blocks of lead measured the same: c1 184.8 vs 184.9 ms)
constexpr int LA_NG = 118;   // Gram values per block: 22 in-block (RkBlk<4> order) + 48 with block - 1 + 48 with block - 2

// (value v of a block) -> (step of the current block, its column, step relative to the block start
// (negative: an earlier block), its column): 22 in-block products in RkBlk<4> order, then X1, X2,
// X3 (4 x 4 each) with block - 1 and the same three with block - 2
__constant__ __align__(4) int8_t la_map[LA_NG][4] = {
    {1, 0, 0, 0}, {2, 0, 0, 0}, {2, 0, 1, 0}, {3, 0, 0, 0}, {3, 0, 1, 0}, {3, 0, 2, 0},                       // AA
    {0, 1, 0, 0}, {1, 1, 0, 0}, {1, 1, 1, 0}, {2, 1, 0, 0}, {2, 1, 1, 0}, {2, 1, 2, 0}, {3, 1, 0, 0},
    {3, 1, 1, 0}, {3, 1, 2, 0}, {3, 1, 3, 0},                                                               // BA
    {1, 1, 0, 1}, {2, 1, 0, 1}, {2, 1, 1, 1}, {3, 1, 0, 1}, {3, 1, 1, 1}, {3, 1, 2, 1},                       // BB
    {0, 0, -4, 0}, {0, 0, -3, 0}, {0, 0, -2, 0}, {0, 0, -1, 0}, {1, 0, -4, 0}, {1, 0, -3, 0}, {1, 0, -2, 0}, {1, 0, -1, 0},
    {2, 0, -4, 0}, {2, 0, -3, 0}, {2, 0, -2, 0}, {2, 0, -1, 0}, {3, 0, -4, 0}, {3, 0, -3, 0}, {3, 0, -2, 0}, {3, 0, -1, 0},   // X1 (block - 1)
    {0, 1, -4, 0}, {0, 1, -3, 0}, {0, 1, -2, 0}, {0, 1, -1, 0}, {1, 1, -4, 0}, {1, 1, -3, 0}, {1, 1, -2, 0}, {1, 1, -1, 0},
    {2, 1, -4, 0}, {2, 1, -3, 0}, {2, 1, -2, 0}, {2, 1, -1, 0}, {3, 1, -4, 0}, {3, 1, -3, 0}, {3, 1, -2, 0}, {3, 1, -1, 0},   // X2 (block - 1)
    {0, 1, -4, 1}, {0, 1, -3, 1}, {0, 1, -2, 1}, {0, 1, -1, 1}, {1, 1, -4, 1}, {1, 1, -3, 1}, {1, 1, -2, 1}, {1, 1, -1, 1},
    {2, 1, -4, 1}, {2, 1, -3, 1}, {2, 1, -2, 1}, {2, 1, -1, 1}, {3, 1, -4, 1}, {3, 1, -3, 1}, {3, 1, -2, 1}, {3, 1, -1, 1},   // X3 (block - 1)
    {0, 0, -8, 0}, {0, 0, -7, 0}, {0, 0, -6, 0}, {0, 0, -5, 0}, {1, 0, -8, 0}, {1, 0, -7, 0}, {1, 0, -6, 0}, {1, 0, -5, 0},
    {2, 0, -8, 0}, {2, 0, -7, 0}, {2, 0, -6, 0}, {2, 0, -5, 0}, {3, 0, -8, 0}, {3, 0, -7, 0}, {3, 0, -6, 0}, {3, 0, -5, 0},   // X1' (block - 2)
    {0, 1, -8, 0}, {0, 1, -7, 0}, {0, 1, -6, 0}, {0, 1, -5, 0}, {1, 1, -8, 0}, {1, 1, -7, 0}, {1, 1, -6, 0}, {1, 1, -5, 0},
    {2, 1, -8, 0}, {2, 1, -7, 0}, {2, 1, -6, 0}, {2, 1, -5, 0}, {3, 1, -8, 0}, {3, 1, -7, 0}, {3, 1, -6, 0}, {3, 1, -5, 0},   // X2' (block - 2)
    {0, 1, -8, 1}, {0, 1, -7, 1}, {0, 1, -6, 1}, {0, 1, -5, 1}, {1, 1, -8, 1}, {1, 1, -7, 1}, {1, 1, -6, 1}, {1, 1, -5, 1},
    {2, 1, -8, 1}, {2, 1, -7, 1}, {2, 1, -6, 1}, {2, 1, -5, 1}, {3, 1, -8, 1}, {3, 1, -7, 1}, {3, 1, -6, 1}, {3, 1, -5, 1}    // X3' (block - 2)
};

// Gram values of 8 blocks from blk0 (one warp): all loads issued before any store
// (map: la_map copied to shared memory -- lanes read different rows, which the constant cache
// would serialise)
__device__ __forceinline__ void la_fill_gram(const RkParams& p, const RkIdx* ring, double (*gring)[LA_NG],
                                             const int8_t (*map)[4], int64_t blk0, int lane) {
  __syncwarp();
  constexpr int PER = (8 * LA_NG + 31) / 32;
  double val[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int e = lane + 32 * q;
    val[q] = 0.0;
    if (e < 8 * LA_NG) {
      const int bl = e / LA_NG, v = e - bl * LA_NG;
      const int64_t b = blk0 + bl;
      const int64_t tb = p.t0 + 4 * b;
      const int sa = map[v][0], ca = map[v][1], sb = map[v][2], cb = map[v][3];
      if (v < 22 || 4 * b + sb >= 0) {   // the earlier block exists in this launch
        const RkIdx ea = ring[(tb + sa) & (RK_RING - 1)];
        const RkIdx ebb = ring[(tb + sb) & (RK_RING - 1)];
        const int ja = ca ? ea.j2 : ea.j1, jb = cb ? ebb.j2 : ebb.j1;
        val[q] = __ldg(p.G + (int64_t)ja * p.npad + jb);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int e = lane + 32 * q;
    if (e < 8 * LA_NG) {
      const int bl = e / LA_NG, v = e - bl * LA_NG;
      gring[(blk0 + bl) & (LA_GR - 1)][v] = val[q];
    }
  }
}

__device__ __forceinline__ void st_async_f64(uint32_t raddr, double a, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr), "d"(a),
               "r"(rbar)
               : "memory");
}

// Warp roles: NWc compute warps (rows), a communication warp (sends the block partials), a reduce
// warp (cluster sum + corrections -> finished products), a fill warp (index + Gram rings ahead),
// a TMA warp (column refills) and a check warp. Compute, communication and reduce warps meet at a
// named barrier per block; the fill and TMA warps run ahead, throttled by progress counters in
// shared memory (release / acquire), so their long operations never stall the step.
// One launch runs the whole inner solve [t0, t1). The inner check (include/ils.h) reads z only, so
// it runs beside the steps: at every check step t_c the communication warp copies z (after exactly
// t_c steps) to a snapshot, the check warp forms its rows of g = A1bar z - b_hat, the 16 partial
// ||g||^2 are exchanged (st.async) and summed in one fixed order in every CTA. On a stop, every
// CTA's communication warp flags its next block message; the first block f whose messages carry a
// flag is the same in every CTA (same messages), and every CTA ends after block f + 2 -- the last
// block any CTA can have sent -- so no message is left in flight. The output is the snapshot z and
// the step count t_c, exactly as if the steps had stopped at t_c.
template <int CC, int U>
__global__ void __launch_bounds__(416, 1) rk_rgs_la_kernel(RkParams p) {
  constexpr int B = 4, NRV = 8;
  static_assert(CC == 16, "the communication warp's cluster sum is written for 16 sources");
  using K = RkBlk<B>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NT = blockDim.x, NW = NT >> 5, NWc = NW - 5, NTc = NWc * 32;
  const bool comm = (warp == NWc), reducer = (warp == NWc + 1), filler = (warp == NWc + 2), tmaw = (warp == NWc + 3);
  const bool checker = (warp == NWc + 4);
  const bool compute = warp < NWc;
  const int rank = (int)cluster_ctarank();
  const int64_t i0 = (int64_t)rank * p.slice;
  const int own = (int)((i0 + p.slice <= p.ppad) ? p.slice : (p.ppad > i0 ? p.ppad - i0 : 0));
  // slot count and slice pitch through shared memory, so that they stay in registers: as kernel
  // parameters they are reloaded from the constant bank (LDC) in every phase of every iteration
  __shared__ int la_cfg[2];
  if (tid == 0) {
    la_cfg[0] = p.nslots;
    la_cfg[1] = p.slicepad;
  }
  __syncthreads();
  const int NS = *(volatile int*)&la_cfg[0], SP = *(volatile int*)&la_cfg[1];
  if (*(volatile int32_t*)&p.st->inner_conv != 0) return;

  uint32_t dyn32 = smem_u32(smem_raw);   // laundered like the static variables below
  asm volatile("" : "+r"(dyn32));
  unsigned char* smem_dyn = reinterpret_cast<unsigned char*>(__cvta_shared_to_generic(dyn32));
  double* slots = reinterpret_cast<double*>(smem_dyn);                 // [NS][2B][slicepad]
  double* zs = slots + (size_t)NS * 2 * B * SP;                        // [npad]
  uint64_t* Ss = reinterpret_cast<uint64_t*>(zs + p.npad);             // [n]
  RkIdx* ring = reinterpret_cast<RkIdx*>(Ss + ((p.n + 1) & ~1));       // [RK_RING]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + RK_RING);        // [NS]
  double* bh_tab = reinterpret_cast<double*>(bars + 8);                 // [n]
  double* rn_tab = bh_tab + ((p.n + 1) & ~1);                          // [n]
  double (*gring)[LA_NG] = reinterpret_cast<double (*)[LA_NG]>(rn_tab + ((p.n + 1) & ~1));   // [LA_GR][LA_NG]
  // The kernel's static shared variables live in one struct reached through a laundered 32-bit shared
  // address: referenced by name, every loop iteration of every role re-derived their cluster-window
  // address with S2UR SR_CgaCtaId (the compiler rematerialises it instead of holding a register), which
  // sat on the step chain (ILS_RK_PROF: ~280 cycles between the axpy barrier and the next products).
  constexpr int NMSG = NRV + 2;                          // 8 products + stop flag + pad
  struct LaSh {
    alignas(16) double wred[2][8][32];   // per warp: value lane & 7 over lane group lane >> 3
    alignas(16) double recv[8][RK_MAXC][NMSG];  // block b in buffer b & 7 (sent two blocks ahead)
    alignas(16) double smail[4][8];   // s1 (0..3), s2 (4..7) of block i, slot i & 3 (reduce -> compute, comm)
    alignas(8) double crecv[2][RK_MAXC];       // check m partials in buffer m & 1
    alignas(8) uint64_t cbar[2];
    alignas(8) int64_t lim_s;      // blocks to run (lowered once on a stop)
    alignas(8) int64_t snap_s;     // z snapshots taken (comm warp)
    alignas(8) int64_t chkd_s;     // checks decided (check warp)
    alignas(8) int64_t stop_t_s;   // step of the check that stopped the solve, -1: none
    alignas(8) uint64_t rbar[8];
    double chkw[16];
    double bnorm_s;
    alignas(8) int64_t filled_s;   // blocks whose index + Gram entries are written
    alignas(8) int64_t done_w[8];  // per compute warp: blocks whose axpy is complete (readers take the minimum)
    // smail[i & 3] written (one arrival by the reduce warp). Four slots: the reduce warp can finish block
    // i + 4 only after its messages were sent, i.e. after every compute thread passed B1 of iteration
    // i + 2 and so its wait for block i
    alignas(8) uint64_t tbar[4];
    int stop_req_s;                  // flag the next block messages
    int zdone_s;                     // the communication warp's last z update is done
    alignas(4) int8_t lam[LA_NG][4];
  };
  __shared__ LaSh la_static;
  uint32_t sh32 = smem_u32(&la_static);
  asm volatile("" : "+r"(sh32));
  LaSh& sh = *reinterpret_cast<LaSh*>(__cvta_shared_to_generic(sh32));
#define wred sh.wred
#define recv sh.recv
#define smail sh.smail
#define crecv sh.crecv
#define cbar sh.cbar
#define lim_s sh.lim_s
#define snap_s sh.snap_s
#define chkd_s sh.chkd_s
#define stop_t_s sh.stop_t_s
#define rbar sh.rbar
#define chkw sh.chkw
#define bnorm_s sh.bnorm_s
#define filled_s sh.filled_s
#define done_w sh.done_w
#define tbar sh.tbar
#define stop_req_s sh.stop_req_s
#define zdone_s sh.zdone_s
#define lam sh.lam
  auto done_min = [&]() {   // blocks finished by every compute warp
    int64_t m = ld_acquire_cta_s64(&done_w[0]);
    for (int w8 = 1; w8 < NWc; ++w8) {
      const int64_t v = ld_acquire_cta_s64(&done_w[w8]);
      m = v < m ? v : m;
    }
    return m;
  };
  if (tid < LA_NG) *reinterpret_cast<int32_t*>(lam[tid]) = *reinterpret_cast<const int32_t*>(la_map[tid]);

  for (int64_t j = tid; j < p.npad; j += NT) zs[j] = p.Z[j];
  for (int j = tid; j < p.n; j += NT) {
    Ss[j] = p.S[j];
    bh_tab[j] = p.bhat[j];
    rn_tab[j] = 1.0 / p.N[j];
  }
  for (int64_t e = tid; e < (int64_t)NS * 2 * B * SP; e += NT) slots[e] = 0.0;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
    for (int s = 0; s < 8; ++s) mbar_init(&rbar[s], 1);
    for (int s = 0; s < 4; ++s) mbar_init(&tbar[s], 1);
    fence_mbar_init();
    for (int s = 0; s < 2; ++s) mbar_init(&cbar[s], 1);
    fence_mbar_init();
    for (int s = 0; s < 8; ++s) mbar_arrive_expect_tx(&rbar[s], CC * NMSG * 8);
    for (int s = 0; s < 2; ++s) mbar_arrive_expect_tx(&cbar[s], CC * 8);
    for (int s = 0; s < 8; ++s) done_w[s] = 0;
    snap_s = 0;
    chkd_s = 0;
    stop_t_s = -1;
    stop_req_s = 0;
    zdone_s = 0;
  }
  double bnorm = 1.0;
  if (p.t0 == 0) {
    double v = 0.0;
    for (int j = tid; j < p.n; j += NT) v = fma(p.bhat[j], p.bhat[j], v);
    v = warp_sum(v);
    if (lane == 0) chkw[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += chkw[w];
      bnorm_s = sqrt(s);
    }
    __syncthreads();
    bnorm = bnorm_s;
  }
  __syncthreads();
  cluster_sync_all();
  if (bnorm == 0.0) {
    if (rank == 0 && tid == 0) {
      p.st->inner_steps = 0;
      p.st->inner_conv = 1;
    }
    return;
  }
  const int64_t nblk = (p.t1 - p.t0 + B - 1) / B;
  if (tid == 0) lim_s = nblk;
  const uint32_t slice_bytes = (uint32_t)own * sizeof(double);
  // 16 blocks ahead before the step loop starts, split over the fill and TMA warps (indices of both
  // halves first: the Gram values of a block read the indices of the two blocks before it)
  if (filler || tmaw) rk_fill_indices(p, Ss, ring, p.t0 + (tmaw ? 32 : 0), lane, bh_tab, rn_tab);
  __syncthreads();
  if (filler || tmaw) la_fill_gram(p, ring, gring, lam, tmaw ? 8 : 0, lane);
  if (filler && lane == 0) filled_s = 16;
  auto issue = [&](int64_t blk, int slot) {   // 2B column slices of block blk (one thread)
    double* dst = slots + (size_t)slot * 2 * B * SP;
    mbar_arrive_expect_tx(&bars[slot], 2 * B * slice_bytes);
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const RkIdx e = ring[(p.t0 + blk * B + i) & (RK_RING - 1)];
      bulk_g2s(dst + (2 * i) * SP, p.A1T + (int64_t)e.j1 * p.ppad + i0, slice_bytes, &bars[slot]);
      bulk_g2s(dst + (2 * i + 1) * SP, p.A1T + (int64_t)e.j2 * p.ppad + i0, slice_bytes, &bars[slot]);
    }
  };
  __syncthreads();
  if (tmaw && lane == 0 && own > 0) {
    fence_proxy_async();
    for (int64_t b = 0; b < NS && b < nblk; ++b) issue(b, (int)b);
  }

  if (filler) {   // ---- fill warp: index + Gram rings, at most 24 blocks ahead of the consumers
    int64_t f = 16;
    bool quit = false;
    const bool fprof = p.prof && lane == 0;
    long long hf[2] = {0, 0};   // throttle wait, fill work
    long long fc0 = fprof ? clock64() : 0;
    while (f < nblk && !quit) {
      while (f + 8 > done_min() + LA_GR) {   // slot of block done must stay
        if (f >= ld_acquire_cta_s64(&lim_s) + 8) {            // stopped: nothing further is needed
          quit = true;
          break;
        }
        if (p.nap) __nanosleep(p.nap);   // leave the issue slots to the compute warp of this SMSP
      }
      if (quit) break;
      if (fprof) {
        const long long c_ = clock64();
        hf[0] += c_ - fc0;
        fc0 = c_;
      }
      rk_fill_indices(p, Ss, ring, p.t0 + 4 * f, lane, bh_tab, rn_tab);
      la_fill_gram(p, ring, gring, lam, f, lane);
      f += 8;
      __syncwarp();
      if (lane == 0) st_release_cta_s64(&filled_s, f);
      if (fprof) {
        const long long c_ = clock64();
        hf[1] += c_ - fc0;
        fc0 = c_;
      }
    }
    if (fprof) {
      p.prof[128 + rank * 8 + 5] += hf[0];
      p.prof[128 + rank * 8 + 6] += hf[1];
    }
  } else if (tmaw) {   // ---- TMA warp: refill slot (b % NS) once block b - NS is done
    if (lane == 0 && own > 0) {
      int slot = 0;
      int64_t b = NS;
      for (; b < nblk; ++b) {
        bool quit = false;
        while (done_min() < b - NS + 1 || ld_acquire_cta_s64(&filled_s) <= b) {
          if (b >= ld_acquire_cta_s64(&lim_s)) {
            quit = true;
            break;
          }
          if (p.nap) __nanosleep(p.nap);
        }
        if (quit) break;
        fence_proxy_async();
        issue(b, slot);
        if (++slot == NS) slot = 0;
      }
      // drain: blocks issued at or past the final limit were never consumed -- their copies must
      // land before the CTA exits (every block below it was waited for by the compute warps)
      const int64_t issued = (b < nblk) ? b : nblk;
      const int64_t lim_end = done_min();
      for (int64_t d = lim_end; d < issued; ++d) mbar_wait(&bars[d % NS], (uint32_t)((d / NS) & 1));
    }
  } else if (checker) {   // ---- check warp: g = A1bar z - b_hat on each snapshot, cluster sum, decide
    const int64_t per = (p.n + CC - 1) / CC;
    const int64_t j0 = (int64_t)rank * per, j1 = (j0 + per < p.n) ? j0 + per : p.n;
    const double* zsn = p.Zsnap + (int64_t)rank * p.npad;
    int64_t m = 0;
    for (int64_t tc = (p.t0 / p.ce + 1) * p.ce; tc < p.t1; tc += p.ce, ++m) {
      bool gone = false;   // the solve ended before this snapshot was taken
      while (ld_acquire_cta_s64(&snap_s) <= m) {
        if (*(volatile int*)&zdone_s) {
          __threadfence_block();
          gone = ld_acquire_cta_s64(&snap_s) <= m;
          break;
        }
        if (p.nap) __nanosleep(4 * p.nap);   // snapshots come every check_every steps
      }
      if (gone) break;
      double part = 0.0;
      for (int64_t j = j0; j < j1; ++j) {   // rows in order, each a warp dot product
        const double* gr = p.G + j * p.npad;
        double a0 = 0.0, a1 = 0.0;
        int64_t c = lane;
        for (; c + 32 < p.npad; c += 64) {
          a0 = fma(gr[c], zsn[c], a0);
          a1 = fma(gr[c + 32], zsn[c + 32], a1);
        }
        if (c < p.npad) a0 = fma(gr[c], zsn[c], a0);
        const double gj = warp_sum(a0 + a1) - bh_tab[j];
        part = fma(gj, gj, part);
      }
      const int bsel = (int)(m & 1);
      if (lane < CC)
        st_async_f64(map_shared_rank(smem_u32(&crecv[bsel][rank]), (uint32_t)lane), part,
                     map_shared_rank(smem_u32(&cbar[bsel]), (uint32_t)lane));
      mbar_wait_cluster(&cbar[bsel], (uint32_t)((m >> 1) & 1));
      double g2 = 0.0;
      for (int c = 0; c < CC; ++c) g2 += crecv[bsel][c];
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&cbar[bsel], CC * 8);   // for check m + 2
      const bool stop = sqrt(g2) <= p.inner_tol * bnorm;
      if (lane == 0) {
        if (stop) {
          stop_t_s = tc;
          stop_req_s = 1;
        }
        st_release_cta_s64(&chkd_s, m + 1);
      }
      if (stop) break;
    }
  } else if (reducer) {   // ---- reduce warp: finished products of block i, then its B-step recurrence
    // The scalars s1, s2 of a block are needed by every compute thread, by the z updates and by the
    // next blocks' corrections: the reduce warp forms them once (every lane redundantly, same
    // operations in the same order as the compute threads did before) and posts them; the compute
    // warps only wait for them and run their axpy (the recurrence and its 30 table loads left their
    // step chain: ~390 of 2140 cycles per block at c1).
    const bool rprof = p.prof && lane == 0;
    long long hr[2] = {0, 0};
    for (int64_t i = 0; i < *(volatile int64_t*)&lim_s; ++i) {
      // in-block Gram values and index entries of block i (filled: block i - 1's messages were sent
      // after the compute warps saw blocks <= i filled), loaded ahead of the message wait
      double T[K::NV];
      {
        const double* gi = gring[i & (LA_GR - 1)];
#pragma unroll
        for (int v = NRV; v < K::NV; ++v) T[v] = gi[v - NRV];
      }
      const int64_t t = p.t0 + i * B;
      double bh1[B], rn1[B], rn2[B];
#pragma unroll
      for (int k = 0; k < B; ++k) {
        const RkIdx ix = ring[(t + k) & (RK_RING - 1)];
        bh1[k] = ix.bh1;
        rn1[k] = ix.rn1;
        rn2[k] = ix.rn2;
      }
      long long rc0 = rprof ? clock64() : 0;
      const int b4 = (int)(i & 7);
      mbar_wait(&rbar[b4], (uint32_t)((i >> 3) & 1));
      if (rprof) {
        const long long c_ = clock64();
        hr[0] += c_ - rc0;
        rc0 = c_;
      }
      // lane (v, g): sources 4g .. 4g+3 of value v (cluster sum in a fixed tree) plus the
      // correction terms of step m = g of blocks i-1 and i-2 (missing from the stale state S_{i-2}),
      // then a butterfly over the four lane groups
      const int v = lane & 7, g = lane >> 3, k = v & 3;
      const bool isq = v >= B;
      const double* gn = gring[i & (LA_GR - 1)];
      double tot = (recv[b4][4 * g][v] + recv[b4][4 * g + 1][v]) + (recv[b4][4 * g + 2][v] + recv[b4][4 * g + 3][v]);
#pragma unroll
      for (int d = 1; d <= 2; ++d) {
        if (i >= d) {
          const double* sm = smail[(i - d) & 3];
          const int o = 22 + 48 * (d - 1) + 4 * k + g;
          const double ga = gn[o + (isq ? 16 : 0)];
          const double gb = isq ? gn[o + 32] : 0.0;
          tot = fma(sm[g], ga, tot);
          tot = fma(-sm[B + g], gb, tot);
        }
      }
      tot += __shfl_xor_sync(0xffffffffu, tot, 8);
      tot += __shfl_xor_sync(0xffffffffu, tot, 16);
#pragma unroll
      for (int q = 0; q < NRV; ++q) T[q] = __shfl_sync(0xffffffffu, tot, q);
      double s1[B], s2[B];
#pragma unroll
      for (int kk = 0; kk < B; ++kk) {
        double dw = T[K::P(kk)];
#pragma unroll
        for (int m = 0; m < kk; ++m) dw = fma(s1[m], T[K::AA(kk, m)], dw);
        s1[kk] = (bh1[kk] - dw) * rn1[kk];
        double dr = T[K::Q(kk)];
#pragma unroll
        for (int m = 0; m < kk; ++m) {
          dr = fma(s1[m], T[K::BA(kk, m)], dr);
          dr = fma(-s2[m], T[K::BB(kk, m)], dr);
        }
        dr = fma(s1[kk], T[K::BA(kk, kk)], dr);
        s2[kk] = dr * rn2[kk];
      }
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < B; ++kk) {
          smail[i & 3][kk] = s1[kk];
          smail[i & 3][B + kk] = s2[kk];
        }
      }
      // stop flags of block i (identical messages in every CTA): end after block i + 2
      const bool flag = __any_sync(0xffffffffu, lane < CC && recv[b4][lane][NRV] != 0.0);
      if (flag && lane == 0 && lim_s > i + 3) lim_s = i + 3;
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&tbar[i & 3]);
        mbar_arrive_expect_tx(&rbar[b4], CC * NMSG * 8);   // for block i + 8
      }
      if (rprof) hr[1] += clock64() - rc0;
    }
    if (rprof) {
      p.prof[128 + rank * 8 + 0] += hr[0];
      p.prof[128 + rank * 8 + 1] += hr[1];
    }
  } else {   // ---- compute warps and the communication warp
    double w[U], r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = tid + u * NTc;
      const bool in = compute && (e < own);
      w[u] = in ? p.W[i0 + e] : 0.0;
      r[u] = in ? p.Rv[i0 + e] : 0.0;
    }
    int64_t known_filled = 0;
    int sl_nb = NS - 1, sl_i = 0;
    uint32_t ph_nb = 1;
    const bool prof = p.prof && tid == 0;
    long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long hx[5] = {0, 0, 0, 0, 0};   // helper-warp timers (lane 0 of the reduce / comm warp)
    long long tc = clock64();
#define LAP(k)                       \
  if (prof) {                        \
    const long long c_ = clock64();  \
    pc[k] += c_ - tc;                \
    tc = c_;                         \
  }
    int64_t next_tc = (p.t0 / p.ce + 1) * p.ce;   // next check step (communication warp)
    int64_t msnap = 0;                            // snapshots taken
    // z updates of block blk in step order (communication warp), with the z snapshot of every check
    // step inside the block taken after exactly that many steps
    auto zupd = [&](int64_t blk) {
      const int64_t tp = p.t0 + blk * B;
      const double* sm = smail[blk & 3];
      int kdone = 0;
      while (next_tc > tp && next_tc <= tp + B && next_tc < p.t1) {
        const int kk = (int)(next_tc - tp);
        if (lane == 0)
          for (int k = kdone; k < kk; ++k) zs[ring[(tp + k) & (RK_RING - 1)].j2] += sm[B + k];
        kdone = kk;
        while (ld_acquire_cta_s64(&chkd_s) < msnap) {   // the previous snapshot is still being read
        }
        if (*(volatile int64_t*)&stop_t_s < 0) {
          __syncwarp();
          double* dst = p.Zsnap + (int64_t)rank * p.npad;
          for (int64_t j = lane; j < p.npad; j += 32) dst[j] = zs[j];
          __threadfence_block();
          __syncwarp();
          if (lane == 0) st_release_cta_s64(&snap_s, msnap + 1);
          ++msnap;
        }
        next_tc += p.ce;
      }
      if (lane == 0)
        for (int k = kdone; k < B; ++k) zs[ring[(tp + k) & (RK_RING - 1)].j2] += sm[B + k];
      __syncwarp();
    };
    for (int64_t i = -2; i < *(volatile int64_t*)&lim_s; ++i) {
      const int64_t nb = i + 2;
      const int64_t lim = *(volatile int64_t*)&lim_s;
      if (++sl_nb == NS) {
        sl_nb = 0;
        ph_nb ^= 1u;
      }
      sl_i = sl_nb - 2 < 0 ? sl_nb - 2 + NS : sl_nb - 2;   // slot of block i (NS >= 3)
      // ---- phase 1 (compute warps): state products of block nb = i + 2 on S_i (blocks i, i+1 not applied)
      LAP(4)
      if (compute && nb < lim) {
        if (known_filled <= nb + 1 && known_filled < nblk) {   // ring + Gram entries of blocks nb, nb+1
          do {
            known_filled = ld_acquire_cta_s64(&filled_s);
          } while (known_filled <= nb + 1 && known_filled < nblk);
        }
        LAP(7)
        if (own > 0) mbar_wait(&bars[sl_nb], ph_nb);
        LAP(6)
        const double* cols = slots + (size_t)sl_nb * 2 * B * SP;
        double acc[NRV];
#pragma unroll
        for (int v = 0; v < NRV; ++v) acc[v] = 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = tid + u * NTc;
#pragma unroll
          for (int k = 0; k < B; ++k) {
            acc[K::P(k)] = fma(cols[(2 * k) * SP + e], w[u], acc[K::P(k)]);
            acc[K::Q(k)] = fma(cols[(2 * k + 1) * SP + e], r[u], acc[K::Q(k)]);
          }
        }
        wred[nb & 1][warp][lane] = warp_reduce_scatter_groups<NRV>(acc, lane);   // groups summed by the comm warp
      }
      LAP(0)
      named_bar_sync(1, NTc + 32);   // B1: compute warps + communication warp
      LAP(1)
      if (comm) {
        const bool cprof = p.prof && lane == 0;
        long long cc0 = cprof ? clock64() : 0;
        if (nb < *(volatile int64_t*)&lim_s) {
          double v = 0.0;
          for (int w8 = 0; w8 < NWc; ++w8) v += wred[nb & 1][w8][lane];
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          const double v0 = __shfl_sync(0xffffffffu, v, (2 * lane) & 7);
          const double v1 = __shfl_sync(0xffffffffu, v, (2 * lane + 1) & 7);
          const int b4 = (int)(nb & 7);
          const uint32_t la = smem_u32(&recv[b4][rank][2 * (lane & 3)]);
          const uint32_t lb = smem_u32(&rbar[b4]);
          const double fl = *(volatile int*)&stop_req_s ? 1.0 : 0.0;   // stop flag (lane NRV / 2)
          const uint32_t la2 = smem_u32(&recv[b4][rank][(lane < NRV / 2) ? 2 * (lane & 3) : NRV]);
          if (lane <= NRV / 2)
            for (int c = 0; c < CC; ++c)
              st_async_v2f64(map_shared_rank(la2, (uint32_t)c), lane < NRV / 2 ? v0 : fl, lane < NRV / 2 ? v1 : 0.0,
                             map_shared_rank(lb, (uint32_t)c));
          __syncwarp();
          if (cprof) {
            const long long c_ = clock64();
            hx[3] += c_ - cc0;
            cc0 = c_;
          }
        }
        if (i >= 1) zupd(i - 1);   // z updates of block i - 1, sequential order
        continue;
      }
      if (i < 0) continue;
      // ---- phase 2 (compute warps): block i, with the scalars posted by the reduce warp
      mbar_wait(&tbar[i & 3], (uint32_t)((i >> 2) & 1));
      LAP(2)
      double s1[B], s2[B];
      {
        const double2* sm2 = reinterpret_cast<const double2*>(smail[i & 3]);
#pragma unroll
        for (int k = 0; k < B; k += 2) {
          const double2 a = sm2[k / 2], b = sm2[(B + k) / 2];
          s1[k] = a.x;
          s1[k + 1] = a.y;
          s2[k] = b.x;
          s2[k + 1] = b.y;
        }
      }
      LAP(3)
      const double* cols = slots + (size_t)sl_i * 2 * B * SP;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = tid + u * NTc;
#pragma unroll
        for (int k = 0; k < B; ++k) {
          const double xa = cols[(2 * k) * SP + e], xb = cols[(2 * k + 1) * SP + e];
          w[u] = fma(s1[k], xa, w[u]);
          r[u] = fma(s1[k], xa, r[u]);
          r[u] = fma(-s2[k], xb, r[u]);
        }
      }
      LAP(5)
      // this warp finished block i's axpy (its loads of slot sl_i have returned: their values were
      // consumed); the slot is reusable once every compute warp says so. No CTA barrier here: the warps
      // meet once per iteration, at B1 (a second barrier cost ~220 cycles of skew per block)
      __syncwarp();
      if (lane == 0) st_relaxed_cta_s64(&done_w[warp], i + 1);
      LAP(5)
    }
#undef LAP
    if (prof)
      for (int k = 0; k < 8; ++k) p.prof[rank * 8 + k] += pc[k];
    if (p.prof && lane == 0 && comm)
      for (int k = 0; k < 5; ++k)
        if (hx[k]) p.prof[128 + rank * 8 + k] += hx[k];
    if (compute) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = tid + u * NTc;
        if (e < own) {
          p.W[i0 + e] = w[u];
          p.Rv[i0 + e] = r[u];
        }
      }
    }
    if (comm) {   // the last block's z updates (and snapshots), once its scalars are posted
      const int64_t lim = *(volatile int64_t*)&lim_s;
      while (done_min() < lim) {
      }
      if (lim >= 1) zupd(lim - 1);
      __threadfence_block();
      if (lane == 0) *(volatile int*)&zdone_s = 1;
    }
  }
  __syncthreads();
  const int64_t tstop = stop_t_s;
  if (rank == 0) {
    const double* zo = (tstop >= 0) ? p.Zsnap : zs;   // a stop returns z after exactly t_c steps
    for (int64_t j = tid; j < p.npad; j += NT) p.Z[j] = zo[j];
    if (tid == 0 && tstop >= 0) {
      p.st->inner_steps = tstop;
      p.st->inner_conv = 1;
    }
  }
  cluster_sync_all();
}

#undef wred
#undef recv
#undef smail
#undef crecv
#undef cbar
#undef lim_s
#undef snap_s
#undef chkd_s
#undef stop_t_s
#undef rbar
#undef chkw
#undef bnorm_s
#undef filled_s
#undef done_w
#undef tbar
#undef stop_req_s
#undef zdone_s
#undef lam

template <int CC, int U>
static int launch_rkla(Handle& h, RkParams& p, int nt, size_t smem) {
  auto kern = rk_rgs_la_kernel<CC, U>;
  ILS_CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ILS_CU(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CC);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ILS_CU(cudaLaunchKernelEx(&cfg, kern, p));
  ILS_LAUNCHED("rk_rgs_la_kernel");
  return ILS_OK;
}

template <int U>
static int dispatch_rk_c(Handle& h, RkParams& p, int nt, size_t smem) {
  switch (p.C) {
    case 1: return launch_rk<1, U>(h, p, nt, smem);
    case 2: return launch_rk<2, U>(h, p, nt, smem);
    case 4: return launch_rk<4, U>(h, p, nt, smem);
    case 8: return launch_rk<8, U>(h, p, nt, smem);
    default: return launch_rk<16, U>(h, p, nt, smem);
  }
}

template <int CC, int U, int B>
static int launch_rkb(Handle& h, RkParams& p, int nt, size_t smem) {
  auto kern = rk_rgs_block_kernel<CC, U, B>;
  ILS_CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CC);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = h.stream;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (CC > 1) {
    ILS_CU(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CC;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    na = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  ILS_CU(cudaLaunchKernelEx(&cfg, kern, p));
  ILS_LAUNCHED("rk_rgs_block_kernel");
  return ILS_OK;
}

template <int U, int B>
static int dispatch_rkb_c(Handle& h, RkParams& p, int nt, size_t smem) {
  switch (p.C) {
    case 1: return launch_rkb<1, U, B>(h, p, nt, smem);
    case 2: return launch_rkb<2, U, B>(h, p, nt, smem);
    case 4: return launch_rkb<4, U, B>(h, p, nt, smem);
    case 8: return launch_rkb<8, U, B>(h, p, nt, smem);
    default: return launch_rkb<16, U, B>(h, p, nt, smem);
  }
}

static int dispatch_rkb(Handle& h, RkParams& p, int U, int B, int nt, size_t smem) {
  if (B == 2) return (U == 4) ? dispatch_rkb_c<4, 2>(h, p, nt, smem) : dispatch_rkb_c<8, 2>(h, p, nt, smem);
  if (U == 2) return dispatch_rkb_c<2, 4>(h, p, nt, smem);
  return (U == 4) ? dispatch_rkb_c<4, 4>(h, p, nt, smem) : dispatch_rkb_c<8, 4>(h, p, nt, smem);
}

static int rk_cluster_size(Handle& h) {
  // one CTA up to 2048 rows; otherwise a cluster of up to 16 CTAs (non-portable size)
  if (h.ppad <= 2048) return 1;
  int c = (int)((h.ppad + 511) / 512);
  return c >= 16 ? 16 : (c >= 8 ? 8 : (c >= 4 ? 4 : 2));
}

int rk_rgs_inner(Handle& h, const double* bhat, double* z, uint64_t seed, int64_t k, int64_t max_inner,
                 int64_t check_every, double inner_tol, int64_t* steps_out) {
  const int64_t ce = check_every > 0 ? check_every : h.n;
  const cudaStream_t st = h.stream;
  {   // w, r, az [ppad], z [npad], z snapshots of the look-ahead kernel [RK_MAXC][npad]
    const size_t words = (size_t)3 * h.ppad + (size_t)(1 + RK_MAXC) * h.npad;
    if (!h.rk_state || h.rk_state_words < words) {
      if (h.rk_state) cudaFreeAsync(h.rk_state, st);
      ILS_CU(cudaMallocAsync(&h.rk_state, words * sizeof(double), st));
      h.rk_state_words = words;
    }
  }
  double* W = h.rk_state;
  double* Rv = W + h.ppad;
  double* AZ = Rv + h.ppad;
  double* Z = AZ + h.ppad;
  ILS_CU(cudaMemsetAsync(h.rk_state, 0, (size_t)(3 * h.ppad + h.npad) * sizeof(double), st));
  ILS_CU(cudaMemsetAsync(&h.dstat->inner_conv, 0, sizeof(int32_t), st));
  ILS_CU(cudaMemsetAsync(&h.dstat->inner_steps, 0, sizeof(int64_t), st));

  RkParams p{};
  p.A1T = h.A1T;
  p.ppad = h.ppad;
  p.npad = h.npad;
  p.n = (int)h.n;
  p.N = h.N;
  p.S = h.S;
  p.bhat = bhat;
  p.W = W;
  p.Rv = Rv;
  p.Z = Z;
  p.seed = seed;
  p.k = (uint32_t)k;
  p.max_inner = max_inner;
  p.st = h.dstat;
  {
    // ns per poll of the look-ahead kernel's helper warps (fill, TMA, check): sleeping polls leave the
    // issue slots of their SMSPs to the compute warps (c1: 198.8 -> 195.1 ms at 300 ns; 0 = spin)
    const char* e = getenv("ILS_RK_NAP");
    p.nap = (e && atoi(e) >= 0) ? atoi(e) : 300;
  }
  // launch geometry (fixed for the whole solve). Blocked kernel (4 steps per reduction) when the
  // CTA has <= 256 threads and >= 2 slots of 8 column slices fit; else the single-step kernel.
  int C = rk_cluster_size(h);
  {
    const char* e = getenv("ILS_RK_CLUSTER");   // experiment override: cluster size 1..16 (power of 2)
    if (e && atoi(e) >= 1) C = atoi(e);
  }
  int Bk = 4;
  {
    const char* e = getenv("ILS_RK_BLOCK");     // experiment override: steps per reduction 1, 2, 4
    if (e && (atoi(e) == 1 || atoi(e) == 2 || atoi(e) == 4)) Bk = atoi(e);
  }
  int U = 8, nt = 32;
  bool blocked = false;
  int Bsel = Bk;   // steps per reduction of the blocked kernel actually launched
  size_t smem = 0;
  for (;;) {
    p.C = C;
    p.slice = (int)(((h.ppad + C - 1) / C + 1) / 2 * 2);
    // rows per thread: one warp with U = 8 for slices <= 256, U = 4 up to 2048, else U = 8
    U = (p.slice <= 256) ? 8 : (p.slice <= 2048 ? 4 : 8);
    {
      const char* e = getenv("ILS_RK_U");   // experiment override of rows per thread (2, 4, 8)
      if (e && (atoi(e) == 2 || atoi(e) == 4 || atoi(e) == 8)) U = atoi(e);
    }
    const int nw = (p.slice + 32 * U - 1) / (32 * U);
    if (nw > RK_MAXW) {
      set_error("RK-RGS: row slice too long for the register-resident kernel (p > 65536)");
      return ILS_ERR_UNSUPPORTED;
    }
    nt = 32 * nw;
    p.slicepad = U * nt;
    const size_t fixed = (size_t)h.npad * 8 + (size_t)((h.n + 1) & ~1) * 8 + RK_RING * sizeof(RkIdx) + 16 * 8 + 256;
    const size_t budget = 200 * 1024;
    const size_t slot1 = (size_t)2 * p.slicepad * 8;
    const size_t fixed4 = fixed + 64 + (size_t)2 * ((h.n + 1) & ~1) * 8;   // + b_hat, 1/N tables
    const size_t fixed_g = (size_t)RK_RING * sizeof(RkIdx) + 16 * 8 + 256;
    // blocked kernel (B steps per cluster reduction): with z / sampling tables in shared memory when
    // two slots of 2B column slices fit next to them, else (long slices at large n, e.g. c2) with
    // those tables in global memory (gmode) and the largest B whose two slots fit; else one step
    // per reduction (rk_rgs_kernel; z in global memory when it does not fit either)
    blocked = false;
    p.gmode = 0;
    Bsel = Bk;
    if (!h.rk_single_step && Bk > 1 && nt <= 512) {
      if (!h.large && fixed4 + 2 * (size_t)Bk * slot1 <= budget) {
        blocked = true;
      } else {
        for (int bb = Bk; bb >= 2 && !blocked; bb /= 2)
          if (fixed_g + 2 * (size_t)bb * slot1 <= budget) {
            blocked = true;
            p.gmode = 1;
            Bsel = bb;
          }
      }
    }
    if (!blocked) p.gmode = (h.large || fixed + 2 * slot1 > budget) ? 1 : 0;
    // gmode blocked: keep the sampler's prefix sums in shared memory when they fit (the fill warp's
    // binary search then runs on shared memory instead of dependent L2 loads)
    const size_t s_bytes = (size_t)((h.n + 1) & ~1) * 8;
    p.s_smem = (blocked && p.gmode && fixed_g + s_bytes + 2 * (size_t)Bsel * slot1 <= budget) ? 1 : 0;
    const size_t slot_bytes = blocked ? (size_t)Bsel * slot1 : slot1;
    const size_t fixed_used = p.gmode ? fixed_g + (p.s_smem ? s_bytes : 0) : (blocked ? fixed4 : fixed);
    if (fixed_used + 2 * slot_bytes > budget) {
      set_error("RK-RGS: shared memory too small for this problem size");
      return ILS_ERR_UNSUPPORTED;
    }
    int NS = (int)((budget - fixed_used) / slot_bytes);
    if (NS > 8) NS = 8;
    p.nslots = NS;
    smem = fixed_used + (size_t)NS * slot_bytes;
    // probe that a cluster of this size can be scheduled
    if (C > 1) {
      int ncl = 0;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C);
      cfg.blockDim = dim3(nt);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a;
      a.id = cudaLaunchAttributeClusterDimension;
      a.val.clusterDim.x = C;
      a.val.clusterDim.y = 1;
      a.val.clusterDim.z = 1;
      cfg.attrs = &a;
      cfg.numAttrs = 1;
      void* kern = blocked ? ((Bsel == 2) ? ((U == 4) ? (void*)rk_rgs_block_kernel<16, 4, 2> : (void*)rk_rgs_block_kernel<16, 8, 2>)
                              : (U == 2) ? (void*)rk_rgs_block_kernel<16, 2, 4>
                              : (U == 4) ? (void*)rk_rgs_block_kernel<16, 4, 4> : (void*)rk_rgs_block_kernel<16, 8, 4>)
                           : ((U == 4) ? (void*)rk_rgs_kernel<16, 4> : (void*)rk_rgs_kernel<16, 8>);
      cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess || ncl < 1) {
        cudaGetLastError();
        if (C > 2) {
          C /= 2;
          continue;
        }
        set_error("RK-RGS: no cluster configuration fits");
        return ILS_ERR_UNSUPPORTED;
      }
    }
    break;
  }

  // look-ahead variant (default for the 16-CTA blocked geometry; ILS_RK_LA=0 disables): three
  // helper warps and a 32-block Gram ring in shared memory, A1bar built once per handle
  bool la = false;
  size_t smem_la = 0;
  {
    const char* e = getenv("ILS_RK_LA");
    if (!(e && e[0] == '0') && blocked && !p.gmode && C == 16 && Bsel == 4 && (U == 2 || U == 4 || U == 8) && nt + 160 <= 416 && !h.large &&
        !h.sparse) {
      // the Gram ring replaces one column slot when both do not fit (>= 3 slots: blocks i .. i+2 live)
      const size_t ring_bytes = (size_t)LA_GR * LA_NG * sizeof(double), slot_la = (size_t)2 * Bsel * p.slicepad * 8;
      smem_la = smem + ring_bytes;
      const size_t cap = 227 * 1024 - 16 * 1024;   // the kernel's static shared memory (~15.4 KB) counts too
      while (smem_la > cap && p.nslots > 4) {
        p.nslots -= 1;
        smem_la -= slot_la;
      }
      if (smem_la <= cap) {
        int rc = build_gram(h);
        if (rc) return rc;
        p.G = h.G;
        la = true;
      }
    }
  }
  // chunks of check_every steps, each followed by the full-GPU inner check; launches are queued
  // ahead (kernels of a stopped solve return at once) and the stop flag is read every kBatch checks
  int kBatch = 8;   // chunks queued between reads of the stop flag
  {
    const char* e = getenv("ILS_RK_KBATCH");   // experiment override
    if (e && atoi(e) >= 1 && atoi(e) <= 256) kBatch = atoi(e);
  }
  long long* prof = nullptr;
  {
    const char* e = getenv("ILS_RK_PROF");
    if (e && e[0] == '1' && blocked) {   // (the look-ahead kernel reports: compute phase1, B1, recv, phase2 | comm B1, send, refill, fill)
      ILS_CU(cudaMallocAsync(&prof, 16 * 16 * sizeof(long long), st));
      ILS_CU(cudaMemsetAsync(prof, 0, 16 * 16 * sizeof(long long), st));
    }
  }
  p.prof = prof;
  {   // one-CTA problems: the whole inner solve in one launch (rk_rgs_small_kernel)
    const char* e = getenv("ILS_RK_SMALL");
    const size_t small_smem = ((size_t)h.npad * h.ppad + h.npad + h.ppad + 3 * (size_t)((h.n + 1) & ~1)) * 8 +
                              RK_RING * sizeof(RkIdx) + 64;
    if (C == 1 && !(e && e[0] == '0') && small_smem <= 200 * 1024 && h.ppad <= 2048 && !prof) {
      // one row per thread up to 256 rows (8 warps share the products and reductions), then U rows
      const int nts = (int)((h.ppad + 31) / 32 * 32);
      int ntc = nts > 256 ? 256 : nts;
      {
        const char* e = getenv("ILS_RK_SMALL_NT");   // experiment override: CTA size (32 .. 256)
        if (e && atoi(e) >= 32 && atoi(e) <= 256 && (atoi(e) & 31) == 0 && (int64_t)atoi(e) * 8 >= h.ppad) ntc = atoi(e);
      }
      const int Us = (int)((h.ppad + ntc - 1) / ntc);
      p.slice = (int)h.p;   // rows >= p are padding (azs)
      p.t0 = 0;
      p.t1 = max_inner;
      // Gram lookups (A1bar staged next to A1) when it fits: 8 reduced values per block instead of 30
      const size_t gs_bytes = (size_t)h.npad * h.npad * 8;
      const char* elk = getenv("ILS_RK_SMALL_LOOKUP");   // experiment override: 0 = reduce all 30 values
      const bool lk = small_smem + gs_bytes <= 200 * 1024 && !(elk && elk[0] == '0');
      if (lk) {
        int rc = build_gram(h);
        if (rc) return rc;
        p.G = h.G;
      }
      const size_t smem_k = small_smem + (lk ? gs_bytes : 0);
      ILS_CU(cudaEventRecord(h.evk0, st));
      void* kern = lk ? ((Us <= 1) ? (void*)rk_rgs_small_kernel<1, true>
                         : (Us <= 2) ? (void*)rk_rgs_small_kernel<2, true>
                         : (Us <= 4) ? (void*)rk_rgs_small_kernel<4, true> : (void*)rk_rgs_small_kernel<8, true>)
                      : ((Us <= 1) ? (void*)rk_rgs_small_kernel<1, false>
                         : (Us <= 2) ? (void*)rk_rgs_small_kernel<2, false>
                         : (Us <= 4) ? (void*)rk_rgs_small_kernel<4, false> : (void*)rk_rgs_small_kernel<8, false>);
      ILS_CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_k));
      double itol = inner_tol;
      int64_t ce64 = ce;
      void* args[] = {&p, &z, &ce64, &itol};
      ILS_CU(cudaLaunchKernel(kern, dim3(1), dim3(ntc), args, smem_k, st));
      ILS_LAUNCHED("rk_rgs_small_kernel");
      ILS_CU(cudaEventRecord(h.evk1, st));
      ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
      ILS_CU(cudaStreamSynchronize(st));
      const int64_t steps = h.hstat->inner_conv ? h.hstat->inner_steps : max_inner;
      if (steps_out) *steps_out = steps;
      const double pd = (double)h.p, nd = (double)h.n;
      hot_account(h, 1, (double)steps * 16.0 * pd + (double)(steps / ce) * 16.0 * pd * nd, 1);
      return ILS_OK;
    }
  }
  ILS_CU(cudaEventRecord(h.evk0, st));
  int64_t t = 0, nchecks = 0;
  int pending = 0;
  bool conv = false;
  if (la) {   // the whole inner solve in one launch, the inner checks inside the kernel
    p.t0 = 0;
    p.t1 = max_inner;
    p.ce = ce;
    p.inner_tol = inner_tol;
    p.Zsnap = Z + h.npad;
    const int r = (U == 2)   ? launch_rkla<16, 2>(h, p, nt + 160, smem_la)
                  : (U == 4) ? launch_rkla<16, 4>(h, p, nt + 160, smem_la)
                             : launch_rkla<16, 8>(h, p, nt + 160, smem_la);
    if (r) return r;
    nchecks = max_inner / ce;
    t = max_inner;
  }
  while (t < max_inner) {
    const int64_t t1 = (t + ce < max_inner) ? t + ce : max_inner;
    p.t0 = t;
    p.t1 = t1;
    const int r = blocked ? dispatch_rkb(h, p, U, Bsel, nt, smem)
                            : ((U == 8) ? dispatch_rk_c<8>(h, p, nt, smem) : dispatch_rk_c<4>(h, p, nt, smem));
    if (r) return r;
    t = t1;
    if (t % ce == 0) {
      const int rc = rk_check(h, Z, bhat, W, Rv, AZ, inner_tol, t);
      if (rc) return rc;
      ++nchecks;
    }
    if (++pending == kBatch || t >= max_inner) {
      ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
      ILS_CU(cudaStreamSynchronize(st));
      pending = 0;
      if (h.hstat->inner_conv) {
        conv = true;
        break;
      }
    }
  }
  ILS_CU(cudaEventRecord(h.evk1, st));
  ILS_CU(cudaMemcpyAsync(z, Z, h.npad * sizeof(double), cudaMemcpyDeviceToDevice, st));
  ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
  ILS_CU(cudaStreamSynchronize(st));
  const int64_t steps = h.hstat->inner_conv ? h.hstat->inner_steps : max_inner;
  (void)conv;
  if (prof) {
    long long hp[16 * 16];
    ILS_CU(cudaMemcpy(hp, prof, sizeof(hp), cudaMemcpyDeviceToHost));
    cudaFree(prof);
    const double nb = (double)((steps + Bsel - 1) / Bsel);
    for (int rk = 0; rk < p.C; ++rk) {
      const long long* q = hp + rk * 8;
      if (la)   // look-ahead kernel phases on compute thread 0 (LAP indices in rk_rgs_la_kernel)
        fprintf(stderr, "ILS_RK_PROF k=%lld rank=%d blocks=%.0f cycles/block: products %.0f B1 %.0f T-wait %.0f T-read %.0f loop-top %.0f axpy %.0f TMA-wait %.0f fill-wait %.0f\n",
                (long long)k, rk, nb, q[0] / nb, q[1] / nb, q[2] / nb, q[3] / nb, q[4] / nb, q[5] / nb, q[6] / nb, q[7] / nb);
      else
        fprintf(stderr, "ILS_RK_PROF k=%lld rank=%d blocks=%.0f cycles/block: wait %.0f local %.0f rscatter %.0f bar %.0f send %.0f recv %.0f sum %.0f rest %.0f\n",
                (long long)k, rk, nb, q[0] / nb, q[1] / nb, q[2] / nb, q[3] / nb, q[4] / nb, q[5] / nb, q[6] / nb, q[7] / nb);
      if (la) {   // look-ahead helper warps: reduce warp (B1 -> data, data -> T posted), comm warp (send issue)
        const long long* r2 = hp + 128 + rk * 8;
        fprintf(stderr, "ILS_RK_PROF_LA rank=%d reduce: data wait %.0f T %.0f rest %.0f | comm: send %.0f z %.0f | fill (per block): throttle %.0f work %.0f\n", rk,
                r2[0] / nb, r2[1] / nb, r2[2] / nb, r2[3] / nb, r2[4] / nb, r2[5] / nb, r2[6] / nb);
      }
    }
  }
  if (steps_out) *steps_out = steps;
  const double pd = (double)h.p, nd = (double)h.n;
  // algorithmic bytes: 16p per inner step (two columns of A1); per inner check
  // 8n^2 (A1bar z, look-ahead kernel) or 16pn (A1^T (A1 z), chunked kernels). Launches: one per
  // inner solve (look-ahead kernel) or one chunk kernel per check interval.
  hot_account(h, 1, (double)steps * 16.0 * pd + (double)(steps / ce) * (la ? 8.0 * nd * nd : 16.0 * pd * nd),
              la ? 1 : (steps + ce - 1) / ce);
  return ILS_OK;
}

}  // namespace ils
