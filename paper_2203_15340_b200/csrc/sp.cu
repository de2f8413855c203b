// sp.cu -- K1 (fused outer right-hand-side stream) and the persistent SP solver (Alg. 1).
//
// One cooperative launch runs the whole SP iteration (Eq. Sec23 :126):
//   phase A  K1: each CTA streams its share of rows a_i of A2 (paper form) or of all of A
//            (correction form / residual) from HBM through a TMA bulk-copy ring in shared
//            memory; the row is staged ONCE and used twice: d_i = a_i^T x - b_i (block
//            reduction) then acc += sigma_i d_i a_i (register accumulators).
//   phase B  c = base + sum_cta partial_cta   (fixed CTA order: deterministic)
//            paper form: c_k = A1^T b1 + A2^T (A2 x_k - b2) = A2bar x_k + A^T J b (Alg. 2 step 5)
//   phase C  x_{k+1} = P c_k (paper form) or x_k + P g_k (correction form, reading R14), the rows
//            of P streamed through the same TMA ring as A2 (one row stream per CTA across phases
//            and outer steps, so HBM stays busy through the grid barriers)
//   phase D  stop test ||x_{k+1} - x_ref|| <= tol ||x_ref|| evaluated redundantly by every CTA.
// rhs_only: phases A+B for one x (b_hat for SP-RK-RGS / SP-SCD, or g = A^T J (b - A x) for RR).
#include <cooperative_groups.h>

#include <vector>
#include "common.cuh"
#include "ils_internal.h"

namespace cg = cooperative_groups;

namespace ils {

constexpr int SPW = 16;                     // consumer warps
constexpr int SP_CONS = SPW * 32;           // consumer threads (own the column pairs of x, c, acc)
constexpr int SP_THREADS = SP_CONS;
constexpr int SP_RMAX = 16;                 // rows per ring stage (max)
constexpr int SP_NRED = 8;                  // partial-dot buffers (>= ring stages: reuse safety)
constexpr int SP_STAGE_TARGET = 65536;      // bytes per ring stage (target)

struct SpParams {
  const double* Arm;
  const double* b;
  int64_t npad, n;
  int64_t row_begin, row_end, p;
  const double* base;     // added in phase B (A1^T b1) or nullptr
  const double* P;
  double* xa;
  double* xb;
  const double* xref;
  double* part;           // [grid][npad]
  double* cvec;           // [npad]
  double* red;            // [grid][2]
  double* x_hist;         // [max_iter][n] or nullptr
  double tol;
  int64_t max_iter;
  int stop, sp_form, rhs_only;
  int rows_per_stage, nstages;
  DevStatus* st;
  // SP-RK-RGS inner check mode (rhs_only = 1, b = nullptr, base = nullptr, x = z): rows [0, p) of
  // A1 give az_i = <A1[i,:], z> (stored to az_out) and c = A1^T az; then g = c - b_hat,
  // stop if ||g|| <= inner_tol ||b_hat|| (inner_steps = t_now); z is only read.
  int check;
  double* az_out;
  const double* bhat;
  const double* wst;
  double* rst;
  int64_t rows_r;          // rows of the r reset (ppad)
  double inner_tol;
  int64_t t_now;
  long long* prof;         // development (ILS_SP_PROF): [grid][8] cycles per phase of thread 0, summed over outer steps
};

// Software grid barrier: one release-add per CTA on a counter that only grows inside a launch (the
// host zeroes it before every launch), and an acquire poll until the count reaches G x (barriers so
// far, `target`, counted by every CTA alike). No last-arriver logic, no returned atomic, no separate
// fences: ~2.2k instead of ~5.5k cycles per barrier at c2 (ILS_SP_TRACE timers; the first version
// read a generation word, fenced, took an atomicAdd round trip, polled, and fenced again). The TMA
// ring keeps filling while the CTA waits. Co-residency is guaranteed by the cooperative launch.
__device__ __forceinline__ void sp_grid_barrier(DevStatus* st, int tid, uint32_t& target) {
  named_bar_sync(1, SP_CONS);
  if (tid == 0) {
    target += gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(&st->gbar_count), "r"(1u) : "memory");
    uint32_t v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&st->gbar_count) : "memory");
    } while ((int32_t)(v - target) < 0);
  }
  named_bar_sync(1, SP_CONS);
}

// Sum of v[c] over c in [0, G) in one fixed order, computed by warp 0 (lane l adds c = l, l+32, ...,
// then a butterfly), result broadcast through shared memory to all consumer threads.
__device__ __forceinline__ void sp_sum2_over_ctas(const double* red, int G, int tid, double* bc, double& a,
                                                  double& b) {
  if (tid < 32) {
    // eight 16-byte loads in flight per lane, added in the order c = tid, tid + 32, ...
    double x = 0.0, y = 0.0;
    const double2* red2 = reinterpret_cast<const double2*>(red);
    for (int c0 = tid; c0 < G; c0 += 8 * 32) {
      double2 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = (c0 + 32 * i < G) ? red2[c0 + 32 * i] : make_double2(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (c0 + 32 * i < G) {
          x += v[i].x;
          y += v[i].y;
        }
    }
    x = warp_sum(x);
    y = warp_sum(y);
    if (tid == 0) {
      bc[0] = x;
      bc[1] = y;
    }
  }
  named_bar_sync(1, SP_CONS);
  a = bc[0];
  b = bc[1];
  named_bar_sync(1, SP_CONS);
}

// Row stream per CTA: the CTA walks its stages (A2 rows of every outer step, then its rows of P)
// through a ring of TMA bulk copies; the 16th warp to release a slot refills it at once. The warps
// never meet at a CTA barrier inside a phase: a stage's per-warp partial dots are posted to a
// split-phase mbarrier (rfull) and the stage is finished -- 16-way sum, axpy from the same smem
// copy, slot release -- only after the NEXT stage's dots are issued, so the cross-warp reduction
// latency hides behind independent work.
template <int NPAIR>
__global__ void __launch_bounds__(SP_THREADS, 1) sp_persistent_kernel(SpParams prm) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, bid = blockIdx.x;
  const int64_t npad = prm.npad, np2 = npad / 2;
  const int R = prm.rows_per_stage, NS = prm.nstages;
  const int64_t stage_dbl = (int64_t)R * npad;
  double* ring = reinterpret_cast<double*>(smem_raw);
  double* reds = ring + NS * stage_dbl;                       // [SP_NRED][SPW][R]
  uint64_t* fullb = reinterpret_cast<uint64_t*>(reds + SP_NRED * SPW * R);
  uint64_t* rfull = fullb + NS;
  __shared__ double chs[SPW * 32];
  __shared__ double wred[SPW][2];
  __shared__ double bc[2];
  __shared__ uint32_t relcnt[SP_NRED];

  if (prm.check && *(volatile int32_t*)&prm.st->inner_conv) return;   // inner solve already stopped
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&fullb[s], 1);
      relcnt[s] = 0;
    }
    for (int s = 0; s < SP_NRED; ++s) mbar_init(&rfull[s], SPW);
    fence_mbar_init();
  }
  __syncthreads();

  // balanced contiguous shares (floor split: shares differ by at most one row, no idle CTA at the tail)
  const int64_t rows = prm.row_end - prm.row_begin;
  const int64_t r0 = prm.row_begin + (int64_t)bid * rows / G;
  const int64_t r1 = prm.row_begin + (int64_t)(bid + 1) * rows / G;
  const int64_t nstA = (r1 > r0) ? (r1 - r0 + R - 1) / R : 0;
  const bool has_c = !prm.rhs_only;
  const int64_t q0 = has_c ? (int64_t)bid * prm.n / G : 0;
  const int64_t q1 = has_c ? (int64_t)(bid + 1) * prm.n / G : 0;
  const int64_t nstP = (has_c && q1 > q0) ? (q1 - q0 + R - 1) / R : 0;
  const int64_t spi = nstA + nstP;
  const int64_t iters = prm.rhs_only ? 1 : prm.max_iter;

  const int64_t total = iters * spi;
  // stage gi of this CTA's row stream -> its ring slot (one TMA bulk copy, completion on fullb)
  auto issue = [&](int64_t gi, int slot) {   // slot = gi mod NS
    if (gi >= total) return;
    const int64_t s = gi % spi;
    const double* src;
    int64_t nr;
    if (s < nstA) {
      const int64_t rs = r0 + s * R;
      nr = (rs + R <= r1) ? R : (r1 - rs);
      src = prm.Arm + rs * npad;
    } else {
      const int64_t rs = q0 + (s - nstA) * R;
      nr = (rs + R <= q1) ? R : (q1 - rs);
      src = prm.P + rs * npad;
    }
    const uint32_t bytes = (uint32_t)(nr * npad * sizeof(double));
    mbar_arrive_expect_tx(&fullb[slot], bytes);
    bulk_g2s(ring + slot * stage_dbl, src, bytes, &fullb[slot]);
  };
  // every warp releases a stage after its last read of the slot; the 16th release refills the slot
  // with stage gg + NS (no producer warp, no CTA barrier)
  auto release = [&](int64_t gg, int slot) {
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      const uint32_t old = atomicAdd(&relcnt[slot], 1u);
      if (old % SPW == SPW - 1) {
        __threadfence_block();
        fence_proxy_async();
        issue(gg + NS, slot);
      }
    }
  };
  if (tid == 0) {
    fence_proxy_async();
    for (int gi = 0; gi < NS; ++gi) issue(gi, gi);
  }

  // ---------------- consumer warps (512 threads)
  int64_t g = 0;   // next stage to consume
  int cslot = 0;        // its ring slot (g mod NS) and phase parity (g / NS mod 2), kept incrementally
  uint32_t cpar = 0;
  auto advance = [&]() {
    ++g;
    if (++cslot == NS) {
      cslot = 0;
      cpar ^= 1u;
    }
  };
  double* xcur = prm.xa;
  double* xnext = prm.xb;
  uint32_t gtarget = 0;   // arrivals expected at the next grid barrier (gbar_count is zero at launch)
  // phase timers (ILS_SP_PROF): 0 phase A, 1 barrier, 2 phase B, 3 barrier, 4 phase C, 5 barrier, 6 phase D
  // (compiled only with -DILS_SP_TRACE: the timers cost registers at 512 threads x 128)
#ifdef ILS_SP_TRACE
  const bool sprof = prm.prof && tid == 0;
  long long spc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long spt = sprof ? clock64() : 0;
#define SPL(i)                       \
  if (sprof) {                       \
    const long long c_ = clock64();  \
    spc[i] += c_ - spt;              \
    spt = c_;                        \
  }
#else
#define SPL(i)
#endif
  for (int64_t k = 0; k < iters; ++k) {
    // ---------------- phase A: fused row stream over this CTA's A2 rows
    double2 vr[NPAIR], acc[NPAIR];
#pragma unroll
    for (int u = 0; u < NPAIR; ++u) {
      const int64_t c = tid + (int64_t)u * SP_CONS;
      vr[u] = (c < np2) ? reinterpret_cast<const double2*>(xcur)[c] : make_double2(0.0, 0.0);
      acc[u] = make_double2(0.0, 0.0);
    }
    double bprev = 0.0;
    auto dots = [&](int64_t gg, int slot, uint32_t par, int nr) {   // partial dots of stage gg -> reds, post rfull
      mbar_wait(&fullb[slot], par);
      const double* st = ring + slot * stage_dbl;
      double* red = reds + (gg & (SP_NRED - 1)) * SPW * R;
      int rr = 0;
      for (; rr + 1 < nr; rr += 2) {
        const double2* row0 = reinterpret_cast<const double2*>(st + rr * npad);
        const double2* row1 = reinterpret_cast<const double2*>(st + (rr + 1) * npad);
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int u = 0; u < NPAIR; ++u) {
          const int64_t c = tid + (int64_t)u * SP_CONS;
          if (c < np2) {
            const double2 v0 = row0[c], v1 = row1[c];
            d0 = fma(v0.x, vr[u].x, d0);
            d1 = fma(v1.x, vr[u].x, d1);
            d0 = fma(v0.y, vr[u].y, d0);
            d1 = fma(v1.y, vr[u].y, d1);
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          d0 += __shfl_xor_sync(0xffffffffu, d0, o);
          d1 += __shfl_xor_sync(0xffffffffu, d1, o);
        }
        if (lane == 0) {
          red[warp * R + rr] = d0;
          red[warp * R + rr + 1] = d1;
        }
      }
      if (rr < nr) {
        const double2* row0 = reinterpret_cast<const double2*>(st + rr * npad);
        double d0 = 0.0;
#pragma unroll
        for (int u = 0; u < NPAIR; ++u) {
          const int64_t c = tid + (int64_t)u * SP_CONS;
          if (c < np2) {
            const double2 v0 = row0[c];
            d0 = fma(v0.x, vr[u].x, d0);
            d0 = fma(v0.y, vr[u].y, d0);
          }
        }
        d0 = warp_sum(d0);
        if (lane == 0) red[warp * R + rr] = d0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&rfull[gg & (SP_NRED - 1)]);
    };
    // 16-way sum of row rr of stage gg (same fixed order in every warp): lane l adds warp l & 15
    auto rowsum = [&](const double* red, int rr) {
      double t = red[(lane & 15) * R + rr];
      t += __shfl_xor_sync(0xffffffffu, t, 8);
      t += __shfl_xor_sync(0xffffffffu, t, 4);
      t += __shfl_xor_sync(0xffffffffu, t, 2);
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      return t;
    };
    auto finish = [&](int64_t gg, int slot, int64_t rs, int nr, double bv) {   // sum, axpy, release slot
      mbar_wait(&rfull[gg & (SP_NRED - 1)], (uint32_t)((gg / SP_NRED) & 1));
      const double* st = ring + slot * stage_dbl;
      const double* red = reds + (gg & (SP_NRED - 1)) * SPW * R;
      for (int rr = 0; rr < nr; ++rr) {
        double d = rowsum(red, rr);
        const int64_t i = rs + rr;
        if (prm.az_out && tid == 0) prm.az_out[i] = d;
        d -= __shfl_sync(0xffffffffu, bv, rr);
        if (i < prm.p) d = -d;          // sigma_i = -1 on A1 rows (correction form only)
        const double2* row = reinterpret_cast<const double2*>(st + rr * npad);
#pragma unroll
        for (int u = 0; u < NPAIR; ++u) {
          const int64_t c = tid + (int64_t)u * SP_CONS;
          if (c < np2) {
            const double2 v = row[c];
            acc[u].x = fma(d, v.x, acc[u].x);
            acc[u].y = fma(d, v.y, acc[u].y);
          }
        }
      }
      release(gg, slot);
    };
    int pslot = 0;
    for (int64_t s = 0; s < nstA; ++s) {
      const int64_t rs = r0 + s * R;
      const int nr = (int)((rs + R <= r1) ? R : (r1 - rs));
      // b_i of this stage's rows (lane rr holds row rr), consumed in finish()
      const double bcur = (prm.b && lane < nr) ? __ldg(prm.b + rs + lane) : 0.0;
      dots(g, cslot, cpar, nr);
      if (s > 0) finish(g - 1, pslot, rs - R, R, bprev);
      bprev = bcur;
      pslot = cslot;
      advance();
    }
    if (nstA > 0) {
      const int64_t rs = r0 + (nstA - 1) * R;
      finish(g - 1, pslot, rs, (int)((rs + R <= r1) ? R : (r1 - rs)), bprev);
    }
    {
      double2* pp = reinterpret_cast<double2*>(prm.part + (int64_t)bid * npad);
#pragma unroll
      for (int u = 0; u < NPAIR; ++u) {
        const int64_t c = tid + (int64_t)u * SP_CONS;
        if (c < np2) pp[c] = acc[u];
      }
    }
    SPL(0)
    sp_grid_barrier(prm.st, tid, gtarget);
    SPL(1)
    // ---------------- phase B: c = base + sum_cta part (fixed order). Every CTA owns a contiguous
    // slice [jb0, jb1) of c; warp w adds partial rows w, w+16, ... (ten loads in flight per thread)
    // for 32 consecutive j, then warp 0 adds the 16 chunk sums.
    const int64_t jb0 = (int64_t)bid * npad / G, jb1 = (int64_t)(bid + 1) * npad / G;
    for (int64_t j0 = jb0; j0 < jb1; j0 += 32) {
      const int64_t j = j0 + lane;
      double sacc = 0.0;
      const double bj = (warp == 0 && j < jb1 && prm.base) ? prm.base[j] : 0.0;   // in flight with the partials
      if (j < jb1) {
        for (int c0 = warp; c0 < G; c0 += 10 * SPW) {
          double v[10];
#pragma unroll
          for (int i = 0; i < 10; ++i) {
            const int c = c0 + i * SPW;
            v[i] = (c < G) ? prm.part[(int64_t)c * npad + j] : 0.0;
          }
#pragma unroll
          for (int i = 0; i < 10; ++i) sacc += v[i];
        }
      }
      chs[warp * 32 + lane] = sacc;
      named_bar_sync(1, SP_CONS);
      if (warp == 0 && j < jb1) {
        double t = bj;
        for (int w = 0; w < SPW; ++w) t += chs[w * 32 + lane];
        prm.cvec[j] = t;
      }
      named_bar_sync(1, SP_CONS);
    }
    if (prm.check) {
      // ||g||^2 and ||b_hat||^2 partials over this CTA's j range (fixed order everywhere)
      double g2 = 0.0, b2 = 0.0;
      const int64_t jb = (jb1 < prm.n) ? jb1 : prm.n;
      for (int64_t j = jb0 + tid; j < jb; j += SP_CONS) {
        const double s = prm.cvec[j];   // this CTA's slice, written above
        const double gg = s - prm.bhat[j];
        g2 = fma(gg, gg, g2);
        b2 = fma(prm.bhat[j], prm.bhat[j], b2);
      }
      g2 = warp_sum(g2);
      b2 = warp_sum(b2);
      if (lane == 0) {
        wred[warp][0] = g2;
        wred[warp][1] = b2;
      }
      named_bar_sync(1, SP_CONS);
      if (tid == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < SPW; ++w) {
          a += wred[w][0];
          b += wred[w][1];
        }
        prm.red[2 * bid] = a;
        prm.red[2 * bid + 1] = b;
      }
      sp_grid_barrier(prm.st, tid, gtarget);
      double Gs, Bs;
      sp_sum2_over_ctas(prm.red, G, tid, bc, Gs, Bs);
      const bool conv = sqrt(Gs) <= prm.inner_tol * sqrt(Bs);
      if (conv && bid == 0 && tid == 0) {
        prm.st->inner_steps = prm.t_now;
        prm.st->inner_conv = 1;
      }
      break;
    }
    if (prm.rhs_only) break;
    SPL(2)
    sp_grid_barrier(prm.st, tid, gtarget);
    SPL(3)
    // ---------------- phase C: x_{k+1} = P c (+ x_k) over this CTA's rows [q0, q1) of P, streamed
    // through the same ring (already in flight); c in registers in the x layout of phase A. The
    // stage's x entries are finished by warp (stage mod 16) once all 16 warps posted their dots.
#pragma unroll
    for (int u = 0; u < NPAIR; ++u) {
      const int64_t c = tid + (int64_t)u * SP_CONS;
      vr[u] = (c < np2) ? reinterpret_cast<const double2*>(prm.cvec)[c] : make_double2(0.0, 0.0);
    }
    double e2 = 0.0, r2 = 0.0;
    for (int64_t s = 0; s < nstP; ++s) {
      const int64_t rs = q0 + s * R;
      const int nr = (int)((rs + R <= q1) ? R : (q1 - rs));
      dots(g, cslot, cpar, nr);
      if (warp == (int)(g & (SPW - 1))) {
        mbar_wait(&rfull[g & (SP_NRED - 1)], (uint32_t)((g / SP_NRED) & 1));
        const double* red = reds + (g & (SP_NRED - 1)) * SPW * R;
        for (int rr = 0; rr < nr; ++rr) {
          const double sum = rowsum(red, rr);
          if (lane == 0) {
            const int64_t i = rs + rr;
            const double xn = prm.sp_form ? xcur[i] + sum : sum;
            xnext[i] = xn;
            if (prm.x_hist) prm.x_hist[k * prm.n + i] = xn;
            if (prm.xref) {
              const double e = xn - prm.xref[i];
              e2 = fma(e, e, e2);
              r2 = fma(prm.xref[i], prm.xref[i], r2);
            }
          }
        }
      }
      release(g, cslot);
      advance();
    }
    if (lane == 0) {
      wred[warp][0] = e2;
      wred[warp][1] = r2;
    }
    named_bar_sync(1, SP_CONS);
    if (tid == 0) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < SPW; ++w) {
        a += wred[w][0];
        b += wred[w][1];
      }
      prm.red[2 * bid] = a;
      prm.red[2 * bid + 1] = b;
    }
    SPL(4)
    sp_grid_barrier(prm.st, tid, gtarget);
    SPL(5)
    // ---------------- phase D: stop decision (identical in every CTA)
    double E, Rr;
    sp_sum2_over_ctas(prm.red, G, tid, bc, E, Rr);
    const double metric = (prm.xref && Rr > 0.0) ? sqrt(E) / sqrt(Rr) : __longlong_as_double(0x7ff8000000000000LL);
    const bool done = (prm.stop == ILS_STOP_XREF) && prm.xref && (metric <= prm.tol);
    if (bid == 0 && tid == 0) {
      prm.st->iters = k + 1;
      prm.st->metric = metric;
      prm.st->flag_stop = done ? 1 : 0;
    }
    double* t = xcur;
    xcur = xnext;
    xnext = t;
    SPL(6)
    if (done) break;
  }
#undef SPL
#ifdef ILS_SP_TRACE
  if (sprof)
    for (int i = 0; i < 8; ++i) prm.prof[(int64_t)bid * 8 + i] = spc[i];
#endif
  // drain: copies already issued into this CTA's ring (stages g .. g+NS-1) land before it exits
  if (tid == 0)
    for (int64_t d = g; d < g + NS && d < total; ++d) {
      mbar_wait(&fullb[cslot], cpar);
      if (++cslot == NS) {
        cslot = 0;
        cpar ^= 1u;
      }
    }
}

// ||x - xref|| / ||xref|| (single block, fixed order) -> st->metric
__global__ void stop_metric_kernel(const double* __restrict__ x, const double* __restrict__ xref, int64_t n,
                                   double* out) {
  __shared__ double s1[32], s2[32];
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double e = x[i] - xref[i];
    a = fma(e, e, a);
    b = fma(xref[i], xref[i], b);
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if ((threadIdx.x & 31) == 0) {
    s1[threadIdx.x >> 5] = a;
    s2[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double A = 0.0, B = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      A += s1[w];
      B += s2[w];
    }
    *out = sqrt(A) / sqrt(B);
  }
}

int stop_metric(Handle& h, const double* x, const double* xref, double* out_dev) {
  stop_metric_kernel<<<1, 1024, 0, h.stream>>>(x, xref, h.n, out_dev);
  ILS_LAUNCHED("stop_metric_kernel");
  return ILS_OK;
}

// TMA ring geometry of the row stream: R whole rows per stage (~SP_STAGE_TARGET bytes), NS stages in
// ~200 KB of shared memory. ILS_SP_STAGE / ILS_SP_NS: experiment overrides (stage bytes, stage cap).
static void sp_ring_geometry(int64_t npad, int& R, int& NS) {
  const int64_t rowbytes = npad * (int64_t)sizeof(double);
  int64_t target = SP_STAGE_TARGET;
  int nscap = 6;
  if (const char* e = getenv("ILS_SP_STAGE")) target = atoll(e) > 0 ? atoll(e) : target;
  if (const char* e = getenv("ILS_SP_NS")) nscap = atoi(e) >= 2 ? atoi(e) : nscap;
  R = (int)(target / rowbytes);
  if (R < 1) R = 1;
  if (R > SP_RMAX) R = SP_RMAX;
  const int64_t stage_bytes = R * rowbytes;
  NS = (int)((200 * 1024) / stage_bytes);
  if (NS > nscap) NS = nscap;
  if (NS > SP_NRED) NS = SP_NRED;
  if (NS < 2) NS = 2;
}

// dynamic shared memory of the row-stream kernel: ring + partial-dot buffers + mbarriers
static size_t sp_smem_bytes(int64_t stage_bytes, int R, int NS) {
  return (size_t)NS * stage_bytes + (size_t)SP_NRED * SPW * R * sizeof(double) +
         (size_t)(NS + SP_NRED) * sizeof(uint64_t);
}

template <int NPAIR>
static int launch_sp(Handle& h, SpParams& prm, size_t smem) {
  ILS_CU(cudaFuncSetAttribute(sp_persistent_kernel<NPAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem));
  if (getenv("ILS_DEBUG_OCC")) {
    int nb = -1;
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, sp_persistent_kernel<NPAIR>);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sp_persistent_kernel<NPAIR>, SP_THREADS, smem);
    fprintf(stderr, "ILS_DEBUG_OCC NPAIR=%d smem=%zu occ=%d (%s) regs=%d maxthr=%d static=%zu maxdyn=%d\n", NPAIR, smem, nb,
            cudaGetErrorString(e), fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes);
  }
  void* args[] = {&prm};
  ILS_CU(cudaLaunchCooperativeKernel((void*)sp_persistent_kernel<NPAIR>, dim3(h.num_sms),
                                     dim3(SP_THREADS), args, smem, h.stream));
  ILS_LAUNCHED("sp_persistent_kernel");
  return ILS_OK;
}

int sp_run(Handle& h, const double* x0_dev, double* x_dev, double tol, int64_t max_iter, int stop,
           const double* xref_dev, int sp_form, double* x_hist_dev, bool rhs_only, double* rhs_out,
           int64_t* iters_out, double* metric_out, int* conv_out) {
  const int64_t npad = h.npad;
  if (h.large) {   // large n: two-pass right-hand side (large.cu); the caller loops for SP
    if (rhs_only) {
      const int full = (sp_form == 1);
      return dense_rhs_twopass(h, x0_dev, rhs_out ? rhs_out : h.vec + 2 * npad, full);
    }
    set_error("internal: the persistent SP kernel needs n <= 8192");
    return ILS_ERR_UNSUPPORTED;
  }
  if (!rhs_only) {
    int r = build_inverse(h);
    if (r) return r;
  }
  double* xa = h.vec;
  double* xb = h.vec + npad;
  double* cvec = h.vec + 2 * npad;
  ILS_CU(cudaMemsetAsync(xa, 0, 2 * npad * sizeof(double), h.stream));
  if (x0_dev) ILS_CU(cudaMemcpyAsync(xa, x0_dev, h.n * sizeof(double), cudaMemcpyDeviceToDevice, h.stream));

  SpParams prm{};
  prm.Arm = h.Arm;
  prm.b = h.b;
  prm.npad = npad;
  prm.n = h.n;
  const bool full = (sp_form == 1);
  prm.row_begin = full ? 0 : h.p;
  prm.row_end = h.m;
  prm.p = full ? h.p : 0;          // sigma = -1 only on A1 rows of the full stream
  prm.base = full ? nullptr : h.a1tb1;
  prm.P = h.P;
  prm.xa = xa;
  prm.xb = xb;
  prm.xref = xref_dev;
  prm.part = h.part;
  prm.cvec = cvec;
  prm.red = h.red;
  prm.x_hist = x_hist_dev;
  prm.tol = tol;
  prm.max_iter = max_iter;
  prm.stop = stop;
  prm.sp_form = sp_form;
  prm.rhs_only = rhs_only ? 1 : 0;
  int R, NS;
  sp_ring_geometry(npad, R, NS);
  const int64_t stage_bytes = R * npad * (int64_t)sizeof(double);
  prm.rows_per_stage = R;
  prm.nstages = NS;
  prm.st = h.dstat;
  size_t smem = sp_smem_bytes(stage_bytes, R, NS);
  if ((size_t)npad * sizeof(double) > (size_t)NS * stage_bytes) return ILS_ERR_UNSUPPORTED;
  ILS_CU(cudaMemsetAsync(h.dstat, 0, sizeof(DevStatus), h.stream));
  const int64_t np2 = npad / 2;
  int r;
  {
    const char* e = getenv("ILS_SP_PROF");
    if (e && e[0] == '1' && !rhs_only) {
      ILS_CU(cudaMallocAsync(&prm.prof, (size_t)h.num_sms * 8 * sizeof(long long), h.stream));
      ILS_CU(cudaMemsetAsync(prm.prof, 0, (size_t)h.num_sms * 8 * sizeof(long long), h.stream));
    }
  }
  ILS_CU(cudaEventRecord(h.evk0, h.stream));
  if (np2 <= SP_CONS) r = launch_sp<1>(h, prm, smem);
  else if (np2 <= 2 * SP_CONS) r = launch_sp<2>(h, prm, smem);
  else if (np2 <= 4 * SP_CONS) r = launch_sp<4>(h, prm, smem);
  else r = launch_sp<8>(h, prm, smem);
  if (r) return r;
  ILS_CU(cudaEventRecord(h.evk1, h.stream));
  const double rows = (double)(prm.row_end - prm.row_begin), nd = (double)h.n;
  if (rhs_only) {
    hot_account(h, 0, 8.0 * rows * (nd + 1.0));
    if (rhs_out) ILS_CU(cudaMemcpyAsync(rhs_out, cvec, npad * sizeof(double), cudaMemcpyDeviceToDevice, h.stream));
    return ILS_OK;
  }
  ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, h.stream));
  ILS_CU(cudaStreamSynchronize(h.stream));
  const int64_t it = h.hstat->iters;
  if (prm.prof) {   // mean and max over CTAs of thread 0's cycles per phase and outer step
    std::vector<long long> hp((size_t)h.num_sms * 8);
    ILS_CU(cudaMemcpy(hp.data(), prm.prof, hp.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(prm.prof);
    static const char* nm[7] = {"A", "bar1", "B", "bar2", "C", "bar3", "D"};
    fprintf(stderr, "ILS_SP_PROF outer=%lld cycles per outer step, mean / max over %d CTAs:", (long long)it, h.num_sms);
    for (int i = 0; i < 7; ++i) {
      double sum = 0.0, mx = 0.0;
      for (int c = 0; c < h.num_sms; ++c) {
        const double v = (double)hp[(size_t)c * 8 + i] / (double)(it > 0 ? it : 1);
        sum += v;
        mx = v > mx ? v : mx;
      }
      fprintf(stderr, " %s %.0f / %.0f", nm[i], sum / h.num_sms, mx);
    }
    fprintf(stderr, "\n");
  }
  hot_account(h, 0, (double)it * (8.0 * rows * (nd + 1.0) + 8.0 * nd * nd));
  const double* xfin = (it % 2 == 1) ? xb : xa;
  if (x_dev) ILS_CU(cudaMemcpyAsync(x_dev, xfin, h.n * sizeof(double), cudaMemcpyDeviceToDevice, h.stream));
  if (iters_out) *iters_out = it;
  if (metric_out) *metric_out = h.hstat->metric;
  if (conv_out) *conv_out = h.hstat->flag_stop;
  return ILS_OK;
}

// SP-RK-RGS inner stop check (include/ils.h "Inner stopping rule"), full grid: az = A1 z,
// g = A1^T az - b_hat, stop if ||g|| <= inner_tol ||b_hat|| (sets st->inner_conv, inner_steps = t_now),
// else r = w - az. No-op if st->inner_conv is already set.
// Small problems (p x n <= 2^20): the same check in ONE CTA (no grid barrier, no 148-CTA launch):
// az = A1 z (thread per row, A1 rows of the row-major copy), g = A1^T az (warp per column),
// ||g|| vs inner_tol ||b_hat||, r = w - az. Fixed-order reductions.
__global__ void __launch_bounds__(1024) rk_check_small_kernel(const double* __restrict__ Arm, int64_t npad, int64_t p,
                                                              int64_t n, int64_t ppad, const double* __restrict__ z,
                                                              const double* __restrict__ bhat,
                                                              const double* __restrict__ w, double* __restrict__ r,
                                                              double* __restrict__ az, double inner_tol, int64_t t_now,
                                                              DevStatus* st) {
  __shared__ double red[32][2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (*(volatile int32_t*)&st->inner_conv) return;
  for (int64_t i = tid; i < p; i += 1024) {
    const double* row = Arm + i * npad;
    double d0 = 0.0, d1 = 0.0;
    int64_t j = 0;
    for (; j + 1 < n; j += 2) {
      d0 = fma(row[j], z[j], d0);
      d1 = fma(row[j + 1], z[j + 1], d1);
    }
    if (j < n) d0 = fma(row[j], z[j], d0);
    az[i] = d0 + d1;
  }
  __syncthreads();
  double g2 = 0.0, b2 = 0.0;
  for (int64_t j = warp; j < n; j += 32) {
    double s = 0.0;
    for (int64_t i = lane; i < p; i += 32) s = fma(Arm[i * npad + j], az[i], s);
    s = warp_sum(s);
    const double g = s - bhat[j];
    g2 = fma(g, g, g2);
    b2 = fma(bhat[j], bhat[j], b2);
  }
  if (lane == 0) {
    red[warp][0] = g2;
    red[warp][1] = b2;
  }
  __syncthreads();
  double G2 = 0.0, B2 = 0.0;
  for (int q = 0; q < 32; ++q) {
    G2 += red[q][0];
    B2 += red[q][1];
  }
  if (sqrt(G2) <= inner_tol * sqrt(B2)) {
    if (tid == 0) {
      st->inner_steps = t_now;
      st->inner_conv = 1;
    }
  } else {
    for (int64_t i = tid; i < ppad; i += 1024) r[i] = w[i] - (i < p ? az[i] : 0.0);
  }
}

int rk_check(Handle& h, const double* z, const double* bhat, const double* w, double* r, double* az,
             double inner_tol, int64_t t_now) {
  if (h.large) return rk_check_twopass(h, z, bhat, w, r, az, inner_tol, t_now);
  if (h.ppad * h.npad <= (int64_t)1 << 20) {
    rk_check_small_kernel<<<1, 1024, 0, h.stream>>>(h.Arm, h.npad, h.p, h.n, h.ppad, z, bhat, w, r, az, inner_tol,
                                                     t_now, h.dstat);
    ILS_LAUNCHED("rk_check_small_kernel");
    return ILS_OK;
  }
  SpParams prm{};
  prm.Arm = h.Arm;
  prm.b = nullptr;
  prm.npad = h.npad;
  prm.n = h.n;
  prm.row_begin = 0;
  prm.row_end = h.p;
  prm.p = 0;
  prm.base = nullptr;
  prm.P = nullptr;
  prm.xa = const_cast<double*>(z);
  prm.xb = nullptr;
  prm.xref = nullptr;
  prm.part = h.part;
  prm.cvec = h.vec + 2 * h.npad;
  prm.red = h.red;
  prm.x_hist = nullptr;
  prm.max_iter = 1;
  prm.stop = ILS_STOP_NONE;
  prm.rhs_only = 1;
  prm.st = h.dstat;
  prm.check = 1;
  prm.az_out = az;
  prm.bhat = bhat;
  prm.wst = w;
  prm.rst = r;
  prm.rows_r = h.ppad;
  prm.inner_tol = inner_tol;
  prm.t_now = t_now;
  int R, NS;
  sp_ring_geometry(h.npad, R, NS);
  const int64_t stage_bytes = R * h.npad * (int64_t)sizeof(double);
  prm.rows_per_stage = R;
  prm.nstages = NS;
  const size_t smem = sp_smem_bytes(stage_bytes, R, NS);
  const int64_t np2 = h.npad / 2;
  // the grid barrier counts arrivals from zero in every launch (the rest of DevStatus carries the
  // inner solve's state across the chunk launches and is kept)
  ILS_CU(cudaMemsetAsync(&h.dstat->gbar_count, 0, 2 * sizeof(uint32_t), h.stream));
  if (np2 <= SP_CONS) return launch_sp<1>(h, prm, smem);
  if (np2 <= 2 * SP_CONS) return launch_sp<2>(h, prm, smem);
  if (np2 <= 4 * SP_CONS) return launch_sp<4>(h, prm, smem);
  return launch_sp<8>(h, prm, smem);
}

// g = A^T J (b - A x) over all m rows (sigma = -1 on A1 rows): correction-form residual.
int full_residual(Handle& h, const double* x_dev, double* g_out) {
  return sp_run(h, x_dev, nullptr, 0.0, 1, ILS_STOP_NONE, nullptr, 1, nullptr, true, g_out, nullptr,
                nullptr, nullptr);
}

}  // namespace ils
