#include <cstdint>
// ingest.cu -- K0: layout and sampling tables built once per handle (ils_create).
//
//   A1T  = column-major copy of A1 (RK/RGS read columns of A1)
//   N_j  = ||A1_(j)||_2^2 summed sequentially in i (include/ils.h "Index stream")
//   S_j  = prefix sums of W_j = max(1, floor(N_j / N_max * 2^32)) (PAPER.md:297 probabilities)
//   A1^T b1 (Alg. 2 step 3 / Alg. 5 step 2)
#include "common.cuh"
#include "ils_internal.h"

namespace ils {

// A1T[j][i] = Arm[i][j], tile 32x32 through shared memory (coalesced both sides).
__global__ void transpose_a1_kernel(const double* __restrict__ Arm, int64_t npad, int64_t p,
                                    double* __restrict__ A1T, int64_t ppad) {
  __shared__ double tile[32][33];
  const int64_t j0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t i = i0 + r, j = j0 + threadIdx.x;
    tile[r][threadIdx.x] = (i < p) ? Arm[i * npad + j] : 0.0;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t j = j0 + r, i = i0 + threadIdx.x;
    if (i < ppad) A1T[j * ppad + i] = tile[threadIdx.x][r];
  }
}

// Fused dense ingest (one pass over A): 32x32 tiles of the padded [A1; A2] region; each tile is
// read once from the caller's A (or in place from Arm after a host upload), written row-major
// into Arm with zero padding (rows >= m, columns >= n), written transposed into A1T for rows < p
// (zeros for p <= row < ppad), and checked for non-finite values (flag). b is checked by the same
// grid. Replaces a memset + 2D copy + finite scan + transpose (4 passes) by one.
__global__ void ingest_dense_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ b,
                                    int64_t m, int64_t n, int64_t p, int64_t rows_pad, int64_t npad, int64_t ppad,
                                    double* Arm, double* __restrict__ A1T, int32_t* flag) {
  __shared__ double tile[32][33];
  const int64_t j0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  bool bad = false;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t i = i0 + r, j = j0 + threadIdx.x;
    double v = 0.0;
    if (i < m && j < n) {
      v = A[i * lda + j];
      bad |= !isfinite(v);
    }
    tile[r][threadIdx.x] = (i < p) ? v : 0.0;
    if (i < rows_pad) Arm[i * npad + j] = v;
  }
  if (blockIdx.x == 0 && blockIdx.y == 0)
    for (int64_t k = threadIdx.y * 32 + threadIdx.x; k < m; k += 256) bad |= !isfinite(b[k]);
  if (bad) atomicExch(flag, 1);
  if (i0 >= ppad) return;
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t j = j0 + r, i = i0 + threadIdx.x;
    if (i < ppad) A1T[j * ppad + i] = tile[threadIdx.x][r];
  }
}

int launch_ingest_dense(Handle& h, const double* A, int64_t lda, const double* b, int32_t* flag) {
  const int64_t rows_pad = h.m + 64;
  dim3 grid((unsigned)(h.npad / 32), (unsigned)((rows_pad + 31) / 32));
  ingest_dense_kernel<<<grid, dim3(32, 8), 0, h.stream>>>(A, lda, b, h.m, h.n, h.p, rows_pad, h.npad, h.ppad,
                                                          h.Arm, h.A1T, flag);
  ILS_LAUNCHED("ingest_dense_kernel");
  return ILS_OK;
}

int launch_transpose_a1(Handle& h) {
  dim3 grid((unsigned)(h.npad / 32), (unsigned)((h.ppad + 31) / 32));
  transpose_a1_kernel<<<grid, dim3(32, 8), 0, h.stream>>>(h.Arm, h.npad, h.p, h.A1T, h.ppad);
  ILS_LAUNCHED("transpose_a1_kernel");
  return ILS_OK;
}

// N_j = (((0 + a_0j^2) + a_1j^2) + ...) with every square rounded (no FMA contraction).
// N_j = sum_i a_ij^2 in sequential row order, each product and sum rounded (no FMA): the oracle's
// definition bit for bit (R7). One CTA per 32 columns: 8 warps stream 32-row tiles of
// the column group into an 8-stage shared-memory ring with 16-byte cp.async (deep memory-level
// parallelism), warp 0 runs the 32 sequential per-column sums out of shared memory.
constexpr int CN_TR = 32;        // rows per tile
constexpr int CN_ST = 8;         // ring stages
__global__ void __launch_bounds__(256) colnorms_kernel(const double* __restrict__ Arm, int64_t npad, int64_t p,
                                                       int64_t n, double* __restrict__ N) {
  extern __shared__ __align__(16) unsigned char cn_smem[];
  double(*ring)[CN_TR][32] = reinterpret_cast<double(*)[CN_TR][32]>(cn_smem);   // [CN_ST][CN_TR][32]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  const int64_t ntiles = (p + CN_TR - 1) / CN_TR;
  auto issue = [&](int64_t t) {
    if (t < ntiles) {
      double(*dst)[32] = ring[t % CN_ST];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int c = tid + 256 * k;   // 512 16-byte chunks: row c / 16, column pair c % 16
        const int64_t i = t * CN_TR + (c >> 4);
        if (i < p) cp_async16(&dst[c >> 4][2 * (c & 15)], Arm + i * npad + j0 + 2 * (c & 15));
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int t = 0; t < CN_ST - 1; ++t) issue(t);
  double s = 0.0;
  for (int64_t t = 0; t < ntiles; ++t) {
    cp_async_wait<CN_ST - 2>();
    __syncthreads();   // tile t visible to warp 0; every thread is done with tile t - 1
    issue(t + CN_ST - 1);
    if (warp == 0) {
      const double(*tile)[32] = ring[t % CN_ST];
      const int rows = (int)((p - t * CN_TR) < CN_TR ? (p - t * CN_TR) : CN_TR);
      for (int r = 0; r < rows; ++r) {
        const double v = tile[r][lane];
        s = __dadd_rn(s, __dmul_rn(v, v));
      }
    }
  }
  cp_async_wait<0>();
  if (warp == 0 && j0 + lane < n) N[j0 + lane] = s;
}

int launch_colnorms(Handle& h) {
  const int smem = CN_ST * CN_TR * 32 * (int)sizeof(double);
  ILS_CU(cudaFuncSetAttribute(colnorms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  colnorms_kernel<<<(unsigned)((h.n + 31) / 32), 256, smem, h.stream>>>(h.Arm, h.npad, h.p, h.n, h.N);
  ILS_LAUNCHED("colnorms_kernel");
  return ILS_OK;
}

// One block: N_max, W_j, zero-column flag, inclusive uint64 scan S.
__global__ void __launch_bounds__(1024) weights_kernel(const double* __restrict__ N, int n,
                                                       uint64_t* __restrict__ S, int32_t* zero_flag) {
  __shared__ double smax[32];
  __shared__ uint64_t ssum[32];
  __shared__ uint64_t sbase[1024];
  const int tid = threadIdx.x, nt = blockDim.x;
  double mx = 0.0;
  int bad = 0;
  for (int j = tid; j < n; j += nt) {
    const double v = N[j];
    mx = fmax(mx, v);
    bad |= (v <= 0.0);
  }
  bad = __syncthreads_or(bad);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((tid & 31) == 0) smax[tid >> 5] = mx;
  __syncthreads();
  if (tid < 32) {
    double v = (tid < (nt >> 5)) ? smax[tid] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (tid == 0) smax[0] = v;
  }
  __syncthreads();
  const double nmax = smax[0];
  if (bad) {
    if (tid == 0) *zero_flag = 1;
    return;
  }
  // contiguous chunk per thread
  const int per = (n + nt - 1) / nt;
  const int j0 = tid * per, j1 = min(n, j0 + per);
  uint64_t local = 0;
  for (int j = j0; j < j1; ++j) {
    const double r = __ddiv_rn(N[j], nmax);
    uint64_t w = (uint64_t)floor(scalbn(r, 32));
    local += (w < 1 ? 1 : w);
  }
  sbase[tid] = local;
  __syncthreads();
  // exclusive scan of sbase (simple Hillis-Steele over 1024 entries, integer exact)
  for (int off = 1; off < nt; off <<= 1) {
    const uint64_t add = (tid >= off) ? sbase[tid - off] : 0;
    __syncthreads();
    sbase[tid] += add;
    __syncthreads();
  }
  uint64_t run = sbase[tid] - local;
  for (int j = j0; j < j1; ++j) {
    const double r = __ddiv_rn(N[j], nmax);
    uint64_t w = (uint64_t)floor(scalbn(r, 32));
    run += (w < 1 ? 1 : w);
    S[j] = run;
  }
  (void)ssum;
}

int launch_weights(Handle& h, int32_t* d_zero_flag) {
  weights_kernel<<<1, 1024, 0, h.stream>>>(h.N, (int)h.n, h.S, d_zero_flag);
  ILS_LAUNCHED("weights_kernel");
  return ILS_OK;
}

// y[i] = alpha * sum_j X[i*ldx + j] v[j] (+ yadd[i]); one warp per row, fixed-order reduction.
__global__ void gemv_rows_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows, int64_t cols,
                                 const double* __restrict__ v, double* __restrict__ y, double alpha,
                                 const double* __restrict__ yadd) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < rows; i += nw) {
    const double* xr = X + i * ldx;
    double s = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;   // four loads in flight per lane
    int64_t j = lane;
    for (; j + 96 < cols; j += 128) {
      s = fma(xr[j], v[j], s);
      s1 = fma(xr[j + 32], v[j + 32], s1);
      s2 = fma(xr[j + 64], v[j + 64], s2);
      s3 = fma(xr[j + 96], v[j + 96], s3);
    }
    for (; j < cols; j += 32) s = fma(xr[j], v[j], s);
    s = warp_sum((s + s1) + (s2 + s3));
    if (lane == 0) y[i] = alpha * s + (yadd ? yadd[i] : 0.0);
  }
}

// The same product with 16-byte loads, eight of them in flight per lane (64 B of the row and 64 B of
// v), for 16-byte-aligned rows (X and the row stride aligned: every caller's padded layout).
__global__ void gemv_rows2_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows, int64_t cols,
                                  const double* __restrict__ v, double* __restrict__ y, double alpha,
                                  const double* __restrict__ yadd) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t c2 = cols >> 1;   // whole double2 entries
  const double2* v2 = reinterpret_cast<const double2*>(v);
  for (int64_t i = warp; i < rows; i += nw) {
    const double2* xr = reinterpret_cast<const double2*>(X + i * ldx);
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = 0.0;
    int64_t k = lane;
    for (; k + 96 < c2; k += 128) {
      double2 xv[4], vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        xv[u] = __ldcs(xr + k + 32 * u);
        vv[u] = __ldg(v2 + k + 32 * u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[2 * u] = fma(xv[u].x, vv[u].x, a[2 * u]);
        a[2 * u + 1] = fma(xv[u].y, vv[u].y, a[2 * u + 1]);
      }
    }
    for (; k < c2; k += 32) {
      const double2 xv = __ldcs(xr + k), vv = __ldg(v2 + k);
      a[0] = fma(xv.x, vv.x, a[0]);
      a[1] = fma(xv.y, vv.y, a[1]);
    }
    if ((cols & 1) && lane == 0) a[2] = fma(X[i * ldx + cols - 1], v[cols - 1], a[2]);
    const double s = warp_sum(((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7])));
    if (lane == 0) y[i] = alpha * s + (yadd ? yadd[i] : 0.0);
  }
}

int launch_gemv_rows(const double* X, int64_t ldx, int64_t rows, int64_t cols, const double* v, double* y,
                     double alpha, const double* yadd, cudaStream_t st) {
  if (rows <= 0) return ILS_OK;
  const int bs = 256;
  int64_t blocks = (rows * 32 + bs - 1) / bs;
  if (blocks > 148 * 16) blocks = 148 * 16;
  const bool al16 = (((uintptr_t)X | (uintptr_t)v) & 15) == 0 && (ldx & 1) == 0;
  if (al16) {
    gemv_rows2_kernel<<<(unsigned)blocks, bs, 0, st>>>(X, ldx, rows, cols, v, y, alpha, yadd);
    ILS_LAUNCHED("gemv_rows2_kernel");
  } else {
    gemv_rows_kernel<<<(unsigned)blocks, bs, 0, st>>>(X, ldx, rows, cols, v, y, alpha, yadd);
    ILS_LAUNCHED("gemv_rows_kernel");
  }
  return ILS_OK;
}

// y[j] = alpha * sum_i X[i*ldx + j] v[i] (+ yadd[j]); thread per column, sequential in i.
__global__ void gemv_cols_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows, int64_t cols,
                                 const double* __restrict__ v, double* __restrict__ y, double alpha,
                                 const double* __restrict__ yadd) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  double s = 0.0;
  for (int64_t i = 0; i < rows; ++i) s = fma(X[i * ldx + j], v[i], s);
  y[j] = alpha * s + (yadd ? yadd[j] : 0.0);
}

int launch_gemv_cols(const double* X, int64_t ldx, int64_t rows, int64_t cols, const double* v, double* y,
                     double alpha, const double* yadd, cudaStream_t st) {
  if (cols <= 0) return ILS_OK;
  const int bs = 128;
  gemv_cols_kernel<<<(unsigned)((cols + bs - 1) / bs), bs, 0, st>>>(X, ldx, rows, cols, v, y, alpha, yadd);
  ILS_LAUNCHED("gemv_cols_kernel");
  return ILS_OK;
}

}  // namespace ils
