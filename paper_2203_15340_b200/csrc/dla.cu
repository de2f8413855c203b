// dla.cu -- K3: the only dense contractions of the method, on fp64 tensor cores (DMMA).
//
//   Gram  A1bar = A1^T A1             (Alg. 1 step 2 / Alg. 5 step 2)
//   Cholesky A1bar = L L^T, Z = L^{-1} (recursive, DMMA GEMMs at every level)
//   P = (A1^T A1)^{-1} = Z^T Z        (Alg. 1 step 2 explicit inverse)
//   M = A1^T A1 - A2^T A2             (normal matrix; reference solve only)
//
// GEMM convention: C[M x N] = alpha * sum_k opA(i,k) * opB(j,k) + beta * C
//   opA(i,k) = A[i*lda + k] (K-contiguous) or A[k*lda + i] (M-contiguous, a_mc)
//   opB(j,k) = B[j*ldb + k] (K-contiguous) or B[k*ldb + j] (N-contiguous, b_nc)
// All dimensions are multiples of 64 (M, N) and 32 (K): the handle pads every dense
// operand with zeros (identity on the padded diagonal), so there are no tails.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "ils_internal.h"

namespace ils {

constexpr int BM = 64, BN = 64, BK = 32, GEMM_THREADS = 128, GEMM_STAGES = 3;
constexpr int LDK = BK + 4;   // K-contiguous smem tile row stride (doubles)
constexpr int LDM = BM + 4;   // M-contiguous smem tile row stride (doubles)
constexpr int TILE_DBL = (BM * LDK > BK * LDM) ? BM * LDK : BK * LDM;   // doubles per operand tile
constexpr size_t GEMM_SMEM = (size_t)GEMM_STAGES * 2 * TILE_DBL * sizeof(double);

template <bool MC>
__device__ __forceinline__ void load_tile(double* __restrict__ s, const double* __restrict__ g, int64_t ld,
                                          int64_t row0, int64_t k0) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int u = 0; u < (BM * BK / 2) / GEMM_THREADS; ++u) {
    const int q = tid + u * GEMM_THREADS;
    if (!MC) {  // rows of 32 k-values: 16 chunks of 2 doubles
      const int r = q >> 4, c = q & 15;
      cp_async16(s + r * LDK + 2 * c, g + (row0 + r) * ld + k0 + 2 * c);
    } else {    // k-rows of 64 m-values: 32 chunks
      const int kk = q >> 5, c = q & 31;
      cp_async16(s + kk * LDM + 2 * c, g + (k0 + kk) * ld + row0 + 2 * c);
    }
  }
}

template <bool MC>
__device__ __forceinline__ double frag(const double* __restrict__ s, int r, int k) {
  return MC ? s[k * LDM + r] : s[r * LDK + k];
}

// grid: (tiles, 1, splits). lower_only: tiles enumerate bm >= bn. kmode restricts each tile's K
// range to where a triangular operand is non-zero (64-aligned blocks): 1 K >= max(row0, col0)
// (Z^T Z), 2 K < col0 + BN (B lower, C = A B^T), 3 K >= col0 (B lower, C = A B),
// 4 K < row0 + BM (A lower, C = A B).
template <bool AMC, bool BNC>
__global__ void __launch_bounds__(GEMM_THREADS) gemm_dmma_kernel(
    int64_t M, int64_t N, int64_t K, double alpha, const double* __restrict__ A, int64_t lda,
    const double* __restrict__ B, int64_t ldb, double beta, double* __restrict__ C, int64_t ldc,
    int lower_only, int kmode, int splits, double* __restrict__ ws) {
  extern __shared__ __align__(128) double smem[];
  const int64_t nt = N / BN;
  int64_t bm, bn;
  const int64_t t = blockIdx.x;
  if (lower_only) {
    bm = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while ((bm + 1) * (bm + 2) / 2 <= t) ++bm;
    while (bm * (bm + 1) / 2 > t) --bm;
    bn = t - bm * (bm + 1) / 2;
  } else {
    bm = t / nt;
    bn = t % nt;
  }
  const int64_t row0 = bm * BM, col0 = bn * BN;
  int64_t kbeg = 0, kend = K;
  if (kmode == 1) kbeg = row0 > col0 ? row0 : col0;
  else if (kmode == 2) kend = (col0 + BN < K) ? col0 + BN : K;
  else if (kmode == 3) kbeg = col0;
  else if (kmode == 4) kend = (row0 + BM < K) ? row0 + BM : K;
  const int64_t klen = kend > kbeg ? kend - kbeg : 0;
  int64_t kc = (klen + splits - 1) / splits;
  kc = (kc + BK - 1) / BK * BK;
  const int64_t z = blockIdx.z;
  const int64_t ks = kbeg + z * kc;
  const int64_t ke = (ks + kc < kend) ? ks + kc : kend;
  const int nk = ke > ks ? (int)((ke - ks) / BK) : 0;

  double* sA = smem;
  double* sB = smem + GEMM_STAGES * TILE_DBL;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int fr = lane >> 2, fk = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < GEMM_STAGES - 1; ++s) {
    if (s < nk) {
      load_tile<AMC>(sA + s * TILE_DBL, A, lda, row0, ks + (int64_t)s * BK);
      load_tile<BNC>(sB + s * TILE_DBL, B, ldb, col0, ks + (int64_t)s * BK);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<GEMM_STAGES - 2>();
    __syncthreads();
    {
      const int pf = kt + GEMM_STAGES - 1;
      if (pf < nk) {
        const int st = pf % GEMM_STAGES;
        load_tile<AMC>(sA + st * TILE_DBL, A, lda, row0, ks + (int64_t)pf * BK);
        load_tile<BNC>(sB + st * TILE_DBL, B, ldb, col0, ks + (int64_t)pf * BK);
      }
      cp_async_commit();
    }
    const double* a = sA + (kt % GEMM_STAGES) * TILE_DBL;
    const double* b = sB + (kt % GEMM_STAGES) * TILE_DBL;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = frag<AMC>(a, wm + 8 * i + fr, kk + fk);
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = frag<BNC>(b, wn + 8 * j + fr, kk + fk);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: lane holds C[8i + fr][8j + 2fk + {0,1}] of the warp tile
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = row0 + wm + 8 * i + fr;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = col0 + wn + 8 * j + 2 * fk;
      if (splits > 1 || ws != nullptr) {
        double2* dst = reinterpret_cast<double2*>(ws + ((int64_t)z * M + r) * N + c);
        *dst = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        double2* dst = reinterpret_cast<double2*>(C + r * ldc + c);
        double2 v = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
        if (beta != 0.0) {
          const double2 o = *dst;
          v.x += beta * o.x;
          v.y += beta * o.y;
        }
        *dst = v;
      }
    }
  }
}

// C = alpha * sum_z ws[z] + beta * C over the tiles in scope (fixed z order: deterministic)
__global__ void splitk_reduce_kernel(int64_t M, int64_t N, int splits, const double* __restrict__ ws,
                                     double alpha, double beta, double* __restrict__ C, int64_t ldc,
                                     int lower_only) {
  const int64_t total = M * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / N, c = e % N;
    if (lower_only && (r / BM) < (c / BN)) continue;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += ws[(int64_t)z * total + e];
    double v = alpha * s;
    if (beta != 0.0) v += beta * C[r * ldc + c];
    C[r * ldc + c] = v;
  }
}

static int ensure_ws(Handle& h, size_t bytes) {
  if (h.wsA_bytes >= bytes) return ILS_OK;
  if (h.wsA) cudaFreeAsync(h.wsA, h.stream);
  h.wsA = nullptr;
  h.wsA_bytes = 0;
  cudaError_t e = cudaMallocAsync(&h.wsA, bytes, h.stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync(ws)");
  h.wsA_bytes = bytes;
  return ILS_OK;
}

template <bool AMC, bool BNC>
static int gemm_launch(Handle& h, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                       int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                       bool lower_only, int kmode, int splits, bool force_ws) {
  static bool attr_set = false;
  if (!attr_set) {
    ILS_CU(cudaFuncSetAttribute(gemm_dmma_kernel<AMC, BNC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)GEMM_SMEM));
    attr_set = true;
  }
  const int64_t mt = M / BM, nt = N / BN;
  const int64_t tiles = lower_only ? mt * (mt + 1) / 2 : mt * nt;
  if (tiles == 0) return ILS_OK;
  double* ws = nullptr;
  if (splits > 1 || force_ws) {
    int r = ensure_ws(h, (size_t)splits * M * N * sizeof(double));
    if (r) return r;
    ws = h.wsA;
  }
  dim3 grid((unsigned)tiles, 1, (unsigned)splits);
  gemm_dmma_kernel<AMC, BNC><<<grid, GEMM_THREADS, GEMM_SMEM, h.stream>>>(
      M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, lower_only ? 1 : 0, kmode, splits, ws);
  ILS_LAUNCHED("gemm_dmma_kernel");
  if (ws) {
    const int64_t total = M * N;
    int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)h.num_sms * 8);
    splitk_reduce_kernel<<<(unsigned)blocks, 256, 0, h.stream>>>(M, N, splits, ws, alpha, beta, C, ldc,
                                                                 lower_only ? 1 : 0);
    ILS_LAUNCHED("splitk_reduce_kernel");
  }
  return ILS_OK;
}

int gemm_dmma(Handle& h, bool a_mc, bool b_nc, int64_t M, int64_t N, int64_t K, double alpha,
              const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
              int64_t ldc, bool lower_only, int splits) {
  if (a_mc && b_nc)
    return gemm_launch<true, true>(h, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, lower_only, 0,
                                   splits, false);
  if (a_mc)
    return gemm_launch<true, false>(h, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, lower_only, 0,
                                    splits, false);
  if (b_nc)
    return gemm_launch<false, true>(h, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, lower_only, 0,
                                    splits, false);
  return gemm_launch<false, false>(h, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, lower_only, 0,
                                   splits, false);
}

// Split count so that the launch covers the SMs ~2x.
static int pick_splits(Handle& h, int64_t tiles, int64_t K) {
  int s = 1;
  while (tiles * s < 2LL * h.num_sms && K / (BK * (s * 2)) >= 8 && s < 32) s *= 2;
  return s;
}

// C[j][i] = C[i][j] for i > j (copy lower -> upper); set C[j][j] = 1 for n_real <= j < n.
__global__ void mirror_kernel(double* C, int64_t ld, int64_t n, int64_t n_real) {
  __shared__ double tile[32][33];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;   // target tile (bi, bj) in upper part: bi < bj
  if (bi > bj) return;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t i = bj * 32 + r, j = bi * 32 + threadIdx.x;   // source: lower tile (bj, bi)
    tile[r][threadIdx.x] = C[i * ld + j];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int64_t i = bi * 32 + r, j = bj * 32 + threadIdx.x;
    if (j > i) C[i * ld + j] = tile[threadIdx.x][r];
    if (j == i && i >= n_real) C[i * ld + j] = 1.0;
  }
}

int mirror_lower(Handle& h, double* C, int64_t ld, int64_t n, int64_t n_real) {
  dim3 grid((unsigned)(n / 32), (unsigned)(n / 32));
  mirror_kernel<<<grid, dim3(32, 8), 0, h.stream>>>(C, ld, n, n_real);
  ILS_LAUNCHED("mirror_kernel");
  return ILS_OK;
}

// ---------------------------------------------------------------- 64x64 base: potf2 + trtri
// Cholesky of the 64x64 diagonal block at (s0, s0) of L (lower, in place) and its inverse into Z,
// fused in one right-looking sweep with both trailing matrices in registers. A 16x16 thread grid
// holds 4x4 elements each (rows ty + 16 u, columns tx + 16 v) of A (-> L) and of W, the working
// right-hand side of L Z = I. Iteration k: the owners of column k of A publish it and the diagonal
// owner publishes 1 / sqrt(a_kk); the owners of row k-1 of W publish Z[k-1][:] = W[k-1][:] / L_{k-1,k-1};
// one barrier; then every thread applies a_ij -= l_ik l_jk (l = published * rs, the arithmetic of a
// textbook potf2) and W_ic -= L[i][k-1] Z[k-1][c]. One barrier per column for both factorisations
// (the shared-memory loop version with a separate trtri pass took ~75 us per block, mostly barrier
// and issue stalls; a fully unrolled 32x32 register version was instruction-fetch bound).
__global__ void __launch_bounds__(256) potf2_trtri_kernel(double* __restrict__ L, double* __restrict__ Z,
                                                          int64_t ld, int64_t s0, int32_t* err) {
  extern __shared__ __align__(16) double potf_smem[];
  double (*a)[65] = reinterpret_cast<double (*)[65]>(potf_smem);            // [64][65] L (lower)
  double (*zi)[65] = reinterpret_cast<double (*)[65]>(potf_smem + 64 * 65);  // [64][65] Z (lower)
  __shared__ double colv[3][64];   // raw column k of the trailing A (rows >= k), buffer k % 3
  __shared__ double rsv[3];        // 1 / L_kk, buffer k % 3
  __shared__ double zrow[2][64];   // row k-1 of Z (columns <= k-1), buffer (k-1) & 1
  __shared__ int bad_s;
  const int tid = threadIdx.x;
  double* blk = L + s0 * ld + s0;
  const int ty = tid >> 4, tx = tid & 15;
  double t[4][4], w[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int i = ty + 16 * u, j = tx + 16 * v;
      t[u][v] = (j <= i) ? blk[i * ld + j] : 0.0;
      w[u][v] = (j == i) ? 1.0 : 0.0;
    }
  if (tid == 0) bad_s = 0;
  int b3 = 0, bm3 = 2;   // k % 3, (k - 1) % 3
  for (int k = 0; k <= 64; ++k) {
    const int m = k - 1;
    // ---- publish
    if (k < 64 && tx == (k & 15)) {   // column k of A (rows >= k); the diagonal owner adds 1 / L_kk
      const int kv = k >> 4;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = ty + 16 * u;
        double val = 0.0;
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (v == kv) val = t[u][v];
        if (i >= k) colv[b3][i] = val;
        if (i == k) {
          const bool ok = val > 0.0 && isfinite(val);
          rsv[b3] = ok ? rsqrt(val) : 0.0;
          if (!ok) bad_s = 1;
        }
      }
    }
    if (m >= 0 && ty == (m & 15)) {   // row m of Z = row m of W scaled by 1 / L_mm
      const int mu = m >> 4;
      const double rm = rsv[bm3];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (u != mu) continue;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c = tx + 16 * v;
          if (c <= m) {
            const double z = w[u][v] * rm;
            zrow[m & 1][c] = z;
            zi[m][c] = z;
          }
        }
      }
    }
    __syncthreads();
    // ---- update
    if (k < 64) {
      const double rs = rsv[b3];
      double lik[4], ljk[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) lik[u] = colv[b3][(ty + 16 * u) & 63] * rs;
#pragma unroll
      for (int v = 0; v < 4; ++v) ljk[v] = colv[b3][(tx + 16 * v) & 63] * rs;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = ty + 16 * u;
        if (i <= k) continue;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int j = tx + 16 * v;
          if (j > k && j <= i) t[u][v] = fma(-lik[u], ljk[v], t[u][v]);
        }
      }
      if (tx == (k & 15)) {   // the finished column k of L
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int i = ty + 16 * u;
          if (i > k) a[i][k] = lik[u];
          if (i == k) a[k][k] = colv[b3][k] * rs;
        }
      }
    }
    if (m >= 0) {   // W_ic -= L[i][m] Z[m][c] for i > m, c <= m
      const double rm = rsv[bm3];
      double zmc[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) zmc[v] = zrow[m & 1][tx + 16 * v];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = ty + 16 * u;
        if (i <= m) continue;
        const double lim = colv[bm3][i] * rm;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int c = tx + 16 * v;
          if (c <= m) w[u][v] = fma(-lim, zmc[v], w[u][v]);
        }
      }
    }
    bm3 = b3;
    b3 = (b3 == 2) ? 0 : b3 + 1;
  }
  __syncthreads();
  double* zb = Z + s0 * ld + s0;
  for (int e = tid; e < 64 * 64; e += 256) {
    const int i = e >> 6, j = e & 63;
    blk[i * ld + j] = (j <= i) ? a[i][j] : 0.0;
    zb[i * ld + j] = (j <= i) ? zi[i][j] : 0.0;
  }
  if (tid == 0 && bad_s) atomicExch(err, 1);
}

// ---------------------------------------------------------------- 64x64 base, blocked (default)
// The same leaf (L = chol(A), Z = L^{-1} of the 64x64 diagonal block at (s0, s0)) as four 16-column
// panels, so that the sequential part is a 16x16 factorisation done by one warp in registers and
// everything else is small dense products on the fp64 tensor cores (DMMA m8n8k4, 8x8 output tiles,
// K = 16) over the whole CTA. Z is built in place of W, the right-hand side of L Z = I (W = I at the
// start), by the same right-looking sweep. Per panel P:
//   (a) warp 0, lane l holding row l of A_PP and column l of W_PP = I. Every lane also carries the
//       16 diagonal entries (updated redundantly with the same fma as their owners, so bitwise equal)
//       and the current column, broadcast once through shared memory right after its owners updated
//       it; column k is then: 1 / sqrt(a_kk) by rsqrt (as potf2_trtri_kernel), L_jk = a_jk * rsqrt
//       for every j locally, the diagonal update, the own row's rank-1 update and Z_PP's row k -- the
//       step chain is rsqrt -> mul -> fma, with the broadcast of column k + 1 beside it;
//   (b) L_iP = A_iP Z_PP^T for the rows below and Z_P,<P = Z_PP W_P,<P (12 DMMA tiles);
//   (c) A_ij -= L_iP L_jP^T (lower tiles) and W_i,<=P -= L_iP Z_P,<=P for the rows below (DMMA).
// 4 barriers per panel (65 in the column-at-a-time sweep).
// Row stride of the leaf's shared-memory tiles: 68 = 4 (mod 16) doubles, so the DMMA fragment loads
// (row fr, column fk of an 8x4 slice, either orientation) hit 16 distinct 8-byte banks per half-warp.
constexpr int LEAF_LD = 68;
constexpr int LEAF_SMEM = 2 * 64 * LEAF_LD * (int)sizeof(double);

__device__ __forceinline__ void leaf_mma_k16(double& c0, double& c1, const double* abase, int astr, int acol,
                                             const double* bbase, int bstr_n, int bstr_k, int lane) {
  const int fr = lane >> 2, fk = lane & 3;
#pragma unroll
  for (int kk = 0; kk < 16; kk += 4) {
    const double av = abase[fr * astr + acol + kk + fk];
    const double bv = bbase[fr * bstr_n + (kk + fk) * bstr_k];
    dmma884(c0, c1, av, bv);
  }
}

__global__ void __launch_bounds__(256) potrf_trtri64_kernel(double* __restrict__ L, double* __restrict__ Z,
                                                            int64_t ld, int64_t s0, int32_t* err) {
  extern __shared__ __align__(16) double leaf_smem[];
  double (*a)[LEAF_LD] = reinterpret_cast<double (*)[LEAF_LD]>(leaf_smem);                  // A -> L (lower)
  double (*z)[LEAF_LD] = reinterpret_cast<double (*)[LEAF_LD]>(leaf_smem + 64 * LEAF_LD);   // W -> Z (lower)
  __shared__ __align__(16) double colbuf[2][16];
  __shared__ int bad_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int fr = lane >> 2, fk = lane & 3;
  double* blk = L + s0 * ld + s0;
  {
    double v[16];   // all 16 loads in flight before the first shared-memory store
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int e = tid + 256 * q, i = e >> 6, j = e & 63;
      v[q] = (j <= i) ? __ldcg(blk + i * ld + j) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int e = tid + 256 * q, i = e >> 6, j = e & 63;
      a[i][j] = v[q];
      z[i][j] = (i == j) ? 1.0 : 0.0;
    }
  }
  if (tid == 0) bad_s = 0;
  __syncthreads();
  for (int P = 0; P < 64; P += 16) {
    // (a) L_PP, Z_PP (warp 0): lane l < 16 holds row l of A_PP, lane 16 + l column l of W_PP = I;
    // both are updated by the same two operations per column (scale by 1 / L_kk, then x_j -= x_k L_jk)
    if (warp == 0) {
      const int l = lane & 15;
      const bool rowlane = lane < 16;
      double x[16], bk[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        x[c] = rowlane ? a[P + l][P + c] : ((c == l) ? 1.0 : 0.0);
        bk[c] = a[P + c][P];   // column 0 of A_PP
      }
      bool bad = false;
      double dk = bk[0];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        bad = bad || !(dk > 0.0 && isfinite(dk));   // off the step chain: a breakdown only flags
        const double rs = rsqrt(dk);
        x[k] *= rs;   // row lanes: L_lk (lane k: sqrt(a_kk)); column lanes: Z_kl final
#pragma unroll
        for (int j = k + 1; j < 16; ++j) x[j] = fma(-x[k], bk[j] * rs, x[j]);   // L_jk = a_jk / sqrt(a_kk)
        if (k < 15) {   // the updated column k + 1 to every lane: its diagonal by a shuffle (the step
                        // chain), the rest through shared memory
          dk = __shfl_sync(0xffffffffu, x[k + 1], k + 1);
          if (rowlane) colbuf[(k + 1) & 1][l] = x[k + 1];
          __syncwarp();
#pragma unroll
          for (int j = k + 2; j < 16; ++j) bk[j] = colbuf[(k + 1) & 1][j];
        }
      }
      if (rowlane) {
#pragma unroll
        for (int c = 0; c < 16; ++c) a[P + l][P + c] = (c <= l) ? x[c] : 0.0;
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) z[P + i][P + l] = (i >= l) ? x[i] : 0.0;
      }
      if (lane == 0 && bad) bad_s = 1;
    }
    __syncthreads();
    // (b) 12 tiles: L_iP = A_iP Z_PP^T (rows below, two column tiles each), then Z_P,<P = Z_PP W_P,<P
    const int R = 48 - P;
    double o0[2], o1[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int t = warp + 8 * q;
      o0[q] = o1[q] = 0.0;
      if (t < R / 4) {
        const int i0 = P + 16 + 8 * (t >> 1), c0 = 8 * (t & 1);
        leaf_mma_k16(o0[q], o1[q], &a[i0][0], LEAF_LD, P, &z[P + c0][P], LEAF_LD, 1, lane);
      } else if (t < 12) {
        const int u = t - R / 4, r0 = 8 * (u & 1), c0 = 8 * (u >> 1);
        leaf_mma_k16(o0[q], o1[q], &z[P + r0][0], LEAF_LD, P, &z[P][c0], 1, LEAF_LD, lane);
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int t = warp + 8 * q;
      if (t < R / 4) {
        const int i0 = P + 16 + 8 * (t >> 1), c0 = 8 * (t & 1);
        a[i0 + fr][P + c0 + 2 * fk] = o0[q];
        a[i0 + fr][P + c0 + 2 * fk + 1] = o1[q];
      } else if (t < 12) {
        const int u = t - R / 4, r0 = 8 * (u & 1), c0 = 8 * (u >> 1);
        z[P + r0 + fr][c0 + 2 * fk] = o0[q];
        z[P + r0 + fr][c0 + 2 * fk + 1] = o1[q];
      }
    }
    __syncthreads();
    if (R == 0) break;
    // (c) lower 8x8 tiles of A below the panel, then W tiles (rows below, columns <= P + 15); a warp
    // takes two tiles per pass and splits K in two, so four independent DMMA chains of two are in flight
    {
      const int nb = R >> 3, nA = nb * (nb + 1) / 2, nW = nb * ((P + 16) >> 3), nT = nA + nW;
      for (int t0 = warp; t0 < nT; t0 += 16) {
        const double* ab[2];
        const double* bb[2];
        int bn[2], bkst[2], i0[2], j0[2];
        bool isA[2], live[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int t = t0 + 8 * h;
          live[h] = t < nT;
          isA[h] = t < nA;
          if (isA[h]) {
            int ti = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);   // exact for t < 21
            ti += ((ti + 1) * (ti + 2) / 2 <= t) ? 1 : 0;
            i0[h] = P + 16 + 8 * ti;
            j0[h] = P + 16 + 8 * (t - ti * (ti + 1) / 2);
            bb[h] = &a[j0[h]][P];
            bn[h] = LEAF_LD;
            bkst[h] = 1;
          } else {
            const int w = live[h] ? t - nA : 0, nc = (P + 16) >> 3, ti = w / nc;
            i0[h] = P + 16 + 8 * ti;
            j0[h] = 8 * (w - ti * nc);
            bb[h] = &z[P][j0[h]];
            bn[h] = 1;
            bkst[h] = LEAF_LD;
          }
          ab[h] = &a[i0[h]][P];
        }
        // all 16 fragment loads first (a dead second tile reads the first one's operands), then the DMMAs
        double af[2][4], bf[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int hh = live[h] ? h : 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            af[h][q] = ab[hh][fr * LEAF_LD + 4 * q + fk];
            bf[h][q] = bb[hh][fr * bn[hh] + (4 * q + fk) * bkst[hh]];
          }
        }
        double c[2][2][2];   // [tile][K half][pair]
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int e = 0; e < 2; ++e) c[h][e][0] = c[h][e][1] = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) dmma884(c[h][q & 1][0], c[h][q & 1][1], af[h][q], bf[h][q]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (!live[h]) continue;
          const double v0 = c[h][0][0] + c[h][1][0], v1 = c[h][0][1] + c[h][1][1];
          const int i = i0[h] + fr, j = j0[h] + 2 * fk;
          if (isA[h]) {
            if (j <= i) a[i][j] -= v0;
            if (j + 1 <= i) a[i][j + 1] -= v1;
          } else {
            z[i][j] -= v0;
            z[i][j + 1] -= v1;
          }
        }
      }
    }
    __syncthreads();
  }
  double* zb = Z + s0 * ld + s0;
  for (int e = tid; e < 64 * 64; e += 256) {
    const int i = e >> 6, j = e & 63;
    blk[i * ld + j] = (j <= i) ? a[i][j] : 0.0;
    zb[i * ld + j] = (j <= i) ? z[i][j] : 0.0;
  }
  if (tid == 0 && bad_s) atomicExch(err, 1);
}

// Recursive Cholesky + inverse on blocks [s, e) (units of 64).
// need_z = true: the node's inverse Z[s:e, s:e] = L[s:e, s:e]^{-1} is formed whole (Z21 = -Z22 L21 Z11,
// two GEMMs per node). need_z = false (top-level call with full_z = false, n >= 8192): only the
// children of at most zt_th blocks get whole inverses (node_full); above them L21 = A21 L11^{-T} is a
// recursive triangular solve over the left child's tree (trsm_rec) and Z is applied to vectors through
// L21 on the same tree (zc_apply_tree), so the Z21 GEMMs of every large node (~n^3/21 flops with the
// left children whole, 18.7 of 125 ms at c3) are never run.
// smallest padded n whose inverse is kept in tree form (sparse / large handles); ILS_ZT_MIN_NPAD is a
// test hook that takes small problems through the same code
static int64_t zt_min_npad() {
  const char* e = getenv("ILS_ZT_MIN_NPAD");
  return (e && atoll(e) >= 64) ? atoll(e) : 8192;
}

static inline bool node_full(const Handle& h, bool need_z, int64_t blocks) { return need_z || blocks <= h.zt_th; }

// B <- B L[s:e, s:e]^{-T} for the m rows of L starting at row0, columns [64 s, 64 e)  (B inside L)
static int trsm_rec(Handle& h, double* L, double* Z, int64_t ld, int64_t s, int64_t e, bool full, int64_t row0,
                    int64_t m, double* tmp) {
  double* Bs = L + row0 * ld + s * 64;
  if (full) {   // X = B Z^T (tmp, then copy back: in-place operands)
    const int64_t nn = (e - s) * 64;
    const int sp = pick_splits(h, (m / 64) * (nn / 64), nn);
    int r = gemm_launch<false, false>(h, m, nn, nn, 1.0, Bs, ld, Z + s * 64 * ld + s * 64, ld, 0.0, tmp, nn, false, 2,
                                      sp, sp > 1);
    if (r) return r;
    ILS_CU(cudaMemcpy2DAsync(Bs, ld * sizeof(double), tmp, nn * sizeof(double), nn * sizeof(double), m,
                             cudaMemcpyDeviceToDevice, h.stream));
    return ILS_OK;
  }
  const int64_t hmid = s + (e - s) / 2;
  const int64_t n1 = (hmid - s) * 64, n2 = (e - hmid) * 64;
  int r = trsm_rec(h, L, Z, ld, s, hmid, node_full(h, false, hmid - s), row0, m, tmp);
  if (r) return r;
  // B2 -= X1 L21^T
  const int sp = pick_splits(h, (m / 64) * (n2 / 64), n1);
  r = gemm_launch<false, false>(h, m, n2, n1, -1.0, Bs, ld, L + hmid * 64 * ld + s * 64, ld, 1.0,
                                L + row0 * ld + hmid * 64, ld, false, 0, sp, false);
  if (r) return r;
  return trsm_rec(h, L, Z, ld, hmid, e, node_full(h, false, e - hmid), row0, m, tmp);
}

static int chol_rec(Handle& h, double* L, double* Z, int64_t ld, int64_t s, int64_t e, double* tmp,
                    bool need_z) {
  if (e - s == 1) {
    const int smem = 2 * 64 * 65 * (int)sizeof(double);
    const char* ev = getenv("ILS_LEAF_OLD");   // experiment override: 1 = the column-at-a-time leaf
    const bool old_leaf = ev && ev[0] == '1';
    if (old_leaf) {
      ILS_CU(cudaFuncSetAttribute(potf2_trtri_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      potf2_trtri_kernel<<<1, 256, smem, h.stream>>>(L, Z, ld, s * 64, &h.dstat->flag_err);
      ILS_LAUNCHED("potf2_trtri_kernel");
    } else {
      ILS_CU(cudaFuncSetAttribute(potrf_trtri64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, LEAF_SMEM));
      potrf_trtri64_kernel<<<1, 256, LEAF_SMEM, h.stream>>>(L, Z, ld, s * 64, &h.dstat->flag_err);
      ILS_LAUNCHED("potrf_trtri64_kernel");
    }
    return ILS_OK;
  }
  const int64_t hmid = s + (e - s) / 2;
  const int64_t n1 = (hmid - s) * 64, n2 = (e - hmid) * 64;
  const bool lfull = node_full(h, need_z, hmid - s), rfull = node_full(h, need_z, e - hmid);
  double* L21 = L + hmid * 64 * ld + s * 64;
  double* L22 = L + hmid * 64 * ld + hmid * 64;
  double* Z11 = Z + s * 64 * ld + s * 64;
  double* Z21 = Z + hmid * 64 * ld + s * 64;
  double* Z22 = Z + hmid * 64 * ld + hmid * 64;
  int r = chol_rec(h, L, Z, ld, s, hmid, tmp, lfull);
  if (r) return r;
  // L21 = A21 L11^{-T}: A21 Z11^T when Z11 is whole, else the recursive solve
  const int sp1 = pick_splits(h, (n2 / 64) * (n1 / 64), n1);
  r = trsm_rec(h, L, Z, ld, s, hmid, lfull, hmid * 64, n2, tmp);
  if (r) return r;
  // A22 -= L21 L21^T (lower tiles)
  const int sp2 = pick_splits(h, (n2 / 64) * (n2 / 64 + 1) / 2, n1);
  r = gemm_launch<false, false>(h, n2, n2, n1, -1.0, L21, ld, L21, ld, 1.0, L22, ld, true, 0, sp2,
                                false);
  if (r) return r;
  r = chol_rec(h, L, Z, ld, hmid, e, tmp, rfull);
  if (r) return r;
  if (!need_z) return ILS_OK;
  // Z21 = -Z22 (L21 Z11): T1 = L21 Z11 -> tmp (opB(j,k) = Z11[k][j], N-contiguous)
  r = gemm_launch<false, true>(h, n2, n1, n1, 1.0, L21, ld, Z11, ld, 0.0, tmp, n1, false, 3, sp1,
                               sp1 > 1);
  if (r) return r;
  const int sp3 = pick_splits(h, (n2 / 64) * (n1 / 64), n2);
  r = gemm_launch<false, true>(h, n2, n1, n2, -1.0, Z22, ld, tmp, n1, 0.0, Z21, ld, false, 4, sp3,
                               false);
  return r;
}

int cholesky_inverse(Handle& h, double* L, double* Z, int64_t npad, bool full_z) {
  ILS_CU(cudaMemsetAsync(Z, 0, (size_t)npad * npad * sizeof(double), h.stream));
  double* tmp = nullptr;
  ILS_CU(cudaMallocAsync(&tmp, (size_t)npad * npad * sizeof(double), h.stream));
  {
    const char* e = getenv("ILS_ZT_TH");   // experiment override: whole inverses up to this many 64-blocks
    h.zt_th = (e && atoll(e) >= 1) ? atoll(e) : 64;
  }
  int r = chol_rec(h, L, Z, npad, 0, npad / 64, tmp, full_z || node_full(h, false, npad / 64));
  cudaFreeAsync(tmp, h.stream);
  return r;
}

// x = Z^T (Z c) with Z = L^{-1} held only as the whole inverses of the tree's full nodes (node_full);
// on a split node (s, mid, e), with Z21 = -Z22 L21 Z11:
//   y = Z w:    y1 = Z11 w1 ; w2 <- w2 - L21 y1 ; y2 = Z22 w2
//   x = Z^T t:  x2 = Z22^T t2 ; t1 <- t1 - L21^T x2 ; x1 = Z11^T t1
// One GEMV launch per node and pass (both updates are element-wise in place).
static int zc_fwd(Handle& h, int64_t s, int64_t e, bool full, double* w, double* y) {
  const int64_t np = h.npad, B = 64;
  if (full) return launch_tri_rows(h.Z + s * B * np + s * B, np, (e - s) * B, w + s * B, y + s * B, h.stream);
  const int64_t m = s + (e - s) / 2;
  int rc = zc_fwd(h, s, m, node_full(h, false, m - s), w, y);
  if (rc) return rc;
  rc = launch_gemv_rows(h.L + m * B * np + s * B, np, (e - m) * B, (m - s) * B, y + s * B, w + m * B, -1.0, w + m * B,
                        h.stream);
  if (rc) return rc;
  return zc_fwd(h, m, e, node_full(h, false, e - m), w, y);
}

static int zc_bwd(Handle& h, int64_t s, int64_t e, bool full, double* t, double* x) {
  const int64_t np = h.npad, B = 64;
  if (full)
    return launch_cols(h.Z + s * B * np + s * B, np, (e - s) * B, (e - s) * B, t + s * B, 1.0, nullptr, x + s * B, 1,
                       h.stream);
  const int64_t m = s + (e - s) / 2;
  int rc = zc_bwd(h, m, e, node_full(h, false, e - m), t, x);
  if (rc) return rc;
  rc = launch_cols(h.L + m * B * np + s * B, np, (e - m) * B, (m - s) * B, x + m * B, -1.0, t + s * B, t + s * B, 0,
                   h.stream);
  if (rc) return rc;
  return zc_bwd(h, s, m, node_full(h, false, m - s), t, x);
}

int zc_apply_tree(Handle& h, const double* c, double* x) {
  const int64_t np = h.npad;
  const cudaStream_t st = h.stream;
  double* w = h.vec + 2 * np;    // working copy of c (updated in place on the split nodes)
  double* y = h.vec + 4 * np;    // Z c (updated in place on the way back)
  ILS_CU(cudaMemcpyAsync(w, c, np * sizeof(double), cudaMemcpyDeviceToDevice, st));
  const bool top = node_full(h, false, np / 64);
  int rc = zc_fwd(h, 0, np / 64, top, w, y);
  if (rc) return rc;
  rc = zc_bwd(h, 0, np / 64, top, y, x);
  if (rc) return rc;
  if (h.n < np) ILS_CU(cudaMemsetAsync(x + h.n, 0, (np - h.n) * sizeof(double), st));
  return ILS_OK;
}

int build_gram(Handle& h) {
  if (h.have_gram) return ILS_OK;
  const int64_t np = h.npad;
  if (!h.G) ILS_CU(cudaMallocAsync(&h.G, (size_t)np * np * sizeof(double), h.stream));
  if (h.sparse) {
    int r = sparse_gram(h, h.G, false);
    if (r) return r;
    h.have_gram = true;
    return ILS_OK;
  }
  const int64_t tiles = (np / 64) * (np / 64 + 1) / 2;
  const int sp = pick_splits(h, tiles, h.ppad);
  int r = gemm_launch<false, false>(h, np, np, h.ppad, 1.0, h.A1T, h.ppad, h.A1T, h.ppad, 0.0, h.G, np,
                                    true, 0, sp, false);
  if (r) return r;
  // row-sharded handle: sum the ranks' lower triangles before the mirror sets the padded diagonal
  r = allreduce_sum(h, h.G, np * np);
  if (r) return r;
  r = mirror_lower(h, h.G, np, np, h.n);
  if (r) return r;
  h.have_gram = true;
  return ILS_OK;
}

int build_inverse(Handle& h) {
  if (h.have_P) return ILS_OK;
  int r = build_gram(h);
  if (r) return r;
  const int64_t np = h.npad;
  const size_t bytes = (size_t)np * np * sizeof(double);
  if (!h.L) ILS_CU(cudaMallocAsync(&h.L, bytes, h.stream));
  if (!h.Z) ILS_CU(cudaMallocAsync(&h.Z, bytes, h.stream));
  ILS_CU(cudaMemcpyAsync(h.L, h.G, bytes, cudaMemcpyDeviceToDevice, h.stream));
  if ((h.sparse || h.large) && np >= zt_min_npad()) {
    // large n (few outer steps, setup-dominated): no n^3 GEMM for P and whole inverses only of the
    // recursion's small diagonal blocks; x = Z^T (Z c) is applied through the tree (zc_apply_tree)
    r = cholesky_inverse(h, h.L, h.Z, np, false);
    if (r) return r;
    h.use_zt = true;
    h.have_P = true;
    return ILS_OK;
  }
  if (!h.P) ILS_CU(cudaMallocAsync(&h.P, bytes, h.stream));
  r = cholesky_inverse(h, h.L, h.Z, np, true);
  if (r) return r;
  // P = Z^T Z: opA(i,k) = Z[k][i] (M-contiguous), opB(j,k) = Z[k][j] (N-contiguous); K from max(i,j)
  const int64_t tiles = (np / 64) * (np / 64 + 1) / 2;
  const int sp = pick_splits(h, tiles, np / 2);
  r = gemm_launch<true, true>(h, np, np, np, 1.0, h.Z, np, h.Z, np, 0.0, h.P, np, true, 1, sp, false);
  if (r) return r;
  r = mirror_lower(h, h.P, np, np, np);
  if (r) return r;
  h.have_P = true;
  return ILS_OK;
}

// Paper-literal precompute (Alg. 1 steps 2-4; Alg. 2 steps 2-3, :291-292):
// A2bar = A2^T A2 (DMMA SYRK over the A2 rows), A^T J b = A1^T b1 - A2^T b2.
int build_a2bar(Handle& h) {
  if (h.have_a2bar) return ILS_OK;
  const int64_t np = h.npad;
  const size_t bytes = (size_t)np * np * sizeof(double);
  if (!h.A2bar) ILS_CU(cudaMallocAsync(&h.A2bar, bytes, h.stream));
  if (!h.lit_vec) ILS_CU(cudaMallocAsync(&h.lit_vec, 2 * (size_t)np * sizeof(double), h.stream));
  if (h.sparse) {
    int r = sparse_a2bar(h, h.A2bar, h.lit_vec);
    if (r) return r;
    h.have_a2bar = true;
    return ILS_OK;
  }
  ILS_CU(cudaMemsetAsync(h.A2bar, 0, bytes, h.stream));
  if (h.q > 0) {
    const int64_t kq = roundup(h.q, 32);
    const int64_t tiles = (np / 64) * (np / 64 + 1) / 2;
    const int sp = pick_splits(h, tiles, kq);
    int r = gemm_launch<true, true>(h, np, np, kq, 1.0, h.Arm + h.p * np, np, h.Arm + h.p * np, np, 0.0, h.A2bar,
                                    np, true, false, sp, false);
    if (r) return r;
    r = mirror_lower(h, h.A2bar, np, np, np);
    if (r) return r;
  }
  int r = launch_gemv_cols(h.Arm + h.p * np, np, h.q, np, h.b + h.p, h.lit_vec, -1.0, h.a1tb1, h.stream);
  if (r) return r;
  h.have_a2bar = true;
  return ILS_OK;
}

// B = P A2bar (DMMA GEMM) and c0 = P A^T J b (Alg. 1 steps 3-4)
int build_explicit_b(Handle& h) {
  if (h.have_B) return ILS_OK;
  if ((h.sparse || h.large) && h.npad >= zt_min_npad()) {
    set_error("sp_form 2 (explicit B = P A2bar) is not supported for n >= 8192 (P is applied implicitly there)");
    return ILS_ERR_UNSUPPORTED;
  }
  int r = build_inverse(h);
  if (!r) r = build_a2bar(h);
  if (r) return r;
  const int64_t np = h.npad;
  if (!h.Bmat) ILS_CU(cudaMallocAsync(&h.Bmat, (size_t)np * np * sizeof(double), h.stream));
  const int sp = pick_splits(h, (np / 64) * (np / 64), np);
  r = gemm_launch<false, true>(h, np, np, np, 1.0, h.P, np, h.A2bar, np, 0.0, h.Bmat, np, false, 0, sp, sp > 1);
  if (r) return r;
  r = launch_gemv_rows(h.P, np, np, np, h.lit_vec, h.lit_vec + np, 1.0, nullptr, h.stream);
  if (r) return r;
  h.have_B = true;
  return ILS_OK;
}

}  // namespace ils
