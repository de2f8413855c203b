// large.cu -- dense inputs with n > 8192 (the paper's own Tables 2-5 sizes): rows of A
// no longer fit a shared-memory ring next to register accumulators, so the outer right-hand side
// runs as two passes (y = A2 x - b2 row pass, c = A1^T b1 + A2^T y column pass), x = P c uses the
// generic P GEMV, and the SP-RK-RGS inner check is a row pass + column pass + a one-CTA decision.
#include "common.cuh"
#include "ils_internal.h"

namespace ils {

// y[i] = sum_j X[i][j] v[j] - b[i] over rows [0, rows), warp per row, two accumulators
__global__ void rows_minus_b_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows, int64_t cols,
                                    const double* __restrict__ v, const double* __restrict__ b,
                                    double* __restrict__ y) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < rows; i += nw) {
    const double* xr = X + i * ldx;
    double s0 = 0.0, s1 = 0.0;
    int64_t j = lane;
    for (; j + 32 < cols; j += 64) {
      s0 = fma(xr[j], v[j], s0);
      s1 = fma(xr[j + 32], v[j + 32], s1);
    }
    if (j < cols) s0 = fma(xr[j], v[j], s0);
    const double s = warp_sum(s0 + s1);
    if (lane == 0) y[i] = b ? s - b[i] : s;
  }
}

// The same row pass with 16-byte loads, four of the row and four of v in flight per lane (16-byte
// aligned rows: every caller's padded layout), as gemv_rows2_kernel (ingest.cu)
__global__ void rows_minus_b2_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows, int64_t cols,
                                     const double* __restrict__ v, const double* __restrict__ b,
                                     double* __restrict__ y) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t c2 = cols >> 1;
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
    if (lane == 0) y[i] = b ? s - b[i] : s;
  }
}

static int launch_rows_minus_b(const double* X, int64_t ldx, int64_t rows, int64_t cols, const double* v,
                                const double* b, double* y, cudaStream_t st) {
  const bool al16 = (((uintptr_t)X | (uintptr_t)v) & 15) == 0 && (ldx & 1) == 0;
  if (al16) {
    rows_minus_b2_kernel<<<148 * 16, 256, 0, st>>>(X, ldx, rows, cols, v, b, y);
    ILS_LAUNCHED("rows_minus_b2_kernel");
  } else {
    rows_minus_b_kernel<<<148 * 16, 256, 0, st>>>(X, ldx, rows, cols, v, b, y);
    ILS_LAUNCHED("rows_minus_b_kernel");
  }
  return ILS_OK;
}

// c[j] = (base[j]) + alpha * sum_i X[i][j] y[i]: columns split over CTAs, rows over warps of a CTA
// (fixed-order combine in shared memory), coalesced row segments
__global__ void __launch_bounds__(256) cols_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows,
                                                   int64_t cols, const double* __restrict__ y, double alpha,
                                                   const double* base, double* c, int tri_lower = 0) {
  __shared__ double part[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t j0 = (int64_t)blockIdx.x * 32; j0 < cols; j0 += (int64_t)gridDim.x * 32) {
    const int64_t j = j0 + lane;
    double s = 0.0;
    if (j < cols) {   // tri_lower: X[i][j] = 0 for i < j, so rows start at the tile's first column
      // eight rows in flight per warp (all eight loads issued before the first fma)
      double a[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] = 0.0;
      int64_t i = (tri_lower ? j0 : 0) + warp;
      for (; i + 56 < rows; i += 64) {
        double xv[8], yv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          xv[u] = __ldcs(X + (i + 8 * u) * ldx + j);
          yv[u] = __ldg(y + i + 8 * u);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = fma(xv[u], yv[u], a[u]);
      }
      for (; i < rows; i += 8) a[0] = fma(X[i * ldx + j], y[i], a[0]);
      s = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    }
    part[warp][lane] = s;
    __syncthreads();
    if (warp == 0 && j < cols) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += part[w][lane];
      c[j] = (base ? base[j] : 0.0) + alpha * t;
    }
    __syncthreads();
  }
}

// y = T c for the lower-triangular m x m block T (row stride ld, 16-byte aligned rows); warp per row
__global__ void __launch_bounds__(256) tri_rows_kernel(const double* __restrict__ T, int64_t ld, int64_t m,
                                                       const double* __restrict__ c, double* __restrict__ y) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double2* c2 = reinterpret_cast<const double2*>(c);
  for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < m; i += (int64_t)gridDim.x * 8) {
    const double2* tr = reinterpret_cast<const double2*>(T + i * ld);
    const int64_t k1 = (i >> 1) + 1;   // double2 entries covering columns 0..i (i + 1 is zero if present)
    double a8[8];   // four 16-byte loads of the row in flight per lane
#pragma unroll
    for (int u = 0; u < 8; ++u) a8[u] = 0.0;
    int64_t k = lane;
    for (; k + 96 < k1; k += 128) {
      double2 tv[4], cv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        tv[u] = __ldcs(tr + k + 32 * u);
        cv[u] = __ldg(c2 + k + 32 * u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a8[2 * u] = fma(tv[u].x, cv[u].x, a8[2 * u]);
        a8[2 * u + 1] = fma(tv[u].y, cv[u].y, a8[2 * u + 1]);
      }
    }
    for (; k < k1; k += 32) {
      const double2 v = __ldcs(tr + k), a = __ldg(c2 + k);
      a8[0] = fma(v.x, a.x, a8[0]);
      a8[1] = fma(v.y, a.y, a8[1]);
    }
    const double s = warp_sum(((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7])));
    if (lane == 0) y[i] = s;
  }
}

static int grid_cols(int64_t cols) {
  int64_t g = (cols + 31) / 32;
  return (int)(g > 148 * 8 ? 148 * 8 : (g < 1 ? 1 : g));
}

static int ensure_y(Handle& h) {
  if (!h.sp_y) ILS_CU(cudaMallocAsync(&h.sp_y, (size_t)(h.m + 64 + h.npad) * sizeof(double), h.stream));
  return ILS_OK;
}

// c = A1^T b1 + A2^T (A2 x - b2) (full = 0) or g = A^T J (b - A x) (full = 1), npad entries
int dense_rhs_twopass(Handle& h, const double* x, double* c, int full) {
  int rc = ensure_y(h);
  if (rc) return rc;
  const cudaStream_t st = h.stream;
  const int64_t np = h.npad;
  ILS_CU(cudaMemsetAsync(c, 0, np * sizeof(double), st));
  if (!full) {
    { const int rr_ = launch_rows_minus_b(h.Arm + h.p * np, np, h.q, h.n, x, h.b + h.p, h.sp_y, st);
      if (rr_) return rr_; }
    { const int rc_ = launch_cols(h.Arm + h.p * np, np, h.q, h.n, h.sp_y, 1.0, h.a1tb1, c, 0, st);
    if (rc_) return rc_; }
    return ILS_OK;
  }
  // g = A1^T (b1 - A1 x) - A2^T (b2 - A2 x) = -A1^T y1 + A2^T y2 with y = A x - b
  { const int rr_ = launch_rows_minus_b(h.Arm, np, h.m, h.n, x, h.b, h.sp_y, st);
    if (rr_) return rr_; }
  { const int rc_ = launch_cols(h.Arm + h.p * np, np, h.q, h.n, h.sp_y + h.p, 1.0, nullptr, c, 0, st);
    if (rc_) return rc_; }
  { const int rc_ = launch_cols(h.Arm, np, h.p, h.n, h.sp_y, -1.0, c, c, 0, st);   // in place per column
    if (rc_) return rc_; }
  return ILS_OK;
}

// stop decision of the SP-RK-RGS inner check from g (already A1^T A1 z), one CTA, fixed order
__global__ void __launch_bounds__(1024) check_finish_kernel(const double* __restrict__ g, const double* __restrict__ bhat,
                                                            int64_t n, const double* __restrict__ az,
                                                            const double* __restrict__ w, double* __restrict__ r,
                                                            int64_t p, int64_t ppad, double inner_tol, int64_t t_now,
                                                            DevStatus* st) {
  __shared__ double red[32][2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (*(volatile int32_t*)&st->inner_conv) return;
  double a = 0.0, b = 0.0;
  for (int64_t j = tid; j < n; j += 1024) {
    const double d = g[j] - bhat[j];
    a = fma(d, d, a);
    b = fma(bhat[j], bhat[j], b);
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) {
    red[warp][0] = a;
    red[warp][1] = b;
  }
  __syncthreads();
  double A = 0.0, B = 0.0;
  for (int q = 0; q < 32; ++q) {
    A += red[q][0];
    B += red[q][1];
  }
  if (sqrt(A) <= inner_tol * sqrt(B)) {
    if (tid == 0) {
      st->inner_steps = t_now;
      st->inner_conv = 1;
    }
  }
}

// the SP-RK-RGS inner check (include/ils.h) for large n: az = A1 z, g = A1^T az, decide (reads z only)
int rk_check_twopass(Handle& h, const double* z, const double* bhat, const double* w, double* r, double* az,
                     double inner_tol, int64_t t_now) {
  int rc = ensure_y(h);
  if (rc) return rc;
  const cudaStream_t st = h.stream;
  const int64_t np = h.npad;
  { const int rr_ = launch_rows_minus_b(h.Arm, np, h.p, h.n, z, nullptr, az, st);
    if (rr_) return rr_; }
  double* g = h.sp_y + h.m + 64;
  { const int rc_ = launch_cols(h.Arm, np, h.p, h.n, az, 1.0, nullptr, g, 0, st);
    if (rc_) return rc_; }
  check_finish_kernel<<<1, 1024, 0, st>>>(g, bhat, h.n, az, w, r, h.p, h.ppad, inner_tol, t_now, h.dstat);
  ILS_LAUNCHED("check_finish_kernel");
  return ILS_OK;
}

__global__ void add_kernel(double* __restrict__ x, const double* __restrict__ y, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] += y[i];
}

// The same product as cols_kernel, tiled for HBM: a CTA owns a tile of 512 columns (two per thread, one
// 16-byte load per row: 4 KB contiguous per row and CTA instead of 256 B per warp) and a chunk of rows,
// eight rows in flight per thread; the per-chunk partial sums go to a workspace [chunks][cols] and
// cols_tile_reduce_kernel adds them in chunk order (fixed geometry: deterministic). tri_lower: rows
// above the tile's first column hold zeros and are skipped.
constexpr int CT_THREADS = 256, CT_COLS = 2 * CT_THREADS;
__global__ void __launch_bounds__(CT_THREADS) cols_tile_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows,
                                                               int64_t cols, const double* __restrict__ y,
                                                               int64_t rc, int tri_lower, double* __restrict__ part) {
  const int64_t j0 = (int64_t)blockIdx.x * CT_COLS, jt = j0 + 2 * threadIdx.x;
  const int64_t chunk = blockIdx.y;
  int64_t ra = chunk * rc, rb = ra + rc < rows ? ra + rc : rows;
  if (tri_lower && ra < j0) ra = j0;
  double sx = 0.0, sy = 0.0;
  if (jt + 1 < cols) {
    const double* xp = X + jt;
    double ax[8], ay[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) ax[u] = ay[u] = 0.0;
    int64_t i = ra;
    for (; i + 8 <= rb; i += 8) {
      double2 xv[8];
      double yv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        xv[u] = __ldcs(reinterpret_cast<const double2*>(xp + (i + u) * ldx));
        yv[u] = __ldg(y + i + u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        ax[u] = fma(xv[u].x, yv[u], ax[u]);
        ay[u] = fma(xv[u].y, yv[u], ay[u]);
      }
    }
    for (; i < rb; ++i) {
      const double2 xv = __ldcs(reinterpret_cast<const double2*>(xp + i * ldx));
      const double yv = __ldg(y + i);
      ax[0] = fma(xv.x, yv, ax[0]);
      ay[0] = fma(xv.y, yv, ay[0]);
    }
    sx = ((ax[0] + ax[1]) + (ax[2] + ax[3])) + ((ax[4] + ax[5]) + (ax[6] + ax[7]));
    sy = ((ay[0] + ay[1]) + (ay[2] + ay[3])) + ((ay[4] + ay[5]) + (ay[6] + ay[7]));
  } else if (jt < cols) {   // odd column count: the last column alone
    for (int64_t i = ra; i < rb; ++i) sx = fma(X[i * ldx + jt], __ldg(y + i), sx);
  }
  if (jt < cols) part[chunk * cols + jt] = sx;
  if (jt + 1 < cols) part[chunk * cols + jt + 1] = sy;
}

// c[j] = base[j] + alpha * sum_k part[k][j]: a CTA of 32 x 8 threads owns 32 columns; thread (lane, g)
// adds the chunks k = g, g + 8, ... (eight loads in flight), then the eight group sums are added in
// group order (fixed geometry: deterministic). One thread per column adding all chunks in turn was
// latency-bound (12.6 us per launch at c3, half of the pass it finishes).
__global__ void __launch_bounds__(256) cols_tile_reduce_kernel(const double* __restrict__ part, int64_t chunks,
                                                               int64_t cols, double alpha, const double* base,
                                                               double* c) {
  __shared__ double gs[8][32];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  double t = 0.0;
  if (j < cols) {
    int64_t k = g;
    for (; k + 56 < chunks; k += 64) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(part + (k + 8 * u) * cols + j);
#pragma unroll
      for (int u = 0; u < 8; ++u) t += v[u];
    }
    for (; k < chunks; k += 8) t += __ldcs(part + k * cols + j);
  }
  gs[g][lane] = t;
  __syncthreads();
  if (g == 0 && j < cols) {
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += gs[u][lane];
    c[j] = (base ? base[j] : 0.0) + alpha * s;
  }
}

// c = base + alpha * X^T y over `rows` rows (tri_lower: X lower triangular, zero rows skipped)
int launch_cols(const double* X, int64_t ldx, int64_t rows, int64_t cols, const double* y, double alpha,
                const double* base, double* c, int tri_lower, cudaStream_t st) {
  if (cols <= 0) return ILS_OK;
  const char* e = getenv("ILS_COLS_TILED");   // override: 0 = the 32-column kernel, 2 = tiled at any size (tests)
  const bool al16 = ((uintptr_t)X & 15) == 0 && (ldx & 1) == 0;
  const bool big = (rows >= 256 && cols >= 64) || (e && e[0] == '2');
  if (al16 && big && !(e && e[0] == '0')) {
    const int64_t nct = (cols + CT_COLS - 1) / CT_COLS;
    int cps = 8;                                           // CTAs per SM over the whole panel (ILS_COLS_CPS: experiment)
    if (const char* ec = getenv("ILS_COLS_CPS")) cps = atoi(ec) > 0 ? atoi(ec) : cps;
    int64_t chunks = ((int64_t)148 * cps + nct - 1) / nct;
    if (chunks > rows / 32) chunks = rows / 32;            // at least 32 rows per chunk
    if (chunks < 1) chunks = 1;
    int64_t rc = (rows + chunks - 1) / chunks;
    if (rc < 1) rc = 1;                                    // rows = 0 (forced mode): one chunk of zeros
    chunks = (rows + rc - 1) / rc;
    if (chunks < 1) chunks = 1;
    double* part = nullptr;
    ILS_CU(cudaMallocAsync(&part, (size_t)chunks * cols * sizeof(double), st));
    cols_tile_kernel<<<dim3((unsigned)nct, (unsigned)chunks), CT_THREADS, 0, st>>>(X, ldx, rows, cols, y, rc, tri_lower,
                                                                                    part);
    ILS_LAUNCHED("cols_tile_kernel");
    cols_tile_reduce_kernel<<<(unsigned)((cols + 31) / 32), 256, 0, st>>>(part, chunks, cols, alpha, base, c);
    ILS_LAUNCHED("cols_tile_reduce_kernel");
    ILS_CU(cudaFreeAsync(part, st));
    return ILS_OK;
  }
  cols_kernel<<<grid_cols(cols), 256, 0, st>>>(X, ldx, rows, cols, y, alpha, base, c, tri_lower);
  ILS_LAUNCHED("cols_kernel");
  return ILS_OK;
}

int launch_tri_rows(const double* T, int64_t ld, int64_t m, const double* c, double* y, cudaStream_t st) {
  if (m <= 0) return ILS_OK;
  int64_t g = (m + 7) / 8;
  if (g > 148 * 8) g = 148 * 8;
  tri_rows_kernel<<<(unsigned)g, 256, 0, st>>>(T, ld, m, c, y);
  ILS_LAUNCHED("tri_rows_kernel");
  return ILS_OK;
}

// x += y over n entries (the correction form x_{k+1} = x_k + P g_k on the two-pass path)
int vec_add(Handle& h, double* x, const double* y, int64_t n) {
  add_kernel<<<148, 256, 0, h.stream>>>(x, y, n);
  ILS_LAUNCHED("add_kernel");
  return ILS_OK;
}

}  // namespace ils
