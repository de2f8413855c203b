// sparse.cu -- K5: the CSR input path (BASELINE.json configs[3]).
//
// Ingest: validation, CSR -> CSC of A1 and of A2 (count, scan, scatter, per-column rank sort by
//         row: a deterministic layout), column norms N_j (sequential in i, no FMA: include/ils.h)
//         and A1^T b1 from the CSC of A1.
// Gram:   A1bar = A1^T A1 formed densely for the exact-inverse SP baseline and the
//         SP-SCD row table: one CTA per column j accumulates row j of A1bar in shared memory from
//         the column's entries (i, v) and the CSR row i (fixed order: deterministic), then writes it.
// Stream: c_k = A1^T b1 + A2^T (A2 x_k - b2) (Alg. 2 step 5) as a CSR row pass (y = A2 x - b2)
//         and a CSC column pass (fixed order per column, no atomics). The "full" variant gives
//         g = A^T J (b - A x) for the RR stop and the correction form.
// SP-RK-RGS: persistent single-CTA chunk kernel; w, r (p-vectors, L2-resident) are gathered /
//         scattered at the ~250 rows of the two sampled columns; <a_j2, a_j1> comes from the dense
//         A1bar (prefetched with the index ring). Check: A1 z (CSR) and A1^T (A1 z) (CSC).
// SP-SCD: A1bar compacted to CSR (~11% dense at c3); one CTA keeps r (n <= 26000) in shared
//         memory; membership masks precomputed per chunk (scd.cu); check r = b_hat - A1bar beta.
#include <cstdio>
#include <climits>

#include <cooperative_groups.h>

#include <cstdlib>

#include <type_traits>

#include "common.cuh"
#include "ils_internal.h"

namespace cg = cooperative_groups;

namespace ils {

// ---------------------------------------------------------------------------------------------
// ingest
__global__ void csr_validate_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                    const double* __restrict__ va, int64_t m, int64_t n, int64_t nnz,
                                    int32_t* flag) {
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = rp[i], b = rp[i + 1];
    if (a > b || a < 0 || b > nnz) {
      bad = 1;
      continue;
    }
    int prev = -1;
    for (int64_t e = a; e < b; ++e) {
      const int c = ci[e];
      if (c <= prev || c >= n) bad = 1;   // in range, strictly increasing (no duplicates)
      if (!isfinite(va[e])) bad = 1;
      prev = c;
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

__global__ void csc_count_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t r0,
                                 int64_t r1, int32_t* __restrict__ cnt) {
  for (int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < r1; i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) atomicAdd(&cnt[ci[e]], 1);
}

// exclusive scan of int32 counts into int64 pointers (one CTA of 1024 threads, chunked)
__global__ void __launch_bounds__(1024) scan_counts_kernel(const int32_t* __restrict__ cnt, int64_t n,
                                                           int64_t* __restrict__ ptr) {
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t a = tid * per, b = (a + per < n) ? a + per : n;
  int64_t s = 0;
  for (int64_t j = a; j < b; ++j) s += cnt[j];
  part[tid] = s;
  __syncthreads();
  if (tid == 0) {
    int64_t acc = 0;
    for (int t = 0; t < 1024; ++t) {
      const int64_t v = part[t];
      part[t] = acc;
      acc += v;
    }
    ptr[n] = acc;
  }
  __syncthreads();
  int64_t acc = part[tid];
  for (int64_t j = a; j < b; ++j) {
    ptr[j] = acc;
    acc += cnt[j];
  }
}

__global__ void csc_scatter_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                   const double* __restrict__ va, int64_t r0, int64_t r1,
                                   const int64_t* __restrict__ cptr, int32_t* __restrict__ cursor,
                                   int32_t* __restrict__ crow, double* __restrict__ cval) {
  for (int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < r1; i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const int c = ci[e];
      const int64_t pos = cptr[c] + atomicAdd(&cursor[c], 1);
      crow[pos] = (int32_t)(i - r0);
      cval[pos] = va[e];
    }
}

// rank sort of each column by row (rows in a column are distinct): a warp per column
constexpr int SORT_CAP = 1024;
__global__ void __launch_bounds__(128) csc_sort_kernel(const int64_t* __restrict__ cptr, int32_t* __restrict__ crow,
                                                       double* __restrict__ cval, int64_t n) {
  __shared__ int32_t srow[4][SORT_CAP];
  __shared__ double sval[4][SORT_CAP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t j = (int64_t)blockIdx.x * 4 + warp; j < n; j += (int64_t)gridDim.x * 4) {
    const int64_t a = cptr[j];
    const int k = (int)(cptr[j + 1] - a);
    if (k <= 1) continue;
    if (k <= SORT_CAP) {
      for (int e = lane; e < k; e += 32) {
        srow[warp][e] = crow[a + e];
        sval[warp][e] = cval[a + e];
      }
      __syncwarp();
      for (int e = lane; e < k; e += 32) {
        const int r = srow[warp][e];
        int rank = 0;
        for (int f = 0; f < k; ++f) rank += (srow[warp][f] < r);
        crow[a + rank] = r;
        cval[a + rank] = sval[warp][e];
      }
      __syncwarp();
    } else if (lane == 0) {   // long column: insertion sort in place
      for (int e = 1; e < k; ++e) {
        const int r = crow[a + e];
        const double v = cval[a + e];
        int f = e - 1;
        while (f >= 0 && crow[a + f] > r) {
          crow[a + f + 1] = crow[a + f];
          cval[a + f + 1] = cval[a + f];
          --f;
        }
        crow[a + f + 1] = r;
        cval[a + f + 1] = v;
      }
    }
  }
}

// N_j = sum_i A1[i,j]^2 in increasing i without FMA (include/ils.h); t_j = sum_i A1[i,j] b_i
__global__ void csc_colnorms_kernel(const int64_t* __restrict__ cptr, const int32_t* __restrict__ crow,
                                    const double* __restrict__ cval, const double* __restrict__ b, int64_t n,
                                    double* __restrict__ N, double* __restrict__ atb) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0, t = 0.0;
    for (int64_t e = cptr[j]; e < cptr[j + 1]; ++e) {
      const double v = cval[e];
      s = __dadd_rn(s, __dmul_rn(v, v));
      t = fma(v, b[crow[e]], t);
    }
    N[j] = s;
    atb[j] = t;
  }
}

// ---------------------------------------------------------------------------------------------
// dense Gram rows from the sparse A (rows [r0, r1)): G[j][:] (+)= alpha * sum_{(i,v) in col j} v A[i,:]
// One CTA per column j (row j of G lives in shared memory); padded rows j >= n get the identity.
__global__ void __launch_bounds__(256) sparse_gram_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                          const double* __restrict__ va, int64_t r0,
                                                          const int64_t* __restrict__ cptr,
                                                          const int32_t* __restrict__ crow,
                                                          const double* __restrict__ cval, int64_t n, int64_t npad,
                                                          double alpha, int accumulate, double* __restrict__ G) {
  extern __shared__ __align__(16) double gs[];
  const int64_t j = blockIdx.x;
  double* grow = G + j * npad;
  if (j >= n) {   // padding: identity row (accumulate mode leaves it untouched)
    if (!accumulate)
      for (int64_t k = threadIdx.x; k < npad; k += blockDim.x) grow[k] = (k == j) ? 1.0 : 0.0;
    return;
  }
  for (int64_t k = threadIdx.x; k < npad; k += blockDim.x) gs[k] = accumulate ? grow[k] : 0.0;
  __syncthreads();
  if (threadIdx.x < 32) {
    // One warp applies the column's entries in their stored order (deterministic sums); the
    // dependent global loads are batched: lane l fetches entry base + l's row, value and row
    // extent, then the first 32 entries of G_ROWS consecutive rows are loaded before any of them
    // is applied (G_ROWS rows in flight instead of one).
    constexpr int G_ROWS = 8;
    const int lane = threadIdx.x;
    const int64_t e0 = cptr[j], e1 = cptr[j + 1];
    for (int64_t base = e0; base < e1; base += 32) {
      const int64_t e = base + lane;
      double v = 0.0;
      int64_t f0 = 0, f1 = 0;
      if (e < e1) {
        const int64_t i = r0 + crow[e];
        v = alpha * cval[e];
        f0 = rp[i];
        f1 = rp[i + 1];
      }
      const int cnt = (int)((e1 - base) < 32 ? (e1 - base) : 32);
      for (int q0 = 0; q0 < cnt; q0 += G_ROWS) {
        int cc[G_ROWS];
        double aa[G_ROWS];
#pragma unroll
        for (int u = 0; u < G_ROWS; ++u) {
          const int64_t g0 = __shfl_sync(0xffffffffu, f0, (q0 + u) & 31);
          const int64_t g1 = __shfl_sync(0xffffffffu, f1, (q0 + u) & 31);
          const bool ok = (q0 + u < cnt) && (g0 + lane < g1);
          cc[u] = ok ? ci[g0 + lane] : -1;
          aa[u] = ok ? va[g0 + lane] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < G_ROWS; ++u) {
          const double vu = __shfl_sync(0xffffffffu, v, (q0 + u) & 31);
          if (cc[u] >= 0) gs[cc[u]] = fma(vu, aa[u], gs[cc[u]]);
          // rows longer than 32 entries: the rest in order (rare on the benchmark data)
          const int64_t g0 = __shfl_sync(0xffffffffu, f0, (q0 + u) & 31);
          const int64_t g1 = __shfl_sync(0xffffffffu, f1, (q0 + u) & 31);
          if (q0 + u < cnt && g1 - g0 > 32) {
            __syncwarp();
            for (int64_t f = g0 + 32 + lane; f < g1; f += 32) gs[ci[f]] = fma(vu, va[f], gs[ci[f]]);
          }
          __syncwarp();
        }
      }
    }
  }
  __syncthreads();
  for (int64_t k = threadIdx.x; k < npad; k += blockDim.x) grow[k] = gs[k];
}

// The same Gram row, with the dependent global loads taken off the applying warp (default; the
// kernel above is kept as ILS_SPGRAM_OLD=1). Entries of column j are handled in chunks of GS_EC:
//   (1) every thread loads one entry's row i, value v and row extent [rp[i], rp[i+1]) (two dependent
//       loads, all entries at once), then a block scan of the extents gives each entry's offset in
//       the chunk's contribution list;
//   (2) the contributions (k, a_ik) are loaded by all threads into shared memory, in windows of
//       ccap (an entry's row may straddle two windows);
//   (3) warp 0 applies them in stored entry order, a row's contributions lane-parallel (distinct k
//       within a row), __syncwarp between rows -- the same per-address fma order as the kernel above,
//       so G is bitwise identical; the next row's (k, a) are read before the current row is applied.
constexpr int GS_EC = 256;
constexpr int GS_T = 256;
__global__ void __launch_bounds__(GS_T) sparse_gram_staged_kernel(
    const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, const double* __restrict__ va, int64_t r0,
    const int64_t* __restrict__ cptr, const int32_t* __restrict__ crow, const double* __restrict__ cval, int64_t n,
    int64_t npad, double alpha, int accumulate, int ccap, double* __restrict__ G) {
  extern __shared__ __align__(16) double gs[];                                    // [npad]
  double* ca = gs + npad;                                                         // [ccap]
  int32_t* ck = reinterpret_cast<int32_t*>(ca + ccap);                            // [ccap]
  __shared__ double ev[GS_EC];
  __shared__ int64_t ers[GS_EC];
  __shared__ int32_t eoff[GS_EC + 1];
  __shared__ int32_t wsum[GS_T / 32];
  const int64_t j = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* grow = G + j * npad;
  if (j >= n) {
    if (!accumulate)
      for (int64_t k = tid; k < npad; k += GS_T) grow[k] = (k == j) ? 1.0 : 0.0;
    return;
  }
  for (int64_t k = tid; k < npad; k += GS_T) gs[k] = accumulate ? grow[k] : 0.0;
  const int64_t e0 = cptr[j], e1 = cptr[j + 1];
  for (int64_t b = e0; b < e1; b += GS_EC) {
    const int cnt = (int)((e1 - b) < GS_EC ? (e1 - b) : GS_EC);
    int len = 0;
    if (tid < cnt) {
      const int64_t i = r0 + crow[b + tid];
      ev[tid] = alpha * cval[b + tid];
      const int64_t f0 = rp[i];
      ers[tid] = f0;
      len = (int)(rp[i + 1] - f0);
    }
    // exclusive block scan of the extents
    int x = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();   // also: the previous chunk's apply is complete (ev / ers / eoff reusable below)
    int wb = 0;
#pragma unroll
    for (int w = 0; w < GS_T / 32; ++w) wb += (w < warp) ? wsum[w] : 0;
    if (tid < GS_EC) eoff[tid] = wb + x - len;
    if (tid == GS_T - 1) eoff[GS_EC] = wb + x;
    __syncthreads();
    const int total = eoff[GS_EC];
    int ebeg = 0;   // first entry overlapping the current window (warp 0's cursor)
    for (int c0 = 0; c0 < total; c0 += ccap) {
      const int c1 = (c0 + ccap < total) ? c0 + ccap : total;
      for (int f = c0 + tid; f < c1; f += GS_T) {   // entry of contribution f: last e with eoff[e] <= f
        int lo = 0, hi = cnt - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (eoff[mid] <= f) lo = mid; else hi = mid - 1;
        }
        const int64_t g = ers[lo] + (f - eoff[lo]);
        ck[f - c0] = ci[g];
        ca[f - c0] = va[g];
      }
      __syncthreads();
      if (warp == 0) {
        int e = ebeg;
        while (e < cnt && eoff[e + 1] <= c0) ++e;   // empty rows / rows finished in the last window
        // software pipeline: (k, a) of row e read before row e - 1 is applied
        auto fetch = [&](int ee, int& k, double& a, double& v, int& lo2, int& hi2) {
          lo2 = eoff[ee] > c0 ? eoff[ee] : c0;
          hi2 = eoff[ee + 1] < c1 ? eoff[ee + 1] : c1;
          v = ev[ee];
          const int f = lo2 + lane;
          k = (f < hi2) ? ck[f - c0] : -1;
          a = (f < hi2) ? ca[f - c0] : 0.0;
        };
        int k = -1, lo2 = 0, hi2 = 0;
        double a = 0.0, v = 0.0;
        if (e < cnt && eoff[e] < c1) fetch(e, k, a, v, lo2, hi2);
        while (e < cnt && eoff[e] < c1) {
          int kn = -1, lon = 0, hin = 0;
          double an = 0.0, vn = 0.0;
          const bool more = (e + 1 < cnt) && eoff[e + 1] < c1;
          if (more) fetch(e + 1, kn, an, vn, lon, hin);
          if (k >= 0) gs[k] = fma(v, a, gs[k]);
          for (int f = lo2 + 32 + lane; f < hi2; f += 32) gs[ck[f - c0]] = fma(v, ca[f - c0], gs[ck[f - c0]]);
          __syncwarp();
          if (eoff[e + 1] > c1) break;   // row continues in the next window
          ++e;
          k = kn;
          a = an;
          v = vn;
          lo2 = lon;
          hi2 = hin;
        }
        ebeg = e;
      }
      __syncthreads();   // window consumed
    }
  }
  __syncthreads();
  for (int64_t k = tid; k < npad; k += GS_T) grow[k] = gs[k];
}

// ---------------------------------------------------------------------------------------------
// right-hand-side stream
// y[i - r0] = sigma_i (A_i x - b_i), sigma = -1 for i < psig (A1 rows of the full residual)
__global__ void spmv_rows_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 const double* __restrict__ va, const double* __restrict__ b,
                                 const double* __restrict__ x, int64_t r0, int64_t r1, int64_t psig,
                                 double* __restrict__ y) {
  for (int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < r1; i += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) d = fma(va[e], x[ci[e]], d);
    d = b ? d - b[i] : d;
    y[i - r0] = (i < psig) ? -d : d;
  }
}

// c_j = (base_j or c_j if accumulate) + sum over the CSC entries (i, v) of column j of v y_i
__global__ void spmv_cols_kernel(const int64_t* __restrict__ cptr, const int32_t* __restrict__ crow,
                                 const double* __restrict__ cval, const double* __restrict__ y,
                                 const double* __restrict__ base, int64_t n, int64_t npad, int accumulate,
                                 double* __restrict__ c) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < npad; j += (int64_t)gridDim.x * blockDim.x) {
    if (j >= n) {
      if (!accumulate) c[j] = 0.0;
      continue;
    }
    double s = accumulate ? c[j] : (base ? base[j] : 0.0);
    for (int64_t e = cptr[j]; e < cptr[j + 1]; ++e) s = fma(cval[e], y[crow[e]], s);
    c[j] = s;
  }
}

static int grid_for(int64_t work, int bs) {
  int64_t g = (work + bs - 1) / bs;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return (int)g;
}

// c = A1^T b1 + A2^T (A2 x - b2) (full = 0) or g = A^T J (b - A x) (full = 1); c has npad entries
int sparse_rhs(Handle& h, const double* x, double* c, int full) {
  const cudaStream_t st = h.stream;
  double* y = h.sp_y;
  if (!full) {
    spmv_rows_kernel<<<grid_for(h.q, 256), 256, 0, st>>>(h.rp, h.ci, h.va, h.b, x, h.p, h.m, 0, y);
    ILS_LAUNCHED("spmv_rows_kernel");
    spmv_cols_kernel<<<grid_for(h.npad, 256), 256, 0, st>>>(h.cp2, h.cr2, h.cv2, y, h.a1tb1, h.n, h.npad, 0, c);
    ILS_LAUNCHED("spmv_cols_kernel");
    return ILS_OK;
  }
  spmv_rows_kernel<<<grid_for(h.m, 256), 256, 0, st>>>(h.rp, h.ci, h.va, h.b, x, 0, h.m, h.p, y);
  ILS_LAUNCHED("spmv_rows_kernel");
  spmv_cols_kernel<<<grid_for(h.npad, 256), 256, 0, st>>>(h.cp1, h.cr1, h.cv1, y, nullptr, h.n, h.npad, 0, c);
  ILS_LAUNCHED("spmv_cols_kernel");
  spmv_cols_kernel<<<grid_for(h.npad, 256), 256, 0, st>>>(h.cp2, h.cr2, h.cv2, y + h.p, nullptr, h.n, h.npad, 1, c);
  ILS_LAUNCHED("spmv_cols_kernel");
  return ILS_OK;
}

// ---------------------------------------------------------------------------------------------
// create-time ingest for CSR input (device arrays already copied into the handle)
static int build_csc(Handle& h, int64_t r0, int64_t r1, int64_t** cptr, int32_t** crow, double** cval,
                     int32_t* cnt) {
  const cudaStream_t st = h.stream;
  const int64_t n = h.n;
  const int64_t nnz = 0;
  (void)nnz;
  ILS_CU(cudaMemsetAsync(cnt, 0, (size_t)n * sizeof(int32_t), st));
  csc_count_kernel<<<grid_for(r1 - r0, 256), 256, 0, st>>>(h.rp, h.ci, r0, r1, cnt);
  ILS_LAUNCHED("csc_count_kernel");
  ILS_CU(cudaMallocAsync(cptr, (size_t)(n + 1) * sizeof(int64_t), st));
  scan_counts_kernel<<<1, 1024, 0, st>>>(cnt, n, *cptr);
  ILS_LAUNCHED("scan_counts_kernel");
  int64_t total = 0;
  ILS_CU(cudaMemcpyAsync(&total, *cptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  ILS_CU(cudaStreamSynchronize(st));
  ILS_CU(cudaMallocAsync(crow, (size_t)(total > 0 ? total : 1) * sizeof(int32_t), st));
  ILS_CU(cudaMallocAsync(cval, (size_t)(total > 0 ? total : 1) * sizeof(double), st));
  ILS_CU(cudaMemsetAsync(cnt, 0, (size_t)n * sizeof(int32_t), st));
  csc_scatter_kernel<<<grid_for(r1 - r0, 256), 256, 0, st>>>(h.rp, h.ci, h.va, r0, r1, *cptr, cnt, *crow, *cval);
  ILS_LAUNCHED("csc_scatter_kernel");
  csc_sort_kernel<<<grid_for(n * 32, 128), 128, 0, st>>>(*cptr, *crow, *cval, n);
  ILS_LAUNCHED("csc_sort_kernel");
  return ILS_OK;
}

int sparse_ingest(Handle& h, int32_t* d_flag, bool* ok) {
  const cudaStream_t st = h.stream;
  ILS_CU(cudaMemsetAsync(d_flag, 0, sizeof(int32_t), st));
  csr_validate_kernel<<<grid_for(h.m, 256), 256, 0, st>>>(h.rp, h.ci, h.va, h.m, h.n, h.nnz, d_flag);
  ILS_LAUNCHED("csr_validate_kernel");
  int32_t f = 0;
  ILS_CU(cudaMemcpyAsync(&f, d_flag, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  ILS_CU(cudaStreamSynchronize(st));
  *ok = (f == 0);
  if (!*ok) return ILS_OK;
  int32_t* cnt = nullptr;
  ILS_CU(cudaMallocAsync(&cnt, (size_t)h.n * sizeof(int32_t), st));
  int rc = build_csc(h, 0, h.p, &h.cp1, &h.cr1, &h.cv1, cnt);
  if (!rc) rc = build_csc(h, h.p, h.m, &h.cp2, &h.cr2, &h.cv2, cnt);
  cudaFreeAsync(cnt, st);
  if (rc) return rc;
  csc_colnorms_kernel<<<grid_for(h.n, 256), 256, 0, st>>>(h.cp1, h.cr1, h.cv1, h.b, h.n, h.N, h.a1tb1);
  ILS_LAUNCHED("csc_colnorms_kernel");
  ILS_CU(cudaMemsetAsync(h.a1tb1 + h.n, 0, (h.npad - h.n) * sizeof(double), st));
  ILS_CU(cudaMallocAsync(&h.sp_y, (size_t)(h.m + 64) * sizeof(double), st));
  return ILS_OK;
}

// Gram rows G[j][:] (+)= alpha * sum over the CSC entries of column j (rows r0 + i of the CSR) --
// the staged kernel by default, the one-warp kernel with ILS_SPGRAM_OLD=1
static int launch_sparse_gram(Handle& h, int64_t r0, const int64_t* cptr, const int32_t* crow, const double* cval,
                              double alpha, int accumulate, double* G) {
  const cudaStream_t st = h.stream;
  const size_t row = (size_t)h.npad * sizeof(double);
  const size_t limit = 227 * 1024 - 6 * 1024;   // dynamic part; the staged kernel's static arrays ~5.2 KB
  const char* ev = getenv("ILS_SPGRAM_OLD");
  const bool old = ev && ev[0] == '1';
  if (!old && row + 256 * 12 <= limit) {
    int64_t ccap = (int64_t)((limit - row) / 12);
    if (ccap > 8192) ccap = 8192;
    const char* ec = getenv("ILS_SPGRAM_CCAP");   // test knob: a small window (rows straddling windows)
    if (ec && atoi(ec) > 0 && atoi(ec) < ccap) ccap = atoi(ec);
    const size_t smem = row + (size_t)ccap * 12;
    ILS_CU(cudaFuncSetAttribute(sparse_gram_staged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    sparse_gram_staged_kernel<<<(unsigned)h.npad, GS_T, smem, st>>>(h.rp, h.ci, h.va, r0, cptr, crow, cval, h.n, h.npad,
                                                                    alpha, accumulate, (int)ccap, G);
    ILS_LAUNCHED("sparse_gram_staged_kernel");
    return ILS_OK;
  }
  if (row > 227 * 1024) {
    set_error("sparse path: n > 29000 does not fit the shared-memory Gram row");
    return ILS_ERR_UNSUPPORTED;
  }
  ILS_CU(cudaFuncSetAttribute(sparse_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row));
  sparse_gram_kernel<<<(unsigned)h.npad, 256, row, st>>>(h.rp, h.ci, h.va, r0, cptr, crow, cval, h.n, h.npad, alpha,
                                                         accumulate, G);
  ILS_LAUNCHED("sparse_gram_kernel");
  return ILS_OK;
}

// dense A1bar (alpha = 1) or M = A1bar - A2^T A2 (into a caller buffer) from the CSR/CSC arrays
int sparse_gram(Handle& h, double* G, bool subtract_a2) {
  if (!subtract_a2) return launch_sparse_gram(h, 0, h.cp1, h.cr1, h.cv1, 1.0, 0, G);
  return launch_sparse_gram(h, h.p, h.cp2, h.cr2, h.cv2, -1.0, 1, G);
}

__global__ void neg_copy_kernel(const double* __restrict__ x, int64_t len, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) y[i] = -x[i];
}

__global__ void zero_pad_diag_kernel(double* __restrict__ G, int64_t n, int64_t npad) {
  for (int64_t j = n + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < npad; j += (int64_t)gridDim.x * blockDim.x)
    G[j * npad + j] = 0.0;
}

// Paper-literal precompute for CSR input (Alg. 1 steps 2-3; Alg. 2 steps 2-3,
// :291-292; Alg. 5 steps 2-4, :689-691): A2bar = A2^T A2 as dense rows from the CSC of A2 (the Gram
// kernel of A1bar run over the A2 rows, zero padding), and A^T J b = A1^T b1 - A2^T b2 by one CSC
// column pass over -b2.
int sparse_a2bar(Handle& h, double* A2bar, double* ajb) {
  const cudaStream_t st = h.stream;
  int rc = launch_sparse_gram(h, h.p, h.cp2, h.cr2, h.cv2, 1.0, 0, A2bar);
  if (rc) return rc;
  if (h.npad > h.n) {   // the Gram kernel writes identity rows for the padding: A2bar is zero there
    zero_pad_diag_kernel<<<1, 64, 0, st>>>(A2bar, h.n, h.npad);
    ILS_LAUNCHED("zero_pad_diag_kernel");
  }
  if (h.q > 0) {
    neg_copy_kernel<<<grid_for(h.q, 256), 256, 0, st>>>(h.b + h.p, h.q, h.sp_y);
    ILS_LAUNCHED("neg_copy_kernel");
    spmv_cols_kernel<<<grid_for(h.npad, 256), 256, 0, st>>>(h.cp2, h.cr2, h.cv2, h.sp_y, h.a1tb1, h.n, h.npad, 0, ajb);
    ILS_LAUNCHED("spmv_cols_kernel");
  } else {
    ILS_CU(cudaMemcpyAsync(ajb, h.a1tb1, h.npad * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  return ILS_OK;
}

// ---------------------------------------------------------------------------------------------
// x = P c (dense, npad x npad): warp per row, 8 outstanding 16-byte loads per lane
__global__ void __launch_bounds__(256) gemv_p_kernel(const double* __restrict__ P, const double* __restrict__ c,
                                                     int64_t npad, int64_t n, double* __restrict__ x) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t np2 = npad / 2;
  const double2* c2 = reinterpret_cast<const double2*>(c);
  for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < npad; i += (int64_t)gridDim.x * 8) {
    const double2* pr = reinterpret_cast<const double2*>(P + i * npad);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t k = lane;
    for (; k + 7 * 32 < np2; k += 8 * 32) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcs(pr + k + 32 * u);
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        const double2 a = __ldg(c2 + k + 32 * u), b = __ldg(c2 + k + 32 * (u + 1));
        s0 = fma(v[u].x, a.x, s0);
        s1 = fma(v[u].y, a.y, s1);
        s2 = fma(v[u + 1].x, b.x, s2);
        s3 = fma(v[u + 1].y, b.y, s3);
      }
    }
    for (; k < np2; k += 32) {
      const double2 v = __ldcs(pr + k), a = __ldg(c2 + k);
      s0 = fma(v.x, a.x, s0);
      s1 = fma(v.y, a.y, s1);
    }
    const double s = warp_sum((s0 + s1) + (s2 + s3));
    if (lane == 0) x[i] = (i < n) ? s : 0.0;
  }
}

int gemv_p(Handle& h, const double* c, double* x) {
  if (h.use_zt) return zc_apply_tree(h, c, x);   // x = Z^T (Z c) through the recursion's spine (dla.cu)
  gemv_p_kernel<<<(unsigned)(h.num_sms * 8), 256, 0, h.stream>>>(h.P, c, h.npad, h.n, x);
  ILS_LAUNCHED("gemv_p_kernel");
  return ILS_OK;
}

// ---------------------------------------------------------------------------------------------
// SP-RK-RGS on CSR input: one CTA; steps [t0, t1) of one inner solve; w, r, z in global memory.
struct SpRkParams {
  const int64_t* cp;    // CSC of A1
  const int32_t* cr;
  const double* cv;
  const double* G;      // dense A1bar (npad x npad): <a_j2, a_j1>
  int64_t npad;
  int n;
  const double* N;
  const uint64_t* S;
  const double* bhat;
  double* W;
  double* Rv;
  double* Z;
  uint64_t seed;
  uint32_t k;
  int64_t t0, t1;
  DevStatus* st;
  long long* prof;      // sparse_rk_la_kernel<true>: per-phase cycles (thread 0), ILS_SRK_PROF=1
};

struct SpRkIdx {
  int32_t j1, j2;
  double bh1, rn1, rn2, g21;
  int64_t a1, a2;    // CSC starts of the two columns
  int32_t k1, k2;    // their lengths
};

constexpr int SRK_RING = 128;
constexpr int SRK_T = 256;

__device__ __forceinline__ void srk_fill(const SpRkParams& p, const uint64_t* Ss, SpRkIdx* ring, int64_t t0, int lane) {
  const int64_t t = t0 + lane;
  if (t < p.t1) {
    const U4 x = draw(p.seed, p.k, (uint64_t)t, kTagRkRgs);
    const int j1 = sample_weighted(((uint64_t)x.y << 32) | x.x, Ss, p.n);
    const int j2 = sample_weighted(((uint64_t)x.w << 32) | x.z, Ss, p.n);
    SpRkIdx e;
    e.j1 = j1;
    e.j2 = j2;
    e.bh1 = p.bhat[j1];
    e.rn1 = 1.0 / p.N[j1];
    e.rn2 = 1.0 / p.N[j2];
    e.g21 = p.G[(int64_t)j2 * p.npad + j1];
    e.a1 = p.cp[j1];
    e.a2 = p.cp[j2];
    e.k1 = (int32_t)(p.cp[j1 + 1] - e.a1);
    e.k2 = (int32_t)(p.cp[j2 + 1] - e.a2);
    ring[t & (SRK_RING - 1)] = e;
  }
}

constexpr int SRK_D = 4;        // column prefetch depth (steps)
constexpr int SRK_MAXK = 512;   // column entries staged per column (longer columns read from global)

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
// first index f in sorted rows[0, k) with rows[f] == r, else -1
__device__ __forceinline__ int find_row(const int32_t* rows, int k, int r) {
  int lo = 0, hi = k;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (rows[mid] < r) lo = mid + 1; else hi = mid;
  }
  return (lo < k && rows[lo] == r) ? lo : -1;
}

// One step needs the entries (i, v) of columns j1 and j2 (CSC, sorted by row). They are staged in
// shared memory SRK_D steps ahead (cp.async; the index stream is data-independent). Per step ONE
// round of independent gathers (w at rows of j1, r at rows of j1 and of j2), one block reduction,
// then plain stores: a row present in both columns is written once, by its j2 entry, as
// (r + s1 a_j1) - s2 a_j2 (the sequential order of Alg. 2 steps 9 and 11); the match is a binary
// search in the other column's staged rows.
__global__ void __launch_bounds__(SRK_T) sparse_rk_kernel(SpRkParams p) {
  extern __shared__ __align__(16) unsigned char srk_smem[];
  double (*cvs)[2][SRK_MAXK] = reinterpret_cast<double (*)[2][SRK_MAXK]>(srk_smem);              // [D][2][MAXK]
  int32_t (*crs)[2][SRK_MAXK] = reinterpret_cast<int32_t (*)[2][SRK_MAXK]>(srk_smem + SRK_D * 2 * SRK_MAXK * 8);
  uint64_t* Ssm = reinterpret_cast<uint64_t*>(srk_smem + SRK_D * 2 * SRK_MAXK * 12);           // [n]
  __shared__ SpRkIdx ring[SRK_RING];
  __shared__ double red[2][SRK_T / 32][2];
  __shared__ double bn_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (*(volatile int32_t*)&p.st->inner_conv) return;
  for (int j = tid; j < p.n; j += SRK_T) Ssm[j] = p.S[j];
  if (p.t0 == 0) {   // b_hat = 0: z = 0 after 0 steps
    double v = 0.0;
    for (int j = tid; j < p.n; j += SRK_T) v = fma(p.bhat[j], p.bhat[j], v);
    v = warp_sum(v);
    if (lane == 0) red[0][warp][0] = v;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < SRK_T / 32; ++w) s += red[0][w][0];
      bn_s = s;
    }
    __syncthreads();
    if (bn_s == 0.0) {
      if (tid == 0) {
        p.st->inner_steps = 0;
        p.st->inner_conv = 1;
      }
      return;
    }
  }
  __syncthreads();
  if (warp == 0) srk_fill(p, Ssm, ring, p.t0, lane);
  if (warp == 1) srk_fill(p, Ssm, ring, p.t0 + 32, lane);
  __syncthreads();
  auto stage = [&](int64_t t) {   // cp.async the two columns of step t into slot t % D
    if (t < p.t1) {
      const SpRkIdx ix = ring[t & (SRK_RING - 1)];
      const int sl = (int)(t % SRK_D);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int64_t a = c ? ix.a2 : ix.a1;
        const int k = min(SRK_MAXK, c ? ix.k2 : ix.k1);
        for (int e = tid; e < k; e += SRK_T) {
          cp_async4(&crs[sl][c][e], p.cr + a + e);
          cp_async8(&cvs[sl][c][e], p.cv + a + e);
        }
      }
    }
    cp_async_commit();
  };
  for (int64_t t = p.t0; t < p.t0 + SRK_D; ++t) stage(t);
  for (int64_t t = p.t0; t < p.t1; ++t) {
    const int pb = (int)(t & 1);
    const int sl = (int)(t % SRK_D);
    if (warp == 7 && ((t - p.t0) & 31) == 0 && t + 64 < p.t1) srk_fill(p, Ssm, ring, t + 64, lane);
    cp_async_wait<SRK_D - 1>();
    __syncthreads();   // slot sl staged by every thread
    const SpRkIdx ix = ring[t & (SRK_RING - 1)];
    const int64_t a1 = ix.a1, a2 = ix.a2;
    const int k1 = ix.k1, k2 = ix.k2;
    // z_{j2}: its load rides with the gathers; the store below follows the previous step's store
    // to the same address in program order of thread 0
    const double zold = (tid == 0) ? p.Z[ix.j2] : 0.0;
    const int32_t* R1 = crs[sl][0];
    const int32_t* R2 = crs[sl][1];
    const bool st1 = k1 <= SRK_MAXK, st2 = k2 <= SRK_MAXK;
    // gathers (one round of independent loads)
    constexpr int EPT = (SRK_MAXK + SRK_T - 1) / SRK_T;
    int i1[EPT], i2[EPT];
    double v1[EPT], v2[EPT], w1[EPT], q1[EPT], q2[EPT];
    double d1 = 0.0, d2 = 0.0;
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
      const int e = tid + u * SRK_T;
      i1[u] = -1;
      i2[u] = -1;
      if (e < k1) {
        i1[u] = st1 ? R1[e] : p.cr[a1 + e];
        v1[u] = st1 ? cvs[sl][0][e] : p.cv[a1 + e];
        w1[u] = p.W[i1[u]];
        q1[u] = p.Rv[i1[u]];
      }
      if (e < k2) {
        i2[u] = st2 ? R2[e] : p.cr[a2 + e];
        v2[u] = st2 ? cvs[sl][1][e] : p.cv[a2 + e];
        q2[u] = p.Rv[i2[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < EPT; ++u) {
      if (i1[u] >= 0) d1 = fma(v1[u], w1[u], d1);
      if (i2[u] >= 0) d2 = fma(v2[u], q2[u], d2);
    }
    for (int e = tid + EPT * SRK_T; e < k1; e += SRK_T) d1 = fma(p.cv[a1 + e], p.W[p.cr[a1 + e]], d1);
    for (int e = tid + EPT * SRK_T; e < k2; e += SRK_T) d2 = fma(p.cv[a2 + e], p.Rv[p.cr[a2 + e]], d2);
    d1 = warp_sum(d1);
    d2 = warp_sum(d2);
    if (lane == 0) {
      red[pb][warp][0] = d1;
      red[pb][warp][1] = d2;
    }
    __syncthreads();
    double D1 = 0.0, D2 = 0.0;
#pragma unroll
    for (int w = 0; w < SRK_T / 32; ++w) {
      D1 += red[pb][w][0];
      D2 += red[pb][w][1];
    }
    const double s1 = (ix.bh1 - D1) * ix.rn1;
    const double s2 = (D2 + s1 * ix.g21) * ix.rn2;
    const bool fast = st1 && st2 && k1 <= EPT * SRK_T && k2 <= EPT * SRK_T;
    if (fast) {
#pragma unroll
      for (int u = 0; u < EPT; ++u) {
        if (i1[u] >= 0) {
          p.W[i1[u]] = fma(s1, v1[u], w1[u]);
          if (find_row(R2, k2, i1[u]) < 0) p.Rv[i1[u]] = fma(s1, v1[u], q1[u]);
        }
        if (i2[u] >= 0) {
          const int f = find_row(R1, k1, i2[u]);
          const double base = (f >= 0) ? fma(s1, cvs[sl][0][f], q2[u]) : q2[u];
          p.Rv[i2[u]] = fma(-s2, v2[u], base);
        }
      }
    } else {   // long columns: the two-phase read-modify-write form
      for (int e = tid; e < k1; e += SRK_T) {
        const int i = p.cr[a1 + e];
        const double v = p.cv[a1 + e];
        p.W[i] = fma(s1, v, p.W[i]);
        p.Rv[i] = fma(s1, v, p.Rv[i]);
      }
      __syncthreads();
      for (int e = tid; e < k2; e += SRK_T) {
        const int i = p.cr[a2 + e];
        p.Rv[i] = fma(-s2, p.cv[a2 + e], p.Rv[i]);
      }
    }
    if (tid == 0) p.Z[ix.j2] = zold + s2;
    __syncthreads();   // next step's gathers see these stores; slot sl is free
    stage(t + SRK_D);
  }
  cp_async_wait<0>();
}

// inner check: az = A1 z (rows, CSR), g = A1^T az - b_hat (CSC), stop (cooperative; reads z only)
__global__ void __launch_bounds__(256) sparse_rk_check_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                              const double* __restrict__ va, int64_t p_rows,
                                                              const int64_t* __restrict__ cp,
                                                              const int32_t* __restrict__ cr,
                                                              const double* __restrict__ cv, int64_t n,
                                                              const double* __restrict__ bhat,
                                                              const double* __restrict__ Z, const double* __restrict__ W,
                                                              double* __restrict__ Rv, double* __restrict__ az,
                                                              double* __restrict__ red, double inner_tol, int64_t t_now,
                                                              DevStatus* st) {
  cg::grid_group grid = cg::this_grid();
  if (*(volatile int32_t*)&st->inner_conv) return;
  __shared__ double sr[8][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gsz = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = gtid; i < p_rows; i += gsz) {
    double d = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) d = fma(va[e], Z[ci[e]], d);
    az[i] = d;
  }
  grid.sync();
  double a = 0.0, b = 0.0;
  for (int64_t j = gtid; j < n; j += gsz) {
    double s = 0.0;
    for (int64_t e = cp[j]; e < cp[j + 1]; ++e) s = fma(cv[e], az[cr[e]], s);
    const double g = s - bhat[j];
    a = fma(g, g, a);
    b = fma(bhat[j], bhat[j], b);
  }
  a = warp_sum(a);
  b = warp_sum(b);
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
  }
}

// ---------------------------------------------------------------------------------------------
// Look-ahead SP-RK-RGS on CSR input (one CTA, all columns staged: <= SRK_LA_K entries each). The
// gathers of w at the rows of a_u = A1_(j1_u) and of r at the rows of b_u = A1_(j2_u) are issued
// two steps ahead, on the state S_g before steps g..u-1 (g = max(t0, u - 2)); the missing updates
// enter the products through A1bar (dense, resident):
//   <a_u, w_u> = <a_u, w_g> + sum_m s1_m <a_u, a_m>
//   <b_u, r_u> = <b_u, r_g> + sum_m (s1_m <b_u, a_m> - s2_m <b_u, b_m>)        (m = g .. u-1)
// (the identity of rk_rgs.cu's look-ahead kernel; Alg. 2 steps 9 and 11). The
// updates are applied as floating-point reductions to global memory (one per address per step: a
// row in both columns is updated once, by its b-entry, with s1 a_i - s2 b_i), ordered across steps
// by the step barrier, so the result is deterministic. Per step: one block reduction of two values,
// the gather latency is off the step chain.
constexpr int SRK_LA_K = 512;   // EPT * SRK_T entries per column
struct SpRkLaIdx {
  int32_t j1, j2;
  double bh1, rn1, rn2, g21;
  double ga1, ga2, gb1, gb2, gbb1, gbb2;   // <a_t, a_{t-1}>, <a_t, a_{t-2}>, <b_t, a_{t-1}>, <b_t, a_{t-2}>,
                                           // <b_t, b_{t-1}>, <b_t, b_{t-2}> (0 before the chunk start)
  int64_t a1, a2;
  int32_t k1, k2;
};

__device__ __forceinline__ void srk_la_fill(const SpRkParams& p, const uint64_t* Ss, SpRkLaIdx* ring, int64_t f0,
                                            int lane) {
  const int64_t t = f0 + lane;
  SpRkLaIdx e{};
  const bool live = t < p.t1;
  if (live) {
    const U4 x = draw(p.seed, p.k, (uint64_t)t, kTagRkRgs);
    e.j1 = sample_weighted(((uint64_t)x.y << 32) | x.x, Ss, p.n);
    e.j2 = sample_weighted(((uint64_t)x.w << 32) | x.z, Ss, p.n);
    e.bh1 = p.bhat[e.j1];
    e.rn1 = 1.0 / p.N[e.j1];
    e.rn2 = 1.0 / p.N[e.j2];
    e.a1 = p.cp[e.j1];
    e.a2 = p.cp[e.j2];
    e.k1 = (int32_t)(p.cp[e.j1 + 1] - e.a1);
    e.k2 = (int32_t)(p.cp[e.j2 + 1] - e.a2);
    ring[t & (SRK_RING - 1)].j1 = e.j1;
    ring[t & (SRK_RING - 1)].j2 = e.j2;
  }
  __syncwarp();
  if (live) {   // indices of steps t-1, t-2 (this fill or the previous one), then the Gram values
    const int64_t np = p.npad;
    const double* Ga = p.G + (int64_t)e.j1 * np;
    const double* Gb = p.G + (int64_t)e.j2 * np;
    e.g21 = Gb[e.j1];
    if (t - 1 >= p.t0) {
      const SpRkLaIdx& q = ring[(t - 1) & (SRK_RING - 1)];
      e.ga1 = Ga[q.j1];
      e.gb1 = Gb[q.j1];
      e.gbb1 = Gb[q.j2];
    }
    if (t - 2 >= p.t0) {
      const SpRkLaIdx& q = ring[(t - 2) & (SRK_RING - 1)];
      e.ga2 = Ga[q.j1];
      e.gb2 = Gb[q.j1];
      e.gbb2 = Gb[q.j2];
    }
  }
  __syncwarp();
  if (live) ring[t & (SRK_RING - 1)] = e;
}

template <bool PROF>
__global__ void __launch_bounds__(SRK_T) sparse_rk_la_kernel(SpRkParams p) {
  long long pc[6] = {0, 0, 0, 0, 0, 0}, tc0 = PROF ? clock64() : 0;
#define SLAP(q)                                      \
  do {                                               \
    if (PROF && threadIdx.x == 0) {                  \
      const long long c_ = clock64();                \
      pc[q] += c_ - tc0;                             \
      tc0 = c_;                                      \
    }                                                \
  } while (0)
  extern __shared__ __align__(16) unsigned char srk_smem[];
  double (*cvs)[2][SRK_MAXK] = reinterpret_cast<double (*)[2][SRK_MAXK]>(srk_smem);              // [D][2][MAXK]
  int32_t (*crs)[2][SRK_MAXK] = reinterpret_cast<int32_t (*)[2][SRK_MAXK]>(srk_smem + SRK_D * 2 * SRK_MAXK * 8);
  uint64_t* Ssm = reinterpret_cast<uint64_t*>(srk_smem + SRK_D * 2 * SRK_MAXK * 12);           // [n]
  __shared__ SpRkLaIdx ring[SRK_RING];
  __shared__ double red[2][SRK_T / 32][2];
  __shared__ double bn_s;
  constexpr int EPT = SRK_LA_K / SRK_T;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (*(volatile int32_t*)&p.st->inner_conv) return;
  for (int j = tid; j < p.n; j += SRK_T) Ssm[j] = p.S[j];
  if (p.t0 == 0) {   // b_hat = 0: z = 0 after 0 steps
    double v = 0.0;
    for (int j = tid; j < p.n; j += SRK_T) v = fma(p.bhat[j], p.bhat[j], v);
    v = warp_sum(v);
    if (lane == 0) red[0][warp][0] = v;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < SRK_T / 32; ++w) s += red[0][w][0];
      bn_s = s;
    }
    __syncthreads();
    if (bn_s == 0.0) {
      if (tid == 0) {
        p.st->inner_steps = 0;
        p.st->inner_conv = 1;
      }
      return;
    }
  }
  __syncthreads();
  if (warp == 0) srk_la_fill(p, Ssm, ring, p.t0, lane);
  __syncthreads();
  if (warp == 0) srk_la_fill(p, Ssm, ring, p.t0 + 32, lane);
  __syncthreads();
  auto stage = [&](int64_t t) {   // cp.async the two columns of step t into slot t % D
    if (t < p.t1) {
      const SpRkLaIdx& ix = ring[t & (SRK_RING - 1)];
      const int sl = (int)(t % SRK_D);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int64_t a = c ? ix.a2 : ix.a1;
        const int k = c ? ix.k2 : ix.k1;
        for (int e = tid; e < k; e += SRK_T) {
          cp_async4(&crs[sl][c][e], p.cr + a + e);
          cp_async8(&cvs[sl][c][e], p.cv + a + e);
        }
      }
    }
    cp_async_commit();
  };
  for (int64_t t = p.t0; t < p.t0 + SRK_D; ++t) stage(t);
  double gw[3][EPT], gq[3][EPT];   // gathered w at rows of a_u, r at rows of b_u: buffer (u - t0) % 3
  auto gather = [&](int64_t u, double (&w)[EPT], double (&q)[EPT]) {
    const SpRkLaIdx& ix = ring[u & (SRK_RING - 1)];
    const int sl = (int)(u % SRK_D);
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const int i = tid + e * SRK_T;
      w[e] = (i < ix.k1) ? p.W[crs[sl][0][i]] : 0.0;
      q[e] = (i < ix.k2) ? p.Rv[crs[sl][1][i]] : 0.0;
    }
  };
  cp_async_wait<SRK_D - 2>();   // slots t0, t0 + 1
  __syncthreads();
  if (p.t0 < p.t1) gather(p.t0, gw[0], gq[0]);
  if (p.t0 + 1 < p.t1) gather(p.t0 + 1, gw[1], gq[1]);
  double s1m1 = 0.0, s1m2 = 0.0, s2m1 = 0.0, s2m2 = 0.0;   // scalars of steps t-1, t-2
  auto body = [&](int64_t t, auto phc) {
    constexpr int PH = decltype(phc)::value, NX = (PH + 2) % 3;
    const int pb = (int)(t & 1);
    if (warp == 7 && ((t - p.t0) & 31) == 0 && t + 64 < p.t1) srk_la_fill(p, Ssm, ring, t + 64, lane);
    SLAP(5);
    cp_async_wait<1>();   // slot of step t + 2 (groups up to t + 3 issued)
    __syncthreads();
    SLAP(0);
    if (t + 2 < p.t1) gather(t + 2, gw[NX], gq[NX]);   // on S_t: corrected for steps t, t+1 later
    const SpRkLaIdx& ix = ring[t & (SRK_RING - 1)];
    const int sl = (int)(t % SRK_D);
    const int32_t* R1 = crs[sl][0];
    const int32_t* R2 = crs[sl][1];
    double d1 = 0.0, d2 = 0.0;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const int i = tid + e * SRK_T;
      if (i < ix.k1) d1 = fma(cvs[sl][0][i], gw[PH][e], d1);
      if (i < ix.k2) d2 = fma(cvs[sl][1][i], gq[PH][e], d2);
    }
    d1 = warp_sum(d1);
    d2 = warp_sum(d2);
    if (lane == 0) {
      red[pb][warp][0] = d1;
      red[pb][warp][1] = d2;
    }
    SLAP(1);
    __syncthreads();
    SLAP(2);
    double D1 = 0.0, D2 = 0.0;
#pragma unroll
    for (int w = 0; w < SRK_T / 32; ++w) {
      D1 += red[pb][w][0];
      D2 += red[pb][w][1];
    }
    // corrections for the steps the gathered state missed (zero Gram values before the chunk start)
    D1 = fma(s1m1, ix.ga1, D1);
    D1 = fma(s1m2, ix.ga2, D1);
    D2 = fma(s1m1, ix.gb1, D2);
    D2 = fma(s1m2, ix.gb2, D2);
    D2 = fma(-s2m1, ix.gbb1, D2);
    D2 = fma(-s2m2, ix.gbb2, D2);
    const double s1 = (ix.bh1 - D1) * ix.rn1;
    const double s2 = (D2 + s1 * ix.g21) * ix.rn2;
    // rows shared by a_t and b_t get one combined update; with <b_t, a_t> = 0 the columns share no
    // row (but for an exact cancellation, where the two updates of a row stay separate reductions)
    const bool shared = ix.g21 != 0.0;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const int i = tid + e * SRK_T;
      if (i < ix.k1) {
        const int row = R1[i];
        const double dv = s1 * cvs[sl][0][i];
        atomicAdd(p.W + row, dv);
        if (!shared || find_row(R2, ix.k2, row) < 0) atomicAdd(p.Rv + row, dv);
      }
      if (i < ix.k2) {
        const int row = R2[i];
        const int f = shared ? find_row(R1, ix.k1, row) : -1;
        const double dv = (f >= 0) ? fma(s1, cvs[sl][0][f], -s2 * cvs[sl][1][i]) : -s2 * cvs[sl][1][i];
        atomicAdd(p.Rv + row, dv);
      }
    }
    if (tid == 0) atomicAdd(p.Z + ix.j2, s2);
    SLAP(3);
    s1m2 = s1m1;
    s1m1 = s1;
    s2m2 = s2m1;
    s2m1 = s2;
    __syncthreads();   // this step's updates precede the next step's gathers; slot sl is free
    SLAP(4);
    stage(t + SRK_D);
  };
  int64_t t = p.t0;
  for (; t + 2 < p.t1; t += 3) {
    body(t, std::integral_constant<int, 0>{});
    body(t + 1, std::integral_constant<int, 1>{});
    body(t + 2, std::integral_constant<int, 2>{});
  }
  if (t < p.t1) body(t, std::integral_constant<int, 0>{});
  if (t + 1 < p.t1) body(t + 1, std::integral_constant<int, 1>{});
  cp_async_wait<0>();
  if (PROF && threadIdx.x == 0)
    for (int q = 0; q < 6; ++q) atomicAdd(reinterpret_cast<unsigned long long*>(p.prof + q), (unsigned long long)pc[q]);
#undef SLAP
}

// ---------------------------------------------------------------------------------------------
// 16-CTA cluster SP-RK-RGS on CSR input (default when the sampling table fits shared memory;
// ILS_SRK_CL=0 keeps the one-CTA look-ahead kernel). CTA c owns rows [c R, (c + 1) R) of w and r
// (global memory, L2-resident); the entries of a column inside those rows are one contiguous range
// of the row-sorted CSC (split table: one lower_bound per column and CTA, built once per handle).
// B = 4 steps per cluster exchange with the blocked recurrence of rk_rgs.cu (RkBlk<4>: identical to
// four single steps of Alg. 2 steps 9 and 11, in exact arithmetic):
//   per block each CTA gathers w at its entries of a_k = A1_(j1_k) and r at those of b_k = A1_(j2_k)
//   (k < 4), forms the 8 partial inner products, sends them to all 16 CTAs (destination-uniform
//   st.async, mbarrier complete_tx); warp 0 sums the 16 partials in rank order, adds the 22 in-block
//   Gram values read from A1bar, runs the recurrence for s1_k, s2_k and publishes them; warp 1 then
//   applies w += s1_k a_k and warp 2 r += s1_k a_k - s2_k b_k to the CTA's rows as floating-point
//   reductions, column by column in step order with __syncwarp between columns (one reduction per
//   address per column, so the result is deterministic); rank 0 adds s2_k to z_(j2_k).
// A fill warp runs up to SRC_NS blocks ahead in rounds of SRC_NS / 2 blocks: indices (Philox +
// weighted inverse CDF on the shared prefix sums), 1/N, b_hat, Gram values, the CTA's segment of
// each column and its entries (row, value) copied into the block's shared-memory slot (entries past
// SRC_CAP per block are read from global memory by the consumers).
constexpr int SRC_C = 16, SRC_T = 256, SRC_NWC = 7, SRC_CAP = 256, SRC_HB = 9;

// named barrier over nthreads threads that also ORs a predicate over them
__device__ __forceinline__ bool bar_red_or(int id, int nthreads, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "bar.red.or.pred q, %2, %3, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)pred), "r"(id), "r"(nthreads)
      : "memory");
  return r != 0;
}
struct SrcSlot {
  int32_t row[SRC_CAP];
  double val[SRC_CAP];
  int64_t gbase[8];   // CSC index of each segment's first entry (segments a0, b0, a1, b1, ...)
  int32_t off[9];     // segment offsets in the block's entry list
  int32_t j1[4], j2[4];
  double gv[22];      // in-block Gram values, RkBlk<4> order (value 8 + v)
  double bh1[4], rn1[4], rn2[4];
};

// (value v < 22 of the in-block Gram) -> the two columns: (step, is_b) pairs in RkBlk<4> order
// (AA(i,k) k < i, BA(i,k) k <= i, BB(i,k) k < i)
__device__ __forceinline__ void src_gram_cols(int v, int& si, int& bi, int& sk, int& bk) {
  if (v < 6) {            // AA: (1,0) (2,0) (2,1) (3,0) (3,1) (3,2)
    si = v < 1 ? 1 : (v < 3 ? 2 : 3);
    sk = v - si * (si - 1) / 2;
    bi = 0;
    bk = 0;
  } else if (v < 16) {    // BA: (0,0) (1,0) (1,1) (2,0) (2,1) (2,2) (3,0) ...
    const int w = v - 6;
    si = w < 1 ? 0 : (w < 3 ? 1 : (w < 6 ? 2 : 3));
    sk = w - si * (si + 1) / 2;
    bi = 1;
    bk = 0;
  } else {                // BB
    const int w = v - 16;
    si = w < 1 ? 1 : (w < 3 ? 2 : 3);
    sk = w - si * (si - 1) / 2;
    bi = 1;
    bk = 1;
  }
}

struct SrcParams {
  SpRkParams b;
  const int32_t* split;   // [n][17]
  int64_t R;              // rows per CTA
  int ns;                 // slots (8 or 16)
};

__global__ void __launch_bounds__(SRC_T, 1) sparse_rk_cl_kernel(SrcParams q) {
  const SpRkParams& p = q.b;
  extern __shared__ __align__(16) unsigned char src_smem[];
  uint64_t* Ssm = reinterpret_cast<uint64_t*>(src_smem);                                   // [n]
  SrcSlot* slots = reinterpret_cast<SrcSlot*>(src_smem + (((size_t)p.n * 8 + 15) & ~(size_t)15));   // [ns]
  __shared__ __align__(16) double recv[2][SRC_C][8];
  __shared__ __align__(8) uint64_t rbar[2];
  __shared__ __align__(8) uint64_t full[16];
  __shared__ double part[SRC_NWC][8];
  __shared__ unsigned long long htab[1 << SRC_HB];   // (block tag << 32) | row of the current block's entries
  __shared__ double sv[2][8];
  __shared__ __align__(8) int64_t done_s;
  __shared__ double red0[SRC_T / 32];
  __shared__ int zero_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)cluster_ctarank();
  const int NS = q.ns, RD = NS / 2;
  if (*(volatile int32_t*)&p.st->inner_conv) return;   // the same flag in every CTA
  for (int j = tid; j < p.n; j += SRC_T) Ssm[j] = p.S[j];
  for (int u = tid; u < (1 << SRC_HB); u += SRC_T) htab[u] = 0ull;
  if (tid == 0) {
    mbar_init(&rbar[0], 1);
    mbar_init(&rbar[1], 1);
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&rbar[0], SRC_C * 64);
    mbar_arrive_expect_tx(&rbar[1], SRC_C * 64);
    done_s = 0;
    zero_s = 0;
  }
  if (p.t0 == 0) {   // b_hat = 0: z = 0 after 0 steps (every CTA decides the same)
    double v = 0.0;
    for (int j = tid; j < p.n; j += SRC_T) v = fma(p.bhat[j], p.bhat[j], v);
    v = warp_sum(v);
    if (lane == 0) red0[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double s_ = 0.0;
      for (int w = 0; w < SRC_T / 32; ++w) s_ += red0[w];
      zero_s = (s_ == 0.0);
    }
  }
  __syncthreads();
  cluster_sync_all();   // barriers initialised everywhere before any remote st.async
  if (zero_s) {
    if (rank == 0 && tid == 0) {
      p.st->inner_steps = 0;
      p.st->inner_conv = 1;
    }
    cluster_sync_all();
    return;
  }
  const int64_t nblk = (p.t1 - p.t0 + 3) / 4;
  if (warp == SRC_NWC) {   // ---- fill warp
    long long fbusy = 0;
    const int NSM = NS - 1;   // NS is a power of two
    for (int64_t f = 0; f < nblk; f += RD) {
      while (f + RD - NS > ld_acquire_cta_s64(&done_s)) {
      }
      const long long fc0 = (p.prof && rank == 0) ? clock64() : 0;
      const int nb = (int)((nblk - f) < RD ? (nblk - f) : RD);
      // (1) indices: lane l -> step 4 f + l (l < 4 nb; RD <= 8), the two inverse-CDF searches interleaved
      int j1 = 0, j2 = 0;
      bool live = false;
      if (lane < 4 * nb) {
        const int64_t t = p.t0 + 4 * f + lane;
        live = t < p.t1;
        double bh = 0.0, r1 = 0.0, r2 = 0.0;
        if (live) {
          const U4 x = draw(p.seed, p.k, (uint64_t)t, kTagRkRgs);
          const uint64_t tot = Ssm[p.n - 1];
          const uint64_t v1 = mulhi64(((uint64_t)x.y << 32) | x.x, tot);
          const uint64_t v2 = mulhi64(((uint64_t)x.w << 32) | x.z, tot);
          int lo1 = 0, hi1 = p.n - 1, lo2 = 0, hi2 = p.n - 1;
          while (lo1 < hi1 || lo2 < hi2) {   // the searches of sample_weighted, side by side
            const int m1 = (lo1 + hi1) >> 1, m2 = (lo2 + hi2) >> 1;
            const uint64_t s1_ = Ssm[m1], s2_ = Ssm[m2];
            if (lo1 < hi1) {
              if (s1_ > v1) hi1 = m1; else lo1 = m1 + 1;
            }
            if (lo2 < hi2) {
              if (s2_ > v2) hi2 = m2; else lo2 = m2 + 1;
            }
          }
          j1 = lo1;
          j2 = lo2;
          bh = p.bhat[j1];
          r1 = 1.0 / p.N[j1];
          r2 = 1.0 / p.N[j2];
        }
        SrcSlot& sl = slots[(f + lane / 4) & NSM];
        sl.j1[lane & 3] = j1;
        sl.j2[lane & 3] = j2;
        sl.bh1[lane & 3] = bh;
        sl.rn1[lane & 3] = r1;
        sl.rn2[lane & 3] = r2;
      }
      // (2) segments: pair (block f + u / 8, segment c = u & 7), u = lane, lane + 32 (loads of both first)
      {
        int64_t cb[2];
        int32_t o0[2], o1[2];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int u = lane + 32 * h2;
          const int bl = u >> 3, c = u & 7;
          const int src = 4 * bl + (c >> 1);
          const int ja = __shfl_sync(0xffffffffu, j1, src & 31), jb = __shfl_sync(0xffffffffu, j2, src & 31);
          const bool lv = __shfl_sync(0xffffffffu, live, src & 31);
          cb[h2] = 0;
          o0[h2] = 0;
          o1[h2] = 0;
          if (bl < nb && lv) {
            const int col = (c & 1) ? jb : ja;
            cb[h2] = p.cp[col];
            const int32_t* spl = q.split + (int64_t)col * (SRC_C + 1) + rank;
            o0[h2] = spl[0];
            o1[h2] = spl[1];
          }
        }
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int u = lane + 32 * h2;
          const int bl = u >> 3, c = u & 7;
          const int len = o1[h2] - o0[h2];
          int x = len;   // inclusive scan inside the 8-lane group
#pragma unroll
          for (int o = 1; o < 8; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o, 8);
            if (c >= o) x += y;
          }
          if (bl < nb) {
            SrcSlot& sl = slots[(f + bl) & NSM];
            sl.gbase[c] = cb[h2] + o0[h2];
            sl.off[c] = x - len;
            if (c == 7) sl.off[8] = x;
          }
        }
      }
      __syncwarp();
      // (3) Gram values: 22 per block, all loads of the round in flight together
      {
        double gq[6];
#pragma unroll
        for (int w = 0; w < 6; ++w) {
          const int u = lane + 32 * w;
          gq[w] = 0.0;
          if (u < 22 * nb) {
            const int bl = u / 22, v = u - 22 * bl;
            const SrcSlot& sl = slots[(f + bl) & NSM];
            int si, bi, sk, bk;
            src_gram_cols(v, si, bi, sk, bk);
            const int ca = bi ? sl.j2[si] : sl.j1[si];
            const int cb = bk ? sl.j2[sk] : sl.j1[sk];
            gq[w] = p.G[(int64_t)ca * p.npad + cb];
          }
        }
#pragma unroll
        for (int w = 0; w < 6; ++w) {
          const int u = lane + 32 * w;
          if (u < 22 * nb) {
            const int bl = u / 22, v = u - 22 * bl;
            slots[(f + bl) & NSM].gv[v] = gq[w];
          }
        }
      }
      // (4) entries (row, value): two blocks per batch, segment by segment (lane = position in the
      // segment; segments longer than 32 entries continue in a second loop), loads before stores
      for (int bl = 0; bl < nb; bl += 2) {
        int32_t rr[16];
        double vv[16];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const SrcSlot& sl = slots[(f + bl + u) & NSM];
          const bool on = bl + u < nb;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int e = (on ? sl.off[c] : 0) + lane;
            const int hi = on ? min(sl.off[c + 1], SRC_CAP) : 0;
            rr[8 * u + c] = 0;
            vv[8 * u + c] = 0.0;
            if (e < hi) {
              const int64_t g = sl.gbase[c] + lane;
              rr[8 * u + c] = p.cr[g];
              vv[8 * u + c] = p.cv[g];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          SrcSlot& sl = slots[(f + bl + u) & NSM];
          const bool on = bl + u < nb;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int e = (on ? sl.off[c] : 0) + lane;
            const int hi = on ? min(sl.off[c + 1], SRC_CAP) : 0;
            if (e < hi) {
              sl.row[e] = rr[8 * u + c];
              sl.val[e] = vv[8 * u + c];
            }
            for (int e2 = e + 32; e2 < hi; e2 += 32) {   // long segments
              const int64_t g = sl.gbase[c] + (e2 - sl.off[c]);
              sl.row[e2] = p.cr[g];
              sl.val[e2] = p.cv[g];
            }
          }
        }
      }
      __syncwarp();
      if (lane < nb) mbar_arrive(&full[(f + lane) & NSM]);
      if (p.prof && rank == 0) fbusy += clock64() - fc0;
    }
    if (p.prof && rank == 0 && lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(p.prof + 6), (unsigned long long)fbusy);
  } else {   // ---- consumer warps (NWC x 32 threads)
    constexpr int NTC = SRC_NWC * 32;
    using K = RkBlk<4>;
    const bool prof = p.prof && tid == 0 && rank == 0;
    long long pc[6] = {0, 0, 0, 0, 0, 0}, tc = prof ? clock64() : 0;
#define CLAP(k_)                      \
  if (prof) {                         \
    const long long c_ = clock64();   \
    pc[k_] += c_ - tc;                \
    tc = c_;                          \
  }
    for (int64_t i = 0; i < nblk; ++i) {
      const int si = (int)(i & (NS - 1));
      mbar_wait(&full[si], (uint32_t)((i / NS) & 1));
      CLAP(0)
      const SrcSlot& sl = slots[si];
      const int tot = sl.off[8];
      double acc[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = 0.0;
      // register path (at most two staged entries per thread): the thread keeps its entries' old w / r
      // and, when no row of the CTA appears in two columns of the block (shared-memory hash of the
      // block's rows, tagged by block), stores the updated values itself (fast update path)
      const bool regp = tot <= SRC_CAP && tot <= 2 * NTC;
      int frow[2] = {-1, -1}, fseg[2] = {0, 0};
      double fv[2] = {0.0, 0.0}, fw[2] = {0.0, 0.0}, fr[2] = {0.0, 0.0};
      bool dup = !regp;
      if (regp) {
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int e = tid + h2 * NTC;
          if (e < tot) {
            int c = 0;
#pragma unroll
            for (int cc = 1; cc < 8; ++cc) c += (sl.off[cc] <= e);
            frow[h2] = sl.row[e];
            fv[h2] = sl.val[e];
            fseg[h2] = c;
            fr[h2] = p.Rv[frow[h2]];
            if (!(c & 1)) fw[h2] = p.W[frow[h2]];
          }
        }
        const unsigned long long tagb = (unsigned long long)(i + 1) << 32;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          if (frow[h2] >= 0) {
            const unsigned long long key = tagb | (unsigned)frow[h2];
            uint32_t hs = ((uint32_t)frow[h2] * 2654435761u) >> (32 - SRC_HB);
            for (int probe = 0;; ++probe) {
              if (probe == (1 << SRC_HB)) {   // table full: take the ordered path
                dup = true;
                break;
              }
              unsigned long long cur = htab[hs];
              if ((cur >> 32) != (tagb >> 32)) {   // stale (an earlier block) or empty: claim it
                const unsigned long long prev = atomicCAS(&htab[hs], cur, key);
                if (prev == cur) break;
                cur = prev;
              }
              if ((cur >> 32) == (tagb >> 32)) {
                if ((uint32_t)cur == (uint32_t)frow[h2]) {   // another column of this block has the row
                  dup = true;
                  break;
                }
                hs = (hs + 1) & ((1u << SRC_HB) - 1);
              }
            }
          }
        }
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          if (frow[h2] >= 0) {
            const double d = fv[h2] * ((fseg[h2] & 1) ? fr[h2] : fw[h2]);
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) acc[cc] += (fseg[h2] == cc) ? d : 0.0;
          }
        }
      } else {
        for (int e = tid; e < tot; e += NTC) {
          int c = 0;
#pragma unroll
          for (int cc = 1; cc < 8; ++cc) c += (sl.off[cc] <= e);
          int row;
          double v;
          if (e < SRC_CAP) {
            row = sl.row[e];
            v = sl.val[e];
          } else {
            const int64_t g = sl.gbase[c] + (e - sl.off[c]);
            row = p.cr[g];
            v = p.cv[g];
          }
          const double xg = (c & 1) ? p.Rv[row] : p.W[row];
          const double d = v * xg;
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) acc[cc] += (c == cc) ? d : 0.0;
        }
      }
      // value order of RkBlk<4>: P(k) = k (a_k, w), Q(k) = 4 + k (b_k, r); segment c = 2k + is_b
      double accv[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        accv[K::P(k)] = acc[2 * k];
        accv[K::Q(k)] = acc[2 * k + 1];
      }
      const double ws = warp_reduce_scatter<8>(accv, lane);
      if (lane < 8) part[warp][lane] = ws;
      CLAP(1)
      const bool fast = !bar_red_or(1, NTC, dup);
      CLAP(2)
      const int b2 = (int)(i & 1);
      if (warp == 0) {
        double v = 0.0;
        if (lane < 8)
#pragma unroll
          for (int w = 0; w < SRC_NWC; ++w) v += part[w][lane];
        double vals[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) vals[m] = __shfl_sync(0xffffffffu, v, m);
        if (lane < SRC_C) {
          const uint32_t bar = map_shared_rank(smem_u32(&rbar[b2]), (uint32_t)lane);
#pragma unroll
          for (int m = 0; m < 4; ++m)
            st_async_v2f64(map_shared_rank(smem_u32(&recv[b2][rank][2 * m]), (uint32_t)lane), vals[2 * m],
                           vals[2 * m + 1], bar);
        }
        mbar_wait_cluster(&rbar[b2], (uint32_t)((i >> 1) & 1));
        CLAP(3)
        double tv = 0.0;
        if (lane < 8)
#pragma unroll
          for (int c = 0; c < SRC_C; ++c) tv += recv[b2][c][lane];
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&rbar[b2], SRC_C * 64);   // for block i + 2
        double T[K::NV];
#pragma unroll
        for (int m = 0; m < 8; ++m) T[m] = __shfl_sync(0xffffffffu, tv, m);
#pragma unroll
        for (int m = 8; m < K::NV; ++m) T[m] = sl.gv[m - 8];
        double s1[4], s2[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double dw = T[K::P(k)];
#pragma unroll
          for (int m = 0; m < k; ++m) dw = fma(s1[m], T[K::AA(k, m)], dw);
          s1[k] = (sl.bh1[k] - dw) * sl.rn1[k];
          double dr = T[K::Q(k)];
#pragma unroll
          for (int m = 0; m < k; ++m) {
            dr = fma(s1[m], T[K::BA(k, m)], dr);
            dr = fma(-s2[m], T[K::BB(k, m)], dr);
          }
          dr = fma(s1[k], T[K::BA(k, k)], dr);
          s2[k] = dr * sl.rn2[k];
        }
        if (lane < 4) {
          sv[b2][lane] = s1[lane & 3];
          sv[b2][4 + lane] = s2[lane & 3];
        }
      }
      named_bar_sync(1, NTC);
      CLAP(4)
      if (fast) {
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          if (frow[h2] >= 0) {
            const int k = fseg[h2] >> 1;
            if (fseg[h2] & 1) {
              p.Rv[frow[h2]] = fma(-sv[b2][4 + k], fv[h2], fr[h2]);
            } else {
              const double s1k = sv[b2][k];
              p.W[frow[h2]] = fma(s1k, fv[h2], fw[h2]);
              p.Rv[frow[h2]] = fma(s1k, fv[h2], fr[h2]);
            }
          }
        }
        if (warp == 3 && lane == 0 && rank == 0) {
          const int64_t tb = p.t0 + 4 * i;
          for (int k = 0; k < 4; ++k)
            if (tb + k < p.t1) atomicAdd(p.Z + sl.j2[k], sv[b2][4 + k]);
        }
      } else if (warp == 1 || warp == 2) {   // w (warp 1) / r (warp 2) updates, column by column in step order
        for (int c = 0; c < 8; ++c) {
          if (warp == 1 && (c & 1)) continue;
          const double sc = (c & 1) ? -sv[b2][4 + (c >> 1)] : sv[b2][c >> 1];
          double* dst = (warp == 1) ? p.W : p.Rv;
          for (int e = sl.off[c] + lane; e < sl.off[c + 1]; e += 32) {
            int row;
            double v;
            if (e < SRC_CAP) {
              row = sl.row[e];
              v = sl.val[e];
            } else {
              const int64_t g = sl.gbase[c] + (e - sl.off[c]);
              row = p.cr[g];
              v = p.cv[g];
            }
            atomicAdd(dst + row, sc * v);
          }
          __syncwarp();
        }
      } else if (warp == 3 && lane == 0 && rank == 0) {
        const int64_t tb = p.t0 + 4 * i;
        for (int k = 0; k < 4; ++k)
          if (tb + k < p.t1) atomicAdd(p.Z + sl.j2[k], sv[b2][4 + k]);
      }
      named_bar_sync(1, NTC);   // this block's updates precede the next block's gathers; slot free
      if (tid == 0) st_relaxed_cta_s64(&done_s, i + 1);   // after the barrier: see common.cuh
      CLAP(5)
    }
#undef CLAP
    if (prof)
      for (int k = 0; k < 6; ++k) atomicAdd(reinterpret_cast<unsigned long long*>(p.prof + k), (unsigned long long)pc[k]);
  }
  __syncthreads();
  cluster_sync_all();
}

// split[j][c] = (first CSC entry of column j with row >= c R) - cp[j], c = 0..16
__global__ void src_split_kernel(const int64_t* __restrict__ cp, const int32_t* __restrict__ cr, int64_t n, int64_t R,
                                 int32_t* __restrict__ split) {
  const int64_t tot = n * (SRC_C + 1);
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < tot; u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = u / (SRC_C + 1);
    const int c = (int)(u - j * (SRC_C + 1));
    const int64_t a = cp[j], b = cp[j + 1];
    const int64_t key = (int64_t)c * R;
    int64_t lo = a, hi = b;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)cr[mid] < key) lo = mid + 1; else hi = mid;
    }
    split[u] = (int32_t)(lo - a);
  }
}

__global__ void max_col_kernel(const int64_t* __restrict__ cp, int64_t n, unsigned long long* out) {
  unsigned long long m = 0;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)(cp[j + 1] - cp[j]));
  m = __reduce_max_sync(0xffffffffu, (unsigned)m);
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

int sparse_rk_inner(Handle& h, const double* bhat, double* z, uint64_t seed, int64_t k, int64_t max_inner,
                    int64_t check_every, double inner_tol, int64_t* steps_out) {
  int rc = build_gram(h);   // <a_j2, a_j1> lookups
  if (rc) return rc;
  const cudaStream_t st = h.stream;
  const int64_t ce = check_every > 0 ? check_every : h.n;
  const size_t words = (size_t)2 * h.ppad + h.ppad + h.npad + 2 * h.num_sms;
  if (!h.rk_state || h.rk_state_words < words) {
    if (h.rk_state) cudaFreeAsync(h.rk_state, st);
    ILS_CU(cudaMallocAsync(&h.rk_state, words * sizeof(double), st));
    h.rk_state_words = words;
  }
  double* W = h.rk_state;
  double* Rv = W + h.ppad;
  double* AZ = Rv + h.ppad;
  double* Z = AZ + h.ppad;
  double* red = Z + h.npad;
  ILS_CU(cudaMemsetAsync(h.rk_state, 0, (size_t)(3 * h.ppad + h.npad) * sizeof(double), st));
  ILS_CU(cudaMemsetAsync(&h.dstat->inner_conv, 0, sizeof(int32_t), st));
  ILS_CU(cudaMemsetAsync(&h.dstat->inner_steps, 0, sizeof(int64_t), st));
  SpRkParams prm{};
  prm.cp = h.cp1;
  prm.cr = h.cr1;
  prm.cv = h.cv1;
  prm.G = h.G;
  prm.npad = h.npad;
  prm.n = (int)h.n;
  prm.N = h.N;
  prm.S = h.S;
  prm.bhat = bhat;
  prm.W = W;
  prm.Rv = Rv;
  prm.Z = Z;
  prm.seed = seed;
  prm.k = (uint32_t)k;
  prm.st = h.dstat;
  const size_t smem = (size_t)SRK_D * 2 * SRK_MAXK * 12 + (size_t)h.n * sizeof(uint64_t);
  if (smem > 227 * 1024) {
    set_error("sparse SP-RK-RGS: n too large for the shared-memory sampling table");
    return ILS_ERR_UNSUPPORTED;
  }
  ILS_CU(cudaFuncSetAttribute(sparse_rk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (h.maxcol1 < 0) {
    unsigned long long* dm = nullptr;
    unsigned long long hm = 0;
    ILS_CU(cudaMallocAsync(&dm, sizeof(unsigned long long), st));
    ILS_CU(cudaMemsetAsync(dm, 0, sizeof(unsigned long long), st));
    max_col_kernel<<<64, 256, 0, st>>>(h.cp1, h.n, dm);
    ILS_LAUNCHED("max_col_kernel");
    ILS_CU(cudaMemcpyAsync(&hm, dm, sizeof(hm), cudaMemcpyDeviceToHost, st));
    ILS_CU(cudaStreamSynchronize(st));
    cudaFreeAsync(dm, st);
    h.maxcol1 = (int64_t)hm;
  }
  // 16-CTA cluster kernel when the sampling table and 8+ slots fit shared memory (ILS_SRK_CL=0: the
  // one-CTA kernels below)
  const char* ecl = getenv("ILS_SRK_CL");
  const size_t cl_base = (((size_t)h.n * 8 + 15) & ~(size_t)15);
  const size_t cl_static = 8 * 1024;
  int cl_ns = 0;
  if (!(ecl && ecl[0] == '0')) {
    if (cl_base + 16 * sizeof(SrcSlot) + cl_static <= 227 * 1024) cl_ns = 16;
    else if (cl_base + 8 * sizeof(SrcSlot) + cl_static <= 227 * 1024) cl_ns = 8;
  }
  if (cl_ns) {
    const size_t cl_smem = cl_base + (size_t)cl_ns * sizeof(SrcSlot);
    const int64_t R = (h.p + SRC_C - 1) / SRC_C;
    if (!h.sp_split) {
      ILS_CU(cudaMallocAsync(&h.sp_split, (size_t)h.n * (SRC_C + 1) * sizeof(int32_t), st));
      src_split_kernel<<<grid_for(h.n * (SRC_C + 1), 256), 256, 0, st>>>(h.cp1, h.cr1, h.n, R, h.sp_split);
      ILS_LAUNCHED("src_split_kernel");
    }
    SrcParams q{};
    q.b = prm;
    q.split = h.sp_split;
    q.R = R;
    q.ns = cl_ns;
    ILS_CU(cudaFuncSetAttribute(sparse_rk_cl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cl_smem));
    ILS_CU(cudaFuncSetAttribute(sparse_rk_cl_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(SRC_C);
    cfg.blockDim = dim3(SRC_T);
    cfg.dynamicSmemBytes = cl_smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = SRC_C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const char* eprof = getenv("ILS_SRK_PROF");
    if (eprof && eprof[0] == '1') {
      ILS_CU(cudaMallocAsync(&q.b.prof, 8 * sizeof(long long), st));
      ILS_CU(cudaMemsetAsync(q.b.prof, 0, 8 * sizeof(long long), st));
    }
    ILS_CU(cudaEventRecord(h.evk0, st));
    int64_t t = 0;
    int pending = 0;
    while (t < max_inner) {
      const int64_t t1 = (t + ce < max_inner) ? t + ce : max_inner;
      q.b.t0 = t;
      q.b.t1 = t1;
      ILS_CU(cudaLaunchKernelEx(&cfg, sparse_rk_cl_kernel, q));
      ILS_LAUNCHED("sparse_rk_cl_kernel");
      t = t1;
      if (t % ce == 0) {
        double itol = inner_tol;
        int64_t tn = t;
        const int64_t prow = h.p, nn = h.n;
        const int64_t* rp = h.rp;
        const int32_t* ci = h.ci;
        const double* va = h.va;
        const int64_t* cp = h.cp1;
        const int32_t* cr = h.cr1;
        const double* cv = h.cv1;
        DevStatus* dst = h.dstat;
        void* args[] = {(void*)&rp, (void*)&ci, (void*)&va, (void*)&prow, (void*)&cp, (void*)&cr, (void*)&cv,
                        (void*)&nn, (void*)&bhat, (void*)&Z, (void*)&W, (void*)&Rv, (void*)&AZ, (void*)&red,
                        (void*)&itol, (void*)&tn, (void*)&dst};
        ILS_CU(cudaLaunchCooperativeKernel((void*)sparse_rk_check_kernel, dim3(h.num_sms), dim3(256), args, 0, st));
        ILS_LAUNCHED("sparse_rk_check_kernel");
      }
      if (++pending == 8 || t >= max_inner) {
        ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
        ILS_CU(cudaStreamSynchronize(st));
        pending = 0;
        if (h.hstat->inner_conv) break;
      }
    }
    ILS_CU(cudaEventRecord(h.evk1, st));
    ILS_CU(cudaMemcpyAsync(z, Z, h.npad * sizeof(double), cudaMemcpyDeviceToDevice, st));
    ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
    ILS_CU(cudaStreamSynchronize(st));
    const int64_t steps = h.hstat->inner_conv ? h.hstat->inner_steps : max_inner;
    if (q.b.prof) {
      long long hp[8];
      cudaMemcpy(hp, q.b.prof, sizeof(hp), cudaMemcpyDeviceToHost);
      cudaFree(q.b.prof);
      const double blk = (double)(steps > 0 ? steps : 1) / 4.0;
      fprintf(stderr, "ILS_SRK_PROF cluster steps=%lld cycles/block: wait-full %.0f products %.0f bar1 %.0f "
              "exchange %.0f recurrence+bar2 %.0f updates+bar3 %.0f | fill busy %.0f\n", (long long)steps, hp[0] / blk,
              hp[1] / blk, hp[2] / blk, hp[3] / blk, hp[4] / blk, hp[5] / blk, hp[6] / blk);
    }
    if (steps_out) *steps_out = steps;
    const double nnz1 = (double)h.nnz1;
    hot_account(h, 1, (double)steps * 2.0 * (nnz1 / (double)h.n) * 28.0 + (double)(steps / ce) * 24.0 * nnz1,
                (steps + ce - 1) / ce);
    return ILS_OK;
  }
  // look-ahead kernel when every column is staged whole (ILS_SRK_LA=0 keeps the one-step kernel)
  const char* ela = getenv("ILS_SRK_LA");
  const bool la = h.maxcol1 <= SRK_LA_K && !(ela && ela[0] == '0');
  const char* eprof = getenv("ILS_SRK_PROF");
  const bool sprof = la && eprof && eprof[0] == '1';
  if (la) {
    ILS_CU(cudaFuncSetAttribute(sparse_rk_la_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ILS_CU(cudaFuncSetAttribute(sparse_rk_la_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  if (sprof) {
    ILS_CU(cudaMallocAsync(&prm.prof, 8 * sizeof(long long), st));
    ILS_CU(cudaMemsetAsync(prm.prof, 0, 8 * sizeof(long long), st));
  }
  const int64_t prow = h.p, nn = h.n;
  const int64_t* rp = h.rp;
  const int32_t* ci = h.ci;
  const double* va = h.va;
  const int64_t* cp = h.cp1;
  const int32_t* cr = h.cr1;
  const double* cv = h.cv1;
  DevStatus* dst = h.dstat;
  constexpr int kBatch = 8;
  ILS_CU(cudaEventRecord(h.evk0, st));
  int64_t t = 0;
  int pending = 0;
  while (t < max_inner) {
    const int64_t t1 = (t + ce < max_inner) ? t + ce : max_inner;
    prm.t0 = t;
    prm.t1 = t1;
    if (la) {
      if (sprof) sparse_rk_la_kernel<true><<<1, SRK_T, smem, st>>>(prm);
      else sparse_rk_la_kernel<false><<<1, SRK_T, smem, st>>>(prm);
      ILS_LAUNCHED("sparse_rk_la_kernel");
    } else {
      sparse_rk_kernel<<<1, SRK_T, smem, st>>>(prm);
      ILS_LAUNCHED("sparse_rk_kernel");
    }
    t = t1;
    if (t % ce == 0) {
      double itol = inner_tol;
      int64_t tn = t;
      void* args[] = {(void*)&rp, (void*)&ci, (void*)&va, (void*)&prow, (void*)&cp, (void*)&cr, (void*)&cv,
                      (void*)&nn, (void*)&bhat, (void*)&Z, (void*)&W, (void*)&Rv, (void*)&AZ, (void*)&red,
                      (void*)&itol, (void*)&tn, (void*)&dst};
      ILS_CU(cudaLaunchCooperativeKernel((void*)sparse_rk_check_kernel, dim3(h.num_sms), dim3(256), args, 0, st));
      ILS_LAUNCHED("sparse_rk_check_kernel");
    }
    if (++pending == kBatch || t >= max_inner) {
      ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
      ILS_CU(cudaStreamSynchronize(st));
      pending = 0;
      if (h.hstat->inner_conv) break;
    }
  }
  ILS_CU(cudaEventRecord(h.evk1, st));
  ILS_CU(cudaMemcpyAsync(z, Z, h.npad * sizeof(double), cudaMemcpyDeviceToDevice, st));
  ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
  ILS_CU(cudaStreamSynchronize(st));
  const int64_t steps = h.hstat->inner_conv ? h.hstat->inner_steps : max_inner;
  if (sprof) {
    long long hp[6];
    cudaMemcpy(hp, prm.prof, sizeof(hp), cudaMemcpyDeviceToHost);
    cudaFree(prm.prof);
    const double st_ = (double)(steps > 0 ? steps : 1);
    fprintf(stderr, "ILS_SRK_PROF steps=%lld cycles/step: top-barrier %.0f gather+dots+reduce %.0f barrier2 %.0f "
            "recurrence+updates %.0f end-barrier %.0f stage+loop %.0f\n", (long long)steps, hp[0] / st_, hp[1] / st_,
            hp[2] / st_, hp[3] / st_, hp[4] / st_, hp[5] / st_);
  }
  if (steps_out) *steps_out = steps;
  const double nnz1 = (double)h.nnz1;
  // bytes per step: the two sampled columns (12 B per entry) and the w / r entries they touch
  hot_account(h, 1, (double)steps * 2.0 * (nnz1 / (double)h.n) * 28.0 + (double)(steps / ce) * 24.0 * nnz1,
              (steps + ce - 1) / ce);
  return ILS_OK;
}

// ---------------------------------------------------------------------------------------------
// SP-SCD on CSR input: A1bar compacted to CSR; one CTA with r in shared memory.
__global__ void gram_count_kernel(const double* __restrict__ G, int64_t npad, int64_t n, int64_t* __restrict__ cnt) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; j < n; j += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    int64_t c = 0;
    for (int64_t k = lane; k < n; k += 32) c += (G[j * npad + k] != 0.0);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[j] = c;
  }
}

__global__ void __launch_bounds__(1024) scan64_kernel(int64_t* __restrict__ a, int64_t n) {   // exclusive, in place, a[n] = total
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t s0 = tid * per, s1 = (s0 + per < n) ? s0 + per : n;
  int64_t s = 0;
  for (int64_t j = s0; j < s1; ++j) s += a[j];
  part[tid] = s;
  __syncthreads();
  if (tid == 0) {
    int64_t acc = 0;
    for (int t = 0; t < 1024; ++t) {
      const int64_t v = part[t];
      part[t] = acc;
      acc += v;
    }
    a[n] = acc;
  }
  __syncthreads();
  int64_t acc = part[tid];
  for (int64_t j = s0; j < s1; ++j) {
    const int64_t v = a[j];
    a[j] = acc;
    acc += v;
  }
}

// ordered compaction of row j of G (ballot within the warp keeps the column order)
__global__ void gram_compact_kernel(const double* __restrict__ G, int64_t npad, int64_t n, const int64_t* __restrict__ ptr,
                                    int32_t* __restrict__ col, double* __restrict__ val) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; j < n; j += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    int64_t pos = ptr[j];
    for (int64_t k0 = 0; k0 < n; k0 += 32) {
      const int64_t k = k0 + lane;
      const double v = (k < n) ? G[j * npad + k] : 0.0;
      const unsigned m = __ballot_sync(0xffffffffu, v != 0.0);
      if (v != 0.0) {
        const int64_t at = pos + __popc(m & ((1u << lane) - 1u));
        col[at] = (int32_t)k;
        val[at] = v;
      }
      pos += __popc(m);
    }
  }
}

int sparse_gram_csr(Handle& h) {
  if (h.gcsr_ptr) return ILS_OK;
  int rc = build_gram(h);
  if (rc) return rc;
  const cudaStream_t st = h.stream;
  ILS_CU(cudaMallocAsync(&h.gcsr_ptr, (size_t)(h.n + 1) * sizeof(int64_t), st));
  gram_count_kernel<<<grid_for(h.n * 32, 256), 256, 0, st>>>(h.G, h.npad, h.n, h.gcsr_ptr);
  ILS_LAUNCHED("gram_count_kernel");
  scan64_kernel<<<1, 1024, 0, st>>>(h.gcsr_ptr, h.n);
  ILS_LAUNCHED("scan64_kernel");
  int64_t total = 0;
  ILS_CU(cudaMemcpyAsync(&total, h.gcsr_ptr + h.n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  ILS_CU(cudaStreamSynchronize(st));
  h.gnnz = total;
  ILS_CU(cudaMallocAsync(&h.gcsr_col, (size_t)(total > 0 ? total : 1) * sizeof(int32_t), st));
  ILS_CU(cudaMallocAsync(&h.gcsr_val, (size_t)(total > 0 ? total : 1) * sizeof(double), st));
  gram_compact_kernel<<<grid_for(h.n * 32, 256), 256, 0, st>>>(h.G, h.npad, h.n, h.gcsr_ptr, h.gcsr_col, h.gcsr_val);
  ILS_LAUNCHED("gram_compact_kernel");
  return ILS_OK;
}

struct SpScdParams {
  const double* Gd;        // dense A1bar rows (npad stride) for dense input with large n, else null
  const int64_t* gp;
  const int32_t* gc;
  const double* gv;
  int n;
  int64_t npad;
  const double* N;
  const double* bhat;
  double* Rv;     // [npad] state r (in/out)
  double* Bv;     // [npad] state beta (in/out)
  const uint32_t* masks;   // [t1 - t0][NT] (V coordinates per thread, s = tid + v*NT)
  int V;
  int all_members;         // alpha_t = n every step (Motzkin): no masks
  const int32_t* jw;       // weighted SP-RCD: j_t for t in [t0, t1) (rcd_index_kernel), else null
  int64_t t0, t1;
  DevStatus* st;
};

constexpr int SSCD_T = 1024;

// SP-RCD: j_t drawn from the column-norm weights, one thread per step of the
// chunk, the same draw (tag kTagRcd) and integer inverse-CDF as the one-CTA kernel (scd.cu)
__global__ void rcd_index_kernel(uint64_t seed, uint32_t k, int64_t t0, int64_t t1, int n,
                                 const uint64_t* __restrict__ S, int32_t* __restrict__ J) {
  const int64_t u = t0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= t1) return;
  const U4 x = draw(seed, k, (uint64_t)u, kTagRcd);
  J[u - t0] = sample_weighted(((uint64_t)x.y << 32) | x.x, S, n);
}

__global__ void __launch_bounds__(SSCD_T, 1) sparse_scd_kernel(SpScdParams p) {
  extern __shared__ __align__(16) double rs[];     // [npad] r
  __shared__ double wv[2][32], wr[2][32];
  __shared__ int wi[2][32];
  __shared__ double red[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = p.n, V = p.V;
  if (*(volatile int32_t*)&p.st->inner_conv) return;
  double nb2 = 0.0;
  for (int s = tid; s < p.npad; s += SSCD_T) {
    rs[s] = (s < n) ? p.Rv[s] : 0.0;
    if (s < n) nb2 = fma(p.bhat[s], p.bhat[s], nb2);
  }
  if (p.t0 == 0) {
    nb2 = warp_sum(nb2);
    if (lane == 0) red[warp] = nb2;
    __syncthreads();
    double B2 = 0.0;
    for (int w = 0; w < 32; ++w) B2 += red[w];
    if (B2 == 0.0) {
      if (tid == 0) {
        p.st->inner_steps = 0;
        p.st->inner_conv = 1;
      }
      return;
    }
  }
  __syncthreads();
  if (p.jw) {   // weighted: j_t is data-independent, r_j read from the shared residual, no argmax
    const int64_t L = p.t1 - p.t0;
    int j0 = __ldcg(p.jw), j1 = (L > 1) ? __ldcg(p.jw + 1) : 0;
    double n0 = p.N[j0];
    for (int64_t u = 0; u < L; ++u) {
      const int j = j0;
      const double sc = rs[j] / n0;
      j0 = j1;
      n0 = p.N[j0];
      j1 = (u + 2 < L) ? __ldcg(p.jw + u + 2) : 0;
      __syncthreads();   // every thread has read r_j before any update of it
      if (p.Gd) {
        const double* grow = p.Gd + (int64_t)j * p.npad;
        for (int c = tid; c < n; c += SSCD_T) rs[c] = fma(-sc, __ldcg(grow + c), rs[c]);
      } else {
        for (int64_t e = p.gp[j] + tid; e < p.gp[j + 1]; e += SSCD_T) {
          const int c = p.gc[e];
          rs[c] = fma(-sc, p.gv[e], rs[c]);
        }
      }
      if (tid == 0) atomicAdd(p.Bv + j, sc);
      __syncthreads();
    }
    for (int s2 = tid; s2 < n; s2 += SSCD_T) p.Rv[s2] = rs[s2];
    return;
  }
  const uint32_t* mk = p.masks + tid;
  uint32_t allbits = 0;
  for (int v = 0; v < V; ++v)
    if (tid + v * SSCD_T < n) allbits |= 1u << v;
  uint32_t q0 = 0, q1 = 0;
  if (!p.all_members) {
    q0 = __ldcg(mk);
    q1 = (p.t1 - p.t0 > 1) ? __ldcg(mk + SSCD_T) : 0u;
  }
  for (int64_t t = p.t0; t < p.t1; ++t) {
    const int pb = (int)(t & 1);
    uint32_t inmask = allbits;
    if (!p.all_members) {
      inmask = q0;
      q0 = q1;
      const int64_t ahead = t - p.t0 + 2;
      q1 = (ahead < p.t1 - p.t0) ? __ldcg(mk + ahead * SSCD_T) : 0u;
    }
    double bv = -1.0, br = 0.0;
    int bi = INT_MAX;
    for (int v = 0; v < V; ++v) {
      if ((inmask >> v) & 1u) {
        const int s = tid + v * SSCD_T;
        const double r = rs[s];
        const double q = r * r;
        if (q > bv) {
          bv = q;
          bi = s;
          br = r;
        }
      }
    }
    // warp argmax by integer warp reductions (common.cuh); the winning thread records it
    if (bi == INT_MAX) bv = 0.0;
    const int wj = warp_argmax_redux(bv, bi);
    if (wj == INT_MAX ? lane == 0 : bi == wj) {
      wv[pb][warp] = bv;
      wi[pb][warp] = wj;
      wr[pb][warp] = br;
    }
    __syncthreads();
    const int j = warp_argmax_redux(wv[pb][lane], wi[pb][lane]);   // 32 warps: one entry per lane
    const double sc = wr[pb][(j % SSCD_T) >> 5] / p.N[j];
    // r -= sc A1bar_(j): the row's columns are distinct
    if (p.Gd) {
      const double* grow = p.Gd + (int64_t)j * p.npad;
      for (int c = tid; c < n; c += SSCD_T) rs[c] = fma(-sc, __ldcg(grow + c), rs[c]);
    } else {
      for (int64_t e = p.gp[j] + tid; e < p.gp[j + 1]; e += SSCD_T) {
        const int c = p.gc[e];
        rs[c] = fma(-sc, p.gv[e], rs[c]);
      }
    }
    if (tid == 0) atomicAdd(p.Bv + j, sc);   // fire-and-forget (program-ordered per address)
    __syncthreads();
  }
  for (int s = tid; s < n; s += SSCD_T) p.Rv[s] = rs[s];
}

// ---------------------------------------------------------------------------------------------
// SP-SCD for dense input with large n (the paper's n = 13000-15000): a 16-CTA cluster of 256
// threads, V = 4 coordinates of r per thread for n <= 16384 (V = 8 up to 32768), r in registers.
// Per step: masked local argmax -> warp butterfly -> CTA winner (barrier + warp reduction) -> the
// CTA winners (r_j^2, j, r_j, N_j) exchanged through DSMEM (destination-uniform st.async with
// mbarrier complete_tx, as in rk_rgs.cu) -> every CTA reduces the 16 candidates in the same order
// (ties to the smallest index) -> each thread updates its coordinates from row j of A1bar (HBM /
// L2, one coalesced pass over the row spread over 16 SMs instead of one).
constexpr int SCDC_C = 16;
constexpr int SCDC_T = 256;   // 8 warps per CTA: the per-step reductions are issue-bound, fewer warps win

struct ScdClParams {
  const double* G;        // A1bar, npad x npad
  int64_t npad;
  int n;
  const double* N;
  const double* bhat;
  double* Rv;             // [npad] state r
  double* Bv;             // [npad] state beta
  const uint32_t* masks;  // [t1 - t0][SCDC_C * SCDC_T], bit v <=> coordinate g + v * SCDC_C * SCDC_T
  int all_members;
  int64_t t0, t1;
  DevStatus* st;
};

template <int V>
__global__ void __cluster_dims__(SCDC_C, 1, 1) __launch_bounds__(SCDC_T, 1) scd_cluster_kernel(ScdClParams p) {
  constexpr int NTT = SCDC_C * SCDC_T;
  __shared__ double wv[2][32], wr[2][32], wn[2][32];
  __shared__ int wi[2][32];
  __shared__ __align__(16) double recv[2][SCDC_C][4];   // [source CTA] (r_j^2, r_j, j, 1 / N_j)
  __shared__ __align__(8) uint64_t rbar[2];
  __shared__ double red[32];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)cluster_ctarank();
  const int g = rank * SCDC_T + tid;
  const int n = p.n;
  if (*(volatile int32_t*)&p.st->inner_conv) return;
  if (p.t0 == 0) {   // b_hat = 0: beta = 0 after 0 steps (every CTA takes the same decision)
    double v = 0.0;
    for (int s = tid; s < n; s += SCDC_T) v = fma(p.bhat[s], p.bhat[s], v);
    v = warp_sum(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double B2 = 0.0;
    for (int w = 0; w < SCDC_T / 32; ++w) B2 += red[w];
    if (B2 == 0.0) {
      if (rank == 0 && tid == 0) {
        p.st->inner_steps = 0;
        p.st->inner_conv = 1;
      }
      return;
    }
  }
  double r[V], nj[V], beta[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int s = g + v * NTT;
    r[v] = (s < n) ? p.Rv[s] : 0.0;
    nj[v] = (s < n) ? 1.0 / p.N[s] : 1.0;   // reciprocal: the step length is one multiply (as scd_chunk_kernel)
    beta[v] = (s < n) ? p.Bv[s] : 0.0;
  }
  uint32_t allbits = 0;
#pragma unroll
  for (int v = 0; v < V; ++v)
    if (g + v * NTT < n) allbits |= 1u << v;
  if (tid == 0) {
    mbar_init(&rbar[0], 1);
    mbar_init(&rbar[1], 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(&rbar[0], SCDC_C * 32);
    mbar_arrive_expect_tx(&rbar[1], SCDC_C * 32);
  }
  __syncthreads();
  cluster_sync_all();
  const uint32_t* mk = p.masks + g;
  const int64_t L = p.t1 - p.t0;
  uint32_t q0 = 0, q1 = 0, q2 = 0, q3 = 0;
  if (!p.all_members) {
    q0 = (0 < L) ? __ldcg(mk) : 0u;
    q1 = (1 < L) ? __ldcg(mk + NTT) : 0u;
    q2 = (2 < L) ? __ldcg(mk + 2 * NTT) : 0u;
    q3 = (3 < L) ? __ldcg(mk + 3 * NTT) : 0u;
  }
  for (int64_t t = p.t0; t < p.t1; ++t) {
    const int pb = (int)(t & 1);
    uint32_t inmask = allbits;
    if (!p.all_members) {
      inmask = q0;
      q0 = q1;
      q1 = q2;
      q2 = q3;
      const int64_t ahead = t - p.t0 + 4;
      q3 = (ahead < L) ? __ldcg(mk + ahead * NTT) : 0u;
    }
    double bv = -1.0, br = 0.0, bn = 1.0;
    int bi = INT_MAX;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const double q = r[v] * r[v];
      if (((inmask >> v) & 1u) && q > bv) {
        bv = q;
        bi = g + v * NTT;
        br = r[v];
        bn = nj[v];
      }
    }
    // warp argmax by integer warp reductions (common.cuh); the winning thread records it
    if (bi == INT_MAX) bv = 0.0;
    const int wj = warp_argmax_redux(bv, bi);
    if (wj == INT_MAX ? lane == 0 : bi == wj) {
      wv[pb][warp] = bv;
      wi[pb][warp] = wj;
      wr[pb][warp] = br;
      wn[pb][warp] = bn;
    }
    __syncthreads();
    if (warp == 0) {   // CTA winner, one message to every CTA
      if (lane == 0 && t > p.t0)   // every warp has read step t-1's messages: re-arm that buffer for t+1
        mbar_arrive_expect_tx(&rbar[pb ^ 1], SCDC_C * 32);
      const double cv0 = (lane < SCDC_T / 32) ? wv[pb][lane] : 0.0;
      const int ci0 = warp_argmax_redux(cv0, (lane < SCDC_T / 32) ? wi[pb][lane] : INT_MAX);
      const int ww = (ci0 == INT_MAX) ? 0 : (((ci0 % NTT) - rank * SCDC_T) >> 5);   // its warp
      const double cv = (ci0 == INT_MAX) ? 0.0 : wv[pb][ww];
      const double cr = wr[pb][ww], cn0 = (ci0 == INT_MAX) ? 1.0 : wn[pb][ww];
      // lane 0 carries (r_j^2, r_j), lane 1 carries (j, 1 / N_j): 32 bytes per destination
      const double m0 = (lane == 0) ? cv : (double)ci0;
      const double m1 = (lane == 0) ? cr : cn0;
      const uint32_t la = smem_u32(&recv[pb][rank][2 * (lane & 1)]);
      const uint32_t lb = smem_u32(&rbar[pb]);
      __syncwarp();   // the re-arm precedes this step's sends (the peers' step t+1 messages follow them)
      if (lane < 2)
#pragma unroll
        for (int c = 0; c < SCDC_C; ++c) st_async_v2f64(map_shared_rank(la, (uint32_t)c), m0, m1, map_shared_rank(lb, (uint32_t)c));
    }
    // every warp waits for the 16 CTA winners and reduces them the same way (no second CTA barrier):
    // lane c holds candidate c, ties to the smallest index
    mbar_wait_cluster(&rbar[pb], (uint32_t)((t - p.t0) >> 1) & 1u);
    const double xv = (lane < SCDC_C) ? recv[pb][lane][0] : 0.0;
    const int j = warp_argmax_redux(xv, (lane < SCDC_C) ? (int)recv[pb][lane][2] : INT_MAX);
    const int wc = (j % NTT) / SCDC_T;   // the CTA that owns coordinate j
    const double sc = recv[pb][wc][1] * recv[pb][wc][3];   // r_j / N_j as r_j * (1 / N_j)
    const double* grow = p.G + (int64_t)j * p.npad;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int s = g + v * NTT;
      if (s < n) r[v] = fma(-sc, __ldg(grow + s), r[v]);
      if (s == j) beta[v] += sc;   // registers: no dependent global load on the step chain
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int s = g + v * NTT;
    if (s < n) {
      p.Rv[s] = r[v];
      p.Bv[s] = beta[v];
    }
  }
  cluster_sync_all();   // no CTA exits while a peer may still write into its shared memory
}

__global__ void __launch_bounds__(256) sparse_scd_check_kernel(const double* __restrict__ Gd, int64_t npad,
                                                               const int64_t* __restrict__ gp, const int32_t* __restrict__ gc,
                                                               const double* __restrict__ gv, int64_t n,
                                                               const double* __restrict__ bhat,
                                                               const double* __restrict__ Bv, double* __restrict__ Rv,
                                                               double* __restrict__ rtmp, double* __restrict__ red,
                                                               double inner_tol, int64_t t_now, DevStatus* st) {
  cg::grid_group grid = cg::this_grid();
  if (*(volatile int32_t*)&st->inner_conv) return;
  __shared__ double sr[8][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double a = 0.0, b = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * 8 + warp; j < n; j += (int64_t)gridDim.x * 8) {
    double s = 0.0;
    if (Gd) {
      for (int64_t c = lane; c < n; c += 32) s = fma(Gd[j * npad + c], Bv[c], s);
    } else {
      for (int64_t e = gp[j] + lane; e < gp[j + 1]; e += 32) s = fma(gv[e], Bv[gc[e]], s);
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
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
      Rv[j] = rtmp[j];
  }
}

int sparse_scd_inner(Handle& h, const double* bhat, double* beta, uint64_t seed, int64_t k, int64_t max_inner,
                     int64_t check_every, double inner_tol, int alpha_mode, int alpha_k, int weighted,
                     int64_t* steps_out) {
  // CSR input: A1bar compacted to CSR; dense input with large n: the dense A1bar rows
  int rc = h.sparse ? sparse_gram_csr(h) : build_gram(h);
  if (rc) return rc;
  const cudaStream_t st = h.stream;
  const int64_t ce = check_every > 0 ? check_every : h.n;
  const int V = (int)((h.n + SSCD_T - 1) / SSCD_T);
  if (V > 32 || (size_t)h.npad * 8 > 227 * 1024) {
    set_error("sparse SP-SCD: n too large for the shared-memory residual");
    return ILS_ERR_UNSUPPORTED;
  }
  const int64_t chunk_cap = (max_inner < ce) ? max_inner : ce;
  // the 16-CTA cluster kernel over dense A1bar rows (dense input with large n; CSR input too: its
  // dense A1bar is resident, built for the SP Cholesky and compacted from), up to 8 coordinates of r
  // per thread in registers (c3: 2.5 us per step against 5.2 for the one-CTA shared-residual kernel)
  const char* ecl = getenv("ILS_SCD_CLUSTER");
  const bool cl = !weighted && h.G && h.n <= 8 * SCDC_C * SCDC_T && !(ecl && ecl[0] == '0');
  const int Vc = (h.n <= 4 * SCDC_C * SCDC_T) ? 4 : 8;
  const int mask_threads = cl ? SCDC_C * SCDC_T : SSCD_T;
  const size_t need = ((size_t)3 * h.npad + 2 * (size_t)h.num_sms) * sizeof(double) +
                      (size_t)chunk_cap * mask_threads * sizeof(uint32_t);
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
  ILS_CU(cudaMemcpyAsync(Rv, bhat, h.n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  ILS_CU(cudaMemsetAsync(&h.dstat->inner_conv, 0, sizeof(int32_t), st));
  ILS_CU(cudaMemsetAsync(&h.dstat->inner_steps, 0, sizeof(int64_t), st));
  SpScdParams prm{};
  prm.Gd = h.sparse ? nullptr : h.G;
  prm.gp = h.gcsr_ptr;
  prm.gc = h.gcsr_col;
  prm.gv = h.gcsr_val;
  prm.n = (int)h.n;
  prm.npad = h.npad;
  prm.N = h.N;
  prm.bhat = bhat;
  prm.Rv = Rv;
  prm.Bv = Bv;
  prm.masks = masks;
  prm.V = V;
  prm.all_members = ((alpha_mode & 0xF) == ILS_ALPHA_FIXED && alpha_k >= h.n) ? 1 : 0;
  prm.jw = weighted ? reinterpret_cast<const int32_t*>(masks) : nullptr;   // chunk_cap <= the mask space
  prm.st = h.dstat;
  const size_t smem = (size_t)h.npad * sizeof(double);
  ILS_CU(cudaFuncSetAttribute(sparse_scd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t* gp = h.gcsr_ptr;
  const int32_t* gc = h.gcsr_col;
  const double* gv = h.gcsr_val;
  const double* Gd = prm.Gd;
  const int64_t npd = h.npad;
  const int64_t nn = h.n;
  DevStatus* dst = h.dstat;
  constexpr int kBatch = 8;
  ILS_CU(cudaEventRecord(h.evk0, st));
  int64_t t = 0;
  int pending = 0;
  while (t < max_inner) {
    const int64_t t1 = (t + ce < max_inner) ? t + ce : max_inner;
    if (weighted) {
      rcd_index_kernel<<<(unsigned)((t1 - t + 255) / 256), 256, 0, st>>>(seed, (uint32_t)k, t, t1, (int)h.n, h.S,
                                                                           reinterpret_cast<int32_t*>(masks));
      ILS_LAUNCHED("rcd_index_kernel");
    } else if (!prm.all_members &&
               (rc = scd_masks(h, seed, k, t, t1, alpha_mode, alpha_k, mask_threads, cl ? Vc : V, masks))) {
      return rc;
    }
    prm.t0 = t;
    prm.t1 = t1;
    if (cl) {
      ScdClParams cp{};
      cp.G = h.G;
      cp.npad = h.npad;
      cp.n = (int)h.n;
      cp.N = h.N;
      cp.bhat = bhat;
      cp.Rv = Rv;
      cp.Bv = Bv;
      cp.masks = masks;
      cp.all_members = prm.all_members;
      cp.t0 = t;
      cp.t1 = t1;
      cp.st = h.dstat;
      if (Vc == 4) {
        ILS_CU(cudaFuncSetAttribute(scd_cluster_kernel<4>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        scd_cluster_kernel<4><<<SCDC_C, SCDC_T, 0, st>>>(cp);
      } else {
        ILS_CU(cudaFuncSetAttribute(scd_cluster_kernel<8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        scd_cluster_kernel<8><<<SCDC_C, SCDC_T, 0, st>>>(cp);
      }
      ILS_LAUNCHED("scd_cluster_kernel");
    } else {
      sparse_scd_kernel<<<1, SSCD_T, smem, st>>>(prm);
      ILS_LAUNCHED("sparse_scd_kernel");
    }
    t = t1;
    if (t % ce == 0) {
      double itol = inner_tol;
      int64_t tn = t;
      void* args[] = {(void*)&Gd, (void*)&npd, (void*)&gp, (void*)&gc, (void*)&gv, (void*)&nn, (void*)&bhat,
                      (void*)&Bv, (void*)&Rv, (void*)&rtmp, (void*)&red, (void*)&itol, (void*)&tn, (void*)&dst};
      ILS_CU(cudaLaunchCooperativeKernel((void*)sparse_scd_check_kernel, dim3(h.num_sms), dim3(256), args, 0, st));
      ILS_LAUNCHED("sparse_scd_check_kernel");
    }
    if (++pending == kBatch || t >= max_inner) {
      ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
      ILS_CU(cudaStreamSynchronize(st));
      pending = 0;
      if (h.hstat->inner_conv) break;
    }
  }
  ILS_CU(cudaEventRecord(h.evk1, st));
  ILS_CU(cudaMemsetAsync(beta, 0, h.npad * sizeof(double), st));
  ILS_CU(cudaMemcpyAsync(beta, Bv, h.n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  ILS_CU(cudaMemcpyAsync(h.hstat, h.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
  ILS_CU(cudaStreamSynchronize(st));
  const int64_t steps = h.hstat->inner_conv ? h.hstat->inner_steps : max_inner;
  if (steps_out) *steps_out = steps;
  const double row = h.sparse ? 12.0 * (double)h.gnnz / (double)h.n : 8.0 * (double)h.n;
  hot_account(h, 2, (double)steps * row + (double)(steps / ce) * row * (double)h.n, (steps + ce - 1) / ce);
  return ILS_OK;
}

}  // namespace ils
