// ils_internal.h -- host-side internals of libils (handle layout, launchers).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/ils.h"

namespace ils {

constexpr int kPad = 64;  // all dense dimensions padded to multiples of 64

inline int64_t roundup(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// Device-side scalars written by kernels and read back once per call.
struct DevStatus {
  int32_t flag_stop;       // outer stop decided
  int32_t flag_err;        // Cholesky breakdown etc.
  int64_t iters;           // outer iterations done
  double metric;           // last stop metric
  int64_t inner_steps;     // inner steps of the last inner solve
  int32_t inner_conv;      // inner solve met its tolerance
  int32_t flag_nonfinite;  // ingest: a non-finite entry in A or b
  uint32_t gbar_count;     // software grid barrier of the SP row-stream kernel: arrivals since the launch (zeroed by the host before every launch)
  uint32_t gbar_gen;       // (unused; keeps the layout)
};

struct ils_comm_impl {
  void* nccl = nullptr;   // ncclComm_t
  int nranks = 1, rank = 0;
};

struct Handle {
  int64_t p = 0, q = 0, n = 0, m = 0, batch = 1;
  int64_t npad = 0, ppad = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;

  // dense single-instance layouts
  double* Arm = nullptr;    // (m + 64) x npad row-major, zero padded  [A1; A2]
  double* A1T = nullptr;    // npad x ppad: row j = column j of A1 (column-major A1)
  double* b = nullptr;      // m (+64 zero tail)
  double* N = nullptr;      // n column norms ||A1_(j)||^2 (sequential order)
  uint64_t* S = nullptr;    // n weight prefix sums
  double* a1tb1 = nullptr;  // npad  A1^T b1
  double* ajb = nullptr;    // npad  A^T J b (lazy)

  // lazy SP / SCD precompute
  double* G = nullptr;      // npad x npad  A1^T A1 (full symmetric, identity padding)
  double* L = nullptr;      // npad x npad  Cholesky workspace
  double* Z = nullptr;      // npad x npad  L^{-1} (lower, zero upper)
  double* P = nullptr;      // npad x npad  (A1^T A1)^{-1}
  bool have_gram = false, have_P = false;
  bool use_zt = false;      // P applied as Z^T (Z c) (n >= 8192): Z holds complete inverses only of the
                            // recursion's diagonal blocks of <= zt_th 64-blocks; above them L21 comes from
                            // a recursive triangular solve and Z is applied through L (dla.cu)
  int64_t zt_th = 64;       // largest node (in 64-blocks) whose inverse is formed whole (ILS_ZT_TH)
  // paper-literal precompute (sp_form = 2): A2bar = A2^T A2, B = P A2bar, c0 = P A^T J b
  double* A2bar = nullptr;
  double* Bmat = nullptr;
  double* lit_vec = nullptr;   // [2][npad]: A^T J b, c0
  bool have_a2bar = false, have_B = false;

  // workspace
  double* part = nullptr;   // partial sums [grid][npad]
  int64_t part_rows = 0;
  double* wsA = nullptr;    // GEMM split-K workspace
  size_t wsA_bytes = 0;
  double* vec = nullptr;    // 8 x npad scratch vectors
  double* rk_state = nullptr;  // SP-RK-RGS chunk state: w, r, az [ppad] each, z [npad]
  void* scd_ws = nullptr;      // SP-SCD chunk state r, beta, r_tmp [npad], reductions, membership masks
  size_t scd_ws_bytes = 0;
  ils_comm_impl* comm = nullptr;   // row-sharded handle (comm.cu): row sums are all-reduced
  bool large = false;          // dense n > 8192 (or ILS_FORCE_LARGE=1): two-pass SP RHS/check, global-z RK, smem-r SCD
  bool rk_single_step = false; // ILS_RK_SINGLE_STEP env: force the one-step-per-reduction RK-RGS kernel
  double* red = nullptr;    // reduction scratch [grid * 4]
  DevStatus* dstat = nullptr;
  DevStatus* hstat = nullptr;  // pinned host mirror

  // CSR input (BASELINE.json configs[3])
  bool sparse = false;
  int64_t nnz = 0, nnz1 = 0;
  double a1_row_sq = 0.0;   // sum over A1 rows of nnz_i^2
  int64_t maxcol1 = -1;     // longest A1 column (CSC entries), computed on first use
  int64_t* rp = nullptr;    // [m+1]
  int32_t* ci = nullptr;    // [nnz]
  double* va = nullptr;     // [nnz]
  int64_t* cp1 = nullptr;   // CSC of A1: [n+1], rows sorted
  int32_t* cr1 = nullptr;
  double* cv1 = nullptr;
  int64_t* cp2 = nullptr;   // CSC of A2 (row indices relative to p)
  int32_t* cr2 = nullptr;
  double* cv2 = nullptr;
  double* sp_y = nullptr;   // [m] row-pass scratch
  int32_t* sp_split = nullptr;   // [n][17]: CSC entry offsets of each A1 column at the 16 row-slice bounds
  int64_t* gcsr_ptr = nullptr;   // A1bar compacted to CSR (SP-SCD)
  int32_t* gcsr_col = nullptr;
  double* gcsr_val = nullptr;
  int64_t gnnz = 0;
  size_t rk_state_words = 0;

  // batched layout
  double* Ab = nullptr;     // [batch][m][n]
  double* bb = nullptr;     // [batch][m]

  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t evk0 = nullptr, evk1 = nullptr;   // per-launch timing of the hot kernels
  // SP-SCD: the membership masks of chunk i + 1 are formed on an auxiliary stream while chunk i runs
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_mask[2] = {nullptr, nullptr}, ev_chunk[2] = {nullptr, nullptr};
  double hot_ms[4] = {0, 0, 0, 0};
  double hot_work[4] = {0, 0, 0, 0};
  int64_t hot_n[4] = {0, 0, 0, 0};
};

// Accumulate the device time between h.evk0 and h.evk1 (already recorded) into class c.
// launches: hot-kernel launches covered by [evk0, evk1] (RK/SCD: chunk kernels, each with its check)
void hot_account(Handle& h, int c, double work, int64_t launches = 1);

// error plumbing
void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
void count_launch(int64_t k = 1);
int64_t launches_now();

#define ILS_CU(call)                                       \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return ::ils::cuda_fail(e_, #call); \
  } while (0)

#define ILS_LAUNCHED(what)                                         \
  do {                                                             \
    ::ils::count_launch();                                         \
    cudaError_t e_ = cudaGetLastError();                           \
    if (e_ != cudaSuccess) return ::ils::cuda_fail(e_, what);      \
  } while (0)

// ---- launchers (each returns ILS_OK or a negative status) ----
// ingest.cu
int launch_transpose_a1(Handle& h);
int launch_ingest_dense(Handle& h, const double* A, int64_t lda, const double* b, int32_t* flag);
int launch_colnorms(Handle& h);
int launch_weights(Handle& h, int32_t* d_zero_flag);
int launch_gemv_rows(const double* X, int64_t ldx, int64_t rows, int64_t cols, const double* v,
                     double* y, double alpha, const double* yadd, cudaStream_t st);
int launch_gemv_cols(const double* X, int64_t ldx, int64_t rows, int64_t cols, const double* v,
                     double* y, double alpha, const double* yadd, cudaStream_t st);

// dla.cu (dense linear algebra on DMMA)
// C[MxN] = alpha * sum_k opA(i,k) opB(j,k) + beta*C ; opA(i,k)=A[i*lda+k] (a_mc=0) or A[k*lda+i] (a_mc=1)
//                                                    opB(j,k)=B[j*ldb+k] (b_nc=0) or B[k*ldb+j] (b_nc=1)
int gemm_dmma(Handle& h, bool a_mc, bool b_nc, int64_t M, int64_t N, int64_t K, double alpha,
              const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
              int64_t ldc, bool lower_only, int splits);
int mirror_lower(Handle& h, double* C, int64_t ld, int64_t n, int64_t n_real);
// Cholesky of the lower triangle of L (npad x npad) in place, Z = L^{-1}. flag_err set on breakdown.
int cholesky_inverse(Handle& h, double* L, double* Z, int64_t npad, bool full_z);
int build_gram(Handle& h);      // G = A1^T A1
int build_inverse(Handle& h);   // L, Z, P from G
int build_a2bar(Handle& h);     // A2bar = A2^T A2 and A^T J b (dense)
int build_explicit_b(Handle& h);   // B = P A2bar, c0 = P A^T J b (dense)

// sp.cu
int sp_run(Handle& h, const double* x0_dev, double* x_dev, double tol, int64_t max_iter, int stop,
           const double* xref_dev, int sp_form, double* x_hist_dev, bool rhs_only, double* rhs_out,
           int64_t* iters_out, double* metric_out, int* conv_out);
int full_residual(Handle& h, const double* x_dev, double* g_out);  // g = A^T J (b - A x)
// SP-RK-RGS inner check (full grid): az = A1 z, g = A1^T az - b_hat, stop flag / r = w - az
int rk_check(Handle& h, const double* z, const double* bhat, const double* w, double* r, double* az,
             double inner_tol, int64_t t_now);

// rk_rgs.cu
int rk_rgs_inner(Handle& h, const double* bhat, double* z, uint64_t seed, int64_t k, int64_t max_inner,
                 int64_t check_every, double inner_tol, int64_t* steps_out);
int rk_indices(Handle& h, uint64_t seed, int64_t k, int64_t t0, int64_t count, int32_t* j1, int32_t* j2);

// scd.cu
int scd_inner(Handle& h, const double* bhat, double* beta, uint64_t seed, int64_t k, int64_t max_inner,
              int64_t check_every, double inner_tol, int alpha_mode, int alpha_k, int weighted,
              int64_t* steps_out);
int scd_subset_mask(int64_t n, uint64_t seed, int64_t k, int64_t t, int alpha_mode, int alpha_k,
                    int32_t* alpha_dev, uint8_t* mask_dev, cudaStream_t st);

// small vector kernels (sp.cu)
int stop_metric(Handle& h, const double* x, const double* xref, double* out_dev);

// sparse.cu (CSR input)
int sparse_ingest(Handle& h, int32_t* d_flag, bool* ok);
int sparse_gram(Handle& h, double* G, bool subtract_a2);
int sparse_a2bar(Handle& h, double* A2bar, double* ajb);   // CSR: A2^T A2 (dense rows), A^T J b
int sparse_rhs(Handle& h, const double* x, double* c, int full);
int gemv_p(Handle& h, const double* c, double* x);
int sparse_rk_inner(Handle& h, const double* bhat, double* z, uint64_t seed, int64_t k, int64_t max_inner,
                    int64_t check_every, double inner_tol, int64_t* steps_out);
int sparse_scd_inner(Handle& h, const double* bhat, double* beta, uint64_t seed, int64_t k, int64_t max_inner,
                     int64_t check_every, double inner_tol, int alpha_mode, int alpha_k, int weighted, int64_t* steps_out);
// scd.cu: membership masks of steps [t0, t1) for NT threads x V coordinates
int scd_masks(Handle& h, uint64_t seed, int64_t k, int64_t t0, int64_t t1, int alpha_mode, int alpha_k, int NT, int V,
              uint32_t* masks);

// comm.cu (row-sharded handles): in-place sum over ranks on h.stream (no-op when unsharded)
int allreduce_sum(Handle& h, double* buf, int64_t count);

// large.cu (dense n > 8192)
int dense_rhs_twopass(Handle& h, const double* x, double* c, int full);
int rk_check_twopass(Handle& h, const double* z, const double* bhat, const double* w, double* r, double* az,
                     double inner_tol, int64_t t_now);
int vec_add(Handle& h, double* x, const double* y, int64_t n);
int launch_cols(const double* X, int64_t ldx, int64_t rows, int64_t cols, const double* y, double alpha,
                const double* base, double* c, int tri_lower, cudaStream_t st);
int launch_tri_rows(const double* T, int64_t ld, int64_t m, const double* c, double* y, cudaStream_t st);
int zc_apply_tree(Handle& h, const double* c, double* x);

// batched.cu
int batched_solve(Handle& h, int method, const double* x0, double* x, double tol, int64_t max_iter,
                  const ils_opts& o, int64_t* inst_iters_dev, int32_t* inst_status_dev);

}  // namespace ils

// the public opaque communicator type (include/ils.h) is the internal one
struct ils_comm_s : public ils::ils_comm_impl {};

