/*
 * ils.h -- C ABI of libils.so: B200 (sm_100a) fp64 solvers for the indefinite least
 * squares (ILS) problem of Zhang & Li, arXiv 2203.15340 ("Splitting-based randomized
 * iterative methods for solving indefinite least squares problem").
 *
 *     min_x (b - A x)^T J (b - A x),  J = diag(I_p, -I_q),  A = [A1; A2]
 *
 * Entry points (BASELINE.json north_star):
 *   ils_create     ingest A, b (layout, column norms, sampling tables, A1^T b1)
 *   ils_sp_solve   Alg. 1, SP:         x_{k+1} = (A1^T A1)^{-1} (A2^T A2 x_k + A^T J b)
 *   ils_rk_solve   Alg. 2, SP-RK-RGS:  RK steps on A1^T w = b_hat interleaved with
 *                                      RGS steps on A1 z = w
 *   ils_rgs_solve  Alg. 5, SP-SCD (and SP-RCD, the j1 = j2 reduction of Alg. 2)
 *   ils_destroy    free the handle
 * plus helpers for the reference solution, RR, diagnostics and replay checks.
 *
 * Conventions (all entry points)
 *   - fp64 throughout. Row-major A (m x n, leading dimension lda >= n), m = p + q.
 *   - Pointers may be HOST or DEVICE memory; the library detects which
 *     (cudaPointerGetAttributes). Host inputs are copied to the device inside the call;
 *     host outputs are written back before the call returns.
 *   - Input arrays are borrowed for the duration of the call only; ils_create makes its
 *     own device copies (it never keeps a caller pointer).
 *   - All device work runs on ext->stream (default stream if NULL). Every call is
 *     synchronous with respect to its return value and report.
 *   - Deterministic: the same inputs and seed give bitwise-identical outputs on the same
 *     GPU (fixed-order reductions, no floating-point atomics).
 *   - Negative return codes are errors and leave outputs unspecified; ILS_NOT_CONVERGED
 *     (= 1) is not an error: x holds the last iterate and the report is filled.
 *   - One handle per host thread.
 *
 * Index stream (normative; the oracle replays it from this text)
 *   Philox4x32-10 (Salmon et al., SC'11): counter (c0,c1,c2,c3) = (t mod 2^32, t >> 32, k, tag),
 *   key = (seed mod 2^32, seed >> 32); t = inner step (0-based), k = outer iteration (0-based).
 *   Output words x0..x3.
 *   Column weights: N_j = sum_{i=0}^{p-1} A1[i,j]^2 accumulated sequentially in i with
 *   each square rounded before the add (no FMA); W_j = max(1, floor(N_j / max_i N_i * 2^32));
 *   S_j = W_0 + ... + W_j (uint64). Weighted draw from a 64-bit U: v = floor(U * S_{n-1} / 2^64),
 *   j = min{ j : S_j > v }. This realises Pr(j) = ||A1_(j)||^2 / ||A1||_F^2 (PAPER.md:199-202,
 *   :227-230) to within 2^-32 relative.
 *   SP-RK-RGS step t (tag 1): j1 from U = x1:x0 (x1 high), j2 from U = x3:x2.
 *   SP-SCD step t: tag 2 draw A, tag 3 draw B, tag 4 draw C.
 *     alpha_t = 1 + floor(A.x0 * n / 2^32) (uniform on {1..n}) or min(alpha_k, n).
 *     Round keys K0..K7 = A.x1, A.x2, A.x3, B.x0, B.x1, B.x2, B.x3, C.x0.
 *     pi = 8-round balanced Feistel permutation of [0, 2^(2h)), h = ceil(ceil(log2 n) / 2),
 *     round (L, R) -> (R, L xor F(R, K_r)), F(R, K) = mix32(R xor K) & (2^h - 1),
 *     mix32(x): x *= 0x85EBCA6B; x ^= x >> 13; x *= 0xC2B2AE35; x ^= x >> 16 (mod 2^32),
 *     value = (L << h) | R, cycle-walked (re-encrypted) until < n; pi = identity for n = 1.
 *     tau_t = { pi(0), ..., pi(alpha_t - 1) } (alpha_mode | ILS_SUBSET_EXACT: see
 *     below); j_t = argmax_{s in tau_t} r_s^2,
 *     ties to the smallest s.
 *   SP-RCD step t (weighted = 1): tag 6, j from U = x1:x0 with the column weights.
 *   Batched instance i uses seed + i.
 *
 * Inner stopping rule (the paper says "until convergence"; R2):
 *   the inner solve of outer iteration k starts from zero. If ||b_hat|| = 0
 *   it returns 0 after 0 steps. After every check_every steps: SP-RK-RGS evaluates
 *   g = A1^T A1 z - b_hat (as A1bar z - b_hat where A1bar = A1^T A1 is resident, else as
 *   A1^T (A1 z) - b_hat: the same vector up to rounding) and stops if ||g||_2 <= inner_tol
 *   ||b_hat||_2; the check reads z only -- the residual r = w - A1 z is maintained by the steps
 *   and never recomputed. SP-SCD recomputes r = b_hat - A1bar beta and stops if
 *   ||r||_2 <= inner_tol ||b_hat||_2. The solve also stops after max_inner steps.
 * Outer stopping rule: after forming x_{k+1}: STOP_XREF ||x_{k+1} - x_ref||_2 <= tol ||x_ref||_2
 *   (BASELINE.json), STOP_RR RR(x_{k+1}) < tol with RR = ||A^T J (A x - b)||^2 / ||A^T J b||^2
 *   (PAPER.md:651-653), STOP_NONE never (fixed horizon). outer_iters counts completed updates.
 */
#ifndef ILS_H_
#define ILS_H_

#include <stdint.h>

#if defined(__GNUC__)
#define ILS_API __attribute__((visibility("default")))
#else
#define ILS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ils_handle_s* ils_handle;
typedef struct ils_comm_s* ils_comm;   /* NCCL communicator for row-sharded handles */
#define ILS_COMM_ID_BYTES 128

enum {
  ILS_OK = 0,
  ILS_NOT_CONVERGED = 1,     /* non-fatal: iteration cap reached, x = last iterate */
  ILS_ERR_ARG = -1,          /* NULL / bad option / non-finite entry / A^T J b = 0 under STOP_RR */
  ILS_ERR_SHAPE = -2,        /* p < 1, q < 0, n < 1, p < n (A1^T A1 must be SPD), lda < n */
  ILS_ERR_ZERO_COLUMN = -3,  /* some column of A1 has N_j = 0 (RK/RGS probability undefined) */
  ILS_ERR_NOT_SPD = -4,      /* Cholesky breakdown of A1^T A1 or of A^T J A (condition 1.3) */
  ILS_ERR_CUDA = -5,         /* CUDA runtime error; ils_last_error() has the message */
  ILS_ERR_NOMEM = -6,        /* device allocation failed */
  ILS_ERR_UNSUPPORTED = -7   /* option combination not implemented */
};

enum { ILS_STOP_XREF = 0, ILS_STOP_RR = 1, ILS_STOP_NONE = 2 };
enum { ILS_FORMAT_DENSE = 0, ILS_FORMAT_CSR = 1 };
enum { ILS_ALPHA_UNIFORM = 0, ILS_ALPHA_FIXED = 1 };
/* OR into alpha_mode: exact uniform subsets instead of the Feistel prefix (the
 * study of reading R9 / Q9): coordinate s at SP-SCD step t gets the key u_s = word (s mod 4) of the
 * Philox draw with counter (t_lo, t_hi, k, 7 + 256 * floor(s / 4)); tau_t = the alpha_t coordinates
 * with the smallest (u_s, s) in lexicographic order. The keys are i.i.d. uniform, so every subset
 * of size alpha_t has probability 1 / C(n, alpha_t) up to equal keys (probability < n^2 / 2^33 per
 * step). Single-instance handles only (batched: ILS_ERR_UNSUPPORTED). */
#define ILS_SUBSET_EXACT 0x10

/* Optional creation extras; NULL = dense, batch 1, lda = n, default stream. */
typedef struct {
  int32_t format;            /* ILS_FORMAT_DENSE or ILS_FORMAT_CSR (BASELINE.json configs[3]) */
  int64_t batch;             /* >= 1. batch > 1: A is [batch][m][lda], b is [batch][m]; one CTA per instance */
  int64_t lda;               /* row stride of A in elements (0 = n) */
  void* stream;              /* cudaStream_t */
  /* ILS_FORMAT_CSR (batch 1): A points to the nnz values; rows 0..p-1 are A1, p..m-1 are A2. */
  const int64_t* row_ptr;    /* [m + 1], row_ptr[0] = 0, non-decreasing, row_ptr[m] = nnz */
  const int32_t* col_idx;    /* [nnz], 0 <= col < n, strictly increasing within each row */
  int64_t nnz;
  /* Row sharding (dense, batch 1): A and b hold THIS rank's row block
   * [A1_r; A2_r] (p = p_r >= 1 rows of A1, q = q_r >= 0 rows of A2; the global p >= n is the
   * caller's to guarantee). Row sums (A1^T A1, column norms, c_k, A^T J (b - A x)) are reduced
   * over comm with NCCL all-reduce; every rank then holds identical iterates. Supported:
   * ils_sp_solve (sp_form 0/1, all stop rules), ils_rgs_solve (SP-SCD/RCD; the inner solve runs
   * replicated), ils_relative_residual. ils_rk_solve (needs whole columns of A1), sp_form 2 and
   * ils_direct_solve return ILS_ERR_UNSUPPORTED. NULL = unsharded. Borrowed until ils_destroy. */
  ils_comm comm;
} ils_ext;

/* Solver options; ils_default_opts() fills the defaults given in brackets. */
typedef struct {
  int32_t stop;              /* [ILS_STOP_XREF] */
  const double* x_ref;       /* [NULL] reference solution ([batch][n]) for ILS_STOP_XREF */
  double inner_tol;          /* [1e-12] inner stopping tolerance (relative) */
  int64_t max_inner;         /* [100000] cap on inner steps per outer iteration */
  int64_t check_every;       /* [0 = n] inner check period */
  uint64_t seed;             /* [0] Philox key */
  int32_t alpha_mode;        /* [ILS_ALPHA_UNIFORM] SCD alpha policy */
  int32_t alpha_k;           /* [1] alpha for ILS_ALPHA_FIXED */
  int32_t weighted;          /* [0] ils_rgs_solve: 1 = SP-RCD (alpha = 1, column-norm weights) */
  int32_t sp_form;           /* [0] 0: x = P (A1^T b1 + A2^T (A2 x - b2)) (Sec23); 1: x += P A^T J (b - A x);
                                2: the paper's literal layout: SP x = B x + c with B = P A2^T A2, c = P A^T J b
                                formed once (Alg. 1 steps 2-6); RK/RGS b_hat = A2bar x + A^T J b
                                with A2bar = A2^T A2 formed once (Alg. 2 steps 2-5, Alg. 5 steps 2-4). CSR input:
                                A2bar from the CSC of A2 (dense rows, n <= 29000); SP's B = P A2bar needs the
                                explicit P, so SP at n >= 8192 (dense or CSR) returns ILS_ERR_UNSUPPORTED.
                                3 (ILS_SP_FORM_AUTO): 2 if its precompute pays off over expected_outer outer
                                steps, else 0 (include/ils.h "Automatic form"). */
  double* x_hist;            /* [NULL] optional [max_iter][n] record of every outer iterate (batch 1) */
  int64_t* inner_hist;       /* [NULL] optional [max_iter] inner step count per outer iteration */
  int64_t expected_outer;    /* [0] outer steps the caller expects, for ILS_SP_FORM_AUTO (0: min(max_iter, 32)) */
} ils_opts;

/* Automatic form (sp_form = ILS_SP_FORM_AUTO, PAPER.md:134-139 vs :291, :689): the literal layout
 * (2) replaces the per-outer-step stream of A2 (8 q (n + 1) bytes) by an n x n GEMV (8 n^2 bytes;
 * SP already applies P, so its per-step saving is the full A2 stream) at the price of a one-time
 * DMMA precompute: A2bar = A2^T A2 (q n (n + 1) flops) and, for SP, B = P A2bar (2 n^3 flops).
 * It is chosen iff K * saved_bytes / 6.0e12 B/s > precompute_flops / 3.0e13 flop/s with
 * K = expected_outer (the measured HBM copy rate and DMMA DGEMM rate of this B200 pool, rounded
 * down). CSR input, n > 8192 and row-sharded handles always take form 0. The report's
 * sp_form_used records the choice. */
#define ILS_SP_FORM_AUTO 3

typedef struct {
  int64_t outer_iters;       /* completed outer updates (max over instances when batched) */
  int64_t inner_iters_total; /* inner steps summed over outer iterations (and instances) */
  int32_t converged;         /* all instances met the stop rule */
  double final_metric;       /* last stop metric (max over instances) */
  double setup_ms;           /* method precompute in this call (Gram / Cholesky / P), device time */
  double solve_ms;           /* iteration time in this call, device time */
  double bytes_touched;      /* algorithmic bytes of A-derived data read by the iterations */
  int64_t kernel_launches;   /* kernels launched by this call */
  /* Per kernel class, measured with CUDA events on the handle's stream around each launch:
   * class 0 = SP persistent solver / K1 right-hand-side stream, 1 = SP-RK-RGS inner kernel,
   * 2 = SP-SCD inner kernel, 3 = setup (Gram, Cholesky, inverse). hot_work is the algorithmic
   * work of those launches: bytes of A-derived data touched (classes 0-2) or
   * flops (class 3). */
  double hot_ms[4];
  double hot_work[4];
  int64_t hot_launches[4];
  int64_t* inst_iters;       /* [NULL] optional host [batch] outer iterations per instance */
  int32_t* inst_status;      /* [NULL] optional host [batch] 1 = converged */
  int32_t sp_form_used;      /* the right-hand-side form this call ran (0, 1 or 2; resolves ILS_SP_FORM_AUTO) */
} ils_report;

ILS_API void ils_default_opts(ils_opts* opts);
ILS_API const char* ils_status_string(int status);
ILS_API const char* ils_last_error(void);

/* Ingest A (m x n, row-major, stride ext->lda) and b (m). Builds the handle's device copies:
 * row-major [A1; A2] padded to a multiple of 64 columns, column-major A1 (for RK/RGS
 * columns), the column norms N_j, the weight prefix sums S_j, and A1^T b1
 * (Alg. 2 step 3 / Alg. 5 step 2).
 * CSR input (ext->format = ILS_FORMAT_CSR): the CSR arrays are validated (ILS_ERR_ARG on an
 * out-of-range / unsorted / duplicated column, a bad row pointer or a non-finite value) and
 * converted to CSC for A1 and A2 (columns sorted by row). SP forms A1^T A1 densely (n <= 29000);
 * SP-SCD/RCD use it compacted to CSR; sp_form = 2 forms A2bar = A2^T A2 from the CSC of A2
 * (and, for SP at n < 8192, B = P A2bar). */
ILS_API int ils_create(ils_handle* h, const double* A, const double* b,
               int64_t p, int64_t q, int64_t n, const ils_ext* ext);

/* Alg. 1: P = (A1^T A1)^{-1} by DMMA Gram + Cholesky + explicit inverse,
 * built on the first call and cached; each iteration streams A2 once (K1) and applies P. */
ILS_API int ils_sp_solve(ils_handle h, const double* x0, double* x, double tol, int64_t max_iter,
                 const ils_opts* opts, ils_report* rep);

/* Alg. 2: SP-RK-RGS. */
ILS_API int ils_rk_solve(ils_handle h, const double* x0, double* x, double tol, int64_t max_iter,
                 const ils_opts* opts, ils_report* rep);

/* Alg. 5: SP-SCD; opts->weighted = 1 gives SP-RCD. */
ILS_API int ils_rgs_solve(ils_handle h, const double* x0, double* x, double tol, int64_t max_iter,
                  const ils_opts* opts, ils_report* rep);

ILS_API void ils_destroy(ils_handle h);

/* ---- helpers (same conventions) ---- */

/* Reference solution of the normal equation A^T J A x = A^T J b by a
 * device Cholesky of M = A1^T A1 - A2^T A2; ILS_ERR_NOT_SPD if (1.3) fails. x: [batch 1][n]. */
ILS_API int ils_direct_solve(ils_handle h, double* x);

/* RR(x) = ||A^T J (A x - b)||^2 / ||A^T J b||^2. */
ILS_API int ils_relative_residual(ils_handle h, const double* x, double* rr);

/* Copy the handle's column norms N (n doubles) and weight prefix sums S (n uint64) out. */
ILS_API int ils_get_sampling_tables(ils_handle h, double* N, uint64_t* S);

/* Replay check: the (j1, j2) pairs of SP-RK-RGS steps t0 .. t0+count-1 of outer iteration k
 * (int32 each), generated by the same device code the inner kernel uses. */
ILS_API int ils_rk_indices(ils_handle h, uint64_t seed, int64_t k, int64_t t0, int64_t count,
                   int32_t* j1, int32_t* j2);

/* Replay check: alpha_t and the membership mask of tau_t (n bytes, 1 = member) for SP-SCD
 * step t of outer iteration k, by the device code the inner kernel uses. */
ILS_API int ils_scd_subset(int64_t n, uint64_t seed, int64_t k, int64_t t, int32_t alpha_mode,
                   int32_t alpha_k, int32_t* alpha, uint8_t* mask);

/* Row-sharded handles (ext->comm): one NCCL communicator per process/GPU. Rank 0 calls
 * ils_comm_unique_id (ILS_COMM_ID_BYTES bytes, host), shares it with the other ranks by any
 * out-of-band means (e.g. torch.distributed broadcast), then every rank calls ils_comm_create
 * with its rank on its own device. NCCL is loaded at run time (ILS_ERR_UNSUPPORTED if absent). */
ILS_API int ils_comm_unique_id(void* id);
ILS_API int ils_comm_create(const void* id, int nranks, int rank, ils_comm* comm);
ILS_API void ils_comm_destroy(ils_comm comm);

/* Total kernels launched by this process through libils (for launch accounting). */
ILS_API int64_t ils_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* ILS_H_ */
