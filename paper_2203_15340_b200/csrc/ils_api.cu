// ils_api.cu -- the C ABI of libils (include/ils.h): validation, handle, host<->device staging,
// outer loops and reports. All arithmetic runs in the kernels of this library.
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "ils_internal.h"

namespace ils {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }
int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  if (e == cudaErrorMemoryAllocation) return ILS_ERR_NOMEM;
  return ILS_ERR_CUDA;
}
void count_launch(int64_t k) { g_launches += k; }

void hot_account(Handle& h, int c, double work, int64_t launches) {
  float ms = 0.f;
  cudaEventSynchronize(h.evk1);
  cudaEventElapsedTime(&ms, h.evk0, h.evk1);
  h.hot_ms[c] += ms;
  h.hot_work[c] += work;
  h.hot_n[c] += launches;
}
int64_t launches_now() { return g_launches.load(); }

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Device view of a caller buffer: the pointer itself if it is device memory, else a staged copy.
struct Staged {
  void* dev = nullptr;
  bool owned = false;
  const void* user = nullptr;
  size_t bytes = 0;
  cudaStream_t st = nullptr;
  int in(const void* u, size_t b, cudaStream_t s) {
    user = u;
    bytes = b;
    st = s;
    if (!u || b == 0) return ILS_OK;
    if (is_device_ptr(u)) {
      dev = const_cast<void*>(u);
      return ILS_OK;
    }
    ILS_CU(cudaMallocAsync(&dev, b, s));
    owned = true;
    ILS_CU(cudaMemcpyAsync(dev, u, b, cudaMemcpyHostToDevice, s));
    return ILS_OK;
  }
  int out(void* u, size_t b, cudaStream_t s) {   // output buffer (not copied in)
    user = u;
    bytes = b;
    st = s;
    if (!u || b == 0) return ILS_OK;
    if (is_device_ptr(u)) {
      dev = u;
      return ILS_OK;
    }
    ILS_CU(cudaMallocAsync(&dev, b, s));
    owned = true;
    return ILS_OK;
  }
  int writeback(size_t b) {
    if (owned && user && b) ILS_CU(cudaMemcpyAsync(const_cast<void*>(user), dev, b, cudaMemcpyDeviceToHost, st));
    return ILS_OK;
  }
  ~Staged() {
    if (owned && dev) cudaFreeAsync(dev, st);
  }
  double* d() const { return static_cast<double*>(dev); }
};

__global__ void nonfinite_kernel(const double* __restrict__ a, int64_t rows, int64_t cols, int64_t ld,
                                 int32_t* flag) {
  int bad = 0;
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const double v = a[(e / cols) * ld + (e % cols)];
    bad |= !isfinite(v);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

// batched ingest: flag an instance whose A1 has an all-zero column (include/ils.h ILS_ERR_ZERO_COLUMN)
__global__ void batched_zero_col_kernel(const double* __restrict__ Ab, int64_t batch, int64_t m, int64_t n,
                                        int64_t p, int32_t* flag) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < batch * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t inst = e / n, j = e - (e / n) * n;
    const double* a = Ab + inst * m * n + j;
    bool nz = false;
    for (int64_t i = 0; i < p && !nz; ++i) nz = a[i * n] != 0.0;
    if (!nz) atomicExch(flag, 1);
  }
}

static int check_finite(Handle& h, const double* a, int64_t rows, int64_t cols, int64_t ld, bool* ok) {
  ILS_CU(cudaMemsetAsync(&h.dstat->flag_err, 0, sizeof(int32_t), h.stream));
  if (rows * cols > 0) {
    nonfinite_kernel<<<h.num_sms * 4, 256, 0, h.stream>>>(a, rows, cols, ld, &h.dstat->flag_err);
    ILS_LAUNCHED("nonfinite_kernel");
  }
  int32_t f = 0;
  ILS_CU(cudaMemcpyAsync(&f, &h.dstat->flag_err, sizeof(int32_t), cudaMemcpyDeviceToHost, h.stream));
  ILS_CU(cudaStreamSynchronize(h.stream));
  *ok = (f == 0);
  return ILS_OK;
}

__global__ void dot_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* out) {
  __shared__ double s[32];
  double v = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v = fma(a[i], b[i], v);
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    *out = t;
  }
}

static int dot_host(Handle& h, const double* a, const double* b, int64_t n, double* res) {
  double* d = &h.dstat->metric;
  dot_kernel<<<1, 1024, 0, h.stream>>>(a, b, n, d);
  ILS_LAUNCHED("dot_kernel");
  ILS_CU(cudaMemcpyAsync(res, d, sizeof(double), cudaMemcpyDeviceToHost, h.stream));
  ILS_CU(cudaStreamSynchronize(h.stream));
  return ILS_OK;
}

// Pinned host status blocks are recycled across handles: cudaMallocHost / cudaFreeHost cost
// milliseconds (and cudaFreeHost synchronises the device), measured at ~1-3 ms per ils_create.
static std::mutex g_pin_mu;
static std::vector<DevStatus*> g_pin_free;
static DevStatus* pinned_status_get() {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (!g_pin_free.empty()) {
      DevStatus* s = g_pin_free.back();
      g_pin_free.pop_back();
      return s;
    }
  }
  void* p = nullptr;
  if (cudaMallocHost(&p, sizeof(DevStatus)) != cudaSuccess) return nullptr;
  return static_cast<DevStatus*>(p);
}
static void pinned_status_put(DevStatus* s) {
  if (!s) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.push_back(s);
}

static void free_handle_impl(Handle* h) {
  if (!h) return;
  cudaStream_t s = h->stream;
  double* bufs[] = {h->Arm, h->A1T, h->b, h->N, h->a1tb1, h->ajb, h->G, h->L, h->Z, h->P,
                    h->part, h->wsA, h->vec, h->red, h->Ab, h->bb, h->rk_state, h->A2bar, h->Bmat, h->lit_vec};
  for (double* p : bufs)
    if (p) cudaFreeAsync(p, s);
  if (h->S) cudaFreeAsync(h->S, s);
  if (h->scd_ws) cudaFreeAsync(h->scd_ws, s);
  {
    void* sb[] = {h->rp, h->ci, h->va, h->cp1, h->cr1, h->cv1, h->cp2, h->cr2, h->cv2, h->sp_y, h->gcsr_ptr,
                  h->gcsr_col, h->gcsr_val, h->sp_split};
    for (void* q : sb)
      if (q) cudaFreeAsync(q, s);
  }
  if (h->dstat) cudaFreeAsync(h->dstat, s);
  cudaStreamSynchronize(s);
  pinned_status_put(h->hstat);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->evk0) cudaEventDestroy(h->evk0);
  if (h->evk1) cudaEventDestroy(h->evk1);
  for (int i = 0; i < 2; ++i) {
    if (h->ev_mask[i]) cudaEventDestroy(h->ev_mask[i]);
    if (h->ev_chunk[i]) cudaEventDestroy(h->ev_chunk[i]);
  }
  if (h->aux) cudaStreamSynchronize(h->aux);   // shared per device (scd.cu), not owned
}

static float elapsed(Handle& h) {
  float ms = 0.f;
  cudaEventSynchronize(h.ev1);
  cudaEventElapsedTime(&ms, h.ev0, h.ev1);
  return ms;
}

}  // namespace ils

using namespace ils;

struct ils_handle_s : public ils::Handle {};

static void free_handle(ils_handle_s* h) {
  if (!h) return;
  free_handle_impl(h);
  delete h;
}

extern "C" {

void ils_default_opts(ils_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->stop = ILS_STOP_XREF;
  o->x_ref = nullptr;
  o->inner_tol = 1e-12;
  o->max_inner = 100000;
  o->check_every = 0;
  o->seed = 0;
  o->alpha_mode = ILS_ALPHA_UNIFORM;
  o->alpha_k = 1;
  o->weighted = 0;
  o->sp_form = 0;
}

const char* ils_status_string(int s) {
  switch (s) {
    case ILS_OK: return "ok";
    case ILS_NOT_CONVERGED: return "not converged (iteration cap reached)";
    case ILS_ERR_ARG: return "invalid argument";
    case ILS_ERR_SHAPE: return "invalid shape";
    case ILS_ERR_ZERO_COLUMN: return "A1 has a zero column";
    case ILS_ERR_NOT_SPD: return "matrix not SPD (condition 1.3 violated)";
    case ILS_ERR_CUDA: return "CUDA error";
    case ILS_ERR_NOMEM: return "out of device memory";
    case ILS_ERR_UNSUPPORTED: return "unsupported option or size";
    default: return "unknown status";
  }
}

const char* ils_last_error(void) { return g_err.c_str(); }

int64_t ils_kernel_launch_count(void) { return launches_now(); }

int ils_create(ils_handle* out, const double* A, const double* b, int64_t p, int64_t q, int64_t n,
               const ils_ext* ext) {
  if (!out || !A || !b) {
    set_error("ils_create: NULL argument");
    return ILS_ERR_ARG;
  }
  *out = nullptr;
  const int64_t lda = (ext && ext->lda) ? ext->lda : n;
  const int64_t batch = (ext && ext->batch > 0) ? ext->batch : 1;
  const bool sharded = ext && ext->comm;
  // a row shard may hold fewer than n rows of A1; the global p >= n is the caller's contract
  if (p < 1 || q < 0 || n < 1 || (!sharded && p < n) || lda < n) {
    set_error("ils_create: need p >= 1, q >= 0, n >= 1, p >= n (unsharded), lda >= n");
    return ILS_ERR_SHAPE;
  }
  const bool csr = ext && ext->format == ILS_FORMAT_CSR;
  if (sharded && (csr || batch != 1)) {
    set_error("ils_create: row sharding (ext->comm) needs dense input and batch 1");
    return ILS_ERR_UNSUPPORTED;
  }
  if (ext && ext->format != ILS_FORMAT_DENSE && !csr) {
    set_error("ils_create: unknown format");
    return ILS_ERR_ARG;
  }
  if (csr && (batch != 1 || !ext->row_ptr || !ext->col_idx || ext->nnz < 0)) {
    set_error("ils_create: CSR input needs batch 1, row_ptr, col_idx and nnz >= 0");
    return ILS_ERR_ARG;
  }
  ils_handle_s* h = new ils_handle_s();
  h->p = p;
  h->q = q;
  h->n = n;
  h->m = p + q;
  h->batch = batch;
  h->stream = ext ? static_cast<cudaStream_t>(ext->stream) : nullptr;
  h->comm = sharded ? static_cast<ils::ils_comm_impl*>(ext->comm) : nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  {   // keep freed stream-ordered allocations cached in the pool: handles of the same size reuse
      // them instead of returning GBs to the OS at every synchronisation
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  }
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev);
  {
    const char* e = getenv("ILS_RK_SINGLE_STEP");
    h->rk_single_step = (e && e[0] == '1');
  }
  int rc = ILS_OK;
  auto fail = [&](int code) {
    free_handle(h);
    return code;
  };
#define CK(call)                              \
  do {                                        \
    rc = (call);                              \
    if (rc != ILS_OK) return fail(rc);        \
  } while (0)
#define CKC(call) CK(((call) == cudaSuccess) ? ILS_OK : cuda_fail(cudaGetLastError(), #call))
  const cudaStream_t st = h->stream;
  CKC(cudaMallocAsync(&h->dstat, sizeof(DevStatus), st));
  CKC(cudaMemsetAsync(h->dstat, 0, sizeof(DevStatus), st));
  h->hstat = pinned_status_get();
  if (!h->hstat) {
    set_error("ils_create: pinned host allocation failed");
    return fail(ILS_ERR_NOMEM);
  }
  CKC(cudaEventCreate(&h->ev0));
  CKC(cudaEventCreate(&h->ev1));
  CKC(cudaEventCreate(&h->evk0));
  CKC(cudaEventCreate(&h->evk1));
  const int64_t m = h->m;
  bool ok = true;
  if (batch > 1) {
    const size_t abytes = (size_t)batch * m * n * sizeof(double);
    CKC(cudaMallocAsync(&h->Ab, abytes, st));
    CKC(cudaMallocAsync(&h->bb, (size_t)batch * m * sizeof(double), st));
    CKC(cudaMemcpy2DAsync(h->Ab, n * sizeof(double), A, lda * sizeof(double), n * sizeof(double),
                          (size_t)batch * m, cudaMemcpyDefault, st));
    CKC(cudaMemcpyAsync(h->bb, b, (size_t)batch * m * sizeof(double), cudaMemcpyDefault, st));
    CK(check_finite(*h, h->Ab, batch * m, n, n, &ok));
    if (ok) CK(check_finite(*h, h->bb, batch, m, m, &ok));
    if (!ok) {
      set_error("ils_create: non-finite entry in A or b");
      return fail(ILS_ERR_ARG);
    }
    {
      int32_t zc = 0;
      CKC(cudaMemsetAsync(&h->dstat->flag_err, 0, sizeof(int32_t), st));
      batched_zero_col_kernel<<<h->num_sms * 4, 256, 0, st>>>(h->Ab, batch, m, n, p, &h->dstat->flag_err);
      ILS_LAUNCHED("batched_zero_col_kernel");
      CKC(cudaMemcpyAsync(&zc, &h->dstat->flag_err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      CKC(cudaStreamSynchronize(st));
      if (zc) {
        set_error("ils_create: an instance's A1 has a zero column (||A1_(j)||^2 = 0)");
        return fail(ILS_ERR_ZERO_COLUMN);
      }
    }
    *out = h;
    return ILS_OK;
  }
  h->npad = roundup(n, kPad);
  {
    const char* e = getenv("ILS_FORCE_LARGE");   // test hook: take the n > 8192 dense paths at any n
    h->large = !csr && (h->npad > 8192 || (e && e[0] == '1'));
  }
  h->ppad = roundup(p, kPad);
  const int64_t np = h->npad;
  if (csr) {   // ---- CSR input (sparse.cu)
    const int64_t nnz = ext->nnz;
    h->sparse = true;
    h->nnz = nnz;
    CKC(cudaMallocAsync(&h->rp, (size_t)(m + 1) * sizeof(int64_t), st));
    CKC(cudaMallocAsync(&h->ci, (size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t), st));
    CKC(cudaMallocAsync(&h->va, (size_t)(nnz > 0 ? nnz : 1) * sizeof(double), st));
    CKC(cudaMemcpyAsync(h->rp, ext->row_ptr, (size_t)(m + 1) * sizeof(int64_t), cudaMemcpyDefault, st));
    if (nnz > 0) {
      CKC(cudaMemcpyAsync(h->ci, ext->col_idx, (size_t)nnz * sizeof(int32_t), cudaMemcpyDefault, st));
      CKC(cudaMemcpyAsync(h->va, A, (size_t)nnz * sizeof(double), cudaMemcpyDefault, st));
    }
    CKC(cudaMallocAsync(&h->b, (size_t)(m + 64) * sizeof(double), st));
    CKC(cudaMemsetAsync(h->b, 0, (size_t)(m + 64) * sizeof(double), st));
    CKC(cudaMemcpyAsync(h->b, b, m * sizeof(double), cudaMemcpyDefault, st));
    {
      int64_t ends[2] = {0, 0};
      CKC(cudaMemcpyAsync(&ends[0], h->rp, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      CKC(cudaMemcpyAsync(&ends[1], h->rp + m, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      CKC(cudaMemcpyAsync(&h->nnz1, h->rp + p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      CKC(cudaStreamSynchronize(st));
      if (ends[0] != 0 || ends[1] != nnz) {
        set_error("ils_create: CSR row_ptr[0] must be 0 and row_ptr[m] = nnz");
        return fail(ILS_ERR_ARG);
      }
    }
    CK(check_finite(*h, h->b, 1, m, m, &ok));
    if (!ok) {
      set_error("ils_create: non-finite entry in b");
      return fail(ILS_ERR_ARG);
    }
    {   // sum of squared row lengths of A1 (Gram flop count)
      std::vector<int64_t> rph((size_t)p + 1);
      CKC(cudaMemcpyAsync(rph.data(), h->rp, (size_t)(p + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      CKC(cudaStreamSynchronize(st));
      double sq = 0.0;
      for (int64_t i = 0; i < p; ++i) {
        const double l = (double)(rph[i + 1] - rph[i]);
        sq += l * l;
      }
      h->a1_row_sq = sq;
    }
    CKC(cudaMallocAsync(&h->N, (size_t)n * sizeof(double), st));
    CKC(cudaMallocAsync(&h->S, (size_t)n * sizeof(uint64_t), st));
    CKC(cudaMallocAsync(&h->a1tb1, (size_t)np * sizeof(double), st));
    CK(sparse_ingest(*h, &h->dstat->flag_err, &ok));
    if (!ok) {
      set_error("ils_create: invalid CSR structure (row_ptr, column order/range) or non-finite value");
      return fail(ILS_ERR_ARG);
    }
    CKC(cudaMemsetAsync(&h->dstat->flag_err, 0, sizeof(int32_t), st));
    CK(launch_weights(*h, &h->dstat->flag_err));
    h->part_rows = h->num_sms > 16 ? h->num_sms : 16;
    CKC(cudaMallocAsync(&h->part, (size_t)h->part_rows * np * sizeof(double), st));
    CKC(cudaMallocAsync(&h->red, (size_t)h->part_rows * 4 * sizeof(double), st));
    CKC(cudaMallocAsync(&h->vec, (size_t)8 * np * sizeof(double), st));
    CKC(cudaMemsetAsync(h->vec, 0, (size_t)8 * np * sizeof(double), st));
    int32_t zf = 0;
    CKC(cudaMemcpyAsync(&zf, &h->dstat->flag_err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CKC(cudaStreamSynchronize(st));
    if (zf) {
      set_error("ils_create: A1 has a zero column");
      return fail(ILS_ERR_ZERO_COLUMN);
    }
    *out = h;
    return ILS_OK;
  }
  CKC(cudaMallocAsync(&h->Arm, (size_t)(m + 64) * np * sizeof(double), st));
  CKC(cudaMallocAsync(&h->b, (size_t)(m + 64) * sizeof(double), st));
  CKC(cudaMemsetAsync(h->b, 0, (size_t)(m + 64) * sizeof(double), st));
  CKC(cudaMemcpyAsync(h->b, b, m * sizeof(double), cudaMemcpyDefault, st));
  CKC(cudaMallocAsync(&h->A1T, (size_t)np * h->ppad * sizeof(double), st));
  CKC(cudaMemsetAsync(&h->dstat->flag_nonfinite, 0, sizeof(int32_t), st));
  // one fused pass: Arm (padded), A1T, finite check (ingest.cu). Host A is uploaded into Arm
  // first and then processed in place.
  const double* Asrc = A;
  int64_t lsrc = lda;
  if (!is_device_ptr(A)) {
    CKC(cudaMemcpy2DAsync(h->Arm, np * sizeof(double), A, lda * sizeof(double), n * sizeof(double), m,
                          cudaMemcpyHostToDevice, st));
    Asrc = h->Arm;
    lsrc = np;
  }
  CK(launch_ingest_dense(*h, Asrc, lsrc, h->b, &h->dstat->flag_nonfinite));
  CKC(cudaMallocAsync(&h->N, (size_t)n * sizeof(double), st));
  CKC(cudaMallocAsync(&h->S, (size_t)n * sizeof(uint64_t), st));
  CK(launch_colnorms(*h));
  CK(allreduce_sum(*h, h->N, n));   // sharded: N_j = sum over ranks (comm.cu)
  CKC(cudaMemsetAsync(&h->dstat->flag_err, 0, sizeof(int32_t), st));
  CK(launch_weights(*h, &h->dstat->flag_err));
  CKC(cudaMallocAsync(&h->a1tb1, (size_t)np * sizeof(double), st));
  CK(launch_gemv_rows(h->A1T, h->ppad, np, p, h->b, h->a1tb1, 1.0, nullptr, st));
  h->part_rows = h->num_sms > 16 ? h->num_sms : 16;
  CKC(cudaMallocAsync(&h->part, (size_t)h->part_rows * np * sizeof(double), st));
  CKC(cudaMallocAsync(&h->red, (size_t)h->part_rows * 4 * sizeof(double), st));
  CKC(cudaMallocAsync(&h->vec, (size_t)8 * np * sizeof(double), st));
  CKC(cudaMemsetAsync(h->vec, 0, (size_t)8 * np * sizeof(double), st));
  CKC(cudaMemcpyAsync(h->hstat, h->dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
  CKC(cudaStreamSynchronize(st));
  if (h->hstat->flag_nonfinite) {
    set_error("ils_create: non-finite entry in A or b");
    return fail(ILS_ERR_ARG);
  }
  if (h->hstat->flag_err) {
    set_error("ils_create: A1 has a zero column");
    return fail(ILS_ERR_ZERO_COLUMN);
  }
#undef CK
#undef CKC
  *out = h;
  return ILS_OK;
}

void ils_destroy(ils_handle h) { free_handle(h); }

// method: 0 SP, 1 SP-RK-RGS, 2 SP-SCD/RCD
// include/ils.h "Automatic form": the literal layout (sp_form 2) iff its one-time DMMA precompute
// costs less than the A2 stream it saves over the expected outer steps.
static int auto_sp_form(const Handle& H, int method, int64_t max_iter, int64_t expected_outer) {
  if (H.sparse || H.large || H.n > 8192 || H.comm != nullptr) return 0;
  const double K = (double)(expected_outer > 0 ? expected_outer : (max_iter < 32 ? max_iter : 32));
  const double n = (double)H.n, q = (double)H.q;
  const double saved = (method == 0) ? 8.0 * q * (n + 1.0) : 8.0 * q * (n + 1.0) - 8.0 * n * n;
  const double flops = q * n * (n + 1.0) + (method == 0 ? 2.0 * n * n * n : 0.0);
  constexpr double kHbm = 6.0e12, kDmma = 3.0e13;
  return (saved > 0.0 && K * saved / kHbm > flops / kDmma) ? 2 : 0;
}

static int solve_common(ils_handle h, int method, const double* x0, double* x, double tol, int64_t max_iter,
                        const ils_opts* opts_in, ils_report* rep) {
  if (!h || !x) {
    set_error("solve: NULL handle or x");
    return ILS_ERR_ARG;
  }
  ils_opts o;
  if (opts_in) o = *opts_in; else ils_default_opts(&o);
  if (max_iter < 0 || o.max_inner < 0 || o.inner_tol < 0 || !(tol >= 0)) {
    set_error("solve: negative cap or tolerance");
    return ILS_ERR_ARG;
  }
  if (o.stop == ILS_STOP_XREF && !o.x_ref) {
    set_error("solve: ILS_STOP_XREF needs opts->x_ref");
    return ILS_ERR_ARG;
  }
  if (o.stop < 0 || o.stop > 2 || (o.alpha_mode & ~(0xF | ILS_SUBSET_EXACT)) || (o.alpha_mode & 0xF) > ILS_ALPHA_FIXED ||
      ((o.alpha_mode & 0xF) == ILS_ALPHA_FIXED && o.alpha_k < 1)) {
    set_error("solve: bad option");
    return ILS_ERR_ARG;
  }
  Handle& H = *h;
  const cudaStream_t st = H.stream;
  const int64_t n = H.n, B = H.batch;
  const int64_t l0 = launches_now();
  for (int c = 0; c < 4; ++c) {
    H.hot_ms[c] = 0.0;
    H.hot_work[c] = 0.0;
    H.hot_n[c] = 0;
  }
  int rc = ILS_OK;
  if (rep) {
    int64_t* ii = rep->inst_iters;
    int32_t* is = rep->inst_status;
    std::memset(rep, 0, sizeof(*rep));
    rep->inst_iters = ii;
    rep->inst_status = is;
  }
  Staged sx0, sx, sxr;
  if ((rc = sx0.in(x0, (size_t)B * n * sizeof(double), st))) return rc;
  if ((rc = sx.out(x, (size_t)B * n * sizeof(double), st))) return rc;
  if ((rc = sxr.in(o.x_ref, (size_t)B * n * sizeof(double), st))) return rc;

  if (B > 1) {
    if (o.stop == ILS_STOP_RR || (method == 2 && (o.alpha_mode & ILS_SUBSET_EXACT))) {
      set_error("batched: ILS_STOP_RR and exact uniform subsets are not supported");
      return ILS_ERR_UNSUPPORTED;
    }
    ils_opts od = o;
    od.x_ref = sxr.d();
    int64_t* it_dev = nullptr;
    int32_t* st_dev = nullptr;
    ILS_CU(cudaMallocAsync(&it_dev, B * sizeof(int64_t), st));
    ILS_CU(cudaMallocAsync(&st_dev, B * sizeof(int32_t), st));
    ILS_CU(cudaMemsetAsync(H.dstat, 0, sizeof(DevStatus), st));
    ILS_CU(cudaEventRecord(H.ev0, st));
    rc = batched_solve(H, method, sx0.d(), sx.d(), tol, max_iter, od, it_dev, st_dev);
    ILS_CU(cudaEventRecord(H.ev1, st));
    if (rc) return rc;
    std::vector<int64_t> its(B);
    std::vector<int32_t> sts(B);
    ILS_CU(cudaMemcpyAsync(its.data(), it_dev, B * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    ILS_CU(cudaMemcpyAsync(sts.data(), st_dev, B * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    ILS_CU(cudaMemcpyAsync(H.hstat, H.dstat, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
    if ((rc = sx.writeback((size_t)B * n * sizeof(double)))) return rc;
    ILS_CU(cudaStreamSynchronize(st));
    cudaFreeAsync(it_dev, st);
    cudaFreeAsync(st_dev, st);
    if (H.hstat->flag_err) {   // batched SP: an instance's A1^T A1 broke down in the Cholesky
      if (rep && rep->inst_status) std::memcpy(rep->inst_status, sts.data(), B * sizeof(int32_t));
      set_error("batched SP: Cholesky of an instance's A1^T A1 broke down (inst_status -1)");
      return ILS_ERR_NOT_SPD;
    }
    int64_t mx = 0;
    bool all = true;
    for (int64_t i = 0; i < B; ++i) {
      mx = its[i] > mx ? its[i] : mx;
      all = all && sts[i];
    }
    if (rep) {
      rep->outer_iters = mx;
      rep->inner_iters_total = H.hstat->inner_steps;
      rep->converged = all ? 1 : 0;
      rep->solve_ms = elapsed(H);
      rep->kernel_launches = launches_now() - l0;
      if (rep->inst_iters) std::memcpy(rep->inst_iters, its.data(), B * sizeof(int64_t));
      if (rep->inst_status) std::memcpy(rep->inst_status, sts.data(), B * sizeof(int32_t));
      // algorithmic bytes: per outer step the A2 stream 8q(n+1) (+ 8n^2 for the P
      // apply of SP), per inner step 16p (RK-RGS: two columns of A1) or 8n (SCD: one row of A1bar)
      double outer_sum = 0.0;
      for (int64_t i = 0; i < B; ++i) outer_sum += (double)its[i];
      const double nd = (double)n, pd = (double)H.p, qd = (double)H.q;
      double byt = outer_sum * 8.0 * qd * (nd + 1.0);
      if (method == 0) byt += outer_sum * 8.0 * nd * nd;
      else if (method == 1) byt += (double)H.hstat->inner_steps * 16.0 * pd;
      else byt += (double)H.hstat->inner_steps * 8.0 * nd;
      rep->bytes_touched = byt;
      rep->hot_ms[method] = rep->solve_ms;
      rep->hot_work[method] = byt;
      rep->hot_launches[method] = 1;
    }
    return all ? ILS_OK : ILS_NOT_CONVERGED;
  }

  const int64_t np = H.npad;
  if (o.sp_form == ILS_SP_FORM_AUTO) o.sp_form = auto_sp_form(H, method, max_iter, o.expected_outer);
  if (rep) rep->sp_form_used = o.sp_form;
  if (o.sp_form < 0 || o.sp_form > 2 || (o.sp_form == 1 && method != 0)) {
    set_error("solve: sp_form must be 0, 2 or 3 (RK/RGS), 0..3 (SP)");
    return ILS_ERR_ARG;
  }
  const bool sharded = H.comm != nullptr;
  if (sharded && (method == 1 || o.sp_form == 2)) {
    set_error("row-sharded handle: SP-RK-RGS (needs whole columns of A1) and sp_form 2 are not supported");
    return ILS_ERR_UNSUPPORTED;
  }
  // full residual g = A^T J (b - A x): dense stream kernel or the sparse row/column passes
  // (sharded: local rows, then the sum over ranks)
  auto full_res = [&](const double* xv, double* gv) -> int {
    const int r = H.sparse ? sparse_rhs(H, xv, gv, 1) : full_residual(H, xv, gv);
    return r ? r : allreduce_sum(H, gv, H.npad);
  };
  // ---- setup (timed separately)
  ILS_CU(cudaMemsetAsync(&H.dstat->flag_err, 0, sizeof(int32_t), st));
  const bool gram_new = !H.have_gram && method != 1, inv_new = !H.have_P && method == 0;
  const bool lit_new = o.sp_form == 2 && (method == 0 ? !H.have_B : !H.have_a2bar);
  ILS_CU(cudaEventRecord(H.ev0, st));
  if (method == 0) rc = (o.sp_form == 2) ? build_explicit_b(H) : build_inverse(H);
  else if (method == 2) rc = build_gram(H);
  if (!rc && method != 0 && o.sp_form == 2) rc = build_a2bar(H);
  ILS_CU(cudaEventRecord(H.ev1, st));
  if (rc) return rc;
  const float setup_ms = elapsed(H);
  if (gram_new || inv_new || lit_new) {
    const double nd = (double)H.n, pd = (double)H.p;
    H.hot_ms[3] += setup_ms;
    // algorithmic flops (LAPACK counts): SYRK p n (n+1) (sparse: 2 sum_i nnz_i^2 over A1 rows),
    // Cholesky n^3/3 + triangular inverse n^3/3 (+ P = Z^T Z n^3/3 when formed)
    const double gram = H.sparse ? 2.0 * H.a1_row_sq : pd * nd * (nd + 1.0);
    // use_zt (n >= 8192): only the Cholesky (n^3 / 3) is counted; the partial inverse formed there
    // replaces triangular solves and is an implementation choice, not algorithmic work
    H.hot_work[3] += (gram_new ? gram : 0.0) + (inv_new ? (H.use_zt ? 1.0 : 3.0) * nd * nd * nd / 3.0 : 0.0) +
                     (lit_new ? (double)H.q * nd * (nd + 1.0) + (method == 0 ? 2.0 * nd * nd * nd : 0.0) : 0.0);
    H.hot_n[3] += 1;
  }
  {
    int32_t f = 0;
    ILS_CU(cudaMemcpy(&f, &H.dstat->flag_err, sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (f) {
      set_error("Cholesky of A1^T A1 broke down");
      return ILS_ERR_NOT_SPD;
    }
  }
  // RR denominator ||A^T J b||^2
  double ajb2 = 0.0;
  double* g = H.vec + 5 * np;
  if (o.stop == ILS_STOP_RR) {
    double* zero = H.vec + 4 * np;
    ILS_CU(cudaMemsetAsync(zero, 0, np * sizeof(double), st));
    if ((rc = full_res(zero, g))) return rc;
    if ((rc = dot_host(H, g, g, n, &ajb2))) return rc;
    if (ajb2 == 0.0) {
      set_error("A^T J b = 0: RR undefined");
      return ILS_ERR_ARG;
    }
  }
  Staged shist;
  const size_t hist_bytes = (size_t)max_iter * n * sizeof(double);
  if (o.x_hist && (rc = shist.out(o.x_hist, hist_bytes, st))) return rc;

  ILS_CU(cudaEventRecord(H.ev0, st));
  int64_t outer = 0, inner_total = 0;
  double metric = NAN;
  int conv = 0;
  double* xk = H.vec + 6 * np;   // current iterate (device, npad)
  double* bhat = H.vec + 3 * np;
  double* xnew = H.vec + 7 * np;
  ILS_CU(cudaMemsetAsync(xk, 0, np * sizeof(double), st));
  if (sx0.d()) ILS_CU(cudaMemcpyAsync(xk, sx0.d(), n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  std::vector<int64_t> inner_hist;

  const bool big = !H.sparse && H.large;   // dense n > 8192: host-looped two-pass SP (large.cu)
  if (method == 0 && o.stop != ILS_STOP_RR && !H.sparse && o.sp_form != 2 && !big && !sharded) {
    // whole SP loop in one persistent cooperative launch
    const int stop = (o.stop == ILS_STOP_XREF) ? ILS_STOP_XREF : ILS_STOP_NONE;
    if (max_iter > 0) {
      if ((rc = sp_run(H, xk, xnew, tol, max_iter, stop, sxr.d(), o.sp_form, shist.d(), false, nullptr, &outer,
                       &metric, &conv)))
        return rc;
      ILS_CU(cudaMemcpyAsync(xk, xnew, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
  } else {
    for (int64_t k = 0; k < max_iter; ++k) {
      int64_t steps = 0;
      if (method == 0 && o.sp_form == 2) {   // Alg. 1 literal: x_{k+1} = B x_k + c0 (one n x n GEMV)
        ILS_CU(cudaEventRecord(H.evk0, st));
        if ((rc = launch_gemv_rows(H.Bmat, np, np, np, xk, xnew, 1.0, H.lit_vec + np, st))) return rc;
        ILS_CU(cudaEventRecord(H.evk1, st));
        hot_account(H, 0, 8.0 * (double)n * (double)n);
      } else if (method == 0 && (H.sparse || big || sharded)) {   // c_k by row/column passes, x = P c_k (+ x_k)
        ILS_CU(cudaEventRecord(H.evk0, st));
        if (H.sparse) {   // paper form c_k, or the correction form's g_k = A^T J (b - A x_k)
          if ((rc = sparse_rhs(H, xk, bhat, o.sp_form == 1))) return rc;
        } else if (big) {
          if ((rc = dense_rhs_twopass(H, xk, bhat, o.sp_form == 1))) return rc;
        } else if ((rc = sp_run(H, xk, nullptr, 0.0, 1, ILS_STOP_NONE, nullptr, o.sp_form, nullptr, true, bhat,
                                nullptr, nullptr, nullptr))) {
          return rc;
        }
        if ((rc = allreduce_sum(H, bhat, np))) return rc;   // sharded: sum of the ranks' partial c_k / g_k
        if ((rc = gemv_p(H, bhat, xnew))) return rc;
        if ((big || sharded || H.sparse) && o.sp_form == 1 && (rc = vec_add(H, xnew, xk, n))) return rc;
        ILS_CU(cudaEventRecord(H.evk1, st));
        if (H.sparse)   // row pass + column pass over A2 (all of A, twice, under the correction form) + P
          hot_account(H, 0, (o.sp_form == 1 ? 24.0 * (double)H.nnz + 16.0 * (double)H.m
                                            : 24.0 * (double)(H.nnz - H.nnz1) + 16.0 * (double)H.q) +
                                8.0 * (double)np * (double)np,
                      o.sp_form == 1 ? 5 : 2);
        else   // two passes over A2 (or all of A under the correction form) + the P sweep
          hot_account(H, 0, 16.0 * (double)(o.sp_form == 1 ? H.m : H.q) * (double)n + 8.0 * (double)np * (double)np,
                      o.sp_form == 1 ? 5 : 3);
      } else if (method == 0) {   // SP under the RR rule: one persistent step at a time
        int64_t one = 0;
        double mm;
        int cc;
        if ((rc = sp_run(H, xk, xnew, 0.0, 1, ILS_STOP_NONE, nullptr, o.sp_form, nullptr, false, nullptr, &one,
                         &mm, &cc)))
          return rc;
      } else {
        // b_hat = A2bar x_k + A^T J b (K1 stream, rhs_only)
        if (o.sp_form == 2) {   // b_hat = A2bar x_k + A^T J b (Alg. 2 step 5 / Alg. 5 step 4, literal)
          if ((rc = launch_gemv_rows(H.A2bar, np, np, np, xk, bhat, 1.0, H.lit_vec, st))) return rc;
        } else if (H.sparse) {
          if ((rc = sparse_rhs(H, xk, bhat, 0))) return rc;
        } else if ((rc = sp_run(H, xk, nullptr, 0.0, 1, ILS_STOP_NONE, nullptr, 0, nullptr, true, bhat, nullptr,
                                nullptr, nullptr))) {
          return rc;
        }
        if ((rc = allreduce_sum(H, bhat, np))) return rc;   // sharded SP-SCD: global b_hat
        if (method == 1)
          rc = H.sparse ? sparse_rk_inner(H, bhat, xnew, o.seed, k, o.max_inner, o.check_every, o.inner_tol, &steps)
                        : rk_rgs_inner(H, bhat, xnew, o.seed, k, o.max_inner, o.check_every, o.inner_tol, &steps);
        else
          rc = H.sparse ? sparse_scd_inner(H, bhat, xnew, o.seed, k, o.max_inner, o.check_every, o.inner_tol,
                                           o.alpha_mode, o.alpha_k, o.weighted, &steps)
                        : scd_inner(H, bhat, xnew, o.seed, k, o.max_inner, o.check_every, o.inner_tol, o.alpha_mode,
                                    o.alpha_k, o.weighted, &steps);
        if (rc) return rc;
      }
      ILS_CU(cudaMemcpyAsync(xk, xnew, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      if (shist.d())
        ILS_CU(cudaMemcpyAsync(shist.d() + k * n, xk, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      inner_total += steps;
      inner_hist.push_back(steps);
      outer = k + 1;
      bool done = false;
      if (o.stop == ILS_STOP_XREF) {
        if ((rc = stop_metric(H, xk, sxr.d(), &H.dstat->metric))) return rc;
        ILS_CU(cudaMemcpyAsync(&metric, &H.dstat->metric, sizeof(double), cudaMemcpyDeviceToHost, st));
        ILS_CU(cudaStreamSynchronize(st));
        done = metric <= tol;
      } else if (o.stop == ILS_STOP_RR) {
        if ((rc = full_res(xk, g))) return rc;
        double gg = 0.0;
        if ((rc = dot_host(H, g, g, n, &gg))) return rc;
        metric = gg / ajb2;
        done = metric < tol;
      }
      if (done) {
        conv = 1;
        break;
      }
    }
  }
  ILS_CU(cudaEventRecord(H.ev1, st));
  const float solve_ms = elapsed(H);
  ILS_CU(cudaMemcpyAsync(sx.d(), xk, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if ((rc = sx.writeback(n * sizeof(double)))) return rc;
  if (shist.d() && (rc = shist.writeback((size_t)outer * n * sizeof(double)))) return rc;
  ILS_CU(cudaStreamSynchronize(st));
  if (o.inner_hist)
    for (size_t i = 0; i < inner_hist.size(); ++i) o.inner_hist[i] = inner_hist[i];
  if (rep) {
    rep->outer_iters = outer;
    rep->inner_iters_total = inner_total;
    rep->converged = conv;
    rep->final_metric = metric;
    rep->setup_ms = setup_ms;
    rep->solve_ms = solve_ms;
    const double q = (double)H.q, p = (double)H.p, nd = (double)n;
    if (H.sparse && o.sp_form != 2) {   // algorithmic bytes of the sparse path (12 B per CSR/CSC entry)
      const double a2 = (method == 0 && o.sp_form == 1) ? 24.0 * (double)H.nnz + 16.0 * (double)H.m
                                                        : 12.0 * (double)(H.nnz - H.nnz1) * 2.0 + 16.0 * q;
      const double rk_step = 2.0 * ((double)H.nnz1 / nd) * 28.0;
      const double scd_step = 12.0 * ((double)H.gnnz / nd);
      rep->bytes_touched = outer * a2 + (method == 0 ? outer * 8.0 * (double)np * (double)np
                                                     : inner_total * (method == 1 ? rk_step : scd_step));
    } else if (o.sp_form == 2) {   // literal forms: one n x n GEMV per outer step
      const double inner_b = (method == 1) ? inner_total * 16.0 * p : (method == 2 ? inner_total * 8.0 * nd : 0.0);
      rep->bytes_touched = outer * 8.0 * nd * nd + inner_b;
    } else if (method == 0)
      rep->bytes_touched = outer * (8.0 * q * (nd + 1) + 8.0 * nd * nd);
    else if (method == 1)
      rep->bytes_touched = outer * 8.0 * q * (nd + 1) + inner_total * 16.0 * p;
    else
      rep->bytes_touched = outer * 8.0 * q * (nd + 1) + inner_total * 8.0 * nd;
    rep->kernel_launches = launches_now() - l0;
    for (int c = 0; c < 4; ++c) {
      rep->hot_ms[c] = H.hot_ms[c];
      rep->hot_work[c] = H.hot_work[c];
      rep->hot_launches[c] = H.hot_n[c];
    }
  }
  return conv ? ILS_OK : ILS_NOT_CONVERGED;
}

int ils_sp_solve(ils_handle h, const double* x0, double* x, double tol, int64_t max_iter, const ils_opts* opts,
                 ils_report* rep) {
  return solve_common(h, 0, x0, x, tol, max_iter, opts, rep);
}

int ils_rk_solve(ils_handle h, const double* x0, double* x, double tol, int64_t max_iter, const ils_opts* opts,
                 ils_report* rep) {
  return solve_common(h, 1, x0, x, tol, max_iter, opts, rep);
}

int ils_rgs_solve(ils_handle h, const double* x0, double* x, double tol, int64_t max_iter, const ils_opts* opts,
                  ils_report* rep) {
  return solve_common(h, 2, x0, x, tol, max_iter, opts, rep);
}

int ils_direct_solve(ils_handle h, double* x) {
  if (!h || !x) return ILS_ERR_ARG;
  Handle& H = *h;
  if (H.batch > 1) return ILS_ERR_UNSUPPORTED;
  if (H.comm) {
    set_error("ils_direct_solve: not supported on a row-sharded handle");
    return ILS_ERR_UNSUPPORTED;
  }
  const cudaStream_t st = H.stream;
  const int64_t np = H.npad, n = H.n;
  int rc = build_gram(H);
  if (rc) return rc;
  const size_t bytes = (size_t)np * np * sizeof(double);
  double *M = nullptr, *Zm = nullptr;
  ILS_CU(cudaMallocAsync(&M, bytes, st));
  ILS_CU(cudaMallocAsync(&Zm, bytes, st));
  ILS_CU(cudaMemcpyAsync(M, H.G, bytes, cudaMemcpyDeviceToDevice, st));
  // M -= A2^T A2 : opA(i,k) = A2[k][i] (M-contiguous), opB(j,k) = A2[k][j] (N-contiguous)
  const int64_t kq = roundup(H.q, 32);
  if (H.sparse) {
    if (H.q > 0) rc = sparse_gram(H, M, true);
  } else if (H.q > 0) {
    rc = gemm_dmma(H, true, true, np, np, kq, -1.0, H.Arm + H.p * np, np, H.Arm + H.p * np, np, 1.0, M, np, true, 1);
    if (!rc) rc = mirror_lower(H, M, np, np, n);
  }
  ILS_CU(cudaMemsetAsync(&H.dstat->flag_err, 0, sizeof(int32_t), st));
  if (!rc) rc = cholesky_inverse(H, M, Zm, np, true);
  // rhs = A^T J b = A1^T b1 - A2^T b2 ; x = Z^T (Z rhs)
  double* rhs = H.vec + 4 * np;
  double* y = H.vec + 5 * np;
  double* xd = H.vec + 6 * np;
  if (!rc) {
    if (H.sparse) {   // A^T J (b - A 0) by the sparse passes
      ILS_CU(cudaMemsetAsync(xd, 0, np * sizeof(double), st));
      rc = sparse_rhs(H, xd, rhs, 1);
    } else {
      rc = launch_gemv_cols(H.Arm + H.p * np, np, H.q, np, H.b + H.p, rhs, -1.0, H.a1tb1, st);
    }
  }
  if (!rc) rc = launch_gemv_rows(Zm, np, np, np, rhs, y, 1.0, nullptr, st);
  if (!rc) rc = launch_gemv_cols(Zm, np, np, np, y, xd, 1.0, nullptr, st);
  int32_t f = 0;
  if (!rc) {
    Staged sx;
    if ((rc = sx.out(x, n * sizeof(double), st)) == ILS_OK) {
      ILS_CU(cudaMemcpyAsync(sx.d(), xd, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      rc = sx.writeback(n * sizeof(double));
      ILS_CU(cudaMemcpyAsync(&f, &H.dstat->flag_err, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      ILS_CU(cudaStreamSynchronize(st));
    }
  }
  cudaFreeAsync(M, st);
  cudaFreeAsync(Zm, st);
  cudaStreamSynchronize(st);
  if (rc) return rc;
  if (f) {
    set_error("A^T J A is not SPD (condition 1.3)");
    return ILS_ERR_NOT_SPD;
  }
  return ILS_OK;
}

int ils_relative_residual(ils_handle h, const double* x, double* rr) {
  if (!h || !x || !rr) return ILS_ERR_ARG;
  Handle& H = *h;
  if (H.batch > 1) return ILS_ERR_UNSUPPORTED;
  const cudaStream_t st = H.stream;
  const int64_t np = H.npad, n = H.n;
  Staged sx;
  int rc = sx.in(x, n * sizeof(double), st);
  if (rc) return rc;
  double* xz = H.vec + 4 * np;
  double* g = H.vec + 5 * np;
  auto fres = [&](const double* xv, double* gv) {
    const int r = H.sparse ? sparse_rhs(H, xv, gv, 1) : full_residual(H, xv, gv);
    return r ? r : allreduce_sum(H, gv, H.npad);   // sharded: sum over ranks
  };
  ILS_CU(cudaMemsetAsync(xz, 0, np * sizeof(double), st));
  if ((rc = fres(xz, g))) return rc;
  double den = 0.0, num = 0.0;
  if ((rc = dot_host(H, g, g, n, &den))) return rc;
  if (den == 0.0) {
    set_error("A^T J b = 0: RR undefined");
    return ILS_ERR_ARG;
  }
  ILS_CU(cudaMemcpyAsync(xz, sx.d(), n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if ((rc = fres(xz, g))) return rc;
  if ((rc = dot_host(H, g, g, n, &num))) return rc;
  *rr = num / den;
  return ILS_OK;
}

int ils_get_sampling_tables(ils_handle h, double* N, uint64_t* S) {
  if (!h) return ILS_ERR_ARG;
  Handle& H = *h;
  if (H.batch > 1) return ILS_ERR_UNSUPPORTED;
  if (N) ILS_CU(cudaMemcpyAsync(N, H.N, H.n * sizeof(double), cudaMemcpyDefault, H.stream));
  if (S) ILS_CU(cudaMemcpyAsync(S, H.S, H.n * sizeof(uint64_t), cudaMemcpyDefault, H.stream));
  ILS_CU(cudaStreamSynchronize(H.stream));
  return ILS_OK;
}

int ils_rk_indices(ils_handle h, uint64_t seed, int64_t k, int64_t t0, int64_t count, int32_t* j1, int32_t* j2) {
  if (!h || !j1 || !j2 || count < 0) return ILS_ERR_ARG;
  Handle& H = *h;
  if (H.batch > 1) return ILS_ERR_UNSUPPORTED;
  Staged s1, s2;
  int rc;
  if ((rc = s1.out(j1, count * sizeof(int32_t), H.stream))) return rc;
  if ((rc = s2.out(j2, count * sizeof(int32_t), H.stream))) return rc;
  if (count > 0 && (rc = rk_indices(H, seed, k, t0, count, static_cast<int32_t*>(s1.dev), static_cast<int32_t*>(s2.dev))))
    return rc;
  if ((rc = s1.writeback(count * sizeof(int32_t)))) return rc;
  if ((rc = s2.writeback(count * sizeof(int32_t)))) return rc;
  ILS_CU(cudaStreamSynchronize(H.stream));
  return ILS_OK;
}

int ils_scd_subset(int64_t n, uint64_t seed, int64_t k, int64_t t, int32_t alpha_mode, int32_t alpha_k,
                   int32_t* alpha, uint8_t* mask) {
  if (n < 1 || !alpha || !mask) return ILS_ERR_ARG;
  cudaStream_t st = nullptr;
  Staged sa, sm;
  int rc;
  if ((rc = sa.out(alpha, sizeof(int32_t), st))) return rc;
  if ((rc = sm.out(mask, n, st))) return rc;
  if ((rc = scd_subset_mask(n, seed, k, t, alpha_mode, alpha_k, static_cast<int32_t*>(sa.dev),
                            static_cast<uint8_t*>(sm.dev), st)))
    return rc;
  if ((rc = sa.writeback(sizeof(int32_t)))) return rc;
  if ((rc = sm.writeback(n))) return rc;
  ILS_CU(cudaStreamSynchronize(st));
  return ILS_OK;
}

}  // extern "C"
