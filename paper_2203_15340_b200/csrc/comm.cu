// comm.cu -- row-sharded handles over NCCL.
//
// One process per GPU; rank r holds a row block [A1_r; A2_r] of A. Everything the SP method
// needs from A is a sum over rows, so a sharded handle computes its local partial and sums it
// across ranks with one NCCL all-reduce on the handle's stream:
//   Gram     A1^T A1 = sum_r A1_r^T A1_r                  (once, before the Cholesky)
//   norms    N_j = sum_r ||A1_r(:, j)||^2                   (once, at create; SP-SCD diagonal)
//   c_k      A1^T b1 + A2^T (A2 x - b2) = sum_r (...)_r      (n doubles per outer step)
//   g        A^T J (b - A x) = sum_r (...)_r                (correction form, RR)
// After each reduction every rank holds bitwise the same vector, runs the same P apply / SP-SCD
// inner solve, and so takes the same stop decision. NCCL is loaded with dlopen on first use, so
// libils.so does not depend on it unless a communicator is created.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "common.cuh"
#include "ils_internal.h"

namespace ils {
namespace {

struct NcclApi {
  bool tried = false, ok = false;
  void* lib = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.tried) return api;
  api.tried = true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    api.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (api.lib) break;
  }
  if (!api.lib) return api;
  api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(api.lib, "ncclGetUniqueId"));
  api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(api.lib, "ncclCommInitRank"));
  api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(api.lib, "ncclCommDestroy"));
  api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(api.lib, "ncclAllReduce"));
  api.getErrorString = reinterpret_cast<decltype(api.getErrorString)>(dlsym(api.lib, "ncclGetErrorString"));
  api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce && api.getErrorString;
  return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
  set_error(std::string(what) + ": " + nccl().getErrorString(r));
  return ILS_ERR_CUDA;
}

}  // namespace

int allreduce_sum(Handle& h, double* buf, int64_t count) {
  if (!h.comm || count <= 0) return ILS_OK;
  const ncclResult_t r = nccl().allReduce(buf, buf, (size_t)count, ncclDouble, ncclSum,
                                          static_cast<ncclComm_t>(h.comm->nccl), h.stream);
  if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
  count_launch();
  return ILS_OK;
}

}  // namespace ils

using namespace ils;

int ils_comm_unique_id(void* id_out) {
  if (!id_out) {
    set_error("ils_comm_unique_id: NULL argument");
    return ILS_ERR_ARG;
  }
  if (!nccl().ok) {
    set_error("ils_comm_unique_id: NCCL (libnccl.so.2) could not be loaded");
    return ILS_ERR_UNSUPPORTED;
  }
  ncclUniqueId id;
  const ncclResult_t r = nccl().getUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == ILS_COMM_ID_BYTES, "ncclUniqueId size");
  std::memcpy(id_out, &id, sizeof(id));
  return ILS_OK;
}

int ils_comm_create(const void* id, int nranks, int rank, ils_comm* out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("ils_comm_create: need id, out, nranks >= 1, 0 <= rank < nranks");
    return ILS_ERR_ARG;
  }
  *out = nullptr;
  if (!nccl().ok) {
    set_error("ils_comm_create: NCCL (libnccl.so.2) could not be loaded");
    return ILS_ERR_UNSUPPORTED;
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  const ncclResult_t r = nccl().commInitRank(&c, nranks, uid, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
  ils_comm_s* cm = new ils_comm_s();
  cm->nccl = c;
  cm->nranks = nranks;
  cm->rank = rank;
  *out = cm;
  return ILS_OK;
}

void ils_comm_destroy(ils_comm c) {
  if (!c) return;
  if (c->nccl && nccl().ok) nccl().commDestroy(static_cast<ncclComm_t>(c->nccl));
  delete c;
}
