// comm.cpp -- serinv_comm_t: an NCCL communicator owned by the library, used for
// the one exchange step of the distributed method (the all-gather of the
// per-partition records, Alg. 3 l.8 P:413 and the Gather/Scatter of
// P:650, replaced by one all-gather).
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <mutex>

struct serinv_comm {
  ncclComm_t nccl = nullptr;
  int P = 0, rank = 0, device = 0;
};

namespace {

struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char *(*errorString)(ncclResult_t) = nullptr;
  bool ok = false;
};

NcclApi &api() {
  static NcclApi A;
  static std::once_flag once;
  std::call_once(once, [] {
    // prefer the NCCL already mapped into the process (torch's), else the loader's
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      fprintf(stderr, "serinv: NCCL not found (libnccl.so.2): %s\n", dlerror());
      return;
    }
    A.getUniqueId = (decltype(A.getUniqueId))dlsym(h, "ncclGetUniqueId");
    A.commInitRank = (decltype(A.commInitRank))dlsym(h, "ncclCommInitRank");
    A.commDestroy = (decltype(A.commDestroy))dlsym(h, "ncclCommDestroy");
    A.allGather = (decltype(A.allGather))dlsym(h, "ncclAllGather");
    A.errorString = (decltype(A.errorString))dlsym(h, "ncclGetErrorString");
    A.ok = A.getUniqueId && A.commInitRank && A.commDestroy && A.allGather && A.errorString;
  });
  return A;
}

int nccl_status(ncclResult_t r, const char *where) {
  if (r == ncclSuccess) return SERINV_OK;
  fprintf(stderr, "serinv: %s failed: %s\n", where, api().errorString ? api().errorString(r) : "?");
  return SERINV_ERR_NCCL;
}

}  // namespace

namespace serinv {
int comm_allgather_f64(serinv_comm_t c, const double *send, double *recv, size_t count, cudaStream_t stream) {
  if (!c) return SERINV_ERR_HANDLE;
  if (c->P == 1 && !c->nccl) {  // a communicator of one rank needs no NCCL
    if (send == recv) return SERINV_OK;
    return cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice, stream) == cudaSuccess
               ? SERINV_OK
               : SERINV_ERR_CUDA;
  }
  return nccl_status(api().allGather(send, recv, count, ncclDouble, c->nccl, stream), "ncclAllGather");
}
int comm_size(serinv_comm_t c) { return c ? c->P : 0; }
int comm_rank(serinv_comm_t c) { return c ? c->rank : -1; }
int comm_device(serinv_comm_t c) { return c ? c->device : -1; }
}  // namespace serinv

extern "C" {

int serinv_nccl_unique_id(unsigned char *id) {
  if (!id) return -1;
  if (!api().ok) return SERINV_ERR_NCCL;
  ncclUniqueId u;
  int rc = nccl_status(api().getUniqueId(&u), "ncclGetUniqueId");
  if (rc) return rc;
  static_assert(sizeof(u.internal) == SERINV_NCCL_ID_BYTES, "NCCL unique id size");
  memcpy(id, u.internal, SERINV_NCCL_ID_BYTES);
  return SERINV_OK;
}

int serinv_comm_init(serinv_comm_t *c, const unsigned char *id, int P, int rank, int cuda_device) {
  if (!c) return -1;
  *c = nullptr;
  if (P < 1) return -3;
  if (rank < 0 || rank >= P) return -4;
  if (cudaSetDevice(cuda_device) != cudaSuccess) return SERINV_ERR_CUDA;
  serinv_comm *k = new serinv_comm();
  k->P = P;
  k->rank = rank;
  k->device = cuda_device;
  if (id) {  // id == NULL is allowed for P == 1 only: no NCCL at all
    if (!api().ok) {
      delete k;
      return SERINV_ERR_NCCL;
    }
    ncclUniqueId u;
    memcpy(u.internal, id, SERINV_NCCL_ID_BYTES);
    int rc = nccl_status(api().commInitRank(&k->nccl, P, u, rank), "ncclCommInitRank");
    if (rc) {
      delete k;
      return rc;
    }
  } else if (P != 1) {
    delete k;
    return -2;
  }
  *c = k;
  return SERINV_OK;
}

int serinv_comm_destroy(serinv_comm_t c) {
  if (!c) return SERINV_ERR_HANDLE;
  int rc = SERINV_OK;
  if (c->nccl) rc = nccl_status(api().commDestroy(c->nccl), "ncclCommDestroy");
  delete c;
  return rc;
}

}  // extern "C"
