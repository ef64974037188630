// comm.cu -- the library-owned NCCL communicator of a multi-GPU run.
//
// The multipole exchange of SURVEY §8(e): every rank runs P2M / M2M for its own source leaves
// only, and one ncclAllReduce(sum) over the per-level multipole tree gives every rank the full
// tree (M2M is linear, so the ranks' partial sums add up to the single-GPU multipoles).  NCCL is
// loaded at run time (dlopen "libnccl.so.2": the copy torch already loaded when there is one), so
// the library itself has no link-time NCCL dependency and loads on hosts without it.
#include <dlfcn.h>
#include <string.h>
#include <nccl.h>  // types only; every call goes through the dlsym'd table below

#include <mutex>
#include <string>

#include "fmm_internal.cuh"

namespace {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*GetVersion)(int*);
  bool ok;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api{};
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("dlopen libnccl.so.2: ") + dlerror();
      return;
    }
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.GetVersion = (decltype(api.GetVersion))dlsym(h, "ncclGetVersion");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.GetErrorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

int nccl_fail(const char* what, ncclResult_t r) {
  fmm_set_error_message(std::string(what) + ": " + nccl().GetErrorString(r));
  return FMM_ENCCL;
}

}  // namespace

struct fmm_comm_s {
  ncclComm_t comm;
  int32_t rank, nranks;
};

int fmm_comm_allreduce_sum_f64(fmm_comm_t c, double* buf, size_t count, cudaStream_t s) {
  if (!c) return FMM_EBADCFG;
  if (count == 0) return FMM_OK;
  ncclResult_t r = nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, s);
  if (r != ncclSuccess) return nccl_fail("ncclAllReduce", r);
  return FMM_OK;
}

int32_t fmm_comm_nranks(fmm_comm_t c) { return c ? c->nranks : 0; }
int32_t fmm_comm_rank(fmm_comm_t c) { return c ? c->rank : -1; }

extern "C" {

int fmm_comm_unique_id(void* id) {
  if (!id) return FMM_EBADCFG;
  const NcclApi& a = nccl();
  if (!a.ok) {
    fmm_set_error_message(a.why);
    return FMM_ENCCL;
  }
  ncclUniqueId u;
  ncclResult_t r = a.GetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
  static_assert(sizeof(ncclUniqueId) == FMM_COMM_ID_BYTES, "ncclUniqueId size");
  memcpy(id, &u, sizeof(u));
  return FMM_OK;
}

int fmm_comm_init(const void* id, int32_t nranks, int32_t rank, fmm_comm_t* out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return FMM_EBADCFG;
  *out = nullptr;
  const NcclApi& a = nccl();
  if (!a.ok) {
    fmm_set_error_message(a.why);
    return FMM_ENCCL;
  }
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  ncclResult_t r = a.CommInitRank(&c, nranks, u, rank);
  if (r != ncclSuccess) return nccl_fail("ncclCommInitRank", r);
  fmm_comm_s* h = new fmm_comm_s{c, rank, nranks};
  *out = h;
  return FMM_OK;
}

int fmm_comm_destroy(fmm_comm_t c) {
  if (!c) return FMM_OK;
  ncclResult_t r = nccl().CommDestroy(c->comm);
  delete c;
  if (r != ncclSuccess) return nccl_fail("ncclCommDestroy", r);
  return FMM_OK;
}

int fmm_nccl_version(void) {
  const NcclApi& a = nccl();
  int v = 0;
  if (!a.ok || !a.GetVersion || a.GetVersion(&v) != ncclSuccess) return 0;
  return v;
}

}  // extern "C"
