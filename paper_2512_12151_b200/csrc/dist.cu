// Communicator of the row-partitioned PCG (internal.cuh, ibf.h "row-
// partitioned PCG"): NCCL across processes (one GPU each), loaded at run
// time so the library needs no NCCL to load, or "local" — every partition in
// this process (pcg.cu does those exchanges as device copies).
//
// The reference is single-process numpy; this replaces the in-process
// matvec / pcg_solve (intact/sparse.py:64-73, :99-150) when one scene is
// spread over several GPUs.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "internal.cuh"
#include "system.cuh"

namespace ibf {
namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the process's NCCL (torch loads libnccl.so.2 for its "nccl" backend)
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.AllGather &&
             api.GetErrorString;
  });
  return api;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return IBF_OK;
  set_error(std::string(what) + ": " + nccl().GetErrorString(r));
  return IBF_ERR_CUDA;
}

}  // namespace

int dist_allreduce_sum(ibf_dist* d, double* buf, int count, cudaStream_t s) {
  if (d->local || d->world == 1) return IBF_OK;
  return nccl_check(nccl().AllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, (ncclComm_t)d->comm, s),
                    "ncclAllReduce");
}

int dist_allgather(ibf_dist* d, const double* send, double* recv, size_t count_per_rank, cudaStream_t s) {
  if (d->local || d->world == 1) return IBF_OK;
  return nccl_check(nccl().AllGather(send, recv, count_per_rank, ncclDouble, (ncclComm_t)d->comm, s),
                    "ncclAllGather");
}

}  // namespace ibf

using namespace ibf;

extern "C" int ibf_dist_unique_id(void* out128) {
  if (!out128) {
    set_error("ibf_dist_unique_id: null output");
    return IBF_ERR_BAD_ARG;
  }
  if (!nccl().ok) {
    set_error("ibf_dist_unique_id: libnccl.so.2 not loadable");
    return IBF_ERR_CUDA;
  }
  ncclUniqueId id;
  IBF_TRY(nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId"));
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
  return IBF_OK;
}

extern "C" int ibf_dist_create(int rank, int world, const void* id128, ibf_dist** out) {
  if (!out || !id128 || world < 1 || rank < 0 || rank >= world) {
    set_error("ibf_dist_create: bad arguments");
    return IBF_ERR_BAD_ARG;
  }
  ibf_dist* d = new ibf_dist();
  d->rank = rank;
  d->world = world;
  d->local = false;
  if (world > 1) {
    if (!nccl().ok) {
      delete d;
      set_error("ibf_dist_create: libnccl.so.2 not loadable");
      return IBF_ERR_CUDA;
    }
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm = nullptr;
    const int st = nccl_check(nccl().CommInitRank(&comm, world, id, rank), "ncclCommInitRank");
    if (st != IBF_OK) {
      delete d;
      return st;
    }
    d->comm = comm;
  }
  *out = d;
  return IBF_OK;
}

extern "C" int ibf_dist_create_local(int parts, ibf_dist** out) {
  if (!out || parts < 1) {
    set_error("ibf_dist_create_local: parts must be >= 1");
    return IBF_ERR_BAD_ARG;
  }
  ibf_dist* d = new ibf_dist();
  d->world = parts;
  d->local = true;
  *out = d;
  return IBF_OK;
}

extern "C" void ibf_dist_destroy(ibf_dist* d) {
  if (!d) return;
  if (d->comm && nccl().ok) nccl().CommDestroy((ncclComm_t)d->comm);
  delete d;
}

extern "C" int ibf_system_set_dist(ibf_system* s, ibf_dist* d) {
  if (!s) {
    set_error("ibf_system_set_dist: null system");
    return IBF_ERR_BAD_ARG;
  }
  s->dist = d;
  return IBF_OK;
}
