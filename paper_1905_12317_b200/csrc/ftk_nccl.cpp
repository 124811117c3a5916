// NCCL glue of the C ABI: the cross-rank all-gather of per-image bests inside ftk_align (SURVEY 8(b),
// 8(e); north star (4): "templates sharded across GPUs, NCCL allgather of per-image bests over NVLink").
// libnccl.so.2 is opened at run time (dlopen) so that the library links no NCCL version of its own: in a
// PyTorch process the NCCL that torch already loaded is the one used.  Types come from nccl.h.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "ftk_nccl.h"

namespace ftk {
namespace {

struct NcclApi {
  bool tried = false, ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (a.tried) return a;
  a.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    a.err = std::string("libnccl.so.2 not found: ") + dlerror();
    return a;
  }
  auto sym = [&](const char* n) { return dlsym(h, n); };
  a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
  a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
  a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
  a.CommCount = reinterpret_cast<decltype(a.CommCount)>(sym("ncclCommCount"));
  a.CommUserRank = reinterpret_cast<decltype(a.CommUserRank)>(sym("ncclCommUserRank"));
  a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
  a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
  a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.CommCount && a.CommUserRank && a.AllGather &&
         a.GetErrorString;
  if (!a.ok) a.err = "libnccl.so.2 lacks a required symbol";
  return a;
}

int fail_nccl(NcclApi& a, ncclResult_t r, const char* what, std::string& msg) {
  msg = std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(r) : "NCCL error");
  return FTK_ENCCL;
}

}  // namespace

int nccl_unique_id(void* id_out, std::string& msg) {
  NcclApi& a = api();
  if (!a.ok) {
    msg = a.err;
    return FTK_ENCCL;
  }
  ncclUniqueId id;
  const ncclResult_t r = a.GetUniqueId(&id);
  if (r != ncclSuccess) return fail_nccl(a, r, "ncclGetUniqueId", msg);
  std::memcpy(id_out, &id, sizeof id);
  return FTK_OK;
}

int nccl_comm_create(const void* id_in, int world, int rank, void** comm_out, std::string& msg) {
  NcclApi& a = api();
  if (!a.ok) {
    msg = a.err;
    return FTK_ENCCL;
  }
  ncclUniqueId id;
  std::memcpy(&id, id_in, sizeof id);
  ncclComm_t c = nullptr;
  const ncclResult_t r = a.CommInitRank(&c, world, id, rank);
  if (r != ncclSuccess) return fail_nccl(a, r, "ncclCommInitRank", msg);
  *comm_out = c;
  return FTK_OK;
}

int nccl_comm_destroy(void* comm) {
  NcclApi& a = api();
  if (!a.ok || !comm) return FTK_OK;
  return a.CommDestroy(reinterpret_cast<ncclComm_t>(comm)) == ncclSuccess ? FTK_OK : FTK_ENCCL;
}

int nccl_comm_check(void* comm, int world, int rank, std::string& msg) {
  NcclApi& a = api();
  if (!a.ok) {
    msg = a.err;
    return FTK_ENCCL;
  }
  int n = 0, r = 0;
  ncclResult_t e = a.CommCount(reinterpret_cast<ncclComm_t>(comm), &n);
  if (e != ncclSuccess) return fail_nccl(a, e, "ncclCommCount", msg);
  e = a.CommUserRank(reinterpret_cast<ncclComm_t>(comm), &r);
  if (e != ncclSuccess) return fail_nccl(a, e, "ncclCommUserRank", msg);
  if (n != world || r != rank) {
    msg = "nccl_comm has " + std::to_string(n) + " ranks (this one " + std::to_string(r) + "), the plan says world " +
          std::to_string(world) + " rank " + std::to_string(rank);
    return FTK_EINVAL;
  }
  return FTK_OK;
}

int nccl_allgather_bests(void* comm, const void* send, void* recv, int64_t n_records, cudaStream_t s,
                         std::string& msg) {
  NcclApi& a = api();
  if (!a.ok) {
    msg = a.err;
    return FTK_ENCCL;
  }
  // 16-byte records as 4 int32 each; recv = [world][n_records]
  const ncclResult_t r = a.AllGather(send, recv, (size_t)n_records * 4, ncclInt32, reinterpret_cast<ncclComm_t>(comm), s);
  if (r != ncclSuccess) return fail_nccl(a, r, "ncclAllGather", msg);
  return FTK_OK;
}

}  // namespace ftk
