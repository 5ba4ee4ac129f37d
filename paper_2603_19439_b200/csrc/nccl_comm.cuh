// The library's own st_comm over NCCL (NVLink / NVSwitch inside one box): the
// sharded step's collectives enqueued straight on the session stream, with
// no host callback. NCCL is resolved at run time (dlopen of libnccl.so.2):
// in a process that already loaded NCCL (e.g. torch.distributed) the same
// instance is used; otherwise the system library. Only the types come from
// nccl.h, so the product library has no link-time NCCL dependency.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "common.cuh"

namespace stg {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!api.CommInitRank) throw CudaError("libnccl.so.2 unavailable: " + err);
  return api;
}

struct NcclCtx {
  ncclComm_t comm = nullptr;
  int rank = 0, size = 1;
};

inline int32_t nccl_allreduce_cb(void* ctx, double* buf, int64_t count, void* stream) {
  auto* c = static_cast<NcclCtx*>(ctx);
  return nccl_api().AllReduce(buf, buf, static_cast<size_t>(count), ncclFloat64, ncclSum, c->comm,
                              static_cast<cudaStream_t>(stream)) == ncclSuccess ? 0 : 1;
}

inline int32_t nccl_allgather_cb(void* ctx, const void* send, void* recv, int64_t bytes, void* stream) {
  auto* c = static_cast<NcclCtx*>(ctx);
  return nccl_api().AllGather(send, recv, static_cast<size_t>(bytes), ncclUint8, c->comm,
                              static_cast<cudaStream_t>(stream)) == ncclSuccess ? 0 : 1;
}

inline int32_t nccl_alltoallv_cb(void* ctx, const void* send, const int64_t* sb, void* recv, const int64_t* rb,
                                 void* stream) {
  auto* c = static_cast<NcclCtx*>(ctx);
  const NcclApi& api = nccl_api();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* s = static_cast<const char*>(send);
  char* r = static_cast<char*>(recv);
  int64_t so = 0, ro = 0;
  if (api.GroupStart() != ncclSuccess) return 1;
  for (int p = 0; p < c->size; ++p) {
    if (p == c->rank) {
      if (sb[p] != rb[p]) return 1;
      if (sb[p] && cudaMemcpyAsync(r + ro, s + so, static_cast<size_t>(sb[p]), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return 1;
    } else {
      if (sb[p] && api.Send(s + so, static_cast<size_t>(sb[p]), ncclUint8, p, c->comm, st) != ncclSuccess) return 1;
      if (rb[p] && api.Recv(r + ro, static_cast<size_t>(rb[p]), ncclUint8, p, c->comm, st) != ncclSuccess) return 1;
    }
    so += sb[p];
    ro += rb[p];
  }
  return api.GroupEnd() == ncclSuccess ? 0 : 1;
}

}  // namespace stg
