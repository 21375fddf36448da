// nccl_shim.h -- NCCL loaded lazily with dlopen (first use: mr_nccl_unique_id /
// mr_comm_init).  Linking libnccl.so.2 at load time would pin whichever NCCL
// the loader finds first; if that is the system 2.27 and PyTorch (which needs
// its bundled 2.28) is imported afterwards, torch fails to resolve symbols.
// Resolving lazily binds to the NCCL already in the process when there is one
// (PyTorch's), else loads libnccl.so.2.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi& nccl_api()
{
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
#define MR_NCCL_SYM(field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name))
    MR_NCCL_SYM(GetUniqueId, "ncclGetUniqueId");
    MR_NCCL_SYM(CommInitRank, "ncclCommInitRank");
    MR_NCCL_SYM(CommDestroy, "ncclCommDestroy");
    MR_NCCL_SYM(GroupStart, "ncclGroupStart");
    MR_NCCL_SYM(GroupEnd, "ncclGroupEnd");
    MR_NCCL_SYM(Send, "ncclSend");
    MR_NCCL_SYM(Recv, "ncclRecv");
    MR_NCCL_SYM(AllReduce, "ncclAllReduce");
    MR_NCCL_SYM(AllGather, "ncclAllGather");
    MR_NCCL_SYM(GetErrorString, "ncclGetErrorString");
#undef MR_NCCL_SYM
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.GroupStart && a.GroupEnd &&
           a.Send && a.Recv && a.AllReduce && a.AllGather && a.GetErrorString;
    return a;
  }();
  return api;
}
