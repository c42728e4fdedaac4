// pp_nccl.h -- NCCL, resolved at run time.
//
// The sharded engine (pp_sharded.cuh) moves strings between GPUs with NCCL
// point-to-point calls and combines scalars with NCCL all-reduces.  The
// library is opened on first use (dlopen of libnccl.so.2: the copy a host
// process already loaded -- e.g. PyTorch's -- or the system one), so
// libppgpu.so has no link-time NCCL dependency and single-GPU use never
// touches it.  Only the types come from <nccl.h>.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

namespace ppgpu {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;

  static NcclApi& get() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] { api.load(); });
    if (!api.error.empty()) throw std::runtime_error(api.error);
    return api;
  }

 private:
  void load() {
    // one NCCL per process: the copy already loaded (e.g. PyTorch's), else
    // PP_NCCL_LIBRARY (the Python package points it at the wheel PyTorch
    // links, so a later `import torch` finds the same soname loaded), else
    // the loader's search path
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    const char* env = std::getenv("PP_NCCL_LIBRARY");
    if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      if (h) break;
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) {
      error = std::string("NCCL not found (dlopen libnccl.so.2): ") + dlerror();
      return;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p && error.empty()) error = std::string("NCCL symbol missing: ") + n;
      return p;
    };
    GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(sym("ncclGetUniqueId"));
    CommInitRank = reinterpret_cast<decltype(CommInitRank)>(sym("ncclCommInitRank"));
    CommDestroy = reinterpret_cast<decltype(CommDestroy)>(sym("ncclCommDestroy"));
    CommAbort = reinterpret_cast<decltype(CommAbort)>(sym("ncclCommAbort"));
    AllReduce = reinterpret_cast<decltype(AllReduce)>(sym("ncclAllReduce"));
    Send = reinterpret_cast<decltype(Send)>(sym("ncclSend"));
    Recv = reinterpret_cast<decltype(Recv)>(sym("ncclRecv"));
    GroupStart = reinterpret_cast<decltype(GroupStart)>(sym("ncclGroupStart"));
    GroupEnd = reinterpret_cast<decltype(GroupEnd)>(sym("ncclGroupEnd"));
    GetErrorString = reinterpret_cast<decltype(GetErrorString)>(sym("ncclGetErrorString"));
  }
};

#define PP_NCCL(x)                                                                                      \
  do {                                                                                                  \
    ncclResult_t r_ = (x);                                                                              \
    if (r_ != ncclSuccess)                                                                              \
      throw EngineError(PP_ERR_INTERNAL, std::string("NCCL: ") + NcclApi::get().GetErrorString(r_) + " at " + #x); \
  } while (0)

}  // namespace ppgpu
