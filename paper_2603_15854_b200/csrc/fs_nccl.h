// fs_nccl.h -- NCCL entry points of the library, resolved at run time (host only).
//
// fs_comm_init / fs_sample_tp (include/flashsample.h) use NCCL for the all-gather of the B x 12-byte
// shard summaries (Alg. A.4 line 4).  The library does not link libnccl: it resolves the few
// symbols it needs from the NCCL already loaded in the process (torch's pip NCCL, RTLD_NOLOAD), else
// from $FS_NCCL_LIB, else from the pip NCCL found at build time, else from libnccl.so.2 on the loader
// path -- so it loads (and every other entry point works) on machines without NCCL; fs_comm_init
// then fails with FS_ERR_UNSUPPORTED.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>

namespace fs {

struct NcclApi {
  bool ok = false;
  const char* why = "not loaded";
  ncclResult_t (*GetVersion)(int*) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // Order matters: a process that later imports torch must end up with torch's NCCL, because a
    // second libnccl.so.2 loaded first would satisfy torch's soname and lack its newer symbols.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h && std::getenv("FS_NCCL_LIB")) h = dlopen(std::getenv("FS_NCCL_LIB"), RTLD_NOW);
#ifdef FS_NCCL_DEFAULT_PATH
    if (!h) h = dlopen(FS_NCCL_DEFAULT_PATH, RTLD_NOW);    // the pip NCCL torch links (build.py)
#endif
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) {
      api.why = "libnccl.so.2 not found (load torch.distributed's NCCL first or set FS_NCCL_LIB)";
      return;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      all = all && fn != nullptr;
    };
    sym(api.GetVersion, "ncclGetVersion");
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.CommAbort, "ncclCommAbort");
    sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
    sym(api.AllGather, "ncclAllGather");
    sym(api.GetErrorString, "ncclGetErrorString");
    api.ok = all;
    api.why = all ? "" : "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

}  // namespace fs
