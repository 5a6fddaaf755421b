// nccl_shim.cuh -- NCCL entry points resolved at run time.
//
// The library is not linked against libnccl: PyTorch ships its own
// libnccl.so.2 (a newer 2.x), and whichever copy is loaded first wins the
// soname for the whole process.  Linking ours would break `import torch`
// after `import paper_2202_09056_b200`.  Instead the first multi-GPU call
// resolves the functions from (1) a libnccl.so.2 already loaded in the
// process, (2) $SAMG_NCCL_LIB, (3) the default search path.  Only the
// types and constants of nccl.h are used at compile time (NCCL 2.x ABI).
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <string>

#include "common.cuh"

namespace samgb {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    const char *(*GetErrorString)(ncclResult_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t);
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t);
};

inline const NcclApi &nccl() {
    static NcclApi api = [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            if (const char *p = std::getenv("SAMG_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) fail(SAMG_NCCL_ERROR, std::string("cannot load libnccl.so.2: ") + dlerror());
        NcclApi a{};
        auto get = [&](const char *name) {
            void *f = dlsym(h, name);
            if (!f) fail(SAMG_NCCL_ERROR, std::string("libnccl.so.2 lacks ") + name);
            return f;
        };
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(get("ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(get("ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(get("ncclCommDestroy"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(get("ncclGetErrorString"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(get("ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(get("ncclGroupEnd"));
        a.Send = reinterpret_cast<decltype(a.Send)>(get("ncclSend"));
        a.Recv = reinterpret_cast<decltype(a.Recv)>(get("ncclRecv"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(get("ncclAllReduce"));
        a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(get("ncclBroadcast"));
        return a;
    }();
    return api;
}

} // namespace samgb
