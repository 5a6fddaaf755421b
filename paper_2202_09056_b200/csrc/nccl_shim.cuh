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

#include <chrono>
#include <cstdlib>
#include <string>
#include <thread>

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
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t);
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *);
    ncclResult_t (*CommAbort)(ncclComm_t);
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
        a.AllGather = reinterpret_cast<decltype(a.AllGather)>(get("ncclAllGather"));
        a.CommGetAsyncError =
            reinterpret_cast<decltype(a.CommGetAsyncError)>(get("ncclCommGetAsyncError"));
        a.CommAbort = reinterpret_cast<decltype(a.CommAbort)>(get("ncclCommAbort"));
        return a;
    }();
    return api;
}

inline void nccl_check(ncclResult_t r, const char *what) {
    if (r != ncclSuccess && r != ncclInProgress)
        fail(SAMG_NCCL_ERROR, std::string(what) + " failed: " + nccl().GetErrorString(r));
}
#define NK(x) ::samgb::nccl_check((x), #x)

// Wait for stream s while polling the communicator for asynchronous errors
// (a dead or failed peer): a plain cudaStreamSynchronize would hang on an
// NCCL kernel that never completes.  On an error the communicator is
// aborted (its kernels return) and SAMG_NCCL_ERROR is raised.
inline void stream_wait(ncclComm_t comm, cudaStream_t s) {
    if (!comm) {
        CK(cudaStreamSynchronize(s));
        return;
    }
    for (int spin = 0;; ++spin) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) CK(q);
        ncclResult_t ar = ncclSuccess;
        NK(nccl().CommGetAsyncError(comm, &ar));
        if (ar != ncclSuccess && ar != ncclInProgress) {
            nccl().CommAbort(comm);
            fail(SAMG_NCCL_ERROR, std::string("NCCL asynchronous error: ") + nccl().GetErrorString(ar));
        }
        if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
}

} // namespace samgb
