// hostcopy.cpp -- host->device copies of pageable user arrays.
//
// The C-ABI takes plain host pointers (the reference's csr arrays), which
// are pageable: a direct cudaMemcpyAsync from them runs at ~11 GB/s on the
// B200 hosts (measured, scripts/h2d_probe.py) versus ~55 GB/s from pinned
// memory.  Large copies are therefore staged: T host threads each own two
// pinned chunk buffers, copy their chunks of the source into them
// (memcpy runs in parallel on the host) and issue the DMA from pinned
// memory on the caller's stream; a buffer is reused once the event recorded
// after its DMA has completed.  The pinned pool is allocated on first use
// and kept for the life of the process.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace samgb {

namespace {

constexpr size_t kChunk = 8u << 20;     // bytes per staging buffer
constexpr int kThreads = 16;  // upper bound; SAMG_H2D_THREADS (default min(12, cores - 2)) uses fewer
constexpr size_t kDirect = 4u << 20;    // below this: plain cudaMemcpyAsync

struct Pool {
    std::mutex mu;                       // one staged copy at a time
    bool ready = false;
    int device = -1;
    char *buf[kThreads][2] = {};
    cudaEvent_t ev[kThreads][2] = {};

    void init() {
        int dev = 0;
        CK(cudaGetDevice(&dev));
        if (ready && dev == device) return;
        release();
        for (int t = 0; t < kThreads; ++t)
            for (int b = 0; b < 2; ++b)
                CK(cudaEventCreateWithFlags(&ev[t][b], cudaEventDisableTiming));
        device = dev;
        ready = true;
    }
    // pin the buffers of the first T thread slots (before the copy threads
    // start: concurrent cudaHostAlloc calls serialise in the driver).  Only
    // the slots in use are pinned (cudaHostAlloc costs ~0.5 ms per MB in a
    // cold process; the pool used to pin all 16 x 2 slots)
    void pin(int T) {
        for (int t = 0; t < T; ++t)
            for (int b = 0; b < 2; ++b)
                if (!buf[t][b]) CK(cudaHostAlloc(reinterpret_cast<void **>(&buf[t][b]), kChunk, cudaHostAllocPortable));
    }
    char *slot(int t, int b) { return buf[t][b]; }
    void release() {
        for (int t = 0; t < kThreads; ++t)
            for (int b = 0; b < 2; ++b) {
                if (buf[t][b]) cudaFreeHost(buf[t][b]);
                if (ev[t][b]) cudaEventDestroy(ev[t][b]);
                buf[t][b] = nullptr;
                ev[t][b] = nullptr;
            }
        ready = false;
    }
};

Pool &pool() {
    static Pool *p = new Pool;  // never destroyed: outlives static CUDA teardown
    return *p;
}

} // namespace

void h2d(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return;
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, src) == cudaSuccess &&
                        (pa.type == cudaMemoryTypeHost || pa.type == cudaMemoryTypeDevice ||
                         pa.type == cudaMemoryTypeManaged);
    cudaGetLastError();
    if (bytes < kDirect || pinned) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    Pool &P = pool();
    std::lock_guard<std::mutex> lock(P.mu);
    P.init();
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const size_t nchunks = (bytes + kChunk - 1) / kChunk;
    // default: 12 staging threads, or all but two of the host's (C1 setup
    // on the 16-thread GPU hosts, scripts/upload_sweep.py: 4 / 8 / 12 / 16
    // threads -> 89.1 / 80.6 / 76.7 / 77.1 ms)
    static const int threads = [] {
        const char *e = std::getenv("SAMG_H2D_THREADS");
        const int hw = static_cast<int>(std::thread::hardware_concurrency());
        const int v = e ? std::atoi(e) : std::min(12, std::max(1, hw - 2));
        return std::min(kThreads, std::max(1, v));
    }();
    const int T = static_cast<int>(std::min<size_t>(threads, nchunks));
    P.pin(T);
    std::vector<std::exception_ptr> errs(T);
    auto work = [&](int t) {
        try {
            CK(cudaSetDevice(dev));
            int b = 0;
            for (size_t c = t; c < nchunks; c += T, b ^= 1) {
                const size_t off = c * kChunk, n = std::min(kChunk, bytes - off);
                CK(cudaEventSynchronize(P.ev[t][b]));  // previous DMA from this buffer done
                std::memcpy(P.slot(t, b), static_cast<const char *>(src) + off, n);
                CK(cudaMemcpyAsync(static_cast<char *>(dst) + off, P.buf[t][b], n,
                                   cudaMemcpyHostToDevice, s));
                CK(cudaEventRecord(P.ev[t][b], s));
            }
        } catch (...) {
            errs[t] = std::current_exception();
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto &x : th) x.join();
    for (auto &e : errs)
        if (e) std::rethrow_exception(e);
    // the pinned buffers are reused by the next call only after their
    // events; the caller's stream already orders the copies before its
    // next work
}

// int64 -> int32 host -> device copy with a range check (the scalar CSR
// column indices of samg_setup: half the PCIe bytes of the int64 array).
// The staging threads narrow while they copy into the pinned buffers;
// returns false if any value lies outside [0, bound).
bool h2d_narrow(int32_t *dst, const int64_t *src, size_t count, int64_t bound, cudaStream_t s) {
    if (count == 0) return true;
    constexpr size_t kElems = kChunk / sizeof(int32_t);
    auto narrow = [bound](int32_t *out, const int64_t *in, size_t n) {
        bool ok = true;
        for (size_t i = 0; i < n; ++i) {
            const int64_t v = in[i];
            ok &= (v >= 0) & (v < bound);
            out[i] = static_cast<int32_t>(v);
        }
        return ok;
    };
    if (count * sizeof(int64_t) < kDirect) {
        std::vector<int32_t> tmp(count);
        const bool ok = narrow(tmp.data(), src, count);
        CK(cudaMemcpyAsync(dst, tmp.data(), sizeof(int32_t) * count, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
        return ok;
    }
    Pool &P = pool();
    std::lock_guard<std::mutex> lock(P.mu);
    P.init();
    int dev = 0;
    CK(cudaGetDevice(&dev));
    const size_t nchunks = (count + kElems - 1) / kElems;
    static const int threads = [] {
        const char *e = std::getenv("SAMG_H2D_THREADS");
        const int hw = static_cast<int>(std::thread::hardware_concurrency());
        const int v = e ? std::atoi(e) : std::min(12, std::max(1, hw - 2));
        return std::min(kThreads, std::max(1, v));
    }();
    const int T = static_cast<int>(std::min<size_t>(threads, nchunks));
    P.pin(T);
    std::vector<std::exception_ptr> errs(T);
    std::vector<char> oks(T, 1);
    auto work = [&](int t) {
        try {
            CK(cudaSetDevice(dev));
            int b = 0;
            for (size_t c = t; c < nchunks; c += T, b ^= 1) {
                const size_t off = c * kElems, n = std::min(kElems, count - off);
                CK(cudaEventSynchronize(P.ev[t][b]));
                if (!narrow(reinterpret_cast<int32_t *>(P.slot(t, b)), src + off, n)) oks[t] = 0;
                CK(cudaMemcpyAsync(dst + off, P.buf[t][b], sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
                CK(cudaEventRecord(P.ev[t][b], s));
            }
        } catch (...) {
            errs[t] = std::current_exception();
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto &x : th) x.join();
    for (auto &e : errs)
        if (e) std::rethrow_exception(e);
    for (char o : oks)
        if (!o) return false;
    return true;
}

// Small pinned objects (CG scalar mirrors, ...): 256-byte slots carved
// from 1 MB pinned slabs, so a hierarchy setup does not pay cudaMallocHost
// (~2 ms each) for a few hundred bytes.
namespace {
constexpr size_t kSlot = 256, kSlab = 1u << 20;
struct SmallPool {
    std::mutex mu;
    std::vector<void *> free_slots;
};
SmallPool &small_pool() {
    static SmallPool *p = new SmallPool;  // slabs live for the process
    return *p;
}
} // namespace

void *pinned_small_alloc(size_t bytes) {
    if (bytes > kSlot) fail(SAMG_INVALID_ARGUMENT, "pinned_small_alloc: object too large");
    SmallPool &P = small_pool();
    std::lock_guard<std::mutex> lock(P.mu);
    if (P.free_slots.empty()) {
        char *slab = nullptr;
        CK(cudaHostAlloc(reinterpret_cast<void **>(&slab), kSlab, cudaHostAllocPortable));
        for (size_t o = 0; o < kSlab; o += kSlot) P.free_slots.push_back(slab + o);
    }
    void *p = P.free_slots.back();
    P.free_slots.pop_back();
    std::memset(p, 0, kSlot);
    return p;
}

void pinned_small_free(void *p) {
    if (!p) return;
    SmallPool &P = small_pool();
    std::lock_guard<std::mutex> lock(P.mu);
    P.free_slots.push_back(p);
}

} // namespace samgb
