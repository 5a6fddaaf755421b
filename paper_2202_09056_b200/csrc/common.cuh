// common.cuh -- error plumbing, device buffers and launch helpers shared by
// the solve kernels (solve.cu), the setup kernels (setup.cu) and the host
// runtime (hierarchy.cu, capi.cu).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>

#include "samg_b200.h"

namespace samgb {

// Typed error carrying a samg_status; thrown by host code, translated at
// the C-ABI edge (capi.cu).  Mirrors samg::error's hierarchy by code.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string &msg) { throw Error(code, msg); }

inline void cuda_check(cudaError_t e, const char *what, const char *file, int line) {
    if (e == cudaSuccess) return;
    char buf[512];
    snprintf(buf, sizeof buf, "%s failed: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
    throw Error(e == cudaErrorMemoryAllocation ? SAMG_OUT_OF_MEMORY : SAMG_CUDA_ERROR, buf);
}
#define CK(x) ::samgb::cuda_check((x), #x, __FILE__, __LINE__)
#define CK_LAUNCH() ::samgb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Device error word written by kernels that detect reference exceptions
// (zero filtered diagonal, singular pivot, ...).  First code wins.
struct DevError {
    int code;
    int64_t where;
};

// RAII device buffer (stream-ordered allocation).
template <class T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    explicit DevBuf(size_t count, cudaStream_t st = nullptr) { alloc(count, st); }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DevBuf &operator=(DevBuf &&o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count, cudaStream_t st = nullptr) {
        release();
        s = st;
        n = count;
        if (count) CK(cudaMallocAsync(&p, count * sizeof(T), st));
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
    T *get() const { return p; }
};

constexpr int kWarp = 32;

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// Host -> device copy on stream s; large pageable sources are staged through
// a pinned buffer pool by parallel host threads (hostcopy.cpp).
void h2d(void *dst, const void *src, size_t bytes, cudaStream_t s);
// int64 -> int32 staged copy; false if a value lies outside [0, bound)
bool h2d_narrow(int32_t *dst, const int64_t *src, size_t count, int64_t bound, cudaStream_t s);
// small (<= 256 B) pinned host objects from a process-wide slab pool
void *pinned_small_alloc(size_t bytes);
void pinned_small_free(void *p);

// Per-device cache of an int computed once per device (function attributes
// such as the dynamic shared-memory opt-in and cluster limits are per
// device: a value cached per process would leave a second device's kernels
// un-opted-in).  Racing first calls on one device both compute f(); harmless.
constexpr int kMaxDevices = 64;
struct DeviceCache {
    std::atomic<int> v[kMaxDevices];
    DeviceCache() { for (auto &x : v) x.store(INT_MIN, std::memory_order_relaxed); }
    template <class F>
    int get(F &&f) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
        std::atomic<int> &slot = v[dev & (kMaxDevices - 1)];
        int x = slot.load(std::memory_order_acquire);
        if (x == INT_MIN) {
            x = f();
            slot.store(x, std::memory_order_release);
        }
        return x;
    }
};

// SM count of the current device (cached per device).
int sm_count();

// NVTX range for the lifetime of the object (setup phases, solves): shows
// in Nsight Systems / ncu --nvtx; header-only NVTX v3, no-op without a tool.
struct NvtxScope {
    explicit NvtxScope(const char *name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
    NvtxScope(const NvtxScope &) = delete;
    NvtxScope &operator=(const NvtxScope &) = delete;
};

} // namespace samgb
