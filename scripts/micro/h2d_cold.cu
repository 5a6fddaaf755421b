// Host->device copies of a 972 MB pageable array (the drop-in setup's scalar
// CSR): cost of allocating pinned staging buffers (cold), staged copies,
// plain pageable cudaMemcpyAsync from 1 and from 12 threads.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
    const size_t bytes = 972ull << 20;
    char *src = static_cast<char *>(malloc(bytes));
    memset(src, 1, bytes);
    char *dst;
    cudaMalloc(&dst, bytes);
    cudaFree(0);
    double t = now();
    std::vector<char *> bufs(32);
    for (auto &b : bufs) cudaHostAlloc(reinterpret_cast<void **>(&b), 8 << 20, cudaHostAllocPortable);
    printf("cudaHostAlloc 32 x 8 MB: %.1f ms\n", (now() - t) * 1e3);
    t = now();
    for (auto &b : bufs) memset(b, 0, 8 << 20);
    printf("first touch of the pinned buffers: %.1f ms\n", (now() - t) * 1e3);
    t = now();
    char *big;
    cudaHostAlloc(reinterpret_cast<void **>(&big), 256 << 20, cudaHostAllocPortable);
    printf("cudaHostAlloc 1 x 256 MB: %.1f ms\n", (now() - t) * 1e3);
    for (int rep = 0; rep < 2; ++rep) {
        t = now();
        cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
        printf("pageable cudaMemcpy, 1 thread: %.1f ms\n", (now() - t) * 1e3);
    }
    for (int T : {4, 8, 12}) {
        for (int rep = 0; rep < 2; ++rep) {
            t = now();
            std::vector<std::thread> th;
            for (int k = 0; k < T; ++k)
                th.emplace_back([&, k] {
                    cudaStream_t s;
                    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
                    const size_t per = (bytes / T + 15) & ~size_t(15);
                    const size_t off = per * k, n = off < bytes ? std::min(per, bytes - off) : 0;
                    if (n) cudaMemcpyAsync(dst + off, src + off, n, cudaMemcpyHostToDevice, s);
                    cudaStreamSynchronize(s);
                    cudaStreamDestroy(s);
                });
            for (auto &x : th) x.join();
            printf("pageable cudaMemcpyAsync, %2d threads: %.1f ms\n", T, (now() - t) * 1e3);
        }
    }
    return 0;
}
