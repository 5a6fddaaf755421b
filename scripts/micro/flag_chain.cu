// Microbenchmark: latency of a release/acquire flag hand-off chain between
// warps (row i waits for row i-1), the critical path of a sync-free sweep.
#include <cuda/atomic>
#include <cstdio>

__device__ int ld_relaxed(int *p) {
    cuda::atomic_ref<int, cuda::thread_scope_device> a(*p);
    return a.load(cuda::memory_order_relaxed);
}

template <int MODE>
__global__ void k_chain(int n, int *flags, int *counter, double *y) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(counter, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= n) return;
        if (t > 0) {
            if (lane == 0)
                while (ld_relaxed(flags + t - 1) == 0) {
                }
            __syncwarp();
            if (MODE >= 1) cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
        }
        double v = t > 0 ? __ldcg(y + t - 1) : 0.0;
        if (lane == 0) y[t] = v + 1.0;
        __syncwarp();
        if (lane == 0) {
            cuda::atomic_ref<int, cuda::thread_scope_device> a(flags[t]);
            if (MODE >= 2) a.store(1, cuda::memory_order_release);
            else { __threadfence(); a.store(1, cuda::memory_order_relaxed); }
        }
    }
}

int main() {
    const int n = 20000;
    int *flags, *counter;
    double *y;
    cudaMalloc(&flags, sizeof(int) * (n + 1));
    cudaMalloc(&counter, sizeof(int));
    cudaMalloc(&y, sizeof(double) * n);
    for (int grid : {1, 148, 296}) {
        for (int mode = 0; mode < 3; ++mode) {
            cudaMemset(flags, 0, sizeof(int) * (n + 1));
            cudaMemset(counter, 0, sizeof(int));
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            if (mode == 0) k_chain<0><<<grid, 256>>>(n, flags, counter, y);
            if (mode == 1) k_chain<1><<<grid, 256>>>(n, flags, counter, y);
            if (mode == 2) k_chain<2><<<grid, 256>>>(n, flags, counter, y);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double hy;
            cudaMemcpy(&hy, y + n - 1, 8, cudaMemcpyDeviceToHost);
            printf("grid %3d mode %d: %.3f us per hop (y=%g) %s\n", grid, mode, 1e3 * ms / n, hy,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
}
