// Microbenchmark: hand-off latency of a dependency chain (row t needs row t-1)
// when the VALUE itself is the flag.  y is pre-filled with a NaN sentinel that
// fp arithmetic never produces; the consumer polls y[t-1] with relaxed
// gpu-scope loads until it is no longer the sentinel -- one L2 round trip per
// poll and no fence on either side -- against the release/acquire flag
// hand-off (flag_chain.cu).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a value_chain.cu -o value_chain
#include <cuda/atomic>
#include <cstdint>
#include <cstdio>

constexpr unsigned long long kSent = 0xffffffffffffffffull;

__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rlx(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// MODE 0: flag + fence (flag_chain mode 0); MODE 1: value polling;
// MODE 2: value polling, 3 components per row (a 3x3-block sweep's y_i).
template <int MODE>
__global__ void k_chain(int n, int *flags, int *counter, unsigned long long *y) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(counter, 1);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= n) return;
        if (MODE == 0) {
            double v = 0.0;
            if (t > 0) {
                if (lane == 0) {
                    cuda::atomic_ref<int, cuda::thread_scope_device> a(flags[t - 1]);
                    while (a.load(cuda::memory_order_relaxed) == 0) {
                    }
                }
                __syncwarp();
                v = __longlong_as_double(__ldcg(reinterpret_cast<const long long *>(y) + t - 1));
            }
            if (lane == 0) {
                y[t] = __double_as_longlong(v + 1.0);
                __threadfence();
                cuda::atomic_ref<int, cuda::thread_scope_device> a(flags[t]);
                a.store(1, cuda::memory_order_relaxed);
            }
        } else if (MODE == 1) {
            double v = 0.0;
            if (t > 0 && lane == 0) {
                unsigned long long b;
                while ((b = ld_rlx(y + t - 1)) == kSent) {
                }
                v = __longlong_as_double(b);
            }
            if (lane == 0) st_rlx(y + t, __double_as_longlong(v + 1.0));
        } else {
            double v = 0.0;
            if (t > 0 && lane < 3) {
                unsigned long long b;
                while ((b = ld_rlx(y + 3LL * (t - 1) + lane)) == kSent) {
                }
                v = __longlong_as_double(b);
            }
            const double s = __shfl_sync(0xffffffffu, v, 0) + __shfl_sync(0xffffffffu, v, 1) +
                             __shfl_sync(0xffffffffu, v, 2);
            if (lane < 3) st_rlx(y + 3LL * t + lane, __double_as_longlong(s + 1.0));
        }
        __syncwarp();
    }
}

int main() {
    const int n = 20000;
    int *flags, *counter;
    unsigned long long *y;
    cudaMalloc(&flags, sizeof(int) * (n + 1));
    cudaMalloc(&counter, sizeof(int));
    cudaMalloc(&y, sizeof(unsigned long long) * 3 * n);
    for (int grid : {1, 148, 296}) {
        for (int mode = 0; mode < 3; ++mode) {
            float best = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
                cudaMemset(flags, 0, sizeof(int) * (n + 1));
                cudaMemset(counter, 0, sizeof(int));
                cudaMemset(y, 0xff, sizeof(unsigned long long) * 3 * n);
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
                if (ms < best) best = ms;
            }
            printf("grid %3d mode %d (%s): %.3f us per hop %s\n", grid, mode,
                   mode == 0 ? "flag+fence" : mode == 1 ? "value poll" : "3-value poll",
                   1e3 * best / n, cudaGetErrorString(cudaGetLastError()));
        }
    }
}
