// Microbenchmark: cost of one grid-wide barrier of a cooperative grid (one
// CTA per SM), for the V-cycle tail kernel's barrier variants:
//   mode 0: relaxed poll + fence.acq_rel on both sides (k_vtail's)
//   mode 1: no fences (lower bound of the counter/flag protocol)
//   mode 2: cooperative_groups grid.sync()
//   mode 3: launch-to-launch: an empty kernel per "barrier" (stream order)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

template <int MODE>
__device__ __forceinline__ void gbar(unsigned *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned gen;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
        if (MODE == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        unsigned prev;
        asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(bar) : "memory");
        if (prev == gridDim.x - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen + 1) : "memory");
        } else {
            unsigned g2;
            do {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g2) : "l"(bar + 1) : "memory");
            } while (g2 == gen);
        }
        if (MODE == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

template <int MODE>
__global__ void k_bar(int iters, unsigned *bar, double *out) {
    double acc = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        if (MODE == 2) cg::this_grid().sync();
        else gbar<MODE>(bar);
        acc += 1.0;
    }
    if (acc < 0) out[0] = acc;
}
__global__ void k_empty(double *out) {
    if (threadIdx.x == 1000000) out[0] = 1.0;
}

template <int MODE>
float run(int sms, int threads, int iters, unsigned *bar, double *out) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    void *args[] = {&iters, &bar, &out};
    cudaLaunchCooperativeKernel((void *)k_bar<MODE>, sms, threads, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void *)k_bar<MODE>, sms, threads, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3f / iters;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned *bar;
    double *out;
    cudaMalloc(&bar, 8);
    cudaMemset(bar, 0, 8);
    cudaMalloc(&out, 8);
    const int iters = 2000;
    for (int threads : {256, 1024}) {
        printf("threads %4d  fenced %.3f us  unfenced %.3f us  cg.sync %.3f us\n", threads,
               run<0>(sms, threads, iters, bar, out), run<1>(sms, threads, iters, bar, out),
               run<2>(sms, threads, iters, bar, out));
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int k = 0; k < 10; ++k) k_empty<<<sms, 1024>>>(out);
    cudaEventRecord(a);
    for (int k = 0; k < iters; ++k) k_empty<<<sms, 1024>>>(out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("empty kernel back to back: %.3f us per launch\n", ms * 1e3f / iters);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
