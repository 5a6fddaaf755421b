// Microbenchmark: cost of cluster.sync() and __syncthreads() per call for
// cluster sizes 1..16 (one cluster on the GPU), 512 threads per CTA.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, int mode, double *out) {
    cg::cluster_group cl = cg::this_cluster();
    double acc = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        if (mode == 0) cl.sync();
        else if (mode == 1) __syncthreads();
        else { cl.barrier_arrive(); cl.barrier_wait(); }
        acc += 1.0;
    }
    if (acc < 0) out[0] = acc;
}

int main() {
    double *out;
    cudaMalloc(&out, 8);
    cudaFuncSetAttribute(k_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const int iters = 20000;
    for (int mode = 0; mode < 3; ++mode)
        for (int C : {1, 2, 4, 8, 16}) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(C);
            cfg.blockDim = dim3(512);
            cudaLaunchAttribute at{};
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = C; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
            cfg.attrs = &at; cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, k_sync, 100, mode, out);
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            cudaLaunchKernelEx(&cfg, k_sync, iters, mode, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("mode %s C=%2d: %.3f us per call (%s)\n", mode == 0 ? "cl.sync      " : mode == 1 ? "syncthreads  " : "arrive+wait  ", C,
                   1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
