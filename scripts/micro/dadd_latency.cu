// Microbenchmark: dependent-chain latency of DADD / DMUL / DFMA and FADD on
// sm_100a (one thread, clock64).  Bounds the ILU(0) sweep's sequential
// subtraction chain (ilu.cu: 3 dependent DADDs per dependency).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a dadd_latency.cu -o dadd_latency
#include <cstdio>

template <int OP>
__global__ void k(double *out, float *outf, long long *cyc, double a, double b, int n) {
    double x = a;
    float xf = static_cast<float>(a);
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (OP == 0) x = __dsub_rn(x, b);
            if (OP == 1) x = __dmul_rn(x, b);
            if (OP == 2) x = __fma_rn(x, b, b);
            if (OP == 3) xf = __fsub_rn(xf, static_cast<float>(b));
        }
    }
    const long long t1 = clock64();
    out[0] = x;
    outf[0] = xf;
    cyc[0] = t1 - t0;
}

int main() {
    double *o; float *of; long long *c;
    cudaMalloc(&o, 8); cudaMalloc(&of, 4); cudaMalloc(&c, 8);
    const int n = 1 << 14;
    const char *names[] = {"DADD", "DMUL", "DFMA", "FADD"};
    for (int op = 0; op < 4; ++op) {
        if (op == 0) k<0><<<1, 1>>>(o, of, c, 1.0, 1e-300, n);
        if (op == 1) k<1><<<1, 1>>>(o, of, c, 1.0, 1.0000000001, n);
        if (op == 2) k<2><<<1, 1>>>(o, of, c, 1.0, 1e-300, n);
        if (op == 3) k<3><<<1, 1>>>(o, of, c, 1.0, 1e-30, n);
        long long h;
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%s dependent latency: %.2f cycles\n", names[op], static_cast<double>(h) / (16.0 * n));
    }
}
