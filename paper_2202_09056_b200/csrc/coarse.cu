// coarse.cu -- coarsest-level direct solver.
//
// The reference factors the coarsest matrix with a dense partially pivoted
// LU and solves with two triangular sweeps per V-cycle
// (dense_lu, hierarchy.hpp:86-129).  Triangular sweeps are sequential in n,
// so on the GPU the setup instead forms the explicit inverse once by
// Gauss-Jordan elimination with the same pivot rule (largest |a_ik|, first
// index on ties, error below 1e-300) and every V-cycle applies it as one
// bandwidth-bound dense GEMV (launch_dense_gemv in solve.cu).
#include "kernels.cuh"

namespace samgb {

namespace {

// scatter A (BSR3) into W = [A | I], row-major n x 2n (to_dense, csr.hpp:370-382)
__global__ void k_scatter(int nrows, const int *ptr, const int *col, const double *val,
                          int64_t n, double *W) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    const int64_t ld = 2 * n;
    for (int r = 0; r < 3; ++r) W[(3 * static_cast<int64_t>(i) + r) * ld + n + 3 * i + r] = 1.0;
    for (int j = ptr[i]; j < ptr[i + 1]; ++j)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                W[(3 * static_cast<int64_t>(i) + r) * ld + 3 * static_cast<int64_t>(col[j]) + c] =
                    val[9 * static_cast<int64_t>(j) + 3 * r + c];
}

// pivot search (first max |a_ik|, i >= k), row swap, row scale, save column k
__global__ void __launch_bounds__(1024) k_gj_pivot(int64_t n, int64_t k, double *W, double *fcol,
                                                   DevError *err) {
    __shared__ double bv[32];
    __shared__ int64_t bi[32];
    __shared__ int64_t piv;
    __shared__ double pval;
    const int64_t ld = 2 * n;
    double best = -1.0;
    int64_t besti = n;
    for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x) {
        const double v = fabs(W[i * ld + k]);
        if (v > best) { best = v; besti = i; }
    }
    for (int off = 16; off >= 1; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, besti, off);
        if (ov > best || (ov == best && oi < besti)) { best = ov; besti = oi; }
    }
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    if (l == 0) { bv[w] = best; bi[w] = besti; }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x / 32;
        best = l < nw ? bv[l] : -1.0;
        besti = l < nw ? bi[l] : n;
        for (int off = 16; off >= 1; off >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, best, off);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, besti, off);
            if (ov > best || (ov == best && oi < besti)) { best = ov; besti = oi; }
        }
        if (l == 0) { piv = besti; pval = W[besti * ld + k]; }
    }
    __syncthreads();
    const int64_t p = piv;
    if (!(fabs(pval) >= 1e-300)) {
        if (threadIdx.x == 0 && atomicCAS(&err->code, 0, SAMG_ERROR) == 0) err->where = k;
        return;
    }
    const double inv = 1.0 / pval;
    for (int64_t j = k + threadIdx.x; j < ld; j += blockDim.x) {
        const double a = W[k * ld + j], b = W[p * ld + j];
        W[p * ld + j] = a;
        W[k * ld + j] = b * inv;
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) fcol[i] = (i == k) ? 0.0 : W[i * ld + k];
}

__global__ void k_gj_elim(int64_t n, int64_t k, double *W, const double *fcol) {
    const int64_t ld = 2 * n;
    const int64_t i = blockIdx.y;
    const double f = fcol[i];
    if (f == 0.0) return;
    const double *rk = W + k * ld;
    double *ri = W + i * ld;
    for (int64_t j = k + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < ld;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        ri[j] = fma(-f, rk[j], ri[j]);
}

__global__ void k_copy_right(int64_t n, const double *W, double *Ainv) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n * n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e / n, j = e - i * n;
        Ainv[e] = W[i * 2 * n + n + j];
    }
}

} // namespace

void dense_inverse(const Bsr3 &A, DevBuf<double> &Ainv, DevError *err, cudaStream_t s) {
    const int64_t n = 3 * A.nrows;
    if (n > 65535) fail(SAMG_UNSUPPORTED, "dense coarse solve: coarsest level above 65535 unknowns");
    Ainv.alloc(n * n, s);
    if (n == 0) return;
    DevBuf<double> W(2 * n * n, s), fcol(n, s);
    CK(cudaMemsetAsync(W.p, 0, W.bytes(), s));
    k_scatter<<<ceil_div(A.nrows, 128), 128, 0, s>>>(static_cast<int>(A.nrows), A.ptr.p, A.col.p,
                                                    A.val.p, n, W.p);
    CK_LAUNCH();
    const int gx = static_cast<int>(std::min<int64_t>((2 * n + 255) / 256, 8));
    for (int64_t k = 0; k < n; ++k) {
        k_gj_pivot<<<1, 1024, 0, s>>>(n, k, W.p, fcol.p, err);
        k_gj_elim<<<dim3(gx, static_cast<unsigned>(n)), 256, 0, s>>>(n, k, W.p, fcol.p);
    }
    CK_LAUNCH();
    k_copy_right<<<ceil_div(n * n, 256) < 4096 ? ceil_div(n * n, 256) : 4096, 256, 0, s>>>(n, W.p, Ainv.p);
    CK_LAUNCH();
    check_dev_error(err, s);
}

} // namespace samgb
