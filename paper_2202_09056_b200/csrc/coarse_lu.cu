// coarse_lu.cu -- the reference's own coarse solver, dense_lu
// (hierarchy.hpp:86-129), bit-exact: partially pivoted LU in the reference's
// k-i-j order and the two triangular sweeps in its summation order.
//
// The default coarse solve is the explicit inverse (coarse.cu) applied as one
// GEMV per V-cycle.  When the coarse operator is numerically singular (cond
// ~1e16 even after equilibration -- e.g. a heterogeneous cantilever whose
// filtered prolongator diagonal nearly cancels, leaving coarse diagonal
// entries of 1e28 next to 0.05), the solution of A_c u = f is not determined
// by fp64 data: the inverse's answer and the LU answer differ at O(1), and
// only the latter reproduces the reference's preconditioner (and its CG
// convergence).  The hierarchy then switches to this solver
// (Hierarchy::coarse_lu), which returns exactly the reference's u.
//
// Cost: the factorization is 2 launches per column (setup); per V-cycle the
// forward sweep is column-oriented (n barrier steps: row i receives its
// terms s -= L_ij u_j in ascending j, the reference's order), the backward
// sweep is the reference's row recurrence, a sequential chain of n^2/2
// dependent subtractions (~8 cycles each) -- used only up to kLuMaxN.
// Compiled with --fmad=false; explicit _rn intrinsics keep the order.
#include <algorithm>
#include <vector>

#include "kernels.cuh"

namespace samgb {

namespace {

__global__ void k_lu_scatter(int nrows, const int *ptr, const int *col, const double *val,
                             int64_t ld, double *X) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    for (int j = ptr[i]; j < ptr[i + 1]; ++j)
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                X[(3 * static_cast<int64_t>(i) + r) * ld + 3 * static_cast<int64_t>(col[j]) + c] =
                    val[9 * static_cast<int64_t>(j) + 3 * r + c];
}

// Step k (hierarchy.hpp:91-102): p = first row of the largest |a_ik|, i >= k;
// swap rows k and p (whole rows); d = a_kk, singular below 1e-300; 1/d.
__global__ void __launch_bounds__(1024) k_lu_pivot(int n, int64_t ld, int k, double *X,
                                                   int64_t *piv, double *dinv, DevError *err) {
    __shared__ double bv[32];
    __shared__ int bi[32];
    __shared__ int P;
    // sequential rule "if (|a_ik| > |a_pk|) p = i" = first index of the max
    double best = -1.0;
    int b = k;
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
        const double v = fabs(X[static_cast<int64_t>(i) * ld + k]);
        if (v > best) { best = v; b = i; }
    }
    for (int off = 16; off >= 1; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int oi = __shfl_xor_sync(0xffffffffu, b, off);
        if (ov > best || (ov == best && oi < b)) { best = ov; b = oi; }
    }
    if (threadIdx.x % 32 == 0) { bv[threadIdx.x / 32] = best; bi[threadIdx.x / 32] = b; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double bb = bv[0];
        int ib = bi[0];
        for (int w = 1; w < static_cast<int>(blockDim.x / 32); ++w)
            if (bv[w] > bb || (bv[w] == bb && bi[w] < ib)) { bb = bv[w]; ib = bi[w]; }
        // the sequential scan keeps p = k unless a strictly larger entry exists
        if (!(bb > fabs(X[static_cast<int64_t>(k) * ld + k]))) ib = k;
        P = ib;
        piv[k] = ib;
    }
    __syncthreads();
    const int p = P;
    if (p != k)
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            double *a = X + static_cast<int64_t>(k) * ld + j, *c = X + static_cast<int64_t>(p) * ld + j;
            const double t = *a;
            *a = *c;
            *c = t;
        }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double d = X[static_cast<int64_t>(k) * ld + k];
        if (fabs(d) < 1e-300 && atomicCAS(&err->code, 0, SAMG_ERROR) == 0) err->where = k;
        *dinv = __ddiv_rn(1.0, d);
    }
}

// Step k, rows i > k (hierarchy.hpp:103-108): l = a_ik * inv; a_ij -= l a_kj
// for j > k; a_ik = l.  One CTA per row.
__global__ void __launch_bounds__(256) k_lu_update(int n, int64_t ld, int k, double *X,
                                                   const double *dinv) {
    const int i = k + 1 + blockIdx.x;
    double *ri = X + static_cast<int64_t>(i) * ld;
    const double *rk = X + static_cast<int64_t>(k) * ld;
    const double l = __dmul_rn(ri[k], *dinv);
    for (int j = k + 1 + threadIdx.x; j < n; j += blockDim.x) ri[j] = __dsub_rn(ri[j], __dmul_rn(l, rk[j]));
    __syncthreads();
    if (threadIdx.x == 0) ri[k] = l;
}

// L transposed (column-major unit lower part) for the column-oriented sweep
__global__ void k_lu_lt(int n, int64_t ld, const double *X, double *Lt) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
         e < static_cast<int64_t>(n) * n; e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / n, i = e - j * n;  // Lt[j*n + i] = L(i, j)
        Lt[e] = i > j ? X[i * ld + j] : 0.0;
    }
}

// solve (hierarchy.hpp:113-129), one CTA: u = P f; forward u_i -= L_ij u_j
// (ascending j, column-oriented: one barrier per j); backward
// u_i = (u_i - sum_{j>i} U_ij u_j) / U_ii, the sum ascending in j -- one
// sequential chain per row (lane 0), the next row staged by the other warps.
constexpr int kLuThreads = 1024;

__global__ void __launch_bounds__(kLuThreads) k_lu_solve(int n, int64_t ld, const double *__restrict__ X,
        const double *__restrict__ Lt, const int64_t *__restrict__ perm,
        const double *__restrict__ f, double *__restrict__ u) {
    extern __shared__ double lsm[];
    double *us = lsm, *row0 = lsm + n, *row1 = lsm + 2 * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) us[i] = f[perm[i]];
    __syncthreads();
    for (int j = 0; j + 1 < n; ++j) {
        const double uj = us[j];
        const double *lc = Lt + static_cast<int64_t>(j) * n;
        for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x)
            us[i] = __dsub_rn(us[i], __dmul_rn(lc[i], uj));
        __syncthreads();
    }
    // backward: row i staged into row buffers (double-buffered)
    for (int q = threadIdx.x; q < n; q += blockDim.x) row0[q] = X[static_cast<int64_t>(n - 1) * ld + q];
    __syncthreads();
    for (int i = n - 1; i >= 0; --i) {
        double *cur = ((n - 1 - i) & 1) ? row1 : row0, *nxt = ((n - 1 - i) & 1) ? row0 : row1;
        if (threadIdx.x >= 32 && i > 0)
            for (int q = threadIdx.x - 32; q < n; q += blockDim.x - 32)
                nxt[q] = X[static_cast<int64_t>(i - 1) * ld + q];
        if (threadIdx.x == 0) {
            double s = us[i];
#pragma unroll 8
            for (int j = i + 1; j < n; ++j) s = __dsub_rn(s, __dmul_rn(cur[j], us[j]));
            us[i] = __ddiv_rn(s, cur[i]);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) u[i] = us[i];
}

} // namespace

void dense_lu_ref(const Bsr3 &A, CoarseLu &lu, DevError *err, cudaStream_t s) {
    const int64_t n = 3 * A.nrows;
    if (n > kLuMaxN) fail(SAMG_UNSUPPORTED, "dense_lu: coarse dimension above the exact-LU limit");
    const int64_t ld = n;
    lu.n = n;
    lu.X.alloc(n * ld + 1, s);
    lu.Lt.alloc(n * n + 1, s);
    lu.perm.alloc(n + 1, s);
    if (n == 0) return;
    DevBuf<int64_t> piv(n, s);
    DevBuf<double> dinv(1, s);
    CK(cudaMemsetAsync(lu.X.p, 0, sizeof(double) * n * ld, s));
    k_lu_scatter<<<ceil_div(A.nrows, 128), 128, 0, s>>>(static_cast<int>(A.nrows), A.ptr.p, A.col.p,
                                                       A.val.p, ld, lu.X.p);
    for (int64_t k = 0; k < n; ++k) {
        k_lu_pivot<<<1, 1024, 0, s>>>(static_cast<int>(n), ld, static_cast<int>(k), lu.X.p, piv.p,
                                      dinv.p, err);
        if (k + 1 < n)
            k_lu_update<<<static_cast<int>(n - k - 1), 256, 0, s>>>(static_cast<int>(n), ld,
                                                                   static_cast<int>(k), lu.X.p, dinv.p);
    }
    CK_LAUNCH();
    k_lu_lt<<<std::max(1, std::min(4096, ceil_div(n * n, 256))), 256, 0, s>>>(static_cast<int>(n), ld,
                                                                              lu.X.p, lu.Lt.p);
    CK_LAUNCH();
    // the solve's row swaps u[k] <-> u[piv[k]], k ascending, composed on the
    // host into one gather u[k] = f[perm[k]]
    std::vector<int64_t> hp(n), hperm(n);
    CK(cudaMemcpyAsync(hp.data(), piv.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int64_t k = 0; k < n; ++k) hperm[k] = k;
    for (int64_t k = 0; k < n; ++k) std::swap(hperm[k], hperm[std::min<int64_t>(std::max<int64_t>(hp[k], 0), n - 1)]);
    CK(cudaMemcpyAsync(lu.perm.p, hperm.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));  // hperm goes out of scope
    check_dev_error(err, s);
}

void launch_lu_solve(const CoarseLu &lu, const double *f, double *u, cudaStream_t s) {
    const int n = static_cast<int>(lu.n);
    if (n == 0) return;
    const int smem = 3 * n * static_cast<int>(sizeof(double));
    static DeviceCache attr;
    attr.get([] {
        CK(cudaFuncSetAttribute(k_lu_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                3 * kLuMaxN * static_cast<int>(sizeof(double))));
        return 1;
    });
    k_lu_solve<<<1, kLuThreads, smem, s>>>(n, lu.n, lu.X.p, lu.Lt.p, lu.perm.p, f, u);
    CK_LAUNCH();
}

} // namespace samgb
