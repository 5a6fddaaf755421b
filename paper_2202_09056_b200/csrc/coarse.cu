// coarse.cu -- coarsest-level direct solver.
//
// The reference factors the coarsest matrix with a dense partially pivoted
// LU and solves with two triangular sweeps per V-cycle
// (dense_lu, hierarchy.hpp:86-129).  Triangular sweeps are sequential in n,
// so on the GPU the setup instead forms the explicit inverse once and every
// V-cycle applies it as one bandwidth-bound dense GEMV (launch_dense_gemv in
// solve.cu).  Pivot rule as the reference: largest |a_ik| over the remaining
// rows (first index on ties); a pivot below 1e-300 raises samg::error
// ("dense_lu: singular coarse matrix").
//
// Blocked Gauss-Jordan on W = [A | I] (n x 2n, row-major), panel width kB:
//  1. the panel's kB columns (Y) plus an accumulator Z (n x kB) are reduced
//     by one cooperative kernel, 2 grid barriers per column (pivot search;
//     pivot-row broadcast), rows of Y/Z swapped physically;
//  2. the panel's row swaps are applied to the trailing columns of W;
//  3. the trailing columns get the rank-kB update
//     W[:, J] += (Z - E_K) W[K, J]  (one FP64 tiled GEMM),
// so the n^3 work streams W once per panel instead of once per column.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace samgb {

namespace {

constexpr int kB = 32;          // panel width
constexpr int kPT = 256;        // panel kernel threads per CTA

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

__global__ void k_panel_load(int64_t n, int64_t k0, int bk, const double *W, double *Pn) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n * 2 * kB;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e / (2 * kB);
        const int q = static_cast<int>(e - i * 2 * kB);
        Pn[e] = (q < bk) ? W[i * 2 * n + k0 + q] : 0.0;
    }
}

// Gauss-Jordan on the n x (Y | Z) panel; rows split into contiguous ranges
// per CTA.  piv[q] = pivot row of panel column q.
__global__ void __launch_bounds__(kPT) k_panel_gj(int64_t n, int64_t k0, int bk, double *Pn,
                                                   double *pval, int64_t *pidx, int64_t *piv,
                                                   DevError *err) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double prow[2 * kB], krow[2 * kB], rk[2 * kB], fs[64];
    __shared__ double wv[kPT / 32];
    __shared__ int64_t wi[kPT / 32];
    __shared__ int64_t s_p;
    __shared__ double s_v;
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = blockIdx.x * per, r1 = min(n, r0 + per);
    const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
    for (int q = 0; q < bk; ++q) {
        const int64_t k = k0 + q;
        // a. local argmax of |Y[i][q]| over own rows i >= k
        double best = -1.0;
        int64_t bi = n;
        for (int64_t i = max(r0, k) + threadIdx.x; i < r1; i += blockDim.x) {
            const double v = fabs(Pn[i * 2 * kB + q]);
            if (v > best) { best = v; bi = i; }
        }
        for (int off = 16; off >= 1; off >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, best, off);
            const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        }
        if (lane == 0) { wv[w] = best; wi[w] = bi; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int t = 1; t < kPT / 32; ++t)
                if (wv[t] > wv[0] || (wv[t] == wv[0] && wi[t] < wi[0])) { wv[0] = wv[t]; wi[0] = wi[t]; }
            pval[blockIdx.x] = wv[0];
            pidx[blockIdx.x] = wi[0];
        }
        grid.sync();
        // b. global pivot (same in every CTA): block-parallel reduction of
        //    the per-CTA candidates, then read pivot row and row k
        {
            double bv = -1.0;
            int64_t bix = n;
            for (unsigned c = threadIdx.x; c < gridDim.x; c += blockDim.x) {
                const double v = pval[c];
                const int64_t i = pidx[c];
                if (v > bv || (v == bv && i < bix)) { bv = v; bix = i; }
            }
            for (int off = 16; off >= 1; off >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
                const int64_t oi = __shfl_xor_sync(0xffffffffu, bix, off);
                if (ov > bv || (ov == bv && oi < bix)) { bv = ov; bix = oi; }
            }
            __syncthreads();
            if (lane == 0) { wv[w] = bv; wi[w] = bix; }
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int t = 1; t < kPT / 32; ++t)
                    if (wv[t] > wv[0] || (wv[t] == wv[0] && wi[t] < wi[0])) { wv[0] = wv[t]; wi[0] = wi[t]; }
                s_p = wi[0];
                s_v = wi[0] < n ? Pn[wi[0] * 2 * kB + q] : 0.0;
            }
        }
        __syncthreads();
        const int64_t p = s_p;
        const double v = s_v;
        if (!(fabs(v) >= 1e-300)) {
            if (blockIdx.x == 0 && threadIdx.x == 0 && atomicCAS(&err->code, 0, SAMG_ERROR) == 0)
                err->where = k;
            return;  // uniform across the grid
        }
        for (int t = threadIdx.x; t < 2 * kB; t += blockDim.x) {
            prow[t] = Pn[p * 2 * kB + t];
            krow[t] = Pn[k * 2 * kB + t];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            prow[kB + q] = 1.0;  // Z column q starts as e_k (after the swap)
            if (blockIdx.x == 0) piv[q] = p;
        }
        __syncthreads();
        const double inv = 1.0 / v;
        for (int t = threadIdx.x; t < 2 * kB; t += blockDim.x) rk[t] = prow[t] * inv;
        grid.sync();  // everyone has read rows p and k
        // c. eliminate column q from own rows (rows k and p swapped), in
        //    chunks of 64 rows: multipliers first, then the 2*kB updates
        for (int64_t c0 = r0; c0 < r1; c0 += 64) {
            const int nr = static_cast<int>(r1 - c0 < 64 ? r1 - c0 : 64);
            for (int t = threadIdx.x; t < nr; t += blockDim.x) {
                const int64_t i = c0 + t;
                fs[t] = (i == k) ? 0.0 : (i == p ? krow[q] : Pn[i * 2 * kB + q]);
            }
            __syncthreads();
            for (int e = threadIdx.x; e < nr * 2 * kB; e += blockDim.x) {
                const int r = e / (2 * kB), t = e % (2 * kB);
                const int64_t i = c0 + r;
                double *dst = Pn + i * 2 * kB + t;
                if (i == k) *dst = rk[t];
                else *dst = fma(-fs[r], rk[t], i == p ? krow[t] : *dst);
            }
            __syncthreads();
        }
    }
}

// apply the panel's row swaps, in order, to columns [j0, 2n)
__global__ void k_apply_swaps(int64_t n, int64_t j0, int64_t k0, int bk, const int64_t *piv,
                              double *W) {
    const int64_t ld = 2 * n;
    for (int64_t j = j0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < ld;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        for (int q = 0; q < bk; ++q) {
            const int64_t a = k0 + q, b = piv[q];
            if (a != b) {
                const double t = W[a * ld + j];
                W[a * ld + j] = W[b * ld + j];
                W[b * ld + j] = t;
            }
        }
}

__global__ void k_copy_rk(int64_t n, int64_t j0, int64_t k0, int bk, const double *W, double *Rk) {
    const int64_t m = 2 * n - j0;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < bk * m;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t q = e / m, j = e - q * m;
        Rk[q * m + j] = W[(k0 + q) * 2 * n + j0 + j];
    }
}

// W[i][j0 + j] += sum_q (Z[i][q] - delta(i, k0+q)) * Rk[q][j]; 64x64 tiles,
// 256 threads x (4x4) outputs, K = bk <= 32 staged in shared memory.
__global__ void __launch_bounds__(256) k_trailing(int64_t n, int64_t j0, int64_t k0, int bk,
                                                  const double *Pn, const double *Rk, double *W) {
    __shared__ double As[kB][64 + 1];
    __shared__ double Bs[kB][64];
    const int64_t m = 2 * n - j0;
    const int64_t i0 = blockIdx.y * 64, jj0 = blockIdx.x * 64;
    for (int t = threadIdx.x; t < kB * 64; t += 256) {
        const int q = t / 64, r = t % 64;
        const int64_t i = i0 + r;
        double a = 0.0;
        if (q < bk && i < n) a = Pn[i * 2 * kB + kB + q] - (i == k0 + q ? 1.0 : 0.0);
        As[q][r] = a;
        const int64_t j = jj0 + r;
        Bs[q][r] = (q < bk && j < m) ? Rk[q * m + j] : 0.0;
    }
    __syncthreads();
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    double acc[4][4] = {};
    for (int q = 0; q < bk; ++q) {
        double a[4], b[4];
        for (int u = 0; u < 4; ++u) { a[u] = As[q][ty + 16 * u]; b[u] = Bs[q][tx + 16 * u]; }
        for (int u = 0; u < 4; ++u)
            for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + ty + 16 * u;
        if (i >= n) continue;
        for (int v = 0; v < 4; ++v) {
            const int64_t j = jj0 + tx + 16 * v;
            if (j < m) W[i * 2 * n + j0 + j] += acc[u][v];
        }
    }
}

__global__ void k_copy_right(int64_t n, int64_t ld, const double *W, double *Ainv) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n * ld;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e / ld, j = e - i * ld;
        Ainv[e] = j < n ? W[i * 2 * n + n + j] : 0.0;
    }
}

int grid_for(int64_t work) {
    const int64_t g = (work + 255) / 256;
    return static_cast<int>(g < 8192 ? (g > 0 ? g : 1) : 8192);
}

} // namespace

void dense_inverse(const Bsr3 &A, DevBuf<double> &Ainv, DevError *err, cudaStream_t s) {
    const int64_t n = 3 * A.nrows;
    const int64_t ld = dense_ld(n);
    Ainv.alloc(n * ld, s);
    if (n == 0) return;
    DevBuf<double> W(2 * n * n, s), Pn(n * 2 * kB, s), Rk(static_cast<int64_t>(kB) * 2 * n, s);
    int dev = 0, nsm = 148, coop = 0, per_sm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
    if (!coop) fail(SAMG_UNSUPPORTED, "dense coarse solve needs cooperative launch");
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_panel_gj, kPT, 0));
    // panel CTAs: fewer CTAs make the two grid barriers per column cheaper,
    // more CTAs spread the row updates (SAMG_GJ_CTAS overrides)
    static const int64_t gj_ctas = [] {
        const char *e = std::getenv("SAMG_GJ_CTAS");
        return e ? std::atoll(e) : 128;
    }();
    const int pgrid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>({static_cast<int64_t>(nsm) * std::max(per_sm, 1), (n + 15) / 16, gj_ctas})));
    DevBuf<double> pval(pgrid, s);
    DevBuf<int64_t> pidx(pgrid, s), piv(kB, s);
    CK(cudaMemsetAsync(W.p, 0, W.bytes(), s));
    k_scatter<<<ceil_div(A.nrows, 128), 128, 0, s>>>(static_cast<int>(A.nrows), A.ptr.p, A.col.p,
                                                    A.val.p, n, W.p);
    CK_LAUNCH();
    for (int64_t k0 = 0; k0 < n; k0 += kB) {
        int bk = static_cast<int>(std::min<int64_t>(kB, n - k0));
        k_panel_load<<<grid_for(n * 2 * kB), 256, 0, s>>>(n, k0, bk, W.p, Pn.p);
        int64_t nn = n, kk0 = k0;
        double *pp = Pn.p, *pv = pval.p;
        int64_t *pi = pidx.p, *pvt = piv.p;
        DevError *e = err;
        void *args[] = {&nn, &kk0, &bk, &pp, &pv, &pi, &pvt, &e};
        CK(cudaLaunchCooperativeKernel(reinterpret_cast<void *>(k_panel_gj), pgrid, kPT, args, 0, s));
        const int64_t j0 = k0 + bk, m = 2 * n - j0;
        k_apply_swaps<<<grid_for(m), 256, 0, s>>>(n, j0, k0, bk, piv.p, W.p);
        k_copy_rk<<<grid_for(bk * m), 256, 0, s>>>(n, j0, k0, bk, W.p, Rk.p);
        dim3 tg(static_cast<unsigned>((m + 63) / 64), static_cast<unsigned>((n + 63) / 64));
        k_trailing<<<tg, 256, 0, s>>>(n, j0, k0, bk, Pn.p, Rk.p, W.p);
        CK_LAUNCH();
    }
    k_copy_right<<<grid_for(n * ld), 256, 0, s>>>(n, ld, W.p, Ainv.p);
    CK_LAUNCH();
    check_dev_error(err, s);
}

} // namespace samgb
