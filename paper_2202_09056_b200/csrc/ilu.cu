// ilu.cu -- block ILU(0) smoother: ilu0<block3> (relaxation.hpp:20-139), the
// reference's default smoother (hierarchy.hpp:52, 295-297).
//
// Compiled with --fmad=false and explicit __d*_rn arithmetic in the
// reference's loop orders, so the factors, the inverted pivots and every
// smoothing application are bit-identical to the reference.
//
// Both the IKJ factorization and the two triangular sweeps are sequential
// chains in row order.  They run as "sync-free" persistent kernels: warps
// take work in increasing row order from an atomic counter and wait only
// for the rows they depend on (one release/acquire flag per row), so the
// critical path is the dependency depth of the pattern (~nx+ny+nz row hops
// for a structured mesh in natural order), not n.
//  * factorization: a warp per row; lanes split the U part of each pivot row
//    (distinct targets per step), steps in the reference's j order;
//  * triangular sweeps: a warp per segment of S consecutive rows, processed
//    in order with the segment's results kept in shared memory, so the
//    (frequent) dependency on the preceding rows costs no flag round trip;
//    lanes 0..2 carry the three row components through the exact
//    subtraction chain; dependencies outside the segment are awaited on flags.
#include <cuda/atomic>

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace samgb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kSegMax = 64;

__device__ __forceinline__ int ld_acquire(int *p) {
    cuda::atomic_ref<int, cuda::thread_scope_device> a(*p);
    return a.load(cuda::memory_order_acquire);
}
__device__ __forceinline__ void st_release(int *p, int v) {
    cuda::atomic_ref<int, cuda::thread_scope_device> a(*p);
    a.store(v, cuda::memory_order_release);
}
__device__ __forceinline__ void wait_flag(int *p) {
    while (ld_acquire(p) == 0) {
    }
}

__device__ void raise_err(DevError *err, int code, int64_t where) {
    if (atomicCAS(&err->code, 0, code) == 0) err->where = where;
}

// inverse (static_block.hpp:119-158); false on a singular pivot
__device__ bool blk_inverse_ref(const double *a, double *inv) {
    double lu[9];
    int piv[3];
    for (int e = 0; e < 9; ++e) lu[e] = a[e];
    for (int k = 0; k < 3; ++k) {
        int p = k;
        for (int r = k + 1; r < 3; ++r)
            if (fabs(lu[r * 3 + k]) > fabs(lu[p * 3 + k])) p = r;
        piv[k] = p;
        if (p != k)
            for (int j = 0; j < 3; ++j) { const double t = lu[k * 3 + j]; lu[k * 3 + j] = lu[p * 3 + j]; lu[p * 3 + j] = t; }
        if (fabs(lu[k * 3 + k]) < 1e-300) return false;
        const double d = __ddiv_rn(1.0, lu[k * 3 + k]);
        for (int r = k + 1; r < 3; ++r) {
            const double l = __dmul_rn(lu[r * 3 + k], d);
            lu[r * 3 + k] = l;
            for (int j = k + 1; j < 3; ++j) lu[r * 3 + j] = __dsub_rn(lu[r * 3 + j], __dmul_rn(l, lu[k * 3 + j]));
        }
    }
    for (int c = 0; c < 3; ++c) {
        double x[3] = {0.0, 0.0, 0.0};
        x[c] = 1.0;
        for (int k = 0; k < 3; ++k)
            if (piv[k] != k) { const double t = x[k]; x[k] = x[piv[k]]; x[piv[k]] = t; }
        for (int r = 1; r < 3; ++r)
            for (int j = 0; j < r; ++j) x[r] = __dsub_rn(x[r], __dmul_rn(lu[r * 3 + j], x[j]));
        for (int r = 2; r >= 0; --r) {
            for (int j = r + 1; j < 3; ++j) x[r] = __dsub_rn(x[r], __dmul_rn(lu[r * 3 + j], x[j]));
            x[r] = __ddiv_rn(x[r], lu[r * 3 + r]);
        }
        for (int r = 0; r < 3; ++r) inv[r * 3 + c] = x[r];
    }
    return true;
}

__global__ void k_ilu_dpos(int n, const int *ptr, const int *col, int *dpos, DevError *err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int d = -1;
    for (int j = ptr[i]; j < ptr[i + 1]; ++j)
        if (col[j] == i) d = j;
    dpos[i] = d;
    if (d < 0) raise_err(err, SAMG_MISSING_DIAGONAL, i);
}

// IKJ factorization (relaxation.hpp:115-132), a warp per row.
__global__ void __launch_bounds__(256) k_ilu_factor(int n, const int *__restrict__ ptr,
        const int *__restrict__ col, const int *__restrict__ dpos, double *lu, double *inv,
        int *done, int *counter, DevError *err) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int i = 0;
        if (lane == 0) i = atomicAdd(counter, 1);
        i = __shfl_sync(kFull, i, 0);
        if (i >= n) return;
        const int b = ptr[i], e = ptr[i + 1], di = dpos[i];
        for (int j = b + lane; j < di; j += 32) wait_flag(done + col[j]);
        __syncwarp();
        for (int j = b; j < di; ++j) {
            const int k = col[j];
            // L_ik = A_ik * U_kk^-1 (operator*, static_block.hpp:68-76)
            double le = 0.0;
            if (lane < 9) {
                const int r = lane / 3, c = lane % 3;
                const double *a = lu + 9LL * j, *d = inv + 9LL * k;
                le = __dadd_rn(le, __dmul_rn(a[r * 3 + 0], __ldcg(d + 0 * 3 + c)));
                le = __dadd_rn(le, __dmul_rn(a[r * 3 + 1], __ldcg(d + 1 * 3 + c)));
                le = __dadd_rn(le, __dmul_rn(a[r * 3 + 2], __ldcg(d + 2 * 3 + c)));
            }
            __syncwarp();
            if (lane < 9) lu[9LL * j + lane] = le;
            double lik[9];
#pragma unroll
            for (int t = 0; t < 9; ++t) lik[t] = __shfl_sync(kFull, le, t);
            // A_i. -= L_ik * U_k. over the U part of row k that hits row i
            const int u0 = __ldg(dpos + k) + 1, u1 = __ldg(ptr + k + 1);
            for (int l = u0 + lane; l < u1; l += 32) {
                const int c = col[l];
                int lo = b, hi = e - 1, q = -1;
                while (lo <= hi) {
                    const int m = (lo + hi) >> 1, cm = col[m];
                    if (cm == c) { q = m; break; }
                    if (cm < c) lo = m + 1;
                    else hi = m - 1;
                }
                if (q < 0) continue;
                double uv[9];
#pragma unroll
                for (int t = 0; t < 9; ++t) uv[t] = __ldcg(lu + 9LL * l + t);
                double *dst = lu + 9LL * q;
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc) {
                        double pr = 0.0;
                        pr = __dadd_rn(pr, __dmul_rn(lik[r * 3 + 0], uv[0 * 3 + cc]));
                        pr = __dadd_rn(pr, __dmul_rn(lik[r * 3 + 1], uv[1 * 3 + cc]));
                        pr = __dadd_rn(pr, __dmul_rn(lik[r * 3 + 2], uv[2 * 3 + cc]));
                        dst[r * 3 + cc] = __dsub_rn(dst[r * 3 + cc], pr);
                    }
            }
            __syncwarp();
        }
        if (lane == 0) {
            double piv[9], out[9];
            for (int t = 0; t < 9; ++t) piv[t] = lu[9LL * di + t];
            if (!blk_inverse_ref(piv, out)) {
                raise_err(err, SAMG_SINGULAR_BLOCK, i);
                for (int t = 0; t < 9; ++t) out[t] = 0.0;
            }
            for (int t = 0; t < 9; ++t) inv[9LL * i + t] = out[t];
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            st_release(done + i, 1);
        }
    }
}

// Forward sweep with the unit lower factor (relaxation.hpp:48-62):
// y_i = r_i - sum_{j<i} L_ij y_j; rin may alias y.
__global__ void __launch_bounds__(256) k_ilu_fwd(int n, int S, const int *__restrict__ ptr,
        const int *__restrict__ col, const int *__restrict__ dpos, const double *__restrict__ lu,
        const double *rin, double *y, int *flags, int *counter) {
    __shared__ double segv[8][3 * kSegMax];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *sv = segv[w];
    for (;;) {
        int sg = 0;
        if (lane == 0) sg = atomicAdd(counter, 1);
        sg = __shfl_sync(kFull, sg, 0);
        const int i0 = sg * S;
        if (i0 >= n) return;
        const int i1 = min(n, i0 + S);
        for (int i = i0; i < i1; ++i) {
            const int b = ptr[i], e = dpos[i];
            for (int j = b + lane; j < e; j += 32) {
                const int k = col[j];
                if (k < i0) wait_flag(flags + k);
            }
            __syncwarp();
            if (lane < 3) {
                double acc = __ldcg(rin + 3LL * i + lane);
                for (int j = b; j < e; ++j) {
                    const int k = col[j];
                    const double *bl = lu + 9LL * j + 3 * lane;
                    double x0, x1, x2;
                    if (k >= i0) {
                        x0 = sv[3 * (k - i0)]; x1 = sv[3 * (k - i0) + 1]; x2 = sv[3 * (k - i0) + 2];
                    } else {
                        const double *g = y + 3LL * k;
                        x0 = __ldcg(g); x1 = __ldcg(g + 1); x2 = __ldcg(g + 2);
                    }
                    acc = __dsub_rn(acc, __dmul_rn(bl[0], x0));
                    acc = __dsub_rn(acc, __dmul_rn(bl[1], x1));
                    acc = __dsub_rn(acc, __dmul_rn(bl[2], x2));
                }
                sv[3 * (i - i0) + lane] = acc;
                y[3LL * i + lane] = acc;
            }
            __syncwarp();
            if (lane == 0) st_release(flags + i, 1);
        }
    }
}

// Backward sweep (relaxation.hpp:63-87): x_i = U_ii^-1 (y_i - sum_{j>i} U_ij
// x_j), in place over y; then u_out = x (zero guess) or u_in + x
// (kernels::axpby(1, x, 1, u)).
template <bool kZero>
__global__ void __launch_bounds__(256) k_ilu_bwd(int n, int S, const int *__restrict__ ptr,
        const int *__restrict__ col, const int *__restrict__ dpos, const double *__restrict__ lu,
        const double *__restrict__ inv, double *y, const double *u_in, double *u_out, int *flags,
        int *counter) {
    __shared__ double segv[8][3 * kSegMax];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *sv = segv[w];
    const int nseg = (n + S - 1) / S;
    for (;;) {
        int sg = 0;
        if (lane == 0) sg = atomicAdd(counter, 1);
        sg = __shfl_sync(kFull, sg, 0);
        if (sg >= nseg) return;
        const int i0 = (nseg - 1 - sg) * S, i1 = min(n, i0 + S);
        for (int i = i1 - 1; i >= i0; --i) {
            const int b = dpos[i] + 1, e = ptr[i + 1];
            for (int j = b + lane; j < e; j += 32) {
                const int k = col[j];
                if (k >= i1) wait_flag(flags + k);
            }
            __syncwarp();
            double acc = 0.0;
            if (lane < 3) {
                acc = __ldcg(y + 3LL * i + lane);
                for (int j = b; j < e; ++j) {
                    const int k = col[j];
                    const double *bl = lu + 9LL * j + 3 * lane;
                    double x0, x1, x2;
                    if (k < i1) {
                        x0 = sv[3 * (k - i0)]; x1 = sv[3 * (k - i0) + 1]; x2 = sv[3 * (k - i0) + 2];
                    } else {
                        const double *g = y + 3LL * k;
                        x0 = __ldcg(g); x1 = __ldcg(g + 1); x2 = __ldcg(g + 2);
                    }
                    acc = __dsub_rn(acc, __dmul_rn(bl[0], x0));
                    acc = __dsub_rn(acc, __dmul_rn(bl[1], x1));
                    acc = __dsub_rn(acc, __dmul_rn(bl[2], x2));
                }
            }
            const double a0 = __shfl_sync(kFull, acc, 0), a1 = __shfl_sync(kFull, acc, 1),
                         a2 = __shfl_sync(kFull, acc, 2);
            if (lane < 3) {
                const double *d = inv + 9LL * i + 3 * lane;
                double t = 0.0;
                t = __dadd_rn(t, __dmul_rn(d[0], a0));
                t = __dadd_rn(t, __dmul_rn(d[1], a1));
                t = __dadd_rn(t, __dmul_rn(d[2], a2));
                sv[3 * (i - i0) + lane] = t;
                y[3LL * i + lane] = t;
                u_out[3LL * i + lane] = kZero ? t : __dadd_rn(t, u_in[3LL * i + lane]);
            }
            __syncwarp();
            if (lane == 0) st_release(flags + i, 1);
        }
    }
}

int persistent_grid(const void *kern, int64_t work_warps) {
    static int sms = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
    const int64_t want = (work_warps + 7) / 8;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, static_cast<int64_t>(std::max(occ, 1)) * sms)));
}

int segment_rows() {
    static const int s = [] {
        const char *e = std::getenv("SAMG_ILU_SEG");
        const int v = e ? std::atoi(e) : 32;
        return std::min(kSegMax, std::max(1, v));
    }();
    return s;
}

} // namespace

void setup_ilu0(const Bsr3 &A, Smoother &M, DevError *err, cudaStream_t s) {
    if (A.nrows != A.ncols) fail(SAMG_NON_SQUARE, "ilu0: matrix must be square");
    const int n = static_cast<int>(A.nrows);
    M.kind = SM_ILU;
    M.ptr = A.ptr.p;
    M.col = A.col.p;
    M.nrows = A.nrows;
    M.nnzb = A.nnzb;
    M.data.alloc(9 * A.nrows + 1, s);
    M.lu.alloc(9 * A.nnzb + 1, s);
    M.tmp.alloc(3 * A.nrows + 3, s);
    M.dpos.alloc(A.nrows + 1, s);
    M.flags.alloc(2 * A.nrows + 2, s);
    if (n == 0) return;
    k_ilu_dpos<<<ceil_div(n, 256), 256, 0, s>>>(n, A.ptr.p, A.col.p, M.dpos.p, err);
    CK_LAUNCH();
    check_dev_error(err, s);  // no factorization without every diagonal
    CK(cudaMemcpyAsync(M.lu.p, A.val.p, sizeof(double) * 9 * A.nnzb, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemsetAsync(M.flags.p, 0, sizeof(int) * (2 * A.nrows + 2), s));
    k_ilu_factor<<<persistent_grid(reinterpret_cast<const void *>(k_ilu_factor), n), 256, 0, s>>>(
        n, A.ptr.p, A.col.p, M.dpos.p, M.lu.p, M.data.p, M.flags.p, M.flags.p + 2 * n, err);
    CK_LAUNCH();
}

void launch_ilu_smooth(const Bsr3 *A, const Smoother &M, const double *f, const double *u_in,
                       double *u_out, cudaStream_t s) {
    const int n = static_cast<int>(M.nrows);
    if (n == 0) return;
    const int S = segment_rows();
    const int nseg = (n + S - 1) / S;
    int *fw = M.flags.p, *bw = M.flags.p + n, *cnt = M.flags.p + 2 * n;
    CK(cudaMemsetAsync(M.flags.p, 0, sizeof(int) * (2 * static_cast<int64_t>(n) + 2), s));
    const double *rin = f;
    if (u_in) {
        launch_residual(*A, f, u_in, M.tmp.p, s);  // r = f - A u (hierarchy.hpp:213-215)
        rin = M.tmp.p;
    }
    static const int gf = persistent_grid(reinterpret_cast<const void *>(k_ilu_fwd), 1 << 30);
    const int grid = std::min(gf, (nseg + 7) / 8);
    k_ilu_fwd<<<grid, 256, 0, s>>>(n, S, M.ptr, M.col, M.dpos.p, M.lu.p, rin, M.tmp.p, fw, cnt);
    if (u_in)
        k_ilu_bwd<false><<<grid, 256, 0, s>>>(n, S, M.ptr, M.col, M.dpos.p, M.lu.p, M.data.p, M.tmp.p,
                                              u_in, u_out, bw, cnt + 1);
    else
        k_ilu_bwd<true><<<grid, 256, 0, s>>>(n, S, M.ptr, M.col, M.dpos.p, M.lu.p, M.data.p, M.tmp.p,
                                             nullptr, u_out, bw, cnt + 1);
    CK_LAUNCH();
}

} // namespace samgb
