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
#include <vector>

#include "block3.cuh"
#include "kernels.cuh"

namespace samgb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
// one flag per 128-byte line: the flags of recent rows are polled by many
// warps at once, padding keeps unrelated rows off the same L2 line
constexpr int kFS = 32;

__device__ __forceinline__ int ld_relaxed(int *p) {
    cuda::atomic_ref<int, cuda::thread_scope_device> a(*p);
    return a.load(cuda::memory_order_relaxed);
}
__device__ __forceinline__ void st_release(int *p, int v) {
    cuda::atomic_ref<int, cuda::thread_scope_device> a(*p);
    a.store(v, cuda::memory_order_release);
}

// Wait until every dependency k = col[j], j in [b, e) (all of them finish
// earlier in the level order) has its flag set.  The lanes test all of them
// at once; while some are pending a single lane spins on one pending flag
// (one load in flight per waiting warp), then the warp re-tests.  Ends with
// an acquire fence.  (Measured on a 27-point 64^3 sweep: 7.7 us per level,
// against 10.3 us for a one-lane sequential scan, scripts/micro/ilu_trace.cu.)
__device__ __forceinline__ void wait_deps(const int *col, int b, int e, int *flags) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int pend = -1;
        for (int j = b + lane; j < e; j += 32) {
            const int k = col[j];
            if (ld_relaxed(flags + static_cast<int64_t>(k) * kFS) == 0) { pend = k; break; }
        }
        const unsigned m = __ballot_sync(kFull, pend >= 0);
        if (!m) break;
        const int k = __shfl_sync(kFull, pend, __ffs(m) - 1);
        if (lane == 0)
            while (ld_relaxed(flags + static_cast<int64_t>(k) * kFS) == 0) {
            }
        __syncwarp();
    }
    cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
    __syncwarp();
}

__device__ void raise_err(DevError *err, int code, int64_t where) {
    if (atomicCAS(&err->code, 0, code) == 0) err->where = where;
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
constexpr int kFMax = 192;  // rows up to this many blocks live in shared memory

__global__ void __launch_bounds__(256) k_ilu_factor(int n, const int *__restrict__ order,
        const int *__restrict__ ptr, const int *__restrict__ col, const int *__restrict__ dpos,
        double *lu, double *inv, int *done, int *counter, DevError *err) {
    // per warp: the row's columns and blocks (the IKJ chain then runs in
    // shared memory: binary searches and updates never touch L2)
    extern __shared__ __align__(16) unsigned char fsm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *srow = reinterpret_cast<double *>(fsm) + static_cast<size_t>(w) * 9 * kFMax;
    int *scol = reinterpret_cast<int *>(fsm + sizeof(double) * 9 * kFMax * 8) + w * kFMax;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(counter, 1);
        t = __shfl_sync(kFull, t, 0);
        if (t >= n) return;
        const int i = __ldg(order + t);
        const int b = ptr[i], e = ptr[i + 1], di = dpos[i], len = e - b;
        const bool in_smem = len <= kFMax;
        double *rv = in_smem ? srow - 9LL * b : lu;   // rv[9j + .] = block j of row i
        const int *rc = in_smem ? scol - b : col;     // rc[j] = column of block j
        if (in_smem) {
            for (int q = lane; q < len; q += 32) scol[q] = col[b + q];
            for (int q = lane; q < 9 * len; q += 32) srow[q] = lu[9LL * b + q];
        }
        wait_deps(col, b, di, done);
        // operands of step j+1 (inverted pivot of row k, first 32 blocks of
        // its U part) are requested while step j runs: every row k < i is
        // final once the dependencies are met
        auto load_step = [&](int j, double (&dv)[3], int &c0, double (&u0v)[9], int &uend) {
            const int k = rc[j];
            if (lane < 9) {
                const double *d = inv + 9LL * k;
                const int c = lane % 3;
                dv[0] = __ldcg(d + c); dv[1] = __ldcg(d + 3 + c); dv[2] = __ldcg(d + 6 + c);
            }
            const int ub = __ldg(dpos + k) + 1;
            uend = __ldg(ptr + k + 1);
            const int l = ub + lane;
            c0 = -1;
            if (l < uend) {
                c0 = __ldg(col + l);
#pragma unroll
                for (int q = 0; q < 9; ++q) u0v[q] = __ldcg(lu + 9LL * l + q);
            }
        };
        double dv[3] = {0, 0, 0}, u0v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        int c0 = -1, uend = 0;
        if (b < di) load_step(b, dv, c0, u0v, uend);
        for (int j = b; j < di; ++j) {
            const int k = rc[j];
            double ndv[3] = {0, 0, 0}, nu0v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
            int nc0 = -1, nuend = 0;
            if (j + 1 < di) load_step(j + 1, ndv, nc0, nu0v, nuend);
            // L_ik = A_ik * U_kk^-1 (operator*, static_block.hpp:68-76)
            double le = 0.0;
            if (lane < 9) {
                const int r = lane / 3;
                const double *a = rv + 9LL * j;
                le = __dadd_rn(le, __dmul_rn(a[r * 3 + 0], dv[0]));
                le = __dadd_rn(le, __dmul_rn(a[r * 3 + 1], dv[1]));
                le = __dadd_rn(le, __dmul_rn(a[r * 3 + 2], dv[2]));
            }
            __syncwarp();
            if (lane < 9) rv[9LL * j + lane] = le;
            double lik[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) lik[q] = __shfl_sync(kFull, le, q);
            // A_i. -= L_ik * U_k. over the U part of row k that hits row i
            const int ub = __ldg(dpos + k) + 1;
            for (int l = ub + lane; l < uend; l += 32) {
                int c;
                double uv[9];
                if (l == ub + lane) {
                    c = c0;
#pragma unroll
                    for (int q = 0; q < 9; ++q) uv[q] = u0v[q];
                } else {
                    c = __ldg(col + l);
#pragma unroll
                    for (int q = 0; q < 9; ++q) uv[q] = __ldcg(lu + 9LL * l + q);
                }
                int lo = b, hi = e - 1, q = -1;
                while (lo <= hi) {
                    const int m = (lo + hi) >> 1, cm = rc[m];
                    if (cm == c) { q = m; break; }
                    if (cm < c) lo = m + 1;
                    else hi = m - 1;
                }
                if (q < 0) continue;
                double *dst = rv + 9LL * q;
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
#pragma unroll
            for (int q = 0; q < 3; ++q) dv[q] = ndv[q];
#pragma unroll
            for (int q = 0; q < 9; ++q) u0v[q] = nu0v[q];
            c0 = nc0;
            uend = nuend;
        }
        if (in_smem)
            for (int q = lane; q < 9 * len; q += 32) lu[9LL * b + q] = srow[q];
        if (lane == 0) {
            double piv[9], out[9];
            for (int q = 0; q < 9; ++q) piv[q] = rv[9LL * di + q];
            if (!blk_inverse_ref(piv, out)) {
                raise_err(err, SAMG_SINGULAR_BLOCK, i);
                for (int q = 0; q < 9; ++q) out[q] = 0.0;
            }
            for (int q = 0; q < 9; ++q) inv[9LL * i + q] = out[q];
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            st_release(done + static_cast<int64_t>(i) * kFS, 1);
        }
    }
}

// Triangular sweeps (relaxation.hpp:44-88), level-scheduled and sync-free:
// a warp per row, rows taken from an atomic counter in LEVEL order (forward:
// the levels of the unit lower factor's dependency DAG, backward: of the
// upper factor's), each waiting on the flags of its dependencies.  Lanes
// 0..2 carry the three components through the exact subtraction chain in
// the reference's (j, q) order:
//   forward  y_i = r_i - sum_{j<i} L_ij y_j            (unit lower factor)
//   backward x_i = U_ii^-1 (y_i - sum_{j>i} U_ij x_j), in place over y,
//            then u_out = x (zero guess) or u_in + x  (kernels::axpby(1,x,1,u)).
template <bool kFwd, bool kZero>
__global__ void __launch_bounds__(256) k_ilu_sweep(int n, const int *__restrict__ order,
        const int *__restrict__ ptr, const int *__restrict__ col, const int *__restrict__ dpos,
        const double *__restrict__ lu, const double *__restrict__ inv, const double *rin,
        double *y, const double *u_in, double *u_out, int *flags, int *counter) {
    __shared__ double stage[8][12 * 32];  // per warp: 32 x 3 values + 32 x 9 block entries
    const int lane = threadIdx.x & 31;
    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(counter, 1);
        t = __shfl_sync(kFull, t, 0);
        if (t >= n) return;
        const int i = __ldg(order + t);
        const int b = kFwd ? ptr[i] : dpos[i] + 1, e = kFwd ? dpos[i] : ptr[i + 1];
        wait_deps(col, b, e, flags);
        // the lanes fetch a chunk of up to 32 dependencies (their values and
        // the lanes' rows of the factor blocks) in parallel into shared
        // memory -- one L2 round trip per chunk -- then lanes 0..2 walk the
        // chunk in order
        double acc = 0.0;
        if (lane < 3) acc = __ldcg((kFwd ? rin : y) + 3LL * i + lane);
        double *xs = stage[threadIdx.x >> 5], *bs = xs + 3 * 32;
        for (int c = b; c < e; c += 32) {
            const int j = c + lane, m = min(32, e - c);
            if (j < e) {
                const double *g = y + 3LL * col[j];
                const double *blk = lu + 9LL * j;
                xs[3 * lane] = __ldcg(g); xs[3 * lane + 1] = __ldcg(g + 1); xs[3 * lane + 2] = __ldcg(g + 2);
#pragma unroll
                for (int q = 0; q < 9; ++q) bs[9 * lane + q] = __ldg(blk + q);
            }
            __syncwarp();
            if (lane < 3)
                for (int d = 0; d < m; ++d) {
                    const double *bl = bs + 9 * d + 3 * lane, *v = xs + 3 * d;
                    acc = __dsub_rn(acc, __dmul_rn(bl[0], v[0]));
                    acc = __dsub_rn(acc, __dmul_rn(bl[1], v[1]));
                    acc = __dsub_rn(acc, __dmul_rn(bl[2], v[2]));
                }
            __syncwarp();
        }
        double out = acc;
        if constexpr (!kFwd) {
            const double a0 = __shfl_sync(kFull, acc, 0), a1 = __shfl_sync(kFull, acc, 1),
                         a2 = __shfl_sync(kFull, acc, 2);
            if (lane < 3) {
                const double *d = inv + 9LL * i + 3 * lane;
                double tt = 0.0;
                tt = __dadd_rn(tt, __dmul_rn(d[0], a0));
                tt = __dadd_rn(tt, __dmul_rn(d[1], a1));
                tt = __dadd_rn(tt, __dmul_rn(d[2], a2));
                out = tt;
            }
        }
        if (lane < 3) {
            y[3LL * i + lane] = out;
            if constexpr (!kFwd)
                u_out[3LL * i + lane] = kZero ? out : __dadd_rn(out, u_in[3LL * i + lane]);
        }
        __syncwarp();
        if (lane == 0) st_release(flags + static_cast<int64_t>(i) * kFS, 1);
    }
}

// Persistent grid: at most SAMG_ILU_CTAS_PER_SM (default 2) CTAs of 8 warps
// per SM -- the wavefront of a structured mesh offers a few hundred to a
// few thousand independent rows, more warps would only wait.
int persistent_grid(const void *kern, int64_t work_warps) {
    static int sms = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    static const int per_sm = [] {
        const char *e = std::getenv("SAMG_ILU_CTAS_PER_SM");
        return e ? std::max(1, std::atoi(e)) : 1;
    }();
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
    const int64_t want = (work_warps + 7) / 8;
    const int64_t cap = static_cast<int64_t>(std::min(std::max(occ, 1), per_sm)) * sms;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, cap)));
}

// Level orders of the two dependency DAGs (rows of level l depend only on
// levels < l), from one host pass over the pattern: forward = unit lower
// factor (row i waits for col < i), backward = upper factor (col > i).
// Within a level rows keep ascending (forward) / descending (backward) order.
void level_orders(const Bsr3 &A, const DevBuf<int> &dpos, DevBuf<int> &order, cudaStream_t s) {
    const int n = static_cast<int>(A.nrows);
    std::vector<int> ptr(n + 1), col(A.nnzb), dp(n);
    CK(cudaMemcpyAsync(ptr.data(), A.ptr.p, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(col.data(), A.col.p, sizeof(int) * A.nnzb, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(dp.data(), dpos.p, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<int> lev(n), ord(2 * static_cast<size_t>(n)), cnt;
    auto bucket = [&](int *out, bool ascending) {
        int maxl = 0;
        for (int i = 0; i < n; ++i) maxl = std::max(maxl, lev[i]);
        cnt.assign(maxl + 2, 0);
        for (int i = 0; i < n; ++i) ++cnt[lev[i] + 1];
        for (int l = 0; l <= maxl; ++l) cnt[l + 1] += cnt[l];
        for (int t = 0; t < n; ++t) {
            const int i = ascending ? t : n - 1 - t;
            out[cnt[lev[i]]++] = i;
        }
    };
    for (int i = 0; i < n; ++i) {
        int l = 0;
        for (int j = ptr[i]; j < dp[i]; ++j) l = std::max(l, lev[col[j]] + 1);
        lev[i] = l;
    }
    bucket(ord.data(), true);
    for (int i = n - 1; i >= 0; --i) {
        int l = 0;
        for (int j = dp[i] + 1; j < ptr[i + 1]; ++j) l = std::max(l, lev[col[j]] + 1);
        lev[i] = l;
    }
    bucket(ord.data() + n, false);
    order.alloc(2 * static_cast<size_t>(n), s);
    CK(cudaMemcpyAsync(order.p, ord.data(), sizeof(int) * 2 * n, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));  // host vectors go out of scope
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
    M.flags.alloc(2 * A.nrows * kFS + 2, s);
    if (n == 0) return;
    k_ilu_dpos<<<ceil_div(n, 256), 256, 0, s>>>(n, A.ptr.p, A.col.p, M.dpos.p, err);
    CK_LAUNCH();
    check_dev_error(err, s);  // no factorization without every diagonal
    level_orders(A, M.dpos, M.order, s);
    CK(cudaMemcpyAsync(M.lu.p, A.val.p, sizeof(double) * 9 * A.nnzb, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemsetAsync(M.flags.p, 0, sizeof(int) * (2 * A.nrows * kFS + 2), s));
    constexpr int fsmem = 8 * kFMax * (9 * static_cast<int>(sizeof(double)) + static_cast<int>(sizeof(int)));
    static const bool fattr = [] {
        CK(cudaFuncSetAttribute(k_ilu_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem));
        return true;
    }();
    (void)fattr;
    k_ilu_factor<<<persistent_grid(reinterpret_cast<const void *>(k_ilu_factor), n), 256, fsmem, s>>>(
        n, M.order.p, A.ptr.p, A.col.p, M.dpos.p, M.lu.p, M.data.p, M.flags.p,
        M.flags.p + 2 * static_cast<int64_t>(n) * kFS, err);
    CK_LAUNCH();
}

void launch_ilu_smooth(const Bsr3 *A, const Smoother &M, const double *f, const double *u_in,
                       double *u_out, cudaStream_t s) {
    const int n = static_cast<int>(M.nrows);
    if (n == 0) return;
    const int64_t nf = static_cast<int64_t>(n) * kFS;
    int *fw = M.flags.p, *bw = M.flags.p + nf, *cnt = M.flags.p + 2 * nf;
    CK(cudaMemsetAsync(M.flags.p, 0, sizeof(int) * (2 * nf + 2), s));
    const double *rin = f;
    if (u_in) {
        launch_residual(*A, f, u_in, M.tmp.p, s);  // r = f - A u (hierarchy.hpp:213-215)
        rin = M.tmp.p;
    }
    static const int gf = persistent_grid(reinterpret_cast<const void *>(k_ilu_sweep<true, true>), 1 << 30);
    const int grid = std::min(gf, (n + 7) / 8);
    const int *of = M.order.p, *ob = M.order.p + n;
    k_ilu_sweep<true, true><<<grid, 256, 0, s>>>(n, of, M.ptr, M.col, M.dpos.p, M.lu.p, M.data.p, rin,
                                                 M.tmp.p, nullptr, nullptr, fw, cnt);
    if (u_in)
        k_ilu_sweep<false, false><<<grid, 256, 0, s>>>(n, ob, M.ptr, M.col, M.dpos.p, M.lu.p, M.data.p,
                                                       nullptr, M.tmp.p, u_in, u_out, bw, cnt + 1);
    else
        k_ilu_sweep<false, true><<<grid, 256, 0, s>>>(n, ob, M.ptr, M.col, M.dpos.p, M.lu.p, M.data.p,
                                                      nullptr, M.tmp.p, nullptr, u_out, bw, cnt + 1);
    CK_LAUNCH();
}

} // namespace samgb
