// ilu.cu -- block ILU(0) smoother: ilu0<block3> (relaxation.hpp:20-139), the
// reference's default smoother (hierarchy.hpp:52, 295-297).
//
// Compiled with --fmad=false and explicit __d*_rn arithmetic in the
// reference's loop orders, so the factors, the inverted pivots and every
// smoothing application are bit-identical to the reference.
//
// Both the IKJ factorization and the two triangular sweeps are sequential
// chains in row order.  They run as "sync-free" persistent kernels: warps
// take rows in dependency-level order from an atomic counter and wait only
// for the rows they depend on, so the critical path is the dependency depth
// of the pattern (~nx+2ny+4nz row hops for a structured mesh in natural
// order), not n.
//  * factorization: a warp per row, one release/acquire flag per row; lanes
//    split the U part of each pivot row (distinct targets per step), steps
//    in the reference's j order;
//  * triangular sweeps: a warp per row, the output value is its own flag
//    (sentinel-filled vector, relaxed polls); lanes 0..2 carry the three row
//    components through the exact subtraction chain over the ready prefix
//    of the dependencies (k_ilu_sweep).
#include <cuda/atomic>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
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
        // Steps run as soon as THEIR pivot row is final, in the reference's
        // j order: [b, rdy) are known complete (flags seen, then an acquire
        // fence).  In natural order the latest dependency (k = i-1) is the
        // last step, so all but the last step overlap the rows before.
        int rdy = b;
        auto advance = [&](int j) {  // make dependency j complete, extend rdy
            for (;;) {
                const int c = j + lane;
                const bool ok = c >= di || ld_relaxed(done + static_cast<int64_t>(rc[c]) * kFS) != 0;
                const unsigned nr = __ballot_sync(kFull, !ok);
                const int pre = nr ? __ffs(nr) - 1 : 32;
                if (pre > 0) { rdy = min(di, j + pre); break; }
                if (lane == 0)
                    while (ld_relaxed(done + static_cast<int64_t>(rc[j]) * kFS) == 0) {
                    }
                __syncwarp();
            }
            cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
            __syncwarp();
        };
        if (in_smem) __syncwarp();  // scol staged
        // operands of step j+1 (inverted pivot of row k, first 32 blocks of
        // its U part) are requested while step j runs when row k is known
        // final
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
        if (b < di) {
            advance(b);
            load_step(b, dv, c0, u0v, uend);
        }
        for (int j = b; j < di; ++j) {
            const int k = rc[j];
            double ndv[3] = {0, 0, 0}, nu0v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
            int nc0 = -1, nuend = 0;
            const bool pre = j + 1 < rdy;
            if (pre) load_step(j + 1, ndv, nc0, nu0v, nuend);
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
            if (j + 1 < di && !pre) {
                advance(j + 1);
                load_step(j + 1, ndv, nc0, nu0v, nuend);
            }
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
// upper factor's).  Lanes 0..2 carry the three components through the exact
// subtraction chain in the reference's (j, q) order:
//   forward  y_i = r_i - sum_{j<i} L_ij y_j            (unit lower factor)
//   backward x_i = U_ii^-1 (y_i - sum_{j>i} U_ij x_j),
//            then u_out = x (zero guess) or u_in + x  (kernels::axpby(1,x,1,u)).
//
// The value is its own flag: the output vector is pre-filled with kSent (all
// bits set, a NaN payload fp arithmetic never returns) and a dependency is
// complete once its three components are not kSent.  A hand-off therefore
// costs one relaxed L2 poll -- no release fence on the producer, no flag
// load + acquire + data load on the consumer (scripts/micro/value_chain.cu:
// 0.36 us per hop against 0.98 us for flag + fence).  The factor blocks of
// the row do not depend on other rows and are staged in shared memory before
// the first poll; every lane polls its own dependencies and, once one is
// complete, forms its 9 products (independent of the chain) in place; lanes
// 0..2 then walk the READY PREFIX of the subtraction chain while later
// dependencies are still pending.  In natural order the latest forward
// dependency (row i-1) is the last in the chain, so only a few subtractions
// follow the hand-off; backward, the latest (row i+1) is the first, and the
// whole chain of 3 dependent subtractions per dependency follows it.
constexpr unsigned long long kSent = ~0ull;
constexpr int kWin = 96;  // dependencies staged per window (3 per lane)

__device__ __forceinline__ unsigned long long ld_poll(const double *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_publish(double *p, double x) {
    unsigned long long v = static_cast<unsigned long long>(__double_as_longlong(x));
    if (v == kSent) v = 0x7fffffffffffffffull;  // a NaN input carrying the sentinel bits
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <bool kFwd, bool kZero, bool kRev = false>
__global__ void __launch_bounds__(256) k_ilu_sweep(int n, const int *__restrict__ order,
        const int *__restrict__ ptr, const int *__restrict__ col, const int *__restrict__ dpos,
        const double *__restrict__ lu, const double *__restrict__ inv, const double *src,
        double *out, const double *u_in, double *u_out, unsigned *counter) {
    extern __shared__ __align__(16) double ssm[];  // per warp: kWin x 9 block entries (then products)
    const int lane = threadIdx.x & 31;
    double *bs = ssm + static_cast<size_t>(threadIdx.x >> 5) * kWin * 9;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(counter, 1u) + 1u;  // counter starts at 0xffffffff
        t = __shfl_sync(kFull, t, 0);
        if (t >= static_cast<unsigned>(n)) return;
        const int i = __ldg(order + t);
        const int b = kFwd ? __ldg(ptr + i) : __ldg(dpos + i) + 1, e = kFwd ? __ldg(dpos + i) : __ldg(ptr + i + 1);
        double acc = 0.0;
        if (lane < 3) acc = src[3LL * i + lane];
        // backward: the row of U_ii^-1 (and u_in) ahead of the chain -- loaded
        // after it they put a memory round trip on every hand-off
        double dv0 = 0.0, dv1 = 0.0, dv2 = 0.0, uin = 0.0;
        if constexpr (!kFwd) {
            if (lane < 3) {
                const double *d = inv + 9LL * i + 3 * lane;
                dv0 = __ldg(d);
                dv1 = __ldg(d + 1);
                dv2 = __ldg(d + 2);
                if constexpr (!kZero) uin = u_in[3LL * i + lane];
            }
        }
        for (int wd = 0; wd < e - b; wd += kWin) {
            const int m = min(kWin, e - b - wd);
            // kRev (backward, relaxed order): the chain runs over descending
            // columns -- windows from the row's end, reversed inside -- so
            // the latest dependency (row i + 1) is its last term
            const int w0 = kRev ? e - wd - m : b + wd;
            if constexpr (kRev) {
                for (int q = lane; q < 9 * m; q += 32) {
                    const int d = q / 9;
                    bs[q] = __ldg(lu + 9LL * (w0 + m - 1 - d) + (q - 9 * d));
                }
            } else {
                for (int q = lane; q < 9 * m; q += 32) bs[q] = __ldg(lu + 9LL * w0 + q);
            }
            int kk[3];
            unsigned pend = 0;
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                const int d = lane + 32 * s;
                kk[s] = 0;
                if (d < m) { kk[s] = __ldg(col + w0 + (kRev ? m - 1 - d : d)); pend |= 1u << s; }
            }
            __syncwarp();  // the staged blocks are multiplied by their dependency's lane
            int done = 0;
            for (;;) {
#pragma unroll
                for (int s = 0; s < 3; ++s)
                    if (pend >> s & 1u) {
                        const double *g = out + 3LL * kk[s];
                        const unsigned long long v0 = ld_poll(g), v1 = ld_poll(g + 1), v2 = ld_poll(g + 2);
                        if (v0 != kSent && v1 != kSent && v2 != kSent) {
                            // the dependency's 9 products, in place over its
                            // block: only the subtractions stay sequential
                            double *bl = bs + 9 * (lane + 32 * s);
                            const double x0 = __longlong_as_double(static_cast<long long>(v0)),
                                         x1 = __longlong_as_double(static_cast<long long>(v1)),
                                         x2 = __longlong_as_double(static_cast<long long>(v2));
#pragma unroll
                            for (int r = 0; r < 3; ++r) {
                                bl[3 * r] = __dmul_rn(bl[3 * r], x0);
                                bl[3 * r + 1] = __dmul_rn(bl[3 * r + 1], x1);
                                bl[3 * r + 2] = __dmul_rn(bl[3 * r + 2], x2);
                            }
                            pend &= ~(1u << s);
                        }
                    }
                __syncwarp();
                const unsigned r0 = __ballot_sync(kFull, !(pend & 1u)), r1 = __ballot_sync(kFull, !(pend & 2u)),
                               r2 = __ballot_sync(kFull, !(pend & 4u));
                int ready = r0 != kFull ? __ffs(~r0) - 1
                          : r1 != kFull ? 32 + __ffs(~r1) - 1
                          : r2 != kFull ? 64 + __ffs(~r2) - 1 : kWin;
                ready = min(ready, m);
                if (lane < 3) {
                    // acc = ((acc - B(r,0) x0) - B(r,1) x1) - B(r,2) x2 per
                    // dependency, in order (relaxation.hpp:60-66); the
                    // products of the next 4 dependencies are loaded while
                    // the current 4 are subtracted (the chain is DADD-latency
                    // bound, shared-memory latency stays off it)
                    const double *pr = bs + 3 * lane;
                    int d = done;
                    double p[12];
                    auto load4 = [&](int d0, double (&q)[12]) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int dd = min(d0 + u, kWin - 1);
                            q[3 * u] = pr[9 * dd]; q[3 * u + 1] = pr[9 * dd + 1]; q[3 * u + 2] = pr[9 * dd + 2];
                        }
                    };
                    if (d + 4 <= ready) load4(d, p);
                    while (d + 4 <= ready) {
                        double q[12];
                        load4(d + 4, q);
#pragma unroll
                        for (int u = 0; u < 12; ++u) acc = __dsub_rn(acc, p[u]);
#pragma unroll
                        for (int u = 0; u < 12; ++u) p[u] = q[u];
                        d += 4;
                    }
                    for (; d < ready; ++d) {
                        acc = __dsub_rn(acc, pr[9 * d]);
                        acc = __dsub_rn(acc, pr[9 * d + 1]);
                        acc = __dsub_rn(acc, pr[9 * d + 2]);
                    }
                }
                done = ready;
                if (done == m) break;
                // only the chain's last term is pending (forward: row i - 1,
                // the usual case): lanes 0..2 poll that dependency themselves
                // and finish the chain from registers -- no product staging,
                // warp vote or shared-memory round trip after the hand-off
                // (the same products and subtractions)
                // (not in the reference-order backward sweep, whose last term
                // is the earliest dependency: there the extra path only cost
                // the chain walk its code shape, 1.19 -> 1.43 ms)
                if ((kFwd || kRev) && done == m - 1 && wd + m == e - b) {
                    const int dl = m - 1;
                    const int ks = dl < 32 ? kk[0] : (dl < 64 ? kk[1] : kk[2]);
                    const int kl = __shfl_sync(kFull, ks, dl & 31);
                    if (lane < 3) {
                        const double *pr = bs + 9 * dl + 3 * lane;  // still the factor block: its lane never saw the value
                        const double b0 = pr[0], b1 = pr[1], b2 = pr[2];
                        const double *g = out + 3LL * kl;
                        unsigned long long v0, v1, v2;
                        do {
                            v0 = ld_poll(g);
                            v1 = ld_poll(g + 1);
                            v2 = ld_poll(g + 2);
                        } while (v0 == kSent || v1 == kSent || v2 == kSent);
                        acc = __dsub_rn(acc, __dmul_rn(b0, __longlong_as_double(static_cast<long long>(v0))));
                        acc = __dsub_rn(acc, __dmul_rn(b1, __longlong_as_double(static_cast<long long>(v1))));
                        acc = __dsub_rn(acc, __dmul_rn(b2, __longlong_as_double(static_cast<long long>(v2))));
                    }
                    break;
                }
            }
            __syncwarp();  // the window's staging is reused
        }
        double res = acc;
        if constexpr (!kFwd) {
            const double a0 = __shfl_sync(kFull, acc, 0), a1 = __shfl_sync(kFull, acc, 1),
                         a2 = __shfl_sync(kFull, acc, 2);
            if (lane < 3) {
                double tt = 0.0;
                tt = __dadd_rn(tt, __dmul_rn(dv0, a0));
                tt = __dadd_rn(tt, __dmul_rn(dv1, a1));
                tt = __dadd_rn(tt, __dmul_rn(dv2, a2));
                res = tt;
            }
        }
        if (lane < 3) {
            st_publish(out + 3LL * i + lane, res);
            if constexpr (!kFwd) u_out[3LL * i + lane] = kZero ? res : __dadd_rn(res, uin);
        }
        __syncwarp();
    }
}

constexpr int kSweepSmem = 8 * kWin * 9 * static_cast<int>(sizeof(double));

// Persistent grid: at most SAMG_ILU_CTAS_PER_SM (default 1; the sweeps: 2) CTAs of 8 warps
// per SM -- the wavefront of a structured mesh offers a few hundred to a
// few thousand independent rows, more warps would only wait.
int persistent_grid(const void *kern, int64_t work_warps, int smem = 0, int per_sm_cap = 0) {
    const int sms = sm_count();
    static const int per_sm = [] {
        const char *e = std::getenv("SAMG_ILU_CTAS_PER_SM");
        return e ? std::max(1, std::atoi(e)) : 1;
    }();
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
    const int64_t want = (work_warps + 7) / 8;
    const int64_t cap = static_cast<int64_t>(std::min(std::max(occ, 1), per_sm_cap ? per_sm_cap : per_sm)) * sms;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, cap)));
}

// Level orders of the two dependency DAGs (rows of level l depend only on
// levels < l), from one host pass over the pattern: forward = unit lower
// factor (row i waits for col < i), backward = upper factor (col > i).
// Within a level rows keep ascending (forward) / descending (backward) order.
// The same level orders on the GPU: a persistent grid claims rows in
// dependency order (forward: ascending i, backward: descending -- a valid
// topological order of each DAG), a warp takes the max level over the row's
// lower (upper) neighbours, polling each until published (levels start at
// -1), and publishes 1 + max; a stable radix sort by level then keeps
// ascending (forward) / descending (backward) rows within a level.  The
// host pass downloaded the pattern and walked it sequentially (C1 level 0:
// 25 ms of a 61 ms ILU(0) setup).
__global__ void __launch_bounds__(256) k_ilu_levels(int n, bool fwd, const int *__restrict__ ptr,
        const int *__restrict__ col, const int *__restrict__ dpos, int *lev, int *keys, int *vals,
        unsigned *counter, int *maxlev) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(counter, 1u);
        t = __shfl_sync(kFull, t, 0);
        if (t >= static_cast<unsigned>(n)) return;
        const int i = fwd ? static_cast<int>(t) : n - 1 - static_cast<int>(t);
        const int b = fwd ? ptr[i] : dpos[i] + 1, e = fwd ? dpos[i] : ptr[i + 1];
        int l = 0;
        for (int j = b + lane; j < e; j += 32) {
            const int c = col[j];
            int v;
            do {
                asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(lev + c) : "memory");
            } while (v < 0);
            l = max(l, v + 1);
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) l = max(l, __shfl_xor_sync(kFull, l, off));
        if (lane == 0) {
            asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(lev + i), "r"(l) : "memory");
            keys[t] = l;
            vals[t] = i;
            atomicMax(maxlev, l);
        }
    }
}

void level_orders_device(const Bsr3 &A, const DevBuf<int> &dpos, DevBuf<int> &order, int (&depth)[2],
                         cudaStream_t s) {
    const int n = static_cast<int>(A.nrows);
    order.alloc(2 * static_cast<size_t>(n), s);
    DevBuf<int> lev(n, s), keys(n, s), vals(n, s), keys2(n, s), mx(2, s);
    DevBuf<unsigned> cnt(2, s);
    CK(cudaMemsetAsync(cnt.p, 0, 2 * sizeof(unsigned), s));
    CK(cudaMemsetAsync(mx.p, 0, 2 * sizeof(int), s));
    const int grid = std::max(1, std::min(sm_count() * 4, (n + 7) / 8));
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys2.p, vals.p, order.p, n, 0, 32, s));
    DevBuf<char> ws(bytes, s);
    for (int d = 0; d < 2; ++d) {
        CK(cudaMemsetAsync(lev.p, 0xff, sizeof(int) * n, s));  // -1: not yet published
        k_ilu_levels<<<grid, 256, 0, s>>>(n, d == 0, A.ptr.p, A.col.p, dpos.p, lev.p, keys.p, vals.p,
                                          cnt.p + d, mx.p + d);
        CK_LAUNCH();
        // stable: the claim order (ascending / descending rows) survives within a level
        CK(cub::DeviceRadixSort::SortPairs(ws.p, bytes, keys.p, keys2.p, vals.p,
                                           order.p + static_cast<size_t>(d) * n, n, 0, 32, s));
    }
    int hm[2];
    CK(cudaMemcpyAsync(hm, mx.p, sizeof hm, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    depth[0] = hm[0] + 1;
    depth[1] = hm[1] + 1;
}

void level_orders(const Bsr3 &A, const DevBuf<int> &dpos, DevBuf<int> &order, int (&depth)[2],
                  cudaStream_t s) {
    static const bool on_device = [] {
        const char *e = std::getenv("SAMG_ILU_LEVELS_HOST");
        return !(e && e[0] == '1');
    }();
    if (on_device && A.nrows > 0) return level_orders_device(A, dpos, order, depth, s);
    const int n = static_cast<int>(A.nrows);
    std::vector<int> ptr(n + 1), col(A.nnzb), dp(n);
    CK(cudaMemcpyAsync(ptr.data(), A.ptr.p, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(col.data(), A.col.p, sizeof(int) * A.nnzb, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(dp.data(), dpos.p, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<int> lev(n), ord(2 * static_cast<size_t>(n)), cnt;
    auto bucket = [&](int *out, bool ascending, int &nlev) {
        int maxl = 0;
        for (int i = 0; i < n; ++i) maxl = std::max(maxl, lev[i]);
        nlev = maxl + 1;
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
    bucket(ord.data(), true, depth[0]);
    for (int i = n - 1; i >= 0; --i) {
        int l = 0;
        for (int j = dp[i] + 1; j < ptr[i + 1]; ++j) l = std::max(l, lev[col[j]] + 1);
        lev[i] = l;
    }
    bucket(ord.data() + n, false, depth[1]);
    order.alloc(2 * static_cast<size_t>(n), s);
    CK(cudaMemcpyAsync(order.p, ord.data(), sizeof(int) * 2 * n, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));  // host vectors go out of scope
}

// ---- ilu0<double> on the scalar view --------------------------------------
// The scalar pipelines (and ns_hybrid1) smooth with the SCALAR ILU(0) of the
// level matrix (hierarchy.hpp:288-291, relaxation.hpp:20-139 with
// V = double).  Its scalar rows 3b, 3b+1, 3b+2 form block row b and the
// pattern is the blocks' entries, so the factors keep the 3x3 block layout
// (entry (3b+r, 3c+q) at lu[9j + 3r + q] for block j = (b, c)).  A scalar
// row depends on the scalar rows of the lower blocks of its block row and on
// the earlier scalar rows of its own block row: one warp per block row, in
// the block rows' dependency-level order (level_orders), its three scalar
// rows in sequence.  Every operation is the reference's, in its order.

// IKJ (relaxation.hpp:115-132) for the three scalar rows of a block row.
// The steps of a scalar row over its LOWER blocks only touch that row, so
// the three rows take them together: per lower block c (ascending) the U
// part of block row c (its diagonal block right of each pivot, then its
// blocks right of the diagonal, with their positions in row i found once)
// is read once and serves the 3 x 3 (row, pivot) steps -- for each scalar
// row the steps still run in ascending pivot order k = 3c + q, and each
// step updates distinct entries.  Then the within-block steps (k = 3i + q,
// q < r) run row by row.
__global__ void __launch_bounds__(256) k_ilu_factor_s(int n, const int *__restrict__ order,
        const int *__restrict__ ptr, const int *__restrict__ col, const int *__restrict__ dpos,
        double *lu, double *inv, int *done, int *counter, DevError *err) {
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
        double *rv = in_smem ? srow - 9LL * b : lu;
        const int *rc = in_smem ? scol - b : col;
        if (in_smem) {
            for (int q = lane; q < len; q += 32) scol[q] = col[b + q];
            for (int q = lane; q < 9 * len; q += 32) srow[q] = lu[9LL * b + q];
        }
        // every lower block row must be factored (flags, then acquire)
        for (int j = b + lane; j < di; j += 32)
            while (ld_relaxed(done + static_cast<int64_t>(col[j]) * kFS) == 0) {
            }
        __syncwarp();
        cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
        __syncwarp();
        for (int j = b; j < di; ++j) {
            const int c = rc[j];
            const int dc = __ldg(dpos + c), ec = __ldg(ptr + c + 1);
            double dg[9], iv[3];
#pragma unroll
            for (int q = 0; q < 9; ++q) dg[q] = __ldcg(lu + 9LL * dc + q);
#pragma unroll
            for (int q = 0; q < 3; ++q) iv[q] = __ldcg(inv + 3LL * c + q);
            // lanes own blocks l = dc+1+lane, +32, ... (up to kUB per lane):
            // their position in row i (or -1) and their 9 values, found /
            // loaded once for the three pivots q
            constexpr int kUB = 4;
            int upos[kUB];
            double uval[kUB][9];
            const bool cached = ec - dc - 1 <= 32 * kUB;
            if (cached) {
#pragma unroll
                for (int u = 0; u < kUB; ++u) {
                    const int l = dc + 1 + lane + 32 * u;
                    upos[u] = -1;
                    if (l < ec) {
                        const int cc = __ldg(col + l);
                        int lo = b, hi = e - 1;
                        while (lo <= hi) {
                            const int m = (lo + hi) >> 1, cm = rc[m];
                            if (cm == cc) { upos[u] = m; break; }
                            if (cm < cc) lo = m + 1;
                            else hi = m - 1;
                        }
                        if (upos[u] >= 0)
#pragma unroll
                            for (int v = 0; v < 9; ++v) uval[u][v] = __ldcg(lu + 9LL * l + v);
                    }
                }
            }
            for (int q = 0; q < 3; ++q) {
                // L_{r,k} for the three rows (k = 3c+q), then row k's entries
                // right of the pivot: diagonal block (q' > q) and higher blocks
                double L[3];
#pragma unroll
                for (int r = 0; r < 3; ++r) L[r] = __dmul_rn(rv[9LL * j + 3 * r + q], iv[q]);
                __syncwarp();
                if (lane < 3) rv[9LL * j + 3 * lane + q] = L[lane];
                if (lane < 3 * (2 - q)) {
                    const int r = lane % 3, qq = q + 1 + lane / 3;
                    double *dst = rv + 9LL * j + 3 * r + qq;
                    *dst = __dsub_rn(*dst, __dmul_rn(L[r], dg[3 * q + qq]));
                }
                auto update = [&](int pos, double u0, double u1, double u2) {
#pragma unroll
                    for (int r = 0; r < 3; ++r) {
                        double *dst = rv + 9LL * pos + 3 * r;
                        dst[0] = __dsub_rn(dst[0], __dmul_rn(L[r], u0));
                        dst[1] = __dsub_rn(dst[1], __dmul_rn(L[r], u1));
                        dst[2] = __dsub_rn(dst[2], __dmul_rn(L[r], u2));
                    }
                };
                if (cached) {
#pragma unroll
                    for (int u = 0; u < kUB; ++u)
                        if (upos[u] >= 0)
                            update(upos[u], uval[u][3 * q], uval[u][3 * q + 1], uval[u][3 * q + 2]);
                } else {
                    for (int l = dc + 1 + lane; l < ec; l += 32) {
                        const int cc = __ldg(col + l);
                        int lo = b, hi = e - 1, pos = -1;
                        while (lo <= hi) {
                            const int m = (lo + hi) >> 1, cm = rc[m];
                            if (cm == cc) { pos = m; break; }
                            if (cm < cc) lo = m + 1;
                            else hi = m - 1;
                        }
                        if (pos < 0) continue;
                        update(pos, __ldcg(lu + 9LL * l + 3 * q), __ldcg(lu + 9LL * l + 3 * q + 1),
                               __ldcg(lu + 9LL * l + 3 * q + 2));
                    }
                }
                __syncwarp();
            }
        }
        double own_inv[3] = {0.0, 0.0, 0.0};
        for (int r = 0; r < 3; ++r) {
            // steps k = 3i + q, q < r: the earlier scalar rows of this block row
            for (int q = 0; q < r; ++q) {
                const double L = __dmul_rn(rv[9LL * di + 3 * r + q], own_inv[q]);
                __syncwarp();
                if (lane == 0) rv[9LL * di + 3 * r + q] = L;
                if (lane < 2 - q) {
                    const int qq = q + 1 + lane;
                    double *dst = rv + 9LL * di + 3 * r + qq;
                    *dst = __dsub_rn(*dst, __dmul_rn(L, rv[9LL * di + 3 * q + qq]));
                }
                for (int l = di + 1 + lane; l < e; l += 32) {
                    double *dst = rv + 9LL * l + 3 * r;
#pragma unroll
                    for (int q2 = 0; q2 < 3; ++q2)
                        dst[q2] = __dsub_rn(dst[q2], __dmul_rn(L, rv[9LL * l + 3 * q + q2]));
                }
                __syncwarp();
            }
            // inverted pivot (value_traits<double>::inverse, static_block.hpp:170-173)
            const double piv = rv[9LL * di + 4 * r];
            if (fabs(piv) < 1e-300) {
                if (lane == 0) raise_err(err, SAMG_SINGULAR_BLOCK, 3LL * i + r);
                own_inv[r] = 0.0;
            } else {
                own_inv[r] = __ddiv_rn(1.0, piv);
            }
            __syncwarp();
        }
        if (in_smem)
            for (int q = lane; q < 9 * len; q += 32) lu[9LL * b + q] = srow[q];
        if (lane < 3) inv[3LL * i + lane] = own_inv[lane];
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            st_release(done + static_cast<int64_t>(i) * kFS, 1);
        }
    }
}

// The scalar triangular sweeps (relaxation.hpp:44-88, V = double), a warp
// per block row in level order, the output value its own flag (as
// k_ilu_sweep).  Forward: lanes 0..2 run the chains of scalar rows 3i+p over
// the lower blocks (ascending scalar columns), then the rows of the own
// block in sequence (their within-block terms come last).  Backward: the
// within-block terms come FIRST in each chain, so the rows run in sequence
// 3i+2, 3i+1, 3i, each over the products of the higher blocks formed in
// parallel per window; x_i = (chain) * inv_i; u_out = x (+ u_in,
// kernels::axpby(1, x, 1, u)).
constexpr int kWinS = 192;
constexpr int kSweepSmemS = 8 * kWinS * 9 * static_cast<int>(sizeof(double));

template <bool kFwd, bool kZero>
__global__ void __launch_bounds__(256) k_ilu_sweep_s(int n, const int *__restrict__ order,
        const int *__restrict__ ptr, const int *__restrict__ col, const int *__restrict__ dpos,
        const double *__restrict__ lu, const double *__restrict__ inv, const double *src,
        double *out, const double *u_in, double *u_out, unsigned *counter) {
    extern __shared__ __align__(16) double ssm[];  // per warp: kWinS x 9 products
    const int lane = threadIdx.x & 31;
    double *bs = ssm + static_cast<size_t>(threadIdx.x >> 5) * kWinS * 9;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(counter, 1u) + 1u;  // counter starts at 0xffffffff
        t = __shfl_sync(kFull, t, 0);
        if (t >= static_cast<unsigned>(n)) return;
        const int i = __ldg(order + t);
        const int di = __ldg(dpos + i);
        const int b = kFwd ? __ldg(ptr + i) : di + 1, e = kFwd ? di : __ldg(ptr + i + 1);
        double res[3];
        const double *dl = lu + 9LL * di;
        if constexpr (kFwd) {
            double a = lane < 3 ? src[3LL * i + lane] : 0.0;  // lane p: the chain of row 3i+p
            const double l10 = __ldg(dl + 3), l20 = __ldg(dl + 6), l21 = __ldg(dl + 7);  // ahead of the chain
            for (int w0 = b; w0 < e; w0 += kWinS) {
                const int m = min(kWinS, e - w0);
                for (int q = lane; q < 9 * m; q += 32) bs[q] = __ldg(lu + 9LL * w0 + q);
                __syncwarp();
                // each dependency: wait for its value, form its 9 products in place
                for (int d = lane; d < m; d += 32) {
                    const double *g = out + 3LL * __ldg(col + w0 + d);
                    unsigned long long v0, v1, v2;
                    do {
                        v0 = ld_poll(g); v1 = ld_poll(g + 1); v2 = ld_poll(g + 2);
                    } while (v0 == kSent || v1 == kSent || v2 == kSent);
                    const double x0 = __longlong_as_double(static_cast<long long>(v0)),
                                 x1 = __longlong_as_double(static_cast<long long>(v1)),
                                 x2 = __longlong_as_double(static_cast<long long>(v2));
                    double *bl = bs + 9 * d;
#pragma unroll
                    for (int r = 0; r < 3; ++r) {
                        bl[3 * r] = __dmul_rn(bl[3 * r], x0);
                        bl[3 * r + 1] = __dmul_rn(bl[3 * r + 1], x1);
                        bl[3 * r + 2] = __dmul_rn(bl[3 * r + 2], x2);
                    }
                }
                __syncwarp();
                if (lane < 3)  // the lower blocks' terms, the three chains in parallel
                    for (int d = 0; d < m; ++d) {
                        a = __dsub_rn(a, bs[9 * d + 3 * lane]);
                        a = __dsub_rn(a, bs[9 * d + 3 * lane + 1]);
                        a = __dsub_rn(a, bs[9 * d + 3 * lane + 2]);
                    }
                __syncwarp();  // the window's staging is reused
            }
            const double a0 = __shfl_sync(kFull, a, 0), a1 = __shfl_sync(kFull, a, 1),
                         a2 = __shfl_sync(kFull, a, 2);
            // own block, unit lower factor: y0; y1 - L10 y0; (y2 - L20 y0) - L21 y1
            res[0] = a0;
            res[1] = __dsub_rn(a1, __dmul_rn(l10, res[0]));
            res[2] = __dsub_rn(__dsub_rn(a2, __dmul_rn(l20, res[0])), __dmul_rn(l21, res[1]));
        } else {
            // rows 3i+2, 3i+1, 3i in sequence; each chain: y, the own block's
            // terms right of the diagonal, then the higher blocks' products
            // (windows of 3*kWinS dependencies, 3 products each); every lane
            // carries the same chain (the products come from shared memory)
            constexpr int kWinB = 3 * kWinS;
            for (int r = 2; r >= 0; --r) {
                double c = __ldcg(src + 3LL * i + r);
                // the pivot and the factor entries are read before the polls:
                // after them they add a memory round trip to every hand-off
                const double piv = __ldg(inv + 3LL * i + r);
                for (int q = r + 1; q < 3; ++q) c = __dsub_rn(c, __dmul_rn(__ldg(dl + 3 * r + q), res[q]));
                for (int w0 = b; w0 < e; w0 += kWinB) {
                    const int m = min(kWinB, e - w0);
                    for (int d = lane; d < m; d += 32) {
                        const double *g = out + 3LL * __ldg(col + w0 + d);
                        const double *u = lu + 9LL * (w0 + d) + 3 * r;
                        const double f0 = __ldg(u), f1 = __ldg(u + 1), f2 = __ldg(u + 2);
                        unsigned long long v0, v1, v2;
                        do {
                            v0 = ld_poll(g); v1 = ld_poll(g + 1); v2 = ld_poll(g + 2);
                        } while (v0 == kSent || v1 == kSent || v2 == kSent);
                        bs[3 * d] = __dmul_rn(f0, __longlong_as_double(static_cast<long long>(v0)));
                        bs[3 * d + 1] = __dmul_rn(f1, __longlong_as_double(static_cast<long long>(v1)));
                        bs[3 * d + 2] = __dmul_rn(f2, __longlong_as_double(static_cast<long long>(v2)));
                    }
                    __syncwarp();
                    for (int d = 0; d < 3 * m; ++d) c = __dsub_rn(c, bs[d]);
                    __syncwarp();
                }
                res[r] = __dmul_rn(c, piv);
            }
        }
        if (lane < 3) {
            st_publish(out + 3LL * i + lane, res[lane]);
            if constexpr (!kFwd)
                u_out[3LL * i + lane] = kZero ? res[lane] : __dadd_rn(res[lane], u_in[3LL * i + lane]);
        }
        __syncwarp();
    }
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
    M.flags.alloc(A.nrows * kFS + 2, s);
    M.sweep.alloc(6 * A.nrows + 1, s);
    if (n == 0) return;
    k_ilu_dpos<<<ceil_div(n, 256), 256, 0, s>>>(n, A.ptr.p, A.col.p, M.dpos.p, err);
    CK_LAUNCH();
    check_dev_error(err, s);  // no factorization without every diagonal
    static const bool timing = [] {
        const char *e = std::getenv("SAMG_SETUP_TIMING");
        return e && e[0] == '1';
    }();
    const auto t0 = std::chrono::steady_clock::now();
    level_orders(A, M.dpos, M.order, M.depth, s);
    const auto t1 = std::chrono::steady_clock::now();
    CK(cudaMemcpyAsync(M.lu.p, A.val.p, sizeof(double) * 9 * A.nnzb, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemsetAsync(M.flags.p, 0, sizeof(int) * (A.nrows * kFS + 2), s));
    constexpr int fsmem = 8 * kFMax * (9 * static_cast<int>(sizeof(double)) + static_cast<int>(sizeof(int)));
    static DeviceCache fattr;
    fattr.get([] {
        CK(cudaFuncSetAttribute(k_ilu_factor, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem));
        return 1;
    });
    k_ilu_factor<<<persistent_grid(reinterpret_cast<const void *>(k_ilu_factor), n), 256, fsmem, s>>>(
        n, M.order.p, A.ptr.p, A.col.p, M.dpos.p, M.lu.p, M.data.p, M.flags.p,
        M.flags.p + static_cast<int64_t>(n) * kFS, err);
    CK_LAUNCH();
    if (timing) {
        CK(cudaStreamSynchronize(s));
        const auto t2 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "  ilu0 %d rows: level orders %.3f ms, factorization %.3f ms (depth %d / %d)\n", n,
                     std::chrono::duration<double, std::milli>(t1 - t0).count(),
                     std::chrono::duration<double, std::milli>(t2 - t1).count(), M.depth[0], M.depth[1]);
    }
}

void setup_ilu0_scalar(const Bsr3 &A, Smoother &M, DevError *err, cudaStream_t s) {
    if (A.nrows != A.ncols) fail(SAMG_NON_SQUARE, "ilu0: matrix must be square");
    const int n = static_cast<int>(A.nrows);
    M.kind = SM_ILU;
    M.scalar = true;
    M.ptr = A.ptr.p;
    M.col = A.col.p;
    M.nrows = A.nrows;
    M.nnzb = A.nnzb;
    M.data.alloc(3 * A.nrows + 3, s);
    M.lu.alloc(9 * A.nnzb + 1, s);
    M.tmp.alloc(3 * A.nrows + 3, s);
    M.dpos.alloc(A.nrows + 1, s);
    M.flags.alloc(A.nrows * kFS + 2, s);
    M.sweep.alloc(6 * A.nrows + 1, s);
    if (n == 0) return;
    k_ilu_dpos<<<ceil_div(n, 256), 256, 0, s>>>(n, A.ptr.p, A.col.p, M.dpos.p, err);
    CK_LAUNCH();
    check_dev_error(err, s);
    level_orders(A, M.dpos, M.order, M.depth, s);
    CK(cudaMemcpyAsync(M.lu.p, A.val.p, sizeof(double) * 9 * A.nnzb, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemsetAsync(M.flags.p, 0, sizeof(int) * (A.nrows * kFS + 2), s));
    constexpr int fsmem = 8 * kFMax * (9 * static_cast<int>(sizeof(double)) + static_cast<int>(sizeof(int)));
    static DeviceCache fattr;
    fattr.get([] {
        CK(cudaFuncSetAttribute(k_ilu_factor_s, cudaFuncAttributeMaxDynamicSharedMemorySize, fsmem));
        return 1;
    });
    k_ilu_factor_s<<<persistent_grid(reinterpret_cast<const void *>(k_ilu_factor_s), n), 256, fsmem, s>>>(
        n, M.order.p, A.ptr.p, A.col.p, M.dpos.p, M.lu.p, M.data.p, M.flags.p,
        M.flags.p + static_cast<int64_t>(n) * kFS, err);
    CK_LAUNCH();
}

void launch_ilu_smooth(const Bsr3 *A, const Smoother &M, const double *f, const double *u_in,
                       double *u_out, cudaStream_t s, bool lowp) {
    const int n = static_cast<int>(M.nrows);
    if (n == 0) return;
    // [y | x | two row counters]: sentinel-filled by one memset (the counters
    // start at 0xffffffff, see k_ilu_sweep)
    double *y = M.sweep.p, *x = M.sweep.p + 3LL * n;
    unsigned *cnt = reinterpret_cast<unsigned *>(M.sweep.p + 6LL * n);
    CK(cudaMemsetAsync(M.sweep.p, 0xff, sizeof(double) * (6LL * n + 1), s));
    const double *rin = f;
    if (u_in) {
        launch_residual(*A, f, u_in, M.tmp.p, s, lowp);  // r = f - A u (hierarchy.hpp:213-215)
        rin = M.tmp.p;
    }
    static DeviceCache gf_cache;
    const int gf = gf_cache.get([] {
        for (const void *k : {reinterpret_cast<const void *>(k_ilu_sweep<true, true>),
                               reinterpret_cast<const void *>(k_ilu_sweep<false, false>),
                               reinterpret_cast<const void *>(k_ilu_sweep<false, true>),
                               reinterpret_cast<const void *>(k_ilu_sweep<false, false, true>),
                               reinterpret_cast<const void *>(k_ilu_sweep<false, true, true>)})
            CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepSmem));
        const char *e = std::getenv("SAMG_ILU_CTAS_PER_SM");
        return persistent_grid(reinterpret_cast<const void *>(k_ilu_sweep<true, true>), 1 << 30, kSweepSmem,
                               e ? 0 : 2);
    });
    // warps for about kAhead dependency levels: a warp spins on the rows it
    // waits for, and warps far ahead of the wavefront only load L2 (coarse
    // levels have a few rows per level)
    static const int ahead = [] {
        const char *e = std::getenv("SAMG_ILU_AHEAD");
        return e ? std::max(1, std::atoi(e)) : 16;
    }();
    // (latest-last order: both sweeps hand off at the chain's end, and twice
    // the rows ahead on 3 CTAs per SM measured 4.6 % faster on C1 -- 0.278 ->
    // 0.265 s; the reference order lost 1 % with it)
    static const bool env_ctas = std::getenv("SAMG_ILU_CTAS_PER_SM") != nullptr;
    static const bool env_ahead = std::getenv("SAMG_ILU_AHEAD") != nullptr;
    const int64_t gcap = M.latest_last && !env_ctas ? gf / 2 * 3 : gf;
    const int64_t look = M.latest_last && !env_ahead ? 2 * ahead : ahead;
    auto grid_for = [&](int depth) {
        const int64_t warps = (look * n + depth - 1) / std::max(depth, 1);
        return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(gcap, (std::min<int64_t>(warps, n) + 7) / 8)));
    };
    const int gridf = grid_for(M.depth[0]), gridb = grid_for(M.depth[1]);
    const int *of = M.order.p, *ob = M.order.p + n;
    if (M.scalar) {  // ilu0<double>
        static DeviceCache sattr;
        sattr.get([] {
            for (const void *k : {reinterpret_cast<const void *>(k_ilu_sweep_s<true, true>),
                                   reinterpret_cast<const void *>(k_ilu_sweep_s<false, false>),
                                   reinterpret_cast<const void *>(k_ilu_sweep_s<false, true>)})
                CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSweepSmemS));
            return 1;
        });
        const int gs = std::max(1, std::min(gridf, sm_count()));  // one 8-warp CTA per SM (110 KB)
        const int gb = std::max(1, std::min(gridb, sm_count()));
        k_ilu_sweep_s<true, true><<<gs, 256, kSweepSmemS, s>>>(n, of, M.ptr, M.col, M.dpos.p, M.lu.p,
                                                              M.data.p, rin, y, nullptr, nullptr, cnt);
        if (u_in)
            k_ilu_sweep_s<false, false><<<gb, 256, kSweepSmemS, s>>>(n, ob, M.ptr, M.col, M.dpos.p, M.lu.p,
                                                                    M.data.p, y, x, u_in, u_out, cnt + 1);
        else
            k_ilu_sweep_s<false, true><<<gb, 256, kSweepSmemS, s>>>(n, ob, M.ptr, M.col, M.dpos.p, M.lu.p,
                                                                   M.data.p, y, x, nullptr, u_out, cnt + 1);
        CK_LAUNCH();
        return;
    }
    k_ilu_sweep<true, true><<<gridf, 256, kSweepSmem, s>>>(n, of, M.ptr, M.col, M.dpos.p, M.lu.p, M.data.p,
                                                          rin, y, nullptr, nullptr, cnt);
    if (M.latest_last) {
        if (u_in)
            k_ilu_sweep<false, false, true><<<gridb, 256, kSweepSmem, s>>>(n, ob, M.ptr, M.col, M.dpos.p, M.lu.p,
                                                                          M.data.p, y, x, u_in, u_out, cnt + 1);
        else
            k_ilu_sweep<false, true, true><<<gridb, 256, kSweepSmem, s>>>(n, ob, M.ptr, M.col, M.dpos.p, M.lu.p,
                                                                         M.data.p, y, x, nullptr, u_out, cnt + 1);
    } else if (u_in)
        k_ilu_sweep<false, false><<<gridb, 256, kSweepSmem, s>>>(n, ob, M.ptr, M.col, M.dpos.p, M.lu.p,
                                                                M.data.p, y, x, u_in, u_out, cnt + 1);
    else
        k_ilu_sweep<false, true><<<gridb, 256, kSweepSmem, s>>>(n, ob, M.ptr, M.col, M.dpos.p, M.lu.p,
                                                               M.data.p, y, x, nullptr, u_out, cnt + 1);
    CK_LAUNCH();
}

} // namespace samgb
