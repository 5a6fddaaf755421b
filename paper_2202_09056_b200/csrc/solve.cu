// solve.cu -- solve-phase kernels: 3x3-BSR SpMV family (spmv, residual,
// fused smoother sweep, fused CG matvec+dot), coarse dense GEMV and the CG
// vector kernels with deterministic, launch-free reductions.
//
// All of these are HBM-bandwidth bound (18 flop per 76 B of matrix; DESIGN.md
// section 5).  A group of G lanes owns one block row; G in {1,...,128} is
// chosen per matrix (choose_group): ~7 blocks per lane, widened until the
// matrix fills 148 SMs (coarse levels, restriction).  Default kernel
// (variant 1): lane l accumulates whole 3x3 blocks beg+l, beg+l+G, ... with
// 16-byte loads, so the row's 72-byte blocks stream as contiguous, coalesced
// bytes; col[] is read once per block and x[3c..3c+2] is a gather that hits
// L1/L2 (structured meshes keep the column window small).  Long rows (a warp
// or two per row, G = 32 / 64) run variant 2: variant 1 with col read one
// iteration ahead (row_sums_pipe); large matrices the TMA-fed persistent
// kernel (variant 3, k_bsr3_tma).  Variant 0 (row
// units: lane l handles scalar row l%3 of every block, G in {8,16,32}) is kept
// for comparison (SAMG_SPMV_VARIANT=0).  The three row sums are combined with
// a width-G butterfly (plus shared memory for G > 32) and the epilogue
// (spmv / residual / smoother sweep / CG dot) is fused.
#include <cuda/atomic>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"

namespace samgb {

namespace {

// ---- programmatic dependent launch (PDL) ------------------------------------
// Back-to-back standalone SpMVs (samg_bsr3_spmv_device: a caller's loop of
// y = A x) are launched with programmatic stream serialization: SpMV k+1 is
// scheduled while the last CTAs of SpMV k run, its TMA producer streams the
// matrix at once (independent of k), and its consumers read x only after
// griddepcontrol.wait (k complete, its writes visible) plus a GPU-scope
// acquire fence.  The fence is needed: a dependent grid is not preceded by
// the launch-time L1 invalidation of a normal launch, and x is gathered
// through L1 (measured: without it CG lost its convergence).  Inside the
// CG graph PDL is not used: the fence and the early-resident dependents cost
// more than the overlapped tails gained (C1 0.521 -> 0.546 ms per
// iteration, C4 13.9 -> 17.7 ms; profiles/README.md).  SAMG_PDL=0 disables.
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("SAMG_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}
thread_local bool g_spmv_pdl = false;  // set around standalone SpMV launches

// L2 cache policies (SAMG_L2_HINTS, default on): the TMA matrix streams
// evict-first, the coarse inverse evict-last (it is re-read every V-cycle)
bool l2_hints() {
    static const bool on = [] {
        const char *e = std::getenv("SAMG_L2_HINTS");
        return !(e && e[0] == '0');
    }();
    return on;
}

// kernel launch, with the PDL attribute if `pdl` (the kernel then calls
// pdl_wait before it reads a predecessor's output)
template <class... KArgs, class... Args>
void launch_k(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
              Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

__device__ __forceinline__ double ld_stream(const double *p) { return __ldcs(p); }

__device__ __forceinline__ double2 ldg2(const double *p) {
    return __ldg(reinterpret_cast<const double2 *>(p));
}

// Sum three values over the G lanes of a group; every lane gets the totals.
// G > 32 spans G/32 warps of the 256-thread CTA (shared memory, CTA barrier:
// every thread of the CTA must call it).
template <int G, int kThreads = 256>
__device__ __forceinline__ void group_reduce3(double &v0, double &v1, double &v2) {
    constexpr int W = G < 32 ? G : 32;
#pragma unroll
    for (int off = W / 2; off >= 1; off >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, off, W);
        v1 += __shfl_xor_sync(0xffffffffu, v1, off, W);
        v2 += __shfl_xor_sync(0xffffffffu, v2, off, W);
    }
    if constexpr (G > 32) {
        __shared__ double red[3][kThreads / 32];
        const int w = threadIdx.x / 32;
        if (threadIdx.x % 32 == 0) { red[0][w] = v0; red[1][w] = v1; red[2][w] = v2; }
        __syncthreads();
        const int g0 = (threadIdx.x / G) * (G / 32);
        v0 = v1 = v2 = 0.0;
#pragma unroll
        for (int k = 0; k < G / 32; ++k) { v0 += red[0][g0 + k]; v1 += red[1][g0 + k]; v2 += red[2][g0 + k]; }
        __syncthreads();
    }
}

// Variant 0: row units (G in {8,16,32}, U = G - G%3 active lanes).
template <int G>
__device__ __forceinline__ void row_sums_units(int row, bool valid, int lane,
        const int *__restrict__ ptr, const int *__restrict__ col,
        const double *__restrict__ val, const double *__restrict__ x,
        double &s0, double &s1, double &s2) {
    constexpr int U = G - G % 3;
    double s = 0.0, t2 = 0.0;
    if (valid && lane < U) {
        const int beg = __ldg(ptr + row), end = __ldg(ptr + row + 1);
        const int nu = 3 * (end - beg);
        const double *v = val + 9 * static_cast<size_t>(beg);
        const int *cc = col + beg;
        int t = lane;
        for (; t + U < nu; t += 2 * U) {
            const int c0 = __ldg(cc + t / 3), c1 = __ldg(cc + (t + U) / 3);
            const double *x0 = x + 3 * c0, *x1 = x + 3 * c1;
            s = fma(ld_stream(v + 3 * t), __ldg(x0), s);
            s = fma(ld_stream(v + 3 * t + 1), __ldg(x0 + 1), s);
            s = fma(ld_stream(v + 3 * t + 2), __ldg(x0 + 2), s);
            t2 = fma(ld_stream(v + 3 * (t + U)), __ldg(x1), t2);
            t2 = fma(ld_stream(v + 3 * (t + U) + 1), __ldg(x1 + 1), t2);
            t2 = fma(ld_stream(v + 3 * (t + U) + 2), __ldg(x1 + 2), t2);
        }
        if (t < nu) {
            const double *x0 = x + 3 * __ldg(cc + t / 3);
            s = fma(ld_stream(v + 3 * t), __ldg(x0), s);
            s = fma(ld_stream(v + 3 * t + 1), __ldg(x0 + 1), s);
            s = fma(ld_stream(v + 3 * t + 2), __ldg(x0 + 2), s);
        }
        s += t2;
    }
    const int r = lane % 3;
    s0 = (r == 0) ? s : 0.0;
    s1 = (r == 1) ? s : 0.0;
    s2 = (r == 2) ? s : 0.0;
    group_reduce3<G>(s0, s1, s2);
}

// Variant 1: block per lane.  A block (72 B) is read with four 16-byte loads
// plus one 8-byte load whose offsets depend only on the parity of j (block j
// starts 16-byte aligned iff j is even), so every lane runs the same
// instruction sequence; x[3c..3c+2] likewise with one 16-byte + one 8-byte
// load.  Per block: 1 col + 5 value + 2 x loads.
// A block as 9 doubles from its 9 stored values v[0..8] (element offset of
// v in its array has parity `odd`): fp64 -- four 16-byte + one 8-byte load;
// fp32 (mixed-precision V-cycle storage) -- four 8-byte + one 4-byte load.
// kNc: read-only global path (ld.global.nc), else a generic (shared) load.
template <bool kNc>
__device__ __forceinline__ void blk9(const double *v, int odd, double (&b)[9]) {
    auto l2 = [](const double *p) {
        if constexpr (kNc) return ldg2(p);
        else return *reinterpret_cast<const double2 *>(p);
    };
    const double2 q0 = l2(v + odd), q1 = l2(v + odd + 2), q2 = l2(v + odd + 4), q3 = l2(v + odd + 6);
    const double e = kNc ? __ldg(v + (odd ? 0 : 8)) : v[odd ? 0 : 8];
    b[0] = odd ? e : q0.x; b[1] = odd ? q0.x : q0.y; b[2] = odd ? q0.y : q1.x;
    b[3] = odd ? q1.x : q1.y; b[4] = odd ? q1.y : q2.x; b[5] = odd ? q2.x : q2.y;
    b[6] = odd ? q2.y : q3.x; b[7] = odd ? q3.x : q3.y; b[8] = odd ? q3.y : e;
}
template <bool kNc>
__device__ __forceinline__ void blk9(const float *v, int odd, double (&b)[9]) {
    auto l2 = [](const float *p) {
        if constexpr (kNc) return __ldg(reinterpret_cast<const float2 *>(p));
        else return *reinterpret_cast<const float2 *>(p);
    };
    const float2 q0 = l2(v + odd), q1 = l2(v + odd + 2), q2 = l2(v + odd + 4), q3 = l2(v + odd + 6);
    const float e = kNc ? __ldg(v + (odd ? 0 : 8)) : v[odd ? 0 : 8];
    b[0] = odd ? e : q0.x; b[1] = odd ? q0.x : q0.y; b[2] = odd ? q0.y : q1.x;
    b[3] = odd ? q1.x : q1.y; b[4] = odd ? q1.y : q2.x; b[5] = odd ? q2.x : q2.y;
    b[6] = odd ? q2.y : q3.x; b[7] = odd ? q3.x : q3.y; b[8] = odd ? q3.y : e;
}

// kNcX = false: x is gathered through L2 only (ld.global.cg) -- inside the
// persistent V-cycle tail x was written by other CTAs of the same launch, so
// neither the read-only path nor L1 may serve it.
template <int G, class VT = double, bool kNcX = true, int kThreads = 256>
__device__ __forceinline__ void row_sums_blocks(int row, bool valid, int lane,
        const int *__restrict__ ptr, const int *__restrict__ col,
        const VT *__restrict__ val, const double *__restrict__ x,
        double &s0, double &s1, double &s2) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    // blocks in flight per lane: fp32 blocks are half the bytes, so twice as many
    constexpr int kUnr = sizeof(VT) == 4 ? 4 : 2;
    if (valid) {
        const int beg = __ldg(ptr + row), end = __ldg(ptr + row + 1);
#pragma unroll kUnr
        for (int j = beg + lane; j < end; j += G) {
            const int c = __ldg(col + j);
            double bb[9];
            blk9<true>(val + 9 * static_cast<size_t>(j), j & 1, bb);
            const double *xp = x + 3 * static_cast<size_t>(c);
            const int xo = c & 1;
            const double2 xq = kNcX ? ldg2(xp + xo) : __ldcg(reinterpret_cast<const double2 *>(xp + xo));
            const double xe = kNcX ? __ldg(xp + (xo ? 0 : 2)) : __ldcg(xp + (xo ? 0 : 2));
            const double x0 = xo ? xe : xq.x, x1 = xo ? xq.x : xq.y, x2 = xo ? xq.y : xe;
            const double b0 = bb[0], b1 = bb[1], b2 = bb[2], b3 = bb[3], b4 = bb[4], b5 = bb[5],
                         b6 = bb[6], b7 = bb[7], b8 = bb[8];
            a0 = fma(b0, x0, a0); a0 = fma(b1, x1, a0); a0 = fma(b2, x2, a0);
            a1 = fma(b3, x0, a1); a1 = fma(b4, x1, a1); a1 = fma(b5, x2, a1);
            a2 = fma(b6, x0, a2); a2 = fma(b7, x1, a2); a2 = fma(b8, x2, a2);
        }
    }
    s0 = a0; s1 = a1; s2 = a2;
    group_reduce3<G, kThreads>(s0, s1, s2);
}

// Variant 2 (long rows, a warp per row; SAMG_LONG_PIPE=0 restores variant 1):
// variant 1 with col read one iteration ahead, so an iteration's x gather is
// issued together with its value loads instead of after a col round trip of
// its own: the row's chain is ptr -> col -> {val, x} -> {val, x} ... instead
// of ptr -> {col, val} -> x -> {col, val} -> x ...  Same blocks per lane in
// the same order: identical sums.  Compiled for 5 CTAs per SM (<= 51
// registers; ptxas otherwise takes 52 for most epilogues and loses a CTA).
// C1's level-1 kernels: 42.6 / 33.3 / 32.6 -> 40.6 / 30.6 / 30.1 us; the
// G = 64 rows of its level 2 gain another 2.5 us per iteration.
template <int G, class VT = double>
__device__ __forceinline__ void row_sums_pipe(int row, bool valid, int lane,
        const int *__restrict__ ptr, const int *__restrict__ col,
        const VT *__restrict__ val, const double *__restrict__ x,
        double &s0, double &s1, double &s2) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    if (valid) {
        const int beg = __ldg(ptr + row), end = __ldg(ptr + row + 1);
        int j = beg + lane;
        int c0 = j < end ? __ldg(col + j) : -1, c1 = j + G < end ? __ldg(col + j + G) : -1;
        // both blocks of a pair in flight together (no branch between them)
        auto load = [&](int jj, int c, double (&bb)[9], double &x0, double &x1, double &x2) {
            blk9<true>(val + 9 * static_cast<size_t>(jj), jj & 1, bb);
            const double *xp = x + 3 * static_cast<size_t>(c);
            const int xo = c & 1;
            const double2 xq = ldg2(xp + xo);
            const double xe = __ldg(xp + (xo ? 0 : 2));
            x0 = xo ? xe : xq.x;
            x1 = xo ? xq.x : xq.y;
            x2 = xo ? xq.y : xe;
        };
        auto acc = [&](const double (&bb)[9], double x0, double x1, double x2) {
            a0 = fma(bb[0], x0, a0); a0 = fma(bb[1], x1, a0); a0 = fma(bb[2], x2, a0);
            a1 = fma(bb[3], x0, a1); a1 = fma(bb[4], x1, a1); a1 = fma(bb[5], x2, a1);
            a2 = fma(bb[6], x0, a2); a2 = fma(bb[7], x1, a2); a2 = fma(bb[8], x2, a2);
        };
        for (; j + G < end; j += 2 * G) {
            const int n0 = j + 2 * G < end ? __ldg(col + j + 2 * G) : -1;
            const int n1 = j + 3 * G < end ? __ldg(col + j + 3 * G) : -1;
            double b0[9], b1[9], p0, p1, p2, q0, q1, q2;
            load(j, c0, b0, p0, p1, p2);
            load(j + G, c1, b1, q0, q1, q2);
            acc(b0, p0, p1, p2);
            acc(b1, q0, q1, q2);
            c0 = n0;
            c1 = n1;
        }
        if (j < end) {
            double b0[9], p0, p1, p2;
            load(j, c0, b0, p0, p1, p2);
            acc(b0, p0, p1, p2);
        }
    }
    s0 = a0; s1 = a1; s2 = a2;
    group_reduce3<G>(s0, s1, s2);
}

template <int G, int V, class VT>
__device__ __forceinline__ void row_sums(int row, bool valid, int lane, const int *__restrict__ ptr,
        const int *__restrict__ col, const VT *__restrict__ val,
        const double *__restrict__ x, double &s0, double &s1, double &s2) {
    if constexpr (V == 0 && std::is_same_v<VT, double>) row_sums_units<G>(row, valid, lane, ptr, col, val, x, s0, s1, s2);
    else if constexpr (V == 2) row_sums_pipe<G, VT>(row, valid, lane, ptr, col, val, x, s0, s1, s2);
    else row_sums_blocks<G, VT>(row, valid, lane, ptr, col, val, x, s0, s1, s2);
}

__device__ __forceinline__ double pick3(int c, double a, double b, double d) {
    return c == 0 ? a : (c == 1 ? b : d);
}

// Run the epilogue for the three components of `row`: lanes 0..2 in
// parallel, or lane 0 for all three when G < 3.  Returns sum over the
// handled components of epi's dot contribution (0 if none).
template <int G, class Epi>
__device__ __forceinline__ double epilogue(const Epi &epi, int row, int lane, double s0, double s1,
                                           double s2) {
    double d = 0.0;
    if constexpr (G >= 3) {
        if (lane < 3) d = epi(row, lane, s0, s1, s2);
    } else {
        if (lane == 0)
            for (int c = 0; c < 3; ++c) d += epi(row, c, s0, s1, s2);
    }
    return d;
}

// Bulk L2 prefetch (cp.async.bulk.prefetch, sm_90+) of `bytes` from p,
// widened to 16-byte bounds: the TMA producer issues it for the rows of a
// chunk it has just scheduled, so the epilogue's per-row vector loads hit L2.
__device__ __forceinline__ void bulk_prefetch(const void *p, size_t bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uintptr_t b = a & ~static_cast<uintptr_t>(15), e = (a + bytes + 15) & ~static_cast<uintptr_t>(15);
    if (e > b)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b), "r"(static_cast<unsigned>(e - b))
                     : "memory");
}

struct EpiSpmv {
    double alpha, beta;
    double *y;
    __device__ void prefetch(int r0, int n) const {
        if (beta != 0.0) bulk_prefetch(y + 3 * static_cast<size_t>(r0), 24 * static_cast<size_t>(n));
    }
    __device__ double operator()(int row, int c, double s0, double s1, double s2) const {
        double *yi = y + 3 * static_cast<size_t>(row) + c;
        const double s = pick3(c, s0, s1, s2);
        *yi = alpha * s + (beta == 0.0 ? 0.0 : beta * *yi);
        return 0.0;
    }
};

struct EpiResidual {
    const double *f;
    double *r;
    __device__ void prefetch(int r0, int n) const {
        bulk_prefetch(f + 3 * static_cast<size_t>(r0), 24 * static_cast<size_t>(n));
    }
    __device__ double operator()(int row, int c, double s0, double s1, double s2) const {
        const size_t i = 3 * static_cast<size_t>(row) + c;
        r[i] = f[i] - pick3(c, s0, s1, s2);
        return 0.0;
    }
};

// u_out = u + (omega/a_cc) * (f - A u); returns f*u_out (for r.z)
struct EpiSmoothPoint {
    const double *f, *u, *m;
    double *out;
    __device__ void prefetch(int r0, int n) const {
        const size_t o = 3 * static_cast<size_t>(r0), b = 24 * static_cast<size_t>(n);
        bulk_prefetch(f + o, b);
        bulk_prefetch(u + o, b);
        bulk_prefetch(m + o, b);
    }
    __device__ double operator()(int row, int c, double s0, double s1, double s2) const {
        const size_t i = 3 * static_cast<size_t>(row) + c;
        const double fi = f[i];
        const double o = u[i] + m[i] * (fi - pick3(c, s0, s1, s2));
        out[i] = o;
        return fi * o;
    }
};

// u_out = u + M_row (f - A u)_row; returns f*u_out
struct EpiSmoothBlock {
    const double *f, *u, *m;
    double *out;
    __device__ void prefetch(int r0, int n) const {
        const size_t o = 3 * static_cast<size_t>(r0), b = 24 * static_cast<size_t>(n);
        bulk_prefetch(f + o, b);
        bulk_prefetch(u + o, b);
        bulk_prefetch(m + 3 * o, 3 * b);
    }
    __device__ double operator()(int row, int c, double s0, double s1, double s2) const {
        const size_t b = 3 * static_cast<size_t>(row);
        const double r0 = f[b] - s0, r1 = f[b + 1] - s1, r2 = f[b + 2] - s2;
        const double *M = m + 9 * static_cast<size_t>(row) + 3 * c;
        const double o = u[b + c] + (M[0] * r0 + M[1] * r1 + M[2] * r2);
        out[b + c] = o;
        return f[b + c] * o;
    }
};

// Restriction fused with the next level's first smoothing sweep from a zero
// guess: f_c = (R r)_row, u_c = M_row f_c (hierarchy.hpp:429 then :426 /
// relaxation.hpp:165-173 with u = 0: the residual is f_c exactly).
// kBlock: 3x3 M_i; else point (3 per row).
template <bool kBlock>
struct EpiRestrictSmooth {
    double *f, *u;
    const double *m;
    __device__ void prefetch(int r0, int n) const {
        bulk_prefetch(m + (kBlock ? 9 : 3) * static_cast<size_t>(r0),
                      (kBlock ? 72 : 24) * static_cast<size_t>(n));
    }
    __device__ double operator()(int row, int c, double s0, double s1, double s2) const {
        const size_t b = 3 * static_cast<size_t>(row);
        f[b + c] = pick3(c, s0, s1, s2);
        if constexpr (kBlock) {
            const double *M = m + 9 * static_cast<size_t>(row) + 3 * c;
            u[b + c] = M[0] * s0 + M[1] * s1 + M[2] * s2;
        } else {
            u[b + c] = m[b + c] * pick3(c, s0, s1, s2);
        }
        return 0.0;
    }
};

// q = A p; returns p*q (CG p'Ap)
struct EpiDot {
    const double *p;
    double *q;
    __device__ void prefetch(int r0, int n) const {
        bulk_prefetch(p + 3 * static_cast<size_t>(r0), 24 * static_cast<size_t>(n));
    }
    __device__ double operator()(int row, int c, double s0, double s1, double s2) const {
        const size_t i = 3 * static_cast<size_t>(row) + c;
        const double qi = pick3(c, s0, s1, s2);
        q[i] = qi;
        return p[i] * qi;
    }
};

template <int G, int V, class Epi, class VT = double>
__global__ void __launch_bounds__(256, V == 2 ? 5 : 0) k_bsr3(int nrows, const int *__restrict__ ptr,
        const int *__restrict__ col, const VT *__restrict__ val,
        const double *__restrict__ x, Epi epi) {
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int row = gtid / G, lane = threadIdx.x % G;
    const bool valid = row < nrows;
    double s0, s1, s2;
    row_sums<G, V, VT>(row, valid, lane, ptr, col, val, x, s0, s1, s2);
    if (valid) epilogue<G>(epi, row, lane, s0, s1, s2);
}

// Same over an explicit row list (interior / boundary rows of a partition).
template <int G, class Epi>
__global__ void __launch_bounds__(256) k_bsr3_rows(int nlist, const int *__restrict__ rows,
        const int *__restrict__ ptr, const int *__restrict__ col,
        const double *__restrict__ val, const double *__restrict__ x, Epi epi) {
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int g = gtid / G, lane = threadIdx.x % G;
    const bool valid = g < nlist;
    const int row = valid ? __ldg(rows + g) : 0;
    double s0, s1, s2;
    row_sums<G, 1, double>(row, valid, lane, ptr, col, val, x, s0, s1, s2);
    if (valid) epilogue<G>(epi, row, lane, s0, s1, s2);
}

// 6x6 node-blocked SpMV family (make_node6): a group of G lanes per node row
// (2 block rows); a lane pair shares a 6x6 block -- lane 2m+h takes its
// half-rows 3h..3h+2 (nine 16-byte loads, 144 B) and the whole 48-byte x
// gather (three 16-byte loads) of blocks beg+m, beg+m+G/2, ...  The three
// half-row sums are combined over the lanes of the same half, then lane h
// runs the epilogue of block row 2 row + h.
template <int G, class Epi>
__global__ void __launch_bounds__(256) k_bsr6(int nrows6, const int *__restrict__ ptr,
        const int *__restrict__ col, const double *__restrict__ val,
        const double *__restrict__ x, Epi epi) {
    static_assert(G >= 2 && G <= 32, "k_bsr6: 2..32 lanes per node row");
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int row = gtid / G, lane = threadIdx.x % G;
    const int half = lane & 1, m = lane >> 1;
    const bool valid = row < nrows6;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    if (valid) {
        const int beg = __ldg(ptr + row), end = __ldg(ptr + row + 1);
#pragma unroll 2
        for (int j = beg + m; j < end; j += G / 2) {
            const int c = __ldg(col + j);
            const double2 *bp =
                reinterpret_cast<const double2 *>(val + 36 * static_cast<size_t>(j) + 18 * half);
            double2 b[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) b[k] = __ldg(bp + k);
            const double2 *xp = reinterpret_cast<const double2 *>(x + 6 * static_cast<size_t>(c));
            const double2 x01 = __ldg(xp), x23 = __ldg(xp + 1), x45 = __ldg(xp + 2);
            a0 = fma(b[0].x, x01.x, a0); a0 = fma(b[0].y, x01.y, a0); a0 = fma(b[1].x, x23.x, a0);
            a0 = fma(b[1].y, x23.y, a0); a0 = fma(b[2].x, x45.x, a0); a0 = fma(b[2].y, x45.y, a0);
            a1 = fma(b[3].x, x01.x, a1); a1 = fma(b[3].y, x01.y, a1); a1 = fma(b[4].x, x23.x, a1);
            a1 = fma(b[4].y, x23.y, a1); a1 = fma(b[5].x, x45.x, a1); a1 = fma(b[5].y, x45.y, a1);
            a2 = fma(b[6].x, x01.x, a2); a2 = fma(b[6].y, x01.y, a2); a2 = fma(b[7].x, x23.x, a2);
            a2 = fma(b[7].y, x23.y, a2); a2 = fma(b[8].x, x45.x, a2); a2 = fma(b[8].y, x45.y, a2);
        }
    }
#pragma unroll
    for (int off = G / 2; off >= 2; off >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, off, G);
        a1 += __shfl_xor_sync(0xffffffffu, a1, off, G);
        a2 += __shfl_xor_sync(0xffffffffu, a2, off, G);
    }
    if (valid && m == 0)
        for (int c = 0; c < 3; ++c) epi(2 * row + half, c, a0, a1, a2);
}

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double red[32];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int w = threadIdx.x / 32, l = threadIdx.x % 32;
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (w == 0) {
        const int nw = blockDim.x / 32;
        t = (l < nw) ? red[l] : 0.0;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    }
    __syncthreads();
    return t;  // valid in thread 0
}

// CG scalar updates (cg.hpp:58-77) applied to a finished dot product s.
__device__ void cg_apply(int what, double s, CgScalars *sc, cudaGraphConditionalHandle h) {
    switch (what) {
        case CG_RR: sc->rr = s; break;
        case CG_PQ:
            sc->pq = s;
            if (!(s > 0.0)) sc->breakdown = 1;
            sc->alpha = sc->rho / s;
            break;
        case CG_RZ:
            sc->rho_new = s;
            sc->beta = s / sc->rho;
            sc->rho = s;
            break;
        case CG_RHO: sc->rho = s; break;
        case CG_STORE: sc->tmp = s; break;
        case CG_STORE2: sc->tmp2 = s; break;
        case CG_ADD: sc->tmp += s; break;  // further row ranges of one product
        case CG_RR_LOOP: {
            sc->rr = s;
            const int it = sc->iter + 1;
            sc->iter = it;
            const bool go = (sqrt(s) / sc->norm_f > sc->tol) && it < sc->max_iter && !sc->breakdown;
            cudaGraphSetConditional(h, go ? 1u : 0u);
            break;
        }
        default: break;
    }
}

// Deterministic grid-wide reduction without a second launch: every CTA
// writes its partial, the last CTA to arrive (ticket) sums all partials in
// index order and applies the CG update.
__device__ void grid_finish(double d, double *partials, CgScalars *sc, int what,
                            cudaGraphConditionalHandle h) {
    __shared__ bool last;
    d = block_sum(d);
    if (threadIdx.x == 0) {
        // release: the partial is visible before the ticket (no L1 flush,
        // unlike __threadfence, so co-resident CTAs keep their cached x)
        __stcg(partials + blockIdx.x, d);
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> t(sc->ticket);
        last = t.fetch_add(1u, cuda::memory_order_release) == gridDim.x - 1;
        if (last) cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
    }
    __syncthreads();
    if (!last) return;
    double s = 0.0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) s += __ldcg(partials + i);
    s = block_sum(s);
    if (threadIdx.x == 0) {
        sc->ticket = 0;
        cg_apply(what, s, sc, h);
    }
}

// SpMV-family kernel whose epilogue also yields a dot product, finished by
// grid_finish: q = A p with p.q (CG), or the last smoothing sweep with r.z.
// Grid-stride over row groups with a fixed grid so partials are few.
template <int G, class Epi, class VT = double>
__global__ void __launch_bounds__(256) k_bsr3_reduce(int nrows, const int *__restrict__ ptr,
        const int *__restrict__ col, const VT *__restrict__ val,
        const double *__restrict__ x, Epi epi, double *__restrict__ partials, CgScalars *sc,
        int what) {
    const int groups = gridDim.x * (blockDim.x / G);
    const int lane = threadIdx.x % G;
    double d = 0.0;
    const int nit = (nrows + groups - 1) / groups;
    for (int it = 0; it < nit; ++it) {
        const int row = (blockIdx.x * blockDim.x + threadIdx.x) / G + it * groups;
        const bool valid = row < nrows;
        double s0, s1, s2;
        row_sums<G, 1, VT>(row, valid, lane, ptr, col, val, x, s0, s1, s2);
        if (valid) d += epilogue<G>(epi, row, lane, s0, s1, s2);
    }
    grid_finish(d, partials, sc, what, 0);
}

// ---- TMA-fed persistent variant (variant 3) ---------------------------------
// The fine-level matrix stream is the whole cost of the SpMV.  Here it is
// moved by the copy engine instead of by per-thread loads: a persistent CTA
// (one per SM) walks chunks of RPC = 256/G consecutive block rows; one
// producer lane issues 1-D bulk copies (cp.async.bulk, completion counted on
// an mbarrier) of the chunk's contiguous val / col / ptr bytes into an
// S-stage shared-memory ring, while 8 consumer warps compute the previous
// chunks from shared memory (x is gathered from L2, as before).  Bytes in
// flight per SM are set by the ring size, not by registers.  A chunk that
// does not fit a stage, or would read past the arrays' ends, is computed
// straight from global memory.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
    unsigned done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// the same with an L2 cache policy (createpolicy): the matrix stream marked
// evict-first, so it does not push the small, re-read operands (vectors, the
// coarse inverse) out of the 126 MB L2
__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, unsigned bytes, uint64_t *bar,
                                              uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double2 ldg2_hint(const double2 *p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}

struct TmaHdr {
    int p0, direct, voff, coff;  // first block, fallback flag, block p0's offset (doubles / ints)
};

struct TmaCfg {
    int nrows, nchunks, stages;
    int pmis;     // ptr's misalignment in ints (a row view of a larger matrix: ptr + r0)
    int pdl;      // launched as a programmatic dependent (consumers wait + fence)
    int per_cta;  // > 0: CTA b owns the contiguous chunks [b*per_cta, (b+1)*per_cta)
                  // (neighbouring rows share x, so the gathers hit L1); 0: strided
    int evict_first;  // stream val / col with an L2 evict-first policy
    unsigned vcap, ccap, pcap;  // stage layout: val | col | ptr (bytes)
    long long nnzb;
};

constexpr int kTmaHdrBytes = 1024;  // barriers + headers of up to 16 stages

// the CTA's k-th chunk, or -1 past its last
__device__ __forceinline__ int chunk_of(const TmaCfg &cfg, int k) {
    if (cfg.per_cta > 0) {
        const int c = blockIdx.x * cfg.per_cta + k;
        return k < cfg.per_cta && c < cfg.nchunks ? c : -1;
    }
    const int c = blockIdx.x + k * gridDim.x;
    return c < cfg.nchunks ? c : -1;
}

template <int G, int TW, int NT, bool kReduce, class Epi, class VT = double>
__global__ void __launch_bounds__(32 * (TW * NT + 1), 1) k_bsr3_tma(TmaCfg cfg, const int *__restrict__ ptr,
        const int *__restrict__ col, const VT *__restrict__ val,
        const double *__restrict__ x, Epi epi, double *partials, CgScalars *sc, int what) {
    static_assert(G >= 1 && G <= 32, "TMA variant: at most one warp per row");
    constexpr int RPC = 32 * TW / G;  // rows per chunk: one team of TW warps per chunk
    extern __shared__ __align__(128) unsigned char sm[];
    const int S = cfg.stages;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm);
    uint64_t *empty = full + 16;
    TmaHdr *hdr = reinterpret_cast<TmaHdr *>(sm + 256);
    unsigned char *data = sm + kTmaHdrBytes;
    const unsigned stage_bytes = cfg.vcap + cfg.ccap + cfg.pcap;
    const int warp = threadIdx.x / 32, lane32 = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, TW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double d = 0.0;
    if (warp == TW * NT) {
        // producer warp: the 32 lanes fetch the row bounds of 32 upcoming
        // chunks at once, lane 0 issues the copies in order
        int st = 0;
        unsigned ph = 0;
        for (int k0 = 0; chunk_of(cfg, k0) >= 0; k0 += 32) {
            const int cl = chunk_of(cfg, k0 + lane32);
            int b0 = 0, b1 = 0;
            if (cl >= 0) {
                const int r0 = cl * RPC, r1 = min(r0 + RPC, cfg.nrows);
                b0 = __ldg(ptr + r0);
                b1 = __ldg(ptr + r1);
            }
            for (int i = 0; i < 32; ++i) {
                const int c = chunk_of(cfg, k0 + i);
                const int p0 = __shfl_sync(0xffffffffu, b0, i), p1 = __shfl_sync(0xffffffffu, b1, i);
                if (c < 0) break;
                if (lane32 == 0) {
                    mbar_wait(empty + st, ph ^ 1);
                    const int r0 = c * RPC;
                    constexpr long long BB = 9 * sizeof(VT);  // bytes per stored block
                    const long long vb = (BB * p0) & ~15LL, ve = (BB * p1 + 15) & ~15LL;
                    const long long cb = (4LL * p0) & ~15LL, ce = (4LL * p1 + 15) & ~15LL;
                    // ptr entries [r0 - pmis, r0 - pmis + RPC + 8): a 16-byte
                    // aligned window holding [r0, r0 + RPC]
                    constexpr int PW = (RPC + 8 + 3) / 4 * 4;  // whole 16-byte units
                    const long long pbytes = 4LL * PW;
                    const bool direct = ve - vb > cfg.vcap || ce - cb > cfg.ccap ||
                                        ve > BB * cfg.nnzb || ce > 4LL * cfg.nnzb ||
                                        r0 - cfg.pmis + PW > cfg.nrows + 1 || p1 == p0;
                    hdr[st] = TmaHdr{p0, direct ? 1 : 0,
                                     static_cast<int>((BB * p0 - vb) / static_cast<long long>(sizeof(VT))),
                                     static_cast<int>((4LL * p0 - cb) / 4)};
                    if (!direct) {
                        unsigned char *sv = data + static_cast<size_t>(st) * stage_bytes;
                        mbar_arrive_tx(full + st, static_cast<unsigned>((ve - vb) + (ce - cb) + pbytes));
                        if (cfg.evict_first) {
                            const uint64_t pol = policy_evict_first();
                            bulk_g2s_hint(sv, reinterpret_cast<const char *>(val) + vb,
                                          static_cast<unsigned>(ve - vb), full + st, pol);
                            bulk_g2s_hint(sv + cfg.vcap, reinterpret_cast<const char *>(col) + cb,
                                          static_cast<unsigned>(ce - cb), full + st, pol);
                        } else {
                            bulk_g2s(sv, reinterpret_cast<const char *>(val) + vb,
                                     static_cast<unsigned>(ve - vb), full + st);
                            bulk_g2s(sv + cfg.vcap, reinterpret_cast<const char *>(col) + cb,
                                     static_cast<unsigned>(ce - cb), full + st);
                        }
                        bulk_g2s(sv + cfg.vcap + cfg.ccap, ptr + r0 - cfg.pmis,
                                 static_cast<unsigned>(pbytes), full + st);
                        // the chunk's epilogue vectors towards L2 (after a
                        // PDL wait only: they may be the previous kernel's output)
                        if (!cfg.pdl) epi.prefetch(r0, min(RPC, cfg.nrows - r0));
                    } else {
                        mbar_arrive(full + st);
                    }
                }
                if (++st == S) { st = 0; ph ^= 1; }
            }
        }
    } else {
        // NT teams of TW consumer warps take the CTA's chunks in turn, so NT
        // chunks are computed concurrently while the ring fills.  The
        // producer streams the matrix (independent of the previous kernel)
        // at once; x / f / u are read only after the PDL wait.
        if (cfg.pdl) pdl_wait();
        const int team = warp / TW, tt = threadIdx.x - 32 * TW * team;
        const int lane = tt % G, grp = tt / G;
        for (int i = team, c = chunk_of(cfg, team); c >= 0; i += NT, c = chunk_of(cfg, i)) {
            const int st = i % S;
            const unsigned ph = (i / S) & 1;
            mbar_wait(full + st, ph);
            const TmaHdr h = hdr[st];
            const int row = c * RPC + grp;
            const bool valid = row < cfg.nrows;
            double s0, s1, s2;
            if (h.direct) {
                row_sums_blocks<G, VT>(row, valid, lane, ptr, col, val, x, s0, s1, s2);
            } else {
                const unsigned char *sv = data + static_cast<size_t>(st) * stage_bytes;
                const VT *svd = reinterpret_cast<const VT *>(sv);
                const int *svc = reinterpret_cast<const int *>(sv + cfg.vcap);
                const int *svp = reinterpret_cast<const int *>(sv + cfg.vcap + cfg.ccap) + cfg.pmis;
                double a0 = 0.0, a1 = 0.0, a2 = 0.0;
                constexpr int kUnr = sizeof(VT) == 4 ? 4 : 2;
                if (valid) {
                    const int beg = svp[grp] - h.p0, end = svp[grp + 1] - h.p0;
#pragma unroll kUnr
                    for (int k = beg + lane; k < end; k += G) {
                        const int c3 = svc[k + h.coff];
                        const int o = 9 * k + h.voff;
                        double bb[9];
                        blk9<false>(svd + o, o & 1, bb);
                        const double *xp = x + 3 * static_cast<size_t>(c3);
                        const int xo = c3 & 1;
                        const double2 xq = ldg2(xp + xo);
                        const double xe = __ldg(xp + (xo ? 0 : 2));
                        const double x0 = xo ? xe : xq.x, x1 = xo ? xq.x : xq.y, x2 = xo ? xq.y : xe;
                        const double b0 = bb[0], b1 = bb[1], b2 = bb[2], b3 = bb[3], b4 = bb[4],
                                     b5 = bb[5], b6 = bb[6], b7 = bb[7], b8 = bb[8];
                        a0 = fma(b0, x0, a0); a0 = fma(b1, x1, a0); a0 = fma(b2, x2, a0);
                        a1 = fma(b3, x0, a1); a1 = fma(b4, x1, a1); a1 = fma(b5, x2, a1);
                        a2 = fma(b6, x0, a2); a2 = fma(b7, x1, a2); a2 = fma(b8, x2, a2);
                    }
                }
                s0 = a0; s1 = a1; s2 = a2;
                group_reduce3<G>(s0, s1, s2);
            }
            __syncwarp();
            if (lane32 == 0) mbar_arrive(empty + st);
            if (valid) {
                const double t = epilogue<G>(epi, row, lane, s0, s1, s2);
                if constexpr (kReduce) d += t;
            }
        }
    }
    if (cfg.pdl) pdl_trigger();
    if constexpr (kReduce) grid_finish(d, partials, sc, what, 0);
}

constexpr int kReduceCtas = 148 * 8;

int spmv_variant() {
    static const int v = [] {
        const char *e = std::getenv("SAMG_SPMV_VARIANT");
        return e ? std::atoi(e) : 3;
    }();
    return v;
}

int choose_group(const Bsr3 &A) {
    static const int forced = [] {
        const char *e = std::getenv("SAMG_SPMV_GROUP");
        return e ? std::atoi(e) : 0;
    }();
    const double bpr = A.nrows ? static_cast<double>(A.nnzb) / A.nrows : 0.0;
    if (spmv_variant() == 0) {
        if (forced == 8 || forced == 16 || forced == 32) return forced;
        return 3.0 * bpr >= 45.0 ? 32 : (3.0 * bpr >= 12.0 ? 16 : 8);
    }
    if (forced >= 1 && forced <= 128 && (forced & (forced - 1)) == 0) return forced;
    // ~7 blocks per lane: enough independent loads per thread to cover HBM
    // latency, several rows per warp (measured on C1, fine rows of ~26
    // blocks: G=4 5.9 TB/s, G=8 5.2, G=16 4.8, G=32 4.2; profiles/)
    static const double per_lane = [] {
        const char *e = std::getenv("SAMG_SPMV_BLOCKS_PER_LANE");
        return e ? std::atof(e) : 7.0;
    }();
    const double want = bpr / per_lane;
    int G = 1;
    while (G < 32 && G < want) G *= 2;
    // long rows (C1's A1, ~102 blocks): a full warp per row beats two rows
    // per warp (33.8 vs 35.7 us, scripts/solve_sweep.sh)
    if (bpr >= 64.0 && G < 32 && forced == 0) G = 32;
    // small (coarse-level / restriction) matrices cannot fill 148 SMs:
    // spend more lanes per row to shorten the serial chains instead
    // (R1 of C1: 3 822 rows; 8 lanes -> 40 us, 32 lanes -> ~6 us).  Keeping
    // the grid within one wave instead (C1's level 2 at 32 lanes: 0.65
    // waves) measured slower than 64 lanes in 1.29 waves (17.3 -> 25.9 us
    // per residual): the shorter per-lane chains win
    while (G < 128 && A.nrows * G < 148LL * 1024) G *= 2;
    return G;
}

// Calls f(std::integral_constant<int, G>) for the runtime G.
template <class F>
void dispatch_group(int G, F f) {
    switch (G) {
        case 1: f(std::integral_constant<int, 1>{}); break;
        case 2: f(std::integral_constant<int, 2>{}); break;
        case 4: f(std::integral_constant<int, 4>{}); break;
        case 8: f(std::integral_constant<int, 8>{}); break;
        case 16: f(std::integral_constant<int, 16>{}); break;
        case 32: f(std::integral_constant<int, 32>{}); break;
        case 64: f(std::integral_constant<int, 64>{}); break;
        default: f(std::integral_constant<int, 128>{}); break;
    }
}

int env_int(const char *name, int dflt) {
    const char *e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

// Variant 3 launch; false if the matrix does not suit it (then the caller
// uses the register-streaming kernel).
template <int G_, int TW_ = 8, int NT_ = 2>
struct TmaShape {
    static constexpr int G = G_, TW = TW_, NT = NT_;
};

// Teams: two of 8 warps by default.  Long rows (G = 32, a warp per row) can
// run as more, smaller teams (tw = 4 or 2 warps per team, 16 / tw teams):
// a chunk is then tw rows, so more chunks fit the ring and more rows are in
// different phases of gather / reduce / epilogue at once.
template <class F>
void dispatch_tma_shape(int G, int tw, F f) {
    switch (G) {
        case 4: f(TmaShape<4>{}); break;
        case 16: f(TmaShape<16>{}); break;
        case 32:
            if (tw == 4) f(TmaShape<32, 4, 4>{});
            else if (tw == 2) f(TmaShape<32, 2, 8>{});
            else f(TmaShape<32>{});
            break;
        default: f(TmaShape<8>{}); break;
    }
}

// CTA cap for the persistent SpMV (0 = one per SM): the host-vector
// pipeline leaves HBM headroom for the concurrent PCIe copies this way
thread_local int g_tma_cta_cap = -1;
int tma_cta_cap() {
    if (g_tma_cta_cap >= 0) return g_tma_cta_cap;
    static const int env = env_int("SAMG_TMA_CTAS", 0);
    return env;
}

template <bool kReduce, class VT, class Epi>
bool launch_tma(const Bsr3 &A, const VT *val, const double *x, Epi epi, double *partials,
                CgScalars *sc, int what, cudaStream_t s) {
    static const int dbg = env_int("SAMG_TMA_DEBUG", 0);
    auto why = [&](const char *r) {
        if (dbg) std::fprintf(stderr, "launch_tma: %lld rows %lld blocks: %s\n", (long long)A.nrows,
                              (long long)A.nnzb, r);
        return false;
    };
    if (A.nrows < 8 || A.nnzb == 0) return why("small");
    // val / col: the full arrays (16-byte aligned allocations); ptr may be a
    // row view's offset pointer (the multi-GPU interior rows), handled in-kernel
    if ((reinterpret_cast<uintptr_t>(val) | reinterpret_cast<uintptr_t>(A.col.p)) & 15 ||
        reinterpret_cast<uintptr_t>(A.ptr.p) & 3)
        return why("alignment");
    static const int forced_g = env_int("SAMG_TMA_G", 0);
    static const int budget64 = env_int("SAMG_TMA_SMEM", 226000);
    static const int budget32 = env_int("SAMG_TMA_SMEM32", 226000);
    const int budget = sizeof(VT) == 4 ? budget32 : budget64;
    int TW = 8, NT = 2;  // two teams of 8 consumer warps (measured best on C1's fine level)
    const double bpr = static_cast<double>(A.nnzb) / A.nrows;
    // ~3 blocks per lane (C1 fine level, 26 blocks per row: G = 8)
    // (fp32 values: twice the blocks per lane, C1 mixed solve 0.080 -> 0.074 s)
    int G = 4;
    while (G < 32 && 3.3 * G * 1.5 * (sizeof(VT) == 4 ? 2 : 1) < bpr) G *= 2;
    if (forced_g == 4 || forced_g == 8 || forced_g == 16 || forced_g == 32) G = forced_g;
    static const int gmax = env_int("SAMG_TMA_GMAX", 32);
    G = std::min(G, std::max(4, gmax));
    static const int tw32 = env_int("SAMG_TMA_TW32", 8);
    if (G == 32 && (tw32 == 4 || tw32 == 2)) {
        TW = tw32;
        NT = 16 / tw32;
    }
    const int rpc = 32 * TW / G;
    auto up = [](long long b) { return static_cast<unsigned>((b + 127) / 128 * 128); };
    // (smaller teams: fewer rows per chunk average out less, so more slack)
    static const double slack_env = [] {
        const char *e = std::getenv("SAMG_TMA_SLACK");
        return e ? std::atof(e) : 0.0;
    }();
    const double slack = slack_env > 1.0 ? slack_env : (TW < 8 ? 1.25 : 1.1);
    long long est = static_cast<long long>(std::ceil(bpr * slack)) + 1;
    // blocks per row a stage holds: ~10 % above the mean, but shrunk (down to
    // the mean + 2 %) so that NT + 1 stages still fit -- C4's fine level (26.7
    // blocks per row) missed the third stage by 1 % and ran without TMA;
    // a rarer chunk above the capacity is computed from global memory
    {
        const long long per_block = 9 * static_cast<long long>(sizeof(VT)) + 4;
        const long long room = (budget - kTmaHdrBytes) / (NT + 1) - 4LL * (rpc + 8) - 3 * 128 - 32;
        const long long fit = room / (rpc * per_block);
        if (fit < est && fit >= static_cast<long long>(std::ceil(bpr * 1.02))) est = fit;
    }
    TmaCfg cfg{};
    cfg.nrows = static_cast<int>(A.nrows);
    cfg.nchunks = static_cast<int>((A.nrows + rpc - 1) / rpc);
    cfg.nnzb = A.nnzb;
    cfg.vcap = up(rpc * est * 9 * static_cast<long long>(sizeof(VT)) + 16);
    cfg.ccap = up(rpc * est * 4 + 16);
    cfg.pcap = up(4LL * (rpc + 8));
    cfg.pmis = static_cast<int>((reinterpret_cast<uintptr_t>(A.ptr.p) & 15) / 4);
    cfg.pdl = g_spmv_pdl && pdl_enabled() ? 1 : 0;
    cfg.evict_first = l2_hints() ? 1 : 0;
    const long long stage = cfg.vcap + cfg.ccap + cfg.pcap;
    cfg.stages = static_cast<int>(std::min<long long>(16, (budget - kTmaHdrBytes) / stage));
    if (cfg.stages < NT + 1) return why("stages");
    const int smem = kTmaHdrBytes + static_cast<int>(cfg.stages * stage);
    const int sms = sm_count();
    // one persistent CTA per SM only pays off when every CTA streams many
    // chunks (C1: fine level 8 064 chunks, P0 4 032 -> TMA; A1 2 580 -> variant 1)
    static const int min_chunks_per_sm = env_int("SAMG_TMA_MIN_CHUNKS", 24);
    if (cfg.nchunks < min_chunks_per_sm * sms) return why("chunks");
    bool ok = false;
    dispatch_tma_shape(G, TW, [&](auto sh) {
        using Sh = decltype(sh);
        auto kern = k_bsr3_tma<Sh::G, Sh::TW, Sh::NT, kReduce, Epi, VT>;
        const int threads = 32 * (Sh::TW * Sh::NT + 1);
        // opt in to the largest dynamic size next to the static shared
        // memory of the reduction helpers
        static DeviceCache max_dyn_cache;
        const int max_dyn = max_dyn_cache.get([&] {
            int dev = 0, optin = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, kern);
            const int m = optin - static_cast<int>(fa.sharedSizeBytes);
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, m) !=
                cudaSuccess) {
                cudaGetLastError();
                return 0;
            }
            return m;
        });
        if (smem > max_dyn) { why("smem"); return; }
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        int grid = std::max(1, std::min(cfg.nchunks, std::max(1, occ) * sms));
        if (tma_cta_cap() > 0) grid = std::min(grid, tma_cta_cap());
        static const int blocked = env_int("SAMG_TMA_BLOCKED", 0);
        cfg.per_cta = blocked ? (cfg.nchunks + grid - 1) / grid : 0;
        launch_k(cfg.pdl != 0, kern, grid, threads, smem, s, cfg, A.ptr.p, A.col.p, val, x, epi, partials, sc, what);
        ok = true;
    });
    if (ok) CK_LAUNCH();
    return ok;
}

bool node6_enabled() { return true; }  // a matrix carries val6 only if setup built it

template <class Epi>
void launch_node6(const Bsr3 &A, const double *x, Epi epi, cudaStream_t s) {
    const double bpr = static_cast<double>(A.nnzb6) / static_cast<double>(A.nrows6);
    int G = 2;  // a lane pair per block, ~2 blocks per pair
    while (G < 32 && G < bpr) G *= 2;
    while (G < 32 && A.nrows6 * G < 148LL * 1024) G *= 2;
    const int grid = ceil_div(A.nrows6 * static_cast<int64_t>(G), 256);
    const int n = static_cast<int>(A.nrows6);
    switch (G) {
        case 2: k_bsr6<2, Epi><<<grid, 256, 0, s>>>(n, A.ptr6.p, A.col6.p, A.val6.p, x, epi); break;
        case 4: k_bsr6<4, Epi><<<grid, 256, 0, s>>>(n, A.ptr6.p, A.col6.p, A.val6.p, x, epi); break;
        case 8: k_bsr6<8, Epi><<<grid, 256, 0, s>>>(n, A.ptr6.p, A.col6.p, A.val6.p, x, epi); break;
        case 16: k_bsr6<16, Epi><<<grid, 256, 0, s>>>(n, A.ptr6.p, A.col6.p, A.val6.p, x, epi); break;
        default: k_bsr6<32, Epi><<<grid, 256, 0, s>>>(n, A.ptr6.p, A.col6.p, A.val6.p, x, epi); break;
    }
    CK_LAUNCH();
}

template <class VT, class Epi>
void launch_rows_t(const Bsr3 &A, const VT *val, const double *x, Epi epi, cudaStream_t s) {
    if (std::is_same_v<VT, double> && A.val6.p && node6_enabled() &&
        reinterpret_cast<const void *>(val) == reinterpret_cast<const void *>(A.val.p)) {
        launch_node6(A, x, epi, s);
        return;
    }
    if (spmv_variant() == 3 && launch_tma<false>(A, val, x, epi, nullptr, nullptr, 0, s)) return;
    const int G = choose_group(A);
    const int grid = ceil_div(A.nrows * static_cast<int64_t>(G), 256);
    const int n = static_cast<int>(A.nrows);
    if (std::is_same_v<VT, double> && spmv_variant() == 0) {
        const double *vd = reinterpret_cast<const double *>(val);
        if (G == 32) launch_k(false, k_bsr3<32, 0, Epi, double>, grid, 256, 0, s, n, A.ptr.p, A.col.p, vd, x, epi);
        else if (G == 16) launch_k(false, k_bsr3<16, 0, Epi, double>, grid, 256, 0, s, n, A.ptr.p, A.col.p, vd, x, epi);
        else launch_k(false, k_bsr3<8, 0, Epi, double>, grid, 256, 0, s, n, A.ptr.p, A.col.p, vd, x, epi);
    } else {
        static const int pipe = env_int("SAMG_LONG_PIPE", 2);  // 0: variant 1; 1: G = 32 only; 2: also G = 64
        if (G == 32 && pipe) {
            launch_k(false, k_bsr3<32, 2, Epi, VT>, grid, 256, 0, s, n, A.ptr.p, A.col.p, val, x, epi);
        } else if (G == 64 && pipe >= 2) {
            launch_k(false, k_bsr3<64, 2, Epi, VT>, grid, 256, 0, s, n, A.ptr.p, A.col.p, val, x, epi);
        } else {
            dispatch_group(G, [&](auto g) {
                constexpr int GG = decltype(g)::value;
                launch_k(false, k_bsr3<GG, 1, Epi, VT>, grid, 256, 0, s, n, A.ptr.p, A.col.p, val, x, epi);
            });
        }
    }
    CK_LAUNCH();
}

// lowp: use the matrix's fp32 value copy (mixed-precision V-cycle) if it has one
template <class Epi>
void launch_rows(const Bsr3 &A, const double *x, Epi epi, cudaStream_t s, bool lowp = false) {
    if (A.nrows == 0) return;
    if (lowp && A.val32.p) launch_rows_t(A, static_cast<const float *>(A.val32.p), x, epi, s);
    else launch_rows_t(A, static_cast<const double *>(A.val.p), x, epi, s);
}

template <class VT, class Epi>
void launch_reduce_t(const Bsr3 &A, const VT *val, const double *x, Epi epi, double *partials,
                     CgScalars *sc, int what, cudaStream_t s) {
    if (spmv_variant() == 3 && launch_tma<true>(A, val, x, epi, partials, sc, what, s)) return;
    const int G = choose_group(A);
    const int n = static_cast<int>(A.nrows);
    dispatch_group(G, [&](auto g) {
        constexpr int GG = decltype(g)::value;
        // persistent grid = exactly one wave of resident CTAs (a second,
        // partial wave cost ~15% on C1's fine level)
        static const int resident = [] {
            int occ = 0, dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bsr3_reduce<GG, Epi, VT>, 256, 0);
            return std::max(1, occ) * sms;
        }();
        const int grid = std::max(1, std::min({kReduceCtas, resident,
                                               ceil_div(A.nrows * static_cast<int64_t>(GG), 256)}));
        launch_k(false, k_bsr3_reduce<GG, Epi, VT>, grid, 256, 0, s, n, A.ptr.p, A.col.p, val, x, epi, partials,
                 sc, what);
    });
    CK_LAUNCH();
}

template <class Epi>
void launch_reduce(const Bsr3 &A, const double *x, Epi epi, double *partials, CgScalars *sc,
                   int what, cudaStream_t s, bool lowp = false) {
    if (lowp && A.val32.p) launch_reduce_t(A, static_cast<const float *>(A.val32.p), x, epi, partials, sc, what, s);
    else launch_reduce_t(A, static_cast<const double *>(A.val.p), x, epi, partials, sc, what, s);
}

// node row i of a pairable matrix: rows 2i, 2i+1 with equal column lists of
// consecutive pairs (2j, 2j+1)
__global__ void k_node6_check(int64_t nr6, const int *ptr, const int *col, int *bad, int *cnt) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= nr6) return;
    const int a0 = ptr[2 * i], a1 = ptr[2 * i + 1], a2 = ptr[2 * i + 2];
    const int n = a1 - a0;
    bool ok = (n == a2 - a1) && !(n & 1);
    for (int k = 0; ok && k < n; k += 2)
        ok = col[a0 + k] == col[a1 + k] && col[a0 + k + 1] == col[a1 + k + 1] &&
             !(col[a0 + k] & 1) && col[a0 + k + 1] == col[a0 + k] + 1;
    if (!ok) atomicExch(bad, 1);
    cnt[i] = n / 2;
}

__global__ void k_node6_fill(int64_t nr6, const int *ptr, const int *col, const double *val,
                             int *ptr6, int *col6, double *val6) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i > nr6) return;
    // block rows 0..2i-1 hold ptr[2i] 3x3 blocks = ptr[2i]/4 6x6 blocks
    ptr6[i] = ptr[2 * i] / 4;
    if (i == nr6) return;
    const int a0 = ptr[2 * i], a1 = ptr[2 * i + 1];
    const int n = a1 - a0;
    const int o6 = ptr[2 * i] / 4;
    for (int k = 0; k < n / 2; ++k) {
        col6[o6 + k] = col[a0 + 2 * k] / 2;
        double *d = val6 + 36 * static_cast<int64_t>(o6 + k);
        for (int hr = 0; hr < 2; ++hr)
            for (int hc = 0; hc < 2; ++hc) {
                const double *b = val + 9 * static_cast<int64_t>((hr ? a1 : a0) + 2 * k + hc);
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c) d[(3 * hr + r) * 6 + 3 * hc + c] = b[3 * r + c];
            }
    }
}

__global__ void k_to_f32(int64_t n, const double *__restrict__ a, float *__restrict__ b) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        b[i] = __double2float_rn(a[i]);
}

__global__ void k_smooth_zero_point(int64_t n, const double *__restrict__ m,
        const double *__restrict__ f, double *__restrict__ u) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        u[i] = m[i] * f[i];
}

// u = M f for 3x3 M: one thread per block row (72 B of M, 24 B of f, 24 B of u)
__global__ void k_smooth_zero_block(int64_t nrows, const double *__restrict__ m,
        const double *__restrict__ f, double *__restrict__ u) {
    for (int64_t row = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; row < nrows;
         row += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double *M = m + 9 * row;
        const double f0 = f[3 * row], f1 = f[3 * row + 1], f2 = f[3 * row + 2];
        double Mv[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) Mv[e] = __ldcs(M + e);
        u[3 * row] = Mv[0] * f0 + Mv[1] * f1 + Mv[2] * f2;
        u[3 * row + 1] = Mv[3] * f0 + Mv[4] * f1 + Mv[5] * f2;
        u[3 * row + 2] = Mv[6] * f0 + Mv[7] * f1 + Mv[8] * f2;
    }
}

// u = Ainv f, Ainv row-major with an even leading dimension (zero padded):
// one 64-thread CTA per row: 2 922 rows at C1 fit in one wave (32 resident
// CTAs per SM; 128-thread CTAs needed 1.23 waves, 20.4 us -> see profiles/),
// eight 16-byte loads in flight per thread.
constexpr int kGemvThreads = 64;
__global__ void __launch_bounds__(kGemvThreads) k_dense_gemv(int n, int64_t ld, const double *__restrict__ A,
        const double *__restrict__ f, double *__restrict__ u, int keep) {
    constexpr int T = kGemvThreads;
    __shared__ double red[T / 32];
    const int row = blockIdx.x;
    const double2 *a = reinterpret_cast<const double2 *>(A + static_cast<size_t>(row) * ld);
    const int n2 = static_cast<int>(ld / 2);
    const uint64_t pol = policy_evict_last();
    double s = 0.0, t = 0.0;
    // f as 16-byte pairs (f is 16-byte aligned; a last odd element alone)
    auto fpair = [&](int j2) {
        const int j = 2 * j2;
        return j + 1 < n ? __ldg(reinterpret_cast<const double2 *>(f) + j2) : make_double2(__ldg(f + j), 0.0);
    };
    // batches of 8 16-byte loads per thread, all issued before the FMAs (32
    // registers: the 2 922 rows of C1 in 0.62 waves; 24 per batch needed 129
    // registers and 2.8 waves)
    constexpr int B = 8;
    for (int j0 = threadIdx.x; j0 < n2; j0 += B * T) {
        double2 av[B];
#pragma unroll
        for (int k = 0; k < B; ++k) {
            const int j2 = j0 + k * T;
            av[k] = j2 < n2 ? (keep ? ldg2_hint(a + j2, pol) : __ldg(a + j2)) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int k = 0; k < B; ++k) {
            const int j2 = j0 + k * T;
            if (j2 < n2) {
                const double2 fk = fpair(j2);
                s = fma(av[k].x, fk.x, s);
                t = fma(av[k].y, fk.y, t);
            }
        }
    }
    s += t;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = s;
    __syncthreads();
    if (threadIdx.x == 0) u[row] = red[0] + red[1];
}

// TMA-fed dense GEMV (the coarse solve u = Ainv f, a 68 MB stream at C1):
// one persistent CTA per SM owns a contiguous range of rows; a producer lane
// streams whole rows (8*ld bytes, contiguous) into an S-stage shared-memory
// ring with cp.async.bulk + mbarriers, after f itself; 8 consumer warps take
// the CTA's rows in turn (warp w: rows w, w+8, ...) and form each dot
// product from shared memory.  The per-thread-load variant (k_dense_gemv)
// keeps one DRAM round trip per batch of 8 loads on every thread's chain
// (3.3 TB/s at C1); here the bytes in flight per SM are set by the ring.
constexpr int kGemvWarps = 8;
__global__ void __launch_bounds__(32 * (kGemvWarps + 1), 1) k_dense_gemv_tma(int n, int64_t ld,
        const double *__restrict__ A, const double *__restrict__ f, double *__restrict__ u, int stages,
        int evict_first) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm);  // [16]
    uint64_t *empty = full + 16;                          // [16]
    uint64_t *fbar = empty + 16;
    double *fs = reinterpret_cast<double *>(sm + 384);
    const unsigned rowb = static_cast<unsigned>(8 * ld);
    double *ring = fs + ld;
    const int r0 = static_cast<int>((static_cast<long long>(n) * blockIdx.x) / gridDim.x);
    const int r1 = static_cast<int>((static_cast<long long>(n) * (blockIdx.x + 1)) / gridDim.x);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int st = 0; st < stages; ++st) {
            mbar_init(full + st, 1);
            mbar_init(empty + st, 1);
        }
        mbar_init(fbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kGemvWarps) {
        if (lane == 0) {
            const uint64_t pol = evict_first ? policy_evict_first() : 0;
            // f's first n & ~1 entries (an odd n's last entry is read from global)
            const unsigned fb = static_cast<unsigned>(8 * (n & ~1));
            mbar_arrive_tx(fbar, fb);
            if (fb) bulk_g2s(fs, f, fb, fbar);
            int st = 0;
            unsigned ph = 0;
            for (int r = r0; r < r1; ++r) {
                mbar_wait(empty + st, ph ^ 1);
                mbar_arrive_tx(full + st, rowb);
                if (evict_first)
                    bulk_g2s_hint(ring + static_cast<size_t>(st) * ld, A + static_cast<size_t>(r) * ld, rowb,
                                  full + st, pol);
                else
                    bulk_g2s(ring + static_cast<size_t>(st) * ld, A + static_cast<size_t>(r) * ld, rowb, full + st);
                if (++st == stages) { st = 0; ph ^= 1; }
            }
        }
        return;
    }
    mbar_wait(fbar, 0);
    const int n2 = static_cast<int>(ld / 2);
    const double2 *f2 = reinterpret_cast<const double2 *>(fs);
    for (int i = warp; r0 + i < r1; i += kGemvWarps) {
        const int st = i % stages;
        mbar_wait(full + st, (i / stages) & 1);
        const double2 *a2 = reinterpret_cast<const double2 *>(ring + static_cast<size_t>(st) * ld);
        double s = 0.0, t = 0.0;
        for (int j = lane; j < n2; j += 32) {
            const double2 av = a2[j];
            const double2 fv = 2 * j + 1 < n ? f2[j] : make_double2(__ldg(f + 2 * j), 0.0);
            s = fma(av.x, fv.x, s);
            t = fma(av.y, fv.y, t);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);
        s += t;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) u[r0 + i] = s;
    }
}

// Vector kernels: 2 elements per thread per step (16-byte loads; the
// vectors are cudaMalloc'd, so 16-byte aligned), grid-stride, tail handled
// by thread 0.
__global__ void __launch_bounds__(256) k_dot(int64_t n, const double *__restrict__ x,
        const double *__restrict__ y, double *__restrict__ partials, CgScalars *sc, int what) {
    const int64_t n2 = n / 2;
    const double2 *x2 = reinterpret_cast<const double2 *>(x), *y2 = reinterpret_cast<const double2 *>(y);
    double s = 0.0, t = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n2;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double2 a = x2[i], b = y2[i];
        s = fma(a.x, b.x, s);
        t = fma(a.y, b.y, t);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) s = fma(x[n - 1], y[n - 1], s);
    grid_finish(s + t, partials, sc, what, 0);
}

// u += alpha p; r -= alpha q; r.r (cg.hpp:68-71), finished in place
__global__ void __launch_bounds__(256) k_cg_update(int64_t n, CgScalars *sc,
        const double *__restrict__ p, const double *__restrict__ q, double *__restrict__ u,
        double *__restrict__ r, double *__restrict__ partials, int what,
        cudaGraphConditionalHandle h) {
    const double a = sc->alpha;
    const int64_t n2 = n / 2;
    const double2 *p2 = reinterpret_cast<const double2 *>(p), *q2 = reinterpret_cast<const double2 *>(q);
    double2 *u2 = reinterpret_cast<double2 *>(u), *r2 = reinterpret_cast<double2 *>(r);
    double s = 0.0, t = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n2;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double2 pp = p2[i], qq = q2[i], uu = u2[i], rr = r2[i];
        u2[i] = make_double2(fma(a, pp.x, uu.x), fma(a, pp.y, uu.y));
        const double ra = fma(-a, qq.x, rr.x), rb = fma(-a, qq.y, rr.y);
        r2[i] = make_double2(ra, rb);
        s = fma(ra, ra, s);
        t = fma(rb, rb, t);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        u[n - 1] = fma(a, p[n - 1], u[n - 1]);
        const double ri = fma(-a, q[n - 1], r[n - 1]);
        r[n - 1] = ri;
        s = fma(ri, ri, s);
    }
    grid_finish(s + t, partials, sc, what, h);
}

__global__ void k_p_update(int64_t n, const CgScalars *__restrict__ sc,
        const double *__restrict__ z, double *__restrict__ p) {
    const double b = sc->beta;
    const int64_t n2 = n / 2;
    const double2 *z2 = reinterpret_cast<const double2 *>(z);
    double2 *p2 = reinterpret_cast<double2 *>(p);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n2;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double2 zz = z2[i], pp = p2[i];
        p2[i] = make_double2(fma(b, pp.x, zz.x), fma(b, pp.y, zz.y));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) p[n - 1] = fma(b, p[n - 1], z[n - 1]);
}

// CG step with the u update deferred (to k_p_update_u) and the V-cycle's
// first level-0 sweep fused (cg.hpp:68-71, then relaxation.hpp:165-173 from
// u = 0): r -= alpha q; r.r; z0 = M r.  Tiles of 256 block rows: q, r and
// the rows' M are staged in shared memory with coalesced 16-byte loads (a
// thread per row reading its own 24 / 72-byte records touched 3x the
// sectors per instruction: C4 1.34 GB at 3.2 TB/s), one thread per row
// computes, and r, z0 leave with coalesced stores.
template <bool kBlock>
__global__ void __launch_bounds__(256) k_cg_update_smooth(int64_t nrows, CgScalars *sc,
        const double *__restrict__ q, double *__restrict__ r, const double *__restrict__ m,
        double *__restrict__ z0, double *__restrict__ partials, int what,
        cudaGraphConditionalHandle h) {
    constexpr int TR = 256, MW = kBlock ? 9 : 3;
    __shared__ __align__(16) double sq[3 * TR], sr[3 * TR], sm[MW * TR];
    const double a = sc->alpha;
    double s = 0.0;
    const int64_t ntiles = (nrows + TR - 1) / TR;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t row0 = t * TR;
        const int nr = nrows - row0 < TR ? static_cast<int>(nrows - row0) : TR;
        const int nv = 3 * nr, nm = MW * nr;
        const double2 *q2 = reinterpret_cast<const double2 *>(q + 3 * row0);
        const double2 *r2 = reinterpret_cast<const double2 *>(r + 3 * row0);
        const double2 *m2 = reinterpret_cast<const double2 *>(m + MW * row0);
        double2 *sq2 = reinterpret_cast<double2 *>(sq), *sr2 = reinterpret_cast<double2 *>(sr);
        double2 *sm2 = reinterpret_cast<double2 *>(sm);
        for (int i = threadIdx.x; i < nv / 2; i += TR) { sq2[i] = q2[i]; sr2[i] = r2[i]; }
        for (int i = threadIdx.x; i < nm / 2; i += TR) sm2[i] = __ldcs(m2 + i);
        if (threadIdx.x == 0) {
            if (nv & 1) { sq[nv - 1] = q[3 * row0 + nv - 1]; sr[nv - 1] = r[3 * row0 + nv - 1]; }
            if (nm & 1) sm[nm - 1] = m[MW * row0 + nm - 1];
        }
        __syncthreads();
        if (threadIdx.x < nr) {
            const int b = 3 * threadIdx.x;
            const double r0 = fma(-a, sq[b], sr[b]), r1 = fma(-a, sq[b + 1], sr[b + 1]),
                         r2v = fma(-a, sq[b + 2], sr[b + 2]);
            s = fma(r0, r0, s); s = fma(r1, r1, s); s = fma(r2v, r2v, s);
            sr[b] = r0; sr[b + 1] = r1; sr[b + 2] = r2v;
            if constexpr (kBlock) {
                const double *M = sm + 9 * threadIdx.x;
                sq[b] = M[0] * r0 + M[1] * r1 + M[2] * r2v;
                sq[b + 1] = M[3] * r0 + M[4] * r1 + M[5] * r2v;
                sq[b + 2] = M[6] * r0 + M[7] * r1 + M[8] * r2v;
            } else {
                sq[b] = sm[b] * r0; sq[b + 1] = sm[b + 1] * r1; sq[b + 2] = sm[b + 2] * r2v;
            }
        }
        __syncthreads();
        double2 *ro2 = reinterpret_cast<double2 *>(r + 3 * row0);
        double2 *zo2 = reinterpret_cast<double2 *>(z0 + 3 * row0);
        for (int i = threadIdx.x; i < nv / 2; i += TR) { ro2[i] = sr2[i]; zo2[i] = sq2[i]; }
        if (threadIdx.x == 0 && (nv & 1)) { r[3 * row0 + nv - 1] = sr[nv - 1]; z0[3 * row0 + nv - 1] = sq[nv - 1]; }
        __syncthreads();
    }
    grid_finish(s, partials, sc, what, h);
}

// p_old -> u += alpha p_old (the deferred update), p = z + beta p_old
__global__ void k_p_update_u(int64_t n, const CgScalars *__restrict__ sc,
        const double *__restrict__ z, double *__restrict__ p, double *__restrict__ u) {
    const double a = sc->alpha, b = sc->beta;
    const int64_t n2 = n / 2;
    const double2 *z2 = reinterpret_cast<const double2 *>(z);
    double2 *p2 = reinterpret_cast<double2 *>(p), *u2 = reinterpret_cast<double2 *>(u);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n2;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double2 zz = z2[i], pp = p2[i], uu = u2[i];
        u2[i] = make_double2(fma(a, pp.x, uu.x), fma(a, pp.y, uu.y));
        p2[i] = make_double2(fma(b, pp.x, zz.x), fma(b, pp.y, zz.y));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        u[n - 1] = fma(a, p[n - 1], u[n - 1]);
        p[n - 1] = fma(b, p[n - 1], z[n - 1]);
    }
}

// u += alpha p (the deferred update of the last iteration, host loop)
__global__ void k_u_update(int64_t n, const CgScalars *__restrict__ sc, const double *__restrict__ p,
                           double *__restrict__ u) {
    const double a = sc->alpha;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        u[i] = fma(a, p[i], u[i]);
}

__global__ void k_fill(int64_t n, double v, double *x) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = v;
}

__global__ void k_cg_finish(CgScalars *sc, int what) {
    cg_apply(what, sc->tmp, sc, 0);
}

__global__ void k_cg_finish2(CgScalars *sc, int rr_what, cudaGraphConditionalHandle h) {
    cg_apply(CG_RZ, sc->tmp2, sc, 0);
    cg_apply(rr_what, sc->tmp, sc, h);
}

// ---- V-cycle tail: the small levels in one persistent launch ----------------
// Below a size threshold a level's operators are a few MB: as separate
// launches each is latency-bound (C1 level 2 and the coarse GEMV: seven
// kernels at 0.2-2.6 TB/s, ~99 us of the 540 us iteration; profiles/
// r02_ncu_cg_iteration.txt).  Here one cooperative grid (every CTA resident)
// runs the whole list of phases -- restriction into the first small level,
// its sweeps and residuals, the coarser levels, the dense coarse solve and
// the prolongations back up -- with a grid barrier between phases, so the
// launch gaps and ramp-downs are paid once.  Vectors written by an earlier
// phase are read through L2 (ld.global.cg gathers) or after the barrier's
// acquire fence (epilogue loads); the matrices stay on the read-only path.

// Generation barrier over the whole grid (bar[0] = arrivals, bar[1] =
// generation; both start at 0 and are left consistent for the next launch).
__device__ __forceinline__ void vt_grid_sync(unsigned *bar, int sleep_ns) {
    __syncthreads();
    if (threadIdx.x == 0) {
        // (relaxed loads for the generation: an acquire load would invalidate
        // this SM's L1 on every poll)
        unsigned gen;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
        asm volatile("fence.acq_rel.gpu;" ::: "memory");  // release this CTA's phase output
        unsigned prev;
        asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(bar) : "memory");
        if (prev == gridDim.x - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(gen + 1) : "memory");
        } else {
            unsigned g2;
            do {
                if (sleep_ns) __nanosleep(sleep_ns);
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g2) : "l"(bar + 1) : "memory");
            } while (g2 == gen);
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire the other CTAs' outputs
    }
    __syncthreads();
}

// One SpMV-family phase: groups of G lanes per block row, consecutive rows
// on consecutive groups of a CTA; uniform trip count (G > 32 reduces with
// CTA barriers).
constexpr int kVtThreads = 1024;  // one CTA per SM: 148 arrivals per grid barrier

template <int G, class Epi>
__device__ __forceinline__ void vt_rows(const VPhase &P, const Epi &epi) {
    constexpr int GPC = kVtThreads / G;
    const int total = gridDim.x * GPC;
    const int nit = (P.nrows + total - 1) / total;
    const int lane = threadIdx.x % G;
    const int g0 = blockIdx.x * GPC + threadIdx.x / G;
    for (int it = 0; it < nit; ++it) {
        const int row = g0 + it * total;
        const bool valid = row < P.nrows;
        double s0, s1, s2;
        row_sums_blocks<G, double, false, kVtThreads>(row, valid, lane, P.ptr, P.col, P.val, P.x, s0, s1, s2);
        if (valid) epilogue<G>(epi, row, lane, s0, s1, s2);
    }
}

template <class Epi>
__device__ __forceinline__ void vt_spmv(const VPhase &P, const Epi &epi) {
    switch (P.G) {
        case 4: vt_rows<4>(P, epi); break;
        case 8: vt_rows<8>(P, epi); break;
        case 16: vt_rows<16>(P, epi); break;
        case 32: vt_rows<32>(P, epi); break;
        case 64: vt_rows<64>(P, epi); break;
        default: vt_rows<128>(P, epi); break;
    }
}

// u = Ainv f: one warp per row, f staged once per CTA in shared memory
// (when it fits: fs != nullptr), eight 16-byte loads in flight per lane.
__device__ __forceinline__ void vt_gemv(const VPhase &P, double *fs, bool keep) {
    const uint64_t pol = policy_evict_last();
    const int n = P.nrows;
    const int n2 = static_cast<int>(P.ld / 2);
    const double *f = P.x;
    if (fs) {
        for (int j = threadIdx.x; j < n; j += blockDim.x) fs[j] = __ldcg(f + j);
        if (threadIdx.x == 0 && (n & 1)) fs[n] = 0.0;
        __syncthreads();
    }
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nw = gridDim.x * (blockDim.x / 32);
    for (int row = blockIdx.x * (blockDim.x / 32) + warp; row < n; row += nw) {
        const double2 *a = reinterpret_cast<const double2 *>(P.val + static_cast<size_t>(row) * P.ld);
        double s = 0.0, t = 0.0;
        constexpr int B = 8;
        for (int j0 = lane; j0 < n2; j0 += B * 32) {
            double2 av[B];
#pragma unroll
            for (int k = 0; k < B; ++k) {
                const int j2 = j0 + k * 32;
                av[k] = j2 < n2 ? (keep ? ldg2_hint(a + j2, pol) : __ldg(a + j2)) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int k = 0; k < B; ++k) {
                const int j2 = j0 + k * 32;
                if (j2 < n2) {
                    const int j = 2 * j2;
                    double2 fk;
                    if (fs) fk = make_double2(fs[j], fs[j + 1]);
                    else fk = make_double2(__ldcg(f + j), j + 1 < n ? __ldcg(f + j + 1) : 0.0);
                    s = fma(av[k].x, fk.x, s);
                    t = fma(av[k].y, fk.y, t);
                }
            }
        }
        s += t;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) P.out[row] = s;
    }
}

__global__ void __launch_bounds__(kVtThreads, 1) k_vtail(const VPhase *__restrict__ phases, int nph,
                                                   unsigned *bar, double *final_out, int flags,
                                                   unsigned long long *trace) {
    extern __shared__ double vt_fs[];
    auto stamp = [&](int slot) {
        if (trace && blockIdx.x == 0 && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace[slot] = t;
        }
    };
    stamp(2 * nph);
    auto stamp_cta = [&](int k) {  // every CTA's end of phase k (k == nph: its start)
        if (trace && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace[2 * nph + 1 + static_cast<size_t>(k) * gridDim.x + blockIdx.x] = t;
        }
    };
    stamp_cta(nph);
    for (int k = 0; k < nph; ++k) {
        VPhase P = phases[k];
        if (P.last_out) P.out = final_out;
        switch (P.kind) {
            case VP_SPMV: vt_spmv(P, EpiSpmv{P.alpha, P.beta, P.out}); break;
            case VP_RESIDUAL: vt_spmv(P, EpiResidual{P.f, P.out}); break;
            case VP_SMOOTH_B: vt_spmv(P, EpiSmoothBlock{P.f, P.x, P.m, P.out}); break;
            case VP_SMOOTH_P: vt_spmv(P, EpiSmoothPoint{P.f, P.x, P.m, P.out}); break;
            case VP_RSMOOTH_B: vt_spmv(P, EpiRestrictSmooth<true>{P.out, P.out2, P.m}); break;
            case VP_RSMOOTH_P: vt_spmv(P, EpiRestrictSmooth<false>{P.out, P.out2, P.m}); break;
            case VP_GEMV: vt_gemv(P, (flags & 1) ? vt_fs : nullptr, (flags & 2) != 0); break;
            case VP_FILL:
                for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
                     i < 3LL * P.nrows; i += static_cast<int64_t>(gridDim.x) * blockDim.x)
                    P.out[i] = P.alpha;
                break;
            default: break;
        }
        stamp(2 * k);
        __syncthreads();
        stamp_cta(k);
        if (k + 1 < nph) vt_grid_sync(bar, flags >> 8);
        stamp(2 * k + 1);
    }
}

int vec_grid(int64_t n) {
    const int64_t g = (n + 255) / 256;
    return static_cast<int>(g < kRedBlocks ? (g > 0 ? g : 1) : kRedBlocks);
}

} // namespace

void set_spmv_cta_cap(int ctas) { g_tma_cta_cap = ctas; }
void set_spmv_pdl(bool on) { g_spmv_pdl = on; }

void launch_spmv(const Bsr3 &A, double alpha, const double *x, double beta, double *y,
                 cudaStream_t s, bool lowp) {
    launch_rows(A, x, EpiSpmv{alpha, beta, y}, s, lowp);
}

// y[rows] = alpha*A[rows,:]*x + beta*y[rows]; group 0 = choose from A
void launch_spmv_rows(const Bsr3 &A, const int *rows, int64_t nlist, int group, double alpha,
                      const double *x, double beta, double *y, cudaStream_t s) {
    if (nlist == 0) return;
    const int G = (group >= 1 && group <= 128 && (group & (group - 1)) == 0) ? group : choose_group(A);
    const int grid = ceil_div(nlist * static_cast<int64_t>(G), 256);
    const int n = static_cast<int>(nlist);
    const EpiSpmv epi{alpha, beta, y};
    dispatch_group(G, [&](auto g) {
        constexpr int GG = decltype(g)::value;
        launch_k(false, k_bsr3_rows<GG, EpiSpmv>, grid, 256, 0, s, n, rows, A.ptr.p, A.col.p, A.val.p, x, epi);
    });
    CK_LAUNCH();
}

void launch_residual(const Bsr3 &A, const double *f, const double *u, double *r,
                     cudaStream_t s, bool lowp) {
    launch_rows(A, u, EpiResidual{f, r}, s, lowp);
}

void launch_smooth(const Bsr3 &A, const Smoother &M, const double *f, const double *u,
                   double *u_out, cudaStream_t s, bool lowp) {
    if (M.kind == SM_ILU) return launch_ilu_smooth(&A, M, f, u, u_out, s, lowp);
    if (M.kind == SM_POINT) launch_rows(A, u, EpiSmoothPoint{f, u, M.data.p, u_out}, s, lowp);
    else launch_rows(A, u, EpiSmoothBlock{f, u, M.data.p, u_out}, s, lowp);
}

// As launch_smooth with the gathered vector x apart from the row-indexed u
// (a row range of a partitioned level: x is the whole halo-extended vector)
void launch_smooth_split(const Bsr3 &A, const Smoother &M, const double *f, const double *x,
                         const double *u, double *u_out, cudaStream_t s) {
    if (M.kind == SM_ILU) fail(SAMG_UNSUPPORTED, "launch_smooth_split: ILU(0) sweeps are not row-separable");
    if (A.nrows == 0) return;
    if (M.kind == SM_POINT) launch_rows(A, x, EpiSmoothPoint{f, u, M.data.p, u_out}, s, false);
    else launch_rows(A, x, EpiSmoothBlock{f, u, M.data.p, u_out}, s, false);
}

void launch_smooth_zero(int64_t nrows, const Smoother &M, const double *f, double *u,
                        cudaStream_t s) {
    if (nrows == 0) return;
    if (M.kind == SM_ILU) return launch_ilu_smooth(nullptr, M, f, nullptr, u, s);
    if (M.kind == SM_POINT) launch_k(false, k_smooth_zero_point, vec_grid(3 * nrows), 256, 0, s, 3 * nrows, M.data.p, f, u);
    else launch_k(false, k_smooth_zero_block, vec_grid(nrows), 256, 0, s, nrows, M.data.p, f, u);
    CK_LAUNCH();
}

void launch_spmv_dot(const Bsr3 &A, const double *p, double *q, double *partials,
                     CgScalars *sc, cudaStream_t s, int what) {
    launch_reduce(A, p, EpiDot{p, q}, partials, sc, what, s);
}

// q = A x and p.q on a row range: x the whole halo-extended vector, p / q
// row-indexed
void launch_spmv_dot_split(const Bsr3 &A, const double *x, const double *p, double *q,
                           double *partials, CgScalars *sc, cudaStream_t s, int what) {
    if (A.nrows == 0) return;
    launch_reduce(A, x, EpiDot{p, q}, partials, sc, what, s);
}

void launch_smooth_dot(const Bsr3 &A, const Smoother &M, const double *f, const double *u,
                       double *u_out, double *partials, CgScalars *sc, cudaStream_t s, int what,
                       bool lowp) {
    if (M.kind == SM_ILU) {
        // f.u_out, as the fused sweeps' epilogues return (r.z inside CG)
        launch_ilu_smooth(&A, M, f, u, u_out, s, lowp);
        launch_dot(3 * A.nrows, f, u_out, partials, sc, what, s);
        return;
    }
    if (M.kind == SM_POINT)
        launch_reduce(A, u, EpiSmoothPoint{f, u, M.data.p, u_out}, partials, sc, what, s, lowp);
    else
        launch_reduce(A, u, EpiSmoothBlock{f, u, M.data.p, u_out}, partials, sc, what, s, lowp);
}

// 6x6 node-blocked copy: node rows i = block rows (2i, 2i+1) whose column
// lists are equal and made of consecutive pairs (2j, 2j+1)
bool make_node6(Bsr3 &A, cudaStream_t s) {
    if (A.nrows < 2 || (A.nrows & 1) || (A.ncols & 1) || A.nnzb == 0 || (A.nnzb & 3)) return false;
    const int64_t nr6 = A.nrows / 2;
    DevBuf<int> bad(1, s), cnt(nr6 + 1, s);
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    const int *ap = A.ptr.p, *ac = A.col.p;
    int *bp = bad.p, *cp = cnt.p;
    k_node6_check<<<ceil_div(nr6, 256), 256, 0, s>>>(nr6, ap, ac, bp, cp);
    CK_LAUNCH();
    int hb = 0;
    CK(cudaMemcpyAsync(&hb, bad.p, sizeof hb, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hb) return false;
    A.nrows6 = nr6;
    A.nnzb6 = A.nnzb / 4;
    A.ptr6.alloc(nr6 + 1, s);
    A.col6.alloc(A.nnzb6, s);
    A.val6.alloc(36 * A.nnzb6, s);
    k_node6_fill<<<ceil_div(nr6, 128), 128, 0, s>>>(nr6, ap, ac, A.val.p, A.ptr6.p, A.col6.p, A.val6.p);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(s));
    return true;
}

void make_lowp(Bsr3 &A, cudaStream_t s) {
    A.val32.alloc(9 * A.nnzb, s);
    if (A.nnzb) k_to_f32<<<vec_grid(9 * A.nnzb), 256, 0, s>>>(9 * A.nnzb, A.val.p, A.val32.p);
    CK_LAUNCH();
}

void launch_dense_gemv(int64_t n, const double *Ainv, const double *f, double *u,
                       cudaStream_t s) {
    if (n == 0) return;
    static const int tma = env_int("SAMG_GEMV_TMA", 1);
    const int64_t ld = dense_ld(n);
    // f and at least 4 row stages in shared memory, 16-byte aligned rows
    if (tma && 8 * ld * 5 + 384 <= 227 * 1024 && (reinterpret_cast<uintptr_t>(Ainv) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(f) & 15) == 0) {
        static DeviceCache attr;
        const int ok = attr.get([] {
            return cudaFuncSetAttribute(k_dense_gemv_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        227 * 1024) == cudaSuccess ? 1 : (cudaGetLastError(), 0);
        });
        if (ok) {
            const int stages = static_cast<int>(std::min<int64_t>(16, (227 * 1024 - 384 - 8 * ld) / (8 * ld)));
            const size_t smem = 384 + static_cast<size_t>(8 * ld) * (stages + 1);
            const int grid = static_cast<int>(std::min<int64_t>(sm_count(), n));
            static const int gemv_ef = env_int("SAMG_GEMV_EVICT_FIRST", 1);
            launch_k(false, k_dense_gemv_tma, grid, 32 * (kGemvWarps + 1), smem, s, static_cast<int>(n), ld, Ainv, f,
                     u, stages, l2_hints() && gemv_ef ? 1 : 0);
            CK_LAUNCH();
            return;
        }
    }
    launch_k(false, k_dense_gemv, static_cast<int>(n), kGemvThreads, 0, s, static_cast<int>(n), dense_ld(n), Ainv, f, u,
             l2_hints() ? 1 : 0);
    CK_LAUNCH();
}

void launch_dot(int64_t n, const double *x, const double *y, double *partials, CgScalars *sc,
                int what, cudaStream_t s) {
    launch_k(false, k_dot, vec_grid(n / 2 + 1), 256, 0, s, n, x, y, partials, sc, what);
    CK_LAUNCH();
}

void launch_cg_update(int64_t n, CgScalars *sc, const double *p, const double *q, double *u,
                      double *r, double *partials, int what, cudaGraphConditionalHandle h,
                      cudaStream_t s) {
    launch_k(false, k_cg_update, vec_grid(n / 2 + 1), 256, 0, s, n, sc, p, q, u, r, partials, what, h);
    CK_LAUNCH();
}

bool launch_cg_update_smooth(int64_t nrows, CgScalars *sc, const double *q, double *r,
                             const Smoother &M, double *z0, double *partials, int what,
                             cudaGraphConditionalHandle h, cudaStream_t s) {
    if (M.kind != SM_POINT && M.kind != SM_BLOCK) return false;
    const int grid = std::max(1, std::min<int>(kRedBlocks, ceil_div(nrows, 256)));
    if (M.kind == SM_BLOCK)
        launch_k(false, k_cg_update_smooth<true>, grid, 256, 0, s, nrows, sc, q, r,
                 static_cast<const double *>(M.data.p), z0, partials, what, h);
    else
        launch_k(false, k_cg_update_smooth<false>, grid, 256, 0, s, nrows, sc, q, r,
                 static_cast<const double *>(M.data.p), z0, partials, what, h);
    CK_LAUNCH();
    return true;
}

void launch_p_update_u(int64_t n, const CgScalars *sc, const double *z, double *p, double *u,
                       cudaStream_t s) {
    launch_k(false, k_p_update_u, vec_grid(n / 2 + 1), 256, 0, s, n, sc, z, p, u);
    CK_LAUNCH();
}

void launch_u_update(int64_t n, const CgScalars *sc, const double *p, double *u, cudaStream_t s) {
    launch_k(false, k_u_update, vec_grid(n), 256, 0, s, n, sc, p, u);
    CK_LAUNCH();
}

bool launch_restrict_smooth(const Bsr3 &R, const double *r, double *f, const Smoother &M, double *u,
                            cudaStream_t s, bool lowp) {
    if (M.kind == SM_BLOCK) launch_rows(R, r, EpiRestrictSmooth<true>{f, u, M.data.p}, s, lowp);
    else if (M.kind == SM_POINT) launch_rows(R, r, EpiRestrictSmooth<false>{f, u, M.data.p}, s, lowp);
    else return false;
    return true;
}

void launch_p_update(int64_t n, const CgScalars *sc, const double *z, double *p,
                     cudaStream_t s) {
    launch_k(false, k_p_update, vec_grid(n / 2 + 1), 256, 0, s, n, static_cast<const CgScalars *>(sc), z, p);
    CK_LAUNCH();
}

void launch_cg_finish(CgScalars *sc, int what, cudaStream_t s) {
    launch_k(false, k_cg_finish, 1, 1, 0, s, sc, what);
    CK_LAUNCH();
}

void launch_cg_finish2(CgScalars *sc, int rr_what, cudaGraphConditionalHandle h, cudaStream_t s) {
    launch_k(false, k_cg_finish2, 1, 1, 0, s, sc, rr_what, h);
    CK_LAUNCH();
}

void launch_fill(int64_t n, double v, double *x, cudaStream_t s) {
    if (n == 0) return;
    launch_k(false, k_fill, vec_grid(n), 256, 0, s, n, v, x);
    CK_LAUNCH();
}


int vtail_group(int64_t nrows, int64_t nnzb, int64_t threads) {
    static const int forced = env_int("SAMG_VTAIL_G", 0);
    if (forced) return forced;
    // ~8 blocks per lane, then as many lanes as the resident grid allows in
    // one pass (shorter per-lane chains), at most 128
    const double bpr = nrows ? static_cast<double>(nnzb) / nrows : 0.0;
    int G = 4;
    while (G < 128 && G * 8.0 < bpr) G *= 2;
    while (G < 128 && nrows * G * 2 <= threads) G *= 2;
    return G;
}

int vtail_grid(size_t smem) {
    static DeviceCache attr;
    const int ok = attr.get([&] {
        int dev = 0, coop = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        if (!coop) return 0;
        // up to 96 KB of staged coarse right-hand side
        return cudaFuncSetAttribute(k_vtail, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024) ==
                       cudaSuccess ? 1 : (cudaGetLastError(), 0);
    });
    if (!ok || smem > 96 * 1024) return 0;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_vtail, kVtThreads, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return occ * sm_count();
}

void launch_vtail(const VPhase *d_ph, int nph, unsigned *bar, int grid, size_t smem, int64_t gemv_ld,
                  double *final_out, cudaStream_t s, unsigned long long *trace) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kVtThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    static const int sleep_ns = env_int("SAMG_VTAIL_SLEEP", 0);
    const int flags = (smem >= static_cast<size_t>(8 * gemv_ld) && gemv_ld > 0 ? 1 : 0) | (l2_hints() ? 2 : 0) |
                      (sleep_ns << 8);
    CK(cudaLaunchKernelEx(&cfg, k_vtail, d_ph, nph, bar, final_out, flags, trace));
}

} // namespace samgb
