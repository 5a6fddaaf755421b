// solve.cu -- solve-phase kernels: 3x3-BSR SpMV family (spmv, residual,
// fused smoother sweep, fused CG matvec+dot), coarse dense GEMV and the CG
// vector kernels with deterministic reductions.
//
// All of these are HBM-bandwidth bound (18 flop per 76 B of matrix; DESIGN.md
// section 3).  A group of G lanes (G in {4,8,16,32}, chosen per matrix from
// its blocks per row) owns one block row.  Default (variant 1): lane l
// accumulates whole 3x3 blocks beg+l, beg+l+G, ... with 16-byte loads, so
// the row's 72-byte blocks stream as contiguous, coalesced bytes; col[] is
// read once per block and x[3c..3c+2] is a gather that hits L1/L2
// (structured meshes keep the column window small).  Variant 0 (row units:
// lane l handles scalar row l%3 of every block) is kept for comparison
// (SAMG_SPMV_VARIANT=0).  The three row sums are combined with a width-G
// butterfly and the epilogue (spmv / residual / smoother sweep / CG dot) is
// fused on lanes 0..2.
#include "kernels.cuh"

#include <algorithm>
#include <cstdlib>

namespace samgb {

namespace {

__device__ __forceinline__ double ld_stream(const double *p) { return __ldcs(p); }

template <int G>
__device__ __forceinline__ void group_reduce3(double &v0, double &v1, double &v2) {
#pragma unroll
    for (int off = G / 2; off >= 1; off >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, off, G);
        v1 += __shfl_xor_sync(0xffffffffu, v1, off, G);
        v2 += __shfl_xor_sync(0xffffffffu, v2, off, G);
    }
}

// Row-unit accumulation shared by every BSR3 kernel.  Returns the three row
// sums (A x)_row in every lane of the group.
template <int G>
__device__ __forceinline__ void bsr3_row_sums(int row, int nrows, int lane,
        const int *__restrict__ ptr, const int *__restrict__ col,
        const double *__restrict__ val, const double *__restrict__ x,
        double &s0, double &s1, double &s2) {
    constexpr int U = G - G % 3;
    double s = 0.0, t2 = 0.0;
    if (row < nrows && lane < U) {
        const int beg = __ldg(ptr + row), end = __ldg(ptr + row + 1);
        const int nu = 3 * (end - beg);
        const double *v = val + 9 * static_cast<size_t>(beg);
        const int *cc = col + beg;
        int t = lane;
        for (; t + U < nu; t += 2 * U) {
            const int b0 = t / 3, b1 = (t + U) / 3;
            const int c0 = __ldg(cc + b0), c1 = __ldg(cc + b1);
            const double a0 = ld_stream(v + 3 * t), a1 = ld_stream(v + 3 * t + 1),
                         a2 = ld_stream(v + 3 * t + 2);
            const double d0 = ld_stream(v + 3 * (t + U)), d1 = ld_stream(v + 3 * (t + U) + 1),
                         d2 = ld_stream(v + 3 * (t + U) + 2);
            const double *x0 = x + 3 * c0, *x1 = x + 3 * c1;
            s = fma(a0, __ldg(x0), s);
            s = fma(a1, __ldg(x0 + 1), s);
            s = fma(a2, __ldg(x0 + 2), s);
            t2 = fma(d0, __ldg(x1), t2);
            t2 = fma(d1, __ldg(x1 + 1), t2);
            t2 = fma(d2, __ldg(x1 + 2), t2);
        }
        if (t < nu) {
            const int c0 = __ldg(cc + t / 3);
            const double *x0 = x + 3 * c0;
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

// Block-per-lane accumulation: lane l of the group handles whole blocks
// j = beg+l, beg+l+G, ...  A block (72 B) is read with four 16-byte loads
// plus one 8-byte load whose offsets depend only on the parity of j (block j
// starts 16-byte aligned iff j is even), so every lane runs the same
// instruction sequence; x[3c..3c+2] likewise with one 16-byte + one 8-byte
// load.  Per block: 1 col + 5 value + 2 x loads (vs 21 scalar loads).
__device__ __forceinline__ double2 ldg2(const double *p) {
    return __ldg(reinterpret_cast<const double2 *>(p));
}

template <int G>
__device__ __forceinline__ void bsr3_row_sums_blk(int row, int nrows, int lane,
        const int *__restrict__ ptr, const int *__restrict__ col,
        const double *__restrict__ val, const double *__restrict__ x,
        double &s0, double &s1, double &s2) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    if (row < nrows) {
        const int beg = __ldg(ptr + row), end = __ldg(ptr + row + 1);
#pragma unroll 2
        for (int j = beg + lane; j < end; j += G) {
            const int c = __ldg(col + j);
            const double *v = val + 9 * static_cast<size_t>(j);
            const int odd = j & 1;
            const double2 q0 = ldg2(v + odd), q1 = ldg2(v + odd + 2), q2 = ldg2(v + odd + 4),
                          q3 = ldg2(v + odd + 6);
            const double e = __ldg(v + (odd ? 0 : 8));
            const double *xp = x + 3 * static_cast<size_t>(c);
            const int xo = c & 1;
            const double2 xq = ldg2(xp + xo);
            const double xe = __ldg(xp + (xo ? 0 : 2));
            const double x0 = xo ? xe : xq.x, x1 = xo ? xq.x : xq.y, x2 = xo ? xq.y : xe;
            const double b0 = odd ? e : q0.x, b1 = odd ? q0.x : q0.y, b2 = odd ? q0.y : q1.x;
            const double b3 = odd ? q1.x : q1.y, b4 = odd ? q1.y : q2.x, b5 = odd ? q2.x : q2.y;
            const double b6 = odd ? q2.y : q3.x, b7 = odd ? q3.x : q3.y, b8 = odd ? q3.y : e;
            a0 = fma(b0, x0, a0); a0 = fma(b1, x1, a0); a0 = fma(b2, x2, a0);
            a1 = fma(b3, x0, a1); a1 = fma(b4, x1, a1); a1 = fma(b5, x2, a1);
            a2 = fma(b6, x0, a2); a2 = fma(b7, x1, a2); a2 = fma(b8, x2, a2);
        }
    }
    s0 = a0; s1 = a1; s2 = a2;
    group_reduce3<G>(s0, s1, s2);
}

int spmv_variant() {
    static const int v = [] {
        const char *e = std::getenv("SAMG_SPMV_VARIANT");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

template <int G, int V>
__device__ __forceinline__ void row_sums(int row, int nrows, int lane, const int *__restrict__ ptr,
        const int *__restrict__ col, const double *__restrict__ val,
        const double *__restrict__ x, double &s0, double &s1, double &s2) {
    if constexpr (V == 1) bsr3_row_sums_blk<G>(row, nrows, lane, ptr, col, val, x, s0, s1, s2);
    else bsr3_row_sums<G>(row, nrows, lane, ptr, col, val, x, s0, s1, s2);
}

__device__ __forceinline__ double pick3(int c, double a, double b, double d) {
    return c == 0 ? a : (c == 1 ? b : d);
}

struct EpiSpmv {
    double alpha, beta;
    double *y;
    __device__ void operator()(int row, int c, double s0, double s1, double s2) const {
        double *yi = y + 3 * static_cast<size_t>(row) + c;
        const double s = pick3(c, s0, s1, s2);
        *yi = alpha * s + (beta == 0.0 ? 0.0 : beta * *yi);
    }
};

struct EpiResidual {
    const double *f;
    double *r;
    __device__ void operator()(int row, int c, double s0, double s1, double s2) const {
        const size_t i = 3 * static_cast<size_t>(row) + c;
        r[i] = f[i] - pick3(c, s0, s1, s2);
    }
};

struct EpiSmoothPoint {  // u_out = u + (omega/a_cc) * (f - A u)
    const double *f, *u, *m;
    double *out;
    __device__ void operator()(int row, int c, double s0, double s1, double s2) const {
        const size_t i = 3 * static_cast<size_t>(row) + c;
        out[i] = u[i] + m[i] * (f[i] - pick3(c, s0, s1, s2));
    }
};

struct EpiSmoothBlock {  // u_out = u + M_row (f - A u)_row
    const double *f, *u, *m;
    double *out;
    __device__ void operator()(int row, int c, double s0, double s1, double s2) const {
        const size_t b = 3 * static_cast<size_t>(row);
        const double r0 = f[b] - s0, r1 = f[b + 1] - s1, r2 = f[b + 2] - s2;
        const double *M = m + 9 * static_cast<size_t>(row) + 3 * c;
        out[b + c] = u[b + c] + (M[0] * r0 + M[1] * r1 + M[2] * r2);
    }
};

// V = 0: row units; V = 1: block per lane; V = 2: block per lane with the
// register budget capped for 6 resident CTAs (48 warps) per SM.
template <int G, int V, class Epi>
__global__ void __launch_bounds__(256, V == 2 ? 6 : 1) k_bsr3(int nrows,
        const int *__restrict__ ptr, const int *__restrict__ col,
        const double *__restrict__ val, const double *__restrict__ x, Epi epi) {
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int row = gtid / G, lane = threadIdx.x % G;
    double s0, s1, s2;
    row_sums<G, (V == 0 ? 0 : 1)>(row, nrows, lane, ptr, col, val, x, s0, s1, s2);
    if (row < nrows && lane < 3) epi(row, lane, s0, s1, s2);
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

// fused CG matvec q = A p with p.q: grid-stride over row groups with a fixed
// grid, so the partial sums (one per CTA) are few and their order fixed.
constexpr int kDotCtas = 148 * 8;

template <int G, int V>
__global__ void __launch_bounds__(256) k_bsr3_dot(int nrows, const int *__restrict__ ptr,
        const int *__restrict__ col, const double *__restrict__ val,
        const double *__restrict__ p, double *__restrict__ q, double *__restrict__ partials) {
    const int groups = gridDim.x * (blockDim.x / G);
    const int lane = threadIdx.x % G;
    double d = 0.0;
    const int nit = (nrows + groups - 1) / groups;
    for (int it = 0; it < nit; ++it) {
        const int row = (blockIdx.x * blockDim.x + threadIdx.x) / G + it * groups;
        double s0, s1, s2;
        row_sums<G, (V == 0 ? 0 : 1)>(row, nrows, lane, ptr, col, val, p, s0, s1, s2);
        if (row < nrows && lane < 3) {
            const size_t i = 3 * static_cast<size_t>(row) + lane;
            const double qi = pick3(lane, s0, s1, s2);
            q[i] = qi;
            d = fma(p[i], qi, d);
        }
    }
    d = block_sum(d);
    if (threadIdx.x == 0) partials[blockIdx.x] = d;
}

int choose_group(const Bsr3 &A) {
    static const int forced = [] {
        const char *e = std::getenv("SAMG_SPMV_GROUP");
        return e ? std::atoi(e) : 0;
    }();
    if (forced == 4 || forced == 8 || forced == 16 || forced == 32) return forced;
    const double bpr = A.nrows ? static_cast<double>(A.nnzb) / A.nrows : 0.0;
    if (spmv_variant() >= 1) {
        // ~7 blocks per lane: enough independent loads per thread to cover
        // HBM latency, several rows per warp (measured on C1, fine rows of
        // ~26 blocks: G=4 5.9 TB/s, G=8 5.2, G=16 4.8, G=32 4.2; profiles/)
        static const double per_lane = [] {
            const char *e = std::getenv("SAMG_SPMV_BLOCKS_PER_LANE");
            return e ? std::atof(e) : 7.0;
        }();
        const double want = bpr / per_lane;
        if (want > 16.0) return 32;
        if (want > 8.0) return 16;
        if (want > 4.0) return 8;
        return 4;
    }
    if (3.0 * bpr >= 45.0) return 32;
    if (3.0 * bpr >= 12.0) return 16;
    return 8;
}

#define SAMG_DISPATCH_G(G, V, ...)                                  \
    if ((V) == 1) {                                                 \
        switch (G) {                                                \
            case 32: { constexpr int GG = 32, VV = 1; __VA_ARGS__; } break; \
            case 16: { constexpr int GG = 16, VV = 1; __VA_ARGS__; } break; \
            case 8: { constexpr int GG = 8, VV = 1; __VA_ARGS__; } break;   \
            default: { constexpr int GG = 4, VV = 1; __VA_ARGS__; } break;  \
        }                                                           \
    } else if ((V) == 2) {                                          \
        switch (G) {                                                \
            case 32: { constexpr int GG = 32, VV = 2; __VA_ARGS__; } break; \
            case 16: { constexpr int GG = 16, VV = 2; __VA_ARGS__; } break; \
            case 8: { constexpr int GG = 8, VV = 2; __VA_ARGS__; } break;   \
            default: { constexpr int GG = 4, VV = 2; __VA_ARGS__; } break;  \
        }                                                           \
    } else {                                                        \
        switch (G) {                                                \
            case 32: { constexpr int GG = 32, VV = 0; __VA_ARGS__; } break; \
            case 16: { constexpr int GG = 16, VV = 0; __VA_ARGS__; } break; \
            default: { constexpr int GG = 8, VV = 0; __VA_ARGS__; } break;  \
        }                                                           \
    }

template <class Epi>
void launch_rows(const Bsr3 &A, const double *x, Epi epi, cudaStream_t s) {
    if (A.nrows == 0) return;
    const int G = choose_group(A);
    const int grid = ceil_div(A.nrows * static_cast<int64_t>(G), 256);
    const int n = static_cast<int>(A.nrows);
    SAMG_DISPATCH_G(G, spmv_variant(),
        (k_bsr3<GG, VV><<<grid, 256, 0, s>>>(n, A.ptr.p, A.col.p, A.val.p, x, epi)));
    CK_LAUNCH();
}

__global__ void k_smooth_zero_point(int64_t n, const double *__restrict__ m,
        const double *__restrict__ f, double *__restrict__ u) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        u[i] = m[i] * f[i];
}

__global__ void k_smooth_zero_block(int64_t nrows, const double *__restrict__ m,
        const double *__restrict__ f, double *__restrict__ u) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < 3 * nrows;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t row = e / 3;
        const int c = static_cast<int>(e - 3 * row);
        const double *M = m + 9 * row + 3 * c;
        const double *fr = f + 3 * row;
        u[e] = M[0] * fr[0] + M[1] * fr[1] + M[2] * fr[2];
    }
}

// u = Ainv f, Ainv row-major with an even leading dimension (zero padded):
// one warp per row, 16-byte loads, 4 in flight per lane.
__global__ void k_dense_gemv(int n, int64_t ld, const double *__restrict__ A,
        const double *__restrict__ f, double *__restrict__ u) {
    const int row = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
    if (row >= n) return;
    const double2 *a = reinterpret_cast<const double2 *>(A + static_cast<size_t>(row) * ld);
    const int n2 = static_cast<int>(ld / 2);
    double s = 0.0, t = 0.0;
    auto fpair = [&](int j2) {
        const int j = 2 * j2;
        return make_double2(__ldg(f + j), j + 1 < n ? __ldg(f + j + 1) : 0.0);
    };
    int j2 = lane;
    for (; j2 + 96 < n2; j2 += 128) {
        const double2 a0 = __ldcs(a + j2), a1 = __ldcs(a + j2 + 32), a2 = __ldcs(a + j2 + 64),
                      a3 = __ldcs(a + j2 + 96);
        const double2 f0 = fpair(j2), f1 = fpair(j2 + 32), f2 = fpair(j2 + 64), f3 = fpair(j2 + 96);
        s = fma(a0.x, f0.x, s); t = fma(a0.y, f0.y, t);
        s = fma(a1.x, f1.x, s); t = fma(a1.y, f1.y, t);
        s = fma(a2.x, f2.x, s); t = fma(a2.y, f2.y, t);
        s = fma(a3.x, f3.x, s); t = fma(a3.y, f3.y, t);
    }
    for (; j2 < n2; j2 += 32) {
        const double2 a0 = __ldcs(a + j2);
        const double2 f0 = fpair(j2);
        s = fma(a0.x, f0.x, s); t = fma(a0.y, f0.y, t);
    }
    s += t;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) u[row] = s;
}

__global__ void __launch_bounds__(256) k_dot(int64_t n, const double *__restrict__ x,
        const double *__restrict__ y, double *__restrict__ partials) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        s = fma(x[i], y[i], s);
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_cg_update(int64_t n, const CgScalars *__restrict__ sc,
        const double *__restrict__ p, const double *__restrict__ q, double *__restrict__ u,
        double *__restrict__ r, double *__restrict__ partials) {
    const double a = sc->alpha;
    double s = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        u[i] = fma(a, p[i], u[i]);
        const double ri = fma(-a, q[i], r[i]);
        r[i] = ri;
        s = fma(ri, ri, s);
    }
    s = block_sum(s);
    if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

__global__ void k_p_update(int64_t n, const CgScalars *__restrict__ sc,
        const double *__restrict__ z, double *__restrict__ p) {
    const double b = sc->beta;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = fma(b, p[i], z[i]);
}

__global__ void k_fill(int64_t n, double v, double *x) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        x[i] = v;
}

__global__ void __launch_bounds__(256) k_finalize(int what, const double *__restrict__ partials,
        int nparts, CgScalars *sc) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partials[i];
    s = block_sum(s);
    if (threadIdx.x != 0) return;
    switch (what) {
        case 0: sc->rr = s; break;
        case 1:
            sc->pq = s;
            if (!(s > 0.0)) sc->breakdown = 1;
            sc->alpha = sc->rho / s;
            break;
        case 2:
            sc->rho_new = s;
            sc->beta = s / sc->rho;
            sc->rho = s;
            break;
        default: sc->rho = s; break;
    }
}

__global__ void __launch_bounds__(256) k_finalize_loop(const double *__restrict__ partials,
        int nparts, CgScalars *sc, cudaGraphConditionalHandle h) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partials[i];
    s = block_sum(s);
    if (threadIdx.x != 0) return;
    sc->rr = s;
    const int it = sc->iter + 1;
    sc->iter = it;
    const bool go = (sqrt(s) / sc->norm_f > sc->tol) && it < sc->max_iter && !sc->breakdown;
    cudaGraphSetConditional(h, go ? 1u : 0u);
}

// norm_f / tol / max_iter are written by the host before the graph launch
__global__ void k_cg_loop_init(CgScalars *sc, cudaGraphConditionalHandle h) {
    sc->iter = 0;
    sc->breakdown = 0;
    // loop condition before the first pass: res_norm = norm_f (cg.hpp:60-62)
    cudaGraphSetConditional(h, (1.0 > sc->tol && 0 < sc->max_iter) ? 1u : 0u);
}

int vec_grid(int64_t n) {
    const int64_t g = (n + 255) / 256;
    return static_cast<int>(g < kRedBlocks ? (g > 0 ? g : 1) : kRedBlocks);
}

} // namespace

void launch_spmv(const Bsr3 &A, double alpha, const double *x, double beta, double *y,
                 cudaStream_t s) {
    launch_rows(A, x, EpiSpmv{alpha, beta, y}, s);
}

void launch_residual(const Bsr3 &A, const double *f, const double *u, double *r,
                     cudaStream_t s) {
    launch_rows(A, u, EpiResidual{f, r}, s);
}

void launch_smooth(const Bsr3 &A, const Smoother &M, const double *f, const double *u,
                   double *u_out, cudaStream_t s) {
    if (M.kind == SM_POINT) launch_rows(A, u, EpiSmoothPoint{f, u, M.data.p, u_out}, s);
    else launch_rows(A, u, EpiSmoothBlock{f, u, M.data.p, u_out}, s);
}

void launch_smooth_zero(int64_t nrows, const Smoother &M, const double *f, double *u,
                        cudaStream_t s) {
    if (nrows == 0) return;
    const int grid = vec_grid(3 * nrows);
    if (M.kind == SM_POINT) k_smooth_zero_point<<<grid, 256, 0, s>>>(3 * nrows, M.data.p, f, u);
    else k_smooth_zero_block<<<grid, 256, 0, s>>>(nrows, M.data.p, f, u);
    CK_LAUNCH();
}

void launch_spmv_dot(const Bsr3 &A, const double *p, double *q, double *partials, int *nparts,
                     cudaStream_t s) {
    const int G = choose_group(A);
    const int grid = std::max(1, std::min(kDotCtas, ceil_div(A.nrows * static_cast<int64_t>(G), 256)));
    const int n = static_cast<int>(A.nrows);
    SAMG_DISPATCH_G(G, spmv_variant(),
        (k_bsr3_dot<GG, VV><<<grid, 256, 0, s>>>(n, A.ptr.p, A.col.p, A.val.p, p, q, partials)));
    CK_LAUNCH();
    *nparts = grid;
}

void launch_dense_gemv(int64_t n, const double *Ainv, const double *f, double *u,
                       cudaStream_t s) {
    if (n == 0) return;
    k_dense_gemv<<<ceil_div(n * 32, 256), 256, 0, s>>>(static_cast<int>(n), dense_ld(n), Ainv, f, u);
    CK_LAUNCH();
}

void launch_dot_partials(int64_t n, const double *x, const double *y, double *partials,
                         cudaStream_t s) {
    k_dot<<<kRedBlocks, 256, 0, s>>>(n, x, y, partials);
    CK_LAUNCH();
}

void launch_finalize(int what, const double *partials, int nparts, CgScalars *sc,
                     cudaStream_t s) {
    k_finalize<<<1, 256, 0, s>>>(what, partials, nparts, sc);
    CK_LAUNCH();
}

void launch_finalize_loop(const double *partials, int nparts, CgScalars *sc,
                          cudaGraphConditionalHandle h, cudaStream_t s) {
    k_finalize_loop<<<1, 256, 0, s>>>(partials, nparts, sc, h);
    CK_LAUNCH();
}

void launch_cg_loop_init(CgScalars *sc, cudaGraphConditionalHandle h, cudaStream_t s) {
    k_cg_loop_init<<<1, 1, 0, s>>>(sc, h);
    CK_LAUNCH();
}

void launch_cg_update(int64_t n, const CgScalars *sc, const double *p, const double *q,
                      double *u, double *r, double *partials, cudaStream_t s) {
    k_cg_update<<<kRedBlocks, 256, 0, s>>>(n, sc, p, q, u, r, partials);
    CK_LAUNCH();
}

void launch_p_update(int64_t n, const CgScalars *sc, const double *z, double *p,
                     cudaStream_t s) {
    k_p_update<<<vec_grid(n), 256, 0, s>>>(n, sc, z, p);
    CK_LAUNCH();
}

void launch_fill(int64_t n, double v, double *x, cudaStream_t s) {
    if (n == 0) return;
    k_fill<<<vec_grid(n), 256, 0, s>>>(n, v, x);
    CK_LAUNCH();
}

} // namespace samgb
