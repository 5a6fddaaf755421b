// setup.cu -- setup-phase kernels of the ns_block pipeline.
//
// COMPILED WITH --fmad=false: the reference's header code is built without
// -mfma, so every product and sum here is a separately rounded
// IEEE operation, and every sum is taken in the reference's order.  With
// identical inputs the strength graph, the aggregates, P, R and the Galerkin
// products are therefore bit-identical to samg::setup (pinned by
// tests/test_gpu_parity.py).
//
// Reference functions restated (paths under proj/include/samg/):
//   to_block<3>            csr.hpp:268-324          -> k_s2b_*
//   condense_weights +
//   strength_graph         coarsening.hpp:52-123    -> k_strength_*
//   aggregate              coarsening.hpp:131-160   -> k_agg_* (parallel, exact)
//   thin_qr +
//   tentative_prolongation coarsening.hpp:167-312   -> k_tentative_qr
//   smooth_prolongation    coarsening.hpp:319-416   -> k_psm_*
//   transpose              csr.hpp:173-194          -> k_tr_*
//   spgemm / galerkin      csr.hpp:199-262          -> k_spgemm_*
//   fix_decoupled_rows     hierarchy.hpp:172-191    -> k_fix_rows
//   damped_jacobi ctor     relaxation.hpp:147-162   -> k_sm_point
//   block smoothers        DESIGN.md section 4      -> k_sm_block
#include "block3.cuh"
#include "kernels.cuh"

#include <cub/cub.cuh>

// the pattern-only (kCols) instances return before the accumulation loops
#pragma nv_diag_suppress 128

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace samgb {

namespace {

constexpr int INF = 0x7fffffff;

__device__ void raise(DevError *err, int code, int64_t where) {
    if (atomicCAS(&err->code, 0, code) == 0) err->where = where;
}

template <class F>
__global__ void k_for(int64_t n, F f) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        f(i);
}

template <class F>
void for_each(int64_t n, F f, cudaStream_t s) {
    if (n <= 0) return;
    int64_t g = (n + 255) / 256;
    if (g > 65535LL * 8) g = 65535LL * 8;
    k_for<<<static_cast<int>(g), 256, 0, s>>>(n, f);
    CK_LAUNCH();
}

// exclusive scan of n ints into out (n+1 entries, out[n] = total); returns total
int64_t scan_counts(const int *in, int *out, int64_t n, cudaStream_t s) {
    DevBuf<int64_t> tmp64(n + 1, s);
    int64_t *t = tmp64.p;
    for_each(n, [=] __device__(int64_t i) { t[i] = in[i]; }, s);
    size_t bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, t, t, n + 1, s));
    DevBuf<char> ws(bytes, s);
    // t[n] must be zero before the scan so that t[n] becomes the total
    CK(cudaMemsetAsync(t + n, 0, sizeof(int64_t), s));
    CK(cub::DeviceScan::ExclusiveSum(ws.p, bytes, t, t, n + 1, s));
    int64_t total = 0;
    CK(cudaMemcpyAsync(&total, t + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (total > INT32_MAX) fail(SAMG_UNSUPPORTED, "setup: more than 2^31-1 entries in one matrix");
    for_each(n + 1, [=] __device__(int64_t i) { out[i] = static_cast<int>(t[i]); }, s);
    return total;
}

__device__ __forceinline__ bool bsearch_int(const int *a, int lo, int hi, int key) {
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const int v = a[mid];
        if (v == key) return true;
        if (v < key) lo = mid + 1;
        else hi = mid;
    }
    return false;
}

__device__ __forceinline__ int lower_bound_int(const int *a, int n, int key) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// 3x3 product, static_block.hpp:104-113 (r = 0; r(i,j) += a(i,k) b(k,j); i,k,j)
__device__ __forceinline__ void blk_mul(const double *a, const double *b, double *r) {
#pragma unroll
    for (int e = 0; e < 9; ++e) r[e] = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double aik = a[i * 3 + k];
#pragma unroll
            for (int j = 0; j < 3; ++j) r[i * 3 + j] = __dadd_rn(r[i * 3 + j], __dmul_rn(aik, b[k * 3 + j]));
        }
}

// c += a*b for the SpGEMM accumulators.  Block arithmetic (csr<block3>):
// the block product first (blk_mul), then added.  Scalar order (csr<double>
// on the full-block scalar view, csr.hpp:237-243): each scalar term goes
// straight into the accumulator, terms of one block in q order.
template <bool kScalar>
__device__ __forceinline__ void accum_block(const double *a, const double *b, double *c) {
    if constexpr (kScalar) {
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                double t = c[p * 3 + q];
                t = __dadd_rn(t, __dmul_rn(a[p * 3 + 0], b[0 * 3 + q]));
                t = __dadd_rn(t, __dmul_rn(a[p * 3 + 1], b[1 * 3 + q]));
                t = __dadd_rn(t, __dmul_rn(a[p * 3 + 2], b[2 * 3 + q]));
                c[p * 3 + q] = t;
            }
    } else {
        double prod[9];
        blk_mul(a, b, prod);
#pragma unroll
        for (int e = 0; e < 9; ++e) c[e] = __dadd_rn(c[e], prod[e]);
    }
}

// ---------------------------------------------------------------------------
// to_block<3> of a sorted scalar CSR (csr.hpp:268-324): 3-way merge of the
// scalar rows' block columns; absent tile entries stay zero.

template <class CT>
__global__ void k_s2b_count(int64_t nb, const int64_t *ptr, const CT *col, int *cnt,
                            DevError *err) {
    for (int64_t bi = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; bi < nb;
         bi += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t h[3], e[3];
        for (int r = 0; r < 3; ++r) { h[r] = ptr[3 * bi + r]; e[r] = ptr[3 * bi + r + 1]; }
        for (int r = 0; r < 3; ++r) {
            if (h[r] < e[r] && (col[h[r]] < 0 || col[e[r] - 1] >= 3 * nb))
                raise(err, SAMG_INVALID_ARGUMENT, 3 * bi + r);  // column out of range
            for (int64_t j = h[r] + 1; j < e[r]; ++j)
                if (col[j] <= col[j - 1]) raise(err, SAMG_INVALID_ARGUMENT, 3 * bi + r);
        }
        int c = 0;
        while (true) {
            int64_t m = INT64_MAX;
            for (int r = 0; r < 3; ++r)
                if (h[r] < e[r]) m = min(m, static_cast<int64_t>(col[h[r]]) / 3);
            if (m == INT64_MAX) break;
            ++c;
            for (int r = 0; r < 3; ++r)
                while (h[r] < e[r] && col[h[r]] / 3 == m) ++h[r];
        }
        cnt[bi] = c;
    }
}

template <class CT>
__global__ void k_s2b_fill(int64_t nb, const int64_t *ptr, const CT *col,
                           const double *val, const int *bptr, int *bcol, double *bval) {
    for (int64_t bi = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; bi < nb;
         bi += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t h[3], e[3];
        for (int r = 0; r < 3; ++r) { h[r] = ptr[3 * bi + r]; e[r] = ptr[3 * bi + r + 1]; }
        int out = bptr[bi];
        while (true) {
            int64_t m = INT64_MAX;
            for (int r = 0; r < 3; ++r)
                if (h[r] < e[r]) m = min(m, static_cast<int64_t>(col[h[r]]) / 3);
            if (m == INT64_MAX) break;
            bcol[out] = static_cast<int>(m);
            double *blk = bval + 9 * static_cast<int64_t>(out);
            for (int e9 = 0; e9 < 9; ++e9) blk[e9] = 0.0;
            for (int r = 0; r < 3; ++r)
                while (h[r] < e[r] && col[h[r]] / 3 == m) {
                    blk[r * 3 + static_cast<int>(col[h[r]] % 3)] = val[h[r]];
                    ++h[r];
                }
            ++out;
        }
    }
}

// ---------------------------------------------------------------------------
// strength graph.  A node is h block rows (pbs = 3h); the weight of node
// tile (i, j) is the max |a| over its scalar entries (condense_weights,
// coarsening.hpp:64-75); edge iff w*w > (eps2*d_i)*d_j (coarsening.hpp:105),
// union-symmetrised.

// per-block max|a| over its 9 entries (read once, coalesced)
__global__ void k_block_maxabs(int64_t nnzb, const double *val, double *wblk) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < nnzb;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double *b = val + 9 * j;
        double w = 0.0;
        for (int e = 0; e < 9; ++e) w = fmax(w, fabs(b[e]));
        wblk[j] = w;
    }
}

// per-block Frobenius norm (static_block.hpp:111-115: sum of squares in
// entry order, then sqrt) -- the block pipeline's strength weight
__global__ void k_block_fnorm(int64_t nnzb, const double *val, double *wblk) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < nnzb;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double *b = val + 9 * j;
        double q = 0.0;
        for (int e = 0; e < 9; ++e) q = __dadd_rn(q, __dmul_rn(b[e], b[e]));
        wblk[j] = __dsqrt_rn(q);
    }
}

template <class F>
__device__ __forceinline__ void for_node_tiles(int node, int h, const int *ptr, const int *col,
                                               const double *wblk, F f) {
    // visit (node column, max|a|) of node row `node` in ascending node column;
    // wblk[j] = max|a| of block j (max is order-independent: exact)
    if (h == 1) {
        for (int j = ptr[node]; j < ptr[node + 1]; ++j) f(col[j], wblk[j]);
        return;
    }
    int hd[4], en[4];
    for (int r = 0; r < h; ++r) { hd[r] = ptr[node * h + r]; en[r] = ptr[node * h + r + 1]; }
    while (true) {
        int m = INF;
        for (int r = 0; r < h; ++r)
            if (hd[r] < en[r]) m = min(m, col[hd[r]] / h);
        if (m == INF) break;
        double w = 0.0;
        for (int r = 0; r < h; ++r)
            while (hd[r] < en[r] && col[hd[r]] / h == m) {
                w = fmax(w, wblk[hd[r]]);
                ++hd[r];
            }
        f(m, w);
    }
}

__global__ void k_strength_diag(int n, int h, const int *ptr, const int *col, const double *val,
                                double *d) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double di = 0.0;
    for_node_tiles(i, h, ptr, col, val, [&](int j, double w) { if (j == i) di = w; });
    d[i] = di;
}

__global__ void k_strength_edges(int n, int h, const int *ptr, const int *col, const double *val,
                                 const double *d, double eps2, int *cnt,
                                 const int *off, unsigned long long *keys) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int c = 0;
    const double di = d[i];
    int64_t o = off ? 2 * static_cast<int64_t>(off[i]) : 0;
    for_node_tiles(i, h, ptr, col, val, [&](int j, double w) {
        if (j == i) return;
        if (__dmul_rn(w, w) > __dmul_rn(__dmul_rn(eps2, di), d[j])) {
            if (keys) {
                keys[o++] = (static_cast<unsigned long long>(i) << 32) | static_cast<unsigned>(j);
                keys[o++] = (static_cast<unsigned long long>(j) << 32) | static_cast<unsigned>(i);
            }
            ++c;
        }
    });
    if (cnt) cnt[i] = c;
}

// ---------------------------------------------------------------------------
// aggregation.  Pass 1 of coarsening.hpp:136-146 seeds node i iff no earlier
// seed lies within graph distance 2, i.e. the seeds are the
// lexicographically-first maximal independent set of G^2.  It is computed
// in rounds: m1[j]/u1[j] = smallest seed / undecided index in the closed
// neighbourhood of j; an undecided i becomes OUT if min m1 over N[i] < i,
// IN if min u1 over N[i] == i (all smaller nodes within distance 2 are
// decided OUT).  Pass 2 (:148-154) joins the first neighbour (ascending)
// that is pass-1 assigned or has a smaller index; chains are resolved by
// pointer jumping.  Pass 3 (:156-157) cannot trigger (isolated nodes seed).

enum { UND = 0, IN = 1, OUT = 2 };

__global__ void k_agg_a(int n, const int *gp, const int *gc, const unsigned char *state,
                        int *m1, int *u1) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const unsigned char sj = state[j];
    int m = sj == IN ? j : INF, u = sj == UND ? j : INF;
    for (int e = gp[j]; e < gp[j + 1]; ++e) {
        const int nb = gc[e];
        const unsigned char s = state[nb];
        if (s == IN) m = min(m, nb);
        else if (s == UND) u = min(u, nb);
    }
    m1[j] = m;
    u1[j] = u;
}

__global__ void k_agg_b(int n, const int *gp, const int *gc, unsigned char *state, const int *m1,
                        const int *u1, int *undecided) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || state[i] != UND) return;
    int m = m1[i], u = u1[i];
    for (int e = gp[i]; e < gp[i + 1]; ++e) {
        const int nb = gc[e];
        m = min(m, m1[nb]);
        u = min(u, u1[nb]);
    }
    if (m < i) state[i] = OUT;
    else if (u == i) state[i] = IN;
    else atomicAdd(undecided, 1);
}

// The same rounds, event-driven: a round only recomputes the nodes whose
// inputs changed in the round before.  The lexicographic front sweeps the
// index order, so far ahead of it nothing can change and behind it
// everything is decided; re-reading the whole graph twice per round made
// C4's level-0 aggregation (7.96 M nodes, ~600 rounds) a 1 TB stream
// (161 ms).  Phase a recomputes (m1, u1) of node j only if a node of N[j]
// changed state (dA[j]); a changed (m1, u1) marks N[j] for phase b (dB);
// phase b re-decides an undecided node i only if dB[i], and a decided node
// marks N[i] for the next phase a.  Each recomputation is the full-scan
// kernels' function of the same inputs, so the result is identical.
__global__ void k_agg_ad(int n, const int *__restrict__ gp, const int *__restrict__ gc,
                         const unsigned char *state, int *m1, int *u1, unsigned char *dA,
                         unsigned char *dB) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n || !dA[j]) return;
    dA[j] = 0;
    const unsigned char sj = state[j];
    int m = sj == IN ? j : INF, u = sj == UND ? j : INF;
    const int e0 = gp[j], e1 = gp[j + 1];
    for (int e = e0; e < e1; ++e) {
        const int nb = gc[e];
        const unsigned char sn = state[nb];
        if (sn == IN) m = min(m, nb);
        else if (sn == UND) u = min(u, nb);
    }
    if (m != m1[j] || u != u1[j]) {
        m1[j] = m;
        u1[j] = u;
        dB[j] = 1;
        for (int e = e0; e < e1; ++e) dB[gc[e]] = 1;
    }
}

__global__ void k_agg_bd(int n, const int *__restrict__ gp, const int *__restrict__ gc,
                         unsigned char *state, const int *m1, const int *u1, unsigned char *dA,
                         unsigned char *dB, int *undecided) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !dB[i]) return;
    dB[i] = 0;
    if (state[i] != UND) return;
    int m = m1[i], u = u1[i];
    const int e0 = gp[i], e1 = gp[i + 1];
    for (int e = e0; e < e1; ++e) {
        const int nb = gc[e];
        m = min(m, m1[nb]);
        u = min(u, u1[nb]);
    }
    const unsigned char ns = m < i ? OUT : (u == i ? IN : UND);
    if (ns != UND) {
        state[i] = ns;
        atomicSub(undecided, 1);
        dA[i] = 1;
        for (int e = e0; e < e1; ++e) dA[gc[e]] = 1;
    }
}

// ---------------------------------------------------------------------------
// tentative prolongation: Householder thin QR per aggregate, loop orders of
// coarsening.hpp:167-229 and :289-309.  A group of 16 lanes owns one
// aggregate: every sum over rows i stays sequential on one lane (lane 0 for
// the column norm, lane c for column c's dot products), so the result is
// bit-identical to the sequential reference; the k <= 12 column updates and
// all elementwise work run in parallel across the lanes.

constexpr int kQrLanes = 16;

// smem_m > 0: the group's m x k work matrix and Q live in shared memory
// (room for m <= smem_m rows each) instead of the global scratch: the
// sequential per-lane sums walk them element by element, and from global
// memory every step waited for an L2 round trip (C4 level 0: 80 ms).  The
// arithmetic and its order are unchanged.
__global__ void __launch_bounds__(256) k_tentative_qr(int64_t naggs, int pbs, int k,
        const int *nodes, const int *agg_ptr, const double *B, int64_t bnrows, double *work,
        double *Qw, double *Pt, double *Bc, int64_t a0, int64_t a1, int smem_m) {
    __shared__ double Rs[256 / kQrLanes][144];
    extern __shared__ double qr_sm[];
    const int64_t a = a0 + (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / kQrLanes;
    const int lane = threadIdx.x % kQrLanes;
    const int base = (threadIdx.x % 32) & ~(kQrLanes - 1);
    const unsigned mask = 0xffffu << base;
    if (a >= a1) return;  // whole group
    double *R = Rs[threadIdx.x / kQrLanes];
    const int n0 = agg_ptr[a], n1 = agg_ptr[a + 1];
    const int64_t m = static_cast<int64_t>(pbs) * (n1 - n0);
    double *A = work + static_cast<int64_t>(pbs) * n0 * k;
    double *Q = Qw + static_cast<int64_t>(pbs) * n0 * k;
    if (smem_m > 0 && m <= smem_m) {
        A = qr_sm + static_cast<size_t>(threadIdx.x / kQrLanes) * 2 * smem_m * k;
        Q = A + static_cast<size_t>(smem_m) * k;
    }
#define a_(i, j) A[(j) * m + (i)]
#define ROW(r) (static_cast<int64_t>(nodes[n0 + (r) / pbs]) * pbs + (r) % pbs)
    double local_max = 0;
    for (int64_t t = lane; t < m * k; t += kQrLanes) {
        const int64_t c = t / m, r = t - c * m;
        const double v = B[c * bnrows + ROW(r)];
        A[t] = v;
        local_max = fmax(local_max, fabs(v));
    }
    for (int off = kQrLanes / 2; off >= 1; off >>= 1)
        local_max = fmax(local_max, __shfl_xor_sync(mask, local_max, off, kQrLanes));
    __syncwarp(mask);
    const double tol = __dmul_rn(1e-12, fmax(local_max, 1.0));
    double tau[12];
    for (int j = 0; j < 12; ++j) tau[j] = 0.0;
    const int64_t steps = m < k ? m : k;
    for (int64_t j = 0; j < steps; ++j) {
        double normx = 0, alpha = 0, v0 = 0;
        int skip = 0;
        if (lane == 0) {
            for (int64_t i = j; i < m; ++i) normx = __dadd_rn(normx, __dmul_rn(a_(i, j), a_(i, j)));
            normx = __dsqrt_rn(normx);
            skip = normx <= tol;
            if (!skip) {
                alpha = a_(j, j) >= 0 ? -normx : normx;
                v0 = __dsub_rn(a_(j, j), alpha);
            }
        }
        skip = __shfl_sync(mask, skip, base);
        if (skip) continue;  // tau[j] stays 0
        alpha = __shfl_sync(mask, alpha, base);
        v0 = __shfl_sync(mask, v0, base);
        tau[j] = __ddiv_rn(-v0, alpha);
        for (int64_t i = j + 1 + lane; i < m; i += kQrLanes) a_(i, j) = __ddiv_rn(a_(i, j), v0);
        __syncwarp(mask);
        if (lane == 0) a_(j, j) = alpha;
        const int c = lane;
        if (c > j && c < k) {
            double s = a_(j, c);
            for (int64_t i = j + 1; i < m; ++i) s = __dadd_rn(s, __dmul_rn(a_(i, j), a_(i, c)));
            s = __dmul_rn(s, tau[j]);
            a_(j, c) = __dsub_rn(a_(j, c), s);
            for (int64_t i = j + 1; i < m; ++i) a_(i, c) = __dsub_rn(a_(i, c), __dmul_rn(s, a_(i, j)));
        }
        __syncwarp(mask);
    }
    for (int t = lane; t < k * k; t += kQrLanes) {
        const int j = t / k, i = t - j * k;  // R[j*k + i] = a(i, j) for i <= min(j, m-1)
        R[t] = (i <= j && i < m) ? a_(i, j) : 0.0;
    }
    for (int64_t t = lane; t < m * k; t += kQrLanes) {
        const int64_t c = t / m, r = t - c * m;
        Q[t] = (r == c) ? 1.0 : 0.0;
    }
    __syncwarp(mask);
    for (int64_t j = steps - 1; j >= 0; --j) {
        if (tau[j] == 0) continue;
        const int c = lane;
        if (c < k) {
            double s = Q[c * m + j];
            for (int64_t i = j + 1; i < m; ++i) s = __dadd_rn(s, __dmul_rn(a_(i, j), Q[c * m + i]));
            s = __dmul_rn(s, tau[j]);
            Q[c * m + j] = __dsub_rn(Q[c * m + j], s);
            for (int64_t i = j + 1; i < m; ++i) Q[c * m + i] = __dsub_rn(Q[c * m + i], __dmul_rn(s, a_(i, j)));
        }
        __syncwarp(mask);
    }
    // rank-deficient columns (coarsening.hpp:222-228): lane j tests column j
    const double lm = fmax(local_max, 1e-300);
    const int j = lane;
    bool drop = false;
    if (j < k) {
        const double rjj = (j < m) ? fabs(R[j * k + j]) : 0.0;
        drop = rjj <= __dmul_rn(1e-12, lm);
    }
    __syncwarp(mask);
    if (drop) {
        for (int64_t i = 0; i < m; ++i) Q[j * m + i] = 0.0;
        for (int c = 0; c < k; ++c) R[c * k + j] = 0.0;
    }
    __syncwarp(mask);
    for (int64_t t = lane; t < m * k; t += kQrLanes) {
        const int64_t r = t / k, c = t - r * k;
        Pt[ROW(r) * k + c] = Q[c * m + r];
    }
    const int64_t bcn = naggs * k;
    for (int t = lane; t < k * k; t += kQrLanes) {
        const int c = t / k, i = t - c * k;
        Bc[c * bcn + a * k + i] = R[c * k + i];
    }
#undef a_
#undef ROW
}

// ---------------------------------------------------------------------------
// prolongator smoothing (coarsening.hpp:319-416) in the scalar semantics the
// ns_block wrapper uses (as_scalar_transfer, :451-464), emitted directly as
// 3x3 blocks (to_block<3> of the scalar P is exact: every node's scalar
// rows share one column set made of whole k-column aggregate groups).

__device__ __forceinline__ bool strong(const int *gp, const int *gc, int node, int cnode) {
    return bsearch_int(gc, gp[node], gp[node + 1], cnode);
}

// touched aggregates of each node: agg(node) + agg(c) for kept node columns
__global__ void k_psm_touch(int nnodes, int h, const int *ptr, const int *col, const int *gp,
                            const int *gc, const int *agg, const int *toff, int *tlist,
                            int *tcnt, int node0 = 0) {
    const int ln = blockIdx.x * blockDim.x + threadIdx.x;  // local node (lists)
    if (ln >= nnodes) return;
    const int node = node0 + ln;                           // global node
    int *L = tlist + toff[ln];
    int n = 0;
    L[n++] = agg[node];
    for (int r = 0; r < h; ++r) {
        const int br = node * h + r;
        for (int j = ptr[br]; j < ptr[br + 1]; ++j) {
            const int cn = col[j] / h;
            if (cn == node || strong(gp, gc, node, cn)) {
                const int g = agg[cn];
                int q = n;
                bool dup = false;
                for (int t = 0; t < n; ++t) if (L[t] == g) { dup = true; break; }
                if (dup) continue;
                // insertion keeping ascending order
                while (q > 0 && L[q - 1] > g) { L[q] = L[q - 1]; --q; }
                L[q] = g;
                ++n;
            }
        }
    }
    // the own aggregate was inserted first; restore ascending order
    for (int t = 1; t < n; ++t) {
        const int v = L[t];
        int q = t;
        while (q > 0 && L[q - 1] > v) { L[q] = L[q - 1]; --q; }
        L[q] = v;
    }
    tcnt[ln] = n;
}

__global__ void k_psm_cols(int nbrows, int h, int kb, const int *toff, const int *tlist,
                           const int *tcnt, const int *pptr, int *pcol) {
    const int br = blockIdx.x * blockDim.x + threadIdx.x;
    if (br >= nbrows) return;
    const int node = br / h;
    const int *L = tlist + toff[node];
    int o = pptr[br];
    for (int t = 0; t < tcnt[node]; ++t)
        for (int q = 0; q < kb; ++q) pcol[o++] = L[t] * kb + q;
}

// filtered scalar diagonal D_f (coarsening.hpp:335-358)
__global__ void k_psm_diag(int64_t nsc, int pbs, const int *ptr, const int *col,
                           const double *val, const int *gp, const int *gc, double *dinv,
                           double *diag, DevError *err, int64_t off = 0) {
    const int64_t li = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (li >= nsc) return;
    const int64_t i = li + off;  // global scalar row
    const int br = static_cast<int>(i / 3), rr = static_cast<int>(i % 3);
    const int node = static_cast<int>(i / pbs);
    double d = 0.0;
    for (int j = ptr[br]; j < ptr[br + 1]; ++j) {
        const int64_t sc0 = 3 * static_cast<int64_t>(col[j]);
        const int cn = static_cast<int>(sc0 / pbs);
        const bool same = cn == node;
        const bool st = same ? false : strong(gp, gc, node, cn);
        const double *b = val + 9 * static_cast<int64_t>(j) + 3 * rr;
        for (int c = 0; c < 3; ++c) {
            const int64_t sc = sc0 + c;
            if (same) {
                if (sc == i) d = __dadd_rn(d, b[c]);
            } else if (!st) {
                d = __dadd_rn(d, b[c]);
            }
        }
    }
    diag[li] = d;
    if (d == 0.0) { raise(err, SAMG_ZERO_DIAGONAL, i); dinv[li] = 0.0; return; }
    if (fabs(d) < 1e-300) { raise(err, SAMG_SINGULAR_BLOCK, i); dinv[li] = 0.0; return; }
    dinv[li] = __ddiv_rn(1.0, d);
}

// P row values: for each touched aggregate g, in ascending scalar column
// order over kept entries k with agg(node(k)) == g (coarsening.hpp:387-414)
__global__ void k_psm_vals(int64_t nsc, int pbs, int h, int k, const int *ptr, const int *col,
                           const double *val, const int *gp, const int *gc, const int *agg,
                           const int *toff, const int *tlist, const int *tcnt,
                           const double *dinv, const double *diag, const double *Pt,
                           double omega, const int *pptr, double *pval, int64_t off = 0) {
    const int64_t li = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (li >= nsc) return;
    const int64_t i = li + off;  // global scalar row
    const int br = static_cast<int>(i / 3), rr = static_cast<int>(i % 3);
    const int node = static_cast<int>(i / pbs);
    const int lnode = static_cast<int>(li / pbs), lbr = static_cast<int>(li / 3);
    const int kb = k / 3;
    const int *L = tlist + toff[lnode];
    const int nt = tcnt[lnode];
    const double di = dinv[li], dg = diag[li];
    const double nom = -omega;
    for (int t = 0; t < nt; ++t) {
        const int g = L[t];
        double acc[12];
        bool touched = agg[node] == g;
        if (touched)
            for (int c = 0; c < k; ++c) acc[c] = Pt[i * k + c];
        for (int j = ptr[br]; j < ptr[br + 1]; ++j) {
            const int64_t sc0 = 3 * static_cast<int64_t>(col[j]);
            const int cn = static_cast<int>(sc0 / pbs);
            if (agg[cn] != g) continue;
            if (cn != node && !strong(gp, gc, node, cn)) continue;
            const double *b = val + 9 * static_cast<int64_t>(j) + 3 * rr;
            for (int c3 = 0; c3 < 3; ++c3) {
                const int64_t sc = sc0 + c3;
                const double coef = (sc == i) ? dg : b[c3];
                const double scaled = __dmul_rn(__dmul_rn(di, coef), nom);
                const double *pk = Pt + sc * k;
                if (touched) {
                    for (int c = 0; c < k; ++c) acc[c] = __dadd_rn(acc[c], __dmul_rn(scaled, pk[c]));
                } else {
                    for (int c = 0; c < k; ++c) acc[c] = __dmul_rn(scaled, pk[c]);
                    touched = true;
                }
            }
        }
        const int64_t base = pptr[lbr] + static_cast<int64_t>(t) * kb;
        for (int c = 0; c < k; ++c) pval[9 * (base + c / 3) + 3 * rr + c % 3] = acc[c];
    }
}

// The same values with a thread per BLOCK row (its three scalar rows share
// the node, the candidate groups, the row's blocks, the strength tests and
// every P_tent row they read): each scalar row's accumulator sees exactly
// the terms of k_psm_vals in the same order -- one third of the index work
// and of the P_tent gathers.  K = the nullspace width (6 for the ns
// pipelines).
template <int K>
__global__ void __launch_bounds__(128) k_psm_vals3(int64_t nbr, int pbs, const int *ptr, const int *col,
        const double *val, const int *gp, const int *gc, const int *agg, const int *toff,
        const int *tlist, const int *tcnt, const double *dinv, const double *diag, const double *Pt,
        double omega, const int *pptr, double *pval, int64_t off) {
    const int64_t lb = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (lb >= nbr) return;
    const int64_t li0 = 3 * lb, i0 = li0 + off;
    const int br = static_cast<int>(i0 / 3);
    const int node = static_cast<int>(i0 / pbs);
    const int lnode = static_cast<int>(li0 / pbs);
    constexpr int kb = K / 3;
    const int *L = tlist + toff[lnode];
    const int nt = tcnt[lnode];
    double di[3], dg[3];
#pragma unroll
    for (int rr = 0; rr < 3; ++rr) { di[rr] = dinv[li0 + rr]; dg[rr] = diag[li0 + rr]; }
    const double nom = -omega;
    const int jb = ptr[br], je = ptr[br + 1];
    const int ownagg = agg[node];
    for (int t = 0; t < nt; ++t) {
        const int g = L[t];
        double acc[3][K];
        bool touched = ownagg == g;  // the same for the three rows throughout
        if (touched) {
#pragma unroll
            for (int rr = 0; rr < 3; ++rr)
#pragma unroll
                for (int c = 0; c < K; ++c) acc[rr][c] = Pt[(i0 + rr) * K + c];
        }
        for (int j = jb; j < je; ++j) {
            const int64_t sc0 = 3 * static_cast<int64_t>(col[j]);
            const int cn = static_cast<int>(sc0 / pbs);
            if (agg[cn] != g) continue;
            if (cn != node && !strong(gp, gc, node, cn)) continue;
            const double *b = val + 9 * static_cast<int64_t>(j);
#pragma unroll
            for (int c3 = 0; c3 < 3; ++c3) {
                const int64_t sc = sc0 + c3;
                double pk[K];
#pragma unroll
                for (int c = 0; c < K; ++c) pk[c] = Pt[sc * K + c];
#pragma unroll
                for (int rr = 0; rr < 3; ++rr) {
                    const double coef = (sc == i0 + rr) ? dg[rr] : b[3 * rr + c3];
                    const double scaled = __dmul_rn(__dmul_rn(di[rr], coef), nom);
                    if (touched) {
#pragma unroll
                        for (int c = 0; c < K; ++c) acc[rr][c] = __dadd_rn(acc[rr][c], __dmul_rn(scaled, pk[c]));
                    } else {
#pragma unroll
                        for (int c = 0; c < K; ++c) acc[rr][c] = __dmul_rn(scaled, pk[c]);
                    }
                }
                touched = true;
            }
        }
        const int64_t base = pptr[lb] + static_cast<int64_t>(t) * kb;
#pragma unroll
        for (int rr = 0; rr < 3; ++rr)
#pragma unroll
            for (int c = 0; c < K; ++c) pval[9 * (base + c / 3) + 3 * rr + c % 3] = acc[rr][c];
    }
}

bool psm_block_rows() {  // SAMG_PSM_BLOCKROW=0 selects the thread-per-scalar-row kernel
    static const bool on = [] {
        const char *e = std::getenv("SAMG_PSM_BLOCKROW");
        return !(e && e[0] == '0');
    }();
    return on;
}

// The `scalar` pipeline's tentative operator has no nullspace: the unit
// aggregate indicator expanded per point-block component
// (coarsening.hpp:249-266), one entry per scalar row -- P_tent(i, agg(i)*3 +
// i%3) = 1/sqrt(|aggregate|), Pt1[i] holds it.  The smoothing then follows
// coarsening.hpp:387-414 with a first touch per column: scalar column sc of
// A's row contributes only to column comp(sc) of the aggregate group.
__global__ void k_tent_indicator(int64_t nnodes, int pbs, const int *agg, const int *cnt,
                                 double *Pt1) {
    const int64_t n = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (n >= nnodes) return;
    const double v = __ddiv_rn(1.0, __dsqrt_rn(static_cast<double>(cnt[agg[n]])));
    for (int c = 0; c < pbs; ++c) Pt1[n * pbs + c] = v;
}

__global__ void k_psm_vals_ind(int64_t nsc, int pbs, int h, const int *ptr, const int *col,
                               const double *val, const int *gp, const int *gc, const int *agg,
                               const int *toff, const int *tlist, const int *tcnt,
                               const double *dinv, const double *diag, const double *Pt1,
                               double omega, const int *pptr, double *pval, int64_t off) {
    const int64_t li = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (li >= nsc) return;
    const int64_t i = li + off;
    const int br = static_cast<int>(i / 3), rr = static_cast<int>(i % 3);
    const int node = static_cast<int>(i / pbs);
    const int lnode = static_cast<int>(li / pbs), lbr = static_cast<int>(li / 3);
    const int *L = tlist + toff[lnode];
    const int nt = tcnt[lnode];
    const double di = dinv[li], dg = diag[li];
    const double nom = -omega;
    for (int t = 0; t < nt; ++t) {
        const int g = L[t];
        double acc[3] = {0.0, 0.0, 0.0};
        bool touched[3] = {false, false, false};
        if (agg[node] == g) {  // P_tent's own entry first
            const int c = static_cast<int>(i % pbs);
            acc[c] = Pt1[i];
            touched[c] = true;
        }
        for (int j = ptr[br]; j < ptr[br + 1]; ++j) {
            const int64_t sc0 = 3 * static_cast<int64_t>(col[j]);
            const int cn = static_cast<int>(sc0 / pbs);
            if (agg[cn] != g) continue;
            if (cn != node && !strong(gp, gc, node, cn)) continue;
            const double *b = val + 9 * static_cast<int64_t>(j) + 3 * rr;
            for (int c3 = 0; c3 < 3; ++c3) {
                const int64_t sc = sc0 + c3;
                const double coef = (sc == i) ? dg : b[c3];
                const double scaled = __dmul_rn(__dmul_rn(di, coef), nom);
                const int c = static_cast<int>(sc % pbs);
                const double pr = __dmul_rn(scaled, Pt1[sc]);
                if (touched[c]) acc[c] = __dadd_rn(acc[c], pr);
                else { acc[c] = pr; touched[c] = true; }
            }
        }
        const int64_t base = pptr[lbr] + t;  // one 3x3 block per touched aggregate
        for (int c = 0; c < 3; ++c) pval[9 * base + 3 * rr + c] = acc[c];
    }
}

// ---------------------------------------------------------------------------
// block pipeline transfer (block_transfer_operators, coarsening.hpp:471-560).
// Tentative: block v_g * I for node i in aggregate g, v_g = 1/sqrt(|g|).
// Filtered diagonal D_i = sum, in row order, of the diagonal block and every
// weak off-diagonal block; P row i = the tentative entry first, then for each
// kept entry k (diagonal or strong) in row order the block
// ((D_i^-1 * coef) * -omega) * Ptent_k, where coef = D_i on the diagonal;
// the first contribution to a column assigns, later ones add.

__global__ void k_bt_count(int n, const int *agg, int *cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicAdd(cnt + agg[i], 1);
}

__global__ void k_bt_scale(int naggs, const int *cnt, double *pv) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < naggs) pv[g] = __ddiv_rn(1.0, __dsqrt_rn(static_cast<double>(cnt[g])));
}

__device__ __forceinline__ void bt_tent(double v, double *t) {
    for (int e = 0; e < 9; ++e) t[e] = __dmul_rn(v, (e % 4 == 0) ? 1.0 : 0.0);
}

// omega == 0: P = P_tent
__global__ void k_bt_tent(int n, const int *agg, const double *pv, int *pptr, int *pcol,
                          double *pval, int row0 = 0) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // local row
    if (i > n) return;
    pptr[i] = i;
    if (i == n) return;
    const int g = agg[row0 + i];
    pcol[i] = g;
    bt_tent(pv[g], pval + 9 * static_cast<int64_t>(i));
}

// lumped filtered diagonal and its inverse, a thread per block row
__global__ void k_bt_diag(int n, const int *ptr, const int *col, const double *val,
                          const int *gp, const int *gc, double *dg, double *dinv, DevError *err,
                          int row0 = 0) {
    const int li = blockIdx.x * blockDim.x + threadIdx.x;  // local row (dg / dinv)
    if (li >= n) return;
    const int i = row0 + li;                                 // global row
    double d[9];
    for (int e = 0; e < 9; ++e) d[e] = 0.0;
    for (int j = ptr[i]; j < ptr[i + 1]; ++j) {
        const int c = col[j];
        if (c != i && strong(gp, gc, i, c)) continue;
        const double *b = val + 9 * static_cast<int64_t>(j);
        for (int e = 0; e < 9; ++e) d[e] = __dadd_rn(d[e], b[e]);
    }
    bool zero = true;
    for (int e = 0; e < 9; ++e) {
        dg[9 * static_cast<int64_t>(li) + e] = d[e];
        if (d[e] != 0.0) zero = false;
    }
    double inv[9];
    if (zero) { raise(err, SAMG_ZERO_DIAGONAL, i); return; }
    if (!blk_inverse_ref(d, inv)) { raise(err, SAMG_SINGULAR_BLOCK, i); return; }
    for (int e = 0; e < 9; ++e) dinv[9 * static_cast<int64_t>(li) + e] = inv[e];
}

// one thread per P entry (row i, aggregate column g)
__global__ void k_bt_vals(int64_t nnzb, int n, const int *ptr, const int *col, const double *val,
                          const int *gp, const int *gc, const int *agg, const double *pv,
                          const double *dg, const double *dinv, double omega, const int *pptr,
                          const int *pcol, double *pval, int row0 = 0) {
    const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= nnzb) return;
    const int li = lower_bound_int(pptr, n + 1, static_cast<int>(e) + 1) - 1;  // local row
    const int i = row0 + li;                                                   // global row
    const int g = pcol[e];
    double acc[9], inv[9];
    bool touched = agg[i] == g;
    if (touched) bt_tent(pv[g], acc);
    for (int q = 0; q < 9; ++q) inv[q] = dinv[9 * static_cast<int64_t>(li) + q];
    const double nom = -omega;
    for (int j = ptr[i]; j < ptr[i + 1]; ++j) {
        const int k = col[j];
        if (agg[k] != g) continue;
        if (k != i && !strong(gp, gc, i, k)) continue;
        const double *coef = k == i ? dg + 9 * static_cast<int64_t>(li) : val + 9 * static_cast<int64_t>(j);
        double sc[9], t[9], prod[9];
        blk_mul_ref(inv, coef, sc);
        for (int q = 0; q < 9; ++q) sc[q] = __dmul_rn(sc[q], nom);
        bt_tent(pv[g], t);
        blk_mul_ref(sc, t, prod);
        if (touched) {
            for (int q = 0; q < 9; ++q) acc[q] = __dadd_rn(acc[q], prod[q]);
        } else {
            for (int q = 0; q < 9; ++q) acc[q] = prod[q];
            touched = true;
        }
    }
    for (int q = 0; q < 9; ++q) pval[9 * e + q] = acc[q];
}

// omega == 0: P is the tentative operator (coarsening.hpp:326)
__global__ void k_ptent_bsr(int nbrows, int h, int k, const int *agg, const double *Pt,
                            int *pptr, int *pcol, double *pval, int row0 = 0) {
    const int br = blockIdx.x * blockDim.x + threadIdx.x;  // local block row
    if (br > nbrows) return;
    const int kb = k / 3;
    pptr[br] = br * kb;
    if (br == nbrows) return;
    const int gb = row0 + br;  // global block row
    const int g = agg[gb / h];
    for (int q = 0; q < kb; ++q) {
        pcol[br * kb + q] = g * kb + q;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c)
                pval[9 * (static_cast<int64_t>(br) * kb + q) + 3 * r + c] =
                    Pt[(3 * static_cast<int64_t>(gb) + r) * k + 3 * q + c];
    }
}

// omega == 0 with the indicator tentative (the `scalar` pipeline; the
// reference's own known-answer case, test_coarsening.cpp:172-180): scalar row
// i holds the single entry P_tent(i, 3 agg(i/3) + i%3) = Pt1[i], i.e. block
// row br is one diagonal 3x3 block in column agg(br)
__global__ void k_ptent_ind_bsr(int nbrows, const int *agg, const double *Pt1, int *pptr,
                                int *pcol, double *pval, int row0) {
    const int br = blockIdx.x * blockDim.x + threadIdx.x;  // local block row
    if (br > nbrows) return;
    pptr[br] = br;
    if (br == nbrows) return;
    const int gb = row0 + br;  // global block row = node (point block size 3)
    pcol[br] = agg[gb];
    double *b = pval + 9 * static_cast<int64_t>(br);
    for (int e = 0; e < 9; ++e) b[e] = 0.0;
    for (int c = 0; c < 3; ++c) b[4 * c] = Pt1[3 * static_cast<int64_t>(gb) + c];
}

// ---------------------------------------------------------------------------
// SpGEMM C = A*B (csr.hpp:199-255).  One CTA per output row; a hash set of
// the row's columns lives in shared memory (or a global scratch slab for
// oversized rows).  Numeric phase: columns are sorted (bitonic), slots
// zeroed, then A's row entries are consumed in ascending order with a CTA
// barrier between them, so every output block receives its products in
// exactly the reference's (ja ascending) order.

__device__ __forceinline__ unsigned hash_u(int key) {
    unsigned x = static_cast<unsigned>(key);
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// returns slot index; inserts if absent; -1 if the table is full
__device__ __forceinline__ int hash_insert(int *keys, int cap, int key, bool &inserted) {
    unsigned h = hash_u(key) & (cap - 1);
    for (int probe = 0; probe < cap; ++probe) {
        const int cur = keys[h];
        if (cur == key) { inserted = false; return static_cast<int>(h); }
        if (cur == -1) {
            const int prev = atomicCAS(keys + h, -1, key);
            if (prev == -1) { inserted = true; return static_cast<int>(h); }
            if (prev == key) { inserted = false; return static_cast<int>(h); }
        }
        h = (h + 1) & (cap - 1);
    }
    inserted = false;
    return -1;
}

__device__ __forceinline__ int hash_find(const int *keys, int cap, int key) {
    unsigned h = hash_u(key) & (cap - 1);
    for (int probe = 0; probe < cap; ++probe) {
        const int cur = keys[h];
        if (cur == key) return static_cast<int>(h);
        if (cur == -1) return -1;
        h = (h + 1) & (cap - 1);
    }
    return -1;
}

// symbolic: count distinct columns per row.  GLOBAL: table in scratch.
template <bool GLOBAL>
__global__ void k_spgemm_count(int nrows, const int *rows, const int *ap, const int *ac,
                               const int *bp, const int *bc, int cap, int *keys_g,
                               const int64_t *goff, int *cnt, int *overflow) {
    extern __shared__ int smem[];
    const int ridx = blockIdx.x;
    if (ridx >= nrows) return;
    const int row = rows ? rows[ridx] : ridx;
    int *keys = GLOBAL ? keys_g + goff[ridx] : smem;
    const int tcap = GLOBAL ? static_cast<int>(goff[ridx + 1] - goff[ridx]) : cap;
    __shared__ int n_s, full_s;
    for (int t = threadIdx.x; t < tcap; t += blockDim.x) keys[t] = -1;
    if (threadIdx.x == 0) { n_s = 0; full_s = 0; }
    __syncthreads();
    const int limit = tcap / 2;
    for (int ja = ap[row]; ja < ap[row + 1]; ++ja) {
        const int kk = ac[ja];
        for (int jb = bp[kk] + threadIdx.x; jb < bp[kk + 1]; jb += blockDim.x) {
            if (full_s) break;
            bool ins;
            const int slot = hash_insert(keys, tcap, bc[jb], ins);
            if (slot < 0) { full_s = 1; break; }
            if (ins && atomicAdd(&n_s, 1) + 1 > limit - 1) full_s = 1;
        }
        if (full_s) break;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (full_s) { cnt[row] = -1; atomicAdd(overflow, 1); }
        else cnt[row] = n_s;
    }
}

template <bool GLOBAL, bool kScalar, bool kCols = false>
__global__ void __launch_bounds__(256) k_spgemm_numeric(
        int nrows, const int *rows, const int *ap, const int *ac, const double *av,
        const int *bp, const int *bc, const double *bv, int cap, int *keys_g, int *vals_g,
        int *list_g, const int64_t *goff, const int *cp, int *ccol, double *cval) {
    extern __shared__ int smem[];
    const int ridx = blockIdx.x;
    if (ridx >= nrows) return;
    const int row = rows ? rows[ridx] : ridx;
    const int tcap = GLOBAL ? static_cast<int>(goff[ridx + 1] - goff[ridx]) : cap;
    int *keys = GLOBAL ? keys_g + goff[ridx] : smem;
    int *vals = GLOBAL ? vals_g + goff[ridx] : smem + cap;
    int *list = GLOBAL ? list_g + goff[ridx] / 2 : smem + 2 * cap;
    const int lcap = tcap / 2;
    // rows too wide for the shared table are done by the GLOBAL instance
    if (!GLOBAL && cp[row + 1] - cp[row] > lcap - 1) return;
    __shared__ int n_s;
    for (int t = threadIdx.x; t < tcap; t += blockDim.x) keys[t] = -1;
    if (threadIdx.x == 0) n_s = 0;
    __syncthreads();
    for (int ja = ap[row]; ja < ap[row + 1]; ++ja) {
        const int kk = ac[ja];
        for (int jb = bp[kk] + threadIdx.x; jb < bp[kk + 1]; jb += blockDim.x) {
            bool ins;
            hash_insert(keys, tcap, bc[jb], ins);
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < tcap; t += blockDim.x)
        if (keys[t] != -1) list[atomicAdd(&n_s, 1)] = keys[t];
    __syncthreads();
    const int n = n_s;
    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (int t = n + threadIdx.x; t < np2 && t < lcap; t += blockDim.x) list[t] = INF;
    __syncthreads();
    // bitonic sort of list[0..np2)
    for (int size = 2; size <= np2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < np2; t += blockDim.x) {
                const int partner = t ^ stride;
                if (partner > t) {
                    const bool up = (t & size) == 0;
                    const int a = list[t], b = list[partner];
                    if ((a > b) == up) { list[t] = b; list[partner] = a; }
                }
            }
            __syncthreads();
        }
    const int64_t base = cp[row];
    if constexpr (kCols) {  // pattern only: values come from k_spgemm_pull
        for (int t = threadIdx.x; t < n; t += blockDim.x) ccol[base + t] = list[t];
        return;
    }
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const int key = list[t];
        ccol[base + t] = key;
        vals[hash_find(keys, tcap, key)] = t;
        double *cb = cval + 9 * (base + t);
        for (int e = 0; e < 9; ++e) cb[e] = 0.0;
    }
    __syncthreads();
    for (int ja = ap[row]; ja < ap[row + 1]; ++ja) {
        const int kk = ac[ja];
        const double *a = av + 9 * static_cast<int64_t>(ja);
        double am[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) am[e] = a[e];
        for (int jb = bp[kk] + threadIdx.x; jb < bp[kk + 1]; jb += blockDim.x) {
            const int slot = vals[hash_find(keys, tcap, bc[jb])];
            accum_block<kScalar>(am, bv + 9 * static_cast<int64_t>(jb), cval + 9 * (base + slot));
        }
        __syncthreads();
    }
}

// Warp-per-row variants (8 rows per CTA) for rows with at most kWCap/2-1
// distinct columns: same hash, same bitonic sort, same in-order
// accumulation, __syncwarp instead of the CTA barrier, so 8 rows progress
// concurrently.  Results are bit-identical to the CTA kernels.
constexpr int kWCap = 1024;
constexpr int kWPB = 8;

__global__ void __launch_bounds__(256) k_spgemm_wcount(int nrows, const int *rows, const int *ap,
                                                       const int *ac, const int *bp, const int *bc,
                                                       int *cnt) {
    __shared__ int keys_all[kWPB][kWCap];
    __shared__ int n_all[kWPB];
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int ridx = blockIdx.x * kWPB + w;
    if (ridx >= nrows) return;  // whole warp
    const int row = rows ? rows[ridx] : ridx;
    int *keys = keys_all[w];
    for (int t = lane; t < kWCap; t += 32) keys[t] = -1;
    if (lane == 0) n_all[w] = 0;
    __syncwarp();
    bool full = false;
    for (int ja = ap[row]; ja < ap[row + 1]; ++ja) {
        const int kk = ac[ja];
        for (int jb = bp[kk] + lane; jb < bp[kk + 1] && !full; jb += 32) {
            bool ins;
            const int slot = hash_insert(keys, kWCap, bc[jb], ins);
            if (slot < 0 || (ins && atomicAdd(n_all + w, 1) + 1 > kWCap / 2 - 1)) full = true;
        }
        if (__any_sync(0xffffffffu, full)) { full = true; break; }
    }
    __syncwarp();
    if (lane == 0) cnt[row] = full ? -1 : n_all[w];
}

template <bool kScalar, bool kCols = false>
__global__ void __launch_bounds__(256) k_spgemm_wnumeric(
        int nrows, const int *ap, const int *ac, const double *av, const int *bp, const int *bc,
        const double *bv, const int *cp, const int *mode, int *ccol, double *cval) {
    extern __shared__ int wsm[];
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int row = blockIdx.x * kWPB + w;
    if (row >= nrows || mode[row]) return;  // bitmap rows: k_spgemm_bnumeric
    const int n = cp[row + 1] - cp[row];
    if (n > kWCap / 2 - 1) return;  // wide row: CTA kernel
    int *keys = wsm + w * (kWCap * 5 / 2);
    int *vals = keys + kWCap;
    int *list = vals + kWCap;
    for (int t = lane; t < kWCap; t += 32) keys[t] = -1;
    __syncwarp();
    for (int ja = ap[row]; ja < ap[row + 1]; ++ja) {
        const int kk = ac[ja];
        for (int jb = bp[kk] + lane; jb < bp[kk + 1]; jb += 32) {
            bool ins;
            hash_insert(keys, kWCap, bc[jb], ins);
        }
    }
    __syncwarp();
    // deterministic compaction: ballot over the table in slot order
    int out = 0;
    for (int t0 = 0; t0 < kWCap; t0 += 32) {
        const int key = keys[t0 + lane];
        const unsigned m = __ballot_sync(0xffffffffu, key != -1);
        if (key != -1) list[out + __popc(m & ((1u << lane) - 1u))] = key;
        out += __popc(m);
    }
    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (int t = n + lane; t < np2; t += 32) list[t] = INF;
    __syncwarp();
    for (int size = 2; size <= np2; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = lane; t < np2; t += 32) {
                const int partner = t ^ stride;
                if (partner > t) {
                    const bool up = (t & size) == 0;
                    const int a = list[t], b = list[partner];
                    if ((a > b) == up) { list[t] = b; list[partner] = a; }
                }
            }
            __syncwarp();
        }
    const int64_t base = cp[row];
    if constexpr (kCols) {  // pattern only: values come from k_spgemm_pull
        for (int t = lane; t < n; t += 32) ccol[base + t] = list[t];
        return;
    }
    for (int t = lane; t < n; t += 32) {
        const int key = list[t];
        ccol[base + t] = key;
        vals[hash_find(keys, kWCap, key)] = t;
        double *cb = cval + 9 * (base + t);
        for (int e = 0; e < 9; ++e) cb[e] = 0.0;
    }
    __syncwarp();
    // In-order accumulation.  The operands of step ja+1 (A block, this lane's
    // first B entry and its column) are loaded while step ja accumulates, so
    // the L2 latency is off the sequential chain; B rows longer than 32
    // entries finish their extra chunks unpipelined in the same step.
    const int ja0 = ap[row], jend = ap[row + 1];
    double am[9], bm[9];
    int cc = -1, jbc = -1, kend = 0;
    auto fetch = [&](int ja, double *a_, double *b_, int &c_, int &jb_, int &kend_) {
        const int kk = ac[ja];
        const double *a = av + 9 * static_cast<int64_t>(ja);
#pragma unroll
        for (int e = 0; e < 9; ++e) a_[e] = a[e];
        jb_ = bp[kk] + lane;
        kend_ = bp[kk + 1];
        c_ = -1;
        if (jb_ < kend_) {
            c_ = bc[jb_];
            const double *b = bv + 9 * static_cast<int64_t>(jb_);
#pragma unroll
            for (int e = 0; e < 9; ++e) b_[e] = b[e];
        }
    };
    if (ja0 < jend) fetch(ja0, am, bm, cc, jbc, kend);
    for (int ja = ja0; ja < jend; ++ja) {
        double an[9], bn[9];
        int cn = -1, jbn = -1, kendn = 0;
        if (ja + 1 < jend) fetch(ja + 1, an, bn, cn, jbn, kendn);
        if (cc >= 0) {
            const int slot = vals[hash_find(keys, kWCap, cc)];
            accum_block<kScalar>(am, bm, cval + 9 * (base + slot));
            for (int jb = jbc + 32; jb < kend; jb += 32) {
                const int sl = vals[hash_find(keys, kWCap, bc[jb])];
                accum_block<kScalar>(am, bv + 9 * static_cast<int64_t>(jb), cval + 9 * (base + sl));
            }
        }
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 9; ++e) { am[e] = an[e]; bm[e] = bn[e]; }
        cc = cn;
        jbc = jbn;
        kend = kendn;
    }
}

// ---------------------------------------------------------------------------
// Window-bitmap SpGEMM (warp per row) for rows whose output columns span a
// window of at most kWinMax columns -- every row of the AMG Galerkin
// products on mesh matrices.  The row's column set is a bitmap over
// [cmin, cmin + W) in shared memory; a per-word prefix popcount gives both
// the sorted column list (no hashing, no sort) and every product's output
// slot (one popcount).  Products are accumulated in the reference's ja order
// into shared memory when the row has <= acc_cap columns (global memory
// otherwise).  Results are bit-identical to the hash kernels.
constexpr int kWinMax = 32768;   // columns of the widest window (bits)
constexpr int kBWPB = 8;         // warps (rows) per CTA

// [cmin, cmax] of row i's products: B rows are column-sorted, so their first
// and last entries bound them.  Empty row: cmin > cmax.
__device__ __forceinline__ void row_window(int i, const int *__restrict__ ap, const int *__restrict__ ac,
                                           const int *__restrict__ bp, const int *__restrict__ bc,
                                           int &cmin, int &cmax) {
    const int lane = threadIdx.x & 31;
    int lo = INT_MAX, hi = -1;
    for (int ja = ap[i] + lane; ja < ap[i + 1]; ja += 32) {
        const int kk = ac[ja], b0 = bp[kk], b1 = bp[kk + 1];
        if (b1 > b0) { lo = min(lo, bc[b0]); hi = max(hi, bc[b1 - 1]); }
    }
    cmin = static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(lo)));
    cmax = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(hi + 1))) - 1;
}

// set the bits of row i's product columns; returns the column count
__device__ int row_bitmap(int i, const int *__restrict__ ap, const int *__restrict__ ac,
                          const int *__restrict__ bp, const int *__restrict__ bc, int cmin,
                          int words, unsigned *bm) {
    const int lane = threadIdx.x & 31;
    for (int w = lane; w < words; w += 32) bm[w] = 0u;
    __syncwarp();
    for (int ja = ap[i]; ja < ap[i + 1]; ++ja) {
        const int kk = ac[ja];
        for (int jb = bp[kk] + lane; jb < bp[kk + 1]; jb += 32) {
            const int c = bc[jb] - cmin;
            atomicOr(bm + (c >> 5), 1u << (c & 31));
        }
    }
    __syncwarp();
    int cnt = 0;
    for (int w = lane; w < words; w += 32) cnt += __popc(bm[w]);
    return __reduce_add_sync(0xffffffffu, cnt);
}

// symbolic pass: count = distinct columns, or -2 when the window is too wide
__global__ void __launch_bounds__(kBWPB * 32) k_spgemm_bcount(int nrows, const int *ap, const int *ac,
        const int *bp, const int *bc, int win_limit, int *cnt, int *win_lo, int *maxwin) {
    __shared__ unsigned bm_all[kBWPB][kWinMax / 32];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * kBWPB + w;
    if (row >= nrows) return;
    int cmin, cmax;
    row_window(row, ap, ac, bp, bc, cmin, cmax);
    if (cmax < cmin) {  // empty row
        if (lane == 0) { cnt[row] = 0; win_lo[row] = 0; }
        return;
    }
    const int width = cmax - cmin + 1;
    if (width > win_limit) {
        if (lane == 0) cnt[row] = -2;
        return;
    }
    const int c = row_bitmap(row, ap, ac, bp, bc, cmin, (width + 31) >> 5, bm_all[w]);
    if (lane == 0) {
        cnt[row] = c;
        win_lo[row] = cmin;
        atomicMax(maxwin, width);
    }
}

// numeric pass for the bitmap rows (cnt >= 0 from k_spgemm_bcount; rows
// marked -2 there are skipped here, the hash kernels do them)
template <bool kScalar, bool kCols = false>
__global__ void __launch_bounds__(kBWPB * 32) k_spgemm_bnumeric(int nrows, const int *ap,
        const int *ac, const double *av, const int *bp, const int *bc, const double *bv,
        const int *cp, const int *mode, const int *win_lo, int words, int acc_cap, int *ccol,
        double *cval) {
    extern __shared__ __align__(16) unsigned char bsm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = blockIdx.x * kBWPB + w;
    if (row >= nrows || mode[row] != 1) return;
    const size_t per = (2 * static_cast<size_t>(words) * 4 + 15) / 16 * 16 + static_cast<size_t>(acc_cap) * 72;
    unsigned *bm = reinterpret_cast<unsigned *>(bsm + w * per);
    int *pre = reinterpret_cast<int *>(bm + words);
    double *acc_s = reinterpret_cast<double *>(bsm + w * per + (2 * static_cast<size_t>(words) * 4 + 15) / 16 * 16);
    const int cmin = win_lo[row];
    const int64_t base = cp[row];
    const int n = cp[row + 1] - cp[row];
    if (n == 0) return;
    row_bitmap(row, ap, ac, bp, bc, cmin, words, bm);
    // exclusive prefix of the word popcounts: lane l owns words [l*wpl, (l+1)*wpl)
    const int wpl = (words + 31) / 32;
    int mine = 0;
    for (int t = 0; t < wpl; ++t) {
        const int wd = lane * wpl + t;
        if (wd < words) mine += __popc(bm[wd]);
    }
    int incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
    }
    int run = incl - mine;
    for (int t = 0; t < wpl; ++t) {
        const int wd = lane * wpl + t;
        if (wd >= words) break;
        unsigned bits = bm[wd];
        pre[wd] = run;
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            ccol[base + run++] = cmin + (wd << 5) + b;
        }
    }
    if constexpr (kCols) return;  // pattern only: values come from k_spgemm_pull
    const bool in_smem = n <= acc_cap;
    double *acc = in_smem ? acc_s : cval + 9 * base;
    for (int e = lane; e < 9 * n; e += 32) acc[e] = 0.0;
    __syncwarp();
    auto slot_of = [&](int col) {
        const int c = col - cmin, wd = c >> 5, b = c & 31;
        return pre[wd] + __popc(bm[wd] & ((1u << b) - 1u));
    };
    // in-order accumulation; operands of step ja+1 fetched during step ja
    const int ja0 = ap[row], jend = ap[row + 1];
    double am[9], bmx[9];
    int cc = -1, jbc = -1, kend = 0;
    auto fetch = [&](int ja, double *a_, double *b_, int &c_, int &jb_, int &kend_) {
        const int kk = ac[ja];
        const double *a = av + 9 * static_cast<int64_t>(ja);
#pragma unroll
        for (int e = 0; e < 9; ++e) a_[e] = a[e];
        jb_ = bp[kk] + lane;
        kend_ = bp[kk + 1];
        c_ = -1;
        if (jb_ < kend_) {
            c_ = bc[jb_];
            const double *b = bv + 9 * static_cast<int64_t>(jb_);
#pragma unroll
            for (int e = 0; e < 9; ++e) b_[e] = b[e];
        }
    };
    if (ja0 < jend) fetch(ja0, am, bmx, cc, jbc, kend);
    for (int ja = ja0; ja < jend; ++ja) {
        double an[9], bn[9];
        int cn = -1, jbn = -1, kendn = 0;
        if (ja + 1 < jend) fetch(ja + 1, an, bn, cn, jbn, kendn);
        if (cc >= 0) {
            accum_block<kScalar>(am, bmx, acc + 9 * slot_of(cc));
            for (int jb = jbc + 32; jb < kend; jb += 32)
                accum_block<kScalar>(am, bv + 9 * static_cast<int64_t>(jb), acc + 9 * slot_of(bc[jb]));
        }
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 9; ++e) { am[e] = an[e]; bmx[e] = bn[e]; }
        cc = cn;
        jbc = jbn;
        kend = kendn;
    }
    if (in_smem)
        for (int e = lane; e < 9 * n; e += 32) cval[9 * base + e] = acc_s[e];
}

// ---------------------------------------------------------------------------
// Pull (inner-product) numeric pass over a known output pattern.  Output
// block (i, c) = sum over the entries of B's column c in ascending row j of
// A(i, j) * B(j, c), restricted to the j present in A's row i.  The reference
// accumulates (i, c) over A's row entries in ascending column order
// (csr.hpp:231-243), i.e. ascending j as well, so every output block gets
// the same terms in the same order as in the row-by-row (push) kernels --
// bit-identical -- but no output depends on another: no in-order chain along
// the row, no shared or global accumulators, every thread owns its outputs.
// A's row i is a shared-memory hash (column -> position); B's columns come
// from BCols (A itself for a structurally symmetric level matrix, through the
// transpose positions; R = P^T for P, through its block transposes).
struct BCols {
    const int *cp = nullptr, *ri = nullptr, *pos = nullptr;
    const double *val = nullptr;
    bool tr = false;  // stored block is B(j, c)^T (R's blocks for P)
};

template <bool kScalar, bool kTr, int NT, int BATCH>
__global__ void __launch_bounds__(NT) k_spgemm_pull(int nrows, int tcap, const int *__restrict__ ap,
        const int *__restrict__ ac, const double *__restrict__ av, BCols bc,
        const int *__restrict__ mode, const int *__restrict__ cp, const int *__restrict__ ccol,
        double *__restrict__ cval) {
    extern __shared__ int psm[];
    int *keys = psm, *vals = psm + tcap;
    const int row = blockIdx.x;
    if (row >= nrows || mode[row] == 2) return;  // 2: global-table rows (k_spgemm_numeric<true>)
    const int64_t base = cp[row];
    const int n = cp[row + 1] - cp[row];
    if (n == 0) return;
    for (int t = threadIdx.x; t < tcap; t += NT) keys[t] = -1;
    __syncthreads();
    const int a0 = ap[row], na = ap[row + 1] - a0;
    for (int t = threadIdx.x; t < na; t += NT) {
        bool ins;
        const int slot = hash_insert(keys, tcap, ac[a0 + t], ins);
        vals[slot] = t;
    }
    __syncthreads();
    const int *__restrict__ bcp = bc.cp;
    const int *__restrict__ bri = bc.ri;
    const int *__restrict__ bpos = bc.pos;
    const double *__restrict__ bval = bc.val;
    for (int t = threadIdx.x; t < n; t += NT) {
        const int c = ccol[base + t];
        double acc[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) acc[e] = 0.0;
        const int e1 = bcp[c + 1];
        // batches of BATCH column entries: the index loads, then the B blocks
        // of the hits are issued together (memory-level parallelism), then
        // the hits are accumulated in ascending row order
        for (int e = bcp[c]; e < e1; e += BATCH) {
            int ja[BATCH], qq[BATCH];
#pragma unroll
            for (int u = 0; u < BATCH; ++u) {
                const int ee = e + u;
                const bool in = ee < e1;
                const int j = in ? bri[ee] : -1;
                qq[u] = in ? (bpos ? bpos[ee] : ee) : 0;
                ja[u] = j;
            }
#pragma unroll
            for (int u = 0; u < BATCH; ++u) {
                const int slot = ja[u] >= 0 ? hash_find(keys, tcap, ja[u]) : -1;
                ja[u] = slot >= 0 ? vals[slot] : -1;
            }
            double bm[BATCH][9];
#pragma unroll
            for (int u = 0; u < BATCH; ++u)
                if (ja[u] >= 0) {
                    const double *b = bval + 9 * static_cast<int64_t>(qq[u]);
#pragma unroll
                    for (int q = 0; q < 9; ++q) bm[u][q] = b[q];
                }
#pragma unroll
            for (int u = 0; u < BATCH; ++u)
                if (ja[u] >= 0) {
                    const double *a = av + 9 * static_cast<int64_t>(a0 + ja[u]);
                    double am[9], bt[9];
#pragma unroll
                    for (int q = 0; q < 9; ++q) am[q] = a[q];
#pragma unroll
                    for (int r = 0; r < 3; ++r)
#pragma unroll
                        for (int q = 0; q < 3; ++q) bt[r * 3 + q] = kTr ? bm[u][q * 3 + r] : bm[u][r * 3 + q];
                    accum_block<kScalar>(am, bt, acc);
                }
        }
        double *o = cval + 9 * (base + t);
#pragma unroll
        for (int q = 0; q < 9; ++q) o[q] = acc[q];
    }
}

// Transpose positions of a structurally symmetric BSR pattern: for entry e =
// (i, j), tpos[e] = the index of entry (j, i); *bad = 1 if one is missing.
__global__ void k_tpos(int nrows, const int *__restrict__ ptr, const int *__restrict__ col,
                       int *__restrict__ tpos, int *bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    for (int e = ptr[i]; e < ptr[i + 1]; ++e) {
        const int j = col[e];
        int lo = ptr[j], hi = ptr[j + 1] - 1, found = -1;
        while (lo <= hi) {
            const int mid = (lo + hi) >> 1, v = col[mid];
            if (v == i) { found = mid; break; }
            if (v < i) lo = mid + 1; else hi = mid - 1;
        }
        tpos[e] = found;
        if (found < 0) *bad = 1;
    }
}

__global__ void k_spgemm_ub(int nrows, const int *ap, const int *ac, const int *bp,
                            int64_t *ub) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    int64_t s = 0;
    for (int ja = ap[i]; ja < ap[i + 1]; ++ja) s += bp[ac[ja] + 1] - bp[ac[ja]];
    ub[i] = s;
}

int next_pow2(int64_t v) {
    int64_t p = 1;
    while (p < v) p <<= 1;
    return static_cast<int>(p);
}

} // namespace

// ============================================================================

void check_dev_error(DevError *err, cudaStream_t s) {
    DevError h{};
    CK(cudaMemcpyAsync(&h, err, sizeof h, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h.code == 0) return;
    CK(cudaMemsetAsync(err, 0, sizeof(DevError), s));
    const char *what = "setup: device-side error";
    switch (h.code) {
        case SAMG_ZERO_DIAGONAL: what = "smooth_prolongation: zero filtered diagonal"; break;
        case SAMG_SINGULAR_BLOCK: what = "singular pivot in block inversion"; break;
        case SAMG_MISSING_DIAGONAL: what = "structurally zero diagonal"; break;
        case SAMG_INVALID_ARGUMENT: what = "input CSR rows must have strictly increasing columns"; break;
        case SAMG_ERROR: what = "dense_lu: singular coarse matrix"; break;
        default: break;
    }
    fail(h.code, std::string(what) + " (at index " + std::to_string(h.where) + ")");
}

template <class CT>
void scalar_to_bsr3_t(int64_t n, const int64_t *d_ptr, const CT *d_col, const double *d_val,
                      Bsr3 &out, cudaStream_t s) {
    const int64_t nb = n / 3;
    DevBuf<int> cnt(nb + 1, s);
    DevBuf<DevError> err(1, s);
    CK(cudaMemsetAsync(err.p, 0, sizeof(DevError), s));
    const int grid = std::max(1, std::min(ceil_div(nb, 256), 65535));
    k_s2b_count<<<grid, 256, 0, s>>>(nb, d_ptr, d_col, cnt.p, err.p);
    CK_LAUNCH();
    check_dev_error(err.p, s);
    DevBuf<int> bptr(nb + 1, s);
    const int64_t nnzb = scan_counts(cnt.p, bptr.p, nb, s);
    out.nrows = out.ncols = nb;
    out.nnzb = nnzb;
    out.ptr = std::move(bptr);
    out.col.alloc(nnzb, s);
    out.val.alloc(9 * nnzb, s);
    k_s2b_fill<<<grid, 256, 0, s>>>(nb, d_ptr, d_col, d_val, out.ptr.p, out.col.p, out.val.p);
    CK_LAUNCH();
}

void scalar_to_bsr3(int64_t n, const int64_t *d_ptr, const int64_t *d_col, const double *d_val,
                    Bsr3 &out, cudaStream_t s) {
    scalar_to_bsr3_t(n, d_ptr, d_col, d_val, out, s);
}

void scalar_to_bsr3(int64_t n, const int64_t *d_ptr, const int32_t *d_col, const double *d_val,
                    Bsr3 &out, cudaStream_t s) {
    scalar_to_bsr3_t(n, d_ptr, d_col, d_val, out, s);
}

void strength_graph(const Bsr3 &A, int h, double eps_strong, Graph &G, cudaStream_t s,
                    bool fnorm) {
    NvtxScope nvtx_scope("samg::strength_graph");
    const int n = static_cast<int>(A.nrows / h);
    const double eps2 = eps_strong * eps_strong;
    DevBuf<double> d(n, s), wblk(A.nnzb + 1, s);
    const int grid = ceil_div(n, 256);
    const int wgrid = std::max(1, std::min(ceil_div(A.nnzb, 256), 65535));
    if (fnorm)
        k_block_fnorm<<<wgrid, 256, 0, s>>>(A.nnzb, A.val.p, wblk.p);
    else
        k_block_maxabs<<<wgrid, 256, 0, s>>>(A.nnzb, A.val.p, wblk.p);
    k_strength_diag<<<grid, 256, 0, s>>>(n, h, A.ptr.p, A.col.p, wblk.p, d.p);
    CK_LAUNCH();
    DevBuf<int> cnt(n + 1, s), off(n + 1, s);
    k_strength_edges<<<grid, 256, 0, s>>>(n, h, A.ptr.p, A.col.p, wblk.p, d.p, eps2, cnt.p,
                                          nullptr, nullptr);
    CK_LAUNCH();
    const int64_t ne = scan_counts(cnt.p, off.p, n, s);
    DevBuf<unsigned long long> keys(2 * ne + 1, s), keys2(2 * ne + 1, s);
    k_strength_edges<<<grid, 256, 0, s>>>(n, h, A.ptr.p, A.col.p, wblk.p, d.p, eps2, nullptr,
                                          off.p, keys.p);
    CK_LAUNCH();
    int bits = 1;
    while ((1LL << bits) < n) ++bits;
    size_t bytes = 0;
    const int64_t nk = 2 * ne;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys.p, keys2.p, nk, 0, 32 + bits, s));
    DevBuf<char> ws(bytes, s);
    CK(cub::DeviceRadixSort::SortKeys(ws.p, bytes, keys.p, keys2.p, nk, 0, 32 + bits, s));
    DevBuf<int64_t> nuniq(1, s);
    size_t b2 = 0;
    CK(cub::DeviceSelect::Unique(nullptr, b2, keys2.p, keys.p, nuniq.p, nk, s));
    DevBuf<char> ws2(b2, s);
    CK(cub::DeviceSelect::Unique(ws2.p, b2, keys2.p, keys.p, nuniq.p, nk, s));
    int64_t nu = 0;
    CK(cudaMemcpyAsync(&nu, nuniq.p, sizeof nu, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    G.nnodes = n;
    G.nedges = nu;
    G.ptr.alloc(n + 1, s);
    G.col.alloc(nu + 1, s);
    int *gp = G.ptr.p, *gc = G.col.p;
    const unsigned long long *kp = keys.p;
    for_each(n + 1, [=] __device__(int64_t i) {
        int64_t lo = 0, hi = nu;
        const unsigned long long key = static_cast<unsigned long long>(i) << 32;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (kp[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        gp[i] = static_cast<int>(lo);
    }, s);
    for_each(nu, [=] __device__(int64_t e) { gc[e] = static_cast<int>(kp[e] & 0xffffffffULL); }, s);
}

int64_t aggregate(const Graph &G, DevBuf<int> &agg, cudaStream_t s, DevBuf<int> *seedno_out) {
    NvtxScope nvtx_scope("samg::aggregate");
    const int n = static_cast<int>(G.nnodes);
    agg.alloc(n, s);
    if (n == 0) return 0;
    DevBuf<unsigned char> state(n, s);
    DevBuf<int> m1(n, s), u1(n, s), und(1, s);
    CK(cudaMemsetAsync(state.p, 0, n, s));
    const int grid = ceil_div(n, 256);
    int h_und = 1;
    int rounds = 0;
    static const bool dirty_rounds = [] {
        const char *e = std::getenv("SAMG_AGG_DIRTY");
        return !(e && e[0] == '0');
    }();
    if (dirty_rounds) {
        // event-driven rounds (k_agg_ad / k_agg_bd): every node dirty at first,
        // (m1, u1) = -1 so the first phase a publishes all of them
        DevBuf<unsigned char> dA(n, s), dB(n, s);
        CK(cudaMemsetAsync(dA.p, 1, n, s));
        CK(cudaMemsetAsync(dB.p, 0, n, s));
        CK(cudaMemsetAsync(m1.p, 0xff, sizeof(int) * n, s));
        CK(cudaMemsetAsync(u1.p, 0xff, sizeof(int) * n, s));
        CK(cudaMemcpyAsync(und.p, &n, sizeof(int), cudaMemcpyHostToDevice, s));
        int last = n, stalled = 0;
        while (h_und) {
            for (int k = 0; k < 8; ++k) {
                k_agg_ad<<<grid, 256, 0, s>>>(n, G.ptr.p, G.col.p, state.p, m1.p, u1.p, dA.p, dB.p);
                k_agg_bd<<<grid, 256, 0, s>>>(n, G.ptr.p, G.col.p, state.p, m1.p, u1.p, dA.p, dB.p, und.p);
                ++rounds;
            }
            CK_LAUNCH();
            CK(cudaMemcpyAsync(&h_und, und.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            // the smallest undecided node decides in every round: 8 rounds
            // without a decision cannot happen
            stalled = h_und == last ? stalled + 1 : 0;
            last = h_und;
            if (stalled > 1 || rounds > 4 * n + 64) fail(SAMG_ERROR, "aggregate: no progress");
        }
    }
    while (!dirty_rounds && h_und) {
        for (int k = 0; k < 8; ++k) {
            k_agg_a<<<grid, 256, 0, s>>>(n, G.ptr.p, G.col.p, state.p, m1.p, u1.p);
            CK(cudaMemsetAsync(und.p, 0, sizeof(int), s));
            k_agg_b<<<grid, 256, 0, s>>>(n, G.ptr.p, G.col.p, state.p, m1.p, u1.p, und.p);
            ++rounds;
        }
        CK_LAUNCH();
        CK(cudaMemcpyAsync(&h_und, und.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (rounds > 4 * n + 64) fail(SAMG_ERROR, "aggregate: no progress");
    }
    // final seed-in-closed-neighbourhood map
    k_agg_a<<<grid, 256, 0, s>>>(n, G.ptr.p, G.col.p, state.p, m1.p, u1.p);
    CK_LAUNCH();
    DevBuf<int> is_in(n + 1, s), seedno(n + 1, s), parent(n, s), changed(1, s);
    const unsigned char *st = state.p;
    int *isin = is_in.p;
    for_each(n, [=] __device__(int64_t i) { isin[i] = st[i] == IN ? 1 : 0; }, s);
    const int64_t count = scan_counts(is_in.p, seedno.p, n, s);
    int *id = agg.p, *par = parent.p;
    const int *mm = m1.p, *sn = seedno.p, *gp = G.ptr.p, *gc = G.col.p;
    DevBuf<DevError> err(1, s);
    CK(cudaMemsetAsync(err.p, 0, sizeof(DevError), s));
    DevError *ep = err.p;
    for_each(n, [=] __device__(int64_t ii) {
        const int i = static_cast<int>(ii);
        if (mm[i] != INF) { id[i] = sn[mm[i]]; par[i] = i; return; }
        id[i] = -1;
        par[i] = -1;
        for (int e = gp[i]; e < gp[i + 1]; ++e) {
            const int nb = gc[e];
            if (mm[nb] != INF || nb < i) { par[i] = nb; return; }
        }
        raise(ep, SAMG_ERROR, i);
    }, s);
    check_dev_error(err.p, s);
    int h_changed = 1;
    int* ch = changed.p;
    while (h_changed) {
        CK(cudaMemsetAsync(changed.p, 0, sizeof(int), s));
        for_each(n, [=] __device__(int64_t i) {
            const int p = par[i];
            const int pp = par[p];
            if (pp != p) { par[i] = pp; *ch = 1; }
        }, s);
        CK(cudaMemcpyAsync(&h_changed, changed.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    for_each(n, [=] __device__(int64_t i) { if (id[i] < 0) id[i] = id[par[i]]; }, s);
    if (seedno_out) *seedno_out = std::move(seedno);
    return count;
}

void tentative(const DevBuf<int> &agg, int64_t nnodes, int64_t naggs, int pbs, const double *B,
               int k, DevBuf<double> &Pt, DevBuf<double> &Bc, DevError *err, cudaStream_t s,
               int64_t a0, int64_t a1) {
    NvtxScope nvtx_scope("samg::tentative_prolongation");
    if (a1 < 0) a1 = naggs;
    const int64_t nfine = nnodes * pbs;
    DevBuf<int> keys2(nnodes, s), iota(nnodes, s), nodes(nnodes, s), agg_ptr(naggs + 1, s);
    int *io = iota.p;
    for_each(nnodes, [=] __device__(int64_t i) { io[i] = static_cast<int>(i); }, s);
    size_t bytes = 0;
    int bits = 1;
    while ((1LL << bits) < naggs + 1) ++bits;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, agg.p, keys2.p, iota.p, nodes.p, nnodes, 0,
                                       bits, s));
    DevBuf<char> ws(bytes, s);
    CK(cub::DeviceRadixSort::SortPairs(ws.p, bytes, agg.p, keys2.p, iota.p, nodes.p, nnodes, 0,
                                       bits, s));
    const int *sk = keys2.p;
    int *ap = agg_ptr.p;
    const int nn = static_cast<int>(nnodes);
    for_each(naggs + 1, [=] __device__(int64_t a) {
        ap[a] = lower_bound_int(sk, nn, static_cast<int>(a));
    }, s);
    Pt.alloc(nfine * k, s);
    Bc.alloc(naggs * k * k, s);
    DevBuf<double> work, Qw;  // global scratch, only without the shared-memory path
    if (a1 > a0) {
        // shared-memory work matrices sized for the 99th-percentile-ish
        // aggregate: room for smem_m rows per group, larger aggregates keep
        // the global scratch (same kernel, same arithmetic)
        static const int use_smem = [] {
            const char *e = std::getenv("SAMG_QR_SMEM");
            return e ? std::atoi(e) : 1;
        }();
        int smem_m = 0, threads = 256;
        bool need_global = false;
        if (use_smem && k > 0) {
            DevBuf<int> dmax(1, s);
            CK(cudaMemsetAsync(dmax.p, 0, sizeof(int), s));
            int *dm = dmax.p;
            const int *apc = agg_ptr.p;
            for_each(a1 - a0, [=] __device__(int64_t t) {
                const int64_t a = a0 + t;
                atomicMax(dm, apc[a + 1] - apc[a]);
            }, s);
            int hmax = 0;
            CK(cudaMemcpyAsync(&hmax, dmax.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            // room for the largest aggregate up to 192 rows (C4 level 0: 78-row
            // aggregates); larger ones keep the global scratch.  At least 4
            // groups of 16 lanes per CTA in <= 110 KB (two CTAs per SM);
            // otherwise the global-scratch kernel's occupancy wins (C4
            // level 1: 2.0 ms global vs 6.9 ms with 2 groups per CTA)
            smem_m = std::min(pbs * hmax, 192);
            const size_t per_group = 2 * static_cast<size_t>(smem_m) * k * sizeof(double);
            int groups = 16;
            while (groups > 4 && groups * per_group > 110 * 1024) groups /= 2;
            if (groups * per_group > 110 * 1024) smem_m = 0;
            else threads = groups * kQrLanes;
            if (smem_m && pbs * hmax > smem_m) need_global = true;
        }
        const size_t dyn = smem_m ? static_cast<size_t>(threads / kQrLanes) * 2 * smem_m * k * sizeof(double) : 0;
        if (!smem_m || need_global) {
            work.alloc(nfine * k, s);
            Qw.alloc(nfine * k, s);
        }
        if (dyn > 48 * 1024) {
            static DeviceCache qattr;
            qattr.get([] {
                CK(cudaFuncSetAttribute(k_tentative_qr, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
                return 1;
            });
        }
        k_tentative_qr<<<ceil_div((a1 - a0) * kQrLanes, threads), threads, dyn, s>>>(
            naggs, pbs, k, nodes.p, agg_ptr.p, B, nfine, work.p, Qw.p, Pt.p, Bc.p, a0, a1, smem_m);
    }
    (void)err;
    CK_LAUNCH();
}

void smooth_prolongation(const Bsr3 &A, const Graph &G, const DevBuf<int> &agg, int64_t naggs,
                         int pbs, int k, const double *Pt, double omega, Bsr3 &P, DevError *err,
                         cudaStream_t s, int64_t node0, int64_t node1) {
    NvtxScope nvtx_scope("samg::smooth_prolongation");
    // k == 0: the indicator tentative operator of the `scalar` pipeline
    // (pbs 3 on every level: one 3x3 block column group per aggregate)
    const bool ind = k == 0;
    if (ind) {
        if (pbs != 3) fail(SAMG_UNSUPPORTED, "smooth_prolongation: indicator tentative needs pbs 3");
        k = 3;
    }
    const int h = pbs / 3, kb = k / 3;
    if (node1 < 0) node1 = A.nrows / h;
    // rows of the nodes [node0, node1): A (global numbering) must hold them
    const int64_t nnodes = node1 - node0, nbrows = nnodes * h, nsc = 3 * nbrows;
    const int64_t row0 = node0 * h;
    if (omega == 0.0) {
        P.alloc(nbrows, naggs * kb, nbrows * kb, s);
        if (ind)
            k_ptent_ind_bsr<<<ceil_div(nbrows + 1, 256), 256, 0, s>>>(static_cast<int>(nbrows), agg.p, Pt,
                                                                     P.ptr.p, P.col.p, P.val.p,
                                                                     static_cast<int>(row0));
        else
            k_ptent_bsr<<<ceil_div(nbrows + 1, 256), 256, 0, s>>>(static_cast<int>(nbrows), h, k, agg.p,
                                                             Pt, P.ptr.p, P.col.p, P.val.p,
                                                             static_cast<int>(row0));
        CK_LAUNCH();
        return;
    }
    // touched-aggregate lists per node, bounded by the node row length + 1
    DevBuf<int> rl(nnodes + 1, s), toff(nnodes + 1, s), tcnt(nnodes + 1, s);
    const int *ap = A.ptr.p;
    int *rlp = rl.p;
    for_each(nnodes, [=] __device__(int64_t nd) {
        rlp[nd] = ap[(node0 + nd + 1) * h] - ap[(node0 + nd) * h] + 1;
    }, s);
    const int64_t tl = scan_counts(rl.p, toff.p, nnodes, s);
    DevBuf<int> tlist(tl + 1, s);
    if (nnodes)
        k_psm_touch<<<ceil_div(nnodes, 128), 128, 0, s>>>(static_cast<int>(nnodes), h, A.ptr.p,
                                                          A.col.p, G.ptr.p, G.col.p, agg.p, toff.p,
                                                          tlist.p, tcnt.p, static_cast<int>(node0));
    CK_LAUNCH();
    DevBuf<int> bcnt(nbrows + 1, s);
    int *bc = bcnt.p;
    const int *tc = tcnt.p;
    for_each(nbrows, [=] __device__(int64_t br) { bc[br] = tc[br / h] * kb; }, s);
    P.nrows = nbrows;
    P.ncols = naggs * kb;
    P.ptr.alloc(nbrows + 1, s);
    P.nnzb = scan_counts(bcnt.p, P.ptr.p, nbrows, s);
    P.col.alloc(P.nnzb, s);
    P.val.alloc(9 * P.nnzb, s);
    if (nbrows == 0) return;
    k_psm_cols<<<ceil_div(nbrows, 256), 256, 0, s>>>(static_cast<int>(nbrows), h, kb, toff.p,
                                                     tlist.p, tcnt.p, P.ptr.p, P.col.p);
    CK_LAUNCH();
    DevBuf<double> dinv(nsc, s), diag(nsc, s);
    k_psm_diag<<<ceil_div(nsc, 256), 256, 0, s>>>(nsc, pbs, A.ptr.p, A.col.p, A.val.p, G.ptr.p,
                                                  G.col.p, dinv.p, diag.p, err, 3 * row0);
    CK_LAUNCH();
    check_dev_error(err, s);
    if (ind)
        k_psm_vals_ind<<<ceil_div(nsc, 128), 128, 0, s>>>(nsc, pbs, h, A.ptr.p, A.col.p, A.val.p,
                                                          G.ptr.p, G.col.p, agg.p, toff.p, tlist.p,
                                                          tcnt.p, dinv.p, diag.p, Pt, omega, P.ptr.p,
                                                          P.val.p, 3 * row0);
    else if (k == 6 && psm_block_rows() && nsc % 3 == 0)
        k_psm_vals3<6><<<ceil_div(nsc / 3, 128), 128, 0, s>>>(nsc / 3, pbs, A.ptr.p, A.col.p, A.val.p,
                                                             G.ptr.p, G.col.p, agg.p, toff.p, tlist.p,
                                                             tcnt.p, dinv.p, diag.p, Pt, omega, P.ptr.p,
                                                             P.val.p, 3 * row0);
    else
        k_psm_vals<<<ceil_div(nsc, 128), 128, 0, s>>>(nsc, pbs, h, k, A.ptr.p, A.col.p, A.val.p,
                                                      G.ptr.p, G.col.p, agg.p, toff.p, tlist.p,
                                                      tcnt.p, dinv.p, diag.p, Pt, omega, P.ptr.p,
                                                      P.val.p, 3 * row0);
    CK_LAUNCH();
}

void tentative_indicator(const DevBuf<int> &agg, int64_t nnodes, int64_t naggs, int pbs,
                         DevBuf<double> &Pt1, cudaStream_t s) {
    NvtxScope nvtx_scope("samg::tentative_prolongation (indicator)");
    DevBuf<int> cnt(naggs + 1, s);
    CK(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (naggs + 1), s));
    if (nnodes) k_bt_count<<<ceil_div(nnodes, 256), 256, 0, s>>>(static_cast<int>(nnodes), agg.p, cnt.p);
    Pt1.alloc(nnodes * pbs + 1, s);
    if (nnodes)
        k_tent_indicator<<<ceil_div(nnodes, 256), 256, 0, s>>>(nnodes, pbs, agg.p, cnt.p, Pt1.p);
    CK_LAUNCH();
}

void block_transfer(const Bsr3 &A, const Graph &G, const DevBuf<int> &agg, int64_t naggs,
                    double omega, Bsr3 &P, DevError *err, cudaStream_t s, int64_t r0, int64_t r1) {
    NvtxScope nvtx_scope("samg::block_transfer_operators");
    const int nall = static_cast<int>(A.nrows);  // aggregate sizes over every node
    if (r1 < 0) r1 = nall;
    const int n = static_cast<int>(r1 - r0);      // rows [r0, r1) of P
    DevBuf<int> cnt(naggs + 1, s);
    DevBuf<double> pv(naggs + 1, s);
    CK(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (naggs + 1), s));
    k_bt_count<<<ceil_div(nall, 256), 256, 0, s>>>(nall, agg.p, cnt.p);
    k_bt_scale<<<ceil_div(naggs, 256), 256, 0, s>>>(static_cast<int>(naggs), cnt.p, pv.p);
    CK_LAUNCH();
    if (omega == 0.0) {
        P.alloc(n, naggs, n, s);
        k_bt_tent<<<ceil_div(n + 1, 256), 256, 0, s>>>(n, agg.p, pv.p, P.ptr.p, P.col.p, P.val.p,
                                                       static_cast<int>(r0));
        CK_LAUNCH();
        return;
    }
    // columns: the sorted distinct aggregates of the row's kept entries and
    // its own (k_psm_touch with one block row per node)
    DevBuf<int> rl(n + 1, s), toff(n + 1, s), tcnt(n + 1, s);
    const int *ap = A.ptr.p;
    int *rlp = rl.p;
    for_each(n, [=] __device__(int64_t i) { rlp[i] = ap[r0 + i + 1] - ap[r0 + i] + 1; }, s);
    const int64_t tl = scan_counts(rl.p, toff.p, n, s);
    DevBuf<int> tlist(tl + 1, s);
    if (n)
        k_psm_touch<<<ceil_div(n, 128), 128, 0, s>>>(n, 1, A.ptr.p, A.col.p, G.ptr.p, G.col.p, agg.p,
                                                     toff.p, tlist.p, tcnt.p, static_cast<int>(r0));
    CK_LAUNCH();
    P.nrows = n;
    P.ncols = naggs;
    P.ptr.alloc(n + 1, s);
    P.nnzb = scan_counts(tcnt.p, P.ptr.p, n, s);
    P.col.alloc(P.nnzb, s);
    P.val.alloc(9 * P.nnzb, s);
    if (n == 0) return;
    k_psm_cols<<<ceil_div(n, 256), 256, 0, s>>>(n, 1, 1, toff.p, tlist.p, tcnt.p, P.ptr.p,
                                                P.col.p);
    DevBuf<double> dg(9 * static_cast<int64_t>(n) + 1, s), dinv(9 * static_cast<int64_t>(n) + 1, s);
    k_bt_diag<<<ceil_div(n, 128), 128, 0, s>>>(n, A.ptr.p, A.col.p, A.val.p, G.ptr.p, G.col.p,
                                               dg.p, dinv.p, err, static_cast<int>(r0));
    CK_LAUNCH();
    check_dev_error(err, s);
    k_bt_vals<<<std::max<int64_t>(1, ceil_div(P.nnzb, 128)), 128, 0, s>>>(
        P.nnzb, n, A.ptr.p, A.col.p, A.val.p, G.ptr.p, G.col.p, agg.p, pv.p, dg.p, dinv.p, omega,
        P.ptr.p, P.col.p, P.val.p, static_cast<int>(r0));
    CK_LAUNCH();
}

void transpose(const Bsr3 &P, Bsr3 &R, cudaStream_t s) {
    NvtxScope nvtx_scope("samg::transpose");
    const int64_t nnz = P.nnzb;
    R.alloc(P.ncols, P.nrows, nnz, s);
    DevBuf<int> rowidx(nnz + 1, s), iota(nnz + 1, s), perm(nnz + 1, s), skeys(nnz + 1, s);
    const int *pp = P.ptr.p;
    int *ri = rowidx.p, *io = iota.p;
    const int nr = static_cast<int>(P.nrows);
    for_each(nnz, [=] __device__(int64_t e) {
        io[e] = static_cast<int>(e);
        ri[e] = lower_bound_int(pp, nr + 1, static_cast<int>(e) + 1) - 1;
    }, s);
    int bits = 1;
    while ((1LL << bits) < P.ncols + 1) ++bits;
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, P.col.p, skeys.p, iota.p, perm.p, nnz, 0,
                                       bits, s));
    DevBuf<char> ws(bytes, s);
    CK(cub::DeviceRadixSort::SortPairs(ws.p, bytes, P.col.p, skeys.p, iota.p, perm.p, nnz, 0, bits,
                                       s));
    const int *sk = skeys.p, *pm = perm.p;
    int *rp = R.ptr.p, *rc = R.col.p;
    double *rv = R.val.p;
    const double *pv = P.val.p;
    const int nz = static_cast<int>(nnz);
    for_each(P.ncols + 1, [=] __device__(int64_t c) {
        rp[c] = lower_bound_int(sk, nz, static_cast<int>(c));
    }, s);
    for_each(nnz, [=] __device__(int64_t k) {
        const int e = pm[k];
        rc[k] = ri[e];
        const double *b = pv + 9 * static_cast<int64_t>(e);
        double *t = rv + 9 * k;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) t[c * 3 + r] = b[r * 3 + c];
    }, s);
}

namespace {
__global__ void k_max_row_len(int nrows, const int *ptr, int *mx) {
    int v = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += gridDim.x * blockDim.x)
        v = max(v, ptr[i + 1] - ptr[i]);
    v = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(v)));
    if ((threadIdx.x & 31) == 0) atomicMax(mx, v);
}

template <bool kScalar>
void spgemm_impl(const Bsr3 &A, const Bsr3 &B, Bsr3 &C, cudaStream_t s, const BCols *bcols) {
    if (A.ncols != B.nrows) fail(SAMG_DIMENSION_MISMATCH, "spgemm: inner dimensions disagree");
    const int n = static_cast<int>(A.nrows);
    // SAMG_SPGEMM_TIMING=1: sub-phase wall times on stderr (diagnosis only)
    static const bool timing = [] {
        const char *e = std::getenv("SAMG_SPGEMM_TIMING");
        return e && e[0] == '1';
    }();
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char *what) {
        if (!timing) return;
        CK(cudaStreamSynchronize(s));
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "  spgemm %8d rows %-10s %8.3f ms\n", n, what,
                     std::chrono::duration<double, std::milli>(t - t_last).count());
        t_last = t;
    };
    C.nrows = A.nrows;
    C.ncols = B.ncols;
    C.ptr.alloc(n + 1, s);
    if (n == 0) { CK(cudaMemsetAsync(C.ptr.p, 0, sizeof(int), s)); C.nnzb = 0; return; }
    DevBuf<int64_t> ub(n, s);
    k_spgemm_ub<<<ceil_div(n, 256), 256, 0, s>>>(n, A.ptr.p, A.col.p, B.ptr.p, ub.p);
    CK_LAUNCH();
    // max upper bound decides the shared table size of the symbolic pass
    DevBuf<int64_t> mx(1, s);
    size_t bytes = 0;
    CK(cub::DeviceReduce::Max(nullptr, bytes, ub.p, mx.p, n, s));
    DevBuf<char> ws(bytes, s);
    CK(cub::DeviceReduce::Max(ws.p, bytes, ub.p, mx.p, n, s));
    int64_t maxub = 0;
    CK(cudaMemcpyAsync(&maxub, mx.p, sizeof maxub, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    constexpr int kMaxCap = 16384;
    const int cap_s = std::min(kMaxCap, std::max(256, next_pow2(2 * std::min<int64_t>(maxub, B.ncols) + 2)));
    DevBuf<int> cnt(n + 1, s), ovf(1, s), winlo(n + 1, s), mode(n + 1, s), maxwin(1, s);
    CK(cudaMemsetAsync(ovf.p, 0, sizeof(int), s));
    CK(cudaMemsetAsync(maxwin.p, 0, sizeof(int), s));
    // 0. window-bitmap symbolic pass (most rows); rows whose product columns
    //    span more than kWinMax columns are marked -2 for the hash kernels
    static const int win_env = [] {
        const char *e = std::getenv("SAMG_SPGEMM_MAXWIN");
        return e ? std::min(kWinMax, std::atoi(e)) : -1;
    }();
    // measured on C1 (profiles/README.md): the bitmap kernels win for
    // products with short B rows (x P: RAP), the hash kernels for long ones
    // (x A: RA, whose many lanes per step amortise the hashing)
    const double b_row = B.nrows ? static_cast<double>(B.nnzb) / B.nrows : 0.0;
    const int win_limit = win_env >= 0 ? win_env : (b_row <= 16.0 ? kWinMax : 0);
    k_spgemm_bcount<<<ceil_div(n, kBWPB), kBWPB * 32, 0, s>>>(n, A.ptr.p, A.col.p, B.ptr.p, B.col.p,
                                                              win_limit, cnt.p, winlo.p, maxwin.p);
    CK_LAUNCH();
    DevBuf<int> fb(n, s), nfb_d(1, s);
    CK(cudaMemsetAsync(nfb_d.p, 0, sizeof(int), s));
    {
        int *cc = cnt.p, *md = mode.p, *fl = fb.p, *nf = nfb_d.p;
        for_each(n, [=] __device__(int64_t i) {
            md[i] = cc[i] >= 0 ? 1 : 0;
            if (cc[i] == -2) fl[atomicAdd(nf, 1)] = static_cast<int>(i);
        }, s);
    }
    int hdr[2] = {0, 0};
    CK(cudaMemcpyAsync(&hdr[0], nfb_d.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&hdr[1], maxwin.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int nfb = hdr[0], wmax = hdr[1];
    // 1. warp-per-row hash symbolic pass for those; rows above kWCap/2-1
    //    columns -> wide list
    if (nfb)
        k_spgemm_wcount<<<ceil_div(nfb, kWPB), 256, 0, s>>>(nfb, fb.p, A.ptr.p, A.col.p, B.ptr.p,
                                                            B.col.p, cnt.p);
    CK_LAUNCH();
    DevBuf<int> wide(n, s), nwide_d(1, s);
    CK(cudaMemsetAsync(nwide_d.p, 0, sizeof(int), s));
    {
        int *cc = cnt.p, *wl = wide.p, *nw = nwide_d.p;
        for_each(n, [=] __device__(int64_t i) {
            if (cc[i] < 0) wl[atomicAdd(nw, 1)] = static_cast<int>(i);
        }, s);
    }
    int nwide = 0;
    CK(cudaMemcpyAsync(&nwide, nwide_d.p, sizeof nwide, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (nwide) {
        // sort the wide list so the CTA passes visit rows in a fixed order
        std::vector<int> hw(nwide);
        CK(cudaMemcpyAsync(hw.data(), wide.p, sizeof(int) * nwide, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::sort(hw.begin(), hw.end());
        CK(cudaMemcpyAsync(wide.p, hw.data(), sizeof(int) * nwide, cudaMemcpyHostToDevice, s));
        CK(cudaFuncSetAttribute(k_spgemm_count<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kMaxCap * 4));
        k_spgemm_count<false><<<nwide, 256, cap_s * 4, s>>>(nwide, wide.p, A.ptr.p, A.col.p, B.ptr.p,
                                                           B.col.p, cap_s, nullptr, nullptr, cnt.p,
                                                           ovf.p);
        CK_LAUNCH();
    }
    int novf = 0;
    CK(cudaMemcpyAsync(&novf, ovf.p, sizeof novf, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    // rows whose distinct count exceeds the shared table: global slabs
    DevBuf<int> orows;
    DevBuf<int64_t> goff;
    DevBuf<int> gkeys, gvals, glist;
    if (novf) {
        std::vector<int> hcnt(n);
        std::vector<int64_t> hub(n);
        CK(cudaMemcpyAsync(hcnt.data(), cnt.p, sizeof(int) * n, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hub.data(), ub.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::vector<int> rows;
        std::vector<int64_t> off{0};
        for (int i = 0; i < n; ++i)
            if (hcnt[i] < 0) {
                rows.push_back(i);
                off.push_back(off.back() + next_pow2(2 * std::min<int64_t>(hub[i], B.ncols) + 2));
            }
        orows.alloc(rows.size(), s);
        goff.alloc(off.size(), s);
        CK(cudaMemcpyAsync(orows.p, rows.data(), sizeof(int) * rows.size(), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(goff.p, off.data(), sizeof(int64_t) * off.size(), cudaMemcpyHostToDevice, s));
        gkeys.alloc(off.back(), s);
        gvals.alloc(off.back(), s);
        glist.alloc(off.back() / 2 + 1, s);
        k_spgemm_count<true><<<static_cast<int>(rows.size()), 256, 0, s>>>(
            static_cast<int>(rows.size()), orows.p, A.ptr.p, A.col.p, B.ptr.p, B.col.p, 0, gkeys.p,
            goff.p, cnt.p, ovf.p);
        CK_LAUNCH();
    }
    mark("symbolic");
    C.nnzb = scan_counts(cnt.p, C.ptr.p, n, s);
    C.col.alloc(C.nnzb, s);
    C.val.alloc(9 * C.nnzb, s);
    mark("alloc");
    // numeric: table sized by the actual max row count
    DevBuf<int> mc(1, s);
    size_t b3 = 0;
    CK(cub::DeviceReduce::Max(nullptr, b3, cnt.p, mc.p, n, s));
    DevBuf<char> ws3(b3, s);
    CK(cub::DeviceReduce::Max(ws3.p, b3, cnt.p, mc.p, n, s));
    int maxc = 0;
    CK(cudaMemcpyAsync(&maxc, mc.p, sizeof maxc, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const int cap_n = std::min(kMaxCap, std::max(256, next_pow2(2 * static_cast<int64_t>(maxc) + 2)));
    // pull numeric (k_spgemm_pull) when B's columns are available and A's
    // longest row fits a shared-memory hash; the row kernels then only write
    // the pattern (kCols)
    static const bool pull_env = [] {
        const char *e = std::getenv("SAMG_SPGEMM_PULL");
        return !e || e[0] != '0';
    }();
    int tcap = 0;
    if (bcols && pull_env) {
        DevBuf<int> mxa(1, s);
        CK(cudaMemsetAsync(mxa.p, 0, sizeof(int), s));
        k_max_row_len<<<std::min(1184, ceil_div(n, 256)), 256, 0, s>>>(n, A.ptr.p, mxa.p);
        CK_LAUNCH();
        int maxa = 0;
        CK(cudaMemcpyAsync(&maxa, mxa.p, sizeof maxa, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        tcap = std::max(64, next_pow2(2 * static_cast<int64_t>(maxa) + 2));
        if (tcap > 16384) tcap = 0;  // 128 KB of hash: use the row kernels
    }
    const bool pull = tcap > 0;
    const size_t smem_n = static_cast<size_t>(cap_n) * 4 * 2 + static_cast<size_t>(cap_n / 2) * 4;
    // 2a. window-bitmap numeric pass (accumulators in shared memory for rows
    //     of up to acc_cap columns)
    if (wmax > 0) {
        static const int budget = [] {  // shared bytes per warp (rows of one CTA)
            const char *e = std::getenv("SAMG_SPGEMM_WARP_SMEM");
            return e ? std::atoi(e) : 20 * 1024;
        }();
        const int words = (wmax + 31) / 32;
        const int bm_bytes = (2 * words * 4 + 15) / 16 * 16;
        const int acc_cap = std::max(0, std::min(512, (budget - bm_bytes) / 72));
        const size_t smem_b = static_cast<size_t>(kBWPB) * (bm_bytes + static_cast<size_t>(acc_cap) * 72);
        static DeviceCache battr;
        battr.get([] {
            CK(cudaFuncSetAttribute(k_spgemm_bnumeric<kScalar>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    220 * 1024));
            CK(cudaFuncSetAttribute(k_spgemm_bnumeric<kScalar, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
            return 1;
        });
        if (pull)
            k_spgemm_bnumeric<kScalar, true><<<ceil_div(n, kBWPB), kBWPB * 32, smem_b, s>>>(
                n, A.ptr.p, A.col.p, A.val.p, B.ptr.p, B.col.p, B.val.p, C.ptr.p, mode.p, winlo.p, words,
                acc_cap, C.col.p, C.val.p);
        else
            k_spgemm_bnumeric<kScalar><<<ceil_div(n, kBWPB), kBWPB * 32, smem_b, s>>>(
                n, A.ptr.p, A.col.p, A.val.p, B.ptr.p, B.col.p, B.val.p, C.ptr.p, mode.p, winlo.p, words,
                acc_cap, C.col.p, C.val.p);
        CK_LAUNCH();
    }
    mark("bnumeric");
    // 2b. warp-per-row hash numeric pass for the other narrow rows
    if (nfb) {
        const size_t smem_w = static_cast<size_t>(kWPB) * kWCap * 5 / 2 * sizeof(int);
        auto kw = pull ? k_spgemm_wnumeric<kScalar, true> : k_spgemm_wnumeric<kScalar>;
        CK(cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem_w)));
        kw<<<ceil_div(n, kWPB), 256, smem_w, s>>>(n, A.ptr.p, A.col.p, A.val.p, B.ptr.p,
                                                  B.col.p, B.val.p, C.ptr.p, mode.p,
                                                  C.col.p, C.val.p);
        CK_LAUNCH();
    }
    mark("wnumeric");
    // 3. CTA-per-row numeric pass for the wide rows
    if (nwide) {
        auto kn = pull ? k_spgemm_numeric<false, kScalar, true> : k_spgemm_numeric<false, kScalar>;
        CK(cudaFuncSetAttribute(kn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxCap * 10));
        kn<<<nwide, 256, smem_n, s>>>(nwide, wide.p, A.ptr.p, A.col.p, A.val.p,
                                      B.ptr.p, B.col.p, B.val.p, cap_n, nullptr,
                                      nullptr, nullptr, nullptr, C.ptr.p, C.col.p,
                                      C.val.p);
        CK_LAUNCH();
    }
    if (novf) {
        const int nr = static_cast<int>(orows.n);
        k_spgemm_numeric<true, kScalar><<<nr, 256, 0, s>>>(nr, orows.p, A.ptr.p, A.col.p, A.val.p, B.ptr.p,
                                                 B.col.p, B.val.p, 0, gkeys.p, gvals.p, glist.p,
                                                 goff.p, C.ptr.p, C.col.p, C.val.p);
        CK_LAUNCH();
        if (pull) {  // these rows are complete: the pull pass skips them
            int *md = mode.p;
            const int *orw = orows.p;
            for_each(nr, [=] __device__(int64_t k) { md[orw[k]] = 2; }, s);
        }
    }
    mark("wide");
    if (pull) {
        const int smem_p = tcap * 8;
        // few rows (coarse levels: long rows, many outputs each): more
        // threads per row
        const bool wide_cta = n < 148 * 16;
        // batch: measured on C4 (scripts/setup_phases.py): 1 for the fine
        // level's 601 526 rows (88 / 100 ms vs 122 / 139 with 4: occupancy),
        // 4 for level 1's 78 162 (37 / 57 ms vs 40 / 83 with 1); C1's level
        // 0 (20 642 rows): 1 (2.3 / 3.0 ms vs 2.8 / 4.0 with 4; ncu: 128
        // registers, 20 % warps active)
        static const int batch_env = [] {
            const char *e = std::getenv("SAMG_PULL_BATCH");
            return e ? std::atoi(e) : 0;
        }();
        // (round 2: C1's level 1 (3 822 rows) 2.02 / 0.85 ms with 1 -> 1.37 /
        // 0.75 with 4: few rows per SM, latency-bound column scans)
        const int batch = batch_env > 0 ? batch_env
                                        : ((n >= 50000 && n < 200000) || (!wide_cta && n < 12000) ? 4 : 1);
        using KP = decltype(&k_spgemm_pull<kScalar, true, 128, 1>);
        KP kp;
        auto pick = [&](auto bt) {
            constexpr int BT = decltype(bt)::value;
            kp = wide_cta ? (bcols->tr ? k_spgemm_pull<kScalar, true, 256, BT> : k_spgemm_pull<kScalar, false, 256, BT>)
                          : (bcols->tr ? k_spgemm_pull<kScalar, true, 128, BT> : k_spgemm_pull<kScalar, false, 128, BT>);
        };
        if (batch >= 4) pick(std::integral_constant<int, 4>{});
        else if (batch == 2) pick(std::integral_constant<int, 2>{});
        else pick(std::integral_constant<int, 1>{});
        if (smem_p > 48 * 1024)
            CK(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_p));
        kp<<<n, wide_cta ? 256 : 128, smem_p, s>>>(n, tcap, A.ptr.p, A.col.p, A.val.p, *bcols, mode.p,
                                                   C.ptr.p, C.col.p, C.val.p);
        CK_LAUNCH();
        mark("pull");
    }
}

} // namespace

void spgemm(const Bsr3 &A, const Bsr3 &B, Bsr3 &C, cudaStream_t s, bool scalar_order) {
    if (scalar_order) spgemm_impl<true>(A, B, C, s, nullptr);
    else spgemm_impl<false>(A, B, C, s, nullptr);
}

// Galerkin product A_c = (R A) P (csr.hpp:259-262), both products with the
// pull numeric pass: B = A through its transpose positions when A's pattern
// is symmetric (every level matrix: R = P^T), B = P through R's blocks.
void galerkin(const Bsr3 &R, const Bsr3 &A, const Bsr3 &P, Bsr3 &Ac, cudaStream_t s,
              bool scalar_order) {
    NvtxScope nvtx_scope("samg::galerkin");
    galerkin_rows(R, A, P, R, Ac, s, scalar_order);
}

// Rows [r0, r1) of M as a matrix of their own (same columns).
void slice_rows(const Bsr3 &M, int64_t r0, int64_t r1, Bsr3 &out, cudaStream_t s) {
    int b[2] = {0, 0};
    CK(cudaMemcpyAsync(&b[0], M.ptr.p + r0, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&b[1], M.ptr.p + r1, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    out.alloc(r1 - r0, M.ncols, b[1] - b[0], s);
    const int *mp = M.ptr.p + r0;
    int *op = out.ptr.p;
    const int b0 = b[0];
    for_each(r1 - r0 + 1, [=] __device__(int64_t i) { op[i] = mp[i] - b0; }, s);
    if (out.nnzb) {
        CK(cudaMemcpyAsync(out.col.p, M.col.p + b0, sizeof(int) * out.nnzb, cudaMemcpyDeviceToDevice, s));
        CK(cudaMemcpyAsync(out.val.p, M.val.p + 9LL * b0, sizeof(double) * 9 * out.nnzb,
                           cudaMemcpyDeviceToDevice, s));
    }
}

// Rows of the Galerkin product for the rows of Rl (a row slice of R, or R):
// (Rl A) P, with P's columns read through the full R = P^T.
void galerkin_rows(const Bsr3 &Rl, const Bsr3 &A, const Bsr3 &P, const Bsr3 &R, Bsr3 &Ac,
                   cudaStream_t s, bool scalar_order, bool subset) {
    NvtxScope nvtx_scope("samg::galerkin");
    Bsr3 RA;
    {
        DevBuf<int> tpos(std::max<int64_t>(1, A.nnzb), s), bad(1, s);
        CK(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
        if (A.nrows)
            k_tpos<<<ceil_div(A.nrows, 256), 256, 0, s>>>(static_cast<int>(A.nrows), A.ptr.p, A.col.p,
                                                          tpos.p, bad.p);
        CK_LAUNCH();
        int hbad = 0;
        CK(cudaMemcpyAsync(&hbad, bad.p, sizeof hbad, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        BCols ba;
        ba.cp = A.ptr.p; ba.ri = A.col.p; ba.pos = tpos.p; ba.val = A.val.p; ba.tr = false;
        // subset: A holds only some rows (global numbering, the others
        // empty), so transpose positions into rows it lacks are missing;
        // they are never read -- a hit needs the row in Rl's pattern, whose
        // rows A holds (dsetup.cu)
        const BCols *pa = ((hbad && !subset) || A.nrows != A.ncols) ? nullptr : &ba;
        if (scalar_order) spgemm_impl<true>(Rl, A, RA, s, pa);
        else spgemm_impl<false>(Rl, A, RA, s, pa);
    }
    BCols bp;
    bp.cp = R.ptr.p; bp.ri = R.col.p; bp.pos = nullptr; bp.val = R.val.p; bp.tr = true;
    if (scalar_order) spgemm_impl<true>(RA, P, Ac, s, &bp);
    else spgemm_impl<false>(RA, P, Ac, s, &bp);
}

// thread per block row: merge the two sorted column lists (to_dense of both,
// compared on the union pattern, hierarchy.hpp:390-396)
__global__ void k_union_diff(int64_t n, const int *ap, const int *ac, const double *av,
                             const int *gp, const int *gc, const double *gv, double *acc) {
    double d = 0.0, r = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int ja = ap[i], jg = gp[i];
        const int ea = ap[i + 1], eg = gp[i + 1];
        while (ja < ea || jg < eg) {
            const int ca = ja < ea ? ac[ja] : INT_MAX, cg = jg < eg ? gc[jg] : INT_MAX;
            const double *x = ca <= cg ? av + 9LL * ja : nullptr;
            const double *y = cg <= ca ? gv + 9LL * jg : nullptr;
            for (int e = 0; e < 9; ++e) {
                const double a = x ? x[e] : 0.0, g = y ? y[e] : 0.0;
                d += (a - g) * (a - g);
                r += g * g;
            }
            if (x) ++ja;
            if (y) ++jg;
        }
    }
    for (int o = 16; o; o >>= 1) {
        d += __shfl_xor_sync(0xffffffffu, d, o);
        r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc, d);
        atomicAdd(acc + 1, r);
    }
}

void union_diff(const Bsr3 &A, const Bsr3 &G, double out[2], cudaStream_t s) {
    if (A.nrows != G.nrows || A.ncols != G.ncols)
        fail(SAMG_ERROR, "setup: Galerkin consistency check: shapes differ");
    DevBuf<double> acc(2, s);
    CK(cudaMemsetAsync(acc.p, 0, 2 * sizeof(double), s));
    if (A.nrows)
        k_union_diff<<<std::min(ceil_div(A.nrows, 256), 4 * sm_count()), 256, 0, s>>>(
            A.nrows, A.ptr.p, A.col.p, A.val.p, G.ptr.p, G.col.p, G.val.p, acc.p);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(out, acc.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
}

void fix_decoupled_rows(Bsr3 &A, cudaStream_t s, int64_t row0) {
    const int *ap = A.ptr.p, *ac = A.col.p;
    double *av = A.val.p;
    const int r0 = static_cast<int>(row0);
    for_each(A.nrows, [=] __device__(int64_t i) {
        int dg = -1;
        for (int j = ap[i]; j < ap[i + 1]; ++j)
            if (ac[j] == r0 + i) { dg = j; break; }
        for (int r = 0; r < 3; ++r) {
            bool zero_row = true;
            for (int j = ap[i]; zero_row && j < ap[i + 1]; ++j)
                for (int c = 0; c < 3; ++c)
                    if (av[9 * static_cast<int64_t>(j) + 3 * r + c] != 0.0) { zero_row = false; break; }
            if (zero_row && dg >= 0) av[9 * static_cast<int64_t>(dg) + 4 * r] = 1.0;
        }
    }, s);
}

void setup_smoother(const Bsr3 &A, int kind, double omega, Smoother &M, DevError *err,
                    cudaStream_t s, int64_t row0) {
    NvtxScope nvtx_scope("samg::smoother_setup");
    const int *ap = A.ptr.p, *ac = A.col.p;
    const int r0 = static_cast<int>(row0);  // global id of local row 0 (diagonal = r0 + i)
    const double *av = A.val.p;
    DevError *ep = err;
    if (kind == SAMG_SMOOTHER_ILU0) {
        setup_ilu0(A, M, err, s);
        return;
    }
    if (kind == SAMG_SMOOTHER_JACOBI) {
        // relaxation.hpp:147-162; the damping is folded in (omega * (1/d)),
        // the same first product as relaxation.hpp:172
        M.kind = SM_POINT;
        M.data.alloc(3 * A.nrows, s);
        double *m = M.data.p;
        for_each(A.nrows, [=] __device__(int64_t i) {
            int dg = -1;
            for (int j = ap[i]; j < ap[i + 1]; ++j) if (ac[j] == r0 + i) { dg = j; break; }
            for (int r = 0; r < 3; ++r) {
                const double d = dg >= 0 ? av[9 * static_cast<int64_t>(dg) + 4 * r] : 0.0;
                if (d == 0.0) { raise(ep, SAMG_ZERO_DIAGONAL, 3 * i + r); m[3 * i + r] = 0.0; continue; }
                m[3 * i + r] = __dmul_rn(omega, __ddiv_rn(1.0, d));
            }
        }, s);
        return;
    }
    M.kind = SM_BLOCK;
    M.data.alloc(9 * A.nrows, s);
    double *m = M.data.p;
    const bool spai = kind == SAMG_SMOOTHER_SPAI0;
    for_each(A.nrows, [=] __device__(int64_t i) {
        int dg = -1;
        double den = 0.0;
        for (int j = ap[i]; j < ap[i + 1]; ++j) {
            if (ac[j] == r0 + i) dg = j;
            const double *b = av + 9 * static_cast<int64_t>(j);
            for (int e = 0; e < 9; ++e) den = __dadd_rn(den, __dmul_rn(b[e], b[e]));
        }
        double *Mi = m + 9 * i;
        if (dg < 0) { raise(ep, SAMG_MISSING_DIAGONAL, i); return; }
        const double *a = av + 9 * static_cast<int64_t>(dg);
        if (spai) {
            if (den == 0.0) { raise(ep, SAMG_ZERO_DIAGONAL, i); return; }
            for (int e = 0; e < 9; ++e) Mi[e] = __ddiv_rn(a[e], den);
            return;
        }
        // inverse (static_block.hpp:155-194)
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
            if (fabs(lu[k * 3 + k]) < 1e-300) { raise(ep, SAMG_SINGULAR_BLOCK, i); return; }
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
            for (int r = 0; r < 3; ++r) Mi[r * 3 + c] = __dmul_rn(omega, x[r]);
        }
    }, s);
}

} // namespace samgb
