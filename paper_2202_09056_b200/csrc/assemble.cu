// assemble.cu -- on-GPU assembly of the synthetic hex8 elasticity problems
// (SURVEY 8f #2): hex8 element blocks -> 3x3 BSR directly in HBM, plus the
// right-hand side, node coordinates and rigid-body modes, so a large problem
// (C4: 23.9 M unknowns) never crosses PCIe.
//
// Same semantics and bitwise the same result as the host assembly
// (generator.cpp, itself the reference generator elasticity.hpp:129-213
// extended): the element matrices and per-element materials come from the
// same host preparation (hex_prepare), and every block is summed in the same
// (ascending element) order with --fmad=false arithmetic.
#include <cub/cub.cuh>

#include <algorithm>

#include "hexgen.cuh"
#include "kernels.cuh"
#include "problem.cuh"

namespace samgb {

namespace {

struct Grid {
    int64_t nx, ny, nz, mx, my, mz, i0, kx, nb, nnodes;
    double hx, hy, hz, nodal_force, traction, noise;
    uint64_t seed;
    int keep, x_slowest, hetero, load;
};

__device__ __forceinline__ int64_t node_id(const Grid &g, int64_t i, int64_t j, int64_t k) {
    const int64_t ii = i - g.i0;
    return g.x_slowest ? k + g.mz * (j + g.my * ii) : ii + g.kx * (j + g.my * k);
}
__device__ __forceinline__ void ijk_of(const Grid &g, int64_t id, int64_t &i, int64_t &j, int64_t &k) {
    if (g.x_slowest) { k = id % g.mz; j = (id / g.mz) % g.my; i = id / (g.mz * g.my) + g.i0; }
    else { i = id % g.kx + g.i0; j = (id / g.kx) % g.my; k = id / (g.kx * g.my); }
}
__device__ __forceinline__ bool inside(const Grid &g, int64_t i, int64_t j, int64_t k) {
    return i >= g.i0 && i < g.mx && j >= 0 && j < g.my && k >= 0 && k < g.mz;
}
__device__ __forceinline__ bool constrained(const Grid &g, int64_t i) { return g.keep && i == 0; }

// neighbour offsets in ascending node-id order (generator.cpp for_nbrs)
__device__ __forceinline__ void nbr(const Grid &g, int t, int &di, int &dj, int &dk) {
    const int a = t / 9 - 1, b = (t / 3) % 3 - 1, c = t % 3 - 1;
    if (g.x_slowest) { di = a; dj = b; dk = c; }
    else { dk = a; dj = b; di = c; }
}

__global__ void k_hex_count(Grid g, int *cnt) {
    const int64_t L = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (L >= g.nnodes) return;
    int64_t i, j, k;
    ijk_of(g, g.nb + L, i, j, k);
    int c = 0;
    if (constrained(g, i)) {
        c = 1;
    } else {
        for (int t = 0; t < 27; ++t) {
            int di, dj, dk;
            nbr(g, t, di, dj, dk);
            if (inside(g, i + di, j + dj, k + dk) && !constrained(g, i + di)) ++c;
        }
    }
    cnt[L] = c;
}

// one thread per node row: blocks in ascending neighbour order, each the sum
// over the shared elements in ascending element index (generator.cpp:199-236)
__global__ void k_hex_fill(Grid g, const int *__restrict__ ptr, const double *__restrict__ K,
                           const double *__restrict__ elam, const double *__restrict__ emu,
                           int *col, double *val, double *rhs, double *xyz) {
    const int64_t L = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (L >= g.nnodes) return;
    const int64_t n = g.nb + L;
    int64_t i, j, k;
    ijk_of(g, n, i, j, k);
    xyz[3 * L] = static_cast<double>(i) * g.hx;
    xyz[3 * L + 1] = static_cast<double>(j) * g.hy;
    xyz[3 * L + 2] = static_cast<double>(k) * g.hz;
    int64_t o = ptr[L];
    if (constrained(g, i)) {
        col[o] = static_cast<int>(n);
        double *blk = val + 9 * o;
        for (int e = 0; e < 9; ++e) blk[e] = (e % 4 == 0) ? 1.0 : 0.0;
    } else {
        const double *Khom = K, *Klam = K + 576, *Kmu = K + 1152;
        for (int t = 0; t < 27; ++t) {
            int di, dj, dk;
            nbr(g, t, di, dj, dk);
            const int64_t a = i + di, b = j + dj, d = k + dk;
            if (!inside(g, a, b, d) || constrained(g, a)) continue;
            col[o] = static_cast<int>(node_id(g, a, b, d));
            double blk[9];
            for (int e = 0; e < 9; ++e) blk[e] = 0.0;
            for (int64_t ez = max(k, d) - 1; ez <= min(k, d); ++ez)
            for (int64_t ey = max(j, b) - 1; ey <= min(j, b); ++ey)
            for (int64_t ex = max(i, a) - 1; ex <= min(i, a); ++ex) {
                if (ex < 0 || ey < 0 || ez < 0 || ex >= g.nx || ey >= g.ny || ez >= g.nz) continue;
                const int la = static_cast<int>((i - ex) + 2 * (j - ey) + 4 * (k - ez));
                const int lb = static_cast<int>((a - ex) + 2 * (b - ey) + 4 * (d - ez));
                const int64_t e = ex + g.nx * (ey + g.ny * ez);
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c) {
                        const int idx = (3 * la + r) * 24 + 3 * lb + c;
                        const double v = g.hetero ? __dadd_rn(__dmul_rn(elam[e], Klam[idx]),
                                                              __dmul_rn(emu[e], Kmu[idx]))
                                                  : Khom[idx];
                        blk[3 * r + c] = __dadd_rn(blk[3 * r + c], v);
                    }
            }
            double *dst = val + 9 * o;
            for (int e = 0; e < 9; ++e) dst[e] = blk[e];
            ++o;
        }
    }
    // loads (generator.cpp:237-261); a kept clamped row has none
    double f[3] = {0.0, 0.0, 0.0};
    if (!constrained(g, i)) {
        if (g.load == SAMG_LOAD_BODY_FORCE) {
            for (int64_t ez = k - 1; ez <= k; ++ez)
            for (int64_t ey = j - 1; ey <= j; ++ey)
            for (int64_t ex = i - 1; ex <= i; ++ex)
                if (ex >= 0 && ey >= 0 && ez >= 0 && ex < g.nx && ey < g.ny && ez < g.nz)
                    f[2] = __dadd_rn(f[2], g.nodal_force);
        } else if (g.load == SAMG_LOAD_TRACTION_XEND) {
            if (i == g.nx)
                for (int64_t ez = k - 1; ez <= k; ++ez)
                for (int64_t ey = j - 1; ey <= j; ++ey)
                    if (ey >= 0 && ez >= 0 && ey < g.ny && ez < g.nz) f[2] = __dadd_rn(f[2], g.traction);
        } else {
            const int64_t gnode = i + g.mx * (j + g.my * k);
            for (int r = 0; r < 3; ++r)
                f[r] = __dsub_rn(__dmul_rn(2.0, uhash(g.seed, 4, 3 * gnode + r)), 1.0);
        }
        if (g.noise != 0.0) {
            const int64_t gnode = i + g.mx * (j + g.my * k);
            for (int r = 0; r < 3; ++r)
                f[r] = __dadd_rn(f[r], __dmul_rn(g.noise, __dsub_rn(__dmul_rn(2.0, uhash(g.seed, 5, 3 * gnode + r)), 1.0)));
        }
    }
    for (int r = 0; r < 3; ++r) rhs[3 * L + r] = f[r];
}

__global__ void k_i64_to_i32(int64_t n, const int64_t *a, int *b) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t < n) b[t] = static_cast<int>(a[t]);
}

// rigid_body_modes (elasticity.hpp:38-52), column-major (3n) x 6
__global__ void k_rbm(int64_t nnodes, const double *xyz, double *B) {
    const int64_t a = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (a >= nnodes) return;
    const int64_t nr = 3 * nnodes, r = 3 * a;
    const double x = xyz[3 * a], y = xyz[3 * a + 1], z = xyz[3 * a + 2];
    double v[6][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {-y, x, 0}, {0, -z, y}, {z, 0, -x}};
    for (int c = 0; c < 6; ++c)
        for (int q = 0; q < 3; ++q) B[c * nr + r + q] = v[c][q];
}

} // namespace

void generate_hex_device(const samg_problem_params &p, Bsr3 &A, DevBuf<double> &rhs,
                         DevBuf<double> &xyz, DevBuf<double> &B, int64_t &nnodes, cudaStream_t s) {
    const HexSetup H = hex_prepare(p);
    Grid g{};
    g.nx = H.nx; g.ny = H.ny; g.nz = H.nz; g.mx = H.mx; g.my = H.my; g.mz = H.mz;
    g.i0 = H.i0; g.kx = H.kx; g.nb = H.nb; g.nnodes = H.ne - H.nb;
    g.hx = H.hx; g.hy = H.hy; g.hz = H.hz; g.nodal_force = H.nodal_force; g.traction = H.traction;
    g.noise = p.noise; g.seed = p.seed; g.keep = H.keep; g.x_slowest = p.x_slowest;
    g.hetero = p.heterogeneous; g.load = p.load;
    nnodes = g.nnodes;
    if (H.nnodes_all > INT32_MAX) fail(SAMG_UNSUPPORTED, "generate_hex_device: more than 2^31-1 nodes");
    const int64_t n = g.nnodes;
    DevBuf<double> K(3 * 576, s), el, em;
    CK(cudaMemcpyAsync(K.p, H.Khom.data(), sizeof(double) * 576, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(K.p + 576, H.Klam.data(), sizeof(double) * 576, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(K.p + 1152, H.Kmu.data(), sizeof(double) * 576, cudaMemcpyHostToDevice, s));
    if (p.heterogeneous) {
        el.alloc(H.elam.size(), s);
        em.alloc(H.emu.size(), s);
        h2d(el.p, H.elam.data(), sizeof(double) * H.elam.size(), s);
        h2d(em.p, H.emu.data(), sizeof(double) * H.emu.size(), s);
    }
    DevBuf<int> cnt(n + 1, s);
    k_hex_count<<<ceil_div(n, 256), 256, 0, s>>>(g, cnt.p);
    CK_LAUNCH();
    // ptr = exclusive scan of the counts (int64 total checked against int32)
    DevBuf<int64_t> ptr64(n + 1, s);
    {
        size_t bytes = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, ptr64.p, n + 1, s));
        DevBuf<char> ws(bytes + 1, s);
        CK(cudaMemsetAsync(cnt.p + n, 0, sizeof(int), s));
        CK(cub::DeviceScan::ExclusiveSum(ws.p, bytes, cnt.p, ptr64.p, n + 1, s));
    }
    int64_t nnzb = 0;
    CK(cudaMemcpyAsync(&nnzb, ptr64.p + n, sizeof nnzb, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    A.alloc(n, H.nnodes_all, nnzb, s);  // throws above 2^31-1 blocks
    k_i64_to_i32<<<ceil_div(n + 1, 256), 256, 0, s>>>(n + 1, ptr64.p, A.ptr.p);
    CK_LAUNCH();
    rhs.alloc(3 * n + 1, s);
    xyz.alloc(3 * n + 1, s);
    B.alloc(18 * n + 1, s);
    k_hex_fill<<<ceil_div(n, 128), 128, 0, s>>>(g, A.ptr.p, K.p, el.p, em.p, A.col.p, A.val.p, rhs.p, xyz.p);
    CK_LAUNCH();
    k_rbm<<<ceil_div(n, 256), 256, 0, s>>>(n, xyz.p, B.p);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(s));
}

} // namespace samgb
