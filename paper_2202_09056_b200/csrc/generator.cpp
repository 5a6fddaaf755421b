// generator.cpp -- synthetic 3D linear-elasticity problems (input tooling).
//
// Restates the reference generator (elasticity.hpp:129-213: trilinear hex8
// elements, 2x2x2 Gauss, isotropic material, interleaved DOFs, unit -z body
// force, x=0 face clamped) and extends it for the BASELINE configs:
// free-DOF elimination of the clamped face, per-element heterogeneous
// materials, a -z traction on the x-end face, seeded noise / random loads,
// non-unit domains (cantilever beam) and x-slowest node numbering.
//
// Assembly is row-wise and direct to 3x3 BSR: block (n, m) is the sum, in
// ascending element order, of the element blocks coupling nodes n and m.
// Every block of a node pair that shares an element is stored (the
// reference stores every Ke entry, zeros included), so the pattern equals
// to_block<3> of the reference's matrix.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "common.cuh"
#include "hexgen.cuh"
#include "problem.cuh"

namespace samgb {

namespace {

template <class F>
void parallel_for(int64_t n, F f) {
    unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    if (n < 4096) nt = 1;
    std::vector<std::thread> th;
    const int64_t chunk = (n + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        const int64_t b = t * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        th.emplace_back([=] { for (int64_t i = b; i < e; ++i) f(i); });
    }
    for (auto &x : th) x.join();
}

} // namespace

// Validated grid, element matrices and per-element materials of a problem:
// shared by the host assembly below and the device assembly (assemble.cu),
// so both use bitwise the same inputs.
HexSetup hex_prepare(const samg_problem_params &p) {
    if (p.nx < 1 || p.ny < 1 || p.nz < 1)
        fail(SAMG_INVALID_MATERIAL, "generate_hex_elasticity: element counts must be >= 1");
    if (!p.heterogeneous && (!(p.E > 0) || !(p.nu > 0 && p.nu < 0.5)))
        fail(SAMG_INVALID_MATERIAL, "generate_hex_elasticity: need E > 0 and 0 < nu < 0.5");
    if (!(p.lx > 0 && p.ly > 0 && p.lz > 0))
        fail(SAMG_INVALID_MATERIAL, "generate_hex_elasticity: domain lengths must be > 0");
    HexSetup h;
    h.p = p;
    h.nx = p.nx; h.ny = p.ny; h.nz = p.nz;
    h.mx = h.nx + 1; h.my = h.ny + 1; h.mz = h.nz + 1;
    h.hx = p.lx / h.nx; h.hy = p.ly / h.ny; h.hz = p.lz / h.nz;
    h.elim = p.dirichlet == SAMG_DIRICHLET_ELIMINATE;
    h.keep = p.dirichlet == SAMG_DIRICHLET_KEEP_ROWS;
    h.i0 = h.elim ? 1 : 0;
    h.kx = h.mx - h.i0;
    h.nnodes_all = h.kx * h.my * h.mz;
    const bool ranged = p.node_end > p.node_begin;
    h.nb = ranged ? p.node_begin : 0;
    h.ne = ranged ? p.node_end : h.nnodes_all;
    if (h.nb < 0 || h.ne > h.nnodes_all)
        fail(SAMG_INVALID_ARGUMENT, "generate_hex: node range outside the grid");
    h.nodal_force = -h.hx * h.hy * h.hz / 8.0;  // elasticity.hpp:189
    h.traction = -h.hy * h.hz / 4.0;
    h.Khom.assign(576, 0.0); h.Klam.assign(576, 0.0); h.Kmu.assign(576, 0.0);
    const int64_t nel = h.nx * h.ny * h.nz;
    if (!p.heterogeneous) {
        double C[6][6];
        iso_C(p.E * p.nu / ((1 + p.nu) * (1 - 2 * p.nu)), p.E / (2 * (1 + p.nu)), C);
        hex8_ke(h.hx, h.hy, h.hz, C, h.Khom.data());
    } else {
        double C[6][6];
        iso_C(1.0, 0.0, C);
        hex8_ke(h.hx, h.hy, h.hz, C, h.Klam.data());
        iso_C(0.0, 1.0, C);
        hex8_ke(h.hx, h.hy, h.hz, C, h.Kmu.data());
        h.elam.resize(nel);
        h.emu.resize(nel);
        double *el = h.elam.data(), *em = h.emu.data();
        const uint64_t seed = p.seed;
        parallel_for(nel, [=](int64_t e) {
            const double u1 = std::max(uhash(seed, 1, e), 1e-300), u2 = uhash(seed, 2, e);
            const double g = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
            const double E = std::exp(g);
            const double nu = 0.25 + 0.1 * uhash(seed, 3, e);
            el[e] = E * nu / ((1 + nu) * (1 - 2 * nu));
            em[e] = E / (2 * (1 + nu));
        });
    }
    return h;
}

samg_problem *generate_hex(const samg_problem_params &p) {
    const HexSetup H = hex_prepare(p);
    const int64_t nx = H.nx, ny = H.ny, nz = H.nz;
    const int64_t mx = H.mx, my = H.my, mz = H.mz;
    const double hx = H.hx, hy = H.hy, hz = H.hz;
    const bool keep = H.keep;
    const int64_t i0 = H.i0, kx = H.kx;
    auto node_id = [&](int64_t i, int64_t j, int64_t k) -> int64_t {
        const int64_t ii = i - i0;
        return p.x_slowest ? k + mz * (j + my * ii) : ii + kx * (j + my * k);
    };
    auto constrained = [&](int64_t i) { return keep && i == 0; };
    const int64_t nb = H.nb, ne = H.ne;
    const int64_t nnodes = ne - nb;

    auto *pb = new samg_problem;
    pb->nnodes = nnodes;
    pb->n = 3 * nnodes;
    const std::vector<double> &Khom = H.Khom, &Klam = H.Klam, &Kmu = H.Kmu;
    const std::vector<double> &elam = H.elam, &emu = H.emu;

    // node -> (i,j,k)
    auto ijk_of = [&](int64_t id, int64_t &i, int64_t &j, int64_t &k) {
        if (p.x_slowest) { k = id % mz; j = (id / mz) % my; i = id / (mz * my) + i0; }
        else { i = id % kx + i0; j = (id / kx) % my; k = id / (kx * my); }
    };
    // neighbour enumeration in ascending id order
    auto for_nbrs = [&](int64_t i, int64_t j, int64_t k, auto f) {
        if (p.x_slowest) {
            for (int di = -1; di <= 1; ++di) for (int dj = -1; dj <= 1; ++dj) for (int dk = -1; dk <= 1; ++dk) f(di, dj, dk);
        } else {
            for (int dk = -1; dk <= 1; ++dk) for (int dj = -1; dj <= 1; ++dj) for (int di = -1; di <= 1; ++di) f(di, dj, dk);
        }
    };
    auto inside = [&](int64_t i, int64_t j, int64_t k) {
        return i >= i0 && i < mx && j >= 0 && j < my && k >= 0 && k < mz;
    };

    std::vector<int64_t> cnt(nnodes + 1, 0);
    parallel_for(nnodes, [&](int64_t L) {
        int64_t i, j, k;
        ijk_of(nb + L, i, j, k);
        if (constrained(i)) { cnt[L + 1] = 1; return; }
        int64_t c = 0;
        for_nbrs(i, j, k, [&](int di, int dj, int dk) {
            const int64_t a = i + di, b = j + dj, d = k + dk;
            if (inside(a, b, d) && !constrained(a)) ++c;
        });
        cnt[L + 1] = c;
    });
    for (int64_t L = 0; L < nnodes; ++L) cnt[L + 1] += cnt[L];
    const int64_t nnzb = cnt[nnodes];
    pb->ptr = cnt;
    pb->col.resize(nnzb);
    pb->val.assign(9 * nnzb, 0.0);
    pb->rhs.assign(3 * nnodes, 0.0);
    pb->xyz.resize(3 * nnodes);

    parallel_for(nnodes, [&](int64_t L) {
        const int64_t n = nb + L;
        int64_t i, j, k;
        ijk_of(n, i, j, k);
        pb->xyz[3 * L] = i * hx;
        pb->xyz[3 * L + 1] = j * hy;
        pb->xyz[3 * L + 2] = k * hz;
        int64_t o = pb->ptr[L];
        if (constrained(i)) {
            pb->col[o] = n;
            double *blk = &pb->val[9 * o];
            blk[0] = blk[4] = blk[8] = 1.0;
            return;
        }
        for_nbrs(i, j, k, [&](int di, int dj, int dk) {
            const int64_t a = i + di, b = j + dj, d = k + dk;
            if (!inside(a, b, d) || constrained(a)) return;
            pb->col[o] = node_id(a, b, d);
            double *blk = &pb->val[9 * o];
            // elements shared by n and m, ascending element index (x fastest)
            for (int64_t ez = std::max(k, d) - 1; ez <= std::min(k, d); ++ez)
            for (int64_t ey = std::max(j, b) - 1; ey <= std::min(j, b); ++ey)
            for (int64_t ex = std::max(i, a) - 1; ex <= std::min(i, a); ++ex) {
                if (ex < 0 || ey < 0 || ez < 0 || ex >= nx || ey >= ny || ez >= nz) continue;
                const int la = static_cast<int>((i - ex) + 2 * (j - ey) + 4 * (k - ez));
                const int lb = static_cast<int>((a - ex) + 2 * (b - ey) + 4 * (d - ez));
                const int64_t e = ex + nx * (ey + ny * ez);
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c) {
                        const int idx = (3 * la + r) * 24 + 3 * lb + c;
                        const double v = p.heterogeneous
                            ? elam[e] * Klam[idx] + emu[e] * Kmu[idx]
                            : Khom[idx];
                        blk[3 * r + c] += v;
                    }
            }
            ++o;
        });
        // loads
        double *f = &pb->rhs[3 * L];
        if (p.load == SAMG_LOAD_BODY_FORCE) {
            const double nodal_force = H.nodal_force;
            for (int64_t ez = k - 1; ez <= k; ++ez)
            for (int64_t ey = j - 1; ey <= j; ++ey)
            for (int64_t ex = i - 1; ex <= i; ++ex)
                if (ex >= 0 && ey >= 0 && ez >= 0 && ex < nx && ey < ny && ez < nz)
                    f[2] += nodal_force;
        } else if (p.load == SAMG_LOAD_TRACTION_XEND) {
            if (i == nx) {
                const double q = H.traction;
                for (int64_t ez = k - 1; ez <= k; ++ez)
                for (int64_t ey = j - 1; ey <= j; ++ey)
                    if (ey >= 0 && ez >= 0 && ey < ny && ez < nz) f[2] += q;
            }
        } else {
            const int64_t gnode = i + mx * (j + my * k);
            for (int r = 0; r < 3; ++r) f[r] = 2.0 * uhash(p.seed, 4, 3 * gnode + r) - 1.0;
        }
        if (p.noise != 0.0) {
            const int64_t gnode = i + mx * (j + my * k);
            for (int r = 0; r < 3; ++r)
                f[r] += p.noise * (2.0 * uhash(p.seed, 5, 3 * gnode + r) - 1.0);
        }
    });
    return pb;
}

void rigid_body_modes(int64_t nnodes, const double *xyz, double *B) {
    // elasticity.hpp:38-52, column-major (3n)-by-6
    const int64_t nr = 3 * nnodes;
    std::fill(B, B + nr * 6, 0.0);
    for (int64_t a = 0; a < nnodes; ++a) {
        const double x = xyz[3 * a], y = xyz[3 * a + 1], z = xyz[3 * a + 2];
        const int64_t r = 3 * a;
        B[0 * nr + r + 0] = 1;
        B[1 * nr + r + 1] = 1;
        B[2 * nr + r + 2] = 1;
        B[3 * nr + r + 0] = -y; B[3 * nr + r + 1] = x;
        B[4 * nr + r + 1] = -z; B[4 * nr + r + 2] = y;
        B[5 * nr + r + 0] = z;  B[5 * nr + r + 2] = -x;
    }
}

} // namespace samgb
