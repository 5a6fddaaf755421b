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
#include "problem.cuh"

namespace samgb {

namespace {

// hex8_stiffness (elasticity.hpp:57-123) for a given isotropic C.
void hex8_ke(double hx, double hy, double hz, const double C[6][6], double *Ke) {
    int off[8][3];
    for (int a = 0; a < 8; ++a) { off[a][0] = a & 1; off[a][1] = (a >> 1) & 1; off[a][2] = (a >> 2) & 1; }
    const double g = 1.0 / std::sqrt(3.0);
    const double gp[2] = {-g, g};
    const double jac[3] = {hx / 2, hy / 2, hz / 2};
    const double detJ = jac[0] * jac[1] * jac[2];
    std::fill(Ke, Ke + 576, 0.0);
    for (int qx = 0; qx < 2; ++qx)
    for (int qy = 0; qy < 2; ++qy)
    for (int qz = 0; qz < 2; ++qz) {
        const double xi = gp[qx], eta = gp[qy], zeta = gp[qz];
        double dN[8][3];
        for (int a = 0; a < 8; ++a) {
            const double sx = off[a][0] ? 1.0 : -1.0, sy = off[a][1] ? 1.0 : -1.0,
                         sz = off[a][2] ? 1.0 : -1.0;
            dN[a][0] = 0.125 * sx * (1 + sy * eta) * (1 + sz * zeta) / jac[0];
            dN[a][1] = 0.125 * (1 + sx * xi) * sy * (1 + sz * zeta) / jac[1];
            dN[a][2] = 0.125 * (1 + sx * xi) * (1 + sy * eta) * sz / jac[2];
        }
        for (int a = 0; a < 8; ++a)
        for (int b = 0; b < 8; ++b) {
            double Ba[6][3] = {}, Bb[6][3] = {};
            auto fill = [](double Bm[6][3], const double d[3]) {
                Bm[0][0] = d[0]; Bm[1][1] = d[1]; Bm[2][2] = d[2];
                Bm[3][0] = d[1]; Bm[3][1] = d[0];
                Bm[4][1] = d[2]; Bm[4][2] = d[1];
                Bm[5][0] = d[2]; Bm[5][2] = d[0];
            };
            fill(Ba, dN[a]);
            fill(Bb, dN[b]);
            for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                double s = 0;
                for (int p = 0; p < 6; ++p)
                for (int q = 0; q < 6; ++q) s += Ba[p][i] * C[p][q] * Bb[q][j];
                Ke[(3 * a + i) * 24 + (3 * b + j)] += s * detJ;
            }
        }
    }
}

void iso_C(double lambda, double mu, double C[6][6]) {
    for (int i = 0; i < 6; ++i) for (int j = 0; j < 6; ++j) C[i][j] = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) C[i][j] = (i == j) ? lambda + 2 * mu : lambda;
    for (int i = 3; i < 6; ++i) C[i][i] = mu;
}

// counter-based uniform in [0,1): splitmix64 of (seed, stream, index)
double uhash(uint64_t seed, uint64_t stream, uint64_t i) {
    uint64_t z = seed * 0x9E3779B97F4A7C15ULL + stream * 0xD1B54A32D192ED03ULL + i + 0x632BE59BD9B4E019ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return static_cast<double>(z >> 11) * (1.0 / 9007199254740992.0);
}

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

samg_problem *generate_hex(const samg_problem_params &p) {
    if (p.nx < 1 || p.ny < 1 || p.nz < 1)
        fail(SAMG_INVALID_MATERIAL, "generate_hex_elasticity: element counts must be >= 1");
    if (!p.heterogeneous && (!(p.E > 0) || !(p.nu > 0 && p.nu < 0.5)))
        fail(SAMG_INVALID_MATERIAL, "generate_hex_elasticity: need E > 0 and 0 < nu < 0.5");
    if (!(p.lx > 0 && p.ly > 0 && p.lz > 0))
        fail(SAMG_INVALID_MATERIAL, "generate_hex_elasticity: domain lengths must be > 0");
    const int64_t nx = p.nx, ny = p.ny, nz = p.nz;
    const int64_t mx = nx + 1, my = ny + 1, mz = nz + 1;
    const double hx = p.lx / nx, hy = p.ly / ny, hz = p.lz / nz;
    const bool elim = p.dirichlet == SAMG_DIRICHLET_ELIMINATE;
    const bool keep = p.dirichlet == SAMG_DIRICHLET_KEEP_ROWS;
    const int64_t i0 = elim ? 1 : 0;  // first kept x index
    const int64_t kx = mx - i0;        // kept nodes along x
    auto node_id = [&](int64_t i, int64_t j, int64_t k) -> int64_t {
        const int64_t ii = i - i0;
        return p.x_slowest ? k + mz * (j + my * ii) : ii + kx * (j + my * k);
    };
    auto constrained = [&](int64_t i) { return keep && i == 0; };
    const int64_t nnodes_all = kx * my * mz;
    // optional row range [node_begin, node_end): one rank's slab of a
    // row-partitioned problem (global column ids)
    const bool ranged = p.node_end > p.node_begin;
    const int64_t nb = ranged ? p.node_begin : 0, ne = ranged ? p.node_end : nnodes_all;
    if (nb < 0 || ne > nnodes_all)
        fail(SAMG_INVALID_ARGUMENT, "generate_hex: node range outside the grid");
    const int64_t nnodes = ne - nb;

    auto *pb = new samg_problem;
    pb->nnodes = nnodes;
    pb->n = 3 * nnodes;

    // element matrices: homogeneous -> one Ke; heterogeneous -> lambda/mu split
    std::vector<double> Khom(576), Klam(576), Kmu(576);
    std::vector<double> elam, emu;
    const int64_t nel = nx * ny * nz;
    if (!p.heterogeneous) {
        double C[6][6];
        iso_C(p.E * p.nu / ((1 + p.nu) * (1 - 2 * p.nu)), p.E / (2 * (1 + p.nu)), C);
        hex8_ke(hx, hy, hz, C, Khom.data());
    } else {
        double C[6][6];
        iso_C(1.0, 0.0, C);
        hex8_ke(hx, hy, hz, C, Klam.data());
        iso_C(0.0, 1.0, C);
        hex8_ke(hx, hy, hz, C, Kmu.data());
        elam.resize(nel);
        emu.resize(nel);
        parallel_for(nel, [&](int64_t e) {
            const double u1 = std::max(uhash(p.seed, 1, e), 1e-300), u2 = uhash(p.seed, 2, e);
            const double g = std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
            const double E = std::exp(g);
            const double nu = 0.25 + 0.1 * uhash(p.seed, 3, e);
            elam[e] = E * nu / ((1 + nu) * (1 - 2 * nu));
            emu[e] = E / (2 * (1 + nu));
        });
    }

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
            const double nodal_force = -hx * hy * hz / 8.0;  // elasticity.hpp:189
            for (int64_t ez = k - 1; ez <= k; ++ez)
            for (int64_t ey = j - 1; ey <= j; ++ey)
            for (int64_t ex = i - 1; ex <= i; ++ex)
                if (ex >= 0 && ey >= 0 && ez >= 0 && ex < nx && ey < ny && ez < nz)
                    f[2] += nodal_force;
        } else if (p.load == SAMG_LOAD_TRACTION_XEND) {
            if (i == nx) {
                const double q = -hy * hz / 4.0;
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
