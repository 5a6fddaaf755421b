// ref_driver.cpp -- C-ABI driver around the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against the headers
// and sources under /root/reference/proj (never copied into this repo) into
// oracle/_ref/libsamg_ref.so, which travels to the GPU box.  Used (a) to pin
// the C restatement in samg_oracle.c, (b) to generate tests/golden fixtures,
// (c) as bench.py's CPU reference arm.
//
// Everything on the setup path is the reference's own public API:
// samg::setup(..., pipeline::ns_block, ...) (hierarchy.hpp:263-405),
// samg::cg_solve (cg.hpp:87-112), samg::vcycle (hierarchy.hpp:408-441).
// Aggregates are re-derived with the public strength_graph + aggregate on
// to_scalar(A_l) exactly as as_scalar_transfer does (coarsening.hpp:451-464).
// The 3x3 block smoothers the reference lacks (SPAI0, block Jacobi) use a
// harness V-cycle that follows hierarchy.hpp:408-441 line by line and the
// reference's generic cg_solve_op (cg.hpp:39-83).
#include <array>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "samg/cg.hpp"
#include "samg/coarsening.hpp"
#include "samg/elasticity.hpp"
#include "samg/hierarchy.hpp"
#include "samg/kernels.hpp"

// The repo's host problem generator (paper_2202_09056_b200/csrc/generator.cpp,
// compiled into this library by oracle/Makefile as host-only C++): the
// reference arm of bench.py and the golden scripts build the BASELINE
// configs (free-DOF, heterogeneous, cantilever) without loading the product
// library.  Input tooling only, not on any measured path.
#include "problem.cuh"
namespace samgb { samg_problem *generate_hex(const samg_problem_params &p); }

using namespace samg;

namespace {

std::string g_err;

int code_of(const std::exception &e) {
    if (dynamic_cast<const dimension_mismatch *>(&e)) return 2;
    if (dynamic_cast<const not_divisible *>(&e)) return 3;
    if (dynamic_cast<const singular_block *>(&e)) return 4;
    if (dynamic_cast<const missing_diagonal *>(&e)) return 5;
    if (dynamic_cast<const zero_diagonal *>(&e)) return 6;
    if (dynamic_cast<const non_square *>(&e)) return 7;
    if (dynamic_cast<const bad_nullspace_shape *>(&e)) return 8;
    if (dynamic_cast<const breakdown_non_spd *>(&e)) return 9;
    if (dynamic_cast<const invalid_material *>(&e)) return 10;
    return 1;
}

#define GUARD_BEGIN try {
#define GUARD_END                                   \
    } catch (const std::exception &e) {             \
        g_err = e.what();                           \
        return code_of(e);                          \
    }                                               \
    return 0;

// smoother kinds, same numbering as samg_oracle.h / samg_b200.h
enum { SM_JACOBI = 0, SM_SPAI0 = 1, SM_BLOCK_JACOBI = 2, SM_ILU0 = 3 };

struct ref_handle {
    hierarchy H;
    int smoother = SM_JACOBI;
    double smoother_omega = 0.72;
    std::vector<std::vector<samg::index>> agg;
    std::vector<samg::index> agg_count;
    std::vector<std::vector<double>> sm;  // block smoother data per level
    double setup_seconds = 0;
    // scalar pipelines: the level matrices as 3x3 blocks (to_block<3>, for
    // the parity taps; the hierarchy itself keeps them scalar)
    std::vector<std::array<csr<block3>, 3>> blockview;
    std::vector<csr<block3>> ilu_blockview;  // ilu0<double> factors as 3x3 blocks
};

using clk = std::chrono::steady_clock;

const csr<block3> &blk(const any_matrix &m) { return std::get<csr<block3>>(m); }

void block_smooth(const ref_handle &h, samg::index l, std::span<const double> f,
        std::span<double> u, std::span<double> r, int sweeps) {
    const csr<block3> &A = blk(h.H.levels[l].A);
    const std::vector<double> &M = h.sm[l];
    for (int s = 0; s < sweeps; ++s) {
        residual(A, f, std::span<const double>(u.data(), u.size()), r);
        for (samg::index i = 0; i < A.nrows; ++i) {
            double t[3];
            for (int p = 0; p < 3; ++p) {
                t[p] = 0;
                for (int q = 0; q < 3; ++q) t[p] += M[i * 9 + p * 3 + q] * r[i * 3 + q];
            }
            for (int p = 0; p < 3; ++p) u[i * 3 + p] += t[p];
        }
    }
}

// Harness V-cycle: hierarchy.hpp:408-441 with the block smoother swapped in.
void harness_vcycle(const ref_handle &h, std::span<const double> f,
        std::span<double> u, vcycle_workspace &ws) {
    const hierarchy &H = h.H;
    const samg::index L = H.nlevels();
    if (L == 1) { H.coarsest.solve(f, u); return; }
    std::copy(f.begin(), f.end(), ws.f[0].begin());
    std::copy(u.begin(), u.end(), ws.u[0].begin());
    for (samg::index i = 0; i < L - 1; ++i) {
        const level &lv = H.levels[i];
        if (i > 0) std::fill(ws.u[i].begin(), ws.u[i].end(), 0.0);
        block_smooth(h, i, ws.f[i], ws.u[i], ws.r[i], H.params.pre_sweeps);
        residual(blk(lv.A), std::span<const double>(ws.f[i]),
                std::span<const double>(ws.u[i]), std::span<double>(ws.r[i]));
        any_spmv(1.0, lv.R, ws.r[i], 0.0, ws.f[i + 1]);
    }
    H.coarsest.solve(ws.f[L - 1], ws.u[L - 1]);
    for (samg::index i = L - 2; i >= 0; --i) {
        const level &lv = H.levels[i];
        any_spmv(1.0, lv.P, ws.u[i + 1], 1.0, ws.u[i]);
        block_smooth(h, i, ws.f[i], ws.u[i], ws.r[i], H.params.post_sweeps);
    }
    std::copy(ws.u[0].begin(), ws.u[0].end(), u.begin());
}

bool uses_harness(const ref_handle &h) {
    return h.smoother == SM_SPAI0 || h.smoother == SM_BLOCK_JACOBI;
}

} // namespace

template <class T>
static T *dup(const std::vector<T> &v) {
    T *p = static_cast<T *>(std::malloc(sizeof(T) * (v.size() ? v.size() : 1)));
    std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

extern "C" {

const char *ref_last_error() { return g_err.c_str(); }
void ref_free_buf(void *p) { std::free(p); }

// The reference generator (elasticity.hpp:129-213) + rigid_body_modes.
int ref_generate_hex(int64_t nx, int64_t ny, int64_t nz, double E, double nu,
        int clamp_x0, int64_t *n, int64_t **ptr, int64_t **col, double **val,
        double **rhs, double **coords) {
    GUARD_BEGIN
    problem_bundle pb = generate_hex_elasticity(nx, ny, nz, E, nu, clamp_x0 != 0);
    *n = pb.A.nrows;
    *ptr = dup(pb.A.ptr);
    *col = dup(pb.A.col);
    *val = dup(pb.A.val);
    *rhs = dup(pb.rhs);
    *coords = dup(pb.coords.xyz);
    GUARD_END
}

// The BASELINE-config generator (see the include above): BSR3 arrays,
// right-hand side and node coordinates, malloc'd (ref_free_buf).
int ref_gen_hex(const samg_problem_params *p, int64_t *n, int64_t *nnodes, int64_t **ptr,
        int64_t **col, double **val, double **rhs, double **xyz) {
    GUARD_BEGIN
    std::unique_ptr<samg_problem> pb(samgb::generate_hex(*p));
    *n = pb->n;
    *nnodes = pb->nnodes;
    *ptr = dup(pb->ptr);
    *col = dup(pb->col);
    *val = dup(pb->val);
    *rhs = dup(pb->rhs);
    *xyz = dup(pb->xyz);
    GUARD_END
}

// kernels::force_isa (kernels.hpp:25-28): 0 = scalar, 1 = avx2 dot/axpby.
// Returns the active ISA after the call (1 avx2, 0 scalar).
int ref_force_isa(int which) {
    kernels::force_isa(which ? kernels::isa::avx2 : kernels::isa::scalar);
    return kernels::active_isa() == kernels::isa::avx2 ? 1 : 0;
}

int ref_rigid_body_modes(int64_t nnodes, const double *xyz, double *B) {
    GUARD_BEGIN
    node_coordinates c;
    c.xyz.assign(xyz, xyz + 3 * nnodes);
    dense_columns D = rigid_body_modes(c);
    std::memcpy(B, D.data.data(), sizeof(double) * D.data.size());
    GUARD_END
}

static void setup_impl(scalar_csr &&A, const double *B, int64_t bcols, double eps_strong,
        double omega, int smoother, double smoother_omega,
        int64_t coarse_enough, double stagnation_ratio, int pipeline_id, void **out) {
    const int64_t n = A.nrows;
    std::optional<dense_columns> Bd;
    if (B) {
        dense_columns D(n, bcols);
        std::memcpy(D.data.data(), B, sizeof(double) * n * bcols);
        Bd = std::move(D);
    }
    amg_params prm;
    prm.coarsening.eps_strong = eps_strong;
    prm.coarsening.omega = omega;
    prm.coarse_enough = coarse_enough;
    prm.stagnation_ratio = stagnation_ratio;
    prm.smoother = smoother == SM_ILU0 ? smoother_kind::ilu0 : smoother_kind::jacobi;

    auto h = std::make_unique<ref_handle>();
    h->smoother = smoother;
    h->smoother_omega = smoother_omega;
    auto t0 = clk::now();
    // samg::pipeline numbering (hierarchy.hpp:30): 0 scalar, 1 block,
    // 2 ns_scalar, 3 ns_hybrid1, 4 ns_hybrid2, 5 ns_block
    const pipeline pl = pipeline_id == 0 ? pipeline::scalar
                      : pipeline_id == 1 ? pipeline::block
                      : pipeline_id == 2 ? pipeline::ns_scalar
                      : pipeline_id == 3 ? pipeline::ns_hybrid1
                      : pipeline_id == 4 ? pipeline::ns_hybrid2 : pipeline::ns_block;
    const bool scalar_levels = pl == pipeline::scalar || pl == pipeline::ns_scalar;
    h->H = setup(A, Bd, pl, prm);
    const samg::index L = h->H.nlevels();
    // Smoother override through the public level members.
    h->sm.resize(L);
    for (samg::index l = 0; l + 1 < L; ++l) {
        if (scalar_levels) {  // the reference's scalar smoothers only
            if (smoother == SM_JACOBI && smoother_omega != damped_jacobi::default_damping)
                h->H.levels[l].smoother =
                    damped_jacobi(std::get<scalar_csr>(h->H.levels[l].A), smoother_omega);
            else if (smoother != SM_JACOBI && smoother != SM_ILU0)
                throw error("scalar pipelines: block smoothers are not defined");
            continue;
        }
        const csr<block3> &Al = blk(h->H.levels[l].A);
        if (smoother == SM_JACOBI && smoother_omega != damped_jacobi::default_damping) {
            h->H.levels[l].smoother = damped_jacobi(Al, smoother_omega);
        } else if (smoother == SM_SPAI0 || smoother == SM_BLOCK_JACOBI) {
            std::vector<double> &M = h->sm[l];
            M.assign(Al.nrows * 9, 0.0);
            for (samg::index i = 0; i < Al.nrows; ++i) {
                samg::index dg = -1;
                double den = 0.0;
                for (samg::index j = Al.ptr[i]; j < Al.ptr[i + 1]; ++j) {
                    if (Al.col[j] == i) dg = j;
                    for (int e = 0; e < 9; ++e) den += Al.val[j].m[e] * Al.val[j].m[e];
                }
                if (dg < 0) throw missing_diagonal("block smoother: structurally zero diagonal");
                if (smoother == SM_SPAI0) {
                    if (den == 0.0) throw zero_diagonal("spai0: zero row");
                    for (int e = 0; e < 9; ++e) M[i * 9 + e] = Al.val[dg].m[e] / den;
                } else {
                    block3 inv = inverse(Al.val[dg]);
                    for (int e = 0; e < 9; ++e) M[i * 9 + e] = smoother_omega * inv.m[e];
                }
            }
        }
    }
    h->setup_seconds = std::chrono::duration<double>(clk::now() - t0).count();
    // Aggregates per level, re-derived with the public API exactly as the
    // as_scalar_transfer wrapper computes them (pbs 3 then 6).
    h->agg.resize(L);
    h->agg_count.assign(L, 0);
    for (samg::index l = 0; l + 1 < L; ++l) {
        adjacency G;
        if (pl == pipeline::block) {  // block_transfer_operators, coarsening.hpp:471
            G = strength_graph(blk(h->H.levels[l].A), eps_strong, 1);
        } else if (scalar_levels) {  // scalar_setup (hierarchy.hpp:234-259)
            const int pbs = (l == 0 || pl == pipeline::scalar) ? 3 : static_cast<int>(bcols);
            G = strength_graph(std::get<scalar_csr>(h->H.levels[l].A), eps_strong, pbs);
        } else {
            scalar_csr S = to_scalar(blk(h->H.levels[l].A));
            const int pbs = l == 0 ? 3 : static_cast<int>(bcols);
            G = strength_graph(S, eps_strong, pbs);
        }
        aggregates a = aggregate(G);
        h->agg[l] = a.id;
        h->agg_count[l] = a.count;
    }
    if (scalar_levels) {
        h->blockview.resize(L);
        for (samg::index l = 0; l < L; ++l) {
            const samg::level &lv = h->H.levels[l];
            h->blockview[l][0] = to_block<3>(std::get<scalar_csr>(lv.A));
            if (lv.has_transfer) {
                h->blockview[l][1] = to_block<3>(std::get<scalar_csr>(lv.P));
                h->blockview[l][2] = to_block<3>(std::get<scalar_csr>(lv.R));
            }
        }
    }
    *out = h.release();
}

int ref_setup(int64_t n, const int64_t *ptr, const int64_t *col,
        const double *val, const double *B, int64_t bcols, double eps_strong,
        double omega, int smoother, double smoother_omega,
        int64_t coarse_enough, double stagnation_ratio, int pipeline_id, void **out) {
    GUARD_BEGIN
    scalar_csr A;
    A.nrows = A.ncols = n;
    A.ptr.assign(ptr, ptr + n + 1);
    A.col.assign(col, col + ptr[n]);
    A.val.assign(val, val + ptr[n]);
    setup_impl(std::move(A), B, bcols, eps_strong, omega, smoother, smoother_omega,
               coarse_enough, stagnation_ratio, pipeline_id, out);
    GUARD_END
}

// The same from a 3x3 BSR input: the scalar CSR the reference's setup takes
// is formed by its own to_scalar (csr.hpp:327-353, every block entry kept),
// which is what the host generator's scalar view is -- without holding a
// second scalar copy on the Python side (C3: 8 GB).
int ref_setup_bsr3(int64_t nbrows, const int64_t *ptr, const int64_t *col,
        const double *val, const double *B, int64_t bcols, double eps_strong,
        double omega, int smoother, double smoother_omega,
        int64_t coarse_enough, double stagnation_ratio, int pipeline_id, void **out) {
    GUARD_BEGIN
    scalar_csr A;
    {
        csr<block3> Ab;
        Ab.nrows = Ab.ncols = nbrows;
        Ab.ptr.assign(ptr, ptr + nbrows + 1);
        Ab.col.assign(col, col + ptr[nbrows]);
        Ab.val.resize(ptr[nbrows]);
        std::memcpy(Ab.val.data(), val, sizeof(double) * 9 * ptr[nbrows]);
        A = to_scalar(Ab);
    }
    setup_impl(std::move(A), B, bcols, eps_strong, omega, smoother, smoother_omega,
               coarse_enough, stagnation_ratio, pipeline_id, out);
    GUARD_END
}

void ref_destroy(void *h) { delete static_cast<ref_handle *>(h); }

int ref_nlevels(void *hp) { return static_cast<int>(static_cast<ref_handle *>(hp)->H.nlevels()); }
double ref_setup_seconds(void *hp) { return static_cast<ref_handle *>(hp)->setup_seconds; }
int64_t ref_coarse_dim(void *hp) { return static_cast<ref_handle *>(hp)->H.coarsest.dim(); }
uint64_t ref_memory_footprint(void *hp) {
    auto *h = static_cast<ref_handle *>(hp);
    uint64_t bytes = memory_footprint(h->H);
    // harness smoothers replace the damped_jacobi placeholders in the count
    if (uses_harness(*h))
        for (samg::index l = 0; l + 1 < h->H.nlevels(); ++l)
            bytes = bytes - blk(h->H.levels[l].A).nrows * 3 * 8 + h->sm[l].size() * 8;
    return bytes;
}

// which: 0=A 1=P 2=R; pointers stay owned by the hierarchy
int ref_level_matrix(void *hp, int level, int which, int64_t *nrows,
        int64_t *ncols, const int64_t **ptr, const int64_t **col,
        const double **val) {
    auto *h = static_cast<ref_handle *>(hp);
    if (level < 0 || level >= h->H.nlevels()) return 1;
    const samg::level &lv = h->H.levels[level];
    if (which != 0 && !lv.has_transfer) return 1;
    const csr<block3> &M = h->blockview.empty() ? blk(which == 0 ? lv.A : which == 1 ? lv.P : lv.R)
                                                : h->blockview[level][which];
    *nrows = M.nrows;
    *ncols = M.ncols;
    *ptr = M.ptr.data();
    *col = M.col.data();
    *val = reinterpret_cast<const double *>(M.val.data());
    static_assert(sizeof(block3) == 72, "block layout");
    return 0;
}

// ilu0<block3> factors and inverted pivots of a level (relaxation.hpp:90-92)
int ref_ilu_factors(void *hp, int level, int64_t *nnz, int64_t *nrows, const double **lu,
        const double **inv) {
    auto *h = static_cast<ref_handle *>(hp);
    if (level < 0 || level + 1 >= h->H.nlevels()) return 1;
    // ilu0<double>: the scalar factors re-blocked (to_block<3>: the scalar
    // pattern is whole blocks), the 3 scalar pivots per block row as they are
    if (const auto *ss = std::get_if<ilu0<double>>(&h->H.levels[level].smoother)) {
        h->ilu_blockview.resize(h->H.nlevels());
        csr<block3> &fb = h->ilu_blockview[level];
        fb = to_block<3>(ss->factors());
        *nnz = static_cast<int64_t>(fb.val.size());
        *nrows = static_cast<int64_t>(ss->inverted_pivots().size()) / 3;
        *lu = reinterpret_cast<const double *>(fb.val.data());
        *inv = ss->inverted_pivots().data();
        return 0;
    }
    const auto *sm = std::get_if<ilu0<block3>>(&h->H.levels[level].smoother);
    if (!sm) return 1;
    *nnz = static_cast<int64_t>(sm->factors().val.size());
    *nrows = static_cast<int64_t>(sm->inverted_pivots().size());
    *lu = reinterpret_cast<const double *>(sm->factors().val.data());
    *inv = reinterpret_cast<const double *>(sm->inverted_pivots().data());
    return 0;
}

int ref_aggregates(void *hp, int level, int64_t *nnodes, const int64_t **id,
        int64_t *count) {
    auto *h = static_cast<ref_handle *>(hp);
    if (level < 0 || level + 1 >= h->H.nlevels()) return 1;
    *nnodes = static_cast<int64_t>(h->agg[level].size());
    *id = h->agg[level].data();
    *count = h->agg_count[level];
    return 0;
}

int ref_vcycle(void *hp, const double *f, double *u) {
    GUARD_BEGIN
    auto *h = static_cast<ref_handle *>(hp);
    const samg::index n = h->H.finest_dim();
    vcycle_workspace ws(h->H);
    if (uses_harness(*h))
        harness_vcycle(*h, std::span<const double>(f, n), std::span<double>(u, n), ws);
    else
        vcycle(h->H, std::span<const double>(f, n), std::span<double>(u, n), ws);
    GUARD_END
}

int ref_cg_solve(void *hp, const double *f, double *u, double tol, int maxit,
        int *iterations, double *rel_res, int *converged, double *solve_s) {
    GUARD_BEGIN
    auto *h = static_cast<ref_handle *>(hp);
    const samg::index n = h->H.finest_dim();
    cg_params prm{tol, maxit};
    std::span<const double> fs(f, n);
    std::span<double> us(u, n);
    auto t0 = clk::now();
    solve_report rep;
    if (!uses_harness(*h)) {
        rep = cg_solve(h->H, fs, us, prm);
    } else {
        vcycle_workspace ws(h->H);
        const any_matrix &A0 = h->H.levels.front().A;
        rep = cg_solve_op(n,
            [&](std::span<const double> x, std::span<double> y) { any_spmv(1.0, A0, x, 0.0, y); },
            [&](std::span<const double> r, std::span<double> z) {
                std::fill(z.begin(), z.end(), 0.0);
                harness_vcycle(*h, r, z, ws);
            },
            fs, us, prm);
        std::vector<double> res(f, f + n);
        any_spmv(-1.0, A0, us, 1.0, res);
        double nf = kernels::norm2(fs);
        rep.relative_residual = nf > 0 ? kernels::norm2(res) / nf : 0.0;
    }
    *solve_s = std::chrono::duration<double>(clk::now() - t0).count();
    *iterations = rep.iterations;
    *rel_res = rep.relative_residual;
    *converged = rep.converged ? 1 : 0;
    GUARD_END
}

// spmv<block3> (csr.hpp:129-160) on a level matrix: the CPU baseline kernel.
int ref_spmv(void *hp, int level, double alpha, const double *x, double beta,
        double *y) {
    GUARD_BEGIN
    auto *h = static_cast<ref_handle *>(hp);
    const csr<block3> &A = blk(h->H.levels[level].A);
    spmv(alpha, A, std::span<const double>(x, A.scalar_cols()), beta,
            std::span<double>(y, A.scalar_rows()));
    GUARD_END
}

// A reference csr<static_block<3>> built once (timed spmv baseline).
void *ref_bsr3_create(int64_t nrows, int64_t ncols, const int64_t *ptr, const int64_t *col,
        const double *val) {
    auto *A = new csr<block3>;
    A->nrows = nrows;
    A->ncols = ncols;
    A->ptr.assign(ptr, ptr + nrows + 1);
    A->col.assign(col + ptr[0], col + ptr[nrows]);
    for (auto &p : A->ptr) p -= ptr[0];
    A->val.resize(A->col.size());
    std::memcpy(A->val.data(), val + 9 * ptr[0], sizeof(double) * 9 * A->col.size());
    return A;
}

void ref_bsr3_destroy(void *A) { delete static_cast<csr<block3> *>(A); }

int ref_bsr3_spmv(void *Ap, double alpha, const double *x, double beta, double *y) {
    GUARD_BEGIN
    const csr<block3> &A = *static_cast<csr<block3> *>(Ap);
    spmv(alpha, A, std::span<const double>(x, A.scalar_cols()), beta,
            std::span<double>(y, A.scalar_rows()));
    GUARD_END
}

// Standalone spmv on caller-owned BSR3 arrays (no hierarchy).
int ref_spmv_bsr3(int64_t nrows, int64_t ncols, const int64_t *ptr,
        const int64_t *col, const double *val, double alpha, const double *x,
        double beta, double *y) {
    GUARD_BEGIN
    csr<block3> A;
    A.nrows = nrows;
    A.ncols = ncols;
    A.ptr.assign(ptr, ptr + nrows + 1);
    A.col.assign(col, col + ptr[nrows]);
    A.val.resize(ptr[nrows]);
    std::memcpy(A.val.data(), val, sizeof(double) * 9 * ptr[nrows]);
    spmv(alpha, A, std::span<const double>(x, ncols * 3), beta,
            std::span<double>(y, nrows * 3));
    GUARD_END
}

} // extern "C"
