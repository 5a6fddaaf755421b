// shim_test.cpp -- the reference-facing C++ interface (include/samg_b200.hpp)
// exercised like the reference's own tests (test_cg.cpp, test_hierarchy.cpp):
// a clamped hex8 problem, setup(ns_block), cg_solve to 1e-8, an independent
// residual check, V-cycle linearity, and the typed exceptions.
#include <cmath>
#include <cstdio>
#include <vector>

#include "samg_b200.hpp"

using namespace samg_b200;

static int failures = 0;
#define EXPECT(c) do { if (!(c)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); ++failures; } } while (0)

int main() {
    samg_problem_params pp;
    samg_default_problem_params(&pp);
    pp.nx = pp.ny = pp.nz = 8;
    pp.dirichlet = SAMG_DIRICHLET_KEEP_ROWS;
    samg_problem *prob = nullptr;
    check(samg_generate_hex(&pp, &prob));
    int64_t n = 0, nnzb = 0, nnodes = 0;
    check(samg_problem_info(prob, &n, &nnzb, &nnodes));
    std::vector<int64_t> ptr(n + 1), col(9 * nnzb);
    std::vector<double> val(9 * nnzb), rhs(n), xyz(3 * nnodes);
    check(samg_problem_get_csr(prob, ptr.data(), col.data(), val.data()));
    check(samg_problem_get_rhs(prob, rhs.data()));
    check(samg_problem_get_coords(prob, xyz.data()));
    samg_problem_destroy(prob);

    scalar_csr A;
    A.nrows = A.ncols = n;
    A.ptr.assign(ptr.begin(), ptr.end());
    A.col.assign(col.begin(), col.end());
    A.val = val;
    dense_columns B(n, 6);
    check(samg_rigid_body_modes(nnodes, xyz.data(), B.data.data()));

    amg_params prm;
    prm.coarse_enough = 300;
    hierarchy H = setup(A, B, pipeline::ns_block, prm);
    EXPECT(H.nlevels() >= 2);
    std::vector<double> u(n, 0.0);
    solve_report rep = cg_solve(H, rhs, u, cg_params{});
    EXPECT(rep.converged);
    EXPECT(rep.relative_residual <= 1e-8);
    EXPECT(rep.preconditioner_bytes == memory_footprint(H));
    // independent residual (test_cg.cpp:73-78)
    double rn = 0, fn = 0;
    for (index i = 0; i < n; ++i) {
        double s = 0;
        for (index j = A.ptr[i]; j < A.ptr[i + 1]; ++j) s += A.val[j] * u[A.col[j]];
        rn += (rhs[i] - s) * (rhs[i] - s);
        fn += rhs[i] * rhs[i];
    }
    EXPECT(std::sqrt(rn / fn) <= 1e-8 * 1.01);
    EXPECT(std::abs(std::sqrt(rn / fn) - rep.relative_residual) <= 1e-10);

    // V-cycle linearity (test_hierarchy.cpp:50-67)
    vcycle_workspace ws(H);
    std::vector<double> u1(n, 0.0), u2(n, 0.0), f2(n);
    for (index i = 0; i < n; ++i) f2[i] = 2.0 * rhs[i];
    vcycle(H, rhs, u1, ws);
    vcycle(H, f2, u2, ws);
    double dmax = 0, umax = 0;
    for (index i = 0; i < n; ++i) {
        dmax = std::fmax(dmax, std::abs(u2[i] - 2.0 * u1[i]));
        umax = std::fmax(umax, std::abs(u1[i]));
    }
    EXPECT(dmax <= 1e-12 * umax);

    // parity tap
    csr<block3> A0 = H.level_matrix(0);
    EXPECT(A0.nrows == n / 3 && A0.nnz() == nnzb);

    // typed errors (test_hierarchy.cpp:392-404)
    bool thrown = false;
    try { setup(A, std::nullopt, pipeline::ns_block, prm); } catch (const bad_nullspace_shape &) { thrown = true; }
    EXPECT(thrown);
    thrown = false;
    try { setup(A, dense_columns(12, 6), pipeline::ns_block, prm); } catch (const bad_nullspace_shape &) { thrown = true; }
    EXPECT(thrown);
    thrown = false;
    {   // block smoothers are defined for block pipelines only
        amg_params ps = prm;
        ps.smoother = smoother_kind::spai0;
        try { setup(A, B, pipeline::ns_scalar, ps); } catch (const unsupported &) { thrown = true; }
    }
    EXPECT(thrown);
    // ns_scalar with its own ilu0<double> smoother (hierarchy.hpp:298-330)
    hierarchy Hs = setup(A, B, pipeline::ns_scalar, prm);
    std::vector<double> us(n, 0.0);
    solve_report rs = cg_solve(Hs, rhs, us, cg_params{});
    EXPECT(rs.converged && rs.relative_residual <= 1e-8);
    EXPECT(rs.variant == pipeline::ns_scalar);
    thrown = false;
    try { std::vector<double> bad(5); cg_solve(H, bad, u, cg_params{}); } catch (const dimension_mismatch &) { thrown = true; }
    EXPECT(thrown);

    // pipeline::block takes no nullspace (hierarchy.hpp:340-347)
    hierarchy Hb = setup(A, std::nullopt, pipeline::block, prm);
    EXPECT(Hb.nlevels() >= 2);
    std::vector<double> ub(n, 0.0);
    solve_report rb = cg_solve(Hb, rhs, ub, cg_params{});
    EXPECT(rb.converged && rb.relative_residual <= 1e-8);
    EXPECT(rb.variant == pipeline::block);

    std::printf("%s: levels=%td iterations=%d relres=%.3e\n", failures ? "FAILED" : "ok",
                H.nlevels(), rep.iterations, rep.relative_residual);
    return failures ? 1 : 0;
}
