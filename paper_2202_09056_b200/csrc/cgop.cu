// cgop.cu -- the generic PCG driver cg_solve_op (cg.hpp:39-83) with caller
// operators: y = A x and z = M r are callbacks on device vectors, the CG
// vector work runs on the device (the fused dot / update kernels of
// solve.cu, deterministic reductions), the scalars are read once per
// iteration (the loop condition needs them on the host to call back).
#include <chrono>
#include <cmath>

#include "kernels.cuh"

namespace samgb {

samg_solve_report cg_solve_op(int64_t n, samg_apply_fn apply_A, samg_apply_fn apply_M, void *ctx,
                              const double *d_f, double *d_u, const samg_cg_params &prm,
                              cudaStream_t s) {
    NvtxScope nvtx_scope("samg::cg_solve_op");
    const auto t0 = std::chrono::steady_clock::now();
    samg_solve_report rep{};
    DevBuf<double> r(n + 2, s), z(n + 2, s), p(n + 2, s), q(n + 2, s), partials(4096, s);
    DevBuf<CgScalars> sc(1, s);
    CgScalars *h = static_cast<CgScalars *>(pinned_small_alloc(sizeof(CgScalars)));
    struct Free { CgScalars *p; ~Free() { pinned_small_free(p); } } free_h{h};
    CK(cudaMemsetAsync(sc.p, 0, sizeof(CgScalars), s));
    CK(cudaMemcpyAsync(r.p, d_f, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    launch_fill(n, 0.0, d_u, s);
    auto read = [&] {
        CK(cudaMemcpyAsync(h, sc.p, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    };
    // the callbacks see their inputs complete; their outputs must be
    // complete on return or enqueued on s
    auto call = [&](samg_apply_fn fn, const double *in, double *out) {
        CK(cudaStreamSynchronize(s));
        if (!fn) {  // identity preconditioner = copy (cg.hpp:37-38)
            CK(cudaMemcpyAsync(out, in, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
            return;
        }
        const int rc = fn(ctx, in, out, s);
        if (rc != 0) fail(rc, "cg_solve_op: operator callback returned an error");
    };
    auto finish = [&] {
        rep.solve_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        CK(cudaStreamSynchronize(s));
        return rep;
    };
    launch_dot(n, d_f, d_f, partials.p, sc.p, CG_RR, s);
    read();
    const double norm_f = std::sqrt(h->rr);
    if (norm_f == 0.0) {
        rep.converged = 1;
        return finish();
    }
    call(apply_M, r.p, z.p);
    CK(cudaMemcpyAsync(p.p, z.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    launch_dot(n, r.p, z.p, partials.p, sc.p, CG_RHO, s);
    double res_norm = norm_f;
    int iter = 0;
    while (res_norm / norm_f > prm.tol && iter < prm.max_iterations) {
        call(apply_A, p.p, q.p);
        launch_dot(n, p.p, q.p, partials.p, sc.p, CG_PQ, s);          // alpha = rho / p'q
        launch_cg_update(n, sc.p, p.p, q.p, d_u, r.p, partials.p, CG_RR, 0, s);
        read();
        if (h->breakdown) fail(SAMG_BREAKDOWN_NON_SPD, "cg: p'Ap <= 0, matrix or preconditioner not SPD");
        ++iter;
        res_norm = std::sqrt(h->rr);
        if (res_norm / norm_f <= prm.tol) break;
        call(apply_M, r.p, z.p);
        launch_dot(n, r.p, z.p, partials.p, sc.p, CG_RZ, s);          // beta, rho
        launch_p_update(n, sc.p, z.p, p.p, s);
    }
    rep.iterations = iter;
    rep.converged = res_norm / norm_f <= prm.tol;
    rep.relative_residual = res_norm / norm_f;  // the recurrence residual (cg.hpp:80)
    return finish();
}

} // namespace samgb
