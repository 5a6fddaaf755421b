"""Which smoother converges on C2 (96^3 heterogeneous cube)?  One JSON line
per (smoother, omega): GPU setup + CG (rtol 1e-8, up to --maxit iterations)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09056_b200 as pb  # noqa: E402

KW = dict(nx=95, ny=95, nz=95, dirichlet="eliminate", heterogeneous=True, load="random", seed=2022)
maxit = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
p = pb.generate_hex(**KW)
B = p.nullspace()
for sm, om in [("jacobi", 0.5), ("jacobi", 0.4), ("jacobi", 0.3), ("jacobi", 0.6),
               ("block_jacobi", 0.5), ("block_jacobi", 0.7), ("spai0", 0.72), ("ilu0", 0.72)]:
    rec = {"smoother": sm, "omega": om}
    try:
        t0 = time.perf_counter()
        h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), B, "ns_block",
                          pb.AmgParams(smoother=sm, smoother_omega=om))
        rec["setup_s"] = time.perf_counter() - t0
        u, rep = h.cg_solve(p.rhs, pb.CgParams(max_iterations=maxit))
        rec.update(iterations=rep["iterations"], converged=rep["converged"],
                   relres=rep["relative_residual"], solve_s=rep["solve_seconds"])
        h.close()
    except Exception as e:
        rec["error"] = str(e)
    print(json.dumps(rec), flush=True)
