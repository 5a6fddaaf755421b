"""ILU(0) convergence on a mid-size cantilever (x slowest), GPU vs reference."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2202_09056_b200 as pb
from oracle.oracle import Ref, Params, SM_ILU0

for kw in [dict(nx=127, ny=31, nz=31, lx=127 / 31, dirichlet="eliminate", load="traction_xend", x_slowest=True),
           dict(nx=127, ny=31, nz=31, lx=127 / 31, dirichlet="eliminate", load="traction_xend", x_slowest=False)]:
    p = pb.generate_hex(**kw)
    A = p.csr(); B = p.nullspace()
    h = pb.setup(A, B, "ns_block", pb.AmgParams(smoother="ilu0"))
    u, rep = h.cg_solve(p.rhs, pb.CgParams(max_iterations=400))
    print("GPU", kw["x_slowest"], [h.level_info(l)[0] for l in range(h.nlevels)], rep["iterations"], rep["relative_residual"], flush=True)
    inv = [np.abs(h.smoother(l)[:9 * h.level_info(l)[0]]).max() for l in range(h.nlevels - 1)]
    print("  max |U_kk^-1| per level (first 9n entries)", ["%.2e" % v for v in inv], flush=True)
    t0 = time.time()
    hr = Ref().setup(A[0], A[1], A[2], A[3], B, Params(smoother=SM_ILU0))
    ur, rr = hr.cg_solve(p.rhs, max_iterations=400)
    print("REF", rr["iterations"], rr["relative_residual"], rr["converged"], "%.0f s" % (time.time() - t0), flush=True)
