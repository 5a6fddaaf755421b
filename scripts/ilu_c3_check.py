"""C3 (512x64x64 cantilever) with ILU(0): factors per level, one V-cycle and
the first CG iterations, GPU against the reference."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2202_09056_b200 as pb
from oracle.oracle import Ref, Params, SM_ILU0

kw = dict(nx=511, ny=63, nz=63, lx=511 / 63, dirichlet="eliminate", load="traction_xend", x_slowest=True)
p = pb.generate_hex(**kw)
A = p.csr(); B = p.nullspace()
h = pb.setup(A, B, "ns_block", pb.AmgParams(smoother="ilu0"))
print("GPU levels", [h.level_info(l)[0] for l in range(h.nlevels)], flush=True)
for its in (1, 2, 5, 20):
    u, rep = h.cg_solve(p.rhs, pb.CgParams(max_iterations=its))
    print("GPU its", its, "relres", rep["relative_residual"], flush=True)
vg = h.vcycle(p.rhs)
print("GPU vcycle norm", np.linalg.norm(vg), "finite", np.isfinite(vg).all(), "max", np.abs(vg).max(), flush=True)
t0 = time.time()
hr = Ref().setup(A[0], A[1], A[2], A[3], B, Params(smoother=SM_ILU0))
print("REF setup %.0f s" % (time.time() - t0), flush=True)
for l in range(h.nlevels - 1):
    g, r = h.smoother(l), hr.ilu(l)
    same = np.array_equal(g, r)
    print("level", l, "factors", "==" if same else "DIFFER", "max|.|", np.abs(g).max(), np.abs(r).max(), flush=True)
    if not same:
        d = np.nonzero(g != r)[0]
        print("   first diffs at", d[:10], g[d[:5]], r[d[:5]], "count", d.size, flush=True)
vr = hr.vcycle(p.rhs)
print("REF vcycle norm", np.linalg.norm(vr), "rel diff", np.linalg.norm(vg - vr) / np.linalg.norm(vr), flush=True)
ur, rr = hr.cg_solve(p.rhs, max_iterations=5)
print("REF 5 its relres", rr["relative_residual"], flush=True)
