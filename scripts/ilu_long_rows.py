"""ILU(0) on hierarchies with long coarse rows (> 96 dependencies per
triangle, > 192 blocks per row): factors vs the reference, and solves."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2202_09056_b200 as pb
from oracle.oracle import Ref, Params, SM_ILU0

for nx, ce in [(12, 30), (16, 30), (20, 60), (24, 60)]:
    p = pb.generate_hex(nx=nx, ny=nx, nz=nx, dirichlet="eliminate", noise=0.01, seed=5)
    A = p.csr(); B = p.nullspace()
    h = pb.setup(A, B, "ns_block", pb.AmgParams(smoother="ilu0", coarse_enough=ce))
    hr = Ref().setup(A[0], A[1], A[2], A[3], B, Params(smoother=SM_ILU0, coarse_enough=ce))
    info = []
    ok = True
    for l in range(h.nlevels - 1):
        nr, nc, ptr, col, val = h.level(l, 0)
        mx = int(np.diff(ptr).max())
        same = np.array_equal(h.smoother(l), hr.ilu(l))
        ok &= same
        info.append(f"L{l}: {nr} rows, max {mx} blocks/row, factors {'==' if same else 'DIFFER'}")
    u, rep = h.cg_solve(p.rhs)
    ur, rr = hr.cg_solve(p.rhs)
    vg, vr = h.vcycle(p.rhs), hr.vcycle(p.rhs)
    print(nx, ce, "; ".join(info), f"| its {rep['iterations']} vs {rr['iterations']}, relres {rep['relative_residual']:.2e}, "
          f"vcycle rel diff {np.linalg.norm(vg - vr) / np.linalg.norm(vr):.1e}", flush=True)
