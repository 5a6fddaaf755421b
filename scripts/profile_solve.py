"""C1 setup + a few CG iterations (host-loop mode so ncu sees every launch)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2202_09056_b200 as pb  # noqa: E402

its = int(sys.argv[1]) if len(sys.argv) > 1 else 5
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
p = pb.generate_hex(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022)
h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), "ns_block",
                  pb.AmgParams(smoother="spai0", vcycle_precision=prec))
u, rep = h.cg_solve(p.rhs, pb.CgParams(max_iterations=its))
print(rep, [h.level_info(l) for l in range(h.nlevels)])
for l in range(h.nlevels - 1):
    print("P", l, h.level_info(l, 1), "R", h.level_info(l, 2))
