"""C1 (or nx^3) ILU(0) V-cycles with every launch visible (host-loop CG) --
run under ncu --metrics gpu__time_duration.sum to get per-level sweep times."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SAMG_CG_GRAPH", "0")
import paper_2202_09056_b200 as pb  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 63
its = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = pb.generate_hex(nx=nx, ny=nx, nz=nx, dirichlet="eliminate", noise=0.01, seed=2022)
h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), "ns_block",
                  pb.AmgParams(smoother="ilu0"))
u, rep = h.cg_solve(p.rhs, pb.CgParams(max_iterations=its))
print(rep, [h.level_info(l) for l in range(h.nlevels)])
