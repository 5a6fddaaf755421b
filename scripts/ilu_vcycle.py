"""A few V-cycles with the ILU(0) smoother (for ncu launch lists)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09056_b200 as pb  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 19
p = pb.generate_hex(nx=nx, ny=nx, nz=nx, dirichlet="eliminate", noise=0.01, seed=2022)
h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), "ns_block",
                  pb.AmgParams(smoother="ilu0"))
for _ in range(2):
    u = h.vcycle(p.rhs)
print("ok", u[:3])
