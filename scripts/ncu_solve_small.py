"""A short host-loop C1 solve (a few CG iterations) for ncu captures of the
V-cycle kernels:  ncu --set full -k regex:... python scripts/ncu_solve_small.py [iters]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SAMG_CG_GRAPH", "0")
import torch  # noqa: E402

import paper_2202_09056_b200 as pb  # noqa: E402

its = int(sys.argv[1]) if len(sys.argv) > 1 else 6
dp = pb.generate_hex_device(pb.ProblemParams(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022), device=0)
sm = sys.argv[2] if len(sys.argv) > 2 else None
h = pb.setup_device(dp.A, dp.nullspace_ptr, 6, "ns_block", pb.AmgParams(smoother=sm) if sm else pb.AmgParams())
u = torch.zeros(dp.n, dtype=torch.float64, device="cuda")
rep = h.cg_solve_device(dp.rhs_ptr, u.data_ptr(), pb.CgParams(max_iterations=its))
torch.cuda.synchronize()
print(rep)
