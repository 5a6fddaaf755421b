"""A short host-loop solve of a BASELINE config (a few CG iterations) for ncu captures:
    ncu --set full -k regex:... python scripts/ncu_solve_cfg.py C4 [iters] [smoother]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SAMG_CG_GRAPH", "0")
import torch  # noqa: E402

import paper_2202_09056_b200 as pb  # noqa: E402
from scripts.configs import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
its = int(sys.argv[2]) if len(sys.argv) > 2 else 4
sm = sys.argv[3] if len(sys.argv) > 3 else "spai0"
kw, _ = CONFIGS[name]
dp = pb.generate_hex_device(pb.ProblemParams(**kw), device=0)
h = pb.setup_device(dp.A, dp.nullspace_ptr, 6, "ns_block", pb.AmgParams(smoother=sm))
u = torch.zeros(dp.n, dtype=torch.float64, device="cuda")
rep = h.cg_solve_device(dp.rhs_ptr, u.data_ptr(), pb.CgParams(max_iterations=its))
torch.cuda.synchronize()
print(rep)
