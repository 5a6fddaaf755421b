"""Device-resident setup of a BASELINE config with per-phase timing
(SAMG_SETUP_TIMING=1 prints the phases on stderr), then one solve.

    SAMG_SETUP_TIMING=1 python scripts/setup_phases.py C4
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2202_09056_b200 as pb  # noqa: E402
from scripts.configs import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
kw, _ = CONFIGS[name]
prm = pb.AmgParams(smoother=os.environ.get("SAMG_PROBE_SMOOTHER", "spai0"))
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dp = pb.generate_hex_device(pb.ProblemParams(**kw), device=0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h = pb.setup_device(dp.A, dp.nullspace_ptr, 6, "ns_block", prm)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name} run {rep}: assemble {t1 - t0:.3f} s setup {t2 - t1:.3f} s levels "
          f"{[h.level_info(l)[0] for l in range(h.nlevels)]}", flush=True)
    if rep == 1:
        u = torch.zeros(dp.n, dtype=torch.float64, device="cuda")
        t0 = time.perf_counter()
        r = h.cg_solve_device(dp.rhs_ptr, u.data_ptr())
        torch.cuda.synchronize()
        print(f"solve {time.perf_counter() - t0:.3f} s its {r['iterations']}", flush=True)
    h.close()
    del dp
