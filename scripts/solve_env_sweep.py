"""C1 SPAI0 solve time under solve-path environment switches, one process
per setting (the switches are read once per process).

    python scripts/solve_env_sweep.py [config=C1] 'ENV=V ENV2=W' ...
Prints one JSON line per setting: median of 5 solves (CUDA-graph CG)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, statistics, sys, time
sys.path.insert(0, %r)
import numpy as np, torch
import paper_2202_09056_b200 as pb
C = {"C1": dict(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022),
     "C3": dict(nx=511, ny=63, nz=63, lx=511 / 63, dirichlet="eliminate", load="traction_xend", x_slowest=True),
     "C4": dict(nx=199, ny=199, nz=199, dirichlet="eliminate", noise=0.01, seed=2022)}[%r]
dp = pb.generate_hex_device(pb.ProblemParams(**C), device=0)
h = pb.setup_device(dp.A, dp.nullspace_ptr, 6, "ns_block", pb.AmgParams(smoother=os.environ.get("SWEEP_SMOOTHER", "spai0"),
                                 ilu_sweep_order=os.environ.get("SAMG_ILU_ORDER", "reference")))
u = torch.zeros(dp.n, dtype=torch.float64, device="cuda")
ts, its = [], None
for k in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rep = h.cg_solve_device(dp.rhs_ptr, u.data_ptr())
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print(json.dumps({"solve_s": statistics.median(ts[1:]), "iterations": rep["iterations"],
                  "ms_per_it": 1e3 * statistics.median(ts[1:]) / rep["iterations"],
                  "relres": rep["relative_residual"], "all": ts}))
'''
cfg = "C1"
args = sys.argv[1:]
if args and args[0] in ("C1", "C3", "C4"):
    cfg, args = args[0], args[1:]
for setting in args or [""]:
    env = dict(os.environ)
    for kv in setting.split():
        k, v = kv.split("=", 1)
        env[k] = v
    out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg)], env=env, capture_output=True,
                         text=True)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
    print(json.dumps({"config": cfg, "env": setting, "result": line}), flush=True)
