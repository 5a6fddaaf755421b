"""C1 setup once, then the SPAI0-PCG solve 5 times: min / median solve seconds
(used by scripts/solve_sweep.sh to compare SpMV dispatch settings)."""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09056_b200 as pb  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
p = pb.generate_hex(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022)
h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), "ns_block",
                  pb.AmgParams(smoother="spai0", vcycle_precision=prec))
ts, its = [], None
for _ in range(6):
    t0 = time.perf_counter()
    u, rep = h.cg_solve(p.rhs)
    ts.append(time.perf_counter() - t0)
    its = rep["iterations"]
ts = ts[1:]
env = {k: v for k, v in os.environ.items() if k.startswith("SAMG_")}
print(f"{env} solve min {min(ts)*1e3:.2f} ms med {statistics.median(ts)*1e3:.2f} ms "
      f"its {its} per-it {min(ts)/its*1e6:.1f} us")
