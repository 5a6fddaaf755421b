"""Per-kernel GPU time of the CG iteration with warm caches (unlike ncu's
per-kernel cache flush): CUPTI kernel records via torch.profiler around one
whole solve in host-loop mode (SAMG_CG_GRAPH=0: the kernels of the graph's
conditional body are not reported by CUPTI).  Kernels are grouped by name; per-iteration time =
total / iterations for kernels launched once per iteration.

    python scripts/iter_timeline.py [C1|C4] [smoother] [--json OUT] [ENV=V ...]"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
args = [a for a in sys.argv[1:]]
out_json = None
if "--json" in args:
    i = args.index("--json")
    out_json = args[i + 1]
    del args[i:i + 2]
os.environ.setdefault("SAMG_CG_GRAPH", "0")
for a in [a for a in args if "=" in a]:
    k, v = a.split("=", 1)
    os.environ[k] = v
    args.remove(a)
cfg = args[0] if args else "C1"
smoother = args[1] if len(args) > 1 else "spai0"
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2202_09056_b200 as pb  # noqa: E402

C = {"C1": dict(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022),
     "C4": dict(nx=199, ny=199, nz=199, dirichlet="eliminate", noise=0.01, seed=2022)}[cfg]
dp = pb.generate_hex_device(pb.ProblemParams(**C), device=0)
h = pb.setup_device(dp.A, dp.nullspace_ptr, 6, "ns_block", pb.AmgParams(smoother=smoother,
                                 ilu_sweep_order=os.environ.get("SAMG_ILU_ORDER", "reference")))
u = torch.zeros(dp.n, dtype=torch.float64, device="cuda")
for _ in range(2):
    rep = h.cg_solve_device(dp.rhs_ptr, u.data_ptr())
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
    rep = h.cg_solve_device(dp.rhs_ptr, u.data_ptr())
    torch.cuda.synchronize()
its = rep["iterations"]
tot = collections.defaultdict(float)
cnt = collections.Counter()
t_first, t_last = None, None
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    name = e.name.replace("(anonymous namespace)::", "").split("(")[0].replace("samgb::", "")
    name = name.replace("<unnamed>::", "").replace("void ", "")
    tot[name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    cnt[name] += 1
    s0 = e.time_range.start
    s1 = e.time_range.end
    t_first = s0 if t_first is None else min(t_first, s0)
    t_last = s1 if t_last is None else max(t_last, s1)
rows = sorted(tot.items(), key=lambda kv: -kv[1])
busy = sum(tot.values())
print(f"{cfg}: {its} iterations, solve {rep['solve_seconds'] * 1e3:.2f} ms, "
      f"kernel busy {busy / 1e3:.2f} ms, span {(t_last - t_first) / 1e3:.2f} ms")
res = []
for n, t in rows:
    print(f"{t / its:9.2f} us/it  n={cnt[n]:6d}  {t / cnt[n]:8.2f} us/launch  {n[:100]}")
    res.append({"kernel": n[:120], "us_per_iteration": t / its, "launches": cnt[n],
                "us_per_launch": t / cnt[n]})
# one iteration in launch order (between the 2nd and 3rd q = A p kernels)
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
marks = [k for k, e in enumerate(evs) if "EpiDot" in e.name]
if len(marks) >= 3:
    print("one iteration in launch order:")
    for e in evs[marks[1]:marks[2]]:
        nm = e.name.replace("(anonymous namespace)::", "").split("(")[0].replace("samgb::", "").replace("void ", "")
        print(f"   {(e.time_range.end - e.time_range.start):9.2f} us  {nm[:90]}")
if out_json:
    json.dump({"config": cfg, "iterations": its, "solve_ms": rep["solve_seconds"] * 1e3,
               "busy_ms": busy / 1e3, "span_ms": (t_last - t_first) / 1e3, "kernels": res},
              open(out_json, "w"), indent=1)
