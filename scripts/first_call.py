"""First-call latency of the drop-in path in a fresh process: library load,
the first samg_setup (staging pool, memory pool growth, lazy module loading
included) and the first samg_cg_solve, then the same calls again.

    python scripts/first_call.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
t0 = time.perf_counter()
import paper_2202_09056_b200 as pb  # noqa: E402
t1 = time.perf_counter()
p = pb.generate_hex(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022)
A, B = p.csr(), p.nullspace()
pb.device_count()
t2 = time.perf_counter()
for k in range(3):
    a = time.perf_counter()
    h = pb.setup(A, B, "ns_block", pb.AmgParams(smoother="spai0"))
    b = time.perf_counter()
    u, rep = h.cg_solve(p.rhs)
    c = time.perf_counter()
    h.close()
    print(f"call {k}: setup {b - a:.4f} s solve {c - b:.4f} s ({rep['iterations']} its)", flush=True)
print(f"import {t1 - t0:.3f} s, generate + device init {t2 - t1:.3f} s")
