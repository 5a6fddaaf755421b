"""ILU(0) setup + a few V-cycles on an nx^3 cube; prints wall times."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09056_b200 as pb  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 63
p = pb.generate_hex(nx=nx, ny=nx, nz=nx, dirichlet="eliminate", noise=0.01, seed=2022)
t0 = time.perf_counter()
h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), "ns_block",
                  pb.AmgParams(smoother="ilu0"))
t1 = time.perf_counter()
h.vcycle(p.rhs)
t2 = time.perf_counter()
for _ in range(3):
    h.vcycle(p.rhs)
t3 = time.perf_counter()
print("nx", nx, "setup %.3f s" % (t1 - t0), "vcycle %.2f ms" % ((t3 - t2) / 3 * 1e3), flush=True)
