"""C1 setup with the ILU(0) smoother (run with SAMG_SETUP_TIMING=1)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09056_b200 as pb  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 63
p = pb.generate_hex(nx=nx, ny=nx, nz=nx, dirichlet="eliminate", noise=0.01, seed=2022)
for _ in range(2):
    t0 = time.perf_counter()
    h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), "ns_block",
                      pb.AmgParams(smoother="ilu0"))
    print("setup %.3f s" % (time.perf_counter() - t0), flush=True)
    h.close()
