"""C1 host-input setup (samg_setup_bsr3 from pageable numpy arrays) timed
several times; run under different SAMG_H2D_THREADS to compare the staged
upload (SAMG_SETUP_TIMING=1 prints the upload phase)."""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09056_b200 as pb  # noqa: E402

p = pb.generate_hex(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022)
B = p.nullspace()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), B, "ns_block", pb.AmgParams())
    ts.append(time.perf_counter() - t0)
    h.close()
print(os.environ.get("SAMG_H2D_THREADS", "8"), "setup median", round(statistics.median(ts[1:]) * 1e3, 2), "ms",
      [round(t * 1e3, 1) for t in ts], flush=True)
