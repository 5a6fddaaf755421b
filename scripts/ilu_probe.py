"""ILU(0) smoother timing on C1: setup (factorization) and CG solve."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09056_b200 as pb  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 63
p = pb.generate_hex(nx=nx, ny=nx, nz=nx, dirichlet="eliminate", noise=0.01, seed=2022)
B = p.nullspace()
for sm in ("ilu0", "spai0"):
    prm = pb.AmgParams(smoother=sm)
    h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), B, "ns_block", prm)
    h.close()
    t0 = time.perf_counter()
    h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), B, "ns_block", prm)
    ts = time.perf_counter() - t0
    u, rep = h.cg_solve(p.rhs, pb.CgParams(max_iterations=3))
    u, rep = h.cg_solve(p.rhs)
    print(sm, "setup %.4f s" % ts, "solve %.4f s" % rep["solve_seconds"], "it", rep["iterations"],
          "%.3f ms/it" % (1e3 * rep["solve_seconds"] / max(rep["iterations"], 1)), flush=True)
    h.close()
