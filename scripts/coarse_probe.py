"""Time the coarsest-level inverse of C1 alone (samg_bsr3_dense_inverse)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2202_09056_b200 as pb  # noqa: E402

p = pb.generate_hex(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022)
h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), "ns_block",
                  pb.AmgParams())
Ac = h.level_matrix(h.nlevels - 1)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for _ in range(reps):
    t0 = time.perf_counter()
    X = Ac.dense_inverse()
    print("dense_inverse n=%d: %.2f ms (incl. D2H of %.0f MB)" % (X.shape[0], 1e3 * (time.perf_counter() - t0), X.nbytes / 1e6))
