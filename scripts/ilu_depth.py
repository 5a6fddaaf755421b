"""Dependency depth of the ILU(0) sweeps per level of the C1 hierarchy."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09056_b200 as pb  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 63
p = pb.generate_hex(nx=nx, ny=nx, nz=nx, dirichlet="eliminate", noise=0.01, seed=2022)
h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), "ns_block",
                  pb.AmgParams())
for l in range(h.nlevels - 1):
    nr, nc, ptr, col, val = h.level(l, 0)
    lev = np.zeros(nr, np.int64)
    for i in range(nr):
        c = col[ptr[i]:ptr[i + 1]]
        d = c[c < i]
        lev[i] = lev[d].max() + 1 if d.size else 0
    print(f"level {l}: rows {nr}, blocks/row {ptr[-1] / nr:.1f}, forward depth {lev.max() + 1}, "
          f"rows per level {nr / (lev.max() + 1):.1f}", flush=True)
