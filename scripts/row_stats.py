"""Row-length statistics (blocks per row) of every operator of the C1
hierarchy: mean, percentiles, max, and the share of 8 / 4 / 2-row chunks
above 1.1x / 1.25x the mean (the TMA stage capacity rule)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09056_b200 as pb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
n = {"C1": 63, "C0": 19, "C4": 199}[cfg]
dp = pb.generate_hex_device(pb.ProblemParams(nx=n, ny=n, nz=n, dirichlet="eliminate", noise=0.01, seed=2022), device=0)
h = pb.setup_device(dp.A, dp.nullspace_ptr, 6, "ns_block", pb.AmgParams())
for l in range(h.nlevels):
    for w, name in ((0, "A"), (1, "P"), (2, "R")):
        if w and l == h.nlevels - 1:
            continue
        M = h.level_matrix(l, w)
        nr, nc, nz = M.shape
        if nz > 50_000_000:
            continue
        _, _, ptr, _, _ = M.download()
        ln = np.diff(ptr)
        mean = ln.mean()
        s = f"{name}{l} rows {nr} mean {mean:.1f} p50 {np.percentile(ln, 50):.0f} p90 {np.percentile(ln, 90):.0f} p99 {np.percentile(ln, 99):.0f} max {ln.max()}"
        for rpc in (8, 4, 2):
            m = nr // rpc * rpc
            ch = ln[:m].reshape(-1, rpc).sum(1)
            s += f" | rpc{rpc}: >1.1x {np.mean(ch > rpc * (np.ceil(mean * 1.1) + 1)):.2f} >1.25x {np.mean(ch > rpc * (np.ceil(mean * 1.25) + 1)):.2f}"
        print(s, flush=True)
