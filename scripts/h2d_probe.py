"""H2D bandwidth probe: pageable vs pinned (torch), and C1 upload vs setup split."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_09056_b200 as pb  # noqa: E402

n = 512 * 2**20 // 8
a = np.random.default_rng(0).uniform(size=n)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for kind in ("pageable", "pinned"):
    src = torch.from_numpy(a) if kind == "pageable" else torch.from_numpy(a).pin_memory()
    for _ in range(2):
        d.copy_(src)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        d.copy_(src)
    torch.cuda.synchronize()
    print(kind, "%.1f GB/s" % (5 * 8 * n / (time.perf_counter() - t0) / 1e9))
p = pb.generate_hex(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022)
v = p.val.reshape(-1)
for _ in range(2):
    A = pb.Bsr3.from_host(p.nbrows, p.nbrows, p.ptr, p.col, v)
    del A
torch.cuda.synchronize()
t0 = time.perf_counter()
A = pb.Bsr3.from_host(p.nbrows, p.nbrows, p.ptr, p.col, v)
torch.cuda.synchronize()
print("upload C1 %.4f s" % (time.perf_counter() - t0))
B = p.nullspace()
prm = pb.AmgParams()
h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, v, B, "ns_block", prm)
h.close()
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, v, B, "ns_block", prm)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    h.close()
print("setup C1", ["%.4f" % t for t in ts])
