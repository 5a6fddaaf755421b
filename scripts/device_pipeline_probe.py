"""Device-resident pipeline on C1: on-GPU assembly, setup_device, solve."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2202_09056_b200 as pb  # noqa: E402

C1 = dict(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dp = pb.generate_hex_device(**C1)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h = pb.setup_device(dp.A, dp.nullspace_ptr, 6, "ns_block", pb.AmgParams())
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("it", it, "assemble %.4f setup %.4f" % (t1 - t0, t2 - t1), flush=True)
    h.close()
    del dp
