"""Time y = A x for every operator of the C1 hierarchy (A_l, P_l, R_l)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2202_09056_b200 as pb  # noqa: E402

p = pb.generate_hex(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022)
h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), "ns_block",
                  pb.AmgParams())
out = []
for l in range(h.nlevels):
    for w, name in ((0, "A"), (1, "P"), (2, "R")):
        if w and l == h.nlevels - 1:
            continue
        M = h.level_matrix(l, w)
        nr, nc, nz = M.shape
        x = torch.rand(3 * nc + 2, dtype=torch.float64, device="cuda")
        y = torch.zeros(3 * nr + 2, dtype=torch.float64, device="cuda")
        for _ in range(5):
            M.spmv_device(x.data_ptr(), y.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            M.spmv_device(x.data_ptr(), y.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 200 * 1e3
        by = M.spmv_bytes()
        out.append(f"{name}{l} {nr}x{nc} nnzb={nz} bpr={nz / nr:.1f}: {us:.1f} us {by / us / 1e3:.0f} GB/s")
print(os.environ.get("SAMG_SPMV_VARIANT", "-"), os.environ.get("SAMG_SPMV_GROUP", "-"),
      os.environ.get("SAMG_TMA_MIN_CHUNKS", "-"))
print("\n".join(out))
