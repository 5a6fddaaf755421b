"""Same-box GPU comparator for the headline kernel: the C1 fine
matrix y = A x through torch's BSR sparse matmul (cuSPARSE bsrmv / bsrmm on
CUDA) next to samg_bsr3_spmv_device, both timed with CUDA events on the
current stream, inputs resident, 527 MB per call (> L2).  A reported
reference only -- the product never calls cuSPARSE."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2202_09056_b200 as pb  # noqa: E402

p = pb.generate_hex(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022)
nb, n = p.nbrows, p.n
nbytes = p.nnzb * 76 + (nb + 1) * 4 + nb * 24 + nb * 24
dev = torch.device("cuda", 0)
x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).to(dev)


def timeit(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


out = {}
for idx in (torch.int32, torch.int64):
    try:
        A = torch.sparse_bsr_tensor(torch.from_numpy(p.ptr).to(idx), torch.from_numpy(p.col).to(idx),
                                    torch.from_numpy(p.val.reshape(-1, 3, 3)), size=(n, n),
                                    dtype=torch.float64).to(dev)
        xc = x.reshape(n, 1)
        y = A @ xc
        t = timeit(lambda: A @ xc)
        out[f"torch_bsr_{str(idx).split('.')[-1]}"] = {"us": t * 1e6, "GBs": nbytes / t / 1e9}
        ref = y.reshape(-1)
    except Exception as e:  # noqa: BLE001
        out[f"torch_bsr_{str(idx).split('.')[-1]}"] = {"error": repr(e)[:200]}
M = pb.Bsr3.from_host(nb, nb, p.ptr, p.col, p.val.reshape(-1))
yb = torch.zeros(n + 2, dtype=torch.float64, device=dev)
t = timeit(lambda: M.spmv_device(x.data_ptr(), yb.data_ptr()))
out["samg_bsr3_spmv_device"] = {"us": t * 1e6, "GBs": nbytes / t / 1e9}
if "ref" in dir():
    out["max_rel_diff"] = float((yb[:n] - ref).abs().max() / ref.abs().max())
print(out)
