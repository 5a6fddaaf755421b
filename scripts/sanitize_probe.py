"""Small end-to-end exercise of every kernel family for compute-sanitizer:
setup (all phases incl. the cluster GJ panel) + CG with SPAI0 and ILU(0),
the TMA SpMV (>= 24 chunks per SM: 50^3 elements), the bitmap/hash SpGEMM,
the batch SpMV, device assembly and the emulated multi-rank solve."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2202_09056_b200 as pb  # noqa: E402
from paper_2202_09056_b200.dist import DistHierarchy  # noqa: E402

p = pb.generate_hex(nx=8, ny=8, nz=8, dirichlet="eliminate", noise=0.01, seed=1)
for sm in ("spai0", "ilu0"):
    h = pb.setup(p.csr(), p.nullspace(), "ns_block", pb.AmgParams(smoother=sm, coarse_enough=300))
    u, rep = h.cg_solve(p.rhs)
    print(sm, rep["iterations"], flush=True)
    h.close()
hh = pb.setup(p.csr(), p.nullspace(), "ns_hybrid2", pb.AmgParams(coarse_enough=300))
print("hybrid2", hh.cg_solve(p.rhs)[1]["iterations"], flush=True)
q = pb.generate_hex(nx=50, ny=50, nz=50, dirichlet="eliminate")
M = pb.Bsr3.from_host(q.nbrows, q.nbrows, q.ptr, q.col, q.val.reshape(-1))
x = np.ones(q.n)
print("tma spmv", float(M.spmv(x).sum()), flush=True)
print("batch", float(M.spmv_batch(np.ones((3, q.n))).sum()), flush=True)
dp = pb.generate_hex_device(nx=6, ny=5, nz=4, dirichlet="eliminate")
print("device assembly", dp.nnzb, flush=True)
dh = DistHierarchy(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), 0, 3,
                   min_rows=1, prm=pb.AmgParams(coarse_enough=300), emulate=True)
print("emulated 3 ranks", dh.cg_solve(p.rhs)[1]["iterations"], flush=True)
# round 2: 6x6 node-blocked level >= 1 operators, the fused CG kernels (graph),
# verify_galerkin, the distributed setup (emulated), PDL back-to-back SpMVs
r = pb.generate_hex(nx=12, ny=10, nz=10, dirichlet="eliminate", noise=0.01, seed=5)
h3 = pb.setup(r.csr(), r.nullspace(), "ns_block",
              pb.AmgParams(coarse_enough=150, verify_galerkin=True))
print("levels", h3.nlevels, "cg", h3.cg_solve(r.rhs)[1]["iterations"], flush=True)
dh2 = DistHierarchy(r.nbrows, r.ptr, r.col, r.val.reshape(-1), r.nullspace(), 0, 4,
                    min_rows=1, prm=pb.AmgParams(coarse_enough=150), emulate=True)
print("distributed setup 4 ranks", dh2.info(), dh2.cg_solve(r.rhs)[1]["iterations"], flush=True)
import torch  # noqa: E402
xd = torch.ones(q.n, dtype=torch.float64, device="cuda")
yd = torch.zeros(q.n, dtype=torch.float64, device="cuda")
for _ in range(3):
    M.spmv_device(xd.data_ptr(), yd.data_ptr())
torch.cuda.synchronize()
print("pdl spmv", float(yd.sum()), flush=True)
