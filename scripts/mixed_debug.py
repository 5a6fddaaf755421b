"""Debug: heterogeneous 16x4x4 beam, GPU vs reference V-cycle / coarse inverse."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2202_09056_b200 as pb
from oracle.oracle import Ref, Params, SM_SPAI0

def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
kw = dict(nx=16, ny=4, nz=4, lx=4.0, dirichlet="eliminate", heterogeneous=True, load="random", seed=9)
p = pb.generate_hex(**kw); A = p.csr(); B = p.nullspace()
h = pb.setup(A, B, "ns_block", pb.AmgParams(smoother="spai0", coarse_enough=150))
hr = Ref().setup(A[0], A[1], A[2], A[3], B, Params(smoother=SM_SPAI0, coarse_enough=150))
print("levels", h.nlevels, hr.nlevels)
vg, vr = h.vcycle(p.rhs), hr.vcycle(p.rhs)
print("vcycle rel diff", rel(vg, vr))
L = h.nlevels - 1
Ac = h.level_matrix(L, 0)
nb, nc, ptr, col, val = h.level(L, 0)
D = np.zeros((3 * nb, 3 * nb))
v = val.reshape(-1, 3, 3)
for i in range(nb):
    for j in range(ptr[i], ptr[i + 1]):
        D[3 * i:3 * i + 3, 3 * col[j]:3 * col[j] + 3] = v[j]
Ainv = Ac.dense_inverse()
print("coarse n", D.shape[0], "cond", np.linalg.cond(D), "||Ainv*A - I||", np.abs(Ainv @ D - np.eye(D.shape[0])).max())
print("diag min/max", np.abs(np.diag(D)).min(), np.abs(np.diag(D)).max())
print("symmetric", np.abs(D - D.T).max() / np.abs(D).max())
w = np.linalg.eigvalsh((D + D.T) / 2); print("eig min/max", w.min(), w.max())
u, rep = h.cg_solve(p.rhs); ur, rr = hr.cg_solve(p.rhs)
print(rep["iterations"], rep["relative_residual"], rr["iterations"], rr["relative_residual"])
