"""Algorithmic bytes of one SPAI0-PCG iteration (graph body: q = A p with
p.q; fused r update + level-0 first sweep; V-cycle with the restriction
fused into the next level's first sweep; last sweep with r.z; p / u update)
from the hierarchy's level sizes -- the numerator of the whole-iteration
roofline.  Each matrix pass counts nnzb*(72+4) + (nrows+1)*4, each vector
once per kernel that reads or writes it (x gathers once).

    python scripts/iter_bytes.py [C1|C4] [ms_per_iteration]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09056_b200 as pb  # noqa: E402

CFG = {"C1": dict(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022),
       "C4": dict(nx=199, ny=199, nz=199, dirichlet="eliminate", noise=0.01, seed=2022)}
name = sys.argv[1] if len(sys.argv) > 1 else "C1"
ms = float(sys.argv[2]) if len(sys.argv) > 2 else None
dp = pb.generate_hex_device(pb.ProblemParams(**CFG[name]))
h = pb.setup_device(dp.A, dp.nullspace_ptr, 6, "ns_block", pb.AmgParams(smoother="spai0"))
L = h.nlevels
A = [h.level_info(l, 0) for l in range(L)]
P = [h.level_info(l, 1) for l in range(L - 1)]
R = [h.level_info(l, 2) for l in range(L - 1)]
n = [a[0] for a in A]  # block rows
V = 24  # bytes per block row of a vector


def mat(m):
    return m[2] * 76 + (m[0] + 1) * 4


items = []
items.append(("q = A0 p, p.q", mat(A[0]) + V * n[0] * 3))
items.append(("r -= a q, r.r, z0 = M0 r", V * n[0] * 4 + 72 * n[0]))
for l in range(L - 1):
    items.append((f"residual A{l}", mat(A[l]) + V * n[l] * 3))
    if l + 2 < L:
        items.append((f"R{l} + first sweep L{l + 1}", mat(R[l]) + V * n[l] + V * n[l + 1] * 2 + 72 * n[l + 1]))
    else:
        items.append((f"R{l}", mat(R[l]) + V * n[l] + V * n[l + 1]))
nc = 3 * n[L - 1]
items.append(("coarse GEMV", nc * ((nc + 1) & ~1) * 8 + 16 * nc))
for l in range(L - 2, -1, -1):
    items.append((f"P{l} (u += P uc)", mat(P[l]) + V * n[l + 1] + V * n[l] * 2))
    items.append((f"last sweep A{l}" + (" + r.z" if l == 0 else ""),
                  mat(A[l]) + V * n[l] * 4 + 72 * n[l]))
items.append(("p = z + b p, u += a p", V * n[0] * 5))
tot = sum(b for _, b in items)
out = {"config": name, "levels": n, "coarse_dim": nc, "items": items, "bytes_per_iteration": tot}
if ms:
    out["ms_per_iteration"] = ms
    out["TBps"] = tot / (ms * 1e-3) / 1e12
print(json.dumps(out))
