"""Symmetry and definiteness of the coarsest operator of a BASELINE config
(decides whether the coarse inverse runs without row exchanges)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2202_09056_b200 as pb  # noqa: E402
from scripts.configs import CONFIGS  # noqa: E402

for name in sys.argv[1:] or ["C1", "C4"]:
    kw, _ = CONFIGS[name]
    dp = pb.generate_hex_device(pb.ProblemParams(**kw), device=0)
    h = pb.setup_device(dp.A, dp.nullspace_ptr, 6, "ns_block", pb.AmgParams(smoother="spai0"))
    L = h.nlevels - 1
    nr, _, ptr, col, val = h.level_matrix(L).download()
    v = val.reshape(-1, 3, 3)
    D = np.zeros((3 * nr, 3 * nr))
    for i in range(nr):
        for j in range(ptr[i], ptr[i + 1]):
            D[3 * i:3 * i + 3, 3 * col[j]:3 * col[j] + 3] = v[j]
    asym = np.abs(D - D.T).max() / np.abs(D).max()
    d = np.sqrt(np.abs(np.diag(D)))
    S = D / np.outer(d, d)
    ev = np.linalg.eigvalsh((S + S.T) / 2)
    print(f"{name}: n={3 * nr} asym/max={asym:.3e} eq. eig min={ev.min():.3e} max={ev.max():.3e} "
          f"coarse solver={h.coarse_solver}", flush=True)
    h.close()
