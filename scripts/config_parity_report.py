"""GPU vs reference at config scale (tests/golden/config_*.json): one JSON
line per golden with the iteration counts, residuals, the solution's
relative difference on the stored sample and on the norm, and whether the
hierarchy hashes matched.  python scripts/config_parity_report.py [names]"""
import glob
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09056_b200 as pb  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def sha(a, dt):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dt).tobytes()).hexdigest()


want = sys.argv[1:]
for path in sorted(glob.glob(os.path.join(GOLD, "config_*.json"))):
    name = os.path.basename(path)[7:-5]
    if want and name not in want:
        continue
    rec = json.load(open(path))
    p = pb.generate_hex(**rec["generator"])
    prm = pb.AmgParams(smoother=rec["smoother"], smoother_omega=rec["smoother_omega"])
    h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), "ns_block", prm)
    same = h.nlevels == rec["nlevels"]
    for l, lv in enumerate(rec["levels"]):
        for w, tag in ((0, "A"), (1, "P"), (2, "R")):
            if tag in lv and same:
                nr, nc, ptr, col, val = h.level(l, w)
                same = same and sha(val, np.float64) == lv[tag]["val"] and sha(col, np.int64) == lv[tag]["col"]
    out = {"config": name, "isa": rec["isa"], "hierarchy_bitwise": bool(same)}
    if "iterations" in rec:
        u, rep = h.cg_solve(p.rhs, pb.CgParams(tol=rec["tol"], max_iterations=rec["max_iterations"]))
        us = np.load(os.path.join(GOLD, f"config_{name}_u.npy"))
        gs = u[::rec["u_stride"]]
        out.update(gpu_iterations=rep["iterations"], ref_iterations=rec["iterations"],
                   gpu_relres=rep["relative_residual"], ref_relres=rec["relative_residual"],
                   gpu_converged=rep["converged"], ref_converged=rec["converged"],
                   u_sample_rel_diff=float(np.linalg.norm(gs - us) / np.linalg.norm(us)),
                   u_norm_rel_diff=float(abs(np.linalg.norm(u) - rec["u_norm"]) / rec["u_norm"]),
                   gpu_solve_s=rep["solve_seconds"], ref_solve_s=rec.get("solve_s"),
                   ref_setup_s=rec.get("setup_s"))
    print(json.dumps(out), flush=True)
    h.close()
