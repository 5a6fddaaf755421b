"""Run the BASELINE.json configs on the B200 path and (where the single-core
reference is affordable) against the reference, one JSON line per run.

    python scripts/configs.py [C0 C0k C1 C2 C3 C4] [--ref] [--out FILE]

C0  20^3-node cube, SPAI0, body force + U[-0.01,0.01] noise (free-DOF form)
C0k same, reference kept-rows form
C1  64^3-node cube (free-DOF), SPAI0
C2  96^3-node cube, heterogeneous E = exp(N(0,1)), nu ~ U[0.25,0.35], random
    RHS U[-1,1]; damped Jacobi omega = 0.72 as specified (divergent, SURVEY
    0.4) and SPAI0 (block Jacobi hits a singular coarse diagonal block here,
    the reference's samg::inverse throws the same singular_block)
C3  512x64x64-node cantilever (x slowest), -z traction on the x-end face
C4  200^3-node cube, SPAI0
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2202_09056_b200 as pb  # noqa: E402

CONFIGS = {
    "C0": (dict(nx=19, ny=19, nz=19, dirichlet="eliminate", noise=0.01, seed=2022), [("spai0", 0.72)]),
    "C0k": (dict(nx=19, ny=19, nz=19, dirichlet="keep_rows", noise=0.01, seed=2022), [("spai0", 0.72)]),
    "C1": (dict(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022), [("spai0", 0.72)]),
    "C2": (dict(nx=95, ny=95, nz=95, dirichlet="eliminate", heterogeneous=True, load="random",
                seed=2022), [("jacobi", 0.72), ("spai0", 0.72)]),
    "C3": (dict(nx=511, ny=63, nz=63, lx=511 / 63, dirichlet="eliminate", load="traction_xend",
                x_slowest=True), [("spai0", 0.72)]),
    "C4": (dict(nx=199, ny=199, nz=199, dirichlet="eliminate", noise=0.01, seed=2022), [("spai0", 0.72)]),
}
SM = {"spai0": 1, "jacobi": 0, "block_jacobi": 2, "ilu0": 3}


PIPE = {"scalar": 0, "block": 1, "ns_scalar": 2, "ns_hybrid1": 3, "ns_hybrid2": 4, "ns_block": 5}


def run(name, ref_on, max_it, out, smoother=None, pipeline="ns_block", precision="fp64"):
    kw, smoothers = CONFIGS[name]
    if smoother:
        smoothers = [(smoother, 0.72)]
    t0 = time.perf_counter()
    p = pb.generate_hex(**kw)
    tgen = time.perf_counter() - t0
    B = None if pipeline in ("block", "scalar") else p.nullspace()
    for sm, om in smoothers:
        rec = {"config": name, "pipeline": pipeline, "smoother": sm, "omega": om, "unknowns": p.n,
               "nnzb": p.nnzb, "generate_s": tgen, "vcycle_precision": precision}
        prm = pb.AmgParams(smoother=sm, smoother_omega=om, vcycle_precision=precision)
        h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), B, pipeline, prm)
        h.close()  # warm-up (lazy module loading, memory pool)
        t0 = time.perf_counter()
        h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), B, pipeline, prm)
        rec["gpu_setup_s"] = time.perf_counter() - t0
        rec["levels_block_rows"] = [h.level_info(l)[0] for l in range(h.nlevels)]
        rec["coarse_dim"] = h.coarse_dim
        u, rep = h.cg_solve(p.rhs, pb.CgParams(max_iterations=max_it))
        u, rep = h.cg_solve(p.rhs, pb.CgParams(max_iterations=max_it))
        rec.update(gpu_solve_s=rep["solve_seconds"], gpu_iterations=rep["iterations"],
                   gpu_converged=rep["converged"], gpu_relres=rep["relative_residual"],
                   preconditioner_bytes=rep["preconditioner_bytes"])
        if ref_on:
            from oracle.oracle import Params, Ref
            ref = Ref()
            n, ptr, col, val = p.csr()
            t0 = time.perf_counter()
            hr = ref.setup(n, ptr, col, val, B, Params(smoother=SM[sm], smoother_omega=om,
                                                         pipeline=PIPE[pipeline]))
            rec["ref_setup_s"] = time.perf_counter() - t0
            same = hr.nlevels == h.nlevels
            agg_same = same
            for l in range(min(h.nlevels, hr.nlevels)):
                for w in (0, 1, 2):
                    if w and l == h.nlevels - 1:
                        continue
                    a, b = h.level(l, w), hr.level(l, w)
                    same = same and a[0] == b[0] and np.array_equal(a[2], b[2]) and \
                        np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4])
                if l < h.nlevels - 1:
                    agg_same = agg_same and np.array_equal(h.aggregates(l)[0], hr.aggregates(l)[0])
            rec["hierarchy_bit_identical"] = bool(same)
            rec["aggregates_bit_identical"] = bool(agg_same)
            rec["footprint_equal"] = h.memory_footprint() == hr.memory_footprint
            if os.environ.get("SAMG_CONFIGS_REF_SOLVE", "1") == "1":
                ur, rr = hr.cg_solve(p.rhs, max_iterations=max_it)
                rec.update(ref_solve_s=rr["solve_seconds"], ref_iterations=rr["iterations"],
                           ref_converged=rr["converged"])
                if rr["converged"] and rep["converged"]:
                    rec["solution_rel_diff"] = float(np.linalg.norm(u - ur) / np.linalg.norm(ur))
        h.close()
        print(json.dumps(rec), flush=True)
        if out:
            with open(out, "a") as f:
                f.write(json.dumps(rec) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C0", "C0k", "C1"])
    ap.add_argument("--ref", action="store_true")
    ap.add_argument("--max-it", type=int, default=1000)
    ap.add_argument("--out", default=None)
    ap.add_argument("--smoother", default=None, help="override the configs' smoothers (e.g. ilu0)")
    ap.add_argument("--pipeline", default="ns_block", choices=sorted(PIPE))
    ap.add_argument("--precision", default="fp64", choices=["fp64", "mixed"],
                    help="V-cycle operator storage (mixed: fp32 copies, DESIGN.md 5.8)")
    a = ap.parse_args()
    for c in a.configs:
        run(c, a.ref, a.max_it, a.out, a.smoother, a.pipeline, a.precision)


if __name__ == "__main__":
    main()
