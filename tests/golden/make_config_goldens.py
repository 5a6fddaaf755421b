"""Config-scale goldens from the UNMODIFIED reference (oracle/_ref).

    python tests/golden/make_config_goldens.py C1 [--isa avx2|scalar] [--tag T]

For one BASELINE config this runs the reference's own ns_block setup
(hierarchy.hpp:263-405) and cg_solve (cg.hpp:87-112; SPAI0 / block Jacobi
through the harness V-cycle + cg_solve_op, oracle/ref_driver.cpp) on the
problem the repo's generator builds for that config (generator.cpp, linked
into oracle/_ref, bitwise the product's generate_hex), and writes

  tests/golden/config_<name>[_<tag>].json   level shapes + sha256 of every
      level's ptr / col / val (A, P, R as int64 / fp64 bytes), aggregate ids,
      coarse dim, footprint, setup and solve seconds, iterations, relative
      residual, ||u||_2 and the sha256 of u;
  tests/golden/config_<name>[_<tag>]_u.npy  u[::stride] (about 20 000
      entries), for the north_star 1e-7 solution bar.

The GPU tests (tests/test_gpu_config_parity.py) rebuild the same problem on
the B200, hash the GPU hierarchy the same way and compare.  Full vectors at
C2 / C3 would be 21 / 50 MB, hence the subsample + norm.

The reference is single-threaded; C1 takes ~1 min, C2 ~10-20 min, C3 1-2 h
on one core.  --isa scalar forces the reference's scalar dot/axpby
(kernels.hpp:25-28) instead of its AVX2-FMA ones: the same reference,
different rounding in CG only -- the spread of its own iteration count
under that change is the anchor for the +-1 bar at ill-conditioned configs.
"""
import argparse
import hashlib
import json
import os
import resource
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Params, Ref  # noqa: E402

SM = {"jacobi": 0, "spai0": 1, "block_jacobi": 2, "ilu0": 3}

# name: (generator keywords, smoother, smoother_omega, max_iterations)
# the same problems as scripts/configs.py / bench.py (BASELINE.json configs)
CONFIGS = {
    "C1": (dict(nx=63, ny=63, nz=63, dirichlet="eliminate", noise=0.01, seed=2022),
           "spai0", 0.72, 1000),
    "C2": (dict(nx=95, ny=95, nz=95, dirichlet="eliminate", heterogeneous=True,
                load="random", seed=2022), "jacobi", 0.5, 5000),
    # C2's ns_block hierarchy has near-singular coarse diagonal blocks (the
    # reference's block inverse throws singular_block there):
    # no smoother converges, so C2 is pinned on the hierarchy and on a
    # fixed number of SPAI0-PCG iterations
    "C2s": (dict(nx=95, ny=95, nz=95, dirichlet="eliminate", heterogeneous=True,
                 load="random", seed=2022), "spai0", 0.72, 100),
    "C3": (dict(nx=511, ny=63, nz=63, lx=511 / 63, dirichlet="eliminate",
                load="traction_xend", x_slowest=True), "spai0", 0.72, 5000),
    "C3i": (dict(nx=511, ny=63, nz=63, lx=511 / 63, dirichlet="eliminate",
                 load="traction_xend", x_slowest=True), "ilu0", 0.72, 1000),
    # 23.88 M unknowns: the reference setup needs ~130 GB and ~6 min, its
    # solve ~1.5 h single-threaded -> hierarchy only (--no-solve), run on
    # the GPU box's host (196 GB)
    "C4": (dict(nx=199, ny=199, nz=199, dirichlet="eliminate", noise=0.01, seed=2022),
           "spai0", 0.72, 1000),
}


def sha(a, dtype):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dtype).tobytes()).hexdigest()


def level_record(nr, nc, ptr, col, val):
    return {"nrows": int(nr), "ncols": int(nc), "nnzb": int(ptr[-1]),
            "ptr": sha(ptr, np.int64), "col": sha(col, np.int64), "val": sha(val, np.float64)}


def stride_for(n):
    return max(1, n // 20000)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CONFIGS))
    ap.add_argument("--isa", choices=["avx2", "scalar"], default="avx2")
    ap.add_argument("--tag", default="")
    ap.add_argument("--smoother", default=None)
    ap.add_argument("--omega", type=float, default=None)
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--outdir", default=HERE)
    ap.add_argument("--maxit", type=int, default=None,
                    help="CG iteration cap (C2: a fixed-iteration comparison)")
    args = ap.parse_args()
    kw, sm, om, maxit = CONFIGS[args.config]
    maxit = args.maxit or maxit
    sm = args.smoother or sm
    om = args.omega if args.omega is not None else om
    ref = Ref()
    avx = ref.force_isa(args.isa == "avx2")
    t0 = time.perf_counter()
    p = ref.gen_hex(**kw)
    tgen = time.perf_counter() - t0
    n = p.n
    B = p.nullspace()
    rec = {"config": args.config, "generator": kw, "smoother": sm, "smoother_omega": om,
           "pipeline": "ns_block", "isa": "avx2" if avx else "scalar", "unknowns": n,
           "nnzb": p.nnzb, "generate_s": tgen, "max_iterations": maxit, "tol": 1e-8}
    print(f"[{args.config}] generated n={n} in {tgen:.1f}s", flush=True)
    # samg::setup on to_scalar(A) (csr.hpp:327-353) -- the scalar view the
    # product's samg_setup receives; formed inside the driver to save memory
    h = ref.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), B,
                       Params(smoother=SM[sm], smoother_omega=om))
    rec["setup_s"] = h.setup_seconds
    rec["nlevels"] = h.nlevels
    rec["coarse_dim"] = h.coarse_dim
    rec["memory_footprint"] = h.memory_footprint
    levels = []
    for l in range(h.nlevels):
        lv = {"A": level_record(*h.level(l, 0))}
        if l < h.nlevels - 1:
            lv["P"] = level_record(*h.level(l, 1))
            lv["R"] = level_record(*h.level(l, 2))
            ids, cnt = h.aggregates(l)
            lv["aggregates"] = {"count": int(cnt), "ids": sha(ids, np.int64)}
        levels.append(lv)
    rec["levels"] = levels
    print(f"[{args.config}] setup {rec['setup_s']:.1f}s levels "
          f"{[x['A']['nrows'] for x in levels]}", flush=True)
    name = f"config_{args.config}{'_' + args.tag if args.tag else ''}"
    if not args.no_solve:
        u, rep = h.cg_solve(p.rhs, tol=1e-8, max_iterations=maxit)
        rec.update(iterations=rep["iterations"], relative_residual=rep["relative_residual"],
                   converged=rep["converged"], solve_s=rep["solve_seconds"],
                   u_norm=float(np.linalg.norm(u)), u_sha=sha(u, np.float64),
                   u_stride=stride_for(n))
        np.save(os.path.join(args.outdir, name + "_u.npy"), u[::stride_for(n)])
        print(f"[{args.config}] solve {rep}", flush=True)
    rec["max_rss_gb"] = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20
    rec["host"] = os.uname().nodename
    with open(os.path.join(args.outdir, name + ".json"), "w") as f:
        json.dump(rec, f, indent=1)
    print(json.dumps({k: v for k, v in rec.items() if k != "levels"}), flush=True)


if __name__ == "__main__":
    main()
