"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs /root/reference to build oracle/_ref):
    make -C oracle ref && python tests/golden/make_golden.py

Every fixture's inputs come from the reference's own generator
(generate_hex_elasticity, elasticity.hpp:129-213) and rigid_body_modes
(elasticity.hpp:38-52); outputs are the reference's samg::setup(ns_block)
hierarchy, aggregates (strength_graph + aggregate on to_scalar(A_l)),
samg::vcycle and samg::cg_solve results.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Params, Ref, SM_JACOBI, SM_SPAI0  # noqa: E402

CASES = {
    # name: (nx, clamp, smoother, smoother_omega, coarse_enough)
    "cube4_keep_spai0": (4, True, SM_SPAI0, 0.72, 100),
    "cube5_keep_jacobi": (5, True, SM_JACOBI, 0.72, 150),
    "cube4_free_jacobi05": (4, False, SM_JACOBI, 0.5, 100),
}


def main():
    ref = Ref()
    for name, (nx, clamp, sm, om, ce) in CASES.items():
        p = ref.generate_hex(nx, nx, nx, 1.0, 0.3, clamp)
        B = ref.rigid_body_modes(p.coords)
        out = dict(n=p.n, ptr=p.ptr, col=p.col, val=p.val, rhs=p.rhs, coords=p.coords, B=B,
                   smoother=sm, smoother_omega=om, coarse_enough=ce)
        if not clamp:
            # free-floating grid is singular: pin setup + V-cycle only
            pass
        h = ref.setup(p.n, p.ptr, p.col, p.val, B, Params(smoother=sm, smoother_omega=om,
                                                         coarse_enough=ce))
        out["nlevels"] = h.nlevels
        out["coarse_dim"] = h.coarse_dim
        out["memory_footprint"] = h.memory_footprint
        for l in range(h.nlevels):
            for w, tag in ((0, "A"), (1, "P"), (2, "R")):
                if w and l == h.nlevels - 1:
                    continue
                nr, nc, ptr, col, val = h.level(l, w)
                out[f"L{l}_{tag}_shape"] = np.array([nr, nc])
                out[f"L{l}_{tag}_ptr"] = ptr
                out[f"L{l}_{tag}_col"] = col
                out[f"L{l}_{tag}_val"] = val
            if l < h.nlevels - 1:
                ids, cnt = h.aggregates(l)
                out[f"L{l}_agg"] = ids
                out[f"L{l}_naggs"] = cnt
        f = p.rhs if clamp else np.random.default_rng(nx).uniform(-1, 1, p.n)
        out["vcycle_f"] = f
        out["vcycle_u"] = h.vcycle(f)
        if clamp:
            u, rep = h.cg_solve(p.rhs)
            out["cg_u"] = u
            out["cg_iterations"] = rep["iterations"]
            out["cg_relres"] = rep["relative_residual"]
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, "levels", h.nlevels, "bytes", os.path.getsize(os.path.join(HERE, name + ".npz")))


if __name__ == "__main__":
    main()
