"""Pin the C restatement oracle (oracle/samg_oracle.c) before trusting it.

1. Against the committed golden fixtures (tests/golden/*.npz), produced by
   the unmodified reference (tests/golden/make_golden.py): bit-exact setup
   hierarchies, aggregates, footprint and V-cycle; CG within +-1 iteration
   (the reference's dot product is AVX2-FMA, the oracle's the scalar
   4-partial-sum variant, kernels_scalar.cpp:15-28 vs kernels_avx2.cpp:35-45).
2. Against the live reference (oracle/_ref) on more shapes, when built.
3. Restated reference unit tests (test_coarsening.cpp, test_hierarchy.cpp,
   test_cg.cpp) on the oracle's kernels.
"""
import glob
import os

import numpy as np
import pytest

from oracle.oracle import Params, SM_BLOCK_JACOBI, SM_JACOBI, SM_SPAI0

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_oracle_matches_golden(orc, path):
    g = np.load(path)
    n = int(g["n"])
    prm = Params(smoother=int(g["smoother"]), smoother_omega=float(g["smoother_omega"]),
                 coarse_enough=int(g["coarse_enough"]))
    h = orc.setup(n, g["ptr"], g["col"], g["val"], g["B"], prm)
    assert h.nlevels == int(g["nlevels"])
    assert h.coarse_dim == int(g["coarse_dim"])
    assert h.memory_footprint == int(g["memory_footprint"])
    for l in range(h.nlevels):
        for w, tag in ((0, "A"), (1, "P"), (2, "R")):
            if w and l == h.nlevels - 1:
                continue
            nr, nc, ptr, col, val = h.level(l, w)
            assert [nr, nc] == list(g[f"L{l}_{tag}_shape"])
            np.testing.assert_array_equal(ptr, g[f"L{l}_{tag}_ptr"])
            np.testing.assert_array_equal(col, g[f"L{l}_{tag}_col"])
            np.testing.assert_array_equal(val, g[f"L{l}_{tag}_val"])
        if l < h.nlevels - 1:
            ids, cnt = h.aggregates(l)
            assert cnt == int(g[f"L{l}_naggs"])
            np.testing.assert_array_equal(ids, g[f"L{l}_agg"])
    np.testing.assert_array_equal(h.vcycle(g["vcycle_f"]), g["vcycle_u"])
    if "cg_u" in g:
        u, rep = h.cg_solve(g["rhs"])
        assert abs(rep["iterations"] - int(g["cg_iterations"])) <= 1
        assert np.linalg.norm(u - g["cg_u"]) <= 1e-7 * np.linalg.norm(g["cg_u"])


@pytest.mark.parametrize("nx,clamp", [(3, True), (4, False), (6, True)])
def test_oracle_generator_matches_golden_generator(orc, nx, clamp):
    """The restated generator equals the reference's to rounding (duplicates
    are summed in a different order: from_triplets uses an unstable sort)."""
    for path in GOLDEN:
        g = np.load(path)
        if int(g["n"]) != 3 * (nx + 1) ** 3:
            continue
        p = orc.generate_hex(nx, nx, nx, 1.0, 0.3, clamp)
        if ("free" in path) == clamp:
            continue
        np.testing.assert_array_equal(p.ptr, g["ptr"])
        np.testing.assert_array_equal(p.col, g["col"])
        assert np.abs(p.val - g["val"]).max() <= 1e-15 * np.abs(g["val"]).max()
        np.testing.assert_array_equal(p.rhs, g["rhs"])
        np.testing.assert_array_equal(p.coords, g["coords"])
        np.testing.assert_array_equal(orc.rigid_body_modes(p.coords), g["B"])


LIVE = [
    (5, True, SM_SPAI0, 0.72, 120),
    (6, True, SM_BLOCK_JACOBI, 0.5, 100),
    (7, True, SM_JACOBI, 0.5, 200),
]


@pytest.mark.parametrize("nx,clamp,sm,om,ce", LIVE)
def test_oracle_matches_live_reference(orc, ref, nx, clamp, sm, om, ce):
    p = ref.generate_hex(nx, nx, nx, 1.0, 0.3, clamp)
    B = ref.rigid_body_modes(p.coords)
    prm = Params(smoother=sm, smoother_omega=om, coarse_enough=ce)
    ho = orc.setup(p.n, p.ptr, p.col, p.val, B, prm)
    hr = ref.setup(p.n, p.ptr, p.col, p.val, B, prm)
    assert ho.nlevels == hr.nlevels
    for l in range(ho.nlevels):
        for w in (0, 1, 2):
            if w and l == ho.nlevels - 1:
                continue
            a, b = ho.level(l, w), hr.level(l, w)
            for x, y in zip(a[2:], b[2:]):
                np.testing.assert_array_equal(x, y)
        if l < ho.nlevels - 1:
            np.testing.assert_array_equal(ho.aggregates(l)[0], hr.aggregates(l)[0])
    assert ho.memory_footprint == hr.memory_footprint
    np.testing.assert_array_equal(ho.vcycle(p.rhs), hr.vcycle(p.rhs))
    uo, ro = ho.cg_solve(p.rhs)
    ur, rr = hr.cg_solve(p.rhs)
    assert abs(ro["iterations"] - rr["iterations"]) <= 1
    assert np.linalg.norm(uo - ur) <= 1e-7 * np.linalg.norm(ur)


# --- restated reference unit tests (doctest suites do not build here) -------

def _lap1d(n):
    ptr, col, val = [0], [], []
    for i in range(n):
        if i > 0:
            col.append(i - 1); val.append(-1.0)
        col.append(i); val.append(2.0)
        if i + 1 < n:
            col.append(i + 1); val.append(-1.0)
        ptr.append(len(col))
    return np.array(ptr), np.array(col), np.array(val)


def test_aggregation_kats(orc):
    # test_coarsening.cpp:18-26: 1D Laplacian edges all strong -> aggregates
    # of three consecutive nodes (seed i, neighbours i-1, i+1)
    ptr, col, val = _lap1d(9)
    ids, cnt = orc.aggregate_scalar(9, ptr, col, val, 0.08, 1)
    # greedy: seeds 0, 3, 6; node 8 joins its assigned neighbour 7 in pass 2
    assert cnt == 3
    np.testing.assert_array_equal(ids, [0, 0, 1, 1, 1, 2, 2, 2, 2])
    # identity: no edges -> singletons (test_coarsening.cpp:58-65)
    n = 5
    ids, cnt = orc.aggregate_scalar(n, np.arange(n + 1), np.arange(n), np.ones(n), 0.08, 1)
    assert cnt == n
    np.testing.assert_array_equal(ids, np.arange(n))


def test_greedy_aggregation_on_path(orc):
    """Path 0-1-2 -> one aggregate (test_coarsening.cpp:67-75)."""
    ptr, col, val = _lap1d(3)
    ids, cnt = orc.aggregate_scalar(3, ptr, col, val, 0.08, 1)
    assert cnt == 1
    np.testing.assert_array_equal(ids, [0, 0, 0])


def test_spmv_row_sums_worked_example(orc):
    """test_csr.cpp:19-27 on a 3x3-block version of the worked example."""
    rng = np.random.default_rng(1)
    nr = 4
    ptr = np.array([0, 2, 3, 5, 6])
    col = np.array([0, 2, 1, 0, 3, 3])
    val = rng.uniform(-1, 1, (6, 3, 3))
    y = orc.spmv_bsr3(nr, nr, ptr, col, val.reshape(-1), np.ones(3 * nr))
    dense = np.zeros((3 * nr, 3 * nr))
    for i in range(nr):
        for j in range(ptr[i], ptr[i + 1]):
            dense[3 * i:3 * i + 3, 3 * col[j]:3 * col[j] + 3] = val[j]
    np.testing.assert_allclose(y, dense.sum(1), rtol=1e-14, atol=1e-14)


def test_galerkin_matches_dense(orc):
    """acceptance.cpp:297-332 (criterion 9): block Galerkin vs dense, 1e-12."""
    rng = np.random.default_rng(223)

    def rand_bsr(nr, nc, dens):
        mask = rng.random((nr, nc)) < dens
        ptr = np.concatenate([[0], np.cumsum(mask.sum(1))]).astype(np.int64)
        col = np.nonzero(mask)[1].astype(np.int64)
        return nr, nc, ptr, col, rng.uniform(-1, 1, (col.size, 3, 3))

    def dense(m):
        nr, nc, ptr, col, val = m
        D = np.zeros((3 * nr, 3 * nc))
        for i in range(nr):
            for j in range(ptr[i], ptr[i + 1]):
                D[3 * i:3 * i + 3, 3 * col[j]:3 * col[j] + 3] = val[j]
        return D

    for _ in range(50):
        nb = int(rng.integers(2, 11))
        mb = max(1, nb // 2)
        R, A, P = rand_bsr(mb, nb, 0.3), rand_bsr(nb, nb, 0.3), rand_bsr(nb, mb, 0.3)
        C = orc.galerkin_bsr3(R, A, P)
        Cd = dense(R) @ dense(A) @ dense(P)
        diff = np.linalg.norm(dense(C) - Cd)
        assert diff <= 1e-12 * max(np.linalg.norm(Cd), 1.0)


def test_breakdown_and_zero_rhs(orc):
    """test_cg.cpp:42-55 and :107-115 on the hierarchy solver."""
    p = orc.generate_hex(3, 3, 3, 1.0, 0.3, True)
    B = orc.rigid_body_modes(p.coords)
    h = orc.setup(p.n, p.ptr, p.col, p.val, B, Params(coarse_enough=60))
    u, rep = h.cg_solve(np.zeros(p.n))
    assert rep["converged"] and rep["iterations"] == 0 and not u.any()
    hn = orc.setup(p.n, p.ptr, p.col, -p.val, B, Params(coarse_enough=60))
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as e:
        hn.cg_solve(p.rhs)
    assert e.value.code == 9


@pytest.mark.parametrize("pipeline", [3, 4])
def test_hybrid_pipelines_match_reference(orc, ref, pipeline):
    """ns_hybrid1 / ns_hybrid2 (hierarchy.hpp:233-260, 300-330): the scalar
    Galerkin path of the restatement equals the reference bit for bit, and
    differs from ns_block at rounding level (so the test has teeth)."""
    p = orc.generate_hex(9, 7, 5, 1.0, 0.3, True)
    n, ptr, col, val = p.n, p.ptr, p.col, p.val
    B = orc.rigid_body_modes(p.coords)
    prm = Params(coarse_enough=150, pipeline=pipeline)
    o = orc.setup(n, ptr, col, val, B, prm)
    r = ref.setup(n, ptr, col, val, B, prm)
    assert o.nlevels == r.nlevels >= 3
    for l in range(o.nlevels):
        for w in ((0, 1, 2) if l < o.nlevels - 1 else (0,)):
            np.testing.assert_array_equal(o.level(l, w)[4], r.level(l, w)[4])
    nb = orc.setup(n, ptr, col, val, B, Params(coarse_enough=150))
    assert not np.array_equal(nb.level(1)[4], o.level(1)[4])
    assert o.memory_footprint == r.memory_footprint
    # +-1: the reference's dot is AVX2-FMA (kernels_avx2.cpp:35-45)
    assert abs(o.cg_solve(p.rhs)[1]["iterations"] - r.cg_solve(p.rhs)[1]["iterations"]) <= 1


@pytest.mark.parametrize("nx,ny,nz,ce,sm", [(9, 7, 5, 150, SM_SPAI0), (10, 10, 10, 300, 2),
                                            (12, 8, 8, 200, SM_BLOCK_JACOBI)])
def test_block_pipeline_matches_reference(orc, ref, nx, ny, nz, ce, sm):
    """pipeline::block (hierarchy.hpp:340-347, coarsening.hpp:471-560): no
    nullspace, Frobenius-norm block strength, identity-block tentative and
    block-diagonal smoothing; bit-identical levels and aggregates."""
    p = orc.generate_hex(nx, ny, nz, 1.0, 0.3, True)
    prm = Params(coarse_enough=ce, pipeline=1, smoother=sm,
                 smoother_omega=0.5 if sm == SM_BLOCK_JACOBI else 0.72)
    o = orc.setup(p.n, p.ptr, p.col, p.val, None, prm)
    r = ref.setup(p.n, p.ptr, p.col, p.val, None, prm)
    assert o.nlevels == r.nlevels >= 3
    for l in range(o.nlevels):
        for w in ((0, 1, 2) if l < o.nlevels - 1 else (0,)):
            for a, b in zip(o.level(l, w), r.level(l, w)):
                np.testing.assert_array_equal(a, b)
        if l < o.nlevels - 1:
            np.testing.assert_array_equal(o.aggregates(l)[0], r.aggregates(l)[0])
    assert o.memory_footprint == r.memory_footprint
    # +-1: the reference's dot is AVX2-FMA (kernels_avx2.cpp:35-45)
    assert abs(o.cg_solve(p.rhs)[1]["iterations"] - r.cg_solve(p.rhs)[1]["iterations"]) <= 1


def test_threaded_reference_spmv_matches_single_thread():
    """bench.py's multi-threaded reference baseline (the reference's own
    spmv on row slices, one thread each) computes the same y as one call."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import paper_2202_09056_b200 as pb
    from oracle.oracle import Ref
    p = pb.generate_hex(nx=9, ny=7, nz=8, dirichlet="eliminate", noise=0.01, seed=5)
    ref = Ref()
    x = np.random.default_rng(1).uniform(-1, 1, p.n)
    y1 = np.zeros(p.n)
    ref.bsr3(p.nbrows, p.nbrows, p.ptr, p.col, p.val.reshape(-1)).spmv(x, y1)
    cuts = [0, p.nbrows // 3, p.nbrows // 2, p.nbrows]
    y2 = np.zeros(p.n)
    for r0, r1 in zip(cuts[:-1], cuts[1:]):
        ref.bsr3(r1 - r0, p.nbrows, p.ptr[r0:r1 + 1], p.col, p.val.reshape(-1)).spmv(
            x, y2[3 * r0:3 * r1])
    assert np.array_equal(y1, y2)
    times, used = bench.cpu_reference_spmv_threaded(p, 3, 0, steps=2)
    assert used == 3 and len(times) == 2
