"""Device side of the row-partitioned operator (dist.cu) on one GPU.

Two and three ranks are emulated in one process, one after the other (no
kernel waits on another rank): each rank packs its send buffers on the GPU,
the "transport" is a device-to-device copy into the receiving rank's ghost
segment, then interior and boundary rows are multiplied.  The concatenated
result must equal the single-GPU SpMV of the global matrix and the
reference's spmv<static_block<3>>.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PROB = dict(nx=15, ny=5, nz=6, lx=2.5, dirichlet="eliminate", load="traction_xend",
            x_slowest=True)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_emulated_ranks_match_global_spmv(gpu, ref, world):
    import torch

    from paper_2202_09056_b200.dist import DistMatrix
    pb = gpu
    pp = pb.ProblemParams(**PROB)
    full = pb.generate_hex(pp)
    per_plane = (pp.ny + 1) * (pp.nz + 1)
    cuts = [round(pp.nx * r / world) for r in range(world + 1)]
    starts = np.array([c * per_plane for c in cuts], dtype=np.int64)
    dms = []
    for r in range(world):
        r0, r1 = int(starts[r]), int(starts[r + 1])
        mine = pb.generate_hex(pb.ProblemParams(**{**PROB, "node_begin": r0, "node_end": r1}))
        dms.append(DistMatrix(mine.ptr, mine.col, mine.val.reshape(-1), starts, r))
    # in-process plan exchange
    for r, dm in enumerate(dms):
        peers, counts, ids = [], [], []
        for q, dq in enumerate(dms):
            if q == r:
                continue
            rp, rc, ro = dq.recv_plan()
            g = dq.ghosts()
            for p, c, o in zip(rp, rc, ro):
                if p == r:
                    peers.append(q)
                    counts.append(c)
                    ids.extend(g[o:o + c])
        dm.set_send(peers, counts, np.array(ids, np.int64))
        dm.to_device(0)
    dev = torch.device("cuda", 0)
    x = np.random.default_rng(3).uniform(-1, 1, full.n)
    xexts, sends, ys = [], [], []
    for r, dm in enumerate(dms):
        inf = dm.info()
        r0 = int(starts[r])
        xe = torch.zeros(3 * (inf["nloc"] + inf["nghost"]) + 3, dtype=torch.float64, device=dev)
        xe[:3 * inf["nloc"]] = torch.from_numpy(x[3 * r0:3 * (r0 + inf["nloc"])]).to(dev)
        _, sc, _, _ = dm.send_plan()
        sb = torch.zeros(3 * int(sc.sum()) + 3, dtype=torch.float64, device=dev)
        dm.pack(xe.data_ptr(), sb.data_ptr())
        xexts.append(xe)
        sends.append(sb)
        ys.append(torch.zeros(3 * inf["nloc"], dtype=torch.float64, device=dev))
    # transport: sender q's segment for r -> r's ghost segment from q
    for r, dm in enumerate(dms):
        nloc = dm.info()["nloc"]
        rp, rc, ro = dm.recv_plan()
        for p, c, o in zip(rp, rc, ro):
            sp, sc, so, _ = dms[p].send_plan()
            k = sp.index(r)
            assert sc[k] == c
            xexts[r][3 * (nloc + o):3 * (nloc + o + c)] = sends[p][3 * so[k]:3 * (so[k] + c)]
    for r, dm in enumerate(dms):
        dm.spmv(0, xexts[r].data_ptr(), ys[r].data_ptr())
        dm.spmv(1, xexts[r].data_ptr(), ys[r].data_ptr())
    torch.cuda.synchronize()
    y = np.concatenate([t.cpu().numpy() for t in ys])
    A = pb.Bsr3.from_host(full.nbrows, full.nbrows, full.ptr, full.col, full.val.reshape(-1))
    yg = A.spmv(x)
    yr = ref.spmv_bsr3(full.nbrows, full.nbrows, full.ptr, full.col, full.val.reshape(-1), x)
    assert np.abs(y - yg).max() <= 1e-14 * np.abs(yg).max()
    assert np.abs(y - yr).max() <= 1e-13 * np.abs(yr).max()


@pytest.mark.parametrize("min_rows", [1, 10**7])
def test_multi_gpu_solver_single_rank(gpu, min_rows):
    """samg_dsetup / samg_dcg_solve on one rank (NCCL communicator of size
    1): the partitioned V-cycle (all levels partitioned, or only the fine
    one) must reproduce the single-GPU solve."""
    from paper_2202_09056_b200.dist import DistHierarchy
    pb = gpu
    p = pb.generate_hex(nx=10, ny=8, nz=7, dirichlet="eliminate", load="traction_xend")
    prm = pb.AmgParams(coarse_enough=150)
    h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), "ns_block", prm)
    u1, r1 = h.cg_solve(p.rhs)
    dh = DistHierarchy(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), 0, 1,
                       min_rows=min_rows, prm=prm)
    inf = dh.info()
    assert inf["row0"] == 0 and inf["row1"] == p.nbrows
    assert 1 <= inf["dist_levels"] <= inf["nlevels"] - 1
    if min_rows == 1:
        assert inf["dist_levels"] == inf["nlevels"] - 1
    u2, r2 = dh.cg_solve(p.rhs)
    assert r2["converged"] and r1["converged"]
    assert abs(r1["iterations"] - r2["iterations"]) <= 1
    assert np.linalg.norm(u1 - u2) <= 1e-10 * np.linalg.norm(u1)
    assert r2["relative_residual"] <= 1e-8 * 1.01


EMU_CASES = [
    # world, min_rows, (pre, post), smoother, uneven row split, pipeline
    (2, 1, (1, 1), "spai0", False, "ns_block"),
    (3, 1, (1, 1), "spai0", True, "ns_block"),
    (4, 8, (2, 2), "spai0", False, "ns_block"),
    (5, 1, (1, 1), "jacobi", True, "ns_block"),
    (2, 1, (1, 1), "block_jacobi", False, "ns_block"),
    (3, 10**7, (1, 1), "spai0", False, "ns_block"),
    (3, 1, (1, 1), "spai0", True, "ns_hybrid2"),
    (2, 1, (1, 1), "spai0", False, "block"),
]


@pytest.mark.parametrize("world,min_rows,sweeps,smoother,uneven,pipeline", EMU_CASES)
def test_emulated_multi_gpu_solver(gpu, world, min_rows, sweeps, smoother, uneven, pipeline):
    """samg_dsetup with id=NULL: all `world` row slices of the partitioned
    hierarchy driven from one process, every NCCL step replaced by device
    copies with the same offsets/counts.  The partitioned PCG must reproduce
    the single-GPU solve (same hierarchy; only dot-product and SpMV
    summation order differ)."""
    from paper_2202_09056_b200.dist import DistHierarchy
    pb = gpu
    p = pb.generate_hex(nx=16, ny=8, nz=8, dirichlet="eliminate", load="traction_xend")
    prm = pb.AmgParams(coarse_enough=60, smoother=smoother, smoother_omega=0.5,
                       pre_sweeps=sweeps[0], post_sweeps=sweeps[1])
    B = None if pipeline == "block" else p.nullspace()
    h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), B, pipeline, prm)
    u1, r1 = h.cg_solve(p.rhs)
    rs = None
    if uneven:
        cuts = np.cumsum([1] + [2 * k + 1 for k in range(world - 1)])
        rs = np.concatenate([[0], np.round(p.nbrows * cuts / cuts[-1] * 0.999).astype(np.int64)])
        rs[-1] = p.nbrows
    dh = DistHierarchy(p.nbrows, p.ptr, p.col, p.val.reshape(-1), B, 0, world,
                       row_starts=rs, min_rows=min_rows, prm=prm, emulate=True, pipeline=pipeline)
    inf = dh.info()
    assert inf["row0"] == 0 and inf["row1"] == p.nbrows
    if min_rows == 1:
        assert inf["dist_levels"] >= 2
    if min_rows >= 10**7:
        assert inf["dist_levels"] == 1
    u2, r2 = dh.cg_solve(p.rhs)
    assert r1["converged"] and r2["converged"]
    assert abs(r1["iterations"] - r2["iterations"]) <= 1
    assert np.linalg.norm(u1 - u2) <= 1e-9 * np.linalg.norm(u1)
    assert r2["relative_residual"] <= 1e-8 * 1.01


def test_emulated_rejects_empty_rank(gpu):
    from paper_2202_09056_b200._lib import InvalidArgument
    from paper_2202_09056_b200.dist import DistHierarchy
    pb = gpu
    p = pb.generate_hex(nx=6, ny=4, nz=4, dirichlet="eliminate")
    with pytest.raises(InvalidArgument):
        DistHierarchy(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), 0, 2,
                      row_starts=[0, 0, p.nbrows], prm=pb.AmgParams(coarse_enough=30),
                      emulate=True)


@pytest.mark.parametrize("world,uneven,pipeline,min_rows", [
    (2, False, "ns_block", 1), (3, True, "ns_block", 1), (4, False, "ns_hybrid2", 1),
    (3, False, "block", 1), (5, True, "ns_block", 1), (3, False, "ns_hybrid1", 1),
    (4, False, "ns_block", 200)])
def test_distributed_setup_is_bit_identical(gpu, world, uneven, pipeline, min_rows):
    """The multi-GPU setup is distributed (dsetup.cu): every rank builds only
    its rows of each level from its own rows plus fetched halo rows; the
    node graph is gathered so that the aggregation is global.  Emulated here
    rank by rank: every level matrix, assembled from the ranks' rows, must
    be bit-identical to the single-GPU setup's (and so to the reference)."""
    from paper_2202_09056_b200.dist import DistHierarchy
    pb = gpu
    p = pb.generate_hex(nx=16, ny=8, nz=8, dirichlet="eliminate", load="traction_xend")
    prm = pb.AmgParams(coarse_enough=60)
    B = None if pipeline == "block" else p.nullspace()
    h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), B, pipeline, prm)
    rs = None
    if uneven:
        cuts = np.cumsum([1] + [2 * k + 1 for k in range(world - 1)])
        rs = np.concatenate([[0], np.round(p.nbrows * cuts / cuts[-1] * 0.999).astype(np.int64)])
        rs[-1] = p.nbrows
    dh = DistHierarchy(p.nbrows, p.ptr, p.col, p.val.reshape(-1), B, 0, world, row_starts=rs,
                       min_rows=min_rows, prm=prm, emulate=True, pipeline=pipeline)
    inf = dh.info()
    assert inf["nlevels"] == h.nlevels
    if min_rows == 1:
        assert inf["dist_levels"] >= 2
    for lvl in range(h.nlevels):
        for w in ((0, 1, 2) if lvl + 1 < h.nlevels else (0,)):
            a, b = h.level(lvl, w), dh.level(lvl, w)
            assert a[0] == b[0] and a[1] == b[1], (lvl, w)
            for x, y in zip(a[2:], b[2:]):
                assert np.array_equal(x, y), (lvl, w)


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_setup_holds_slab_plus_halo(gpu, world):
    """No rank holds more of A_0 than its slab plus the halo layers the
    setup needs (strength: one node layer; Galerkin: the rows within the
    support of its aggregates' prolongator columns and their neighbours).
    A slender x-slowest beam: every rank owns 10 x-planes of 49 nodes."""
    from paper_2202_09056_b200.dist import DistHierarchy
    pb = gpu
    p = pb.generate_hex(nx=10 * world, ny=6, nz=6, lx=10.0 * world / 6, dirichlet="eliminate",
                        load="traction_xend", x_slowest=True)
    plane = 7 * 7
    rs = np.array([10 * plane * r for r in range(world + 1)], np.int64)
    prm = pb.AmgParams(coarse_enough=60)
    h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), "ns_block", prm)
    dh = DistHierarchy(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), 0, world,
                       row_starts=rs, min_rows=1, prm=prm, emulate=True)
    inf = dh.info()
    # rank 0: its 10 planes + at most 6 halo planes on its one neighbour side
    assert 10 * plane < inf["held_rows"] <= 16 * plane, inf
    assert inf["held_rows"] < p.nbrows
    for lvl in range(h.nlevels):
        for w in ((0, 1, 2) if lvl + 1 < h.nlevels else (0,)):
            a, b = h.level(lvl, w), dh.level(lvl, w)
            for x, y in zip(a[2:], b[2:]):
                assert np.array_equal(x, y), (lvl, w)
    u1, r1 = h.cg_solve(p.rhs)
    u2, r2 = dh.cg_solve(p.rhs)
    assert r1["converged"] and r2["converged"]
    assert abs(r1["iterations"] - r2["iterations"]) <= 1
    assert np.linalg.norm(u1 - u2) <= 1e-9 * np.linalg.norm(u1)


@pytest.mark.parametrize("mode", ["device", "local"])
def test_rank_local_input_single_rank(gpu, mode):
    """samg_dsetup_device / samg_dsetup_local: the rank passes only its own
    rows (here, one NCCL rank: all of them) -- from the on-GPU assembly or
    from host arrays -- and the distributed setup + graph-captured PCG
    reproduce the single-GPU hierarchy and solve."""
    import torch

    from paper_2202_09056_b200.dist import DistHierarchy
    pb = gpu
    kw = dict(nx=12, ny=6, nz=6, lx=2.0, dirichlet="eliminate", load="traction_xend", x_slowest=True)
    host = pb.generate_hex(**kw)
    prm = pb.AmgParams(coarse_enough=60)
    h = pb.setup_bsr3(host.nbrows, host.ptr, host.col, host.val.reshape(-1), host.nullspace(),
                      "ns_block", prm)
    u1, r1 = h.cg_solve(host.rhs)
    rs = np.array([0, host.nbrows], np.int64)
    if mode == "device":
        dp = pb.generate_hex_device(**kw)
        dh = DistHierarchy(0, None, None, None, None, 0, 1, row_starts=rs, min_rows=1, prm=prm,
                           device=(dp.A, dp.nullspace_ptr))
    else:
        dh = DistHierarchy(0, None, None, None, None, 0, 1, row_starts=rs, min_rows=1, prm=prm,
                           local=(host.ptr, host.col, host.val.reshape(-1), host.nullspace()))
    inf = dh.info()
    assert inf["nlevels"] == h.nlevels and inf["dist_levels"] >= 1
    for lvl in range(h.nlevels):
        for w in ((0, 1, 2) if lvl + 1 < h.nlevels else (0,)):
            a, b = h.level(lvl, w), dh.level(lvl, w)
            for x, y in zip(a[2:], b[2:]):
                assert np.array_equal(x, y), (lvl, w)
    f = torch.from_numpy(host.rhs).cuda()
    u = torch.zeros_like(f)
    r2 = dh.cg_solve_device(f.data_ptr(), u.data_ptr())
    assert r1["converged"] and r2["converged"]
    assert abs(r1["iterations"] - r2["iterations"]) <= 1
    assert np.linalg.norm(u1 - u.cpu().numpy()) <= 1e-9 * np.linalg.norm(u1)
