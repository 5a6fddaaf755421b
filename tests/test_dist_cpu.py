"""Multi-rank host logic of the row-partitioned operator, on CPU with gloo.

world_size 2 and 3 processes each build their slab of a cantilever (x
slowest, so slabs are contiguous x-planes) with the native partition/halo
plan (samg_dist_*), exchange ghost-id lists over gloo, then run the halo
exchange for real (pack by the send plan, isend/irecv into the ghost
segments) and multiply with the renumbered local matrix on the host.  The
distributed product must equal the global product, and the plan must be
consistent (interior + boundary = all rows, ghosts = off-rank columns).
The device side of the same plan is covered by tests/test_gpu_dist.py.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

PROB = dict(nx=11, ny=3, nz=4, lx=3.0, dirichlet="eliminate", load="traction_xend",
            x_slowest=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def bsr_mv(ptr, col, val, x):
    nr = len(ptr) - 1
    y = np.zeros(3 * nr)
    for i in range(nr):
        for j in range(ptr[i], ptr[i + 1]):
            y[3 * i:3 * i + 3] += val[j] @ x[3 * col[j]:3 * col[j] + 3]
    return y


def row_starts_for(pp, world):
    planes = pp.nx  # eliminate: kept x-planes = nx
    per_plane = (pp.ny + 1) * (pp.nz + 1)
    cuts = [round(planes * r / world) for r in range(world + 1)]
    return np.array([c * per_plane for c in cuts], dtype=np.int64)


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    import paper_2202_09056_b200 as pb
    from paper_2202_09056_b200.dist import DistMatrix, exchange_plan

    pp = pb.ProblemParams(**PROB)
    full = pb.generate_hex(pp)
    starts = row_starts_for(pp, world)
    r0, r1 = int(starts[rank]), int(starts[rank + 1])
    mine = pb.generate_hex(pb.ProblemParams(**{**PROB, "node_begin": r0, "node_end": r1}))
    # the slab is exactly the full problem's rows
    np.testing.assert_array_equal(mine.ptr, full.ptr[r0:r1 + 1] - full.ptr[r0])
    np.testing.assert_array_equal(mine.col, full.col[full.ptr[r0]:full.ptr[r1]])
    np.testing.assert_array_equal(mine.val, full.val[full.ptr[r0]:full.ptr[r1]])

    dm = DistMatrix(mine.ptr, mine.col, mine.val.reshape(-1), starts, rank)
    # the rule the distributed setup / solve use (dsolve.cu build_local_rows):
    # the owner derives what each peer reads from its own rows ...
    dm.derive_send()
    derived = dm.send_plan()
    # ... and it must equal what the peers' ghost lists say (gloo exchange)
    exchange_plan(dm, dist)
    got = dm.send_plan()
    assert derived[0] == got[0]
    for a, b in zip(derived[1:], got[1:]):
        np.testing.assert_array_equal(a, b)
    inf = dm.info()
    assert inf["nloc"] == r1 - r0
    assert inf["ninterior"] + inf["nboundary"] == inf["nloc"]
    ghosts = dm.ghosts()
    off = np.unique(mine.col[(mine.col < r0) | (mine.col >= r1)])
    np.testing.assert_array_equal(ghosts, off)

    # halo exchange for real: pack by the send plan, isend/irecv over gloo
    x = np.random.default_rng(7).uniform(-1, 1, full.n)
    xloc = x[3 * r0:3 * r1]
    speers, scounts, soffs, srows = dm.send_plan()
    rpeers, rcounts, roffs = dm.recv_plan()
    send = np.concatenate([xloc.reshape(-1, 3)[srows].reshape(-1)]) if len(srows) else np.zeros(0)
    xext = np.zeros(3 * (inf["nloc"] + inf["nghost"]))
    xext[:3 * inf["nloc"]] = xloc
    sbuf = torch.from_numpy(send.copy())
    rbuf = torch.zeros(3 * inf["nghost"], dtype=torch.float64)
    ops = [dist.P2POp(dist.isend, sbuf[3 * o:3 * (o + c)], p) for p, c, o in zip(speers, scounts, soffs)]
    ops += [dist.P2POp(dist.irecv, rbuf[3 * o:3 * (o + c)], p) for p, c, o in zip(rpeers, rcounts, roffs)]
    for r in (dist.batch_isend_irecv(ops) if ops else []):
        r.wait()
    xext[3 * inf["nloc"]:] = rbuf.numpy()
    # ghost values are the owners' x entries
    np.testing.assert_array_equal(xext[3 * inf["nloc"]:].reshape(-1, 3), x.reshape(-1, 3)[ghosts])
    lptr, lcol, lval = dm.local_csr()
    y = bsr_mv(lptr, lcol, lval, xext)
    yref = bsr_mv(full.ptr[r0:r1 + 1] - full.ptr[r0], full.col[full.ptr[r0]:full.ptr[r1]],
                  full.val[full.ptr[r0]:full.ptr[r1]], x)
    # same per-row block order -> identical sums
    np.testing.assert_array_equal(y, yref)
    np.save(os.path.join(outdir, f"y{rank}.npy"), y)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_spmv_gloo(tmp_path, world):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    import paper_2202_09056_b200 as pb
    full = pb.generate_hex(pb.ProblemParams(**PROB))
    x = np.random.default_rng(7).uniform(-1, 1, full.n)
    y = np.concatenate([np.load(tmp_path / f"y{r}.npy") for r in range(world)])
    np.testing.assert_allclose(y, bsr_mv(full.ptr, full.col, full.val, x), rtol=0, atol=1e-13)


def test_partition_validation():
    import paper_2202_09056_b200 as pb
    from paper_2202_09056_b200.dist import DistMatrix
    p = pb.generate_hex(pb.ProblemParams(**PROB))
    starts = np.array([0, p.nbrows // 2, p.nbrows])
    with pytest.raises(pb.InvalidArgument):
        DistMatrix(p.ptr[:10], p.col, p.val.reshape(-1), starts, 0)  # wrong row range
    dm = DistMatrix(p.ptr[:starts[1] + 1], p.col[:p.ptr[starts[1]]],
                    p.val[:p.ptr[starts[1]]].reshape(-1), starts, 0)
    with pytest.raises(pb.InvalidArgument):
        dm.set_send([1], [1], [p.nbrows - 1])  # rank 0 does not own that row
    with pytest.raises(pb.InvalidArgument):
        dm.to_device(0)  # send plan not set
