"""Row-partitioned BSR3 operator across ranks (one process per GPU).

The partition and halo plan are native (dist.cu, behind the C-ABI
``samg_dist_*``); this module only moves data with ``torch.distributed``
(NCCL between GPUs, gloo for the CPU tests): the ghost-id lists once, then
per SpMV the packed send buffers into the ghost segments of ``x_ext``.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, f64p, i64p, lib, vp


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class DistMatrix:
    """A rank's rows [row_starts[rank], row_starts[rank+1]) of a global
    3x3-BSR matrix (global column ids in ``col``)."""

    def __init__(self, ptr, col, val, row_starts, rank):
        row_starts = _i64(row_starts)
        ptr, col = _i64(ptr), _i64(col)
        val = np.ascontiguousarray(val, dtype=np.float64)
        self.rank, self.nranks = rank, len(row_starts) - 1
        self.row_starts = row_starts
        from ._lib import InvalidArgument
        nrows = int(row_starts[rank + 1] - row_starts[rank])
        if len(ptr) != nrows + 1 or len(col) < ptr[-1] - ptr[0] or val.size < 9 * (ptr[-1] - ptr[0]):
            raise InvalidArgument("dist: ptr/col/val do not match the rank's row range", 105)
        h = vp()
        check(lib.samg_dist_create(int(row_starts[rank]), int(row_starts[rank + 1]),
                                   ptr.ctypes.data_as(i64p), col.ctypes.data_as(i64p),
                                   val.ctypes.data_as(f64p), self.nranks,
                                   row_starts.ctypes.data_as(i64p), rank, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib.samg_dist_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def info(self):
        a, b, c, d = (C.c_int64() for _ in range(4))
        e, f = C.c_int(), C.c_int()
        check(lib.samg_dist_info(self.h, C.byref(a), C.byref(b), C.byref(c), C.byref(d),
                                 C.byref(e), C.byref(f)))
        return dict(nloc=a.value, nghost=b.value, ninterior=c.value, nboundary=d.value,
                    nrecv=e.value, nsend=f.value)

    def recv_plan(self):
        n = self.info()["nrecv"]
        peers = (C.c_int * max(n, 1))()
        counts, offsets = np.zeros(n, np.int64), np.zeros(n, np.int64)
        check(lib.samg_dist_recv_plan(self.h, peers, counts.ctypes.data_as(i64p),
                                      offsets.ctypes.data_as(i64p)))
        return [peers[i] for i in range(n)], counts, offsets

    def ghosts(self):
        g = np.zeros(self.info()["nghost"], np.int64)
        check(lib.samg_dist_ghosts(self.h, g.ctypes.data_as(i64p)))
        return g

    def set_send(self, peers, counts, ids):
        peers = list(peers)
        arr = (C.c_int * max(len(peers), 1))(*peers)
        counts, ids = _i64(counts), _i64(ids)
        check(lib.samg_dist_set_send(self.h, len(peers), arr, counts.ctypes.data_as(i64p),
                                     ids.ctypes.data_as(i64p)))

    def derive_send(self):
        """The send plan from the rank's own rows (structural symmetry; no
        transport): samg_dist_derive_send."""
        check(lib.samg_dist_derive_send(self.h))

    def send_plan(self):
        """(peers, counts, offsets, local block rows) of the send side."""
        n = self.info()["nsend"]
        peers = (C.c_int * max(n, 1))()
        counts, offsets = np.zeros(n, np.int64), np.zeros(n, np.int64)
        check(lib.samg_dist_send_plan(self.h, peers, counts.ctypes.data_as(i64p),
                                      offsets.ctypes.data_as(i64p), None))
        rows = np.zeros(int(counts.sum()) + 1, np.int64)
        check(lib.samg_dist_send_plan(self.h, peers, counts.ctypes.data_as(i64p),
                                      offsets.ctypes.data_as(i64p), rows.ctypes.data_as(i64p)))
        return [peers[i] for i in range(n)], counts, offsets, rows[:int(counts.sum())]

    def local_csr(self):
        """The renumbered local matrix: columns [0,nloc) owned, nloc+g ghosts."""
        nl = self.info()["nloc"]
        ptr = np.zeros(nl + 1, np.int64)
        check(lib.samg_dist_local_matrix(self.h, ptr.ctypes.data_as(i64p), None, None))
        nnzb = int(ptr[-1])
        col, val = np.zeros(nnzb, np.int64), np.zeros(9 * nnzb)
        check(lib.samg_dist_local_matrix(self.h, ptr.ctypes.data_as(i64p),
                                         col.ctypes.data_as(i64p), val.ctypes.data_as(f64p)))
        return ptr, col, val.reshape(-1, 3, 3)

    def to_device(self, device, group=0):
        check(lib.samg_dist_to_device(self.h, device, group))

    def pack(self, x_ptr, buf_ptr, stream=0):
        check(lib.samg_dist_pack(self.h, x_ptr, buf_ptr, stream or None))

    def spmv(self, part, x_ext_ptr, y_ptr, alpha=1.0, beta=0.0, stream=0):
        check(lib.samg_dist_spmv(self.h, part, alpha, x_ext_ptr, beta, y_ptr, stream or None))


def exchange_plan(dm: DistMatrix, dist, device=None):
    """Tell every owner which of its rows this rank needs (ghost ids), and
    install the resulting send plan.  Works with gloo (CPU tensors) and NCCL
    (``device`` tensors)."""
    import torch
    rank, world = dm.rank, dm.nranks
    peers, counts, offsets = dm.recv_plan()
    ghosts = dm.ghosts()
    need = np.zeros(world, np.int64)
    for p, c in zip(peers, counts):
        need[p] = c
    t = torch.from_numpy(need)
    if device is not None:
        t = t.to(device)
    allc = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(allc, t)
    send_counts = [int(allc[q][rank]) for q in range(world)]
    ops, recvbufs = [], {}
    for p, c, o in zip(peers, counts, offsets):
        buf = torch.from_numpy(np.ascontiguousarray(ghosts[o:o + c]))
        if device is not None:
            buf = buf.to(device)
        ops.append(dist.P2POp(dist.isend, buf, p))
    for q in range(world):
        if send_counts[q]:
            rb = torch.zeros(send_counts[q], dtype=torch.int64,
                             device=device if device is not None else "cpu")
            recvbufs[q] = rb
            ops.append(dist.P2POp(dist.irecv, rb, q))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    speers = sorted(recvbufs)
    scounts = [send_counts[q] for q in speers]
    ids = np.concatenate([recvbufs[q].cpu().numpy() for q in speers]) if speers else \
        np.zeros(0, np.int64)
    dm.set_send(speers, scounts, ids)


class Halo:
    """Per-SpMV halo exchange of a device vector (torch tensors on the rank's
    GPU): pack owned entries, send to peers, receive into the ghost part of
    ``x_ext``."""

    def __init__(self, dm: DistMatrix, dist, device):
        import torch
        self.dm, self.dist = dm, dist
        inf = dm.info()
        self.nloc, self.nghost = inf["nloc"], inf["nghost"]
        self.rpeers, self.rcounts, self.roffs = dm.recv_plan()
        self.speers, self.scounts, self.soffs, _ = dm.send_plan()
        self.sendbuf = torch.zeros(3 * int(self.scounts.sum()) + 3, dtype=torch.float64,
                                   device=device)
        self.x_ext = torch.zeros(3 * (self.nloc + self.nghost) + 3, dtype=torch.float64,
                                 device=device)

    def start(self, stream_handle=0):
        """pack + post the sends/receives; returns the request list"""
        dist = self.dist
        self.dm.pack(self.x_ext.data_ptr(), self.sendbuf.data_ptr(), stream_handle)
        ops = []
        for p, c, o in zip(self.speers, self.scounts, self.soffs):
            ops.append(dist.P2POp(dist.isend, self.sendbuf[3 * o:3 * (o + c)], p))
        base = 3 * self.nloc
        for p, c, o in zip(self.rpeers, self.rcounts, self.roffs):
            ops.append(dist.P2POp(dist.irecv, self.x_ext[base + 3 * o:base + 3 * (o + c)], p))
        return dist.batch_isend_irecv(ops) if ops else []


def _load_torch_nccl():
    """The library resolves NCCL at first use from the libnccl.so.2 already in
    the process (nccl_shim.cuh); importing torch first makes that torch's own
    copy, so both share one NCCL."""
    import torch  # noqa: F401


def nccl_unique_id() -> bytes:
    _load_torch_nccl()
    buf = (C.c_ubyte * 128)()
    check(lib.samg_nccl_unique_id(buf))
    return bytes(buf)


class DistHierarchy:
    """Multi-GPU hierarchy with a distributed setup (samg_dsetup*): every
    rank builds only its rows of the large levels (dsetup.cu); the solve runs
    on the rank's rows with NCCL halos.  The NCCL id is created on rank 0 and
    broadcast with torch.distributed.

    Input, one of:
      * the global matrix (nbrows, ptr, col, val) and nullspace B on every
        rank -- only the rank's rows are uploaded (samg_dsetup);
      * ``local=(ptr, col, val, B_local)``: the rank's own rows (ptr from 0,
        global column ids) and nullspace rows, with ``row_starts``
        (samg_dsetup_local);
      * ``device=(bsr3, d_B_ptr)``: the rank's rows as a device Bsr3 and
        its nullspace rows in device memory (samg_dsetup_device).
    ``emulate=True`` drives all ``nranks`` slices from this process on one
    GPU without NCCL (every exchange a device copy); f and u are then the
    global vectors."""

    def __init__(self, nbrows, ptr, col, val, B, rank, nranks, dist=None, row_starts=None,
                 min_rows=4096, prm=None, uid=None, emulate=False, pipeline="ns_block",
                 local=None, device=None, b_cols=6):
        from .api import AmgParams, _nullspace, _pipeline
        prm = prm or AmgParams()
        idbuf = None
        if emulate:
            rank = 0
        else:
            _load_torch_nccl()
            if uid is None:
                obj = [nccl_unique_id() if rank == 0 else None]
                if dist is not None and nranks > 1:
                    dist.broadcast_object_list(obj, src=0)
                uid = obj[0]
            idbuf = (C.c_ubyte * 128).from_buffer_copy(uid)
        rs = None if row_starts is None else _i64(row_starts)
        pc = prm.c()
        h = vp()
        if local is not None or device is not None:
            if emulate or rs is None:
                raise ValueError("local / device input needs NCCL and row_starts")
            if device is not None:
                A, bptr = device
                check(lib.samg_dsetup_device(idbuf, nranks, rank, rs.ctypes.data_as(i64p), A.h,
                                             bptr or None, b_cols, min_rows, _pipeline(pipeline),
                                             C.byref(pc), C.byref(h)))
            else:
                lp, lc, lv, lb = local
                lp, lc = _i64(lp), _i64(lc)
                lv = np.ascontiguousarray(lv, dtype=np.float64)
                lb = None if lb is None else np.ascontiguousarray(lb, dtype=np.float64)
                check(lib.samg_dsetup_local(idbuf, nranks, rank, rs.ctypes.data_as(i64p),
                                            lp.ctypes.data_as(i64p), lc.ctypes.data_as(i64p),
                                            lv.ctypes.data_as(f64p),
                                            lb.ctypes.data_as(f64p) if lb is not None else None,
                                            b_cols, min_rows, _pipeline(pipeline), C.byref(pc),
                                            C.byref(h)))
        else:
            ptr, col = _i64(ptr), _i64(col)
            val = np.ascontiguousarray(val, dtype=np.float64)
            Bv, brows, k = _nullspace(B, 3 * nbrows)
            check(lib.samg_dsetup(idbuf, nranks, rank, nbrows, ptr.ctypes.data_as(i64p),
                                  col.ctypes.data_as(i64p), val.ctypes.data_as(f64p),
                                  Bv.ctypes.data_as(f64p) if Bv is not None else None, brows, k,
                                  rs.ctypes.data_as(i64p) if rs is not None else None, min_rows,
                                  _pipeline(pipeline),
                                  C.byref(pc), C.byref(h)))
        self.h = h
        self.rank, self.nranks = rank, nranks

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib.samg_ddestroy(self.h)
            except Exception:
                pass
            self.h = None

    def close(self):
        self.__del__()

    def info(self):
        r0, r1 = C.c_int64(), C.c_int64()
        nl, dl = C.c_int(), C.c_int()
        ss = C.c_double()
        check(lib.samg_dinfo(self.h, C.byref(r0), C.byref(r1), C.byref(nl), C.byref(dl),
                             C.byref(ss)))
        hr = C.c_int64()
        check(lib.samg_dheld_rows(self.h, C.byref(hr)))
        return dict(row0=r0.value, row1=r1.value, nlevels=nl.value, dist_levels=dl.value,
                    setup_seconds=ss.value, held_rows=hr.value)

    def level(self, level, which=0):
        """(nrows, ncols, ptr, col, val[nnzb,3,3]) of the global A (0), P (1)
        or R (2) of `level`, assembled from every rank's rows (collective)."""
        import numpy as np
        nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.samg_dlevel_info(self.h, level, which, C.byref(nr), C.byref(nc), C.byref(nz)))
        ptr, col = np.zeros(nr.value + 1, np.int64), np.zeros(nz.value, np.int64)
        val = np.zeros(9 * nz.value)
        check(lib.samg_dget_level(self.h, level, which, ptr.ctypes.data_as(C.POINTER(C.c_int64)),
                                  col.ctypes.data_as(C.POINTER(C.c_int64)),
                                  val.ctypes.data_as(C.POINTER(C.c_double))))
        return nr.value, nc.value, ptr, col, val.reshape(-1, 3, 3)

    def cg_solve(self, f_local, prm=None):
        from ._lib import CgParamsC, ReportC
        from .api import CgParams, _report
        prm = prm or CgParams()
        f = np.ascontiguousarray(f_local, dtype=np.float64)
        u = np.zeros_like(f)
        rep = ReportC()
        cp = CgParamsC(prm.tol, prm.max_iterations)
        check(lib.samg_dcg_solve(self.h, f.ctypes.data_as(f64p), u.ctypes.data_as(f64p),
                                 C.byref(cp), C.byref(rep)))
        return u, _report(rep)

    def cg_solve_device(self, f_ptr, u_ptr, prm=None):
        from ._lib import CgParamsC, ReportC
        from .api import CgParams, _report
        prm = prm or CgParams()
        rep = ReportC()
        cp = CgParamsC(prm.tol, prm.max_iterations)
        check(lib.samg_dcg_solve_device(self.h, f_ptr, u_ptr, C.byref(cp), C.byref(rep)))
        return _report(rep)
