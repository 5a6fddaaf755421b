"""Pythonic mirror of the reference interface over the C-ABI.

Names follow proj/include/samg: ``setup`` / ``vcycle`` / ``cg_solve`` /
``memory_footprint``; parameters mirror ``amg_params`` (hierarchy.hpp:50-58),
``coarsening_params`` (coarsening.hpp:26-31) and ``cg_params`` (cg.hpp:32-35).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import (AmgParamsC, CgParamsC, ProblemParamsC, ReportC, check, f64p, i64p, lib, vp)

PIPELINES = {"scalar": 0, "block": 1, "ns_scalar": 2, "ns_hybrid1": 3, "ns_hybrid2": 4,
             "ns_block": 5}
SMOOTHERS = {"jacobi": 0, "spai0": 1, "block_jacobi": 2, "ilu0": 3}
PRECISIONS = {"fp64": 0, "mixed": 1}
ILU_ORDERS = {"reference": 0, "latest_last": 1}


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t=f64p):
    return a.ctypes.data_as(t)


def device_count() -> int:
    n = C.c_int()
    check(lib.samg_device_count(C.byref(n)))
    return n.value


@dataclass
class AmgParams:
    eps_strong: float = 0.08
    omega: float = 2.0 / 3.0
    point_block_size: int = 3
    smoother: str = "spai0"
    smoother_omega: float = 0.72
    pre_sweeps: int = 1
    post_sweeps: int = 1
    coarse_enough: int = 3000
    stagnation_ratio: float = 0.8
    device: int = 0
    # "fp64" (the reference) or "mixed": fp32 operator copies for the V-cycle
    vcycle_precision: str = "fp64"
    # hierarchy.hpp:382-401: recompute each coarse operator and compare
    verify_galerkin: bool = False
    # block ILU(0) backward sweep: "reference" (bit-identical applications) or
    # "latest_last" (descending columns: same sums up to rounding, shorter chain
    # after the last hand-off)
    ilu_sweep_order: str = "reference"

    def c(self) -> AmgParamsC:
        return AmgParamsC(self.eps_strong, self.omega, self.point_block_size,
                          SMOOTHERS[self.smoother] if isinstance(self.smoother, str)
                          else int(self.smoother), self.smoother_omega, self.pre_sweeps,
                          self.post_sweeps, self.coarse_enough, self.stagnation_ratio,
                          int(self.verify_galerkin),
                          self.device, PRECISIONS[self.vcycle_precision],
                          ILU_ORDERS[self.ilu_sweep_order])


@dataclass
class CgParams:
    tol: float = 1e-8
    max_iterations: int = 1000


def _report(r: ReportC) -> dict:
    return dict(iterations=r.iterations, relative_residual=r.relative_residual,
                setup_seconds=r.setup_seconds, solve_seconds=r.solve_seconds,
                preconditioner_bytes=r.preconditioner_bytes, variant=r.variant,
                converged=bool(r.converged))


class Bsr3:
    """A device-resident 3x3 BSR matrix (csr<static_block<3>>, csr.hpp:26-40)."""

    def __init__(self, handle, owner=None):
        self.h = handle
        self._owner = owner  # a Hierarchy for borrowed level matrices

    @classmethod
    def from_host(cls, nrows, ncols, ptr, col, val, device=0) -> "Bsr3":
        ptr, col, val = _i64(ptr), _i64(col), _f64(val)
        h = vp()
        check(lib.samg_bsr3_create(nrows, ncols, _p(ptr, i64p), _p(col, i64p), _p(val),
                                   device, C.byref(h)))
        return cls(h)

    def __del__(self):
        if self._owner is None and getattr(self, "h", None):
            try:
                lib.samg_bsr3_destroy(self.h)
            except Exception:
                pass
            self.h = None

    @property
    def shape(self):
        nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.samg_bsr3_info(self.h, C.byref(nr), C.byref(nc), C.byref(nz)))
        return nr.value, nc.value, nz.value

    def download(self):
        nr, nc, nz = self.shape
        ptr, col = np.zeros(nr + 1, np.int64), np.zeros(nz, np.int64)
        val = np.zeros(9 * nz)
        check(lib.samg_bsr3_download(self.h, _p(ptr, i64p), _p(col, i64p), _p(val)))
        return nr, nc, ptr, col, val.reshape(-1, 3, 3)

    def spmv(self, x, alpha=1.0, beta=0.0, y=None):
        """Host vectors (H2D, kernel, D2H) -- the e2e path."""
        nr, nc, _ = self.shape
        x = _f64(x)
        y = np.zeros(3 * nr) if y is None else _f64(y).copy()
        check(lib.samg_bsr3_spmv(self.h, alpha, _p(x), beta, _p(y)))
        return y

    def spmv_batch(self, X, alpha=1.0, beta=0.0, Y=None):
        """Rows of X (count x 3*ncols host array) -> rows of Y, each product
        with its own H2D/D2H, pipelined (samg_bsr3_spmv_batch)."""
        nr, nc, _ = self.shape
        X = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, 3 * nc)
        Y = np.zeros((X.shape[0], 3 * nr)) if Y is None else np.ascontiguousarray(Y, dtype=np.float64)
        check(lib.samg_bsr3_spmv_batch(self.h, alpha, X.ctypes.data, beta, Y.ctypes.data, X.shape[0]))
        return Y

    def spmv_device(self, x_ptr: int, y_ptr: int, alpha=1.0, beta=0.0, stream: int = 0):
        check(lib.samg_bsr3_spmv_device(self.h, alpha, x_ptr, beta, y_ptr, stream or None))

    def spmv_bytes(self, beta_nonzero=False) -> int:
        b = C.c_uint64()
        check(lib.samg_bsr3_spmv_bytes(self.h, int(beta_nonzero), C.byref(b)))
        return b.value

    def dense_inverse(self) -> np.ndarray:
        """A^-1 as a dense host array (the coarsest-level solver, coarse.cu)."""
        nr, nc, _ = self.shape
        n = 3 * nr
        out = np.zeros((n, n))
        check(lib.samg_bsr3_dense_inverse(self.h, out.ctypes.data_as(f64p)))
        return out

    @staticmethod
    def galerkin(R: "Bsr3", A: "Bsr3", P: "Bsr3") -> "Bsr3":
        h = vp()
        check(lib.samg_bsr3_galerkin(R.h, A.h, P.h, C.byref(h)))
        return Bsr3(h)


class Hierarchy:
    """Device-resident AMG hierarchy (samg::hierarchy, hierarchy.hpp:140-148)."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib.samg_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def close(self):
        self.__del__()

    @property
    def finest_dim(self) -> int:
        n = C.c_int64()
        check(lib.samg_finest_dim(self.h, C.byref(n)))
        return n.value

    @property
    def nlevels(self) -> int:
        n = C.c_int()
        check(lib.samg_num_levels(self.h, C.byref(n)))
        return n.value

    @property
    def coarse_dim(self) -> int:
        n = C.c_int64()
        check(lib.samg_coarse_dim(self.h, C.byref(n)))
        return n.value

    @property
    def coarse_solver(self) -> str:
        """"inverse" (GEMV with the explicit inverse) or "lu" (the reference's
        dense LU, bit-exact; numerically singular coarse operators)."""
        k = C.c_int()
        check(lib.samg_coarse_solver(self.h, C.byref(k)))
        return "lu" if k.value == 1 else "inverse"

    @property
    def setup_seconds(self) -> float:
        s = C.c_double()
        check(lib.samg_setup_seconds(self.h, C.byref(s)))
        return s.value

    def memory_footprint(self) -> int:
        b = C.c_uint64()
        check(lib.samg_memory_footprint(self.h, C.byref(b)))
        return b.value

    def level_info(self, level, which=0):
        nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.samg_level_info(self.h, level, which, C.byref(nr), C.byref(nc), C.byref(nz)))
        return nr.value, nc.value, nz.value

    def level(self, level, which=0):
        """(nrows, ncols, ptr, col, val[nnzb,3,3]) of A (0), P (1) or R (2)."""
        nr, nc, nz = self.level_info(level, which)
        ptr, col = np.zeros(nr + 1, np.int64), np.zeros(nz, np.int64)
        val = np.zeros(9 * nz)
        check(lib.samg_get_level(self.h, level, which, _p(ptr, i64p), _p(col, i64p), _p(val)))
        return nr, nc, ptr, col, val.reshape(-1, 3, 3)

    def level_matrix(self, level, which=0) -> Bsr3:
        m = vp()
        check(lib.samg_level_matrix(self.h, level, which, C.byref(m)))
        return Bsr3(m, owner=self)

    def aggregates(self, level):
        nn, cnt = C.c_int64(), C.c_int64()
        check(lib.samg_aggregates_info(self.h, level, C.byref(nn), C.byref(cnt)))
        ids = np.zeros(nn.value, np.int64)
        check(lib.samg_get_aggregates(self.h, level, _p(ids, i64p)))
        return ids, cnt.value

    def smoother(self, level):
        n = C.c_int64()
        check(lib.samg_smoother_info(self.h, level, C.byref(n)))
        d = np.zeros(n.value)
        check(lib.samg_get_smoother(self.h, level, _p(d)))
        return d

    def vcycle(self, f, u=None):
        """One V-cycle; u is the initial approximation (zeros by default)."""
        f = _f64(f)
        u = np.zeros_like(f) if u is None else _f64(u).copy()
        check(lib.samg_vcycle(self.h, _p(f), _p(u)))
        return u

    def vcycle_device(self, f_ptr: int, u_ptr: int):
        check(lib.samg_vcycle_device(self.h, f_ptr, u_ptr))

    def cg_solve(self, f, prm: CgParams = CgParams()):
        f = _f64(f)
        u = np.zeros_like(f)
        rep = ReportC()
        cp = CgParamsC(prm.tol, prm.max_iterations)
        check(lib.samg_cg_solve(self.h, _p(f), _p(u), C.byref(cp), C.byref(rep)))
        return u, _report(rep)

    def cg_solve_device(self, f_ptr: int, u_ptr: int, prm: CgParams = CgParams()):
        rep = ReportC()
        cp = CgParamsC(prm.tol, prm.max_iterations)
        check(lib.samg_cg_solve_device(self.h, f_ptr, u_ptr, C.byref(cp), C.byref(rep)))
        return _report(rep)


def _pipeline(p) -> int:
    return PIPELINES[p] if isinstance(p, str) else int(p)


def _nullspace(B, n):
    """B as column-major (dense_columns, csr.hpp:46-55): accepts a flat
    column-major vector or an (n, k) array."""
    if B is None:
        return None, n, 0
    B = np.asarray(B, dtype=np.float64)
    if B.ndim == 2:
        rows, k = B.shape
        return np.ascontiguousarray(B.T).reshape(-1), rows, k
    k = B.size // n if n else 0
    return np.ascontiguousarray(B), n, k


def setup(A, B, pipeline="ns_block", prm: AmgParams = AmgParams()) -> Hierarchy:
    """samg::setup (hierarchy.hpp:263-405) from a scalar CSR ``(n, ptr, col, val)``
    or a scipy.sparse matrix."""
    if hasattr(A, "indptr"):
        A = A.tocsr()
        A.sort_indices()
        n, ptr, col, val = A.shape[0], A.indptr, A.indices, A.data
    else:
        n, ptr, col, val = A
    ptr, col, val = _i64(ptr), _i64(col), _f64(val)
    Bv, brows, k = _nullspace(B, n)
    h = vp()
    pc = prm.c()
    check(lib.samg_setup(n, _p(ptr, i64p), _p(col, i64p), _p(val),
                         _p(Bv) if Bv is not None else None, brows, k, _pipeline(pipeline),
                         C.byref(pc), C.byref(h)))
    return Hierarchy(h)


def setup_bsr3(nbrows, ptr, col, val, B, pipeline="ns_block",
               prm: AmgParams = AmgParams()) -> Hierarchy:
    ptr, col, val = _i64(ptr), _i64(col), _f64(val)
    Bv, brows, k = _nullspace(B, 3 * nbrows)
    h = vp()
    pc = prm.c()
    check(lib.samg_setup_bsr3(nbrows, _p(ptr, i64p), _p(col, i64p), _p(val),
                              _p(Bv) if Bv is not None else None, brows, k,
                              _pipeline(pipeline), C.byref(pc), C.byref(h)))
    return Hierarchy(h)


@dataclass
class ProblemParams:
    nx: int = 19
    ny: int = 19
    nz: int = 19
    lx: float = 1.0
    ly: float = 1.0
    lz: float = 1.0
    E: float = 1.0
    nu: float = 0.3
    heterogeneous: bool = False
    dirichlet: str = "eliminate"   # none | keep_rows | eliminate
    load: str = "body_force"       # body_force | traction_xend | random
    noise: float = 0.0
    seed: int = 12345
    x_slowest: bool = False
    node_begin: int = 0            # node_end > node_begin: rows of that node
    node_end: int = 0              # range only (global column ids)

    def c(self) -> ProblemParamsC:
        d = {"none": 0, "keep_rows": 1, "eliminate": 2}[self.dirichlet]
        ld = {"body_force": 0, "traction_xend": 1, "random": 2}[self.load]
        return ProblemParamsC(self.nx, self.ny, self.nz, self.lx, self.ly, self.lz, self.E,
                              self.nu, int(self.heterogeneous), d, ld, self.noise, self.seed,
                              int(self.x_slowest), self.node_begin, self.node_end)

    def total_nodes(self) -> int:
        kx = self.nx + (0 if self.dirichlet == "eliminate" else 1)
        return kx * (self.ny + 1) * (self.nz + 1)


@dataclass
class Problem:
    n: int
    nnodes: int
    ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray          # (nnzb, 3, 3)
    rhs: np.ndarray
    xyz: np.ndarray
    _csr: tuple | None = field(default=None, repr=False)

    @property
    def nbrows(self):
        return self.n // 3

    @property
    def nnzb(self):
        return int(self.ptr[-1])

    def nullspace(self):
        return rigid_body_modes(self.xyz)

    def csr(self):
        """Scalar CSR with every block entry kept (to_scalar, csr.hpp:327-353)."""
        if self._csr is None:
            nb = self.nbrows
            lens = np.diff(self.ptr)
            ptr = np.zeros(self.n + 1, np.int64)
            ptr[1:] = np.repeat(3 * lens, 3).cumsum()
            rows_blocks = np.repeat(np.arange(nb), lens)
            jpos = np.arange(self.nnzb) - self.ptr[rows_blocks]
            col = np.empty(9 * self.nnzb, np.int64)
            val = np.empty(9 * self.nnzb)
            # scalar row 3*bi + r lists the blocks of row bi in order, c = 0..2
            for r in range(3):
                base = ptr[3 * rows_blocks + r] + 3 * jpos
                for c in range(3):
                    col[base + c] = 3 * self.col + c
                    val[base + c] = self.val[:, r, c]
            self._csr = (self.n, ptr, col, val)
        return self._csr


def generate_hex(prm: ProblemParams = ProblemParams(), **kw) -> Problem:
    """Synthetic hex8 elasticity (elasticity.hpp:129-213, extended)."""
    if kw:
        prm = ProblemParams(**{**prm.__dict__, **kw})
    pc = prm.c()
    h = vp()
    check(lib.samg_generate_hex(C.byref(pc), C.byref(h)))
    try:
        n, nz, nn = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.samg_problem_info(h, C.byref(n), C.byref(nz), C.byref(nn)))
        ptr = np.zeros(nn.value + 1, np.int64)
        col = np.zeros(nz.value, np.int64)
        val = np.zeros(9 * nz.value)
        check(lib.samg_problem_get_bsr3(h, _p(ptr, i64p), _p(col, i64p), _p(val)))
        rhs = np.zeros(n.value)
        check(lib.samg_problem_get_rhs(h, _p(rhs)))
        xyz = np.zeros(3 * nn.value)
        check(lib.samg_problem_get_coords(h, _p(xyz)))
    finally:
        lib.samg_problem_destroy(h)
    return Problem(n.value, nn.value, ptr, col, val.reshape(-1, 3, 3), rhs, xyz)


class DeviceProblem:
    """A problem assembled on the GPU (samg_generate_hex_device): the matrix
    as a device Bsr3 view, rhs / nullspace / coordinates as device pointers."""

    def __init__(self, handle):
        self.h = handle
        n, nb, nz = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.samg_dproblem_info(handle, C.byref(n), C.byref(nb), C.byref(nz)))
        self.n, self.nbrows, self.nnzb = n.value, nb.value, nz.value
        a = vp()
        check(lib.samg_dproblem_matrix(handle, C.byref(a)))
        self._a = a
        r, b, x = vp(), vp(), vp()
        check(lib.samg_dproblem_vectors(handle, C.byref(r), C.byref(b), C.byref(x)))
        self.rhs_ptr, self.nullspace_ptr, self.xyz_ptr = r.value, b.value, x.value

    @property
    def A(self) -> "Bsr3":
        # a fresh borrowed view per access: storing one on the problem would
        # make a reference cycle (view -> owner -> view) and leave the device
        # memory to the cyclic collector instead of `del` / scope exit
        return Bsr3(self._a, owner=self)

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib.samg_dproblem_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def close(self):
        self.__del__()

    def download(self):
        """(rhs, nullspace (6 x 3n column-major blocks, flat), xyz) on the host"""
        rhs, B, xyz = np.zeros(self.n), np.zeros(6 * self.n), np.zeros(self.n)
        check(lib.samg_dproblem_download(self.h, _p(rhs), _p(B), _p(xyz)))
        return rhs, B, xyz


def generate_hex_device(prm: ProblemParams = ProblemParams(), device: int = 0, **kw) -> DeviceProblem:
    """generate_hex assembled directly in device memory (bitwise equal)."""
    if kw:
        prm = ProblemParams(**{**prm.__dict__, **kw})
    pc = prm.c()
    h = vp()
    check(lib.samg_generate_hex_device(C.byref(pc), device, C.byref(h)))
    return DeviceProblem(h)


def setup_device(A: "Bsr3", B_ptr: int, b_cols: int = 6, pipeline="ns_block",
                 prm: AmgParams = AmgParams()) -> Hierarchy:
    """samg_setup_device: hierarchy from a device matrix and a device (or
    host, by address) nullspace of 3*nrows x b_cols, column-major."""
    nr, _, _ = A.shape
    h = vp()
    pc = prm.c()
    check(lib.samg_setup_device(A.h, B_ptr, 3 * nr, b_cols, _pipeline(pipeline), C.byref(pc),
                                C.byref(h)))
    return Hierarchy(h)


def rigid_body_modes(xyz) -> np.ndarray:
    """rigid_body_modes (elasticity.hpp:38-52): column-major (3n x 6), flat."""
    xyz = _f64(xyz)
    nn = xyz.size // 3
    B = np.zeros(3 * nn * 6)
    check(lib.samg_rigid_body_modes(nn, _p(xyz), _p(B)))
    return B


# samg_apply_fn: int fn(void *ctx, const double *d_in, double *d_out, void *stream)
APPLY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)


def cg_solve_op(n: int, apply_A, apply_M, f_ptr: int, u_ptr: int, prm: CgParams = CgParams(),
                device: int = 0) -> dict:
    """cg_solve_op(n, apply_A, apply_M, f, u, prm) (cg.hpp:39-83) with caller
    operators on device vectors: apply_A(in_ptr, out_ptr, stream) -> None
    computes out = A in, apply_M (None = identity) out = M in; both must
    finish their work on return or enqueue it on `stream`.  f / u: device
    pointers of n doubles (u is overwritten)."""
    keep = []

    def wrap(fn):
        if fn is None:
            return None

        def cb(ctx, x, y, stream):
            try:
                fn(x, y, stream)
                return 0
            except SamgError as e:  # noqa: F821 (imported below)
                return e.code
            except Exception:
                return 1
        c = APPLY_FN(cb)
        keep.append(c)
        return c

    from ._lib import SamgError  # noqa: F401
    globals()["SamgError"] = SamgError
    rep = ReportC()
    cp = CgParamsC(prm.tol, prm.max_iterations)
    check(lib.samg_cg_solve_op(n, wrap(apply_A), wrap(apply_M), None, f_ptr, u_ptr, C.byref(cp),
                               device, C.byref(rep)))
    return _report(rep)
