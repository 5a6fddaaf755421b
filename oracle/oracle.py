"""ctypes front-end for the parity checkers (TEST INFRASTRUCTURE ONLY).

Two back-ends with the same Python surface:
  * ``Oracle`` -- the C restatement in samg_oracle.c (libsamg_oracle.so)
  * ``Ref``    -- the unmodified reference compiled by oracle/Makefile
                  (oracle/_ref/libsamg_ref.so)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libsamg_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsamg_ref.so")

SM_JACOBI, SM_SPAI0, SM_BLOCK_JACOBI, SM_ILU0 = 0, 1, 2, 3

i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


def build(ref: bool = True) -> None:
    """Compile the restatement (always) and the reference (when present)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _p(a, t=f64p):
    return a.ctypes.data_as(t) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


@dataclass
class Problem:
    n: int
    ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray
    rhs: np.ndarray
    coords: np.ndarray


@dataclass
class Params:
    eps_strong: float = 0.08
    omega: float = 2.0 / 3.0
    smoother: int = SM_SPAI0
    smoother_omega: float = 0.72
    coarse_enough: int = 3000
    stagnation_ratio: float = 0.8
    pipeline: int = 5  # samg::pipeline: 3 ns_hybrid1, 4 ns_hybrid2, 5 ns_block


class _problem_params(C.Structure):
    """samg_problem_params (include/samg_b200.h), for ref_gen_hex."""
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("lx", C.c_double), ("ly", C.c_double), ("lz", C.c_double),
                ("E", C.c_double), ("nu", C.c_double), ("heterogeneous", C.c_int),
                ("dirichlet", C.c_int), ("load", C.c_int), ("noise", C.c_double),
                ("seed", C.c_uint64), ("x_slowest", C.c_int), ("node_begin", C.c_int64),
                ("node_end", C.c_int64)]


_DIRICHLET = {"none": 0, "keep_rows": 1, "eliminate": 2}
_LOAD = {"body_force": 0, "traction_xend": 1, "random": 2}


@dataclass
class GenProblem:
    """A BASELINE-config problem from the repo's host generator as compiled
    into oracle/_ref (same fields as paper_2202_09056_b200.Problem)."""
    n: int
    nnodes: int
    ptr: np.ndarray
    col: np.ndarray
    val: np.ndarray          # (nnzb, 3, 3)
    rhs: np.ndarray
    xyz: np.ndarray
    ref: object = None

    @property
    def nbrows(self):
        return self.n // 3

    @property
    def nnzb(self):
        return int(self.ptr[-1])

    def nullspace(self):
        """rigid_body_modes (elasticity.hpp:38-52), the reference's own."""
        return self.ref.rigid_body_modes(self.xyz)

    def csr(self):
        """Scalar CSR with every block entry kept (to_scalar, csr.hpp:327-353)."""
        nb = self.nbrows
        lens = np.diff(self.ptr)
        ptr = np.zeros(self.n + 1, np.int64)
        ptr[1:] = np.repeat(3 * lens, 3).cumsum()
        rows_blocks = np.repeat(np.arange(nb), lens)
        jpos = np.arange(self.nnzb) - self.ptr[rows_blocks]
        col = np.empty(9 * self.nnzb, np.int64)
        val = np.empty(9 * self.nnzb)
        for r in range(3):
            base = ptr[3 * rows_blocks + r] + 3 * jpos
            for c in range(3):
                col[base + c] = 3 * self.col + c
                val[base + c] = self.val[:, r, c]
        return self.n, ptr, col, val


class _orc_mat(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("b", C.c_int),
                ("ptr", i64p), ("col", i64p), ("val", f64p)]


class _orc_params(C.Structure):
    _fields_ = [("eps_strong", C.c_double), ("omega", C.c_double),
                ("smoother", C.c_int), ("smoother_omega", C.c_double),
                ("pre_sweeps", C.c_int), ("post_sweeps", C.c_int),
                ("coarse_enough", C.c_int64), ("stagnation_ratio", C.c_double),
                ("pipeline", C.c_int)]


class _orc_report(C.Structure):
    _fields_ = [("iterations", C.c_int), ("relative_residual", C.c_double),
                ("converged", C.c_int)]


def _copy(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


class _Backend:
    lib: C.CDLL

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._err().decode())


class Oracle(_Backend):
    """The C restatement."""

    def __init__(self, path: str = ORACLE_SO):
        lib = C.CDLL(path)
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_generate_hex.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                         C.c_double, C.c_int, i64p, C.POINTER(i64p),
                                         C.POINTER(i64p), C.POINTER(f64p), C.POINTER(f64p),
                                         C.POINTER(f64p)]
        lib.orc_rigid_body_modes.argtypes = [C.c_int64, f64p, f64p]
        lib.orc_hex8_stiffness.argtypes = [C.c_double] * 5 + [f64p]
        lib.orc_free.argtypes = [vp]
        lib.orc_setup_ns_block.argtypes = [C.c_int64, i64p, i64p, f64p, f64p, C.c_int64,
                                           C.POINTER(_orc_params), C.POINTER(vp)]
        lib.orc_hier_free.argtypes = [vp]
        lib.orc_hier_nlevels.argtypes = [vp]
        lib.orc_hier_matrix.argtypes = [vp, C.c_int, C.c_int, C.POINTER(_orc_mat)]
        lib.orc_hier_aggregates.argtypes = [vp, C.c_int, i64p, C.POINTER(i64p), i64p]
        lib.orc_hier_smoother.argtypes = [vp, C.c_int, i64p, C.POINTER(f64p)]
        lib.orc_hier_coarse_dim.argtypes = [vp]
        lib.orc_hier_coarse_dim.restype = C.c_int64
        lib.orc_hier_memory_footprint.argtypes = [vp]
        lib.orc_hier_memory_footprint.restype = C.c_uint64
        lib.orc_vcycle.argtypes = [vp, f64p, f64p]
        lib.orc_cg_solve.argtypes = [vp, f64p, f64p, C.c_double, C.c_int,
                                     C.POINTER(_orc_report)]
        lib.orc_spmv_bsr3.argtypes = [C.c_int64, C.c_int64, i64p, i64p, f64p, C.c_double,
                                      f64p, C.c_double, f64p]
        lib.orc_galerkin_bsr3.argtypes = [C.POINTER(_orc_mat)] * 4
        lib.orc_aggregate_scalar.argtypes = [C.c_int64, i64p, i64p, f64p, C.c_double,
                                             C.c_int, i64p, i64p]
        self.lib = lib
        self._err = lib.orc_last_error

    def generate_hex(self, nx, ny, nz, E=1.0, nu=0.3, clamp_x0=True) -> Problem:
        n = C.c_int64()
        ptr, col = i64p(), i64p()
        val, rhs, xyz = f64p(), f64p(), f64p()
        self._check(self.lib.orc_generate_hex(nx, ny, nz, E, nu, int(clamp_x0), C.byref(n),
                                              C.byref(ptr), C.byref(col), C.byref(val),
                                              C.byref(rhs), C.byref(xyz)))
        N = n.value
        nnz = int(np.ctypeslib.as_array(ptr, shape=(N + 1,))[N])
        nn = (nx + 1) * (ny + 1) * (nz + 1)
        out = Problem(N, _copy(ptr, N + 1, np.int64), _copy(col, nnz, np.int64),
                      _copy(val, nnz, np.float64), _copy(rhs, N, np.float64),
                      _copy(xyz, 3 * nn, np.float64))
        for p in (ptr, col, val, rhs, xyz):
            self.lib.orc_free(C.cast(p, vp))
        return out

    def hex8_stiffness(self, hx, hy, hz, E, nu):
        Ke = np.zeros(576)
        self.lib.orc_hex8_stiffness(hx, hy, hz, E, nu, _p(Ke))
        return Ke.reshape(24, 24)

    def rigid_body_modes(self, coords):
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        nn = coords.size // 3
        B = np.zeros(3 * nn * 6)
        self.lib.orc_rigid_body_modes(nn, _p(coords), _p(B))
        return B

    def setup(self, n, ptr, col, val, B, params: Params = Params()):
        pr = _orc_params(params.eps_strong, params.omega, params.smoother,
                         params.smoother_omega, 1, 1, params.coarse_enough,
                         params.stagnation_ratio, params.pipeline)
        ptr = np.ascontiguousarray(ptr, np.int64)
        col = np.ascontiguousarray(col, np.int64)
        val = np.ascontiguousarray(val, np.float64)
        Bp, bc = (None, 0) if B is None else (_p(B := np.ascontiguousarray(B, np.float64)),
                                               B.size // n)
        h = vp()
        self._check(self.lib.orc_setup_ns_block(n, _p(ptr, i64p), _p(col, i64p), _p(val),
                                                Bp, bc, C.byref(pr), C.byref(h)))
        return OracleHier(self, h, n)

    def spmv_bsr3(self, nrows, ncols, ptr, col, val, x, alpha=1.0, beta=0.0, y=None):
        y = np.zeros(3 * nrows) if y is None else np.array(y, dtype=np.float64)
        ptr = np.ascontiguousarray(ptr, np.int64)
        col = np.ascontiguousarray(col, np.int64)
        val = np.ascontiguousarray(val, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        self._check(self.lib.orc_spmv_bsr3(nrows, ncols, _p(ptr, i64p), _p(col, i64p),
                                           _p(val), alpha, _p(x), beta, _p(y)))
        return y

    def galerkin_bsr3(self, R, A, P):
        """R, A, P: (nrows, ncols, ptr, col, val) tuples in 3x3 blocks."""
        keep = []

        def mk(m):
            nr, nc, ptr, col, val = m
            ptr = np.ascontiguousarray(ptr, np.int64)
            col = np.ascontiguousarray(col, np.int64)
            val = np.ascontiguousarray(val, np.float64)
            keep.extend([ptr, col, val])
            return _orc_mat(nr, nc, 3, _p(ptr, i64p), _p(col, i64p), _p(val))

        r, a, p = mk(R), mk(A), mk(P)
        c = _orc_mat()
        self._check(self.lib.orc_galerkin_bsr3(C.byref(r), C.byref(a), C.byref(p), C.byref(c)))
        nnz = int(np.ctypeslib.as_array(c.ptr, shape=(c.nrows + 1,))[c.nrows])
        out = (c.nrows, c.ncols, _copy(c.ptr, c.nrows + 1, np.int64),
               _copy(c.col, nnz, np.int64), _copy(c.val, nnz * 9, np.float64).reshape(-1, 3, 3))
        for q in (c.ptr, c.col, c.val):
            self.lib.orc_free(C.cast(q, vp))
        return out

    def aggregate_scalar(self, n, ptr, col, val, eps=0.08, pbs=1):
        ptr = np.ascontiguousarray(ptr, np.int64)
        col = np.ascontiguousarray(col, np.int64)
        val = np.ascontiguousarray(val, np.float64)
        idv = np.zeros(n // pbs, dtype=np.int64)
        cnt = C.c_int64()
        self._check(self.lib.orc_aggregate_scalar(n, _p(ptr, i64p), _p(col, i64p), _p(val),
                                                  eps, pbs, _p(idv, i64p), C.byref(cnt)))
        return idv, cnt.value


class OracleHier:
    def __init__(self, be: Oracle, h, n):
        self.be, self.h, self.n = be, h, n

    def __del__(self):
        try:
            self.be.lib.orc_hier_free(self.h)
        except Exception:
            pass

    @property
    def nlevels(self):
        return self.be.lib.orc_hier_nlevels(self.h)

    @property
    def coarse_dim(self):
        return self.be.lib.orc_hier_coarse_dim(self.h)

    @property
    def memory_footprint(self):
        return self.be.lib.orc_hier_memory_footprint(self.h)

    def level(self, l, which=0):
        m = _orc_mat()
        if self.be.lib.orc_hier_matrix(self.h, l, which, C.byref(m)) != 0:
            raise IndexError((l, which))
        nnz = int(np.ctypeslib.as_array(m.ptr, shape=(m.nrows + 1,))[m.nrows])
        return (m.nrows, m.ncols, _copy(m.ptr, m.nrows + 1, np.int64),
                _copy(m.col, nnz, np.int64), _copy(m.val, nnz * 9, np.float64).reshape(-1, 3, 3))

    def aggregates(self, l):
        nn, cnt, idp = C.c_int64(), C.c_int64(), i64p()
        if self.be.lib.orc_hier_aggregates(self.h, l, C.byref(nn), C.byref(idp), C.byref(cnt)):
            raise IndexError(l)
        return _copy(idp, nn.value, np.int64), cnt.value

    def smoother(self, l):
        ln, dp = C.c_int64(), f64p()
        if self.be.lib.orc_hier_smoother(self.h, l, C.byref(ln), C.byref(dp)):
            raise IndexError(l)
        return _copy(dp, ln.value, np.float64)

    def vcycle(self, f):
        f = np.ascontiguousarray(f, np.float64)
        u = np.zeros_like(f)
        self.be._check(self.be.lib.orc_vcycle(self.h, _p(f), _p(u)))
        return u

    def cg_solve(self, f, tol=1e-8, max_iterations=1000):
        f = np.ascontiguousarray(f, np.float64)
        u = np.zeros_like(f)
        rep = _orc_report()
        self.be._check(self.be.lib.orc_cg_solve(self.h, _p(f), _p(u), tol, max_iterations,
                                                C.byref(rep)))
        return u, dict(iterations=rep.iterations, relative_residual=rep.relative_residual,
                       converged=bool(rep.converged))


class Ref(_Backend):
    """The unmodified reference, via oracle/ref_driver.cpp."""

    def __init__(self, path: str = REF_SO):
        lib = C.CDLL(path)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_free_buf.argtypes = [vp]
        lib.ref_generate_hex.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                         C.c_double, C.c_int, i64p, C.POINTER(i64p),
                                         C.POINTER(i64p), C.POINTER(f64p), C.POINTER(f64p),
                                         C.POINTER(f64p)]
        lib.ref_rigid_body_modes.argtypes = [C.c_int64, f64p, f64p]
        lib.ref_gen_hex.argtypes = [C.POINTER(_problem_params), i64p, i64p, C.POINTER(i64p),
                                    C.POINTER(i64p), C.POINTER(f64p), C.POINTER(f64p),
                                    C.POINTER(f64p)]
        lib.ref_force_isa.argtypes = [C.c_int]
        lib.ref_setup.argtypes = [C.c_int64, i64p, i64p, f64p, f64p, C.c_int64, C.c_double,
                                  C.c_double, C.c_int, C.c_double, C.c_int64, C.c_double,
                                  C.c_int, C.POINTER(vp)]
        lib.ref_setup_bsr3.argtypes = lib.ref_setup.argtypes
        lib.ref_destroy.argtypes = [vp]
        lib.ref_nlevels.argtypes = [vp]
        lib.ref_setup_seconds.argtypes = [vp]
        lib.ref_setup_seconds.restype = C.c_double
        lib.ref_coarse_dim.argtypes = [vp]
        lib.ref_coarse_dim.restype = C.c_int64
        lib.ref_memory_footprint.argtypes = [vp]
        lib.ref_memory_footprint.restype = C.c_uint64
        lib.ref_level_matrix.argtypes = [vp, C.c_int, C.c_int, i64p, i64p, C.POINTER(i64p),
                                         C.POINTER(i64p), C.POINTER(f64p)]
        lib.ref_aggregates.argtypes = [vp, C.c_int, i64p, C.POINTER(i64p), i64p]
        lib.ref_ilu_factors.argtypes = [vp, C.c_int, i64p, i64p, C.POINTER(f64p), C.POINTER(f64p)]
        lib.ref_vcycle.argtypes = [vp, f64p, f64p]
        lib.ref_cg_solve.argtypes = [vp, f64p, f64p, C.c_double, C.c_int, C.POINTER(C.c_int),
                                     f64p, C.POINTER(C.c_int), f64p]
        lib.ref_spmv.argtypes = [vp, C.c_int, C.c_double, f64p, C.c_double, f64p]
        lib.ref_spmv_bsr3.argtypes = [C.c_int64, C.c_int64, i64p, i64p, f64p, C.c_double,
                                      f64p, C.c_double, f64p]
        lib.ref_bsr3_create.argtypes = [C.c_int64, C.c_int64, i64p, i64p, f64p]
        lib.ref_bsr3_create.restype = vp
        lib.ref_bsr3_destroy.argtypes = [vp]
        lib.ref_bsr3_spmv.argtypes = [vp, C.c_double, f64p, C.c_double, f64p]
        self.lib = lib
        self._err = lib.ref_last_error

    def bsr3(self, nrows, ncols, ptr, col, val):
        """A reference csr<static_block<3>> (rows [0, nrows) of the arrays;
        ptr may be a slice of a larger matrix's ptr)."""
        return RefBsr3(self, nrows, ncols, ptr, col, val)

    def generate_hex(self, nx, ny, nz, E=1.0, nu=0.3, clamp_x0=True) -> Problem:
        n = C.c_int64()
        ptr, col = i64p(), i64p()
        val, rhs, xyz = f64p(), f64p(), f64p()
        self._check(self.lib.ref_generate_hex(nx, ny, nz, E, nu, int(clamp_x0), C.byref(n),
                                              C.byref(ptr), C.byref(col), C.byref(val),
                                              C.byref(rhs), C.byref(xyz)))
        N = n.value
        nnz = int(np.ctypeslib.as_array(ptr, shape=(N + 1,))[N])
        nn = (nx + 1) * (ny + 1) * (nz + 1)
        out = Problem(N, _copy(ptr, N + 1, np.int64), _copy(col, nnz, np.int64),
                      _copy(val, nnz, np.float64), _copy(rhs, N, np.float64),
                      _copy(xyz, 3 * nn, np.float64))
        for p in (ptr, col, val, rhs, xyz):
            self.lib.ref_free_buf(C.cast(p, vp))
        return out

    def rigid_body_modes(self, coords):
        coords = np.ascontiguousarray(coords, dtype=np.float64)
        nn = coords.size // 3
        B = np.zeros(3 * nn * 6)
        self._check(self.lib.ref_rigid_body_modes(nn, _p(coords), _p(B)))
        return B

    def gen_hex(self, nx=19, ny=19, nz=19, lx=1.0, ly=1.0, lz=1.0, E=1.0, nu=0.3,
                heterogeneous=False, dirichlet="eliminate", load="body_force", noise=0.0,
                seed=12345, x_slowest=False, node_begin=0, node_end=0) -> GenProblem:
        """The repo's BASELINE-config generator (generator.cpp, host-only,
        linked into oracle/_ref); keywords as paper_2202_09056_b200.ProblemParams."""
        pc = _problem_params(nx, ny, nz, lx, ly, lz, E, nu, int(heterogeneous),
                             _DIRICHLET[dirichlet], _LOAD[load], noise, seed, int(x_slowest),
                             node_begin, node_end)
        n, nn = C.c_int64(), C.c_int64()
        ptr, col = i64p(), i64p()
        val, rhs, xyz = f64p(), f64p(), f64p()
        self._check(self.lib.ref_gen_hex(C.byref(pc), C.byref(n), C.byref(nn), C.byref(ptr),
                                         C.byref(col), C.byref(val), C.byref(rhs), C.byref(xyz)))
        N, NN = n.value, nn.value
        nnzb = int(np.ctypeslib.as_array(ptr, shape=(NN + 1,))[NN])
        out = GenProblem(N, NN, _copy(ptr, NN + 1, np.int64), _copy(col, nnzb, np.int64),
                         _copy(val, 9 * nnzb, np.float64).reshape(-1, 3, 3),
                         _copy(rhs, N, np.float64), _copy(xyz, 3 * NN, np.float64), self)
        for p in (ptr, col, val, rhs, xyz):
            self.lib.ref_free_buf(C.cast(p, vp))
        return out

    def force_isa(self, avx2: bool) -> bool:
        """kernels::force_isa (kernels.hpp:25-28) for the CG dot/axpby;
        returns whether AVX2 is active afterwards."""
        return bool(self.lib.ref_force_isa(int(avx2)))

    def setup(self, n, ptr, col, val, B, params: Params = Params()):
        ptr = np.ascontiguousarray(ptr, np.int64)
        col = np.ascontiguousarray(col, np.int64)
        val = np.ascontiguousarray(val, np.float64)
        Bp, bc = (None, 0) if B is None else (_p(B := np.ascontiguousarray(B, np.float64)),
                                               B.size // n)
        h = vp()
        self._check(self.lib.ref_setup(n, _p(ptr, i64p), _p(col, i64p), _p(val), Bp,
                                       bc, params.eps_strong, params.omega,
                                       params.smoother, params.smoother_omega,
                                       params.coarse_enough, params.stagnation_ratio,
                                       params.pipeline, C.byref(h)))
        return RefHier(self, h, n)

    def setup_bsr3(self, nbrows, ptr, col, val, B, params: Params = Params()):
        """setup() of to_scalar(BSR3 input) (csr.hpp:327-353), formed inside
        the reference driver."""
        ptr = np.ascontiguousarray(ptr, np.int64)
        col = np.ascontiguousarray(col, np.int64)
        val = np.ascontiguousarray(val, np.float64)
        n = 3 * nbrows
        Bp, bc = (None, 0) if B is None else (_p(B := np.ascontiguousarray(B, np.float64)),
                                               B.size // n)
        h = vp()
        self._check(self.lib.ref_setup_bsr3(nbrows, _p(ptr, i64p), _p(col, i64p), _p(val), Bp,
                                            bc, params.eps_strong, params.omega,
                                            params.smoother, params.smoother_omega,
                                            params.coarse_enough, params.stagnation_ratio,
                                            params.pipeline, C.byref(h)))
        return RefHier(self, h, n)

    def spmv_bsr3(self, nrows, ncols, ptr, col, val, x, alpha=1.0, beta=0.0, y=None):
        y = np.zeros(3 * nrows) if y is None else np.array(y, dtype=np.float64)
        ptr = np.ascontiguousarray(ptr, np.int64)
        col = np.ascontiguousarray(col, np.int64)
        val = np.ascontiguousarray(val, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        self._check(self.lib.ref_spmv_bsr3(nrows, ncols, _p(ptr, i64p), _p(col, i64p),
                                           _p(val), alpha, _p(x), beta, _p(y)))
        return y


class RefHier:
    def __init__(self, be: Ref, h, n):
        self.be, self.h, self.n = be, h, n

    def __del__(self):
        try:
            self.be.lib.ref_destroy(self.h)
        except Exception:
            pass

    @property
    def nlevels(self):
        return self.be.lib.ref_nlevels(self.h)

    @property
    def coarse_dim(self):
        return self.be.lib.ref_coarse_dim(self.h)

    @property
    def memory_footprint(self):
        return self.be.lib.ref_memory_footprint(self.h)

    @property
    def setup_seconds(self):
        return self.be.lib.ref_setup_seconds(self.h)

    def level(self, l, which=0):
        nr, nc = C.c_int64(), C.c_int64()
        ptr, col, val = i64p(), i64p(), f64p()
        if self.be.lib.ref_level_matrix(self.h, l, which, C.byref(nr), C.byref(nc),
                                        C.byref(ptr), C.byref(col), C.byref(val)):
            raise IndexError((l, which))
        nrows = nr.value
        nnz = int(np.ctypeslib.as_array(ptr, shape=(nrows + 1,))[nrows])
        return (nrows, nc.value, _copy(ptr, nrows + 1, np.int64), _copy(col, nnz, np.int64),
                _copy(val, nnz * 9, np.float64).reshape(-1, 3, 3))

    def ilu(self, l, scalar=False):
        """[factors (9*nnzb) | inverted pivots (9*nrows)] of level l's
        ilu0<block3>; scalar: ilu0<double>'s factors re-blocked and its 3
        pivots per block row"""
        nz, nr = C.c_int64(), C.c_int64()
        lp, ip = f64p(), f64p()
        if self.be.lib.ref_ilu_factors(self.h, l, C.byref(nz), C.byref(nr), C.byref(lp), C.byref(ip)):
            raise KeyError(l)
        return np.concatenate([np.ctypeslib.as_array(lp, (9 * nz.value,)).copy(),
                               np.ctypeslib.as_array(ip, ((3 if scalar else 9) * nr.value,)).copy()])

    def aggregates(self, l):
        nn, cnt, idp = C.c_int64(), C.c_int64(), i64p()
        if self.be.lib.ref_aggregates(self.h, l, C.byref(nn), C.byref(idp), C.byref(cnt)):
            raise IndexError(l)
        return _copy(idp, nn.value, np.int64), cnt.value

    def vcycle(self, f):
        f = np.ascontiguousarray(f, np.float64)
        u = np.zeros_like(f)
        self.be._check(self.be.lib.ref_vcycle(self.h, _p(f), _p(u)))
        return u

    def cg_solve(self, f, tol=1e-8, max_iterations=1000):
        f = np.ascontiguousarray(f, np.float64)
        u = np.zeros_like(f)
        it, conv = C.c_int(), C.c_int()
        rr, ss = C.c_double(), C.c_double()
        self.be._check(self.be.lib.ref_cg_solve(self.h, _p(f), _p(u), tol, max_iterations,
                                                C.byref(it), C.byref(rr), C.byref(conv),
                                                C.byref(ss)))
        return u, dict(iterations=it.value, relative_residual=rr.value,
                       converged=bool(conv.value), solve_seconds=ss.value)

    def spmv(self, x, level=0, alpha=1.0, beta=0.0, y=None):
        x = np.ascontiguousarray(x, np.float64)
        nr = self.level(level)[0]
        y = np.zeros(3 * nr) if y is None else np.array(y, dtype=np.float64)
        self.be._check(self.be.lib.ref_spmv(self.h, level, alpha, _p(x), beta, _p(y)))
        return y


class RefBsr3:
    """Handle to a reference csr<block3>; spmv is samg::spmv (csr.hpp:129-160)."""

    def __init__(self, be: Ref, nrows, ncols, ptr, col, val):
        self.be = be
        self.nrows, self.ncols = nrows, ncols
        ptr = np.ascontiguousarray(ptr, np.int64)
        col = np.ascontiguousarray(col, np.int64)
        val = np.ascontiguousarray(val, np.float64)
        self.h = be.lib.ref_bsr3_create(nrows, ncols, _p(ptr, i64p), _p(col, i64p), _p(val))

    def __del__(self):
        try:
            self.be.lib.ref_bsr3_destroy(self.h)
        except Exception:
            pass

    def spmv(self, x, y, alpha=1.0, beta=0.0):
        self.be._check(self.be.lib.ref_bsr3_spmv(self.h, alpha, _p(x), beta, _p(y)))
        return y
