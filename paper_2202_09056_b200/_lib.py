"""Loader and ctypes prototypes for libsamg_b200.so (include/samg_b200.h)."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsamg_b200.so")

i64 = C.c_int64
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


class SamgError(RuntimeError):
    """samg::error (common.hpp:12); ``code`` is the C-ABI status."""
    code = 1

    def __init__(self, msg: str, code: int | None = None):
        super().__init__(msg)
        if code is not None:
            self.code = code


class DimensionMismatch(SamgError): code = 2
class NotDivisible(SamgError): code = 3
class SingularBlock(SamgError): code = 4
class MissingDiagonal(SamgError): code = 5
class ZeroDiagonal(SamgError): code = 6
class NonSquare(SamgError): code = 7
class BadNullspaceShape(SamgError): code = 8
class BreakdownNonSpd(SamgError): code = 9
class InvalidMaterial(SamgError): code = 10
class ShapeMismatch(SamgError): code = 11
class CudaError(SamgError): code = 100
class NcclError(SamgError): code = 101
class OutOfMemory(SamgError): code = 102
class NoDevice(SamgError): code = 103
class Unsupported(SamgError): code = 104
class InvalidArgument(SamgError): code = 105


_BY_CODE = {cls.code: cls for cls in (
    SamgError, DimensionMismatch, NotDivisible, SingularBlock, MissingDiagonal, ZeroDiagonal,
    NonSquare, BadNullspaceShape, BreakdownNonSpd, InvalidMaterial, ShapeMismatch, CudaError,
    NcclError, OutOfMemory, NoDevice, Unsupported, InvalidArgument)}


class AmgParamsC(C.Structure):
    _fields_ = [("eps_strong", C.c_double), ("omega", C.c_double),
                ("point_block_size", C.c_int), ("smoother", C.c_int),
                ("smoother_omega", C.c_double), ("pre_sweeps", C.c_int),
                ("post_sweeps", C.c_int), ("coarse_enough", C.c_int64),
                ("stagnation_ratio", C.c_double), ("verify_galerkin", C.c_int),
                ("device", C.c_int), ("vcycle_precision", C.c_int),
                ("ilu_sweep_order", C.c_int)]


class CgParamsC(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iterations", C.c_int)]


class ReportC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("relative_residual", C.c_double),
                ("setup_seconds", C.c_double), ("solve_seconds", C.c_double),
                ("preconditioner_bytes", C.c_uint64), ("variant", C.c_int),
                ("converged", C.c_int)]


class ProblemParamsC(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("lx", C.c_double), ("ly", C.c_double), ("lz", C.c_double),
                ("E", C.c_double), ("nu", C.c_double), ("heterogeneous", C.c_int),
                ("dirichlet", C.c_int), ("load", C.c_int), ("noise", C.c_double),
                ("seed", C.c_uint64), ("x_slowest", C.c_int),
                ("node_begin", C.c_int64), ("node_end", C.c_int64)]


# (name, argtypes) of every exported function; restype int unless noted
PROTOTYPES = {
    "samg_default_amg_params": ([C.POINTER(AmgParamsC)], None),
    "samg_default_cg_params": ([C.POINTER(CgParamsC)], None),
    "samg_last_error": ([], C.c_char_p),
    "samg_status_name": ([C.c_int], C.c_char_p),
    "samg_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "samg_setup": ([i64, i64p, i64p, f64p, f64p, i64, i64, C.c_int, C.POINTER(AmgParamsC),
                    C.POINTER(vp)], C.c_int),
    "samg_setup_bsr3": ([i64, i64p, i64p, f64p, f64p, i64, i64, C.c_int,
                         C.POINTER(AmgParamsC), C.POINTER(vp)], C.c_int),
    "samg_destroy": ([vp], C.c_int),
    "samg_cg_solve": ([vp, f64p, f64p, C.POINTER(CgParamsC), C.POINTER(ReportC)], C.c_int),
    "samg_cg_solve_device": ([vp, vp, vp, C.POINTER(CgParamsC), C.POINTER(ReportC)], C.c_int),
    "samg_vcycle": ([vp, f64p, f64p], C.c_int),
    "samg_vcycle_device": ([vp, vp, vp], C.c_int),
    "samg_cg_solve_op": ([i64, vp, vp, vp, vp, vp, C.POINTER(CgParamsC), C.c_int, C.POINTER(ReportC)],
                         C.c_int),
    "samg_memory_footprint": ([vp, C.POINTER(C.c_uint64)], C.c_int),
    "samg_finest_dim": ([vp, i64p], C.c_int),
    "samg_num_levels": ([vp, C.POINTER(C.c_int)], C.c_int),
    "samg_coarse_dim": ([vp, i64p], C.c_int),
    "samg_coarse_solver": ([vp, C.POINTER(C.c_int)], C.c_int),
    "samg_setup_seconds": ([vp, f64p], C.c_int),
    "samg_level_info": ([vp, C.c_int, C.c_int, i64p, i64p, i64p], C.c_int),
    "samg_get_level": ([vp, C.c_int, C.c_int, i64p, i64p, f64p], C.c_int),
    "samg_level_matrix": ([vp, C.c_int, C.c_int, C.POINTER(vp)], C.c_int),
    "samg_aggregates_info": ([vp, C.c_int, i64p, i64p], C.c_int),
    "samg_get_aggregates": ([vp, C.c_int, i64p], C.c_int),
    "samg_smoother_info": ([vp, C.c_int, i64p], C.c_int),
    "samg_get_smoother": ([vp, C.c_int, f64p], C.c_int),
    "samg_bsr3_create": ([i64, i64, i64p, i64p, f64p, C.c_int, C.POINTER(vp)], C.c_int),
    "samg_bsr3_destroy": ([vp], C.c_int),
    "samg_bsr3_info": ([vp, i64p, i64p, i64p], C.c_int),
    "samg_bsr3_download": ([vp, i64p, i64p, f64p], C.c_int),
    "samg_bsr3_spmv_device": ([vp, C.c_double, vp, C.c_double, vp, vp], C.c_int),
    "samg_bsr3_spmv": ([vp, C.c_double, f64p, C.c_double, f64p], C.c_int),
    "samg_bsr3_spmv_batch": ([vp, C.c_double, vp, C.c_double, vp, i64], C.c_int),
    "samg_bsr3_galerkin": ([vp, vp, vp, C.POINTER(vp)], C.c_int),
    "samg_bsr3_dense_inverse": ([vp, f64p], C.c_int),
    "samg_bsr3_spmv_bytes": ([vp, C.c_int, C.POINTER(C.c_uint64)], C.c_int),
    "samg_default_problem_params": ([C.POINTER(ProblemParamsC)], None),
    "samg_generate_hex": ([C.POINTER(ProblemParamsC), C.POINTER(vp)], C.c_int),
    "samg_problem_destroy": ([vp], C.c_int),
    "samg_problem_info": ([vp, i64p, i64p, i64p], C.c_int),
    "samg_problem_get_bsr3": ([vp, i64p, i64p, f64p], C.c_int),
    "samg_problem_get_csr": ([vp, i64p, i64p, f64p], C.c_int),
    "samg_problem_get_rhs": ([vp, f64p], C.c_int),
    "samg_problem_get_coords": ([vp, f64p], C.c_int),
    "samg_rigid_body_modes": ([i64, f64p, f64p], C.c_int),
    "samg_problem_bsr3_view": ([vp, C.POINTER(i64p), C.POINTER(i64p), C.POINTER(f64p)], C.c_int),
    "samg_dist_create": ([i64, i64, i64p, i64p, f64p, C.c_int, i64p, C.c_int, C.POINTER(vp)],
                         C.c_int),
    "samg_dist_destroy": ([vp], C.c_int),
    "samg_dist_info": ([vp, i64p, i64p, i64p, i64p, C.POINTER(C.c_int), C.POINTER(C.c_int)],
                       C.c_int),
    "samg_dist_recv_plan": ([vp, C.POINTER(C.c_int), i64p, i64p], C.c_int),
    "samg_dist_ghosts": ([vp, i64p], C.c_int),
    "samg_dist_set_send": ([vp, C.c_int, C.POINTER(C.c_int), i64p, i64p], C.c_int),
    "samg_dist_send_plan": ([vp, C.POINTER(C.c_int), i64p, i64p, i64p], C.c_int),
    "samg_dist_derive_send": ([vp], C.c_int),
    "samg_dist_local_matrix": ([vp, i64p, i64p, f64p], C.c_int),
    "samg_dist_to_device": ([vp, C.c_int, C.c_int], C.c_int),
    "samg_dist_pack": ([vp, vp, vp, vp], C.c_int),
    "samg_dist_spmv": ([vp, C.c_int, C.c_double, vp, C.c_double, vp, vp], C.c_int),
    "samg_generate_hex_device": ([C.POINTER(ProblemParamsC), C.c_int, C.POINTER(vp)], C.c_int),
    "samg_dproblem_destroy": ([vp], C.c_int),
    "samg_dproblem_info": ([vp, i64p, i64p, i64p], C.c_int),
    "samg_dproblem_matrix": ([vp, C.POINTER(vp)], C.c_int),
    "samg_dproblem_vectors": ([vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)], C.c_int),
    "samg_dproblem_download": ([vp, f64p, f64p, f64p], C.c_int),
    "samg_setup_device": ([vp, vp, i64, i64, C.c_int, C.POINTER(AmgParamsC), C.POINTER(vp)], C.c_int),
    "samg_nccl_unique_id": ([C.POINTER(C.c_ubyte)], C.c_int),
    "samg_dsetup": ([C.POINTER(C.c_ubyte), C.c_int, C.c_int, i64, i64p, i64p, f64p, f64p, i64,
                     i64, i64p, i64, C.c_int, C.POINTER(AmgParamsC), C.POINTER(vp)], C.c_int),
    "samg_ddestroy": ([vp], C.c_int),
    "samg_dinfo": ([vp, i64p, i64p, C.POINTER(C.c_int), C.POINTER(C.c_int), f64p], C.c_int),
    "samg_dheld_rows": ([vp, i64p], C.c_int),
    "samg_dsetup_local": ([C.POINTER(C.c_ubyte), C.c_int, C.c_int, i64p, i64p, i64p, f64p, f64p,
                           i64, i64, C.c_int, C.POINTER(AmgParamsC), C.POINTER(vp)], C.c_int),
    "samg_dsetup_device": ([C.POINTER(C.c_ubyte), C.c_int, C.c_int, i64p, vp, vp, i64, i64,
                            C.c_int, C.POINTER(AmgParamsC), C.POINTER(vp)], C.c_int),
    "samg_dlevel_info": ([vp, C.c_int, C.c_int, i64p, i64p, i64p], C.c_int),
    "samg_dget_level": ([vp, C.c_int, C.c_int, i64p, i64p, f64p], C.c_int),
    "samg_dcg_solve_device": ([vp, vp, vp, C.POINTER(CgParamsC), C.POINTER(ReportC)], C.c_int),
    "samg_dcg_solve": ([vp, f64p, f64p, C.POINTER(CgParamsC), C.POINTER(ReportC)], C.c_int),
}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (args, res) in PROTOTYPES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc != 0:
        msg = lib.samg_last_error().decode(errors="replace")
        raise _BY_CODE.get(rc, SamgError)(msg, rc)
