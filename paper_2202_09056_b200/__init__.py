"""B200-native SA-AMG "NS Block" solver (arXiv 2202.09056 hot path).

Python mirror of the reference's C++ interface (proj/include/samg):
``setup`` (hierarchy.hpp:263), ``Hierarchy.vcycle`` (hierarchy.hpp:408),
``Hierarchy.cg_solve`` (cg.hpp:87), ``Hierarchy.memory_footprint``
(hierarchy.hpp:443), with the reference's typed errors as exception
subclasses.  Every call goes through the C-ABI of libsamg_b200.so
(include/samg_b200.h); there is no CPU fallback -- importing without the
built library raises, and compute calls without a GPU raise ``NoDevice``.
"""
from ._lib import (  # noqa: F401
    LIB_PATH,
    BadNullspaceShape,
    BreakdownNonSpd,
    CudaError,
    DimensionMismatch,
    InvalidArgument,
    InvalidMaterial,
    MissingDiagonal,
    NoDevice,
    NonSquare,
    NotDivisible,
    SamgError,
    SingularBlock,
    Unsupported,
    ZeroDiagonal,
    lib,
)
from .api import (  # noqa: F401
    PIPELINES,
    SMOOTHERS,
    AmgParams,
    Bsr3,
    CgParams,
    DeviceProblem,
    Hierarchy,
    Problem,
    ProblemParams,
    cg_solve_op,
    device_count,
    generate_hex,
    generate_hex_device,
    rigid_body_modes,
    setup,
    setup_bsr3,
    setup_device,
)

__all__ = [
    "setup", "setup_bsr3", "Hierarchy", "AmgParams", "CgParams", "Bsr3", "Problem",
    "ProblemParams", "generate_hex", "rigid_body_modes", "device_count", "SamgError",
    "DeviceProblem", "generate_hex_device", "setup_device", "cg_solve_op",
]
