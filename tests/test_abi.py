"""CPU-side checks of the C-ABI library (no GPU compute).

* libsamg_b200.so loads and exports every function include/samg_b200.h
  declares;
* host-side validation raises the reference's typed errors before any
  device work (hierarchy.hpp:267-282), and compute calls without a device
  fail loudly with NoDevice (no CPU fallback);
* the host problem generator equals the reference generator
  (elasticity.hpp:129-213) to rounding, in both Dirichlet forms.
"""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2202_09056_b200 as pb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "samg_b200.h")


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"SAMG_API\s+[\w\s\*]*?\b(samg_\w+)\s*\(", src)))


def test_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 40
    out = subprocess.run(["nm", "-D", "--defined-only", pb.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        assert hasattr(pb.lib, n)


def test_library_has_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", pb.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_validation_before_device():
    p = pb.generate_hex(nx=2, ny=2, nz=2, dirichlet="eliminate")
    A, B = p.csr(), p.nullspace()
    with pytest.raises(pb.BadNullspaceShape):
        pb.setup(A, None)
    with pytest.raises(pb.BadNullspaceShape):
        pb.setup(A, np.zeros((A[0] - 3, 6)))
    n, ptr, col, val = A
    with pytest.raises(pb.NotDivisible):
        pb.setup((n - 1, ptr[:-1], col[:ptr[n - 1]], val[:ptr[n - 1]]), np.zeros((n - 1, 6)))
    with pytest.raises(pb.Unsupported):  # scalar pipelines: damped Jacobi only
        pb.setup(A, B, "ns_scalar", pb.AmgParams(smoother="spai0"))
    with pytest.raises(pb.InvalidArgument):
        pb.setup(A, B, "ns_block", pb.AmgParams(smoother=7))
    with pytest.raises(pb.NotDivisible):
        pb.setup(A, np.zeros((n, 4)))
    prm = pb.AmgParams()
    prm.vcycle_precision = "mixed"
    c = prm.c()
    c.vcycle_precision = 5
    with pytest.raises(pb.InvalidArgument):
        pb.setup(A, B, "ns_block", type("P", (), {"c": lambda self: c})())
    c2 = pb.AmgParams(smoother="ilu0", ilu_sweep_order="latest_last").c()
    assert c2.ilu_sweep_order == 1
    c2.ilu_sweep_order = 4
    with pytest.raises(pb.InvalidArgument):
        pb.setup(A, B, "ns_block", type("P", (), {"c": lambda self: c2})())


def test_no_cpu_fallback():
    if pb.device_count() > 0:
        pytest.skip("a device is visible")
    p = pb.generate_hex(nx=2, ny=2, nz=2, dirichlet="eliminate")
    with pytest.raises(pb.NoDevice):
        pb.setup(p.csr(), p.nullspace())
    with pytest.raises(pb.NoDevice):
        pb.Bsr3.from_host(p.nbrows, p.nbrows, p.ptr, p.col, p.val.reshape(-1))


def test_status_names():
    assert pb.lib.samg_status_name(9) == b"breakdown_non_spd"
    assert pb.lib.samg_status_name(103) == b"no_device"


@pytest.mark.parametrize("nx,ny,nz,clamp", [(3, 3, 3, True), (4, 3, 2, False), (5, 5, 5, True)])
def test_generator_matches_reference(ref, nx, ny, nz, clamp):
    r = ref.generate_hex(nx, ny, nz, 1.0, 0.3, clamp)
    p = pb.generate_hex(nx=nx, ny=ny, nz=nz, dirichlet="keep_rows" if clamp else "none")
    n, ptr, col, val = p.csr()
    import scipy.sparse as sp
    Ar = sp.csr_matrix((r.val, r.col, r.ptr), shape=(r.n, r.n)).toarray()
    Ag = sp.csr_matrix((val, col, ptr), shape=(n, n)).toarray()
    assert np.abs(Ar - Ag).max() <= 1e-15 * np.abs(Ar).max()
    np.testing.assert_array_equal(p.rhs, r.rhs)
    np.testing.assert_array_equal(p.xyz, r.coords)
    np.testing.assert_array_equal(p.nullspace(), ref.rigid_body_modes(r.coords))


def test_generator_free_dof_is_kept_rows_minus_face():
    """Eliminating the x=0 face equals deleting its rows/cols from the
    kept-rows matrix (same physics)."""
    k = pb.generate_hex(nx=4, ny=3, nz=3, dirichlet="keep_rows")
    e = pb.generate_hex(nx=4, ny=3, nz=3, dirichlet="eliminate")
    import scipy.sparse as sp
    Ak = sp.csr_matrix(k.csr()[3:0:-1] if False else (k.csr()[3], k.csr()[2], k.csr()[1]),
                       shape=(k.n, k.n)).toarray()
    Ae = sp.csr_matrix((e.csr()[3], e.csr()[2], e.csr()[1]), shape=(e.n, e.n)).toarray()
    keep = np.array([(i % 5) != 0 for i in range(k.nnodes)])
    dofs = np.repeat(keep, 3)
    np.testing.assert_array_equal(Ak[np.ix_(dofs, dofs)], Ae)
    np.testing.assert_array_equal(k.rhs[dofs], e.rhs)


def test_generator_configs_shapes():
    """Block counts of the BASELINE configs (SURVEY 8d formula)."""
    def blocks_free(mx, my, mz):
        return (3 * (mx - 1) - 2) * (3 * my - 2) * (3 * mz - 2)
    p = pb.generate_hex(nx=19, ny=19, nz=19, dirichlet="eliminate")
    assert p.nnzb == blocks_free(20, 20, 20) == 185020
    q = pb.generate_hex(nx=19, ny=19, nz=19, dirichlet="keep_rows")
    assert q.nnzb == (3 * 20 - 5) * (3 * 20 - 2) * (3 * 20 - 2) + 20 * 20 == 185420
    h = pb.generate_hex(nx=6, ny=5, nz=4, dirichlet="eliminate", heterogeneous=True,
                        load="random", seed=9)
    assert np.all(np.isfinite(h.val)) and np.abs(h.rhs).max() <= 1.0
    b = pb.generate_hex(nx=8, ny=2, nz=2, lx=4.0, dirichlet="eliminate", load="traction_xend",
                        x_slowest=True)
    # traction total = -area of the end face
    assert abs(b.rhs[2::3].sum() + 1.0) <= 1e-14


def test_mixed_precision_is_single_gpu_only():
    """The partitioned solver keeps fp64 operators: dsetup refuses MIXED
    before touching a device (include/samg_b200.h samg_precision)."""
    from paper_2202_09056_b200.dist import DistHierarchy
    p = pb.generate_hex(nx=3, ny=2, nz=2, dirichlet="eliminate")
    with pytest.raises(pb.Unsupported):
        DistHierarchy(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), 0, 2,
                      prm=pb.AmgParams(vcycle_precision="mixed"), emulate=True)


def test_bench_and_entry_compile():
    """bench.py and __graft_entry__.py are at least valid Python (the driver
    runs them on the GPU box only)."""
    import ast
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for f in ("bench.py", "__graft_entry__.py"):
        with open(os.path.join(root, f)) as fh:
            ast.parse(fh.read(), f)
