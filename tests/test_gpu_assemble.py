"""On-GPU assembly (assemble.cu): bitwise equal to the host
generator (itself the reference generator, elasticity.hpp:129-213, extended)
for every problem family, and a hierarchy set up from the device problem
equals the one from the host problem."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FAMILIES = [
    dict(nx=4, ny=4, nz=4, dirichlet="keep_rows"),
    dict(nx=5, ny=4, nz=3, dirichlet="eliminate", noise=0.01, seed=3),
    dict(nx=9, ny=7, nz=5, dirichlet="eliminate", load="traction_xend"),
    dict(nx=7, ny=7, nz=7, dirichlet="eliminate", heterogeneous=True, load="random", seed=7),
    dict(nx=12, ny=4, nz=4, lx=3.0, dirichlet="eliminate", load="traction_xend", x_slowest=True),
    dict(nx=6, ny=5, nz=4, dirichlet="none", E=2.5, nu=0.25),
    dict(nx=8, ny=6, nz=5, dirichlet="eliminate", node_begin=40, node_end=170),
]


@pytest.mark.parametrize("kw", FAMILIES)
def test_device_assembly_bitwise(gpu, kw):
    pb = gpu
    host = pb.generate_hex(**kw)
    dev = pb.generate_hex_device(**kw)
    assert dev.nbrows == host.nbrows and dev.nnzb == host.nnzb and dev.n == host.n
    nr, nc, ptr, col, val = dev.A.download()
    np.testing.assert_array_equal(ptr, host.ptr)
    np.testing.assert_array_equal(col, host.col)
    np.testing.assert_array_equal(val.reshape(-1), host.val.reshape(-1))
    rhs, B, xyz = dev.download()
    np.testing.assert_array_equal(rhs, host.rhs)
    np.testing.assert_array_equal(xyz, host.xyz)
    np.testing.assert_array_equal(B, pb.rigid_body_modes(host.xyz))


def test_setup_from_device_problem(gpu):
    pb = gpu
    kw = dict(nx=10, ny=8, nz=7, dirichlet="eliminate", load="traction_xend")
    host = pb.generate_hex(**kw)
    dev = pb.generate_hex_device(**kw)
    prm = pb.AmgParams(coarse_enough=150)
    h1 = pb.setup_bsr3(host.nbrows, host.ptr, host.col, host.val.reshape(-1), host.nullspace(),
                       "ns_block", prm)
    h2 = pb.setup_device(dev.A, dev.nullspace_ptr, 6, "ns_block", prm)
    assert h1.nlevels == h2.nlevels
    for l in range(h1.nlevels):
        for w in ((0, 1, 2) if l < h1.nlevels - 1 else (0,)):
            a, b = h1.level(l, w), h2.level(l, w)
            for x, y in zip(a[2:], b[2:]):
                np.testing.assert_array_equal(x, y)
    u1, r1 = h1.cg_solve(host.rhs)
    u2, r2 = h2.cg_solve(host.rhs)
    assert r1["iterations"] == r2["iterations"]
    np.testing.assert_array_equal(u1, u2)


def test_device_problem_is_released_without_the_cyclic_collector(gpu):
    """A dropped DeviceProblem frees its device memory at once: the borrowed
    matrix view is made per access, not stored on the problem (a stored view
    -> owner -> view cycle left C4's 17 GB to the cyclic collector and the next
    setup grew the memory pool by as much)."""
    import gc
    import weakref
    pb = gpu
    gc.disable()
    try:
        dev = pb.generate_hex_device(nx=4, ny=4, nz=4, dirichlet="eliminate")
        view = dev.A
        assert view.shape[0] == dev.nbrows
        ref = weakref.ref(dev)
        del view, dev
        assert ref() is None
    finally:
        gc.enable()
