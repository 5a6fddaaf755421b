"""Coarsest-level direct solver (coarse.cu, samg_bsr3_dense_inverse): the
in-place blocked Gauss-Jordan with partial pivoting against numpy, across
panel widths/cluster sizes, pivoting-heavy matrices and the singular case
(dense_lu, hierarchy.hpp:86-129)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def random_bsr3(nb, density, rng, diag=0.0):
    ptr, col, val = [0], [], []
    for i in range(nb):
        cols = sorted(set(rng.choice(nb, size=max(1, int(density * nb)), replace=False)) | {i})
        for c in cols:
            col.append(c)
            b = rng.standard_normal((3, 3))
            if c == i:
                b += diag * np.eye(3)
            val.append(b)
        ptr.append(len(col))
    return (np.array(ptr, np.int64), np.array(col, np.int64), np.array(val).reshape(-1))


def dense_of(nb, ptr, col, val):
    D = np.zeros((3 * nb, 3 * nb))
    v = val.reshape(-1, 3, 3)
    for i in range(nb):
        for j in range(ptr[i], ptr[i + 1]):
            D[3 * i:3 * i + 3, 3 * col[j]:3 * col[j] + 3] = v[j]
    return D


@pytest.mark.parametrize("nb,density,diag", [(1, 1.0, 0.0), (10, 1.0, 0.0), (33, 0.3, 0.0),
                                             (700, 0.01, 8.0), (1100, 0.004, 0.0)])
def test_dense_inverse_matches_numpy(gpu, nb, density, diag):
    pb = gpu
    rng = np.random.default_rng(nb)
    ptr, col, val = random_bsr3(nb, density, rng, diag)
    A = pb.Bsr3.from_host(nb, nb, ptr, col, val)
    X = A.dense_inverse()
    D = dense_of(nb, ptr, col, val)
    ref = np.linalg.inv(D)
    cond = np.linalg.cond(D)
    err = np.abs(X - ref).max() / np.abs(ref).max()
    assert err <= 1e-15 * cond * 3 * nb + 1e-13, (err, cond)
    assert np.abs(D @ X - np.eye(3 * nb)).max() <= 1e-14 * cond * 3 * nb + 1e-12


def test_dense_inverse_needs_pivoting(gpu):
    """Zero diagonal blocks: only row exchanges make it solvable."""
    pb = gpu
    nb = 40
    rng = np.random.default_rng(5)
    ptr, col, val = [0], [], []
    for i in range(nb):
        for c in sorted({(i + 1) % nb, (i + 7) % nb, i}):
            col.append(c)
            val.append(np.zeros((3, 3)) if c == i else rng.standard_normal((3, 3)))
        ptr.append(len(col))
    ptr, col, val = np.array(ptr, np.int64), np.array(col, np.int64), np.array(val).reshape(-1)
    A = pb.Bsr3.from_host(nb, nb, ptr, col, val)
    X = A.dense_inverse()
    D = dense_of(nb, ptr, col, val)
    assert np.abs(D @ X - np.eye(3 * nb)).max() <= 1e-14 * np.linalg.cond(D) * 3 * nb


def test_dense_inverse_singular_raises(gpu):
    from paper_2202_09056_b200._lib import SamgError
    pb = gpu
    nb = 20
    rng = np.random.default_rng(2)
    ptr, col, val = random_bsr3(nb, 0.2, rng, 4.0)
    v = val.reshape(-1, 3, 3)
    for j in range(ptr[7], ptr[8]):  # block row 7 identically zero
        v[j] = 0.0
    A = pb.Bsr3.from_host(nb, nb, ptr, col, v.reshape(-1))
    with pytest.raises(SamgError) as e:
        A.dense_inverse()
    assert e.value.code == 1


def test_coarse_level_inverse(gpu):
    """The coarsest matrix of a real hierarchy (C0-like cube)."""
    pb = gpu
    p = pb.generate_hex(nx=12, ny=12, nz=12, dirichlet="eliminate")
    h = pb.setup_bsr3(p.nbrows, p.ptr, p.col, p.val.reshape(-1), p.nullspace(), "ns_block",
                      pb.AmgParams())
    L = h.nlevels - 1
    Ac = h.level_matrix(L)
    nr, _, ptr, col, val = Ac.download()
    D = dense_of(nr, ptr, col, val.reshape(-1))
    X = Ac.dense_inverse()
    assert np.abs(D @ X - np.eye(3 * nr)).max() <= 1e-9


def spd_bsr3(nb, density, rng, shift):
    """Symmetric block pattern and values (A = M + M^T + shift I): SPD for a
    large enough shift, indefinite for a small one."""
    D = np.zeros((3 * nb, 3 * nb))
    for i in range(nb):
        for c in set(rng.choice(nb, size=max(1, int(density * nb)), replace=False)) | {i}:
            D[3 * i:3 * i + 3, 3 * c:3 * c + 3] += rng.standard_normal((3, 3))
    D = D + D.T + shift * np.eye(3 * nb)
    ptr, col, val = [0], [], []
    for i in range(nb):
        for c in range(nb):
            blk = D[3 * i:3 * i + 3, 3 * c:3 * c + 3]
            if np.any(blk != 0.0):
                col.append(c)
                val.append(blk)
        ptr.append(len(col))
    return np.array(ptr, np.int64), np.array(col, np.int64), np.array(val).reshape(-1), D


@pytest.mark.parametrize("nb,shift", [(700, 40.0), (973, 60.0), (500, 0.5)])
def test_dense_inverse_symmetric(gpu, nb, shift):
    """Symmetric coarse operators take the Gauss-Jordan path without row
    exchanges (k_panel_reg<.., false>) when every pivot of the equilibrated
    matrix stays positive (SPD; large shift, odd and even n), and fall back to
    partial pivoting when one does not (indefinite; small shift): the inverse
    is accurate either way."""
    pb = gpu
    rng = np.random.default_rng(nb)
    ptr, col, val, D = spd_bsr3(nb, 0.01, rng, shift)
    if shift > 1.0:
        assert np.linalg.eigvalsh(D).min() > 0.0
    else:
        assert np.linalg.eigvalsh(D).min() < 0.0
    A = pb.Bsr3.from_host(nb, nb, ptr, col, val)
    X = A.dense_inverse()
    cond = np.linalg.cond(D)
    ref = np.linalg.inv(D)
    assert np.abs(X - ref).max() <= (1e-15 * cond * 3 * nb + 1e-13) * np.abs(ref).max(), cond
    assert np.abs(D @ X - np.eye(3 * nb)).max() <= 1e-14 * cond * 3 * nb + 1e-12
