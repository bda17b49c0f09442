"""Dense GPU LU (vb_zgetrf / vb_zgetrs) vs numpy.linalg.solve; residual contract
of solvers.py:62-78 (||Ax-b||/||b|| <= 1e-10, tests/test_solvers.py:65-69)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _c(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.mark.parametrize("n,s", [(1, 1), (5, 2), (64, 1), (65, 3), (200, 16), (1000, 4), (3001, 1)])
def test_dense_lu_random(cuda, n, s):
    import torch
    from paper_2310_04734_b200.solvers import DenseLU
    rng = np.random.default_rng(n)
    A = _c(rng, n, n)
    b = _c(rng, n, s)
    lu = DenseLU(torch.as_tensor(A, device=cuda), copy=True)
    assert lu.info == 0
    x = lu.solve(torch.as_tensor(b, device=cuda)).cpu().numpy()
    res = np.linalg.norm(A @ x - b) / np.linalg.norm(b)
    assert res <= 1e-10, res
    xr = np.linalg.solve(A, b)
    assert np.abs(x - xr).max() <= 1e-9 * np.abs(xr).max()


def test_dense_lu_pivots_match_lapack_semantics(cuda):
    """Row interchanges are required (zero leading diagonal) and follow izamax."""
    import scipy.linalg as sla
    import torch
    from paper_2310_04734_b200.solvers import DenseLU
    rng = np.random.default_rng(5)
    n = 150
    A = _c(rng, n, n)
    A[np.arange(n), np.arange(n)] = 0.0
    lu = DenseLU(torch.as_tensor(A, device=cuda), copy=True)
    lu_ref, piv_ref = sla.lu_factor(A)
    ipiv = lu.ipiv.cpu().numpy()
    # identical pivot sequence on a generic matrix (no near-ties)
    np.testing.assert_array_equal(ipiv, piv_ref)
    np.testing.assert_allclose(lu.A.cpu().numpy(), lu_ref, rtol=0, atol=1e-10 * np.abs(lu_ref).max())
    b = _c(rng, n)
    x = lu.solve(torch.as_tensor(b, device=cuda)).cpu().numpy()
    assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) <= 1e-12


def test_dense_lu_singular(cuda):
    import torch
    from paper_2310_04734_b200.solvers import DenseLU
    n = 70
    A = np.eye(n, dtype=complex)
    A[40, 40] = 0.0
    lu = DenseLU(torch.as_tensor(A, device=cuda), copy=True)
    assert lu.info == 41
    with pytest.raises(RuntimeError, match="singular"):
        lu.solve(torch.ones(n, dtype=torch.complex128, device=cuda))


def test_dense_lu_cfg1_operator(cuda):
    """The cfg1 full-order operator K - w^2 M + i w D (n = 4641) at 87.5 Hz."""
    import torch
    from paper_2310_04734_b200 import assembly, linalg
    from paper_2310_04734_b200.solvers import DenseLU
    box, ne = (0.0, 0.0, 0.0, 2.0, 1.6, 1.2), (10, 8, 6)
    xyz, conn = assembly.hex27_box(box, *ne)
    Kg, Mn = assembly.assemble_helmholtz(xyz, conn)
    F = assembly.assemble_face_mass(xyz, assembly.hex27_box_face(ne, "z0", conn))
    rho, c = 1.21, 343.0
    w = 2 * np.pi * 87.5
    n = Kg.n
    A = torch.zeros((n, n), dtype=torch.complex128, device=cuda)
    linalg.axpy_dense(Kg, 1 / rho, A)
    linalg.axpy_dense(Mn, -w * w / (rho * c * c), A)
    linalg.axpy_dense(F, 1j * w / (rho * c * (5 + 1j)), A)
    Ah = A.cpu().numpy()
    b = np.zeros(n, complex)
    b[2000] = 1.0
    lu = DenseLU(A, copy=True)
    x = lu.solve(torch.as_tensor(b, device=cuda)).cpu().numpy()
    assert np.linalg.norm(Ah @ x - b) / np.linalg.norm(b) <= 1e-10


@pytest.mark.parametrize("n", [700, 3001, 4641, 8102])
def test_lookahead_lu_equals_plain_kernel(cuda, n):
    """The look-ahead LU (panel CTAs factor panel k+1 while the rest run the
    trailing update of panel k) takes the same izamax pivots as the plain
    kernel, and the same operations per element (up to the compiler's FMA
    contraction at the two call sites: factors equal to ~1e-13 relative)."""
    import torch
    from paper_2310_04734_b200 import _lib
    from paper_2310_04734_b200.solvers import DenseLU
    lib = _lib.load()
    rng = np.random.default_rng(n + 3)
    A = torch.as_tensor(_c(rng, n, n), device=cuda)
    out = {}
    for la in (0, 1):
        lib.vb_set_lu_lookahead(la)
        try:
            lu = DenseLU(A, copy=True)
            torch.cuda.synchronize()
        finally:
            lib.vb_set_lu_lookahead(1)
        out[la] = (lu.A.clone(), lu.ipiv.clone(), lu.info)
    assert out[0][2] == out[1][2] == 0
    assert torch.equal(out[0][1], out[1][1])
    d = float((out[0][0] - out[1][0]).abs().max() / out[0][0].abs().max())
    assert d <= 1e-10, d
    b = torch.as_tensor(_c(rng, n, 2), device=cuda)
    lu = DenseLU(A, copy=True)
    x = lu.solve(b)
    res = float(torch.linalg.norm(A @ x - b) / torch.linalg.norm(b))
    assert res <= 1e-10, res


def test_lookahead_lu_singular_column(cuda):
    import torch
    from paper_2310_04734_b200.solvers import DenseLU
    n = 3200
    A = np.eye(n, dtype=complex) * 2.0
    A[2500, 2500] = 0.0
    lu = DenseLU(torch.as_tensor(A, device=cuda), copy=True)
    assert lu.info == 2501
