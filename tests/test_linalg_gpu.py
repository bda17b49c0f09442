"""GPU SpMM / dense scatter / DMMA ZGEMM / column norms vs numpy/scipy."""

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


def _dev_csr(A, cuda):
    import torch
    from paper_2310_04734_b200.assembly import DeviceCSR
    A = sp.csr_matrix(A)
    return DeviceCSR(A.shape[0], torch.as_tensor(A.indptr.astype(np.int32), device=cuda),
                     torch.as_tensor(A.indices.astype(np.int32), device=cuda),
                     torch.as_tensor(A.data, device=cuda))


def _c(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.mark.parametrize("k", [1, 3, 32, 45])
def test_spmm(cuda, k):
    import torch
    from paper_2310_04734_b200 import linalg
    rng = np.random.default_rng(k)
    A = sp.random(300, 300, density=0.05, random_state=k, format="csr")
    X = _c(rng, 300, k)
    Y0 = _c(rng, 300, k)
    alpha, beta = 0.5 - 2j, 1.5 + 0.25j
    Xd = torch.as_tensor(X, device=cuda)
    Yd = torch.as_tensor(Y0, device=cuda)
    linalg.spmm(_dev_csr(A, cuda), Xd if k > 1 else Xd[:, 0], alpha, beta, Yd if k > 1 else Yd[:, 0].contiguous())
    if k > 1:
        np.testing.assert_allclose(Yd.cpu().numpy(), alpha * (A @ X) + beta * Y0, rtol=1e-13, atol=1e-12)
    out = linalg.spmm(_dev_csr(A, cuda), Xd)
    np.testing.assert_allclose(out.cpu().numpy(), A @ X, rtol=1e-13, atol=1e-12)


def test_axpy_dense(cuda):
    import torch
    from paper_2310_04734_b200 import linalg
    rng = np.random.default_rng(1)
    A = sp.random(50, 50, density=0.2, random_state=1, format="csr")
    D0 = _c(rng, 50, 50)
    Dd = torch.as_tensor(D0, device=cuda)
    linalg.axpy_dense(_dev_csr(A, cuda), 2 - 1j, Dd)
    np.testing.assert_allclose(Dd.cpu().numpy(), D0 + (2 - 1j) * A.toarray(), rtol=1e-14, atol=1e-14)


@pytest.mark.parametrize("m,n,k", [(32, 32, 4641), (76, 76, 8102), (5, 1, 1000), (400, 40, 3000), (1, 7, 13),
                                   (33, 1, 5000), (64, 1, 100), (65, 1, 300), (300, 10, 20000), (17, 16, 2000)])
def test_zgemm_conj(cuda, m, n, k):
    import torch
    from paper_2310_04734_b200 import linalg
    rng = np.random.default_rng(m + n + k)
    A, B, C0 = _c(rng, k, m), _c(rng, k, n), _c(rng, m, n)
    Cd = torch.as_tensor(C0, device=cuda)
    linalg.zgemm("C", torch.as_tensor(A, device=cuda), torch.as_tensor(B, device=cuda), 2.0, 0.5j, Cd)
    ref = 2.0 * A.conj().T @ B + 0.5j * C0
    np.testing.assert_allclose(Cd.cpu().numpy(), ref, rtol=1e-12, atol=1e-10 * np.abs(ref).max())


@pytest.mark.parametrize("m,n,k", [(4641, 8, 32), (100, 33, 70), (1, 1, 1), (257, 16, 513),
                                   (20000, 1, 33), (5000, 1, 64), (300, 1, 65), (20000, 10, 300)])
def test_zgemm_nn(cuda, m, n, k):
    import torch
    from paper_2310_04734_b200 import linalg
    rng = np.random.default_rng(m * n + k)
    A, B, C0 = _c(rng, m, k), _c(rng, k, n), _c(rng, m, n)
    Cd = torch.as_tensor(C0, device=cuda)
    linalg.zgemm("N", torch.as_tensor(A, device=cuda), torch.as_tensor(B, device=cuda), -1.0, 1.0, Cd)
    ref = C0 - A @ B
    np.testing.assert_allclose(Cd.cpu().numpy(), ref, rtol=1e-12, atol=1e-11 * np.abs(ref).max())
    out = linalg.zgemm("N", torch.as_tensor(A, device=cuda), torch.as_tensor(B, device=cuda))
    np.testing.assert_allclose(out.cpu().numpy(), A @ B, rtol=1e-12, atol=1e-11 * np.abs(ref).max())


def test_zgemm_strided_views(cuda):
    """Column slices of a wider buffer (ld > columns), as the basis build uses."""
    import torch
    from paper_2310_04734_b200 import linalg
    rng = np.random.default_rng(7)
    Vb = torch.as_tensor(_c(rng, 3000, 48), device=cuda)
    Xb = torch.as_tensor(_c(rng, 3000, 12), device=cuda)
    for nv, nx in ((40, 1), (40, 10), (9, 1)):
        V, X = Vb[:, :nv], Xb[:, 2:2 + nx]
        G = linalg.zgemm("C", V, X)
        ref = V.conj().T @ X
        assert float((G - ref).abs().max()) <= 1e-12 * float(ref.abs().max())
        Y = X.clone()
        linalg.zgemm("N", V, G, -1.0, 1.0, Y)
        ref2 = X - V @ G
        assert float((Y - ref2).abs().max()) <= 1e-12 * float(ref2.abs().max())


def test_column_norms_and_scale(cuda):
    import torch
    from paper_2310_04734_b200 import linalg
    rng = np.random.default_rng(3)
    W = _c(rng, 5000, 7)
    Wd = torch.as_tensor(W, device=cuda)
    nr = linalg.column_norms(Wd).cpu().numpy()
    np.testing.assert_allclose(nr, np.linalg.norm(W, axis=0), rtol=1e-14)
    linalg.scale_columns(Wd, torch.as_tensor(1 / nr, device=cuda))
    np.testing.assert_allclose(np.linalg.norm(Wd.cpu().numpy(), axis=0), 1.0, rtol=1e-14)


@pytest.mark.parametrize("n,kb", [(5000, 10), (37, 16), (100000, 3)])
def test_block_gs_matches_reference_drop_rule(cuda, n, kb):
    """vb_block_gs (fused in-block CGS2 + drop rule, mor.py:122-135) against the
    oracle's MGS2 on a block with an exact duplicate, a near-dependent column
    (1e-12 residual: dropped) and a weakly dependent one (1e-6: kept)."""
    import torch
    from oracle import mor as omor
    from paper_2310_04734_b200 import linalg, mor
    rng = np.random.default_rng(n + kb)
    B = _c(rng, n, kb)
    if kb >= 3:
        B[:, 1] = B[:, 0]
        B[:, 2] = B[:, 0] + 1e-12 * _c(rng, n)
    if kb >= 5:
        B[:, 4] = B[:, 3] + 1e-6 * _c(rng, n)
    Wd = torch.as_tensor(B, device=cuda).clone()
    Qd = torch.empty((n, kb), dtype=torch.complex128, device=cuda)
    refs = linalg.column_norms(torch.as_tensor(B, device=cuda))
    nk, kept = linalg.block_gs(Wd, Qd, refs, mor.ORTH_DROP_TOL, mor.REORTH_RATIO)
    Qo = omor.orthonormalise(None, B)
    assert nk == Qo.shape[1]
    Q = Qd[:, :nk].cpu().numpy()
    assert np.abs(Q.conj().T @ Q - np.eye(nk)).max() <= 1e-12
    # same span as the reference's basis
    assert np.abs(Qo - Q @ (Q.conj().T @ Qo)).max() <= 1e-8
    if kb >= 3:
        assert list(kept[:3]) == [1, 0, 0]
    # no_drop, in place: re-orthonormalise an orthonormal-ish block
    P = torch.as_tensor(Q + 1e-9 * _c(rng, n, nk), device=cuda)
    linalg.block_gs(P, P, no_drop=True)
    Pn = P.cpu().numpy()
    assert np.abs(Pn.conj().T @ Pn - np.eye(nk)).max() <= 1e-12


def test_orthonormalise_blocks_equals_sequential_appends(cuda):
    """mor.orthonormalise_blocks (one V sweep pair per pass for a group of
    blocks) keeps the same columns as _orthonormalise block by block
    (mor.py:122-135), incl. a column that is dependent on an EARLIER block of
    the same group, and spans the same subspace with an orthonormal basis."""
    import torch
    from paper_2310_04734_b200 import mor
    g = torch.Generator(device="cuda").manual_seed(11)
    n = 5000
    V0 = mor._orthonormalise(None, torch.randn((n, 30), dtype=torch.complex128, device=cuda, generator=g))
    blocks = [torch.randn((n, 10), dtype=torch.complex128, device=cuda, generator=g) for _ in range(4)]
    blocks[2][:, 3] = blocks[0][:, 1] - 2j * blocks[1][:, 4] + 0.5 * V0[:, 7]   # dependent across blocks
    blocks[3][:, 0] = V0[:, 2]                                                    # inside the old basis
    Vs = V0.clone()
    for b in blocks:
        Vs = mor._orthonormalise(Vs, b.clone())
    Vg = mor.orthonormalise_blocks(V0.clone(), [b.clone() for b in blocks])
    assert Vs.shape == Vg.shape == (n, 30 + 38)
    eye = torch.eye(Vg.shape[1], dtype=torch.complex128, device=cuda)
    assert float((Vg.conj().T @ Vg - eye).abs().max()) <= 1e-12
    assert float((Vg[:, :30] - V0).abs().max()) == 0.0
    R = Vs - Vg @ (Vg.conj().T @ Vs)
    assert float(R.abs().max()) <= 1e-10


def test_orthonormalise_cholqr_fast_path_decisions(cuda):
    """_orthonormalise takes the Cholesky-QR fast path only when every column
    is provably kept, and then matches the reference MGS2 basis (same span,
    orthonormal to 1e-12); a block with a column near the drop threshold —
    or a weakly dependent one the Gram matrix cannot resolve — goes through
    the exact Gram-Schmidt with the reference's decisions (mor.py:122-135)."""
    import torch
    from oracle import mor as omor
    from paper_2310_04734_b200 import linalg, mor
    rng = np.random.default_rng(7)
    n = 20000
    V0 = np.linalg.qr(_c(rng, n, 12))[0]
    cases = {"fast": _c(rng, n, 24),
             "dropped": _c(rng, n, 6),
             "weak": _c(rng, n, 6)}
    cases["dropped"][:, 3] = cases["dropped"][:, 1] + 1e-12 * _c(rng, n)     # residual 1e-12: dropped
    cases["weak"][:, 4] = cases["weak"][:, 0] + 1e-7 * _c(rng, n)            # 1e-7: kept, but unresolved by the Gram
    calls = []
    orig = mor._cholqr_keep_all
    mor._cholqr_keep_all = lambda W, r: calls.append(orig(W, r) is not None) or orig(W, r)
    try:
        for name, B in cases.items():
            calls.clear()
            V = mor._orthonormalise(torch.as_tensor(V0, device=cuda), torch.as_tensor(B, device=cuda))
            Vo = omor.orthonormalise(V0, B)
            assert calls == [name == "fast"], (name, calls)
            Vn = V.cpu().numpy()
            assert Vn.shape == Vo.shape, name
            assert np.abs(Vn.conj().T @ Vn - np.eye(Vn.shape[1])).max() <= 1e-12
            assert np.abs(Vo - Vn @ (Vn.conj().T @ Vo)).max() <= 1e-8
    finally:
        mor._cholqr_keep_all = orig
    assert linalg.BLOCK_GS_MAX == 16
