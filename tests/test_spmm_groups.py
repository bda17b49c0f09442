"""Row-group SpMM format (vb_csr_row_groups, host C++ in libvibro_b200.so):
the grouping is exact (a partition of the rows, every member a subset of its
leader, masks/vmap reproduce the CSR) and, on lexicographic hex27 boxes,
finds the 2x2x2 node blocks.  GPU part: vb_rg_spmm and the sub-warp CSR
kernels against scipy (A @ X, mor.py:81-85) and against each other."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fe


def _groups(A):
    import torch
    from paper_2310_04734_b200 import linalg
    A = sp.csr_matrix(A)
    return linalg.RowGroups(A.shape[0], torch.as_tensor(A.indptr.astype(np.int32)),
                            torch.as_tensor(A.indices.astype(np.int32)))


def _emulate(A, rg, X):
    """numpy restatement of rg_spmm_kernel: per group, walk the leader's
    columns, update member i where mask bit i is set."""
    A = sp.csr_matrix(A)
    lead, rows, uoff = rg.leader.numpy(), rg.rows.numpy(), rg.uoff.numpy()
    masks, vmap = rg.masks.numpy(), rg.vmap.numpy()
    Y = np.zeros((A.shape[0], X.shape[1]), complex)
    for g in range(rg.n_groups):
        if lead[g] < 0:       # group of empty rows
            continue
        b, e = A.indptr[lead[g]], A.indptr[lead[g] + 1]
        for j in range(e - b):
            col, m = A.indices[b + j], masks[uoff[g] + j]
            for i in range(8):
                if m >> i & 1:
                    Y[rows[g, i]] += A.data[vmap[uoff[g] + j, i]] * X[col]
    return Y


def _check_structure(A, rg):
    A = sp.csr_matrix(A)
    n = A.shape[0]
    rows = rg.rows.numpy()
    members = rows[rows >= 0]
    assert np.array_equal(np.sort(members), np.arange(n))          # a partition of the rows
    lead, uoff = rg.leader.numpy(), rg.uoff.numpy()
    full = lead >= 0
    assert np.array_equal(rows[full, 0], lead[full])
    # leaderless groups hold exactly the empty rows, after all others
    empty = np.flatnonzero(np.diff(A.indptr) == 0)
    er = rows[~full]
    assert np.array_equal(np.sort(er[er >= 0]), empty)
    assert full[:full.sum()].all()
    masks, vmap = rg.masks.numpy(), rg.vmap.numpy()
    seen = np.zeros(A.nnz, bool)
    for g in np.flatnonzero(full):
        lc = A.indices[A.indptr[lead[g]]:A.indptr[lead[g] + 1]]
        for i, r in enumerate(rows[g]):
            if r < 0:
                assert not (masks[uoff[g]:uoff[g] + lc.size] >> i & 1).any()
                continue
            rc = A.indices[A.indptr[r]:A.indptr[r + 1]]
            assert set(rc) <= set(lc)                               # member ⊆ leader
            sl = slice(uoff[g], uoff[g] + lc.size)
            bits = (masks[sl] >> i & 1).astype(bool)
            assert np.array_equal(lc[bits], rc)
            pos = vmap[sl, i][bits]
            assert np.array_equal(pos, np.arange(A.indptr[r], A.indptr[r + 1]))
            assert (vmap[sl, i][~bits] == -1).all()
            seen[pos] = True
    assert seen.all()
    assert rg.n_union == sum(A.indptr[l + 1] - A.indptr[l] for l in lead[full])


def test_row_groups_hex27_box_are_node_blocks():
    nx, ny, nz = 4, 3, 3
    P = fe.kron_pattern(nx, ny, nz)
    rg = _groups(P)
    _check_structure(P, rg)
    # interior leaders are vertex nodes adopting their 2x2x2 node block:
    # mostly full groups, ~n/8 of them, 512 nonzeros over 125 leader columns
    sizes = (rg.rows.numpy() >= 0).sum(1)
    assert (sizes == 8).sum() >= nx * ny * nz
    assert rg.n_groups <= (nx + 1) * (ny + 1) * (nz + 1)
    reuse = P.nnz / rg.n_union
    assert reuse > 4.0, reuse


@pytest.mark.parametrize("seed", [0, 1])
def test_row_groups_general_pattern_reproduces_product(seed):
    rng = np.random.default_rng(seed)
    A = sp.random(120, 120, density=0.06, random_state=seed, format="csr") + sp.eye(120, format="csr")
    Kg, _ = fe.kron_box((0, 0, 0, 1.0, 0.8, 0.6), 3, 2, 2)
    for M in (sp.csr_matrix(A), Kg):
        M.sort_indices()
        rg = _groups(M)
        _check_structure(M, rg)
        X = rng.standard_normal((M.shape[1], 3)) + 1j * rng.standard_normal((M.shape[1], 3))
        np.testing.assert_allclose(_emulate(M, rg, X), M @ X, rtol=1e-13, atol=1e-13)


def test_row_groups_empty_rows_and_rectangular():
    A = sp.csr_matrix(np.array([[0, 0, 0, 0], [1.0, 0, 2, 0], [0, 0, 0, 0], [0, 3, 0, 0.0]]))
    A.eliminate_zeros()
    rg = _groups(A)
    _check_structure(A, rg)
    R = sp.random(30, 50, density=0.1, random_state=3, format="csr")
    rg = _groups(R)
    _check_structure(R, rg)


# ---------------------------------------------------------------- GPU ------

def _dev_csr(A, dev):
    import torch
    from paper_2310_04734_b200.assembly import DeviceCSR
    A = sp.csr_matrix(A)
    return DeviceCSR(A.shape[0], torch.as_tensor(A.indptr.astype(np.int32), device=dev),
                     torch.as_tensor(A.indices.astype(np.int32), device=dev),
                     torch.as_tensor(A.data, device=dev))


@pytest.mark.gpu
@pytest.mark.parametrize("k", [2, 3, 5, 8, 11, 16, 17, 32, 33, 64, 100])
@pytest.mark.parametrize("kind", ["random", "hex27", "wall"])
def test_spmm_paths_match_scipy_and_each_other(cuda, k, kind):
    import torch
    from paper_2310_04734_b200 import linalg
    rng = np.random.default_rng(k)
    if kind == "random":
        A = sp.random(700, 700, density=0.03, random_state=k, format="csr")
    elif kind == "hex27":
        A, _ = fe.kron_box((0, 0, 0, 1.2, 0.9, 0.7), 5, 4, 3)
        A = sp.csr_matrix(A)
        A.sort_indices()
    else:   # boundary primitive: rows of one wall only (most rows empty)
        A, _ = fe.kron_box((0, 0, 0, 1.2, 0.9, 0.7), 5, 4, 3)
        A = sp.csr_matrix(A)
        keep = np.zeros(A.shape[0])
        keep[: 11 * 9] = 1.0          # the z = 0 node layer
        A = sp.csr_matrix(sp.diags(keep) @ A @ sp.diags(keep))
        A.eliminate_zeros()
        A.sort_indices()
    n = A.shape[0]
    X = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    Y0 = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    alpha, beta = 0.5 - 2j, 1.5 + 0.25j
    Ad = _dev_csr(A, cuda)
    Xd = torch.as_tensor(X, device=cuda)
    outs = {}
    from paper_2310_04734_b200 import _lib
    lib = _lib.load()
    for path, mode in (("csr", 0), ("rg", 1), ("rg", 2), ("rg", 3)):   # DMMA / staged CUDA-core / direct CUDA-core
        lib.vb_set_rg_spmm_mode(mode)
        try:
            Yd = torch.as_tensor(Y0, device=cuda).clone()
            linalg.spmm(Ad, Xd, alpha, beta, Yd, path=path)
        finally:
            lib.vb_set_rg_spmm_mode(0)
        outs[(path, mode)] = Yd.cpu().numpy()
        np.testing.assert_allclose(outs[(path, mode)], alpha * (A @ X) + beta * Y0, rtol=1e-13, atol=1e-12)
    np.testing.assert_allclose(outs[("rg", 1)], outs[("csr", 0)], rtol=1e-14, atol=1e-13)
    np.testing.assert_allclose(outs[("rg", 2)], outs[("csr", 0)], rtol=1e-14, atol=1e-13)
    np.testing.assert_allclose(outs[("rg", 3)], outs[("csr", 0)], rtol=1e-14, atol=1e-13)
    # strided views (ldx, ldy > k) through the auto path
    Xw = torch.zeros((n, k + 3), dtype=torch.complex128, device=cuda)
    Xw[:, :k] = Xd
    Yw = torch.zeros((n, k + 5), dtype=torch.complex128, device=cuda)
    linalg.spmm(Ad, Xw[:, :k], 1.0, 0.0, Yw[:, :k])
    np.testing.assert_allclose(Yw[:, :k].cpu().numpy(), A @ X, rtol=1e-13, atol=1e-12)
    assert (Yw[:, k:] == 0).all()
