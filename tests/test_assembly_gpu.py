"""GPU FE primitives vs the oracle restatement of assembly.py:77-175:
CSR indptr/indices bit-exact, values to rounding; impedance faces; Jacobian check."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fe

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("box,ne", [((0.0, 0.0, 0.0, 0.6, 0.4, 0.3), (3, 2, 2)),
                                    ((0.0, 0.0, 0.0, 2.0, 1.6, 1.2), (10, 8, 6)),
                                    ((0.1, -0.2, 0.3, 0.4, 0.5, 0.9), (1, 1, 1))])
def test_hex27_assembly_matches_oracle(cuda, box, ne):
    from paper_2310_04734_b200 import assembly
    xyz, conn = assembly.hex27_box(box, *ne)
    nodes, elems = fe.structured_hex27(box, *ne)
    np.testing.assert_array_equal(conn, elems)
    np.testing.assert_array_equal(xyz, nodes)
    Kg, Mn = assembly.assemble_helmholtz(xyz, conn)
    Kr, Mr = fe.assemble_helmholtz(nodes, elems, fe.HEX27_IDX)
    n, nnz = fe.hex27_pattern_counts(*ne)
    assert Kg.nnz == nnz
    for D, R in ((Kg, Kr), (Mn, Mr)):
        S = D.to_scipy()
        np.testing.assert_array_equal(S.indptr, R.indptr)      # bit-exact pattern
        np.testing.assert_array_equal(S.indices, R.indices)
        np.testing.assert_allclose(S.data, R.data, rtol=0, atol=1e-13 * np.abs(R.data).max())


def test_assembly_is_deterministic(cuda):
    from paper_2310_04734_b200 import assembly
    xyz, conn = assembly.hex27_box((0, 0, 0, 1.0, 0.8, 0.5), 5, 4, 3)
    a = assembly.assemble_helmholtz(xyz, conn)[0].data.cpu().numpy()
    b = assembly.assemble_helmholtz(xyz, conn)[0].data.cpu().numpy()
    assert np.array_equal(a, b)


def test_face_mass_matches_oracle(cuda):
    from paper_2310_04734_b200 import assembly
    box, ne = (0.0, 0.0, 0.0, 0.6, 0.4, 0.3), (3, 2, 2)
    xyz, conn = assembly.hex27_box(box, *ne)
    for side in ("z0", "x1", "y0"):
        fc = assembly.hex27_box_face(ne, side, conn)
        F = assembly.assemble_face_mass(xyz, fc).to_scipy()
        el, loc = fe.hex27_face(ne, side)
        R = fe.face_mass_hex27(xyz, conn.astype(np.int64), el, loc)
        np.testing.assert_array_equal(F.indptr, R.indptr)
        np.testing.assert_array_equal(F.indices, R.indices)
        np.testing.assert_allclose(F.data, R.data, rtol=0, atol=1e-15)


def test_generic_pattern_random_connectivity(cuda):
    """Arbitrary element lists (repeated dofs inside an element, unsorted ids)."""
    import torch
    from paper_2310_04734_b200 import assembly
    rng = np.random.default_rng(0)
    n, ne, npe = 57, 40, 5
    conn = rng.integers(0, n, size=(ne, npe)).astype(np.int32)
    vals = rng.standard_normal((ne, npe * npe))
    pat = assembly.pattern_from_elements(n, torch.as_tensor(conn, device=cuda))
    D = pat.gather(torch.as_tensor(vals, device=cuda)).to_scipy()
    R = fe.triplets_to_csr(n, conn.astype(np.int64), [vals])[0]
    np.testing.assert_array_equal(D.indptr, R.indptr)
    np.testing.assert_array_equal(D.indices, R.indices)
    np.testing.assert_allclose(D.data, R.data, atol=1e-14)


def test_negative_jacobian_raises(cuda):
    from paper_2310_04734_b200 import assembly
    xyz, conn = assembly.hex27_box((0, 0, 0, 1, 1, 1), 2, 1, 1)
    conn = conn.copy()
    conn[1] = conn[1][::-1]  # mirrored element: detJ < 0
    with pytest.raises(ValueError, match="element 1"):
        assembly.assemble_helmholtz(xyz, conn)


@pytest.mark.parametrize("ne", [(3, 2, 2), (10, 8, 6), (1, 1, 1), (4, 1, 3)])
def test_box_fast_path_equals_general_assembly(cuda, ne):
    """vb_hex27_box_csr (analytic pattern, shared element matrix) == the general
    sort/gather path: pattern bit-exact, values to rounding."""
    from paper_2310_04734_b200 import assembly
    box = (0.0, 0.0, 0.0, 2.0, 1.6, 1.2)
    Kb, Mb = assembly.assemble_helmholtz_box(box, ne)
    xyz, conn = assembly.hex27_box(box, *ne)
    Kg, Mg = assembly.assemble_helmholtz(xyz, conn)
    for A, B in ((Kb, Kg), (Mb, Mg)):
        Sa, Sb = A.to_scipy(), B.to_scipy()
        np.testing.assert_array_equal(Sa.indptr, Sb.indptr)
        np.testing.assert_array_equal(Sa.indices, Sb.indices)
        np.testing.assert_allclose(Sa.data, Sb.data, rtol=0, atol=1e-13 * np.abs(Sb.data).max())


@pytest.mark.gpu
@pytest.mark.parametrize("ne,k", [((1, 1, 1), 2), ((3, 2, 2), 3), ((10, 8, 6), 5), ((17, 5, 3), 33)])
def test_kron_apply_equals_csr_spmm(cuda, ne, k):
    """vb_kron3_apply (matrix-free Kronecker form of the box primitives) == the
    assembled CSR product to rounding, incl. alpha/beta, strided X/Y, ragged
    x-y tiles and k not a multiple of the column chunk."""
    import torch
    from paper_2310_04734_b200 import assembly, linalg
    box = (0.0, 0.0, 0.0, 2.0, 1.6, 1.2)
    Kb, Mb = assembly.assemble_helmholtz_box(box, ne)
    assert Kb.kron is not None and Mb.kron is not None
    g = torch.Generator(device="cuda").manual_seed(sum(ne) + k)
    n = Kb.n
    Xs = torch.randn(n, k + 3, dtype=torch.complex128, device="cuda", generator=g)
    X = Xs[:, 1:k + 1]                      # strided view (ldx = k + 3)
    Y0 = torch.randn(n, k, dtype=torch.complex128, device="cuda", generator=g)
    alpha, beta = 0.7 - 0.2j, -0.3 + 0.5j
    for A in (Kb, Mb):
        ref = linalg.spmm(A.with_data(A.data), X, alpha, beta, Y0.clone())   # CSR path
        Yk = torch.empty(n, k + 2, dtype=torch.complex128, device="cuda")
        Yv = Yk[:, :k]
        Yv.copy_(Y0)
        out = linalg.spmm(A, X, alpha, beta, Yv)                            # Kronecker path
        scale = float(ref.abs().max())
        assert float((out - ref).abs().max()) <= 1e-13 * scale
        # a single column (k = 1) stays on the CSR SpMV
        y1 = linalg.spmm(A, X[:, :1].contiguous())
        r1 = linalg.spmm(A.with_data(A.data), X[:, :1].contiguous())
        assert torch.equal(y1, r1)


def test_cfg3_full_size_pattern_bit_exact(cuda):
    """cfg3 at its BASELINE size (60 x 30 x 25 hex27, n = 376,431, nnz =
    23,300,121): both the general element sort/gather builder and the box
    fast path give indptr/indices bit-identical to the independent Kronecker
    pattern (oracle/fe.kron_pattern) = scipy's coo -> csr -> sum_duplicates
    structure of assembly.py:166-173."""
    import torch
    from paper_2310_04734_b200 import assembly, workloads
    ne = workloads.CFG3_NE
    R = fe.kron_pattern(*ne)
    n, nnz = fe.hex27_pattern_counts(*ne)
    assert R.shape == (n, n) and R.nnz == nnz == 23_300_121
    Kb, _ = assembly.assemble_helmholtz_box(workloads.CFG3_BOX, ne)
    np.testing.assert_array_equal(Kb.indptr.cpu().numpy(), R.indptr)
    np.testing.assert_array_equal(Kb.indices.cpu().numpy(), R.indices)
    del Kb
    xyz, conn = assembly.hex27_box(workloads.CFG3_BOX, *ne)
    pat = assembly.pattern_from_elements(n, torch.as_tensor(conn, device=cuda))
    np.testing.assert_array_equal(pat.indptr.cpu().numpy(), R.indptr)
    np.testing.assert_array_equal(pat.indices.cpu().numpy(), R.indices)
