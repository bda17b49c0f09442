"""The oracle restatement reproduces the unmodified reference (golden fixtures
from tests/golden/make_golden.py) — CPU only."""

import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fe, mor as omor


def _csr(z, prefix):
    n = len(z[f"{prefix}_indptr"]) - 1
    return sp.csr_matrix((z[f"{prefix}_data"], z[f"{prefix}_indices"], z[f"{prefix}_indptr"]), shape=(n, n))


@pytest.fixture(scope="module")
def frozen(golden_dir):
    z = np.load(golden_dir / "frozen_fom.npz")
    K, M, b, c = sp.csc_matrix(z["K"]), sp.csc_matrix(z["M"]), z["b"], z["c"]
    fom = omor.Fom(stiffness=lambda f: K, mass=lambda f: M, load=lambda f: b, c_out=c, n=len(b))
    return z, fom


def test_krylov_block_matches_reference(frozen):
    z, fom = frozen
    Q1, br = omor.krylov_block(fom, 35.0, 5)
    assert not br
    np.testing.assert_allclose(Q1, z["Q1"], atol=1e-12)
    Q2, _ = omor.krylov_block(fom, 55.0, 4)
    np.testing.assert_allclose(Q2, z["Q2"], atol=1e-12)
    V = omor.orthonormalise(Q1, Q2)
    np.testing.assert_allclose(V, z["V"], atol=1e-11)


def test_reduced_output_matches_reference(frozen):
    z, fom = frozen
    for f, yr, yf in zip(z["freqs"], z["y_rom"], z["y_fom"]):
        y = omor.reduced_output(fom, z["V"], f)
        assert abs(y - yr) <= 1e-11 * abs(yr)
        assert abs(fom.output(fom.solve(f)) - yf) <= 1e-12 * abs(yf)


def test_orthonormalise_drop_rule(golden_dir):
    z = np.load(golden_dir / "frozen_fom.npz")
    Q = omor.orthonormalise(None, z["drop_block"])
    assert Q.shape == z["drop_Q"].shape == (30, 2)
    np.testing.assert_allclose(Q, z["drop_Q"], atol=1e-13)


def test_quad9_assembly_matches_reference(golden_dir):
    z = np.load(golden_dir / "assembly_2d.npz")
    Ke, Me = fe.helmholtz_element_parts(fe.QUAD9_IDX, z["coords"])
    np.testing.assert_allclose(Ke, z["Ke"], rtol=0, atol=1e-14 * np.abs(z["Ke"]).max())
    np.testing.assert_allclose(Me, z["Me"], rtol=0, atol=1e-14 * np.abs(z["Me"]).max())
    nodes, elems = fe.structured_quad9((0.0, 0.0, 0.9, 0.6), 3, 3)
    np.testing.assert_array_equal(nodes, z["nodes"])
    np.testing.assert_array_equal(elems, z["elements"])
    Kg, Mn = fe.assemble_helmholtz(nodes, elems, fe.QUAD9_IDX)
    for A, p in ((Kg, "Kgrad"), (Mn, "Mnn")):
        R = _csr(z, p)
        np.testing.assert_array_equal(A.indptr, R.indptr)      # bit-exact pattern
        np.testing.assert_array_equal(A.indices, R.indices)
        np.testing.assert_allclose(A.data, R.data, rtol=0, atol=1e-15 * np.abs(R.data).max())


def test_hex27_assembly_equals_kronecker_sum():
    box, ne = (0.0, 0.0, 0.0, 1.0, 0.7, 0.45), (3, 2, 2)
    nodes, elems = fe.structured_hex27(box, *ne)
    Kg, Mn = fe.assemble_helmholtz(nodes, elems, fe.HEX27_IDX)
    Kk, Mk = fe.kron_box(box, *ne)
    n, nnz = fe.hex27_pattern_counts(*ne)
    assert Kg.shape == (n, n) and Kg.nnz == nnz == Mn.nnz
    for A, B in ((Kg, Kk), (Mn, Mk)):
        B = B.tocsr()
        B.sort_indices()
        np.testing.assert_allclose((A - B).toarray(), 0.0, atol=1e-13 * abs(A).max())
    # canonical CSR pattern == Kronecker product of the 1D element-block patterns
    P = fe.kron_pattern(*ne)
    np.testing.assert_array_equal(Kg.indptr, P.indptr)
    np.testing.assert_array_equal(Kg.indices, P.indices)
    np.testing.assert_array_equal(Mn.indices, P.indices)


def test_hex27_partition_of_unity_and_volume():
    coords = fe.structured_hex27((0.2, 0.1, 0.0, 0.5, 0.3, 0.4), 1, 1, 1)[0]
    Ke, Me = fe.helmholtz_element_parts(fe.HEX27_IDX, coords)
    np.testing.assert_allclose(Ke @ np.ones(27), 0.0, atol=1e-13)
    assert Me.sum() == pytest.approx(0.3 * 0.2 * 0.4, rel=1e-13)


def test_rigid_box_resonances_against_analytic():
    """assembly.py conventions in 3D: f_lmn = c/2 sqrt((l/Lx)^2+(m/Ly)^2+(n/Lz)^2)
    within 1% (pattern of reference tests/test_assembly.py:101-116)."""
    import scipy.linalg as la
    L = (1.0, 0.8, 0.6)
    nodes, elems = fe.structured_hex27((0, 0, 0) + L, 4, 3, 3)
    Kg, Mn = fe.assemble_helmholtz(nodes, elems, fe.HEX27_IDX)
    lam = la.eigh(Kg.toarray(), Mn.toarray(), eigvals_only=True)
    c = 343.0
    f_num = np.sort(c * np.sqrt(np.clip(lam, 0, None)) / (2 * np.pi))
    f_num = f_num[f_num > 1.0][:8]
    f_ex = sorted(c / 2 * math.sqrt((a / L[0]) ** 2 + (b / L[1]) ** 2 + (d / L[2]) ** 2)
                  for a in range(4) for b in range(4) for d in range(4) if a or b or d)[:8]
    for fe_, fn in zip(f_ex, f_num):
        assert abs(fn - fe_) <= 0.01 * fe_


def test_face_mass_area():
    box, ne = (0.0, 0.0, 0.0, 0.6, 0.4, 0.3), (3, 2, 2)
    nodes, elems = fe.structured_hex27(box, *ne)
    for side, area in (("z0", 0.24), ("x1", 0.12), ("y0", 0.18)):
        el, loc = fe.hex27_face(ne, side)
        F = fe.face_mass_hex27(nodes, elems, el, loc)
        assert F.sum() == pytest.approx(area, rel=1e-13)
        ax = "xyz".index(side[0])
        val = box[ax + 3] if side[1] == "1" else box[ax]
        touched = np.unique(F.tocoo().row)
        assert np.allclose(nodes[touched, ax], val)


def _box_fom(z):
    rho, c = 1.21, 343.0
    K = (_csr(z, "Kg") / rho).astype(complex)
    M = (_csr(z, "Mn") / (rho * c * c)).astype(complex)
    D = _csr(z, "Fz") / (rho * c * (5 + 1j))
    n = K.shape[0]
    C = np.zeros((len(z["rec"]), n))
    C[np.arange(len(z["rec"])), z["rec"]] = 1.0
    return omor.Fom(stiffness=lambda f: K, mass=lambda f: M, load=lambda f: z["b"], c_out=C, n=n,
                    damping=lambda f: D)


def test_box_mor_matches_reference(golden_dir):
    z = np.load(golden_dir / "box_mor.npz")
    # the oracle's restated box assembly is exactly what the golden run consumed
    nodes, elems = fe.structured_hex27((0.0, 0.0, 0.0, 0.6, 0.4, 0.3), 3, 2, 2)
    Kg, Mn = fe.assemble_helmholtz(nodes, elems, fe.HEX27_IDX)
    np.testing.assert_array_equal(Kg.indptr, z["Kg_indptr"])
    np.testing.assert_array_equal(Kg.indices, z["Kg_indices"])
    np.testing.assert_allclose(Kg.data, z["Kg_data"], atol=0)
    fom = _box_fom(z)
    V = None
    for f0 in z["points"]:
        Q, _ = omor.krylov_block(fom, f0, 4, second_order=True)
        V = omor.orthonormalise(V, Q)
    np.testing.assert_allclose(np.abs(V), np.abs(z["V"]), atol=1e-10)
    own, seams = omor.window_owners([(200.0, 600.0), (600.0, 1000.0)], list(z["grid"]))
    np.testing.assert_array_equal(own, z["window_index"])
    for i, f in enumerate(z["grid"]):
        Vw = V if own[i] == 0 else V[:, :6]
        y = omor.reduced_output(fom, Vw, f)
        _, e, _, _ = omor.relative_error(z["y"][i], y)
        assert e <= 1e-9
        assert abs(omor.mean_spl(y) - z["spl"][i]) <= 1e-9
    assert [z["grid"][i] for i, _ in seams] == list(z["seam_f"])


def test_affine_sweep_matches_reference_literal_path(golden_dir):
    from paper_2310_04734_b200 import workloads
    z = np.load(golden_dir / "reduced_dense.npz")
    w = workloads.cfg5(r=int(z["r"]), n_freq=int(z["n_freq"]), s=int(z["s"]), n_out=int(z["n_out"]),
                       seed=int(z["seed"]))
    y, spl = omor.affine_sweep(w.prims, w.alpha(z["freqs"]), w.b, w.c_r)
    for i in range(len(z["freqs"])):
        _, e, _, _ = omor.relative_error(z["y"][i].ravel(), y[i].ravel())
        assert e <= 1e-10
    np.testing.assert_allclose(spl, z["spl"], atol=1e-9)


def test_mean_spl_values(golden_dir):
    z = np.load(golden_dir / "spl.npz")
    assert omor.mean_spl(np.ones(64, complex)) == z["ones"]
    assert omor.mean_spl(np.zeros(5, complex)) == z["zeros"]
    assert omor.mean_spl(z["p"]) == pytest.approx(float(z["random"]), abs=1e-12)
    assert z["ones"] == pytest.approx(20 * np.log10(1 / np.sqrt(2) / 20e-6))


def test_relative_error_semantics():
    y = np.array([1.0, 2.0, 3.0])
    eps, emax, k, flag = omor.relative_error(y, 1.01 * y)
    assert emax == pytest.approx(0.01) and not flag
    eps, emax, k, flag = omor.relative_error([0.0, 2.0], [0.5, 2.0])
    assert flag and eps[0] == pytest.approx(0.5)
