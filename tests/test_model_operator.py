"""The ModelOperator drop-in (model_operator.affine_from_operator) on the CPU:
the device CSR terms x scalar coefficients it produces sum to exactly the
reference's K(f) and M(f) (assembly.py:259-284), and the tier-0 fixture's
tabulated scalars are the ones the reference computes.  Needs the reference
package (importable only in the build container): skipped elsewhere."""

import math
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

REF = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def ref_op():
    if not REF.exists():
        pytest.skip("reference package not present")
    import sys
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import vibrofem
    from vibrofem.cli import _mor_fom
    from vibrofem.config import load_config
    cfg = load_config(Path(vibrofem.__file__).parent / "data" / "fuselage_slice.cfg")
    fom, op = _mor_fom(cfg)
    return cfg, fom, op


def _host(terms, f):
    A = None
    for t in terms:
        S = t.P.to_scipy() * t.at(f)
        A = S if A is None else A + S
    return A


def test_affine_terms_sum_to_reference_operator(ref_op):
    from paper_2310_04734_b200.model_operator import affine_from_operator
    cfg, fom, op = ref_op
    aff = affine_from_operator(op, device="cpu")
    for f in (10.0, 316.0, 1000.0):
        K, M = op.K(f), op.M(f)
        Ka, Ma = _host(aff.K, f), _host(aff.M, f)
        for A, B in ((K, Ka), (M, Ma)):
            D = (A - B).tocoo()
            assert D.shape == A.shape
            assert (np.abs(D.data).max() if D.nnz else 0.0) <= 1e-12 * np.abs(A.data).max()
        np.testing.assert_array_equal(aff.load.host(f), op.load(f))
    assert fom.n == aff.n == 8102


def test_fixture_scalars_are_the_reference_values(ref_op, golden_dir):
    """The coefficient tables stored in fuselage_slice.npz equal the scalars
    reference_coefficients() resolves from the operator's module (the same
    calls _domain_KM / system make)."""
    from paper_2310_04734_b200.model_operator import reference_coefficients
    cfg, fom, op = ref_op
    z = np.load(golden_dir / "fuselage_slice.npz")
    co = reference_coefficients(op)
    grid = z["grid"]
    for i in (0, 123, 495):
        f = float(grid[i])
        for d in cfg.domains:
            assert co.kscale(d.id, f) == z[f"scale__{d.id}"][i]
            if d.kind != "elastic":
                rho, c = co.fluid(d.id, f)
                assert rho == z[f"rho_eff__{d.id}"][i] and c == z[f"c_eff__{d.id}"][i]
        for k in range(len(op.couplings)):
            assert co.rho_f(k, f) == z[f"rho_f{k}"][i]
        v = np.zeros(fom.n, complex)
        v[z["load_rows"]] = z["load_vals"][i]
        np.testing.assert_array_equal(v, op.load(f))
    assert int(z["probe"]) == int(np.argmax(fom.c_out))
    assert math.isclose(float(z["grid"][1] - z["grid"][0]), 2.0)


def test_device_csr_terms_split_complex():
    from paper_2310_04734_b200.model_operator import device_csr_terms
    rng = np.random.default_rng(0)
    A = sp.random(30, 20, density=0.2, random_state=1) + 1j * sp.random(30, 20, density=0.2, random_state=2)
    terms = device_csr_terms(A, "cpu", 5, 7, 40)
    assert len(terms) == 2
    S = sum(P.to_scipy() * fac for P, fac in terms)
    E = np.zeros((40, 40), complex)
    E[5:35, 7:27] = A.toarray()
    np.testing.assert_array_equal(S.toarray(), E)
    R = device_csr_terms(sp.csr_matrix(rng.standard_normal((4, 4))), "cpu")
    assert len(R) == 1
