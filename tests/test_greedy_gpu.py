"""Greedy certification and local-ROM windows on the GPU pinned to the
UNMODIFIED reference (tests/golden/make_golden.py `greedy` ->
greedy_ref.npz): greedy_expand (mor.py:224-295) and build_local_roms with
explicit and auto-bisected windows (mor.py:298-353) must take the same
decisions — expansion points in order, reduced order r, converged / stalled /
budget flags, window boundaries — with the same candidate error logs, and
rom_sweep must reproduce the reference FRF.  Models: the reference's own test
fixtures oscillator_chain and frozen_fom (tests/test_mor.py:26-52)."""

import math

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu


class Settings:
    def __init__(self, tol=1e-2, max_points=20, moments_per_point=4, candidate_stride=4, windows="auto"):
        self.tol, self.max_points, self.moments_per_point = tol, max_points, moments_per_point
        self.candidate_stride, self.windows = candidate_stride, windows


def oscillator_chain(n=120, damping=0.02):
    from paper_2310_04734_b200 import mor
    main = 2.0 * np.ones(n)
    off = -np.ones(n - 1)
    K = sp.diags([off, main, off], [-1, 0, 1], format="csc") * 1e6 * (1 + 1j * damping)
    M = sp.identity(n, format="csc") * 1.0
    b = np.zeros(n)
    b[0] = 1.0
    c = np.zeros(n)
    c[-1] = 1.0
    return mor.FullOrderModel(stiffness=lambda f: K, mass=lambda f: M, load=lambda f: b, c_out=c, n=n)


def frozen_fom(n=200, seed=0, damping=0.02):
    from paper_2310_04734_b200 import mor
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, n))
    K = sp.csc_matrix((X @ X.T + n * np.eye(n)) * (1 + 1j * damping))
    Y = rng.standard_normal((n, n)) * 0.05
    M = sp.csc_matrix(Y @ Y.T + np.eye(n))
    b = rng.standard_normal(n)
    c = np.zeros(n)
    c[n // 3] = 1.0
    return mor.FullOrderModel(stiffness=lambda f: K, mass=lambda f: M, load=lambda f: b, c_out=c, n=n)


CASES = {
    "chain_tol1e-3": ("chain", (10.0, 120.0, 56), dict(tol=1e-3, max_points=15, candidate_stride=3), "greedy"),
    "chain_tol1e-4_budget10": ("chain", (10.0, 120.0, 56), dict(tol=1e-4, max_points=10, candidate_stride=3),
                               "greedy"),
    "chain_tol_inf": ("chain", (10.0, 60.0, 26), dict(tol=math.inf), "greedy"),
    "chain_two_windows": ("chain", (10.0, 120.0, 56),
                          dict(tol=1e-3, max_points=15, candidate_stride=3, windows=[(10.0, 60.0), (60.0, 120.0)]),
                          "local"),
    "chain_auto_bisect": ("chain", (10.0, 200.0, 96), dict(tol=1e-7, max_points=3, moments_per_point=2,
                                                           candidate_stride=3), "local"),
    "frozen_tol1e-6": ("frozen", (10.0, 100.0, 46), dict(tol=1e-6, max_points=8, moments_per_point=3,
                                                          candidate_stride=2), "greedy"),
}


@pytest.mark.parametrize("name", list(CASES))
def test_greedy_decisions_match_reference(cuda, golden_dir, name):
    from oracle import mor as omor
    from paper_2310_04734_b200 import mor
    z = np.load(golden_dir / "greedy_ref.npz")
    model, (g0, g1, ng), kw, entry = CASES[name]
    fom = oscillator_chain() if model == "chain" else frozen_fom()
    grid = list(np.linspace(g0, g1, ng))
    st = Settings(**kw)
    if entry == "greedy":
        roms = [mor.greedy_expand(fom, grid, st, (g0, g1))]
    else:
        roms = mor.build_local_roms(fom, grid, st, (g0, g1))
    nw = int(z[f"{name}__n_windows"])
    assert len(roms) == nw
    for k, r in enumerate(roms):
        assert tuple(r.window) == tuple(z[f"{name}__window{k}"]), k
        assert list(r.expansion_points) == list(z[f"{name}__points{k}"]), k
        assert r.r == int(z[f"{name}__r{k}"]), k
        assert [r.converged, r.stalled, r.budget_exhausted] == list(z[f"{name}__flags{k}"]), k
        ref_log = z[f"{name}__errlog{k}"]
        log = np.array(r.error_log)
        assert log.shape == ref_log.shape
        np.testing.assert_array_equal(log[:, 0], ref_log[:, 0])          # same candidates
        # candidate errors: the ROM outputs agree to ~1e-12 relative, so each
        # eps agrees to that absolute level (rounding-level eps included)
        assert np.all(np.abs(log[:, 1] - ref_log[:, 1]) <= 1e-9 + 1e-8 * np.abs(ref_log[:, 1])), k
    sw = mor.rom_sweep(roms, grid)
    assert sw.window_index == [int(w) for w in z[f"{name}__window_index"]]
    _, e, _, _ = omor.relative_error(z[f"{name}__frf"], np.array(sw.frf))
    assert e <= 1e-8, e
