"""cfg2 plate-cavity model: GPU Reissner-Mindlin elements, constrained /
rectangular CSR builder, coupling and plane-wave load vs the oracle
restatement; full-order and MOR chain at reduced size vs the oracle; full
cfg2 size residual and ROM checks."""

import math

import numpy as np
import pytest

from oracle import mor as omor, shell

pytestmark = pytest.mark.gpu
SMALL = ((0.0, 0.0, 0.0, 0.8, 0.6, 0.5), (4, 3, 3))


def test_plate_element_matches_oracle(cuda):
    import torch
    from paper_2310_04734_b200 import plate
    P = dict(E=60e9, nu=0.3, rho=1550.0, t=0.003)
    xyz, conn = plate.plate_mesh((0.1, 0.2, 0.35, 0.3), 1, 1, 0.5)
    Ke, Me = plate.plate_elements(torch.as_tensor(xyz, device=cuda), torch.as_tensor(conn, device=cuda), **P)
    Kr, Mr = shell.plate_element(P["E"], P["nu"], P["rho"], P["t"], xyz[conn[0]][:, :2])
    np.testing.assert_allclose(Ke[0].cpu().numpy(), Kr, rtol=0, atol=1e-12 * np.abs(Kr).max())
    np.testing.assert_allclose(Me[0].cpu().numpy(), Mr, rtol=0, atol=1e-12 * np.abs(Mr).max())


def _small(cuda):
    from paper_2310_04734_b200 import workloads
    box, ne = SMALL
    fom, lay = workloads.cfg2_model(box=box, ne=ne, n_rec=12)
    P = workloads.CFG2_PLATE
    prims = shell.cfg2_primitives(box, ne, P["E"], P["nu"], P["rho"], P["t"], workloads.AIR_RHO, workloads.AIR_C,
                                  workloads.CFG2_THETA)
    return fom, lay, prims


def test_cfg2_primitives_match_oracle(cuda):
    fom, lay, prims = _small(cuda)
    for name in ("Kg", "Mn", "Kp", "Mp", "Fsf", "Ffs"):
        G, R = lay[name].to_scipy(), prims[name]
        np.testing.assert_array_equal(G.indptr, R.indptr, err_msg=name)     # bit-exact pattern
        np.testing.assert_array_equal(G.indices, R.indices, err_msg=name)
        np.testing.assert_allclose(G.data, R.data, rtol=0, atol=1e-12 * np.abs(R.data).max(), err_msg=name)
    for f in (37.0, 401.5):
        np.testing.assert_allclose(lay["load"].host(f), prims["load"](f), rtol=0, atol=1e-14)
        np.testing.assert_allclose(lay["load"].at(f).cpu().numpy()[:, 0], prims["load"](f), rtol=0, atol=1e-14)


def test_cfg2_full_size_primitives_match_oracle(cuda):
    """BASELINE cfg2 size (16 x 12 plate, 16 x 12 x 10 cavity, n = 20,890): all
    six primitives' CSR indptr/indices bit-identical to the oracle's
    coo -> csr -> sum_duplicates of the same triplets, values to rounding."""
    from paper_2310_04734_b200 import workloads
    fom, lay = workloads.cfg2_model(use_schur=False)
    P = workloads.CFG2_PLATE
    prims = shell.cfg2_primitives(workloads.CFG2_BOX, workloads.CFG2_NE, P["E"], P["nu"], P["rho"], P["t"],
                                  workloads.AIR_RHO, workloads.AIR_C, workloads.CFG2_THETA)
    assert fom.n == prims["n"] == 20_890
    for name in ("Kg", "Mn", "Kp", "Mp", "Fsf", "Ffs"):
        G, R = lay[name].to_scipy(), prims[name]
        np.testing.assert_array_equal(G.indptr, R.indptr, err_msg=name)
        np.testing.assert_array_equal(G.indices, R.indices, err_msg=name)
        np.testing.assert_allclose(G.data, R.data, rtol=0, atol=1e-12 * np.abs(R.data).max(), err_msg=name)


def test_cfg2_small_chain_matches_oracle(cuda):
    """Stage-by-stage parity on identical inputs (the coupled operator has
    cond ~ 2e12, so an unconverged ROM's output is rounding-sensitive to the
    basis itself; each stage is therefore compared on the same inputs):
    FOM outputs, Krylov spans, and the GPU sweep vs the oracle's literal
    per-frequency re-projection + zgesv on the GPU basis (TF <= 1e-8)."""
    from paper_2310_04734_b200 import mor, plate, workloads
    fom, lay, prims = _small(cuda)
    ofom = shell.cfg2_fom(prims, lay["rec"], workloads.AIR_RHO, workloads.AIR_C, plate.eta_cfg2)
    for f in (55.0, 333.0):
        yg = fom.output(fom.solve(f))
        yo = ofom.output(ofom.solve(f))
        _, e, _, _ = omor.relative_error(yo, yg)
        assert e <= 1e-8, e
    pts, m = (60.0, 220.0, 380.0), 4
    V = None
    for f0 in pts:
        Q, _ = mor.krylov_block_dev(fom, f0, m)
        Qo, _ = omor.krylov_block(ofom, f0, m)
        Qh = Q.cpu().numpy()
        assert np.linalg.norm(Qo - Qh @ (Qh.conj().T @ Qo)) <= 1e-8
        V = mor._orthonormalise(V, Q)
    Vh = V.cpu().numpy()
    rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 500.0))
    grid = list(np.arange(20.0, 500.1, 40.0))
    res = mor.rom_sweep([rom], grid)
    # the oracle's own rounding sensitivity on these inputs: the same reduction
    # with V perturbed by ~1 ulp (2 seeded trials); near the coupled system's
    # resonances it reaches the 1e-8 level (cond(A) ~ 2e12), so the tolerance is
    # floored at 4x that noise
    rng = np.random.default_rng(0)
    Vp = [Vh * (1 + 2.2e-16 * (rng.standard_normal(Vh.shape) + 1j * rng.standard_normal(Vh.shape)))
          for _ in range(2)]
    for i, f in enumerate(grid):
        yo = omor.reduced_output(ofom, Vh, f)
        sens = max(omor.relative_error(yo, omor.reduced_output(ofom, V2, f))[1] for V2 in Vp)
        _, e, _, _ = omor.relative_error(yo, res.frf[i])
        assert e <= max(1e-8, 4.0 * sens), (f, e, sens)
        assert abs(omor.mean_spl(yo) - res.spl[i][0]) <= 0.01
    # moment matching: the ROM reproduces the FOM at the expansion points, to the
    # accuracy the unscaled coupled operator allows (cond(A) ~ 2e12: measured
    # 3e-7 with the GPU basis, 3e-9 with the oracle's)
    for f0 in pts:
        _, e, _, _ = omor.relative_error(ofom.output(ofom.solve(f0)), rom.output(f0))
        assert e <= 1e-6, (f0, e)


def test_clamped_plate_fundamental(cuda):
    """Uncoupled clamped 0.8 x 0.6 x 0.003 m plate: first mode 71.65 Hz (16 x 12
    RM mesh; converged to 3e-5 against 32 x 24; Leissa C-C-C-C ~72 Hz)."""
    import scipy.linalg as sla
    from paper_2310_04734_b200 import workloads
    fom, lay = workloads.cfg2_model()
    n_p = lay["n_plate"]
    K = lay["Kp"].to_scipy()[:n_p, :n_p].toarray()
    M = lay["Mp"].to_scipy()[:n_p, :n_p].toarray()
    w2 = sla.eigh(K, M, eigvals_only=True, subset_by_index=[0, 2])
    f = np.sqrt(w2) / (2 * math.pi)
    assert abs(f[0] - 71.65) <= 0.05
    assert 70.0 <= f[0] <= 74.0


def test_cfg2_full_size_fom_and_rom(cuda):
    """n = 20,890 coupled non-symmetric system: GPU dense LU residual <= 1e-10
    (host check), and the r = 60 ROM certified against full-order solves."""
    import torch
    from paper_2310_04734_b200 import mor, workloads
    fom, lay = workloads.cfg2_model()
    assert fom.n == 20_890
    f = 143.5
    lu = fom.factor(f)
    b = fom.load_dev(f)
    x = lu.solve(b).cpu().numpy()[:, 0]
    A = fom.operator(f)
    bh = lay["load"].host(f)
    assert np.linalg.norm(A @ x - bh) / np.linalg.norm(bh) <= 1e-10
    V, _ = mor.krylov_basis(fom, lay["points"], lay["moments"])
    assert V.shape[1] == 60
    rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 500.0))
    grid = list(lay["freqs"])
    res = mor.rom_sweep([rom], grid)
    assert len(res.spl) == 961
    # the GPU sweep of all 961 frequencies == the oracle's zgesv on the same
    # reduced operator (frequency-dependent plane-wave b_r), TF <= 1e-8
    P, kinds, _ = rom._projected()
    alpha = rom._alpha(np.array(grid), kinds)
    br = rom._br(grid).cpu().numpy()
    Ph, cR = P.cpu().numpy(), rom._cR.cpu().numpy()
    yo, splo = omor.affine_sweep(Ph, alpha, br, cR)
    yg = np.array([np.atleast_1d(y) for y in res.frf])
    # the reduced coupled operator inherits the coupled system's scaling
    # (cond ~1e10 across much of the band, so zgesv itself is determined only
    # to ~1e-8..1e-6 there):
    # floor the 1e-8 tolerance at 16x the oracle's own change under 1-ulp
    # elementwise perturbations of A_r (4 seeded trials per frequency; an LU
    # solve's backward error is ~r eps ||L|| ||U||, i.e. up to O(r) such ulps)
    rng = np.random.default_rng(1)
    for i in range(len(grid)):
        A = np.tensordot(alpha[i], Ph, 1)
        sens = 0.0
        for _ in range(4):
            E = 2.2e-16 * (rng.standard_normal(A.shape) + 1j * rng.standard_normal(A.shape))
            y1 = cR @ np.linalg.solve(A * (1 + E), br[i])
            sens = max(sens, omor.relative_error(yo[i].ravel(), y1.ravel())[1])
        e = omor.relative_error(yo[i].ravel(), yg[i].ravel())[1]
        assert e <= max(1e-8, 16.0 * sens), (grid[i], e, sens)
    assert np.abs(np.array(res.spl)[:, 0] - splo[:, 0]).max() <= 0.01
    # certification at the reference tolerance on a grid disjoint from the
    # expansion points (tests/test_acceptance.py:272-305: eps_max <= 1e-2),
    # pointwise over all 50 receivers (mor.py:194-208)
    ver = [i for i in range(0, len(grid), 9) if grid[i] not in lay["points"]]
    worst = 0.0
    for i in ver:
        yf = fom.output(fom.solve(grid[i]))
        _, e, _, _ = mor.relative_error(yf, res.frf[i])
        worst = max(worst, e)
    assert len(ver) >= 100 and worst <= 1e-2, worst


def test_cfg2_schur_solver_matches_dense_lu(cuda):
    """Schur complement on the plate + fast-diagonalisation cavity == the dense
    whole-system LU (both refined to ||b - A x|| / ||b|| <= 1e-10)."""
    import torch
    from paper_2310_04734_b200 import workloads
    box, ne = SMALL
    fom_s, lay = workloads.cfg2_model(box=box, ne=ne, n_rec=12)
    fom_d, _ = workloads.cfg2_model(box=box, ne=ne, n_rec=12, use_schur=False)
    assert fom_s.schur is not None and fom_d.schur is None
    g = torch.Generator(device="cuda").manual_seed(5)
    B = torch.randn(fom_s.n, 3, dtype=torch.complex128, device="cuda", generator=g)
    for f in (33.0, 250.0, 487.5):
        fs, fd = fom_s.factor(f), fom_d.factor(f)
        Xs, Xd = fs.solve(B), fd.solve(B)
        assert fs.last_residual <= 1e-10 and fd.last_residual <= 1e-10
        rel = float((Xs - Xd).abs().max() / Xd.abs().max())
        assert rel <= 1e-8, (f, rel)
