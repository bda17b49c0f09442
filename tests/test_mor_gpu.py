"""GPU MOR pipeline (paper_2310_04734_b200.mor) against the unmodified reference
(golden fixtures) and the oracle restatement: Krylov blocks, MGS2/drop rule,
ROM outputs, rom_sweep tie rule, greedy expansion, and cfg1 end to end."""

import math
from dataclasses import dataclass

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fe, mor as omor

pytestmark = pytest.mark.gpu
TF_TOL = 1e-8


@dataclass
class Settings:
    tol: float = 1e-2
    max_points: int = 20
    moments_per_point: int = 4
    candidate_stride: int = 4
    windows: object = "auto"


@pytest.fixture(scope="module")
def frozen(golden_dir):
    from paper_2310_04734_b200 import mor
    z = np.load(golden_dir / "frozen_fom.npz")
    K, M, b, c = sp.csc_matrix(z["K"]), sp.csc_matrix(z["M"]), z["b"], z["c"]
    fom = mor.FullOrderModel(stiffness=lambda f: K, mass=lambda f: M, load=lambda f: b, c_out=c, n=len(b))
    return z, fom


def test_krylov_and_orthonormalise_match_reference(cuda, frozen):
    from paper_2310_04734_b200 import mor
    z, fom = frozen
    Q1, br = mor.krylov_block(fom, 35.0, 5)
    assert not br and Q1.shape == (60, 5)
    np.testing.assert_allclose(Q1, z["Q1"], atol=1e-11)
    Q2, _ = mor.krylov_block(fom, 55.0, 4)
    np.testing.assert_allclose(Q2, z["Q2"], atol=1e-11)
    V = mor._orthonormalise(Q1, Q2)
    # same drop decisions (residual ratios 4e-16, 1.3e-12 | 3.4e-9, 2.9e-9 vs the
    # 1e-10 threshold) and an orthonormal basis; the two kept columns are
    # determined only to ~1e-7 by the data (near-dependent moment blocks), so
    # the basis is compared through what it is used for: the ROM outputs.
    assert V.shape == z["V"].shape
    np.testing.assert_allclose(V[:, :5], z["V"][:, :5], atol=1e-11)
    assert np.abs(V.conj().T @ V - np.eye(V.shape[1])).max() <= 1e-12
    rom = mor.ReducedModel(fom=fom, V=V, window=(10.0, 100.0))
    ys = rom.outputs(list(z["freqs"]))
    for y, yr in zip(ys, z["y_rom"]):
        assert abs(y - yr) <= 1e-8 * abs(yr)


def test_drop_rule_matches_reference(cuda, golden_dir):
    from paper_2310_04734_b200 import mor
    z = np.load(golden_dir / "frozen_fom.npz")
    Q = mor._orthonormalise(None, z["drop_block"])
    assert Q.shape == (30, 2)
    np.testing.assert_allclose(Q, z["drop_Q"], atol=1e-12)


def test_rom_and_fom_outputs_match_reference(cuda, frozen):
    from paper_2310_04734_b200 import mor
    z, fom = frozen
    rom = mor.ReducedModel(fom=fom, V=z["V"], window=(10.0, 100.0))
    for f, yr, yf in zip(z["freqs"], z["y_rom"], z["y_fom"]):
        assert abs(rom.output(f) - yr) <= 1e-10 * abs(yr)
        assert abs(fom.output(fom.solve(f)) - yf) <= 1e-10 * abs(yf)
    ys = rom.outputs(list(z["freqs"]))
    np.testing.assert_allclose(ys, z["y_rom"], rtol=1e-10)


def test_single_moment_exact_at_expansion_point(cuda, frozen):
    """tests/test_mor.py:55-66 on the GPU path."""
    from paper_2310_04734_b200 import mor
    _, fom = frozen
    Q, br = mor.krylov_block(fom, 40.0, 1)
    x = fom.solve(40.0)
    xd = x / np.linalg.norm(x)
    assert min(np.linalg.norm(Q[:, 0] - xd), np.linalg.norm(Q[:, 0] + xd)) <= 1e-10
    rom = mor.ReducedModel(fom=fom, V=Q, window=(30.0, 50.0))
    assert abs(rom.output(40.0) - fom.output(x)) <= 1e-10 * abs(fom.output(x))


def test_identity_basis_reproduces_fom(cuda, frozen):
    """tests/test_mor.py:119-125."""
    from paper_2310_04734_b200 import mor
    _, fom = frozen
    rom = mor.ReducedModel(fom=fom, V=np.eye(60, dtype=complex), window=(10.0, 100.0))
    for f in (12.0, 47.0, 93.0):
        yf = fom.output(fom.solve(f))
        assert abs(rom.output(f) - yf) <= 1e-11 * abs(yf)


def test_moment_matching(cuda, frozen):
    """tests/test_mor.py:76-106: the projected model reproduces 5 shifted moments."""
    from paper_2310_04734_b200 import mor
    _, fom = frozen
    f0, m = 35.0, 5
    Q, _ = mor.krylov_block(fom, f0, m)
    At = fom.operator(f0).toarray()
    Md = fom.mass(f0).toarray()
    b = fom.load(f0)
    v = np.linalg.solve(At, b)
    mom_full = []
    for _ in range(m):
        mom_full.append(fom.c_out @ v)
        v = np.linalg.solve(At, Md @ v)
    Vh = Q.conj().T
    AtR, MR, bR, cR = Vh @ At @ Q, Vh @ Md @ Q, Vh @ b, fom.c_out @ Q
    vr = np.linalg.solve(AtR, bR)
    for j in range(m):
        mr = cR @ vr
        assert abs(mom_full[j] - mr) <= 1e-8 * max(abs(mom_full[j]), 1e-30), j
        vr = np.linalg.solve(AtR, MR @ vr)


def _box_fom_gpu(z):
    import torch
    from paper_2310_04734_b200 import assembly, mor
    box, ne = (0.0, 0.0, 0.0, 0.6, 0.4, 0.3), (3, 2, 2)
    xyz, conn = assembly.hex27_box(box, *ne)
    Kg, Mn = assembly.assemble_helmholtz(xyz, conn)
    F = assembly.assemble_face_mass(xyz, assembly.hex27_box_face(ne, "z0", conn))
    rho, c = 1.21, 343.0
    n = Kg.n
    C = np.zeros((len(z["rec"]), n))
    C[np.arange(len(z["rec"])), z["rec"]] = 1.0
    aff = mor.AffineOperator(K=[mor.AffineTerm(Kg, 1 / rho)], M=[mor.AffineTerm(Mn, 1 / (rho * c * c))],
                             D=[mor.AffineTerm(F, 1 / (rho * c * (5 + 1j)))],
                             load=torch.as_tensor(z["b"], device="cuda"))
    return mor.FullOrderModel(c_out=C, n=n, affine=aff)


def test_box_mor_pipeline_matches_reference(cuda, golden_dir):
    """Reference second-order Krylov + _orthonormalise + 2 windows + rom_sweep
    (tie rule, seam log) + mean_spl on the restated hex27 box (box_mor.npz)."""
    from paper_2310_04734_b200 import mor
    z = np.load(golden_dir / "box_mor.npz")
    fom = _box_fom_gpu(z)
    V = None
    for f0 in z["points"]:
        Q, _ = mor.krylov_block_dev(fom, f0, 4, second_order=True)
        V = mor._orthonormalise(V, Q)
    Vh = V.cpu().numpy()
    assert Vh.shape == z["V"].shape
    assert np.abs(Vh.conj().T @ Vh - np.eye(Vh.shape[1])).max() <= 1e-12
    roms = [mor.ReducedModel(fom=fom, V=V[:, :6].contiguous(), window=(600.0, 1000.0)),
            mor.ReducedModel(fom=fom, V=V, window=(200.0, 600.0))]
    res = mor.rom_sweep(roms, list(z["grid"]))
    np.testing.assert_array_equal(res.window_index, z["window_index"])
    # TF_TOL, floored at twice the reference's own rounding sensitivity at that
    # frequency (y_sens: the reference pipeline rerun on ~1-ulp perturbed K, M;
    # 1.3e-8 at 950 Hz, <= 2.4e-9 everywhere else — make_golden.gold_box_mor)
    for i in range(len(z["grid"])):
        _, e, _, _ = mor.relative_error(z["y"][i], res.frf[i])
        assert e <= max(TF_TOL, 2.0 * z["y_sens"][i]), (i, e, z["y_sens"][i])
        assert abs(res.spl[i][0] - z["spl"][i]) <= 0.01
    assert [s[0] for s in res.seam_log] == list(z["seam_f"])
    np.testing.assert_allclose([np.max(s[1]) for s in res.seam_log], z["seam_gap"], rtol=1e-6)
    # full-order GPU solves reproduce the reference splu outputs
    for i in (0, 7, 16):
        y = fom.output(fom.solve(z["grid"][i]))
        _, e, _, _ = mor.relative_error(z["y_fom"][i], y)
        assert e <= 1e-10


def oscillator_chain(n=120, damping=0.02):
    """tests/test_mor.py:40-52."""
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


def test_greedy_converges_on_oscillator_chain(cuda):
    """tests/test_mor.py:148-160 on the GPU path."""
    from paper_2310_04734_b200 import mor
    fom = oscillator_chain()
    grid = list(np.linspace(10.0, 120.0, 56))
    settings = Settings(tol=1e-3, max_points=15, moments_per_point=4, candidate_stride=3)
    rom = mor.greedy_expand(fom, grid, settings, (10.0, 120.0))
    assert rom.converged
    assert rom.r <= settings.max_points * settings.moments_per_point
    cand = set(mor.candidate_frequencies(grid, (10.0, 120.0), 3))
    others = [f for f in grid if f not in cand]
    y_full = np.array([fom.output(fom.solve(f)) for f in others])
    y_red = np.array(rom.outputs(others))
    _, eps_max, _, _ = mor.relative_error(y_full, y_red)
    assert eps_max <= 1e-2


def test_local_roms_tie_rule_and_seam(cuda):
    """tests/test_mor.py:180-197 on the GPU path."""
    from paper_2310_04734_b200 import mor
    fom = oscillator_chain()
    grid = list(np.linspace(10.0, 120.0, 56))
    settings = Settings(tol=1e-3, max_points=15, candidate_stride=3, windows=[(10.0, 60.0), (60.0, 120.0)])
    roms = mor.build_local_roms(fom, grid, settings, (10.0, 120.0))
    assert [r.window for r in roms] == [(10.0, 60.0), (60.0, 120.0)]
    sw = mor.rom_sweep(roms, grid)
    assert sw.freqs == grid
    assert sw.window_index[grid.index(60.0)] == 0
    assert len(sw.seam_log) == 1 and sw.seam_log[0][0] == 60.0
    y_ref = abs(fom.output(fom.solve(60.0)))
    assert sw.seam_log[0][1] <= 2 * settings.tol * y_ref
    with pytest.raises(ValueError):
        mor.rom_sweep(roms, [200.0])


@pytest.mark.parametrize("fdm", [False, True])
def test_cfg1_end_to_end_matches_oracle(cuda, fdm):
    """cfg1 (n = 4641, 4 points x 8 moments, second order, 50 receivers, 181
    frequencies): GPU assembly -> GPU LU (or the box FDM solver) -> Krylov ->
    CGS2 -> projection -> batched sweep -> SPL, against the oracle running the
    reference algorithm (splu, MGS2, literal per-frequency re-projection, zgesv)
    on the oracle's own assembly of the same box."""
    from paper_2310_04734_b200 import mor, workloads
    fom, lay = workloads.cfg1_model(fdm=fdm)
    V = None
    for f0 in lay["points"]:
        Q, _ = mor.krylov_block_dev(fom, f0, lay["moments"], second_order=True)
        V = mor._orthonormalise(V, Q)
    assert V.shape[1] == 32
    rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 200.0))
    res = mor.rom_sweep([rom], list(lay["freqs"]))
    # oracle
    nodes, elems = fe.structured_hex27(workloads.CFG1_BOX, *workloads.CFG1_NE)
    Kg, Mn = fe.assemble_helmholtz(nodes, elems, fe.HEX27_IDX)
    el, loc = fe.hex27_face(workloads.CFG1_NE, "z0")
    Fz = fe.face_mass_hex27(nodes, elems, el, loc)
    rho, c = workloads.AIR_RHO, workloads.AIR_C
    K, M, D = (Kg / rho).astype(complex), (Mn / (rho * c * c)).astype(complex), Fz / workloads.CFG1_Z
    n = K.shape[0]
    b = np.zeros(n, complex)
    b[lay["src"]] = 1.0
    C = np.zeros((len(lay["rec"]), n))
    C[np.arange(len(lay["rec"])), lay["rec"]] = 1.0
    ofom = omor.Fom(stiffness=lambda f: K, mass=lambda f: M, load=lambda f: b, c_out=C, n=n,
                    damping=lambda f: D)
    Vo = None
    for f0 in lay["points"]:
        Qo, _ = omor.krylov_block(ofom, f0, lay["moments"], second_order=True)
        Vo = omor.orthonormalise(Vo, Qo)
    assert Vo.shape[1] == 32
    worst, worst_spl = 0.0, 0.0
    for i, f in enumerate(lay["freqs"]):  # the full 181-point grid
        yo = omor.reduced_output(ofom, Vo, f)
        _, e, _, _ = omor.relative_error(yo, res.frf[i])
        worst = max(worst, e)
        worst_spl = max(worst_spl, abs(omor.mean_spl(yo) - res.spl[i][0]))
    assert worst <= TF_TOL, worst
    assert worst_spl <= 0.01


@pytest.mark.parametrize("model", ["cfg1", "cfg2"])
def test_concurrent_krylov_matches_sequential(cuda, model):
    """krylov_blocks_concurrent (each expansion point on its own stream / host
    thread, LU kernels on a share of the SMs) returns the blocks of the
    sequential krylov_block_dev loop (mor.py:138-191 per point)."""
    import torch
    from paper_2310_04734_b200 import mor, workloads
    if model == "cfg1":
        fom, lay = workloads.cfg1_model()
        pts, m, so = lay["points"], lay["moments"], True
    else:
        fom, lay = workloads.cfg2_model()
        pts, m, so = lay["points"][:3], 4, False
    seq = [mor.krylov_block_dev(fom, f, m, second_order=so) for f in pts]
    conc = mor.krylov_blocks_concurrent(fom, pts, m, second_order=so)
    # the capped concurrent grid runs the plain LU kernel, the full grid the
    # look-ahead one: same pivots, factors equal to ~1e-13; the moment
    # recurrence amplifies that (cfg2's coupled operator: cond ~1e12) to
    # ~1e-10 in the last moments
    for (Qs, bs), (Qc, bc) in zip(seq, conc):
        assert bs == bc and Qs.shape == Qc.shape
        assert float((Qs - Qc).abs().max()) <= 1e-9
    V, flags = mor.krylov_basis(fom, pts, m, second_order=so)
    Vs = None
    for Q, _ in seq:
        Vs = mor._orthonormalise(Vs, Q)
    assert V.shape == Vs.shape
    # the late columns are nearly dependent moment vectors, determined only to
    # ~1e-7 by the data: the two bases span the same subspace
    # to that level (outputs of an unconverged r = 12 ROM near its own
    # resonances are too sensitive to compare)
    R = Vs - V @ (V.conj().T @ Vs)
    assert float(R.abs().max()) <= 1e-6, float(R.abs().max())


def test_project_lift_and_c_out_reduced(cuda, frozen):
    """project (mor.py:112-119), ReducedModel.lift (104-105) and c_out_reduced
    (100-102) against their numpy definitions, for a provider model (sparse
    providers uploaded as device CSR, no dense n x n) and for an affine one
    (sum_k alpha_k V^H P_k V)."""
    from paper_2310_04734_b200 import mor
    z, fom = frozen
    K, M, b, c = sp.csc_matrix(z["K"]), sp.csc_matrix(z["M"]), z["b"], z["c"]
    rng = np.random.default_rng(4)
    V = np.linalg.qr(rng.standard_normal((60, 7)) + 1j * rng.standard_normal((60, 7)))[0]
    f = 47.5
    w = 2 * math.pi * f
    AR_ref = V.conj().T @ ((K - w * w * M) @ V)
    bR_ref = V.conj().T @ b
    AR, bR = mor.project(fom, V, f)
    assert np.abs(AR - AR_ref).max() <= 1e-12 * np.abs(AR_ref).max()
    assert bR.shape == bR_ref.shape and np.abs(bR - bR_ref).max() <= 1e-12 * np.abs(bR_ref).max()
    with pytest.raises(ValueError):
        mor.project(fom, V[:50], f)
    rom = mor.ReducedModel(fom=fom, V=V, window=(10.0, 100.0))
    xr = rng.standard_normal(7) + 1j * rng.standard_normal(7)
    x = rom.lift(xr)
    assert x.shape == (60,) and np.abs(x - V @ xr).max() <= 1e-13
    X = rom.lift(np.stack([xr, 2 * xr], 1))
    assert X.shape == (60, 2)
    cr = rom.c_out_reduced
    assert cr.shape == (7,) and np.abs(cr - c @ V).max() <= 1e-14
    # the same through the affine description (K, M as real CSR primitives)
    import torch
    from paper_2310_04734_b200.model_operator import device_csr_terms
    Kt = [mor.AffineTerm(P, fac) for P, fac in device_csr_terms(K, cuda)]
    Mt = [mor.AffineTerm(P, fac) for P, fac in device_csr_terms(M, cuda)]
    afom = mor.FullOrderModel(c_out=c, n=60, affine=mor.AffineOperator(K=Kt, M=Mt, load=torch.as_tensor(b)))
    AR2, bR2 = mor.project(afom, V, f)
    assert np.abs(AR2 - AR_ref).max() <= 1e-12 * np.abs(AR_ref).max()
    assert np.abs(bR2 - bR_ref).max() <= 1e-12 * np.abs(bR_ref).max()
