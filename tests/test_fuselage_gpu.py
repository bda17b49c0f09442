"""Tier-0 parity gate: the reference's OWN benchmark model
(vibrofem/data/fuselage_slice.cfg, finest mesh level, n = 8,102; the model
`vibrofem mor` and tests/test_acceptance.py:86-94 build) through the GPU
drop-in, against outputs of the unmodified reference
(tests/golden/make_fuselage_golden.py -> fuselage_slice.npz).

The fixture carries the reference's primitives, couplings, block map, the
per-frequency scalars its ModelOperator computes, its load vectors, the V of
every window build_local_roms produced and the rom_sweep FRF.  The GPU side
reads the primitives as data (model_operator.affine_from_operator with the
tabulated scalars), projects them once and sweeps all 496 frequencies in one
launch per window."""

import types

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import mor as omor

pytestmark = pytest.mark.gpu
TF_TOL = 1e-8


def _csr(z, key):
    return sp.csr_matrix((z[f"{key}__data"], z[f"{key}__indices"], z[f"{key}__indptr"]),
                         shape=tuple(z[f"{key}__shape"]))


def fixture_operator(z):
    """A ModelOperator look-alike (the attributes affine_from_operator reads)
    plus tabulated coefficient callables and load, from the fixture."""
    from paper_2310_04734_b200.model_operator import OperatorCoefficients
    grid = z["grid"]
    pos = {float(f): i for i, f in enumerate(grid)}
    doms = [str(d) for d in z["domains"]]
    kinds = {d: str(k) for d, k in zip(doms, z["kinds"])}
    prims = {}
    for d in doms:
        names = ("Kmat", "Kgeo", "M") if kinds[d] == "elastic" else ("Kgrad", "Mnn")
        prims[d] = {nm: _csr(z, f"prim__{d}__{nm}") for nm in names}
    couplings = [(str(s), str(f), _csr(z, f"coupling{k}")) for k, (s, f) in enumerate(z["couplings"])]
    block_map = {d: tuple(int(v) for v in z["block_map"][i]) for i, d in enumerate(doms)}
    cfg = types.SimpleNamespace(domains=[types.SimpleNamespace(id=d, kind=kinds[d]) for d in doms])
    op = types.SimpleNamespace(config=cfg, kinds=kinds, primitives=prims, couplings=couplings,
                               block_map=block_map)
    coeffs = OperatorCoefficients(
        kscale=lambda d, f: complex(z[f"scale__{d}"][pos[float(f)]]),
        fluid=lambda d, f: (complex(z[f"rho_eff__{d}"][pos[float(f)]]), complex(z[f"c_eff__{d}"][pos[float(f)]])),
        rho_f=lambda k, f: complex(z[f"rho_f{k}"][pos[float(f)]]))
    n = int(z["n"])
    rows, vals = z["load_rows"], z["load_vals"]

    def load(f):
        v = np.zeros(n, complex)
        v[rows] = vals[pos[float(f)]]
        return v
    return op, coeffs, load


def _emb(A, r0, c0, n):
    E = sp.coo_matrix(A)
    return sp.csr_matrix((E.data, (E.row + r0, E.col + c0)), shape=(n, n))


@pytest.fixture(scope="module")
def fuselage(golden_dir, cuda):
    from paper_2310_04734_b200 import mor
    from paper_2310_04734_b200.model_operator import load_operator_npz
    z = dict(np.load(golden_dir / "fuselage_slice.npz"))
    fom, _, _ = load_operator_npz(golden_dir / "fuselage_slice.npz", cuda)
    roms = []
    for k in range(int(z["n_windows"])):
        fl = z[f"flags{k}"]
        roms.append(mor.ReducedModel(fom=fom, V=z[f"V{k}"], window=tuple(z["windows"][k]),
                                     expansion_points=list(z[f"points{k}"]),
                                     error_log=[tuple(e) for e in z[f"errlog{k}"]],
                                     converged=bool(fl[0]), stalled=bool(fl[1]), budget_exhausted=bool(fl[2])))
    return z, fom, roms


def test_fuselage_rom_sweep_matches_reference(fuselage):
    """rom_sweep over the benchmark's full 496-point grid with the reference's
    own bases: FRF relative error <= 1e-8 at every frequency, |dB| <= 0.01,
    same owner windows and seam log (mor.py:366-394)."""
    from paper_2310_04734_b200 import mor
    z, fom, roms = fuselage
    grid = [float(f) for f in z["grid"]]
    res = mor.rom_sweep(roms, grid)
    frf = np.array(res.frf)
    ref = z["frf"]
    assert frf.shape == ref.shape == (496,)
    eps, eps_max, k, _ = omor.relative_error(ref, frf)
    # 1e-8 (north_star), floored at twice the reference's own rounding
    # sensitivity at that frequency (fixture y_sens: the reference output's
    # change under 1-ulp perturbations of its reduced system; > 5e-9 only at
    # a few of the highest frequencies, where the reduced system is worst
    # conditioned)
    tol = np.maximum(TF_TOL, 2.0 * z["y_sens"])
    bad = np.nonzero(eps > tol)[0]
    assert bad.size == 0, [(grid[i], eps[i], z["y_sens"][i]) for i in bad]
    assert np.sum(eps > TF_TOL) <= np.sum(z["y_sens"] > 0.5 * TF_TOL)
    db = lambda y: 20 * np.log10(np.maximum(np.abs(y), 1e-300) / 20e-6)  # noqa: E731  (cli.py:273-278)
    assert np.abs(db(frf) - db(ref)).max() <= 0.01
    # mean_spl of the single probe output (solvers.py:334-338), fused in the sweep kernel
    spl_ref = np.array([omor.mean_spl(np.array([y])) for y in ref])
    assert np.abs(np.array(res.spl)[:, 0] - spl_ref).max() <= 0.01
    assert res.window_index == [int(w) for w in z["window_index"]]
    assert [f for f, _ in res.seam_log] == [float(f) for f in z["seam_f"]]
    for (_, g), gr in zip(res.seam_log, z["seam_gap"]):
        assert abs(g - gr) <= 1e-8 * max(abs(gr), abs(ref).max() * 1e-6)


def test_fuselage_fom_solve_matches_reference_splu(fuselage):
    """FullOrderModel.solve on the GPU (dense LU of the n = 8,102 coupled,
    non-symmetric operator + refinement against the device CSR primitives)
    equals the reference's splu output at the probe (mor.py:48-53)."""
    z, fom, _ = fuselage
    for f, yr in zip(z["fom_f"], z["fom_y"]):
        y = fom.output(fom.solve(float(f)))
        assert abs(y - yr) <= TF_TOL * abs(yr), (f, y, yr)


def test_fuselage_reduced_system_matches_literal_projection(fuselage):
    """The affine reduced operator sum_k alpha_k(f) V^H P_k V equals the
    reference's literal re-projection V^H (K(f) - w^2 M(f)) V (mor.py:73-90),
    rebuilt on the host from the fixture's primitives and scalars."""
    import math
    z, fom, roms = fuselage
    op, coeffs, load = fixture_operator(z)
    rom = roms[0]
    V = z["V0"]
    n = int(z["n"])
    for f in (float(z["grid"][3]), float(z["grid"][250])):
        Kf = sp.csr_matrix((n, n), dtype=complex)
        Mf = sp.csr_matrix((n, n), dtype=complex)
        for d in op.config.domains:
            o, s = op.block_map[d.id]
            P = op.primitives[d.id]
            if d.kind == "elastic":
                Kd = coeffs.kscale(d.id, f) * P["Kmat"] + P["Kgeo"]
                Md = P["M"]
            else:
                rho, c = coeffs.fluid(d.id, f)
                Kd = coeffs.kscale(d.id, f) / rho * P["Kgrad"]
                Md = P["Mnn"] / (rho * c * c)
            Kf = Kf + _emb(Kd, o, o, n)
            Mf = Mf + _emb(Md, o, o, n)
        for k, (sid, fid, C) in enumerate(op.couplings):
            so, ss = op.block_map[sid]
            fo, fs = op.block_map[fid]
            E = sp.coo_matrix(C)
            Kf = Kf + sp.csr_matrix((-E.data, (E.row + so, E.col + fo)), shape=(n, n))
            Mf = Mf + sp.csr_matrix((coeffs.rho_f(k, f) * E.data, (E.col + fo, E.row + so)), shape=(n, n))
        w = 2 * math.pi * f
        AR_ref = V.conj().T @ ((Kf - w * w * Mf) @ V)
        AR, bR = rom.reduced_system(f)
        assert np.abs(AR - AR_ref).max() <= 1e-10 * np.abs(AR_ref).max()
        assert np.abs(bR - V.conj().T @ load(f)).max() <= 1e-12 * np.abs(bR).max()


class _MorSettings:
    """fuselage_slice.cfg `mor:` block (config.py:172-184 MorSettings)."""
    tol, max_points, moments_per_point, candidate_stride, windows = 1e-2, 20, 4, 4, "auto"


def test_fuselage_build_local_roms_matches_reference(fuselage):
    """The whole offline phase on the reference's benchmark through the drop-in:
    build_local_roms (mor.py:322-353: greedy expansion, auto windows) takes the
    reference's decisions — same windows, expansion points in order, r, flags
    and candidate error log — with every FOM solve a GPU LU and every
    candidate ROM evaluation batched (reference: 183.6 s on 8 cores)."""
    import time
    import torch
    from paper_2310_04734_b200 import mor
    z, fom, _ = fuselage
    grid = [float(f) for f in z["grid"]]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    roms = mor.build_local_roms(fom, grid, _MorSettings(), (grid[0], grid[-1]))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"GPU build_local_roms on the reference benchmark: {dt:.2f} s "
          f"(reference {float(z['build_s']):.1f} s)")
    assert len(roms) == int(z["n_windows"])
    for k, r in enumerate(roms):
        assert tuple(r.window) == tuple(z["windows"][k])
        assert [float(p) for p in r.expansion_points] == [float(p) for p in z[f"points{k}"]]
        assert r.r == z[f"V{k}"].shape[1]
        assert [r.converged, r.stalled, r.budget_exhausted] == list(z[f"flags{k}"])
        log, ref = np.array(r.error_log), z[f"errlog{k}"]
        np.testing.assert_array_equal(log[:, 0], ref[:, 0])
        # eps = |y_full - y_rom| / |y_full| is the ROM's own truncation error;
        # the late Krylov columns of a window are nearly dependent moment
        # vectors, determined by the data only to ~1e-7, so two
        # correct builds (splu + MGS2 vs GPU LU + CGS2) give ROMs whose errors
        # agree to a fraction of eps (measured <= 40 %), not to rounding.  The
        # reference is itself this sensitive: rebuilt with its primitives
        # perturbed by 1 ulp it changes its error log by up to 2.9e-3 and
        # even its expansion points (fixture errlog_sens0,
        # errlog_sens_same_decisions = False).  The decisions above are what
        # the candidate errors drive, and they are identical; the sweep with
        # the reference's OWN bases matches to 1e-8
        # (test_fuselage_rom_sweep_matches_reference).
        assert not bool(z["errlog_sens_same_decisions"])
        d = np.abs(log[:, 1] - ref[:, 1])
        bad = d > 5e-8 + 0.5 * np.abs(ref[:, 1])
        assert not bad.any(), list(zip(ref[bad, 0], ref[bad, 1], d[bad]))
