"""Tier-0 parity fixture: the UNMODIFIED reference on its own bundled benchmark
(`vibrofem/data/fuselage_slice.cfg`, finest mesh level, n = 8,102), the model
`vibrofem mor build/sweep` runs (cli.py:211-218, 251-282) and the reference's
`benchmark_roms` acceptance fixture builds (tests/test_acceptance.py:86-94).

Run in the build container (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fuselage_golden.py

Writes tests/golden/fuselage_slice.npz holding, all produced by reference code:
  * the frequency-independent primitives of every domain (assembly.py:142-175)
    and the coupling matrices (mortar.py:183-197), block map, domain kinds;
  * per grid frequency the scalars ModelOperator._domain_KM / system use
    (assembly.py:242-257, 262-265): complex_stiffness_scale per elastic
    domain, (rho_eff, c_eff) per fluid domain, rho_f per coupling;
  * the load op.load(f) on the grid (nonzero rows only; plane_wave_load);
  * build_local_roms (mor.py:322-353): windows, V per window, expansion
    points, error logs, flags;
  * rom_sweep (mor.py:366-394) over the 496-point grid: FRF, owner window,
    seam log; the probe output of FullOrderModel.solve (splu) at a few
    frequencies;
  * the build / sweep wall times (reference CPU baseline on this container).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np
import scipy.sparse as sp

HERE = Path(__file__).resolve().parent

import vibrofem  # noqa: E402  (reference)
from vibrofem import materials as rmats  # noqa: E402
from vibrofem import mor as rmor  # noqa: E402
from vibrofem.assembly import fluid_density  # noqa: E402
from vibrofem.cli import _mor_fom  # noqa: E402
from vibrofem.config import frequency_grid, load_config  # noqa: E402


def main(out=HERE / "fuselage_slice.npz"):
    cfg = load_config(Path(vibrofem.__file__).parent / "data" / "fuselage_slice.cfg")
    fom, op = _mor_fom(cfg)
    grid = frequency_grid(cfg.frequency)
    band = (cfg.frequency.f_min, cfg.frequency.f_max)
    pay = {"n": np.array(fom.n), "grid": np.array(grid), "probe": np.array(int(np.argmax(fom.c_out)))}
    order = [d.id for d in cfg.domains]
    pay["domains"] = np.array(order)
    pay["kinds"] = np.array([op.kinds[d] for d in order])
    pay["block_map"] = np.array([op.block_map[d] for d in order], dtype=np.int64)
    for d in order:
        for name, A in op.primitives[d].items():
            A = sp.csr_matrix(A)
            pay[f"prim__{d}__{name}__data"] = A.data
            pay[f"prim__{d}__{name}__indices"] = A.indices.astype(np.int32)
            pay[f"prim__{d}__{name}__indptr"] = A.indptr.astype(np.int32)
            pay[f"prim__{d}__{name}__shape"] = np.array(A.shape)
    pay["couplings"] = np.array([[sid, fid] for sid, fid, _ in op.couplings])
    for k, (_, _, C) in enumerate(op.couplings):
        C = sp.csr_matrix(C)
        pay[f"coupling{k}__data"] = C.data
        pay[f"coupling{k}__indices"] = C.indices.astype(np.int32)
        pay[f"coupling{k}__indptr"] = C.indptr.astype(np.int32)
        pay[f"coupling{k}__shape"] = np.array(C.shape)
    # per-frequency scalars exactly as _domain_KM / system compute them
    for d in cfg.domains:
        mat = cfg.materials[d.material_id]
        table = cfg.damping_tables.get(d.damping_table_id)
        pay[f"scale__{d.id}"] = np.array([rmats.complex_stiffness_scale(table, f) if table else 1.0 + 0j
                                          for f in grid])
        if d.kind != "elastic":
            rc = [rmats.jca_effective(mat, f) if d.kind == "equivalent_fluid" else
                  (complex(mat.rho), complex(mat.c)) for f in grid]
            pay[f"rho_eff__{d.id}"] = np.array([a for a, _ in rc])
            pay[f"c_eff__{d.id}"] = np.array([b for _, b in rc])
    for k, (sid, fid, _) in enumerate(op.couplings):
        pay[f"rho_f{k}"] = np.array([fluid_density(op.kinds[fid], cfg.material_of(fid), f) for f in grid])
    loads = np.stack([op.load(f) for f in grid])
    rows = np.nonzero(np.any(loads != 0, axis=0))[0]
    pay["load_rows"] = rows
    pay["load_vals"] = loads[:, rows]
    # the reference MOR build and sweep
    t0 = time.perf_counter()
    roms = rmor.build_local_roms(fom, grid, cfg.mor, band)
    pay["build_s"] = np.array(time.perf_counter() - t0)
    pay["n_windows"] = np.array(len(roms))
    pay["windows"] = np.array([r.window for r in roms])
    for k, r in enumerate(roms):
        pay[f"V{k}"] = r.V
        pay[f"points{k}"] = np.array(r.expansion_points)
        pay[f"errlog{k}"] = np.array(r.error_log)
        pay[f"flags{k}"] = np.array([r.converged, r.stalled, r.budget_exhausted])
    t0 = time.perf_counter()
    sw = rmor.rom_sweep(roms, grid)
    pay["sweep_s"] = np.array(time.perf_counter() - t0)
    pay["frf"] = np.array(sw.frf)
    pay["window_index"] = np.array(sw.window_index)
    pay["seam_f"] = np.array([f for f, _ in sw.seam_log])
    pay["seam_gap"] = np.array([g for _, g in sw.seam_log])
    fom_f = [grid[7], grid[200], grid[401]]
    pay["fom_f"] = np.array(fom_f)
    pay["fom_y"] = np.array([fom.output(fom.solve(f)) for f in fom_f])
    np.savez_compressed(out, **pay)
    add_sensitivity(out)
    print(f"wrote {out}: n = {fom.n}, windows = {len(roms)}, r = {[r.r for r in roms]}, "
          f"build {float(pay['build_s']):.1f} s, sweep {float(pay['sweep_s']):.1f} s")


def add_sensitivity(path=HERE / "fuselage_slice.npz", trials: int = 8):
    """Conditioning of the reference's own FRF: for every grid frequency, the
    reference reduced system (ReducedModel.reduced_system, mor.py:73-90) is
    solved again with AR perturbed by ~1 ulp (seeded, `trials` times); the
    largest relative change of the output is the level to which the reference
    result is determined by its own rounding.  Parity tests floor their 1e-8
    tolerance at twice this value."""
    cfg = load_config(Path(vibrofem.__file__).parent / "data" / "fuselage_slice.cfg")
    fom, op = _mor_fom(cfg)
    z = dict(np.load(path))
    grid = [float(f) for f in z["grid"]]
    rng = np.random.default_rng(4242)
    sens = np.zeros(len(grid))
    roms = [rmor.ReducedModel(fom=fom, V=z[f"V{k}"], window=tuple(z["windows"][k]))
            for k in range(int(z["n_windows"]))]
    for i, f in enumerate(grid):
        rom = roms[int(z["window_index"][i])]
        AR, bR = rom.reduced_system(f)
        cR = rom.c_out_reduced
        y0 = cR @ np.linalg.solve(AR, bR)
        for _ in range(trials):
            E = 2.2e-16 * (rng.standard_normal(AR.shape) + 1j * rng.standard_normal(AR.shape))
            y1 = cR @ np.linalg.solve(AR * (1 + E), bR)
            sens[i] = max(sens[i], abs(y1 - y0) / abs(y0))
    z["y_sens"] = sens
    np.savez_compressed(path, **z)
    print(f"y_sens: max {sens.max():.3e} at {grid[int(np.argmax(sens))]} Hz; "
          f"{int(np.sum(sens > 0.5e-8))} frequencies above 5e-9")


def add_errlog_sensitivity(path=HERE / "fuselage_slice.npz", trials: int = 2):
    """How well the reference's own greedy error log is determined by its
    inputs: build_local_roms rerun with every primitive value perturbed by ~1
    ulp (seeded); errlog_sens = the largest |delta eps| per candidate over the
    trials (the decisions must not change, or the run is flagged)."""
    cfg = load_config(Path(vibrofem.__file__).parent / "data" / "fuselage_slice.cfg")
    z = dict(np.load(path))
    grid = [float(f) for f in z["grid"]]
    band = (cfg.frequency.f_min, cfg.frequency.f_max)
    rng = np.random.default_rng(777)
    sens = [np.zeros(len(z[f"errlog{k}"])) for k in range(int(z["n_windows"]))]
    same = True
    for _ in range(trials):
        fom, op = _mor_fom(cfg)
        for prims in op.primitives.values():
            for A in prims.values():
                A.data = A.data * (1 + 2.2e-16 * rng.standard_normal(A.data.shape))
        roms = rmor.build_local_roms(fom, grid, cfg.mor, band)
        same &= len(roms) == int(z["n_windows"])
        for k, r in enumerate(roms[:len(sens)]):
            same &= list(r.expansion_points) == list(z[f"points{k}"])
            log = np.array(r.error_log)
            if log.shape == z[f"errlog{k}"].shape:
                sens[k] = np.maximum(sens[k], np.abs(log[:, 1] - z[f"errlog{k}"][:, 1]))
    for k, sv in enumerate(sens):
        z[f"errlog_sens{k}"] = sv
    z["errlog_sens_same_decisions"] = np.array(same)
    np.savez_compressed(path, **z)
    print(f"errlog_sens: max {max(v.max() for v in sens):.3e}, same decisions {same}")


if __name__ == "__main__":
    if "--errlog-sens" in sys.argv:
        sys.exit(add_errlog_sensitivity())
    if "--sens" in sys.argv:
        sys.exit(add_sensitivity())
    sys.exit(main())
