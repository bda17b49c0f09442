"""Generate the golden fixtures that pin the oracle (and through it the GPU path)
to the UNMODIFIED reference `vibrofem`.

Run in the build container (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array written here is an output of reference code (vibrofem.*) on
seeded inputs; inputs that the reference cannot build itself (hex27 boxes,
impedance faces, point sources — SURVEY §8a "not in the reference") come from
the oracle restatement and are recorded next to the outputs.
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np
import scipy.sparse as sp

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from vibrofem import mor as rmor  # noqa: E402  (reference)
from vibrofem import shape as rshape  # noqa: E402
from vibrofem.assembly import _assemble_primitives, helmholtz_element_parts  # noqa: E402
from vibrofem.config import DomainSpec  # noqa: E402
from vibrofem.materials import AcousticMaterial  # noqa: E402
from vibrofem.meshing import generate_mesh  # noqa: E402
from vibrofem.solvers import mean_spl  # noqa: E402

from paper_2310_04734_b200 import workloads  # noqa: E402  (seeded input generator)
from oracle import fe  # noqa: E402  (restated hex27 inputs)


def csr_dict(prefix, A):
    A = sp.csr_matrix(A)
    return {f"{prefix}_indptr": A.indptr.astype(np.int64), f"{prefix}_indices": A.indices.astype(np.int64),
            f"{prefix}_data": A.data}


def frozen_fom(n=60, seed=0, damping=0.02):
    """tests/test_mor.py:26-37 (reference test fixture, restated here verbatim in behaviour)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, n))
    K = sp.csc_matrix((X @ X.T + n * np.eye(n)) * (1 + 1j * damping))
    Y = rng.standard_normal((n, n)) * 0.05
    M = sp.csc_matrix(Y @ Y.T + np.eye(n))
    b = rng.standard_normal(n)
    c = np.zeros(n)
    c[n // 3] = 1.0
    return rmor.FullOrderModel(stiffness=lambda f: K, mass=lambda f: M, load=lambda f: b,
                               c_out=c, n=n), K, M, b, c


def gold_frozen():
    fom, K, M, b, c = frozen_fom()
    Q1, br1 = rmor.krylov_block(fom, 35.0, 5)
    Q2, br2 = rmor.krylov_block(fom, 55.0, 4)
    V = rmor._orthonormalise(Q1, Q2)
    rom = rmor.ReducedModel(fom=fom, V=V, window=(10.0, 100.0))
    freqs = np.array([12.0, 35.0, 47.0, 55.0, 93.0])
    y_rom = np.array([rom.output(f) for f in freqs])
    y_fom = np.array([fom.output(fom.solve(f)) for f in freqs])
    out = {"K": K.toarray(), "M": M.toarray(), "b": b, "c": c, "Q1": Q1, "Q2": Q2, "V": V,
           "freqs": freqs, "y_rom": y_rom, "y_fom": y_fom}
    # drop rule (tests/test_mor.py:109-116)
    rng = np.random.default_rng(1)
    blk = rng.standard_normal((30, 3))
    blk[:, 2] = blk[:, 0] + blk[:, 1]
    out["drop_block"] = blk
    out["drop_Q"] = rmor._orthonormalise(None, blk)
    np.savez_compressed(HERE / "frozen_fom.npz", **out)


def gold_assembly_2d():
    """Reference _assemble_primitives (assembly.py:142-175) on a 2D acoustic mesh."""
    dom = DomainSpec(id="c", kind="acoustic", rect=(0.0, 0.0, 0.9, 0.6), material_id="air")
    mesh = generate_mesh(dom, (0.3, 0.2))
    prim = _assemble_primitives(mesh, "acoustic", AcousticMaterial(c=343.0, rho=1.21))
    coords = 0.5 * (np.array(rshape.LOCAL_NODES) + 1.0) * [0.7, 0.4] + [0.1, 0.2]
    Ke, Me = helmholtz_element_parts(coords)
    out = {"nodes": mesh.nodes, "elements": mesh.elements, "Ke": Ke, "Me": Me, "coords": coords,
           **csr_dict("Kgrad", prim["Kgrad"]), **csr_dict("Mnn", prim["Mnn"])}
    np.savez_compressed(HERE / "assembly_2d.npz", **out)


def small_box_fom():
    """Restated cfg1-style box (oracle hex27 assembly): the reference MOR then runs on it."""
    box = (0.0, 0.0, 0.0, 0.6, 0.4, 0.3)
    ne = (3, 2, 2)
    nodes, elems = fe.structured_hex27(box, *ne)
    Kg, Mn = fe.assemble_helmholtz(nodes, elems, fe.HEX27_IDX)
    fel, floc = fe.hex27_face(ne, "z0")
    Fz = fe.face_mass_hex27(nodes, elems, fel, floc)
    rho, c = 1.21, 343.0
    Z = rho * c * (5 + 1j)
    K = (Kg / rho).astype(complex)
    M = (Mn / (rho * c * c)).astype(complex)
    D = Fz / Z
    n = nodes.shape[0]
    b = np.zeros(n, complex)
    b[87] = 1.0
    rec = np.array([12, 40, 66, 101, 150, 160, 33, 121])
    C = np.zeros((len(rec), n))
    C[np.arange(len(rec)), rec] = 1.0
    return dict(K=K, M=M, D=D, b=b, C=C, rec=rec, Kg=Kg, Mn=Mn, Fz=Fz, nodes=nodes, elems=elems)


def gold_box_mor():
    d = small_box_fom()
    fom = rmor.FullOrderModel(stiffness=lambda f: d["K"], mass=lambda f: d["M"],
                              load=lambda f: d["b"], c_out=d["C"], n=d["K"].shape[0],
                              damping=lambda f: d["D"])
    pts = [300.0, 900.0]
    V = None
    for f0 in pts:
        Q, _ = rmor.krylov_block(fom, f0, 4, second_order=True)
        V = rmor._orthonormalise(V, Q)
    rom_lo = rmor.ReducedModel(fom=fom, V=V, window=(200.0, 600.0))
    rom_hi = rmor.ReducedModel(fom=fom, V=V[:, :6], window=(600.0, 1000.0))
    grid = list(np.arange(200.0, 1000.1, 50.0))
    sw = rmor.rom_sweep([rom_hi, rom_lo], grid)
    y = np.array(sw.frf)
    spl = np.array([mean_spl(v) for v in y])
    y_fom = np.array([fom.output(fom.solve(f)) for f in grid])
    # Conditioning of the reference output itself: rerun the reference pipeline on
    # K, M with every stored value perturbed by ~1 ulp (8 seeded trials) and keep
    # the largest relative change per frequency.  Where this exceeds the 1e-8
    # spec tolerance the reference result is only determined to that level by
    # its own inputs, and the parity test uses it as the floor.
    rng = np.random.default_rng(12345)
    sens = np.zeros(len(grid))
    for _ in range(8):
        Kp, Mp = sp.csr_matrix(d["K"]), sp.csr_matrix(d["M"])
        Kp.data = Kp.data * (1 + 2.2e-16 * rng.standard_normal(Kp.nnz))
        Mp.data = Mp.data * (1 + 2.2e-16 * rng.standard_normal(Mp.nnz))
        fp = rmor.FullOrderModel(stiffness=lambda f, K=Kp: K, mass=lambda f, M=Mp: M,
                                 load=lambda f: d["b"], c_out=d["C"], n=d["K"].shape[0],
                                 damping=lambda f: d["D"])
        Vp = None
        for f0 in pts:
            Qp, _ = rmor.krylov_block(fp, f0, 4, second_order=True)
            Vp = rmor._orthonormalise(Vp, Qp)
        swp = rmor.rom_sweep([rmor.ReducedModel(fom=fp, V=Vp[:, :6], window=(600.0, 1000.0)),
                              rmor.ReducedModel(fom=fp, V=Vp, window=(200.0, 600.0))], grid)
        sens = np.maximum(sens, [rmor.relative_error(y[i], swp.frf[i])[1] for i in range(len(grid))])
    out = {"V": V, "grid": np.array(grid), "y": y, "spl": spl, "y_fom": y_fom, "y_sens": sens,
           "window_index": np.array(sw.window_index),
           "seam_f": np.array([s[0] for s in sw.seam_log]),
           "seam_gap": np.array([np.max(np.abs(s[1])) for s in sw.seam_log]),
           "points": np.array(pts), **csr_dict("Kg", d["Kg"]), **csr_dict("Mn", d["Mn"]),
           **csr_dict("Fz", d["Fz"]), "b": d["b"], "rec": d["rec"]}
    np.savez_compressed(HERE / "box_mor.npz", **out)


def gold_reduced_dense():
    """cfg5-style dense reduced matrices through ReducedModel with V = I
    (tests/test_mor.py:119-125 pattern) and mean_spl — the literal reference path."""
    w = workloads.cfg5(r=48, n_freq=2000, s=3, n_out=7, seed=9)
    Kd, Dd, Md = (sp.csr_matrix(P) for P in w.prims)
    idx = np.arange(0, 2000, 97)
    freqs = w.freqs[idx]
    ys, spls = [], []
    for col in range(w.b.shape[1]):
        fom = rmor.FullOrderModel(stiffness=lambda f: Kd, mass=lambda f: Md,
                                  load=lambda f, c=col: w.b[:, c], c_out=w.c_r, n=w.r,
                                  damping=lambda f: Dd)
        rom = rmor.ReducedModel(fom=fom, V=np.eye(w.r, dtype=complex), window=(0.0, 2000.0))
        yc = np.array([rom.output(f) for f in freqs])
        ys.append(yc)
        spls.append([mean_spl(v) for v in yc])
    y = np.stack(ys, axis=-1)           # (F, n_out, s)
    spl = np.array(spls).T              # (F, s)
    np.savez_compressed(HERE / "reduced_dense.npz", freqs=freqs, y=y, spl=spl,
                        r=w.r, s=w.b.shape[1], n_out=w.c_r.shape[0], seed=w.seed, n_freq=2000)


def gold_artifacts():
    """Reference rom.npz (cli.save_roms) and frf_mor.csv (cli.write_csv) bytes."""
    from vibrofem import cli as rcli
    fom, K, M, b, c = frozen_fom()
    Q, _ = rmor.krylov_block(fom, 35.0, 4)
    roms = [rmor.ReducedModel(fom=fom, V=Q, window=(10.0, 50.0), expansion_points=[35.0],
                              error_log=[(10.0, 1e-3), (50.0, 2e-3)], converged=True),
            rmor.ReducedModel(fom=fom, V=Q[:, :2], window=(50.0, 100.0), expansion_points=[35.0],
                              error_log=[(50.0, 5e-2)], stalled=True)]
    rcli.save_roms(HERE / "rom_ref.npz", roms)
    grid = [10.0, 30.0, 50.0, 75.0, 100.0]
    sw = rmor.rom_sweep(roms, grid)
    rows = [[f, y.real, y.imag, 20.0 * np.log10(max(abs(y), 1e-300) / 20e-6), w]
            for f, y, w in zip(sw.freqs, sw.frf, sw.window_index)]
    rcli.write_csv(HERE / "frf_ref.csv", ["f_hz", "re_p", "im_p", "abs_db", "window"], rows)
    np.savez_compressed(HERE / "frf_ref_values.npz", freqs=np.array(grid), frf=np.array(sw.frf),
                        window_index=np.array(sw.window_index))


def gold_spl():
    vals = {"ones": mean_spl(np.ones(64, complex)), "zeros": mean_spl(np.zeros(5, complex))}
    rng = np.random.default_rng(4)
    p = rng.standard_normal(50) + 1j * rng.standard_normal(50)
    vals["random"] = mean_spl(p)
    np.savez_compressed(HERE / "spl.npz", p=p, **vals)


def oscillator_chain(n=120, damping=0.02):
    """tests/test_mor.py:40-52 (reference test fixture): spring-mass chain with
    structural damping, forced at one end, observed at the other."""
    main = 2.0 * np.ones(n)
    off = -np.ones(n - 1)
    K = sp.diags([off, main, off], [-1, 0, 1], format="csc") * 1e6 * (1 + 1j * damping)
    M = sp.identity(n, format="csc") * 1.0
    b = np.zeros(n)
    b[0] = 1.0
    c = np.zeros(n)
    c[-1] = 1.0
    return rmor.FullOrderModel(stiffness=lambda f: K, mass=lambda f: M, load=lambda f: b, c_out=c, n=n)


class Settings:
    """MorSettings duck type (config.py:172-184; tests/test_mor.py:17-23)."""

    def __init__(self, tol=1e-2, max_points=20, moments_per_point=4, candidate_stride=4, windows="auto"):
        self.tol, self.max_points, self.moments_per_point = tol, max_points, moments_per_point
        self.candidate_stride, self.windows = candidate_stride, windows


GREEDY_CASES = {
    # name: (model, grid, settings kwargs, band or window, entry)
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


def gold_greedy():
    """Reference greedy_expand / build_local_roms (mor.py:224-353) decisions:
    expansion points, r, error logs, converged/stalled/budget flags,
    auto-bisected windows, and the rom_sweep FRF of the result."""
    out = {"cases": np.array(list(GREEDY_CASES))}
    for name, (model, (g0, g1, ng), kw, entry) in GREEDY_CASES.items():
        fom = oscillator_chain() if model == "chain" else frozen_fom(n=200)[0]
        grid = list(np.linspace(g0, g1, ng))
        st = Settings(**kw)
        if entry == "greedy":
            roms = [rmor.greedy_expand(fom, grid, st, (g0, g1))]
        else:
            roms = rmor.build_local_roms(fom, grid, st, (g0, g1))
        out[f"{name}__n_windows"] = np.array(len(roms))
        for k, r in enumerate(roms):
            out[f"{name}__window{k}"] = np.array(r.window)
            out[f"{name}__points{k}"] = np.array(r.expansion_points)
            out[f"{name}__r{k}"] = np.array(r.r)
            out[f"{name}__errlog{k}"] = np.array(r.error_log)
            out[f"{name}__flags{k}"] = np.array([r.converged, r.stalled, r.budget_exhausted])
        sw = rmor.rom_sweep(roms, grid)
        out[f"{name}__frf"] = np.array(sw.frf)
        out[f"{name}__window_index"] = np.array(sw.window_index)
    np.savez_compressed(HERE / "greedy_ref.npz", **out)


ALL = {"frozen": gold_frozen, "assembly_2d": gold_assembly_2d, "box_mor": gold_box_mor,
       "reduced_dense": gold_reduced_dense, "spl": gold_spl, "artifacts": gold_artifacts,
       "greedy": gold_greedy}


if __name__ == "__main__":
    for name in (sys.argv[1:] or list(ALL)):
        ALL[name]()
    for f in sorted(HERE.glob("*.npz")):
        print(f.name, f.stat().st_size)
