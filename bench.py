#!/usr/bin/env python
"""Benchmark of the north-star path: the MOR reduced frequency sweep.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--r 1024] [--batch B]

Workload (BASELINE.json configs[4], "cfg5"): seeded dense complex128 reduced
matrices K_r, D_r, M_r of order r (default 1024, the middle of {256, 1024,
2048}), 16 RHS, 50 output rows, frequencies from linspace(1, 1000, 100000).
A step = one batch of B frequencies per rank (default 16 per SM): form
A_r(f) = K_r + i w D_r - w^2 M_r, batched complex LU solve, y = C_R x, SPL —
i.e. vibrofem/mor.py:73-102 + solvers.py:334-338 for every frequency.
Each rank sweeps its own frequency slices (weak scaling, no data-path
collective); the step's SPL shard is all-gathered at the end of each step.

Prints ONE JSON line (rank 0).  See DESIGN.md §5 for the roofline counts.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frequency points/sec (MOR sweep)"
UNIT = "freq/s"


def flops_per_freq(r: int, nprim: int, s: int, n_out: int) -> float:
    """Algorithmic real flops per frequency (complex MAC = 8 flops):
    form nprim r^2, LU 8/3 r^3, two triangular solves 8 r^2 s, output 8 n_out r s."""
    return 8.0 * nprim * r * r + 8.0 / 3.0 * r ** 3 + 8.0 * r * r * s + 8.0 * n_out * r * s


def bytes_per_freq(r: int, nprim: int, s: int, n_out: int) -> float:
    """Algorithmic HBM bytes per frequency for the small (shared-memory) path:
    each frequency reads its coefficients and writes y and SPL; the
    primitives are shared (read once per launch)."""
    return 16.0 * nprim + 16.0 * n_out * s + 8.0 * s


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.hw_power_brake_slowdown")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.idx)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "hw_power_brake_slowdown"]
        sm, smax, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        n = [i.get("num_threads", 1) for i in info if i.get("user_api") == "blas"]
        return int(max(n)) if n else 1
    except Exception:
        return os.cpu_count() or 1


def cpu_sweep_rate(w, freqs_sample):
    """Oracle port (mor.py:73-102 restated, numpy.linalg.solve per frequency) on
    the host cores.  Returns freq/s."""
    from oracle import mor as omor
    alpha = w.alpha(freqs_sample)
    t0 = time.perf_counter()
    omor.affine_sweep(w.prims, alpha, w.b, w.c_r)
    dt = time.perf_counter() - t0
    return len(freqs_sample) / dt, dt


def cpu_literal_rate(w, n_freq: int = 20):
    """SURVEY §8(d) CPU baseline (1): the literal reference path,
    ReducedModel.output (mor.py:73-98: per-frequency re-projection V^H K V,
    V^H M V, V^H D V, then zgesv) with FOM providers that return the dense
    reduced matrices and V = I (the tests/test_mor.py:119-125 construction).
    Reported for completeness next to the affine-sweep port (baseline (2))."""
    from oracle import mor as omor
    K, D, M = (np.asarray(p) for p in w.prims)
    r = K.shape[0]
    fom = omor.Fom(stiffness=lambda f: K, mass=lambda f: M, load=lambda f: w.b, c_out=w.c_r, n=r,
                   damping=lambda f: D)
    V = np.eye(r, dtype=complex)
    rng = np.random.default_rng(13)
    fs = w.freqs[np.sort(rng.choice(len(w.freqs), n_freq, replace=False))]
    omor.reduced_output(fom, V, float(fs[0]))  # warm-up
    t0 = time.perf_counter()
    for f in fs:
        omor.reduced_output(fom, V, float(f))
    dt = time.perf_counter() - t0
    return n_freq / dt, dt, n_freq


def cpu_cfg1_pipeline():
    """SURVEY §8(d) offline CPU baselines: the reference algorithm end to end on
    cfg1 (oracle restatement: hex27 assembly, scipy splu per expansion point +
    second-order Krylov, MGS2 _orthonormalise, the literal per-frequency
    re-projection + zgesv of ReducedModel.output over all 181 frequencies, SPL),
    stage by stage, on the host cores.  Compare with offline.cfg1_pipeline_s /
    cfg1_pipeline_fdm_s (the same chain on the GPU)."""
    from oracle import fe
    from oracle import mor as omor
    from paper_2310_04734_b200 import workloads
    t = {}
    t0 = time.perf_counter()
    nodes, elems = fe.structured_hex27(workloads.CFG1_BOX, *workloads.CFG1_NE)
    Kg, Mn = fe.assemble_helmholtz(nodes, elems, fe.HEX27_IDX)
    el, loc = fe.hex27_face(workloads.CFG1_NE, "z0")
    Fz = fe.face_mass_hex27(nodes, elems, el, loc)
    rho, c = workloads.AIR_RHO, workloads.AIR_C
    K, M, D = (Kg / rho).astype(complex), (Mn / (rho * c * c)).astype(complex), Fz / workloads.CFG1_Z
    t["assembly_s"] = time.perf_counter() - t0
    _, _, src, rec = workloads.cfg1_layout()
    lay = {"src": src, "rec": rec, "freqs": np.arange(20.0, 200.5, 1.0), "points": workloads.CFG1_POINTS,
           "moments": workloads.CFG1_MOMENTS}
    n = K.shape[0]
    b = np.zeros(n, complex)
    b[lay["src"]] = 1.0
    C = np.zeros((len(lay["rec"]), n))
    C[np.arange(len(lay["rec"])), lay["rec"]] = 1.0
    fom = omor.Fom(stiffness=lambda f: K, mass=lambda f: M, load=lambda f: b, c_out=C, n=n, damping=lambda f: D)
    V, tk, to = None, 0.0, 0.0
    for f0 in lay["points"]:
        a = time.perf_counter()
        Q, _ = omor.krylov_block(fom, f0, lay["moments"], second_order=True)
        bb = time.perf_counter()
        V = omor.orthonormalise(V, Q)
        tk += bb - a
        to += time.perf_counter() - bb
    t["krylov_splu_s"], t["orthonormalise_s"] = tk, to
    a = time.perf_counter()
    for f in lay["freqs"]:
        omor.mean_spl(omor.reduced_output(fom, V, float(f)))
    t["sweep_s"] = time.perf_counter() - a
    t["total_s"] = t["assembly_s"] + tk + to + t["sweep_s"]
    t["r"] = int(V.shape[1])
    t["n"] = int(n)
    t["freqs"] = len(lay["freqs"])
    return t


def cpu_sample_size(w, budget_s: float) -> int:
    """Number of frequencies the CPU port finishes in about budget_s seconds
    (pilot of 8 frequencies after a warm-up call)."""
    cpu_sweep_rate(w, w.freqs[:2])
    rate, _ = cpu_sweep_rate(w, w.freqs[2:10])
    return int(max(4, min(len(w.freqs), rate * budget_s)))


def bench_config(r: int, s: int, n_out: int, nprim: int, B: int, ws: int) -> dict:
    """The workload both arms report (identical dict, so the driver can pair them)."""
    return {"workload": f"cfg5_r{r}", "r": r, "rhs": s, "n_out": n_out, "n_prim": nprim,
            "freqs_per_step_per_rank": B, "grid": "linspace(1,1000,100000), rank-disjoint slices",
            "l2": "flushed between timed steps (512 MiB write)",
            "parallelism": f"frequency-sharded x{ws}"}


def default_batch(args) -> int:
    """16 frequencies per SM per rank (148 SMs on B200 when no GPU is visible)."""
    if args.batch:
        return args.batch
    nsm = 148
    try:
        import torch
        if torch.cuda.is_available():
            nsm = torch.cuda.get_device_properties(0).multi_processor_count
    except Exception:
        pass
    return 16 * nsm


def parity_sample(w, freqs_timed: np.ndarray, n: int = 64, n_res: int = 16, seed: int = 17) -> np.ndarray:
    """Indices into freqs_timed to check against the oracle: the n_res timed
    frequencies nearest the workload's undamped eigenfrequencies (where the
    LU pivots hardest) plus seeded random others, n in total."""
    from paper_2310_04734_b200 import workloads
    ef = workloads.cfg5_eigenfrequencies(w)
    order = np.argsort(freqs_timed)
    fs = freqs_timed[order]
    lo, hi = fs[0], fs[-1]
    ef = ef[(ef >= lo) & (ef <= hi)]
    pick = []
    if ef.size:
        pos = np.clip(np.searchsorted(fs, ef), 1, len(fs) - 1)
        near = np.where(np.abs(fs[pos - 1] - ef) <= np.abs(fs[pos] - ef), pos - 1, pos)
        dist = np.abs(fs[near] - ef)
        for j in near[np.argsort(dist)]:
            if order[j] not in pick:
                pick.append(int(order[j]))
            if len(pick) >= n_res:
                break
    rng = np.random.default_rng(seed)
    rest = np.setdiff1d(np.arange(len(freqs_timed)), pick)
    extra = rng.choice(rest, min(len(rest), n - len(pick)), replace=False)
    return np.array(sorted(pick + [int(i) for i in extra]), dtype=np.int64)


def parity_check(w, freqs, y, spl, n_res_probe: int = 16) -> dict:
    """Compare GPU outputs y (F, n_out, s) / spl (F, s) at `freqs` with the oracle
    (oracle.mor.affine_sweep = mor.py:73-102 restated, LAPACK zgesv): the
    reference's pointwise relative_error (mor.py:194-208) and |dSPL|."""
    from oracle import mor as omor
    y_ref, spl_ref = omor.affine_sweep(w.prims, w.alpha(freqs), w.b, w.c_r)
    pt = max(omor.relative_error(y_ref[i].ravel(), y[i].ravel())[1] for i in range(len(freqs)))
    nw = max(float(np.linalg.norm(y_ref[i] - y[i]) / np.linalg.norm(y_ref[i])) for i in range(len(freqs)))
    return {"n": int(len(freqs)), "n_near_resonance": int(n_res_probe),
            "max_tf_rel_err": float(pt), "max_tf_rel_err_normwise": nw,
            "max_dspl_db": float(np.abs(spl - spl_ref).max()),
            "tol": {"tf_rel": 1e-8, "dspl_db": 0.01},
            "pass": bool(pt <= 1e-8 and np.abs(spl - spl_ref).max() <= 0.01),
            "oracle": "oracle.mor.affine_sweep (numpy.linalg.solve = LAPACK zgesv per frequency)"}


def probe_peak(n: int = 5) -> tuple[float, list]:
    """FP64 DMMA peak: median of n live probes (one figure for every fraction)."""
    from paper_2310_04734_b200 import _lib
    vals = [_lib.probe_fp64_peak() for _ in range(n)]
    return float(np.median(vals)), vals


def all_host_threads():
    """BLAS thread pool opened to every host core (torchrun exports
    OMP_NUM_THREADS=1 to its ranks; the CPU baseline uses the whole host)."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=os.cpu_count() or 1, user_api="blas")
    except Exception:  # no threadpoolctl: keep the defaults
        import contextlib
        return contextlib.nullcontext()


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port; the reference is
    pure Python and cannot travel to the GPU box) on the host cores."""
    with all_host_threads():
        return _run_reference(args)


def _run_reference(args):
    from paper_2310_04734_b200 import dist as vdist, workloads
    rank, ws, _ = vdist.world()
    if rank != 0:
        return 0
    w = workloads.cfg5(r=args.r)
    B = default_batch(args)
    n_per_step = cpu_sample_size(w, args.cpu_step_s)
    rng = np.random.default_rng(11)
    times, count = [], 0
    for step in range(args.warmup + args.steps):
        idx = np.sort(rng.choice(len(w.freqs), n_per_step, replace=False))
        rate, dt = cpu_sweep_rate(w, w.freqs[idx])
        if step >= args.warmup:
            times.append(dt)
            count += n_per_step
    value = count / sum(times)
    cores = blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "complex128",
        "data": "synthetic (seeded cfg5)",
        "config": bench_config(args.r, w.b.shape[1], w.c_r.shape[0], w.prims.shape[0], B, ws),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"bounded sample of each {B}-frequency step: {n_per_step} seeded random "
                                   f"grid frequencies per step, numpy.linalg.solve (LAPACK zgesv) per "
                                   f"frequency, BLAS threads={cores}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def offline_measurements(w, peak_fp64=None):
    """Secondary numbers (not the headline): the other stages of the MOR chain at
    BASELINE sizes, CUDA-event timed — cfg3 assembly / SpMM / projection / FDM
    solve (tools/bench_offline.py) and the cfg1 pipeline end to end."""
    import importlib.util
    import torch
    spec = importlib.util.spec_from_file_location("bench_offline", ROOT / "tools" / "bench_offline.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    out = mod.measure(peak_fp64)
    from paper_2310_04734_b200 import mor, workloads

    def cfg1(fdm):
        fom, lay = workloads.cfg1_model(fdm=fdm)
        V, _ = mor.krylov_basis(fom, lay["points"], lay["moments"], second_order=True)
        rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 200.0))
        mor.rom_sweep([rom], list(lay["freqs"]))
        return fom, V

    def cfg2():
        fom, lay = workloads.cfg2_model()
        V, _ = mor.krylov_basis(fom, lay["points"], lay["moments"])
        rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 500.0))
        mor.rom_sweep([rom], list(lay["freqs"]))
        return fom, V

    def cfg3():
        fom, lay = workloads.cfg3_model()
        V, _ = mor.krylov_basis(fom, lay["points"], lay["moments"], second_order=True, mimo=True)
        rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 300.0))
        mor.rom_sweep([rom], list(lay["freqs"]))
        return fom, V

    def timed_twice(fn, reps: int = 5):
        """(first run, median of the next `reps` runs) wall clock incl. host
        orchestration; the median is the reported number (first runs include
        one-off module loading, thread-pool and allocator warm-up)."""
        ts = []
        for _ in range(1 + reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return (ts[0], float(np.median(ts[1:]))), res

    (t1, t1w), (_, V) = timed_twice(lambda: cfg1(False))
    out["cfg1_pipeline_s"], out["cfg1_pipeline_first_s"], out["cfg1_r"] = t1w, t1, int(V.shape[1])
    out["cfg1_note"] = ("GPU assembly + 4 dense LUs (n=4641, the 4 expansion points concurrent on their own "
                        "streams) + 2nd-order Krylov + CGS2 + projection + 181-frequency sweep + SPL, wall clock "
                        "incl. host orchestration (median of 5 warm runs; *_first_s = first run in the process)")
    (t1, t1w), (_, V) = timed_twice(lambda: cfg1(True))
    out["cfg1_pipeline_fdm_s"], out["cfg1_pipeline_fdm_first_s"], out["cfg1_fdm_r"] = t1w, t1, int(V.shape[1])
    (t2, t2w), (fom, V) = timed_twice(cfg2)
    out["cfg2_pipeline_s"], out["cfg2_pipeline_first_s"] = t2w, t2
    out["cfg2_n"], out["cfg2_r"] = int(fom.n), int(V.shape[1])
    out["cfg2_note"] = ("GPU plate+cavity assembly (n=20890) + 6 Schur-complement (plate) / fast-diagonalisation "
                        "(cavity) factorisations with refinement (expansion points concurrent) + Krylov + CGS2 + "
                        "projection + batched plane-wave RHS + 961-frequency sweep + SPL")
    # the reference's OWN benchmark model (tier 0: fuselage_slice.cfg, n = 8,102)
    # through the drop-in, from the arrays the reference wrote
    # (tests/golden/fuselage_slice.npz): rom_sweep of the 496-frequency grid
    # with the reference's basis, and the whole build_local_roms (greedy,
    # auto windows) — reference on the build container's 8 cores: 39.7 s and
    # 183.6 s (fixture sweep_s / build_s)
    from paper_2310_04734_b200.model_operator import load_operator_npz
    fx = ROOT / "tests" / "golden" / "fuselage_slice.npz"
    if fx.exists():
        zf = np.load(fx)
        fomf, gridf, _ = load_operator_npz(fx)
        romf = [mor.ReducedModel(fom=fomf, V=zf[f"V{k}"], window=tuple(zf["windows"][k]))
                for k in range(int(zf["n_windows"]))]

        class _Mor:
            tol, max_points, moments_per_point, candidate_stride, windows = 1e-2, 20, 4, 4, "auto"
        (ts, tsw), _ = timed_twice(lambda: mor.rom_sweep(romf, gridf))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rb = mor.build_local_roms(fomf, gridf, _Mor(), (gridf[0], gridf[-1]))
        torch.cuda.synchronize()
        out["fuselage_sweep_s"], out["fuselage_sweep_first_s"] = tsw, ts
        out["fuselage_build_s"] = time.perf_counter() - t0
        out["fuselage_build_same_points"] = bool(all(
            [float(p) for p in r.expansion_points] == [float(p) for p in zf[f"points{k}"]] for k, r in enumerate(rb)))
        out["fuselage_reference_s"] = {"sweep": float(zf["sweep_s"]), "build": float(zf["build_s"]),
                                       "where": "build container, 8 cores (fixture)"}
        out["fuselage_note"] = ("reference benchmark fuselage_slice.cfg (n=8102, r=76, 496 freqs) through the "
                                "ModelOperator drop-in: rom_sweep with the reference's basis; build_local_roms "
                                "(greedy, GPU dense LU FOM solves, batched candidate sweeps)")
    def cfg3_pe():
        fom, lay = workloads.cfg3_model(per_element_z=True)
        V, _ = mor.krylov_basis(fom, lay["points"], lay["moments"], second_order=True, mimo=True)
        rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 300.0))
        mor.rom_sweep([rom], list(lay["freqs"]))
        return fom, V
    (tp, tpw), (fom, V) = timed_twice(cfg3_pe, reps=3)
    out["cfg3_per_element_pipeline_s"], out["cfg3_per_element_pipeline_first_s"] = tpw, tp
    out["cfg3_per_element_note"] = ("cfg3 with per-element wall impedances Z_e = rho c U[2,10] (no Kronecker form): "
                                    "full-order solves by GPU GMRES preconditioned by the box FDM with harmonic-mean "
                                    "walls (~8 iterations, residual <= 1e-10), r = 400, 1121 frequencies")
    (t3, t3w), (fom, V) = timed_twice(cfg3)
    out["cfg3_pipeline_s"], out["cfg3_pipeline_first_s"] = t3w, t3
    out["cfg3_n"], out["cfg3_r"] = int(fom.n), int(V.shape[1])
    out["cfg3_note"] = ("GPU box assembly (n=376431) + fast-diagonalisation FOM solves at 5 points x 10 "
                        "second-order moments x 8 sources + block CGS2 + Kronecker-apply projection + "
                        "1121-frequency sweep (8 RHS) + SPL")
    out.update(cfg4_measurements())
    return out


def cfg4_measurements():
    """cfg4 synthetic fuselage (BASELINE configs[3]): the whole MOR pipeline at
    the reduced resolution the plane-block solver covers (n = 84,189, r ~ 2000,
    461 frequencies, one run: ~40 s), its ROM accuracy on a disjoint grid, and
    generator + GPU assembly at the full ~2.4M-DoF resolution."""
    import torch
    from paper_2310_04734_b200 import fuselage as fz, mor
    out = {}
    sync = torch.cuda.synchronize
    sync()
    t0 = time.perf_counter()
    fom, info = fz.fuselage_model(fz.FuselageSpec())
    sync()
    t_build = time.perf_counter() - t0
    V, _ = mor.krylov_basis(fom, list(fz.CFG4_POINTS), fz.CFG4_MOMENTS)
    rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 250.0))
    res = mor.rom_sweep([rom], list(info["freqs"]))
    sync()
    out["cfg4_pipeline_s"] = time.perf_counter() - t0
    out["cfg4_model_build_s"] = t_build
    out["cfg4_n"], out["cfg4_r"], out["cfg4_freqs"] = int(fom.n), int(V.shape[1]), len(info["freqs"])
    tf, ts = [], []
    for f in (61.0, 173.0):
        sync()
        t1 = time.perf_counter()
        fac = fom.factor(f)
        sync()
        tf.append(time.perf_counter() - t1)
        b = fom.load_dev(f)
        sync()
        t1 = time.perf_counter()
        fac.solve(b)
        sync()
        ts.append(time.perf_counter() - t1)
        del fac
    out["cfg4_factor_s"], out["cfg4_solve_ms"] = float(np.median(tf)), 1e3 * float(np.median(ts))
    ver = [33.1, 97.7, 142.2, 211.9, 247.3]
    y, _, _, _ = rom.sweep(ver)
    y = y.cpu().numpy()
    worst = 0.0
    for i, f in enumerate(ver):
        yf = fom.c_out @ fom.factor(f).solve(fom.load_dev(f)).cpu().numpy()
        _, e, _, _ = mor.relative_error(yf.ravel(), y[i].ravel())
        worst = max(worst, float(e))
    out["cfg4_eps_max"] = worst
    del fom, info, V, rom, res
    torch.cuda.empty_cache()
    sync()
    t0 = time.perf_counter()
    fomF, infoF = fz.fuselage_model(fz.cfg4_spec_full(), solver=False)
    sync()
    out["cfg4_full_build_s"] = time.perf_counter() - t0
    out["cfg4_full_n"] = int(fomF.n)
    out["cfg4_full_nnz"] = int(sum(t.P.nnz for t in fomF.affine.K + fomF.affine.M))
    out["cfg4_note"] = ("synthetic fuselage (cylinder R 1.5 m x 3 m: skin, Miki/Delany-Bazley insulation, lining, floor, "
                        "6 frame webs, 40 U-stringers, cabin air; facet shells + chain-rule hex27). Pipeline at the "
                        "reduced resolution n=84189: GPU assembly + 20 plane-block factorisations (block inverses, "
                        "residual <= 1e-10) x 100 moments + CGS2 + projection + 461-frequency sweep at r~2000, one "
                        "run; eps_max vs full-order solves at 5 disjoint frequencies. cfg4_full_*: host mesh tables "
                        "+ GPU element kernels + CSR assembly at the BASELINE ~2.4M-DoF resolution (no solver)")
    return out


def sweep_timed(w, B, steps, warmup, dev, flush, rank=0, ws=1, keep=False, gather=None):
    """Device-resident sweep of `steps` timed batches of B frequencies (after
    `warmup` untimed ones): returns (step ms list, kernel ms list, kept outputs).
    Each step's frequencies are a rank-disjoint slice of the 100k grid; L2 is
    flushed before every timed step (outside the events)."""
    import torch
    from paper_2310_04734_b200 import sweep
    nF = len(w.freqs)
    freqs_dev = torch.from_numpy(w.freqs).to(dev)
    rs = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds, device=dev)
    stream = torch.cuda.current_stream(dev)

    def idx_of(step):
        start = ((step * ws + rank) * B) % nF
        return (np.arange(B) + start) % nF

    def one_step(step, ev=None):
        f = freqs_dev[torch.from_numpy(idx_of(step)).to(dev)]
        alpha = rs.alpha(f)
        if ev is not None:
            ev[0].record(stream)
        out = sweep.rom_sweep_affine(rs.P, alpha, rs.b, rs.c, want_y=True, want_spl=True)
        if ev is not None:
            ev[1].record(stream)
        if gather is not None:
            gather(out)
        return out

    for i in range(warmup):
        one_step(i)
    torch.cuda.synchronize()
    sweep.raise_if_singular(one_step(0).info)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
    kept = []
    from paper_2310_04734_b200 import dist as vdist
    vdist.barrier()
    torch.cuda.synchronize()
    from paper_2310_04734_b200 import _lib
    n0 = _lib.launch_count()
    for i in range(steps):
        flush.zero_()
        e = evs[i]
        e[0].record(stream)
        out = one_step(warmup + i, ev=(e[2], e[3]))
        e[1].record(stream)
        if keep:
            kept.append((idx_of(warmup + i), out))
    torch.cuda.synchronize()
    launches = _lib.launch_count() - n0
    vdist.barrier()
    step_ms = [e[0].elapsed_time(e[1]) for e in evs]
    kern_ms = [e[2].elapsed_time(e[3]) for e in evs]
    for _, o in kept:
        sweep.raise_if_singular(o.info)
    sweep_timed.launches = launches
    return step_ms, kern_ms, kept


def parity_of_kept(w, kept, n=64):
    """Parity of >= n of the frequencies the timed steps produced (bench's own
    outputs), n_res of them next to the eigenfrequencies."""
    idx = np.concatenate([i for i, _ in kept])
    freqs = w.freqs[idx]
    pick = parity_sample(w, freqs, n=n)
    # outputs of the picked rows (step, row within step)
    B = len(kept[0][0])
    ys = np.stack([kept[p // B][1].y[p % B].cpu().numpy() for p in pick])
    spls = np.stack([kept[p // B][1].spl[p % B].cpu().numpy() for p in pick])
    res = parity_check(w, freqs[pick], ys, spls)
    res["freq_range_hz"] = [float(freqs.min()), float(freqs.max())]
    return res


def per_order(args, dev, flush, peak, nsm):
    """The other cfg5 orders (BASELINE configs[4]: r in {256, 1024, 2048}) on
    the same kernel: throughput, roofline fraction and parity of 64 of their
    own timed frequencies (16 next to resonances)."""
    from paper_2310_04734_b200 import _lib, workloads
    out = {}
    for r in args.orders:
        if r == args.r:
            continue
        w = workloads.cfg5(r=r)
        B = 16 * nsm
        steps = 8 if r <= 512 else 3
        step_ms, kern_ms, kept = sweep_timed(w, B, steps, 2, dev, flush, keep=True)
        fl = flops_per_freq(r, w.prims.shape[0], w.b.shape[1], w.c_r.shape[0])
        kavg = sum(kern_ms) / len(kern_ms)
        ach = fl * B / (kavg * 1e-3) / 1e12
        out[f"r{r}"] = {"value": B * steps / (sum(step_ms) * 1e-3), "unit": UNIT, "freqs_per_step": B,
                        "steps": steps, "kernel_ms": kavg, "achieved_TFLOPs": ach, "frac": ach / peak,
                        "path": "blocked" if _lib.load().vb_rom_sweep_path(r, 3, 16, 50) == 1 else "shared-memory",
                        "parity": parity_of_kept(w, kept)}
        del kept
    return out


def run_ours(args):
    import torch
    from paper_2310_04734_b200 import _lib, dist as vdist, sweep, workloads

    share = os.environ.get("VB_BENCH_SHARE_GPU") == "1"  # test hook: ranks share the visible GPUs (gloo)
    if share:
        os.environ.setdefault("VB_DIST_BACKEND", "gloo")
    rank, ws, local = vdist.init()
    _lib.require_cuda()
    if share:
        local = local % torch.cuda.device_count()
    elif torch.cuda.device_count() < ws:
        raise SystemExit(f"bench.py: {ws} ranks but only {torch.cuda.device_count()} visible GPUs")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _lib.load()
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count

    w = workloads.cfg5(r=args.r)
    r, s, n_out, nprim = w.r, w.b.shape[1], w.c_r.shape[0], w.prims.shape[0]
    B = args.batch or 16 * nsm
    nF = len(w.freqs)
    flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)
    path = lib.vb_rom_sweep_path(r, nprim, s, n_out)
    gather = (lambda out: vdist.gather_rows(out.spl, B * ws, ws)) if ws > 1 else None

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    n0 = _lib.launch_count()
    persist = sweep.persist_primitives_in_l2() if args.l2_persist else None
    if persist:
        persist.__enter__()
    try:
        step_ms, kern_ms, kept = sweep_timed(w, B, args.steps, args.warmup, dev, flush, rank, ws,
                                             keep=(rank == 0 and not args.no_parity), gather=gather)
    finally:
        if persist:
            persist.__exit__(None, None, None)
    launches = _lib.launch_count() - n0  # warm-up + timed
    launches_timed = sweep_timed.launches
    clocks = sampler.stop() if sampler else None
    total_ms = vdist.max_over_ranks(sum(step_ms), dev)
    kern_avg_ms = vdist.max_over_ranks(sum(kern_ms) / len(kern_ms), dev)
    value = ws * B * args.steps / (total_ms * 1e-3)

    # ---- end to end through the public API, host buffers ----
    e2e = None
    if not args.no_e2e:
        P_h = torch.from_numpy(w.prims).pin_memory()
        b_h = torch.from_numpy(w.b).pin_memory()
        c_h = torch.from_numpy(w.c_r).pin_memory()
        f_h = torch.from_numpy(w.freqs).pin_memory()
        y_h = torch.empty((B, n_out, s), dtype=torch.complex128).pin_memory()
        spl_h = torch.empty((B, s), dtype=torch.float64).pin_memory()
        stream = torch.cuda.current_stream(dev)

        def e2e_step(step):
            start = ((step * ws + rank) * B) % nF
            idx = (np.arange(B) + start) % nF
            fs = f_h[torch.from_numpy(idx)].pin_memory()
            rs2 = sweep.ReducedSweep(P_h, b_h, c_h, kinds=w.kinds, device=dev)
            out = rs2.sweep_device(fs.to(dev, non_blocking=True))
            y_h.copy_(out.y, non_blocking=True)
            spl_h.copy_(out.spl, non_blocking=True)
            return out

        for i in range(args.warmup):
            e2e_step(i)
        torch.cuda.synchronize()
        vdist.barrier()
        e_ms = []
        for i in range(args.steps):
            flush.zero_()
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            e2e_step(args.warmup + i)
            b_.record(stream)
            b_.synchronize()
            e_ms.append(a.elapsed_time(b_))
        vdist.barrier()
        e_tot = vdist.max_over_ranks(sum(e_ms), dev)
        h2d = (w.prims.nbytes + w.b.nbytes + w.c_r.nbytes + B * 8)
        d2h = B * n_out * s * 16 + B * s * 8
        e2e = {"value": ws * B * args.steps / (e_tot * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "api": "paper_2310_04734_b200.sweep.ReducedSweep(host pinned arrays).sweep_device"}

    if rank != 0:
        return 0
    # FP64 roofline denominator: measured after the timed regions (the probe's
    # DMMA load does not precede the timed sweep)
    peak, peak_probes = probe_peak()
    # ---- parity of the headline's own outputs ----
    parity = parity_of_kept(w, kept) if kept else None
    del kept

    # ---- roofline of the dominant kernel ----
    fl = flops_per_freq(r, nprim, s, n_out)
    achieved = fl * B / (kern_avg_ms * 1e-3) / 1e12
    traffic = None
    tfile = ROOT / "profiles" / f"traffic_cfg5_r{r}.json"
    if tfile.exists():  # ncu --set full capture of the same kernel (profiles/), per launch
        try:
            traffic = json.loads(tfile.read_text())["dram_bytes_per_freq"] * B
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "rom_sweep_blocked_kernel" if path == 1 else "rom_sweep_small_kernel",
                "peak_source": "FP64 DMMA (mma.sync.m8n8k4.f64) throughput measured live by "
                               "vb_probe_fp64_peak on this GPU, median of 5 probes "
                               "(MEASURED_PEAKS.json has no FP64)",
                "peak_probes": peak_probes,
                "flops_per_freq": fl, "freqs_per_launch": B,
                "traffic_unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, ncu)"}

    orders = None
    if ws == 1 and not args.no_per_order:
        orders = per_order(args, dev, flush, peak, nsm)
        orders[f"r{r}"] = {"value": value, "frac": achieved / peak, "kernel_ms": kern_avg_ms,
                           "note": "headline (this line's value / roofline / parity)"}

    cpu = None
    if ws == 1 and not args.no_cpu:
        _threads = all_host_threads()
        _threads.__enter__()
        n = cpu_sample_size(w, args.cpu_budget_s)
        rng = np.random.default_rng(12)
        idx = np.sort(rng.choice(nF, n, replace=False))
        rate, dt = cpu_sweep_rate(w, w.freqs[idx])
        cpu = {"value": rate, "unit": UNIT, "cores": blas_threads(), "kind": "port",
               "sample": f"{n} random grid frequencies in {dt:.1f} s, oracle.mor.affine_sweep "
                         f"(numpy.linalg.solve = LAPACK zgesv per frequency, BLAS threads)"}
        lrate, ldt, ln = cpu_literal_rate(w)
        cpu["literal_path"] = {"value": lrate, "unit": UNIT, "sample": f"{ln} random grid frequencies in "
                               f"{ldt:.1f} s", "path": "oracle.mor.reduced_output = ReducedModel.output "
                               "(mor.py:73-98) with dense reduced providers and V = I"}
        cpu["cfg1_pipeline"] = cpu_cfg1_pipeline()
        _threads.__exit__(None, None, None)

    offline = None
    if ws == 1 and not args.no_offline:
        offline = offline_measurements(w, peak)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "complex128 (f64)",
        "data": "synthetic (seeded cfg5: K_r, D_r, M_r, 16 RHS, 50 outputs)",
        "config": bench_config(r, s, n_out, nprim, B, ws),
        "method": {"sweep_path": "blocked" if path == 1 else "shared-memory",
                   "l2_persistence": bool(args.l2_persist),
                   "timing": "CUDA events on the launching stream, L2 flushed before each timed step, "
                             "max over ranks"},
        "roofline": roofline, "parity": parity, "per_order": orders, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": int(launches_timed), "gpu_launches_incl_warmup": int(launches),
        "clocks": clocks, "offline": offline,
    }
    print(json.dumps(line), flush=True)
    return 0


def spawn_ranks(args, argv) -> int | None:
    """`python bench.py --gpus N` without a torchrun environment: re-launch
    this script under torch.distributed.run with N ranks on this node (one
    process per GPU) and return its exit code.  Under torchrun, WORLD_SIZE
    must equal --gpus."""
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is not None:
        if int(ws_env) != args.gpus:
            raise SystemExit(f"bench.py: WORLD_SIZE={ws_env} but --gpus {args.gpus}")
        return None
    if args.gpus <= 1:
        return None
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + list(argv)
    return subprocess.call(cmd)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--r", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=0, help="frequencies per step per rank")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-offline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    ap.add_argument("--cpu-step-s", type=float, default=4.0)
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-per-order", action="store_true")
    ap.add_argument("--orders", type=int, nargs="*", default=[256, 1024, 2048])
    ap.add_argument("--l2-persist", type=int, default=1, help="pin the primitives in L2 during the sweep")
    argv = sys.argv[1:] if argv is None else argv
    args = ap.parse_args(argv)
    rc = spawn_ranks(args, argv)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
