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


def run_reference(args):
    """--impl reference: the reference's CPU path (oracle port; the reference is
    pure Python and cannot travel to the GPU box) on the host cores."""
    from paper_2310_04734_b200 import dist as vdist, workloads
    rank, ws, _ = vdist.world()
    if rank != 0:
        return 0
    w = workloads.cfg5(r=args.r)
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
        "config": {"workload": f"cfg5_r{args.r}", "r": args.r, "rhs": w.b.shape[1],
                   "n_out": w.c_r.shape[0], "freqs_per_step": n_per_step,
                   "grid": "linspace(1,1000,100000) (seeded random sample per step)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{n_per_step} random grid frequencies per step, numpy.linalg.solve "
                                   f"(LAPACK zgesv) per frequency, BLAS threads={cores}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def offline_measurements(w):
    """Secondary numbers (not the headline): the other stages of the MOR chain at
    BASELINE sizes, CUDA-event timed — cfg3 assembly / SpMM / projection / FDM
    solve (tools/bench_offline.py) and the cfg1 pipeline end to end."""
    import importlib.util
    import torch
    spec = importlib.util.spec_from_file_location("bench_offline", ROOT / "tools" / "bench_offline.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    out = mod.measure()
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

    def timed_twice(fn):
        """(first run, warm run) wall clock incl. host orchestration; the warm
        run is the reported number (first runs include one-off module loading,
        thread-pool and allocator warm-up)."""
        ts = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return ts, res

    (t1, t1w), (_, V) = timed_twice(lambda: cfg1(False))
    out["cfg1_pipeline_s"], out["cfg1_pipeline_first_s"], out["cfg1_r"] = t1w, t1, int(V.shape[1])
    out["cfg1_note"] = ("GPU assembly + 4 dense LUs (n=4641, the 4 expansion points concurrent on their own "
                        "streams) + 2nd-order Krylov + CGS2 + projection + 181-frequency sweep + SPL, wall clock "
                        "incl. host orchestration (warm run; *_first_s = first run in the process)")
    (t1, t1w), (_, V) = timed_twice(lambda: cfg1(True))
    out["cfg1_pipeline_fdm_s"], out["cfg1_pipeline_fdm_first_s"], out["cfg1_fdm_r"] = t1w, t1, int(V.shape[1])
    (t2, t2w), (fom, V) = timed_twice(cfg2)
    out["cfg2_pipeline_s"], out["cfg2_pipeline_first_s"] = t2w, t2
    out["cfg2_n"], out["cfg2_r"] = int(fom.n), int(V.shape[1])
    out["cfg2_note"] = ("GPU plate+cavity assembly (n=20890) + 6 Schur-complement (plate) / fast-diagonalisation "
                        "(cavity) factorisations with refinement (expansion points concurrent) + Krylov + CGS2 + "
                        "projection + batched plane-wave RHS + 961-frequency sweep + SPL")
    (t3, t3w), (fom, V) = timed_twice(cfg3)
    out["cfg3_pipeline_s"], out["cfg3_pipeline_first_s"] = t3w, t3
    out["cfg3_n"], out["cfg3_r"] = int(fom.n), int(V.shape[1])
    out["cfg3_note"] = ("GPU box assembly (n=376431) + fast-diagonalisation FOM solves at 5 points x 10 "
                        "second-order moments x 8 sources + block CGS2 + Kronecker-apply projection + "
                        "1121-frequency sweep (8 RHS) + SPL")
    return out


def run_ours(args):
    import torch
    from paper_2310_04734_b200 import _lib, dist as vdist, sweep, workloads

    rank, ws, local = vdist.init()
    _lib.require_cuda()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _lib.load()
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count

    w = workloads.cfg5(r=args.r)
    r, s, n_out, nprim = w.r, w.b.shape[1], w.c_r.shape[0], w.prims.shape[0]
    B = args.batch or 16 * nsm
    nF = len(w.freqs)
    freqs_dev = torch.from_numpy(w.freqs).to(dev)

    def step_freqs(step):
        # rank-disjoint slices walking the 100k grid (weak scaling)
        start = ((step * ws + rank) * B) % nF
        idx = (torch.arange(B, device=dev) + start) % nF
        return freqs_dev[idx]

    rs = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds, device=dev)
    flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)
    path = lib.vb_rom_sweep_path(r, nprim, s, n_out)
    stream = torch.cuda.current_stream(dev)

    def one_step(step, ev=None):
        f = step_freqs(step)
        alpha = rs.alpha(f)
        if ev is not None:
            ev[0].record(stream)
        out = sweep.rom_sweep_affine(rs.P, alpha, rs.b, rs.c, want_y=True, want_spl=True)
        if ev is not None:
            ev[1].record(stream)
        if ws > 1:
            vdist.gather_rows(out.spl, B * ws, ws)
        return out

    for i in range(args.warmup):
        one_step(i)
    torch.cuda.synchronize()
    sweep.raise_if_singular(one_step(0).info)

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    vdist.barrier()
    torch.cuda.synchronize()
    n0 = _lib.launch_count()
    for i in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        e = evs[i]
        e[0].record(stream)
        one_step(args.warmup + i, ev=(e[2], e[3]))
        e[1].record(stream)
    torch.cuda.synchronize()
    vdist.barrier()
    launches = _lib.launch_count() - n0
    clocks = sampler.stop() if sampler else None
    step_ms = [e[0].elapsed_time(e[1]) for e in evs]
    kern_ms = [e[2].elapsed_time(e[3]) for e in evs]
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
    # ---- roofline of the dominant kernel ----
    peak = _lib.probe_fp64_peak()
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
                               "vb_probe_fp64_peak on this GPU (MEASURED_PEAKS.json has no FP64)",
                "flops_per_freq": fl, "freqs_per_launch": B,
                "traffic_unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, ncu)"}

    cpu = None
    if ws == 1 and not args.no_cpu:
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

    offline = None
    if ws == 1 and not args.no_offline:
        offline = offline_measurements(w)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "complex128 (f64)",
        "data": "synthetic (seeded cfg5: K_r, D_r, M_r, 16 RHS, 50 outputs)",
        "config": {"workload": f"cfg5_r{r}", "r": r, "rhs": s, "n_out": n_out, "n_prim": nprim,
                   "freqs_per_step_per_rank": B,
                   "grid": "linspace(1,1000,100000), rank-disjoint slices",
                   "sweep_path": "blocked" if path == 1 else "shared-memory",
                   "l2": "flushed between timed steps (512 MiB write)",
                   "parallelism": f"frequency-sharded x{ws}"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clocks, "offline": offline,
    }
    print(json.dumps(line), flush=True)
    return 0


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
    args = ap.parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
