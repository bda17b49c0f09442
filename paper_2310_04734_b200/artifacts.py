"""Artefact drop-in for `vibrofem mor {build,sweep,verify}`:
the `rom.npz` container (ROM_FORMAT_VERSION = 1, vibrofem/cli.py:221-248) and
the CSV writers (cli.py:39-50, 259-303) — byte-compatible formats, so files
written here load in the reference and vice versa."""

from __future__ import annotations

import csv
import math
from pathlib import Path

import numpy as np

ROM_FORMAT_VERSION = 1  # cli.py:32


def _fmt(value) -> str:
    """cli.py:39-42: floats as .12e, everything else str()."""
    if isinstance(value, (float, np.floating)):
        return format(float(value), ".12e")
    return str(value)


def write_csv(path, header, rows):
    """cli.py:45-50 (LF line endings, utf-8)."""
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(header)
        for row in rows:
            w.writerow([_fmt(v) for v in row])


def _host(V):
    try:
        import torch
        if isinstance(V, torch.Tensor):
            return V.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(V)


def save_roms(path, roms):
    """cli.py:221-231."""
    payload = {"version": np.array(ROM_FORMAT_VERSION), "n_windows": np.array(len(roms)),
               "windows": np.array([r.window for r in roms])}
    for k, r in enumerate(roms):
        payload[f"V{k}"] = _host(r.V)
        payload[f"points{k}"] = np.array(r.expansion_points)
        payload[f"errlog{k}"] = np.array(r.error_log)
        payload[f"flags{k}"] = np.array([r.converged, r.stalled, r.budget_exhausted])
    np.savez_compressed(path, **payload)


def load_roms(path, fom) -> list:
    """cli.py:234-248; raises ValueError (the reference's ConfigError) on a
    version mismatch."""
    from .mor import ReducedModel
    data = np.load(path)
    if int(data["version"]) != ROM_FORMAT_VERSION:
        raise ValueError(f"unsupported ROM container version in {path}")
    roms = []
    for k in range(int(data["n_windows"])):
        flags = data[f"flags{k}"]
        roms.append(ReducedModel(fom=fom, V=data[f"V{k}"], window=tuple(data["windows"][k]),
                                 expansion_points=list(data[f"points{k}"]),
                                 error_log=[tuple(e) for e in data[f"errlog{k}"]],
                                 converged=bool(flags[0]), stalled=bool(flags[1]),
                                 budget_exhausted=bool(flags[2])))
    return roms


def write_build_artifacts(out, roms) -> list:
    """`mor build` outputs (cli.py:256-269): rom.npz, rom_summary.csv, windows.csv."""
    out = Path(out)
    rom_path = out / "rom.npz"
    save_roms(rom_path, roms)
    summary = out / "rom_summary.csv"
    write_csv(summary, ["window_lo_hz", "window_hi_hz", "r", "n_points", "eps_max_candidates", "converged"],
              [[r.window[0], r.window[1], r.r, len(r.expansion_points),
                max((e for _, e in r.error_log), default=0.0), int(r.converged)] for r in roms])
    windows = out / "windows.csv"
    write_csv(windows, ["window_lo_hz", "window_hi_hz"], [[r.window[0], r.window[1]] for r in roms])
    return [rom_path, summary, windows]


def write_sweep_artifacts(out, sweep) -> list:
    """`mor sweep` outputs (cli.py:270-282): frf_mor.csv (scalar outputs, the
    reference format) or spl_mor.csv (multi-output receivers: mean SPL per
    frequency, solvers.py:334-338), and timings_mor.csv."""
    out = Path(out)
    files = []
    if all(np.ndim(y) == 0 for y in sweep.frf):
        frf = out / "frf_mor.csv"
        write_csv(frf, ["f_hz", "re_p", "im_p", "abs_db", "window"],
                  [[f, complex(y).real, complex(y).imag, 20.0 * np.log10(max(abs(y), 1e-300) / 20e-6), w]
                   for f, y, w in zip(sweep.freqs, sweep.frf, sweep.window_index)])
        files.append(frf)
    else:
        spl = out / "spl_mor.csv"
        write_csv(spl, ["f_hz", "spl_db", "window"],
                  [[f, float(np.ravel(s)[0]), w] for f, s, w in zip(sweep.freqs, sweep.spl, sweep.window_index)])
        files.append(spl)
    timings = out / "timings_mor.csv"
    write_csv(timings, ["f_hz", "solve_time_s"], list(zip(sweep.freqs, sweep.rom_time)))
    files.append(timings)
    return files


def write_verify_artifacts(out, ver, eps, sweep) -> list:
    """`mor verify` outputs (cli.py:283-298)."""
    out = Path(out)
    err = out / "error_mor.csv"
    write_csv(err, ["f_hz", "rel_error"], list(zip(ver, eps)))
    speed = out / "speedup_mor.csv"
    write_csv(speed, ["f_hz", "rom_time_s", "direct_time_s"], list(zip(ver, sweep.rom_time, sweep.fom_time)))
    return [err, speed]
