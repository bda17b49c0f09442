"""ROM accuracy at the reference's certification tolerance (tests/test_acceptance.py:
272-305: eps_max <= tol = 1e-2 on frequencies disjoint from the candidate /
expansion set): for cfg1, cfg2 and cfg3 build the window basis, sweep, and
compare the ROM outputs with GPU full-order solves (residual <= 1e-10) on a
disjoint grid (every `stride`-th grid frequency, expansion points excluded).
Prints one JSON object per config."""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch


class Settings:
    def __init__(self, tol, max_points, moments_per_point, candidate_stride, windows="auto"):
        self.tol, self.max_points, self.moments_per_point = tol, max_points, moments_per_point
        self.candidate_stride, self.windows = candidate_stride, windows


def eps_disjoint(fom, V, freqs, window, points, stride):
    from paper_2310_04734_b200 import mor
    rom = mor.ReducedModel(fom=fom, V=V, window=window)
    ver = [f for f in freqs[::stride] if f not in set(points)]
    y, _, _, info = rom.sweep(ver)
    yr = y.cpu().numpy()
    C = np.atleast_2d(fom.c_out)
    worst, wf, worst_n, wfn = 0.0, None, 0.0, None
    for i, f in enumerate(ver):
        X = fom.factor(f).solve(fom.load_dev(f)).cpu().numpy()
        yf = C @ X
        _, e, _, _ = mor.relative_error(yf.ravel(), yr[i].ravel())
        en = float(np.linalg.norm(yf - yr[i]) / np.linalg.norm(yf))
        if e > worst:
            worst, wf = e, f
        if en > worst_n:
            worst_n, wfn = en, f
    return worst, wf, len(ver), worst_n, wfn


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="*", default=["cfg1", "cfg2", "cfg3"])
    ap.add_argument("--stride", type=int, default=7)
    ap.add_argument("--points", type=str, default="")
    ap.add_argument("--moments", type=int, default=0)
    ap.add_argument("--greedy", action="store_true")
    ap.add_argument("--tol", type=float, default=1e-2)
    ap.add_argument("--max-points", type=int, default=12)
    ap.add_argument("--cand-stride", type=int, default=10)
    a = ap.parse_args()
    from paper_2310_04734_b200 import mor, workloads
    for cfg in a.configs:
        t0 = time.perf_counter()
        if cfg == "cfg1":
            fom, lay = workloads.cfg1_model(fdm=True)
            kw = dict(second_order=True)
            win = (20.0, 200.0)
        elif cfg == "cfg2":
            fom, lay = workloads.cfg2_model()
            kw = {}
            win = (20.0, 500.0)
        else:
            fom, lay = workloads.cfg3_model()
            kw = dict(second_order=True, mimo=True)
            win = (20.0, 300.0)
        pts = [float(p) for p in a.points.split(",")] if a.points else list(lay["points"])
        m = a.moments or lay["moments"]
        if a.greedy:
            st = Settings(tol=a.tol, max_points=a.max_points, moments_per_point=m, candidate_stride=a.cand_stride)
            rom = mor.greedy_expand(fom, list(lay["freqs"]), st, win, second_order=kw.get("second_order", False))
            V, pts = rom.V, [float(p) for p in rom.expansion_points]
        else:
            V, _ = mor.krylov_basis(fom, pts, m, **kw)
        torch.cuda.synchronize()
        tb = time.perf_counter() - t0
        e, wf, nv, en, wfn = eps_disjoint(fom, V, list(lay["freqs"]), win, pts, a.stride)
        print(json.dumps({"config": cfg, "r": int(V.shape[1]), "points": pts, "moments": m, "eps_max": e,
                          "at_hz": wf, "eps_max_normwise": en, "normwise_at_hz": wfn, "n_verify": nv,
                          "build_s": tb}), flush=True)


if __name__ == "__main__":
    main()
