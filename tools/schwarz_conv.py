"""Convergence of GPU GMRES + additive Schwarz on the reference benchmark
(n = 8,102) for several overlaps / restart lengths: iterations, true residual
per restart, wall time."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2310_04734_b200.gmres import GmresFactor
from paper_2310_04734_b200.model_operator import load_operator_npz
from paper_2310_04734_b200.schwarz import AdditiveSchwarz

root = Path(__file__).resolve().parents[1]
fom, grid, op = load_operator_npz(root / "tests" / "golden" / "fuselage_slice.npz")
sets = [np.arange(o, o + s) for o, s in op.block_map.values()]
for ov in (1, 2, 4):
    asm = AdditiveSchwarz(fom, sets, overlap=ov)
    for f in (24.0, 410.0, 812.0):
        for restart in (50, 200):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fa = GmresFactor(fom, f, asm.factor(f), 1e-10, 800, restart)
            x = fa.solve(fom.load_dev(f), check=False)
            torch.cuda.synchronize()
            print(f"overlap {ov} f {f} restart {restart}: it {fa.iterations} res {fa.last_residual:.2e} "
                  f"{time.perf_counter() - t0:.2f} s hist {[f'{h:.1e}' for h in fa.stats.history]}", flush=True)
