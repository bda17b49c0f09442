"""One reduced-sweep launch (cfg5 shapes) for ncu captures: warm-up launch, then the profiled one."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2310_04734_b200 import sweep, workloads

ap = argparse.ArgumentParser()
ap.add_argument("--r", type=int, default=1024)
ap.add_argument("--F", type=int, default=148)
a = ap.parse_args()
w = workloads.cfg5(r=a.r)
dev = torch.device("cuda:0")
rs = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds, device=dev)
f = torch.from_numpy(w.freqs[np.linspace(0, len(w.freqs) - 1, a.F).astype(int)]).to(dev)
for _ in range(2):
    out = rs.sweep_device(f)
torch.cuda.synchronize()
sweep.raise_if_singular(out.info)
print("ok", a.r, a.F, float(out.spl.mean()))
