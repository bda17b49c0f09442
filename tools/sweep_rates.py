"""Device-resident reduced-sweep throughput at several cfg5 orders (same timing
as bench.py: L2 flushed, CUDA events, kernel time), for A/B of library builds
(VB_LIB_PATH)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import bench
from paper_2310_04734_b200 import workloads

dev = torch.device("cuda", 0)
flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)
nsm = torch.cuda.get_device_properties(dev).multi_processor_count
tag = Path(os.environ.get("VB_LIB_PATH", "default")).stem
orders = [int(x) for x in sys.argv[1:]] or [256, 400, 1024, 2048]
out = []
for r in orders:
    w = workloads.cfg5(r=r)
    B = 16 * nsm
    steps = 6 if r <= 512 else (3 if r <= 1024 else 2)
    _, kern, kept = bench.sweep_timed(w, B, steps, 2, dev, flush, keep=True)
    fl = bench.flops_per_freq(r, 3, 16, 50)
    k = float(np.median(kern))
    par = bench.parity_of_kept(w, kept, n=16)
    out.append(f"r={r} {B / k * 1e3:.0f} freq/s frac {fl * B / (k * 1e-3) / 37.08e12:.3f} err {par['max_tf_rel_err']:.1e}")
print(tag, " | ".join(out), flush=True)
