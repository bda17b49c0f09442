"""Does the nvidia-smi clock sampler (bench.ClockSampler) slow the timed sweep?
Alternates timed loops with and without it."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import bench
from paper_2310_04734_b200 import workloads

dev = torch.device("cuda", 0)
w = workloads.cfg5(r=1024)
B = 16 * torch.cuda.get_device_properties(dev).multi_processor_count
flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)
for rep in range(3):
    for samp in (False, True):
        s = bench.ClockSampler(0) if samp else None
        if s:
            s.start()
        _, kern, _ = bench.sweep_timed(w, B, 5, 3, dev, flush)
        c = s.stop() if s else None
        print(f"rep {rep} sampler {samp}: kernel {np.mean(kern):.1f} ms {[round(k, 1) for k in kern]} {c}", flush=True)
