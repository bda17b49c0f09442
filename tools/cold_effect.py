"""Is the first timed sweep after an idle period slower (GPU / HBM power
state)?  Idle 0 / 30 / 90 s, then 8 timed steps each; memory and SM clocks
sampled by nvidia-smi during the loop."""
import subprocess
import sys
import threading
import time
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


def run(tag):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory",
                          "--format=csv,noheader,nounits", "-lms", "250"], stdout=subprocess.PIPE, text=True)
    lines = []
    th = threading.Thread(target=lambda: lines.extend(l.strip() for l in p.stdout), daemon=True)
    th.start()
    _, kern, _ = bench.sweep_timed(w, B, 8, 0, dev, flush)
    p.terminate()
    time.sleep(0.3)
    print(f"{tag}: kernel per step {[round(k, 1) for k in kern]}; clocks {lines[:3]} ... {lines[-2:]}", flush=True)


run("start")
for idle in (30, 90):
    time.sleep(idle)
    run(f"after {idle} s idle")
