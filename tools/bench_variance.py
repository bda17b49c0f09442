"""Where does the spread between bench.py's device-resident `value` and its
e2e number come from?  Runs the bench's timed sweep loop several times in a
row (L2 persistence on / off) and the e2e loop, printing kernel ms per step."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import bench
from paper_2310_04734_b200 import sweep, workloads


def main():
    dev = torch.device("cuda", 0)
    w = workloads.cfg5(r=1024)
    B = 16 * torch.cuda.get_device_properties(dev).multi_processor_count
    flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)
    for rep in range(3):
        for persist in (0, 1):
            ctx = sweep.persist_primitives_in_l2() if persist else None
            if ctx:
                ctx.__enter__()
            step_ms, kern_ms, _ = bench.sweep_timed(w, B, 5, 3, dev, flush)
            if ctx:
                ctx.__exit__(None, None, None)
            print(f"rep {rep} persist {persist}: step {np.mean(step_ms):.2f} ms kernel {np.mean(kern_ms):.2f} ms "
                  f"-> {B / np.mean(step_ms) * 1e3:.0f} freq/s; per step {[round(x, 1) for x in kern_ms]}",
                  flush=True)
    # no flush between steps
    step_ms, kern_ms, _ = bench.sweep_timed(w, B, 5, 3, dev, torch.empty(1, dtype=torch.uint8, device=dev))
    print(f"no flush: kernel {np.mean(kern_ms):.2f} ms", flush=True)


if __name__ == "__main__":
    main()
