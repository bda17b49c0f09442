"""Kernel / host split of one 8-RHS GMRES solve on cfg3 with per-element walls."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2310_04734_b200 import workloads

fom, lay = workloads.cfg3_model(per_element_z=True)
b = fom.load_dev(150.0)
fa = fom.factor(150.0)
fa.solve(b)
torch.cuda.synchronize()
t0 = time.perf_counter()
fa2 = fom.factor(151.0)
torch.cuda.synchronize()
t1 = time.perf_counter()
x = fa2.solve(b)
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"factor (host eig + uploads) {1e3 * (t1 - t0):.1f} ms; solve {1e3 * (t2 - t1):.1f} ms, {fa2.iterations} it, "
      f"restarts {fa2.stats.restarts}, history {fa2.stats.history}")
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    fa2.solve(b)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15, max_name_column_width=55))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=12, max_name_column_width=55))
