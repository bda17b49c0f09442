"""One cfg3 pipeline run after a warm-up (for ncu launch lists)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_04734_b200 import mor, workloads  # noqa: E402


def run():
    fom, lay = workloads.cfg3_model()
    V = None
    for f0 in lay["points"]:
        for Q, _ in mor.krylov_blocks_mimo_dev(fom, f0, lay["moments"], second_order=True):
            V = mor._orthonormalise(V, Q)
    rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 300.0))
    rom._projected()
    mor.rom_sweep([rom], list(lay["freqs"]))
    torch.cuda.synchronize()


run()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=60))
