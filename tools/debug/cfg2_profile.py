"""cfg2 pipeline: stage times, host cProfile and GPU kernel breakdown (warm)."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2310_04734_b200 import mor, workloads  # noqa: E402


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


def run(verbose=False):
    t0 = T()
    fom, lay = workloads.cfg2_model()
    t1 = T()
    V, tk, to = None, 0.0, 0.0
    for f0 in lay["points"]:
        a = T()
        Q, _ = mor.krylov_block_dev(fom, f0, lay["moments"])
        b = T()
        V = mor._orthonormalise(V, Q)
        c = T()
        tk += b - a
        to += c - b
    a = T()
    rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 500.0))
    mor.rom_sweep([rom], list(lay["freqs"]))
    b = T()
    if verbose:
        print(f"assembly {t1 - t0:.3f} krylov {tk:.3f} orth {to:.3f} proj+sweep {b - a:.3f} total {b - t0:.3f}")


run()
run(True)
pr = cProfile.Profile()
pr.enable()
run()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=18, max_name_column_width=60))
