"""Wall-clock split of the cfg3 pipeline (model build / Krylov basis /
projection + sweep), warm, median of 3."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2310_04734_b200 import mor, workloads


def stages():
    t = [time.perf_counter()]
    fom, lay = workloads.cfg3_model()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    V, _ = mor.krylov_basis(fom, lay["points"], lay["moments"], second_order=True, mimo=True)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 300.0))
    rom._projected()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    mor.rom_sweep([rom], list(lay["freqs"]))
    torch.cuda.synchronize(); t.append(time.perf_counter())
    return np.diff(t)


stages()
res = np.median([stages() for _ in range(3)], axis=0)
print("model %.3f  krylov+orth %.3f  projection %.3f  sweep %.3f  total %.3f s" % (*res, res.sum()))
import cProfile, pstats  # noqa: E401,E402
pr = cProfile.Profile()
pr.enable()
fom, lay = workloads.cfg3_model()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
