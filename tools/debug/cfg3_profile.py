"""cProfile of one warm cfg3 pipeline run (host-side hot spots)."""
import cProfile
import pstats
import sys
import time

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
t = time.perf_counter()
run()
print("warm", time.perf_counter() - t)
pr = cProfile.Profile()
pr.enable()
run()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
