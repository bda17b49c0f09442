"""Krylov basis build, sequential vs concurrent expansion points (cfg1 dense LU, cfg2 Schur, cfg3 FDM MIMO)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2310_04734_b200 import mor, workloads  # noqa: E402


def T():
    torch.cuda.synchronize()
    return time.perf_counter()


for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg3"]:
    fom, lay = getattr(workloads, name + "_model")()
    so = name != "cfg2"
    mimo = name == "cfg3"
    for conc in (False, True, False, True):
        a = T()
        V, _ = mor.krylov_basis(fom, lay["points"], lay["moments"], second_order=so, mimo=mimo, concurrent=conc)
        b = T()
        print(f"{name} concurrent={conc}: {b - a:.3f} s  r={V.shape[1]}")
