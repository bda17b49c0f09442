"""Kernel-level split of the cfg3 basis build's orthonormalisation (torch
profiler / CUPTI activity records; kernel names from libvibro_b200.so):
GPU time per kernel vs the wall time of the appends."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
from torch.profiler import ProfilerActivity, profile


def main():
    from paper_2310_04734_b200 import mor, workloads
    fom, lay = workloads.cfg3_model()
    per = [[Q for Q, _ in mor.krylov_blocks_mimo_dev(fom, f0, lay["moments"], second_order=True)]
           for f0 in lay["points"]]
    groups, g = [], []
    for blocks in per:  # mor.krylov_basis grouping
        g += blocks
        if sum(Q.shape[1] for Q in g) >= mor.GROUP_COLS:
            groups.append(g)
            g = []
    if g:
        groups.append(g)
    V = None
    for g in groups:  # warm-up
        V = mor.orthonormalise_blocks(V, g)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        V = None
        for g in groups:
            V = mor.orthonormalise_blocks(V, g)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    print(f"wall {wall * 1e3:.1f} ms, r = {V.shape[1]}")
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))


if __name__ == "__main__":
    main()
