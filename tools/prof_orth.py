"""Time the cfg3 basis build stage by stage (CUDA-event + wall clock): FDM
factorisations, MIMO Krylov moments, and the _orthonormalise appends, with
the per-call split of the appends.  Prints one JSON object."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch


def _grouped(blocks):
    from paper_2310_04734_b200 import mor
    V = None
    for p in range(0, len(blocks), 8):  # the 8 source blocks of each expansion point together
        V = mor.orthonormalise_blocks(V, blocks[p:p + 8])
    return V


def main():
    from paper_2310_04734_b200 import mor, workloads
    fom, lay = workloads.cfg3_model()
    out = {}
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        blocks = []
        for f0 in lay["points"]:
            blocks += [Q for Q, _ in mor.krylov_blocks_mimo_dev(fom, f0, lay["moments"], second_order=True)]
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        V = None
        per = []
        for Q in blocks:
            a = time.perf_counter()
            V = mor._orthonormalise(V, Q)
            torch.cuda.synchronize()
            per.append(time.perf_counter() - a)
        t2 = time.perf_counter()
        if "--grouped" in sys.argv:
            torch.cuda.synchronize()
            a = time.perf_counter()
            V2 = _grouped(blocks)
            torch.cuda.synchronize()
            out["grouped_s"] = time.perf_counter() - a
            out["grouped_r"] = int(V2.shape[1])
        out.update({"krylov_s": t1 - t0, "orthonormalise_s": t2 - t1, "r": int(V.shape[1]),
                    "per_block_ms": [round(1e3 * p, 2) for p in per]})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
