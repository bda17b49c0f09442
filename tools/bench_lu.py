"""Whole-GPU dense complex LU (vb_zgetrf) throughput at FOM sizes: cfg1 n = 4641,
10k, cfg2 n = 20890 — CUDA-event timed, flops = 8/3 n^3 (complex LU)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2310_04734_b200 import _lib, solvers

peak = _lib.probe_fp64_peak()
for n in [int(x) for x in sys.argv[1:]] or [4641, 10000, 20890]:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(n, n, dtype=torch.complex128, device="cuda", generator=g)
    A.diagonal().add_(n ** 0.5)
    lu = solvers.DenseLU(A, copy=True)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lu = solvers.DenseLU(A, copy=True)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    tf = 8 / 3 * n ** 3 / (best * 1e-3) / 1e12
    print(f"n={n}: {best:.1f} ms  {tf:.2f} TFLOP/s  {tf / peak:.3f} of DMMA peak {peak:.1f}")
    del A, lu
    torch.cuda.empty_cache()
