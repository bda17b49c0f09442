"""vb_zgetrs (triangular solves from vb_zgetrf factors) at FOM sizes, 1 and 8
right-hand sides: CUDA-event timed, residual checked."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2310_04734_b200 import solvers

for n in [int(x) for x in sys.argv[1:]] or [3565, 4641, 10000]:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(n, n, dtype=torch.complex128, device="cuda", generator=g)
    A.diagonal().add_(n ** 0.5)
    lu = solvers.DenseLU(A, copy=True)
    for s in (1, 8):
        B = torch.randn(n, s, dtype=torch.complex128, device="cuda", generator=g)
        X = lu.solve(B, check=False)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            X = lu.solve(B, check=False)
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        res = float(torch.linalg.norm(A @ X - B) / torch.linalg.norm(B))
        gbs = n * n * 16 / (best * 1e-3) / 1e9
        print(f"n={n} nrhs={s}: {best:.3f} ms  (factor bytes {gbs:.0f} GB/s)  residual {res:.2e}")
