"""One dense LU factorisation (vb_zgetrf) for ncu captures: warm-up + profiled."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2310_04734_b200 import solvers

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(n, n, dtype=torch.complex128, device="cuda", generator=g)
A.diagonal().add_(n ** 0.5)
for _ in range(2):
    lu = solvers.DenseLU(A, copy=True)
torch.cuda.synchronize()
print("ok", n, lu.info)
