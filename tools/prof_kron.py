"""cfg3-size Kronecker box apply (k = 400) for ncu: warm-up + profiled launch."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2310_04734_b200 import assembly, linalg, workloads

K, _ = assembly.assemble_helmholtz_box(workloads.CFG3_BOX, workloads.CFG3_NE)
k = int(sys.argv[1]) if len(sys.argv) > 1 else 400
X = torch.randn(K.n, k, dtype=torch.complex128, device="cuda")
for _ in range(2):
    Y = linalg.spmm(K, X)
torch.cuda.synchronize()
print("ok", float(Y.abs().sum()))
