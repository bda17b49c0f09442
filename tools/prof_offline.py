"""Offline-stage kernels at cfg3 size for ncu captures: structured box CSR
assembly and CSR SpMM (k = 32), each run twice (warm-up + profiled)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2310_04734_b200 import assembly, linalg, workloads

box, ne = workloads.CFG3_BOX, workloads.CFG3_NE
for _ in range(2):
    K, M = assembly.assemble_helmholtz_box(box, ne)
torch.cuda.synchronize()
X = torch.randn(K.n, 32, dtype=torch.complex128, device="cuda")
for _ in range(2):
    Y = linalg.spmm(K, X)
torch.cuda.synchronize()
print("ok", K.n, K.nnz, float(Y.abs().sum()))
