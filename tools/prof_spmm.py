"""CSR SpMM at cfg3 size (general CSR of the box Kgrad, n = 376,431, nnz = 23.3M)
for ncu captures: k = 8 (sub-warp kernel), k = 32 and 400 (row-group kernel),
each run twice (warm-up + profiled)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2310_04734_b200 import assembly, linalg, workloads

box, ne = workloads.CFG3_BOX, workloads.CFG3_NE
K, _ = assembly.assemble_helmholtz_box(box, ne)
K = K.with_data(K.data)          # drop the Kronecker form: the general CSR path
linalg.row_groups(K)
for k in [int(a) for a in (sys.argv[1:] or ["8", "32", "400"])]:
    X = torch.randn(K.n, k, dtype=torch.complex128, device="cuda")
    for _ in range(2):
        Y = linalg.spmm(K, X)
    torch.cuda.synchronize()
    print("ok", k, K.n, K.nnz, float(Y.abs().sum()))
