"""Kronecker apply vs row-group CSR SpMM on the cfg3 box Kgrad."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

from paper_2310_04734_b200 import assembly, linalg, workloads

K, _ = assembly.assemble_helmholtz_box(workloads.CFG3_BOX, workloads.CFG3_NE)
Kc = K.with_data(K.data)
linalg.row_groups(Kc)
n, nnz = K.n, K.nnz
for k in [int(a) for a in (sys.argv[1:] or ["2", "8", "32", "400"])]:
    X = torch.randn(n, k, dtype=torch.complex128, device="cuda")
    for name, A in (("kron", K), ("rg", Kc)):
        f = lambda: linalg.spmm(A, X)  # noqa: E731
        f(); torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record(); b.synchronize()
            best = min(best, a.elapsed_time(b))
        print(f"k={k:4d} {name:5s} {best:8.3f} ms")
