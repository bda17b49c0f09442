"""Quick CUDA-event timing of the CSR SpMM paths at cfg3 size (general CSR)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch

from paper_2310_04734_b200 import assembly, linalg, workloads

K, _ = assembly.assemble_helmholtz_box(workloads.CFG3_BOX, workloads.CFG3_NE)
K = K.with_data(K.data)
linalg.row_groups(K)
n, nnz = K.n, K.nnz
for k in [int(a) for a in (sys.argv[1:] or ["1", "8", "32", "64", "400"])]:
    X = torch.randn(n, k, dtype=torch.complex128, device="cuda")
    for path in ("csr", "rg"):
        f = lambda: linalg.spmm(K, X, path=path)  # noqa: E731
        f(); torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record(); b.synchronize()
            best = min(best, a.elapsed_time(b))
        alg = nnz * 12 + 2 * n * k * 16
        print(f"k={k:4d} {path:5s} {best:8.3f} ms  {alg / best / 1e6:7.0f} GB/s  {4 * nnz * k / best / 1e9:6.2f} TF/s")
