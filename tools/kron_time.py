"""Time the matrix-free Kronecker apply (vb_kron3_apply) at cfg3 size for a few
column counts, and check it against the CSR SpMM of the same primitive."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2310_04734_b200 import assembly, linalg, workloads


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


K, _ = assembly.assemble_helmholtz_box(workloads.CFG3_BOX, workloads.CFG3_NE)
n = K.n
tag = Path(os.environ.get("VB_LIB_PATH", "default")).stem
for k in (8, 32, 400):
    X = torch.randn(n, k, dtype=torch.complex128, device="cuda")
    t = timed(lambda: linalg.spmm(K, X))
    Y = linalg.spmm(K, X)
    R = linalg.spmm(K.with_data(K.data), X, path="csr")
    err = float((Y - R).abs().max() / R.abs().max())
    print(f"{tag} k={k}: {t:.3f} ms  {2 * n * k * 16 / (t * 1e-3) / 1e9:.0f} GB/s (X+Y)  err {err:.1e}", flush=True)
