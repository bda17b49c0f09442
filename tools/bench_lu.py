"""Whole-GPU dense complex LU (vb_zgetrf) throughput at FOM sizes: cfg1 n = 4641,
the reference benchmark n = 8102, 10k, cfg2 n = 20890 — CUDA-event timed,
flops = 8/3 n^3 (complex LU); plain kernel vs look-ahead kernel, and the
vendor library on the same matrix (torch.linalg.lu_factor -> cuSOLVER) as the
comparator."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2310_04734_b200 import _lib, solvers


def timed(fn, reps=3):
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


peak = _lib.probe_fp64_peak()
lib = _lib.load()
for n in [int(x) for x in sys.argv[1:]] or [4641, 8102, 10000, 20890]:
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(n, n, dtype=torch.complex128, device="cuda", generator=g)
    A.diagonal().add_(n ** 0.5)
    res = {}
    for la in (0, 1):
        lib.vb_set_lu_lookahead(la)
        res[la] = timed(lambda: solvers.DenseLU(A, copy=True))
    lib.vb_set_lu_lookahead(1)
    cus = timed(lambda: torch.linalg.lu_factor(A))
    fl = 8 / 3 * n ** 3
    print(f"n={n}: plain {res[0]:.1f} ms ({fl / res[0] / 1e9 / peak:.3f} of peak), look-ahead {res[1]:.1f} ms "
          f"({fl / res[1] / 1e9 / peak:.3f}), cuSOLVER {cus:.1f} ms; DMMA peak {peak:.1f} TF/s", flush=True)
    del A
    torch.cuda.empty_cache()
