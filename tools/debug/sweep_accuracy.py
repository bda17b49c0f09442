"""Max TF relative error / SPL difference of the blocked sweep vs the oracle
(numpy zgesv) on seeded cfg5 samples, and normwise backward errors."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import mor as omor
from paper_2310_04734_b200 import sweep, workloads
for r, nf in ((256, 16), (1024, 8), (2048, 3)):
    w = workloads.cfg5(r=r, n_freq=100_000)
    f = w.freqs[np.sort(np.random.default_rng(r).choice(100_000, nf, replace=False))]
    alpha = w.alpha(f)
    y_ref, spl_ref = omor.affine_sweep(w.prims, alpha, w.b, w.c_r)
    out = sweep.rom_sweep_affine(sweep.as_ctensor(w.prims, "cuda"), sweep.as_ctensor(alpha, "cuda"),
                                 sweep.as_ctensor(w.b, "cuda"), sweep.as_ctensor(w.c_r, "cuda"), want_x=True)
    y = out.y.cpu().numpy()
    rel = np.abs(y - y_ref) / np.abs(y_ref)
    P = sweep.as_ctensor(w.prims, "cuda"); B = sweep.as_ctensor(w.b, "cuda"); Al = sweep.as_ctensor(alpha, "cuda")
    be = 0.0
    for i in range(nf):
        A = torch.einsum("k,kij->ij", Al[i], P); X = out.x[i]
        be = max(be, float(torch.linalg.matrix_norm(A @ X - B) / (torch.linalg.matrix_norm(A) * torch.linalg.matrix_norm(X))))
    print(f"r={r}: max TF rel err {rel.max():.2e} (median {np.median(rel):.2e}), max |dSPL| "
          f"{np.abs(out.spl.cpu().numpy() - spl_ref).max():.2e} dB, max backward error {be:.2e}")
