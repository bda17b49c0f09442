"""cfg3 with per-element wall impedances (FDM-preconditioned GMRES full-order
solver): pipeline stage times, GMRES iterations, ROM certification on a
disjoint grid."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2310_04734_b200 import mor, workloads

t0 = time.perf_counter()
fom, lay = workloads.cfg3_model(per_element_z=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
fa = fom.factor(150.0)
x = fa.solve(fom.load_dev(150.0))
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"assembly {t1 - t0:.2f} s; one 8-RHS GMRES solve {t2 - t1:.3f} s, {fa.iterations} it, res {fa.last_residual:.1e}",
      flush=True)
V, _ = mor.krylov_basis(fom, lay["points"], lay["moments"], second_order=True, mimo=True)
torch.cuda.synchronize()
t3 = time.perf_counter()
rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 300.0))
res = mor.rom_sweep([rom], list(lay["freqs"]))
torch.cuda.synchronize()
t4 = time.perf_counter()
print(f"krylov+orth {t3 - t2:.2f} s (r = {V.shape[1]}); projection+sweep {t4 - t3:.2f} s", flush=True)
grid = list(lay["freqs"])
C = np.atleast_2d(fom.c_out)
worst = 0.0
for i in range(3, len(grid), 37):
    f = grid[i]
    X = fom.factor(f).solve(fom.load_dev(f)).cpu().numpy()
    _, e, _, _ = mor.relative_error((C @ X).ravel(), np.asarray(res.frf[i]).ravel())
    worst = max(worst, e)
print(f"eps_max over {len(range(3, len(grid), 37))} disjoint frequencies: {worst:.2e}", flush=True)
