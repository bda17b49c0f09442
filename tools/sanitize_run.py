"""Small end-to-end run for compute-sanitizer: both sweep paths, dense LU,
assembly (general + box + plate), SpMM/GEMM, FDM on a small box."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import __graft_entry__ as g
from paper_2310_04734_b200 import _lib, assembly, linalg, mor, sweep, workloads
from paper_2310_04734_b200.solvers import DenseLU

g.smoke()
dev = torch.device("cuda")
lib = _lib.load()
# blocked path at a non-multiple-of-64 order
w = workloads.cfg5(r=130, n_freq=40, s=3, n_out=5, seed=1)
out = sweep.rom_sweep_affine(sweep.as_ctensor(w.prims, dev), sweep.as_ctensor(w.alpha(), dev),
                             sweep.as_ctensor(w.b, dev), sweep.as_ctensor(w.c_r, dev), want_x=True)
torch.cuda.synchronize()
# assembly + LU + Krylov on a small box, FDM
fom, lay = workloads.cfg3_model(box=(0, 0, 0, 1.0, 0.8, 0.6), ne=(4, 3, 3), n_src=2, n_rec=5)
fom.prefer_fdm = True
Q = mor.krylov_blocks_mimo_dev(fom, 150.0, 3, second_order=True)
V = None
for q, _ in Q:
    V = mor._orthonormalise(V, q)
rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 300.0))
res = mor.rom_sweep([rom], [20.0, 100.0, 300.0])
lu = DenseLU(fom.operator_dense(77.0))
x = lu.solve(fom.load_dev(77.0))
Kb, Mb = assembly.assemble_helmholtz_box((0, 0, 0, 1, 1, 1), (3, 2, 2))
fom2, lay2 = workloads.cfg2_model(box=(0, 0, 0, 0.8, 0.6, 0.5), ne=(4, 3, 3), n_rec=4)
y = fom2.output(fom2.solve(123.0))
torch.cuda.synchronize()
print("sanitize run ok", V.shape, float(np.abs(y).max()))
