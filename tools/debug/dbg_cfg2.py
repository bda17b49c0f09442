import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, "tests"); import test_plate_gpu as T
from oracle import mor as omor, shell
from paper_2310_04734_b200 import mor, plate, workloads
import torch
fom, lay, prims = T._small("cuda")
ofom = shell.cfg2_fom(prims, lay["rec"], workloads.AIR_RHO, workloads.AIR_C, plate.eta_cfg2)
A = ofom.operator(60.0).toarray(); print("cond A(60)", np.linalg.cond(A))
pts, m = (60.0, 220.0, 380.0), 4
V, Vo = None, None
for f0 in pts:
    Q, _ = mor.krylov_block_dev(fom, f0, m); V = mor._orthonormalise(V, Q)
    Qo, _ = omor.krylov_block(ofom, f0, m); Vo = omor.orthonormalise(Vo, Qo)
    Qh = Q.cpu().numpy()
    print(f0, "block span diff", np.linalg.norm(Qo - Qh @ (Qh.conj().T @ Qo)))
Vh = V.cpu().numpy()
print("V span diff", np.linalg.norm(Vo - Vh @ (Vh.conj().T @ Vo)))
rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 500.0))
grid = list(np.arange(20.0, 500.1, 40.0))
res = mor.rom_sweep([rom], grid)
for i, f in enumerate(grid):
    yo = omor.reduced_output(ofom, Vo, f); yg = omor.reduced_output(ofom, Vh, f)
    e1 = omor.relative_error(yo, res.frf[i])[1]; e2 = omor.relative_error(yg, res.frf[i])[1]
    yf = ofom.output(ofom.solve(f)); e3 = omor.relative_error(yf, yo)[1]
    print(f, "gpu vs oracle-basis %.2e  gpu vs same-basis %.2e  rom err %.2e" % (e1, e2, e3))
