"""cfg4 kernels for ncu: the reduced-resolution fuselage model's GPU assembly
(facet shells, chain-rule hex27, CSR pattern/gather), one plane-block
factorisation and a few solves (batched block GEMVs).  Prints CUDA-event
times of the element kernels and of one solve."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2310_04734_b200 import fuselage as fz

dev = torch.device("cuda:0")
spec = fz.FuselageSpec()
fom, info = fz.fuselage_model(spec, dev)
T = info["tables"]
props = torch.as_tensor(np.array([spec.skin, spec.lining, spec.floor, spec.frame, spec.stringer]), device=dev)
sx = torch.as_tensor(T.s_xyz, device=dev)
sc = torch.as_tensor(T.sh_conn.astype(np.int32), device=dev)
sm = torch.as_tensor(T.sh_mat, device=dev)
fx = torch.as_tensor(T.f_xyz, device=dev)
cc = torch.as_tensor(T.cab_conn.astype(np.int32), device=dev)


def ev_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


t_sh = ev_time(lambda: fz.shell_elements(sx, sc, sm, props, spec.drill))
t_hx = ev_time(lambda: fz.helmholtz_chain(fx, cc))
fac = fom.factor(137.0)
b = fom.load_dev(137.0)
t_solve = ev_time(lambda: fac.lu.solve(b))
print(f"shells {len(T.sh_conn)}: {t_sh:.3f} ms; cabin hex27 {len(T.cab_conn)}: {t_hx:.3f} ms; "
      f"plane-block solve (no refinement): {t_solve:.3f} ms")
