"""The reference's full-order solve (scipy splu, vibrofem/mor.py:48-49 /
solvers.py:62-78) of the cfg4 model (n = 84,189) on the host cores, timed
next to the GPU plane-block factorisation of the same operator, with the
solutions compared.  Prints one JSON object."""
import json
import math
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import scipy.sparse.linalg as spl
import torch

from paper_2310_04734_b200 import fuselage as fz

f = float(sys.argv[1]) if len(sys.argv) > 1 else 137.0
fom, info = fz.fuselage_model(fz.FuselageSpec())
fom.factor(61.0)  # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
fac = fom.factor(f)
torch.cuda.synchronize()
t_gpu_factor = time.perf_counter() - t0
b = fom.load_dev(f)
x_gpu = fac.solve(b).cpu().numpy().ravel()
A = fom.operator(f).tocsc()
bh = fom.load(f)
t0 = time.perf_counter()
lu = spl.splu(A)
t_splu = time.perf_counter() - t0
t0 = time.perf_counter()
x_cpu = lu.solve(bh)
t_solve = time.perf_counter() - t0
res = float(np.linalg.norm(A @ x_cpu - bh) / np.linalg.norm(bh))
print(json.dumps({"n": int(fom.n), "nnz": int(A.nnz), "f_hz": f, "splu_s": t_splu, "splu_solve_s": t_solve,
                  "splu_fill_nnz": int(lu.L.nnz + lu.U.nnz), "splu_residual": res,
                  "gpu_factor_s": t_gpu_factor, "gpu_residual": fac.last_residual,
                  "rel_diff": float(np.linalg.norm(x_gpu - x_cpu) / np.linalg.norm(x_cpu)),
                  "host_cpus": os.cpu_count(), "note": "SuperLU is single-threaded"}))
