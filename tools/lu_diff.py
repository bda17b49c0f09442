"""Where do the plain and look-ahead LU factors differ?"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2310_04734_b200 import _lib
from paper_2310_04734_b200.solvers import DenseLU

lib = _lib.load()
for n in (700, 3001):
    rng = np.random.default_rng(n + 3)
    A = torch.as_tensor(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)), device="cuda")
    outs = []
    for la in (0, 1, 1, 0):
        lib.vb_set_lu_lookahead(la)
        lu = DenseLU(A, copy=True)
        torch.cuda.synchronize()
        outs.append(lu.A.cpu().numpy())
    lib.vb_set_lu_lookahead(1)
    for a, b, name in ((outs[0], outs[3], "plain vs plain"), (outs[1], outs[2], "la vs la"), (outs[0], outs[1], "plain vs la")):
        d = np.abs(a - b)
        idx = np.argwhere(d > 0)
        print(n, name, "ndiff", len(idx), "max", d.max(), "rel", d.max() / np.abs(a).max(),
              "rows", (idx[:, 0].min(), idx[:, 0].max()) if len(idx) else None,
              "cols", (idx[:, 1].min(), idx[:, 1].max()) if len(idx) else None)
