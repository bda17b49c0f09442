import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2310_04734_b200.solvers import DenseLU
rng = np.random.default_rng(5)
for n in (60, 64, 100, 128, 150, 200, 300, 1000):
    A = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    lu = DenseLU(torch.as_tensor(A, device="cuda"), copy=True)
    for s in (1, 3):
        b = rng.standard_normal((n, s)) + 1j * rng.standard_normal((n, s))
        x = lu.solve(torch.as_tensor(b, device="cuda")).cpu().numpy()
        print(n, s, np.linalg.norm(A @ x - b) / np.linalg.norm(b))
