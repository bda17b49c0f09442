import sys, math, numpy as np, torch
sys.path.insert(0, '.')
from paper_2310_04734_b200 import workloads, linalg
fom, lay = workloads.cfg3_model()
Kg = lay["Kg"]
S = Kg.to_scipy()
print("nnz", S.nnz, Kg.nnz, S.shape)
rng = np.random.default_rng(0)
x = rng.standard_normal((fom.n, 3)) + 1j * rng.standard_normal((fom.n, 3))
xd = torch.as_tensor(x, device="cuda")
yg = linalg.spmm(Kg, xd).cpu().numpy()
yh = S @ x
print("spmm k=3 rel err", np.abs(yg - yh).max() / np.abs(yh).max())
yg1 = linalg.spmm(Kg, xd[:, 0].contiguous()).cpu().numpy()
print("spmv rel err", np.abs(yg1 - yh[:, 0]).max() / np.abs(yh).max())
x8 = torch.as_tensor(rng.standard_normal((fom.n, 8)) + 0j, device="cuda")
y8 = linalg.spmm(Kg, x8).cpu().numpy()
print("spmm k=8 rel err", np.abs(y8 - S @ x8.cpu().numpy()).max() / np.abs(y8).max())
# indptr sanity
ip = Kg.indptr.cpu().numpy(); print("indptr last", ip[-1], "monotone", np.all(np.diff(ip) >= 0))
