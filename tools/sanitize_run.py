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
# CSR SpMV / sub-warp / row-group SpMM (incl. a boundary matrix with empty rows)
import scipy.sparse as sp  # noqa: E402

from oracle import fe  # noqa: E402

A, _ = fe.kron_box((0, 0, 0, 1.2, 0.9, 0.7), 3, 2, 2)
A = sp.csr_matrix(A)
keep = np.zeros(A.shape[0])
keep[:20] = 1.0
for M in (A, sp.csr_matrix(sp.diags(keep) @ A @ sp.diags(keep))):
    M.eliminate_zeros()
    M.sort_indices()
    Ad = assembly.DeviceCSR(M.shape[0], torch.as_tensor(M.indptr.astype(np.int32), device=dev),
                            torch.as_tensor(M.indices.astype(np.int32), device=dev), torch.as_tensor(M.data, device=dev))
    for k in (1, 2, 5, 8, 13, 33, 70):
        X = torch.randn(M.shape[0], k, dtype=torch.complex128, device=dev)
        for path in ("csr", "rg"):
            linalg.spmm(Ad, X, 1.0 - 0.5j, 0.0, None, path=path)
# fused in-block Gram-Schmidt (drops + no_drop in place)
B = torch.randn(500, 7, dtype=torch.complex128, device=dev)
B[:, 3] = B[:, 1]
Qb = torch.empty_like(B)
nk, _ = linalg.block_gs(B.clone(), Qb, linalg.column_norms(B), 1e-10, 1e-4)
linalg.block_gs(Qb[:, :nk].contiguous(), Qb[:, :nk].contiguous(), no_drop=True)
# concurrent expansion points (streams + thread-local LU CTA cap)
fom1, lay1 = workloads.cfg1_model(box=(0, 0, 0, 1.0, 0.8, 0.6), ne=(3, 3, 2), n_rec=4)
V1, _ = mor.krylov_basis(fom1, [40.0, 90.0, 150.0], 3, second_order=True, concurrent=True)
# round 2: GPU GMRES (batched CGS kernels) on a per-element-impedance box,
# grouped appends (chunked block GS + Cholesky QR), CUDA-core row groups
fom3, lay3 = workloads.cfg3_model(box=(0, 0, 0, 1.0, 0.8, 0.6), ne=(4, 3, 3), n_src=2, n_rec=5, per_element_z=True)
xg = fom3.factor(140.0).solve(fom3.load_dev(140.0))
V3, _ = mor.krylov_basis(fom3, [60.0, 200.0], 3, second_order=True, mimo=True)
lib.vb_set_rg_spmm_mode(2)
linalg.spmm(Ad, torch.randn(Ad.n, 40, dtype=torch.complex128, device=dev), 1.0, 0.0, None, path="rg")
lib.vb_set_rg_spmm_mode(0)
torch.cuda.synchronize()
print("sanitize run ok", V.shape, V1.shape, V3.shape, float(np.abs(y).max()))
