"""Overlapping additive Schwarz preconditioner with exact GPU LU per subdomain
— the reference's `AdditiveSchwarzPrecond` / `BlockJacobiPrecond`
(solvers.py:98-176: subdomains from a grouping of the physical domains,
`overlap` adjacency layers of the sparsity graph of A + A^T
(`_expand_overlap`, solvers.py:122-134), restricted or full combination) on
the device, as the preconditioner of the GPU GMRES (gmres.py) for models no
direct factorisation covers: general meshes beyond the dense-LU size, where
the box fast diagonalisation does not apply.

Per frequency the subdomain matrices A(f)[ext, ext] = sum_k alpha_k(f)
P_k[ext, ext] are assembled densely on the device from the affine model's CSR
primitives (sub-blocks sliced once on the host) and factored by the
whole-GPU LU (vb_zgetrf); an application gathers the residual's subdomain
rows, runs the subdomain solves and scatters the owned rows back
(restricted) or sums them (full).

Deviation: the overlap graph is the structural union of the primitives'
patterns, a superset of the reference's |A(f)| + |A(f)^T| (scipy's
K - w^2 M drops numerically cancelled entries); this only changes the
preconditioner, never the solution (GMRES residual <= 1e-10).
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import torch

from . import linalg
from .assembly import DeviceCSR
from .solvers import DenseLU

CDT = torch.complex128


def _expand_overlap(G: sp.csr_matrix, idx: np.ndarray, layers: int) -> np.ndarray:
    """`layers` adjacency layers around idx in the graph G (solvers.py:122-134)."""
    if layers == 0:
        return np.sort(idx)
    cur = np.zeros(G.shape[0], dtype=bool)
    cur[idx] = True
    for _ in range(layers):
        frontier = np.nonzero(cur)[0]
        cur[np.unique(G[frontier].indices)] = True
    return np.nonzero(cur)[0]


class AdditiveSchwarz:
    """Subdomain setup (once per model): index sets, overlap extension,
    per-term CSR sub-blocks on the device."""

    def __init__(self, fom, index_sets, overlap: int = 1, variant: str = "restricted"):
        if fom.affine is None:
            raise ValueError("AdditiveSchwarz needs an affine model (device CSR primitives)")
        if variant not in ("restricted", "full"):
            raise ValueError("variant must be 'restricted' or 'full'")
        n = fom.n
        sets = [np.asarray(s, dtype=np.int64) for s in index_sets]
        cov = np.concatenate(sets)
        if len(cov) != n or len(np.unique(cov)) != n:
            raise ValueError("grouping must partition all DoFs")  # solvers.py:104-106
        aff = fom.affine
        self.terms = [("K", t) for t in aff.K] + [("M", t) for t in aff.M] + [("D", t) for t in aff.D]
        host = [t.P.to_scipy() for _, t in self.terms]
        pat = None
        for H in host:
            S = sp.csr_matrix((np.ones(H.nnz), H.indices, H.indptr), shape=H.shape)
            pat = S if pat is None else pat + S
        G = (pat + pat.T).tocsr()
        self.fom, self.n, self.variant = fom, n, variant
        self.ext, self.own = [], []
        self.blocks = []          # per subdomain: [device CSR sub-block per term]
        dev = self.terms[0][1].P.data.device
        for base in sets:
            ext = _expand_overlap(G, base, overlap)
            inbase = np.zeros(n, dtype=bool)
            inbase[base] = True
            mask = inbase[ext]
            self.ext.append(torch.as_tensor(ext, device=dev))
            self.own.append((torch.as_tensor(np.nonzero(mask)[0], device=dev), torch.as_tensor(ext[mask], device=dev)))
            blk = []
            for H in host:
                Hs = H[ext][:, ext].tocsr()
                Hs.sort_indices()
                blk.append(DeviceCSR(len(ext), torch.as_tensor(Hs.indptr.astype(np.int32), device=dev),
                                     torch.as_tensor(Hs.indices.astype(np.int32), device=dev),
                                     torch.as_tensor(Hs.data, device=dev)))
            self.blocks.append(blk)

    def factor(self, f: float) -> "SchwarzFactor":
        return SchwarzFactor(self, f)


class SchwarzFactor:
    """The preconditioner at one frequency: dense GPU LU of every subdomain
    matrix A(f)[ext, ext]; `_apply_inverse(R)` = sum_d R_d^T A_d^-1 R_d R."""

    def __init__(self, asm: AdditiveSchwarz, f: float):
        self.asm, self.f = asm, f
        w = 2.0 * math.pi * f
        scale = {"K": 1.0, "M": -w * w, "D": 1j * w}
        self.lus = []
        for ext, blk in zip(asm.ext, asm.blocks):
            m = int(ext.numel())
            D = torch.zeros((m, m), dtype=CDT, device=ext.device)
            for (kind, t), P in zip(asm.terms, blk):
                linalg.axpy_dense(P, scale[kind] * t.at(f), D)
            self.lus.append(DenseLU(D))

    def _apply_inverse(self, R: torch.Tensor) -> torch.Tensor:
        R2 = R.view(-1, 1) if R.dim() == 1 else R
        out = torch.zeros((self.asm.n, R2.shape[1]), dtype=CDT, device=R2.device)
        for ext, (loc, glob), lu in zip(self.asm.ext, self.asm.own, self.lus):
            X = lu.solve(R2.index_select(0, ext).contiguous(), check=False)
            if self.asm.variant == "restricted":
                out.index_copy_(0, glob, X.index_select(0, loc))
            else:
                out.index_add_(0, ext, X)
        return out.view(-1) if R.dim() == 1 else out


class SchwarzGmres:
    """FullOrderModel.iterative hook: GPU GMRES right-preconditioned by the
    additive Schwarz inverse at the solve frequency (solvers.py:191-264 with
    AdditiveSchwarzPrecond, solvers.py:137-176), residual <= tol."""

    def __init__(self, asm: AdditiveSchwarz, tol: float = 1e-10, max_it: int = 600, restart: int = 100):
        self.asm, self.tol, self.max_it, self.restart = asm, tol, max_it, restart

    def factor(self, f: float, fom):
        from .gmres import GmresFactor
        return GmresFactor(fom, f, self.asm.factor(f), self.tol, self.max_it, self.restart)
