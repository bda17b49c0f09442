"""Full-order solver for a structure coupled to a box cavity (cfg2, SURVEY §8f
row 4): Schur complement on the structure block, fast diagonalisation for the
cavity block.

With the DoFs ordered [structure | cavity] (plate.py numbering),

    A = [[A_pp, A_pf],        A_ff = K_g/rho - w^2 M_n/(rho c^2) (+ wall terms)
         [A_fp, A_ff]]        is the box Kronecker-sum operator (fdm.BoxFDM),

so A^-1 needs one dense LU of the structure-sized Schur complement
S = A_pp - A_pf A_ff^-1 A_fp and fast-diagonalisation solves for A_ff: A_fp is
nonzero only in the structure columns that touch the wet face (the plate's
normal displacements), so A_ff^-1 A_fp is nc << n_p cavity solves.  At cfg2
(n_p = 3,565, n_f = 17,325, nc = 713) one factorisation is an FDM block solve
and a 3,565 dense LU instead of a 20,890 dense LU.  The factor is wrapped in
mor.RefinedSolver (iterative refinement against the assembled operator to
||b - A x|| / ||b|| <= 1e-10), the same contract as the dense path
(solvers.py:72-73; mor.py:48-49 replaces scipy splu).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import linalg
from .assembly import DeviceCSR
from .solvers import DenseLU

CDT = torch.complex128


def _dev_csr(S, device) -> DeviceCSR | None:
    S = S.tocsr()
    S.sum_duplicates()
    if S.nnz == 0:
        return None
    return DeviceCSR(S.shape[0], torch.as_tensor(S.indptr.astype(np.int32), device=device),
                     torch.as_tensor(S.indices.astype(np.int32), device=device),
                     torch.as_tensor(S.data.astype(np.float64), device=device))


class CoupledBoxSchur:
    """Block-sliced primitives of an affine FOM whose trailing n_f DoFs are a
    BoxFDM cavity (`fdm` describes the cavity block exactly; a mismatch shows up
    as refinement failure, never as a wrong answer)."""

    def __init__(self, affine, n_p: int, fdm, device=None):
        self.n_p, self.fdm = n_p, fdm
        self.dev = torch.device(device or "cuda")
        self.terms = []   # (kind, term, pp, pf) device CSRs of the structure rows
        fp_cols = []
        fp_host = []
        for kind, lst in (("K", affine.K), ("M", affine.M), ("D", affine.D)):
            for t in lst:
                S = t.P.to_scipy().tocsr()
                pp, pf, fp = S[:n_p, :n_p], S[:n_p, n_p:], S[n_p:, :n_p]
                self.terms.append((kind, t, _dev_csr(pp, self.dev), _dev_csr(pf, self.dev)))
                fp = fp.tocsr()
                fp.sum_duplicates()
                fp_host.append(fp)
                if fp.nnz:
                    fp_cols.append(np.unique(fp.indices))
        self.cols = np.unique(np.concatenate(fp_cols)) if fp_cols else np.zeros(0, dtype=np.int64)
        self.cols_d = torch.as_tensor(self.cols, device=self.dev)
        # A_fp restricted to the coupled structure columns, one dense real block per term
        self.fp_dense = [torch.as_tensor(fp[:, self.cols].toarray(), device=self.dev) if fp.nnz else None
                         for fp in fp_host]

    @staticmethod
    def _scale(kind: str, t, f: float):
        w = 2.0 * math.pi * f
        c = t.at(f)
        return c if kind == "K" else (-w * w * c if kind == "M" else 1j * w * c)

    def factor(self, f: float) -> "SchurFactor":
        n_p, nc = self.n_p, len(self.cols)
        S = torch.zeros((n_p, n_p), dtype=CDT, device=self.dev)
        Afp = torch.zeros((self.fdm.n, nc), dtype=CDT, device=self.dev)
        scales = []
        for (kind, t, pp, pf), D in zip(self.terms, self.fp_dense):
            a = self._scale(kind, t, f)
            scales.append(a)
            if pp is not None:
                linalg.axpy_dense(pp, a, S)
            if D is not None:
                Afp.add_(D.to(CDT), alpha=a)
        fd = self.fdm.factor(f)          # no fom: the global refinement checks the result
        X = fd._apply_inverse(Afp)       # A_ff^-1 A_fp[:, cols]   (n_f x nc)
        T = torch.zeros((n_p, nc), dtype=CDT, device=self.dev)
        for (kind, t, pp, pf), a in zip(self.terms, scales):
            if pf is not None:
                linalg.spmm(pf, X, a, 1.0, T)
        S[:, self.cols_d] -= T
        return SchurFactor(self, DenseLU(S), fd, X, scales)


class SchurFactor:
    """Solver object with the DenseLU interface (`solve`, `info`)."""

    def __init__(self, owner: CoupledBoxSchur, lu: DenseLU, fd, X: torch.Tensor, scales):
        self.o, self.lu, self.fd, self.X, self.scales = owner, lu, fd, X, scales

    @property
    def info(self) -> int:
        return self.lu.info

    def solve(self, B: torch.Tensor, check: bool = True) -> torch.Tensor:
        vec = B.dim() == 1
        B2 = (B.view(-1, 1) if vec else B).to(CDT)
        n_p = self.o.n_p
        Bp, Bf = B2[:n_p].contiguous(), B2[n_p:].contiguous()
        yf = self.fd._apply_inverse(Bf)                       # A_ff^-1 b_f
        rp = Bp.clone()
        for (kind, t, pp, pf), a in zip(self.o.terms, self.scales):
            if pf is not None:
                linalg.spmm(pf, yf, -a, 1.0, rp)               # b_p - A_pf A_ff^-1 b_f
        xp = self.lu.solve(rp, check=check)                   # S x_p = r_p
        xc = xp[self.o.cols_d].contiguous()
        xf = linalg.zgemm("N", self.X, xc, -1.0, 1.0, yf)     # x_f = A_ff^-1 (b_f - A_fp x_p)
        X = torch.cat([xp, xf], dim=0)
        return X.view(-1) if vec else X
