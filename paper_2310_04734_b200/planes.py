"""Full-order direct solver for plane-major z-extruded models (cfg4 fuselage,
fuselage.py): block elimination over the node planes of a quadratic
(27-node / 9-node) mesh extruded along z.

With the DoFs numbered plane by plane, plane p couples only to planes
p +- 1, p +- 2 (one element layer = planes 2e, 2e+1, 2e+2), and a mid plane
2e+1 only to its own layer.  So

  1. every mid plane O_e is eliminated on its own (independent layers):
     dense LU of A[O_e, O_e] (vb_zgetrf), X = A[O,O]^-1 [A[O,E_e] A[O,E_e+1]]
     (lu_solve_many: DMMA block substitution), and the Schur updates
     S[E_a, E_b] -= A[E_a, O] X_b of the two corner planes (vb_zgemm);
  2. the corner planes then form a block-tridiagonal system, factored in one
     sweep: D_j = S[j, j] - S[j, j-1] D_{j-1}^-1 S[j-1, j].

The interior couplings are the affine primitives' sub-blocks, sliced once per
model and summed densely per frequency (vb_csr_axpy_dense).  Pivoting is
partial inside each diagonal block; the factor is wrapped in
mor.RefinedSolver (iterative refinement against the assembled operator to
||b - A x|| / ||b|| <= 1e-10, the direct_solve contract solvers.py:62-78 —
it replaces scipy's splu at mor.py:48-49, 153-156 for models no dense LU
covers).  Cost per factorisation ~ n_z * 70 N^3 flops for N DoFs per plane,
instead of (8/3) n^3 for a dense LU of the whole system.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import linalg
from .assembly import DeviceCSR
from .solvers import DenseLU, lu_solve_many

CDT = torch.complex128


def _dev_csr(S, device) -> DeviceCSR | None:
    S = S.tocsr()
    S.sum_duplicates()
    if S.nnz == 0:
        return None
    return DeviceCSR(S.shape[0], torch.as_tensor(S.indptr.astype(np.int32), device=device),
                     torch.as_tensor(S.indices.astype(np.int32), device=device),
                     torch.as_tensor(S.data.astype(np.float64), device=device))


class PlaneBlockSolver:
    """Sub-blocks of an affine operator over its node planes (set up once)."""

    def __init__(self, affine, plane_off, device=None):
        off = np.asarray(plane_off, dtype=np.int64)
        self.P = P = len(off) - 1
        if P < 3 or P % 2 == 0:
            raise ValueError("an odd number (>= 3) of node planes expected")
        self.nz = (P - 1) // 2
        self.off = off
        self.aff = affine
        dev = torch.device(device or "cuda")
        self.dev = dev
        self.terms = [(kind, t) for kind, lst in (("K", affine.K), ("M", affine.M), ("D", affine.D)) for t in lst]
        host = [t.P.to_scipy().tocsr() for _, t in self.terms]
        pairs = set()
        for e in range(self.nz):
            o, a, b = 2 * e + 1, 2 * e, 2 * e + 2
            pairs |= {(o, o), (o, a), (o, b), (a, o), (b, o), (a, b), (b, a)}
        for j in range(self.nz + 1):
            pairs.add((2 * j, 2 * j))
        self.blocks = {}
        for (p, q) in sorted(pairs):
            lst = []
            for ti, H in enumerate(host):
                sub = H[off[p]:off[p + 1], off[q]:off[q + 1]]
                d = _dev_csr(sub, dev)
                if d is not None:
                    lst.append((ti, d, off[q + 1] - off[q]))
            self.blocks[(p, q)] = lst

    def size(self, p: int) -> int:
        return int(self.off[p + 1] - self.off[p])

    def scales(self, f: float):
        w = 2.0 * math.pi * f
        fac = {"K": 1.0, "M": -w * w, "D": 1j * w}
        return [fac[kind] * t.at(f) for kind, t in self.terms]

    def dense(self, p: int, q: int, sc) -> torch.Tensor:
        D = torch.zeros((self.size(p), self.size(q)), dtype=CDT, device=self.dev)
        for ti, sub, _ in self.blocks.get((p, q), ()):
            linalg.axpy_dense(sub, sc[ti], D)
        return D

    def factor(self, f: float) -> "PlaneBlockFactor":
        return PlaneBlockFactor(self, f)


class PlaneBlockFactor:
    """Factors of A(f): mid-plane LUs, corner-plane Schur chain (D_j LUs, the
    sub-diagonal blocks S[j, j-1] and Y_j = D_j^-1 S[j, j+1])."""

    def __init__(self, owner: PlaneBlockSolver, f: float):
        self.o, self.f = owner, f
        o = owner
        sc = o.scales(f)
        self.sc = sc
        nz = o.nz
        S = {}
        for j in range(nz + 1):
            S[(j, j)] = o.dense(2 * j, 2 * j, sc)
        for j in range(nz):
            S[(j, j + 1)] = o.dense(2 * j, 2 * j + 2, sc)
            S[(j + 1, j)] = o.dense(2 * j + 2, 2 * j, sc)
        self.lu_mid = []
        for e in range(nz):
            m, a, b = 2 * e + 1, 2 * e, 2 * e + 2
            lu = DenseLU(o.dense(m, m, sc))
            na = o.size(a)
            X = lu_solve_many(lu, torch.cat([o.dense(m, a, sc), o.dense(m, b, sc)], dim=1))
            for (j, p) in ((e, a), (e + 1, b)):
                Ap = o.dense(p, m, sc)
                linalg.zgemm("N", Ap, X[:, :na], -1.0, 1.0, C=S[(j, e)])
                linalg.zgemm("N", Ap, X[:, na:], -1.0, 1.0, C=S[(j, e + 1)])
            del X
            self.lu_mid.append(lu)
        self.lu_c, self.Y, self.L = [], [], []
        for j in range(nz + 1):
            Dj = S.pop((j, j))
            if j > 0:
                Lj = S.pop((j, j - 1))
                linalg.zgemm("N", Lj, self.Y[j - 1], -1.0, 1.0, C=Dj)
                self.L.append(Lj)
            lu = DenseLU(Dj)
            self.lu_c.append(lu)
            if j < nz:
                self.Y.append(lu_solve_many(lu, S.pop((j, j + 1))))

    @property
    def info(self) -> int:
        for lu in self.lu_mid + self.lu_c:
            if lu.info != 0:
                return lu.info
        return 0

    def _apply_masked(self, V: torch.Tensor) -> torch.Tensor:
        """A(f) V with the affine primitives (SpMM)."""
        o = self.o
        out = torch.zeros_like(V)
        for ti, (kind, t) in enumerate(o.terms):
            linalg.spmm(t.P, V, self.sc[ti], 1.0, out)
        return out

    def _lu_solve(self, lu: DenseLU, B: torch.Tensor) -> torch.Tensor:
        if B.shape[1] <= 16:
            return lu.solve(B.contiguous(), check=False)
        return lu_solve_many(lu, B)

    def solve(self, B: torch.Tensor, check: bool = True) -> torch.Tensor:
        o = self.o
        if check and self.info != 0:
            raise RuntimeError("Factor is exactly singular")
        vec = B.dim() == 1
        B2 = (B.view(-1, 1) if vec else B).to(CDT).contiguous()
        off, nz = o.off, o.nz
        rng = lambda p: slice(int(off[p]), int(off[p + 1]))
        # 1. mid planes: c = A_OO^-1 b_O, and the corner right-hand side g = b_E - A_EO c
        V = torch.zeros_like(B2)
        for e in range(nz):
            V[rng(2 * e + 1)] = self._lu_solve(self.lu_mid[e], B2[rng(2 * e + 1)])
        G = B2 - self._apply_masked(V)
        # 2. corner chain forward / backward
        Z = []
        for j in range(nz + 1):
            g = G[rng(2 * j)]
            if j > 0:
                g = g - linalg.zgemm("N", self.L[j - 1], Z[j - 1])
            Z.append(self._lu_solve(self.lu_c[j], g))
        X = torch.zeros_like(B2)
        X[rng(2 * nz)] = Z[nz]
        for j in range(nz - 1, -1, -1):
            X[rng(2 * j)] = Z[j] - linalg.zgemm("N", self.Y[j], X[rng(2 * j + 2)])
        # 3. mid planes: x_O = A_OO^-1 (b_O - A_OE x_E)
        W = B2 - self._apply_masked(X)
        for e in range(nz):
            X[rng(2 * e + 1)] = self._lu_solve(self.lu_mid[e], W[rng(2 * e + 1)])
        return X.view(-1) if vec else X
