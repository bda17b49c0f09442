"""Full-order direct solver for plane-major z-extruded models (cfg4 fuselage,
fuselage.py): block elimination over the node planes of a quadratic
(27-node / 9-node) mesh extruded along z.

With the DoFs numbered plane by plane, plane p couples only to planes
p +- 1, p +- 2 (one element layer = planes 2e, 2e+1, 2e+2), and a mid plane
2e+1 only to its own layer.  So

  1. every mid plane O_e is eliminated on its own (independent layers):
     A[O_e, O_e]^-1 from a dense LU (vb_zgetrf) and DMMA block substitution
     (solvers.lu_inverse); the Schur updates S[E_a, E_b] -= A[E_a, O] A[O,O]^-1
     A[O, E_b] of the two corner planes are sparse products (vb_rg_spmm /
     vb_csr_spmm of the coupling blocks) since the couplings are sparse;
  2. the corner planes then form a block-tridiagonal system, factored in one
     sweep: D_j = S[j, j] - S[j, j-1] D_{j-1}^-1 S[j-1, j].

The interior couplings are the affine primitives' sub-blocks, sliced once per
model and summed densely per frequency (vb_csr_axpy_dense).  Pivoting is
partial inside each diagonal block; the factor is wrapped in
mor.RefinedSolver (iterative refinement against the assembled operator to
||b - A x|| / ||b|| <= 1e-10, the direct_solve contract solvers.py:62-78 —
it replaces scipy's splu at mor.py:48-49, 153-156 for models no dense LU
covers).  Cost per factorisation ~ n_z * 40 N^3 flops for N DoFs per plane
(two block LUs + inverses, two corner-chain GEMMs per layer) instead of
(8/3) n^3 for a dense LU of the whole system; a solve is ~4 n_z block GEMVs.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import linalg
from .assembly import DeviceCSR
from .solvers import DenseLU, lu_inverse

CDT = torch.complex128


def _dev_csr(S, device) -> DeviceCSR | None:
    S = S.tocsr()
    S.sum_duplicates()
    if S.nnz == 0:
        return None
    return DeviceCSR(S.shape[0], torch.as_tensor(S.indptr.astype(np.int32), device=device),
                     torch.as_tensor(S.indices.astype(np.int32), device=device),
                     torch.as_tensor(S.data.astype(np.float64), device=device))


def _check_plane_structure(mats, off):
    """Every coupling must stay inside one element layer: |p - q| <= 1, or
    |p - q| = 2 between the two corner planes of a layer (even p, q).  Anything
    else would be silently dropped by the block elimination."""
    for H in mats:
        H = H.tocoo()
        p = np.searchsorted(off, H.row, side="right") - 1
        q = np.searchsorted(off, H.col, side="right") - 1
        d = np.abs(p - q)
        bad = (d > 2) | ((d == 2) & ((p % 2 == 1) | (q % 2 == 1)))
        if np.any(bad):
            i = int(np.argmax(bad))
            raise ValueError(f"operator couples node planes {int(p[i])} and {int(q[i])}: not a plane-major "
                             "z-extruded quadratic model")


class PlaneBlockSolver:
    """Sub-blocks of an affine operator over its node planes (set up once):
    per term, the dense-assembled blocks (mid-mid, corner-corner) and the
    sparse mid-corner couplings used by the SpMM Schur updates."""

    def __init__(self, affine, plane_off, device=None):
        import scipy.sparse as sp
        off = np.asarray(plane_off, dtype=np.int64)
        self.P = P = len(off) - 1
        if P < 3 or P % 2 == 0:
            raise ValueError("an odd number (>= 3) of node planes expected")
        self.nz = nz = (P - 1) // 2
        self.off = off
        self.aff = affine
        dev = torch.device(device or "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        self.terms = [(kind, t) for kind, lst in (("K", affine.K), ("M", affine.M), ("D", affine.D)) for t in lst]
        host = [t.P.to_scipy().tocsr() for _, t in self.terms]
        _check_plane_structure(host, off)
        blk = lambda H, p, q: H[off[p]:off[p + 1], off[q]:off[q + 1]]
        self.blocks = {}
        pairs = [(2 * e + 1, 2 * e + 1) for e in range(nz)] + [(2 * j, 2 * j) for j in range(nz + 1)]
        pairs += [(2 * j, 2 * j + 2) for j in range(nz)] + [(2 * j + 2, 2 * j) for j in range(nz)]
        for (p, q) in pairs:
            lst = []
            for ti, H in enumerate(host):
                d = _dev_csr(blk(H, p, q), dev)
                if d is not None:
                    lst.append((ti, d))
            self.blocks[(p, q)] = lst
        # per layer e: A[E_a, O] (a = 2e, 2e+2) and [A[O, 2e]^T ; A[O, 2e+2]^T] per term
        self.c_eo, self.c_oeT = [], []
        for e in range(nz):
            m, a, b = 2 * e + 1, 2 * e, 2 * e + 2
            eo = {a: [], b: []}
            oeT = []
            for ti, H in enumerate(host):
                for p in (a, b):
                    d = _dev_csr(blk(H, p, m), dev)
                    if d is not None:
                        eo[p].append((ti, d))
                T = sp.vstack([blk(H, m, a).T, blk(H, m, b).T]).tocsr()
                d = _dev_csr(T, dev)
                if d is not None:
                    oeT.append((ti, d))
            self.c_eo.append(eo)
            self.c_oeT.append(oeT)

    def size(self, p: int) -> int:
        return int(self.off[p + 1] - self.off[p])

    def scales(self, f: float):
        w = 2.0 * math.pi * f
        fac = {"K": 1.0, "M": -w * w, "D": 1j * w}
        return [fac[kind] * t.at(f) for kind, t in self.terms]

    def dense(self, p: int, q: int, sc, out: torch.Tensor | None = None) -> torch.Tensor:
        D = out if out is not None else torch.zeros((self.size(p), self.size(q)), dtype=CDT, device=self.dev)
        for ti, sub in self.blocks.get((p, q), ()):
            linalg.axpy_dense(sub, sc[ti], D)
        return D

    def factor(self, f: float) -> "PlaneBlockFactor":
        return PlaneBlockFactor(self, f)


def _inverse(D: torch.Tensor) -> torch.Tensor:
    """D^-1 from the GPU LU (vb_zgetrf + DMMA block substitution, solvers.lu_inverse)."""
    return lu_inverse(DenseLU(D))


class PlaneBlockFactor:
    """Factors of A(f) as explicit block inverses, so that every solve is a
    chain of HBM-bound block GEMVs (vb_zgemv_batched) instead of latency-bound
    triangular solves:
      * mid planes: A[O_e, O_e]^-1; the Schur updates of the two corner
        planes, S[E_a, E_b] -= A[E_a, O] (A[O,O]^-1 A[O, E_b]), are two sparse
        products (SpMM of the coupling CSR blocks, X^T = A[O, E]^T A[O,O]^-T);
      * corner chain: D_j = S[j, j] - S[j, j-1] Y_{j-1}, D_j^-1 and
        Y_j = D_j^-1 S[j, j+1] (DMMA GEMMs).
    mor.RefinedSolver absorbs the inverses' forward error (residual <= 1e-10)."""

    def __init__(self, owner: PlaneBlockSolver, f: float):
        self.o, self.f = owner, f
        o = owner
        sc = o.scales(f)
        self.sc = sc
        nz = o.nz
        N = [o.size(2 * j) for j in range(nz + 1)]
        # corner rows [S(j, j-1) | S(j, j) | S(j, j+1)] in one tensor per j
        rows, lo = [], []
        for j in range(nz + 1):
            nl = N[j - 1] if j > 0 else 0
            nr = N[j + 1] if j < nz else 0
            R = torch.zeros((N[j], nl + N[j] + nr), dtype=CDT, device=o.dev)
            if j > 0:
                o.dense(2 * j, 2 * j - 2, sc, R[:, :nl])
            o.dense(2 * j, 2 * j, sc, R[:, nl:nl + N[j]])
            if j < nz:
                o.dense(2 * j, 2 * j + 2, sc, R[:, nl + N[j]:])
            rows.append(R)
            lo.append(nl)
        self.inv_mid = []
        for e in range(nz):
            m = 2 * e + 1
            Ai = _inverse(o.dense(m, m, sc))
            AiT = Ai.transpose(0, 1).contiguous()
            XT = torch.zeros((N[e] + N[e + 1], o.size(m)), dtype=CDT, device=o.dev)
            for ti, T in o.c_oeT[e]:
                linalg.spmm(T, AiT, sc[ti], 1.0, XT)
            del AiT
            X = XT.transpose(0, 1).contiguous()
            del XT
            for j, p, c0 in ((e, 2 * e, lo[e]), (e + 1, 2 * e + 2, 0)):
                view = rows[j][:, c0:c0 + N[e] + N[e + 1]]
                for ti, A in o.c_eo[e][p]:
                    linalg.spmm(A, X, -sc[ti], 1.0, view)
            del X
            self.inv_mid.append(Ai)
        self.inv_c, self.Y, self.L = [], [], []
        for j in range(nz + 1):
            R = rows[j]
            nl = lo[j]
            D = R[:, nl:nl + N[j]].contiguous()
            if j > 0:
                L = R[:, :nl].contiguous()
                linalg.zgemm("N", L, self.Y[j - 1], -1.0, 1.0, C=D)
                self.L.append(L)
            Di = _inverse(D)
            del D
            self.inv_c.append(Di)
            if j < nz:
                self.Y.append(linalg.zgemm("N", Di, R[:, nl + N[j]:].contiguous()))
            rows[j] = None

    @property
    def info(self) -> int:
        return 0  # exactly singular blocks raise in _inverse

    def _apply(self, V: torch.Tensor) -> torch.Tensor:
        """A(f) V with the affine primitives (SpMM)."""
        out = torch.zeros_like(V)
        for ti, (kind, t) in enumerate(self.o.terms):
            linalg.spmm(t.P, V, self.sc[ti], 1.0, out)
        return out

    def solve(self, B: torch.Tensor, check: bool = True) -> torch.Tensor:
        vec = B.dim() == 1
        B2 = (B.view(-1, 1) if vec else B).to(CDT).contiguous()
        if B2.shape[1] > 16:
            X = torch.cat([self._solve16(B2[:, c:c + 16].contiguous()) for c in range(0, B2.shape[1], 16)], dim=1)
        else:
            X = self._solve16(B2)
        return X.view(-1) if vec else X

    def _solve16(self, B2: torch.Tensor) -> torch.Tensor:
        o = self.o
        off, nz = o.off, o.nz
        rng = lambda p: slice(int(off[p]), int(off[p + 1]))
        gemv = linalg.zgemv_batched
        # 1. mid planes c = A_OO^-1 b_O (one batched launch), g = b - A c
        V = torch.zeros_like(B2)
        gemv([(self.inv_mid[e], B2[rng(2 * e + 1)], V[rng(2 * e + 1)], 1.0, 0.0) for e in range(nz)])
        G = B2 - self._apply(V)
        # 2. corner chain: z_j = D_j^-1 (g_j - L_j z_{j-1}); x_j = z_j - Y_j x_{j+1}
        X = torch.zeros_like(B2)
        for j in range(nz + 1):
            g = G[rng(2 * j)]
            if j > 0:
                gemv([(self.L[j - 1], X[rng(2 * j - 2)], g, -1.0, 1.0)])
            gemv([(self.inv_c[j], g, X[rng(2 * j)], 1.0, 0.0)])
        for j in range(nz - 1, -1, -1):
            gemv([(self.Y[j], X[rng(2 * j + 2)], X[rng(2 * j)], -1.0, 1.0)])
        # 3. mid planes x_O = A_OO^-1 (b_O - A_OE x_E) (one batched launch)
        W = B2 - self._apply(X)
        gemv([(self.inv_mid[e], W[rng(2 * e + 1)], X[rng(2 * e + 1)], 1.0, 0.0) for e in range(nz)])
        return X
