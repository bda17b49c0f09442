"""Fast-diagonalisation full-order solver for structured hex27 boxes
(SURVEY §7.2 L7, §8f row 2 — the cfg3 solver, n = 376,431).

The box Helmholtz operator with per-wall constant impedances,
    A(w) = K/rho - w^2 M/(rho c^2) + i w sum_walls F_w / Z_w,
is EXACTLY a Kronecker sum of 1D quadratic-FE operators (Kgrad = Mz(x)My(x)Kx
+ Mz(x)Ky(x)Mx + Kz(x)My(x)Mx, Mnn = Mz(x)My(x)Mx, a z-wall face mass =
e e^T (x) My (x) Mx; checked against the assembled CSR in the tests).  With
per-direction generalised eigenpairs (A_d V = M_d V Lambda, V^T M_d V = I)
    A^-1 = V (Lz (+) Ly (+) Lx + sigma)^-1 V^T,  V = Vz (x) Vy (x) Vx,
applied on the GPU by axis transforms (vb_axis_apply, vb_fdm_diag).  Each
solve is refined against the assembled operator (SpMV of the GPU-assembled
CSR primitives) to a relative residual <= 1e-10 (solvers.py:72-73 metric).
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.linalg as sla
import torch

from . import _lib, linalg

CDT = torch.complex128
_POOL = ThreadPoolExecutor(3, thread_name_prefix="vb_fdm_eig")  # the three axes of a factorisation
GAUSS3 = (np.array([-math.sqrt(0.6), 0.0, math.sqrt(0.6)]), np.array([5 / 9, 8 / 9, 5 / 9]))


def line_matrices(L: float, ne: int):
    """Assembled 1D quadratic Lagrange stiffness/mass on [0, L] (shape.py:20-26
    bases, 3-point Gauss)."""
    n = 2 * ne + 1
    h = L / ne
    ke = np.zeros((3, 3))
    me = np.zeros((3, 3))
    for x, w in zip(*GAUSS3):
        N = np.array([0.5 * x * (x - 1.0), 1.0 - x * x, 0.5 * x * (x + 1.0)])
        dN = np.array([x - 0.5, -2.0 * x, x + 0.5]) * 2.0 / h
        ke += w * (h / 2) * np.outer(dN, dN)
        me += w * (h / 2) * np.outer(N, N)
    K = np.zeros((n, n))
    M = np.zeros((n, n))
    for e in range(ne):
        s = slice(2 * e, 2 * e + 3)
        K[s, s] += ke
        M[s, s] += me
    return K, M


class BoxFDM:
    """Separable description of a box model: geometry, fluid, wall impedances."""

    def __init__(self, box, ne, rho: float, c: float, walls: dict):
        x0, y0, z0, x1, y1, z1 = box
        self.ne = tuple(ne)
        self.rho, self.c = rho, c
        self.walls = dict(walls)  # side ('x0', ..., 'z1') -> complex Z
        self.lines = [line_matrices(L, m) for L, m in zip((x1 - x0, y1 - y0, z1 - z0), ne)]
        self.shape = tuple(2 * m + 1 for m in ne)  # (npx, npy, npz)
        self._chol_inv: dict[int, np.ndarray] = {}

    @property
    def n(self) -> int:
        return int(np.prod(self.shape))

    def direction_operator(self, d: int, f: float) -> np.ndarray:
        K, _ = self.lines[d]
        A = K.astype(complex) / self.rho
        w = 2.0 * math.pi * f
        for side, Z in self.walls.items():
            if "xyz".index(side[0]) == d:
                i = 0 if side[1] == "0" else A.shape[0] - 1
                A[i, i] += 1j * w / Z
        return A

    def axis_eig(self, d: int, f: float):
        """Generalised eigenpairs A_d V = M_d V Lambda with V^T M_d V = I.  M_d
        is SPD: with M_d = L L^T (cached, frequency independent) this is the
        standard complex-symmetric problem C W = W Lambda, C = L^-1 A_d L^-T,
        V = L^-T W (zgeev on C: ~2.5x faster than the QZ of zggev at these
        sizes).  One BLAS thread: the three axes run concurrently."""
        from threadpoolctl import threadpool_limits
        Li = self._chol_inv.get(d)
        if Li is None:
            L = np.linalg.cholesky(self.lines[d][1])
            Li = self._chol_inv[d] = sla.solve_triangular(L, np.eye(L.shape[0]), lower=True)
        with threadpool_limits(1):
            C = Li @ self.direction_operator(d, f) @ Li.T
            lam, W = np.linalg.eig(C)
            nrm = np.sqrt(np.einsum("ij,ij->j", W, W))  # complex-symmetric normalisation: V^T M V = W^T W
            V = (Li.T @ W) / nrm
        return lam, V

    def factor(self, f: float, fom=None, device=None, tol: float = 1e-10, max_refine: int = 8):
        return FdmFactor(self, f, fom, device, tol, max_refine)


class FdmFactor:
    """Solver object with the DenseLU interface (`solve`, `info`)."""

    info = 0

    def __init__(self, box: BoxFDM, f: float, fom, device, tol, max_refine):
        _lib.require_cuda()
        self.box, self.f, self.fom = box, f, fom
        self.tol, self.max_refine = tol, max_refine
        self.dev = torch.device(device or "cuda")
        w = 2.0 * math.pi * f
        self.sigma = -w * w / (box.rho * box.c * box.c)
        self.V, self.VT, self.lam = [], [], []
        for lam, V in _POOL.map(lambda d: box.axis_eig(d, f), range(3)):
            self.V.append(torch.as_tensor(np.ascontiguousarray(V), device=self.dev))
            self.VT.append(torch.as_tensor(np.ascontiguousarray(V.T), device=self.dev))
            self.lam.append(torch.as_tensor(lam.astype(complex), device=self.dev))
        self.last_residual = None
        self.iterations = 0

    def _apply_inverse(self, B: torch.Tensor) -> torch.Tensor:
        """X = A^-1 B through vb_fdm_solve (tensor-core transforms)."""
        lib = _lib.load()
        npx, npy, npz = self.box.shape
        B2 = B if B.dim() == 2 and B.stride(1) == 1 else B.reshape(B.shape[0], -1).contiguous()
        s = B2.shape[1]
        X = torch.empty((B2.shape[0], s), dtype=B2.dtype, device=B2.device)
        wb = lib.vb_fdm_solve_workspace_bytes(npz, npy, npx, s)
        work = torch.empty(max(wb, 1), dtype=torch.uint8, device=B2.device)
        P = _lib.ptr
        _lib.check(lib.vb_fdm_solve(npz, npy, npx, s, P(self.V[0]), P(self.V[1]), P(self.V[2]), P(self.VT[0]),
                                    P(self.VT[1]), P(self.VT[2]), P(self.lam[0]), P(self.lam[1]), P(self.lam[2]),
                                    _lib.zc(self.sigma), linalg.C_ptr(B2), B2.stride(0), P(X), X.stride(0), P(work), wb,
                                    _lib.stream_handle()), "vb_fdm_solve")
        return X

    def _apply_inverse_axes(self, B: torch.Tensor) -> torch.Tensor:
        """Same operator through the per-axis CUDA-core kernels (cross-check)."""
        lib = _lib.load()
        npx, npy, npz = self.box.shape
        s = B.shape[1]
        st = _lib.stream_handle()
        X = B.contiguous().clone()  # ping-pong buffers: never write into the caller's B
        T = torch.empty_like(X)
        for axis, S in ((0, self.VT[0]), (1, self.VT[1]), (2, self.VT[2])):
            _lib.check(lib.vb_axis_apply(npz, npy, npx, s, axis, _lib.ptr(S), _lib.ptr(X), _lib.ptr(T), st),
                       "vb_axis_apply")
            X, T = T, X
        _lib.check(lib.vb_fdm_diag(npz, npy, npx, s, _lib.ptr(self.lam[2]), _lib.ptr(self.lam[1]),
                                   _lib.ptr(self.lam[0]), _lib.zc(self.sigma), _lib.ptr(X), st), "vb_fdm_diag")
        for axis, S in ((0, self.V[0]), (1, self.V[1]), (2, self.V[2])):
            _lib.check(lib.vb_axis_apply(npz, npy, npx, s, axis, _lib.ptr(S), _lib.ptr(X), _lib.ptr(T), st),
                       "vb_axis_apply")
            X, T = T, X
        return X

    def residual(self, X: torch.Tensor, B: torch.Tensor) -> torch.Tensor:
        """R = B - A X with A from the FOM's assembled primitives (SpMV)."""
        fom, f = self.fom, self.f
        w = 2.0 * math.pi * f
        R = B.clone()
        fom.apply("K", f, X, scale=-1.0, out=R, beta=1.0)
        fom.apply("M", f, X, scale=w * w, out=R, beta=1.0)
        if fom.affine is not None and fom.affine.D:
            fom.apply("D", f, X, scale=-1j * w, out=R, beta=1.0)
        return R

    def solve(self, B: torch.Tensor, check: bool = True) -> torch.Tensor:
        vec = B.dim() == 1
        B2 = (B.view(-1, 1) if vec else B).to(CDT).contiguous()
        X = self._apply_inverse(B2)
        if self.fom is not None:
            nb = linalg.column_norms(B2).max().item()
            it = 0
            while True:
                R = self.residual(X, B2)
                rel = linalg.column_norms(R).max().item() / (nb if nb > 0 else 1.0)
                self.last_residual = rel
                if rel <= self.tol or it >= self.max_refine:
                    break
                X = X + self._apply_inverse(R)
                it += 1
            self.iterations = it
            if check and self.last_residual > self.tol:
                raise RuntimeError(f"FDM solve did not reach residual {self.tol:g} "
                                   f"(got {self.last_residual:.3e} after {it} refinements)")
        return X.view(-1) if vec else X
