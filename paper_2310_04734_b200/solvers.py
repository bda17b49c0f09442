"""Full-order direct solver on the GPU and the SPL helper.

`DenseLU` wraps vb_zgetrf / vb_zgetrs (one matrix on the whole GPU, partial
pivoting with LAPACK izamax semantics).  It replaces the scipy SuperLU
factorisation of the reference (`splu`, vibrofem/mor.py:48-49, 153-156,
solvers.py:62-78) for the n ≲ 25k full-order models of cfg1/cfg2.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib

CDT = torch.complex128
P_REF = 20e-6  # Pa, solvers.py:25


def mean_spl(p) -> float:
    """Mean SPL of one output vector: 20 log10(sqrt(mean|p|^2/2) / 20 uPa)
    with a 1e-300 floor (vibrofem/solvers.py:334-338)."""
    p = np.asarray(p)
    p_rms = math.sqrt(float(np.mean(np.abs(p) ** 2)) / 2.0)
    return 20.0 * math.log10(max(p_rms, 1e-300) / P_REF)


@dataclass
class SolveStats:
    """solvers.py:28-36 (the fields the direct path fills)."""

    iterations: int = 0
    residual_history: list = field(default_factory=list)
    factor_time: float = 0.0
    solve_time: float = 0.0
    factor_memory: int = 0
    converged: bool = True


class DenseLU:
    """In-place dense LU of an n x n complex128 CUDA matrix (row-major).

    `A` is overwritten with L\\U unless copy=True.  Exactly singular pivots set
    `info` (LAPACK INFO); `solve` then raises like scipy's splu would
    (RuntimeError "Factor is exactly singular")."""

    def __init__(self, A: torch.Tensor, copy: bool = False, stream=None):
        _lib.require_cuda()
        lib = _lib.load()
        if A.dim() != 2 or A.shape[0] != A.shape[1]:
            raise ValueError("square matrix expected")
        self.n = n = A.shape[0]
        self.A = A.clone() if copy else A
        if self.A.dtype != CDT or not self.A.is_contiguous():
            raise ValueError("contiguous complex128 matrix expected")
        dev = self.A.device
        self.ipiv = torch.empty(n, dtype=torch.int32, device=dev)
        self._info = torch.zeros(1, dtype=torch.int32, device=dev)
        ab = lib.vb_zgetrf_aux_bytes(n)
        self.aux = torch.empty(ab, dtype=torch.uint8, device=dev)
        wb = lib.vb_zgetrf_workspace_bytes(n)
        work = torch.empty(wb, dtype=torch.uint8, device=dev)
        self.stream = stream
        _lib.check(lib.vb_zgetrf(n, _lib.ptr(self.A), n, _lib.ptr(self.ipiv), _lib.ptr(self._info),
                                 _lib.ptr(self.aux), ab, _lib.ptr(work), wb, _lib.stream_handle(stream)),
                   "vb_zgetrf")
        self._info_host = None

    @property
    def info(self) -> int:
        if self._info_host is None:
            self._info_host = int(self._info.item())
        return self._info_host

    def solve(self, B: torch.Tensor, out: torch.Tensor | None = None, check: bool = True) -> torch.Tensor:
        """X = A^-1 B for B (n,) or (n, s<=16) on the device."""
        if check and self.info != 0:
            raise RuntimeError("Factor is exactly singular")
        lib = _lib.load()
        vec = B.dim() == 1
        B2 = B.view(-1, 1) if vec else B
        if B2.dtype != CDT:
            B2 = B2.to(CDT)
        B2 = B2.contiguous()
        s = B2.shape[1]
        X = out if out is not None else torch.empty_like(B2)
        wb = lib.vb_zgetrs_workspace_bytes(self.n, s)
        work = torch.empty(wb, dtype=torch.uint8, device=B2.device)
        _lib.check(lib.vb_zgetrs(self.n, s, _lib.ptr(self.A), self.n, _lib.ptr(self.aux), _lib.ptr(B2), s,
                                 _lib.ptr(X), X.stride(0) if X.dim() == 2 else 1, _lib.ptr(work), wb,
                                 _lib.stream_handle(self.stream)), "vb_zgetrs")
        return X.view(-1) if vec else X


LU_NB = 64  # diagonal block size of vb_zgetrf's aux inverses (csrc/lu.cu)


def _lu_aux_views(lu: DenseLU):
    """(Linv, Uinv, perm) views of vb_zgetrf's aux block: per 64-row diagonal
    block the inverse of the unit-lower / upper factor (masked to its
    triangle) and the final row permutation."""
    cached = getattr(lu, "_aux_views", None)
    if cached is not None:
        return cached
    n, nb = lu.n, LU_NB
    nblk = (n + nb - 1) // nb
    zb = nblk * nb * nb * 16
    inv = lu.aux[:2 * zb].view(CDT).view(2, nblk, nb, nb)
    Linv = torch.tril(inv[0])
    Uinv = torch.triu(inv[1])
    perm = lu.aux[2 * zb:2 * zb + 4 * n].view(torch.int32).long()
    lu._aux_views = (Linv, Uinv, perm)
    return lu._aux_views


def lu_solve_many(lu: DenseLU, B: torch.Tensor) -> torch.Tensor:
    """X = A^-1 B for any number of right-hand sides from vb_zgetrf factors:
    block forward / backward substitution over the factor's 64-row diagonal
    blocks, each step two DMMA GEMMs (vb_zgemm) — the diagonal-block inverse
    times the block rows, then a rank-64 update of the rows still to solve."""
    from . import linalg
    if lu.info != 0:
        raise RuntimeError("Factor is exactly singular")
    n, nb = lu.n, LU_NB
    Linv, Uinv, perm = _lu_aux_views(lu)
    Y = B.to(CDT).index_select(0, perm).contiguous()
    s = Y.shape[1]
    T = torch.empty((nb, s), dtype=CDT, device=Y.device)
    nblk = (n + nb - 1) // nb
    A = lu.A
    for kb in range(nblk):
        k0 = kb * nb
        w = min(nb, n - k0)
        linalg.zgemm("N", Linv[kb, :w, :w], Y[k0:k0 + w], C=T[:w])
        Y[k0:k0 + w].copy_(T[:w])
        if k0 + w < n:
            linalg.zgemm("N", A[k0 + w:, k0:k0 + w], T[:w], -1.0, 1.0, C=Y[k0 + w:])
    for kb in range(nblk - 1, -1, -1):
        k0 = kb * nb
        w = min(nb, n - k0)
        linalg.zgemm("N", Uinv[kb, :w, :w], Y[k0:k0 + w], C=T[:w])
        Y[k0:k0 + w].copy_(T[:w])
        if k0 > 0:
            linalg.zgemm("N", A[:k0, k0:k0 + w], T[:w], -1.0, 1.0, C=Y[:k0])
    return Y


def lu_inverse(lu: DenseLU) -> torch.Tensor:
    """A^-1 from vb_zgetrf factors (P A = L U): L^-1 is lower triangular, so
    the forward substitution of the identity only touches the columns left of
    the current block (1/3 of a full forward pass); then the backward pass
    X = U^-1 L^-1 = (P A)^-1 and the column permutation A^-1[:, perm] = X."""
    from . import linalg
    if lu.info != 0:
        raise RuntimeError("Factor is exactly singular")
    n, nb = lu.n, LU_NB
    Linv, Uinv, perm = _lu_aux_views(lu)
    Y = torch.eye(n, dtype=CDT, device=lu.A.device)
    T = torch.empty((nb, n), dtype=CDT, device=Y.device)
    nblk = (n + nb - 1) // nb
    A = lu.A
    for kb in range(nblk):
        k0 = kb * nb
        w = min(nb, n - k0)
        ke = k0 + w
        linalg.zgemm("N", Linv[kb, :w, :w], Y[k0:ke, :ke], C=T[:w, :ke])
        Y[k0:ke, :ke].copy_(T[:w, :ke])
        if ke < n:
            linalg.zgemm("N", A[ke:, k0:ke], T[:w, :ke], -1.0, 1.0, C=Y[ke:, :ke])
    for kb in range(nblk - 1, -1, -1):
        k0 = kb * nb
        w = min(nb, n - k0)
        linalg.zgemm("N", Uinv[kb, :w, :w], Y[k0:k0 + w], C=T[:w])
        Y[k0:k0 + w].copy_(T[:w])
        if k0 > 0:
            linalg.zgemm("N", A[:k0, k0:k0 + w], T[:w], -1.0, 1.0, C=Y[:k0])
    out = torch.empty_like(Y)
    out[:, perm] = Y
    return out
