"""Batched reduced sweep on the GPU (C-ABI `vb_rom_sweep`).

This is the north-star hot loop: for every frequency of a window,
A_r(f) = sum_k alpha_k(f) P_k,  x_r = A_r^-1 b_r,  y = C_R x_r,  SPL(y)
(vibrofem/mor.py:73-102 + vibrofem/solvers.py:334-338), one launch for all
frequencies instead of one Python call per frequency (mor.py:376-393).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

CDT = torch.complex128


def as_ctensor(a, device) -> torch.Tensor:
    """complex128 contiguous CUDA tensor view/copy of a numpy array or tensor."""
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=CDT).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.complex128)).to(device)


def affine_coefficients(freqs: torch.Tensor, terms) -> torch.Tensor:
    """alpha[i, k] for the standard second-order form used by the reference:
    terms is a list of ('K'|'D'|'M', complex scale or callable(f)->complex array).
    K -> scale, D -> i w scale, M -> -w^2 scale (mor.py:41-46, 79-85)."""
    w = 2.0 * math.pi * freqs.to(torch.float64)
    cols = []
    for kind, scale in terms:
        sc = scale(freqs) if callable(scale) else torch.full_like(w, 1.0, dtype=CDT) * complex(scale)
        sc = sc.to(CDT)
        if kind == "K":
            cols.append(sc)
        elif kind == "D":
            cols.append(1j * w.to(CDT) * sc)
        elif kind == "M":
            cols.append(-(w * w).to(CDT) * sc)
        else:
            raise ValueError(f"unknown term kind {kind!r}")
    return torch.stack(cols, dim=1).contiguous()


@dataclass
class SweepOut:
    y: torch.Tensor | None       # (F, n_out, s) complex128
    spl: torch.Tensor | None     # (F, s) float64
    x: torch.Tensor | None       # (F, r, s) complex128
    info: torch.Tensor           # (F,) int32


def rom_sweep_affine(prims: torch.Tensor, alpha: torch.Tensor, b: torch.Tensor, c_r: torch.Tensor,
                     want_y: bool = True, want_spl: bool = True, want_x: bool = False,
                     stream=None, out: SweepOut | None = None) -> SweepOut:
    """One launch sequence for all F frequencies.  All inputs are CUDA tensors:
    prims (K, r, r), alpha (F, K), b (r, s) or (F, r, s), c_r (n_out, r)."""
    lib = _lib.load()
    K, r, r2 = prims.shape
    if r != r2:
        raise ValueError("primitives must be square")
    F = alpha.shape[0]
    if alpha.shape[1] != K:
        raise ValueError("alpha must be (F, n_prim)")
    if b.dim() == 2:
        s = b.shape[1]
        bstride = 0
    else:
        s = b.shape[2]
        if b.shape[0] != F:
            raise ValueError("frequency-dependent b must be (F, r, s)")
        bstride = r * s
    if b.shape[-2] != r:
        raise ValueError("b row count does not match reduced order")
    n_out = c_r.shape[0] if c_r is not None else 0
    if n_out and c_r.shape[1] != r:
        raise ValueError("c_r column count does not match reduced order")
    dev = prims.device
    for t in (prims, alpha, b) + ((c_r,) if n_out else ()):
        if t.dtype != CDT or not t.is_cuda or not t.is_contiguous():
            raise ValueError("rom_sweep_affine expects contiguous complex128 CUDA tensors")
    if out is None:
        out = SweepOut(
            y=torch.empty((F, n_out, s), dtype=CDT, device=dev) if want_y and n_out else None,
            spl=torch.empty((F, s), dtype=torch.float64, device=dev) if want_spl and n_out else None,
            x=torch.empty((F, r, s), dtype=CDT, device=dev) if want_x else None,
            info=torch.empty((F,), dtype=torch.int32, device=dev))
    wbytes = lib.vb_rom_sweep_workspace_bytes(r, K, s, n_out, F)
    work = torch.empty((max(wbytes, 1),), dtype=torch.uint8, device=dev)
    rc = lib.vb_rom_sweep(r, K, s, n_out, F, _lib.ptr(prims), _lib.ptr(alpha), _lib.ptr(b), bstride,
                          _lib.ptr(c_r) if n_out else None, _lib.ptr(out.y), _lib.ptr(out.spl),
                          _lib.ptr(out.x), _lib.ptr(out.info), _lib.ptr(work), wbytes,
                          _lib.stream_handle(stream))
    _lib.check(rc, "vb_rom_sweep")
    return out


def raise_if_singular(info: torch.Tensor):
    """numpy.linalg.solve raises LinAlgError on an exactly singular pivot (mor.py:94)."""
    bad = torch.nonzero(info).flatten()
    if bad.numel():
        i = int(bad[0])
        raise np.linalg.LinAlgError(f"Singular matrix (frequency index {i}, zero pivot "
                                    f"{int(info[i])})")
