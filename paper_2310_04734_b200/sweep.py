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
    if s > MAX_RHS_BLOCKED and lib.vb_rom_sweep_path(r, K, s, n_out) == 1:
        return _sweep_rhs_groups(prims, alpha, b, c_r, want_y, want_spl, want_x, stream, out)
    if out is None:
        out = SweepOut(
            y=torch.empty((F, n_out, s), dtype=CDT, device=dev) if want_y and n_out else None,
            spl=torch.empty((F, s), dtype=torch.float64, device=dev) if want_spl and n_out else None,
            x=torch.empty((F, r, s), dtype=CDT, device=dev) if want_x else None,
            info=torch.empty((F,), dtype=torch.int32, device=dev))
    wbytes = lib.vb_rom_sweep_workspace_bytes(r, K, s, n_out, F)
    work = torch.empty((max(wbytes, 1),), dtype=torch.uint8, device=dev)
    side = stream is not None and stream != torch.cuda.current_stream(dev)
    if side:
        # inputs, outputs and workspace come from the current stream: order the
        # launch after them, and keep the caching allocator from recycling any
        # of them before the side stream is done with them
        stream.wait_stream(torch.cuda.current_stream(dev))
    rc = lib.vb_rom_sweep(r, K, s, n_out, F, _lib.ptr(prims), _lib.ptr(alpha), _lib.ptr(b), bstride,
                          _lib.ptr(c_r) if n_out else None, _lib.ptr(out.y), _lib.ptr(out.spl),
                          _lib.ptr(out.x), _lib.ptr(out.info), _lib.ptr(work), wbytes,
                          _lib.stream_handle(stream))
    _lib.check(rc, "vb_rom_sweep")
    if side:
        for t in (work, prims, alpha, b, c_r, out.y, out.spl, out.x, out.info):
            if t is not None:
                t.record_stream(stream)
    return out


class persist_primitives_in_l2:
    """Context manager: blocked sweeps launched inside it pin their reduced
    primitives in L2 (persisting access-policy window); on exit the persisting
    lines are reset and the device's persisting-L2 limit is restored."""

    def __enter__(self):
        _lib.load().vb_set_l2_persistence(1)
        return self

    def __exit__(self, *exc):
        lib = _lib.load()
        lib.vb_set_l2_persistence(0)
        torch.cuda.synchronize()
        _lib.check(lib.vb_release_l2_persistence(), "vb_release_l2_persistence")
        return False


MAX_RHS_BLOCKED = 16  # right-hand sides per launch on the blocked path


def _sweep_rhs_groups(prims, alpha, b, c_r, want_y, want_spl, want_x, stream, out):
    """More than 16 right-hand sides on the blocked path: one launch per group
    of 16 columns (each column's outputs and SPL are independent; every group
    refactors A(f), so the result equals one launch over all columns)."""
    F, r = alpha.shape[0], prims.shape[1]
    s = b.shape[-1]
    n_out = c_r.shape[0] if c_r is not None else 0
    dev = prims.device
    if out is None:
        out = SweepOut(
            y=torch.empty((F, n_out, s), dtype=CDT, device=dev) if want_y and n_out else None,
            spl=torch.empty((F, s), dtype=torch.float64, device=dev) if want_spl and n_out else None,
            x=torch.empty((F, r, s), dtype=CDT, device=dev) if want_x else None,
            info=torch.empty((F,), dtype=torch.int32, device=dev))
    for g0 in range(0, s, MAX_RHS_BLOCKED):
        g1 = min(s, g0 + MAX_RHS_BLOCKED)
        bg = b[..., g0:g1].contiguous()
        o = rom_sweep_affine(prims, alpha, bg, c_r, want_y, want_spl, want_x, stream)
        if out.y is not None:
            out.y[:, :, g0:g1] = o.y
        if out.spl is not None:
            out.spl[:, g0:g1] = o.spl
        if out.x is not None:
            out.x[:, :, g0:g1] = o.x
        if g0 == 0:
            out.info.copy_(o.info)
    return out


def raise_if_singular(info: torch.Tensor):
    """numpy.linalg.solve raises LinAlgError on an exactly singular pivot (mor.py:94)."""
    bad = torch.nonzero(info).flatten()
    if bad.numel():
        i = int(bad[0])
        raise np.linalg.LinAlgError(f"Singular matrix (frequency index {i}, zero pivot "
                                    f"{int(info[i])})")


class ReducedSweep:
    """Affine reduced operator on the device and its batched frequency sweep.

    A_r(f) = sum_k alpha_k(f) P_k with alpha from `kinds` (K -> 1, D -> i w,
    M -> -w^2, mor.py:79-85) or an explicit `coeff_fn(freqs) -> (F, n_prim)`;
    b_r (r, s) and c_r (n_out, r) as in ReducedModel.reduced_system / output.
    Host numpy inputs are copied to the device once here (pinned staging).
    """

    def __init__(self, prims, b_r, c_r, kinds=None, coeff_fn=None, device=None, stream=None):
        _lib.require_cuda()
        self.device = torch.device(device or "cuda")
        self.stream = stream
        self.P = _to_dev(prims, self.device)
        self.b = _to_dev(b_r if np.ndim(b_r) != 1 else np.asarray(b_r)[:, None], self.device)
        self.c = _to_dev(np.atleast_2d(c_r) if not isinstance(c_r, torch.Tensor) else c_r, self.device)
        if (kinds is None) == (coeff_fn is None):
            raise ValueError("give exactly one of kinds / coeff_fn")
        self.kinds = tuple(kinds) if kinds is not None else None
        self.coeff_fn = coeff_fn

    @property
    def r(self):
        return self.P.shape[1]

    def alpha(self, freqs: torch.Tensor) -> torch.Tensor:
        if self.coeff_fn is not None:
            return _to_dev(self.coeff_fn(freqs), self.device)
        return affine_coefficients(freqs, [(k, 1.0) for k in self.kinds])

    def sweep_device(self, freqs: torch.Tensor, want_y=True, want_spl=True, want_x=False) -> SweepOut:
        f = freqs.to(self.device, torch.float64)
        return rom_sweep_affine(self.P, self.alpha(f), self.b, self.c, want_y=want_y,
                                want_spl=want_spl, want_x=want_x, stream=self.stream)

    def sweep(self, freqs, check_singular=True):
        """Host in, host out: (y (F, n_out, s), spl (F, s)) numpy arrays."""
        f = torch.as_tensor(np.asarray(freqs, dtype=np.float64)).pin_memory().to(self.device, non_blocking=True)
        out = self.sweep_device(f)
        y = torch.empty(out.y.shape, dtype=out.y.dtype, pin_memory=True)
        spl = torch.empty(out.spl.shape, dtype=out.spl.dtype, pin_memory=True)
        st = self.stream if self.stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(st):  # the kernel's stream: copy after it, then wait for it
            y.copy_(out.y, non_blocking=True)
            spl.copy_(out.spl, non_blocking=True)
            info = out.info.to("cpu", non_blocking=True)
        st.synchronize()
        if check_singular:
            raise_if_singular(info)
        return y.numpy(), spl.numpy()


def _to_dev(a, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        if a.device.type == "cpu" and not a.is_pinned():
            a = a.pin_memory()
        return a.to(device=device, dtype=CDT, non_blocking=True).contiguous()
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.complex128)).pin_memory()
    return t.to(device, non_blocking=True)
