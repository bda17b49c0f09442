"""Oracle restatement of the rational-Arnoldi MOR sweep algebra (SURVEY §8a
A6–A15) — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reference anchors (vibrofem/):
  mor.py:22        ORTH_DROP_TOL = 1e-10
  mor.py:41-53     FullOrderModel.operator / solve (splu per call) / output
  mor.py:73-98     ReducedModel.reduced_system / solve (LAPACK zgesv) / output
  mor.py:122-135   _orthonormalise (MGS, two passes, relative drop)
  mor.py:138-191   krylov_block + _arnoldi_step (first/second-order recurrences)
  mor.py:194-208   relative_error
  mor.py:366-394   rom_sweep (first containing window owns f; seam log)
  solvers.py:25,334-338  P_REF, mean_spl
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

ORTH_DROP_TOL = 1e-10
P_REF = 20e-6


@dataclass
class Fom:
    """Provider container with the reference's FullOrderModel semantics (mor.py:25-53)."""

    stiffness: object
    mass: object
    load: object
    c_out: np.ndarray
    n: int
    damping: object = None

    def operator(self, f):
        w = 2.0 * math.pi * f
        A = self.stiffness(f) - w * w * self.mass(f)
        if self.damping is not None:
            A = A + 1j * w * self.damping(f)
        return A

    def solve(self, f):
        return spla.splu(sp.csc_matrix(self.operator(f))).solve(self.load(f))

    def output(self, x):
        y = self.c_out @ x
        return complex(y) if np.ndim(y) == 0 else y


def mgs2_against(cols, w):
    """Two passes of modified Gram–Schmidt of w against cols (mor.py:129-131, 185-187)."""
    for _ in range(2):
        for q in cols:
            w = w - np.vdot(q, w) * q
    return w


def orthonormalise(V, block):
    """mor.py:122-135."""
    cols = [] if V is None or V.size == 0 else list(V.T)
    for j in range(block.shape[1]):
        w = block[:, j].astype(complex)
        ref = np.linalg.norm(w)
        w = mgs2_against(cols, w)
        nw = np.linalg.norm(w)
        if ref > 0 and nw > ORTH_DROP_TOL * ref:
            cols.append(w / nw)
    return np.column_stack(cols) if cols else np.zeros((block.shape[0], 0), complex)


def krylov_block(fom: Fom, f_j, m, second_order=False):
    """mor.py:138-191: one factorisation at f_j, m moment vectors, MGS2 within the block."""
    if m < 1:
        raise ValueError("moment count must be >= 1")
    lu = spla.splu(sp.csc_matrix(fom.operator(f_j)))
    Mt = fom.mass(f_j)
    v = lu.solve(fom.load(f_j))
    nv = np.linalg.norm(v)
    if nv == 0:
        raise ValueError("zero load at expansion point")
    cols = [v / nv]
    use2 = second_order and fom.damping is not None
    if use2:
        w0 = 2.0 * math.pi * f_j
        Dt = fom.damping(f_j) + 2j * w0 * fom.mass(f_j)
        prev = np.zeros_like(v)
    breakdown = False
    for _ in range(1, m):
        if use2:
            w = -lu.solve(Dt @ cols[-1] + Mt @ prev)
            prev = cols[-1]
        else:
            w = -lu.solve(Mt @ cols[-1])
        ref = np.linalg.norm(w)
        w = mgs2_against(cols, w)
        nw = np.linalg.norm(w)
        if ref == 0 or nw <= ORTH_DROP_TOL * ref:
            breakdown = True
            break
        cols.append(w / nw)
    return np.column_stack(cols), breakdown


def reduced_output(fom: Fom, V, f, rayleigh=None):
    """ReducedModel.output (mor.py:73-98): literal per-frequency re-projection."""
    w = 2.0 * math.pi * f
    Vh = V.conj().T
    KR = Vh @ (fom.stiffness(f) @ V)
    MR = Vh @ (fom.mass(f) @ V)
    AR = KR - w * w * MR
    if fom.damping is not None:
        AR = AR + 1j * w * (Vh @ (fom.damping(f) @ V))
    if rayleigh is not None:
        a, b = rayleigh
        AR = AR + 1j * w * (a * MR + b * KR)
    bR = Vh @ fom.load(f)
    y = (fom.c_out @ V) @ np.linalg.solve(AR, bR)
    return complex(y) if np.ndim(y) == 0 else y


def affine_sweep(prims, alpha, b, c_r):
    """Reduced sweep over an affine operator A(f_i) = sum_k alpha[i,k] prims[k]
    (algebraically mor.py:73-90 with frequency dependence factored into scalars,
    SURVEY §0 finding 4), then numpy.linalg.solve (mor.py:94 = LAPACK zgesv),
    y = c_r @ x (mor.py:96-102) and mean_spl per RHS column (solvers.py:334-338).

    prims: (K, r, r); alpha: (F, K); b: (r, s) or (F, r, s); c_r: (n_o, r).
    Returns (y (F, n_o, s), spl (F, s)).
    """
    F = alpha.shape[0]
    r = prims.shape[1]
    b = np.asarray(b, complex)
    s = b.shape[-1]
    y = np.empty((F, c_r.shape[0], s), complex)
    spl = np.empty((F, s))
    for i in range(F):
        A = np.tensordot(alpha[i], prims, axes=1)
        x = np.linalg.solve(A, b[i] if b.ndim == 3 else b)
        y[i] = c_r @ x
        for c in range(s):
            spl[i, c] = mean_spl(y[i, :, c])
    return y, spl


def relative_error(y_full, y_rom):
    """mor.py:194-208."""
    y_full = np.asarray(y_full, dtype=complex)
    y_rom = np.asarray(y_rom, dtype=complex)
    denom = np.abs(y_full)
    absolute = denom == 0
    eps = np.abs(y_full - y_rom)
    eps = np.where(absolute, eps, eps / np.where(absolute, 1.0, denom))
    k = int(np.argmax(eps)) if eps.size else 0
    return eps, (float(eps[k]) if eps.size else 0.0), k, bool(absolute.any())


def mean_spl(p):
    """solvers.py:334-338."""
    p_rms = math.sqrt(float(np.mean(np.abs(p) ** 2)) / 2.0)
    return 20.0 * math.log10(max(p_rms, 1e-300) / P_REF)


def window_owners(windows, grid):
    """rom_sweep owner rule (mor.py:376-385): lower window wins at seams;
    returns (owner index per f, [(f index, upper owner)] at seams)."""
    windows = sorted(windows)
    own, seams = [], []
    for i, f in enumerate(grid):
        ks = [k for k, (lo, hi) in enumerate(windows) if lo <= f <= hi]
        if not ks:
            raise ValueError(f"frequency {f} outside every ROM window")
        own.append(ks[0])
        if len(ks) > 1:
            seams.append((i, ks[1]))
    return own, seams
