"""Seeded synthetic inputs with the shapes of BASELINE.json's configs (host-side
input generation; no datasets exist for this path).

cfg5 "reduced-sweep throughput stress": dense complex128 reduced matrices
  K_r = sigma_K (X X^H / r + I) (1 + i eta)     Hermitian PD plus i eta K
  M_r = Y Y^H / r + I                            Hermitian PD
  D_r = sigma_D U U^H / r,   U: r x 32           low rank 32
  B   : r x 16 RHS, entries N(0,1) + i N(0,1)
  C_R : 50 x r output rows, entries N(0,1) + i N(0,1)
  f   = linspace(1, 1000, 100000)
The construction mirrors tests/test_mor.py:26-37 (frozen_fom); sigma_K places
the undamped eigenfrequencies (~134–670 Hz) inside the swept band so the LU
pivots through resonances, and sigma_D is a 5 %-of-critical viscous scale.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

CFG5_ORDERS = (256, 1024, 2048)
CFG5_NFREQ = 100_000
CFG5_RHS = 16
CFG5_NOUT = 50
CFG5_DRANK = 32
CFG5_ETA = 0.02


@dataclass
class ReducedWorkload:
    name: str
    prims: np.ndarray      # (3, r, r): [K_r (1+i eta), D_r, M_r]
    kinds: tuple           # ('K', 'D', 'M') — alpha = [1, i w, -w^2]
    b: np.ndarray          # (r, s)
    c_r: np.ndarray        # (n_out, r)
    freqs: np.ndarray      # (F,)
    seed: int

    @property
    def r(self):
        return self.prims.shape[1]

    def alpha(self, freqs=None) -> np.ndarray:
        f = self.freqs if freqs is None else np.asarray(freqs, float)
        w = 2.0 * math.pi * f
        cols = {"K": np.ones_like(w, dtype=complex), "D": 1j * w, "M": -(w * w) + 0j}
        return np.stack([cols[k] for k in self.kinds], axis=1)


def _cn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def cfg5(r: int = 1024, n_freq: int = CFG5_NFREQ, s: int = CFG5_RHS, n_out: int = CFG5_NOUT,
         seed: int = 5, f_lo: float = 1.0, f_hi: float = 1000.0) -> ReducedWorkload:
    rng = np.random.default_rng(seed)
    sig_k = (2.0 * math.pi * 300.0) ** 2
    X = _cn(rng, r, r)
    Y = _cn(rng, r, r)
    M = Y @ Y.conj().T / r + np.eye(r)
    U = _cn(rng, r, CFG5_DRANK)
    sig_d = 2 * 0.05 * (2.0 * math.pi * 300.0)
    D = sig_d * (U @ U.conj().T) / r
    # enforce exact Hermitian symmetry of the PD parts (rounding of X X^H)
    M = 0.5 * (M + M.conj().T)
    D = 0.5 * (D + D.conj().T)
    Kh = sig_k * (X @ X.conj().T / r + np.eye(r))
    K = 0.5 * (Kh + Kh.conj().T) * (1 + 1j * CFG5_ETA)
    B = _cn(rng, r, s)
    C = _cn(rng, n_out, r)
    freqs = np.linspace(f_lo, f_hi, n_freq)
    return ReducedWorkload(name=f"cfg5_r{r}", prims=np.stack([K, D, M]), kinds=("K", "D", "M"),
                           b=B, c_r=C, freqs=freqs, seed=seed)
