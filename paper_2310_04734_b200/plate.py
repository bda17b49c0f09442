"""cfg2 plate–cavity model on the GPU: 9-node Reissner–Mindlin
+ membrane plate with clamped edges (vb_rm_plate_elements), conforming
fluid–structure coupling (vb_quad9_face_mass on the wet face), and the 30°
plane-wave load, all assembled with the deterministic CSR builder
(vb_csr_pattern_from_blocks + vb_csr_gather) in one global DoF numbering
[plate free DoFs | cavity pressures].

Conventions follow the reference (no RM element exists there): coupling
C = int N_s N_f n dGamma on the normal DoF with n the structure->fluid normal,
-C in K (structure rows) and +rho_f C^T in M (fluid rows)
(vibrofem/assembly.py:4-8, 193-207; docs/formulas.md:20-25); hysteretic
damping (1 + i eta(f)) on the plate stiffness (materials.py:170-172); plane
wave p e^{-i k sin(theta) x} along the inward normal of the loaded face
(assembly.py:108-139).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib, assembly, linalg
from .assembly import DeviceCSR

NDOF = 5  # u, v, w, bx, by


def plate_mesh(rect, nx: int, ny: int, z: float):
    """Structured lexicographic quad9 plate in the plane z: xyz (n, 3), conn (n_e, 9)."""
    x0, y0, x1, y1 = rect
    npx, npy = 2 * nx + 1, 2 * ny + 1
    xs = x0 + (x1 - x0) * np.arange(npx) / (npx - 1)
    ys = y0 + (y1 - y0) * np.arange(npy) / (npy - 1)
    Y, X = np.meshgrid(ys, xs, indexing="ij")
    xyz = np.column_stack([X.ravel(), Y.ravel(), np.full(npx * npy, z)])
    ey, ex = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    base = (2 * ey * npx + 2 * ex).reshape(-1, 1)
    b, a = np.meshgrid(np.arange(3), np.arange(3), indexing="ij")
    conn = (base + (b * npx + a).reshape(1, -1)).astype(np.int32)
    return xyz, conn


def clamped_dof_map(nx: int, ny: int):
    """Free-DoF number of (node, dof); -1 on the clamped boundary nodes."""
    npx, npy = 2 * nx + 1, 2 * ny + 1
    j, i = np.meshgrid(np.arange(npy), np.arange(npx), indexing="ij")
    free = ((i > 0) & (i < npx - 1) & (j > 0) & (j < npy - 1)).ravel()
    dmap = -np.ones((npx * npy, NDOF), dtype=np.int64)
    nf = int(free.sum())
    dmap[free] = np.arange(nf * NDOF).reshape(nf, NDOF)
    return dmap.astype(np.int32), nf * NDOF


def assemble_blocks(n_rows: int, n_cols: int, rdofs: np.ndarray, cdofs: np.ndarray, vals: torch.Tensor,
                    device) -> DeviceCSR:
    """Canonical CSR of element blocks (rows = repeat(rdofs), cols = tile(cdofs),
    negative DoFs dropped) with element-order sums (assembly.py:160-175)."""
    lib = _lib.load()
    ne, nr = rdofs.shape
    nc = cdofs.shape[1]
    rd = torch.as_tensor(np.ascontiguousarray(rdofs, dtype=np.int32), device=device)
    cd = torch.as_tensor(np.ascontiguousarray(cdofs, dtype=np.int32), device=device)
    T = ne * nr * nc
    indptr = torch.empty(n_rows + 1, dtype=torch.int32, device=device)
    indices = torch.empty(T, dtype=torch.int32, device=device)
    gptr = torch.empty(T + 1, dtype=torch.int64, device=device)
    gidx = torch.empty(T, dtype=torch.int32, device=device)
    wb = lib.vb_csr_pattern_blocks_workspace_bytes(n_rows, n_cols, ne, nr, nc)
    work = torch.empty(wb, dtype=torch.uint8, device=device)
    nnz = C.c_int64(0)
    _lib.check(lib.vb_csr_pattern_from_blocks(n_rows, n_cols, ne, nr, nc, _lib.ptr(rd), _lib.ptr(cd),
                                              _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(gptr), _lib.ptr(gidx),
                                              C.byref(nnz), _lib.ptr(work), wb, _lib.stream_handle()),
               "vb_csr_pattern_from_blocks")
    k = int(nnz.value)
    pat = assembly.Pattern(n_rows, indptr, indices[:k].clone(), gptr[:k + 1].clone(), gidx)
    return pat.gather(vals.reshape(-1).contiguous())


def plate_elements(xyz_d: torch.Tensor, conn_d: torch.Tensor, E, nu, rho, t):
    lib = _lib.load()
    ne = conn_d.shape[0]
    Ke = torch.empty((ne, 45, 45), dtype=torch.float64, device=xyz_d.device)
    Me = torch.empty_like(Ke)
    bad = C.c_int32(-1)
    _lib.check(lib.vb_rm_plate_elements(ne, _lib.ptr(xyz_d), _lib.ptr(conn_d), float(E), float(nu), float(rho),
                                        float(t), _lib.ptr(Ke), _lib.ptr(Me), C.byref(bad), _lib.stream_handle()),
               "vb_rm_plate_elements")
    if bad.value >= 0:
        raise ValueError(f"non-positive Jacobian in plate element {bad.value}")
    return Ke, Me


class PlaneWaveLoad:
    """p_hat e^{-i k sin(theta) (x - x0)} on the plate's exterior face, acting
    along the inward normal (-z): f = G e(k) with G[w-DoF, gauss point] =
    -w det N_a (a constant real CSR on the device) and e(k) the phase at the
    Gauss points — one SpMM evaluates any batch of frequencies."""

    def __init__(self, xyz, conn, dmap, n_total: int, c0: float, theta: float, amp: float = 1.0,
                 device=None):
        dev = torch.device(device or "cuda")
        g1 = np.array([-math.sqrt(0.6), 0.0, math.sqrt(0.6)])
        w1 = np.array([5 / 9, 8 / 9, 5 / 9])
        L = lambda x: np.array([0.5 * x * (x - 1.0), 1.0 - x * x, 0.5 * x * (x + 1.0)])
        dL = lambda x: np.array([x - 0.5, -2.0 * x, x + 0.5])
        rows, cols, vals, xg = [], [], [], []
        g = 0
        for e, cn in enumerate(conn):
            X = xyz[cn][:, :2]
            for gy in range(3):
                for gx in range(3):
                    Nx, Ny, dNx, dNy = L(g1[gx]), L(g1[gy]), dL(g1[gx]), dL(g1[gy])
                    N = np.array([Nx[a] * Ny[b] for b in range(3) for a in range(3)])
                    dS = np.array([[dNx[a] * Ny[b], Nx[a] * dNy[b]] for b in range(3) for a in range(3)])
                    det = np.linalg.det(dS.T @ X)
                    xg.append(N @ X[:, 0])
                    for a in range(9):
                        d = dmap[cn[a], 2]
                        if d >= 0:
                            rows.append(d)
                            cols.append(g)
                            vals.append(-amp * w1[gx] * w1[gy] * det * N[a])
                    g += 1
        import scipy.sparse as sp
        G = sp.csr_matrix((vals, (rows, cols)), shape=(n_total, g))
        G.sum_duplicates()
        self.G = DeviceCSR(n_total, torch.as_tensor(G.indptr.astype(np.int32), device=dev),
                           torch.as_tensor(G.indices.astype(np.int32), device=dev),
                           torch.as_tensor(G.data, device=dev))
        self.xg = torch.as_tensor(np.array(xg) - xyz[:, 0].min(), device=dev)
        self.c0, self.theta, self.n = c0, theta, n_total
        self.G_host = G
        self.xg_host = self.xg.cpu().numpy()

    def phases(self, freqs) -> torch.Tensor:
        k = 2.0 * math.pi * torch.as_tensor(np.asarray(freqs, float), device=self.xg.device) / self.c0 \
            * math.sin(self.theta)
        return torch.exp(-1j * torch.outer(self.xg, k).to(torch.complex128)).contiguous()  # (n_gp, F)

    def batch(self, freqs) -> torch.Tensor:
        """(n, F) load block for a batch of frequencies (one SpMM)."""
        return linalg.spmm(self.G, self.phases(freqs))

    def at(self, f: float) -> torch.Tensor:
        return self.batch([f])

    def host(self, f: float) -> np.ndarray:
        k = 2.0 * math.pi * f / self.c0 * math.sin(self.theta)
        return self.G_host @ np.exp(-1j * k * self.xg_host)


def eta_cfg2(f, f0: float = 20.0, f1: float = 500.0) -> float:
    """eta(f) = 0.01 + 2e-5 f as a two-sample LossFactorTable (materials.py:99-109)."""
    e0, e1 = 0.01 + 2e-5 * f0, 0.01 + 2e-5 * f1
    if f <= f0:
        return e0
    if f >= f1:
        return e1
    return e0 + (e1 - e0) * (f - f0) / (f1 - f0)
