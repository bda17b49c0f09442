"""FE primitives on the GPU: structured hex27 boxes, Helmholtz Kgrad/Mnn, impedance
face matrices, point sources, deterministic CSR (SURVEY §8a A1–A3, A6).

Host side of `vb_csr_pattern_from_elements`, `vb_hex27_helmholtz_elements`,
`vb_quad9_face_mass`, `vb_csr_gather`.  Mesh generation is host plumbing (the
reference's meshing.py:44-95, generalised lexicographically to 3D).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


# ------------------------------------------------------------- meshing -----
def hex27_box(box, nx: int, ny: int, nz: int):
    """Structured 27-node hexahedra over an axis-aligned box (meshing.py:44-95
    in 3D): node id k*npx*npy + j*npx + i, element (ez*ny + ey)*nx + ex, local
    node a + 3b + 9c.  Returns (xyz (n, 3) float64, conn (n_elem, 27) int32)."""
    x0, y0, z0, x1, y1, z1 = box
    npx, npy, npz = 2 * nx + 1, 2 * ny + 1, 2 * nz + 1
    xs = x0 + (x1 - x0) * np.arange(npx) / (npx - 1)
    ys = y0 + (y1 - y0) * np.arange(npy) / (npy - 1)
    zs = z0 + (z1 - z0) * np.arange(npz) / (npz - 1)
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    xyz = np.column_stack([X.ravel(), Y.ravel(), Z.ravel()])
    ez, ey, ex = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    base = ((2 * ez) * npy + 2 * ey) * npx + 2 * ex            # (nz, ny, nx)
    c, b, a = np.meshgrid(np.arange(3), np.arange(3), np.arange(3), indexing="ij")
    loc = (c * npy + b) * npx + a                               # (3, 3, 3) -> a + 3b + 9c order
    conn = (base.reshape(-1, 1) + loc.reshape(1, -1)).astype(np.int32)
    return xyz, conn


def hex27_box_face(ne, side: str, conn: np.ndarray):
    """9-node face connectivity (lexicographic in the two free axes) of one box
    side ('x0','x1','y0','y1','z0','z1')."""
    nx, ny, nz = ne
    axis = "xyz".index(side[0])
    hi = side[1] == "1"
    e3 = np.stack(np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij"), -1)
    e3 = e3.reshape(-1, 3)[:, ::-1]  # (ex, ey, ez) in element order
    sel = e3[:, axis] == ((nx, ny, nz)[axis] - 1 if hi else 0)
    elems = np.nonzero(sel)[0]
    free = [d for d in range(3) if d != axis]
    loc = []
    for t in range(3):
        for s in range(3):
            abc = [0, 0, 0]
            abc[axis] = 2 if hi else 0
            abc[free[0]] = s
            abc[free[1]] = t
            loc.append(abc[0] + 3 * abc[1] + 9 * abc[2])
    return conn[elems][:, loc].astype(np.int32)


def interior_nodes(xyz: np.ndarray, box, tol=1e-12):
    x0, y0, z0, x1, y1, z1 = box
    lo = np.array([x0, y0, z0]) + tol
    hi = np.array([x1, y1, z1]) - tol
    return np.nonzero(np.all((xyz > lo) & (xyz < hi), axis=1))[0]


# ----------------------------------------------------------------- CSR -----
@dataclass
class KronBox:
    """Kronecker form of a uniform-box primitive (vb_kron3_apply): node grid,
    [3][maxnp][5] band tables of the 1D stiffness/mass, stiff = Kgrad (1) or Mnn (0)."""

    npx: int
    npy: int
    npz: int
    K1: torch.Tensor
    M1: torch.Tensor
    maxnp: int
    stiff: int


@dataclass
class DeviceCSR:
    """Square CSR on the device: int32 indptr/indices, float64 values (one
    primitive) — the scipy canonical layout of assembly.py:172-173.  `kron`,
    when set, is the same operator in Kronecker form (uniform boxes): products
    with it run matrix-free (linalg.spmm)."""

    n: int
    indptr: torch.Tensor
    indices: torch.Tensor
    data: torch.Tensor
    kron: KronBox | None = None

    @property
    def nnz(self) -> int:
        return int(self.indices.numel())

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.data.cpu().numpy(), self.indices.cpu().numpy(),
                              self.indptr.cpu().numpy()), shape=(self.n, self.n))

    def with_data(self, data: torch.Tensor) -> "DeviceCSR":
        return DeviceCSR(self.n, self.indptr, self.indices, data)


@dataclass
class Pattern:
    n: int
    indptr: torch.Tensor
    indices: torch.Tensor
    gather_ptr: torch.Tensor
    gather_idx: torch.Tensor

    @property
    def nnz(self) -> int:
        return int(self.indices.numel())

    def gather(self, triplet_vals: torch.Tensor) -> DeviceCSR:
        lib = _lib.load()
        vals = torch.empty(self.nnz, dtype=torch.float64, device=self.indptr.device)
        tv = triplet_vals.contiguous()  # alive through the launch (a temporary copy otherwise)
        _lib.check(lib.vb_csr_gather(self.nnz, _lib.ptr(self.gather_ptr), _lib.ptr(self.gather_idx),
                                     _lib.ptr(tv), _lib.ptr(vals), _lib.stream_handle()), "vb_csr_gather")
        return DeviceCSR(self.n, self.indptr, self.indices, vals)

    def gather2(self, tv0: torch.Tensor, tv1: torch.Tensor):
        """Two primitives on this pattern in one pass over the gather map."""
        lib = _lib.load()
        v0 = torch.empty(self.nnz, dtype=torch.float64, device=self.indptr.device)
        v1 = torch.empty_like(v0)
        t0, t1 = tv0.contiguous(), tv1.contiguous()  # alive through the launch
        _lib.check(lib.vb_csr_gather2(self.nnz, _lib.ptr(self.gather_ptr), _lib.ptr(self.gather_idx),
                                      _lib.ptr(t0), _lib.ptr(t1), _lib.ptr(v0), _lib.ptr(v1),
                                      _lib.stream_handle()), "vb_csr_gather2")
        return (DeviceCSR(self.n, self.indptr, self.indices, v0), DeviceCSR(self.n, self.indptr, self.indices, v1))


def pattern_from_elements(n: int, conn_dev: torch.Tensor) -> Pattern:
    """vb_csr_pattern_from_elements: canonical CSR pattern + element-order gather map."""
    lib = _lib.load()
    ne, npe = conn_dev.shape
    T = ne * npe * npe
    dev = conn_dev.device
    indptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    indices = torch.empty(T, dtype=torch.int32, device=dev)
    gptr = torch.empty(T + 1, dtype=torch.int64, device=dev)
    gidx = torch.empty(T, dtype=torch.int32, device=dev)
    wb = lib.vb_csr_pattern_workspace_bytes(n, ne, npe)
    work = torch.empty(wb, dtype=torch.uint8, device=dev)
    nnz = C.c_int64(0)
    _lib.check(lib.vb_csr_pattern_from_elements(n, ne, npe, _lib.ptr(conn_dev), _lib.ptr(indptr),
                                                _lib.ptr(indices), _lib.ptr(gptr), _lib.ptr(gidx),
                                                C.byref(nnz), _lib.ptr(work), wb, _lib.stream_handle()),
               "vb_csr_pattern_from_elements")
    k = int(nnz.value)
    return Pattern(n, indptr, indices[:k].clone(), gptr[:k + 1].clone(), gidx)


def hex27_helmholtz(xyz_dev: torch.Tensor, conn_dev: torch.Tensor):
    """Per-element Kgrad_e, Mnn_e (n_elem, 27, 27) on the device (assembly.py:77-91)."""
    lib = _lib.load()
    ne = conn_dev.shape[0]
    Ke = torch.empty((ne, 27, 27), dtype=torch.float64, device=xyz_dev.device)
    Me = torch.empty_like(Ke)
    bad = C.c_int32(-1)
    _lib.check(lib.vb_hex27_helmholtz_elements(ne, _lib.ptr(xyz_dev), _lib.ptr(conn_dev), _lib.ptr(Ke),
                                               _lib.ptr(Me), C.byref(bad), _lib.stream_handle()),
               "vb_hex27_helmholtz_elements")
    if bad.value >= 0:
        raise ValueError(f"non-positive Jacobian in Helmholtz element {bad.value}")
    return Ke, Me


def face_mass(xyz_dev: torch.Tensor, fconn_dev: torch.Tensor) -> torch.Tensor:
    lib = _lib.load()
    nf = fconn_dev.shape[0]
    Fe = torch.empty((nf, 9, 9), dtype=torch.float64, device=xyz_dev.device)
    _lib.check(lib.vb_quad9_face_mass(nf, _lib.ptr(xyz_dev), _lib.ptr(fconn_dev), _lib.ptr(Fe),
                                      _lib.stream_handle()), "vb_quad9_face_mass")
    return Fe


def assemble_helmholtz(xyz, conn, device=None):
    """_assemble_primitives(kind='acoustic') on the GPU (assembly.py:142-175):
    returns (Kgrad, Mnn) DeviceCSR sharing one pattern."""
    _lib.require_cuda()
    dev = torch.device(device or "cuda")
    xyz_d = torch.as_tensor(np.ascontiguousarray(xyz, dtype=np.float64), device=dev)
    conn_d = torch.as_tensor(np.ascontiguousarray(conn, dtype=np.int32), device=dev)
    pat = pattern_from_elements(xyz.shape[0], conn_d)
    Ke, Me = hex27_helmholtz(xyz_d, conn_d)
    return pat.gather2(Ke, Me)


def assemble_face_mass(xyz, face_conn, device=None) -> DeviceCSR:
    dev = torch.device(device or "cuda")
    xyz_d = torch.as_tensor(np.ascontiguousarray(xyz, dtype=np.float64), device=dev)
    f_d = torch.as_tensor(np.ascontiguousarray(face_conn, dtype=np.int32), device=dev)
    pat = pattern_from_elements(xyz.shape[0], f_d)
    return pat.gather(face_mass(xyz_d, f_d))


def assemble_weighted_face_mass(xyz, face_conn, weights, device=None) -> DeviceCSR:
    """sum_e w_e int_{Gamma_e} N N^T dGamma over the given 9-node faces (real
    per-element weights, e.g. 1 / Z_e of an impedance wall whose impedance
    varies per element): element matrices scaled before the deterministic
    element-order gather, so the CSR pattern is the unweighted face mass's."""
    dev = torch.device(device or "cuda")
    xyz_d = torch.as_tensor(np.ascontiguousarray(xyz, dtype=np.float64), device=dev)
    f_d = torch.as_tensor(np.ascontiguousarray(face_conn, dtype=np.int32), device=dev)
    pat = pattern_from_elements(xyz.shape[0], f_d)
    Fe = face_mass(xyz_d, f_d)
    w = torch.as_tensor(np.asarray(weights, dtype=np.float64), device=dev).view(-1, *([1] * (Fe.dim() - 1)))
    return pat.gather((Fe * w).contiguous())


def box_band_tables(box, ne):
    """[3][maxnp][5] band entries of the assembled 1D quadratic stiffness / mass
    along x, y, z (host; a few KB)."""
    from .fdm import line_matrices
    x0, y0, z0, x1, y1, z1 = box
    maxnp = 2 * max(ne) + 1
    K1 = np.zeros((3, maxnp, 5))
    M1 = np.zeros((3, maxnp, 5))
    for d, (L, m) in enumerate(zip((x1 - x0, y1 - y0, z1 - z0), ne)):
        K, M = line_matrices(L, m)
        npd = 2 * m + 1
        for i in range(npd):
            for o in range(5):
                j = i + o - 2
                if 0 <= j < npd:
                    K1[d, i, o] = K[i, j]
                    M1[d, i, o] = M[i, j]
    return K1, M1, maxnp


def assemble_helmholtz_box(box, ne, device=None):
    """Structured fast path for a uniform box (vb_hex27_box_csr): analytic
    canonical pattern, Kronecker-form values.  Same CSR as
    assemble_helmholtz(hex27_box(...)) (pattern bit-exact, values to rounding)."""
    _lib.require_cuda()
    lib = _lib.load()
    dev = torch.device(device or "cuda")
    nx, ny, nz = ne
    K1, M1, maxnp = box_band_tables(box, ne)
    K1d = torch.as_tensor(K1, device=dev)
    M1d = torch.as_tensor(M1, device=dev)
    n = (2 * nx + 1) * (2 * ny + 1) * (2 * nz + 1)
    nnz = int(lib.vb_hex27_box_nnz(nx, ny, nz))
    indptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    indices = torch.empty(nnz, dtype=torch.int32, device=dev)
    Kv = torch.empty(nnz, dtype=torch.float64, device=dev)
    Mv = torch.empty(nnz, dtype=torch.float64, device=dev)
    _lib.check(lib.vb_hex27_box_csr(nx, ny, nz, _lib.ptr(K1d), _lib.ptr(M1d), maxnp, _lib.ptr(indptr),
                                    _lib.ptr(indices), _lib.ptr(Kv), _lib.ptr(Mv), _lib.stream_handle()),
               "vb_hex27_box_csr")
    grid = (2 * nx + 1, 2 * ny + 1, 2 * nz + 1)
    return (DeviceCSR(n, indptr, indices, Kv, KronBox(*grid, K1d, M1d, maxnp, 1)),
            DeviceCSR(n, indptr, indices, Mv, KronBox(*grid, K1d, M1d, maxnp, 0)))
