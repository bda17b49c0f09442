"""Oracle restatement of the FE primitives feeding the MOR path (SURVEY §8a A1–A3,
A6): 1D quadratic Lagrange bases, Gauss rules, 9-node quad / 27-node hex
Helmholtz element integrals, structured meshes, triplet → canonical CSR,
impedance face matrices and point sources.  TEST INFRASTRUCTURE ONLY (see
oracle/__init__.py).

Reference anchors (vibrofem/):
  shape.py:20-26      _lag1d / _dlag1d (quadratic Lagrange at -1, 0, 1)
  shape.py:9-13,30    LOCAL_NODES / _IDX (quad9 local node order)
  shape.py:56-65      gauss1d / gauss2d (numpy leggauss, x fastest)
  shape.py:73-75      jacobian = dshape^T @ coords
  assembly.py:77-91   helmholtz_element_parts (dN = dshape @ inv(J))
  assembly.py:142-175 _assemble_primitives (repeat/tile triplets, COO->CSR)
  meshing.py:44-95    generate_mesh (node id j*npx+i, element ey*nx+ex)
The 3D hex27 pieces generalise these lexicographically (SURVEY §8a "Not in the
reference"): node id k*npx*npy + j*npx + i, element ez*nx*ny + ey*nx + ex,
local node a + 3b + 9c, Gauss points x fastest.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

QUAD_ORDER = 3  # assembly.py:28


def lag1d(x: float) -> np.ndarray:
    """shape.py:20-22."""
    return np.array([0.5 * x * (x - 1.0), 1.0 - x * x, 0.5 * x * (x + 1.0)])


def dlag1d(x: float) -> np.ndarray:
    """shape.py:25-26."""
    return np.array([x - 0.5, -2.0 * x, x + 0.5])


def gauss1d(n: int = QUAD_ORDER):
    """shape.py:56-57."""
    return np.polynomial.legendre.leggauss(n)


def gauss_nd(dim: int, n: int = QUAD_ORDER):
    """Tensor-product rule, first coordinate fastest (shape.py:60-65 in 2D)."""
    x, w = gauss1d(n)
    idx = np.indices((n,) * dim).reshape(dim, -1)[::-1]  # idx[0] fastest
    pts = x[idx].T
    wts = np.prod(w[idx], axis=0)
    return pts, wts


# local node tables: 1D index (0,1,2) <-> reference coordinate (-1,0,1)
QUAD9_IDX = np.array([(0, 0), (2, 0), (2, 2), (0, 2), (1, 0), (2, 1), (1, 2), (0, 1), (1, 1)])  # shape.py:9-13
HEX27_IDX = np.array([(a, b, c) for c in range(3) for b in range(3) for a in range(3)])
QUAD9_LEX_IDX = np.array([(a, b) for b in range(3) for a in range(3)])  # hex27 face order


def shape_nd(idx: np.ndarray, xi) -> np.ndarray:
    """N_i(xi) = prod_d lag1d(xi_d)[idx_d(i)] (shape.py:32-35)."""
    L = [lag1d(x) for x in xi]
    return np.array([np.prod([L[d][row[d]] for d in range(len(xi))]) for row in idx])


def dshape_nd(idx: np.ndarray, xi) -> np.ndarray:
    """dN_i/dxi_a (shape.py:38-47); shape (nn, dim)."""
    dim = len(xi)
    L = [lag1d(x) for x in xi]
    D = [dlag1d(x) for x in xi]
    out = np.empty((idx.shape[0], dim))
    for i, row in enumerate(idx):
        for a in range(dim):
            out[i, a] = np.prod([(D if d == a else L)[d][row[d]] for d in range(dim)])
    return out


def helmholtz_element_parts(idx: np.ndarray, coords: np.ndarray):
    """Unscaled Laplacian and mass integrals of one Lagrange element
    (assembly.py:77-91, generalised to dim = coords.shape[1]).

    Follows the reference exactly: J = dshape^T @ coords, dN = dshape @ inv(J).
    """
    dim = coords.shape[1]
    pts, wts = gauss_nd(dim)
    nn = idx.shape[0]
    Kgrad = np.zeros((nn, nn))
    Mnn = np.zeros((nn, nn))
    for xi, w in zip(pts, wts):
        dS = dshape_nd(idx, xi)
        J = dS.T @ coords
        detJ = np.linalg.det(J)
        if detJ <= 0:
            raise ValueError("non-positive Jacobian in Helmholtz element")
        dN = dS @ np.linalg.inv(J)
        N = shape_nd(idx, xi)
        Kgrad += w * detJ * (dN @ dN.T)
        Mnn += w * detJ * np.outer(N, N)
    return Kgrad, Mnn


def structured_quad9(rect, nx: int, ny: int):
    """meshing.py:44-95 for given element counts: nodes (npx*npy, 2), elements (nx*ny, 9)."""
    x0, y0, x1, y1 = rect
    npx, npy = 2 * nx + 1, 2 * ny + 1
    xs = x0 + (x1 - x0) * np.arange(npx) / (npx - 1)
    ys = y0 + (y1 - y0) * np.arange(npy) / (npy - 1)
    X, Y = np.meshgrid(xs, ys, indexing="xy")
    nodes = np.column_stack([X.ravel(), Y.ravel()])
    elements = np.empty((nx * ny, 9), dtype=np.int64)
    for ey in range(ny):
        for ex in range(nx):
            i0, j0 = 2 * ex, 2 * ey
            elements[ey * nx + ex] = [(j0 + b) * npx + (i0 + a) for a, b in QUAD9_IDX]
    return nodes, elements


def structured_hex27(box, nx: int, ny: int, nz: int):
    """3D lexicographic generalisation of meshing.py:44-95."""
    x0, y0, z0, x1, y1, z1 = box
    npx, npy, npz = 2 * nx + 1, 2 * ny + 1, 2 * nz + 1
    xs = x0 + (x1 - x0) * np.arange(npx) / (npx - 1)
    ys = y0 + (y1 - y0) * np.arange(npy) / (npy - 1)
    zs = z0 + (z1 - z0) * np.arange(npz) / (npz - 1)
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    nodes = np.column_stack([X.ravel(), Y.ravel(), Z.ravel()])
    elements = np.empty((nx * ny * nz, 27), dtype=np.int64)
    for ez in range(nz):
        for ey in range(ny):
            for ex in range(nx):
                e = (ez * ny + ey) * nx + ex
                elements[e] = [((2 * ez + c) * npy + 2 * ey + b) * npx + 2 * ex + a
                               for a, b, c in HEX27_IDX]
    return nodes, elements


def triplets_to_csr(n: int, dofs: np.ndarray, vals: list[np.ndarray]):
    """assembly.py:160-175: rows = repeat(dofs, e), cols = tile(dofs, e) per
    element in index order; COO -> CSR; sum_duplicates.  Explicit zeros kept."""
    ne, es = dofs.shape
    rows = np.repeat(dofs, es, axis=1).ravel()
    cols = np.tile(dofs, (1, es)).ravel()
    out = []
    for v in vals:
        A = sp.coo_matrix((v.ravel(), (rows, cols)), shape=(n, n)).tocsr()
        A.sum_duplicates()
        out.append(A)
    return out


def assemble_helmholtz(nodes: np.ndarray, elements: np.ndarray, idx: np.ndarray):
    """_assemble_primitives for kind='acoustic' (assembly.py:142-175):
    returns (Kgrad, Mnn) canonical CSR."""
    ne, es = elements.shape
    Kv = np.empty((ne, es * es))
    Mv = np.empty((ne, es * es))
    cache = {}
    for e in range(ne):
        coords = nodes[elements[e]]
        key = np.round(coords - coords[0], 14).tobytes()  # translation-invariant reuse
        if key not in cache:
            cache[key] = helmholtz_element_parts(idx, coords)
        Ke, Me = cache[key]
        Kv[e] = Ke.ravel()
        Mv[e] = Me.ravel()
    return tuple(triplets_to_csr(nodes.shape[0], elements, [Kv, Mv]))


def face_mass_hex27(nodes: np.ndarray, elements: np.ndarray, face_elems: np.ndarray,
                    face_local: np.ndarray):
    """Impedance wall primitive int_Gamma N N^T dGamma over 9-node faces of hex27
    elements (restated: no reference counterpart; convention SURVEY §8c tier 1).

    face_local: 9 local node ids of the face in lexicographic (a, b) order.
    Returns the (n x n) canonical CSR of the face triplets (faces in given order).
    """
    pts, wts = gauss_nd(2)
    dofs = elements[face_elems][:, face_local]
    vals = np.empty((len(face_elems), 81))
    for f, e in enumerate(face_elems):
        X = nodes[dofs[f]]
        Me = np.zeros((9, 9))
        for xi, w in zip(pts, wts):
            dS = dshape_nd(QUAD9_LEX_IDX, xi)
            T = dS.T @ X  # (2, 3) tangents
            dA = np.linalg.norm(np.cross(T[0], T[1]))
            N = shape_nd(QUAD9_LEX_IDX, xi)
            Me += w * dA * np.outer(N, N)
        vals[f] = Me.ravel()
    return triplets_to_csr(nodes.shape[0], dofs, [vals])[0]


def hex27_face(elements_shape, side: str):
    """Element indices and local node ids of one box side ('z0', 'z1', 'x0', ...)."""
    nx, ny, nz = elements_shape
    axis = "xyz".index(side[0])
    hi = side[1] == "1"
    es = []
    for ez in range(nz):
        for ey in range(ny):
            for ex in range(nx):
                e3 = (ex, ey, ez)
                if e3[axis] == ((nx, ny, nz)[axis] - 1 if hi else 0):
                    es.append((ez * ny + ey) * nx + ex)
    fixed = 2 if hi else 0
    loc = []
    for t in range(3):
        for s in range(3):
            abc = [None, None, None]
            free = [d for d in range(3) if d != axis]
            abc[axis] = fixed
            abc[free[0]] = s
            abc[free[1]] = t
            loc.append(abc[0] + 3 * abc[1] + 9 * abc[2])
    return np.array(es, dtype=np.int64), np.array(loc, dtype=np.int64)


def line_matrices_1d(L: float, ne: int):
    """Assembled 1D quadratic stiffness/mass on [0, L] with ne elements (shape.py:20-26,
    gauss1d): building block of the independent Kronecker cross-check."""
    n = 2 * ne + 1
    h = L / ne
    x, w = gauss1d()
    ke = np.zeros((3, 3))
    me = np.zeros((3, 3))
    for xi, wi in zip(x, w):
        N = lag1d(xi)
        dN = dlag1d(xi) * 2.0 / h
        ke += wi * (h / 2) * np.outer(dN, dN)
        me += wi * (h / 2) * np.outer(N, N)
    K = np.zeros((n, n))
    M = np.zeros((n, n))
    for e in range(ne):
        s = slice(2 * e, 2 * e + 3)
        K[s, s] += ke
        M[s, s] += me
    return K, M


def kron_box(box, nx, ny, nz):
    """Independent hex27 cross-check: Kgrad = Kx⊗My⊗Mz + ..., node order z,y,x."""
    x0, y0, z0, x1, y1, z1 = box
    Kx, Mx = line_matrices_1d(x1 - x0, nx)
    Ky, My = line_matrices_1d(y1 - y0, ny)
    Kz, Mz = line_matrices_1d(z1 - z0, nz)
    k = lambda a, b, c: sp.kron(sp.kron(sp.csr_matrix(a), sp.csr_matrix(b)), sp.csr_matrix(c))
    Kg = k(Mz, My, Kx) + k(Mz, Ky, Mx) + k(Kz, My, Mx)
    Mn = k(Mz, My, Mx)
    return Kg.tocsr(), Mn.tocsr()


def kron_pattern(nx, ny, nz):
    """Structural hex27 box pattern as a Kronecker product of 1D element-block
    patterns (independent of values): canonical CSR of ones."""
    def p1(ne):
        n = 2 * ne + 1
        P = np.zeros((n, n))
        for e in range(ne):
            P[2 * e:2 * e + 3, 2 * e:2 * e + 3] = 1.0
        return sp.csr_matrix(P)
    K = sp.kron(sp.kron(p1(nz), p1(ny), format="csr"), p1(nx), format="csr")
    K.sum_duplicates()
    K.sort_indices()
    return K


def hex27_pattern_counts(nx, ny, nz):
    """n and structural nnz of a structured hex27 box (SURVEY §8 shared numbers)."""
    return (2 * nx + 1) * (2 * ny + 1) * (2 * nz + 1), (8 * nx + 1) * (8 * ny + 1) * (8 * nz + 1)
