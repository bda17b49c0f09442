"""Oracle restatement of the cfg2 plate–cavity model (SURVEY §8c tier 2 / §8f
row 4) — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference has no Reissner–Mindlin element, so this
is a restatement that follows the reference's conventions:
  * membrane ("disc") part = the reference's plane-stress 9-node element
    (assembly.py:31-67: D = E/(1-nu^2)[[1,nu,0],[nu,1,0],[0,0,(1-nu)/2]],
    Kmat += w detJ t B^T D B, consistent mass rho t N N^T per component,
    J = dshape^T X, dN = dshape inv(J), 3x3 Gauss);
  * bending/shear = textbook Reissner–Mindlin with the same bases:
    kappa = [d bx/dx, d by/dy, d bx/dy + d by/dx], D_b = E t^3/(12(1-nu^2)) (...),
    gamma = [dw/dx + bx, dw/dy + by], D_s = (5/6) G t I with 2x2 (reduced)
    shear quadrature; rotary inertia rho t^3/12;
  * hysteretic damping (1 + i eta(f)) on the plate stiffness
    (materials.py:170-172), eta(f) a two-sample LossFactorTable (99-109);
  * coupling: C = int N_s N_f n dGamma on the normal DoF, n = structure->fluid
    normal component; -C in K (structure rows, fluid cols), +rho_f C^T in M
    (fluid rows, structure cols) (assembly.py:4-8, 193-207; mortar.py:131-162;
    docs/formulas.md:20-25);
  * plane-wave load p e^{-i k sin(theta) s} along the inward normal of the
    loaded face (assembly.py:108-139 generalised to a 2D plate face).
Node DoFs (u, v, w, bx, by); clamped edges eliminate every DoF of boundary nodes.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

from . import fe

NDOF = 5  # u, v, w, bx, by


def plate_element(E, nu, rho, t, coords):
    """(K, M) 45 x 45 of one 9-node RM + disc plate element (lexicographic local nodes)."""
    idx = fe.QUAD9_LEX_IDX
    Dm = E * t / (1 - nu * nu) * np.array([[1, nu, 0], [nu, 1, 0], [0, 0, 0.5 * (1 - nu)]])
    Db = E * t ** 3 / (12 * (1 - nu * nu)) * np.array([[1, nu, 0], [nu, 1, 0], [0, 0, 0.5 * (1 - nu)]])
    Gs = 5.0 / 6.0 * E / (2 * (1 + nu)) * t
    K = np.zeros((45, 45))
    M = np.zeros((45, 45))
    u, v, w, bx, by = (np.arange(9) * NDOF + k for k in range(5))
    for order, part in ((3, "full"), (2, "shear")):
        pts, wts = fe.gauss_nd(2, order)
        for xi, wq in zip(pts, wts):
            dS = fe.dshape_nd(idx, xi)
            J = dS.T @ coords
            detJ = np.linalg.det(J)
            if detJ <= 0:
                raise ValueError("non-positive Jacobian in plate element")
            dN = dS @ np.linalg.inv(J)
            N = fe.shape_nd(idx, xi)
            if part == "full":
                Bm = np.zeros((3, 45))
                Bm[0, u] = dN[:, 0]
                Bm[1, v] = dN[:, 1]
                Bm[2, u] = dN[:, 1]
                Bm[2, v] = dN[:, 0]
                Bb = np.zeros((3, 45))
                Bb[0, bx] = dN[:, 0]
                Bb[1, by] = dN[:, 1]
                Bb[2, bx] = dN[:, 1]
                Bb[2, by] = dN[:, 0]
                K += wq * detJ * (Bm.T @ Dm @ Bm + Bb.T @ Db @ Bb)
                nn = np.outer(N, N)
                for comp, mass in ((u, rho * t), (v, rho * t), (w, rho * t),
                                   (bx, rho * t ** 3 / 12), (by, rho * t ** 3 / 12)):
                    M[np.ix_(comp, comp)] += wq * detJ * mass * nn
            else:
                Bs = np.zeros((2, 45))
                Bs[0, w] = dN[:, 0]
                Bs[0, bx] = N
                Bs[1, w] = dN[:, 1]
                Bs[1, by] = N
                K += wq * detJ * Gs * (Bs.T @ Bs)
    return K, M


def plate_mesh(rect, nx, ny, z):
    """Structured lexicographic quad9 plate: nodes (npx*npy, 3), elements (n, 9) local a + 3b."""
    x0, y0, x1, y1 = rect
    nodes2, _ = fe.structured_quad9(rect, nx, ny)
    npx = 2 * nx + 1
    elems = np.empty((nx * ny, 9), dtype=np.int64)
    for ey in range(ny):
        for ex in range(nx):
            elems[ey * nx + ex] = [(2 * ey + b) * npx + 2 * ex + a for b in range(3) for a in range(3)]
    nodes = np.column_stack([nodes2, np.full(nodes2.shape[0], z)])
    return nodes, elems


def clamped_dof_map(nx, ny):
    """Global free-DoF number of (node, dof) or -1 for clamped boundary nodes."""
    npx, npy = 2 * nx + 1, 2 * ny + 1
    dmap = -np.ones((npx * npy, NDOF), dtype=np.int64)
    k = 0
    for j in range(npy):
        for i in range(npx):
            if 0 < i < npx - 1 and 0 < j < npy - 1:
                dmap[j * npx + i] = np.arange(k, k + NDOF)
                k += NDOF
    return dmap, k


def eta_table(f, f0=20.0, f1=500.0):
    """cfg2 loss factor eta(f) = 0.01 + 2e-5 f as a two-sample LossFactorTable
    (clamped outside [f0, f1], materials.py:99-109)."""
    e0, e1 = 0.01 + 2e-5 * f0, 0.01 + 2e-5 * f1
    if f <= f0:
        return e0
    if f >= f1:
        return e1
    return e0 + (e1 - e0) * (f - f0) / (f1 - f0)


def rect_triplets(nrow, ncol, rdofs, cdofs, vals):
    """Triplets rows = repeat(rdofs), cols = tile(cdofs) per element in index
    order, -1 DoFs dropped, COO -> CSR + sum_duplicates (assembly.py:160-175)."""
    ne, er = rdofs.shape
    ec = cdofs.shape[1]
    rows = np.repeat(rdofs, ec, axis=1).ravel()
    cols = np.tile(cdofs, (1, er)).ravel()
    v = vals.reshape(ne, er * ec).ravel()
    keep = (rows >= 0) & (cols >= 0)
    A = sp.coo_matrix((v[keep], (rows[keep], cols[keep])), shape=(nrow, ncol)).tocsr()
    A.sum_duplicates()
    return A


def plane_wave_plate(f, c0, theta, nodes, elems, dmap, n_total, amp=1.0):
    """Consistent nodal w-forces of p e^{-i k sin(theta) x} acting along the inward
    normal of the plate's exterior face (-z for a plate on top of a cavity)."""
    k = 2 * math.pi * f / c0 * math.sin(theta)
    fvec = np.zeros(n_total, complex)
    pts, wts = fe.gauss_nd(2)
    x0 = nodes[:, 0].min()
    for e, conn in enumerate(elems):
        X = nodes[conn][:, :2]
        for xi, wq in zip(pts, wts):
            dS = fe.dshape_nd(fe.QUAD9_LEX_IDX, xi)
            detJ = np.linalg.det(dS.T @ X)
            N = fe.shape_nd(fe.QUAD9_LEX_IDX, xi)
            x = N @ X[:, 0]
            p = amp * np.exp(-1j * k * (x - x0))
            for a in range(9):
                d = dmap[conn[a], 2]
                if d >= 0:
                    fvec[d] += -wq * detJ * N[a] * p
    return fvec


def cfg2_primitives(box, ne, E, nu, rho, t, rho_f, c0, theta):
    """scipy restatement of the cfg2 primitives in the global numbering
    [plate free DoFs | cavity pressures]: dict of CSR matrices + load(f)."""
    nx, ny, nz = ne
    x0, y0, z0, x1, y1, z1 = box
    nodes_f, elems_f = fe.structured_hex27(box, *ne)
    pnodes, pelems = plate_mesh((x0, y0, x1, y1), nx, ny, z1)
    dmap, n_p = clamped_dof_map(nx, ny)
    n_f = nodes_f.shape[0]
    n = n_p + n_f
    Kg, Mn = fe.assemble_helmholtz(nodes_f, elems_f, fe.HEX27_IDX)
    ne3 = len(elems_f)
    cg = elems_f + n_p
    # re-assemble the fluid blocks in the global numbering with the same triplet order
    Kv = np.empty((ne3, 729))
    Mv = np.empty((ne3, 729))
    cache = {}
    for e in range(ne3):
        X = nodes_f[elems_f[e]]
        key = np.round(X - X[0], 14).tobytes()
        if key not in cache:
            cache[key] = fe.helmholtz_element_parts(fe.HEX27_IDX, X)
        Kv[e], Mv[e] = cache[key][0].ravel(), cache[key][1].ravel()
    KgG = rect_triplets(n, n, cg, cg, Kv)
    MnG = rect_triplets(n, n, cg, cg, Mv)
    Ke, Me = plate_element(E, nu, rho, t, pnodes[pelems[0]][:, :2])
    npl = len(pelems)
    pd = dmap[pelems].reshape(npl, 45)
    Kp = rect_triplets(n, n, pd, pd, np.tile(Ke.ravel(), (npl, 1)))
    Mp = rect_triplets(n, n, pd, pd, np.tile(Me.ravel(), (npl, 1)))
    fel, floc = fe.hex27_face(ne, "z1")
    fconn = elems_f[fel][:, floc]
    F = face_mass_quads(pnodes, pelems)
    wd = dmap[pelems][:, :, 2]
    Fsf = rect_triplets(n, n, wd, fconn + n_p, F)
    Ffs = rect_triplets(n, n, fconn + n_p, wd, np.transpose(F, (0, 2, 1)).copy())
    load = lambda f: plane_wave_plate(f, c0, theta, pnodes, pelems, dmap, n)
    return dict(n=n, n_p=n_p, n_f=n_f, Kg=KgG, Mn=MnG, Kp=Kp, Mp=Mp, Fsf=Fsf, Ffs=Ffs, load=load,
                dmap=dmap)


def face_mass_quads(nodes, elems):
    """int N N^T dGamma of each 9-node plate face (elements, 9, 9)."""
    pts, wts = fe.gauss_nd(2)
    out = np.empty((len(elems), 9, 9))
    for e, cn in enumerate(elems):
        X = nodes[cn]
        Me = np.zeros((9, 9))
        for xi, w in zip(pts, wts):
            dS = fe.dshape_nd(fe.QUAD9_LEX_IDX, xi)
            T = dS.T @ X
            dA = np.linalg.norm(np.cross(T[0], T[1]))
            N = fe.shape_nd(fe.QUAD9_LEX_IDX, xi)
            Me += w * dA * np.outer(N, N)
        out[e] = Me
    return out


def cfg2_fom(prims, rec, rho_f, c0, eta):
    """oracle.mor.Fom of the coupled operator with the reference conventions:
    K = Kgrad/rho + (1 + i eta(f)) Kp - C, M = Mnn/(rho c^2) + Mp + rho_f C^T,
    C = -F (structure->fluid normal -z)."""
    from .mor import Fom
    P = prims
    sgn = -1.0
    stiff = lambda f: (P["Kg"] / rho_f + (1 + 1j * eta(f)) * P["Kp"] - sgn * P["Fsf"]).astype(complex)
    mass = lambda f: (P["Mn"] / (rho_f * c0 * c0) + P["Mp"] + rho_f * sgn * P["Ffs"]).astype(complex)
    C = np.zeros((len(rec), P["n"]))
    C[np.arange(len(rec)), rec] = 1.0
    return Fom(stiffness=stiff, mass=mass, load=P["load"], c_out=C, n=P["n"])
