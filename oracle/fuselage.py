"""Oracle restatement of the cfg4 synthetic-fuselage element primitives
(BASELINE configs[3]; SURVEY §8c tier 2 / §8d "cfg4: stretch") — TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference has no shell or curved-solid element, so this is a
restatement in the reference's conventions, pinned by analytic properties in
the tests (rigid-body null spaces, symmetry, patch/rotation invariance) and
used as the checker of the GPU element kernels and of the assembled CSR:

  * fluids (cabin air, equivalent-fluid insulation): the Helmholtz integrals of
    assembly.py:77-91 on 27-node hexahedra, but with the chain rule
    dN/dx = dshape inv(J)^T (the reference's dshape inv(J) — see DESIGN §3
    "Known reference quirk" — equals it only for diagonal J; the fuselage's
    cylindrical mapping has non-diagonal J everywhere);
  * shells (skin, lining, floor, frames, stringers): flat 9-node facets,
    membrane + Reissner–Mindlin bending/shear exactly as oracle/shell.py's
    plate (the reference's plane-stress element assembly.py:31-67 for the
    membrane), with the chain rule above, a Hughes–Brezzi drilling term
    gamma int (theta_3 - (v,x - u,y)/2)^2 dA (gamma = drill * G t) and the
    node rotation from the facet frame to global (u, v, w, theta_x, theta_y,
    theta_z);
  * equivalent fluid: Delany–Bazley-type (Miki) characteristic impedance and wavenumber
    mapped to (rho_eff, c_eff) and used like the reference's JCA fluid
    (assembly.py:242-257: K = Kgrad / rho_eff, M = Mnn / (rho_eff c_eff^2);
    coupling M term rho_eff C^T, assembly.py:199-207, 290-294), in the
    reference's e^{+i w t} convention (materials.py:112-167).
"""

from __future__ import annotations

import math

import numpy as np

from . import fe

NDOF = 6  # u_x, u_y, u_z, theta_x, theta_y, theta_z (global)


def helmholtz_element_chain(idx: np.ndarray, coords: np.ndarray):
    """assembly.py:77-91 with the chain rule dN = dshape inv(J)^T."""
    pts, wts = fe.gauss_nd(coords.shape[1])
    nn = idx.shape[0]
    Kg = np.zeros((nn, nn))
    Mn = np.zeros((nn, nn))
    for xi, w in zip(pts, wts):
        dS = fe.dshape_nd(idx, xi)
        J = dS.T @ coords
        det = np.linalg.det(J)
        if det <= 0:
            raise ValueError("non-positive Jacobian in Helmholtz element")
        dN = dS @ np.linalg.inv(J).T
        N = fe.shape_nd(idx, xi)
        Kg += w * det * (dN @ dN.T)
        Mn += w * det * np.outer(N, N)
    return Kg, Mn


def facet_frame(X3: np.ndarray):
    """Rows e1, e2, e3 of the facet frame: e1 along the local xi edge (node 0 ->
    node 2), e3 the normal of the corner plane, e2 = e3 x e1."""
    e1 = X3[2] - X3[0]
    e1 = e1 / np.linalg.norm(e1)
    n = np.cross(X3[2] - X3[0], X3[6] - X3[0])
    e3 = n / np.linalg.norm(n)
    e2 = np.cross(e3, e1)
    return np.array([e1, e2, e3])


def facet_local_matrices(E, nu, rho, t, X2, drill=1e-3):
    """54 x 54 local (u, v, w, bx, by, t3) per node: the plate of oracle/shell.py
    (bx, by with u = z bx, v = z by; 3x3 rule, 2x2 shear rule) with the chain
    rule, plus the drilling term and rotary inertia rho t^3/12 on t3."""
    idx = fe.QUAD9_LEX_IDX
    nd = 6
    Dm = E * t / (1 - nu * nu) * np.array([[1, nu, 0], [nu, 1, 0], [0, 0, 0.5 * (1 - nu)]])
    Db = E * t ** 3 / (12 * (1 - nu * nu)) * np.array([[1, nu, 0], [nu, 1, 0], [0, 0, 0.5 * (1 - nu)]])
    G = E / (2 * (1 + nu))
    Gs = 5.0 / 6.0 * G * t
    gam = drill * G * t
    K = np.zeros((54, 54))
    M = np.zeros((54, 54))
    u, v, w, bx, by, t3 = (np.arange(9) * nd + k for k in range(6))
    for order, part in ((3, "full"), (2, "shear")):
        pts, wts = fe.gauss_nd(2, order)
        for xi, wq in zip(pts, wts):
            dS = fe.dshape_nd(idx, xi)
            J = dS.T @ X2
            det = np.linalg.det(J)
            if det <= 0:
                raise ValueError("non-positive Jacobian in shell element")
            dN = dS @ np.linalg.inv(J).T
            N = fe.shape_nd(idx, xi)
            if part == "full":
                Bm = np.zeros((3, 54))
                Bm[0, u] = dN[:, 0]
                Bm[1, v] = dN[:, 1]
                Bm[2, u] = dN[:, 1]
                Bm[2, v] = dN[:, 0]
                Bb = np.zeros((3, 54))
                Bb[0, bx] = dN[:, 0]
                Bb[1, by] = dN[:, 1]
                Bb[2, bx] = dN[:, 1]
                Bb[2, by] = dN[:, 0]
                Bd = np.zeros(54)
                Bd[t3] = N
                Bd[v] = -0.5 * dN[:, 0]
                Bd[u] = 0.5 * dN[:, 1]
                K += wq * det * (Bm.T @ Dm @ Bm + Bb.T @ Db @ Bb + gam * np.outer(Bd, Bd))
                nn = np.outer(N, N)
                for comp, mass in ((u, rho * t), (v, rho * t), (w, rho * t), (bx, rho * t ** 3 / 12),
                                   (by, rho * t ** 3 / 12), (t3, rho * t ** 3 / 12)):
                    M[np.ix_(comp, comp)] += wq * det * mass * nn
            else:
                Bs = np.zeros((2, 54))
                Bs[0, w] = dN[:, 0]
                Bs[0, bx] = N
                Bs[1, w] = dN[:, 1]
                Bs[1, by] = N
                K += wq * det * Gs * (Bs.T @ Bs)
    return K, M


def node_rotation(R: np.ndarray) -> np.ndarray:
    """6 x 6 map global (u_x,u_y,u_z,th_x,th_y,th_z) -> local (u1,u2,u3,bx,by,t3):
    u_loc = R u, th_loc = R th, bx = th_2, by = -th_1, t3 = th_3."""
    T = np.zeros((6, 6))
    T[:3, :3] = R
    T[3, 3:] = R[1]
    T[4, 3:] = -R[0]
    T[5, 3:] = R[2]
    return T


def facet_shell_element(E, nu, rho, t, X3, drill=1e-3):
    """(K, M) 54 x 54 in the global node DoFs of one flat 9-node facet whose
    nodes X3 (9, 3) may lie slightly off the corner plane (projected)."""
    R = facet_frame(X3)
    X2 = (X3 - X3[0]) @ R[:2].T
    Kl, Ml = facet_local_matrices(E, nu, rho, t, X2, drill)
    T = np.kron(np.eye(9), node_rotation(R))
    return T.T @ Kl @ T, T.T @ Ml @ T


def delany_bazley(f, sigma, rho0=1.21, c0=343.0):
    """(rho_eff, c_eff) of a Delany–Bazley-type equivalent fluid in Miki's
    passive form (the original Delany–Bazley fit gives Im K_eff < 0, i.e. an
    active bulk modulus, for f / sigma below its 0.01 validity bound — most of
    20-250 Hz at sigma ~ 1e4): X = f / sigma,
    Zc = rho0 c0 (1 + 0.070 X^-0.632 - 0.107i X^-0.632),
    kc = w / c0 (1 + 0.109 X^-0.618 - 0.160i X^-0.618);
    rho_eff = Zc kc / w, c_eff = w / kc (e^{+i w t}: Im rho_eff < 0,
    Im rho_eff c_eff^2 >= 0)."""
    w = 2.0 * math.pi * f
    X = f / sigma
    Zc = rho0 * c0 * (1 + 0.070 * X ** -0.632 - 0.107j * X ** -0.632)
    kc = w / c0 * (1 + 0.109 * X ** -0.618 - 0.160j * X ** -0.618)
    return Zc * kc / w, w / kc


def rigid_body_modes(xyz: np.ndarray) -> np.ndarray:
    """(6 n, 6) global rigid-body displacement fields of shell nodes xyz."""
    n = xyz.shape[0]
    Rm = np.zeros((n * 6, 6))
    for i in range(3):
        Rm[i::6, i] = 1.0
    for a in range(3):  # rotation about axis a: u = e_a x x, theta = e_a
        ea = np.eye(3)[a]
        Rm[np.arange(n)[:, None] * 6 + np.arange(3), 3 + a] = np.cross(ea, xyz)
        Rm[np.arange(n) * 6 + 3 + a, 3 + a] = 1.0
    return Rm


def assemble_cfg4(tables, props, drill=1e-3):
    """scipy restatement of the cfg4 primitives from the mesh tables of
    paper_2310_04734_b200.fuselage (node coordinates, element connectivity,
    element DoF maps): per-element oracle matrices, triplets rows =
    repeat(dofs), cols = tile(dofs) in element order, COO -> CSR +
    sum_duplicates (assembly.py:142-175).  Returns a dict of CSR matrices
    Ks, Ms, Kc, Mc, Ki, Mi, Cs, CTi, CTc (the device model's primitives)."""
    from .shell import face_mass_quads, rect_triplets
    T = tables
    n = int(max(T.s_dof0.max() + 6, T.f_dof.max() + 1))
    out = {}
    sd = T.shell_dofs()
    Ke = np.empty((len(T.sh_conn), 54 * 54))
    Me = np.empty_like(Ke)
    for e, cn in enumerate(T.sh_conn):
        K, M = facet_shell_element(*props[T.sh_mat[e]], T.s_xyz[cn], drill)
        Ke[e], Me[e] = K.ravel(), M.ravel()
    out["Ks"] = rect_triplets(n, n, sd, sd, Ke)
    out["Ms"] = rect_triplets(n, n, sd, sd, Me)
    for name, conn in (("c", T.cab_conn), ("i", T.ins_conn)):
        Kh = np.empty((len(conn), 729))
        Mh = np.empty_like(Kh)
        for e, cn in enumerate(conn):
            K, M = helmholtz_element_chain(fe.HEX27_IDX, T.f_xyz[cn])
            Kh[e], Mh[e] = K.ravel(), M.ravel()
        d = T.f_dof[conn]
        out["K" + name] = rect_triplets(n, n, d, d, Kh)
        out["M" + name] = rect_triplets(n, n, d, d, Mh)
    F = face_mass_quads(T.f_xyz, T.cp_f)                                   # (E, 9, 9)
    Ce = (F[:, :, None, :] * T.cp_n[:, None, :, None]).reshape(len(F), 27, 9)
    sr = T.face_struct_dofs()
    fc = T.f_dof[T.cp_f]
    out["Cs"] = rect_triplets(n, n, sr, fc, Ce.reshape(len(F), -1))
    for kind, name in ((0, "i"), (1, "c")):
        sel = T.cp_kind == kind
        out["CT" + name] = rect_triplets(n, n, fc[sel], sr[sel],
                                         np.transpose(Ce[sel], (0, 2, 1)).reshape(int(sel.sum()), -1))
    return out


def plane_wave_cfg4(tables, n, d, f, c0=343.0, amp=1.0):
    """Consistent nodal forces of p e^{-i k d.x} on the illuminated flat skin
    facets (d.n_out < 0) along the inward normal (assembly.py:108-139 in 3D)."""
    T = tables
    d = np.asarray(d, float) / np.linalg.norm(d)
    k = 2 * math.pi * f / c0
    fvec = np.zeros(n, complex)
    pts, wts = fe.gauss_nd(2)
    for e in T.skin_el:
        cn = T.sh_conn[e]
        X = T.s_xyz[cn]
        e3 = np.cross(X[2] - X[0], X[6] - X[0])
        e3 /= np.linalg.norm(e3)
        if e3 @ d >= 0:
            continue
        for xi, w in zip(pts, wts):
            dS = fe.dshape_nd(fe.QUAD9_LEX_IDX, xi)
            t = dS.T @ X
            dA = np.linalg.norm(np.cross(t[0], t[1]))
            N = fe.shape_nd(fe.QUAD9_LEX_IDX, xi)
            p = amp * np.exp(-1j * k * (d @ (N @ X)))
            for a in range(9):
                d0 = T.s_dof0[cn[a]]
                if d0 >= 0:
                    fvec[d0:d0 + 3] += -w * dA * N[a] * p * e3
    return fvec
