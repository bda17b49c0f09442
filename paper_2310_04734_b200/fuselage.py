"""cfg4 synthetic fuselage segment (BASELINE.json configs[3]) on the GPU.

A cylinder barrel (radius R = 1.5 m, length L = 3 m): 3 mm skin, 10 cm
Delany–Bazley equivalent-fluid insulation layer, 2 mm lining, a floor, 6
I-frame webs (0.1 m) and 40 U-stringers (0.05 m), the cabin air above the
floor in 27-node hexahedra; eta(f) = 0.01 + 2e-5 f on every shell, a generic
oblique plane wave on the illuminated skin, 50 seeded cabin receivers.

There is no reference element for any of this (SURVEY §8c tier 2, §8d
"cfg4: stretch"): the physics follows the
reference's conventions and is restated in oracle/fuselage.py:
  * fluids: K = Kgrad / rho_eff, M = Mnn / (rho_eff c_eff^2) per domain
    (assembly.py:242-257), the equivalent fluid with frequency-dependent
    complex (rho_eff, c_eff) like the reference's JCA layer;
  * structure: K = (1 + i eta(f)) Kmat (materials.py:170-172), M;
  * coupling: C = int N_s (n . u) N_f dGamma with n the structure -> fluid
    normal, -C in K, +rho_f C^T in M (assembly.py:193-207, 290-294);
  * plane wave p e^{-i k d.x} along the inward skin normal (assembly.py:108-139
    generalised to a 3D direction d).

Mesh (all structured, z-extruded except the frame webs):
  * cross-section angle nodes theta_j = j pi / n_th (corners even j); the
    cabin is the circular segment above the floor chord, meshed by four
    transfinite (Coons) blocks — centre rectangle, left/right side blocks,
    top block — whose arc sides are the lining nodes; the insulation is the
    annulus [R - 0.1, R] with n_r_ins elements through the thickness;
  * shell nodes at the skin / lining corners lie on the circle and the
    mid-side nodes on the chords, so every facet is exactly flat (the fluid's
    nodes stay on the circle: isoparametric curved hexahedra);
  * stringer s hangs from skin nodes 2 j_s and 2 j_s + 1 (two webs and a flat
    bottom at R - 0.05); frames are annular webs in the planes
    z = (i + 1/2) L / 6, sharing the skin, lining and stringer-bottom nodes;
  * structure DoFs (u_x, u_y, u_z, th_x, th_y, th_z) are clamped at z = 0, L
    (rigid bulkheads); the air has rigid end walls.

DoFs are numbered plane by plane along z (all structure, insulation and cabin
DoFs of node plane k, then plane k + 1 ...): every operator is block
penta-diagonal over planes, which the full-order solver (planes.py) uses.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, assembly, linalg
from .assembly import DeviceCSR, Pattern

AIR_RHO, AIR_C = 1.21, 343.0
NDS = 6  # structure DoFs per node


@dataclass
class FuselageSpec:
    R: float = 1.5
    L: float = 3.0
    ins: float = 0.10            # insulation thickness (skin -> lining)
    n_frames: int = 6
    n_stringers: int = 40
    stringer_h: float = 0.05
    n_th: int = 40               # skin elements around (multiple of 8 and of n_stringers)
    n_z: int = 12                # elements along the axis (multiple of n_frames)
    n_r_ins: int = 1             # insulation elements through the thickness
    floor_k: int = 2             # floor corners at theta = -floor_k * 2pi/n_th and pi + floor_k * 2pi/n_th
    n_side: int = 6              # cabin side-block elements along the floor (= top-block rows)
    a_frac: float = 0.36         # centre-block half width / R_lining
    yt_frac: float = 0.36        # centre-block top / R_lining
    # (E, nu, rho, t) per shell family
    skin: tuple = (60e9, 0.3, 1550.0, 3e-3)
    lining: tuple = (60e9, 0.3, 1550.0, 2e-3)
    floor: tuple = (60e9, 0.3, 1550.0, 10e-3)
    frame: tuple = (60e9, 0.3, 1550.0, 4e-3)
    stringer: tuple = (60e9, 0.3, 1550.0, 2e-3)
    drill: float = 1e-3
    clamped: bool = True         # structure clamped at z = 0, L (False: free, for rigid-body checks)
    sigma_range: tuple = (5e3, 15e3)   # flow resistivity (Pa s / m^2), seeded
    f_band: tuple = (20.0, 250.0)
    d_wave: tuple = (-math.cos(math.radians(30.0)), 0.0, math.sin(math.radians(30.0)))
    n_rec: int = 50
    seed: int = 4

    def check(self):
        if self.n_th % 8 or self.n_th % self.n_stringers or self.n_z % self.n_frames:
            raise ValueError("n_th must be a multiple of 8 and of n_stringers, n_z of n_frames")
        if self.n_side < 1 or self.n_r_ins < 1 or not (0 < self.floor_k < self.n_th // 8):
            raise ValueError("bad fuselage resolution")


def cfg4_spec_full() -> FuselageSpec:
    """The resolution whose DoF count matches BASELINE cfg4 (~2.4M: n =
    2,408,303): 5.9 cm skin facets, 5 cm axial elements, 2 insulation layers.
    Generated and assembled on the GPU; its full-order solve is out of reach
    of the plane-block solver (~20k DoFs per plane), see DESIGN §8."""
    return FuselageSpec(n_th=160, n_z=60, n_r_ins=2, n_side=20, floor_k=8)


# the reduced-resolution cfg4 the pipeline runs end to end (n = 84,189) and its
# Krylov layout: 20 equispaced expansion points x 100 moments (r ~ 2000, BASELINE
# cfg4's order), certified eps_max <= 1e-2 against full-order solves on a
# disjoint grid (tests/test_cfg4_gpu.py)
CFG4_POINTS = tuple(20.0 + 230.0 * (np.arange(20) + 0.5) / 20)
CFG4_MOMENTS = 100


def eta_cfg4(f, band=(20.0, 250.0)) -> float:
    """eta(f) = 0.01 + 2e-5 f as a two-sample LossFactorTable over the band
    (materials.py:99-109)."""
    f0, f1 = band
    f = min(max(f, f0), f1)
    return 0.01 + 2e-5 * f


def delany_bazley(f, sigma, rho0=AIR_RHO, c0=AIR_C):
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


# ---------------------------------------------------------------- mesh -----
def _coons(bot, top, lft, rgt, nu: int, nv: int):
    """Transfinite node grid (2 nv + 1, 2 nu + 1, 2) of a 4-sided block whose
    sides are callables of the side parameter in [0, 1]."""
    us = np.arange(2 * nu + 1) / (2 * nu)
    vs = np.arange(2 * nv + 1) / (2 * nv)
    P00, P10, P01, P11 = bot(0.0), bot(1.0), top(0.0), top(1.0)
    X = np.empty((len(vs), len(us), 2))
    for j, v in enumerate(vs):
        for i, u in enumerate(us):
            X[j, i] = ((1 - v) * bot(u) + v * top(u) + (1 - u) * lft(v) + u * rgt(v)
                       - ((1 - u) * (1 - v) * P00 + u * (1 - v) * P10 + (1 - u) * v * P01 + u * v * P11))
    return X


class _NodeSet:
    """Merge 2D nodes by position (shared block sides)."""

    def __init__(self):
        self.key, self.xy = {}, []

    def add(self, p) -> int:
        k = (round(float(p[0]) * 1e9), round(float(p[1]) * 1e9))
        i = self.key.get(k)
        if i is None:
            i = len(self.xy)
            self.key[k] = i
            self.xy.append((float(p[0]), float(p[1])))
        return i

    def find(self, p) -> int:
        return self.key[(round(float(p[0]) * 1e9), round(float(p[1]) * 1e9))]


def _block_elems(ids: np.ndarray, nu: int, nv: int) -> list:
    out = []
    for ev in range(nv):
        for eu in range(nu):
            out.append([ids[2 * ev + b, 2 * eu + a] for b in range(3) for a in range(3)])
    return out


@dataclass
class FuselageMesh:
    spec: FuselageSpec
    th: np.ndarray                # (2 n_th,) node angles
    cab_xy: np.ndarray            # (N_c2, 2) cabin cross-section nodes
    cab_el: np.ndarray            # (E_c2, 9)
    cab_arc: dict                 # lining angle node j -> cabin 2D node
    cab_floor: np.ndarray         # cabin 2D nodes on the floor, by x
    cab_boundary: np.ndarray      # bool (N_c2,)
    ins_xy: np.ndarray            # (N_i2, 2)
    ins_el: np.ndarray            # (E_i2, 9)
    s2_xy: np.ndarray             # (N_s2, 2) structure nodes present in every plane
    fr_xy: np.ndarray             # (N_fr, 2) frame-only nodes (frame planes)
    skin_ids: np.ndarray          # angle node j -> structure 2D id
    lin_ids: np.ndarray
    floor_ids: np.ndarray         # floor structure nodes by x (ends = lining nodes)
    mid_ids: np.ndarray           # angle node j -> mid-radius node (stringer bottom or frame-only id)
    stringer_nodes: list          # per stringer: (j0, j1, web_mid0, web_mid1, bot0, botm, bot1)
    frame_planes: np.ndarray
    plane_off: np.ndarray         # (P + 1,) DoF offsets of the node planes
    plane_nstruct: np.ndarray     # structure DoFs per plane
    z: np.ndarray                 # (P,) plane coordinates
    extra: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.plane_off[-1])

    @property
    def P(self) -> int:
        return len(self.z)


def fuselage_mesh(spec: FuselageSpec) -> FuselageMesh:
    spec.check()
    R, Rl, nth = spec.R, spec.R - spec.ins, spec.n_th
    nj = 2 * nth
    dth = 2.0 * math.pi / nth
    th = np.arange(nj) * (math.pi / nth)
    er = lambda t: np.array([math.cos(t), math.sin(t)])
    arc = lambda t: Rl * er(t)

    # ---- cabin cross-section: four Coons blocks
    kf = spec.floor_k
    t_fr, t_fl = -kf * dth, math.pi + kf * dth
    y_f, w_f = Rl * math.sin(t_fr), Rl * math.cos(t_fr)
    a, y_t = spec.a_frac * Rl, spec.yt_frac * Rl
    n_c, n_v, n_s = nth // 4, nth // 8 + kf, spec.n_side
    lin = lambda p, q: (lambda s: (1 - s) * np.asarray(p) + s * np.asarray(q))
    P45, P135 = arc(math.pi / 4), arc(3 * math.pi / 4)
    blocks = [
        # centre rectangle
        (lin((-a, y_f), (a, y_f)), lin((-a, y_t), (a, y_t)), lin((-a, y_f), (-a, y_t)), lin((a, y_f), (a, y_t)),
         n_c, n_v),
        # left side block: u from the arc to the rectangle, v up from the floor
        (lin((-w_f, y_f), (-a, y_f)), lin(P135, (-a, y_t)),
         lambda v: arc(t_fl + (3 * math.pi / 4 - t_fl) * v), lin((-a, y_f), (-a, y_t)), n_s, n_v),
        # right side block: u from the rectangle to the arc
        (lin((a, y_f), (w_f, y_f)), lin((a, y_t), P45), lin((a, y_f), (a, y_t)),
         lambda v: arc(t_fr + (math.pi / 4 - t_fr) * v), n_s, n_v),
        # top block: u left -> right, v from the rectangle up to the arc
        (lin((-a, y_t), (a, y_t)), lambda u: arc(3 * math.pi / 4 - (math.pi / 2) * u), lin((-a, y_t), P135),
         lin((a, y_t), P45), n_c, n_s),
    ]
    ns = _NodeSet()
    cab_el = []
    for bot, top, lft, rgt, nu_, nv_ in blocks:
        X = _coons(bot, top, lft, rgt, nu_, nv_)
        ids = np.array([[ns.add(X[j, i]) for i in range(X.shape[1])] for j in range(X.shape[0])])
        cab_el += _block_elems(ids, nu_, nv_)
    cab_xy = np.array(ns.xy)
    cab_el = np.array(cab_el, dtype=np.int64)
    j_fr, j_fl = nj - 2 * kf, nth + 2 * kf
    cab_arc = {}
    for j in list(range(j_fr, nj)) + list(range(0, j_fl + 1)):
        cab_arc[j] = ns.find(arc(th[j]) if j != j_fr else arc(t_fr))
    on_floor = np.abs(cab_xy[:, 1] - y_f) < 1e-9
    cab_floor = np.nonzero(on_floor)[0]
    cab_floor = cab_floor[np.argsort(cab_xy[cab_floor, 0])]
    bnd = on_floor.copy()
    bnd[list(cab_arc.values())] = True

    # ---- insulation annulus: node (i radial, j angle) -> i + nri * j
    nri = 2 * spec.n_r_ins + 1
    rr = Rl + spec.ins * np.arange(nri) / (nri - 1)
    ins_xy = np.array([rr[i] * er(th[j]) for j in range(nj) for i in range(nri)])
    ins_el = []
    for e in range(nth):
        for er_ in range(spec.n_r_ins):
            ins_el.append([(2 * er_ + aa) + nri * ((2 * e + bb) % nj) for bb in range(3) for aa in range(3)])
    ins_el = np.array(ins_el, dtype=np.int64)

    # ---- structure cross-section nodes
    def ring(rad):
        p = np.array([rad * er(t) for t in th])
        p[1::2] = 0.5 * (p[0::2] + np.roll(p[0::2], -1, axis=0))  # mid-side nodes on the chords
        return p
    skin_p, lin_p = ring(R), ring(Rl)
    s2 = []
    skin_ids = np.arange(nj)
    s2 += list(skin_p)
    lin_ids = nj + np.arange(nj)
    s2 += list(lin_p)
    floor_x = cab_xy[cab_floor, 0]
    floor_ids = np.empty(len(cab_floor), dtype=np.int64)
    floor_ids[0], floor_ids[-1] = lin_ids[j_fl], lin_ids[j_fr]
    for q in range(1, len(cab_floor) - 1):
        floor_ids[q] = len(s2)
        s2.append(np.array([floor_x[q], y_f]))
    h = spec.stringer_h
    r_mid_frame = 0.5 * (R + Rl)
    merge = abs(r_mid_frame - (R - h)) < 1e-12
    mid_ids = -np.ones(nj, dtype=np.int64)
    stringer_nodes = []
    step = nth // spec.n_stringers
    for s in range(spec.n_stringers):
        j0 = 2 * s * step
        j1 = j0 + 1
        ids = []
        bots = []
        for jw in (j0, j1):
            e_r = er(th[jw])
            ids.append(len(s2))
            s2.append(skin_p[jw] - 0.5 * h * e_r)
            bots.append(skin_p[jw] - h * e_r)
        b0, b1 = len(s2), len(s2) + 2
        s2 += [bots[0], 0.5 * (bots[0] + bots[1]), bots[1]]
        stringer_nodes.append((j0, j1, ids[0], ids[1], b0, b0 + 1, b1))
        if merge:
            mid_ids[j0], mid_ids[j1] = b0, b1
    s2_xy = np.array(s2)
    fr = []
    n_s2 = len(s2_xy)
    for j in range(nj):
        if mid_ids[j] < 0:
            mid_ids[j] = n_s2 + len(fr)
            fr.append(0.5 * (skin_p[j] + lin_p[j]))
    fr_xy = np.array(fr).reshape(-1, 2)

    # ---- planes and DoF offsets
    P = 2 * spec.n_z + 1
    z = spec.L * np.arange(P) / (P - 1)
    frame_planes = np.array([(2 * i + 1) * spec.n_z // spec.n_frames for i in range(spec.n_frames)])
    is_frame = np.zeros(P, dtype=bool)
    is_frame[frame_planes] = True
    ends = (0, P - 1) if spec.clamped else ()
    nstr = np.array([0 if k in ends else NDS * (n_s2 + (len(fr_xy) if is_frame[k] else 0))
                     for k in range(P)], dtype=np.int64)
    nfl = len(ins_xy) + len(cab_xy)
    plane_off = np.concatenate([[0], np.cumsum(nstr + nfl)]).astype(np.int64)
    return FuselageMesh(spec=spec, th=th, cab_xy=cab_xy, cab_el=cab_el, cab_arc=cab_arc, cab_floor=cab_floor,
                        cab_boundary=bnd, ins_xy=ins_xy, ins_el=ins_el, s2_xy=s2_xy, fr_xy=fr_xy,
                        skin_ids=skin_ids, lin_ids=lin_ids, floor_ids=floor_ids, mid_ids=mid_ids,
                        stringer_nodes=stringer_nodes, frame_planes=frame_planes, plane_off=plane_off,
                        plane_nstruct=nstr, z=z,
                        extra={"y_f": y_f, "w_f": w_f, "j_fl": j_fl, "j_fr": j_fr, "is_frame": is_frame})


# ------------------------------------------------------- element tables ----
@dataclass
class FuselageTables:
    """Node coordinates, element connectivity and element DoF tables (host)."""
    s_xyz: np.ndarray      # (N_s, 3) structure nodes (plane-major: plane k block of that plane's nodes)
    s_dof0: np.ndarray     # (N_s,) first DoF of the node or -1 (clamped)
    f_xyz: np.ndarray      # (N_f, 3) fluid nodes
    f_dof: np.ndarray      # (N_f,)
    sh_conn: np.ndarray    # (E_sh, 9) into s_xyz
    sh_mat: np.ndarray     # (E_sh,) 0 skin, 1 lining, 2 floor, 3 frame, 4 stringer
    cab_conn: np.ndarray   # (E_c, 27) into f_xyz
    ins_conn: np.ndarray   # (E_i, 27)
    cp_s: np.ndarray       # (E_cp, 9) structure face nodes (into s_xyz)
    cp_f: np.ndarray       # (E_cp, 9) fluid face nodes (into f_xyz)
    cp_n: np.ndarray       # (E_cp, 3) unit normal structure -> fluid
    cp_kind: np.ndarray    # (E_cp,) 0 insulation, 1 cabin
    skin_el: np.ndarray    # indices of skin elements in sh_conn

    def shell_dofs(self) -> np.ndarray:
        d0 = self.s_dof0[self.sh_conn]                                 # (E, 9)
        d = d0[:, :, None] + np.arange(NDS)[None, None, :]
        d[d0 < 0] = -1
        return d.reshape(len(d0), 9 * NDS)

    def face_struct_dofs(self) -> np.ndarray:
        d0 = self.s_dof0[self.cp_s]
        d = d0[:, :, None] + np.arange(3)[None, None, :]
        d[d0 < 0] = -1
        return d.reshape(len(d0), 27)


def fuselage_tables(m: FuselageMesh) -> FuselageTables:
    sp_ = m.spec
    P, nth, nj = m.P, sp_.n_th, 2 * sp_.n_th
    n_s2, n_fr = len(m.s2_xy), len(m.fr_xy)
    is_frame = m.extra["is_frame"]
    # structure nodes: plane k holds the n_s2 common nodes (+ n_fr frame-only nodes on frame planes)
    s_base = np.zeros(P + 1, dtype=np.int64)
    for k in range(P):
        s_base[k + 1] = s_base[k] + n_s2 + (n_fr if is_frame[k] else 0)
    s_xyz = np.empty((s_base[-1], 3))
    s_dof0 = np.empty(s_base[-1], dtype=np.int64)
    for k in range(P):
        cnt = s_base[k + 1] - s_base[k]
        xy = m.s2_xy if cnt == n_s2 else np.vstack([m.s2_xy, m.fr_xy])
        s_xyz[s_base[k]:s_base[k + 1], :2] = xy
        s_xyz[s_base[k]:s_base[k + 1], 2] = m.z[k]
        s_dof0[s_base[k]:s_base[k + 1]] = (m.plane_off[k] + NDS * np.arange(cnt)) if m.plane_nstruct[k] else -1

    # structure node (plane-local id, plane k) -> s_base[k] + id; fluid node
    # (insulation 2D id, plane k) -> k nfl + id, cabin 2D id -> k nfl + n_i2 + id
    n_i2, n_c2 = len(m.ins_xy), len(m.cab_xy)
    nfl = n_i2 + n_c2
    f_xy = np.vstack([m.ins_xy, m.cab_xy])
    f_xyz = np.empty((P * nfl, 3))
    f_dof = np.empty(P * nfl, dtype=np.int64)
    for k in range(P):
        f_xyz[k * nfl:(k + 1) * nfl, :2] = f_xy
        f_xyz[k * nfl:(k + 1) * nfl, 2] = m.z[k]
        f_dof[k * nfl:(k + 1) * nfl] = m.plane_off[k] + m.plane_nstruct[k] + np.arange(nfl)

    # element tables, vectorised per z layer in the element order of the
    # original per-element loops: per layer [skin e, lining e] for each e,
    # floor elements, stringers (web 0, web 1, bottom), then the fluids; the
    # frames (one plane each) after all layers.  Coupling faces per layer:
    # [skin-ins e, lining-ins e, (lining-cabin e)] for each e, then floor.
    i_out = 2 * sp_.n_r_ins
    nri = i_out + 1
    e_ = np.arange(nth)
    js = (2 * e_[:, None] + np.arange(3)[None, :]) % nj                  # (nth, 3) angle nodes a
    arc = m.cab_arc
    in_arc = np.array([all(int(j) in arc for j in row) for row in js])
    arc_node = np.full(nj, -1, dtype=np.int64)
    for j, q in arc.items():
        arc_node[j] = q
    nfloor = (len(m.floor_ids) - 1) // 2
    fq = 2 * np.arange(nfloor)[:, None] + np.arange(3)[None, :]          # (nfloor, 3)
    strg = np.array(m.stringer_nodes, dtype=np.int64).reshape(-1, 7)       # j0, j1, w0, w1, b0, bm, b1
    sh_l, mat_l, skin_l, cp_s_l, cp_f_l, cp_k_l, cp_g_l, ins_l, cab_l = ([] for _ in range(9))
    n_sh = 0
    ab = lambda nodes_a, ks: (nodes_a[..., None, :] + s_base[np.asarray(ks)][None, :, None]).reshape(
        nodes_a.shape[0], 9)                                               # [a + 3b] = node(a) in plane ks[b]
    for lay in range(sp_.n_z):
        ks = np.array([2 * lay, 2 * lay + 1, 2 * lay + 2])
        skin = ab(m.skin_ids[js], ks)
        lining = ab(m.lin_ids[js], ks)
        per_e = np.stack([skin, lining], axis=1).reshape(-1, 9)           # skin e, lining e, ...
        sh_l.append(per_e)
        mat_l.append(np.tile([0, 1], nth))
        skin_l.append(n_sh + 2 * e_)
        n_sh += 2 * nth
        fins_out = (i_out + nri * js)[:, None, :] + (ks * nfl)[None, :, None]   # (nth, 3 b, 3 a)
        fins_in = (nri * js)[:, None, :] + (ks * nfl)[None, :, None]
        fcab = (n_i2 + arc_node[js])[:, None, :] + (ks * nfl)[None, :, None]
        for e in range(nth):
            cp_s_l += [skin[e], lining[e]]
            cp_f_l += [fins_out[e].ravel(), fins_in[e].ravel()]
            cp_k_l += [0, 0]
            cp_g_l += [-1.0, 1.0]
            if in_arc[e]:
                cp_s_l.append(lining[e])
                cp_f_l.append(fcab[e].ravel())
                cp_k_l.append(1)
                cp_g_l.append(-1.0)
        fl = ab(m.floor_ids[fq], ks)
        sh_l.append(fl)
        mat_l.append(np.full(nfloor, 2))
        n_sh += nfloor
        for q in range(nfloor):
            cp_s_l.append(fl[q])
            cp_f_l.append(((n_i2 + m.cab_floor[fq[q]])[None, :] + (ks * nfl)[:, None]).ravel())
            cp_k_l.append(1)
            cp_g_l.append(-1.0)   # floor e3 = -y, the cabin is above: n = +y
        if len(strg):
            web0 = ab(np.stack([m.skin_ids[strg[:, 0]], strg[:, 2], strg[:, 4]], 1), ks)
            web1 = ab(np.stack([m.skin_ids[strg[:, 1]], strg[:, 3], strg[:, 6]], 1), ks)
            bot = ab(strg[:, 4:7], ks)
            sh_l.append(np.stack([web0, web1, bot], 1).reshape(-1, 9))
            mat_l.append(np.full(3 * len(strg), 4))
            n_sh += 3 * len(strg)
        q27 = np.arange(27)
        ins_l.append(m.ins_el[:, q27 % 9] + (ks[q27 // 9] * nfl)[None, :])
        cab_l.append(n_i2 + m.cab_el[:, q27 % 9] + (ks[q27 // 9] * nfl)[None, :])
    for k in m.frame_planes:
        jb = js                                                               # b along the angle
        nodes = np.stack([m.lin_ids[jb], m.mid_ids[jb], m.skin_ids[jb]], 2)   # (nth, 3 b, 3 a)
        sh_l.append((nodes + s_base[k]).reshape(nth, 9))
        mat_l.append(np.full(nth, 3))
        n_sh += nth
    c = lambda a: np.ascontiguousarray(a, dtype=np.int64)  # row-major (fancy indexing may give F order)
    sh = c(np.concatenate(sh_l))
    mat = np.concatenate(mat_l)
    skin_el = np.concatenate(skin_l)
    cab = c(np.concatenate(cab_l))
    ins = c(np.concatenate(ins_l))
    cp_s = c(np.array(cp_s_l))
    cp_f = c(np.array(cp_f_l))
    cp_kind, cp_sign = cp_k_l, cp_g_l
    # normals from the flat structure facets: e3 = (x2 - x0) x (x6 - x0) / |.|, n = sign * e3
    X = s_xyz[cp_s]
    e3 = np.cross(X[:, 2] - X[:, 0], X[:, 6] - X[:, 0])
    e3 /= np.linalg.norm(e3, axis=1, keepdims=True)
    cp_n = e3 * np.array(cp_sign)[:, None]
    return FuselageTables(s_xyz=s_xyz, s_dof0=s_dof0, f_xyz=f_xyz, f_dof=f_dof, sh_conn=sh,
                          sh_mat=np.array(mat, dtype=np.int32), cab_conn=np.array(cab, dtype=np.int64),
                          ins_conn=np.array(ins, dtype=np.int64), cp_s=cp_s, cp_f=cp_f,
                          cp_n=cp_n, cp_kind=np.array(cp_kind, dtype=np.int32),
                          skin_el=np.array(skin_el, dtype=np.int64))


# ------------------------------------------------------------ assembly ----
def _quad9_gauss_tables():
    """Quad9 shape values / reference gradients / weights at the 3x3 Gauss
    points (x fastest; local node a + 3b; shape.py:20-26, 56-65)."""
    g1 = np.array([-math.sqrt(0.6), 0.0, math.sqrt(0.6)])
    w1 = np.array([5 / 9, 8 / 9, 5 / 9])
    L = lambda x: np.array([0.5 * x * (x - 1.0), 1.0 - x * x, 0.5 * x * (x + 1.0)])
    dL = lambda x: np.array([x - 0.5, -2.0 * x, x + 0.5])
    N, dN, w = np.empty((9, 9)), np.empty((9, 9, 2)), np.empty(9)
    for gy in range(3):
        for gx in range(3):
            g = 3 * gy + gx
            w[g] = w1[gx] * w1[gy]
            for b in range(3):
                for a in range(3):
                    N[g, a + 3 * b] = L(g1[gx])[a] * L(g1[gy])[b]
                    dN[g, a + 3 * b] = (dL(g1[gx])[a] * L(g1[gy])[b], L(g1[gx])[a] * dL(g1[gy])[b])
    return N, dN, w


def _pattern_blocks(n_rows: int, n_cols: int, rd: np.ndarray, cd: np.ndarray, device) -> Pattern:
    """vb_csr_pattern_from_blocks: canonical CSR pattern + element-order gather
    map of element blocks rows = repeat(rd), cols = tile(cd), -1 dropped
    (assembly.py:160-175)."""
    lib = _lib.load()
    ne, nr = rd.shape
    nc = cd.shape[1]
    rd_d = torch.as_tensor(np.ascontiguousarray(rd, dtype=np.int32), device=device)
    cd_d = torch.as_tensor(np.ascontiguousarray(cd, dtype=np.int32), device=device)
    T = ne * nr * nc
    indptr = torch.empty(n_rows + 1, dtype=torch.int32, device=device)
    indices = torch.empty(T, dtype=torch.int32, device=device)
    gptr = torch.empty(T + 1, dtype=torch.int64, device=device)
    gidx = torch.empty(T, dtype=torch.int32, device=device)
    wb = lib.vb_csr_pattern_blocks_workspace_bytes(n_rows, n_cols, ne, nr, nc)
    work = torch.empty(wb, dtype=torch.uint8, device=device)
    nnz = C.c_int64(0)
    _lib.check(lib.vb_csr_pattern_from_blocks(n_rows, n_cols, ne, nr, nc, _lib.ptr(rd_d), _lib.ptr(cd_d),
                                              _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(gptr), _lib.ptr(gidx),
                                              C.byref(nnz), _lib.ptr(work), wb, _lib.stream_handle()),
               "vb_csr_pattern_from_blocks")
    k = int(nnz.value)
    return Pattern(n_rows, indptr, indices[:k].clone(), gptr[:k + 1].clone(), gidx)


def shell_elements(s_xyz_d: torch.Tensor, conn_d: torch.Tensor, mat_d: torch.Tensor, props_d: torch.Tensor,
                   drill: float):
    """vb_facet_shell_elements: (Ke, Me) (E, 54, 54) in global node DoFs."""
    lib = _lib.load()
    ne = conn_d.shape[0]
    Ke = torch.empty((ne, 54, 54), dtype=torch.float64, device=s_xyz_d.device)
    Me = torch.empty_like(Ke)
    bad = C.c_int32(-1)
    _lib.check(lib.vb_facet_shell_elements(ne, _lib.ptr(s_xyz_d), _lib.ptr(conn_d), _lib.ptr(mat_d),
                                           _lib.ptr(props_d), int(props_d.shape[0]), float(drill), _lib.ptr(Ke),
                                           _lib.ptr(Me),
                                           C.byref(bad), _lib.stream_handle()), "vb_facet_shell_elements")
    if bad.value >= 0:
        raise ValueError(f"non-positive Jacobian or bad material index in shell element {bad.value}")
    return Ke, Me


def helmholtz_chain(xyz_d: torch.Tensor, conn_d: torch.Tensor):
    """vb_hex27_helmholtz_elements_chain: (Kgrad_e, Mnn_e) (E, 27, 27)."""
    lib = _lib.load()
    ne = conn_d.shape[0]
    Ke = torch.empty((ne, 27, 27), dtype=torch.float64, device=xyz_d.device)
    Me = torch.empty_like(Ke)
    bad = C.c_int32(-1)
    _lib.check(lib.vb_hex27_helmholtz_elements_chain(ne, _lib.ptr(xyz_d), _lib.ptr(conn_d), _lib.ptr(Ke),
                                                     _lib.ptr(Me), C.byref(bad), _lib.stream_handle()),
               "vb_hex27_helmholtz_elements_chain")
    if bad.value >= 0:
        raise ValueError(f"non-positive Jacobian in Helmholtz element {bad.value}")
    return Ke, Me


class PlaneWaveLoad3D:
    """p e^{-i k d.x} on the illuminated skin (d.n_out < 0) along the inward
    normal: f = G e(k), G[(node, comp), gauss point] = -w dA N_a n_comp (a
    constant real CSR on the device), e(k) the phases at the Gauss points —
    one SpMM evaluates any batch of frequencies (assembly.py:108-139 in 3D)."""

    def __init__(self, tables: FuselageTables, n: int, d, c0: float = AIR_C, amp: float = 1.0, device=None):
        import scipy.sparse as sp
        dev = torch.device(device or "cuda")
        d = np.asarray(d, float) / np.linalg.norm(d)
        el = tables.sh_conn[tables.skin_el]
        X = tables.s_xyz[el]                                      # (E, 9, 3)
        N, dN, w = _quad9_gauss_tables()                          # (9g, 9), (9g, 9, 2), (9g,)
        e3 = np.cross(X[:, 2] - X[:, 0], X[:, 6] - X[:, 0])
        e3 /= np.linalg.norm(e3, axis=1, keepdims=True)            # outward skin normal
        lit = (e3 @ d) < 0.0
        X, e3, el = X[lit], e3[lit], el[lit]
        t0 = np.einsum("gi,eic->egc", dN[:, :, 0], X)
        t1 = np.einsum("gi,eic->egc", dN[:, :, 1], X)
        dA = np.linalg.norm(np.cross(t0, t1), axis=2) * w[None, :]  # (E, 9g)
        xg = np.einsum("gi,eic->egc", N, X)                       # (E, 9g, 3)
        d0 = tables.s_dof0[el]                                    # (E, 9)
        E = len(el)
        vals = -amp * dA[:, :, None, None] * N[None, :, :, None] * e3[:, None, None, :]  # (E, g, a, c)
        rows = np.broadcast_to(d0[:, None, :, None] + np.arange(3)[None, None, None, :], vals.shape)
        cols = np.broadcast_to(np.arange(E * 9).reshape(E, 9)[:, :, None, None], vals.shape)
        keep = np.broadcast_to((d0 >= 0)[:, None, :, None], vals.shape)
        G = sp.csr_matrix((vals[keep], (rows[keep], cols[keep])), shape=(n, E * 9))
        G.sum_duplicates()
        self.G = DeviceCSR(n, torch.as_tensor(G.indptr.astype(np.int32), device=dev),
                           torch.as_tensor(G.indices.astype(np.int32), device=dev),
                           torch.as_tensor(G.data, device=dev))
        s = (xg.reshape(-1, 3) @ d)
        self.s = torch.as_tensor(s, device=dev)
        self.c0, self.n, self.G_host, self.s_host = c0, n, G, s

    def phases(self, freqs) -> torch.Tensor:
        k = 2.0 * math.pi * torch.as_tensor(np.asarray(freqs, float), device=self.s.device) / self.c0
        return torch.exp(-1j * torch.outer(self.s, k).to(torch.complex128)).contiguous()

    def batch(self, freqs) -> torch.Tensor:
        return linalg.spmm(self.G, self.phases(freqs))

    def at(self, f: float) -> torch.Tensor:
        return self.batch([f])

    def host(self, f: float) -> np.ndarray:
        return self.G_host @ np.exp(-1j * (2.0 * math.pi * f / self.c0) * self.s_host)


def fuselage_model(spec: FuselageSpec | None = None, device=None, solver: bool = True):
    """cfg4 affine full-order model on the GPU.

    Primitives (all real CSR on the device, one global plane-major numbering):
      Ks (1 + i eta(f)), Ms — every shell;  Kc 1/rho0, Mc 1/(rho0 c0^2) — cabin
      air;  Ki 1/rho_eff(f), Mi 1/(rho_eff c_eff^2) — Delany–Bazley insulation;
      Cs -1 (all wet faces, structure rows);  CTi rho_eff(f), CTc rho0
      (fluid rows).  Returns (FullOrderModel, info)."""
    from .mor import AffineOperator, AffineTerm, FullOrderModel
    from .planes import PlaneBlockSolver
    spec = spec or FuselageSpec()
    dev = torch.device(device or "cuda")
    m = fuselage_mesh(spec)
    T = fuselage_tables(m)
    n = m.n
    rng = np.random.default_rng(spec.seed)
    sigma = float(rng.uniform(*spec.sigma_range))
    # shells
    props = torch.as_tensor(np.array([spec.skin, spec.lining, spec.floor, spec.frame, spec.stringer], float),
                            device=dev)
    s_xyz_d = torch.as_tensor(T.s_xyz, device=dev)
    sh_d = torch.as_tensor(T.sh_conn.astype(np.int32), device=dev)
    Kse, Mse = shell_elements(s_xyz_d, sh_d, torch.as_tensor(T.sh_mat, device=dev), props, spec.drill)
    sd = T.shell_dofs()
    Ks, Ms = _pattern_blocks(n, n, sd, sd, dev).gather2(Kse, Mse)
    del Kse, Mse
    # fluids
    f_xyz_d = torch.as_tensor(T.f_xyz, device=dev)
    prims = {}
    for name, conn in (("c", T.cab_conn), ("i", T.ins_conn)):
        Ke, Me = helmholtz_chain(f_xyz_d, torch.as_tensor(conn.astype(np.int32), device=dev))
        dofs = T.f_dof[conn]
        prims["K" + name], prims["M" + name] = _pattern_blocks(n, n, dofs, dofs, dev).gather2(Ke, Me)
        del Ke, Me
    # wet faces: C_e[(a, comp), b] = n_comp int N_a N_b dGamma (fluid face geometry)
    Fe = assembly.face_mass(f_xyz_d, torch.as_tensor(T.cp_f.astype(np.int32), device=dev))   # (E, 9, 9)
    nrm = torch.as_tensor(T.cp_n, device=dev)
    Ce = (Fe[:, :, None, :] * nrm[:, None, :, None]).reshape(-1, 27, 9).contiguous()
    srows = T.face_struct_dofs()
    fcols = T.f_dof[T.cp_f]
    Cs = _pattern_blocks(n, n, srows, fcols, dev).gather(Ce)
    CT = {}
    for kind, name in ((0, "i"), (1, "c")):
        sel = np.nonzero(T.cp_kind == kind)[0]
        CeT = Ce[torch.as_tensor(sel, device=dev)].transpose(1, 2).contiguous()
        CT[name] = _pattern_blocks(n, n, fcols[sel], srows[sel], dev).gather(CeT)
    load = PlaneWaveLoad3D(T, n, spec.d_wave, AIR_C, 1.0, dev)
    # receivers: interior cabin nodes of interior planes
    n_i2 = len(m.ins_xy)
    nfl = n_i2 + len(m.cab_xy)
    inner2 = np.nonzero(~m.cab_boundary)[0]
    ks = np.arange(1, m.P - 1)
    cand = ((m.plane_off[ks] + m.plane_nstruct[ks] + n_i2)[:, None] + inner2[None, :]).ravel()
    rec = np.sort(rng.choice(cand, spec.n_rec, replace=False)).astype(np.int64)
    Cmat = np.zeros((spec.n_rec, n))
    Cmat[np.arange(spec.n_rec), rec] = 1.0
    band = spec.f_band
    rho_eff = lambda f: delany_bazley(f, sigma)[0]
    k_eff = lambda f: (lambda r, c: r * c * c)(*delany_bazley(f, sigma))
    aff = AffineOperator(
        K=[AffineTerm(Ks, lambda f: 1.0 + 1j * eta_cfg4(f, band)),
           AffineTerm(prims["Kc"], 1.0 / AIR_RHO),
           AffineTerm(prims["Ki"], lambda f: 1.0 / rho_eff(f)),
           AffineTerm(Cs, -1.0)],
        M=[AffineTerm(Ms, 1.0),
           AffineTerm(prims["Mc"], 1.0 / (AIR_RHO * AIR_C * AIR_C)),
           AffineTerm(prims["Mi"], lambda f: 1.0 / k_eff(f)),
           AffineTerm(CT["i"], rho_eff),
           AffineTerm(CT["c"], AIR_RHO)],
        D=[], load=load)
    planes = PlaneBlockSolver(aff, m.plane_off, dev) if solver else None
    fom = FullOrderModel(c_out=Cmat, n=n, affine=aff, planes=planes)
    info = {"mesh": m, "tables": T, "sigma": sigma, "rec": rec, "load": load, "Ks": Ks, "Ms": Ms,
            "Kc": prims["Kc"], "Mc": prims["Mc"], "Ki": prims["Ki"], "Mi": prims["Mi"], "Cs": Cs,
            "CTi": CT["i"], "CTc": CT["c"], "freqs": np.arange(band[0], band[1] + 1e-9, 0.5)}
    return fom, info
