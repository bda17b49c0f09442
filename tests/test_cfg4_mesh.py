"""cfg4 synthetic fuselage (BASELINE configs[3]) on the CPU: the oracle's
facet-shell / chain-rule Helmholtz elements against analytic properties
(there is no reference element, SURVEY §8c tier 2), and the host mesh /
DoF-table generator (conformity, orientation, plane-major numbering)."""

import math

import numpy as np
import pytest

from oracle import fe, fuselage as ofu, shell


def _cyl_facet(R=1.5, th0=0.1, dth=0.2, z0=0.0, dz=0.4, project=True):
    th = th0 + dth * np.arange(3) / 2
    X = np.array([[R * math.cos(th[a]), R * math.sin(th[a]), z0 + dz * b / 2] for b in range(3) for a in range(3)])
    if project:  # mid-side node on the chord, as the generator places shell nodes
        X[1::3] = 0.5 * (X[0::3] + X[2::3])
    return X


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_facet_shell_rigid_body_modes_and_symmetry(seed):
    rng = np.random.default_rng(seed)
    X = _cyl_facet(th0=rng.uniform(0, 6), dth=rng.uniform(0.05, 0.3), dz=rng.uniform(0.05, 0.5))
    Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    X = X @ Q.T + rng.standard_normal(3)        # arbitrary rigid placement
    K, M = ofu.facet_shell_element(60e9, 0.3, 1550.0, 3e-3, X)
    R = ofu.rigid_body_modes(X)
    assert np.abs(K @ R).max() <= 1e-10 * np.abs(K).max()
    assert np.abs(K - K.T).max() <= 1e-12 * np.abs(K).max()
    ev = np.linalg.eigvalsh(K)
    # six rigid-body modes + the single-element w mode of the 2x2 shear rule
    # (the 9-node selective-reduced RM element of the cfg2 plate, oracle/shell.py)
    assert ev[7] > 1e-9 * ev[-1]
    assert np.linalg.eigvalsh(M)[0] > 0


def test_facet_shell_in_plane_equals_plate():
    """A facet in the xy plane is oracle/shell.py's plate (membrane + RM) plus
    the drilling term: with drill = 0 the (u, v, w, bx, by) block is the plate
    (bx = theta_y, by = -theta_x)."""
    X = np.array([[0.1 * a + 0.02 * b, 0.15 * b, 0.0] for b in range(3) for a in range(3)])
    K, M = ofu.facet_shell_element(60e9, 0.3, 1550.0, 3e-3, X, drill=0.0)
    Kp, Mp = shell.plate_element(60e9, 0.3, 1550.0, 3e-3, X[:, :2])
    S = np.zeros((54, 45))
    for i in range(9):
        for g, l, sgn in ((0, 0, 1), (1, 1, 1), (2, 2, 1), (4, 3, 1), (3, 4, -1)):
            S[6 * i + g, 5 * i + l] = sgn
    # a sheared (non-rectangular) facet: the plate uses dshape inv(J) (reference
    # quirk), the facet the chain rule; they agree only where J is diagonal
    Xr = np.array([[0.1 * a, 0.15 * b, 0.0] for b in range(3) for a in range(3)])
    Kr, Mr = ofu.facet_shell_element(60e9, 0.3, 1550.0, 3e-3, Xr, drill=0.0)
    Kpr, Mpr = shell.plate_element(60e9, 0.3, 1550.0, 3e-3, Xr[:, :2])
    np.testing.assert_allclose(S.T @ Kr @ S, Kpr, rtol=0, atol=1e-13 * np.abs(Kpr).max())
    np.testing.assert_allclose(S.T @ Mr @ S, Mpr, rtol=0, atol=1e-13 * np.abs(Mpr).max())
    assert np.abs(S.T @ K @ S - Kp).max() > 1e-6 * np.abs(Kp).max()


def test_helmholtz_chain_rule():
    """Chain-rule Laplacian: equal to the reference element on a box (diagonal
    J), constants in its null space and exact on linear fields (patch test) on
    a curved cylindrical element."""
    box = np.array([[0.2 * a, 0.3 * b, 0.25 * c] for c in range(3) for b in range(3) for a in range(3)])
    K0, M0 = fe.helmholtz_element_parts(fe.HEX27_IDX, box)
    K1, M1 = ofu.helmholtz_element_chain(fe.HEX27_IDX, box)
    np.testing.assert_allclose(K1, K0, rtol=0, atol=1e-14 * np.abs(K0).max())
    th = 0.3 + 0.1 * np.arange(3) / 2
    r = 1.2 + 0.1 * np.arange(3) / 2
    X = np.array([[r[a] * math.cos(th[b]), r[a] * math.sin(th[b]), 0.2 * c / 2]
                  for c in range(3) for b in range(3) for a in range(3)])
    K, M = ofu.helmholtz_element_chain(fe.HEX27_IDX, X)
    assert np.abs(K @ np.ones(27)).max() <= 1e-12 * np.abs(K).max()
    # energy of a linear field p = g.x is |g|^2 * volume
    g = np.array([0.3, -1.1, 0.7])
    p = X @ g
    vol = np.ones(27) @ M @ np.ones(27)
    assert abs(p @ K @ p - (g @ g) * vol) <= 1e-9 * (g @ g) * vol


def test_delany_bazley_passive():
    for f in (20.0, 100.0, 250.0):
        rho, c = ofu.delany_bazley(f, 15e3)
        K = rho * c * c
        assert rho.imag < 0 and K.imag >= -1e-12 * abs(K) and c.real > 0  # e^{+iwt}: passive


def test_cfg4_mesh_generator():
    from paper_2310_04734_b200 import fuselage as fz
    spec = fz.FuselageSpec()
    m = fz.fuselage_mesh(spec)
    T = fz.fuselage_tables(m)
    assert m.n == 84_189 and m.P == 2 * spec.n_z + 1
    # positive Jacobians everywhere (cabin Coons blocks + annulus), flat shells
    for el, xy in ((m.cab_el, m.cab_xy), (m.ins_el, m.ins_xy)):
        for e in el:
            for xi in fe.gauss_nd(2)[0]:
                assert np.linalg.det(fe.dshape_nd(fe.QUAD9_LEX_IDX, xi).T @ xy[e]) > 0
    X = T.s_xyz[T.sh_conn]
    n = np.cross(X[:, 2] - X[:, 0], X[:, 6] - X[:, 0])
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    assert np.abs(np.einsum("eic,ec->ei", X - X[:, :1], n)).max() <= 1e-12   # every facet is flat
    # wet faces: structure and fluid nodes coincide up to the chord sagitta
    sag = spec.R * (1 - math.cos(math.pi / spec.n_th)) + 1e-12
    gap = np.linalg.norm(T.s_xyz[T.cp_s] - T.f_xyz[T.cp_f], axis=2)
    assert gap.max() <= sag
    # normals point from the structure into the fluid: skin -> insulation inward,
    # lining -> insulation outward, lining -> cabin inward, floor -> cabin up
    c = T.s_xyz[T.cp_s].mean(axis=1)
    rad = np.linalg.norm(c[:, :2], axis=1)
    er = np.column_stack([c[:, :2] / rad[:, None], np.zeros(len(c))])
    dot = np.einsum("ec,ec->e", T.cp_n, er)
    floor = np.abs(c[:, 1] - m.extra["y_f"]) < 1e-12
    skin = ~floor & (rad > spec.R - 0.01)
    lin = ~floor & ~skin
    assert np.all(dot[skin] < -0.99) and np.all(T.cp_kind[skin] == 0)
    assert np.all(dot[lin & (T.cp_kind == 0)] > 0.99) and np.all(dot[lin & (T.cp_kind == 1)] < -0.99)
    assert np.allclose(T.cp_n[floor], [0.0, 1.0, 0.0]) and np.all(T.cp_kind[floor] == 1)
    # plane-major numbering: every element's DoFs lie in <= 3 consecutive planes
    off = m.plane_off
    plane = lambda d: np.searchsorted(off, d, side="right") - 1
    for dofs in (T.shell_dofs(), T.f_dof[T.cab_conn], T.f_dof[T.ins_conn]):
        p = np.where(dofs >= 0, plane(np.maximum(dofs, 0)), -1)
        lo = np.where(p >= 0, p, 10 ** 9).min(axis=1)
        assert np.all(p.max(axis=1) - lo <= 2)
    # clamped ends: no structure DoFs on the first / last plane; fluid DoFs everywhere
    assert m.plane_nstruct[0] == 0 and m.plane_nstruct[-1] == 0
    assert np.all(np.diff(np.sort(T.f_dof)) == 1) or len(np.unique(T.f_dof)) == len(T.f_dof)
    # stringer bottoms are shared with the frame webs (merged mid-radius nodes)
    assert len(m.fr_xy) == 0


def test_cfg4_full_size_dofs():
    from paper_2310_04734_b200 import fuselage as fz
    m = fz.fuselage_mesh(fz.cfg4_spec_full())
    assert m.n == 2_408_303      # BASELINE cfg4: ~2.4M DoFs


@pytest.mark.parametrize("kw", [dict(n_th=16, n_stringers=8, n_z=6, floor_k=1, n_side=2),
                                dict(n_th=80, n_z=6, n_r_ins=2, floor_k=3, n_side=4),
                                dict(n_th=40, n_z=12, n_r_ins=2, stringer_h=0.04, n_side=5)])
def test_cfg4_mesh_variants(kw):
    """Other valid resolutions: positive Jacobians, flat facets, every DoF
    used by some element, wet faces conforming; a stringer height that does
    not meet the frame's mid radius gives frame-only nodes instead of merges."""
    from paper_2310_04734_b200 import fuselage as fz
    spec = fz.FuselageSpec(**kw)
    m = fz.fuselage_mesh(spec)
    T = fz.fuselage_tables(m)
    for el, xy in ((m.cab_el, m.cab_xy), (m.ins_el, m.ins_xy)):
        J = np.array([[np.linalg.det(fe.dshape_nd(fe.QUAD9_LEX_IDX, xi).T @ xy[e]) for xi in fe.gauss_nd(2)[0]]
                      for e in el])
        assert J.min() > 0
    X = T.s_xyz[T.sh_conn]
    nrm = np.cross(X[:, 2] - X[:, 0], X[:, 6] - X[:, 0])
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    assert np.abs(np.einsum("eic,ec->ei", X - X[:, :1], nrm)).max() <= 1e-12
    used = np.zeros(m.n, dtype=bool)
    sd = T.shell_dofs()
    used[sd[sd >= 0]] = True
    used[T.f_dof[T.cab_conn].ravel()] = True
    used[T.f_dof[T.ins_conn].ravel()] = True
    assert used.all()
    sag = spec.R * (1 - math.cos(math.pi / spec.n_th)) + 1e-12
    assert np.linalg.norm(T.s_xyz[T.cp_s] - T.f_xyz[T.cp_f], axis=2).max() <= sag
    merged = abs(0.5 * (spec.R + spec.R - spec.ins) - (spec.R - spec.stringer_h)) < 1e-12
    n_str_cols = 2 * spec.n_stringers
    assert len(m.fr_xy) == (2 * spec.n_th - n_str_cols if merged else 2 * spec.n_th)


def test_cfg4_tables_are_row_major():
    """Element tables go to the C ABI: row-major int64 (the vectorised builder
    uses fancy indexing, which can return Fortran-ordered arrays)."""
    from paper_2310_04734_b200 import fuselage as fz
    T = fz.fuselage_tables(fz.fuselage_mesh(fz.FuselageSpec(n_th=16, n_stringers=8, n_z=6, floor_k=1, n_side=2)))
    for name in ("sh_conn", "cab_conn", "ins_conn", "cp_s", "cp_f"):
        a = getattr(T, name)
        assert a.flags["C_CONTIGUOUS"] and a.dtype == np.int64, name
        assert a.astype(np.int32).flags["C_CONTIGUOUS"], name
