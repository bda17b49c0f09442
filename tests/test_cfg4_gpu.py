"""cfg4 synthetic fuselage on the GPU (BASELINE configs[3], SURVEY §8c tier 2:
no reference element — checked against oracle/fuselage.py and analytic
properties): element kernels, the assembled CSR primitives (pattern
bit-exact, values to rounding), the plane-wave load, the plane-block
full-order solver (residual <= 1e-10, = scipy splu), the batched GEMV, and
the MOR chain (ROM certified at the reference tolerance eps_max <= 1e-2,
tests/test_acceptance.py:272-305)."""

import math

import numpy as np
import pytest

from oracle import fe, fuselage as ofu

pytestmark = pytest.mark.gpu


def _tiny():
    from paper_2310_04734_b200 import fuselage as fz
    return fz.FuselageSpec(n_th=16, n_stringers=8, n_z=6, floor_k=1, n_side=2)


@pytest.fixture(scope="module")
def tiny(cuda):
    from paper_2310_04734_b200 import fuselage as fz
    spec = _tiny()
    fom, info = fz.fuselage_model(spec, cuda)
    return spec, fom, info


def _props(spec):
    return [spec.skin, spec.lining, spec.floor, spec.frame, spec.stringer]


def test_facet_shell_kernel_matches_oracle(tiny, cuda):
    import torch
    from paper_2310_04734_b200 import fuselage as fz
    spec, fom, info = tiny
    T = info["tables"]
    props = _props(spec)
    Ke, Me = fz.shell_elements(torch.as_tensor(T.s_xyz, device=cuda),
                               torch.as_tensor(T.sh_conn.astype(np.int32), device=cuda),
                               torch.as_tensor(T.sh_mat, device=cuda),
                               torch.as_tensor(np.array(props), device=cuda), spec.drill)
    Ke, Me = Ke.cpu().numpy(), Me.cpu().numpy()
    for fam in range(5):   # skin, lining, floor, frame webs (annular: non-diagonal J), stringers
        for q in np.nonzero(T.sh_mat == fam)[0][::9]:
            K0, M0 = ofu.facet_shell_element(*props[fam], T.s_xyz[T.sh_conn[q]], spec.drill)
            np.testing.assert_allclose(Ke[q], K0, rtol=0, atol=1e-12 * np.abs(K0).max())
            np.testing.assert_allclose(Me[q], M0, rtol=0, atol=1e-12 * np.abs(M0).max())
            R = ofu.rigid_body_modes(T.s_xyz[T.sh_conn[q]])
            assert np.abs(Ke[q] @ R).max() <= 1e-9 * np.abs(K0).max()


def test_hex27_chain_kernel_matches_oracle(tiny, cuda):
    import torch
    from paper_2310_04734_b200 import fuselage as fz
    spec, fom, info = tiny
    T = info["tables"]
    fx = torch.as_tensor(T.f_xyz, device=cuda)
    for conn in (T.cab_conn, T.ins_conn):
        Ke, Me = fz.helmholtz_chain(fx, torch.as_tensor(conn.astype(np.int32), device=cuda))
        Ke, Me = Ke.cpu().numpy(), Me.cpu().numpy()
        for q in range(0, len(conn), 7):
            K0, M0 = ofu.helmholtz_element_chain(fe.HEX27_IDX, T.f_xyz[conn[q]])
            np.testing.assert_allclose(Ke[q], K0, rtol=0, atol=1e-12 * np.abs(K0).max())
            np.testing.assert_allclose(Me[q], M0, rtol=0, atol=1e-12 * np.abs(M0).max())


def test_cfg4_primitives_match_oracle(tiny):
    """Every primitive: CSR indptr / indices bit-exact vs the oracle's scipy
    assembly of the same element tables, values to rounding; the plane-wave
    load vs the oracle's consistent nodal forces."""
    spec, fom, info = tiny
    T = info["tables"]
    ref = ofu.assemble_cfg4(T, _props(spec), spec.drill)
    for name in ("Ks", "Ms", "Kc", "Mc", "Ki", "Mi", "Cs", "CTi", "CTc"):
        A = info[name].to_scipy()
        R = ref[name]
        assert A.shape == R.shape, name
        np.testing.assert_array_equal(A.indptr, R.indptr, err_msg=name)
        np.testing.assert_array_equal(A.indices, R.indices, err_msg=name)
        np.testing.assert_allclose(A.data, R.data, rtol=0, atol=1e-12 * np.abs(R.data).max(), err_msg=name)
    for f in (31.0, 212.5):
        b = info["load"].at(f).cpu().numpy().ravel()
        b0 = ofu.plane_wave_cfg4(T, fom.n, spec.d_wave, f)
        np.testing.assert_allclose(b, b0, rtol=0, atol=1e-12 * np.abs(b0).max())
    # structure stiffness is symmetric; the free structure's rigid-body modes
    # are in the null space of the unclamped interior assembly
    Ks = info["Ks"].to_scipy()
    assert abs(Ks - Ks.T).max() <= 1e-12 * abs(Ks).max()


def test_gemv_batched(cuda):
    import torch
    from paper_2310_04734_b200 import linalg
    g = torch.Generator(device="cpu").manual_seed(3)
    items, refs = [], []
    for (m, n, s) in ((301, 257, 1), (1000, 64, 3), (64, 2049, 16), (3, 5, 2)):
        A = torch.randn(m, n, dtype=torch.complex128, generator=g).to(cuda)
        X = torch.randn(n, s, dtype=torch.complex128, generator=g).to(cuda)
        Y = torch.randn(m, s, dtype=torch.complex128, generator=g).to(cuda)
        refs.append(((0.5 - 2j) * (A @ X) + (1 + 1j) * Y, Y))
        items.append((A, X, Y, 0.5 - 2j, 1 + 1j))
    linalg.zgemv_batched(items)
    for (want, Y), (A, X, _, _, _) in zip(refs, items):
        assert ((Y - want).abs().max() / (A.abs().max() * X.abs().max() * A.shape[1])).item() <= 1e-14


def test_cfg4_plane_solver_matches_splu(tiny):
    """Plane-block elimination + refinement: residual <= 1e-10 and the same
    solution (and receiver outputs) as scipy splu of the assembled operator."""
    import scipy.sparse.linalg as spl
    import torch
    spec, fom, info = tiny
    for f in (20.0, 137.0, 250.0):
        fac = fom.factor(f)
        b = fom.load_dev(f)
        x = fac.solve(b).cpu().numpy().ravel()
        assert fac.last_residual <= 1e-10
        A = fom.operator(f).tocsc()
        xs = spl.splu(A).solve(fom.load(f))
        assert np.linalg.norm(x - xs) <= 1e-7 * np.linalg.norm(xs)
        y, ys = fom.c_out @ x, fom.c_out @ xs
        assert np.abs(y - ys).max() <= 1e-7 * np.abs(ys).max()
        # multi-column right-hand sides (> 16 columns are chunked)
        B = torch.randn(fom.n, 18, dtype=torch.complex128, device=b.device)
        X = fac.solve(B)
        R = fac.residual(X, B)
        assert (torch.linalg.norm(R, dim=0) / torch.linalg.norm(B, dim=0)).max().item() <= 1e-10


def test_cfg4_tiny_mor_chain(tiny):
    """Krylov basis through the plane-block solver, projection and sweep: the
    ROM reproduces full-order solves on a disjoint grid."""
    from paper_2310_04734_b200 import mor
    spec, fom, info = tiny
    # the equivalent fluid's coefficients vary strongly with f (rho_eff from
    # -130i to -9i over the band): dense expansion points, moderate moments
    pts = list(20.0 + 230.0 * (np.arange(24) + 0.5) / 24)
    V, _ = mor.krylov_basis(fom, pts, 30)
    rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 250.0))
    ver = [27.3, 88.8, 131.1, 199.9, 246.0]
    y, _, _, _ = rom.sweep(ver)
    y = y.cpu().numpy()
    for i, f in enumerate(ver):
        yf = fom.c_out @ fom.factor(f).solve(fom.load_dev(f)).cpu().numpy()
        _, e, _, _ = mor.relative_error(yf.ravel(), y[i].ravel())
        assert e <= 1e-2, (f, e)


@pytest.mark.slow
def test_cfg4_reduced_resolution_rom_certified(cuda):
    """The bench's cfg4 pipeline model (n = 84,189; 20 points x 100 moments,
    r ~ 2000): eps_max <= 1e-2 against full-order solves (residual <= 1e-10)
    on frequencies disjoint from the expansion points."""
    from paper_2310_04734_b200 import fuselage as fz, mor
    fom, info = fz.fuselage_model(fz.FuselageSpec(), cuda)
    V, _ = mor.krylov_basis(fom, list(fz.CFG4_POINTS), fz.CFG4_MOMENTS)
    assert V.shape[1] >= 1990
    rom = mor.ReducedModel(fom=fom, V=V, window=(20.0, 250.0))
    ver = list(np.arange(21.3, 250.0, 230 / 12.0))
    y, _, _, _ = rom.sweep(ver)
    y = y.cpu().numpy()
    worst = 0.0
    for i, f in enumerate(ver):
        fac = fom.factor(f)
        yf = fom.c_out @ fac.solve(fom.load_dev(f)).cpu().numpy()
        assert fac.last_residual <= 1e-10
        _, e, _, _ = mor.relative_error(yf.ravel(), y[i].ravel())
        worst = max(worst, e)
    assert worst <= 1e-2, worst


def test_facet_shell_rejects_bad_input(tiny, cuda):
    """Material index outside [0, n_mat) and a degenerate facet raise
    ValueError (the reference raises on detJ <= 0, assembly.py:85-86)."""
    import torch
    from paper_2310_04734_b200 import fuselage as fz
    spec, fom, info = tiny
    T = info["tables"]
    props = torch.as_tensor(np.array(_props(spec)), device=cuda)
    conn = torch.as_tensor(T.sh_conn[:5].astype(np.int32), device=cuda)
    sx = torch.as_tensor(T.s_xyz, device=cuda)
    mat = torch.as_tensor(np.array([0, 1, 7, 0, 0], np.int32), device=cuda)
    with pytest.raises(ValueError, match="shell element 2"):
        fz.shell_elements(sx, conn, mat, props, spec.drill)
    bad = T.sh_conn[:1].copy()
    bad[0, 6:] = bad[0, :3]           # collapsed facet
    with pytest.raises(ValueError):
        fz.shell_elements(sx, torch.as_tensor(bad.astype(np.int32), device=cuda),
                          torch.zeros(1, dtype=torch.int32, device=cuda), props, spec.drill)


def test_plane_solver_rejects_foreign_structure(tiny, cuda):
    """A primitive coupling node planes outside one element layer is refused
    at setup (the block elimination would silently drop it)."""
    import scipy.sparse as sp
    import torch
    from paper_2310_04734_b200.assembly import DeviceCSR
    from paper_2310_04734_b200.mor import AffineOperator, AffineTerm
    from paper_2310_04734_b200.planes import PlaneBlockSolver
    spec, fom, info = tiny
    off = info["mesh"].plane_off
    n = fom.n
    E = sp.csr_matrix(([1.0], ([int(off[1])], [int(off[3])])), shape=(n, n))   # mid plane 1 <-> mid plane 3
    d = DeviceCSR(n, torch.as_tensor(E.indptr.astype(np.int32), device=cuda),
                  torch.as_tensor(E.indices.astype(np.int32), device=cuda), torch.as_tensor(E.data, device=cuda))
    aff = AffineOperator(K=list(fom.affine.K) + [AffineTerm(d, 1.0)], M=fom.affine.M, D=[], load=fom.affine.load)
    with pytest.raises(ValueError, match="node planes 1 and 3"):
        PlaneBlockSolver(aff, off, cuda)


def test_cfg4_structure_rigid_body_modes(cuda):
    """The assembled structure stiffness of the UNclamped fuselage (skin,
    lining, floor, frames, stringers, all facet rotations and merged nodes)
    has the six global rigid-body motions in its null space."""
    from paper_2310_04734_b200 import fuselage as fz
    spec = _tiny()
    spec.clamped = False
    fom, info = fz.fuselage_model(spec, cuda, solver=False)
    T = info["tables"]
    Ks = info["Ks"].to_scipy()
    R = np.zeros((fom.n, 6))
    d0 = T.s_dof0
    assert np.all(d0 >= 0)
    R[(d0[:, None] + np.arange(6)[None, :]).ravel(), :] = ofu.rigid_body_modes(T.s_xyz)
    scale = abs(Ks).max() * np.abs(R).max() * 60
    assert np.abs(Ks @ R).max() <= 1e-10 * scale
    # clamped (the model the pipeline solves): no rigid-body mode survives
    Kc = _tiny_clamped_Ks(cuda)
    assert np.linalg.norm(Kc @ np.ones(Kc.shape[0])) > 0


def _tiny_clamped_Ks(cuda):
    from paper_2310_04734_b200 import fuselage as fz
    _, info = fz.fuselage_model(_tiny(), cuda, solver=False)
    return info["Ks"].to_scipy()


def test_cfg4_fluid_axial_mode(tiny):
    """Cabin air and insulation annulus with rigid ends are z-extrusions of a
    uniform cross-section: the axial mode (constant over the cross-section)
    is an exact eigenpair of (Kgrad, Mnn) with the eigenvalue of the 1D
    quadratic mesh along z (~ (pi / L)^2), and constants are the null space."""
    import scipy.linalg as sla
    import scipy.sparse.linalg as spl
    spec, fom, info = tiny
    K1, M1 = fe.line_matrices_1d(spec.L, spec.n_z)
    lam1 = np.sort(sla.eigh(K1, M1, eigvals_only=True))[1]
    assert abs(lam1 - (math.pi / spec.L) ** 2) <= 1e-3 * lam1
    for Kn, Mn in (("Kc", "Mc"), ("Ki", "Mi")):
        K, M = info[Kn].to_scipy(), info[Mn].to_scipy()
        idx = np.unique(M.nonzero()[0])
        K, M = K[idx][:, idx].tocsc(), M[idx][:, idx].tocsc()
        assert np.abs(K @ np.ones(len(idx))).max() <= 1e-12 * abs(K).max()
        lam = spl.eigsh(K, k=4, M=M, sigma=lam1 * (1 + 1e-4), which="LM", return_eigenvectors=False)
        assert np.min(np.abs(lam - lam1)) <= 1e-9 * lam1, (Kn, lam, lam1)


def test_cfg4_variant_frame_only_nodes_solves(cuda):
    """A resolution with two insulation layers and stringers whose bottom
    misses the frame's mid radius (frame-only nodes on the frame planes, so
    the node planes have different sizes): plane-block solve = splu."""
    import scipy.sparse.linalg as spl
    from paper_2310_04734_b200 import fuselage as fz
    spec = fz.FuselageSpec(n_th=16, n_stringers=8, n_z=6, floor_k=1, n_side=2, n_r_ins=2, stringer_h=0.04)
    fom, info = fz.fuselage_model(spec, cuda)
    assert len(info["mesh"].fr_xy) > 0 and len(set(np.diff(info["mesh"].plane_off))) > 2
    f = 151.0
    fac = fom.factor(f)
    x = fac.solve(fom.load_dev(f)).cpu().numpy().ravel()
    assert fac.last_residual <= 1e-10
    xs = spl.splu(fom.operator(f).tocsc()).solve(fom.load(f))
    assert np.linalg.norm(x - xs) <= 1e-7 * np.linalg.norm(xs)


@pytest.mark.slow
def test_cfg4_full_size_assembly(cuda):
    """BASELINE cfg4 resolution (~2.4M DoFs): the generator, element kernels
    and CSR builder run at full size; the assembled operator applies (K and
    M SpMV of the nine primitives) and the structure stiffness is symmetric
    on a random probe (x^T K y = y^T K x)."""
    import torch
    from paper_2310_04734_b200 import fuselage as fz
    fom, info = fz.fuselage_model(fz.cfg4_spec_full(), cuda, solver=False)
    assert fom.n == 2_408_303
    assert sum(t.P.nnz for t in fom.affine.K + fom.affine.M) == 363_502_858
    g = torch.Generator(device="cpu").manual_seed(5)
    x = torch.randn(fom.n, 1, dtype=torch.complex128, generator=g).to(cuda)
    y = torch.randn(fom.n, 1, dtype=torch.complex128, generator=g).to(cuda)
    for kind in ("K", "M"):
        r = fom.apply(kind, 137.0, x)
        assert bool(torch.isfinite(torch.view_as_real(r)).all())
    from paper_2310_04734_b200 import linalg
    Ks = info["Ks"]
    a = (y.T @ linalg.spmm(Ks, x)).item()
    b = (x.T @ linalg.spmm(Ks, y)).item()
    assert abs(a - b) <= 1e-12 * abs(a)
