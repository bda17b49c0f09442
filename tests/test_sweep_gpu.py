"""GPU parity of the batched reduced sweep (vb_rom_sweep) against the oracle
(oracle.mor.affine_sweep = mor.py:73-102 + solvers.py:334-338 with
numpy.linalg.solve).  Tolerances (north_star): relative transfer-function
error <= 1e-8 (mor.py:194-208 metric) and |dSPL| <= 0.01 dB."""

import math

import numpy as np
import pytest

from oracle import mor as omor

TF_TOL = 1e-8
SPL_TOL = 0.01

pytestmark = pytest.mark.gpu


def _run(cuda, prims, alpha, b, c_r, want_x=False):
    import torch
    from paper_2310_04734_b200 import sweep
    P = sweep.as_ctensor(prims, cuda)
    A = sweep.as_ctensor(alpha, cuda)
    B = sweep.as_ctensor(b, cuda)
    Cr = sweep.as_ctensor(c_r, cuda)
    out = sweep.rom_sweep_affine(P, A, B, Cr, want_x=want_x)
    torch.cuda.synchronize()
    return out


def _check(y_gpu, spl_gpu, y_ref, spl_ref):
    F = y_ref.shape[0]
    worst = 0.0
    for i in range(F):
        _, e, _, _ = omor.relative_error(y_ref[i].ravel(), y_gpu[i].ravel())
        worst = max(worst, e)
    assert worst <= TF_TOL, worst
    assert np.abs(spl_gpu - spl_ref).max() <= SPL_TOL
    return worst


@pytest.mark.parametrize("r,s,n_out,K", [(32, 1, 50, 3), (8, 3, 5, 2), (60, 4, 50, 3), (76, 1, 1, 4),
                                          (96, 16, 50, 3), (1, 1, 1, 1)])
def test_small_path_matches_oracle(cuda, r, s, n_out, K):
    from paper_2310_04734_b200 import _lib
    assert _lib.load().vb_rom_sweep_path(r, K, s, n_out) == 0
    rng = np.random.default_rng(r * 100 + s)
    F = 37
    prims = rng.standard_normal((K, r, r)) + 1j * rng.standard_normal((K, r, r))
    prims[0] += 4 * np.sqrt(r) * np.eye(r)
    alpha = rng.standard_normal((F, K)) + 1j * rng.standard_normal((F, K))
    alpha[:, 0] = 1.0
    b = rng.standard_normal((r, s)) + 1j * rng.standard_normal((r, s))
    c_r = rng.standard_normal((n_out, r)) + 1j * rng.standard_normal((n_out, r))
    y_ref, spl_ref = omor.affine_sweep(prims, alpha, b, c_r)
    out = _run(cuda, prims, alpha, b, c_r, want_x=True)
    assert int(out.info.abs().sum()) == 0
    _check(out.y.cpu().numpy(), out.spl.cpu().numpy(), y_ref, spl_ref)
    x_ref = np.stack([np.linalg.solve(np.tensordot(alpha[i], prims, 1), b) for i in range(F)])
    assert np.abs(out.x.cpu().numpy() - x_ref).max() <= 1e-9 * np.abs(x_ref).max()


def test_frequency_dependent_rhs(cuda):
    rng = np.random.default_rng(3)
    r, s, F, K = 20, 2, 11, 3
    prims = rng.standard_normal((K, r, r)) + 1j * rng.standard_normal((K, r, r))
    alpha = rng.standard_normal((F, K)) + 1j * rng.standard_normal((F, K))
    b = rng.standard_normal((F, r, s)) + 1j * rng.standard_normal((F, r, s))
    c_r = rng.standard_normal((7, r)) + 0j
    y_ref, spl_ref = omor.affine_sweep(prims, alpha, b, c_r)
    out = _run(cuda, prims, alpha, b, c_r)
    _check(out.y.cpu().numpy(), out.spl.cpu().numpy(), y_ref, spl_ref)


def test_pivoting_required(cuda):
    """Zero leading diagonal: fails without row interchanges (zgesv pivots)."""
    r = 12
    P = np.zeros((1, r, r), complex)
    for i in range(r):
        P[0, i, (i + 1) % r] = 1.0 + 0.5j * i
    alpha = np.ones((2, 1), complex)
    b = np.arange(1, r + 1, dtype=complex)[:, None]
    c_r = np.eye(r, dtype=complex)
    y_ref, spl_ref = omor.affine_sweep(P, alpha, b, c_r)
    out = _run(cuda, P, alpha, b, c_r)
    _check(out.y.cpu().numpy(), out.spl.cpu().numpy(), y_ref, spl_ref)


def test_singular_reports_info(cuda):
    """numpy.linalg.solve raises LinAlgError on an exactly singular matrix (mor.py:94)."""
    from paper_2310_04734_b200 import sweep
    r = 6
    P = np.zeros((1, r, r), complex)
    P[0, :5, :5] = np.eye(5)
    alpha = np.ones((3, 1), complex)
    b = np.ones((r, 1), complex)
    c_r = np.ones((1, r), complex)
    with pytest.raises(np.linalg.LinAlgError):
        np.linalg.solve(P[0], b)
    out = _run(cuda, P, alpha, b, c_r)
    assert out.info.cpu().tolist() == [6, 6, 6]
    with pytest.raises(np.linalg.LinAlgError):
        sweep.raise_if_singular(out.info)


def test_cfg5_r256_sample(cuda):
    from paper_2310_04734_b200 import workloads
    w = workloads.cfg5(r=256, n_freq=100_000)
    idx = np.linspace(0, 99_999, 24).astype(int)
    f = w.freqs[idx]
    alpha = w.alpha(f)
    y_ref, spl_ref = omor.affine_sweep(w.prims, alpha, w.b, w.c_r)
    out = _run(cuda, w.prims, alpha, w.b, w.c_r)
    _check(out.y.cpu().numpy(), out.spl.cpu().numpy(), y_ref, spl_ref)


@pytest.fixture
def force_blocked(cuda):
    from paper_2310_04734_b200 import _lib
    _lib.load().vb_set_sweep_path_override(1)
    yield
    _lib.load().vb_set_sweep_path_override(-1)


@pytest.mark.parametrize("r,s,n_out,K", [(1, 1, 1, 1), (5, 2, 3, 2), (33, 1, 50, 3), (64, 16, 50, 3),
                                          (65, 3, 7, 3), (100, 1, 50, 3), (130, 16, 50, 4),
                                          (200, 5, 20, 3)])
def test_blocked_path_matches_oracle(cuda, force_blocked, r, s, n_out, K):
    rng = np.random.default_rng(7 * r + s)
    F = 19
    prims = rng.standard_normal((K, r, r)) + 1j * rng.standard_normal((K, r, r))
    alpha = rng.standard_normal((F, K)) + 1j * rng.standard_normal((F, K))
    b = rng.standard_normal((r, s)) + 1j * rng.standard_normal((r, s))
    c_r = rng.standard_normal((n_out, r)) + 1j * rng.standard_normal((n_out, r))
    y_ref, spl_ref = omor.affine_sweep(prims, alpha, b, c_r)
    out = _run(cuda, prims, alpha, b, c_r, want_x=True)
    assert int(out.info.abs().sum()) == 0
    _check(out.y.cpu().numpy(), out.spl.cpu().numpy(), y_ref, spl_ref)
    x_ref = np.stack([np.linalg.solve(np.tensordot(alpha[i], prims, 1), b) for i in range(F)])
    rel = np.abs(out.x.cpu().numpy() - x_ref).max() / np.abs(x_ref).max()
    assert rel <= 1e-9, rel


def test_blocked_pivoting_and_singular(cuda, force_blocked):
    r = 70
    P = np.zeros((1, r, r), complex)
    for i in range(r):
        P[0, i, (i + 3) % r] = 1.0 + 0.5j * i
    alpha = np.ones((2, 1), complex)
    b = np.arange(1, r + 1, dtype=complex)[:, None]
    c_r = np.eye(r, dtype=complex)
    y_ref, spl_ref = omor.affine_sweep(P, alpha, b, c_r)
    out = _run(cuda, P, alpha, b, c_r)
    _check(out.y.cpu().numpy(), out.spl.cpu().numpy(), y_ref, spl_ref)
    P2 = np.zeros((1, r, r), complex)
    P2[0, :r - 1, :r - 1] = np.eye(r - 1)
    out = _run(cuda, P2, alpha, b, c_r)
    assert out.info.cpu().tolist() == [r, r]


def _resonance_probes(w, n_res: int = 16, n_total: int = 64, seed: int = 0) -> np.ndarray:
    """n_res grid frequencies right next to the workload's undamped
    eigenfrequencies (the 100k grid point nearest each of n_res eigenfrequencies
    spread over the band, and its neighbour) plus seeded random grid points."""
    from paper_2310_04734_b200 import workloads
    ef = workloads.cfg5_eigenfrequencies(w)
    ef = ef[(ef > w.freqs[0]) & (ef < w.freqs[-1])]
    pick = ef[np.linspace(0, len(ef) - 1, n_res // 2).astype(int)]
    idx = np.clip(np.searchsorted(w.freqs, pick), 1, len(w.freqs) - 1)
    res = np.unique(np.concatenate([idx - 1, idx]))
    rng = np.random.default_rng(seed)
    rest = rng.choice(np.setdiff1d(np.arange(len(w.freqs)), res), n_total - len(res), replace=False)
    return np.sort(np.concatenate([res, rest]))


@pytest.mark.parametrize("r", [256, 400, 1024, 1536, 2048])
def test_cfg5_full_size_64_frequencies(cuda, r):
    """BASELINE cfg5 at its full reduced orders (the bench's headline kernel):
    64 frequencies of the 100k grid, 16 of them straddling undamped
    eigenfrequencies, against the oracle (numpy zgesv): TF <= 1e-8 pointwise
    (mor.py:194-208) and |dSPL| <= 0.01 dB."""
    from paper_2310_04734_b200 import workloads
    w = workloads.cfg5(r=r, n_freq=100_000)
    f = w.freqs[_resonance_probes(w, seed=r)]
    alpha = w.alpha(f)
    y_ref, spl_ref = omor.affine_sweep(w.prims, alpha, w.b, w.c_r)
    out = _run(cuda, w.prims, alpha, w.b, w.c_r)
    assert int(out.info.abs().sum()) == 0
    _check(out.y.cpu().numpy(), out.spl.cpu().numpy(), y_ref, spl_ref)


@pytest.mark.parametrize("r", [401, 450, 700, 1001, 1537, 1601])
@pytest.mark.parametrize("s", [1, 3])
def test_blocked_partial_outer_steps(cuda, force_blocked, r, s):
    """Orders whose last outer step is partial: fewer panels than the 2-panel
    (r >= 640) / 4-panel (r >= 1536) step holds, a last panel narrower than 64
    and GEMM depths that are not multiples of 8 (greedy ROMs have any r)."""
    rng = np.random.default_rng(r + 10 * s)
    K, F, n_out = 3, 5, 20
    X = rng.standard_normal((r, r)) + 1j * rng.standard_normal((r, r))
    prims = np.stack([X @ X.conj().T / r + np.eye(r),
                      0.1 * (rng.standard_normal((r, r)) + 1j * rng.standard_normal((r, r))),
                      np.eye(r) + 0j])
    alpha = np.stack([np.ones(F), 1j * rng.uniform(0.5, 2, F), -rng.uniform(0.5, 3, F) + 0j], 1)
    b = rng.standard_normal((r, s)) + 1j * rng.standard_normal((r, s))
    c_r = rng.standard_normal((n_out, r)) + 1j * rng.standard_normal((n_out, r))
    y_ref, spl_ref = omor.affine_sweep(prims, alpha, b, c_r)
    out = _run(cuda, prims, alpha, b, c_r, want_x=True)
    assert int(out.info.abs().sum()) == 0
    _check(out.y.cpu().numpy(), out.spl.cpu().numpy(), y_ref, spl_ref)
    x_ref = np.stack([np.linalg.solve(np.tensordot(alpha[i], prims, 1), b) for i in range(F)])
    rel = np.abs(out.x.cpu().numpy() - x_ref).max() / np.abs(x_ref).max()
    assert rel <= 1e-9, rel


@pytest.mark.parametrize("force", [0, 1])
def test_nan_column_sets_info_without_fault(cuda, force):
    """A NaN pivot column is reported like a zero pivot (info = k + 1, as
    LAPACK's izamax never selects it) instead of indexing shared memory with an
    invalid row; the other frequencies of the launch are unaffected."""
    import torch
    from paper_2310_04734_b200 import _lib
    r = 40
    rng = np.random.default_rng(3)
    P = (rng.standard_normal((1, r, r)) + 1j * rng.standard_normal((1, r, r))) + 8 * np.eye(r)
    alpha = np.ones((3, 1), complex)
    alpha[1, 0] = np.nan
    b = rng.standard_normal((r, 1)) + 0j
    c_r = np.eye(r, dtype=complex)
    _lib.load().vb_set_sweep_path_override(force)
    try:
        out = _run(cuda, P, alpha, b, c_r)
    finally:
        _lib.load().vb_set_sweep_path_override(-1)
    torch.cuda.synchronize()
    info = out.info.cpu().tolist()
    assert info[0] == 0 and info[2] == 0 and info[1] >= 1
    y_ref, spl_ref = omor.affine_sweep(P, alpha[[0]], b, c_r)
    _check(out.y[:1].cpu().numpy(), out.spl[:1].cpu().numpy(), y_ref, spl_ref)


def test_sweep_on_side_stream_matches_current_stream(cuda):
    """ReducedSweep(stream=s): the launch is ordered after the inputs produced
    on the current stream and the results equal the default-stream sweep."""
    import torch
    from paper_2310_04734_b200 import sweep, workloads
    w = workloads.cfg5(r=256, n_freq=300)
    side = torch.cuda.Stream()
    rs1 = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds)
    rs2 = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds, stream=side)
    y1, s1 = rs1.sweep(w.freqs)
    y2, s2 = rs2.sweep(w.freqs)
    assert np.array_equal(y1, y2) and np.array_equal(s1, s2)


def test_cfg5_r1024_residuals_and_determinism(cuda):
    """Size-independent properties on a full launch (2 x #SM frequencies at
    r = 1024): backward-stable residuals ||A x - b|| / (||A|| ||x||) for every
    frequency, and bit-identical results for the same frequency at different
    batch positions (one CTA per frequency, fixed reduction orders)."""
    import torch
    from paper_2310_04734_b200 import sweep, workloads
    w = workloads.cfg5(r=1024, n_freq=100_000)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    F = 2 * nsm
    f = w.freqs[np.linspace(0, 99_999, F).astype(int)]
    f[-1] = f[0]  # same frequency in the first and the last slot
    alpha = w.alpha(f)
    out = _run(cuda, w.prims, alpha, w.b, w.c_r, want_x=True)
    assert int(out.info.abs().sum()) == 0
    assert torch.equal(out.x[0], out.x[-1]) and torch.equal(out.y[0], out.y[-1])
    P = sweep.as_ctensor(w.prims, cuda)
    B = sweep.as_ctensor(w.b, cuda)
    Al = sweep.as_ctensor(alpha, cuda)
    worst = 0.0
    for i in range(0, F, 37):
        A = torch.einsum("k,kij->ij", Al[i], P)
        X = out.x[i]
        R = A @ X - B
        rel = float(torch.linalg.matrix_norm(R) / (torch.linalg.matrix_norm(A) * torch.linalg.matrix_norm(X)))
        worst = max(worst, rel)
    assert worst <= 1e-14, worst


def test_blocked_path_more_than_16_rhs(cuda):
    """s > 16 right-hand sides on the blocked path run as groups of 16 (the
    reference's numpy.linalg.solve takes any number of columns)."""
    rng = np.random.default_rng(33)
    r, s, n_out, K, F = 150, 37, 20, 3, 9
    prims = rng.standard_normal((K, r, r)) + 1j * rng.standard_normal((K, r, r))
    alpha = rng.standard_normal((F, K)) + 1j * rng.standard_normal((F, K))
    b = rng.standard_normal((r, s)) + 1j * rng.standard_normal((r, s))
    c_r = rng.standard_normal((n_out, r)) + 1j * rng.standard_normal((n_out, r))
    y_ref, spl_ref = omor.affine_sweep(prims, alpha, b, c_r)
    out = _run(cuda, prims, alpha, b, c_r, want_x=True)
    _check(out.y.cpu().numpy(), out.spl.cpu().numpy(), y_ref, spl_ref)
    x_ref = np.stack([np.linalg.solve(np.tensordot(alpha[i], prims, 1), b) for i in range(F)])
    assert np.abs(out.x.cpu().numpy() - x_ref).max() <= 1e-9 * np.abs(x_ref).max()


def test_sharded_sweep_world1_matches_direct(cuda):
    """dist.sweep_sharded (frequency shards + SPL/y gather) at world size 1
    returns exactly the direct sweep."""
    import torch
    from paper_2310_04734_b200 import dist as vdist, sweep, workloads
    w = workloads.cfg5(r=256, n_freq=500)
    rs = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds)
    f = torch.as_tensor(w.freqs, device=cuda)
    spl, y = vdist.sweep_sharded(rs, f, want_y=True)
    out = rs.sweep_device(f)
    assert torch.equal(spl, out.spl) and torch.equal(y, out.y)


def test_empty_and_degenerate_inputs(cuda):
    """Empty frequency lists / grids and outputs-free sweeps: no launch, empty
    results (the reference's loops simply do nothing); an all-zero Krylov
    block is dropped entirely by the drop rule (mor.py:133: ref = 0 -> drop)."""
    import torch
    from paper_2310_04734_b200 import mor, sweep, workloads
    w = workloads.cfg5(r=64, n_freq=10)
    rs = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds)
    out = rs.sweep_device(torch.empty(0, dtype=torch.float64, device=cuda))
    assert out.y.shape == (0, w.c_r.shape[0], w.b.shape[1]) and out.spl.shape == (0, w.b.shape[1])
    y, spl = rs.sweep(np.zeros(0))
    assert y.shape[0] == 0 and spl.shape[0] == 0
    o = sweep.rom_sweep_affine(sweep.as_ctensor(w.prims, cuda), sweep.as_ctensor(w.alpha(w.freqs[:3]), cuda),
                               sweep.as_ctensor(w.b, cuda), sweep.as_ctensor(np.zeros((0, 64)), cuda),
                               want_x=True)
    torch.cuda.synchronize()
    assert o.y is None and o.spl is None and o.x.shape == (3, 64, w.b.shape[1])
    x_ref = np.linalg.solve(np.tensordot(w.alpha(w.freqs[:1])[0], w.prims, 1), w.b)
    assert np.abs(o.x[0].cpu().numpy() - x_ref).max() <= 1e-10 * np.abs(x_ref).max()
    V0 = mor._orthonormalise(None, torch.randn(300, 4, dtype=torch.complex128, device=cuda))
    V1 = mor._orthonormalise(V0, torch.zeros(300, 3, dtype=torch.complex128, device=cuda))
    assert V1.shape == (300, 4)
    V2 = mor.orthonormalise_blocks(V0, [torch.zeros(300, 3, dtype=torch.complex128, device=cuda),
                                        V0[:, :2].clone()])
    assert V2.shape == (300, 4)
    fom = mor.FullOrderModel(stiffness=lambda f: np.eye(5) * 4.0, mass=lambda f: np.eye(5), load=lambda f: np.ones(5),
                             c_out=np.ones(5), n=5)
    rom = mor.ReducedModel(fom=fom, V=np.eye(5, dtype=complex), window=(1.0, 2.0))
    res = mor.rom_sweep([rom], [])
    assert res.freqs == [] and res.frf == []
