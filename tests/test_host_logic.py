"""Host-side logic of the product package (no GPU): certification helpers,
window rules, frequency sharding and the SPL gather over a 2-rank gloo group."""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def test_relative_error_and_candidates_follow_reference():
    from paper_2310_04734_b200 import mor
    y = np.array([1.0, 2.0, 3.0])
    eps, emax, k, flag = mor.relative_error(y, 1.01 * y)
    assert emax == pytest.approx(0.01) and not flag
    eps, emax, k, flag = mor.relative_error([0.0, 2.0], [0.5, 2.0])
    assert flag and eps[0] == pytest.approx(0.5)
    grid = [float(f) for f in range(10, 101, 10)]
    cand = mor.candidate_frequencies(grid, (10.0, 100.0), 4)
    assert cand[0] == 10.0 and cand[-1] == 100.0
    with pytest.raises(ValueError):
        mor.candidate_frequencies(grid, (101.0, 102.0), 4)


def test_window_plan_validation():
    from paper_2310_04734_b200 import mor
    band = (10.0, 100.0)
    assert mor.window_plan(band, "auto") == [(10.0, 100.0)]
    assert mor.window_plan(band, [(10.0, 40.0), (40.0, 100.0)]) == [(10.0, 40.0), (40.0, 100.0)]
    for bad in ([(10.0, 40.0), (50.0, 100.0)], [(10.0, 90.0)]):
        with pytest.raises(ValueError):
            mor.window_plan(band, bad)
    with pytest.raises(ValueError):
        mor.window_plan((100.0, 100.0), "auto")


def test_mean_spl_product_matches_reference_value():
    from paper_2310_04734_b200.solvers import mean_spl
    assert mean_spl(np.ones(64, complex)) == pytest.approx(20 * np.log10(1 / np.sqrt(2) / 20e-6))
    assert mean_spl(np.zeros(3)) == pytest.approx(20 * math.log10(1e-300 / 20e-6))


def test_shard_range_covers_and_balances():
    from paper_2310_04734_b200.dist import shard_range
    for n in (0, 1, 7, 100_000, 181):
        for ws in (1, 2, 3, 8):
            parts = [shard_range(n, r, ws) for r in range(ws)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1


def test_affine_coefficients_form():
    from paper_2310_04734_b200.sweep import affine_coefficients
    f = torch.tensor([1.0, 10.0])
    a = affine_coefficients(f, [("K", 1.0), ("D", 2.0), ("M", 3.0)])
    w = 2 * math.pi * f.numpy()
    np.testing.assert_allclose(a.numpy(), np.stack([np.ones(2), 2j * w, -3 * w * w], 1))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws), LOCAL_RANK=str(rank))
    from paper_2310_04734_b200 import dist as vdist
    vdist.init(backend="gloo")
    lo, hi = vdist.shard_range(n, rank, ws)
    # each rank "sweeps" its frequency block: SPL rows tagged by the global index
    local = torch.arange(lo, hi, dtype=torch.float64).unsqueeze(1).repeat(1, 3) * 10 + rank
    full = vdist.gather_rows(local, n, ws)
    t = vdist.max_over_ranks(float(rank + 1))
    q.put((rank, full.numpy(), t))
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 10])
def test_frequency_shards_gather_over_gloo(n):
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, n, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2310_04734_b200.dist import shard_range
    for rank, full, t in out:
        assert full.shape == (n, 3)
        for r in range(ws):
            lo, hi = shard_range(n, r, ws)
            np.testing.assert_array_equal(full[lo:hi, 0], np.arange(lo, hi) * 10 + r)
        assert t == 2.0


def _blocks_worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws), LOCAL_RANK=str(rank))
    from paper_2310_04734_b200 import dist as vdist
    vdist.init(backend="gloo")
    counts = [3, 2]
    g = torch.Generator().manual_seed(100 + rank)
    local = [torch.randn((6, 1 + (rank + i) % 4), dtype=torch.complex128, generator=g) for i in range(counts[rank])]
    full = vdist.gather_blocks(local, counts, 6, 4, torch.complex128, torch.device("cpu"))
    q.put((rank, [b.numpy().copy() for b in local], [b.numpy().copy() for b in full]))
    dist.destroy_process_group()


def test_gather_variable_width_blocks_over_gloo():
    """Offline sharding by expansion point: Krylov blocks of different widths
    (breakdowns) all-gathered in rank order on every rank."""
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_blocks_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(ws):
        rank, local, full = q.get(timeout=120)
        out[rank] = (local, full)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = out[0][0] + out[1][0]
    for rank in range(ws):
        full = out[rank][1]
        assert len(full) == 5
        for a, b in zip(full, expect):
            np.testing.assert_array_equal(a, b)


def test_fdm_axis_eigenpairs_diagonalise_the_pencil():
    """BoxFDM.axis_eig (Cholesky-reduced zgeev): A_d V = M_d V Lambda and
    V^T M_d V = I (the complex-symmetric normalisation fdm.py relies on)."""
    import numpy as np
    from paper_2310_04734_b200.fdm import BoxFDM
    box = BoxFDM((0, 0, 0, 2.0, 1.6, 1.2), (10, 8, 6), 1.21, 343.0, {"x0": 2000.0 + 300j, "z1": 900.0})
    for d in range(3):
        for f in (20.0, 180.0):
            lam, V = box.axis_eig(d, f)
            A, M = box.direction_operator(d, f), box.lines[d][1]
            assert np.abs(A @ V - M @ V * lam).max() <= 1e-9 * np.abs(A).max()
            assert np.abs(V.T @ M @ V - np.eye(len(lam))).max() <= 1e-10
