"""World-size-2 runs of the sharded entry points on the one-GPU box: two
processes (gloo, device tensors staged through the host) share cuda:0, each
rank runs its own shard with the same kernels, and the gathered results must
equal the serial path bit for bit (frequency sharding of the
sweep, expansion-point sharding of the basis build; the reference itself is
serial)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _env(rank, ws, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws), LOCAL_RANK="0")


def _sweep_worker(rank, ws, port, data, q):
    _env(rank, ws, port)
    import torch
    import torch.distributed as dist
    from paper_2310_04734_b200 import dist as vdist, sweep
    vdist.init(backend="gloo")
    torch.cuda.set_device(0)
    # the parent's inputs (regenerating them here could differ in the last bit:
    # multithreaded BLAS in the workload generator sums in a thread-count-
    # dependent order)
    prims, b, c_r, kinds, freqs = data
    rs = sweep.ReducedSweep(prims, b, c_r, kinds=kinds)
    f = torch.as_tensor(freqs, device="cuda:0")
    spl, y = vdist.sweep_sharded(rs, f, want_y=True)
    q.put((rank, spl.cpu().numpy(), y.cpu().numpy()))
    dist.destroy_process_group()


def _krylov_worker(rank, ws, port, q):
    _env(rank, ws, port)
    import torch
    import torch.distributed as dist
    from paper_2310_04734_b200 import dist as vdist
    vdist.init(backend="gloo")
    torch.cuda.set_device(0)
    from test_fdm_gpu import _small_box
    fom, _ = _small_box(torch.device("cuda:0"))
    V = vdist.krylov_basis_sharded(fom, (80.0, 190.0, 300.0), 4, second_order=True)
    q.put((rank, V.cpu().numpy()))
    dist.destroy_process_group()


CFG4_PTS = (45.0, 110.0, 170.0, 230.0)


def _cfg4_tiny(dev):
    from paper_2310_04734_b200 import fuselage as fz
    spec = fz.FuselageSpec(n_th=16, n_stringers=8, n_z=6, floor_k=1, n_side=2)
    return fz.fuselage_model(spec, dev)[0]


def _krylov_cfg4_worker(rank, ws, port, q):
    _env(rank, ws, port)
    import torch
    import torch.distributed as dist
    from paper_2310_04734_b200 import dist as vdist
    vdist.init(backend="gloo")
    torch.cuda.set_device(0)
    fom = _cfg4_tiny(torch.device("cuda:0"))
    V = vdist.krylov_basis_sharded(fom, CFG4_PTS, 8)
    q.put((rank, V.cpu().numpy()))
    dist.destroy_process_group()


def _singular_worker(rank, ws, port, q):
    _env(rank, ws, port)
    import torch
    import torch.distributed as dist
    from paper_2310_04734_b200 import dist as vdist, sweep
    vdist.init(backend="gloo")
    torch.cuda.set_device(0)
    r = 12
    P = np.zeros((1, r, r), complex)
    P[0, :r - 1, :r - 1] = np.eye(r - 1)
    P[0, r - 1, r - 1] = 1.0
    # coefficient table: frequency index 5 (rank 1's shard) gets a zero operator
    coeff = lambda f: torch.where(f == 5.0, 0.0, 1.0).to(torch.complex128).view(-1, 1)  # noqa: E731
    rs = sweep.ReducedSweep(P, np.ones((r, 1)), np.eye(r), coeff_fn=coeff)
    f = torch.arange(8, dtype=torch.float64, device="cuda:0")
    try:
        vdist.sweep_sharded(rs, f)
        q.put((rank, "no error"))
    except np.linalg.LinAlgError as e:
        q.put((rank, f"LinAlgError: {e}"))
    dist.destroy_process_group()


def _run(target, *args, ws=2, timeout=600):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, ws, port) + args + (q,)) for r in range(ws)]
    for p in procs:
        p.start()
    import queue
    import time
    out = {}
    t_end = time.monotonic() + timeout
    while len(out) < ws:
        try:
            item = q.get(timeout=5)
            out[item[0]] = item[1:]
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            if dead or time.monotonic() > t_end:
                for p in procs:
                    p.kill()
                raise AssertionError(f"rank process failed (exit codes {[p.exitcode for p in procs]})")
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("r", [64, 300])
def test_sharded_sweep_world2_equals_serial(cuda, r):
    """Two ranks sweep disjoint frequency blocks (shared-memory path r = 64,
    blocked path r = 300); the all-gathered SPL and y equal one serial launch
    over all frequencies exactly (one CTA per frequency, fixed reductions)."""
    import torch
    from paper_2310_04734_b200 import sweep, workloads
    w = workloads.cfg5(r=r, n_freq=301)
    out = _run(_sweep_worker, (w.prims, w.b, w.c_r, w.kinds, w.freqs))
    rs = sweep.ReducedSweep(w.prims, w.b, w.c_r, kinds=w.kinds)
    o = rs.sweep_device(torch.as_tensor(w.freqs, device=cuda))
    spl, y = o.spl.cpu().numpy(), o.y.cpu().numpy()
    for rank in (0, 1):
        assert np.array_equal(out[rank][0], spl)
        assert np.array_equal(out[rank][1], y)


def test_sharded_krylov_world2_equals_serial(cuda):
    """Expansion points split over two ranks, blocks all-gathered and appended
    in point order on both ranks: the same basis as the serial MIMO build."""
    from paper_2310_04734_b200 import mor
    from test_fdm_gpu import _small_box
    out = _run(_krylov_worker)
    fom, _ = _small_box(cuda)
    V2, _ = mor.krylov_basis(fom, (80.0, 190.0, 300.0), 4, second_order=True, mimo=True)
    V2 = V2.cpu().numpy()
    for rank in (0, 1):
        assert out[rank][0].shape == V2.shape
        assert np.array_equal(out[rank][0], V2)


def test_sharded_sweep_singular_raises_on_every_rank(cuda):
    """A zero pivot in one rank's shard raises LinAlgError on BOTH ranks (the
    info vector is gathered before the check), instead of leaving the healthy
    rank waiting in the gather."""
    out = _run(_singular_worker, timeout=300)
    for rank in (0, 1):
        assert out[rank][0].startswith("LinAlgError"), out[rank]


def test_sharded_krylov_cfg4_world2_equals_serial(cuda):
    """cfg4 (plane-block full-order solver): expansion points split over two
    ranks give the serial basis bit for bit."""
    from paper_2310_04734_b200 import mor
    out = _run(_krylov_cfg4_worker)
    V2, _ = mor.krylov_basis(_cfg4_tiny(cuda), CFG4_PTS, 8, mimo=True)
    V2 = V2.cpu().numpy()
    for rank in (0, 1):
        assert out[rank][0].shape == V2.shape
        assert np.array_equal(out[rank][0], V2)
