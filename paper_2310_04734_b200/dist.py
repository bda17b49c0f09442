"""Frequency sharding across GPUs: one process per GPU, contiguous
frequency blocks per rank, no exchange during the sweep, and one final gather
of the SPL curves (NCCL over NVLink on B200; gloo in the CPU tests).

The reference has no parallelism at all (SPEC.md:552 only states that the ROM
sweep is embarrassingly parallel over frequencies); this module is new.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str | None = None):
    rank, ws, local = world()
    if ws > 1 and not dist.is_initialized():
        if backend is None:  # VB_DIST_BACKEND: e.g. gloo for ranks sharing one GPU in tests
            backend = os.environ.get("VB_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend, rank=rank, world_size=ws)
    return rank, ws, local


def shard_range(n: int, rank: int, world_size: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items owned by `rank`; sizes differ by <= 1."""
    q, rem = divmod(n, world_size)
    lo = rank * q + min(rank, rem)
    hi = lo + q + (1 if rank < rem else 0)
    return lo, hi


def _host_staged() -> bool:
    """gloo has no CUDA all-gather: device tensors travel through host copies
    (the CPU tests and the world-2-on-one-GPU tests use gloo; NCCL moves device
    memory directly)."""
    return dist.is_initialized() and dist.get_backend() == "gloo"


def _all_gather_into(out: torch.Tensor, inp: torch.Tensor):
    if inp.is_cuda and _host_staged():
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(o, inp.cpu())
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp)


def gather_rows(local: torch.Tensor, n_total: int, world_size: int) -> torch.Tensor:
    """Concatenate per-rank row blocks (shard_range layout) on every rank.

    Pads each shard to the largest block so one all_gather_into_tensor moves
    everything; trims back afterwards.
    """
    if world_size == 1:
        return local
    sizes = [shard_range(n_total, r, world_size) for r in range(world_size)]
    width = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world_size * width,) + tuple(local.shape[1:]), dtype=local.dtype,
                      device=local.device)
    _all_gather_into(out, pad)
    parts = [out[r * width: r * width + (hi - lo)] for r, (lo, hi) in enumerate(sizes)]
    return torch.cat(parts, dim=0)


def max_over_ranks(x: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=None if _host_staged() else device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def gather_blocks(local: list, counts: list[int], n_rows: int, max_cols: int, dtype, device) -> list:
    """All-gather variable-width column blocks: rank q contributes `counts[q]`
    blocks (n_rows x w, w <= max_cols, row-major); every rank receives all
    sum(counts) blocks in rank order.  One padded all_gather_into_tensor for
    the payload and one for the widths (complex payloads travel as real
    pairs, which every backend supports)."""
    ws = len(counts)
    if ws == 1:
        return list(local)
    cmax = max(max(counts), 1)
    buf = torch.zeros((cmax, n_rows, max_cols), dtype=dtype, device=device)
    widths = torch.zeros(cmax, dtype=torch.int64, device=device)
    for i, b in enumerate(local):
        b2 = b if b.dim() == 2 else b.view(-1, 1)
        buf[i, :, : b2.shape[1]] = b2
        widths[i] = b2.shape[1]
    real = torch.view_as_real(buf) if buf.is_complex() else buf
    out = torch.empty((ws * cmax,) + tuple(real.shape[1:]), dtype=real.dtype, device=device)
    _all_gather_into(out, real.contiguous())
    wout = torch.empty(ws * cmax, dtype=torch.int64, device=device)
    _all_gather_into(wout, widths)
    full = torch.view_as_complex(out) if buf.is_complex() else out
    wl = wout.cpu().tolist()
    return [full[q * cmax + i, :, : wl[q * cmax + i]] for q in range(ws) for i in range(counts[q])]


def krylov_basis_sharded(fom, points, moments: int, second_order: bool = False):
    """Offline phase sharded by expansion point: each rank
    factors the FOM and builds the Krylov blocks of its contiguous share of
    `points` (mor.krylov_block, mor.py:138-180, per load column for a block
    RHS), the blocks are all-gathered, and every rank appends them with
    mor.orthonormalise_blocks point by point — the serial build's sequence
    (mor.krylov_basis), so every rank holds the same basis.  Returns V (n x r, device)."""
    from . import mor
    rank, ws, _ = world()
    if ws > 1 and not (dist.is_available() and dist.is_initialized()):
        raise RuntimeError("krylov_basis_sharded: call dist.init() first")
    points = list(points)
    lo, hi = shard_range(len(points), rank, ws)
    mine = []
    n_load = None
    local = points[lo:hi]
    per_point = (mor.krylov_blocks_concurrent(fom, local, moments, second_order, mimo=True)
                 if mor._lu_factored(fom) else
                 [mor.krylov_blocks_mimo_dev(fom, f, moments, second_order=second_order) for f in local])
    for blocks in per_point:
        n_load = len(blocks)
        mine += [Q for Q, _ in blocks]
    if n_load is None:  # a rank without points still needs the per-point block count
        n_load = int(fom.load_dev(points[0], mor._device()).shape[1]) if points else 0
    counts = [(b - a) * n_load for a, b in (shard_range(len(points), q, ws) for q in range(ws))]
    dev = mor._device()
    allq = gather_blocks(mine, counts, fom.n, moments, mor.CDT, dev)
    V, group = None, []
    for p in range(len(points)):  # the grouping of mor.krylov_basis (same basis as the serial build)
        group += [Q.contiguous() for Q in allq[p * n_load:(p + 1) * n_load]]
        if sum(Q.shape[1] for Q in group) >= mor.GROUP_COLS:
            V = mor.orthonormalise_blocks(V, group)
            group = []
    if group:
        V = mor.orthonormalise_blocks(V, group)
    return V


def sweep_sharded(rs, freqs: torch.Tensor, want_y: bool = False):
    """Reduced sweep sharded by frequency: rank q sweeps its
    contiguous block of `freqs` with `rs` (sweep.ReducedSweep, primitives
    already on its GPU), then the SPL rows (and optionally the outputs y) are
    all-gathered; returns (spl (F, s), y (F, n_out, s) or None) on every rank."""
    from .sweep import raise_if_singular
    rank, ws, _ = world()
    F = int(freqs.shape[0])
    lo, hi = shard_range(F, rank, ws)
    s, n_out = int(rs.b.shape[-1]), int(rs.c.shape[0])
    if hi > lo:
        out = rs.sweep_device(freqs[lo:hi], want_y=want_y)
        spl_l, y_l, info_l = out.spl, out.y, out.info
    else:  # more ranks than frequencies
        spl_l = torch.empty((0, s), dtype=torch.float64, device=rs.device)
        y_l = torch.empty((0, n_out, s), dtype=torch.complex128, device=rs.device) if want_y else None
        info_l = torch.empty((0,), dtype=torch.int32, device=rs.device)
    # gather first, then every rank checks the same full info vector: a zero
    # pivot on one rank raises LinAlgError on all of them (no rank is left
    # waiting in a collective the failing rank never reaches)
    info = gather_rows(info_l, F, ws)
    spl = gather_rows(spl_l, F, ws)
    y = gather_rows(y_l, F, ws) if want_y else None
    raise_if_singular(info)
    return spl, y
