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
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
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
    dist.all_gather_into_tensor(out, pad)
    parts = [out[r * width: r * width + (hi - lo)] for r, (lo, hi) in enumerate(sizes)]
    return torch.cat(parts, dim=0)


def max_over_ranks(x: float, device=None) -> float:
    if not (dist.is_available() and dist.is_initialized()):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    if dist.is_available() and dist.is_initialized():
        dist.barrier()
