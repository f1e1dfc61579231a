"""Batch sharding across GPUs (one process per GPU).

Matrices are independent, so a rank exponentiates its own slice of the global
batch with no collective on the data path -- the same decomposition as the
reference's process pool (bench.py:303-309: independent tasks, results in
task order).  The only collectives are bookkeeping: the max-over-ranks step
time and, when results must come home, one gather to rank 0 in rank order.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(rank: int, world: int, global_batch: int) -> tuple[int, int]:
    """Contiguous [start, stop) slice of the global batch owned by ``rank``;
    sizes differ by at most one and concatenating slices in rank order
    restores the global order."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the step time) over the process group."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_to_rank0(local: torch.Tensor, global_batch: int):
    """Rank-ordered concatenation of every rank's results on rank 0 (None
    elsewhere).  Handles uneven shards by padding to the largest shard."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    sizes = [shard_range(r, world, global_batch) for r in range(world)]
    cap = max(b - a for a, b in sizes)
    pad = local
    if local.shape[0] < cap:
        pad = torch.cat([local, local.new_zeros((cap - local.shape[0],) + tuple(local.shape[1:]))])
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    dist.gather(pad.contiguous(), bufs, dst=0)
    if rank != 0:
        return None
    return torch.cat([bufs[r][: b - a] for r, (a, b) in enumerate(sizes)])
