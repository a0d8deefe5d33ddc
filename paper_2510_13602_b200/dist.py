"""Multi-GPU plumbing for the batch-sharded decode step.

Sequences never interact on this path, so GPU g owns a contiguous shard of the batch, its own
HBM cache, its own pinned host pool and its own PCIe link.  There is no data-path collective:
torch.distributed is used only for a start barrier and a max-over-ranks reduction of the timed
region, and the per-rank counters are summed for reporting.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    seq_begin: int     # first global sequence id owned by this rank
    seq_count: int     # sequences on this rank
    global_batch: int


def shard_batch(batch: int, world: int, rank: int, strong: bool) -> Shard:
    """Weak scaling: every rank owns `batch` sequences.  Strong scaling: the global batch
    `batch` is split into contiguous, as-equal-as-possible shards."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    if not strong:
        return Shard(rank, world, rank * batch, batch, batch * world)
    if batch < world:
        raise ValueError(f"global batch {batch} smaller than {world} ranks")
    base, extra = divmod(batch, world)
    begin = rank * base + min(rank, extra)
    return Shard(rank, world, begin, base + (1 if rank < extra else 0), batch)


def rank_seed(seed: int, rank: int) -> int:
    """Distinct, reproducible input streams per rank (a rank's shard is independent data)."""
    return seed * 1000003 + rank * 7919


def max_over_ranks(value: float, device=None) -> float:
    """The slowest rank's time (multi-GPU numbers are timed as the max over ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(values: list[float], device=None) -> list[float]:
    """Element-wise sum of per-rank counters (hits, misses, bytes)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()
