"""Multi-GPU plumbing for the batch-sharded decode step.

Sequences never interact on this path, so GPU g owns a contiguous shard of the batch, its own
HBM cache, its own pinned host pool and its own PCIe link.  There is no data-path collective:
torch.distributed is used only for a start barrier and a max-over-ranks reduction of the timed
region, and the per-rank counters are summed for reporting.
"""

from __future__ import annotations

import os
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


def gpu_numa_node(device_index: int, sysfs: str = "/sys") -> int | None:
    """NUMA node of a GPU's PCIe function (sysfs), or None when unknown."""
    try:
        import pynvml
        pynvml.nvmlInit()
        bus = pynvml.nvmlDeviceGetPciInfo(pynvml.nvmlDeviceGetHandleByIndex(device_index)).busId
        bus = bus.decode() if isinstance(bus, bytes) else bus
    except Exception:
        return None
    bdf = bus.lower()
    if bdf.count(":") == 2 and len(bdf.split(":")[0]) == 8:  # NVML pads the domain to 8 digits
        bdf = bdf[4:]
    try:
        node = int(open(os.path.join(sysfs, "bus/pci/devices", bdf, "numa_node")).read().strip())
    except (OSError, ValueError):
        return None
    return node if node >= 0 else None


def parse_cpulist(text: str) -> set[int]:
    """'0-3,8,10-11' -> {0, 1, 2, 3, 8, 10, 11} (the sysfs cpulist format)."""
    cpus: set[int] = set()
    for part in text.strip().split(","):
        if not part:
            continue
        lo, _, hi = part.partition("-")
        cpus.update(range(int(lo), int(hi or lo) + 1))
    return cpus


def bind_to_gpu_numa_node(device_index: int, sysfs: str = "/sys") -> int | None:
    """Pin this process to the CPUs of its GPU's NUMA node before the pinned slow tier is
    allocated, so the pages (first touch) and the host threads sit next to the GPU's PCIe root:
    with one process per GPU, every rank then streams its misses from local DRAM.  Returns the
    node, or None (nothing changed) when the topology is unknown or the CPUs are not allowed."""
    node = gpu_numa_node(device_index, sysfs)
    if node is None:
        return None
    try:
        cpus = parse_cpulist(open(os.path.join(sysfs, f"devices/system/node/node{node}/cpulist")).read())
        allowed = cpus & os.sched_getaffinity(0)
        if not allowed:
            return None
        os.sched_setaffinity(0, allowed)
    except (OSError, ValueError, AttributeError):
        return None
    return node
