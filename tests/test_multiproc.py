"""The N > 1 path on CPU: world_size-2 gloo process group, batch sharding, max-over-ranks timing
and counter sums exactly as bench.py uses them (no data-path collective exists)."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2510_13602_b200.dist import Shard, max_over_ranks, rank_seed, shard_batch, sum_over_ranks


def test_shards_cover_the_batch():
    for world in (1, 2, 3, 4, 8):
        shards = [shard_batch(512, world, r, strong=True) for r in range(world)]
        assert sum(s.seq_count for s in shards) == 512
        assert [s.seq_begin for s in shards] == [sum(x.seq_count for x in shards[:r]) for r in range(world)]
        weak = [shard_batch(128, world, r, strong=False) for r in range(world)]
        assert all(s.seq_count == 128 and s.global_batch == 128 * world for s in weak)
    with pytest.raises(ValueError):
        shard_batch(1, 2, 0, strong=True)
    assert len({rank_seed(0, r) for r in range(8)}) == 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = shard_batch(512, world, rank, strong=True)
    t = max_over_ranks(10.0 + rank)                       # rank 1 is the slow one
    sums = sum_over_ranks([shard.seq_count, 100.0 * (rank + 1)])
    dist.barrier()
    out[rank] = (shard, t, sums)
    dist.destroy_process_group()


def test_gloo_world_size_two():
    world, port = 2, _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][1] == res[1][1] == 11.0
    assert res[0][2] == res[1][2] == [512.0, 300.0]
    assert res[0][0] == Shard(0, 2, 0, 256, 512) and res[1][0] == Shard(1, 2, 256, 256, 512)


def test_cpulist_parsing_and_numa_binding(tmp_path):
    from paper_2510_13602_b200.dist import bind_to_gpu_numa_node, parse_cpulist
    assert parse_cpulist("0-3,8,10-11\n") == {0, 1, 2, 3, 8, 10, 11}
    assert parse_cpulist("") == set()
    # no GPU / NVML here: the binder must leave the affinity alone and report None
    before = os.sched_getaffinity(0)
    assert bind_to_gpu_numa_node(0, sysfs=str(tmp_path)) is None
    assert os.sched_getaffinity(0) == before
