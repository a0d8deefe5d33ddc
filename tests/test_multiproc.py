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


def _bench_shard_worker(rank, world, port, out):
    """bench.workload_dims under a 2-rank gloo group whose ranks see different free host RAM."""
    import sys
    from argparse import Namespace
    from pathlib import Path
    import torch.distributed as dist
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), LOCAL_RANK=str(rank),
                      LOCAL_WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    per_seq = 28 * 2 * 517 * 32768  # cfg3 slow tier per sequence (bench.workload_dims)
    bench.host_mem_available = lambda: int((40 + 30 * rank) * per_seq * world / 0.8)  # rank 0 fits 40, rank 1 70
    args = Namespace(workload="cfg3", layers=None, batch=None, impl="native", slow_tier="host")
    w = bench.workload_dims(args, world)
    out[rank] = (w["batch_local"], w["global_batch"], w["host_limited"])
    dist.destroy_process_group()


def test_bench_ranks_agree_on_the_host_limited_shard():
    world, port = 2, _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_bench_shard_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0] == res[1] == (40, 80, True)


def test_bench_burn_in_defaults(monkeypatch):
    """Untimed burn-in before the warm-up: 32 steps, 128 for cfg5 (256 slots over a 1007-block
    pool settle later); an explicit --burn-in wins."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    for argv, want in ((["bench.py"], 32), (["bench.py", "--workload", "cfg5"], 128),
                       (["bench.py", "--workload", "cfg5", "--burn-in", "7"], 7)):
        monkeypatch.setattr(sys, "argv", argv)
        assert bench.parse().burn_in == want


def test_torchrun_two_ranks_reference_arm():
    """The driver's N>1 launch (torch.distributed.run, 2 ranks on 127.0.0.1) of the reference arm:
    rank 0 alone prints one JSON line with n_gpus = 2, rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl", "reference",
           "--workload", "cfg1", "--gpus", "2", "--steps", "1", "--warmup", "0"]
    p = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, p.stdout
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
