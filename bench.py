#!/usr/bin/env python
"""Batched NOSA offloaded sparse-attention decode throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3] [--impl native|reference]

A step is one decode step of every sequence through every layer: per layer, selection + cache
plan (K1+K2), miss gather pinned-host -> HBM (K3, side stream), block-sparse attention + append
(K4+K5).  Default workload = BASELINE config 3: 1B-class attention shape (16 q / 2 kv heads,
d_head 128, 28 layers), 32K context, batch 128 per GPU, HBM cache holding 25% of the KV blocks
(128 slots per sequence and head), rest in pinned host memory, high-locality AR(1) query stream.

Under torchrun each rank owns its own batch shard, host KV pool and PCIe link (no data-path
collective; one barrier + max-over-ranks timing reduce).  `--impl reference` times the
reference CPU algorithm (the oracle port, oracle/nosa_oracle.py) on the host cores instead.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "batched decode tokens/s at 32K ctx w/ KV offload; H2D miss GB/s; % roofline"

# AttentionConfig fields of the two attention shapes (config.one_b_config / cfg1_config), kept as
# plain dicts so the reference arm never imports the package (which loads libnosa_b200.so)
SHAPES = {
    "cfg1": dict(n=16384, d=1024, n_head=8, n_kv_head=2, d_head=128, n_b=64, n_s=64, n_w=512, k=1024, k_q=256,
                 k_e=768, accounting="exclusive"),
    "1b": dict(n=65536 + 4096, d=2048, n_head=16, n_kv_head=2, d_head=128, n_b=64, n_s=64, n_w=1024, k=4096,
               k_q=1024, k_e=3072, accounting="inclusive"),
}


def shape_text(c: dict) -> str:
    return (f"{c['n_head']} q / {c['n_kv_head']} kv heads, d_head {c['d_head']}, block {c['n_b']}, sink {c['n_s']}, "
            f"window {c['n_w']}, k {c['k']}, k_q {c['k_q']}, k_e {c['k_e']}, {c['accounting']} accounting")


def load_path(name: str, rel: str):
    """A pure-Python module of the package loaded by file path: no package __init__, so no
    libnosa_b200.so (the reference arm and the CPU legs use the input generator this way)."""
    import importlib.util
    if name in sys.modules:
        return sys.modules[name]
    spec = importlib.util.spec_from_file_location(name, ROOT / rel)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod  # (dataclasses look their module up here)
    spec.loader.exec_module(mod)
    return mod

WORKLOADS = {
    "cfg1": dict(desc="single NOSA sparse-attention decode layer, batch 4, 8q/2kv, d128, 8K ctx, block 64, top-k 16",
                 shape="cfg1", layers=1, batch=4, context=8192, cache="resident", rho=0.95),
    "cfg2": dict(desc="1B-class shape, 28 layers, batch 32, 16K ctx, all KV resident in HBM, high locality",
                 shape="1b", layers=28, batch=32, context=16384, cache="resident", rho=0.95),
    "cfg3": dict(desc="1B-class shape, 28 layers, 32K ctx, batch 128, HBM cache = 25% of KV blocks, rest pinned host",
                 shape="1b", layers=28, batch=128, context=32768, cache=0.25, rho=0.95),
    "cfg4": dict(desc="1B-class shape, 28 layers, 32K ctx, batch 128, 25% HBM cache, adversarial random queries (rho=0)",
                 shape="1b", layers=28, batch=128, context=32768, cache=0.25, rho=0.0),
    "cfg5": dict(desc="1B-class shape, 64K ctx, batch 512 total batch-sharded over GPUs, 25% HBM cache, per-GPU host pools",
                 shape="1b", layers=28, batch=512, context=65536, cache=0.25, rho=0.95, strong=True,
                 burn_in=128,  # 256 slots over a 1007-block pool: the miss rate settles after ~100 steps
                 parity_steps=72, parity_pairs=3),  # the parity sample reaches the first evictions
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg3")
    ap.add_argument("--selector", choices=["nosa", "infllmv2"], default="nosa")
    ap.add_argument("--dtype", choices=["bf16", "fp32"], default="bf16",
                    help="KV / query storage: bf16 (tensor-core attention) or fp32 (the 1e-5 parity path)")
    ap.add_argument("--layers", type=int, default=None, help="override (for quick local checks only)")
    ap.add_argument("--batch", type=int, default=None, help="override (for quick local checks only)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--gather", choices=["auto", "uva", "tma", "memcpy", "hostpack", "hybrid"], default="auto",
                    help="auto = copy-engine batches when blocks are offloaded, graph-replayed UVA otherwise")
    ap.add_argument("--schedule", choices=["pipelined", "serial"], default="pipelined")
    ap.add_argument("--burn-in", type=int, default=None,
                    help="untimed decode steps before the warm-up so the HBM cache is in steady state "
                         "(default 32; 128 for cfg5)")
    ap.add_argument("--cpu-pairs", type=int, default=None,
                    help="(sequence, layer) pairs in the CPU baseline / parity sample (default 6)")
    ap.add_argument("--parity-steps", type=int, default=None,
                    help="first decode steps replayed through the oracle for the CPU baseline and the parity "
                         "check (default: the burn-in + warm-up, at most 40; 72 for cfg5)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--trace-out", default=None, help="write the device timeline of one instrumented step here")
    ap.add_argument("--report-dir", default=None,
                    help="also write the run as a reference sim-report (sim_report.json / .csv) into this directory")
    ap.add_argument("--slow-tier", default="host",
                    help="'host' (pinned host memory over PCIe) or 'peer' (another GPU's HBM over NVLink: "
                         "device (local_rank + 1) %% GPUs on the node, the own device when alone = loopback)")
    ap.add_argument("--per-step", action="store_true", help="print each timed step's ms to stderr (diagnostics)")
    ap.add_argument("--inputs", choices=["qkv", "hidden"], default="qkv",
                    help="qkv: the step's q/k/v are given (BASELINE's synthetic Q/K/V); hidden: hidden states "
                         "h [layers][batch][d] with per-layer random projections, q/k/v projected on the tensor "
                         "cores inside the step (DecodeEngine.step(h_t) at batch scale)")
    ap.add_argument("--eager", action="store_true",
                    help="launch every kernel from the host instead of replaying the captured step graph")
    a = ap.parse_args()
    if a.burn_in is None:
        a.burn_in = WORKLOADS[a.workload].get("burn_in", 32)
    if a.cpu_pairs is None:
        a.cpu_pairs = WORKLOADS[a.workload].get("parity_pairs", 6)
    if a.parity_steps is None:
        a.parity_steps = WORKLOADS[a.workload].get("parity_steps", 40)
    a.parity_steps = min(a.parity_steps, a.burn_in + a.warmup)
    return a


def attention_config(shape):
    from paper_2510_13602_b200 import AttentionConfig
    return AttentionConfig(**SHAPES[shape])


def token_budget(args, w) -> tuple[int, int, int]:
    """(max_tokens, blocks per (sequence, head), fast slots) of a run: both arms size the cache
    the same way, so the reference arm decodes the identical configuration."""
    total_steps = args.burn_in + args.warmup + args.steps * (2 if args.no_e2e else 3)
    max_tokens = w["context"] + total_steps + 8  # + the device-clock pass, e2e graph warm-up, traced step
    nblk = -(-max_tokens // SHAPES[w["shape"]]["n_b"])
    fast = nblk if w["cache"] == "resident" else int(w["cache"] * nblk)
    return max_tokens, nblk, fast


def bench_config(args, w, world) -> dict:
    """The `config` object of the JSON line, identical for the native and the reference arm."""
    _, nblk, fast = token_budget(args, w)
    return {"workload": f"{args.workload}: {w['desc']}", "attention_shape": shape_text(SHAPES[w["shape"]]),
            "global_batch": w["global_batch"], "seq_len": w["context"], "layers": w["layers"],
            "selector": args.selector, "rho": w["rho"], "fast_slots_per_seq_head": fast, "blocks_per_seq_head": nblk,
            "parallelism": f"dp{world} (batch-sharded, no data-path collective)",
            "inputs": f"counter-based synthetic q / k_new / v_new and prefix K/V (seed {args.seed}), identical bits "
                      f"on the GPU and in the CPU oracle",
            "kv_storage": getattr(args, "dtype", "bf16"),
            "host_memory_limited_batch": w["host_limited"],
            "l2": "no flush needed: attended KV per layer-step exceeds the 126 MB L2"}


def elem_bytes(args) -> int:
    return 4 if getattr(args, "dtype", "bf16") == "fp32" else 2


def workload_dims(args, world):
    w = dict(WORKLOADS[args.workload])
    if args.layers:
        w["layers"] = args.layers
    if args.batch:
        w["batch"] = args.batch
    shard_batch = load_path("nosa_dist", "paper_2510_13602_b200/dist.py").shard_batch
    rank = int(os.environ.get("RANK", "0"))
    shard = shard_batch(w["batch"], world, rank, bool(w.get("strong")))
    w["batch_local"], w["global_batch"], w["seq0"] = shard.seq_count, shard.global_batch, shard.seq_begin
    w["host_limited"] = False
    if args.impl == "native" and args.slow_tier == "peer":  # slow tier + cache + K_c must fit in HBM
        import torch
        n_blocks = -(-(w["context"] + 256) // 64)
        frac = 1.0 if w["cache"] == "resident" else 1.0 + w["cache"]
        per_seq = w["layers"] * 2 * n_blocks * (2 * 64 * 128 * elem_bytes(args) * frac + 128 * 10)
        budget = int(0.55 * torch.cuda.get_device_properties(0).total_memory)
        if per_seq * w["batch_local"] > budget:
            w["batch_local"] = max(1, budget // int(per_seq))
            w["global_batch"] = w["batch_local"] * world
            w["host_limited"] = True
    elif args.slow_tier != "peer":  # the pinned slow tier of every rank on this node must fit in RAM
        # (the reference arm sizes the same way, so both arms name the same batch)
        local = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
        n_blocks = -(-(w["context"] + 256) // 64)
        per_seq = w["layers"] * 2 * n_blocks * 2 * 64 * 128 * elem_bytes(args)  # [layers][kv heads][blocks] x 32 KiB
        avail = host_mem_available()
        budget = int(0.8 * avail / local) if avail else None
        if budget is not None and per_seq * w["batch_local"] > budget:
            fit = max(1, budget // per_seq)
            print(f"bench: host RAM {avail / 2**30:.0f} GiB for {local} ranks holds {fit} of "
                  f"{w['batch_local']} sequences per rank; batch reduced", file=sys.stderr)
            w["batch_local"] = fit
            w["global_batch"] = fit * world
            w["host_limited"] = True
    if world > 1 and args.impl == "native":  # every rank runs the smallest shard any rank fits
        import torch
        import torch.distributed as dist
        if dist.is_initialized():
            dev = (torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))) if dist.get_backend() == "nccl"
                   else torch.device("cpu"))
            t = torch.tensor([w["batch_local"], int(w["host_limited"])], dtype=torch.int64, device=dev)
            dist.all_reduce(t[:1], op=dist.ReduceOp.MIN)
            dist.all_reduce(t[1:], op=dist.ReduceOp.MAX)
            if not w.get("strong") or int(t[1]):
                w["batch_local"], w["host_limited"] = int(t[0]), bool(t[1])
                w["global_batch"] = w["batch_local"] * world
                w["seq0"] = rank * w["batch_local"]
    return w


def host_mem_available() -> int | None:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return None


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and throttle reasons polled through NVML every 20 ms during the timed region
    (the same counters `nvidia-smi --query-gpu=clocks.sm,clocks_event_reasons.*` reports)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index):
        self.index, self.rows, self.stop = index, [], threading.Event()

    def __enter__(self):
        if os.environ.get("NOSA_BENCH_NO_CLOCKS"):  # diagnostics: no sampling thread
            self.nvml = None
            return self
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception as exc:  # NVML missing: report unsampled rather than guess
            self.nvml, self.err = None, str(exc)
        return self

    def _poll(self):
        n = self.nvml
        while not self.stop.is_set():
            try:
                sm = n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM)
                mask = n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, mask))
            except Exception:
                pass
            self.stop.wait(float(os.environ.get("NOSA_CLOCK_POLL_S", "0.02")))

    def __exit__(self, *exc):
        self.stop.set()
        if getattr(self, "nvml", None):
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({name for _, m in self.rows for bit, name in self.REASONS.items() if m & bit})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.max_sm,
                "reasons": reasons, "samples": len(self.rows), "source": "NVML, 20 ms polling"}


class PcieSampler:
    """Hardware PCIe throughput during the timed region: NVML's per-device PCIe counters
    (nvmlDeviceGetPcieThroughput, each call integrates a 20 ms window; RX = bytes the GPU
    receives, i.e. host -> device; the same counters as `nvidia-smi dmon -s t`).  Independent of
    the bench's own byte accounting, so it checks the H2D figure the step roofline is built on."""

    def __init__(self, index):
        self.index, self.rx, self.tx, self.stop = index, [], [], threading.Event()

    def __enter__(self):
        self.nvml = None
        if os.environ.get("NOSA_BENCH_NO_CLOCKS"):
            return self
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception as exc:
            self.nvml, self.err = None, str(exc)
        return self

    def _poll(self):
        n = self.nvml
        while not self.stop.is_set():
            try:  # KB/s over the call's 20 ms window
                self.rx.append(n.nvmlDeviceGetPcieThroughput(self.h, n.NVML_PCIE_UTIL_RX_BYTES) * 1e3 / 1e9)
                self.tx.append(n.nvmlDeviceGetPcieThroughput(self.h, n.NVML_PCIE_UTIL_TX_BYTES) * 1e3 / 1e9)
            except Exception:
                return

    def __exit__(self, *exc):
        self.stop.set()
        if self.nvml:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rx:
            return None
        return {"rx_h2d_gbs_median": round(statistics.median(self.rx), 2), "rx_h2d_gbs_max": round(max(self.rx), 2),
                "tx_d2h_gbs_median": round(statistics.median(self.tx), 2), "samples": len(self.rx),
                "source": "NVML nvmlDeviceGetPcieThroughput (device PCIe counters, 20 ms windows) during the "
                          "timed region"}


# ------------------------------------------------------------------------------ native arm
def measure_link_gbs(torch, device, src_device=None):
    """Best of 10 1 GiB copies into `device`: from pinned host memory, or from `src_device`'s HBM
    (the peer slow tier; the same device = a local HBM copy)."""
    if src_device is None:
        x = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    else:
        x = torch.empty(1 << 30, dtype=torch.uint8, device=torch.device("cuda", src_device))
    y = torch.empty(1 << 30, dtype=torch.uint8, device=device)
    for _ in range(2):
        y.copy_(x, non_blocking=True)
    torch.cuda.synchronize(device)
    best = 0.0
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); y.copy_(x, non_blocking=True); b.record(); b.synchronize()
        best = max(best, (1 << 30) / (a.elapsed_time(b) * 1e-3) / 1e9)
    del x, y
    return best


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], "measured"
    return 6650.0, "fallback"


def run_native(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2510_13602_b200 import NosaEngine, synth, workload
    from paper_2510_13602_b200.dist import max_over_ranks, rank_seed

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    from paper_2510_13602_b200.dist import bind_to_gpu_numa_node
    numa_node = bind_to_gpu_numa_node(local_rank)  # before the pinned slow tier is allocated
    w = workload_dims(args, world)
    if args.gather == "auto":  # the device-driven SM gather: the whole step replays as one CUDA graph
        args.gather = "uva"
    cfg = attention_config(w["shape"])
    L, B, ctx_len, seq0 = w["layers"], w["batch_local"], w["context"], w["seq0"]
    max_tokens, nblk, fast = token_budget(args, w)
    dtype = torch.float32 if args.dtype == "fp32" else torch.bfloat16
    if args.dtype == "fp32" and args.inputs == "hidden":
        raise SystemExit("bench: --inputs hidden projects in bf16 on the tensor cores; use --dtype bf16")
    peer_dev = None
    if args.slow_tier == "peer":  # the slow tier in another GPU's HBM (alone on the box: loopback)
        ngpu = torch.cuda.device_count()
        peer_dev = (local_rank + 1) % ngpu if ngpu > 1 else local_rank
        slow_tier = f"peer:{peer_dev}"
    else:
        slow_tier = "host"
    link_gbs = measure_link_gbs(torch, device, peer_dev)

    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, args.seed)
    t_setup = time.time()
    # strong scaling splits a fixed global batch: pin the split-K chunk (the automatic one follows
    # the local batch) so every sequence's outputs are bit-identical at 1, 2, 4 and 8 GPUs
    chunk = 8 if w.get("strong") else 0
    eng = NosaEngine(cfg, batch=B, layers=L, max_tokens=max_tokens, fast_slots=fast, w1=w1, w2=w2, dtype=args.dtype,
                     device=local_rank, slow_tier=slow_tier, attend_chunk=chunk)
    t_alloc = time.time() - t_setup
    # inputs: counter-based draws addressed by GLOBAL sequence id (a rank's shard draws the same
    # bits a single GPU would), reproduced exactly by the CPU oracle (workload.synth_*)
    for l in range(L):
        k, v = synth.prefix_kv(args.seed, l, seq0, B, cfg.n_kv_head, ctx_len, cfg.d_head, device, dtype)
        eng.prefill(k, v, layer=l, resident=w["cache"] == "resident")
        del k, v
    eng.start_run()
    torch.cuda.synchronize(device)
    t_prefill = time.time() - t_setup - t_alloc

    hidden = args.inputs == "hidden"
    if hidden:  # AR(1) hidden states through random per-layer projections (q keeps the 1/d_head scale)
        import numpy as np
        seed_base = rank_seed(args.seed, rank)
        prng = np.random.default_rng(seed_base + 4242)
        for l in range(L):
            eng.set_projection(l, prng.standard_normal((cfg.d, cfg.n_head * cfg.d_head)) / np.sqrt(cfg.d * cfg.d_head),
                               prng.standard_normal((cfg.d, cfg.n_kv_head * cfg.d_head)) / np.sqrt(cfg.d),
                               prng.standard_normal((cfg.d, cfg.n_kv_head * cfg.d_head)) / np.sqrt(cfg.d))
        stream = workload.TorchHiddenStream(seed_base + 99991, L, B, cfg.d, w["rho"], device, dtype)
    else:
        stream = synth.GpuQueryStream(args.seed, L, seq0, B, cfg.n_head, cfg.n_kv_head, cfg.d_head, w["rho"], device,
                                      dtype)
    out = torch.empty((L, B, cfg.n_head, cfg.d_head), dtype=torch.float32, device=device)

    def do_step(inp, check=True):
        """One decode step of every layer on device inputs: (q, k_new, v_new) or (h,)."""
        if hidden:
            eng.step_hidden(inp[0], selector=args.selector, out=out, gather=args.gather, check=check,
                            schedule=args.schedule)
        else:
            eng.step(*inp, selector=args.selector, out=out, gather=args.gather, check=check, schedule=args.schedule)
    # residency burn-in (the HBM cache fills to its steady state), then the W warm-up steps; for a
    # random sample of (layer, sequence) pairs the first parity_steps steps' inputs, outputs,
    # selections and cache plans are recorded for the oracle replay (CPU baseline + parity)
    import numpy as np
    prng_pairs = np.random.default_rng(5)
    pairs = [] if hidden or rank != 0 or world != 1 or args.no_cpu_baseline else \
        sorted({(int(prng_pairs.integers(L)), int(prng_pairs.integers(B))) for _ in range(args.cpu_pairs)})
    rec = {p: [] for p in pairs}
    for i in range(args.burn_in + args.warmup):
        inp = stream.next()
        do_step(inp)
        if i < args.parity_steps and pairs:
            for l in sorted({p[0] for p in pairs}):
                bq, nq, be, ne, rq, nr, _ = eng.raw_selection(l)
                plans = eng.plans(l)
                o = out[l].cpu().numpy()
                for (pl, b) in pairs:
                    if pl != l:
                        continue
                    H = cfg.n_kv_head
                    rec[(l, b)].append(dict(
                        inputs=tuple(x[l, b].float().cpu().numpy() for x in inp), out=o[b].copy(),
                        blocks_q=[bq[b, h, :nq[b, h]].tolist() for h in range(H)],
                        blocks_e=[be[b, h, :ne[b, h]].tolist() for h in range(H)],
                        required=[rq[b, h, :nr[b, h]].tolist() for h in range(H)],
                        fetch=[plans[b][h].fetch for h in range(H)], evict=[plans[b][h].evict for h in range(H)],
                        hits=[plans[b][h].hits for h in range(H)]))
    # K steps for the clean timed region, K for the instrumented pass, K for the e2e pass
    # K steps for the timed region, K for the instrumented pass, then (e2e) one warm-up + K, all
    # consecutive in the query stream
    inputs = [stream.next() for _ in range(args.steps * 2 + (0 if args.no_e2e else args.steps + 1))]
    torch.cuda.synchronize(device)
    eng.reset_stats()
    use_graph = args.gather not in ("memcpy", "hostpack", "hybrid") and not args.eager
    if use_graph:  # the whole step as one CUDA graph on fixed buffers, fed by D2D copies
        gbufs = tuple(torch.empty_like(x) for x in inputs[0])
        if hidden:
            eng.capture_hidden(gbufs[0], out, selector=args.selector, gather=args.gather, schedule=args.schedule)
        else:
            eng.capture(*gbufs, out, selector=args.selector, gather=args.gather, schedule=args.schedule)

    step_events = []

    def run_steps(batch_inputs, per_step=False):
        for inp in batch_inputs:
            if per_step:
                step_events.append(torch.cuda.Event(enable_timing=True))
                step_events[-1].record()
            if use_graph:
                for buf, x in zip(gbufs, inp):
                    buf.copy_(x)
                eng.replay()
            else:
                do_step(inp, check=False)

    # ---------------- timed region (value): inputs resident in HBM, no instrumentation
    eng.timing_enable(0)
    launches0 = eng.launch_count
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(device)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks, PcieSampler(local_rank) as pcie:
        ev0.record()
        run_steps(inputs[:args.steps], per_step=args.per_step)
        ev1.record()
        torch.cuda.synchronize(device)
    if args.per_step:
        marks = step_events + [ev1]
        print("per-step ms:", [round(a.elapsed_time(b), 3) for a, b in zip(marks, marks[1:])], file=sys.stderr)
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = eng.launch_count - launches0
    eng.check_errors()
    st = eng.residency_stats()
    ms_max = max_over_ranks(ms, device)  # the slowest rank bounds the whole job
    tokens = w["global_batch"] * args.steps

    # ---------------- instrumented pass: the next K steps with every kernel bracketed by CUDA
    # events on its own stream (event nodes inside the graph); gives the per-kernel durations
    eng.reset_stats()
    eng.timing_enable(4 * L * args.steps + 8)
    ei0, ei1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ei0.record()
    run_steps(inputs[args.steps:2 * args.steps])
    ei1.record()
    torch.cuda.synchronize(device)
    kern = eng.timing_read()
    if args.trace_out:  # device timeline of the last instrumented step (one line per kernel)
        tr = eng.timing_trace()
        last = tr[-(len(tr) // args.steps):]
        base, seen = min(x[1] for x in last), {}
        with open(args.trace_out, "w") as f:
            f.write("kind layer start_us end_us dur_us\n")
            for k, s0, s1 in last:
                seen[k] = seen.get(k, -1) + 1
                f.write(f"{k} {seen[k]} {1000 * (s0 - base):.1f} {1000 * (s1 - base):.1f} {1000 * (s1 - s0):.1f}\n")
    st_i = eng.residency_stats()
    instrumented_ms = ei0.elapsed_time(ei1) / args.steps
    eng.timing_enable(0)
    inputs_e2e = inputs[2 * args.steps + 1:]

    # ---------------- end to end: host inputs H2D + step + D2H of the outputs, every step
    e2e = None
    if not args.no_e2e:
        def pinned(x):  # page-locked buffer from cudaHostAlloc (torch's pin_memory() path is slower)
            h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
            h.copy_(x)
            return h
        host_in = [tuple(pinned(x) for x in step_in) for step_in in inputs_e2e]
        host_out = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
        if world > 1:
            dist.barrier()
        warm = tuple(pinned(x) for x in inputs[2 * args.steps])  # untimed first host-buffer step
        if hidden:  # hidden states: each group's rows staged inside the step, outputs back per batch
            e2e_step = lambda hin: eng.step_hidden_host(hin[0], selector=args.selector, out=host_out,
                                                        gather=args.gather, schedule=args.schedule, sync=False)
        elif use_graph:  # the host-buffer step as a CUDA graph, re-pointed at each step's buffers;
            # the warm-up replay uploads the new executable graph
            eng.capture_host(*host_in[0], host_out, selector=args.selector, gather=args.gather,
                             schedule=args.schedule)
            e2e_step = lambda hin: eng.replay_host(*hin, host_out)
        else:  # the host-buffer C ABI call: inputs staged and outputs copied back inside the step
            e2e_step = lambda hin: eng.step_host(*hin, selector=args.selector, out=host_out, gather=args.gather,
                                                 schedule=args.schedule, sync=False)
        e2e_step(warm)
        eng.reset_stats()  # the e2e pass's own miss traffic is reported beside its rate
        torch.cuda.synchronize(device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        e2e_marks, e2e_host = [], []
        for hin in host_in:
            if args.per_step:
                e2e_marks.append(torch.cuda.Event(enable_timing=True))
                e2e_marks[-1].record()
                e2e_host.append(time.perf_counter())
            e2e_step(hin)
        e1.record()
        torch.cuda.synchronize(device)
        if args.per_step:
            marks = e2e_marks + [e1]
            print("e2e per-step ms:", [round(a.elapsed_time(b), 3) for a, b in zip(marks, marks[1:])],
                  "host enqueue ms:", [round(1e3 * (b - a), 3) for a, b in zip(e2e_host, e2e_host[1:])], file=sys.stderr)
        e_ms = max_over_ranks(e0.elapsed_time(e1), device)
        st_e = eng.residency_stats()
        h2d = sum(x.numel() * x.element_size() for x in host_in[0])
        e2e = {"value": round(tokens / (e_ms * 1e-3), 2), "unit": "tokens/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": host_out.numel() * 4,
               "miss_bytes_per_step": int((st_e.misses - st_e.new_blocks) * eng.bytes_per_block / args.steps),
               "ms_per_step": round(e_ms / args.steps, 4),
               "api": ("NosaEngine.step_hidden_host (C ABI nosa_decode_step_hidden_host: h staged per selection "
                       "group by an SM zero-copy kernel, outputs copied back per attention batch)" if hidden else
                       "NosaEngine.capture_host/replay_host (C ABI nosa_step_graph_launch_host)" if use_graph else
                       "NosaEngine.step_host (C ABI nosa_decode_step_host: q/k/v staged per selection group by "
                       "an SM zero-copy kernel, outputs copied back per attention batch while later layers run)") +
                      " on inputs in pinned host memory"}
        eng.check_errors()
        if args.trace_out and not hidden:  # one more host-buffer step, instrumented, for the timeline
            eng.timing_enable(8 * L + 8)
            hq, hk, hv = (pinned(x) for x in stream.next())  # fresh queries: real misses
            eng.step_host(hq, hk, hv, selector=args.selector, out=host_out, gather=args.gather,
                          schedule=args.schedule)
            tr = eng.timing_trace()
            base, seen = min(x[1] for x in tr), {}
            with open(args.trace_out + ".e2e", "w") as f:
                f.write("kind layer start_us end_us dur_us\n")
                for k, s0, s1 in tr:
                    seen[k] = seen.get(k, -1) + 1
                    f.write(f"{k} {seen[k]} {1000 * (s0 - base):.1f} {1000 * (s1 - base):.1f} {1000 * (s1 - s0):.1f}\n")
            eng.timing_enable(0)

    # device-clock span of the attention launches (diagnostic, untimed, after the e2e pass so the
    # query stream stays in order): first CTA start to last
    # CTA end, read back after each step; the event-timed launch also holds the launch latency
    # after the cross-stream wait on the layer's miss transfer
    eng.ktime_enable(True)
    spans = []
    for _ in range(3):  # eager launches (a captured graph holds the pre-diagnostic kernel arguments)
        do_step(stream.next(), check=False)
        spans += [x for x in eng.ktime_read() if x > 0]
    eng.ktime_enable(False)
    attend_exec_ms = statistics.mean(spans) * 1e-3 if spans else None

    # ---------------- roofline arithmetic (algorithmic bytes, SURVEY.md §8d / DESIGN.md)
    hbm_peak, peak_kind = peaks()
    bpb = eng.bytes_per_block
    calls = L * args.steps  # launches per kernel kind in the instrumented pass
    R_total = st.hits + st.misses                     # attended blocks, summed (timed region)
    R_inst = st_i.hits + st_i.misses                  # the same over the instrumented pass
    P = eng.geometry[0].pool_blocks.stop - eng.geometry[0].pool_blocks.start
    per_launch = {
        # K1+K2: screened pool scan (bf16 K_c + the f32 rounding-error bound per row) + f64 rows of
        # the candidates + q read (reads of required-list metadata are small); exact scan: f64 K_c
        "select_plan": ((B * cfg.n_kv_head * P * (cfg.d_head * 2 + 4) + st_i.candidates * cfg.d_head * 8 / calls)
                        if eng.screened else B * cfg.n_kv_head * P * cfg.d_head * 8) + B * cfg.n_head * cfg.d_head * 2,
        # K3: each missed block crosses PCIe once and is written to HBM once
        "gather": (st_i.misses - st_i.new_blocks) * bpb / calls,
        # K4: K|V of every attended block + its bias + the query rows
        "attend": (R_inst * (bpb + 4)) / calls + B * cfg.n_head * cfg.d_head * 2,
        # K4 merge + K5: f32 outputs + the appended K/V row (HBM slot)
        "finalize": B * cfg.n_head * cfg.d_head * 4 + B * cfg.n_kv_head * 2 * cfg.d_head * 2,
        # projection (hidden inputs): the layer's bf16 weights, its hidden states, its q/k/v
        "project": ((cfg.n_head + 2 * cfg.n_kv_head) * cfg.d_head * (cfg.d + B) * 2 + B * cfg.d * 2),
    }
    for k_ in kern:  # per_launch holds bytes per layer; selection may cover several layers per launch
        kern[k_]["bytes_per_launch"] = per_launch[k_] * calls / max(kern[k_]["launches"], 1)
        kern[k_]["gbs"] = per_launch[k_] * calls / (kern[k_]["total_ms"] * 1e-3) / 1e9 if kern[k_]["total_ms"] else None
    traffic = None
    tpath = ROOT / "profiles" / "traffic.json"
    if tpath.exists():
        traffic = json.loads(tpath.read_text()).get(f"{args.workload}:attend" + ("" if args.dtype == "bf16" else ":fp32"))
    att = kern["attend"]
    roofline = {"bound": "hbm", "kernel": "attend_f32_kernel (K4+K5, fp32 CUDA cores)" if args.dtype == "fp32" else
                "attend_bf16_kernel (K4+K5)", "achieved": round(att["gbs"], 1),
                "peak": hbm_peak, "unit": "GB/s", "frac": round(att["gbs"] / hbm_peak, 4), "traffic": traffic,
                "peak_kind": peak_kind, "bytes_per_launch": int(per_launch["attend"]),
                "avg_launch_ms": round(att["avg_ms"], 5),
                "device_clock": None if attend_exec_ms is None else {
                    "exec_span_ms": round(attend_exec_ms, 5),
                    "achieved": round(per_launch["attend"] * calls / max(att["launches"], 1) / (attend_exec_ms * 1e-3) / 1e9, 1),
                    "frac": round(per_launch["attend"] * calls / max(att["launches"], 1) / (attend_exec_ms * 1e-3) / 1e9 / hbm_peak, 4),
                    "note": "first CTA start to last CTA end (%globaltimer), 3 untimed steps; the event-timed "
                            "launch above also holds the dependency-resolution and launch latency"}}
    # step-level bytes from the uninstrumented timed region; blocks born by an append are rebuilt
    # on the device and never cross PCIe (the reference still counts them as misses)
    h2d_step = (st.misses - st.new_blocks) * bpb / args.steps
    hbm_step = (per_launch["select_plan"] + per_launch["finalize"]) * L + \
        (R_total * (bpb + 4) / args.steps + L * B * cfg.n_head * cfg.d_head * 2) + h2d_step
    if hidden:  # + the projection: every layer's bf16 weights, hidden states in, q/k/v out
        n_qkv = (cfg.n_head + 2 * cfg.n_kv_head) * cfg.d_head
        hbm_step += L * (n_qkv * cfg.d * 2 + B * cfg.d * 2 + B * n_qkv * 2)
    t_roof = max(hbm_step / 8e12, h2d_step / (link_gbs * 1e9))
    step_ms = ms_max / args.steps
    g = kern["gather"]
    gather_name = {"uva": "gather_kernel (K3, UVA zero-copy SM loads)", "tma": "gather_tma_kernel (K3, TMA bulk)",
                   "memcpy": "cudaMemcpyAsync per block (K3, copy engine)",
                   "hostpack": "host-packed 2 MiB chunks, one DMA each + scatter_kernel (K3, copy engine)",
                   "hybrid": "host-packed DMAs + gather_kernel (K3, copy engine and SM loads)"}[args.gather]
    link_roofline = {"bound": "pcie-h2d" if peer_dev is None else "peer-hbm", "kernel": gather_name,
                     "achieved": round(g["gbs"], 2) if g["gbs"] else 0.0, "peak": round(link_gbs, 2), "unit": "GB/s",
                     "frac": round(g["gbs"] / link_gbs, 4) if g["gbs"] else 0.0,
                     "peak_kind": ("measured pinned 1 GiB H2D cudaMemcpyAsync, best of 10" if peer_dev is None else
                                   f"measured 1 GiB device {peer_dev} -> {local_rank} cudaMemcpyAsync, best of 10")}
    step_roofline = {"definition": "t_roof = max(HBM bytes / 8 TB/s, H2D miss bytes / measured link GB/s)",
                     "hbm_bytes_per_step": int(hbm_step), "h2d_bytes_per_step": int(h2d_step),
                     "t_roof_ms": round(t_roof * 1e3, 4), "t_step_ms": round(step_ms, 4),
                     "frac": round(t_roof * 1e3 / step_ms, 4),
                     "bound": "h2d" if h2d_step / (link_gbs * 1e9) > hbm_step / 8e12 else "hbm",
                     "frac_at_measured_hbm": round(max(hbm_step / (hbm_peak * 1e9), h2d_step / (link_gbs * 1e9))
                                                   * 1e3 / step_ms, 4)}

    # ---------------- the run as a reference SimReport row (offload_sim.py:175-192; cli.py:214-218)
    from paper_2510_13602_b200 import reports
    from paper_2510_13602_b200.dist import sum_over_ranks
    from paper_2510_13602_b200.engine import ResidencyStats
    tot = sum_over_ranks([st.hits, st.misses, st.bytes_up, st.bytes_down, st.topk_required, st.topk_misses], device)
    st_all = ResidencyStats(hits=int(tot[0]), misses=int(tot[1]), bytes_up=int(tot[2]), bytes_down=int(tot[3]),
                            topk_required=int(tot[4]), topk_misses=int(tot[5]))
    sim = reports.row_dict(reports.report_from_run(
        selector=args.selector, resident=w["cache"] == "resident", batch=w["global_batch"], context=ctx_len,
        steps=args.steps, seed=args.seed, stats=st_all, tokens_per_s=tokens / (ms_max * 1e-3),
        attn_ms_per_step=kern["attend"]["total_ms"] / args.steps, ms_per_step=step_ms,
        fast_slots_per_seq=fast, config=cfg.to_dict()))
    if args.report_dir and rank == 0:
        reports.write_sim_report([sim], args.report_dir,
                                 params={"measured": True, "link_gbs": link_gbs, "hbm_gbs": hbm_peak,
                                         "layers": L, "workload": args.workload})

    # ---------------- CPU baseline: the oracle (reference algorithm) on a bounded sample
    cpu, parity = None, None
    if pairs:
        cpu, parity = cpu_baseline_sample(args, cfg, w, rec, device, fast, max_tokens)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(tokens / (ms_max * 1e-3), 2), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 4),
            "higher_is_better": True, "scaling": "strong" if w.get("strong") else "weak", "vs_baseline": None,
            "dtype": args.dtype,
            "data": (f"synthetic: K/V ~ N(0,1) bf16 (counter-based), AR(1) hidden states rho={w['rho']} through "
                     f"random per-layer projections (torch Philox / numpy PCG64, seed {args.seed})" if hidden else
                     f"synthetic: K/V ~ N(0,1) {args.dtype}, AR(1) queries rho={w['rho']} (counter-based generator, seed "
                     f"{args.seed}: the same bits on the GPU and in the CPU oracle)"),
            "config": bench_config(args, w, world),
            "run": {"gather": args.gather, "schedule": args.schedule, "burn_in_steps": args.burn_in,
                    "cuda_graph": use_graph,
                    "inputs": ("hidden states [layers][batch][d], QKV projection (tcgen05) inside the step"
                               if hidden else "q / k_new / v_new per layer"),
                    "kernel_timing": "instrumented pass: the K steps after the timed region with CUDA events "
                                     "around every kernel on its own stream (event nodes in the graph); "
                                     "value comes from the uninstrumented region",
                    "numa_node": numa_node, "seq_range": [seq0, seq0 + B],
                    "attend_chunk": chunk or "auto (from the local batch)",
                    "slow_tier": slow_tier + (" (loopback: the own HBM stands in for a peer)"
                                              if peer_dev == local_rank else "")},
            "parity": parity,
            "h2d_miss_gbs": round(h2d_step / (step_ms * 1e-3) / 1e9, 3),
            "hit_rate": round(st.hit_rate, 4),
            "sim_report": sim,
            "misses_per_seq_head_step": round(st.misses / (B * cfg.n_kv_head * L * args.steps), 3),
            "attended_blocks_per_seq_head": round(R_total / (B * cfg.n_kv_head * L * args.steps), 2),
            "selection": {"scan": "screened: bf16 K_c pre-scan with a proven error bound, f64 rescoring of "
                                  "the candidates (same picks as a full f64 scan)" if eng.screened else "full f64",
                          "pool_blocks": P,
                          "f64_rows_per_selection": round(st.candidates / (B * cfg.n_kv_head * L * args.steps), 2)},
            "link_gbs_measured": round(link_gbs, 2),
            "roofline": roofline, "link_roofline": link_roofline, "step_roofline": step_roofline,
            "kernels": {k_: {"avg_ms": round(v["avg_ms"], 5), "launches": v["launches"],
                             "gbs": round(v["gbs"], 2) if v["gbs"] else None} for k_, v in kern.items()},
            "instrumented_ms_per_step": round(instrumented_ms, 4),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks.summary(),
            "pcie_counters": pcie.summary(),
            "setup_s": {"alloc_and_pin": round(t_alloc, 1), "prefill": round(t_prefill, 1)},
        }
        print(json.dumps(line), flush=True)
    eng.close()


def cpu_baseline_sample(args, cfg, w, rec, device, fast, max_tokens):
    """Replay the recorded first steps of a few (layer, sequence) pairs through the oracle on one
    host core: the reference algorithm (attend_biased dense over every cached token, K re-pooled
    every step, TieredBlockManager with 32 KiB payload copies) on the identical inputs.  Times it
    (cpu_baseline) and compares every decision with the GPU's (parity): blocks_q, blocks_e,
    required, fetch (plan order), evict (LRR order), hits exactly; outputs within 2e-2 (bf16 storage) or
    1e-5 (fp32 storage)."""
    import numpy as np
    import torch

    from oracle import nosa_oracle as O
    from paper_2510_13602_b200 import synth, workload

    oc = O.OracleConfig.from_attention_config(cfg)
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, args.seed)
    L, H = w["layers"], cfg.n_kv_head
    worst, prefill_s, step_s, n_steps = 0.0, 0.0, 0.0, 0
    mism = {"blocks_q": 0, "blocks_e": 0, "required": 0, "fetch": 0, "evict": 0, "hits": 0}
    ties = evictions = fetches = 0
    for (l, b), steps in rec.items():
        k, v = synth.prefix_kv(args.seed, l, w["seq0"] + b, 1, H, w["context"], cfg.d_head, device,
                               torch.float32 if args.dtype == "fp32" else torch.bfloat16)
        k, v = k[0].float().cpu().numpy(), v[0].float().cpu().numpy()
        orc = O.OracleEngine(oc, 1, 1, max_tokens, fast, w1, w2, store_payload=True, dense=True)
        t0 = time.perf_counter()
        orc.prefill(0, 0, k, v)
        orc.start_run()
        if w["cache"] == "resident":
            for h in range(H):
                orc.managers[0][0].make_resident(h, -(-w["context"] // cfg.n_b))
        prefill_s += time.perf_counter() - t0
        for g in steps:
            q, kn, vn = g["inputs"]
            ts = time.perf_counter()
            ref, recs = orc.step_seq(0, 0, q, kn, vn, args.selector)
            step_s += time.perf_counter() - ts
            n_steps += 1
            worst = max(worst, float(np.max(np.abs(g["out"] - ref)) / np.max(np.abs(ref))))
            for h, r in enumerate(recs):
                for key, want in (("blocks_q", r.blocks_q.tolist()), ("blocks_e", r.blocks_e.tolist()),
                                  ("required", r.required), ("fetch", r.fetch), ("evict", r.evict), ("hits", r.hits)):
                    if g[key][h] != want:
                        if key in ("blocks_q", "blocks_e"):  # an exact score tie is reported, not a mismatch
                            sc = dict(zip(range(*orc.geom[0].pool), r.s_q if key == "blocks_q" else r.s_e_c))
                            if len({sc.get(x) for x in set(g[key][h]) ^ set(want)}) == 1:
                                ties += 1
                                continue
                        mism[key] += 1
                evictions += len(r.evict)
                fetches += len(r.fetch)
    per_pair_step = step_s / max(n_steps, 1)
    cpu = {"value": round(1.0 / (L * per_pair_step), 4), "unit": "tokens/s", "cores": 1, "kind": "port",
           "sample": f"{len(rec)} random (layer, sequence) pairs x their first {n_steps // max(len(rec), 1)} decode "
                     f"steps through the oracle (the reference algorithm: attend_biased dense over every cached token, "
                     f"K re-pooled every step, per-sequence TieredBlockManager with 32 KiB payload copies) on the "
                     f"same inputs, one host core; tokens/s = 1 / (layers x seconds per pair-step)",
           "seconds_per_pair_step": round(per_pair_step, 5), "prefill_seconds_per_pair": round(prefill_s / len(rec), 3)}
    parity = {"pairs": len(rec), "steps": n_steps // max(len(rec), 1), "heads_checked": n_steps * H,
              "sel_mismatch": mism["blocks_q"] + mism["blocks_e"], "required_mismatch": mism["required"],
              "fetch_mismatch": mism["fetch"], "evict_mismatch": mism["evict"], "hit_mismatch": mism["hits"],
              "ties_reported": ties, "fetches_checked": fetches, "evictions_checked": evictions,
              "max_rel_err": worst, "tolerance": 1e-5 if args.dtype == "fp32" else 2e-2,
              "what": "GPU vs oracle on identical inputs, every (step, head) of the sampled pairs: blocks_q, "
                      "blocks_e, required, fetch list, evict list, hits exactly; outputs max|o-o_ref|/max|o_ref|"}
    return cpu, parity


# ------------------------------------------------------------------------------ reference arm
def _ref_worker(conn, pairs, cfg_d, context, max_tokens, fast, resident, rho, seed, selector, bf16=True):
    """One host process of the reference arm: the oracle (the reference algorithm) for its
    (layer, global sequence) pairs, on the exact inputs the GPU arm decodes for those pairs."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import nosa_oracle as O
    wl = load_path("nosa_workload", "paper_2510_13602_b200/workload.py")
    oc = O.OracleConfig(**{k: cfg_d[k] for k in ("n_head", "n_kv_head", "d_head", "n_b", "n_s", "n_w", "k", "k_q",
                                                 "k_e", "accounting")})
    w1, w2 = wl.eviction_head(oc.n_head, oc.d_head, seed)
    units = []
    for (l, gb) in pairs:
        K, V = wl.synth_prefix_kv(seed, l, [gb], oc.n_kv_head, context, oc.d_head, bf16=bf16)
        orc = O.OracleEngine(oc, 1, 1, max_tokens, fast, w1, w2, store_payload=True, dense=True)
        orc.prefill(0, 0, K[0], V[0])
        orc.start_run()
        if resident:
            for h in range(oc.n_kv_head):
                orc.managers[0][0].make_resident(h, -(-context // oc.n_b))
        stream = wl.SynthQueryStream(seed, [l], [gb], oc.n_head, oc.n_kv_head, oc.d_head, rho, bf16=bf16)
        units.append((orc, stream))
        del K, V
    conn.send("ready")
    while True:
        cmd = conn.recv()
        if cmd == "stop":
            break
        for orc, stream in units:
            q, kn, vn = stream.next()
            orc.step_seq(0, 0, q[0, 0], kn[0, 0], vn[0, 0], selector)
        conn.send("done")


def run_reference(args, rank, world):
    """The reference arm: the reference's CPU algorithm (oracle/nosa_oracle.py, attend_biased dense
    over every cached token, re-pooled K, TieredBlockManager with payload copies; the reference
    package itself cannot travel to the GPU box) on this host's cores.  A step decodes `S` whole
    sequences of the workload through all layers, S chosen so the (layer, sequence) pairs spread
    evenly over the cores; the inputs are the GPU arm's, bit for bit.  Does not import the package."""
    import math
    import multiprocessing as mp

    if rank != 0:
        return
    w = workload_dims(args, world)
    cfg_d = SHAPES[w["shape"]]
    cores = len(os.sched_getaffinity(0))
    max_tokens, nblk, fast = token_budget(args, w)
    L = w["layers"]
    S = max(1, cores // math.gcd(cores, L))          # S x L pairs = a whole number of rounds per core
    per_pair = 2 * cfg_d["n_kv_head"] * max_tokens * cfg_d["d_head"] * 8 * 2   # oracle K, V (f64) + payloads
    S = max(1, min(S, w["global_batch"], int(0.25 * (host_mem_available() or 8 << 30) // (per_pair * L))))
    seqs = sorted(random_sample(w["global_batch"], S, args.seed))
    pairs = [(l, gb) for gb in seqs for l in range(L)]
    nproc = min(cores, len(pairs))
    ctx = mp.get_context("spawn")
    procs, conns = [], []
    t_setup = time.perf_counter()
    for i in range(nproc):
        a, b = ctx.Pipe()
        p = ctx.Process(target=_ref_worker, args=(b, pairs[i::nproc], cfg_d, w["context"], max_tokens, fast,
                                                  w["cache"] == "resident", w["rho"], args.seed, args.selector,
                                                  args.dtype == "bf16"),
                        daemon=True)
        p.start()
        procs.append(p)
        conns.append(a)
    for c in conns:
        assert c.recv() == "ready"
    setup_s = time.perf_counter() - t_setup

    def one_step():
        for c in conns:
            c.send("step")
        for c in conns:
            assert c.recv() == "done"

    for _ in range(args.warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step()
    dt = time.perf_counter() - t0
    for c in conns:
        c.send("stop")
    for p in procs:
        p.join(timeout=10)
    step_s = dt / args.steps
    value = S / step_s                       # tokens/s: S sequences advance one token per step
    sample = (f"each step decodes {S} of the {w['global_batch']} sequences (global ids {seqs}) through all {L} "
              f"layers: {len(pairs)} (layer, sequence) pairs over {nproc} host processes (multiprocessing, "
              f"OPENBLAS_NUM_THREADS=1), on the GPU arm's inputs for those pairs; sequences are independent, so "
              f"tokens/s does not depend on how many of the batch a step holds")
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_s * 1e3, 2),
            "higher_is_better": True, "scaling": "strong" if w.get("strong") else "weak", "vs_baseline": None,
            "dtype": "f64",
            "data": f"synthetic: K/V ~ N(0,1) {args.dtype}, AR(1) queries rho={w['rho']} (counter-based generator, seed "
                    f"{args.seed}: the same bits on the GPU and in the CPU oracle)",
            "config": bench_config(args, w, world),
            "sample_batch": S,
            "ms_per_full_step_extrapolated": round(step_s * 1e3 * w["global_batch"] / S, 1),
            "setup_s": round(setup_s, 1),
            "cpu_baseline": {"value": round(value, 4), "unit": "tokens/s", "cores": nproc, "kind": "port",
                             "sample": sample},
            "e2e": {"value": round(value, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def random_sample(n: int, k: int, seed: int) -> list[int]:
    """k distinct ids of range(n), seeded (pure Python: the reference arm imports no NumPy here)."""
    import random
    return random.Random(seed * 7 + 3).sample(range(n), min(k, n))


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_native(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
