"""Time replays of the host-buffer step graph: same buffers vs a new set each step (not product code)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2510_13602_b200 import NosaEngine, one_b_config, workload

dev = torch.device("cuda", 0)
cfg = one_b_config(65536)
B, L, T = 32, 28, 16384
max_tokens = T + 64
nblk = -(-max_tokens // 64)
w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, 0)
eng = NosaEngine(cfg, batch=B, layers=L, max_tokens=max_tokens, fast_slots=nblk, w1=w1, w2=w2)
for l in range(L):
    shape = (B, cfg.n_kv_head, T, cfg.d_head)
    eng.prefill(workload.torch_prefix_kv(2 * l, shape, dev, torch.bfloat16),
                workload.torch_prefix_kv(2 * l + 1, shape, dev, torch.bfloat16), layer=l, resident=True)
eng.start_run()
qs = workload.TorchQueryStream(7, L, B, cfg.n_head, cfg.n_kv_head, cfg.d_head, 0.95, dev, torch.bfloat16)
def pinned(x):
    h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True); h.copy_(x); return h
sets = [tuple(pinned(x) for x in qs.next()) for _ in range(4)]
outs = [torch.empty((L, B, cfg.n_head, cfg.d_head), dtype=torch.float32, pin_memory=True) for _ in range(4)]
eng.capture_host(*sets[0], outs[0])
for mode in ("same", "rotate", "same"):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record()
    for i in range(12):
        k = 0 if mode == "same" else i % 4
        eng.replay_host(*sets[k], outs[k])
    t1 = time.perf_counter(); b.record(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"{mode:7s} gpu {a.elapsed_time(b) / 12:.3f} ms/step  host enqueue {1e3 * (t1 - t0) / 12:.3f} ms/step  wall {1e3 * (t2 - t0) / 12:.3f}")
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); a.record()
for i in range(12):
    eng.step_host(*sets[i % 4], out=outs[i % 4], gather="uva", sync=False)
b.record(); torch.cuda.synchronize()
print(f"eager step_host gpu {a.elapsed_time(b) / 12:.3f} ms/step wall {1e3 * (time.perf_counter() - t0) / 12:.3f}")
eng.close()
