"""Probe: which re-pointing of captured event-record nodes does the driver accept?"""
import sys
import traceback
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2510_13602_b200 import NosaEngine, one_b_config, workload  # noqa: E402

cfg = one_b_config(8192)
w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, 0)
K, V = workload.prefix_kv(0, 2, 2, 3000, 128)
for case in ("replay_without_timing", "timing_then_disable", "timing_then_more"):
    eng = NosaEngine(cfg, batch=1, layers=2, max_tokens=3200, fast_slots=70, w1=w1, w2=w2)
    eng.prefill(torch.from_numpy(K.reshape(2, 1, 2, 3000, 128)), torch.from_numpy(V.reshape(2, 1, 2, 3000, 128)))
    eng.start_run()
    qs = workload.QueryStream(0, 2, 1, cfg.n_head, 2, 128, 0.5)
    dev = eng.device
    q, k, v = (torch.from_numpy(x).to(dev, torch.bfloat16).contiguous() for x in qs.next())
    out = torch.empty((2, 1, cfg.n_head, 128), dtype=torch.float32, device=dev)
    try:
        eng.capture(q, k, v, out)
        if case == "replay_without_timing":
            eng.replay(); eng.replay()
        elif case == "timing_then_disable":
            eng.timing_enable(8); eng.replay(); eng.timing_enable(0); eng.replay()
        else:
            eng.timing_enable(8); eng.replay(); eng.replay(); eng.replay()
        torch.cuda.synchronize()
        print(case, "OK", flush=True)
    except Exception:
        print(case, "FAILED", flush=True)
        traceback.print_exc()
    eng.close()
