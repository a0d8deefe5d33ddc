"""Run a few decode steps of one workload shape for ncu / timing experiments.

    python tools/profile_step.py --batch 128 --layers 2 --context 32768 --cache 0.25 --steps 6
Prints per-kernel device times (CUDA events bracketing each launch on its stream)."""

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2510_13602_b200 import NosaEngine, one_b_config, workload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--context", type=int, default=32768)
    ap.add_argument("--cache", type=float, default=0.25, help="fraction of blocks in HBM; 1 = resident")
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--rho", type=float, default=0.95)
    ap.add_argument("--selector", default="nosa")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--gather", default="uva")
    ap.add_argument("--layer-by-layer", action="store_true", help="use the per-layer C-ABI calls")
    ap.add_argument("--trace", action="store_true", help="print the device timeline of the last step")
    ap.add_argument("--sel-prof", action="store_true", help="print the selection kernel's cycles per phase")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg = one_b_config(65536)
    max_tokens = a.context + a.steps + 4
    nblk = -(-max_tokens // cfg.n_b)
    fast = nblk if a.cache >= 1 else int(a.cache * nblk)
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, 0)
    t0 = time.time()
    tdt = torch.float32 if a.dtype == "fp32" else torch.bfloat16
    eng = NosaEngine(cfg, batch=a.batch, layers=a.layers, max_tokens=max_tokens, fast_slots=fast, w1=w1, w2=w2,
                     dtype=a.dtype)
    for l in range(a.layers):
        shape = (a.batch, cfg.n_kv_head, a.context, cfg.d_head)
        eng.prefill(workload.torch_prefix_kv(2 * l, shape, dev, tdt),
                    workload.torch_prefix_kv(2 * l + 1, shape, dev, tdt), layer=l, resident=a.cache >= 1)
    eng.start_run()
    torch.cuda.synchronize()
    print(f"setup {time.time() - t0:.1f}s", flush=True)
    qs = workload.TorchQueryStream(7, a.layers, a.batch, cfg.n_head, cfg.n_kv_head, cfg.d_head, a.rho, dev, tdt)
    out = torch.empty((a.layers, a.batch, cfg.n_head, cfg.d_head), dtype=torch.float32, device=dev)
    eng.timing_enable(4 * a.layers * a.steps + 8)
    for s in range(a.steps):
        q, k, v = qs.next()
        if s == 2:
            eng.reset_stats()
            eng.timing_enable(4 * a.layers * a.steps + 8)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
        if a.layer_by_layer:
            for l in range(a.layers):
                eng.step_layer(l, q[l], k[l], v[l], selector=a.selector, out=out[l], gather=a.gather)
            eng._t[:] = eng._t[0]  # step_layer advances per layer
        else:
            eng.step(q, k, v, selector=a.selector, out=out, gather=a.gather, check=False)
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record()
    torch.cuda.synchronize()
    if a.sel_prof:  # one more step with the phase profiler on
        import ctypes
        import numpy as np
        from paper_2510_13602_b200 import _lib
        cyc = np.zeros(16)
        P = lambda: cyc.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        eng._call(_lib.lib.nosa_select_profile, 1, None)
        q, k, v = qs.next()
        eng.step(q, k, v, selector=a.selector, out=out, gather=a.gather, check=False)
        eng._call(_lib.lib.nosa_select_profile, 0, P())
        names = {1: "q_sum", 2: "screen scan", 3: "radix threshold", 4: "f64 rescoring", 5: "ranking", 6: "NOSA walk",
                 7: "outputs+required", 8: "hit test", 9: "victims", 11: "apply+writes"}
        n = max(cyc[15], 1)
        tot = sum(cyc[i] for i in names)
        print(f"select_plan: {int(cyc[15])} CTAs, {tot / n:.0f} cycles per CTA ({tot / n / 1.965e3:.1f} us at 1965 MHz)")
        for i, nm in names.items():
            print(f"  {nm:18s} {cyc[i] / n:8.0f} cycles  {100 * cyc[i] / max(tot, 1):5.1f}%")
    st = eng.residency_stats()
    res = {"ms_per_step": e0.elapsed_time(e1) / (a.steps - 2), "kernels": eng.timing_read(),
           "hit_rate": st.hit_rate, "misses": st.misses, "hits": st.hits}
    print(json.dumps(res, indent=1))
    if a.trace:
        tr = eng.timing_trace()
        per_step = len(tr) // (a.steps - 2)
        last = tr[-per_step:]
        base = min(x[1] for x in last)
        seen = {}
        print("kind        layer   start_us   end_us   dur_us")
        for k, s0, s1 in last:
            l = seen.get(k, 0)
            seen[k] = l + 1
            print(f"{k:11s} {l:5d} {1000 * (s0 - base):10.1f} {1000 * (s1 - base):8.1f} {1000 * (s1 - s0):8.1f}")
    eng.check_errors()
    eng.close()


if __name__ == "__main__":
    main()
