"""Time the tcgen05 QKV projection (nosa_project_qkv) against cuBLAS (torch bf16 matmul) on the
1B attention shape: d = 2048, n = (16 + 2 + 2) x 128 = 2560 (not product code)."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2510_13602_b200.projection import QKVProjection, _splits

d, hq, hkv, dh = 2048, 16, 2, 128
rng = np.random.default_rng(0)
w_q, w_k, w_v = (rng.standard_normal((d, h * dh)) / np.sqrt(d) for h in (hq, hkv, hkv))
proj = QKVProjection(w_q, w_k, w_v)
wt = proj.w_t
rows = []
for m in (1, 32, 128, 512, 3584):
    h = torch.randn(m, d, device="cuda").to(torch.bfloat16)
    def timeit(fn, it=50):
        """GPU time per call: `it` calls captured in one CUDA graph (no host launch overhead)."""
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(it):
                    fn()
        torch.cuda.synchronize()
        g.replay(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record(); torch.cuda.synchronize()
        return a.elapsed_time(b) / it * 1e3
    per_split = {sp: round(timeit(lambda: proj(h, sp)), 2) for sp in (1, 2, 4, 8)}
    ours = timeit(lambda: proj(h))
    cub = timeit(lambda: h @ wt.T)
    byts = wt.numel() * 2 + h.numel() * 2 + m * wt.shape[0] * 2
    flops = 2 * m * d * wt.shape[0]
    rows.append({"m": m, "splits": _splits(m, wt.shape[0], d), "tcgen05_us": round(ours, 2), "by_splits_us": per_split,
                 "cublas_us": round(cub, 2),
                 "tcgen05_GBps": round(byts / ours / 1e3, 1), "tcgen05_TFLOPs": round(flops / ours / 1e6, 2)})
print(json.dumps(rows, indent=1))
