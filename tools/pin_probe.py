"""H2D rate of torch pinned tensors of the bench's input sizes (not product code)."""
import torch

dev = torch.device("cuda", 0)
for mb in (0.6, 2.6, 5.2, 8, 32):
    n = int(mb * 2**20) // 2
    for how in ("pin_memory()", "empty(pin_memory=True)"):
        h = torch.randn(n).to(torch.bfloat16).pin_memory() if how == "pin_memory()" else \
            torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
        d = torch.empty(n, dtype=torch.bfloat16, device=dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            a.record(); d.copy_(h, non_blocking=True); b.record(); torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        print(f"{mb:5.1f} MB {how:24s} {n * 2 / best / 1e6:7.1f} GB/s ({best * 1000:.1f} us)")
