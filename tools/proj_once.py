"""One tcgen05 QKV projection launch per (m, splits) on the 1B shape, for ncu (not product code)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2510_13602_b200.projection import QKVProjection

d, dh = 2048, 128
rng = np.random.default_rng(0)
proj = QKVProjection(*(rng.standard_normal((d, h * dh)) / np.sqrt(d) for h in (16, 2, 2)))
for arg in sys.argv[1:]:
    m, sp = (int(x) for x in arg.split(":"))
    h = torch.randn(m, d, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        proj(h, sp)
torch.cuda.synchronize()
