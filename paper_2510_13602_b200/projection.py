"""QKV projection on the tensor cores (project_qkv, attention.py:67-90).

`QKVProjection` holds [W_q | W_k | W_v] as one bf16 [n][d] matrix on the device (each output
column's weights contiguous, the K-major operand of the tcgen05 GEMM in csrc/nosa_project.cu)
and maps hidden states h [m][d] to bf16 q [m][n_q], k [m][n_kv], v [m][n_kv] through the C ABI
`nosa_project_qkv`.  fp32 accumulation in TMEM; the split-K partials of a thread-block cluster
are summed through distributed shared memory in rank order, so a projection is bitwise
reproducible.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

NUM_SMS = 148


def _splits(m: int, n: int, k: int) -> int:
    """K splits per output tile (a cluster of that many CTAs).  Measured on the 1B shape
    (d = 2048, n = 2560, profiles/r1_projection.txt): 4 splits are fastest while the tiles fill
    well under a wave (m <= 128: 9 us; 8 splits 15 us, 1 split 15-19 us), one split once the
    tiles alone fill the SMs."""
    tiles = (n // 128) * -(-m // 128)
    kt = k // 64
    want = 4 if tiles * 4 <= 2 * NUM_SMS else 1
    want = max(1, min(want, kt))
    while kt % want:
        want -= 1
    return want


class QKVProjection:
    def __init__(self, w_q, w_k, w_v, device=0):
        w = np.concatenate([np.asarray(w_q), np.asarray(w_k), np.asarray(w_v)], axis=1)  # [d][n]
        self.d, self.n = w.shape
        self.nq, self.nk = np.asarray(w_q).shape[1], np.asarray(w_k).shape[1]
        if self.n % 128 or self.d % 64:
            raise ValueError(f"tensor-core projection needs n % 128 == 0 and d % 64 == 0 (n={self.n}, d={self.d})")
        self.device = torch.device("cuda", device)
        self.w_t = torch.as_tensor(np.ascontiguousarray(w.T), dtype=torch.float32).to(
            device=self.device, dtype=torch.bfloat16).contiguous()

    def __call__(self, h: torch.Tensor, splits: int | None = None):
        """h: [m][d] (any float dtype, on the device) -> bf16 (q, k, v) on the same device."""
        h = h.to(device=self.device, dtype=torch.bfloat16).contiguous()
        m = h.shape[0]
        splits = splits or _splits(m, self.n, self.d)
        nv = self.n - self.nq - self.nk
        q = torch.empty((m, self.nq), dtype=torch.bfloat16, device=self.device)
        k = torch.empty((m, self.nk), dtype=torch.bfloat16, device=self.device)
        v = torch.empty((m, nv), dtype=torch.bfloat16, device=self.device)
        with torch.cuda.device(self.device):
            _lib.check(_lib.lib.nosa_project_qkv(h.data_ptr(), m, self.d, self.w_t.data_ptr(), self.n, self.nq, self.nk,
                                                 q.data_ptr(), k.data_ptr(), v.data_ptr(), splits,
                                                 _lib.stream_ptr()))
        return q, k, v
