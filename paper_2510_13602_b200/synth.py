"""GPU side of the counter-based synthetic inputs (workload.synth_* is the NumPy twin).

Bench-size prefixes and query streams are drawn on the device by nosa_synth_normal /
nosa_synth_ar1_step with the same bits the NumPy code yields for any (layer, sequence) subset,
so the CPU oracle and the reference arm see exactly the inputs the GPU arm decodes.
Sequences are addressed by GLOBAL id: a rank owning [seq0, seq0 + n) draws the same values as a
single GPU owning the whole batch.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .workload import KIND_K, KIND_KNEW, KIND_Q0, KIND_V, KIND_VNEW, synth_scale

_DT = {torch.bfloat16: _lib.DTYPE["bf16"], torch.float32: _lib.DTYPE["fp32"]}


def normal(seed: int, kind: int, layer0: int, n_layers: int, seq0: int, n_seq: int, heads: int, pos0: int,
           n_pos: int, d: int, device, dtype=torch.bfloat16, scale=None, out: torch.Tensor | None = None):
    """[n_layers][n_seq][heads][n_pos][d] draws of `kind` on `device`."""
    if out is None:
        out = torch.empty((n_layers, n_seq, heads, n_pos, d), dtype=dtype, device=device)
    sc = float(synth_scale() if scale is None else np.float32(scale))
    with torch.cuda.device(out.device):
        _lib.check(_lib.lib.nosa_synth_normal(seed, kind, layer0, n_layers, seq0, n_seq, heads, pos0, n_pos, d, sc,
                                              _DT[out.dtype], out.data_ptr(), _lib.stream_ptr()))
    return out


def prefix_kv(seed: int, layer: int, seq0: int, n_seq: int, heads: int, t: int, d: int, device,
              dtype=torch.bfloat16):
    """Prefix K, V [n_seq][heads][t][d] of one layer (workload.synth_prefix_kv's values)."""
    k = normal(seed, KIND_K, layer, 1, seq0, n_seq, heads, 0, t, d, device, dtype)[0]
    v = normal(seed, KIND_V, layer, 1, seq0, n_seq, heads, 0, t, d, device, dtype)[0]
    return k, v


class GpuQueryStream:
    """workload.SynthQueryStream on the device for layers [0, layers) x sequences
    [seq0, seq0 + batch): next() -> (q [L][B][n_head][d], k_new, v_new [L][B][n_kv_head][d])."""

    def __init__(self, seed: int, layers: int, seq0: int, batch: int, n_head: int, n_kv_head: int, d_head: int,
                 rho: float, device, dtype=torch.bfloat16):
        if not 0.0 <= rho < 1.0:
            raise ValueError("rho must be in [0, 1)")
        self.seed, self.L, self.seq0, self.B = seed, layers, seq0, batch
        self.n_head, self.n_kv_head, self.d_head, self.dtype, self.device = n_head, n_kv_head, d_head, dtype, device
        self.rho32 = float(np.float32(rho))
        self.sig32 = float(np.float32(np.sqrt(1.0 - rho * rho)))
        self.qscale = float(synth_scale(d_head))
        self.step = 0
        self.state = normal(seed, KIND_Q0, 0, layers, seq0, batch, n_head, 0, 1, d_head, device, torch.float32,
                            scale=self.qscale).reshape(layers, batch, n_head, d_head).contiguous()

    def next(self):
        L, B, D = self.L, self.B, self.d_head
        q = torch.empty((L, B, self.n_head, D), dtype=self.dtype, device=self.device)
        with torch.cuda.device(q.device):
            _lib.check(_lib.lib.nosa_synth_ar1_step(self.seed, 0, L, self.seq0, B, self.n_head, self.step, D,
                                                    self.rho32, self.sig32, self.qscale, self.state.data_ptr(),
                                                    _DT[self.dtype], q.data_ptr(), _lib.stream_ptr()))
        k = normal(self.seed, KIND_KNEW, 0, L, self.seq0, B, self.n_kv_head, self.step, 1, D, self.device,
                   self.dtype).reshape(L, B, self.n_kv_head, D)
        v = normal(self.seed, KIND_VNEW, 0, L, self.seq0, B, self.n_kv_head, self.step, 1, D, self.device,
                   self.dtype).reshape(L, B, self.n_kv_head, D)
        self.step += 1
        return q, k, v
