"""Seeded synthetic inputs of the decode step.

* K, V ~ N(0, 1) rounded to bf16-representable float32 (so the f64 oracle sees the exact
  values the GPU stores).
* Query stream per (sequence, query head): AR(1), q_t = rho q_{t-1} + sqrt(1 - rho^2) eps_t,
  eps ~ N(0, I / d_head).  s_q = K_c . q_sum is linear in q, so every block score follows the
  same AR(1) as the reference's scripted traces (decode.py:252-260); rho = 0 is the
  adversarial, low-locality regime (decode.py:232-234), rho = 0.95 the high-locality one.
* ED-DMA eviction head as ModelWeights.random draws it (decode.py:50-52):
  W1 ~ N(0, 1/d_head), W2 ~ N(0, 1/n_head).
Small sizes use NumPy PCG64 (what the oracle and golden files use); bench-size inputs are drawn
on the GPU with torch's Philox generator.
"""

from __future__ import annotations

import numpy as np


def bf16_round(x) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even), returned as float32."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    u = a.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return rounded.astype(np.uint32).view(np.float32).reshape(a.shape)


def eviction_head(n_head: int, d_head: int, seed: int):
    rng = np.random.default_rng(np.random.SeedSequence([seed, 7]))
    w1 = rng.standard_normal((d_head, n_head)) / np.sqrt(d_head)
    w2 = rng.standard_normal(n_head) / np.sqrt(n_head)
    return w1, w2


def prefix_kv(seed: int, batch: int, n_kv_head: int, t: int, d_head: int, bf16: bool = True):
    """K, V of shape [batch][n_kv_head][t][d_head] float32."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 1]))
    k = rng.standard_normal((batch, n_kv_head, t, d_head), dtype=np.float32)
    v = rng.standard_normal((batch, n_kv_head, t, d_head), dtype=np.float32)
    return (bf16_round(k), bf16_round(v)) if bf16 else (k, v)


class QueryStream:
    """AR(1) per-(layer, sequence, head) query stream plus fresh K/V rows for each step."""

    def __init__(self, seed: int, layers: int, batch: int, n_head: int, n_kv_head: int, d_head: int,
                 rho: float, bf16: bool = True):
        if not 0.0 <= rho < 1.0:
            raise ValueError("rho must be in [0, 1)")
        self.rng = np.random.default_rng(np.random.SeedSequence([seed, 2]))
        self.shape_q = (layers, batch, n_head, d_head)
        self.shape_kv = (layers, batch, n_kv_head, d_head)
        self.rho, self.bf16, self.d_head = rho, bf16, d_head
        self.state = self.rng.standard_normal(self.shape_q) / np.sqrt(d_head)

    def _round(self, x):
        return bf16_round(x) if self.bf16 else x.astype(np.float32)

    def next(self):
        """(q, k_new, v_new) for one step, float32 arrays."""
        q = self._round(self.state)
        k = self._round(self.rng.standard_normal(self.shape_kv))
        v = self._round(self.rng.standard_normal(self.shape_kv))
        eps = self.rng.standard_normal(self.shape_q) / np.sqrt(self.d_head)
        self.state = self.rho * self.state + np.sqrt(1.0 - self.rho ** 2) * eps
        return q, k, v


# ------------------------------------------------------------------------------------------------
# Counter-based synthetic inputs: every value is a pure function of (seed, kind, layer, sequence,
# head, position, dim), so the GPU (nosa_synth_* in libnosa_b200.so) and this NumPy code produce the
# SAME bits, for any batch sharding and any subset.  Both bench arms and the headline-config parity
# tests draw their inputs here.  A normal is the Irwin-Hall sum of the four 16-bit fields of one
# splitmix64 hash (mean 0, variance 1, support +-3.46), scaled in one fp32 multiply; the AR(1)
# update is fl32(fl32(rho * x) + fl32(sigma * eps)) (no fused multiply-add on either side).
KIND_K, KIND_V, KIND_Q0, KIND_QEPS, KIND_KNEW, KIND_VNEW = 0, 1, 2, 3, 4, 5
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1, _M2 = np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB)


def _mix64(z):
    """splitmix64 finalizer on uint64 arrays (wrapping arithmetic)."""
    z = z ^ (z >> np.uint64(30))
    z = z * _M1
    z = z ^ (z >> np.uint64(27))
    z = z * _M2
    return z ^ (z >> np.uint64(31))


def synth_scale(d_head: int | None = None) -> np.float32:
    """fp32 multiplier of the integer Irwin-Hall sum: unit variance, or 1/d_head (queries)."""
    s = np.sqrt(3.0) / 65536.0
    return np.float32(s if d_head is None else s / np.sqrt(float(d_head)))


def synth_normal(seed: int, kind: int, layer: int, seqs, heads: int, pos0: int, n_pos: int, d: int,
                 scale=None) -> np.ndarray:
    """float32 [len(seqs)][heads][n_pos][d] normals of (layer, global sequence ids `seqs`)."""
    scale = synth_scale() if scale is None else np.float32(scale)
    seqs = np.asarray(seqs, dtype=np.uint64).reshape(-1, 1, 1, 1)
    hh = np.arange(heads, dtype=np.uint64).reshape(1, -1, 1, 1)
    pos = np.arange(pos0, pos0 + n_pos, dtype=np.uint64).reshape(1, 1, -1, 1)
    dd = np.arange(d, dtype=np.uint64).reshape(1, 1, 1, -1)
    with np.errstate(over="ignore"):
        k0 = _mix64(np.uint64(seed) * _GOLD + np.uint64(kind))
        row = (np.uint64(layer) << np.uint64(32)) | (seqs << np.uint64(12)) | hh
        krow = _mix64(k0 ^ row)
        h = _mix64(krow + ((pos << np.uint64(10)) | dd) * _GOLD)
    m = np.uint64(0xFFFF)
    s = ((h & m) + ((h >> np.uint64(16)) & m) + ((h >> np.uint64(32)) & m) + (h >> np.uint64(48))).astype(np.int64)
    return (s - 131070).astype(np.float32) * scale


def synth_prefix_kv(seed: int, layer: int, seqs, heads: int, t: int, d: int, bf16: bool = True):
    """Prefix K, V [len(seqs)][heads][t][d] float32: bf16-representable (bf16 storage) or as drawn
    (fp32 storage)."""
    k = synth_normal(seed, KIND_K, layer, seqs, heads, 0, t, d)
    v = synth_normal(seed, KIND_V, layer, seqs, heads, 0, t, d)
    return (bf16_round(k), bf16_round(v)) if bf16 else (k, v)


class SynthQueryStream:
    """NumPy twin of the GPU stream (paper_2510_13602_b200.synth.GpuQueryStream) for a subset of
    layers x global sequences: step s yields q = bf16(x_s), k_new, v_new = bf16(N(0,1)) drawn at
    position s, then x_{s+1} = rho x_s + sqrt(1 - rho^2) eps_s with eps ~ N(0, I/d_head)."""

    def __init__(self, seed: int, layers, seqs, n_head: int, n_kv_head: int, d_head: int, rho: float,
                 bf16: bool = True):
        if not 0.0 <= rho < 1.0:
            raise ValueError("rho must be in [0, 1)")
        self.seed, self.layers, self.seqs = seed, list(layers), list(seqs)
        self.n_head, self.n_kv_head, self.d_head, self.bf16 = n_head, n_kv_head, d_head, bf16
        self.rho32 = np.float32(rho)
        self.sig32 = np.float32(np.sqrt(1.0 - rho * rho))
        self.qscale = synth_scale(d_head)
        self.step = 0
        self.state = np.stack([synth_normal(seed, KIND_Q0, l, self.seqs, n_head, 0, 1, d_head, self.qscale)[:, :, 0]
                               for l in self.layers])

    def _round(self, x):
        return bf16_round(x) if self.bf16 else x

    def next(self):
        """(q [L][B][n_head][d], k_new, v_new [L][B][n_kv_head][d]) float32 for one step."""
        s, H, D = self.step, self.n_kv_head, self.d_head
        q = self._round(self.state.copy())
        k = np.stack([synth_normal(self.seed, KIND_KNEW, l, self.seqs, H, s, 1, D)[:, :, 0] for l in self.layers])
        v = np.stack([synth_normal(self.seed, KIND_VNEW, l, self.seqs, H, s, 1, D)[:, :, 0] for l in self.layers])
        eps = np.stack([synth_normal(self.seed, KIND_QEPS, l, self.seqs, self.n_head, s, 1, D, self.qscale)[:, :, 0]
                        for l in self.layers])
        self.state = (self.rho32 * self.state).astype(np.float32) + (self.sig32 * eps).astype(np.float32)
        self.step += 1
        return q, self._round(k), self._round(v)


def torch_prefix_kv(seed: int, shape, device, dtype):
    """Bench-size K or V drawn on the GPU: N(0, 1) in `dtype` (torch Philox, seeded)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return torch.randn(shape, generator=g, device=device, dtype=torch.float32).to(dtype)


class TorchQueryStream:
    """GPU-side AR(1) query stream of bench size (same process as QueryStream)."""

    def __init__(self, seed: int, layers: int, batch: int, n_head: int, n_kv_head: int, d_head: int,
                 rho: float, device, dtype):
        import torch
        self.torch = torch
        self.g = torch.Generator(device=device)
        self.g.manual_seed(seed)
        self.shape_q = (layers, batch, n_head, d_head)
        self.shape_kv = (layers, batch, n_kv_head, d_head)
        self.rho, self.d_head, self.device, self.dtype = rho, d_head, device, dtype
        self.state = torch.randn(self.shape_q, generator=self.g, device=device) / d_head ** 0.5

    def next(self):
        t = self.torch
        q = self.state.to(self.dtype)
        k = t.randn(self.shape_kv, generator=self.g, device=self.device).to(self.dtype)
        v = t.randn(self.shape_kv, generator=self.g, device=self.device).to(self.dtype)
        eps = t.randn(self.shape_q, generator=self.g, device=self.device) / self.d_head ** 0.5
        self.state = self.rho * self.state + (1.0 - self.rho ** 2) ** 0.5 * eps
        return q, k, v


class TorchHiddenStream:
    """GPU-side AR(1) hidden states h [layers][batch][d] (unit variance): q = h W_q inherits the
    same per-block AR(1) score process as TorchQueryStream's queries (the projection is linear)."""

    def __init__(self, seed: int, layers: int, batch: int, d: int, rho: float, device, dtype):
        import torch
        self.torch = torch
        self.g = torch.Generator(device=device)
        self.g.manual_seed(seed)
        self.shape = (layers, batch, d)
        self.rho, self.device, self.dtype = rho, device, dtype
        self.state = torch.randn(self.shape, generator=self.g, device=device)

    def next(self):
        t = self.torch
        h = self.state.to(self.dtype)
        eps = t.randn(self.shape, generator=self.g, device=self.device)
        self.state = self.rho * self.state + (1.0 - self.rho ** 2) ** 0.5 * eps
        return (h,)
