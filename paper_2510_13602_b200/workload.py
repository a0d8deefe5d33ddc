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
