"""Drop-in `DecodeEngine` for the reference API.

`DecodeEngine(config, weights, capacity)` with `prefill(h)`, `start_run()` and
`step(h_t, selector) -> StepOutput` keeps the reference signatures and meanings
(decode.py:106-194): hidden states in, per-KV-head `SelectionResult`s and
(n_head, d_head) outputs out, the new token appended after attention.  The QKV projection
(project_qkv, attention.py:67-90) runs on the GPU: for bf16 caches on the tensor cores
(`projection.QKVProjection`, the tcgen05 GEMM behind `nosa_project_qkv`) when the shapes
tile (n % 128 == 0, d % 64 == 0), otherwise and for fp32 caches as an fp32 CUDA-core GEMM
(`nosa_project_f32`); selection, attention, the eviction score and the append run in the
sm_100a kernels behind the C ABI.  Like the reference engine, all KV stays
resident (every block is placed in an HBM slot at prefill).

`ModelWeights.random` and `EvictionHead` mirror decode.py:32-53 and attention.py:104-118
(same fields, same seeded draws), so weights built for the reference load unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .config import AttentionConfig
from .engine import NosaEngine
from .projection import QKVProjection
from .selection import SelectionResult

VARIANTS = ("retaining", "dma", "ed-dma", "s-dma")
SELECTORS = ("nosa", "infllmv2")


@dataclass(frozen=True)
class EvictionHead:
    variant: str
    w1: np.ndarray
    w2: np.ndarray

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown eviction head variant {self.variant!r}")


@dataclass(frozen=True)
class ModelWeights:
    w_q: np.ndarray
    w_k: np.ndarray
    w_v: np.ndarray
    eviction: EvictionHead
    seed: int

    @classmethod
    def random(cls, config: AttentionConfig, variant: str, seed: int) -> "ModelWeights":
        """Seeded synthetic weights: five PCG64 child streams, 1/sqrt(fan-in) scaling."""
        streams = [np.random.default_rng(s) for s in np.random.SeedSequence(seed).spawn(5)]
        inv = 1.0 / np.sqrt(config.d)
        w_q = streams[0].standard_normal((config.d, config.n_head * config.d_head)) * inv
        w_k = streams[1].standard_normal((config.d, config.n_kv_head * config.d_head)) * inv
        w_v = streams[2].standard_normal((config.d, config.n_kv_head * config.d_head)) * inv
        fan = config.d if variant == "retaining" else config.d_head
        w1 = streams[3].standard_normal((fan, config.n_head)) / np.sqrt(fan)
        w2 = streams[4].standard_normal(config.n_head) / np.sqrt(config.n_head)
        return cls(w_q, w_k, w_v, EvictionHead(variant, w1, w2), seed)


@dataclass
class StepOutput:
    step: int
    selections: list[SelectionResult]
    outputs: np.ndarray


class DecodeEngine:
    """One sequence, one layer, all KV resident: the reference engine's contract on a B200."""

    def __init__(self, config: AttentionConfig, weights: ModelWeights, capacity: int, device: int = 0,
                 dtype: str = "bf16"):
        if weights.eviction.variant == "retaining":
            raise ValueError("the retaining eviction head scores hidden states; this path scores value rows "
                             "(ed-dma, s-dma, dma)")
        self.config, self.weights, self.capacity = config, weights, capacity
        blocks = -(-capacity // config.n_b)
        self._eng = NosaEngine(config, batch=1, layers=1, max_tokens=capacity, fast_slots=blocks,
                               w1=weights.eviction.w1, w2=weights.eviction.w2, variant=weights.eviction.variant,
                               dtype=dtype, device=device)
        dev = self._eng.device
        w = np.concatenate([weights.w_q, weights.w_k, weights.w_v], axis=1)
        if w.shape[0] != config.d:
            raise ValueError(f"weights expect width {w.shape[0]}, config.d is {config.d}")
        self._split = (config.n_head * config.d_head, config.n_kv_head * config.d_head)
        self._tc = None
        if dtype == "bf16" and w.shape[1] % 128 == 0 and config.d % 64 == 0:
            self._tc = QKVProjection(weights.w_q, weights.w_k, weights.w_v, device=dev.index or 0)
        else:
            self._w = torch.as_tensor(w, dtype=torch.float32, device=dev)
        self.geometry = None

    @property
    def t(self) -> int:
        return int(self._eng._t[0, 0])

    def _project(self, h: np.ndarray):
        if self._tc is not None:  # tcgen05 GEMM, bf16 operands, fp32 accumulation
            return self._tc(torch.as_tensor(np.asarray(h, dtype=np.float32)).to(self._tc.device))
        x = torch.as_tensor(np.asarray(h, dtype=np.float32), device=self._w.device).reshape(-1, self._w.shape[0])
        y = torch.empty(x.shape[0], self._w.shape[1], dtype=torch.float32, device=x.device)
        _lib.check(_lib.lib.nosa_project_f32(x.data_ptr(), x.shape[0], x.shape[1], self._w.data_ptr(),
                                             self._w.shape[1], y.data_ptr(), _lib.stream_ptr()))
        y = y.reshape(*np.shape(h)[:-1], self._w.shape[1])  # the projection GEMM (fp32, CUDA cores)
        q, k, v = torch.split(y, [self._split[0], self._split[1], self._split[1]], dim=-1)
        return q, k, v

    def prefill(self, h: np.ndarray):
        """Project and cache hidden states [t, d] without attending (decode.py:139-146)."""
        h = np.asarray(h)
        if self.t + h.shape[0] > self.capacity:
            raise ValueError("head cache capacity exhausted")
        if self.t:
            raise ValueError("this engine caches one prefix; prefill before any step")
        _, k, v = self._project(h)
        c = self.config
        k = k.reshape(h.shape[0], c.n_kv_head, c.d_head).permute(1, 0, 2).unsqueeze(0)
        v = v.reshape(h.shape[0], c.n_kv_head, c.d_head).permute(1, 0, 2).unsqueeze(0)
        self._eng.prefill(k, v, layer=0, resident=True)

    def start_run(self):
        self._eng.start_run()
        self.geometry = self._eng.geometry[0]

    def step(self, h_t: np.ndarray, selector: str = "nosa") -> StepOutput:
        """Select, attend over the cached tokens, append the new row (decode.py:152-190)."""
        if selector not in SELECTORS:
            raise ValueError(f"selector must be one of {SELECTORS}")
        if self.geometry is None:
            self.start_run()
        t = self.t
        q, k, v = self._project(np.asarray(h_t).reshape(1, -1))
        out = self._eng.step(q, k, v, selector=selector)
        return StepOutput(step=t, selections=self._eng.selections(0)[0],
                          outputs=out[0, 0].double().cpu().numpy())

    def close(self):
        self._eng.close()
