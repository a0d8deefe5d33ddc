"""Block geometry, selection results and the GPU selectors.

`BlockGeometry`, `SelectionResult` and `build_token_mask` keep the reference's definitions
(selection.py:36-118, 181-191) — they are host-side bookkeeping.  `nosa_select` and
`infllmv2_select` keep the reference signatures (selection.py:130-136, 163-168) but the top-k
runs in the sm_100a kernel behind `nosa_select_scores` (block-level bitonic sort with the
argtopk order: score descending, block index ascending, -0.0 == +0.0).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .config import AttentionConfig

NEG_INF = float("-inf")


@dataclass(frozen=True)
class BlockGeometry:
    """Sink / pool / recent layout of one decode run; recent edge frozen at t0."""

    n_b: int
    n_s: int
    t0: int
    recent_start: int

    @classmethod
    def for_run(cls, config: AttentionConfig, t0: int) -> "BlockGeometry":
        if t0 < 0:
            raise ValueError("t0 must be non-negative")
        return cls(n_b=config.n_b, n_s=config.n_s, t0=t0,
                   recent_start=max(0, t0 - config.n_w + 1))

    @property
    def sink_blocks(self) -> range:
        return range(self.n_s // self.n_b)

    @property
    def pool_blocks(self) -> range:
        first = self.n_s // self.n_b
        return range(first, max(first, self.recent_start // self.n_b))

    def n_blocks(self, t: int) -> int:
        return (t + self.n_b - 1) // self.n_b

    def recent_blocks(self, t: int) -> range:
        end = self.n_blocks(t)
        return range(min(self.recent_start // self.n_b, end), end)

    def fixed_blocks(self, t: int) -> tuple[int, ...]:
        end = self.n_blocks(t)
        blocks = set(self.sink_blocks).union(self.recent_blocks(t))
        return tuple(sorted(b for b in blocks if b < end))


@dataclass(frozen=True)
class SelectionResult:
    """One step's selected blocks for one KV head (selection.py:79-101)."""

    step: int
    blocks_q: tuple[int, ...]
    blocks_e: tuple[int, ...]
    blocks_fixed: tuple[int, ...]
    gamma_tokens: frozenset[int]

    @property
    def topk_blocks(self) -> frozenset[int]:
        return frozenset(self.blocks_q).union(self.blocks_e)

    @property
    def attended_blocks(self) -> frozenset[int]:
        return self.topk_blocks.union(self.blocks_fixed)


def make_result(t: int, n_b: int, blocks_q, blocks_e, fixed) -> SelectionResult:
    """Assemble a SelectionResult; Gamma(t) clips the last block at t (selection.py:104-118)."""
    tokens = set()
    for b in set(blocks_q) | set(blocks_e) | set(fixed):
        tokens.update(range(b * n_b, min(b * n_b + n_b, t)))
    return SelectionResult(step=t, blocks_q=tuple(sorted(int(b) for b in blocks_q)),
                           blocks_e=tuple(sorted(int(b) for b in blocks_e)),
                           blocks_fixed=tuple(int(b) for b in fixed),
                           gamma_tokens=frozenset(tokens))


def _scores(arr, geometry: BlockGeometry, t: int, name: str) -> np.ndarray:
    s = np.asarray(arr, dtype=np.float64)
    if s.ndim != 1 or s.size < geometry.n_blocks(t):
        raise ValueError(f"{name} must cover all {geometry.n_blocks(t)} blocks at t={t}, got length {s.size}")
    if np.isnan(s).any():
        raise ValueError(f"{name} contains NaN")
    return s


def select_batch(s_q: np.ndarray, s_e: np.ndarray | None, pool_lo: np.ndarray, pool_hi: np.ndarray,
                 m_q: int, m_e: int, selector: str, device: int = 0):
    """Run the GPU selector on a batch of score rows.

    s_q, s_e: [n, stride] float64; pool ranges [n].  Returns (list of picked_q, list of
    picked_e) as sorted int arrays (absolute block ids)."""
    import torch

    n, stride = s_q.shape
    dev = torch.device("cuda", device)
    tq = torch.as_tensor(np.ascontiguousarray(s_q, dtype=np.float64), device=dev)
    te = torch.as_tensor(np.ascontiguousarray(s_e if s_e is not None else s_q, dtype=np.float64), device=dev)
    lo = torch.as_tensor(np.asarray(pool_lo, dtype=np.int32), device=dev)
    hi = torch.as_tensor(np.asarray(pool_hi, dtype=np.int32), device=dev)
    oq = torch.empty((n, max(m_q, 1)), dtype=torch.int32, device=dev)
    oe = torch.empty((n, max(m_e, 1)), dtype=torch.int32, device=dev)
    nq = torch.empty(n, dtype=torch.int32, device=dev)
    ne = torch.empty(n, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        rc = _lib.lib.nosa_select_scores(n, tq.data_ptr(), te.data_ptr(), stride, lo.data_ptr(), hi.data_ptr(),
                                         m_q, m_e, _lib.SELECTOR[selector], oq.data_ptr(), nq.data_ptr(),
                                         oe.data_ptr(), ne.data_ptr(), _lib.stream_ptr())
        _lib.check(rc)
        oq, oe, nq, ne = oq.cpu().numpy(), oe.cpu().numpy(), nq.cpu().numpy(), ne.cpu().numpy()
    return [oq[i, :nq[i]] for i in range(n)], [oe[i, :ne[i]] for i in range(n)]


def nosa_select(s_q_blocks, s_e_blocks, t: int, config: AttentionConfig,
                geometry: BlockGeometry | None = None) -> SelectionResult:
    """Two-phase NOSA selection on the GPU (reference: selection.py:130-160)."""
    if geometry is None:
        geometry = BlockGeometry.for_run(config, t)
    s_q = _scores(s_q_blocks, geometry, t, "s_q_blocks")
    s_e = _scores(s_e_blocks, geometry, t, "s_e_blocks")
    stride = max(s_q.size, s_e.size)
    sq = np.zeros((1, stride)); sq[0, :s_q.size] = s_q
    se = np.zeros((1, stride)); se[0, :s_e.size] = s_e
    pool = geometry.pool_blocks
    picked_q, picked_e = select_batch(sq, se, [pool.start], [pool.stop], config.blocks_q, config.blocks_e, "nosa")
    return make_result(t, config.n_b, picked_q[0], picked_e[0], geometry.fixed_blocks(t))


def infllmv2_select(s_q_blocks, t: int, config: AttentionConfig,
                    geometry: BlockGeometry | None = None) -> SelectionResult:
    """InfLLM-V2 baseline: top blocks by query score alone (reference: selection.py:163-178)."""
    if geometry is None:
        geometry = BlockGeometry.for_run(config, t)
    s_q = _scores(s_q_blocks, geometry, t, "s_q_blocks")
    pool = geometry.pool_blocks
    picked, _ = select_batch(s_q[None, :], None, [pool.start], [pool.stop], config.blocks_topk, 0, "infllmv2")
    return make_result(t, config.n_b, picked[0], (), geometry.fixed_blocks(t))


def build_token_mask(sel: SelectionResult, t: int) -> np.ndarray:
    """Length-t additive mask, 0 on Gamma(t) and -inf elsewhere (selection.py:181-191)."""
    if sel.step != t:
        raise ValueError(f"selection was taken at step {sel.step}, not {t}")
    mask = np.full(t, NEG_INF)
    open_positions = np.fromiter((j for j in sel.gamma_tokens if j < t), dtype=np.int64)
    mask[open_positions] = 0.0
    return mask

