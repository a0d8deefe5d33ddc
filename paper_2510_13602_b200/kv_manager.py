"""GPU-resident two-tier block manager.

`GpuTieredBlockManager` keeps the TieredBlockManager planning API (kv_manager.py:130-305) for
the residency semantics the decode path uses: every logical block (batch, head, block_index)
exists in the slow tier (the pinned host mirror), the fast tier is a per-(batch, head) pool of
HBM slots, and `plan_transfers` fetches exactly the missing required blocks, evicting
least-recently-required non-required blocks (kv_manager.py:125-127) only as far as capacity
demands, reusing freed slots LIFO (kv_manager.py:147-150, 281-298).

The planner runs in the K2 kernel, which plans and applies in one pass (a GPU plan is never
observed half-applied), so `plan_transfers` returns an executed plan; `apply_transfers`
validates it against the table version exactly like the reference (StalePlan) and moves the
payload (K3) when the manager holds one.  One kernel launch serves any number of
(batch, head) managers: see `plan_batch`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .config import AttentionConfig
from .engine import NosaEngine, ResidencyStats
from .errors import CapacityExceeded, UnknownKey
from . import _lib

FAST, SLOW = "fast", "slow"


@dataclass
class TransferPlan:
    fetch: list[tuple]
    evict: list[tuple]
    bytes_up: int
    bytes_down: int
    hits: int
    misses: int
    version: int

    @property
    def empty(self) -> bool:
        return not self.fetch and not self.evict


class GpuTieredBlockManager:
    """fast_blocks: fast slots per head of each sequence's manager, or with shared=True the size
    of the one per-head pool the whole batch shares (the reference simulator's layout,
    offload_sim.py:254-256; planned in batch order).  slow_blocks: blocks per (sequence, head)."""

    def __init__(self, fast_blocks: int, slow_blocks: int, heads: int = 1, batch: int = 1, n_b: int = 16,
                 d_head: int = 64, element_width: int = 2, device: int = 0, shared: bool = False):
        if element_width not in (2, 4):
            raise ValueError("element_width must be 2 or 4 bytes")
        if shared and fast_blocks % batch:
            raise ValueError("a shared pool is allocated as batch equal shares: fast_blocks % batch must be 0")
        self.heads, self.batch, self.fast_blocks, self.slow_blocks = heads, batch, fast_blocks, slow_blocks
        self.shared = shared
        self.per_seq = fast_blocks // batch if shared else fast_blocks
        # a selection-free engine: the budgets are irrelevant to explicit required sets
        cfg = AttentionConfig(n=max(slow_blocks * n_b, n_b), d=d_head, n_head=heads, n_kv_head=heads, d_head=d_head,
                              n_b=n_b, n_s=0, n_w=0, k=0, k_q=0, k_e=0)
        self._engine = NosaEngine(cfg, batch=batch, max_tokens=slow_blocks * n_b, fast_slots=self.per_seq,
                                  w1=np.zeros((d_head, heads)), w2=np.zeros(heads),
                                  dtype="bf16" if element_width == 2 else "fp32", device=device,
                                  residency="shared" if shared else "per-sequence")
        self.bytes_per_block = self._engine.bytes_per_block
        self.version = 0

    def close(self):
        self._engine.close()

    def plan_batch(self, required: dict[tuple[int, int], set]) -> dict[tuple[int, int], TransferPlan]:
        """Plan + apply for several (batch, head) managers in one kernel launch."""
        B, H, C = self.batch, self.heads, self.per_seq
        req = np.zeros((B, H, C), np.int32)
        n = np.full((B, H), -1, np.int32)
        for (b, h), blocks in required.items():
            blocks = sorted({int(x) for x in blocks})
            if len(blocks) > C:
                raise CapacityExceeded(
                    f"step requires {len(blocks)} blocks but the fast tier holds {C} per head"
                    + (" per sequence share" if self.shared else ""))
            if blocks and (blocks[0] < 0 or blocks[-1] >= self.slow_blocks):
                raise UnknownKey(f"required block {(b, h, blocks[-1])} exists in no tier")
            req[b, h, :len(blocks)] = blocks
            n[b, h] = len(blocks)
        dev = self._engine.device
        treq = torch.as_tensor(req, device=dev)
        tn = torch.as_tensor(n, device=dev)
        with torch.cuda.device(dev):
            self._engine._call(_lib.lib.nosa_cache_plan, 0, treq.data_ptr(), tn.data_ptr(), _lib.stream_ptr())
        self._engine.check_errors()
        views = self._engine.plans(0)
        self.version += 1
        out = {}
        NB = self._engine.max_blocks
        for (b, h) in required:
            v = views[b][h]
            # shared pool: a victim may belong to another sequence (key = owner * NB + block)
            evict = [(x // NB, h, x % NB) for x in v.evict] if self.shared else [(b, h, x) for x in v.evict]
            out[(b, h)] = TransferPlan(fetch=[(b, h, x) for x in v.fetch], evict=evict,
                                       bytes_up=v.bytes_up, bytes_down=v.bytes_down, hits=v.hits,
                                       misses=v.misses, version=self.version)
        return out

    def plan_transfers(self, required, batch: int, head: int) -> TransferPlan:
        return self.plan_batch({(batch, head): set(required)})[(batch, head)]

    def apply_transfers(self, plan: TransferPlan, mover=None):
        from .errors import StalePlan
        if plan.version != self.version:
            raise StalePlan(f"plan was built at table version {plan.version}, manager is at {self.version}")
        if mover is not None:
            for key in plan.evict:
                mover(key, (FAST, key[1], None), (SLOW, key[1], None))
            for key in plan.fetch:
                mover(key, (SLOW, key[1], None), (FAST, key[1], self.lookup(*key)[2]))
        if plan.fetch:  # move the payload of this plan's misses (K3)
            with torch.cuda.device(self._engine.device):
                self._engine._call(_lib.lib.nosa_gather, 0, _lib.GATHER["uva"], _lib.stream_ptr())

    def lookup(self, batch: int, head: int, block_index: int):
        if not 0 <= block_index < self.slow_blocks:
            return None
        slot_of, _ = self._engine.residency(0, batch, head)
        s = int(slot_of[block_index])
        return (FAST, head, s) if s >= 0 else (SLOW, head, block_index)

    def fast_resident(self, batch: int, head: int) -> set[int]:
        return self._engine.fast_resident(0, batch, head)

    def residency_stats(self) -> ResidencyStats:
        return self._engine.residency_stats()

    def reset_stats(self):
        self._engine.reset_stats()
