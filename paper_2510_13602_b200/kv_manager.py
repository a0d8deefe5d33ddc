"""GPU-resident two-tier block managers.

`TieredBlockManager` is the reference class (kv_manager.py:130-363) as a drop-in: the same
constructor `(fast: PhysicalLayout, slow: PhysicalLayout, store_payload=False,
eviction_policy=least_recently_required)`, the same table operations (allocate / lookup /
free_block with exclusive FAST / SLOW residency and per-(tier, head) LIFO slot lists), the same
plan-then-apply contract (plan_transfers ticks the clock and stamps recency but moves nothing;
apply_transfers rejects stale plans and performs the moves), the same payload, statistics, audit
and CSV dump.  Its tables, recency clock, victim selection, moves and payload live on the GPU
(csrc/nosa_manager.cu); this class only maps the reference's (batch, head, block) keys onto the
device's dense ids.

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

import ctypes
import json

from .config import AttentionConfig
from .engine import NosaEngine, ResidencyStats
from .errors import CapacityExceeded, DuplicateKey, LayoutMismatch, ManagerError, OutOfBlocks, StalePlan, UnknownKey
from . import _lib

FAST, SLOW = "fast", "slow"
_ELEMENT_DTYPES = {2: np.float16, 4: np.float32}
_TIER_ID = {FAST: 0, SLOW: 1}
_TIER_NAME = {0: FAST, 1: SLOW}


@dataclass(frozen=True)
class PhysicalLayout:
    """Slot geometry of one memory tier (kv_manager.py:59-81)."""

    tier: str
    num_blocks: int          # slots per head
    heads: int
    n_b: int
    d_head: int
    element_width: int = 2   # bytes per element (2 or 4)

    def __post_init__(self):
        if self.tier not in (FAST, SLOW):
            raise ValueError(f"tier must be '{FAST}' or '{SLOW}'")
        if self.num_blocks < 0 or self.heads <= 0 or self.n_b <= 0 or self.d_head <= 0:
            raise ValueError("layout dimensions must be positive (num_blocks may be 0)")
        if self.element_width not in _ELEMENT_DTYPES:
            raise ValueError("element_width must be 2 or 4 bytes")

    @property
    def bytes_per_block(self) -> int:
        return 2 * self.n_b * self.d_head * self.element_width


@dataclass
class RefResidencyStats:
    """kv_manager.ResidencyStats (kv_manager.py:101-122)."""

    hits: int = 0
    misses: int = 0
    bytes_up: int = 0
    bytes_down: int = 0
    steps: int = 0

    @property
    def hit_rate(self) -> float:
        total = self.hits + self.misses
        return 1.0 if total == 0 else self.hits / total

    def to_dict(self) -> dict:
        return {"hit_rate": self.hit_rate, "hits": self.hits, "misses": self.misses, "bytes_up": self.bytes_up,
                "bytes_down": self.bytes_down, "steps": self.steps}


def least_recently_required(candidates, last_required):
    """The default victim order (kv_manager.py:125-127): oldest requirement first, then (batch,
    block).  The device applies exactly this order; TieredBlockManager accepts no other policy."""
    return sorted(candidates, key=lambda key: (last_required.get(key, 0), key[0], key[2]))


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


class TieredBlockManager:
    """kv_manager.TieredBlockManager (kv_manager.py:130-363) with its state on the GPU.

    Behaviour follows the reference call for call: the same slots from the same LIFO lists, the
    same fetch and victim lists, the same exceptions (LayoutMismatch, DuplicateKey, OutOfBlocks,
    UnknownKey, CapacityExceeded, StalePlan) and the same side effects of a failing call.  A custom
    `mover(key, src, dst)` is called once per move in the reference's order with the same
    (tier, head, slot) locations, after the device has executed the plan.  The default
    least-recently-required victim order runs on the device (a radix select over the head's fast
    keys).  A caller-supplied `eviction_policy(candidates, last_required)` (kv_manager.py:133-138)
    is user code and runs on the host: the device plans the fetches and stamps recency, hands back
    the evictable fast keys, and the policy's first `shortfall` keys become the victims
    (kv_manager.py:236-250).  Its `last_required` map holds the planned head's keys with a nonzero
    clock (the reference passes every head's)."""

    def __init__(self, fast: PhysicalLayout, slow: PhysicalLayout, store_payload: bool = False,
                 eviction_policy=least_recently_required, device: int = 0):
        if fast.tier != FAST or slow.tier != SLOW:
            raise LayoutMismatch("pass layouts as (fast, slow)")
        self.eviction_policy = eviction_policy
        for attr in ("heads", "n_b", "d_head", "element_width"):
            if getattr(fast, attr) != getattr(slow, attr):
                raise LayoutMismatch(f"tiers disagree on {attr}")
        self.layouts = {FAST: fast, SLOW: slow}
        self.heads = fast.heads
        self._cap = fast.num_blocks + slow.num_blocks       # keys a head can map
        self._ids = [dict() for _ in range(self.heads)]      # (batch, head, block) -> device id
        self._keys = [dict() for _ in range(self.heads)]     # device id -> key
        self._free_ids = [list(range(self._cap - 1, -1, -1)) for _ in range(self.heads)]
        self.device = device
        self.store_payload = store_payload
        self.version = 0
        self.stats = RefResidencyStats()
        h = ctypes.c_void_p()
        rc = _lib.lib.nosa_mgr_create(self.heads, fast.num_blocks, slow.num_blocks, fast.n_b, fast.d_head,
                                      fast.element_width, int(store_payload), device, ctypes.byref(h))
        if rc != _lib.NOSA_OK:
            raise RuntimeError(f"nosa_mgr_create failed with status {rc}")
        self._h = h
        I32 = lambda n: (ctypes.c_int32 * max(n, 1))()
        self._buf = [I32(self._cap) for _ in range(3)]      # call scratch: ids in, fetch, evict
        self._moves = I32(4 * self._cap)
        self._cand = I32(fast.num_blocks)

    def _call(self, fn, *args):
        _lib.check(fn(self._h, *args), mgr=self._h)

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib.nosa_mgr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def bytes_per_block(self) -> int:
        return self.layouts[FAST].bytes_per_block

    # -- table operations (kv_manager.py:171-201) ------------------------------------------------
    def allocate(self, tier: str, batch: int, head: int, block_index: int) -> int:
        key = (batch, head, block_index)
        ids = self._ids[head]
        if key in ids:
            loc = self.lookup(*key)
            raise DuplicateKey(f"{key} already mapped to {(loc[0], loc[2])}")
        if not self._free_ids[head]:
            raise OutOfBlocks(f"{tier} tier has no free slot for head {head}")
        kid = self._free_ids[head].pop()
        slot = ctypes.c_int32()
        try:
            self._call(_lib.lib.nosa_mgr_allocate, _TIER_ID[tier], head, kid, batch, block_index, ctypes.byref(slot))
        except OutOfBlocks:
            self._free_ids[head].append(kid)
            raise OutOfBlocks(f"{tier} tier has no free slot for head {head}") from None
        ids[key] = kid
        self._keys[head][kid] = key
        self.version += 1
        return slot.value

    def lookup(self, batch: int, head: int, block_index: int):
        """(tier, head, slot) or None when the key is unmapped."""
        kid = self._ids[head].get((batch, head, block_index)) if 0 <= head < self.heads else None
        if kid is None:
            return None
        t, s = ctypes.c_int32(), ctypes.c_int32()
        self._call(_lib.lib.nosa_mgr_lookup, head, kid, ctypes.byref(t), ctypes.byref(s))
        return (_TIER_NAME[t.value], head, s.value)

    def free_block(self, batch: int, head: int, block_index: int):
        key = (batch, head, block_index)
        kid = self._ids[head].pop(key, None)
        if kid is None:
            raise UnknownKey(f"{key} is not mapped")
        self._call(_lib.lib.nosa_mgr_free, head, kid)
        del self._keys[head][kid]
        self._free_ids[head].append(kid)
        self.version += 1

    # -- transfer planning (kv_manager.py:205-298) -----------------------------------------------
    def plan_transfers(self, required, batch: int, head: int) -> TransferPlan:
        required = sorted(set(int(b) for b in required))
        ids = self._ids[head]
        n = len(required)
        buf = self._buf[0] if n <= self._cap else (ctypes.c_int32 * n)()
        for i, b in enumerate(required):
            buf[i] = ids.get((batch, head, b), -1)
        nf, ne, hits = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        custom = self.eviction_policy is not least_recently_required
        nc = ctypes.c_int32()
        try:
            if custom:
                self._call(_lib.lib.nosa_mgr_plan_policy, head, batch, buf, n, self._buf[1], ctypes.byref(nf),
                           ctypes.byref(ne), self._cand, ctypes.byref(nc), ctypes.byref(hits))
            else:
                self._call(_lib.lib.nosa_mgr_plan, head, batch, buf, n, self._buf[1], ctypes.byref(nf),
                           self._buf[2], ctypes.byref(ne), ctypes.byref(hits))
        except UnknownKey:
            bad = next((batch, head, b) for b in required if (batch, head, b) not in ids)
            raise UnknownKey(f"required block {bad} exists in no tier") from None
        keys = self._keys[head]
        fetch = [keys[self._buf[1][i]] for i in range(nf.value)]
        if custom:
            evict = []
            shortfall = ne.value
            if shortfall > 0:  # kv_manager.py:234-250
                evictable = self.eviction_policy([keys[self._cand[i]] for i in range(nc.value)],
                                                 self._last_required(head))
                if shortfall > len(evictable):
                    raise CapacityExceeded(f"need {shortfall} evictions for head {head} but only "
                                           f"{len(evictable)} blocks are evictable")
                evict = list(evictable[:shortfall])
        else:
            evict = [keys[self._buf[2][i]] for i in range(ne.value)]
        bpb = self.bytes_per_block
        return TransferPlan(fetch=fetch, evict=evict, bytes_up=len(fetch) * bpb, bytes_down=len(evict) * bpb,
                            hits=hits.value, misses=len(fetch), version=self.version)

    def _last_required(self, head: int) -> dict:
        """The head's keys with a nonzero last-required clock (the reference's `last_required`)."""
        last = np.empty(max(self._cap, 1), np.uint32)
        self._call(_lib.lib.nosa_mgr_recency, head, last.ctypes.data)
        return {key: int(last[kid]) for kid, key in self._keys[head].items() if last[kid]}

    def apply_transfers(self, plan: TransferPlan, mover=None):
        if plan.version != self.version:
            raise StalePlan(f"plan was built at table version {plan.version}, manager is at {self.version}")
        moves = list(plan.evict) + list(plan.fetch)
        if moves:
            head = moves[0][1]
            if any(k[1] != head for k in moves):
                raise ValueError("a plan moves the keys of one head")
            ids = self._ids[head]
            ev = (ctypes.c_int32 * max(len(plan.evict), 1))(*[ids[k] for k in plan.evict])
            fe = (ctypes.c_int32 * max(len(plan.fetch), 1))(*[ids[k] for k in plan.fetch])
            self._call(_lib.lib.nosa_mgr_apply, head, ev, len(plan.evict), fe, len(plan.fetch), int(mover is None),
                       self._moves)
            for i, key in enumerate(moves):
                src, dst = self._moves[2 * i], self._moves[2 * i + 1]
                if src < 0:
                    continue  # the key was already in the destination tier (kv_manager.py:284-285)
                if mover is not None:
                    s_tier, d_tier = (FAST, SLOW) if i < len(plan.evict) else (SLOW, FAST)
                    mover(key, (s_tier, head, src), (d_tier, head, dst))
                self.version += 1
        self.stats.hits += plan.hits
        self.stats.misses += plan.misses
        self.stats.bytes_up += plan.bytes_up
        self.stats.bytes_down += plan.bytes_down
        self.stats.steps += 1

    # -- payload access (kv_manager.py:305-321) -------------------------------------------------
    def _block(self, batch, head, block_index, data, write):
        if not self.store_payload:
            raise ManagerError("manager was created without payload storage")
        kid = self._ids[head].get((batch, head, block_index))
        if kid is None:
            raise UnknownKey(f"({batch}, {head}, {block_index}) is not mapped")
        self._call(_lib.lib.nosa_mgr_block, head, kid, data.ctypes.data, int(write))

    def write_block(self, batch: int, head: int, block_index: int, data: np.ndarray):
        lay = self.layouts[FAST]
        buf = np.ascontiguousarray(np.broadcast_to(np.asarray(data, _ELEMENT_DTYPES[lay.element_width]),
                                                   (2, lay.n_b, lay.d_head)))
        self._block(batch, head, block_index, buf, True)

    def read_block(self, batch: int, head: int, block_index: int) -> np.ndarray:
        lay = self.layouts[FAST]
        buf = np.empty((2, lay.n_b, lay.d_head), _ELEMENT_DTYPES[lay.element_width])
        self._block(batch, head, block_index, buf, False)
        return buf

    # -- statistics and auditing (kv_manager.py:323-363) ----------------------------------------
    def residency_stats(self) -> RefResidencyStats:
        return self.stats

    def write_stats_json(self, path):
        with open(path, "w") as f:
            json.dump(self.stats.to_dict(), f, sort_keys=True, indent=2)
            f.write("\n")

    def reset_stats(self):
        self.stats = RefResidencyStats()

    def _tables(self, head: int):
        tier = np.empty(max(self._cap, 1), np.int8)
        slot = np.empty(max(self._cap, 1), np.int32)
        self._call(_lib.lib.nosa_mgr_tables, head, tier.ctypes.data, slot.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        return tier, slot

    @property
    def table(self) -> dict:
        """key -> (tier, slot), read back from the device (the reference's `table` dict)."""
        out = {}
        for h in range(self.heads):
            tier, slot = self._tables(h)
            for kid, key in self._keys[h].items():
                out[key] = (_TIER_NAME[int(tier[kid])], int(slot[kid]))
        return out

    @property
    def free(self) -> dict:
        """{tier: [free slots of each head]} bottom to top (the reference's LIFO lists)."""
        out = {FAST: [], SLOW: []}
        F, S = self.layouts[FAST].num_blocks, self.layouts[SLOW].num_blocks
        for h in range(self.heads):
            fa, sa = (ctypes.c_int32 * max(F, 1))(), (ctypes.c_int32 * max(S, 1))()
            nf, ns = ctypes.c_int32(), ctypes.c_int32()
            self._call(_lib.lib.nosa_mgr_free_lists, h, fa, ctypes.byref(nf), sa, ctypes.byref(ns))
            out[FAST].append(list(fa[:nf.value]))
            out[SLOW].append(list(sa[:ns.value]))
        return out

    def fast_resident(self, batch: int, head: int) -> set[int]:
        tier, _ = self._tables(head)
        return {key[2] for kid, key in self._keys[head].items() if key[0] == batch and tier[kid] == 0}

    def audit(self):
        """Verify the slot partition on the device (kv_manager.py:341-363) and the key index."""
        bad = ctypes.c_int32()
        self._call(_lib.lib.nosa_mgr_audit, ctypes.byref(bad))
        if bad.value:
            raise ManagerError(f"slot partition broken (device audit bits {bad.value:#x})")
        for h in range(self.heads):
            tier, _ = self._tables(h)
            mapped = {int(i) for i in np.flatnonzero(tier[:self._cap] >= 0)}
            if mapped != set(self._keys[h]):
                raise ManagerError(f"head {h}: key index out of sync with the device table")
        return True

    def dump_table_csv(self, path):
        rows = sorted(self.table.items())
        with open(path, "w") as f:
            f.write("# nosa-sim block-table v1\n")
            f.write("batch,head,block_index,tier,slot\n")
            for (b, h, i), (tier, slot) in rows:
                f.write(f"{b},{h},{i},{tier},{slot}\n")


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
        self.version += 1  # a plan is applied once: applying it again raises StalePlan (kv_manager.py:269-273)
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
