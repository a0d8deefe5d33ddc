"""NosaEngine — the batched, GPU-resident NOSA offloaded decode step.

One engine owns a batch of sequences x layers x KV heads on one GPU and replaces, for all of
them at once:
  * DecodeEngine.prefill / start_run / step   (decode.py:106-194)
  * the residency loop of simulate_decode      (offload_sim.py:254-299) with one
    TieredBlockManager per sequence             (kv_manager.py:130-305)
Each step runs, per layer: K1+K2 selection + cache plan, K3 miss gather (pinned host ->
HBM on a side stream), K4+K5 block-sparse attention + append.  Q/K/V are supplied directly
(the engine starts after the projections; SURVEY.md §8f row 1 moves them in).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .config import AttentionConfig
from .selection import BlockGeometry, SelectionResult, make_result

SELECTORS = ("nosa", "infllmv2")
_TORCH_DTYPE = {"bf16": torch.bfloat16, "fp32": torch.float32}


@dataclass
class ResidencyStats:
    """kv_manager.ResidencyStats (kv_manager.py:101-122) plus the new-block and eviction counts."""

    hits: int = 0
    misses: int = 0
    bytes_up: int = 0
    bytes_down: int = 0
    steps: int = 0
    new_blocks: int = 0
    evictions: int = 0
    candidates: int = 0   # pool rows rescored in f64 by the screened selector
    topk_required: int = 0  # required blocks picked from the selection pool (top-k)
    topk_misses: int = 0    # fetches among them

    @property
    def hit_rate(self) -> float:
        total = self.hits + self.misses
        return 1.0 if total == 0 else self.hits / total

    @property
    def hit_rate_topk(self) -> float:
        """Top-k blocks that were already fast-resident (offload_sim.py:291-293, 314)."""
        return 1.0 if self.topk_required == 0 else 1.0 - self.topk_misses / self.topk_required

    def to_dict(self) -> dict:
        return {"hit_rate": self.hit_rate, "hits": self.hits, "misses": self.misses,
                "bytes_up": self.bytes_up, "bytes_down": self.bytes_down, "steps": self.steps}


@dataclass
class TransferPlanView:
    """Executed TransferPlan of one (layer, sequence, head) (kv_manager.py:84-98)."""

    fetch: list[int]
    evict: list[int]
    hits: int
    bytes_per_block: int

    @property
    def misses(self) -> int:
        return len(self.fetch)

    @property
    def bytes_up(self) -> int:
        return len(self.fetch) * self.bytes_per_block

    @property
    def bytes_down(self) -> int:
        return len(self.evict) * self.bytes_per_block


@dataclass
class StepOutput:
    """decode.StepOutput (decode.py:78-82) for a whole batch and all layers."""

    step: list[int]
    outputs: torch.Tensor                     # [layers][batch][n_head][d_head] float32
    selections: list = field(default_factory=list)


class NosaEngine:
    def __init__(self, config: AttentionConfig, *, batch: int, max_tokens: int, fast_slots: int,
                 w1, w2, layers: int = 1, variant: str = "ed-dma", dtype: str = "bf16",
                 device: int = 0, residency: str = "per-sequence", attend_chunk: int = 0,
                 attend_layers: int = 0, exact_scan: bool = False, slow_tier: str = "host"):
        """residency "per-sequence": one manager per (layer, sequence, head) with `fast_slots`
        slots; "shared": one pool of batch*fast_slots slots per (layer, head)
        shared by the batch and planned in batch order, the reference simulator's residency.
        attend_chunk: KV blocks per split-K attention work item (1..8, 0 = chosen from the
        batch size); outputs are bit-identical across runs with the same value.
        attend_layers: layers per persistent attention launch in the pipelined schedule (0 =
        8 when every block fits in HBM, else 1); results do not depend on it.
        exact_scan: score the whole pool in f64 instead of the screened selector (bf16 pre-scan,
        f64 rescoring of the candidates); both pick the same blocks.
        slow_tier: "host" (pinned host memory over PCIe, the reference's SLOW tier) or
        "peer:<device>" (that GPU's HBM over NVLink; the engine's own device = loopback)."""
        if variant not in _lib.VARIANT:
            raise ValueError(f"variant must be one of {tuple(_lib.VARIANT)} (retaining needs hidden states)")
        if residency not in _lib.RESIDENCY:
            raise ValueError(f"residency must be one of {tuple(_lib.RESIDENCY)}")
        self.residency_mode = residency
        if dtype not in _lib.DTYPE:
            raise ValueError(f"dtype must be one of {tuple(_lib.DTYPE)}")
        self.config = config
        self.batch, self.layers, self.max_tokens, self.fast_slots = batch, layers, max_tokens, fast_slots
        self.variant, self.dtype = variant, dtype
        self.device = torch.device("cuda", device)
        self.tdtype = _TORCH_DTYPE[dtype]
        c = _lib.NosaConfig()
        for name in ("n", "d", "n_head", "n_kv_head", "d_head", "n_b", "n_s", "n_w", "k", "k_q", "k_e"):
            setattr(c, name, getattr(config, name))
        c.accounting = 0 if config.accounting == "inclusive" else 1
        c.batch, c.layers, c.max_tokens, c.fast_slots = batch, layers, max_tokens, fast_slots
        c.dtype, c.variant = _lib.DTYPE[dtype], _lib.VARIANT[variant]
        c.residency = _lib.RESIDENCY[residency]
        c.attend_chunk = attend_chunk
        c.attend_layers = attend_layers
        c.exact_scan = int(exact_scan)
        if slow_tier == "host":
            c.slow_tier_device = -1
        elif slow_tier.startswith("peer:") and slow_tier[5:].isdigit():
            c.slow_tier_device = int(slow_tier[5:])
        else:
            raise ValueError(f"slow_tier must be 'host' or 'peer:<device>', got {slow_tier!r}")
        self.slow_tier = slow_tier
        self._cfg = c
        msg = ctypes.create_string_buffer(512)
        if _lib.lib.nosa_config_validate(ctypes.byref(c), msg, 512) != _lib.NOSA_OK:
            raise ValueError(msg.value.decode())
        handle = ctypes.c_void_p()
        _lib.check(_lib.lib.nosa_ctx_create(ctypes.byref(c), device, ctypes.byref(handle)))
        self._ctx = handle
        w1 = np.ascontiguousarray(w1, dtype=np.float64)
        w2 = np.ascontiguousarray(w2, dtype=np.float64).reshape(-1)
        if w1.shape != (config.d_head, config.n_head) or w2.shape != (config.n_head,):
            raise ValueError(f"eviction head must be w1 ({config.d_head}, {config.n_head}) and w2 ({config.n_head},)")
        self._call(_lib.lib.nosa_set_eviction_head,
                   w1.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                   w2.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        self.max_blocks = -(-max_tokens // config.n_b)
        self.bytes_per_block = 2 * config.n_b * config.d_head * (2 if dtype == "bf16" else 4)
        self.geometry: list[BlockGeometry | None] = [None] * batch
        self._t = np.zeros((layers, batch), dtype=np.int64)
        self._graph_io = None
        self.screened = not exact_scan and config.d_head in (64, 128) and not os.environ.get("NOSA_EXACT_SCAN")

    # ------------------------------------------------------------------ plumbing
    def _call(self, fn, *args):
        _lib.check(fn(self._ctx, *args), self._ctx)

    def close(self):
        if getattr(self, "_ctx", None):
            torch.cuda.synchronize(self.device)
            _lib.lib.nosa_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _dev(self, x, dtype=None) -> torch.Tensor:
        dtype = dtype or self.tdtype
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x))
        return x.to(device=self.device, dtype=dtype).contiguous()

    @property
    def launch_count(self) -> int:
        return int(_lib.lib.nosa_launch_count(self._ctx))

    def memory(self) -> tuple[int, int]:
        d, h = ctypes.c_int64(), ctypes.c_int64()
        self._call(_lib.lib.nosa_ctx_memory, ctypes.byref(d), ctypes.byref(h))
        return d.value, h.value

    # ------------------------------------------------------------------ run setup
    def prefill(self, k, v, layer: int | None = None, seq_begin: int = 0, resident: bool = False):
        """Cache a prefix (DecodeEngine.prefill, decode.py:139-146).

        k, v: [layers][S][n_kv_head][t][d_head] (layer=None) or [S][n_kv_head][t][d_head].
        Every block starts in the slow tier (offload_sim.py:262-266); resident=True also places
        all of them in HBM slots (the all-resident configuration)."""
        k = self._dev(k)
        v = self._dev(v)
        if layer is None:
            if k.dim() != 5:
                raise ValueError("prefill over all layers expects [layers][S][H][t][D]")
            for l in range(k.shape[0]):
                self.prefill(k[l], v[l], layer=l, seq_begin=seq_begin, resident=resident)
            return
        if k.dim() != 4 or k.shape != v.shape:
            raise ValueError("prefill expects k, v of shape [S][n_kv_head][t][d_head]")
        S, H, t, D = k.shape
        if H != self.config.n_kv_head or D != self.config.d_head:
            raise ValueError(f"k has {H} heads of width {D}, expected {self.config.n_kv_head} x {self.config.d_head}")
        if t > self.max_tokens:
            raise ValueError("head cache capacity exhausted")
        with torch.cuda.device(self.device):
            fn = _lib.lib.nosa_prefill_resident if resident else _lib.lib.nosa_prefill
            self._call(fn, layer, seq_begin, S, k.data_ptr(), v.data_ptr(), t, _lib.stream_ptr())
            torch.cuda.current_stream().synchronize()
        self._t[layer, seq_begin:seq_begin + S] = t
        for b in range(seq_begin, seq_begin + S):
            self.geometry[b] = None

    def start_run(self, seq_begin: int = 0, seq_count: int | None = None):
        """Freeze the geometry at the current length (DecodeEngine.start_run, decode.py:148-150)."""
        seq_count = self.batch - seq_begin if seq_count is None else seq_count
        if (self._t[:, seq_begin:seq_begin + seq_count] != self._t[0:1, seq_begin:seq_begin + seq_count]).any():
            raise RuntimeError("all layers of a sequence must hold the same number of tokens")
        with torch.cuda.device(self.device):
            self._call(_lib.lib.nosa_start_run, seq_begin, seq_count, _lib.stream_ptr())
        for b in range(seq_begin, seq_begin + seq_count):
            self.geometry[b] = BlockGeometry.for_run(self.config, int(self._t[0, b]))

    # ------------------------------------------------------------------ decode step
    def _check_step(self):
        if any(g is None for g in self.geometry):
            self.start_run()
        if (self._t <= 0).any():
            raise ValueError("softmax over empty support: all scores are -inf (empty cache)")
        if (self._t >= self.max_tokens).any():
            raise ValueError("head cache capacity exhausted")

    def _mover(self, gather: str, graph: bool = False) -> str:
        """"auto": the SM zero-copy gather (`uva`), device-driven and graph-capturable, for every
        tier.  `hostpack` (host-packed chunks over the copy engine, eager steps only), `memcpy`
        (one host-submitted copy-engine copy per block, host-bound) and `tma` stay selectable
        (DESIGN.md §5)."""
        return "uva" if gather == "auto" else gather

    def step(self, q, k_new, v_new, selector: str = "nosa", out: torch.Tensor | None = None,
             gather: str = "auto", check: bool = True, schedule: str = "pipelined") -> torch.Tensor:
        """One decode step of every layer (DecodeEngine.step, decode.py:152-190).

        q: [layers][batch][n_head][d_head]; k_new, v_new: [layers][batch][n_kv_head][d_head].
        Returns out [layers][batch][n_head][d_head] float32 (attention over tokens [0, t)).
        gather: "auto" (see _mover), "uva" (zero-copy SM kernel), "tma" (TMA bulk kernel),
        "hostpack" (host threads pack the misses into 2 MiB chunks, one DMA each) or "memcpy"
        (one copy-engine copy per block).
        schedule: "pipelined" overlaps layer l's gather with the scoring of later layers;
        "serial" runs layer by layer (results are identical)."""
        if selector not in SELECTORS:
            raise ValueError(f"selector must be one of {SELECTORS}")
        gather = self._mover(gather)
        if gather not in _lib.GATHER or schedule not in _lib.SCHEDULE:
            raise ValueError(f"gather must be one of {tuple(_lib.GATHER)}, schedule one of {tuple(_lib.SCHEDULE)}")
        self._check_step()
        L, B, cfg = self.layers, self.batch, self.config
        q = self._dev(q).reshape(L, B, cfg.n_head, cfg.d_head)
        k_new = self._dev(k_new).reshape(L, B, cfg.n_kv_head, cfg.d_head)
        v_new = self._dev(v_new).reshape(L, B, cfg.n_kv_head, cfg.d_head)
        if out is None:
            out = torch.empty((L, B, cfg.n_head, cfg.d_head), dtype=torch.float32, device=self.device)
        io = _lib.NosaStepIO(q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), out.data_ptr(),
                             _lib.SELECTOR[selector], _lib.GATHER[gather], _lib.SCHEDULE[schedule])
        with torch.cuda.device(self.device):
            self._call(_lib.lib.nosa_decode_step, ctypes.byref(io), _lib.stream_ptr())
        self._t += 1
        if check:
            self.check_errors()
        return out

    def step_host(self, q, k_new, v_new, selector: str = "nosa", out: torch.Tensor | None = None,
                  gather: str = "auto", schedule: str = "pipelined", sync: bool = True) -> torch.Tensor:
        """`step` on host tensors (the reference's calling convention: host arrays in, host
        array out).  q/k_new/v_new: CPU tensors of the engine dtype in the `step` layouts, pinned
        for asynchronous copies.  Layer l's inputs are copied in ahead of the miss gathers and
        its output is copied back while later layers run.  Returns `out`, a CPU float32
        [layers][batch][n_head][d_head] (pinned if allocated here); with sync=False it is only
        complete once torch's current stream reaches this point."""
        if selector not in SELECTORS:
            raise ValueError(f"selector must be one of {SELECTORS}")
        gather = self._mover(gather)
        if gather not in _lib.GATHER or schedule not in _lib.SCHEDULE:
            raise ValueError(f"gather must be one of {tuple(_lib.GATHER)}, schedule one of {tuple(_lib.SCHEDULE)}")
        self._check_step()
        L, B, cfg = self.layers, self.batch, self.config
        dt = _TORCH_DTYPE[self.dtype]
        shapes = ((L, B, cfg.n_head, cfg.d_head), (L, B, cfg.n_kv_head, cfg.d_head), (L, B, cfg.n_kv_head, cfg.d_head))
        host = []
        for name, x, shp in zip(("q", "k_new", "v_new"), (q, k_new, v_new), shapes):
            if isinstance(x, np.ndarray):
                x = torch.from_numpy(np.ascontiguousarray(x))
            if not isinstance(x, torch.Tensor) or x.device.type != "cpu":
                raise ValueError(f"{name} must be a host array or CPU tensor")
            if x.dtype != dt or not x.is_contiguous():  # converted once here; pass pinned dt tensors to avoid it
                x = x.to(dt).contiguous().pin_memory()
            if x.numel() != int(np.prod(shp)):
                raise ValueError(f"{name} has {x.numel()} elements, expected {shp}")
            host.append(x)
        q, k_new, v_new = host
        # the staging kernel reads these after this call returns (sync=False): converted copies
        # must outlive the step, or the caching host allocator could hand their pages out again
        self._host_keep = host
        if out is None:
            out = torch.empty((L, B, cfg.n_head, cfg.d_head), dtype=torch.float32, pin_memory=True)
        elif out.device.type != "cpu" or out.dtype != torch.float32 or not out.is_contiguous() \
                or out.numel() != L * B * cfg.n_head * cfg.d_head:
            raise ValueError("out must be a contiguous CPU float32 tensor of the output shape")
        io = _lib.NosaHostStepIO(q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), out.data_ptr(),
                                 _lib.SELECTOR[selector], _lib.GATHER[gather], _lib.SCHEDULE[schedule])
        with torch.cuda.device(self.device):
            self._call(_lib.lib.nosa_decode_step_host, ctypes.byref(io), _lib.stream_ptr())
            self._t += 1
            if sync:
                torch.cuda.current_stream().synchronize()
                self.check_errors()
        return out

    def set_projection(self, layer: int, w_q, w_k, w_v):
        """The QKV projection of one layer for step_hidden (project_qkv, attention.py:67-90):
        w_q [d][n_head*d_head], w_k, w_v [d][n_kv_head*d_head], kept on the device as one bf16
        [n][d] matrix (the K-major operand of the tcgen05 GEMM)."""
        w = np.concatenate([np.asarray(w_q), np.asarray(w_k), np.asarray(w_v)], axis=1)
        w_t = torch.as_tensor(np.ascontiguousarray(w.T), dtype=torch.float32).to(
            device=self.device, dtype=torch.bfloat16).contiguous()
        if not hasattr(self, "_proj_w"):
            self._proj_w = [None] * self.layers
        self._call(_lib.lib.nosa_set_projection, layer, w_t.data_ptr(), w.shape[0], w.shape[1],
                   np.asarray(w_q).shape[1], np.asarray(w_k).shape[1])
        self._proj_w[layer] = w_t  # (the context keeps its own copy)
        self.hidden_dim = w.shape[0]

    def _hidden_io(self, h, out, selector, gather, schedule):
        L, B, cfg = self.layers, self.batch, self.config
        h = self._dev(h, torch.bfloat16).reshape(L, B, self.hidden_dim)
        if out is None:
            out = torch.empty((L, B, cfg.n_head, cfg.d_head), dtype=torch.float32, device=self.device)
        io = _lib.NosaHiddenStepIO(h.data_ptr(), out.data_ptr(), _lib.SELECTOR[selector], _lib.GATHER[gather],
                                   _lib.SCHEDULE[schedule])
        return h, out, io

    def step_hidden(self, h, selector: str = "nosa", out: torch.Tensor | None = None, gather: str = "auto",
                    check: bool = True, schedule: str = "pipelined") -> torch.Tensor:
        """One decode step of every layer from hidden states h [layers][batch][d] (the input of
        DecodeEngine.step, decode.py:152-190): q/k/v are projected on the tensor cores with the
        weights of set_projection, then the step runs as `step` would on them."""
        if selector not in SELECTORS:
            raise ValueError(f"selector must be one of {SELECTORS}")
        gather = self._mover(gather)
        self._check_step()
        h, out, io = self._hidden_io(h, out, selector, gather, schedule)
        self._hidden_keep = h
        with torch.cuda.device(self.device):
            self._call(_lib.lib.nosa_decode_step_hidden, ctypes.byref(io), _lib.stream_ptr())
        self._t += 1
        if check:
            self.check_errors()
        return out

    def step_hidden_host(self, h, selector: str = "nosa", out: torch.Tensor | None = None, gather: str = "auto",
                         schedule: str = "pipelined", sync: bool = True) -> torch.Tensor:
        """`step_hidden` on host tensors (DecodeEngine.step(h_t)'s convention, decode.py:152-190):
        h a CPU bf16 [layers][batch][d] (pinned: the GPU stages each selection group's rows with
        zero-copy loads), out a CPU float32 [layers][batch][n_head][d_head] filled per attention
        batch while later layers run.  With sync=False `out` is complete once torch's current
        stream reaches this point."""
        if selector not in SELECTORS:
            raise ValueError(f"selector must be one of {SELECTORS}")
        gather = self._mover(gather)
        self._check_step()
        L, B, cfg = self.layers, self.batch, self.config
        if isinstance(h, np.ndarray):
            h = torch.from_numpy(np.ascontiguousarray(h))
        if not isinstance(h, torch.Tensor) or h.device.type != "cpu":
            raise ValueError("h must be a host array or CPU tensor")
        if h.dtype != torch.bfloat16 or not h.is_contiguous():
            h = h.to(torch.bfloat16).contiguous().pin_memory()
        if h.numel() != L * B * self.hidden_dim:
            raise ValueError(f"h has {h.numel()} elements, expected {(L, B, self.hidden_dim)}")
        if out is None:
            out = torch.empty((L, B, cfg.n_head, cfg.d_head), dtype=torch.float32, pin_memory=True)
        elif out.device.type != "cpu" or out.dtype != torch.float32 or not out.is_contiguous() \
                or out.numel() != L * B * cfg.n_head * cfg.d_head:
            raise ValueError("out must be a contiguous CPU float32 tensor of the output shape")
        io = _lib.NosaHiddenStepIO(h.data_ptr(), out.data_ptr(), _lib.SELECTOR[selector], _lib.GATHER[gather],
                                   _lib.SCHEDULE[schedule])
        self._hidden_keep = h
        with torch.cuda.device(self.device):
            self._call(_lib.lib.nosa_decode_step_hidden_host, ctypes.byref(io), _lib.stream_ptr())
            self._t += 1
            if sync:
                torch.cuda.current_stream().synchronize()
                self.check_errors()
        return out

    def capture_hidden(self, h: torch.Tensor, out: torch.Tensor, selector: str = "nosa", gather: str = "auto",
                       schedule: str = "pipelined"):
        """Capture one step_hidden on fixed device buffers as a CUDA graph; replay() re-runs it."""
        self._check_step()
        gather = self._mover(gather, graph=True)
        h, out, io = self._hidden_io(h, out, selector, gather, schedule)
        self._graph_bufs = (h, out)
        with torch.cuda.device(self.device):
            self._call(_lib.lib.nosa_step_graph_capture_hidden, ctypes.byref(io))

    def step_layer(self, layer: int, q, k_new, v_new, selector: str = "nosa", out=None,
                   gather: str = "auto") -> torch.Tensor:
        """The same step for one layer, stage by stage through the C ABI."""
        if selector not in SELECTORS:
            raise ValueError(f"selector must be one of {SELECTORS}")
        self._check_step()
        cfg = self.config
        q = self._dev(q).reshape(self.batch, cfg.n_head, cfg.d_head)
        k_new = self._dev(k_new).reshape(self.batch, cfg.n_kv_head, cfg.d_head)
        v_new = self._dev(v_new).reshape(self.batch, cfg.n_kv_head, cfg.d_head)
        if out is None:
            out = torch.empty((self.batch, cfg.n_head, cfg.d_head), dtype=torch.float32, device=self.device)
        s = _lib.stream_ptr
        gather = self._mover(gather)
        with torch.cuda.device(self.device):
            self._call(_lib.lib.nosa_select_plan, layer, q.data_ptr(), _lib.SELECTOR[selector], s())
            self._call(_lib.lib.nosa_gather, layer, _lib.GATHER[gather], s())
            self._call(_lib.lib.nosa_attend, layer, q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(),
                       out.data_ptr(), s())
        self._t[layer] += 1
        return out

    # ------------------------------------------------------------------ CUDA graph
    def capture(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor, out: torch.Tensor,
                selector: str = "nosa", gather: str = "auto", schedule: str = "pipelined"):
        """Capture one full step on fixed device buffers; replay() re-runs it."""
        gather = self._mover(gather, graph=True)
        self._check_step()
        for x in (q, k_new, v_new, out):
            if not x.is_contiguous() or x.device != self.device:
                raise ValueError("graph buffers must be contiguous tensors on the engine's device")
        self._graph_io = _lib.NosaStepIO(q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), out.data_ptr(),
                                         _lib.SELECTOR[selector], _lib.GATHER[gather], _lib.SCHEDULE[schedule])
        self._graph_bufs = (q, k_new, v_new, out)
        with torch.cuda.device(self.device):
            self._call(_lib.lib.nosa_step_graph_capture, ctypes.byref(self._graph_io))

    def _host_io(self, q, k_new, v_new, out, selector, gather, schedule):
        L, B, cfg = self.layers, self.batch, self.config
        dt = _TORCH_DTYPE[self.dtype]
        for name, x, h in (("q", q, cfg.n_head), ("k_new", k_new, cfg.n_kv_head), ("v_new", v_new, cfg.n_kv_head)):
            if not (isinstance(x, torch.Tensor) and x.device.type == "cpu" and x.is_pinned() and x.dtype == dt
                    and x.is_contiguous() and x.numel() == L * B * h * cfg.d_head):
                raise ValueError(f"{name} must be a pinned contiguous CPU tensor of {dt} with the step's shape")
        if not (out.device.type == "cpu" and out.is_pinned() and out.dtype == torch.float32 and out.is_contiguous()
                and out.numel() == L * B * cfg.n_head * cfg.d_head):
            raise ValueError("out must be a pinned contiguous CPU float32 tensor of the output shape")
        return _lib.NosaHostStepIO(q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), out.data_ptr(),
                                   _lib.SELECTOR[selector], _lib.GATHER[gather], _lib.SCHEDULE[schedule])

    def capture_host(self, q, k_new, v_new, out, selector: str = "nosa", gather: str = "auto",
                     schedule: str = "pipelined"):
        """Capture one host-buffer step (step_host) as a CUDA graph; replay_host() re-runs it on
        these or other pinned buffers of the same shapes."""
        self._check_step()
        gather = self._mover(gather, graph=True)
        io = self._host_io(q, k_new, v_new, out, selector, gather, schedule)
        with torch.cuda.device(self.device):
            self._call(_lib.lib.nosa_step_graph_capture_host, ctypes.byref(io))
        self._host_graph_cfg = (selector, gather, schedule)

    def _check_capacity(self):
        # the graph replays append one token per (layer, seq, head) without a host-side check
        # of their own; the device append also refuses (NOSA_FLAG_CAPACITY) past max_tokens
        if (self._t >= self.max_tokens).any():
            raise ValueError("head cache capacity exhausted")

    def replay_host(self, q, k_new, v_new, out, stream=None):
        self._check_capacity()
        io = self._host_io(q, k_new, v_new, out, *self._host_graph_cfg)
        with torch.cuda.device(self.device):
            self._call(_lib.lib.nosa_step_graph_launch_host, ctypes.byref(io), _lib.stream_ptr(stream))
        self._t += 1
        return out

    def replay(self, stream=None):
        self._check_capacity()
        with torch.cuda.device(self.device):
            self._call(_lib.lib.nosa_step_graph_launch, _lib.stream_ptr(stream))
        self._t += 1

    # ------------------------------------------------------------------ readback
    def check_errors(self):
        flags = ctypes.c_uint32()
        self._call(_lib.lib.nosa_check_errors, ctypes.byref(flags))

    def lengths(self) -> np.ndarray:
        out = np.zeros((self.layers, self.batch), dtype=np.int32)
        self._call(_lib.lib.nosa_read_lengths, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        return out

    def raw_selection(self, layer: int):
        """Arrays of the last selection of a layer: blocks_q, n_q, blocks_e, n_e, required, n_req
        ([batch][n_kv_head][cap]) and the pool scores s_q ([batch][n_kv_head][max_blocks])."""
        B, H = self.batch, self.config.n_kv_head
        cap = max(self.fast_slots, self.config.blocks_topk, 1)
        P = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        bq, be, rq = (np.zeros((B, H, cap), np.int32) for _ in range(3))
        nq, ne, nr = (np.zeros((B, H), np.int32) for _ in range(3))
        sq = np.zeros((B, H, self.max_blocks), np.float64)
        self._call(_lib.lib.nosa_read_selection, layer, cap, P(bq), P(nq), P(be), P(ne), P(rq), P(nr),
                   sq.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        return bq, nq, be, ne, rq, nr, sq

    def selections(self, layer: int = 0) -> list[list[SelectionResult]]:
        """SelectionResult per (sequence, kv head) of the last step of `layer`."""
        bq, nq, be, ne, _, _, _ = self.raw_selection(layer)
        out = []
        for b in range(self.batch):
            t = int(self._t[layer, b]) - 1  # the step was taken before the append
            geom = self.geometry[b]
            row = []
            for h in range(self.config.n_kv_head):
                row.append(make_result(t, self.config.n_b, bq[b, h, :nq[b, h]], be[b, h, :ne[b, h]],
                                       geom.fixed_blocks(t)))
            out.append(row)
        return out

    def plans(self, layer: int = 0) -> list[list[TransferPlanView]]:
        B, H, C = self.batch, self.config.n_kv_head, self.fast_slots
        P = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        f, e = np.zeros((B, H, C), np.int32), np.zeros((B, H, C), np.int32)
        nf, ne, nh = (np.zeros((B, H), np.int32) for _ in range(3))
        self._call(_lib.lib.nosa_read_plan, layer, P(f), P(nf), P(e), P(ne), P(nh))
        return [[TransferPlanView(f[b, h, :nf[b, h]].tolist(), e[b, h, :ne[b, h]].tolist(), int(nh[b, h]),
                                  self.bytes_per_block) for h in range(H)] for b in range(B)]

    def residency(self, layer: int, seq: int, head: int) -> tuple[np.ndarray, np.ndarray]:
        slot_of = np.zeros(self.max_blocks, np.int32)
        block_of = np.zeros(self.fast_slots, np.int32)
        P = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        self._call(_lib.lib.nosa_read_residency, layer, seq, head, P(slot_of), P(block_of))
        return slot_of, block_of

    def fast_resident(self, layer: int, seq: int, head: int) -> set[int]:
        """TieredBlockManager.fast_resident (kv_manager.py:338-339)."""
        slot_of, _ = self.residency(layer, seq, head)
        return {int(b) for b in np.flatnonzero(slot_of >= 0)}

    def block_scores(self, layer: int) -> np.ndarray:
        out = np.zeros((self.batch, self.config.n_kv_head, self.max_blocks), np.float64)
        self._call(_lib.lib.nosa_read_block_scores, layer, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        return out

    def read_kv(self, layer: int, seq: int, head: int, t: int | None = None):
        t = int(self._t[layer, seq]) if t is None else t
        npdt = np.uint16 if self.dtype == "bf16" else np.float32
        k = np.zeros((t, self.config.d_head), npdt)
        v = np.zeros((t, self.config.d_head), npdt)
        self._call(_lib.lib.nosa_read_kv, layer, seq, head, t, k.ctypes.data, v.ctypes.data)
        if self.dtype == "bf16":
            k = (k.astype(np.uint32) << 16).view(np.float32)
            v = (v.astype(np.uint32) << 16).view(np.float32)
        return k, v

    def read_slot(self, layer: int, seq: int, head: int, slot: int) -> np.ndarray:
        npdt = np.uint16 if self.dtype == "bf16" else np.float32
        buf = np.zeros((2, self.config.n_b, self.config.d_head), npdt)
        self._call(_lib.lib.nosa_read_slot, layer, seq, head, slot, buf.ctypes.data)
        if self.dtype == "bf16":
            buf = (buf.astype(np.uint32) << 16).view(np.float32)
        return buf

    def residency_stats(self, layers: range | None = None, seqs: range | None = None) -> ResidencyStats:
        layers = layers or range(self.layers)
        seqs = seqs or range(self.batch)
        st = _lib.NosaStats()
        self._call(_lib.lib.nosa_read_stats, layers.start, layers.stop, seqs.start, seqs.stop, ctypes.byref(st))
        return ResidencyStats(hits=st.hits, misses=st.misses, bytes_up=st.bytes_up, bytes_down=st.bytes_down,
                              steps=st.steps, new_blocks=st.new_blocks, evictions=st.evictions,
                              candidates=st.candidates, topk_required=st.topk_required,
                              topk_misses=st.topk_misses)

    def reset_stats(self):
        with torch.cuda.device(self.device):
            self._call(_lib.lib.nosa_reset_stats, _lib.stream_ptr())

    # ------------------------------------------------------------------ device timing
    KERNEL_KINDS = ("select_plan", "gather", "attend", "finalize")
    COPY_KINDS = ("h2d_in", "d2h_out")  # host-buffer step copies (timing kinds 4, 5)
    PROJECT_KIND = "project"            # QKV projection of step_hidden (timing kind 6)

    def timing_enable(self, max_launches: int):
        """Bracket every kernel of the following eager steps with CUDA events on its stream."""
        self._call(_lib.lib.nosa_timing_enable, max_launches)

    def timing_read(self) -> dict:
        ms = (ctypes.c_double * 7)()
        n = (ctypes.c_int64 * 7)()
        self._call(_lib.lib.nosa_timing_read, ms, n)
        kinds = {k: i for i, k in enumerate(self.KERNEL_KINDS)}
        if n[6]:
            kinds[self.PROJECT_KIND] = 6
        return {k: {"total_ms": ms[i], "launches": n[i], "avg_ms": ms[i] / n[i] if n[i] else 0.0}
                for k, i in kinds.items()}

    def copy_timing_read(self) -> dict:
        """Host<->device copy time of nosa_decode_step_host (kinds 4, 5) since timing_enable."""
        ms = (ctypes.c_double * 7)()
        n = (ctypes.c_int64 * 7)()
        self._call(_lib.lib.nosa_timing_read, ms, n)
        return {k: {"total_ms": ms[4 + i], "copies": n[4 + i]} for i, k in enumerate(self.COPY_KINDS)}

    def ktime_enable(self, on: bool = True):
        """Diagnostics: record the device-clock span of every attention launch."""
        self._call(_lib.lib.nosa_ktime_enable, int(on))

    def ktime_read(self) -> list[float]:
        """Microseconds from the first CTA's start to the last CTA's end of the last attention
        launch of each layer (0.0 = no launch started at that layer); resets."""
        out = np.zeros(self.layers, np.float64)
        self._call(_lib.lib.nosa_ktime_read, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        return out.tolist()

    def timing_trace(self, cap: int = 65536) -> list[tuple[str, float, float]]:
        """(kind, start_ms, end_ms) of every timed launch since timing_enable, in issue order,
        relative to the first launch: the device timeline of the step's streams."""
        kind = np.zeros(cap, np.int32)
        t0, t1 = np.zeros(cap, np.float32), np.zeros(cap, np.float32)
        n = ctypes.c_int32()
        F = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        self._call(_lib.lib.nosa_timing_trace, cap, kind.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), F(t0), F(t1),
                   ctypes.byref(n))
        names = self.KERNEL_KINDS + self.COPY_KINDS + (self.PROJECT_KIND,)
        return [(names[kind[i]], float(t0[i]), float(t1[i])) for i in range(n.value)]
