"""ctypes binding of libnosa_b200.so (include/nosa_b200.h).

This is the reference-side binding INTEGRATION.md describes: plain pointers and sizes, int
status codes mapped onto the reference's exception types (kv_manager.py:31-56, ValueError
for config/shape problems).  There is no fallback: if the shared library is missing the import
fails loudly, and every compute entry point needs a CUDA device.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import CapacityExceeded, OutOfBlocks, UnknownKey

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("NOSA_B200_LIB", _HERE / "libnosa_b200.so"))

NOSA_OK = 0
NOSA_ERR_VALUE = 1
NOSA_ERR_CAPACITY = 2
NOSA_ERR_UNKNOWN_KEY = 3
NOSA_ERR_OUT_OF_BLOCKS = 4
NOSA_ERR_CUDA = 5
NOSA_ERR_STATE = 6

SELECTOR = {"nosa": 0, "infllmv2": 1}
VARIANT = {"ed-dma": 0, "s-dma": 1, "dma": 2}
DTYPE = {"bf16": 0, "fp32": 1}
GATHER = {"uva": 0, "memcpy": 1, "tma": 2, "hostpack": 3, "hybrid": 4}
SCHEDULE = {"pipelined": 0, "serial": 1}
RESIDENCY = {"per-sequence": 0, "shared": 1}


class NosaConfig(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int32) for name in (
        "n", "d", "n_head", "n_kv_head", "d_head", "n_b", "n_s", "n_w", "k", "k_q", "k_e",
        "accounting", "batch", "layers", "max_tokens", "fast_slots", "dtype", "variant", "residency",
        "attend_chunk", "attend_layers", "exact_scan", "slow_tier_device")]


class NosaStats(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int64) for name in (
        "hits", "misses", "new_blocks", "evictions", "steps", "bytes_up", "bytes_down", "candidates",
        "topk_required", "topk_misses")]


class NosaStepIO(ctypes.Structure):
    _fields_ = [("q", ctypes.c_void_p), ("k_new", ctypes.c_void_p), ("v_new", ctypes.c_void_p),
                ("out", ctypes.c_void_p), ("selector", ctypes.c_int32), ("gather_mode", ctypes.c_int32),
                ("schedule", ctypes.c_int32)]


class NosaHostStepIO(NosaStepIO):
    """Same fields as NosaStepIO; the pointers are host addresses (nosa_decode_step_host)."""


class NosaHiddenStepIO(ctypes.Structure):
    _fields_ = [("h", ctypes.c_void_p), ("out", ctypes.c_void_p), ("selector", ctypes.c_int32),
                ("gather_mode", ctypes.c_int32), ("schedule", ctypes.c_int32)]


# every symbol include/nosa_b200.h declares, with its ctypes signature
_P = ctypes.c_void_p
_I = ctypes.c_int
_I32P = ctypes.POINTER(ctypes.c_int32)
_F64P = ctypes.POINTER(ctypes.c_double)
SIGNATURES = {
    "nosa_config_validate": (_I, [ctypes.POINTER(NosaConfig), ctypes.c_char_p, _I]),
    "nosa_config_budgets": (_I, [ctypes.POINTER(NosaConfig), _I32P, _I32P, _I32P]),
    "nosa_ctx_create": (_I, [ctypes.POINTER(NosaConfig), _I, ctypes.POINTER(_P)]),
    "nosa_ctx_destroy": (None, [_P]),
    "nosa_last_error": (ctypes.c_char_p, [_P]),
    "nosa_ctx_memory": (_I, [_P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]),
    "nosa_set_eviction_head": (_I, [_P, _F64P, _F64P]),
    "nosa_prefill": (_I, [_P, _I, _I, _I, _P, _P, _I, _P]),
    "nosa_prefill_resident": (_I, [_P, _I, _I, _I, _P, _P, _I, _P]),
    "nosa_start_run": (_I, [_P, _I, _I, _P]),
    "nosa_select_plan": (_I, [_P, _I, _P, _I, _P]),
    "nosa_select": (_I, [_P, _I, _P, _I, _P]),
    "nosa_cache_plan": (_I, [_P, _I, _P, _P, _P]),
    "nosa_gather": (_I, [_P, _I, _I, _P]),
    "nosa_attend": (_I, [_P, _I, _P, _P, _P, _P, _P]),
    "nosa_decode_step": (_I, [_P, ctypes.POINTER(NosaStepIO), _P]),
    "nosa_decode_step_host": (_I, [_P, ctypes.POINTER(NosaHostStepIO), _P]),
    "nosa_step_graph_capture_host": (_I, [_P, ctypes.POINTER(NosaHostStepIO)]),
    "nosa_set_projection": (_I, [_P, _I, _P, _I, _I, _I, _I]),
    "nosa_decode_step_hidden": (_I, [_P, ctypes.POINTER(NosaHiddenStepIO), _P]),
    "nosa_decode_step_hidden_host": (_I, [_P, ctypes.POINTER(NosaHiddenStepIO), _P]),
    "nosa_step_graph_capture_hidden": (_I, [_P, ctypes.POINTER(NosaHiddenStepIO)]),
    "nosa_step_graph_launch_host": (_I, [_P, ctypes.POINTER(NosaHostStepIO), _P]),
    "nosa_step_graph_capture": (_I, [_P, ctypes.POINTER(NosaStepIO)]),
    "nosa_step_graph_launch": (_I, [_P, _P]),
    "nosa_project_qkv": (_I, [_P, _I, _I, _P, _I, _I, _I, _P, _P, _P, _I, _P]),
    "nosa_project_f32": (_I, [_P, _I, _I, _P, _I, _P, _P]),
    "nosa_select_scores": (_I, [_I, _P, _P, _I, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P]),
    "nosa_read_selection": (_I, [_P, _I, _I, _I32P, _I32P, _I32P, _I32P, _I32P, _I32P, _F64P]),
    "nosa_read_plan": (_I, [_P, _I, _I32P, _I32P, _I32P, _I32P, _I32P]),
    "nosa_read_residency": (_I, [_P, _I, _I, _I, _I32P, _I32P]),
    "nosa_read_block_scores": (_I, [_P, _I, _F64P]),
    "nosa_read_kv": (_I, [_P, _I, _I, _I, _I, _P, _P]),
    "nosa_read_slot": (_I, [_P, _I, _I, _I, _I, _P]),
    "nosa_read_stats": (_I, [_P, _I, _I, _I, _I, ctypes.POINTER(NosaStats)]),
    "nosa_reset_stats": (_I, [_P, _P]),
    "nosa_read_lengths": (_I, [_P, _I32P]),
    "nosa_check_errors": (_I, [_P, ctypes.POINTER(ctypes.c_uint32)]),
    "nosa_launch_count": (ctypes.c_int64, [_P]),
    "nosa_timing_enable": (_I, [_P, _I]),
    "nosa_timing_read": (_I, [_P, _F64P, ctypes.POINTER(ctypes.c_int64)]),
    "nosa_ktime_enable": (_I, [_P, _I]),
    "nosa_select_profile": (_I, [_P, _I, _F64P]),
    "nosa_ktime_read": (_I, [_P, _F64P]),
    "nosa_mgr_create": (_I, [_I, _I, _I, _I, _I, _I, _I, _I, ctypes.POINTER(_P)]),
    "nosa_mgr_destroy": (None, [_P]),
    "nosa_mgr_last_error": (ctypes.c_char_p, [_P]),
    "nosa_mgr_allocate": (_I, [_P, _I, _I, _I, _I, _I, _I32P]),
    "nosa_mgr_free": (_I, [_P, _I, _I]),
    "nosa_mgr_plan": (_I, [_P, _I, _I, _I32P, _I, _I32P, _I32P, _I32P, _I32P, _I32P]),
    "nosa_mgr_apply": (_I, [_P, _I, _I32P, _I, _I32P, _I, _I, _I32P]),
    "nosa_mgr_plan_policy": (_I, [_P, _I, _I, _I32P, _I, _I32P, _I32P, _I32P, _I32P, _I32P, _I32P]),
    "nosa_mgr_recency": (_I, [_P, _I, _P]),
    "nosa_mgr_lookup": (_I, [_P, _I, _I, _I32P, _I32P]),
    "nosa_mgr_tables": (_I, [_P, _I, _P, _I32P]),
    "nosa_mgr_audit": (_I, [_P, _I32P]),
    "nosa_mgr_free_lists": (_I, [_P, _I, _I32P, _I32P, _I32P, _I32P]),
    "nosa_mgr_block": (_I, [_P, _I, _I, _P, _I]),
    "nosa_synth_normal": (_I, [ctypes.c_uint64, _I, _I, _I, _I, _I, _I, ctypes.c_longlong, ctypes.c_longlong, _I,
                               ctypes.c_float, _I, _P, _P]),
    "nosa_synth_ar1_step": (_I, [ctypes.c_uint64, _I, _I, _I, _I, _I, ctypes.c_longlong, _I, ctypes.c_float,
                                 ctypes.c_float, ctypes.c_float, _P, _I, _P, _P]),
    "nosa_timing_trace": (_I, [_P, _I, _I32P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float), _I32P]),
}


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2510_13602_b200/csrc); this package has no CPU fallback")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int, ctx=None, mgr=None) -> None:
    """Raise the reference exception type matching a status code."""
    if rc == NOSA_OK:
        return
    msg = lib.nosa_mgr_last_error(mgr) if mgr is not None else lib.nosa_last_error(ctx)
    msg = msg.decode() if msg else f"status {rc}"
    if rc == NOSA_ERR_VALUE:
        raise ValueError(msg)
    if rc == NOSA_ERR_CAPACITY:
        raise CapacityExceeded(msg)
    if rc == NOSA_ERR_UNKNOWN_KEY:
        raise UnknownKey(msg)
    if rc == NOSA_ERR_OUT_OF_BLOCKS:
        raise OutOfBlocks(msg)
    raise RuntimeError(msg)


def stream_ptr(stream=None) -> int:
    """cudaStream_t of a torch stream (default: torch's current stream)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
