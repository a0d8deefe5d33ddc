"""B200-native NOSA offloaded sparse-attention decode step (arXiv 2510.13602).

Host-side mirror of the reference decode API (AttentionConfig, BlockGeometry, SelectionResult,
nosa_select / infllmv2_select, the DecodeEngine step and TieredBlockManager residency) over the
C ABI of libnosa_b200.so (include/nosa_b200.h): hand-written sm_100a kernels for selection, the
GPU-resident block cache, the pinned-host miss gather and block-sparse attention.  There is no
CPU fallback: importing the package loads the shared library or fails.
"""

from . import _lib  # noqa: F401  (loads libnosa_b200.so; fails loudly when it is missing)
from .config import AttentionConfig, cfg1_config, one_b_config
from .engine import NosaEngine, ResidencyStats, StepOutput, TransferPlanView
from .errors import (CapacityExceeded, DuplicateKey, LayoutMismatch, ManagerError, OutOfBlocks, StalePlan,
                     UnknownKey)
from .kv_manager import (FAST, SLOW, GpuTieredBlockManager, PhysicalLayout, TieredBlockManager, TransferPlan,
                         least_recently_required)
from .selection import BlockGeometry, SelectionResult, build_token_mask, infllmv2_select, nosa_select

__all__ = [
    "AttentionConfig", "BlockGeometry", "CapacityExceeded", "DuplicateKey", "GpuTieredBlockManager",
    "LayoutMismatch", "ManagerError", "NosaEngine", "OutOfBlocks", "ResidencyStats", "SelectionResult",
    "StalePlan", "StepOutput", "TransferPlan", "TransferPlanView", "UnknownKey", "build_token_mask",
    "cfg1_config", "infllmv2_select", "nosa_select", "one_b_config",
]
