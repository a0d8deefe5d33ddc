"""Shared drivers for the parity tests: run the GPU engine and the CPU oracle on identical
seeded inputs and compare selections, residency and outputs."""

from __future__ import annotations

import numpy as np

from oracle import nosa_oracle as O


def rel_err(got, want) -> float:
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-30))


def boundary_gap(scores: np.ndarray, chosen: list, pool: list) -> float:
    """Smallest |score(chosen) - score(not chosen)| across the selection boundary: the
    margin that a flip would have to beat (0.0 = an exact tie)."""
    chosen = set(chosen)
    inside = [scores[p] for p in pool if p in chosen]
    outside = [scores[p] for p in pool if p not in chosen]
    if not inside or not outside:
        return float("inf")
    return float(min(inside) - max(outside))


def assert_same_selection(got: list, want: list, scores: np.ndarray, pool: list, what: str, tie_tol=1e-12):
    """Sets must be equal; a mismatch is accepted only as a reported exact/near tie."""
    if list(got) == list(want):
        return None
    gap = abs(boundary_gap(scores, want, pool))
    scale = max(np.max(np.abs(scores)), 1.0)
    assert gap <= tie_tol * scale, f"{what}: GPU {list(got)} != oracle {list(want)}, boundary gap {gap:.3e}"
    return gap


def oracle_for(cfg, batch, layers, capacity, fast_slots, w1, w2, variant="ed-dma", shared=False):
    oc = O.OracleConfig.from_attention_config(cfg, variant)
    return O.OracleEngine(oc, batch, layers, capacity, fast_slots, w1, w2, shared=shared)
