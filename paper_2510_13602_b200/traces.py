"""Selection traces of GPU runs in the reference's on-disk format.

`TraceRecorder` collects the per-step `SelectionResult`s of one (layer, sequence) of a
`NosaEngine` run and writes them as a ``decode-trace`` JSON document with the reference's
schema (serde.py:103-126: kind, version 1, seed, t0, selector, scripted, query_smoothness,
variant, config, steps[step][head] = {step, blocks_q, blocks_e, blocks_fixed}), so
``nosa-sim check-theorem`` (cli.py:117-151) can verify Theorem 1 on GPU traces.  Writes are
atomic (temp file + rename) and byte-deterministic (sorted keys).
`verify_locality_bound` restates the checker (locality.py:16-22, 66-91) for the same files.
"""

from __future__ import annotations

import json
import os
import tempfile

from .selection import SelectionResult

TRACE_VERSION = 1


def dump_json(obj, path) -> None:
    path = os.fspath(path)
    fd, tmp = tempfile.mkstemp(dir=os.path.dirname(path) or ".", prefix=".tmp-", suffix=".part")
    try:
        with os.fdopen(fd, "w") as f:
            f.write(json.dumps(obj, sort_keys=True, indent=2) + "\n")
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


class TraceRecorder:
    def __init__(self, engine, layer: int = 0, seq: int = 0, selector: str = "nosa", seed: int = 0,
                 scripted: bool = False, query_smoothness: float = 0.0):
        self.engine, self.layer, self.seq = engine, layer, seq
        self.selector, self.seed = selector, seed
        self.scripted, self.query_smoothness = scripted, query_smoothness
        self.steps: list[list[SelectionResult]] = []
        self.t0 = None

    def record(self) -> list[SelectionResult]:
        """Append the selections of the engine's last step (one per KV head)."""
        row = self.engine.selections(self.layer)[self.seq]
        if self.t0 is None:
            self.t0 = self.engine.geometry[self.seq].t0
        self.steps.append(row)
        return row

    def to_json(self) -> dict:
        return {
            "kind": "decode-trace",
            "version": TRACE_VERSION,
            "seed": self.seed,
            "t0": self.t0,
            "selector": self.selector,
            "scripted": self.scripted,
            "query_smoothness": self.query_smoothness,
            "variant": self.engine.variant,
            "config": self.engine.config.to_dict(),
            "steps": [[{"step": s.step, "blocks_q": list(s.blocks_q), "blocks_e": list(s.blocks_e),
                        "blocks_fixed": list(s.blocks_fixed)} for s in row] for row in self.steps],
        }

    def dump(self, path) -> None:
        dump_json(self.to_json(), path)


def gamma(prev, cur) -> float:
    """|prev & cur| / |cur| (locality.py:16-22)."""
    prev, cur = frozenset(prev), frozenset(cur)
    if not cur:
        raise ValueError("gamma is undefined for an empty current set")
    return len(prev & cur) / len(cur)


def verify_locality_bound(trace: dict, head: int = 0) -> dict:
    """Theorem-1 check on a decode-trace document: gamma of consecutive top-k sets must stay
    >= k_e_topk / (k_q + k_e_topk); an empty top-k set counts as full overlap
    (locality.py:66-91).  Returns {bound, min_gamma, gammas, violations, steps}."""
    from .config import AttentionConfig
    cfg = AttentionConfig.from_dict(trace["config"])
    bound = cfg.locality_bound
    sets = [frozenset(s[head]["blocks_q"]) | frozenset(s[head]["blocks_e"]) for s in trace["steps"]]
    pos = [s[head]["step"] for s in trace["steps"]]
    gammas, violations, steps = [], [], []
    for i in range(1, len(sets)):
        g = 1.0 if not sets[i] else gamma(sets[i - 1], sets[i])
        gammas.append(g)
        steps.append(pos[i])
        if g < bound:
            violations.append(i)
    return {"bound": bound, "min_gamma": min(gammas) if gammas else 1.0, "gammas": gammas,
            "violations": violations, "steps": steps}
