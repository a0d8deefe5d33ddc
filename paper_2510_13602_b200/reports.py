"""SimReport rows from measured GPU runs.

The reference prices scripted selection traces with a cost model and reports one `SimReport` per
(policy, context, budget) point (offload_sim.py:175-192), written by ``nosa-sim simulate`` as a
``sim-report`` JSON document and a CSV with fixed columns (cli.py:189-194, 208-231).  This module
emits the same rows from a real decode run: the selections, residency counters and bytes come
from the GPU engine's device counters over the timed steps, and ``tokens_per_s`` is the measured
throughput instead of a modelled one, so the reference's ``report`` / plotting tools read GPU
results unchanged.

Field meanings on a GPU run:
  policy           "nosa", "infllmv2-offload" or "infllmv2-resident" (offload_sim.py:30), from
                   the selector and whether every block fits the fast tier
  hit_rate         hits / (hits + misses) over every (layer, sequence, head) plan of the timed
                   steps (ResidencyStats.hit_rate, kv_manager.py:112-115)
  hit_rate_topk    top-k blocks already fast-resident / top-k blocks required
                   (offload_sim.py:291-293, 314); device counters ST_TOPK / ST_TOPK_MISS
  bytes_up/down    miss / eviction payload bytes of the timed steps, all layers
  tokens_per_s     measured (bench.py `value`)
  attn_ratio_mean  attention-kernel time per step / step time (the cost model's attn / t_total,
                   offload_sim.py:124-139, measured instead of modelled)
  fast_blocks_per_head  fast slots per KV head over the whole batch (the reference's shared
                   pool size, offload_sim.py:268)
"""

from __future__ import annotations

import csv
import hashlib
import io
import json
import os
import tempfile
from dataclasses import asdict, dataclass

POLICIES = ("nosa", "infllmv2-offload", "infllmv2-resident")

# cli.py:214-218
SIM_CSV_COLUMNS = (
    "policy", "batch", "context", "steps", "seed", "memory_budget", "fast_blocks_per_head",
    "hit_rate", "hit_rate_topk", "bytes_up", "bytes_down", "tokens_per_s", "attn_ratio_mean",
    "config_hash",
)


@dataclass
class SimReport:
    """offload_sim.SimReport (offload_sim.py:175-192), same fields in the same order."""

    policy: str
    batch: int
    context: int
    steps: int
    seed: int
    hit_rate: float
    hit_rate_topk: float
    bytes_up: int
    bytes_down: int
    tokens_per_s: float
    attn_ratio_mean: float
    fast_blocks_per_head: int
    config: dict

    def to_dict(self) -> dict:
        return asdict(self)


def policy_for(selector: str, resident: bool) -> str:
    if selector == "nosa":
        return "nosa"
    return "infllmv2-resident" if resident else "infllmv2-offload"


def config_hash(config_dict: dict) -> str:
    """serde.config_hash (serde.py:50-52): first 16 hex digits of sha256 of the sorted JSON."""
    return hashlib.sha256(json.dumps(config_dict, sort_keys=True).encode()).hexdigest()[:16]


def report_from_run(*, selector: str, resident: bool, batch: int, context: int, steps: int, seed: int, stats,
                    tokens_per_s: float, attn_ms_per_step: float, ms_per_step: float, fast_slots_per_seq: int,
                    config: dict) -> SimReport:
    """One row from a measured run; `stats` is the engine's ResidencyStats over the timed steps."""
    return SimReport(policy=policy_for(selector, resident), batch=batch, context=context, steps=steps, seed=seed,
                     hit_rate=float(stats.hit_rate), hit_rate_topk=float(stats.hit_rate_topk),
                     bytes_up=int(stats.bytes_up), bytes_down=int(stats.bytes_down),
                     tokens_per_s=float(tokens_per_s),
                     attn_ratio_mean=float(min(1.0, attn_ms_per_step / ms_per_step)) if ms_per_step > 0 else 0.0,
                     fast_blocks_per_head=int(batch * fast_slots_per_seq), config=dict(config))


def row_dict(report: SimReport, memory_budget=None) -> dict:
    """A grid row as ``nosa-sim simulate`` stores it (cli.py:184-187)."""
    row = report.to_dict()
    row["memory_budget"] = memory_budget
    row["config_hash"] = config_hash(row["config"])
    return row


def _csv_cell(v):
    if isinstance(v, float):
        return repr(v)
    return "" if v is None else v


def sim_rows_csv(rows) -> str:
    """cli._sim_rows_csv (cli.py:221-231): version header, fixed columns, repr() floats."""
    buf = io.StringIO()
    buf.write("# nosa-sim grid v1\n")
    w = csv.writer(buf)
    w.writerow(SIM_CSV_COLUMNS)
    for row in rows:
        w.writerow([_csv_cell(row.get(c)) for c in SIM_CSV_COLUMNS])
    return buf.getvalue()


def _atomic_write(path, text: str):
    path = os.fspath(path)
    fd, tmp = tempfile.mkstemp(dir=os.path.dirname(path) or ".", prefix=".tmp-", suffix=".part")
    try:
        with os.fdopen(fd, "w") as f:
            f.write(text)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def write_sim_report(rows, out_dir, params: dict | None = None) -> tuple[str, str]:
    """sim_report.json ({"kind": "sim-report", "version": 1, "params", "rows"}) and sim_report.csv
    (cli.py:189-194).  `params` records the measured link and HBM rates in place of the cost
    model's CostModelParams."""
    os.makedirs(out_dir, exist_ok=True)
    js = os.path.join(out_dir, "sim_report.json")
    _atomic_write(js, json.dumps({"kind": "sim-report", "version": 1, "params": params or {}, "rows": list(rows)},
                                 sort_keys=True, indent=2) + "\n")
    cs = os.path.join(out_dir, "sim_report.csv")
    _atomic_write(cs, sim_rows_csv(rows))
    return js, cs
