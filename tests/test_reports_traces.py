"""GPU-run results in the reference's file formats, checked on CPU:

* SimReport rows (paper_2510_13602_b200.reports) have the reference's fields, CSV columns and
  config hash, and the unmodified reference ``nosa-sim report`` merges them;
* decode traces recorded on the B200 (tests/golden/gpu_trace_*.json, tools/make_gpu_traces.py)
  load through the reference's serde.trace_from_json, pass its Theorem-1 checker, and every
  recorded selection equals the oracle's on the same counter-based inputs.

The reference tests skip when /root/reference is absent (the GPU box); the oracle replay does not
need it.
"""

import dataclasses
import json
import sys
from pathlib import Path

import pytest

from oracle import nosa_oracle as O
from paper_2510_13602_b200 import one_b_config, reports, workload
from paper_2510_13602_b200.engine import ResidencyStats
from paper_2510_13602_b200.traces import verify_locality_bound

GOLDEN = Path(__file__).resolve().parent / "golden"
REF_SRC = Path("/root/reference/pkg/src")
TRACES = {"nosa": GOLDEN / "gpu_trace_nosa.json", "infllmv2": GOLDEN / "gpu_trace_infllmv2.json"}
SPEC = dict(t0=8192, steps=24, fast=96, seed=3, seq=1, layer=0)   # tools/make_gpu_traces.py


def _nosa_sim():
    if not REF_SRC.exists():
        pytest.skip("reference sources not present")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import nosa_sim
    return nosa_sim


def _traces():
    if not all(p.exists() for p in TRACES.values()):
        pytest.skip("GPU trace fixtures not recorded yet (tools/make_gpu_traces.py)")


def _row():
    st = ResidencyStats(hits=900, misses=100, bytes_up=100 * 32768, bytes_down=60 * 32768, topk_required=600,
                        topk_misses=90)
    rep = reports.report_from_run(selector="nosa", resident=False, batch=128, context=32768, steps=20, seed=0,
                                  stats=st, tokens_per_s=14863.9, attn_ms_per_step=3.1, ms_per_step=8.6,
                                  fast_slots_per_seq=128, config=one_b_config(32768).to_dict())
    return reports.row_dict(rep)


def test_sim_report_row_semantics():
    row = _row()
    assert row["policy"] == "nosa" and row["fast_blocks_per_head"] == 128 * 128
    assert row["hit_rate"] == 0.9 and row["hit_rate_topk"] == 1.0 - 90 / 600
    assert 0.0 < row["attn_ratio_mean"] <= 1.0
    assert reports.policy_for("infllmv2", False) == "infllmv2-offload"
    assert reports.policy_for("infllmv2", True) == "infllmv2-resident"
    lines = reports.sim_rows_csv([row]).splitlines()
    assert lines[0] == "# nosa-sim grid v1" and lines[1].split(",") == list(reports.SIM_CSV_COLUMNS)
    assert ResidencyStats().hit_rate_topk == 1.0


def test_sim_report_schema_matches_reference():
    _nosa_sim()
    from nosa_sim import cli, offload_sim, serde
    assert [f.name for f in dataclasses.fields(reports.SimReport)] == \
        [f.name for f in dataclasses.fields(offload_sim.SimReport)]
    assert reports.SIM_CSV_COLUMNS == cli.SIM_CSV_COLUMNS
    assert reports.POLICIES == offload_sim.POLICIES
    cfg = one_b_config(32768).to_dict()
    assert reports.config_hash(cfg) == serde.config_hash(cfg)
    row = _row()
    assert reports.sim_rows_csv([row]) == cli._sim_rows_csv([row])


def test_reference_report_merges_gpu_rows_and_traces(tmp_path):
    _nosa_sim()
    _traces()
    from nosa_sim import cli
    js, _ = reports.write_sim_report([_row()], tmp_path, params={"measured": True})
    rc = cli.main(["report", "--inputs", js, str(TRACES["nosa"]), str(TRACES["infllmv2"]),
                   "--out", str(tmp_path / "merged.csv"), "--json", str(tmp_path / "merged.json")])
    assert rc == 0
    merged = json.loads((tmp_path / "merged.json").read_text())["rows"]
    assert [r["source"] for r in merged] == ["simulate", "locality", "locality"]
    assert merged[0]["tokens_per_s"] == 14863.9 and merged[0]["hit_rate"] == 0.9
    assert merged[1]["violations"] == 0


@pytest.mark.parametrize("selector", ["nosa", "infllmv2"])
def test_gpu_trace_loads_in_reference_serde(selector):
    _nosa_sim()
    _traces()
    from nosa_sim import cli, locality, serde
    doc = json.loads(TRACES[selector].read_text())
    trace = serde.trace_from_json(doc)
    assert trace.selector == selector and len(trace.steps) == SPEC["steps"] and trace.t0 == SPEC["t0"]
    assert serde.trace_to_json(trace)["steps"] == doc["steps"]        # lossless round trip
    for h in range(trace.config.n_kv_head):
        ours = verify_locality_bound(doc, head=h)
        if selector == "nosa":                                          # Theorem 1 holds on GPU runs
            ref = locality.verify_locality_bound(trace, head=h)
            assert ref.violations == [] and ours["violations"] == []
        else:
            ref = locality.baseline_locality(trace, head=h)
        assert ours["min_gamma"] == ref.min_gamma
    if selector == "nosa":
        assert cli.main(["check-theorem", str(TRACES[selector])]) == 0


@pytest.mark.parametrize("selector,rho", [("nosa", 0.95), ("infllmv2", 0.0)])
def test_gpu_trace_matches_oracle(selector, rho):
    """Every selection the B200 recorded equals the oracle's on the same inputs."""
    _traces()
    s = SPEC
    doc = json.loads(TRACES[selector].read_text())
    assert doc["query_smoothness"] == rho
    cfg = one_b_config(65536)
    H, Hq, D = cfg.n_kv_head, cfg.n_head, cfg.d_head
    w1, w2 = workload.eviction_head(Hq, D, s["seed"])
    orc = O.OracleEngine(O.OracleConfig.from_attention_config(cfg), 1, 1, s["t0"] + s["steps"] + 2, s["fast"], w1, w2)
    K, V = workload.synth_prefix_kv(s["seed"], s["layer"], [s["seq"]], H, s["t0"], D)
    orc.prefill(0, 0, K[0], V[0])
    orc.start_run()
    stream = workload.SynthQueryStream(s["seed"], [s["layer"]], [s["seq"]], Hq, H, D, rho)
    for step in range(s["steps"]):
        q, kn, vn = stream.next()
        _, recs = orc.step_seq(0, 0, q[0, 0], kn[0, 0], vn[0, 0], selector)
        for h in range(H):
            got = doc["steps"][step][h]
            assert got["step"] == s["t0"] + step
            assert got["blocks_q"] == recs[h].blocks_q.tolist(), f"step {step} head {h} blocks_q"
            assert got["blocks_e"] == recs[h].blocks_e.tolist(), f"step {step} head {h} blocks_e"
            fixed = sorted(set(recs[h].required) - set(recs[h].blocks_q.tolist()) - set(recs[h].blocks_e.tolist()))
            assert got["blocks_fixed"] == fixed, f"step {step} head {h} blocks_fixed"
