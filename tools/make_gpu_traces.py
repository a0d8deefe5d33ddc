"""Record GPU decode traces as committed fixtures (tests/golden/gpu_trace_*.json).

Runs the GPU engine on the counter-based synthetic inputs (the 1B attention shape at 8K context,
one (layer, sequence), both selectors) and writes each run's selections with traces.TraceRecorder
in the reference's decode-trace schema (serde.py:103-126).  CPU tests then load these files with
the unmodified reference (serde.trace_from_json, locality.verify_locality_bound, `nosa-sim
report`) and replay the same inputs through the oracle to check every recorded selection.
Usage (on a GPU box): python tools/make_gpu_traces.py OUT_DIR
"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2510_13602_b200 import NosaEngine, one_b_config, synth, workload  # noqa: E402
from paper_2510_13602_b200.traces import TraceRecorder  # noqa: E402

SPEC = dict(t0=8192, steps=24, fast=96, seed=3, seq=1, layer=0)


def record(selector: str, rho: float, out: Path):
    s = SPEC
    cfg = one_b_config(65536)
    H, Hq, D = cfg.n_kv_head, cfg.n_head, cfg.d_head
    dev = torch.device("cuda", 0)
    w1, w2 = workload.eviction_head(Hq, D, s["seed"])
    eng = NosaEngine(cfg, batch=1, layers=1, max_tokens=s["t0"] + s["steps"] + 2, fast_slots=s["fast"], w1=w1, w2=w2)
    k, v = synth.prefix_kv(s["seed"], s["layer"], s["seq"], 1, H, s["t0"], D, dev)
    eng.prefill(k, v, layer=0)
    eng.start_run()
    stream = synth.GpuQueryStream(s["seed"], 1, s["seq"], 1, Hq, H, D, rho, dev)
    rec = TraceRecorder(eng, layer=0, seq=0, selector=selector, seed=s["seed"], scripted=False,
                        query_smoothness=rho)
    for _ in range(s["steps"]):
        q, kn, vn = stream.next()
        eng.step(q, kn, vn, selector=selector)
        rec.record()
    eng.close()
    rec.dump(out)


if __name__ == "__main__":
    out = Path(sys.argv[1] if len(sys.argv) > 1 else ROOT / "tests" / "golden")
    out.mkdir(parents=True, exist_ok=True)
    record("nosa", 0.95, out / "gpu_trace_nosa.json")
    record("infllmv2", 0.0, out / "gpu_trace_infllmv2.json")
    print("wrote", sorted(p.name for p in out.glob("gpu_trace_*.json")))
