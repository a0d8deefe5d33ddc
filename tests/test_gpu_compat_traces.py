"""The reference-signature DecodeEngine (hidden states in, projection on the GPU) and
GPU-run decode traces in the reference's JSON format with the Theorem-1 check."""

import json

import numpy as np
import pytest
import torch

from oracle import nosa_oracle as O
from paper_2510_13602_b200 import AttentionConfig, NosaEngine, workload
from paper_2510_13602_b200.compat import DecodeEngine, EvictionHead, ModelWeights
from paper_2510_13602_b200.traces import TraceRecorder, verify_locality_bound

from helpers import assert_same_selection, rel_err

pytestmark = pytest.mark.gpu


def _cfg(row):
    n, d, n_head, n_kv, d_head, n_b, n_s, n_w, k, k_q, k_e, excl = (int(x) for x in row)
    return AttentionConfig(n=n, d=d, n_head=n_head, n_kv_head=n_kv, d_head=d_head, n_b=n_b, n_s=n_s, n_w=n_w,
                           k=k, k_q=k_q, k_e=k_e, accounting="exclusive" if excl else "inclusive")


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_decode_engine_dropin_vs_reference_golden(golden, dtype):
    """h_t = concat(q, k, v) through 0/1 projections, exactly how the golden reference run was
    driven: the drop-in must reproduce its selections bit for bit and its outputs in tolerance."""
    g = golden("engine_small")
    cfg = _cfg(g["cfg"])
    B, t0, steps, seed = (int(g[k]) for k in ("batch", "t0", "steps", "seed"))
    Hq, Hk, D = cfg.n_head, cfg.n_kv_head, cfg.d_head
    eye = np.eye((Hq + 2 * Hk) * D)
    w1, w2 = workload.eviction_head(Hq, D, seed)
    weights = ModelWeights(eye[:, :Hq * D], eye[:, Hq * D:(Hq + Hk) * D], eye[:, (Hq + Hk) * D:],
                           EvictionHead("ed-dma", w1, w2), 0)
    K, V = workload.prefix_kv(seed, B, Hk, t0, D)
    stream = workload.QueryStream(seed, 1, B, Hq, Hk, D, float(g["rho"]))
    inputs = [stream.next() for _ in range(steps)]
    tol = 2e-2 if dtype == "bf16" else 1e-5
    for b in range(B):
        eng = DecodeEngine(cfg, weights, capacity=t0 + steps + 1, dtype=dtype)
        h = np.concatenate([np.zeros((t0, Hq * D)), K[b].transpose(1, 0, 2).reshape(t0, Hk * D),
                            V[b].transpose(1, 0, 2).reshape(t0, Hk * D)], axis=1)
        eng.prefill(h)
        eng.start_run()
        for s in range(steps):
            q, kn, vn = inputs[s]
            out = eng.step(np.concatenate([q[0, b].ravel(), kn[0, b].ravel(), vn[0, b].ravel()]))
            assert out.step == t0 + s
            for hh, sel in enumerate(out.selections):
                assert list(sel.blocks_q) == [x for x in g["sel_q"][s, b, hh] if x >= 0]
                assert list(sel.blocks_e) == [x for x in g["sel_e"][s, b, hh] if x >= 0]
            assert rel_err(out.outputs, g["outputs"][s, b]) <= tol
        eng.close()


def test_decode_engine_random_weights_fp32():
    """Dense random projections (the reference's ModelWeights.random draws): the GPU projects in
    fp32, the oracle in fp64, so selections agree up to reported near-ties."""
    cfg = AttentionConfig(n=4096, d=256, n_head=4, n_kv_head=2, d_head=64, n_b=16, n_s=32, n_w=128, k=512, k_q=128,
                          k_e=384)
    weights = ModelWeights.random(cfg, "ed-dma", 3)
    rng = np.random.default_rng(5)
    t0, steps = 900, 10
    hidden = rng.standard_normal((t0 + steps, cfg.d))
    eng = DecodeEngine(cfg, weights, capacity=t0 + steps + 1, dtype="fp32")
    eng.prefill(hidden[:t0])
    eng.start_run()
    orc = O.OracleEngine(O.OracleConfig.from_attention_config(cfg), 1, 1, t0 + steps + 1, 80, weights.eviction.w1,
                         weights.eviction.w2)
    proj = lambda h, w: (h @ w)
    Kf, Vf = proj(hidden[:t0], weights.w_k), proj(hidden[:t0], weights.w_v)
    orc.prefill(0, 0, Kf.reshape(t0, 2, 64).transpose(1, 0, 2), Vf.reshape(t0, 2, 64).transpose(1, 0, 2))
    orc.start_run()
    for s in range(steps):
        h = hidden[t0 + s]
        out = eng.step(h)
        ref, recs = orc.step_seq(0, 0, proj(h, weights.w_q).reshape(4, 64), proj(h, weights.w_k).reshape(2, 64),
                                 proj(h, weights.w_v).reshape(2, 64))
        lo, hi = orc.geom[0].pool
        for hh in range(2):
            sq = np.zeros(hi)
            sq[lo:hi] = recs[hh].s_q
            assert_same_selection(out.selections[hh].blocks_q, recs[hh].blocks_q.tolist(), sq, list(range(lo, hi)),
                                  f"step {s} head {hh}", tie_tol=1e-5)
        assert rel_err(out.outputs, ref) <= 1e-4
    eng.close()


def test_gpu_trace_json_and_theorem_one(tmp_path):
    cfg = AttentionConfig(n=8192, d=2048, n_head=16, n_kv_head=2, d_head=128, n_b=64, n_s=64, n_w=1024, k=4096,
                          k_q=1024, k_e=3072)
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, 4)
    K, V = workload.prefix_kv(4, 2, 2, 6000, 128)
    eng = NosaEngine(cfg, batch=2, max_tokens=6100, fast_slots=100, w1=w1, w2=w2)
    eng.prefill(torch.from_numpy(K), torch.from_numpy(V), layer=0)
    eng.start_run()
    stream = workload.QueryStream(4, 1, 2, cfg.n_head, 2, 128, 0.0)  # adversarial: fresh queries
    recs = [TraceRecorder(eng, 0, b, seed=4) for b in range(2)]
    for _ in range(40):
        eng.step(*stream.next())
        for r in recs:
            r.record()
    for b, r in enumerate(recs):
        path = tmp_path / f"trace{b}.json"
        r.dump(path)
        doc = json.loads(path.read_text())
        assert doc["kind"] == "decode-trace" and doc["version"] == 1 and len(doc["steps"]) == 40
        assert set(doc["steps"][0][0]) == {"step", "blocks_q", "blocks_e", "blocks_fixed"}
        for head in range(2):
            rep = verify_locality_bound(doc, head)
            assert rep["violations"] == [], rep  # Theorem 1 holds on GPU selections
            assert rep["min_gamma"] >= cfg.locality_bound
        # byte-deterministic writer (serde.py:27-47)
        r.dump(tmp_path / "again.json")
        assert (tmp_path / "again.json").read_bytes() == path.read_bytes()
    eng.close()


def test_recorded_gpu_traces_are_reproducible(tmp_path):
    """tools/make_gpu_traces.py re-run on this box reproduces the committed fixtures byte for byte
    (the CPU suite checks those against the oracle and the reference's serde / Theorem-1 checker)."""
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    subprocess.run([sys.executable, str(root / "tools" / "make_gpu_traces.py"), str(tmp_path)], check=True)
    for name in ("gpu_trace_nosa.json", "gpu_trace_infllmv2.json"):
        fixture = root / "tests" / "golden" / name
        if not fixture.exists():
            pytest.skip("fixtures not recorded yet")
        assert (tmp_path / name).read_bytes() == fixture.read_bytes(), name
