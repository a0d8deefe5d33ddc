"""The CPU oracle against the golden fixtures generated from the unmodified reference
(tests/golden/make_golden.py).  This pins the oracle before any GPU result is compared with it."""

import numpy as np
import pytest

from oracle import nosa_oracle as O


def _cfg(row):
    n, d, n_head, n_kv, d_head, n_b, n_s, n_w, k, k_q, k_e, excl = (int(x) for x in row)
    return dict(n=n, d=d, n_head=n_head, n_kv_head=n_kv, d_head=d_head, n_b=n_b, n_s=n_s, n_w=n_w, k=k, k_q=k_q,
                k_e=k_e, accounting="exclusive" if excl else "inclusive")


def test_selection_kats_bit_exact(golden):
    g = golden("selection_kats")
    for i in range(len(g["t"])):
        c = _cfg(g["cfg_rows"][g["cfg"][i]])
        t, nblk = int(g["t"][i]), int(g["nblk"][i])
        s_q, s_e = g["s_q"][i][:nblk], g["s_e"][i][:nblk]
        geom = O.Geometry.for_run(c["n_b"], c["n_s"], c["n_w"], t)
        m_q, m_e, m_topk = O.budgets(c["n_b"], c["n_s"], c["n_w"], c["k"], c["k_q"], c["k_e"], c["accounting"])
        bq, be = O.select(s_q, s_e, geom, m_q, m_e, "nosa")
        want = lambda key: [x for x in g[key][i] if x >= 0]
        assert bq.tolist() == want("nosa_q"), i
        assert be.tolist() == want("nosa_e"), i
        assert geom.fixed(t) == want("fixed"), i
        iq, _ = O.select(s_q, None, geom, m_topk, 0, "infllmv2")
        assert iq.tolist() == want("inf_q"), i


def test_manager_trace_bit_exact(golden):
    g = golden("manager_trace")
    C = int(g["capacity"])
    steps, H, _ = g["req"].shape
    mgr = O.SequenceManager(H, C)
    for s in range(steps):
        for h in range(H):
            req = [x for x in g["req"][s, h] if x >= 0]
            fetch, evict, hits = mgr.plan_apply(req, h)
            assert fetch == [x for x in g["fetch"][s, h] if x >= 0], (s, h)
            assert evict == [x for x in g["evict"][s, h] if x >= 0], (s, h)
            assert hits == g["hits"][s, h]
            assert [mgr.slot_of[h][b] for b in req] == [x for x in g["slots"][s, h] if x >= 0]
    hits, misses, _, calls = g["stats"]
    assert (mgr.hits, mgr.misses, mgr.steps) == (hits, misses, calls)


@pytest.mark.parametrize("tag", ["nosa", "infllmv2"])
def test_shared_pool_matches_reference_simulator(golden, tag):
    """One manager shared by the batch, b-major calls: the reference simulate_decode's residency."""
    g = golden("shared_pool_sim")
    B, H, slots, _, _, steps = (int(x) for x in g[f"{tag}_shape"])
    mgr = O.SharedManager(H, B * slots)
    topk_hits = topk_total = 0
    for i in range(steps + 1):
        if i == 1:
            mgr.hits = mgr.misses = mgr.evictions = mgr.steps = 0
        for b in range(B):
            for h in range(H):
                req = [x for x in g[f"{tag}_req"][i, b, h] if x >= 0]
                fetch, evict, _ = mgr.plan_apply(req, b, h)
                assert fetch == [x for x in g[f"{tag}_fetch"][i, b, h] if x >= 0], (i, b, h)
                assert [list(k) for k in evict] == [list(e) for e in g[f"{tag}_evict"][i, b, h] if e[0] >= 0]
                if i:
                    tk = {x for x in g[f"{tag}_topk"][i, b, h] if x >= 0}
                    topk_hits += len(tk - set(fetch))
                    topk_total += len(tk)
    hit_rate, hit_rate_topk, bytes_up, _ = g[f"{tag}_report"]
    assert mgr.hits / (mgr.hits + mgr.misses) == hit_rate
    assert mgr.misses * 2 * 16 * 8 * 2 == bytes_up
    assert topk_hits / topk_total == hit_rate_topk


def _workload():
    """The input generator, loaded by path (pure NumPy; importing the package would load the .so)."""
    import importlib.util
    from pathlib import Path
    spec = importlib.util.spec_from_file_location(
        "nosa_workload", Path(__file__).resolve().parents[1] / "paper_2510_13602_b200" / "workload.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("name,dense", [("engine_small", False), ("engine_small", True),
                                        ("engine_small_infllmv2", False), ("engine_cfg1", False),
                                        ("engine_cfg1", True), ("engine_1b_32k", False), ("engine_1b_32k", True),
                                        ("engine_1b_32k_infllmv2_rho0", False)])
def test_engine_matches_reference(golden, name, dense):
    """dense=True: the oracle's attend_biased restatement over every cached token (the reference's
    own form, timed by bench.py's CPU legs); False: the live-token gather the tests use."""
    workload = _workload()
    g = golden(name)
    c = _cfg(g["cfg"])
    B, t0, steps, C, seed = (int(g[k]) for k in ("batch", "t0", "steps", "fast_slots", "seed"))
    rho, selector = float(g["rho"]), str(g["selector"])
    oc = O.OracleConfig(c["n_head"], c["n_kv_head"], c["d_head"], c["n_b"], c["n_s"], c["n_w"], c["k"], c["k_q"],
                        c["k_e"], c["accounting"])
    w1, w2 = workload.eviction_head(c["n_head"], c["d_head"], seed)
    if int(g.get("synth", 0)):
        K, V = workload.synth_prefix_kv(seed, 0, range(B), c["n_kv_head"], t0, c["d_head"])
        stream = workload.SynthQueryStream(seed, [0], range(B), c["n_head"], c["n_kv_head"], c["d_head"], rho)
    else:
        K, V = workload.prefix_kv(seed, B, c["n_kv_head"], t0, c["d_head"])
        stream = workload.QueryStream(seed, 1, B, c["n_head"], c["n_kv_head"], c["d_head"], rho)
    eng = O.OracleEngine(oc, B, 1, t0 + steps + 1, C, w1, w2, dense=dense)
    for b in range(B):
        eng.prefill(0, b, K[b], V[b])
    eng.start_run()
    lo, hi = (int(x) for x in g["pool"])
    for s in range(steps):
        q, kn, vn = stream.next()
        out, recs = eng.step(q, kn, vn, selector)
        for b in range(B):
            for h in range(c["n_kv_head"]):
                r = recs[0][b][h]
                assert r.blocks_q.tolist() == [x for x in g["sel_q"][s, b, h] if x >= 0], (s, b, h)
                assert r.blocks_e.tolist() == [x for x in g["sel_e"][s, b, h] if x >= 0], (s, b, h)
                assert r.fetch == [x for x in g["fetch"][s, b, h] if x >= 0], (s, b, h)
                assert r.evict == [x for x in g["evict"][s, b, h] if x >= 0], (s, b, h)
                assert r.hits == g["hits"][s, b, h]
                np.testing.assert_allclose(r.s_q, g["s_q"][s, b, h], rtol=1e-12, atol=1e-12)
                if s == 0:
                    np.testing.assert_allclose(r.s_e_c, g["s_e_pool"][b, h], rtol=1e-12, atol=1e-14)
        tol = 1e-6 if g["outputs"].dtype == np.float32 else 1e-10
        np.testing.assert_allclose(out[0], g["outputs"][s], rtol=0, atol=tol)


# synth_normal(7, KIND_K, layer 3, seq [5], 2 heads, pos 10..11, d 8)[0, 1, 1, :4], recorded when the
# generator was written (it is the bench's input contract: changing it changes every bench input)
KNOWN_SYNTH = [0.8848428130149841, 0.3378947377204895, 1.2868279218673706, -0.8827285170555115]


def test_synth_generator_known_answers():
    """The counter-based generator is pinned: fixed values (the GPU kernels are checked against this
    NumPy twin bit for bit in tests/test_gpu_synth.py) and unit-variance statistics."""
    W = _workload()
    x = W.synth_normal(7, W.KIND_K, 3, [5], 2, 10, 2, 8)
    assert x.dtype == np.float32 and x.shape == (1, 2, 2, 8)
    assert [float(v) for v in x[0, 1, 1, :4]] == KNOWN_SYNTH
    big = W.synth_normal(1, W.KIND_V, 0, range(4), 2, 0, 4096, 128).astype(np.float64)
    assert abs(big.mean()) < 5e-3 and abs(big.var() - 1.0) < 5e-3
    # the same values whatever subset is drawn (sharding invariance of the inputs)
    sub = W.synth_normal(1, W.KIND_V, 0, [2, 3], 2, 100, 50, 128)
    assert np.array_equal(sub, big[2:4, :, 100:150].astype(np.float32))
    st = W.SynthQueryStream(3, [0, 1], [0, 1, 2], 16, 2, 128, 0.95)
    q0, k0, v0 = st.next()
    q1, _, _ = st.next()
    assert q0.shape == (2, 3, 16, 128) and k0.shape == (2, 3, 2, 128)
    assert np.array_equal(W.bf16_round(q0), q0) and not np.array_equal(q0, q1)
    st2 = W.SynthQueryStream(3, [1], [2], 16, 2, 128, 0.95)
    a, b, c = st2.next()
    assert np.array_equal(a[0, 0], q0[1, 2]) and np.array_equal(b[0, 0], k0[1, 2]) and np.array_equal(c[0, 0], v0[1, 2])
    assert np.array_equal(st2.next()[0][0, 0], q1[1, 2])
