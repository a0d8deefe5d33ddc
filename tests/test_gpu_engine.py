"""GPU decode step (select -> cache plan -> gather -> attend -> append) against the golden
reference runs and the CPU oracle, through the C ABI.

Tolerances (north star): selected blocks and hit/miss sets bit-exact (exact ties excepted and
reported); outputs max|o - o_ref| / max|o_ref| <= 2e-2 in bf16 storage, <= 1e-5 in fp32."""

import numpy as np
import pytest
import torch

from oracle import nosa_oracle as O
from paper_2510_13602_b200 import AttentionConfig, CapacityExceeded, NosaEngine, workload

from helpers import assert_same_selection, oracle_for, rel_err

pytestmark = pytest.mark.gpu

TOL = {"bf16": 2e-2, "fp32": 1e-5}


def _cfg(row):
    n, d, n_head, n_kv, d_head, n_b, n_s, n_w, k, k_q, k_e, excl = (int(x) for x in row)
    return AttentionConfig(n=n, d=d, n_head=n_head, n_kv_head=n_kv, d_head=d_head, n_b=n_b, n_s=n_s, n_w=n_w,
                           k=k, k_q=k_q, k_e=k_e, accounting="exclusive" if excl else "inclusive")


@pytest.mark.parametrize("name", ["engine_small", "engine_small_infllmv2", "engine_cfg1"])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_engine_vs_reference_golden(golden, name, dtype):
    g = golden(name)
    cfg = _cfg(g["cfg"])
    B, t0, steps, C, seed = (int(g[k]) for k in ("batch", "t0", "steps", "fast_slots", "seed"))
    rho, selector = float(g["rho"]), str(g["selector"])
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, seed)
    K, V = workload.prefix_kv(seed, B, cfg.n_kv_head, t0, cfg.d_head)
    stream = workload.QueryStream(seed, 1, B, cfg.n_head, cfg.n_kv_head, cfg.d_head, rho)
    eng = NosaEngine(cfg, batch=B, max_tokens=t0 + steps + 1, fast_slots=C, w1=w1, w2=w2, dtype=dtype)
    eng.prefill(torch.from_numpy(K), torch.from_numpy(V), layer=0)
    eng.start_run()
    lo, hi = (int(x) for x in g["pool"])
    pool = list(range(lo, hi))
    worst = 0.0
    for s in range(steps):
        q, kn, vn = stream.next()
        out = eng.step(q, kn, vn, selector=selector).cpu().numpy()
        sels = eng.selections(0)
        plans = eng.plans(0)
        _, _, _, _, _, _, s_q = eng.raw_selection(0)
        for b in range(B):
            for h in range(cfg.n_kv_head):
                want_q = [x for x in g["sel_q"][s, b, h] if x >= 0]
                want_e = [x for x in g["sel_e"][s, b, h] if x >= 0]
                sq = np.zeros(hi)
                sq[lo:hi] = g["s_q"][s, b, h]
                assert_same_selection(sels[b][h].blocks_q, want_q, sq, pool, f"step {s} seq {b} head {h} blocks_q")
                assert list(sels[b][h].blocks_e) == want_e, (s, b, h)
                assert plans[b][h].fetch == [x for x in g["fetch"][s, b, h] if x >= 0], (s, b, h)
                assert plans[b][h].evict == [x for x in g["evict"][s, b, h] if x >= 0], (s, b, h)
                assert plans[b][h].hits == g["hits"][s, b, h]
                # GPU pool scores agree with the f64 reference to f64 rounding
                np.testing.assert_allclose(s_q[b, h, lo:hi], g["s_q"][s, b, h], rtol=1e-12, atol=1e-12)
        err = rel_err(out[0], g["outputs"][s])
        worst = max(worst, err)
        assert err <= TOL[dtype], f"step {s}: relative error {err:.3e} > {TOL[dtype]}"
    # the append path wrote every token through to the slow tier
    for b in range(B):
        k, v = eng.read_kv(0, b, 0)
        assert k.shape[0] == t0 + steps
        np.testing.assert_array_equal(k[:t0], K[b, 0])
    eng.close()
    print(f"{name} {dtype}: worst relative output error {worst:.3e}")


def _run_pair(cfg, *, batch, t0s, steps, fast_slots, seed, rho, selector="nosa", dtype="bf16", layers=1,
              variant="ed-dma", check_residency=True, gather="uva", schedule="pipelined", resident=False,
              shared=False, attend_chunk=0, slow_tier="host", attend_layers=0):
    """GPU engine and oracle on identical inputs; returns the worst relative output error."""
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, seed)
    if variant == "dma":
        w2 = w2 * 0.2
    tmax = max(t0s)
    cap = tmax + steps + 1
    eng = NosaEngine(cfg, batch=batch, layers=layers, max_tokens=cap, fast_slots=fast_slots, w1=w1, w2=w2,
                     dtype=dtype, variant=variant, residency="shared" if shared else "per-sequence",
                     attend_chunk=attend_chunk, slow_tier=slow_tier, attend_layers=attend_layers)
    orc = oracle_for(cfg, batch, layers, cap, fast_slots, w1, w2, variant, shared=shared)
    K, V = workload.prefix_kv(seed, batch * layers, cfg.n_kv_head, tmax, cfg.d_head)
    K = K.reshape(layers, batch, cfg.n_kv_head, tmax, cfg.d_head)
    V = V.reshape(layers, batch, cfg.n_kv_head, tmax, cfg.d_head)
    if shared:  # one pool per (layer, head): the whole batch is prefilled at once
        assert len(set(t0s)) == 1
        for l in range(layers):
            eng.prefill(torch.from_numpy(np.ascontiguousarray(K[l])), torch.from_numpy(np.ascontiguousarray(V[l])),
                        layer=l)
            for b in range(batch):
                orc.prefill(l, b, K[l, b], V[l, b])
    for l in range(layers if not shared else 0):
        for b in range(batch):
            t = t0s[b]
            eng.prefill(torch.from_numpy(np.ascontiguousarray(K[l, b:b + 1, :, :t])),
                        torch.from_numpy(np.ascontiguousarray(V[l, b:b + 1, :, :t])), layer=l, seq_begin=b,
                        resident=resident)
            orc.prefill(l, b, K[l, b, :, :t], V[l, b, :, :t])
            if resident:
                for h in range(cfg.n_kv_head):
                    orc.managers[l][b].make_resident(h, -(-t // cfg.n_b))
    eng.start_run()
    orc.start_run()
    stream = workload.QueryStream(seed, layers, batch, cfg.n_head, cfg.n_kv_head, cfg.d_head, rho)
    worst = 0.0
    for s in range(steps):
        q, kn, vn = stream.next()
        out = eng.step(q, kn, vn, selector=selector, gather=gather, schedule=schedule).cpu().numpy()
        ref, recs = orc.step(q, kn, vn, selector)
        for l in range(layers):
            sels, plans = eng.selections(l), eng.plans(l)
            _, _, _, _, req, nreq, s_q = eng.raw_selection(l)
            for b in range(batch):
                geom = orc.geom[b]
                lo, hi = geom.pool
                pool = list(range(lo, hi))
                for h in range(cfg.n_kv_head):
                    r = recs[l][b][h]
                    sq = np.zeros(max(hi, 1))
                    sq[lo:hi] = r.s_q
                    assert_same_selection(sels[b][h].blocks_q, r.blocks_q.tolist(), sq, pool, f"l{l} s{s} b{b} h{h} q")
                    assert list(sels[b][h].blocks_e) == r.blocks_e.tolist(), (l, s, b, h)
                    assert req[b, h, :nreq[b, h]].tolist() == r.required, (l, s, b, h)
                    assert plans[b][h].fetch == r.fetch, (l, s, b, h)
                    want_evict = [o * eng.max_blocks + x for o, x in r.evict] if shared else r.evict
                    assert plans[b][h].evict == want_evict, (l, s, b, h)
                    assert plans[b][h].hits == r.hits
                    np.testing.assert_allclose(s_q[b, h, lo:hi], r.s_q, rtol=1e-12, atol=1e-12)
                    if check_residency and s == steps - 1:
                        slot_of, block_of = eng.residency(l, b, h)
                        want = orc.managers[l][b].slot_of[h]
                        if shared:  # shared-pool slot ids of this sequence's blocks
                            want = {blk: sl for (ob, blk), sl in want.items() if ob == b}
                        got = {int(blk): int(sl) for blk, sl in enumerate(slot_of) if sl >= 0}
                        assert got == want, (l, b, h)
        worst = max(worst, rel_err(out, ref))
        assert worst <= TOL[dtype], f"step {s}: relative error {worst:.3e}"
    st = eng.residency_stats()
    ost = orc.stats()
    assert (st.hits, st.misses, st.evictions, st.steps) == (ost["hits"], ost["misses"], ost["evictions"], ost["steps"])
    assert (st.topk_required, st.topk_misses) == (ost["topk_required"], ost["topk_misses"])  # hit_rate_topk
    assert st.bytes_up == st.misses * eng.bytes_per_block
    assert (eng.lengths() == np.array([[t + steps for t in t0s]] * layers)).all()
    eng.close()
    return worst


SMALL = AttentionConfig(n=4096, d=512, n_head=4, n_kv_head=2, d_head=64, n_b=16, n_s=32, n_w=128, k=512, k_q=128,
                        k_e=384)
ONE_B_SMALL = AttentionConfig(n=8192, d=2048, n_head=16, n_kv_head=2, d_head=128, n_b=64, n_s=64, n_w=1024, k=4096,
                              k_q=1024, k_e=3072)


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_eviction_pressure_low_locality(dtype):
    # rho = 0: adversarial stream, fast tier barely above the requirement -> evictions every step
    _run_pair(SMALL, batch=3, t0s=[1000, 1000, 1000], steps=12, fast_slots=36, seed=3, rho=0.0, dtype=dtype)


def test_ragged_batch_and_partial_tails():
    # different cache lengths per sequence, partial tail blocks, one sequence with an empty pool
    _run_pair(SMALL, batch=4, t0s=[1000, 517, 160, 2049], steps=20, fast_slots=48, seed=4, rho=0.5)


def test_tiny_contexts_everything_fixed():
    # t <= n_s + n_w: the pool is empty, every cached block is attended (test_decode.py:123-134)
    _run_pair(SMALL, batch=2, t0s=[1, 100], steps=40, fast_slots=16, seed=5, rho=0.9)


def test_short_pool_selects_everything():
    # pool smaller than the top-k budget (test_selection.py:109-115)
    _run_pair(SMALL, batch=2, t0s=[300, 250], steps=6, fast_slots=40, seed=6, rho=0.3)


@pytest.mark.parametrize("selector", ["nosa", "infllmv2"])
def test_one_b_shape_multi_layer(selector):
    _run_pair(ONE_B_SMALL, batch=2, t0s=[6000, 4100], steps=4, fast_slots=80, seed=7, rho=0.95, layers=2,
              selector=selector)


@pytest.mark.parametrize("variant", ["s-dma", "dma"])
def test_other_eviction_variants(variant):
    _run_pair(SMALL, batch=2, t0s=[700, 900], steps=6, fast_slots=40, seed=8, rho=0.5, variant=variant)


def test_exclusive_accounting():
    cfg = AttentionConfig(n=4096, d=512, n_head=8, n_kv_head=2, d_head=64, n_b=32, n_s=32, n_w=256, k=768, k_q=256,
                          k_e=512, accounting="exclusive")
    _run_pair(cfg, batch=2, t0s=[1500, 1200], steps=6, fast_slots=40, seed=9, rho=0.5)


@pytest.mark.parametrize("n_b", [16, 32, 128])
def test_block_sizes(n_b):
    cfg = AttentionConfig(n=8192, d=1024, n_head=4, n_kv_head=2, d_head=128, n_b=n_b, n_s=n_b, n_w=4 * n_b,
                          k=16 * n_b, k_q=4 * n_b, k_e=12 * n_b)
    _run_pair(cfg, batch=2, t0s=[40 * n_b + 3, 30 * n_b], steps=5, fast_slots=20, seed=10, rho=0.5)


@pytest.mark.parametrize("chunk", [1, 2, 4, 8])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_split_k_chunk_sizes(chunk, dtype):
    """Every split-K granularity (blocks per attention work item) against the oracle."""
    a = _run_pair(ONE_B_SMALL, batch=3, t0s=[3000, 2500, 1700], steps=6, fast_slots=70, seed=21, rho=0.5,
                  dtype=dtype, layers=2, attend_chunk=chunk)
    assert a <= TOL[dtype]


@pytest.mark.parametrize("selector", ["nosa", "infllmv2"])
def test_shared_pool_residency_vs_oracle(selector):
    """The reference simulator's residency: one pool per (layer, head) shared by the batch,
    planned in batch order; victims may belong to other sequences."""
    _run_pair(SMALL, batch=4, t0s=[1000] * 4, steps=16, fast_slots=36, seed=14, rho=0.0, layers=2,
              selector=selector, shared=True)


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_resident_prefill(dtype):
    # all-resident configuration: every prefix block placed in HBM at prefill (allocate(FAST))
    _run_pair(SMALL, batch=2, t0s=[1000, 777], steps=30, fast_slots=70, seed=13, rho=0.0, dtype=dtype,
              resident=True)


@pytest.mark.parametrize("selector,dtype,kscale,qscale", [
    ("nosa", "bf16", 1.0, 1.0), ("infllmv2", "bf16", 1.0, 1.0), ("nosa", "fp32", 1.0, 1.0),
    ("infllmv2", "fp32", 1.0, 1.0),
    ("nosa", "fp32", 3e4, 1e-4),   # large keys, tiny queries: the bound's relative terms dominate
    ("nosa", "fp32", 1.0, 0.0),    # zero queries: every pool score ties at 0, lowest blocks win
])
def test_screened_selection_equals_full_f64_scan(selector, dtype, kscale, qscale, monkeypatch):
    """The screened selector (bf16 pre-scan + f64 rescoring of the candidates) picks exactly the
    blocks a full f64 scan of the pool picks, so every later quantity is bitwise identical; the
    pre-scan fused into select_plan (default) and as its own kernel (NOSA_SPLIT_SCAN) alike."""
    cfg = ONE_B_SMALL
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, 4)
    K, V = workload.prefix_kv(4, 6, cfg.n_kv_head, 6000, cfg.d_head)
    K = (K * kscale).astype(np.float32)
    K, V = K.reshape(2, 3, cfg.n_kv_head, 6000, cfg.d_head), V.reshape(2, 3, cfg.n_kv_head, 6000, cfg.d_head)
    runs = []
    for exact, split in ((True, False), (False, False), (False, True)):
        if split:
            monkeypatch.setenv("NOSA_SPLIT_SCAN", "1")  # read when the context is created
        else:
            monkeypatch.delenv("NOSA_SPLIT_SCAN", raising=False)
        eng = NosaEngine(cfg, batch=3, layers=2, max_tokens=6100, fast_slots=75, w1=w1, w2=w2, dtype=dtype,
                         exact_scan=exact)
        eng.prefill(torch.from_numpy(K), torch.from_numpy(V))
        eng.start_run()
        stream = workload.QueryStream(4, 2, 3, cfg.n_head, cfg.n_kv_head, cfg.d_head, 0.2)
        outs, sels = [], []
        for _ in range(25):
            q, kn, vn = stream.next()
            outs.append(eng.step((q * qscale).astype(np.float32), kn, vn, selector=selector).cpu().numpy())
            sels.append([eng.raw_selection(l)[:4] for l in range(2)])
        st = eng.residency_stats()
        runs.append((np.stack(outs), sels, (st.hits, st.misses, st.evictions)))
        eng.close()
    for other in runs[1:]:
        np.testing.assert_array_equal(runs[0][0], other[0])
        assert runs[0][2] == other[2]
        for a, b in zip(runs[0][1], other[1]):
            for la, lb in zip(a, b):
                for x, y in zip(la, lb):
                    np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("gather", ["memcpy", "uva", "tma"])
def test_peer_slow_tier_loopback(gather):
    """The slow tier in GPU memory (misses served from a peer's HBM over NVLink);
    on one GPU the peer is the engine's own device.  Same selections, residency and outputs."""
    a = _run_pair(ONE_B_SMALL, batch=2, t0s=[3000, 2600], steps=12, fast_slots=70, seed=19, rho=0.0, layers=2,
                  gather=gather, slow_tier="peer:0")
    assert a <= TOL["bf16"]


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("selector", ["nosa", "infllmv2"])
def test_exact_score_ties_pick_the_lower_block(exact, selector):
    """Duplicated KV blocks have bitwise equal block means, so their scores tie exactly; the
    selectors must break the tie by the lower block index like argtopk (numerics.py:59-73),
    with no tolerance (selection given scores is pinned exactly)."""
    cfg = ONE_B_SMALL
    B, t0, steps, C, seed = 2, 5000, 10, 72, 31
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, seed)
    K, V = workload.prefix_kv(seed, B, cfg.n_kv_head, t0, cfg.d_head)
    n_b = cfg.n_b
    for b in range(B):  # blocks 10..39 copy block 9, blocks 45..64 copy block 44 (pool = 1..62)
        for src, dsts in ((9, range(10, 40)), (44, range(45, 65))):
            for d in dsts:
                K[b, :, d * n_b:(d + 1) * n_b] = K[b, :, src * n_b:(src + 1) * n_b]
                V[b, :, d * n_b:(d + 1) * n_b] = V[b, :, src * n_b:(src + 1) * n_b]
    eng = NosaEngine(cfg, batch=B, max_tokens=t0 + steps + 1, fast_slots=C, w1=w1, w2=w2, exact_scan=exact)
    orc = oracle_for(cfg, B, 1, t0 + steps + 1, C, w1, w2)
    eng.prefill(torch.from_numpy(K), torch.from_numpy(V), layer=0)
    for b in range(B):
        orc.prefill(0, b, K[b], V[b])
    eng.start_run()
    orc.start_run()
    stream = workload.QueryStream(seed, 1, B, cfg.n_head, cfg.n_kv_head, cfg.d_head, 0.0)
    ties_at_boundary = 0
    for _ in range(steps):
        q, kn, vn = stream.next()
        out = eng.step(q, kn, vn, selector=selector).cpu().numpy()
        ref, recs = orc.step(q, kn, vn, selector)
        sels = eng.selections(0)
        for b in range(B):
            for h in range(cfg.n_kv_head):
                r = recs[0][b][h]
                assert list(sels[b][h].blocks_q) == r.blocks_q.tolist()
                assert list(sels[b][h].blocks_e) == r.blocks_e.tolist()
                lo = orc.geom[b].pool[0]
                chosen = set(r.blocks_q.tolist())
                inside = [r.s_q[p - lo] for p in chosen]
                outside = [r.s_q[i] for i in range(len(r.s_q)) if i + lo not in chosen]
                ties_at_boundary += bool(inside and outside and min(inside) == max(outside))
        assert rel_err(out, ref) <= TOL["bf16"]
    assert ties_at_boundary > 0  # the duplicates did straddle the top-k boundary
    eng.close()


def test_resident_multilayer_batched_attention():
    """All blocks in HBM: several layers per persistent attention launch (6 layers = 4 + 2 here;
    the default batch is 8)."""
    a = _run_pair(ONE_B_SMALL, batch=2, t0s=[3000, 2900], steps=8, fast_slots=48, seed=17, rho=0.3, layers=6,
                  resident=True, attend_layers=4)
    assert a <= TOL["bf16"]
    a = _run_pair(ONE_B_SMALL, batch=2, t0s=[3000, 2900], steps=8, fast_slots=48, seed=17, rho=0.3, layers=6,
                  resident=True)
    assert a <= TOL["bf16"]


@pytest.mark.parametrize("gather", ["memcpy", "tma", "hostpack", "hybrid"])
def test_other_gather_paths_vs_oracle(gather):
    a = _run_pair(SMALL, batch=2, t0s=[900, 800], steps=20, fast_slots=36, seed=12, rho=0.0, gather=gather)
    assert a <= TOL["bf16"]


def test_gather_paths_and_schedules_bitwise_identical():
    """The mover and the layer schedule change when bytes move, never what is computed."""
    cfg = ONE_B_SMALL
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, 2)
    K, V = workload.prefix_kv(2, 6, cfg.n_kv_head, 3000, cfg.d_head)
    K, V = K.reshape(3, 2, cfg.n_kv_head, 3000, cfg.d_head), V.reshape(3, 2, cfg.n_kv_head, 3000, cfg.d_head)
    results = []
    runs = [("uva", "pipelined", False, 1), ("tma", "pipelined", False, 1), ("memcpy", "pipelined", False, 1),
            ("uva", "serial", False, 1), ("memcpy", "pipelined", True, 1), ("uva", "serial", True, 1),
            ("uva", "pipelined", False, 2), ("memcpy", "pipelined", True, 3), ("hostpack", "pipelined", False, 1),
            ("hostpack", "serial", False, 1), ("hostpack", "pipelined", True, 3), ("hybrid", "pipelined", False, 1),
            ("hybrid", "serial", False, 2), ("hybrid", "pipelined", True, 3)]
    for gather, schedule, host, att_layers in runs:
        eng = NosaEngine(cfg, batch=2, layers=3, max_tokens=3100, fast_slots=70, w1=w1, w2=w2,
                         attend_layers=att_layers)
        eng.prefill(torch.from_numpy(K), torch.from_numpy(V))
        eng.start_run()
        stream = workload.QueryStream(2, 3, 2, cfg.n_head, cfg.n_kv_head, cfg.d_head, 0.0)
        if host:  # nosa_decode_step_host: pinned host tensors in, host outputs back
            outs = [eng.step_host(*stream.next(), gather=gather,
                                  schedule=schedule).clone().numpy() for _ in range(70)]
        else:
            outs = [eng.step(*stream.next(), gather=gather, schedule=schedule).cpu().numpy() for _ in range(70)]
        st = eng.residency_stats()
        results.append((np.stack(outs), st.hits, st.misses, st.evictions))
        eng.close()
    for r in results[1:]:
        np.testing.assert_array_equal(r[0], results[0][0])
        assert r[1:] == results[0][1:]


def test_host_step_graph_replay_matches_eager():
    """nosa_step_graph_launch_host re-points the captured graph at each step's pinned buffers."""
    cfg = ONE_B_SMALL
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, 5)
    K, V = workload.prefix_kv(5, 4, cfg.n_kv_head, 4000, cfg.d_head)
    K, V = K.reshape(2, 2, cfg.n_kv_head, 4000, cfg.d_head), V.reshape(2, 2, cfg.n_kv_head, 4000, cfg.d_head)
    outs = []
    for use_graph in (False, True):
        eng = NosaEngine(cfg, batch=2, layers=2, max_tokens=4100, fast_slots=70, w1=w1, w2=w2)
        eng.prefill(torch.from_numpy(K), torch.from_numpy(V))
        eng.start_run()
        stream = workload.QueryStream(5, 2, 2, cfg.n_head, cfg.n_kv_head, cfg.d_head, 0.3)
        res = []
        for s in range(8):
            hq, hk, hv = (torch.from_numpy(x).to(torch.bfloat16).pin_memory() for x in stream.next())
            ho = torch.empty((2, 2, cfg.n_head, cfg.d_head), dtype=torch.float32, pin_memory=True)
            if use_graph:
                if s == 0:
                    eng.capture_host(hq, hk, hv, ho)
                eng.replay_host(hq, hk, hv, ho)  # new buffers every step
                torch.cuda.synchronize()
            else:
                eng.step_host(hq, hk, hv, out=ho, gather="uva")
            res.append(ho.numpy().copy())
        outs.append(np.stack(res))
        eng.close()
    np.testing.assert_array_equal(outs[0], outs[1])


def test_capacity_exceeded_is_raised():
    w1, w2 = workload.eviction_head(SMALL.n_head, SMALL.d_head, 0)
    eng = NosaEngine(SMALL, batch=1, max_tokens=1100, fast_slots=10, w1=w1, w2=w2)
    K, V = workload.prefix_kv(0, 1, SMALL.n_kv_head, 1000, SMALL.d_head)
    eng.prefill(torch.from_numpy(K), torch.from_numpy(V), layer=0)
    q, kn, vn = workload.QueryStream(0, 1, 1, SMALL.n_head, SMALL.n_kv_head, SMALL.d_head, 0.5).next()
    with pytest.raises(CapacityExceeded):
        eng.step(q, kn, vn)
    eng.close()


def test_full_head_cache_append_refused(monkeypatch):
    """A step past the head capacity (HeadState, decode.py:65-71): the host entry points refuse it,
    and with the host check bypassed the device append refuses it too (NOSA_FLAG_FULL) instead of
    writing into the next row's block 0."""
    cfg = ONE_B_SMALL
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, 0)
    t0 = 64 * 80 - 1                       # one step fills the last block exactly
    eng = NosaEngine(cfg, batch=2, layers=1, max_tokens=t0 + 1, fast_slots=81, w1=w1, w2=w2)
    K, V = workload.prefix_kv(0, 2, cfg.n_kv_head, t0, cfg.d_head)
    eng.prefill(torch.from_numpy(K), torch.from_numpy(V), layer=0)
    eng.start_run()
    stream = workload.QueryStream(0, 1, 2, cfg.n_head, cfg.n_kv_head, cfg.d_head, 0.9)
    eng.step(*stream.next())
    rows = [(b, h) for b in range(2) for h in range(cfg.n_kv_head)]
    before = [eng.read_kv(0, b, h, t=t0 + 1) for b, h in rows]
    with pytest.raises(ValueError, match="capacity exhausted"):
        eng.step(*stream.next())
    with pytest.raises(ValueError, match="capacity exhausted"):
        eng.replay()
    monkeypatch.setattr(eng, "_check_step", lambda: None)
    with pytest.raises(ValueError, match="capacity exhausted"):
        eng.step(*stream.next())                               # device flag, raised by check_errors
    assert list(eng.lengths()[0]) == [t0 + 1, t0 + 1]
    for (b, h), (k0, v0) in zip(rows, before):                 # no row was overwritten
        k1, v1 = eng.read_kv(0, b, h, t=t0 + 1)
        np.testing.assert_array_equal(k1, k0)
        np.testing.assert_array_equal(v1, v0)
    eng.close()


def test_empty_cache_rejected():
    w1, w2 = workload.eviction_head(SMALL.n_head, SMALL.d_head, 0)
    eng = NosaEngine(SMALL, batch=1, max_tokens=100, fast_slots=10, w1=w1, w2=w2)
    q, kn, vn = workload.QueryStream(0, 1, 1, SMALL.n_head, SMALL.n_kv_head, SMALL.d_head, 0.5).next()
    with pytest.raises(ValueError, match="empty support"):
        eng.step(q, kn, vn)
    eng.close()


def test_graph_replay_matches_eager():
    cfg = ONE_B_SMALL
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, 1)
    K, V = workload.prefix_kv(1, 2, cfg.n_kv_head, 5000, cfg.d_head)
    outs = []
    for use_graph in (False, True):
        eng = NosaEngine(cfg, batch=2, layers=1, max_tokens=5100, fast_slots=70, w1=w1, w2=w2)
        eng.prefill(torch.from_numpy(K), torch.from_numpy(V), layer=0)
        eng.start_run()
        stream = workload.QueryStream(1, 1, 2, cfg.n_head, cfg.n_kv_head, cfg.d_head, 0.9)
        dev = eng.device
        qb = torch.empty((1, 2, cfg.n_head, cfg.d_head), dtype=torch.bfloat16, device=dev)
        kb = torch.empty((1, 2, cfg.n_kv_head, cfg.d_head), dtype=torch.bfloat16, device=dev)
        vb = torch.empty_like(kb)
        ob = torch.empty((1, 2, cfg.n_head, cfg.d_head), dtype=torch.float32, device=dev)
        res = []
        for s in range(6):
            q, kn, vn = stream.next()
            qb.copy_(torch.from_numpy(q)); kb.copy_(torch.from_numpy(kn)); vb.copy_(torch.from_numpy(vn))
            if use_graph:
                if s == 0:
                    eng.capture(qb, kb, vb, ob)
                    eng.timing_enable(4 * 3 + 1)  # room for three timed replays
                eng.replay()
            else:
                eng.step(qb, kb, vb, out=ob)
            res.append(ob.cpu().numpy().copy())
        if use_graph:  # replays are timed per kernel through the re-pointed event-record nodes
            timing = eng.timing_read()
            assert [timing[k]["launches"] for k in eng.KERNEL_KINDS] == [3, 3, 3, 3]
            assert all(timing[k]["total_ms"] > 0 for k in ("select_plan", "attend", "finalize"))
        outs.append(np.stack(res))
        eng.close()
    np.testing.assert_array_equal(outs[0], outs[1])  # same kernels, same decomposition: bitwise equal


@pytest.mark.parametrize("selector", ["nosa", "infllmv2"])
def test_full_context_invariants(selector):
    """BASELINE config 3's context (32K tokens, 25% of blocks in HBM) through size-independent
    properties: the picks are the argtopk of the exact f64 pool scores (read back), required =
    sink U picks U recent, every required block is resident after the plan, the slot table is a
    bijection on at most C slots, hits + misses = |required| and misses = |fetch|."""
    from paper_2510_13602_b200 import one_b_config
    cfg = one_b_config(65536)
    B, L, T, steps = 4, 2, 32768, 4
    max_tokens = T + steps + 2
    nblk = -(-max_tokens // cfg.n_b)
    C = nblk // 4
    dev = torch.device("cuda", 0)
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, 3)
    eng = NosaEngine(cfg, batch=B, layers=L, max_tokens=max_tokens, fast_slots=C, w1=w1, w2=w2)
    for l in range(L):
        shape = (B, cfg.n_kv_head, T, cfg.d_head)
        eng.prefill(workload.torch_prefix_kv(10 + 2 * l, shape, dev, torch.bfloat16),
                    workload.torch_prefix_kv(11 + 2 * l, shape, dev, torch.bfloat16), layer=l)
    eng.start_run()
    qs = workload.TorchQueryStream(5, L, B, cfg.n_head, cfg.n_kv_head, cfg.d_head, 0.5, dev, torch.bfloat16)
    m_q = cfg.blocks_q if selector == "nosa" else cfg.blocks_topk
    for _ in range(steps):
        q, kn, vn = qs.next()
        eng.step(q, kn, vn, selector=selector, gather="memcpy")
        for l in range(L):
            bq, nq, be, ne, rq, nr, s_q = eng.raw_selection(l)
            plans = eng.plans(l)
            for b in range(B):
                geom = eng.geometry[b]
                lo, hi = geom.pool_blocks.start, geom.pool_blocks.stop
                t = int(eng._t[l, b]) - 1
                for h in range(cfg.n_kv_head):
                    scores = s_q[b, h, lo:hi]
                    want = sorted(lo + i for i in sorted(range(hi - lo), key=lambda i: (-scores[i], i))[:m_q])
                    assert bq[b, h, :nq[b, h]].tolist() == want, (l, b, h)
                    picks = set(bq[b, h, :nq[b, h]].tolist()) | set(be[b, h, :ne[b, h]].tolist())
                    fixed = set(geom.fixed_blocks(t))
                    req = rq[b, h, :nr[b, h]].tolist()
                    assert req == sorted(fixed | picks) and not (fixed & picks)
                    slot_of, block_of = eng.residency(l, b, h)
                    resident = {blk: int(sl) for blk, sl in enumerate(slot_of) if sl >= 0}
                    assert all(r in resident for r in req)
                    assert len(resident) <= C and len(set(resident.values())) == len(resident)
                    assert all(block_of[sl] == blk for blk, sl in resident.items())
                    p = plans[b][h]
                    assert p.hits + len(p.fetch) == len(req) and not (set(p.fetch) & set(p.evict))
    eng.close()


def test_all_resident_run_launches_no_gather(monkeypatch):
    """Resident prefill and room for every block the run can create: nothing is ever evicted,
    the only misses are newborn blocks, the planner writes those itself and the step launches no
    gather.  Bitwise the same outputs, selections, plans and residency as the run that gathers
    (NOSA_GATHER_ALWAYS) and as the captured step graph's replays, across block boundaries of
    both sequences, with no device error flag."""
    cfg = ONE_B_SMALL
    B, L, steps, seed = 2, 3, 24, 23
    t0s = [3000, 2990]  # both cross the 3008 boundary inside the run
    cap = max(t0s) + steps + 1
    nblk = -(-cap // cfg.n_b)
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, seed)
    K, V = workload.prefix_kv(seed, B * L, cfg.n_kv_head, max(t0s), cfg.d_head)
    K = K.reshape(L, B, cfg.n_kv_head, max(t0s), cfg.d_head)
    V = V.reshape(L, B, cfg.n_kv_head, max(t0s), cfg.d_head)
    runs = []
    for mode in ("local", "always", "graph"):
        if mode == "always":
            monkeypatch.setenv("NOSA_GATHER_ALWAYS", "1")
        else:
            monkeypatch.delenv("NOSA_GATHER_ALWAYS", raising=False)
        eng = NosaEngine(cfg, batch=B, layers=L, max_tokens=cap, fast_slots=nblk, w1=w1, w2=w2)
        for l in range(L):
            for b in range(B):
                t = t0s[b]
                eng.prefill(torch.from_numpy(np.ascontiguousarray(K[l, b:b + 1, :, :t])),
                            torch.from_numpy(np.ascontiguousarray(V[l, b:b + 1, :, :t])), layer=l, seq_begin=b,
                            resident=True)
        eng.start_run()
        eng.timing_enable(4096)
        stream = workload.QueryStream(seed, L, B, cfg.n_head, cfg.n_kv_head, cfg.d_head, 0.3)
        dev = eng.device
        qb = torch.empty((L, B, cfg.n_head, cfg.d_head), dtype=torch.bfloat16, device=dev)
        kb = torch.empty((L, B, cfg.n_kv_head, cfg.d_head), dtype=torch.bfloat16, device=dev)
        vb = torch.empty_like(kb)
        ob = torch.empty((L, B, cfg.n_head, cfg.d_head), dtype=torch.float32, device=dev)
        outs, plans = [], []
        for s in range(steps):
            q, kn, vn = stream.next()
            if mode == "graph":
                qb.copy_(torch.from_numpy(q)); kb.copy_(torch.from_numpy(kn)); vb.copy_(torch.from_numpy(vn))
                if s == 0:
                    eng.capture(qb, kb, vb, ob)
                eng.replay()
                outs.append(ob.cpu().numpy().copy())
            else:
                outs.append(eng.step(q, kn, vn).cpu().numpy())
            plans.append([[(p.fetch, p.evict, p.hits) for p in row] for l in range(L) for row in eng.plans(l)])
        eng.check_errors()
        st = eng.residency_stats()
        gathers = eng.timing_read()["gather"]["launches"] if mode != "graph" else None
        res = [eng.residency(l, b, h) for l in range(L) for b in range(B) for h in range(cfg.n_kv_head)]
        runs.append((np.stack(outs), plans, (st.hits, st.misses, st.evictions), gathers, res))
        eng.close()
    (o0, p0, s0, g0, r0) = runs[0]
    assert g0 == 0 and runs[1][3] > 0
    assert s0[2] == 0 and s0[1] > 0  # the newborn blocks are counted as misses
    for o1, p1, s1, _, r1 in runs[1:]:
        assert s0 == s1
        assert p0 == p1
        np.testing.assert_array_equal(o0, o1)
        for a, b in zip(r0, r1):
            for x, y in zip(a, b):
                np.testing.assert_array_equal(np.asarray(x), np.asarray(y))


def test_fp32_multilayer_batched_attention():
    """fp32 storage, the warp-group CUDA-core kernel over several layers per persistent launch,
    against the oracle at the fp32 tolerance (offloaded and resident)."""
    a = _run_pair(ONE_B_SMALL, batch=2, t0s=[3000, 2900], steps=8, fast_slots=48, seed=17, rho=0.3, layers=6,
                  resident=True, attend_layers=4, dtype="fp32")
    assert a <= TOL["fp32"]
    a = _run_pair(ONE_B_SMALL, batch=3, t0s=[2000, 2500, 1700], steps=10, fast_slots=40, seed=18, rho=0.0,
                  layers=3, attend_layers=3, dtype="fp32")
    assert a <= TOL["fp32"]


def test_fp32_attention_bitwise_independent_of_launch_grouping():
    """The fp32 kernel's result depends on the fixed chunking and its fixed reduction tree only:
    layers per launch, mover and host-buffer staging leave every output bit unchanged."""
    cfg = ONE_B_SMALL
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, 4)
    K, V = workload.prefix_kv(4, 6, cfg.n_kv_head, 2600, cfg.d_head, bf16=False)
    K, V = K.reshape(3, 2, cfg.n_kv_head, 2600, cfg.d_head), V.reshape(3, 2, cfg.n_kv_head, 2600, cfg.d_head)
    results = []
    for gather, host, att_layers in [("uva", False, 1), ("uva", False, 3), ("memcpy", False, 2), ("uva", True, 3)]:
        eng = NosaEngine(cfg, batch=2, layers=3, max_tokens=2700, fast_slots=60, w1=w1, w2=w2, dtype="fp32",
                         attend_layers=att_layers)
        eng.prefill(torch.from_numpy(K), torch.from_numpy(V))
        eng.start_run()
        stream = workload.QueryStream(4, 3, 2, cfg.n_head, cfg.n_kv_head, cfg.d_head, 0.0, bf16=False)
        if host:
            outs = [eng.step_host(*stream.next(), gather=gather).clone().numpy() for _ in range(30)]
        else:
            outs = [eng.step(*stream.next(), gather=gather).cpu().numpy() for _ in range(30)]
        results.append(np.stack(outs))
        eng.close()
    for r in results[1:]:
        np.testing.assert_array_equal(r, results[0])


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("n_head,d_head", [(12, 128), (10, 64), (32, 64)])
def test_padded_and_wide_query_groups(dtype, n_head, d_head):
    """Query groups the kernels pad (G = 6 and 5 of 8 columns: the fp32 tensor-core QK with zero
    query rows) or split (G = 16: the fp32 CUDA-core reduce-scatter, two bf16 N tiles) against
    the oracle at each dtype's tolerance."""
    cfg = AttentionConfig(n=8192, d=n_head * d_head, n_head=n_head, n_kv_head=2, d_head=d_head, n_b=64, n_s=64,
                          n_w=1024, k=4096, k_q=1024, k_e=3072)
    a = _run_pair(cfg, batch=2, t0s=[2600, 2400], steps=6, fast_slots=48, seed=23, rho=0.2, layers=2,
                  dtype=dtype)
    assert a <= TOL[dtype]
