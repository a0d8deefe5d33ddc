"""The drop-in selectors (nosa_select / infllmv2_select on given scores) and the GPU block
manager against the reference's golden vectors and its own known-answer tests."""

import numpy as np
import pytest

from paper_2510_13602_b200 import (AttentionConfig, BlockGeometry, CapacityExceeded, GpuTieredBlockManager,
                                   StalePlan, UnknownKey, infllmv2_select, nosa_select)
from paper_2510_13602_b200.selection import select_batch

pytestmark = pytest.mark.gpu


def _cfg(row):
    n, d, n_head, n_kv, d_head, n_b, n_s, n_w, k, k_q, k_e, excl = (int(x) for x in row)
    return AttentionConfig(n=n, d=d, n_head=n_head, n_kv_head=n_kv, d_head=d_head, n_b=n_b, n_s=n_s, n_w=n_w,
                           k=k, k_q=k_q, k_e=k_e, accounting="exclusive" if excl else "inclusive")


def test_selector_golden_kats_bit_exact(golden):
    g = golden("selection_kats")
    for i in range(len(g["t"])):
        cfg = _cfg(g["cfg_rows"][g["cfg"][i]])
        t, nblk = int(g["t"][i]), int(g["nblk"][i])
        s_q, s_e = g["s_q"][i][:nblk], g["s_e"][i][:nblk]
        want = lambda key: tuple(int(x) for x in g[key][i] if x >= 0)
        a = nosa_select(s_q, s_e, t, cfg)
        assert a.blocks_q == want("nosa_q") and a.blocks_e == want("nosa_e"), i
        assert a.blocks_fixed == want("fixed"), i
        b = infllmv2_select(s_q, t, cfg)
        assert b.blocks_q == want("inf_q") and b.blocks_e == (), i


def test_tie_rule_and_negative_zero():
    # argtopk([1,1,1], 2) -> {0,1} (test_numerics.py:96-97); -0.0 == +0.0 ties go to the lower index
    sq, _ = select_batch(np.array([[1.0, 1.0, 1.0]]), None, [0], [3], 2, 0, "infllmv2")
    assert sq[0].tolist() == [0, 1]
    sq, _ = select_batch(np.array([[0.0, -0.0, 1.0]]), None, [0], [3], 2, 0, "infllmv2")
    assert sq[0].tolist() == [0, 2]
    sq, _ = select_batch(np.array([[-0.0, 0.0, -1.0]]), None, [0], [3], 1, 0, "infllmv2")
    assert sq[0].tolist() == [0]


def test_lift_oracle_random_batches(rng):
    # nosa_select == single top-k over the lifted score (test_selection.py:14-24, 100-107)
    n, P, m_q, m_e = 500, 300, 16, 31
    s_q = np.round(rng.standard_normal((n, P)), 1)
    s_e = np.round(rng.standard_normal((n, P)), 1)
    got_q, got_e = select_batch(s_q, s_e, np.zeros(n), np.full(n, P), m_q, m_e, "nosa")
    for i in range(n):
        pool = list(range(P))
        picked_q = set(sorted(pool, key=lambda b: (-s_q[i, b], b))[:m_q])
        lifted = {b: (np.inf if b in picked_q else s_e[i, b]) for b in pool}
        want = set(sorted(pool, key=lambda b: (-lifted[b], b))[:m_q + m_e])
        assert set(got_q[i]) | set(got_e[i]) == want
        assert set(got_q[i]) == picked_q


def test_short_score_vector_rejected():
    cfg = AttentionConfig(n=2048, d=8, n_head=1, n_kv_head=1, d_head=8, n_b=16, n_s=32, n_w=64, k=288, k_q=64,
                          k_e=224)
    with pytest.raises(ValueError, match="cover all"):
        nosa_select(np.zeros(3), np.zeros(3), 1024, cfg)


# ---------------------------------------------------------------- manager KATs (test_kv_manager.py)
def _mgr(fast=6, slow=32, heads=1, batch=1):
    return GpuTieredBlockManager(fast, slow, heads=heads, batch=batch, n_b=16, d_head=64)


def test_cold_start_fetches_everything():
    m = _mgr()
    p = m.plan_transfers({1, 2, 3}, 0, 0)
    assert sorted(k[2] for k in p.fetch) == [1, 2, 3] and p.hits == 0
    assert p.bytes_up == 3 * m.bytes_per_block


def test_resident_set_is_noop_and_plan_minimal():
    m = _mgr()
    m.apply_transfers(m.plan_transfers({1, 2, 3}, 0, 0))
    p = m.plan_transfers({1, 2, 3}, 0, 0)
    assert p.empty and p.hits == 3
    m.apply_transfers(p)
    p = m.plan_transfers({1, 2, 5, 7}, 0, 0)
    assert sorted(k[2] for k in p.fetch) == [5, 7] and p.evict == []


def test_lrr_victim():
    m = _mgr(fast=3)
    m.apply_transfers(m.plan_transfers({0, 1, 2}, 0, 0))
    m.apply_transfers(m.plan_transfers({1, 2}, 0, 0))
    p = m.plan_transfers({1, 2, 5}, 0, 0)
    assert [k[2] for k in p.evict] == [0]
    m.apply_transfers(p)
    assert m.fast_resident(0, 0) == {1, 2, 5}
    assert m.lookup(0, 0, 0)[0] == "slow"


def test_hand_counted_trace():
    # test_kv_manager.py:290-302: hits 8, misses 9, bytes_up 9 blocks
    m = _mgr(fast=4, slow=16)
    for req in [{0, 1}, {0, 1}, {1, 2, 3}, {3, 4}, {0, 4}, {0, 4}, {5, 6, 7}, {7}]:
        m.apply_transfers(m.plan_transfers(req, 0, 0))
    s = m.residency_stats()
    assert (s.hits, s.misses, s.steps) == (8, 9, 8)
    assert s.hit_rate == 8 / 17 and s.bytes_up == 9 * m.bytes_per_block


def test_errors():
    m = _mgr(fast=2)
    with pytest.raises(CapacityExceeded):
        m.plan_transfers({1, 2, 3}, 0, 0)
    with pytest.raises(UnknownKey):
        m.plan_transfers({99}, 0, 0)
    p = m.plan_transfers({1}, 0, 0)
    m.plan_transfers({2}, 0, 0)
    with pytest.raises(StalePlan):
        m.apply_transfers(p)


def test_manager_golden_trace_bit_exact(golden):
    g = golden("manager_trace")
    C, nblk = int(g["capacity"]), int(g["nblk"])
    steps, H, _ = g["req"].shape
    m = GpuTieredBlockManager(C, nblk, heads=H, batch=1, n_b=16, d_head=64)
    for s in range(steps):
        for h in range(H):
            req = [int(x) for x in g["req"][s, h] if x >= 0]
            p = m.plan_transfers(req, 0, h)
            assert [k[2] for k in p.fetch] == [x for x in g["fetch"][s, h] if x >= 0], (s, h)
            assert [k[2] for k in p.evict] == [x for x in g["evict"][s, h] if x >= 0], (s, h)
            assert p.hits == g["hits"][s, h]
        if s % 50 == 0:
            for h in range(H):
                req = [int(x) for x in g["req"][s, h] if x >= 0]
                assert [m.lookup(0, h, b)[2] for b in req] == [x for x in g["slots"][s, h] if x >= 0]
    hits, misses, _, calls = g["stats"]
    st = m.residency_stats()
    assert (st.hits, st.misses, st.steps) == (hits, misses, calls)


def test_payload_round_trip_through_gather():
    # bytes written to the slow tier arrive unchanged in the fetched fast slot (test_kv_manager.py:252-267)
    import torch
    from paper_2510_13602_b200 import NosaEngine, workload
    cfg = AttentionConfig(n=4096, d=512, n_head=4, n_kv_head=2, d_head=64, n_b=16, n_s=32, n_w=128, k=512, k_q=128,
                          k_e=384)
    w1, w2 = workload.eviction_head(4, 64, 0)
    eng = NosaEngine(cfg, batch=1, max_tokens=1100, fast_slots=40, w1=w1, w2=w2)
    K, V = workload.prefix_kv(0, 1, 2, 1000, 64)
    eng.prefill(torch.from_numpy(K), torch.from_numpy(V), layer=0)
    q, kn, vn = workload.QueryStream(0, 1, 1, 4, 2, 64, 0.5).next()
    eng.step(q, kn, vn)
    for h in range(2):
        slot_of, _ = eng.residency(0, 0, h)
        for blk in np.flatnonzero(slot_of >= 0):
            kv = eng.read_slot(0, 0, h, int(slot_of[blk]))
            rows = slice(blk * 16, min(blk * 16 + 16, 1000))
            n = rows.stop - rows.start
            np.testing.assert_array_equal(kv[0, :n], K[0, h, rows])
            np.testing.assert_array_equal(kv[1, :n], V[0, h, rows])
    eng.close()


@pytest.mark.parametrize("tag", ["nosa", "infllmv2"])
def test_shared_pool_manager_reproduces_reference_simulator(golden, tag):
    """GPU shared-pool planner fed the reference simulator's own required sets
    (offload_sim.simulate_decode, scripted AR(1) selections): identical fetch and evict lists
    (victims across sequences) and the simulator's SimReport hit rates and bytes."""
    g = golden("shared_pool_sim")
    B, H, slots, total, _, steps = (int(x) for x in g[f"{tag}_shape"])
    m = GpuTieredBlockManager(B * slots, total, heads=H, batch=B, n_b=16, d_head=64, shared=True)
    topk_hits = topk_total = 0
    for i in range(steps + 1):
        if i == 1:
            m.reset_stats()  # warm-up with step 0 (offload_sim.py:268-274)
        req = {(b, h): {int(x) for x in g[f"{tag}_req"][i, b, h] if x >= 0} for b in range(B) for h in range(H)}
        plans = m.plan_batch(req)
        for b in range(B):
            for h in range(H):
                p = plans[(b, h)]
                assert [k[2] for k in p.fetch] == [x for x in g[f"{tag}_fetch"][i, b, h] if x >= 0], (i, b, h)
                assert [[k[0], k[2]] for k in p.evict] == [list(e) for e in g[f"{tag}_evict"][i, b, h] if e[0] >= 0]
                if i:
                    tk = {x for x in g[f"{tag}_topk"][i, b, h] if x >= 0}
                    topk_hits += len(tk - {k[2] for k in p.fetch})
                    topk_total += len(tk)
    hit_rate, hit_rate_topk, bytes_up, bytes_down = g[f"{tag}_report"]
    st = m.residency_stats()
    assert st.hit_rate == hit_rate
    assert topk_hits / topk_total == hit_rate_topk
    # the reference's layout counts 2 bytes per element for a d_head-8 head; scale by block size
    assert st.misses * (2 * 16 * 8 * 2) == bytes_up and st.evictions * (2 * 16 * 8 * 2) == bytes_down
    m.close()
