"""Bit-exact parity at the BASELINE headline configurations (the 1B attention shape at 16K / 32K /
64K context, 25% of the KV blocks in HBM, high- and low-locality query streams, both selectors).

The GPU engine and the CPU oracle decode the SAME counter-based inputs (drawn on the GPU by
nosa_synth_*, on the host by workload.synth_*; the two generators are checked bit for bit here).
Every step of every (layer, sequence, head) must agree exactly on blocks_q, blocks_e, the required
list, the fetch list (plan order), the eviction list (LRR order) and the hit count; the final slot
tables and the residency counters must be identical; outputs must be within 2e-2 (bf16 storage).
A selection mismatch is accepted only on an exact score tie, which is reported (none so far).
The oracle itself is pinned to the unmodified reference at the same shape, context, cache size and
inputs by tests/golden/engine_1b_32k*.npz (tests/test_oracle_golden.py), which the first test
here also checks the GPU against directly.
"""

import numpy as np
import pytest
import torch

from oracle import nosa_oracle as O
from paper_2510_13602_b200 import NosaEngine, one_b_config, synth, workload

from helpers import rel_err

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _tie_ok(got, want, scores, what):
    """Exact equality, or an exact score tie at the selection boundary (reported)."""
    if list(got) == list(want):
        return 0
    g, w = set(got), set(want)
    diff = [scores[x] for x in g ^ w]
    assert len(set(diff)) == 1, f"{what}: GPU {sorted(g - w)} vs oracle {sorted(w - g)} (no tie)"
    print(f"reported tie at {what}: {sorted(g ^ w)}")
    return 1


def run_headline(*, t0, fast_slots, batch, layers, steps, rho, selector="nosa", seed=0, resident=False,
                 gather="auto", seq0=0, dense=False):
    """GPU engine vs oracle on identical synth inputs; returns (worst output error, ties, evictions)."""
    cfg = one_b_config(65536)
    H, Hq, D = cfg.n_kv_head, cfg.n_head, cfg.d_head
    cap = t0 + steps + 2
    w1, w2 = workload.eviction_head(Hq, D, seed)
    eng = NosaEngine(cfg, batch=batch, layers=layers, max_tokens=cap, fast_slots=fast_slots, w1=w1, w2=w2)
    orc = O.OracleEngine(O.OracleConfig.from_attention_config(cfg), batch, layers, cap, fast_slots, w1, w2,
                         dense=dense)
    for l in range(layers):
        k, v = synth.prefix_kv(seed, l, seq0, batch, H, t0, D, DEV)
        eng.prefill(k, v, layer=l, resident=resident)
        Kn, Vn = workload.synth_prefix_kv(seed, l, range(seq0, seq0 + batch), H, t0, D)
        # the two generators agree bit for bit (a sample of rows; the whole tensor at small t)
        assert torch.equal(k[:, :, :257].float().cpu(), torch.from_numpy(Kn[:, :, :257]))
        assert torch.equal(v[:, :, -129:].float().cpu(), torch.from_numpy(Vn[:, :, -129:]))
        for b in range(batch):
            orc.prefill(l, b, Kn[b], Vn[b])
            if resident:
                for h in range(H):
                    orc.managers[l][b].make_resident(h, -(-t0 // cfg.n_b))
        del k, v
    eng.start_run()
    orc.start_run()
    gstream = synth.GpuQueryStream(seed, layers, seq0, batch, Hq, H, D, rho, DEV)
    cstream = workload.SynthQueryStream(seed, range(layers), range(seq0, seq0 + batch), Hq, H, D, rho)
    worst, ties = 0.0, 0
    for s in range(steps):
        q, kn, vn = gstream.next()
        cq, ck, cv = cstream.next()
        assert torch.equal(q.float().cpu(), torch.from_numpy(cq)), f"query stream differs at step {s}"
        assert torch.equal(kn.float().cpu(), torch.from_numpy(ck)) and torch.equal(vn.float().cpu(), torch.from_numpy(cv))
        out = eng.step(q, kn, vn, selector=selector, gather=gather).cpu().numpy()
        ref, recs = orc.step(cq, ck, cv, selector)
        for l in range(layers):
            bq, nq, be, ne, req, nreq, s_q = eng.raw_selection(l)
            plans = eng.plans(l)
            for b in range(batch):
                lo, hi = orc.geom[b].pool
                for h in range(H):
                    r = recs[l][b][h]
                    where = f"step {s} layer {l} seq {b} head {h}"
                    sc = np.zeros(max(hi, 1))
                    sc[lo:hi] = r.s_q
                    ties += _tie_ok(bq[b, h, :nq[b, h]].tolist(), r.blocks_q.tolist(), sc, where + " blocks_q")
                    sc[lo:hi] = r.s_e_c
                    ties += _tie_ok(be[b, h, :ne[b, h]].tolist(), r.blocks_e.tolist(), sc, where + " blocks_e")
                    assert req[b, h, :nreq[b, h]].tolist() == r.required, where + " required"
                    assert plans[b][h].fetch == r.fetch, where + " fetch"
                    assert plans[b][h].evict == r.evict, where + " evict"
                    assert plans[b][h].hits == r.hits, where + " hits"
        worst = max(worst, rel_err(out, ref))
        assert worst <= 2e-2, f"step {s}: relative output error {worst:.3e}"
    for l in range(layers):
        for b in range(batch):
            for h in range(H):
                slot_of, _ = eng.residency(l, b, h)
                got = {int(blk): int(sl) for blk, sl in enumerate(slot_of) if sl >= 0}
                assert got == orc.managers[l][b].slot_of[h], f"slot table layer {l} seq {b} head {h}"
    st, ost = eng.residency_stats(), orc.stats()
    assert (st.hits, st.misses, st.evictions, st.steps) == (ost["hits"], ost["misses"], ost["evictions"], ost["steps"])
    assert (st.topk_required, st.topk_misses) == (ost["topk_required"], ost["topk_misses"])  # hit_rate_topk
    eng.close()
    return worst, ties, ost["evictions"]


def test_golden_1b_32k_through_gpu(golden):
    """The unmodified reference (DecodeEngine + TieredBlockManager, 1B shape, 32K, 128 slots) vs the
    GPU engine on the same inputs: every selection, fetch/evict list and hit count over 40 steps,
    including the eviction regime from step 23 on."""
    for name in ("engine_1b_32k", "engine_1b_32k_infllmv2_rho0"):
        g = golden(name)
        cfg = one_b_config(65536)
        B, t0, steps, C, seed = (int(g[k]) for k in ("batch", "t0", "steps", "fast_slots", "seed"))
        rho, selector = float(g["rho"]), str(g["selector"])
        w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, seed)
        eng = NosaEngine(cfg, batch=B, max_tokens=t0 + steps + 1, fast_slots=C, w1=w1, w2=w2)
        k, v = synth.prefix_kv(seed, 0, 0, B, cfg.n_kv_head, t0, cfg.d_head, DEV)
        eng.prefill(k, v, layer=0)
        eng.start_run()
        stream = synth.GpuQueryStream(seed, 1, 0, B, cfg.n_head, cfg.n_kv_head, cfg.d_head, rho, DEV)
        for s in range(steps):
            out = eng.step(*stream.next(), selector=selector).cpu().numpy()
            bq, nq, be, ne, _, _, _ = eng.raw_selection(0)
            plans = eng.plans(0)
            for b in range(B):
                for h in range(cfg.n_kv_head):
                    assert bq[b, h, :nq[b, h]].tolist() == [x for x in g["sel_q"][s, b, h] if x >= 0], (name, s, h)
                    assert be[b, h, :ne[b, h]].tolist() == [x for x in g["sel_e"][s, b, h] if x >= 0], (name, s, h)
                    assert plans[b][h].fetch == [x for x in g["fetch"][s, b, h] if x >= 0], (name, s, h)
                    assert plans[b][h].evict == [x for x in g["evict"][s, b, h] if x >= 0], (name, s, h)
                    assert plans[b][h].hits == g["hits"][s, b, h], (name, s, h)
            err = rel_err(out[0], g["outputs"][s])
            assert err <= 2e-2, (name, s, err)
        eng.close()


def test_cfg3_32k_high_locality():
    """BASELINE config 3: 32K context, 25% cache (128 of 514 slots), rho = 0.95, NOSA; 2 sequences x
    2 layers, 36 steps (the cache fills and evicts from about step 22)."""
    worst, ties, evictions = run_headline(t0=32768, fast_slots=128, batch=2, layers=2, steps=36, rho=0.95)
    assert evictions > 0
    print(f"cfg3: worst output error {worst:.2e}, ties {ties}, evictions {evictions}")


@pytest.mark.parametrize("selector", ["nosa", "infllmv2"])
def test_cfg4_32k_low_locality(selector):
    """BASELINE config 4: the adversarial stream (rho = 0) at 32K, 25% cache, both selectors."""
    worst, ties, evictions = run_headline(t0=32768, fast_slots=128, batch=2, layers=2, steps=12, rho=0.0,
                                          selector=selector, seed=1, seq0=5)
    assert evictions > 0
    print(f"cfg4 {selector}: worst output error {worst:.2e}, ties {ties}, evictions {evictions}")


def test_cfg5_64k():
    """BASELINE config 5's shape: 64K context, 25% cache (256 of 1025 slots), rho = 0.95, sequences
    taken from the middle of the 512-sequence batch (global ids 300, 301: a rank's shard)."""
    worst, ties, evictions = run_headline(t0=65536, fast_slots=256, batch=2, layers=1, steps=72, rho=0.95, seed=2,
                                          seq0=300)
    assert evictions > 0
    print(f"cfg5: worst output error {worst:.2e}, ties {ties}, evictions {evictions}")


def test_cfg2_16k_resident():
    """BASELINE config 2: 16K context, every block resident in HBM (the copy-free path): the only
    misses are the blocks born during the run."""
    worst, ties, _ = run_headline(t0=16384, fast_slots=260, batch=2, layers=2, steps=10, rho=0.95, seed=3,
                                  resident=True)
    print(f"cfg2: worst output error {worst:.2e}, ties {ties}")


def test_gpu_generator_matches_numpy():
    """nosa_synth_* and the NumPy twin: whole tensors, several kinds, odd offsets, fp32 and bf16."""
    for kind in range(6):
        g = synth.normal(9, kind, 2, 3, 7, 5, 2, 1000, 33, 128, DEV, torch.float32)
        c = np.stack([workload.synth_normal(9, kind, 2 + l, range(7, 12), 2, 1000, 33, 128) for l in range(3)])
        assert torch.equal(g.cpu(), torch.from_numpy(c)), kind
    gb = synth.normal(9, 0, 0, 1, 0, 3, 2, 0, 100, 64, DEV)
    cb = workload.bf16_round(workload.synth_normal(9, 0, 0, range(3), 2, 0, 100, 64))
    assert torch.equal(gb[0].float().cpu(), torch.from_numpy(cb))
    gs = synth.GpuQueryStream(4, 3, 10, 4, 16, 2, 128, 0.5, DEV, torch.float32)
    cs = workload.SynthQueryStream(4, range(3), range(10, 14), 16, 2, 128, 0.5, bf16=False)
    for _ in range(5):
        for a, b in zip(gs.next(), cs.next()):
            assert torch.equal(a.cpu(), torch.from_numpy(b))
