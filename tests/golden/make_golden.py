"""Generate the golden fixtures from the UNMODIFIED reference package.

Run in the build container (the reference is not on the GPU box):
    NOSA_REF_PATH=/root/reference/pkg/src python tests/golden/make_golden.py
Writes tests/golden/*.npz.  Nothing here is imported by the product or by the GPU tests at run
time; the tests read only the .npz files.

Fixtures
  selection_kats.npz   nosa_select / infllmv2_select (selection.py:130-178) on random and
                       coarse-quantised scores (ties, -0.0) over several geometries
  manager_trace.npz    TieredBlockManager plan/apply (kv_manager.py:205-305) on random
                       required-set traces, one manager per sequence, all blocks slow at start
  engine_small.npz     DecodeEngine.step (decode.py:152-190) driven by 0/1 selection-matrix
                       projections so q/k/v are exact, ed-dma head built directly
                       (attention.py:104-118); selections, outputs, pool scores, plus the
                       per-sequence residency trace of the required sets (offload_sim.py:279-299)
  engine_cfg1.npz      the same at BASELINE config 1 (8q/2kv, d_head 128, 8K, block 64, top-k 16)
  engine_1b_32k*.npz   the same at the 1B shape, 32K context, 25% fast tier (128 slots), on the
                       counter-based inputs the bench draws (`make_golden.py headline`)
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("NOSA_REF_PATH", "/root/reference/pkg/src")
sys.path.insert(0, REF)
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from nosa_sim.attention import EvictionHead, compress_blocks  # noqa: E402
from nosa_sim.config import AttentionConfig  # noqa: E402
from nosa_sim.decode import DecodeEngine, ModelWeights  # noqa: E402
from nosa_sim.kv_manager import FAST, SLOW, PhysicalLayout, TieredBlockManager  # noqa: E402
from nosa_sim.selection import BlockGeometry, infllmv2_select, nosa_select  # noqa: E402

# the synthetic-input generator of the product (pure NumPy, no GPU needed)
import importlib.util  # noqa: E402

_spec = importlib.util.spec_from_file_location("workload", ROOT / "paper_2510_13602_b200" / "workload.py")
workload = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(workload)

OUT = Path(__file__).resolve().parent


def selection_kats():
    rows = []
    cfgs = [
        dict(n=4096, d=8, n_head=1, n_kv_head=1, d_head=8, n_b=16, n_s=32, n_w=64, k=288, k_q=64, k_e=224),
        dict(n=4096, d=8, n_head=1, n_kv_head=1, d_head=8, n_b=16, n_s=32, n_w=64, k=288, k_q=64, k_e=224,
             accounting="exclusive"),
        dict(n=65536, d=2048, n_head=16, n_kv_head=2, d_head=128, n_b=64, n_s=64, n_w=1024, k=4096, k_q=1024,
             k_e=3072),
        dict(n=16384, d=1024, n_head=8, n_kv_head=2, d_head=128, n_b=64, n_s=64, n_w=512, k=1024, k_q=256,
             k_e=768, accounting="exclusive"),
    ]
    rng = np.random.default_rng(20261017)
    for ci, c in enumerate(cfgs):
        cfg = AttentionConfig(**c)
        ts = [200, 1000, 2047] if cfg.n_b == 16 else [3000, 8192, 32768 + 5]
        for t in ts:
            if t > cfg.n:
                continue
            geom = BlockGeometry.for_run(cfg, t)
            nblk = geom.n_blocks(t)
            for mode in ("gauss", "coarse", "zeros"):
                s_q = rng.standard_normal(nblk)
                s_e = rng.standard_normal(nblk)
                if mode == "coarse":
                    s_q = np.round(s_q, 1)
                    s_e = np.round(s_e, 1)
                if mode == "zeros":  # -0.0 / +0.0 and heavy ties
                    s_q = np.where(rng.random(nblk) < 0.5, -0.0, 0.0) + np.round(rng.random(nblk)) * 0.5
                    s_e = np.where(rng.random(nblk) < 0.5, -0.0, 0.0)
                a = nosa_select(s_q, s_e, t, cfg, geometry=geom)
                b = infllmv2_select(s_q, t, cfg, geometry=geom)
                rows.append(dict(cfg=ci, t=t, s_q=s_q, s_e=s_e, nosa_q=a.blocks_q, nosa_e=a.blocks_e,
                                 fixed=a.blocks_fixed, inf_q=b.blocks_q))
    n = len(rows)
    L = max(len(r["s_q"]) for r in rows)
    pad = lambda key, width: np.array([list(r[key]) + [-1] * (width - len(r[key])) for r in rows], np.int64)
    np.savez_compressed(
        OUT / "selection_kats.npz",
        cfg_rows=np.array([[c.get(k) for k in ("n", "d", "n_head", "n_kv_head", "d_head", "n_b", "n_s", "n_w", "k",
                                                "k_q", "k_e")] + [1 if c.get("accounting") == "exclusive" else 0]
                           for c in cfgs], np.int64),
        cfg=np.array([r["cfg"] for r in rows]), t=np.array([r["t"] for r in rows]),
        nblk=np.array([len(r["s_q"]) for r in rows]),
        s_q=np.array([np.pad(r["s_q"], (0, L - len(r["s_q"]))) for r in rows]),
        s_e=np.array([np.pad(r["s_e"], (0, L - len(r["s_e"]))) for r in rows]),
        nosa_q=pad("nosa_q", 64), nosa_e=pad("nosa_e", 64), inf_q=pad("inf_q", 64), fixed=pad("fixed", 64))
    print("selection_kats:", n, "cases")


def manager_trace():
    """Random required sets over 2 heads, capacity 6 per head, 24 blocks, 300 calls per head."""
    rng = np.random.default_rng(77)
    H, C, NBLK, STEPS = 2, 6, 24, 300
    fast = PhysicalLayout(FAST, C, H, 4, 8)
    slow = PhysicalLayout(SLOW, NBLK, H, 4, 8)
    mgr = TieredBlockManager(fast, slow)
    for h in range(H):
        for i in range(NBLK):
            mgr.allocate(SLOW, 0, h, i)
    req = np.full((STEPS, H, C), -1, np.int64)
    fetch = np.full((STEPS, H, C), -1, np.int64)
    evict = np.full((STEPS, H, C), -1, np.int64)
    hits = np.zeros((STEPS, H), np.int64)
    slots = np.full((STEPS, H, C), -1, np.int64)  # fast slot of each required block after apply
    for s in range(STEPS):
        for h in range(H):
            k = int(rng.integers(1, C + 1))
            # locality: half of the set from a slowly moving window
            base = (s // 10) % (NBLK - C)
            cand = list(range(base, base + C)) if rng.random() < 0.6 else list(range(NBLK))
            r = sorted(set(int(x) for x in rng.choice(cand, size=k, replace=False)))
            plan = mgr.plan_transfers(set(r), 0, h)
            mgr.apply_transfers(plan)
            req[s, h, :len(r)] = r
            fetch[s, h, :len(plan.fetch)] = [key[2] for key in plan.fetch]
            evict[s, h, :len(plan.evict)] = [key[2] for key in plan.evict]
            hits[s, h] = plan.hits
            slots[s, h, :len(r)] = [mgr.lookup(0, h, b)[2] for b in r]
    st = mgr.residency_stats()
    np.savez_compressed(OUT / "manager_trace.npz", req=req, fetch=fetch, evict=evict, hits=hits, slots=slots,
                        capacity=C, nblk=NBLK, stats=np.array([st.hits, st.misses, st.bytes_up, st.steps]))
    print("manager_trace: hit rate", st.hit_rate)


def engine_run(name, cfg_kw, batch, t0, steps, fast_slots, seed, rho, selector="nosa", out_dtype=np.float64,
               synth=False):
    """synth=True: the counter-based inputs (workload.synth_prefix_kv / SynthQueryStream) that the
    GPU bench and the headline-config parity tests draw, for sequences 0..batch-1 of layer 0."""
    cfg = AttentionConfig(**cfg_kw)
    Hq, Hk, D = cfg.n_head, cfg.n_kv_head, cfg.d_head
    d = (Hq + 2 * Hk) * D
    eye = np.eye(d)
    w1, w2 = workload.eviction_head(Hq, D, seed)
    weights = ModelWeights(w_q=eye[:, :Hq * D], w_k=eye[:, Hq * D:(Hq + Hk) * D], w_v=eye[:, (Hq + Hk) * D:],
                           eviction=EvictionHead("ed-dma", w1, w2), seed=0)
    if synth:
        K, V = workload.synth_prefix_kv(seed, 0, range(batch), Hk, t0, D)
        stream = workload.SynthQueryStream(seed, [0], range(batch), Hq, Hk, D, rho)
    else:
        K, V = workload.prefix_kv(seed, batch, Hk, t0, D)
        stream = workload.QueryStream(seed, 1, batch, Hq, Hk, D, rho)
    inputs = [stream.next() for _ in range(steps)]
    engines = []
    for b in range(batch):
        eng = DecodeEngine(cfg, weights, capacity=t0 + steps + 1)
        h = np.concatenate([np.zeros((t0, Hq * D)), K[b].transpose(1, 0, 2).reshape(t0, Hk * D),
                            V[b].transpose(1, 0, 2).reshape(t0, Hk * D)], axis=1)
        eng.prefill(h)
        eng.start_run()
        engines.append(eng)
    nblk_max = -(-(t0 + steps) // cfg.n_b)
    geom = BlockGeometry.for_run(cfg, t0)
    lo, hi = geom.pool_blocks.start, geom.pool_blocks.stop
    sel_q = np.full((steps, batch, Hk, 64), -1, np.int64)
    sel_e = np.full((steps, batch, Hk, 64), -1, np.int64)
    outs = np.zeros((steps, batch, Hq, D), out_dtype)
    s_q_all = np.zeros((steps, batch, Hk, hi - lo))
    s_e_pool = np.zeros((batch, Hk, hi - lo))
    fetch = np.full((steps, batch, Hk, fast_slots), -1, np.int64)
    evict = np.full((steps, batch, Hk, fast_slots), -1, np.int64)
    hits = np.zeros((steps, batch, Hk), np.int64)
    # one reference TieredBlockManager per sequence (SURVEY.md §8a recommendation)
    mgrs = []
    for b in range(batch):
        m = TieredBlockManager(PhysicalLayout(FAST, fast_slots, Hk, cfg.n_b, D),
                               PhysicalLayout(SLOW, nblk_max + 1, Hk, cfg.n_b, D))
        for h in range(Hk):
            for i in range(geom.n_blocks(t0)):
                m.allocate(SLOW, 0, h, i)
        mgrs.append(m)
    for s in range(steps):
        q, kn, vn = inputs[s]
        for b in range(batch):
            eng = engines[b]
            t = eng.t
            # pool scores as the engine computes them (decode.py:170-172), before the step
            for h in range(Hk):
                k_c, s_e_c = eng.heads[h].compressed(cfg.n_b)
                qs = q[0, b, h * cfg.group_size:(h + 1) * cfg.group_size].astype(np.float64).sum(axis=0)
                s_q_all[s, b, h] = (k_c @ qs)[lo:hi]
                if s == 0:
                    s_e_pool[b, h] = s_e_c[lo:hi]
            h_t = np.concatenate([q[0, b].reshape(-1), kn[0, b].reshape(-1), vn[0, b].reshape(-1)])
            out = eng.step(h_t, selector=selector)
            outs[s, b] = out.outputs
            for h, sel in enumerate(out.selections):
                sel_q[s, b, h, :len(sel.blocks_q)] = sel.blocks_q
                sel_e[s, b, h, :len(sel.blocks_e)] = sel.blocks_e
                required = set(sel.blocks_fixed) | sel.topk_blocks
                for blk in required:
                    if mgrs[b].lookup(0, h, blk) is None:  # born during the run (offload_sim.py:286-289)
                        mgrs[b].allocate(SLOW, 0, h, blk)
                plan = mgrs[b].plan_transfers(required, 0, h)
                mgrs[b].apply_transfers(plan)
                fetch[s, b, h, :len(plan.fetch)] = [key[2] for key in plan.fetch]
                evict[s, b, h, :len(plan.evict)] = [key[2] for key in plan.evict]
                hits[s, b, h] = plan.hits
            assert eng.t == t + 1
    np.savez_compressed(OUT / f"{name}.npz", cfg=np.array([cfg_kw[k] for k in ("n", "d", "n_head", "n_kv_head",
                        "d_head", "n_b", "n_s", "n_w", "k", "k_q", "k_e")] + [1 if cfg.accounting == "exclusive" else 0]),
                        batch=batch, t0=t0, steps=steps, fast_slots=fast_slots, seed=seed, rho=rho,
                        selector=selector, synth=int(synth), sel_q=sel_q, sel_e=sel_e, outputs=outs, s_q=s_q_all, s_e_pool=s_e_pool,
                        fetch=fetch, evict=evict, hits=hits, pool=np.array([lo, hi]))
    print(name, "done")


def shared_pool_simulation():
    """The reference simulator itself (offload_sim.simulate_decode, shared per-head pool across
    the batch, scripted AR(1) selections): its SimReport plus every per-(step, b, h) required set
    and the fetch/evict lists of a replay through one shared TieredBlockManager, b-major order."""
    from nosa_sim.decode import scripted_selection_trace
    from nosa_sim.offload_sim import DEFAULT_PARAMS, fast_slots_per_seq, simulate_decode
    cfg = AttentionConfig(n=4096, d=8, n_head=2, n_kv_head=2, d_head=8, n_b=16, n_s=32, n_w=64, k=288,
                          k_q=64, k_e=224)
    out = {}
    for policy, rho in (("nosa", 0.5), ("infllmv2-offload", 0.0)):
        B, t0, steps, seed = 4, 1000, 8, 3
        rep = simulate_decode(cfg, DEFAULT_PARAMS, policy, batch=B, t0=t0, steps=steps, seed=seed,
                              query_smoothness=rho)
        # replay the same loop to record the required sets and plans (offload_sim.py:224-299)
        selector = "nosa" if policy == "nosa" else "infllmv2"
        geom = BlockGeometry.for_run(cfg, t0)
        seeds = np.random.SeedSequence(seed).generate_state(B)
        traces = [scripted_selection_trace(cfg, int(s), t0, steps + 1, selector=selector, query_smoothness=rho,
                                           n_heads=cfg.n_kv_head) for s in seeds]
        slots = fast_slots_per_seq(cfg, t0, steps + 1)
        H, total = cfg.n_kv_head, geom.n_blocks(t0 + steps + 1)
        mgr = TieredBlockManager(PhysicalLayout(FAST, B * slots, H, cfg.n_b, cfg.d_head),
                                 PhysicalLayout(SLOW, B * total, H, cfg.n_b, cfg.d_head))
        for b in range(B):
            for h in range(H):
                for i in range(geom.n_blocks(t0)):
                    mgr.allocate(SLOW, b, h, i)
        R = 64
        req = np.full((steps + 1, B, H, R), -1, np.int64)
        fetch = np.full((steps + 1, B, H, R), -1, np.int64)
        evict = np.full((steps + 1, B, H, R, 2), -1, np.int64)  # (batch, block) of each victim
        topk = np.full((steps + 1, B, H, R), -1, np.int64)
        for i in range(steps + 1):
            for b in range(B):
                for h in range(H):
                    sel = traces[b].steps[i][h]
                    r = sorted(set(sel.blocks_fixed) | sel.topk_blocks)
                    for blk in r:
                        if mgr.lookup(b, h, blk) is None:
                            mgr.allocate(SLOW, b, h, blk)
                    plan = mgr.plan_transfers(set(r), b, h)
                    mgr.apply_transfers(plan)
                    req[i, b, h, :len(r)] = r
                    tk = sorted(sel.topk_blocks)
                    topk[i, b, h, :len(tk)] = tk
                    fetch[i, b, h, :len(plan.fetch)] = [k[2] for k in plan.fetch]
                    for j, key in enumerate(plan.evict):
                        evict[i, b, h, j] = (key[0], key[2])
            if i == 0:
                mgr.reset_stats()
        st = mgr.residency_stats()
        assert st.hit_rate == rep.hit_rate and st.bytes_up == rep.bytes_up
        tag = "nosa" if policy == "nosa" else "infllmv2"
        out.update({f"{tag}_req": req, f"{tag}_fetch": fetch, f"{tag}_evict": evict, f"{tag}_topk": topk,
                    f"{tag}_report": np.array([rep.hit_rate, rep.hit_rate_topk, rep.bytes_up, rep.bytes_down]),
                    f"{tag}_shape": np.array([B, H, slots, total, t0, steps])})
    np.savez_compressed(OUT / "shared_pool_sim.npz", **out)
    print("shared_pool_sim: nosa hit", out["nosa_report"][0], "infllmv2 hit", out["infllmv2_report"][0])


def headline():
    """The 1B attention shape at 32K context with 25% of the blocks in the fast tier (BASELINE config
    3 / 4 per sequence), on the counter-based inputs: long enough for the cache to fill and evict."""
    one_b = dict(n=65536, d=2560, n_head=16, n_kv_head=2, d_head=128, n_b=64, n_s=64, n_w=1024, k=4096, k_q=1024,
                 k_e=3072)
    engine_run("engine_1b_32k", one_b, batch=1, t0=32768, steps=40, fast_slots=128, seed=21, rho=0.95,
               out_dtype=np.float32, synth=True)
    engine_run("engine_1b_32k_infllmv2_rho0", one_b, batch=1, t0=32768, steps=12, fast_slots=128, seed=22, rho=0.0,
               selector="infllmv2", out_dtype=np.float32, synth=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "headline":
        headline()
        return
    selection_kats()
    manager_trace()
    shared_pool_simulation()
    small = dict(n=4096, d=512, n_head=4, n_kv_head=2, d_head=64, n_b=16, n_s=32, n_w=128, k=512, k_q=128, k_e=384)
    engine_run("engine_small", small, batch=2, t0=1000, steps=24, fast_slots=40, seed=5, rho=0.5)
    engine_run("engine_small_infllmv2", small, batch=2, t0=1000, steps=8, fast_slots=40, seed=6, rho=0.0,
               selector="infllmv2")
    cfg1 = dict(n=16384, d=1536, n_head=8, n_kv_head=2, d_head=128, n_b=64, n_s=64, n_w=512, k=1024, k_q=256,
                k_e=768, accounting="exclusive")
    engine_run("engine_cfg1", cfg1, batch=4, t0=8192, steps=16, fast_slots=32, seed=11, rho=0.95,
               out_dtype=np.float32)


if __name__ == "__main__":
    main()
