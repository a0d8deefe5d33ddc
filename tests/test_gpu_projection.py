"""The tcgen05 QKV projection (csrc/nosa_project.cu) against a plain PyTorch fp32 GEMM of the
same bf16 operands."""

import numpy as np
import pytest
import torch

from paper_2510_13602_b200.projection import QKVProjection, _splits

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,d,hq,hkv,dh", [(1, 512, 4, 2, 64), (200, 512, 4, 2, 64), (128, 2048, 16, 2, 128),
                                           (300, 1024, 8, 2, 128)])
def test_projection_matches_fp32_reference(m, d, hq, hkv, dh):
    rng = np.random.default_rng(m + d)
    w_q, w_k, w_v = (rng.standard_normal((d, h * dh)) / np.sqrt(d) for h in (hq, hkv, hkv))
    proj = QKVProjection(w_q, w_k, w_v)
    h = torch.randn(m, d, device="cuda").to(torch.bfloat16)
    q, k, v = proj(h)
    w = torch.cat([proj.w_t.float()], 0)  # [n][d], the bf16 weights as used
    ref = h.float() @ w.T                 # fp32 reference of the same bf16 operands
    got = torch.cat([q, k, v], 1).float()
    assert got.shape == ref.shape
    # fp32 accumulation in a different order, then one bf16 rounding
    err = (got - ref).abs().max().item() / ref.abs().max().item()
    assert err < 8e-3, err
    # deterministic: the same call twice is bitwise equal; every split count agrees in tolerance
    q2, k2, v2 = proj(h)
    assert torch.equal(q, q2) and torch.equal(k, k2) and torch.equal(v, v2)
    for sp in (1, 2, 8):
        if (d // 64) % sp == 0:
            alt = torch.cat(proj(h, sp), 1).float()
            assert (alt - ref).abs().max().item() / ref.abs().max().item() < 8e-3


def test_split_choice_and_exact_identity():
    assert _splits(128, 2560, 2048) == 4 and _splits(3584, 2560, 2048) == 1
    assert (2048 // 64) % _splits(128, 2560, 2048) == 0
    # 0/1 weights and bf16 inputs: every output is one input element, exactly
    d, n = 512, 512
    eye = np.eye(d)
    proj = QKVProjection(eye[:, :256], eye[:, 256:384], eye[:, 384:])
    h = torch.randn(77, d, device="cuda").to(torch.bfloat16)
    q, k, v = proj(h)
    assert torch.equal(torch.cat([q, k, v], 1), h)


@pytest.mark.parametrize("schedule,graph,host", [("pipelined", False, False), ("serial", False, False),
                                                 ("pipelined", True, False), ("pipelined", False, True),
                                                 ("serial", False, True)])
def test_hidden_state_step_matches_projected_step(schedule, graph, host):
    """nosa_decode_step_hidden (projection of every layer inside the step, on the selection
    stream) gives bitwise the outputs, selections and residency of nosa_decode_step fed with the
    same tcgen05 projections computed outside."""
    from paper_2510_13602_b200 import AttentionConfig, NosaEngine, workload
    cfg = AttentionConfig(n=8192, d=1024, n_head=16, n_kv_head=2, d_head=128, n_b=64, n_s=64, n_w=1024, k=4096,
                          k_q=1024, k_e=3072)
    L, B, T, steps = 3, 4, 3000, 6
    rng = np.random.default_rng(7)
    ws = [[rng.standard_normal((cfg.d, h * cfg.d_head)) / np.sqrt(cfg.d) for h in (16, 2, 2)] for _ in range(L)]
    w1, w2 = workload.eviction_head(cfg.n_head, cfg.d_head, 7)
    K, V = workload.prefix_kv(7, L * B, cfg.n_kv_head, T, cfg.d_head)
    K, V = K.reshape(L, B, cfg.n_kv_head, T, cfg.d_head), V.reshape(L, B, cfg.n_kv_head, T, cfg.d_head)
    hs = [torch.randn(L, B, cfg.d, device="cuda").to(torch.bfloat16) for _ in range(steps)]
    runs = []
    for hidden in (False, True):
        eng = NosaEngine(cfg, batch=B, layers=L, max_tokens=T + steps + 1, fast_slots=70, w1=w1, w2=w2)
        eng.prefill(torch.from_numpy(K), torch.from_numpy(V))
        eng.start_run()
        projs = [QKVProjection(*w) for w in ws]
        for l in range(L):
            eng.set_projection(l, *ws[l])
        outs = []
        if hidden and graph:
            hb = torch.empty_like(hs[0])
            ob = torch.empty((L, B, cfg.n_head, cfg.d_head), dtype=torch.float32, device="cuda")
            eng.capture_hidden(hb, ob)
        for s in range(steps):
            if hidden and graph:
                hb.copy_(hs[s])
                eng.replay()
                out = ob
            elif hidden and host:  # host buffers in and out (nosa_decode_step_hidden_host): pinned
                # (SM staging) in the pipelined case, pageable (cudaMemcpyAsync) in the serial one
                h_host = hs[s].cpu()
                out = eng.step_hidden_host(h_host.pin_memory() if schedule == "pipelined" else h_host,
                                           schedule=schedule)
            elif hidden:
                out = eng.step_hidden(hs[s], schedule=schedule)
            else:
                qkv = [p(hs[s][l], 1) for l, p in enumerate(projs)]  # the step's split count
                q = torch.stack([x[0] for x in qkv]).reshape(L, B, cfg.n_head, cfg.d_head)
                k = torch.stack([x[1] for x in qkv]).reshape(L, B, cfg.n_kv_head, cfg.d_head)
                v = torch.stack([x[2] for x in qkv]).reshape(L, B, cfg.n_kv_head, cfg.d_head)
                out = eng.step(q, k, v, schedule=schedule)
            outs.append(out.cpu().numpy().copy())
        st = eng.residency_stats()
        runs.append((np.stack(outs), (st.hits, st.misses, st.evictions), [eng.raw_selection(l)[:4] for l in range(L)]))
        eng.close()
    np.testing.assert_array_equal(runs[0][0], runs[1][0])
    assert runs[0][1] == runs[1][1]
    for a, b in zip(runs[0][2], runs[1][2]):
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("m,k,n", [(1, 512, 512), (1, 2048, 2560), (37, 300, 130), (513, 1024, 384)])
def test_fp32_projection_matches_fp64_reference(m, k, n):
    """nosa_project_f32 (the fp32-cache projection of compat.DecodeEngine) against an fp64 GEMM of
    the same fp32 operands: fp32 FMA chains in k order, relative error ~ k * 2^-24."""
    from paper_2510_13602_b200 import _lib
    g = torch.Generator(device="cpu").manual_seed(m * 7 + n)
    h = torch.randn(m, k, generator=g).cuda()
    w = (torch.randn(k, n, generator=g) / k ** 0.5).cuda()
    out = torch.empty(m, n, device="cuda")
    _lib.check(_lib.lib.nosa_project_f32(h.data_ptr(), m, k, w.data_ptr(), n, out.data_ptr(), _lib.stream_ptr()))
    ref = (h.double() @ w.double())
    err = ((out.double() - ref).abs().max() / ref.abs().max()).item()
    assert err < 1e-5, err
    out2 = torch.empty_like(out)
    _lib.check(_lib.lib.nosa_project_f32(h.data_ptr(), m, k, w.data_ptr(), n, out2.data_ptr(), _lib.stream_ptr()))
    assert torch.equal(out, out2)
