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
