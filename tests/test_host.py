"""CPU-only checks: the C ABI loads and exports what include/nosa_b200.h declares, the host-side
mirror of the reference API (config validation, geometry), the synthetic workload and the
oracle's own known-answer tests (restated from the reference test-suite)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import nosa_oracle as O
from paper_2510_13602_b200 import AttentionConfig, BlockGeometry, _lib, workload
from paper_2510_13602_b200.selection import build_token_mask, make_result

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "nosa_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|void|int64_t|const char\*)\s+\**(nosa_\w+)\(", header, re.M))
    assert len(declared) >= 25
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)


def _header_struct_fields(header: str, name: str) -> list[str]:
    body = re.search(r"typedef struct " + name + r" \{(.*?)\} " + name + ";", header, re.S).group(1)
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        fields += [re.search(r"(\w+)\s*$", part).group(1) for part in decl.split(",")]
    return fields


@pytest.mark.parametrize("name", ["NosaConfig", "NosaStats", "NosaStepIO", "NosaHostStepIO"])
def test_ctypes_structs_match_header(name):
    """The ctypes mirrors (and INTEGRATION.md's stub) lay the structs out as the header does."""
    header = (ROOT / "include" / "nosa_b200.h").read_text()
    want = _header_struct_fields(header, name)
    got = [f for f, _ in getattr(_lib, name)._fields_]
    assert got == want


def test_integration_stub_config_fields_match_header():
    header = (ROOT / "include" / "nosa_b200.h").read_text()
    doc = (ROOT / "INTEGRATION.md").read_text()
    stub = re.search(r"class NosaConfig\(ctypes.Structure\):.*?_fields_ = \[.*?for f in \((.*?)\)\]", doc, re.S)
    names = re.findall(r'"(\w+)"', stub.group(1))
    assert names == _header_struct_fields(header, "NosaConfig")


def _c_config(**over):
    c = _lib.NosaConfig()
    base = dict(n=16384, d=1024, n_head=8, n_kv_head=2, d_head=128, n_b=64, n_s=64, n_w=512, k=1024, k_q=256,
                k_e=768, accounting=1, batch=4, layers=1, max_tokens=9000, fast_slots=32, dtype=0, variant=0)
    base.update(over)
    for k, v in base.items():
        setattr(c, k, v)
    return c


@pytest.mark.parametrize("over,msg", [
    (dict(k=1000), "k must equal k_q + k_e"),
    (dict(n_s=10), "n_s=10 must be divisible by n_b=64"),
    (dict(n=512), "need n_s + n_w <= k <= n"),
    (dict(n_head=7), "n_head=7 must be a positive multiple of n_kv_head=2"),
    (dict(accounting=0, k_q=512, k_e=512), "inclusive accounting needs k_q <= k - n_s - n_w"),
    (dict(d_head=96), "unsupported"),
    (dict(batch=0), "batch and layers must be positive"),
    (dict(attend_chunk=9), "attend_chunk must be in 0..8"),
    (dict(attend_layers=-1), "attend_layers must be >= 0"),
    (dict(exact_scan=2), "exact_scan must be 0 or 1"),
    (dict(slow_tier_device=-2), "slow_tier_device must be -1"),
])
def test_c_config_validation_messages(over, msg):
    buf = ctypes.create_string_buffer(512)
    assert _lib.lib.nosa_config_validate(ctypes.byref(_c_config(**over)), buf, 512) == _lib.NOSA_ERR_VALUE
    assert msg in buf.value.decode()


def test_c_budgets_match_python_config():
    for acc in (0, 1):
        c = _c_config(accounting=acc, k=2048, k_q=512, k_e=1536)
        q, e, t = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        assert _lib.lib.nosa_config_validate(ctypes.byref(c), None, 0) == 0
        _lib.lib.nosa_config_budgets(ctypes.byref(c), ctypes.byref(q), ctypes.byref(e), ctypes.byref(t))
        py = AttentionConfig(n=16384, d=1024, n_head=8, n_kv_head=2, d_head=128, n_b=64, n_s=64, n_w=512, k=2048,
                             k_q=512, k_e=1536, accounting="inclusive" if acc == 0 else "exclusive")
        assert (q.value, e.value, t.value) == (py.blocks_q, py.blocks_e, py.blocks_topk)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    h = ctypes.c_void_p()
    rc = _lib.lib.nosa_ctx_create(ctypes.byref(_c_config()), 0, ctypes.byref(h))
    assert rc == _lib.NOSA_ERR_CUDA and b"no CPU fallback" in _lib.lib.nosa_last_error(None)


def test_attention_config_validation_mirrors_reference():
    with pytest.raises(ValueError, match="k must equal"):
        AttentionConfig(n=1024, d=8, n_head=1, n_kv_head=1, d_head=8, n_b=16, n_s=32, n_w=64, k=256, k_q=64, k_e=100)
    with pytest.raises(ValueError, match="divisible"):
        AttentionConfig(n=1024, d=8, n_head=1, n_kv_head=1, d_head=8, n_b=16, n_s=30, n_w=64, k=256, k_q=64, k_e=192)
    c = AttentionConfig(n=65536, d=2048, n_head=16, n_kv_head=2, d_head=128, n_b=64, n_s=64, n_w=1024, k=4096,
                        k_q=1024, k_e=3072)
    assert (c.blocks_q, c.blocks_e, c.group_size) == (16, 31, 8)
    assert abs(c.locality_bound - 1984 / 3008) < 1e-15


def test_geometry_kats():
    # test_selection.py:28-38
    cfg = AttentionConfig(n=1024, d=8, n_head=1, n_kv_head=1, d_head=8, n_b=16, n_s=32, n_w=64, k=256, k_q=64,
                          k_e=192)
    g = BlockGeometry.for_run(cfg, 512)
    assert g.recent_start == 449 and g.pool_blocks == range(2, 28)
    assert set(g.fixed_blocks(512)) == {0, 1} | set(range(28, 32))
    og = O.Geometry.for_run(16, 32, 64, 512)
    assert og.pool == (2, 28) and og.fixed(512) == list(g.fixed_blocks(512))
    # every cached block is fixed or pool (test_selection.py:50-57)
    for t0 in (47, 64, 200, 511):
        g = BlockGeometry.for_run(cfg, t0)
        for t in (t0, t0 + 5, t0 + 40):
            assert set(g.fixed_blocks(t)) | set(g.pool_blocks) == set(range(g.n_blocks(t)))
    g = BlockGeometry.for_run(cfg, 80)
    assert len(g.pool_blocks) == 0


def test_token_mask():
    sel = make_result(40, 16, (), (), (0, 1, 2))
    assert np.array_equal(build_token_mask(sel, 40), np.zeros(40))
    with pytest.raises(ValueError, match="step"):
        build_token_mask(sel, 41)


def test_oracle_argtopk_tie_rule():
    assert set(O.argtopk(np.array([1.0, 1.0, 1.0]), 2)) == {0, 1}
    assert O.argtopk(np.array([0.0, -0.0, 1.0]), 2).tolist() == [0, 2]
    rng = np.random.default_rng(3)
    for _ in range(100):
        s = np.round(rng.standard_normal(40), 1)
        k = int(rng.integers(0, 41))
        want = sorted(sorted(range(40), key=lambda i: (-s[i], i))[:k])
        assert O.argtopk(s, k).tolist() == want


def test_oracle_manager_kats():
    m = O.SequenceManager(1, 4)
    for req in [{0, 1}, {0, 1}, {1, 2, 3}, {3, 4}, {0, 4}, {0, 4}, {5, 6, 7}, {7}]:
        m.plan_apply(req, 0)
    assert (m.hits, m.misses, m.steps) == (8, 9, 8)
    m = O.SequenceManager(1, 3)
    m.plan_apply({0, 1, 2}, 0)
    m.plan_apply({1, 2}, 0)
    assert m.plan_apply({1, 2, 5}, 0)[1] == [0]
    with pytest.raises(O.CapacityExceededOracle):
        O.SequenceManager(1, 2).plan_apply({1, 2, 3}, 0)


def test_bf16_round_matches_torch():
    x = np.random.default_rng(0).standard_normal(10000).astype(np.float32) * 10
    want = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(workload.bf16_round(x), want)


def test_query_stream_locality():
    a = workload.QueryStream(1, 1, 2, 4, 2, 64, 0.95)
    b = workload.QueryStream(1, 1, 2, 4, 2, 64, 0.0)
    qa = [a.next()[0] for _ in range(6)]
    qb = [b.next()[0] for _ in range(6)]
    corr = lambda qs: np.mean([np.corrcoef(qs[i].ravel(), qs[i + 1].ravel())[0, 1] for i in range(5)])
    assert corr(qa) > 0.8 and abs(corr(qb)) < 0.2


def test_projection_rejects_untileable_shapes_without_a_gpu():
    """nosa_project_qkv validates shapes before touching the device (ValueError-class status)."""
    lib = _lib.lib
    p = ctypes.c_void_p(16)  # never dereferenced: the shape checks fail first
    assert lib.nosa_project_qkv(p, 4, 2048, p, 2500, 2048, 256, p, p, p, 4, None) == _lib.NOSA_ERR_VALUE
    assert b"N % 128" in lib.nosa_last_error(None)
    assert lib.nosa_project_qkv(p, 4, 2048, p, 2560, 2048, 256, p, p, p, 9, None) == _lib.NOSA_ERR_VALUE
    assert lib.nosa_project_qkv(None, 4, 2048, p, 2560, 2048, 256, p, p, p, 4, None) == _lib.NOSA_ERR_VALUE


def test_tiered_block_manager_constructor_contract():
    """The drop-in TieredBlockManager validates like the reference before touching the device
    (kv_manager.py:59-81, 138-146): layout checks and tier order; the default policy."""
    from paper_2510_13602_b200 import FAST, SLOW, LayoutMismatch, PhysicalLayout, TieredBlockManager
    from paper_2510_13602_b200.kv_manager import least_recently_required
    with pytest.raises(ValueError):
        PhysicalLayout("warm", 4, 1, 4, 8)
    with pytest.raises(ValueError):
        PhysicalLayout(FAST, 4, 1, 4, 8, element_width=3)
    assert PhysicalLayout(FAST, 4, 2, 4, 8).bytes_per_block == 2 * 4 * 8 * 2
    fast, slow = PhysicalLayout(FAST, 4, 2, 4, 8), PhysicalLayout(SLOW, 8, 2, 4, 8)
    with pytest.raises(LayoutMismatch):
        TieredBlockManager(slow, fast)
    with pytest.raises(LayoutMismatch, match="disagree"):
        TieredBlockManager(fast, PhysicalLayout(SLOW, 8, 3, 4, 8))
    keys = [(1, 0, 5), (0, 0, 9), (0, 0, 2)]
    assert least_recently_required(keys, {(0, 0, 9): 3}) == [(0, 0, 2), (1, 0, 5), (0, 0, 9)]
