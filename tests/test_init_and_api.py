"""Host-side contract tests (no GPU): pinned init == oracle init bit-for-bit, device layout helpers,
scoring API, config invariants, and the C-ABI library's exported symbols."""

import ctypes
import re
import os

import numpy as np
import pytest

import oracle.model as OM
from paper_2510_22101_b200 import (CONFIGS, ModelConfig, init_weights, rank_items, relevance_score,
                                   top_k)
from paper_2510_22101_b200 import _lib
from paper_2510_22101_b200.weights import bf16_round, interleave_gate_up, rope_tables

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", ["C1", "TINY", "TINY_GQA"])
def test_init_matches_oracle_bitwise(name):
    cfg = CONFIGS[name]
    pw, ow = init_weights(cfg, 0), OM.init_weights(cfg, 0)
    assert np.array_equal(pw.token_embedding, ow.token_embedding)
    assert np.array_equal(pw.head, ow.head)
    for l in range(cfg.n_layers):
        for f in OM.LAYER_FIELDS:
            assert np.array_equal(getattr(pw.layers[l], f), ow.layers[l][f]), (l, f)
    assert pw.param_count() == cfg.param_count() == OM.param_count(cfg)


def test_bf16_round_rne():
    x = np.array([1.0, 1.00390625, 1.01171875, -2.5, 3.0e38, 1e-40, 0.0, -0.0], dtype=np.float32)
    # 1 + 2^-8 is a tie -> even (1.0); 1 + 3*2^-8 tie -> 1 + 2^-6 (even mantissa)
    y = bf16_round(x)
    assert y[0] == 1.0 and y[1] == 1.0 and y[2] == np.float32(1.015625)
    assert np.array_equal(y, OM.bf16_round(x))
    r = np.random.default_rng(0).standard_normal(100000).astype(np.float32) * 7
    assert np.array_equal(bf16_round(r), OM.bf16_round(r))
    assert np.all((bf16_round(r).view(np.uint32) & 0xFFFF) == 0)


def test_rope_tables_match_oracle():
    cfg = CONFIGS["TINY"]
    c, s = rope_tables(cfg)
    oc, os_ = OM.rope_tables(cfg, np.float32)
    assert np.array_equal(c, oc) and np.array_equal(s, os_)


def test_interleave_gate_up_layout():
    F, d = 300, 8
    g = np.arange(F * d, dtype=np.float32).reshape(F, d)
    u = -g - 1
    Fp = 384
    out = interleave_gate_up(g, u, Fp)
    assert out.shape == (2 * Fp, d)
    for j in range(Fp // 128):
        blk = out[256 * j: 256 * (j + 1)]
        n0, n1 = 128 * j, min(128 * (j + 1), F)
        np.testing.assert_array_equal(blk[: n1 - n0], g[n0:n1])
        np.testing.assert_array_equal(blk[128: 128 + n1 - n0], u[n0:n1])
        assert not blk[n1 - n0:128].any() and not blk[128 + n1 - n0:].any()


def test_config_invariants_and_flops():
    with pytest.raises(ValueError):
        ModelConfig(d_model=66, n_heads=4)
    with pytest.raises(ValueError):
        ModelConfig(n_heads=4, n_kv_heads=3)
    c4 = CONFIGS["C4"]
    assert c4.d_ff_pad == 3712 and c4.q_width == 1280
    # SURVEY.md §8d per-item figure for C4 (~172.5 GF/item at P=64, S=100, 256 items)
    import bench
    f = bench.algorithmic_flops(c4, 64, [100] * 256) / 256
    assert abs(f / 1e9 - 172.5) < 1.0


def test_scoring_api():
    r = relevance_score([2.0, 0.0])
    assert abs(r.p_yes - 0.880797) < 1e-6 and abs(r.p_yes + r.p_no - 1) < 1e-12
    full = np.zeros(32)
    full[1] = 2.0
    assert abs(relevance_score(full, CONFIGS["TINY"]).p_yes - 0.880797) < 1e-6
    with pytest.raises(ValueError):
        relevance_score([np.inf, 0.0])
    assert rank_items([0.2, 0.9, 0.9], ["c", "b", "a"]).item_ids == ["a", "b", "c"]
    assert top_k([0.1, 0.5, 0.3], 2) == [1, 2]


def header_symbols():
    src = open(os.path.join(ROOT, "include", "prefill_sm100.h")).read()
    return set(re.findall(r"PF_API\s+[\w\s\*]*?\b(pf_\w+)\s*\(", src))


def test_capi_exports_every_declared_symbol():
    syms = header_symbols()
    assert syms == set(_lib.EXPORTED_SYMBOLS)
    lib = _lib.load()   # dlopen works without a GPU
    for s in syms:
        assert hasattr(lib, s), s
    assert "sm_100a" in _lib.version()


def test_capi_argument_errors_without_gpu():
    lib = _lib.load()
    assert lib.pf_model_create(None, None) == _lib.PF_EARG
    assert "null" in lib.pf_last_error().decode()
    assert lib.pf_workspace_bytes(None, 10, 1) == 0
    rc = lib.pf_score(None, None, None, None, 1, None, 1, None, 1, 1, None, 0, None, None, None, None)
    assert rc == _lib.PF_EARG
    with pytest.raises(_lib.PfError):
        _lib.check(rc)
