"""Pin the CPU oracle against the reference spec's known answers and invariants
(ACCEPTANCE CRITERIA 1-2).  No reference-executed model outputs exist (the
reference ships no model code), so these KATs are the oracle's pin for the model path."""

import math

import numpy as np
import pytest

import oracle.model as OM
import oracle.prefixcache as OP
import oracle.scoring as OS
from paper_2510_22101_b200.config import ModelConfig

SPEC_DEFAULT = ModelConfig(precision="f32")   # SPEC.md:178 defaults: L8 d64 H4 Hkv2 d_ff256
SMALL = ModelConfig(n_layers=2, d_model=64, n_heads=4, n_kv_heads=2, d_ff=128, vocab_size=512,
                    max_seq=256, precision="f32")


@pytest.fixture(scope="module")
def w32():
    return OM.init_weights(SPEC_DEFAULT, 0)


@pytest.fixture(scope="module")
def w64(w32):
    return w32.astype(np.float64)


# ----------------------------------------------------------------------------- scoring
def test_relevance_score_kats():
    logits = np.zeros(16)
    logits[1], logits[2] = 2.0, 0.0
    p, q = OS.relevance_score(logits)
    assert abs(p - 0.880797) < 1e-6 and abs(p + q - 1) < 1e-12
    logits[1] = logits[2] = 0.3
    assert OS.relevance_score(logits) == (0.5, 0.5)
    logits[1], logits[2] = 1.5, -0.7
    a = OS.relevance_score(logits)
    logits[1], logits[2] = -0.7, 1.5
    b = OS.relevance_score(logits)
    assert abs(a[0] - b[1]) < 1e-15 and abs(a[1] - b[0]) < 1e-15
    with pytest.raises(ValueError):
        OS.relevance_score(np.array([0, np.nan, 0.0]))


def test_softmax2_equals_sigmoid():
    rng = np.random.default_rng(0)
    for a, b in rng.normal(0, 5, size=(2000, 2)):
        p = OS.relevance_score(np.array([0.0, a, b]))[0]
        assert abs(p - 1 / (1 + math.exp(-(a - b)))) < 1e-12


def test_rank_items_rules():
    assert OS.rank_items([0.5, 0.5, 0.5]) == [0, 1, 2]
    assert OS.rank_items([0.9, 0.5, 0.1]) == [0, 1, 2]
    rng = np.random.default_rng(1)
    s = rng.random(50)
    assert OS.rank_items(s) == sorted(range(50), key=lambda i: (-s[i], i))
    # monotone-transform invariance
    assert OS.rank_items(np.tanh(3 * s)) == OS.rank_items(s)


# ----------------------------------------------------------------------------- prefixcache
def test_throughput_gain_kats():
    assert abs(OP.throughput_gain(50, 150) - 1.3333333333) < 1e-9
    assert OP.throughput_gain(0, 100) == 1.0 and OP.throughput_gain(100, 100) == 2.0
    with pytest.raises(ValueError):
        OP.throughput_gain(10, 0)


def test_split_shared_prefix_rules():
    sb = OP.split_shared_prefix([[1, 2, 3], [1, 2, 3]])
    assert sb.prefix_tokens == [1, 2] and sb.suffixes == [[3], [3]]
    sb = OP.split_shared_prefix([[1, 2], [5, 6, 7]])
    assert sb.prefix_tokens == [] and sb.suffixes == [[1, 2], [5, 6, 7]]
    sb = OP.split_shared_prefix([[4, 5, 6, 7], [4, 5, 9], [4, 5]])           # boundary moves left
    assert sb.prefix_tokens == [4] and sb.suffixes == [[5, 6, 7], [5, 9], [5]]
    with pytest.raises(ValueError):
        OP.split_shared_prefix([])


def test_merge_attention_algebra():
    rng = np.random.default_rng(2)
    for _ in range(200):
        H, S, Np, dh = 2, int(rng.integers(1, 6)), int(rng.integers(1, 7)), 8
        q = rng.normal(size=(S, H, dh))
        kp, vp = rng.normal(size=(Np, H, dh)), rng.normal(size=(Np, H, dh))
        ks, vs = rng.normal(size=(S, H, dh)), rng.normal(size=(S, H, dh))
        pre = OM.attention_partial(q, kp, vp, causal=False, n_rep=1)
        suf = OM.attention_partial(q, ks, vs, causal=True, n_rep=1)
        merged = OM.merge_attention(pre, suf)
        # dense single pass over concatenated keys
        k = np.concatenate([kp, ks]); v = np.concatenate([vp, vs])
        s = np.einsum("shd,nhd->hsn", q, k) / np.sqrt(dh)
        mask = np.zeros((S, Np + S), dtype=bool)
        mask[:, Np:] = np.triu(np.ones((S, S), dtype=bool), 1)
        s = np.where(mask[None], -np.inf, s)
        p = np.exp(s - s.max(-1, keepdims=True)); p /= p.sum(-1, keepdims=True)
        dense = np.einsum("hsn,nhd->hsd", p, v)
        assert np.max(np.abs(merged - dense)) < 1e-6
        # shift invariance
        c = rng.normal() * 10
        shifted = OM.merge_attention(OM.AttentionPartial(pre.output, pre.lse + c),
                                     OM.AttentionPartial(suf.output, suf.lse + c))
        assert np.max(np.abs(shifted - merged)) < 1e-9
    # lse_p = -inf -> suffix output; equal inputs -> same
    o = rng.normal(size=(2, 3, 4)); l = rng.normal(size=(2, 3))
    out = OM.merge_attention(OM.AttentionPartial(rng.normal(size=(2, 3, 4)), np.full((2, 3), -np.inf)),
                             OM.AttentionPartial(o, l))
    assert np.array_equal(out, o)
    assert np.allclose(OM.merge_attention(OM.AttentionPartial(o, l), OM.AttentionPartial(o, l)), o)


def test_merge_associative():
    rng = np.random.default_rng(3)
    parts = [OM.AttentionPartial(rng.normal(size=(2, 3, 4)), rng.normal(size=(2, 3))) for _ in range(3)]

    def lse_merge(a, b):
        o = OM.merge_attention(a, b)
        return OM.AttentionPartial(o, np.logaddexp(a.lse, b.lse))

    x = lse_merge(lse_merge(parts[0], parts[1]), parts[2])
    y = lse_merge(parts[0], lse_merge(parts[1], parts[2]))
    assert np.max(np.abs(x.output - y.output)) < 1e-9


# ----------------------------------------------------------------------------- model
def test_forward_known_answers(w32):
    logits, cache = OM.forward_prefill(w32, [7])
    assert np.all(np.isfinite(logits)) and cache.seq_len == 1
    with pytest.raises(ValueError):
        OM.forward_prefill(w32, [])
    with pytest.raises(ValueError):
        OM.forward_prefill(w32, [5] * (SPEC_DEFAULT.max_seq + 1))


def test_split_at_25_of_40(w32):
    rng = np.random.default_rng(4)
    toks = list(rng.integers(16, 32768, 40))
    full, _ = OM.forward_prefill(w32, toks)
    _, kv = OM.forward_prefill(w32, toks[:25])
    part, _ = OM.forward_with_prefix(w32, kv, toks[25:])
    assert np.max(np.abs(full - part)) < 1e-5


def test_prefix_split_equivalence_f32_f64(w32, w64):
    """ACCEPTANCE 1: shared-prefix scoring == independent full passes."""
    rng = np.random.default_rng(5)
    worst32 = worst64 = 0.0
    for r in range(24):
        n = int(rng.integers(2, 17))
        P = int(rng.integers(0, 64))
        prefix = list(rng.integers(16, 32768, P))
        prompts = [prefix + list(rng.integers(16, 32768, int(rng.integers(1, 128 - P + 1))))
                   for _ in range(n)]
        prompts = [p[:128] for p in prompts]
        sb = OP.split_shared_prefix(prompts)
        ws = [w32] + ([w64] if r < 6 else [])
        for w in ws:
            shared = OP.score_shared_batch(w, OP.SharedBatch(sb.prefix_tokens, sb.suffixes))
            for i, p in enumerate(prompts):
                full, _ = OM.forward_prefill(w, p)
                d = float(np.max(np.abs(full - shared[i])))
                if w is w32:
                    worst32 = max(worst32, d)
                else:
                    worst64 = max(worst64, d)
    assert worst32 < 1e-5 and worst64 < 1e-10, (worst32, worst64)


def test_determinism_and_position_sensitivity(w64):
    rng = np.random.default_rng(6)
    toks = list(rng.integers(16, 32768, 20))
    a, _ = OM.forward_prefill(w64, toks)
    b, _ = OM.forward_prefill(w64, toks)
    assert np.array_equal(a, b)
    swapped = toks.copy()
    swapped[3], swapped[9] = swapped[9], swapped[3]
    c, _ = OM.forward_prefill(w64, swapped)
    assert not np.allclose(a, c)


def test_f32_f64_argmax_agreement():
    w32 = OM.init_weights(SMALL, 1)
    w64 = w32.astype(np.float64)
    rng = np.random.default_rng(7)
    agree, n = 0, 200
    for _ in range(n):
        toks = list(rng.integers(16, SMALL.vocab_size, int(rng.integers(1, 40))))
        agree += int(np.argmax(OM.forward_prefill(w32, toks)[0]) == np.argmax(OM.forward_prefill(w64, toks)[0]))
    assert agree >= 0.99 * n


def test_param_count_closed_form(w32):
    n = w32.token_embedding.size + w32.final_norm.size + w32.head.size
    n += sum(a.size for lw in w32.layers for a in lw.values())
    assert n == OM.param_count(SPEC_DEFAULT) == SPEC_DEFAULT.param_count()


def test_init_determinism_and_seed():
    a = OM.init_weights(SMALL, 3)
    b = OM.init_weights(SMALL, 3)
    c = OM.init_weights(SMALL, 4)
    assert np.array_equal(a.layers[1]["W_down"], b.layers[1]["W_down"])
    assert not np.array_equal(a.layers[1]["W_down"], c.layers[1]["W_down"])
