"""Packing / prefix indexing: bit-exact against the oracle packer, on random batches and on the
golden Eq-1 prompts produced by the reference tokenizer + corpus (tests/golden/prompts.json)."""

import json
import os

import numpy as np
import pytest

import oracle.prefixcache as OP
from paper_2510_22101_b200 import prefixcache as PC

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "prompts.json")))


def assert_packed_equal(pk, batches):
    ids, pos, segs, last = OP.pack([OP.SharedBatch(b.prefix_tokens, b.suffixes) for b in batches])
    np.testing.assert_array_equal(pk.ids, ids)
    np.testing.assert_array_equal(pk.pos, pos)
    np.testing.assert_array_equal(pk.segs, segs)
    np.testing.assert_array_equal(pk.last_idx, last)
    assert pk.ids.dtype == np.int32 and pk.segs.dtype == np.int32


def check_work(pk):
    seen = set()
    for seg, tile, _, _ in pk.work.tolist():
        assert (seg, tile) not in seen
        seen.add((seg, tile))
        assert 0 <= tile * 128 < pk.segs[seg, 3]
    assert len(seen) == int(sum((q + 127) // 128 for q in pk.segs[:, 3]))


def test_split_matches_oracle_random():
    rng = np.random.default_rng(0)
    for _ in range(300):
        n = int(rng.integers(1, 12))
        P = int(rng.integers(0, 40))
        base = list(rng.integers(0, 6, P))
        lists = [base[: int(rng.integers(0, P + 1))] + list(rng.integers(0, 6, int(rng.integers(0, 6))))
                 for _ in range(n)]
        lists = [l if l else [1] for l in lists]
        a = PC.split_shared_prefix(lists)
        b = OP.split_shared_prefix(lists)
        assert a.prefix_tokens == b.prefix_tokens and a.suffixes == b.suffixes
        assert all(len(s) >= 1 for s in a.suffixes)
        assert all(a.prompt(i) == lists[i] for i in range(n))


def test_pack_bit_exact_random():
    rng = np.random.default_rng(1)
    for _ in range(100):
        batches = []
        for _ in range(int(rng.integers(1, 5))):
            P = int(rng.integers(0, 300))
            pre = list(rng.integers(16, 32768, P))
            sufs = [list(rng.integers(16, 32768, int(rng.integers(1, 400)))) for _ in range(int(rng.integers(1, 20)))]
            batches.append(PC.SharedBatch(pre, sufs))
        pk = PC.pack_requests(batches)
        assert_packed_equal(pk, batches)
        check_work(pk)
        # every item's last row holds its last token; positions restart per suffix at P
        for r, b in enumerate(batches):
            pass
        k = 0
        for b in batches:
            for s in b.suffixes:
                assert pk.ids[pk.last_idx[k]] == s[-1]
                assert pk.pos[pk.last_idx[k]] == len(b.prefix_tokens) + len(s) - 1
                k += 1


def test_golden_prompts_split_and_pack():
    """Eq-1 prompts from the reference: the LCP covers system prefix + query block (+ the
    <|meta|> tag, which every item shares) and every packed item ends on <|ans|> (id 11)."""
    ans = GOLDEN["vocab"]["specials"]["<|ans|>"]
    meta = GOLDEN["vocab"]["specials"]["<|meta|>"]
    batches = []
    for req in GOLDEN["requests"]:
        prompts = req["prompts"]
        sb = PC.split_shared_prefix(prompts)
        sys_q = req["segment_lens"][0][0] + req["segment_lens"][0][1]
        assert len(sb.prefix_tokens) >= sys_q
        assert sb.prefix_tokens[:sys_q] == prompts[0][:sys_q]
        if len(sb.prefix_tokens) > sys_q:
            assert sb.prefix_tokens[sys_q] == meta
        batches.append(sb)
    pk = PC.pack_requests(batches)
    assert_packed_equal(pk, batches)
    assert np.all(pk.ids[pk.last_idx] == ans)
    flat = np.concatenate([np.concatenate([np.asarray(b.prefix_tokens, dtype=np.int64)] +
                                          [np.asarray(s) for s in b.suffixes]) for b in batches])
    np.testing.assert_array_equal(pk.ids, flat)
    assert pk.pos.max() < 2048


def test_pack_errors():
    with pytest.raises(ValueError):
        PC.pack_requests([])
    with pytest.raises(ValueError):
        PC.pack_requests([PC.SharedBatch([1, 2], [])])
    with pytest.raises(ValueError):
        PC.pack_requests([PC.SharedBatch([1] * 2000, [[2] * 49])])
    with pytest.raises(ValueError):
        PC.split_shared_prefix([])


def test_throughput_gain_and_merge_product():
    assert abs(PC.throughput_gain(50, 150) - 4 / 3) < 1e-12
    rng = np.random.default_rng(2)
    a = PC.AttentionPartial(rng.normal(size=(2, 3, 4)), rng.normal(size=(2, 3)))
    b = PC.AttentionPartial(rng.normal(size=(2, 3, 4)), rng.normal(size=(2, 3)))
    import oracle.model as OM
    np.testing.assert_allclose(PC.merge_attention(a, b),
                               OM.merge_attention(OM.AttentionPartial(a.output, a.lse),
                                                  OM.AttentionPartial(b.output, b.lse)), atol=1e-12)
    c = PC.merge_attention(PC.AttentionPartial(a.output, np.full((2, 3), -np.inf)), b)
    np.testing.assert_array_equal(c, b.output)


def test_concat_packed_equals_joint_packing():
    """Requests packed one by one (at arrival) and joined per launch give the same arrays as
    packing the whole batch at once: segments, work order, last rows, request ids."""
    from paper_2510_22101_b200 import SharedBatch, concat_packed, pack_requests

    rng = np.random.default_rng(21)
    reqs = []
    for _ in range(5):
        P = int(rng.integers(0, 80))
        sufs = [list(rng.integers(16, 1000, int(rng.integers(1, 300)))) for _ in range(int(rng.integers(1, 9)))]
        reqs.append(SharedBatch(list(rng.integers(16, 1000, P)), sufs))
    joint = pack_requests(reqs)
    joined = concat_packed([pack_requests([r]) for r in reqs])
    for f in ("ids", "pos", "segs", "work", "last_idx", "item_request", "prefix_lens", "suffix_lens"):
        a, b = getattr(joint, f), getattr(joined, f)
        assert a.dtype == b.dtype and np.array_equal(a, b), f
