"""Property-based parity (hypothesis) for the bit-exact host contracts, beyond the fixed goldens:
the C++ tokenizer vs the oracle restatement on arbitrary Unicode text; the C++ and Python packers vs
the oracle packer on random shared-prefix requests; the calibration sampler vs the oracle."""

import json
import os

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle.calibration as OC
import oracle.prefixcache as OP
import oracle.tokenizer as OT
from paper_2510_22101_b200 import ingest
from paper_2510_22101_b200.calibration import sample_positions
from paper_2510_22101_b200.prefixcache import pack_requests, split_shared_prefix

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "prompts.json")))
SETTINGS = settings(max_examples=300, deadline=None, suppress_health_check=[HealthCheck.too_slow])

# text from pieces that stress the scanner: tags (also partial / upper-case), words, digits,
# punctuation, the two special lowercase code points (U+0130, U+212A), other non-ASCII letters
PIECES = st.sampled_from(["<|sys|>", "<|/SYS|>", "<|q|>", "<|/q|>", "<|meta|>", "<|/Meta|>", "<|desc|>",
                          "<|/desc|>", "<|ans|>", "<|", "|>", "<", ">", "|", "/", "yes", "NO", "No",
                          "rust", "Engineer", "9a", "a9", "x", " ", "\n", "\t", ".", ",", "-", "_",
                          "İ", "K", "K", "ß", "é", "ı", "Σ", "\U0001f600", "Å"])
TEXT = st.one_of(st.lists(PIECES, max_size=60).map("".join), st.text(max_size=200))


def test_oracle_tokenizer_pinned_to_reference_goldens():
    for text, ids in GOLDEN["texts"][:200]:
        assert OT.encode(text) == ids
    for s, ids in GOLDEN["encode"].items():
        assert OT.encode(s) == ids
    for w, i in GOLDEN["word_id"].items():
        assert OT.word_id(w) == i
    for text, spans in GOLDEN["spans"]:
        assert [list(x) for x in OT.encode_with_spans(text)] == [list(x) for x in spans]


@SETTINGS
@given(TEXT)
def test_native_tokenizer_equals_oracle(text):
    assert ingest.encode(text) == OT.encode(text)


@SETTINGS
@given(st.lists(TEXT, min_size=1, max_size=8))
def test_native_batch_tokenizer_equals_oracle(texts):
    assert ingest.encode_batch(texts, n_threads=3) == [OT.encode(t) for t in texts]


@SETTINGS
@given(TEXT)
def test_native_spans_equal_oracle(text):
    from paper_2510_22101_b200.serving import _spans

    ids, ends = _spans(text, ingest.DEFAULT_VOCAB)
    ref = OT.encode_with_spans(text)
    assert ids.tolist() == [t for t, _, _ in ref] and ends.tolist() == [e for _, _, e in ref]


@st.composite
def requests(draw):
    """1-4 requests; each: a shared prefix (possibly empty) + 1-6 lists that may extend it, share
    more than it, or equal it (the LCP-moves-left rule)."""
    out = []
    for _ in range(draw(st.integers(1, 4))):
        prefix = draw(st.lists(st.integers(0, 50), max_size=12))
        lists = []
        for _ in range(draw(st.integers(1, 6))):
            tail = draw(st.lists(st.integers(0, 50), max_size=10))
            lst = prefix + tail
            if not lst:
                lst = [draw(st.integers(0, 50))]
            lists.append(lst)
        out.append(lists)
    return out


@SETTINGS
@given(requests())
def test_packers_equal_oracle(reqs):
    ids, pos, segs, last = OP.pack([OP.split_shared_prefix(r) for r in reqs])
    py = pack_requests([split_shared_prefix(r) for r in reqs])
    nat = ingest.pack_token_lists_native(reqs)
    for got in (py, nat):
        np.testing.assert_array_equal(got.ids, ids)
        np.testing.assert_array_equal(got.pos, pos)
        np.testing.assert_array_equal(got.segs, segs)
        np.testing.assert_array_equal(got.last_idx, last)


@SETTINGS
@given(st.lists(st.integers(1, 300), min_size=1, max_size=20), st.integers(1, 3000), st.integers(0, 2**31))
def test_sampler_equals_oracle(lens, budget, seed):
    np.testing.assert_array_equal(sample_positions(lens, budget, seed), OC.sample_positions(lens, budget, seed))
