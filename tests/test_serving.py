"""Serving wrapper: prompt contract against the reference golden outputs, cache /
PID / shaper known answers, and handle_score_request with a CPU test double for the scorer."""

import json
import os

import numpy as np
import pytest

from paper_2510_22101_b200 import ingest
from paper_2510_22101_b200.serving import (JobItem, PidController, PromptBudgetError, Query, ScoreCache,
                                           ScoreRequest, ScoringService, TokenBucketShaper, assemble_prompt,
                                           query_hash, truncate_description)

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "prompts.json")))


def test_assembly_and_truncation_match_reference():
    for case in GOLDEN["assembly"]:
        q, it = Query(**case["query"]), JobItem(**case["item"])
        seg = assemble_prompt(q, it)
        assert seg.__dict__ == case["segments"]
        for budget, want in case["truncated"].items():
            if isinstance(want, dict):
                with pytest.raises(PromptBudgetError) as e:
                    truncate_description(seg, int(budget))
                assert str(e.value) == want["error"]
            else:
                got = truncate_description(seg, int(budget)).full_prompt()
                assert got == want, budget
                assert len(ingest.encode(got)) <= int(budget)


def test_native_spans_match_reference():
    from paper_2510_22101_b200.serving import _spans

    for text, spans in GOLDEN["spans"]:
        ids, ends = _spans(text, ingest.DEFAULT_VOCAB)
        assert ids.tolist() == [s[0] for s in spans]
        assert ends.tolist() == [s[2] for s in spans]


def test_cache_kats():
    c = ScoreCache(capacity=2, ttl=900)
    c.insert("a", 0.7, now=0.0)
    assert c.lookup("a", now=899.0) == 0.7
    assert c.lookup("a", now=900.0 + 1e-6) is None
    c.insert("a", 0.1, 1000.0); c.insert("b", 0.2, 1000.0); c.insert("c", 0.3, 1000.0)
    assert c.lookup("a", 1000.0) is None and len(c) == 2        # SPEC.md:674 (LRU evicted)
    c.insert("x", 0.5, 2000.0)
    c.lookup("x", 2500.0)                                       # hit refreshes LRU, not TTL
    assert c.lookup("x", 2901.0) is None


def test_pid_kats():
    p = PidController()
    assert p.update(500.0, 500.0, 1.0) == 250
    p = PidController()
    depths = [p.update(1000.0, 500.0, 1.0) for _ in range(40)]
    assert all(b <= a for a, b in zip(depths, depths[1:])) and depths[-1] == 50
    p = PidController()
    depths = [p.update(50.0, 500.0, 1.0) for _ in range(40)]
    assert max(depths) == 1000 and all(d <= 1000 for d in depths)
    z = PidController(kp=0, ki=0, kd=0)
    assert all(z.update(o, 500.0, 1.0) == 250 for o in (10.0, 900.0, 5000.0))


def test_shaper_kats():
    s = TokenBucketShaper(rate=10.0, burst=3, max_defer=0.5)
    assert s.admit(0.0) == 0.0                                  # SPEC.md:690 idle bucket
    s = TokenBucketShaper(rate=10.0, burst=3, max_defer=0.5)
    adm = [s.admit(1.0) for _ in range(4)]
    assert adm[:3] == [1.0, 1.0, 1.0] and abs(adm[3] - 1.1) < 1e-12
    s = TokenBucketShaper(rate=1.0, burst=1, max_defer=0.25)
    s.admit(0.0)
    assert s.admit(0.0) == 0.25                                 # SPEC.md:692 SLA clamp
    rng = np.random.default_rng(0)
    s = TokenBucketShaper(rate=50.0, burst=5, max_defer=0.2)
    arr = np.sort(rng.uniform(0, 2.0, 300))
    adm = [s.admit(a) for a in arr]
    assert len(adm) == 300 and all(b - a <= 0.2 + 1e-9 for a, b in zip(arr, adm))  # no drops, bounded


class FakeScorer:
    """Test double for the device scorer: deterministic p_yes from each item's token ids."""

    def __init__(self):
        self.calls = 0

    def score_packed(self, packed):
        self.calls += 1

        class R:
            pass

        r = R()
        r.p_yes = np.array([((int(packed.ids[i - 1]) * 7919 + int(packed.ids[i])) % 997) / 997.0
                            for i in packed.last_idx], dtype=np.float32)
        return r


def items(n, seed=0):
    rng = np.random.default_rng(seed)
    return [JobItem(f"j{i:04d}", f"engineer {rng.integers(100)}", "acme", "berlin", "full_time", bool(i % 2),
                    " ".join(f"w{int(x)}" for x in rng.integers(0, 500, int(rng.integers(5, 60))))) for i in range(n)]


def test_service_cache_repeat_and_depth():
    fs = FakeScorer()
    svc = ScoringService(fs, model_version="v1", pid=PidController(depth=131))
    req = ScoreRequest(Query("q1", "Rust Engineer"), items(1000), "r1")
    r1 = svc.handle_score_request(req)
    assert r1.depth_used == 131 and len(r1.scores) == 131 and len(r1.unscored) == 869
    assert all(s["source"] == "model" for s in r1.scores) and fs.calls == 1
    ps = [s["p_yes"] for s in r1.scores]
    assert ps == sorted(ps, reverse=True)
    r2 = svc.handle_score_request(ScoreRequest(Query("q1", "rust   ENGINEER"), items(1000), "r2"))
    assert fs.calls == 1 and all(s["source"] == "cache" for s in r2.scores)
    assert [(s["item_id"], s["p_yes"]) for s in r2.scores] == [(s["item_id"], s["p_yes"]) for s in r1.scores]  # :700
    m = svc.metrics()
    assert m["cache"]["hits"] == 131 and m["engine"]["items_scored"] == 131


def test_service_per_item_budget_error():
    svc = ScoringService(FakeScorer(), model_version="v1", token_budget=24)
    r = svc.handle_score_request(ScoreRequest(Query("q", "data"), items(3), "r"))
    assert len(r.errors) == 3 and r.scores == []                # rejected per item, not the request


def test_query_hash_normalizes():
    assert query_hash("Rust  Engineer ") == query_hash("rust engineer") != query_hash("rust engineers")
