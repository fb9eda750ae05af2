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


# ----------------------------------------------------------------------------- concurrency model
class SlowScorer(FakeScorer):
    """Fake scorer that takes ``delay`` seconds per call (to exercise overlap and the PID loop)."""

    def __init__(self, delay):
        super().__init__()
        self.delay = delay
        self.active = self.max_active = 0
        import threading
        self.lock = threading.Lock()

    def score_packed(self, packed):
        import time
        with self.lock:
            self.active += 1
            self.max_active = max(self.max_active, self.active)
        time.sleep(self.delay)
        with self.lock:
            self.active -= 1
        return super().score_packed(packed)


def test_submit_is_concurrent_and_matches_sync():
    """requests are processed concurrently up to the worker-pool limit; results equal
    the synchronous path's."""
    fs = SlowScorer(0.05)
    svc = ScoringService(fs, model_version="v1", workers=4)
    reqs = [ScoreRequest(Query(f"q{i}", f"query {i}"), items(20, seed=i), f"r{i}") for i in range(8)]
    futs = [svc.submit(r) for r in reqs]
    got = [f.result(timeout=30) for f in futs]
    assert fs.max_active > 1 and fs.calls == 8
    ref = ScoringService(FakeScorer(), model_version="v1")
    for r, g in zip(reqs, got):
        want = ref.handle_score_request(r)
        assert [(s["item_id"], s["p_yes"]) for s in g.scores] == [(s["item_id"], s["p_yes"]) for s in want.scores]
    svc.close(); ref.close()


def test_shaper_defers_without_blocking_the_caller():
    """A deferred admission waits in the admission queue, not in submit(): submit returns at once
    and the deferred request still completes, after its admit time."""
    import time

    svc = ScoringService(FakeScorer(), model_version="v1",
                         shaper=TokenBucketShaper(rate=5.0, burst=1, max_defer=0.5), workers=2)
    t0 = time.monotonic()
    futs = [svc.submit(ScoreRequest(Query("q", "x"), items(3, seed=i), f"r{i}", arrival=t0)) for i in range(3)]
    assert time.monotonic() - t0 < 0.1                      # no sleep in the caller
    resp = [f.result(timeout=10) for f in futs]
    queue = [r.timings_ms["queue"] for r in resp]
    assert queue[0] < 50 and 150 <= queue[1] and 350 <= queue[2] <= 700     # 1/R = 200 ms, clamp 500 ms
    assert svc.metrics()["shaper"]["deferred"] == 2
    svc.close()


def test_metrics_loop_drives_the_pid_depth():
    """The single metrics loop feeds the sliding-window p95 to the PID: with every
    request slower than the target, depth falls from its initial value."""
    import time

    svc = ScoringService(SlowScorer(0.03), model_version="v1", pid=PidController(depth=250),
                         target_p95_ms=10.0, pid_interval=0.05, window_s=5.0, workers=2)
    for i in range(6):
        svc.handle_score_request(ScoreRequest(Query(f"q{i}", f"w {i}"), items(5, seed=i), f"r{i}"))
    time.sleep(0.3)
    m = svc.metrics()
    assert m["pid"]["p95_ms"] >= 30 and svc.pid.depth < 250
    svc.close()


def test_metrics_engine_fields():
    """GET /v1/metrics engine block: items_per_sec over the window and the FLOPs saved
    by computing each prefix once (W1 accounting)."""
    from paper_2510_22101_b200 import CONFIGS
    from paper_2510_22101_b200.prefixcache import request_flops, throughput_gain

    cfg = CONFIGS["TINY"]
    svc = ScoringService(FakeScorer(), model_version="v1", model_config=cfg, window_s=60.0)
    r = svc.handle_score_request(ScoreRequest(Query("q", "data engineer"), items(10), "r"))
    m = svc.metrics()["engine"]
    assert m["items_scored"] == 10 and m["items_per_sec"] > 0
    assert 0 < m["flops_saved_pct"] < 100
    # uniform suffixes: counted-FLOP ratio vs independent passes ~ throughput_gain (5%)
    for P, S in ((50, 150), (64, 100), (100, 100)):
        ratio = request_flops(cfg, P, [S] * 64, False) / request_flops(cfg, P, [S] * 64, True)
        assert abs(ratio / throughput_gain(P, S) - 1) < 0.05, (P, S, ratio)
    svc.close()


def test_shadow_scoring_checks_hits_within_tolerance():
    svc = ScoringService(FakeScorer(), model_version="v1", shadow_rate=1.0)
    req = ScoreRequest(Query("q", "rust"), items(12), "r")
    svc.handle_score_request(req)
    r2 = svc.handle_score_request(req)
    assert all(s["source"] == "cache" for s in r2.scores)
    sh = svc.metrics()["shadow"]
    assert sh["checked"] == 12 and sh["violations"] == 0
    svc.close()


def test_batched_tokenize_equals_per_item_truncation():
    """The service's one-batch tokenization equals the per-item pipeline (assemble -> truncate ->
    encode, corpus.py:302-345) for items below, at and above the budget, and rejects the same items."""
    svc = ScoringService(FakeScorer(), model_version="v1", token_budget=60)
    its = items(40, seed=3)
    q = Query("q", "rust systems engineer")
    errors = []
    ids, offs, ok = svc._tokenize(q, its, errors)
    want, want_err = [], []
    for it in its:
        try:
            want.append(ingest.encode(truncate_description(assemble_prompt(q, it), 60).full_prompt()))
        except PromptBudgetError:
            want_err.append(it.id)
    assert [e["item_id"] for e in errors] == want_err
    assert [ids[offs[i]:offs[i + 1]].tolist() for i in range(len(ok))] == want
    assert any(len(w) == 60 for w in want) and any(len(w) < 60 for w in want)
    svc.close()
