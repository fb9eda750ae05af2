"""ReplicaPool and the service on top of it, on the device.

* batched + pipelined launches give the scores of one launch per request (rows are independent);
* item-split shards come back in the request's item order;
* ScoringService.submit over the pool matches the CPU oracle on golden reference prompts.
On a one-GPU box the pool holds two replicas on cuda:0 (two scorers, two worker threads, two
streams): the multi-replica code path, not a scaling measurement.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2510_22101_b200 import CONFIGS, init_weights, pack_requests  # noqa: E402
from paper_2510_22101_b200.engine import PrefillScorer  # noqa: E402
from paper_2510_22101_b200.replicas import ReplicaPool  # noqa: E402
from tests.synth import make_shared  # noqa: E402


def _pool(n=2, **kw):
    w = init_weights(CONFIGS["TINY_GQA"], 0)
    devs = [f"cuda:{i % torch.cuda.device_count()}" for i in range(n)]
    return ReplicaPool([PrefillScorer(w, d) for d in devs], **kw)


def test_pool_batches_equal_single_launches():
    pool = _pool(2, token_budget=4096)
    rng = np.random.default_rng(50)
    reqs = [make_shared(rng, int(rng.integers(0, 80)), list(rng.integers(1, 300, int(rng.integers(1, 20)))),
                        "spread") for _ in range(24)]
    futs = [pool.submit_shared(sb) for sb in reqs]      # queued together: coalesced into few launches
    got = [f.result(timeout=60) for f in futs]
    ref = PrefillScorer(init_weights(CONFIGS["TINY_GQA"], 0))
    for sb, g in zip(reqs, got):
        want = ref.score_packed(pack_requests([sb]))
        np.testing.assert_allclose(g.p_yes, want.p_yes, rtol=0, atol=1e-6)
        np.testing.assert_allclose(g.logits2, want.logits2, rtol=0, atol=1e-5)
    st = pool.stats()
    assert sum(st["items_scored"]) == sum(sb.n_items for sb in reqs)
    assert sum(st["launches"]) < len(reqs)               # batching happened
    pool.close()


def test_item_split_shards_keep_item_order():
    pool = _pool(2, max_shard_items=7)
    rng = np.random.default_rng(51)
    sb = make_shared(rng, 40, list(rng.integers(1, 200, 30)), "spread")
    got = pool.submit_shared(sb).result(timeout=60)
    want = PrefillScorer(init_weights(CONFIGS["TINY_GQA"], 0)).score_packed(pack_requests([sb]))
    np.testing.assert_allclose(got.p_yes, want.p_yes, rtol=0, atol=1e-6)
    assert len(got) == 30
    pool.close()


def test_service_over_pool_matches_oracle():
    import json
    import os

    import oracle.model as OM
    import oracle.prefixcache as OP
    import oracle.scoring as OS
    from paper_2510_22101_b200 import ingest
    from paper_2510_22101_b200.serving import JobItem, Query, ScoreRequest, ScoringService

    golden = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "prompts.json")))
    cfg = CONFIGS["TINY"]
    w = init_weights(cfg, 0)
    pool = ReplicaPool([PrefillScorer(w), PrefillScorer(w)])
    svc = ScoringService(pool, model_version="tiny", token_budget=300)
    case = golden["assembly"]
    queries = {}
    for c in case:
        queries.setdefault(json.dumps(c["query"], sort_keys=True), []).append(c)
    ow = OM.init_weights(cfg, 0)
    futs = []
    for k, cs in queries.items():
        futs.append((cs, svc.submit(ScoreRequest(Query(**cs[0]["query"]), [JobItem(**c["item"]) for c in cs], k))))
    for cs, f in futs:
        got = {s["item_id"]: s["p_yes"] for s in f.result(timeout=60).scores}
        prompts = [ingest.encode(c["truncated"]["300"]) for c in cs]
        ref = [OS.relevance_score(l)[0] for l in OP.score_shared_batch(ow, OP.split_shared_prefix(prompts))]
        for c, p in zip(cs, ref):
            assert abs(got[c["item"]["id"]] - p) <= 1e-2
    m = svc.metrics()
    assert m["engine"]["items_scored"] == len(case) and m["engine"]["flops_saved_pct"] >= 0
    svc.close()
    pool.close()
