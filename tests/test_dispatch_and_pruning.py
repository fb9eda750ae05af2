"""Host-side multi-replica logic (gloo, world_size 2, CPU) and the pruning shape contract."""

import os
import socket

import numpy as np
import pytest

from paper_2510_22101_b200 import CONFIGS, init_weights
from paper_2510_22101_b200.dispatch import (assign_least_loaded, request_tokens, score_local,
                                            split_request)
from paper_2510_22101_b200.prefixcache import SharedBatch, pack_requests
from paper_2510_22101_b200.pruning import (PruneRecipe, apply_recipe, kept_width, prune_kv_groups,
                                           prune_mlp_neurons, remove_layers, select_keep_by_norm)


class _Res:
    def __init__(self, p):
        self.p_yes = p


def fake_score_packed(packed):
    """Deterministic stand-in for the GPU scorer (test double): a hash of each item's tokens."""
    p = []
    start = 0
    for seg in packed.segs:
        pass
    ids = packed.ids.astype(np.int64)
    for k, last in enumerate(packed.last_idx):
        p.append(((int(ids[last]) * 2654435761 + int(packed.pos[last])) % 1000) / 1000.0)
    return _Res(np.asarray(p, dtype=np.float32))


def make_requests(seed, n):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        P = int(rng.integers(1, 40))
        pre = list(rng.integers(16, 1000, P))
        out.append(SharedBatch(pre, [list(rng.integers(16, 1000, int(rng.integers(1, 60))))
                                     for _ in range(int(rng.integers(1, 12)))]))
    return out


def test_assign_least_loaded():
    assert assign_least_loaded([10, 10, 10, 10], 2) == [[0, 2], [1, 3]]
    assert assign_least_loaded([100, 1, 1, 1], 2) == [[0], [1, 2, 3]]
    a = assign_least_loaded([5, 3, 8, 1, 9, 2], 3)
    assert sorted(sum(a, [])) == list(range(6))
    with pytest.raises(ValueError):
        assign_least_loaded([1], 0)


def test_split_request_and_local_scoring():
    reqs = make_requests(0, 6)
    big = SharedBatch([1, 2, 3], [[7, 8]] * 25)
    parts = split_request(big, 10)
    assert [p.n_items for p in parts] == [10, 10, 5] and all(p.prefix_tokens == [1, 2, 3] for p in parts)
    whole = score_local(fake_score_packed, reqs, 2048)
    tiny = score_local(fake_score_packed, reqs, 2048, max_tokens_per_launch=1)
    for a, b, r in zip(whole, tiny, reqs):
        assert len(a) == r.n_items
        np.testing.assert_array_equal(a, b)


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2510_22101_b200.dispatch import ReplicaGroup

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grp = ReplicaGroup(fake_score_packed)
        reqs = make_requests(1, 9) if rank == 0 else None
        out = grp.score(reqs)
        if rank == 0:
            ref = score_local(fake_score_packed, make_requests(1, 9), 2048)
            q.put(all(np.array_equal(a, b) for a, b in zip(out, ref)) and len(out) == 9)
        else:
            q.put(out is None)
    finally:
        dist.destroy_process_group()


def test_replica_group_gloo_world2():
    import multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) and q.get(timeout=5)


# ----------------------------------------------------------------------------- pruning
def test_prune_mlp_and_layers_contract():
    cfg = CONFIGS["TINY_GQA"]
    w = init_weights(cfg, 0)
    k = kept_width(cfg.d_ff, 0.4)
    assert k == round(0.6 * cfg.d_ff)
    keep = select_keep_by_norm(w, 0.4)
    pw = prune_mlp_neurons(w, keep)
    assert pw.config.d_ff == k
    for l in range(cfg.n_layers):
        np.testing.assert_array_equal(pw.layers[l].W_gate, w.layers[l].W_gate[:, keep[l]])
        np.testing.assert_array_equal(pw.layers[l].W_down, w.layers[l].W_down[keep[l]])
    removed = cfg.params_per_layer() - pw.config.params_per_layer()
    assert removed == 3 * cfg.d_model * (cfg.d_ff - k)
    rl = remove_layers(pw, [cfg.n_layers - 1])
    assert rl.config.n_layers == cfg.n_layers - 1
    assert rl.param_count() == pw.param_count() - pw.config.params_per_layer()
    assert rl.param_count() == rl.config.param_count()
    with pytest.raises(ValueError):
        remove_layers(pw, range(cfg.n_layers))
    with pytest.raises(ValueError):
        prune_mlp_neurons(w, [keep[0], keep[1][:-1], keep[2]])              # non-uniform
    with pytest.raises(ValueError):
        PruneRecipe(mlp_sparsity=1.0)


def test_refit_rows_follow_the_callers_keep_order():
    """refit W_down rows aligned with an unsorted keep-set stay paired with their neurons."""
    cfg = CONFIGS["TINY_GQA"]
    w = init_weights(cfg, 0)
    k = kept_width(cfg.d_ff, 0.5)
    rng = np.random.default_rng(3)
    keep = [rng.permutation(cfg.d_ff)[:k] for _ in range(cfg.n_layers)]           # unsorted
    rows = [w.layers[l].W_down[keep[l]] * 2.0 for l in range(cfg.n_layers)]      # aligned with keep
    pw = prune_mlp_neurons(w, keep, rows)
    for l in range(cfg.n_layers):
        order = np.sort(keep[l])
        np.testing.assert_array_equal(pw.layers[l].W_gate, w.layers[l].W_gate[:, order])
        np.testing.assert_array_equal(pw.layers[l].W_down, w.layers[l].W_down[order] * 2.0)


def test_prune_kv_groups_keeps_gqa_invariant():
    cfg = CONFIGS["C3"].with_(n_layers=1, vocab_size=64)
    w = init_weights(cfg, 0)
    pw = prune_kv_groups(w, range(5))
    assert (pw.config.n_heads, pw.config.n_kv_heads) == (10, 5)
    assert pw.layers[0].W_q.shape == (2048, 1280) and pw.layers[0].W_o.shape == (1280, 2048)
    np.testing.assert_array_equal(pw.layers[0].W_k, w.layers[0].W_k[:, : 5 * 128])
    c4 = apply_recipe(w, PruneRecipe(mlp_sparsity=0.4, kv_groups_to_keep=5))
    assert c4.config.d_ff == 3686 and c4.config.n_heads == 10                # config C4 widths


def test_shard_bounds_balance_tokens_and_cover_items():
    """ReplicaPool.shard_bounds: contiguous item ranges covering the request, at most shard_tokens
    tokens per shard (unless one item alone exceeds it), at least one shard per replica when the
    request has min_shard_items items per replica."""
    from paper_2510_22101_b200.replicas import ReplicaPool

    pool = ReplicaPool.__new__(ReplicaPool)
    pool.workers = [None] * 4
    pool.shard_tokens, pool.min_shard_items = 1000, 8
    rng = np.random.default_rng(0)
    for n in (1, 5, 31, 32, 200):
        toks = rng.integers(64, 400, n)
        b = pool.shard_bounds(toks)
        assert b[0][0] == 0 and b[-1][1] == n and all(x[1] == y[0] for x, y in zip(b, b[1:]))
        assert all(hi > lo for lo, hi in b)
        if n >= 32:
            assert len(b) >= 4
        sums = [int(toks[lo:hi].sum()) for lo, hi in b]
        assert max(sums) <= 1000 + int(toks.max())


def test_bench_gpus_n_self_launches_torchrun():
    """`bench.py --gpus N` without a torchrun environment re-runs itself under torch.distributed.run
    with N ranks (127.0.0.1 rendezvous); rank 0 alone prints the line (reference arm: CPU only)."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--config", "C1", "--steps", "1", "--warmup", "1", "--ref-items", "2"],
                         capture_output=True, text=True, env=env, timeout=600, check=True).stdout
    lines = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
