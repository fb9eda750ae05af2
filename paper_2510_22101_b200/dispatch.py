"""Host dispatcher for request-sharded replicas: one process per GPU, each owning
a full weight replica; no collective on the data path — requests go out, scores come back.

* ``assign_least_loaded`` — whole requests to the replica with the fewest outstanding tokens
  (ties -> lowest replica index), in arrival order.
* ``split_request`` — a request with more items than ``max_items`` is item-split; every shard
  keeps the (short) prefix, which is recomputed per shard (+P tokens per shard).
* ``ReplicaGroup`` — the torch.distributed form: rank 0 holds the requests, scatters the
  assignment (object scatter, control plane only), every rank packs + scores its share on its own
  GPU, rank 0 gathers the per-request score vectors in the original order.
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

from .prefixcache import SharedBatch, pack_requests


def request_tokens(sb: SharedBatch) -> int:
    return len(sb.prefix_tokens) + sum(len(s) for s in sb.suffixes)


def assign_least_loaded(token_counts: Sequence[int], n_replicas: int,
                        outstanding: Sequence[int] | None = None) -> list[list[int]]:
    if n_replicas < 1:
        raise ValueError("n_replicas must be >= 1")
    load = list(outstanding) if outstanding is not None else [0] * n_replicas
    out: list[list[int]] = [[] for _ in range(n_replicas)]
    for i, t in enumerate(token_counts):
        r = min(range(n_replicas), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += int(t)
    return out


def split_request(sb: SharedBatch, max_items: int) -> list[SharedBatch]:
    if max_items < 1:
        raise ValueError("max_items must be >= 1")
    return [SharedBatch(list(sb.prefix_tokens), sb.suffixes[i:i + max_items])
            for i in range(0, len(sb.suffixes), max_items)]


def score_local(score_packed: Callable, requests: Sequence[SharedBatch], max_seq: int,
                max_tokens_per_launch: int = 1 << 17) -> list[np.ndarray]:
    """Pack several requests per launch (bounded by ``max_tokens_per_launch``) and return one
    p_yes vector per request, in order."""
    out: list[np.ndarray] = []
    batch: list[SharedBatch] = []
    tokens = 0

    def flush():
        if not batch:
            return
        res = score_packed(pack_requests(batch, max_seq))
        off = 0
        for sb in batch:
            out.append(np.asarray(res.p_yes[off:off + sb.n_items], dtype=np.float32))
            off += sb.n_items
        batch.clear()

    for sb in requests:
        t = request_tokens(sb)
        if batch and tokens + t > max_tokens_per_launch:
            flush()
            tokens = 0
        batch.append(sb)
        tokens += t
    flush()
    return out


class ReplicaGroup:
    """Request-sharded scoring across the ranks of a torch.distributed group."""

    def __init__(self, score_packed: Callable, max_seq: int = 2048, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.score_packed = score_packed
        self.max_seq = max_seq
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def score(self, requests: Sequence[SharedBatch] | None) -> list[np.ndarray] | None:
        """Collective over the group.  Rank 0 passes the requests (others pass None); rank 0 gets
        one p_yes vector per request in input order, other ranks get None."""
        dist = self.dist
        if self.rank == 0:
            reqs = list(requests)
            assign = assign_least_loaded([request_tokens(r) for r in reqs], self.world)
            shares = [[(i, reqs[i]) for i in idx] for idx in assign]
        else:
            shares = None
        mine = [None]
        dist.scatter_object_list(mine, shares, src=0, group=self.group)
        mine = mine[0]
        scores = score_local(self.score_packed, [sb for _, sb in mine], self.max_seq) if mine else []
        result = [(i, s) for (i, _), s in zip(mine, scores)]
        gathered = [None] * self.world if self.rank == 0 else None
        dist.gather_object(result, gathered, dst=0, group=self.group)
        if self.rank != 0:
            return None
        out: list = [None] * len(reqs)
        for part in gathered:
            for i, s in part:
                out[i] = s
        return out
