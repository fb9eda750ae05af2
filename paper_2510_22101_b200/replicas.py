"""Replica pool: one worker thread per GPU replica, batching and pipelining packed requests.

SURVEY.md §8e (replicas only, no collective) and the serving module's concurrency model
("processes requests concurrently up to a worker-pool limit ... model
weights are immutable and shared").  One process drives every local GPU: each replica is a
``PrefillScorer`` on its own device with its own CUDA stream, served by one host thread.  The
ctypes calls into libprefill_sm100.so and the stream synchronisations release the GIL, so the
threads overlap host work (joining packed requests, pinned copies, splitting results) with the
forwards of every device.

* ``submit(packed)`` -> Future[ScoredBatch] for one request (already split + packed on the caller's
  thread).  Requests larger than ``max_shard_items`` are item-split into shards that may land on
  different replicas (each shard recomputes the short prefix); the future resolves
  when every shard is back, with scores in the request's item order.
* Dispatch: the replica with the fewest outstanding tokens (ties: lowest index).
* Sharding (``submit_token_arrays``): a request is item-split into shards of at most
  ``shard_tokens`` tokens, and into at least one shard per replica when it has enough items, so a
  large request runs on every replica at once and no launch grows past the budget; shards complete
  into one future in item order.
* Each worker coalesces queued jobs, up to ``token_budget`` tokens, into one ``pf_score`` launch
  (``concat_packed``), oldest first (``policy="fifo"``; "sjf" = smallest first), and keeps up to
  two launches in flight: while the device runs launch k, the thread joins and enqueues launch k+1
  (H2D from pinned memory on the same stream), then waits for k and hands its scores out.
"""

from __future__ import annotations

import threading
import time
from concurrent.futures import Future
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from .prefixcache import PackedBatch, SharedBatch, concat_packed, pack_requests


@dataclass
class _Job:
    packed: PackedBatch
    future: Future
    tokens: int
    seq: int
    t_submit: float = field(default_factory=time.perf_counter)


class _Shards:
    """Joins the shard results of one item-split request."""

    def __init__(self, n_shards: int, sizes: list[int], future: Future):
        self.left = n_shards
        self.parts: list = [None] * n_shards
        self.sizes = sizes
        self.future = future
        self.lock = threading.Lock()

    def done(self, k: int, fut: Future):
        from .engine import ScoredBatch

        try:
            res = fut.result()
        except BaseException as e:            # first failure fails the request
            if not self.future.done():
                self.future.set_exception(e)
            return
        with self.lock:
            self.parts[k] = res
            self.left -= 1
            last = self.left == 0
        if last and not self.future.done():
            self.future.set_result(ScoredBatch(np.concatenate([p.logits2 for p in self.parts]),
                                               np.concatenate([p.p_yes for p in self.parts])))


class ReplicaWorker(threading.Thread):
    """Serves one PrefillScorer: a queue of packed jobs -> batched, pipelined pf_score launches."""

    def __init__(self, scorer, token_budget: int = 1 << 18, name: str | None = None, policy: str = "fifo"):
        import torch

        super().__init__(name=name or f"replica-{scorer.device}", daemon=True)
        if policy not in ("fifo", "sjf"):
            raise ValueError("policy must be 'fifo' or 'sjf'")
        self.scorer = scorer
        self.token_budget = int(token_budget)
        self.policy = policy
        with torch.cuda.device(scorer.device):
            self.stream = torch.cuda.Stream(scorer.device)
        self._jobs: list[_Job] = []
        self._cv = threading.Condition()
        self._stopping = False
        self.outstanding_tokens = 0
        self.launches = 0
        self.items_scored = 0
        self.busy_s = 0.0

    # ------------------------------------------------------------------ queue
    def enqueue(self, job: _Job) -> None:
        with self._cv:
            if self._stopping:
                raise RuntimeError("replica worker stopped")
            self._jobs.append(job)
            self.outstanding_tokens += job.tokens
            self._cv.notify()

    def stop(self) -> None:
        with self._cv:
            self._stopping = True
            self._cv.notify()

    def _take(self, block: bool) -> list[_Job]:
        """Pending jobs in policy order (oldest or smallest first), up to the token budget (always
        at least one job)."""
        with self._cv:
            while block and not self._jobs and not self._stopping:
                self._cv.wait()
            if not self._jobs:
                return []
            if self.policy == "sjf":
                self._jobs.sort(key=lambda j: (j.tokens, j.seq))
            else:
                self._jobs.sort(key=lambda j: j.seq)
            batch, toks = [], 0
            while self._jobs and (not batch or toks + self._jobs[0].tokens <= self.token_budget):
                j = self._jobs.pop(0)
                batch.append(j)
                toks += j.tokens
            return batch

    # ------------------------------------------------------------------ device side
    def _launch(self, jobs: list[_Job]):
        """Join the jobs, copy them in from pinned memory and enqueue the forward and the score
        copy-out on this replica's stream.  Returns the in-flight record."""
        import torch

        from .engine import DevicePacked

        sc = self.scorer
        packed = concat_packed([j.packed for j in jobs])
        sc.validate(packed)
        n = packed.n_items
        with torch.cuda.device(sc.device), torch.cuda.stream(self.stream):
            pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            host = [pin(packed.ids), pin(packed.pos), pin(packed.segs), pin(packed.work), pin(packed.last_idx)]
            dev = [h.to(sc.device, non_blocking=True) for h in host]
            dp = DevicePacked.__new__(DevicePacked)
            dp.packed = packed
            dp.ids, dp.pos, dp.segs, dp.work, dp.last_idx = dev
            logits2, p_yes = sc.score_device(dp, stream=self.stream)
            out_l = torch.empty((n, 2), dtype=torch.float32).pin_memory()
            out_p = torch.empty((n,), dtype=torch.float32).pin_memory()
            out_l.copy_(logits2, non_blocking=True)
            out_p.copy_(p_yes, non_blocking=True)
            bad = torch.empty(1, dtype=torch.int32).pin_memory()
            bad.copy_(sc.bad_flag(self.stream)[:1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.stream)
        return (jobs, packed, ev, out_l, out_p, bad, host, dev, time.perf_counter())

    def _finish(self, rec) -> None:
        from .engine import ScoredBatch

        jobs, packed, ev, out_l, out_p, bad, _, _, t0 = rec
        ev.synchronize()
        self.busy_s += time.perf_counter() - t0
        self.launches += 1
        self.items_scored += packed.n_items
        with self._cv:
            self.outstanding_tokens -= sum(j.tokens for j in jobs)
        if int(bad[0]) != 0:
            err = ValueError("relevance_score: non-finite logits (SPEC.md:330)")
            for j in jobs:
                j.future.set_exception(err)
            return
        lg, py = out_l.numpy(), out_p.numpy()
        off = 0
        for j in jobs:
            n = j.packed.n_items
            j.future.set_result(ScoredBatch(lg[off:off + n].copy(), py[off:off + n].copy()))
            off += n

    def run(self) -> None:
        inflight = None
        while True:
            jobs = self._take(block=inflight is None)
            if not jobs and inflight is None:
                if self._stopping:
                    return
                continue
            nxt = None
            if jobs:
                try:
                    nxt = self._launch(jobs)
                except BaseException as e:     # a bad batch fails its own jobs only
                    with self._cv:
                        self.outstanding_tokens -= sum(j.tokens for j in jobs)
                    for j in jobs:
                        j.future.set_exception(e)
            if inflight is not None:
                try:
                    self._finish(inflight)
                except BaseException as e:
                    for j in inflight[0]:
                        if not j.future.done():
                            j.future.set_exception(e)
            inflight = nxt


class ReplicaPool:
    """Request-sharded scoring over local GPU replicas: no collective, one host
    thread per replica, scores gathered host-side in request order."""

    def __init__(self, scorers: Sequence, token_budget: int = 1 << 18, max_shard_items: int | None = None,
                 shard_tokens: int = 1 << 16, min_shard_items: int = 8, policy: str = "fifo"):
        if not scorers:
            raise ValueError("ReplicaPool: need >= 1 scorer")
        self.workers = [ReplicaWorker(s, token_budget, policy=policy) for s in scorers]
        self.shard_tokens, self.min_shard_items = int(shard_tokens), int(min_shard_items)
        self.max_seq = scorers[0].config.max_seq
        self.config = scorers[0].config
        # default: split so a request can spread over every replica once it is larger than ~1 launch
        self.max_shard_items = max_shard_items
        self._seq = 0
        self._lock = threading.Lock()
        for w in self.workers:
            w.start()

    @classmethod
    def from_weights(cls, weights_factory, devices: Sequence, **kw) -> "ReplicaPool":
        """One replica per device; ``weights_factory(device)`` returns its DeviceWeights."""
        from .engine import PrefillScorer

        return cls([PrefillScorer(weights_factory(d), d) for d in devices], **kw)

    def __len__(self) -> int:
        return len(self.workers)

    def _pick(self) -> ReplicaWorker:
        return min(self.workers, key=lambda w: (w.outstanding_tokens, self.workers.index(w)))

    def _enqueue(self, packed: PackedBatch) -> Future:
        fut: Future = Future()
        with self._lock:
            self._seq += 1
            seq = self._seq
            w = self._pick()
            w.enqueue(_Job(packed, fut, packed.T, seq))
        return fut

    def submit_shared(self, sb: SharedBatch) -> Future:
        """Score one request; item-split across replicas when it exceeds ``max_shard_items``."""
        k = self.max_shard_items
        if k is None or sb.n_items <= k or len(self.workers) == 1:
            return self._enqueue(pack_requests([sb], self.max_seq))
        n_sh = -(-sb.n_items // k)
        # balance the shards: equal item counts, at most one more
        bounds = np.linspace(0, sb.n_items, n_sh + 1).round().astype(int)
        shards = [SharedBatch(list(sb.prefix_tokens), sb.suffixes[a:b]) for a, b in zip(bounds, bounds[1:])]
        return self.submit_shards([pack_requests([s], self.max_seq) for s in shards])

    def submit_packed(self, packed: PackedBatch) -> Future:
        return self._enqueue(packed)

    def shard_bounds(self, item_tokens: np.ndarray) -> list[tuple[int, int]]:
        """Item ranges of the shards of one request (see the module docstring)."""
        n = len(item_tokens)
        total = int(np.sum(item_tokens))
        k = max(1, -(-total // self.shard_tokens))
        k = max(k, min(len(self.workers), n // max(1, self.min_shard_items)))
        k = min(k, n)
        if k == 1:
            return [(0, n)]
        # cut at equal token quantiles (balanced shard cost)
        cum = np.cumsum(item_tokens)
        cuts = np.searchsorted(cum, total * np.arange(1, k) / k, side="left") + 1
        b = [0] + sorted(set(int(c) for c in cuts if 0 < c < n)) + [n]
        return list(zip(b[:-1], b[1:]))

    def submit_token_arrays(self, ids: np.ndarray, offsets: np.ndarray) -> Future:
        """One request given as its items' full prompts (flat token ids + offsets, what
        ingest.encode_batch_arrays returns): sharded, packed natively (LCP split per shard) and
        scored; the future holds the request's ScoredBatch in item order."""
        from . import ingest

        offsets = np.asarray(offsets, dtype=np.int64)
        bounds = self.shard_bounds(np.diff(offsets))
        shards = []
        for a, b in bounds:
            sub = offsets[a:b + 1] - offsets[a]
            shards.append(ingest.pack_flat_native(ids[offsets[a]:offsets[b]], sub, None, self.max_seq))
        return self.submit_shards(shards)

    def submit_shards(self, shards: Sequence[PackedBatch]) -> Future:
        fut: Future = Future()
        if len(shards) == 1:
            return self._enqueue(shards[0])
        join = _Shards(len(shards), [s.n_items for s in shards], fut)
        for i, s in enumerate(shards):
            self._enqueue(s).add_done_callback(lambda f, i=i: join.done(i, f))
        return fut

    def score_packed(self, packed: PackedBatch):
        """Synchronous form (the ScoringService scorer protocol)."""
        return self._enqueue(packed).result()

    def stats(self) -> dict:
        return {"replicas": len(self.workers),
                "launches": [w.launches for w in self.workers],
                "items_scored": [w.items_scored for w in self.workers],
                "busy_s": [round(w.busy_s, 3) for w in self.workers]}

    def close(self) -> None:
        for w in self.workers:
            w.stop()
        for w in self.workers:
            w.join(timeout=10)
