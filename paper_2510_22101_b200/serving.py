"""Serving wrapper around the B200 scoring path.

Reference: serving module, and the prompt contract of
corpus.py:10-31,74-89,302-345.  ``handle_score_request`` runs the spec's pipeline:

    shape_admit -> truncate candidates to the PID depth -> cache lookup per item ->
    assemble Eq-1 prompts for misses -> truncate descriptions to the token budget ->
    encode_batch (native C++ tokenizer) -> split_shared_prefix + pack (native) ->
    one pf_score call (prefix-shared batch scoring) -> cache fill -> merge and rank

Pinned choices the spec leaves open: cache key = (model_version,
FNV-1a-64(normalized query), item id) with normalization = lowercase + whitespace collapse; TTL is
write-time (hits refresh LRU position only); PID error signal
e = (target - observed)/target with gains (100, 10, 20) and anti-windup; the
shaper is a token bucket that defers but never drops.
"""

from __future__ import annotations

import time
from collections import OrderedDict
from dataclasses import asdict, dataclass, field
from typing import Callable, Sequence

import numpy as np

from . import ingest
from .scoring import rank_items

SYSTEM_PREFIX = "<|sys|>Decide if the job matches the query. Answer yes or no.<|/sys|>"
SUFFIX = "<|ans|>"


class PromptBudgetError(ValueError):
    """Token budget too small for the non-description prompt segments (corpus.py:44-45)."""


@dataclass(frozen=True)
class Query:
    id: str
    text: str


@dataclass(frozen=True)
class JobItem:
    id: str
    title: str
    company: str
    location: str
    employment_type: str
    remote_eligible: bool
    description: str


@dataclass(frozen=True)
class PromptSegments:
    system_prefix: str
    query_text: str
    metadata_text: str
    description_text: str
    suffix: str

    def full_prompt(self) -> str:
        return self.system_prefix + self.query_text + self.metadata_text + self.description_text + self.suffix


def assemble_prompt(query: Query, item: JobItem) -> PromptSegments:
    """Eq 1 (corpus.py:302-311)."""
    remote = "true" if item.remote_eligible else "false"
    return PromptSegments(
        SYSTEM_PREFIX, f"<|q|>{query.text}<|/q|>",
        f"<|meta|>{item.title}|{item.company}|{item.location}|{item.employment_type}|{remote}<|/meta|>",
        f"<|desc|>{item.description}<|/desc|>", SUFFIX)


def _spans(text: str, vocab: ingest.Vocab):
    import ctypes

    from . import _lib

    lib = _lib.load()
    raw = text.encode("utf-8", errors="surrogatepass")
    ids = np.empty(max(1, len(raw)), dtype=np.int32)
    ends = np.empty(max(1, len(raw)), dtype=np.int64)
    n = ctypes.c_int64()
    _lib.check(lib.pf_tokenize_spans(raw, len(raw), vocab.size, vocab.reserved, ids.ctypes.data,
                                     ends.ctypes.data, ids.size, ctypes.byref(n)))
    return ids[: n.value], ends[: n.value]


def truncate_description(seg: PromptSegments, token_budget: int, vocab: ingest.Vocab = ingest.DEFAULT_VOCAB
                         ) -> PromptSegments:
    """corpus.py:314-345: trim description words from the end until the prompt fits; other segments
    byte-identical; <|desc|> tags kept while any content remains."""
    enc = lambda s: ingest.encode(s, vocab)
    base = (len(enc(seg.system_prefix)) + len(enc(seg.query_text)) + len(enc(seg.metadata_text))
            + len(enc(seg.suffix)))
    if token_budget < base:
        raise PromptBudgetError(f"budget {token_budget} below non-description length {base}")
    desc_budget = token_budget - base
    if len(enc(seg.description_text)) <= desc_budget:
        return seg
    if desc_budget < 2:
        return PromptSegments(seg.system_prefix, seg.query_text, seg.metadata_text, "", seg.suffix)
    content = seg.description_text
    if not (content.startswith("<|desc|>") and content.endswith("<|/desc|>")):
        raise ValueError("truncate_description: malformed description segment")
    content = content[len("<|desc|>"):-len("<|/desc|>")]
    _, ends = _spans(content, vocab)
    keep = ends[: desc_budget - 2]
    kept = content[: int(keep[-1])] if len(keep) else ""
    return PromptSegments(seg.system_prefix, seg.query_text, seg.metadata_text, f"<|desc|>{kept}<|/desc|>",
                          seg.suffix)


def query_hash(text: str) -> int:
    """FNV-1a-64 of the normalized query text."""
    norm = " ".join(text.lower().split()).encode("utf-8")
    h = ingest.FNV_OFFSET
    for b in norm:
        h = ((h ^ b) * ingest.FNV_PRIME) & 0xFFFFFFFFFFFFFFFF
    return h


# ----------------------------------------------------------------------------- cache
class ScoreCache:
    """TTL + LRU score cache: never exceeds capacity; entries older than ttl are
    never returned; a hit refreshes the LRU position, not the TTL."""

    def __init__(self, capacity: int = 1_000_000, ttl: float = 900.0):
        if capacity < 1 or ttl < 0:
            raise ValueError("capacity >= 1 and ttl >= 0 required")
        self.capacity, self.ttl = capacity, ttl
        self._d: OrderedDict = OrderedDict()
        self.hits = self.misses = 0

    def lookup(self, key, now: float):
        v = self._d.get(key)
        if v is None:
            self.misses += 1
            return None
        p, t = v
        if now - t > self.ttl:
            del self._d[key]
            self.misses += 1
            return None
        self._d.move_to_end(key)
        self.hits += 1
        return p

    def insert(self, key, p_yes: float, now: float) -> None:
        self._d[key] = (float(p_yes), now)
        self._d.move_to_end(key)
        while len(self._d) > self.capacity:
            self._d.popitem(last=False)

    def __len__(self):
        return len(self._d)

    def stats(self) -> dict:
        tot = self.hits + self.misses
        return {"hits": self.hits, "misses": self.misses, "hit_rate": self.hits / tot if tot else 0.0}


# ----------------------------------------------------------------------------- PID depth
@dataclass
class PidController:
    """Scoring-depth controller."""

    depth: int = 250
    d_min: int = 50
    d_max: int = 1000
    kp: float = 100.0
    ki: float = 10.0
    kd: float = 20.0
    i_clamp: float = 100.0
    integral: float = 0.0
    e_prev: float = 0.0

    def update(self, observed_p95_ms: float, target_p95_ms: float, dt: float) -> int:
        if dt <= 0:
            raise ValueError("dt must be > 0")
        e = (target_p95_ms - observed_p95_ms) / target_p95_ms
        raw = self.depth + self.kp * e + self.ki * (self.integral + e * dt) + self.kd * (e - self.e_prev) / dt
        new = int(min(self.d_max, max(self.d_min, round(raw))))
        # anti-windup: freeze the integral while pushing against the active bound
        clamped = (raw > self.d_max and e > 0) or (raw < self.d_min and e < 0)
        if not clamped:
            self.integral = float(np.clip(self.integral + e * dt, -self.i_clamp, self.i_clamp))
        self.e_prev = e
        self.depth = new
        return new


# ----------------------------------------------------------------------------- shaper
@dataclass
class TokenBucketShaper:
    """Token bucket (rate R req/s, burst B) that defers admissions by at most max_defer and never
    drops."""

    rate: float
    burst: float
    max_defer: float
    level: float = field(default=None)
    t_last: float = field(default=None)
    deferred: int = 0
    total_defer: float = 0.0
    admitted: int = 0

    def __post_init__(self):
        if self.rate <= 0 or self.burst < 1 or self.max_defer < 0:
            raise ValueError("rate > 0, burst >= 1, max_defer >= 0 required")
        if self.level is None:
            self.level = float(self.burst)

    def admit(self, arrival: float) -> float:
        if self.t_last is not None and arrival < self.t_last:
            arrival_eff = self.t_last          # admissions are serialized through one queue
        else:
            arrival_eff = arrival
        if self.t_last is not None:
            self.level = min(self.burst, self.level + self.rate * (arrival_eff - self.t_last))
        self.t_last = arrival_eff
        if self.level >= 1.0:
            admit = arrival_eff
        else:
            t_tok = arrival_eff + (1.0 - self.level) / self.rate
            admit = min(t_tok, arrival + self.max_defer)
            self.level = min(self.burst, self.level + self.rate * (admit - arrival_eff))
            self.t_last = max(self.t_last, admit)
        self.level -= 1.0
        self.admitted += 1
        if admit > arrival:
            self.deferred += 1
            self.total_defer += admit - arrival
        return admit

    def stats(self) -> dict:
        return {"deferred": self.deferred,
                "mean_defer_ms": 1e3 * self.total_defer / self.deferred if self.deferred else 0.0}


# ----------------------------------------------------------------------------- service
@dataclass
class ScoreRequest:
    query: Query
    items: list
    request_id: str = ""
    arrival: float | None = None


@dataclass
class ScoreResponse:
    request_id: str
    depth_used: int
    scores: list            # [{"item_id", "p_yes", "source"}], descending p_yes, ties by item id
    timings_ms: dict
    unscored: list = field(default_factory=list)
    errors: list = field(default_factory=list)


class ScoringService:
    """handle_score_request with the spec's concurrency model.

    * ``submit(req) -> Future[ScoreResponse]`` never blocks the caller.  Admission goes through the
      token-bucket shaper under one lock (the spec's "serializes admissions through one queue");
      a deferred request waits in a timer queue served by one admission thread, not in a handler.
    * Admitted requests run on a pool of ``workers`` handler threads: PID depth, cache lookups,
      Eq-1 assembly, truncation, native tokenization and packing.  The packed request then goes to
      the scorer: a ``ReplicaPool`` (asynchronous, batched and pipelined across GPU replicas) or
      any object with ``score_packed(PackedBatch) -> ScoredBatch`` (called on the handler thread).
    * The cache is guarded by one lock (a lookup moves the LRU position, so reads write too).
    * One metrics loop owns the PID: every ``pid_interval`` s it feeds the p95 latency of the
      requests completed in the last ``window_s`` s to ``PidController.update``;
      handlers read ``pid.depth`` (an int, read atomically).
    * ``handle_score_request(req)`` is the synchronous form: ``submit(req).result()``.

    Cache tolerance ("a hit returns exactly the value the model would produce"): a
    device score depends on its item's prompt only up to bf16 rounding of how the co-batched items
    split the shared prefix, so a fresh score may differ from a cached one in the low bits.  With
    ``shadow_rate`` > 0 (test mode) that fraction of hits is re-scored with the misses and the
    difference is checked against ``shadow_tol`` (1e-2, the parity contract); ``metrics()``
    reports the checks."""

    def __init__(self, scorer, model_version: str, vocab: ingest.Vocab = ingest.DEFAULT_VOCAB,
                 cache: ScoreCache | None = None, pid: PidController | None = None,
                 shaper: TokenBucketShaper | None = None, token_budget: int = 2048, max_seq: int = 2048,
                 clock: Callable[[], float] = time.monotonic, workers: int = 8, target_p95_ms: float = 500.0,
                 pid_interval: float = 1.0, window_s: float = 10.0, shadow_rate: float = 0.0,
                 shadow_tol: float = 1e-2, model_config=None, seed: int = 0):
        import threading

        self.scorer, self.model_version, self.vocab = scorer, model_version, vocab
        self.cache = cache if cache is not None else ScoreCache()
        self.pid, self.shaper = pid, shaper
        self.token_budget, self.max_seq, self.clock = token_budget, max_seq, clock
        self.workers, self.target_p95_ms = int(workers), float(target_p95_ms)
        self.pid_interval, self.window_s = float(pid_interval), float(window_s)
        self.shadow_rate, self.shadow_tol = float(shadow_rate), float(shadow_tol)
        self.model_config = model_config if model_config is not None else getattr(scorer, "config", None)
        self._rng = np.random.default_rng(seed)
        self.model_calls = self.items_scored = 0
        self._flops_shared = self._flops_indep = 0.0
        self._shadow = {"checked": 0, "max_abs_diff": 0.0, "violations": 0}
        self._lock = threading.Lock()          # cache, counters, latency log
        self._adm_lock = threading.Lock()      # shaper: admissions serialized
        self._lat: list = []                   # (t_done, total_ms) of completed requests
        self._item_log: list = []              # (t_done, n_items scored by the model)
        self._pool = None
        self._timer = None
        self._metrics_thread = None
        self._closed = False

    # ------------------------------------------------------------------ threads
    def _ensure_threads(self):
        import heapq
        import threading
        from concurrent.futures import ThreadPoolExecutor

        if self._pool is not None:
            return
        with self._adm_lock:
            if self._pool is not None:
                return
            self._heap: list = []
            self._heap_cv = threading.Condition()
            self._heapq = heapq

            def admission_loop():
                while True:
                    with self._heap_cv:
                        while not self._heap and not self._closed:
                            self._heap_cv.wait()
                        if self._closed and not self._heap:
                            return
                        t_adm, k, item = self._heap[0]
                        wait = t_adm - self.clock()
                        if wait > 0:
                            self._heap_cv.wait(timeout=wait)
                            continue
                        heapq.heappop(self._heap)
                    self._pool.submit(self._run, *item)

            self._timer = threading.Thread(target=admission_loop, name="shaper-admission", daemon=True)
            self._pool = ThreadPoolExecutor(max_workers=self.workers, thread_name_prefix="score-handler")
            self._timer.start()
            if self.pid is not None and self.pid_interval > 0:
                self._metrics_thread = threading.Thread(target=self._metrics_loop, name="metrics-pid", daemon=True)
                self._metrics_thread.start()

    def close(self):
        self._closed = True
        if self._pool is not None:
            with self._heap_cv:
                self._heap_cv.notify_all()
            self._timer.join(timeout=5)
            self._pool.shutdown(wait=True)
            if self._metrics_thread is not None:
                self._metrics_thread.join(timeout=5)

    def _metrics_loop(self):
        t_prev = self.clock()
        while not self._closed:
            time.sleep(self.pid_interval)
            now = self.clock()
            p95 = self.p95_ms(now)
            if p95 is not None:
                self.pid.update(p95, self.target_p95_ms, max(now - t_prev, 1e-6))
            t_prev = now

    # ------------------------------------------------------------------ request path
    def submit(self, req: ScoreRequest):
        from concurrent.futures import Future

        self._ensure_threads()
        fut: Future = Future()
        t0 = self.clock()
        arrival = req.arrival if req.arrival is not None else t0
        with self._adm_lock:
            admit = self.shaper.admit(arrival) if self.shaper else arrival
        if admit > self.clock():
            with self._heap_cv:
                self._heapq.heappush(self._heap, (admit, id(fut), (req, t0, arrival, fut)))
                self._heap_cv.notify()
        else:
            self._pool.submit(self._run, req, t0, arrival, fut)
        return fut

    def handle_score_request(self, req: ScoreRequest) -> ScoreResponse:
        return self.submit(req).result()

    def _run(self, req, t0, arrival, fut):
        try:
            self._prepare(req, t0, arrival, fut)
        except BaseException as e:       # pragma: no cover - surfaced to the caller
            if not fut.done():
                fut.set_exception(e)

    def _prepare(self, req, t0, arrival, fut):
        t_admit = self.clock()
        depth = self.pid.depth if self.pid else len(req.items)
        cands, unscored = list(req.items[:depth]), [it.id for it in req.items[depth:]]
        qh = query_hash(req.query.text)
        scores, misses, errors, shadow = {}, [], [], []
        with self._lock:
            for it in cands:
                p = self.cache.lookup((self.model_version, qh, it.id), t_admit)
                if p is None:
                    misses.append(it)
                else:
                    scores[it.id] = (p, "cache")
                    if self.shadow_rate > 0 and self._rng.random() < self.shadow_rate:
                        shadow.append(it)
        ctx = {"req": req, "t0": t0, "arrival": arrival, "t_admit": t_admit, "depth": depth, "qh": qh,
               "scores": scores, "unscored": unscored, "errors": errors, "ok": [], "shadow": 0,
               "t_tok": 0.0, "t_pre0": None}
        to_score = misses + shadow
        if not to_score:
            self._respond(ctx, None, fut)
            return
        t1 = self.clock()
        ids, offs, ok = self._tokenize(req.query, to_score, errors)
        n_shadow = sum(1 for it in ok if it in shadow)
        ctx["ok"], ctx["shadow"] = ok, n_shadow
        t2 = self.clock()
        ctx["t_tok"], ctx["t_pre0"] = t2 - t1, t2
        if not ok:
            self._respond(ctx, None, fut)
            return
        if hasattr(self.scorer, "submit_token_arrays"):      # ReplicaPool: sharded, asynchronous
            ctx["flops"] = self._work_flops_arrays(ids, offs)
            inner = self.scorer.submit_token_arrays(ids, offs)
            inner.add_done_callback(lambda f: self._after_model(ctx, f, fut))
        else:
            packed = ingest.pack_flat_native(ids, offs, None, self.max_seq)
            ctx["flops"] = self._work_flops(packed)
            res = self.scorer.score_packed(packed)
            self._respond(ctx, res, fut)

    def _tokenize(self, query: Query, items: list, errors: list):
        """Eq-1 prompts of ``items`` -> (flat ids, offsets, items kept), tokenized in one native batch.
        Segments begin and end with tags, so a prompt's token count is the sum of its segments'
        counts: a prompt within the budget is exactly what truncate_description would return
        unchanged, and only over-budget prompts take the per-item truncation path (corpus.py:314-345)."""
        prompts = [assemble_prompt(query, it).full_prompt() for it in items]
        ids, offs = ingest.encode_batch_arrays(prompts, self.vocab)
        lens = np.diff(offs)
        over = np.nonzero(lens > self.token_budget)[0]
        if len(over) == 0:
            return ids, offs, list(items)
        keep, fixed = [], {}
        for i in over:
            try:
                fixed[int(i)] = truncate_description(assemble_prompt(query, items[i]), self.token_budget,
                                                     self.vocab).full_prompt()
            except PromptBudgetError as e:          # per-item rejection
                errors.append({"item_id": items[i].id, "error": str(e)})
                fixed[int(i)] = None
        for i in range(len(items)):
            if fixed.get(i, "") is not None:
                keep.append(i)
        prompts = [fixed.get(i) or prompts[i] for i in keep]
        if not prompts:
            return ids[:0], np.zeros(1, np.int64), []
        ids, offs = ingest.encode_batch_arrays(prompts, self.vocab)
        return ids, offs, [items[i] for i in keep]

    def _after_model(self, ctx, f, fut):
        try:
            res = f.result()
        except BaseException as e:
            fut.set_exception(e)
            return
        try:
            self._respond(ctx, res, fut)
        except BaseException as e:       # pragma: no cover
            fut.set_exception(e)

    def _work_flops(self, packed):
        cfg = self.model_config
        if cfg is None:
            return None
        from .prefixcache import request_flops

        P = int(packed.prefix_lens[0])
        return (request_flops(cfg, P, packed.suffix_lens, True), request_flops(cfg, P, packed.suffix_lens, False))

    def _work_flops_arrays(self, ids, offs):
        """(shared, independent) FLOPs of one request from its flat prompt tokens: the LCP of the
        prompts is the shared prefix (split_shared_prefix rule)."""
        cfg = self.model_config
        if cfg is None:
            return None
        from .prefixcache import request_flops

        lens = np.diff(offs)
        first = ids[offs[0]:offs[1]]
        P = len(first)
        for i in range(1, len(lens)):
            row = ids[offs[i]:offs[i + 1]]
            n = min(P, len(row))
            neq = np.nonzero(first[:n] != row[:n])[0]
            P = int(neq[0]) if len(neq) else n
        if (lens == P).any():
            P -= 1
        return (request_flops(cfg, P, lens - P, True), request_flops(cfg, P, lens - P, False))

    def _respond(self, ctx, res, fut):
        req, scores = ctx["req"], ctx["scores"]
        now = self.clock()
        t_pre = (now - ctx["t_pre0"]) if ctx["t_pre0"] is not None else 0.0
        with self._lock:
            if res is not None:
                self.model_calls += 1
                n_model = len(ctx["ok"]) - ctx["shadow"]
                self.items_scored += n_model
                self._item_log.append((now, n_model))
                fl = ctx.get("flops")
                if fl is not None:
                    self._flops_shared += fl[0]
                    self._flops_indep += fl[1]
                for it, p in zip(ctx["ok"], res.p_yes):
                    p = float(p)
                    if it.id in scores:                       # shadow re-score of a cache hit
                        diff = abs(p - scores[it.id][0])
                        self._shadow["checked"] += 1
                        self._shadow["max_abs_diff"] = max(self._shadow["max_abs_diff"], diff)
                        self._shadow["violations"] += int(diff > self.shadow_tol)
                        continue
                    scores[it.id] = (p, "model")
                    self.cache.insert((self.model_version, ctx["qh"], it.id), p, now)
        ids = list(scores.keys())
        out = []
        if ids:
            ranked = rank_items([scores[i][0] for i in ids], ids)
            out = [{"item_id": i, "p_yes": p, "source": scores[i][1]} for i, p in zip(ranked.item_ids, ranked.scores)]
        t_end = self.clock()
        arrival = ctx["arrival"]
        total = 1e3 * (t_end - (arrival if req.arrival is not None else ctx["t0"]))
        resp = ScoreResponse(req.request_id, ctx["depth"], out,
                             {"queue": 1e3 * (ctx["t_admit"] - (arrival if req.arrival is not None else ctx["t0"])),
                              "tokenize": 1e3 * ctx["t_tok"], "prefill": 1e3 * t_pre, "total": total},
                             ctx["unscored"], ctx["errors"])
        with self._lock:
            self._lat.append((t_end, total))
        fut.set_result(resp)

    # ------------------------------------------------------------------ metrics
    def _prune(self, now):
        lo = now - self.window_s
        while self._lat and self._lat[0][0] < lo:
            self._lat.pop(0)
        while self._item_log and self._item_log[0][0] < lo:
            self._item_log.pop(0)

    def p95_ms(self, now: float | None = None):
        """Nearest-rank p95 of request latency over the sliding window."""
        now = self.clock() if now is None else now
        with self._lock:
            self._prune(now)
            lat = sorted(x for _, x in self._lat)
        if not lat:
            return None
        return lat[max(1, int(np.ceil(0.95 * len(lat)))) - 1]

    def metrics(self) -> dict:
        """GET /v1/metrics shape."""
        now = self.clock()
        p95 = self.p95_ms(now)
        with self._lock:
            items_window = sum(n for _, n in self._item_log)
            saved = (100.0 * (1.0 - self._flops_shared / self._flops_indep)) if self._flops_indep > 0 else 0.0
            return {"cache": self.cache.stats(),
                    "pid": {"depth": self.pid.depth if self.pid else None, "p95_ms": p95},
                    "shaper": self.shaper.stats() if self.shaper else {"deferred": 0, "mean_defer_ms": 0.0},
                    "engine": {"items_per_sec": items_window / self.window_s if self._item_log else 0.0,
                               "flops_saved_pct": saved, "model_calls": self.model_calls,
                               "items_scored": self.items_scored},
                    "shadow": dict(self._shadow)}
