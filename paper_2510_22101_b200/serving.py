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
    """handle_score_request over a device scorer (``score_packed(PackedBatch) ->
    ScoredBatch``: a PrefillScorer, or a dispatcher over several replicas)."""

    def __init__(self, scorer, model_version: str, vocab: ingest.Vocab = ingest.DEFAULT_VOCAB,
                 cache: ScoreCache | None = None, pid: PidController | None = None,
                 shaper: TokenBucketShaper | None = None, token_budget: int = 2048, max_seq: int = 2048,
                 clock: Callable[[], float] = time.monotonic):
        self.scorer, self.model_version, self.vocab = scorer, model_version, vocab
        self.cache = cache if cache is not None else ScoreCache()
        self.pid, self.shaper = pid, shaper
        self.token_budget, self.max_seq, self.clock = token_budget, max_seq, clock
        self.model_calls = self.items_scored = 0

    def handle_score_request(self, req: ScoreRequest) -> ScoreResponse:
        t0 = self.clock()
        arrival = req.arrival if req.arrival is not None else t0
        admit = self.shaper.admit(arrival) if self.shaper else arrival
        if admit > t0:
            time.sleep(admit - t0)
        t_admit = self.clock()
        depth = self.pid.depth if self.pid else len(req.items)
        cands, unscored = list(req.items[:depth]), [it.id for it in req.items[depth:]]
        qh = query_hash(req.query.text)
        scores, misses, errors = {}, [], []
        for it in cands:
            p = self.cache.lookup((self.model_version, qh, it.id), t_admit)
            if p is None:
                misses.append(it)
            else:
                scores[it.id] = (p, "cache")
        t_tok = t_pre = 0.0
        if misses:
            t1 = self.clock()
            prompts, ok = [], []
            for it in misses:
                try:
                    prompts.append(truncate_description(assemble_prompt(req.query, it), self.token_budget,
                                                        self.vocab).full_prompt())
                    ok.append(it)
                except PromptBudgetError as e:          # per-item rejection
                    errors.append({"item_id": it.id, "error": str(e)})
            token_lists = ingest.encode_batch(prompts, self.vocab) if prompts else []
            t2 = self.clock()
            t_tok = t2 - t1
            if token_lists:
                packed = ingest.pack_token_lists_native([token_lists], self.max_seq)
                res = self.scorer.score_packed(packed)
                self.model_calls += 1
                self.items_scored += len(ok)
                now = self.clock()
                for it, p in zip(ok, res.p_yes):
                    scores[it.id] = (float(p), "model")
                    self.cache.insert((self.model_version, qh, it.id), float(p), now)
            t_pre = self.clock() - t2
        ids = list(scores.keys())
        out = []
        if ids:
            ranked = rank_items([scores[i][0] for i in ids], ids)
            out = [{"item_id": i, "p_yes": p, "source": scores[i][1]} for i, p in zip(ranked.item_ids, ranked.scores)]
        t_end = self.clock()
        return ScoreResponse(req.request_id, depth, out,
                             {"queue": 1e3 * (t_admit - arrival) if req.arrival is not None else 1e3 * (t_admit - t0),
                              "tokenize": 1e3 * t_tok, "prefill": 1e3 * t_pre, "total": 1e3 * (t_end - t0)},
                             unscored, errors)

    def metrics(self) -> dict:
        """GET /v1/metrics shape."""
        return {"cache": self.cache.stats(),
                "pid": {"depth": self.pid.depth if self.pid else None},
                "shaper": self.shaper.stats() if self.shaper else {"deferred": 0, "mean_defer_ms": 0.0},
                "engine": {"model_calls": self.model_calls, "items_scored": self.items_scored}}
