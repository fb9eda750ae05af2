"""Relevance scoring (Eq 2) and ranking — reference scoring module.

``relevance_score`` accepts either a full [vocab] logit vector (the spec's form) or the
2-logit (yes, no) view the B200 path returns (north_star: full-vocab logits are never formed).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np


@dataclass(frozen=True)
class RelevanceScore:
    p_yes: float
    p_no: float


def _sigmoid(x: float) -> float:
    if x >= 0:
        return 1.0 / (1.0 + math.exp(-x))
    e = math.exp(x)
    return e / (1.0 + e)


def relevance_score(logits, vocab=None, *, yes_id: int | None = None, no_id: int | None = None) -> RelevanceScore:
    """Two-way softmax over (logits[yes_id], logits[no_id]) == sigmoid(l_yes - l_no)
    (SPEC.md:326-334, :366).  ``vocab`` supplies yes_id/no_id (reference Vocab or ModelConfig);
    a length-2 input is read as (logit_yes, logit_no)."""
    arr = np.asarray(logits, dtype=np.float64).reshape(-1)
    if arr.shape[0] == 2:
        ly, ln = float(arr[0]), float(arr[1])
    else:
        y = yes_id if yes_id is not None else getattr(vocab, "yes_id", 1)
        n = no_id if no_id is not None else getattr(vocab, "no_id", 2)
        ly, ln = float(arr[y]), float(arr[n])
    if not (math.isfinite(ly) and math.isfinite(ln)):
        raise ValueError("relevance_score: non-finite logits")
    p = _sigmoid(ly - ln)
    return RelevanceScore(p_yes=p, p_no=1.0 - p)


@dataclass(frozen=True)
class RankedList:
    item_ids: list
    scores: list


def rank_items(scores: Sequence[float], item_ids: Sequence | None = None) -> RankedList:
    """Stable sort by p_yes descending, ties by ascending item id."""
    if len(scores) == 0:
        raise ValueError("rank_items: need >= 1 item")
    ids = list(range(len(scores))) if item_ids is None else list(item_ids)
    order = sorted(range(len(scores)), key=lambda i: (-float(scores[i]), ids[i]))
    return RankedList([ids[i] for i in order], [float(scores[i]) for i in order])


def top_k(scores: Sequence[float], k: int = 10, item_ids: Sequence | None = None) -> list:
    return rank_items(scores, item_ids).item_ids[:k]
