"""Oracle restatement of the reference ``scoring`` module.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""

from __future__ import annotations

import math

import numpy as np


def relevance_score(logits, yes_id: int = 1, no_id: int = 2):
    """Eq 2: 2-way softmax over (logits[yes], logits[no]) -> (p_yes, p_no)."""
    a, b = float(logits[yes_id]), float(logits[no_id])
    if not (math.isfinite(a) and math.isfinite(b)):
        raise ValueError("non-finite logits")
    m = max(a, b)
    ea, eb = math.exp(a - m), math.exp(b - m)
    return ea / (ea + eb), eb / (ea + eb)


def rank_items(p_yes, item_ids=None):
    """stable sort, p_yes descending, ties by ascending item id."""
    ids = list(range(len(p_yes))) if item_ids is None else list(item_ids)
    return [ids[i] for i in sorted(range(len(p_yes)), key=lambda i: (-float(p_yes[i]), ids[i]))]


def near_tie_pairs(p_yes, k: int, gap: float) -> int:
    """Number of adjacent pairs within the oracle's top-(k+1) whose score gap is below ``gap``
    (declared near-ties for the template-faithful parity family)."""
    order = rank_items(p_yes)
    top = [float(p_yes[i]) for i in order[: k + 1]]
    return sum(1 for a, b in zip(top, top[1:]) if abs(a - b) < gap)


def topk_equal_modulo_ties(p_ref, p_test, k: int, gap: float) -> bool:
    """Top-k identical after treating oracle near-ties (|Δ| < gap) as unordered: the oracle's
    top-k, grouped into runs of near-tied scores, must map onto the test's top-k with the same
    group sequence."""
    ref_order = rank_items(p_ref)
    test_order = rank_items(p_test)
    p_ref = np.asarray(p_ref, dtype=np.float64)
    # the item at test position j must be near-tied with the oracle item at position j
    for j in range(min(k, len(ref_order))):
        if abs(p_ref[test_order[j]] - p_ref[ref_order[j]]) >= gap:
            return False
    return True
