"""Oracle restatement of the reference ``prefixcache`` module and of the flat
packed layout the device consumes.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import model as M


@dataclass
class SharedBatch:
    prefix_tokens: list
    suffixes: list
    prefix_kv: object = None


def split_shared_prefix(token_lists) -> SharedBatch:
    """SPEC.md:255-263.  Longest common prefix; boundary moved one token left if any suffix would
    be empty; empty batch is an error."""
    if not token_lists:
        raise ValueError("empty batch")
    lists = [list(t) for t in token_lists]
    if any(len(t) == 0 for t in lists):
        raise ValueError("all lists must be non-empty")
    n = 0
    shortest = min(len(t) for t in lists)
    while n < shortest and all(t[n] == lists[0][n] for t in lists):
        n += 1
    if any(len(t) == n for t in lists):
        n -= 1
    return SharedBatch(lists[0][:n], [t[n:] for t in lists])


def throughput_gain(n_query_tokens, n_item_tokens) -> float:
    """T = 1 + N_q / N_i."""
    if n_item_tokens <= 0:
        raise ValueError("zero item tokens")
    return 1.0 + n_query_tokens / n_item_tokens


def score_shared_batch(W: M.OracleWeights, shared: SharedBatch, eps: float = 1e-6):
    """one prefix prefill populates prefix_kv; each suffix via
    forward_with_prefix (LSE merge inside).  Returns list of [vocab] logit vectors."""
    if len(shared.prefix_tokens) > 0:
        _, kv = M.forward_prefill(W, shared.prefix_tokens, eps)
        shared.prefix_kv = kv
    else:
        kv = None
    out = []
    for s in shared.suffixes:
        if kv is None:
            logits, _ = M.forward_prefill(W, s, eps)
        else:
            logits, _ = M.forward_with_prefix(W, kv, s, eps)
        out.append(logits)
    return out


def pack(batches, max_seq: int = 2048):
    """Flat varlen layout, restated: per request prefix rows then each suffix's
    rows; positions prefix 0..P-1 and P..P+S-1 for every suffix; segments
    {kv_off, kv_len, q_off, q_len}; last_idx = last row of each suffix."""
    ids, pos, segs, last = [], [], [], []
    row = 0
    for sb in batches:
        P = len(sb.prefix_tokens)
        base = row
        if P:
            ids += list(sb.prefix_tokens)
            pos += list(range(P))
            segs.append([base, 0, base, P])
            row += P
        for s in sb.suffixes:
            if len(s) == 0 or P + len(s) > max_seq:
                raise ValueError("bad suffix length")
            ids += list(s)
            pos += list(range(P, P + len(s)))
            segs.append([base, P, row, len(s)])
            row += len(s)
            last.append(row - 1)
    return (np.asarray(ids, dtype=np.int32), np.asarray(pos, dtype=np.int32),
            np.asarray(segs, dtype=np.int32).reshape(-1, 4), np.asarray(last, dtype=np.int32))
