"""In-batch prefix sharing: the LCP split and the varlen packer (no padding).

Reference: prefixcache module.

* ``split_shared_prefix`` — SPEC.md:255-263: prefix = longest common prefix of all token lists,
  moved one token left if any suffix would be empty; empty batch is an error.
* ``throughput_gain`` — SPEC.md:282-291 (T = 1 + N_q/N_i).
* ``merge_attention`` — SPEC.md:264-272 (LSE merge).  On the device the merge is fused into the
  online softmax of the shared-prefix attention kernel; this host version serves the algebra
  tests and documents the identity.
* ``pack_requests`` — B200 layout: for each request the prefix rows then every
  item's suffix rows, contiguous; positions continue at P for every suffix;
  per-segment descriptors and 128-row attention work tiles; ``last_idx`` = last row per item.
  Bit-exact contract, checked against the oracle packer.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

ATTN_TILE = 128


@dataclass
class SharedBatch:
    """SPEC.md:245-248.  ``prefix_kv`` is always None on the B200 path: the prefix KV lives only
    inside one pf_score call (north_star: no KV retained after the request)."""

    prefix_tokens: list[int]
    suffixes: list[list[int]]
    prefix_kv: object = None

    @property
    def n_items(self) -> int:
        return len(self.suffixes)

    def prompt(self, i: int) -> list[int]:
        return list(self.prefix_tokens) + list(self.suffixes[i])


def split_shared_prefix(token_lists: Sequence[Sequence[int]]) -> SharedBatch:
    if len(token_lists) == 0:
        raise ValueError("split_shared_prefix: empty batch")
    lists = [list(map(int, t)) for t in token_lists]
    if any(len(t) == 0 for t in lists):
        raise ValueError("split_shared_prefix: every token list must be non-empty")
    lcp = min(len(t) for t in lists)
    first = lists[0]
    for t in lists[1:]:
        n = 0
        lim = min(lcp, len(t))
        while n < lim and t[n] == first[n]:
            n += 1
        lcp = n
        if lcp == 0:
            break
    # every suffix must keep >= 1 token
    if any(len(t) == lcp for t in lists):
        lcp -= 1
    return SharedBatch(prefix_tokens=first[:lcp], suffixes=[t[lcp:] for t in lists])


def throughput_gain(n_query_tokens: int, n_item_tokens: int) -> float:
    if n_item_tokens <= 0:
        raise ValueError("throughput_gain: n_item_tokens must be >= 1")
    return 1.0 + n_query_tokens / n_item_tokens


def request_flops(cfg, prefix_len: int, suffix_lens: Sequence[int], shared: bool = True) -> float:
    """Algorithmic FLOPs of scoring one request (SPEC.md:295 work accounting):
    L * [tokens * linear_flops_per_token + 4*H*dh * causal (q, k) pairs] at true widths.
    ``shared``: the prefix is computed once and every suffix attends to it (score_shared_batch);
    otherwise every item is an independent full pass over prefix + suffix (forward_prefill)."""
    P = float(prefix_len)
    S = np.asarray(suffix_lens, dtype=np.float64)
    if shared:
        tokens = P + S.sum()
        pairs = P * (P + 1) / 2 + np.sum(S * P + S * (S + 1) / 2)
    else:
        tokens = np.sum(P + S)
        pairs = np.sum((P + S) * (P + S + 1) / 2)
    return float(cfg.n_layers * (tokens * cfg.linear_flops_per_token() + 4 * cfg.n_heads * cfg.d_head * pairs))


@dataclass
class AttentionPartial:
    """output [heads x S x d_head], lse [heads x S]."""

    output: np.ndarray
    lse: np.ndarray


def merge_attention(prefix_part: AttentionPartial, suffix_part: AttentionPartial) -> np.ndarray:
    """(e^{lse_p} o_p + e^{lse_s} o_s) / (e^{lse_p} + e^{lse_s}) with max-subtraction."""
    op, lp = np.asarray(prefix_part.output), np.asarray(prefix_part.lse)
    os_, ls = np.asarray(suffix_part.output), np.asarray(suffix_part.lse)
    if op.shape != os_.shape or lp.shape != ls.shape or op.shape[:-1] != lp.shape:
        raise ValueError("merge_attention: shape mismatch")
    if not (np.all(np.isfinite(op)) and np.all(np.isfinite(os_)) and np.all(np.isfinite(ls))
            and not np.any(np.isnan(lp)) and not np.any(np.isposinf(lp))):
        raise ValueError("merge_attention: non-finite inputs")
    m = np.maximum(lp, ls)
    wp = np.exp(lp - m)
    ws = np.exp(ls - m)
    return (wp[..., None] * op + ws[..., None] * os_) / (wp + ws)[..., None]


@dataclass
class PackedBatch:
    """Flat device inputs of one pf_score call (include/prefill_sm100.h)."""

    ids: np.ndarray        # int32 [T]
    pos: np.ndarray        # int32 [T]
    segs: np.ndarray       # int32 [n_seg, 4]  {kv_off, kv_len, q_off, q_len}
    work: np.ndarray       # int32 [n_work, 4] {seg, q_tile, 0, 0}
    last_idx: np.ndarray   # int32 [N]
    item_request: np.ndarray  # int32 [N] request index of each item
    prefix_lens: np.ndarray   # int32 [R]
    suffix_lens: np.ndarray   # int32 [N]

    @property
    def T(self) -> int:
        return int(self.ids.shape[0])

    @property
    def n_items(self) -> int:
        return int(self.last_idx.shape[0])

    def nbytes(self) -> int:
        return sum(a.nbytes for a in (self.ids, self.pos, self.segs, self.work, self.last_idx))


def pack_requests(batches: Sequence[SharedBatch], max_seq: int = 2048) -> PackedBatch:
    """Pack one or more SharedBatches (requests) into one varlen launch."""
    if len(batches) == 0:
        raise ValueError("pack_requests: no requests")
    ids_parts, pos_parts, segs, last, item_req, plens, slens = [], [], [], [], [], [], []
    off = 0
    for r, sb in enumerate(batches):
        P = len(sb.prefix_tokens)
        if sb.n_items == 0:
            raise ValueError(f"pack_requests: request {r} has no items")
        plens.append(P)
        pre_off = off
        if P > 0:
            ids_parts.append(np.asarray(sb.prefix_tokens, dtype=np.int32))
            pos_parts.append(np.arange(P, dtype=np.int32))
            segs.append((pre_off, 0, pre_off, P))
            off += P
        for s in sb.suffixes:
            S = len(s)
            if S == 0:
                raise ValueError(f"pack_requests: request {r} has an empty suffix")
            if P + S > max_seq:
                raise ValueError(f"pack_requests: prompt length {P + S} exceeds max_seq {max_seq}")
            ids_parts.append(np.asarray(s, dtype=np.int32))
            pos_parts.append(np.arange(P, P + S, dtype=np.int32))
            segs.append((pre_off, P, off, S))
            last.append(off + S - 1)
            item_req.append(r)
            slens.append(S)
            off += S
    segs_a = np.asarray(segs, dtype=np.int32).reshape(-1, 4)
    work = make_work(segs_a)
    return PackedBatch(
        ids=np.concatenate(ids_parts).astype(np.int32, copy=False),
        pos=np.concatenate(pos_parts).astype(np.int32, copy=False),
        segs=segs_a, work=work,
        last_idx=np.asarray(last, dtype=np.int32),
        item_request=np.asarray(item_req, dtype=np.int32),
        prefix_lens=np.asarray(plens, dtype=np.int32),
        suffix_lens=np.asarray(slens, dtype=np.int32),
    )


def concat_packed(parts: Sequence[PackedBatch]) -> PackedBatch:
    """Join requests packed separately (e.g. at arrival, off the serving loop) into one launch.
    Row offsets in segs / last_idx shift by the preceding parts' T, request indices by their request
    counts, and the work list is rebuilt over the joined segments; the result equals
    ``pack_requests`` over the concatenated request list, array for array."""
    if len(parts) == 0:
        raise ValueError("concat_packed: no requests")
    if len(parts) == 1:
        return parts[0]
    t_off = np.cumsum([0] + [p.T for p in parts[:-1]]).astype(np.int32)
    r_off = np.cumsum([0] + [len(p.prefix_lens) for p in parts[:-1]]).astype(np.int32)
    segs = np.concatenate([p.segs + np.array([o, 0, o, 0], dtype=np.int32) for p, o in zip(parts, t_off)])
    return PackedBatch(
        ids=np.concatenate([p.ids for p in parts]),
        pos=np.concatenate([p.pos for p in parts]),
        segs=segs, work=make_work(segs),
        last_idx=np.concatenate([p.last_idx + o for p, o in zip(parts, t_off)]).astype(np.int32),
        item_request=np.concatenate([p.item_request + o for p, o in zip(parts, r_off)]).astype(np.int32),
        prefix_lens=np.concatenate([p.prefix_lens for p in parts]),
        suffix_lens=np.concatenate([p.suffix_lens for p in parts]),
    )


# Query rows per attention work group: the K/V of a group's segments (C3: 4 KB per row over all kv
# heads, 32 MB per group) stay in the 126 MB L2 while its tiles run (4096-8192 rows measured best at
# C3: step 152.7 -> 150.8 ms, same box).  PF_WORK_GROUP_ROWS overrides
# (0 = one group: plain longest-first order over the whole batch).
WORK_GROUP_ROWS = 8192


def make_work(segs: np.ndarray, group_rows: int | None = None) -> np.ndarray:
    """One work entry per 128-row query tile.  Segments are cut into consecutive groups of at most
    ``group_rows`` query rows, taken from the last segment backwards (the QKV GEMM writes rows in
    ascending order, so the first attention units read the rows it wrote last, while they are still
    in L2).  Inside a group the heaviest tiles (most key blocks) go first so the longest CTAs start
    early; ties in descending segment order.  Grouping keeps each group's K/V resident in L2 across
    its tiles: ordering all tiles of a long-item batch (C3) by cost alone cycles through every
    item's K/V once per tile index and re-reads ~2.6x the QKV buffer from DRAM."""
    import os

    if group_rows is None:
        group_rows = int(os.environ.get("PF_WORK_GROUP_ROWS", WORK_GROUP_ROWS))
    q_len = segs[:, 3].astype(np.int64)
    kv_len = segs[:, 1].astype(np.int64)
    n = len(segs)
    ntile = (q_len + ATTN_TILE - 1) // ATTN_TILE
    # group id per segment, counting from the last segment
    group = np.zeros(n, dtype=np.int64)
    if group_rows > 0:
        g, acc = 0, 0
        for i in range(n - 1, -1, -1):
            if acc > 0 and acc + q_len[i] > group_rows:
                g, acc = g + 1, 0
            acc += int(q_len[i])
            group[i] = g
    seg_idx = np.repeat(np.arange(n, dtype=np.int64), ntile)
    starts = np.cumsum(ntile) - ntile
    tile = np.arange(int(ntile.sum()), dtype=np.int64) - np.repeat(starts, ntile)
    cost = (kv_len[seg_idx] + ATTN_TILE - 1) // ATTN_TILE + tile + 1
    order = np.lexsort((tile, -seg_idx, -cost, group[seg_idx]))
    work = np.zeros((len(seg_idx), 4), dtype=np.int32)
    work[:, 0] = seg_idx[order]
    work[:, 1] = tile[order]
    return work


def pack_token_lists(token_lists: Sequence[Sequence[int]], max_seq: int = 2048) -> PackedBatch:
    """split_shared_prefix + pack for a single request."""
    return pack_requests([split_shared_prefix(token_lists)], max_seq)
