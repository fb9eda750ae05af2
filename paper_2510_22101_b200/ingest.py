"""Host ingest: tokenizer + packer running in C++ inside libprefill_sm100.so.

``Vocab``/``encode``/``encode_batch`` mirror the reference tokenizer
(/root/reference/pkg/src/prefrank/tokenizer.py:49-161): FNV-1a-64 word hashing into
[reserved, size), template tags and yes/no as reserved ids.  Output is bit-identical to the
reference (tests/test_host_ingest.py, against tests/golden/prompts.json).
``pack_token_lists_native`` is the C++ twin of ``prefixcache.pack_requests``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from .prefixcache import PackedBatch, make_work

TEMPLATE_TAGS = ("<|sys|>", "<|/sys|>", "<|q|>", "<|/q|>", "<|meta|>", "<|/meta|>", "<|desc|>",
                 "<|/desc|>", "<|ans|>")
FNV_OFFSET = 14695981039346656037
FNV_PRIME = 1099511628211


@dataclass(frozen=True)
class Vocab:
    """tokenizer.py:49-70: id space and reserved-id table (the C++ scanner hard-wires this table)."""

    size: int = 32768
    reserved: int = 16
    yes_id: int = 1
    no_id: int = 2
    specials: dict = field(default_factory=lambda: {"yes": 1, "no": 2,
                                                    **{t: 3 + i for i, t in enumerate(TEMPLATE_TAGS)}})

    def __post_init__(self):
        if self.yes_id == self.no_id:
            raise ValueError("yes_id and no_id must differ")
        if max(self.specials.values()) >= self.reserved:
            raise ValueError("special ids must fit in the reserved range")
        if self.reserved >= self.size:
            raise ValueError("vocab size must exceed reserved range")
        if (self.yes_id, self.no_id) != (1, 2) or self.specials.get("<|ans|>") != 11:
            raise ValueError("the native tokenizer implements the reference special-id table only")

    def word_id(self, word: str) -> int:
        s = self.specials.get(word)
        if s is not None:
            return s
        h = FNV_OFFSET
        for b in word.encode("utf-8"):
            h = ((h ^ b) * FNV_PRIME) & 0xFFFFFFFFFFFFFFFF
        return self.reserved + h % (self.size - self.reserved)


DEFAULT_VOCAB = Vocab()


def encode(text: str, vocab: Vocab = DEFAULT_VOCAB) -> list[int]:
    lib = _lib.load()
    raw = text.encode("utf-8", errors="surrogatepass")
    out = np.empty(max(1, len(raw)), dtype=np.int32)
    n = ctypes.c_int64()
    _lib.check(lib.pf_tokenize(raw, len(raw), vocab.size, vocab.reserved, out.ctypes.data, out.size,
                               ctypes.byref(n)))
    return out[: n.value].tolist()


def encode_batch_arrays(texts: Sequence[str], vocab: Vocab = DEFAULT_VOCAB, n_threads: int = 0):
    """-> (ids int32 [total], offsets int64 [n+1])."""
    lib = _lib.load()
    raws = [t.encode("utf-8", errors="surrogatepass") for t in texts]
    lens = np.fromiter((len(r) for r in raws), dtype=np.int64, count=len(raws))
    offs = np.zeros(len(raws) + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    data = b"".join(raws)
    buf = ctypes.create_string_buffer(data, len(data) + 1)
    out = np.empty(max(1, int(offs[-1])), dtype=np.int32)
    out_offs = np.empty(len(raws) + 1, dtype=np.int64)
    _lib.check(lib.pf_tokenize_batch(ctypes.addressof(buf), offs.ctypes.data, len(raws), vocab.size,
                                     vocab.reserved, out.ctypes.data, out.size, out_offs.ctypes.data, n_threads))
    return out[: out_offs[-1]], out_offs


def encode_batch(texts: Sequence[str], vocab: Vocab = DEFAULT_VOCAB, n_threads: int = 0) -> list[list[int]]:
    ids, offs = encode_batch_arrays(texts, vocab, n_threads)
    return [ids[offs[i]:offs[i + 1]].tolist() for i in range(len(texts))]


def pack_token_lists_native(requests: Sequence[Sequence[Sequence[int]]], max_seq: int = 2048) -> PackedBatch:
    """requests[r] = the token lists of request r (one per item); split_shared_prefix + packing in
    C++.  Same PackedBatch as prefixcache.pack_requests([split_shared_prefix(l) for l in requests])."""
    lists = [np.asarray(l, dtype=np.int32) for req in requests for l in req]
    begin = np.zeros(len(requests) + 1, dtype=np.int32)
    np.cumsum([len(req) for req in requests], out=begin[1:])
    loffs = np.zeros(len(lists) + 1, dtype=np.int64)
    np.cumsum([len(l) for l in lists], out=loffs[1:])
    flat = np.concatenate(lists) if lists else np.zeros(0, np.int32)
    return pack_flat_native(flat, loffs, begin, max_seq)


def pack_flat_native(flat: np.ndarray, loffs: np.ndarray, begin: np.ndarray | None = None,
                     max_seq: int = 2048) -> PackedBatch:
    """The same from flat arrays (what encode_batch_arrays returns): token list i is
    flat[loffs[i]:loffs[i+1]]; request r owns lists begin[r]..begin[r+1]-1 (default: one request)."""
    lib = _lib.load()
    flat = np.ascontiguousarray(flat, dtype=np.int32)
    loffs = np.ascontiguousarray(loffs, dtype=np.int64)
    if begin is None:
        begin = np.array([0, len(loffs) - 1], dtype=np.int32)
    begin = np.ascontiguousarray(begin, dtype=np.int32)
    requests = [range(int(begin[r]), int(begin[r + 1])) for r in range(len(begin) - 1)]
    T, S, N = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.check(lib.pf_pack_sizes(loffs.ctypes.data, begin.ctypes.data, len(requests), ctypes.byref(T),
                                 ctypes.byref(S), ctypes.byref(N)))
    ids = np.empty(max(1, T.value), np.int32)
    pos = np.empty(max(1, T.value), np.int32)
    segs = np.empty((max(1, S.value), 4), np.int32)
    last = np.empty(max(1, N.value), np.int32)
    plen = np.empty(max(1, len(requests)), np.int32)
    t_out, s_out = ctypes.c_int64(), ctypes.c_int64()
    rc = lib.pf_pack_requests(flat.ctypes.data, loffs.ctypes.data, begin.ctypes.data, len(requests), max_seq,
                              ids.ctypes.data, pos.ctypes.data, segs.ctypes.data, last.ctypes.data,
                              plen.ctypes.data, ctypes.byref(t_out), ctypes.byref(s_out))
    if rc == -2:
        raise ValueError(f"pack: prompt length exceeds max_seq {max_seq}")
    if rc == -1:
        raise ValueError("pack: empty request or empty token list")
    _lib.check(rc)
    segs = segs[: s_out.value].copy()
    n_items = N.value
    item_req = np.repeat(np.arange(len(requests), dtype=np.int32), [len(r) for r in requests])
    return PackedBatch(ids=ids[: t_out.value].copy(), pos=pos[: t_out.value].copy(), segs=segs,
                       work=make_work(segs), last_idx=last[:n_items].copy(), item_request=item_req,
                       prefix_lens=plen[: len(requests)].copy(),
                       suffix_lens=_suffix_lens(segs, plen[: len(requests)], [len(r) for r in requests]))


def _suffix_lens(segs, plen, n_items_per_req):
    out = []
    k = 0
    for P, n in zip(plen, n_items_per_req):
        if P > 0:
            k += 1            # the request's prefix segment
        out.extend(int(s) for s in segs[k:k + n, 3])
        k += n
    return np.asarray(out, dtype=np.int32)
