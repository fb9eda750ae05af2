"""Device scorer: owns the pf_model handle, the workspace and the call into pf_score.

This is the host side of the drop-in boundary.  ``score_shared_batch`` keeps the
reference name and meaning: one prefix, many suffixes, results order-aligned
with the input batch.  Every call goes through libprefill_sm100.so; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .config import ModelConfig
from .prefixcache import PackedBatch, SharedBatch, pack_requests
from .scoring import RelevanceScore
from .weights import DeviceWeights, Weights, to_device


def _ptr(t) -> int:
    return int(t.data_ptr())


def _ptr_array(ts) -> ctypes.Array:
    return (ctypes.c_void_p * len(ts))(*[_ptr(t) for t in ts])


@dataclass
class ScoredBatch:
    """Per-item (logit_yes, logit_no) and p_yes, order-aligned with the packed items."""

    logits2: np.ndarray   # float32 [N, 2]
    p_yes: np.ndarray     # float32 [N]

    def relevance(self, i: int) -> RelevanceScore:
        p = float(self.p_yes[i])
        return RelevanceScore(p_yes=p, p_no=1.0 - p)

    # the spec's "list of last-token logits": item i -> its (logit_yes, logit_no)
    def __len__(self) -> int:
        return int(self.p_yes.shape[0])

    def __getitem__(self, i):
        return self.logits2[i]

    def __iter__(self):
        return iter(self.logits2)


class DevicePacked:
    """A PackedBatch resident on the device (torch int32 tensors)."""

    def __init__(self, packed: PackedBatch, device="cuda"):
        import torch

        self.packed = packed
        self.ids = torch.from_numpy(packed.ids).to(device)
        self.pos = torch.from_numpy(packed.pos).to(device)
        self.segs = torch.from_numpy(np.ascontiguousarray(packed.segs)).to(device)
        self.work = torch.from_numpy(np.ascontiguousarray(packed.work)).to(device)
        self.last_idx = torch.from_numpy(packed.last_idx).to(device)


class PinnedPacked:
    """A PackedBatch in page-locked host memory (for the end-to-end host-buffer path)."""

    def __init__(self, packed: PackedBatch):
        import torch

        self.packed = packed
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        self.ids, self.pos = pin(packed.ids), pin(packed.pos)
        self.segs, self.work, self.last_idx = pin(packed.segs), pin(packed.work), pin(packed.last_idx)
        n = packed.n_items
        self.logits2 = torch.empty((n, 2), dtype=torch.float32).pin_memory()
        self.p_yes = torch.empty((n,), dtype=torch.float32).pin_memory()

    def h2d_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.ids, self.pos, self.segs, self.work, self.last_idx))

    def d2h_bytes(self) -> int:
        return (self.logits2.numel() + self.p_yes.numel()) * 4


class _StreamState:
    """Workspace and non-finite flag owned by one CUDA stream.  Calls on distinct streams never share
    activations, and a workspace that must grow is replaced only by calls on its own stream, whose
    earlier kernels the caching allocator orders before any reuse of the old block."""

    __slots__ = ("ws", "bad")

    def __init__(self, bad):
        self.ws = None
        self.bad = bad


class PrefillScorer:
    """Model replica on one GPU: device weights + pf_model handle + per-stream workspaces.

    Thread-safety: the handle and weights are read-only after construction ("weights
    shareable read-only across threads").  Each CUDA stream gets its own workspace and non-finite
    flag, so concurrent calls are safe as long as each thread scores on its own stream."""

    def __init__(self, weights: DeviceWeights | Weights, device=None):
        import threading

        import torch

        self.lib = _lib.load()
        if isinstance(weights, Weights):
            weights = to_device(weights, device or "cuda")
        self.device = torch.device(device) if device is not None else weights.embedding.device
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.weights = weights
        self.config: ModelConfig = weights.config
        check_device_weights(weights, self.device)
        cfg = self.config
        w = weights
        self._keep = [_ptr_array(w.w_qkv), _ptr_array(w.w_o), _ptr_array(w.w_gu), _ptr_array(w.w_down)]
        desc = _lib.PfModelDesc()
        desc.n_layers, desc.d_model = cfg.n_layers, cfg.d_model
        desc.n_heads, desc.n_kv_heads, desc.d_head = cfg.n_heads, cfg.n_kv_heads, cfg.d_head
        desc.d_ff, desc.d_ff_pad = cfg.d_ff, cfg.d_ff_pad
        desc.vocab_size, desc.max_seq, desc.rms_eps = cfg.vocab_size, cfg.max_seq, cfg.rms_eps
        desc.embedding = _ptr(w.embedding)
        (desc.w_qkv, desc.w_o, desc.w_gu, desc.w_down) = [
            ctypes.cast(a, ctypes.POINTER(ctypes.c_void_p)) for a in self._keep]
        desc.ln_final, desc.w_yes, desc.w_no = _ptr(w.ln_final), _ptr(w.w_yes), _ptr(w.w_no)
        desc.rope_cos, desc.rope_sin = _ptr(w.rope_cos), _ptr(w.rope_sin)
        self._desc = desc
        handle = ctypes.c_void_p()
        with self.device_guard():
            _lib.check(self.lib.pf_model_create(ctypes.byref(desc), ctypes.byref(handle)))
        self.handle = handle
        self._states: dict[int, _StreamState] = {}
        self._lock = threading.Lock()

    # ------------------------------------------------------------------ device / stream plumbing
    def device_guard(self):
        """Make this replica's device current for the C-ABI calls (kernel attributes, SM counts and
        launches are per device)."""
        import torch

        return torch.cuda.device(self.device)

    def _torch_stream(self, stream):
        import torch

        return stream if stream is not None else torch.cuda.current_stream(self.device)

    def _state(self, stream) -> _StreamState:
        import torch

        key = int(self._torch_stream(stream).cuda_stream)
        st = self._states.get(key)
        if st is None:
            with self._lock:
                st = self._states.get(key)
                if st is None:
                    st = _StreamState(torch.zeros(4, dtype=torch.int32, device=self.device))
                    self._states[key] = st
        return st

    def bad_flag(self, stream=None):
        """Device int32[4]; element 0 is non-zero after a non-finite logit on ``stream``."""
        return self._state(stream).bad

    # ------------------------------------------------------------------ workspace
    def workspace(self, T: int, n_items: int, stream=None):
        import torch

        need = int(self.lib.pf_workspace_bytes(self.handle, T, n_items))
        st = self._state(stream)
        if st.ws is None or st.ws.numel() < need:
            st.ws = None   # freed on this stream; the allocator orders reuse after its pending kernels
            with torch.cuda.stream(self._torch_stream(stream)):
                st.ws = torch.empty(need + 4096, dtype=torch.uint8, device=self.device)
        base = _ptr(st.ws)
        aligned = (base + 1023) & ~1023
        return aligned, st.ws.numel() - (aligned - base)

    def _stream(self, stream):
        return ctypes.c_void_p(self._torch_stream(stream).cuda_stream)

    # ------------------------------------------------------------------ scoring
    def validate_device(self, dp: DevicePacked, stream=None) -> None:
        """Bounds-check a device-resident batch on the device (pf_validate_packed) and raise
        ValueError on the first violation.  Synchronises ``stream``."""
        import torch

        pk = dp.packed
        err = torch.zeros(2, dtype=torch.int32, device=self.device)
        with self.device_guard():
            _lib.check(self.lib.pf_validate_packed(self.handle, _ptr(dp.ids), _ptr(dp.pos), _ptr(dp.segs),
                                                   len(pk.segs), _ptr(dp.work), len(pk.work), _ptr(dp.last_idx),
                                                   pk.n_items, pk.T, _ptr(err), self._stream(stream)))
        self._torch_stream(stream).synchronize()
        code, idx = (int(x) for x in err.cpu())
        if code:
            what = {1: "token id", 2: "position", 3: "segment", 4: "work tile", 5: "last_idx"}.get(code, "?")
            raise ValueError(f"packed batch invalid: {what} at index {idx}")

    def score_device(self, dp: DevicePacked, logits2=None, p_yes=None, stream=None, check=True,
                     workspace=None, validate=False, bad=None):
        """Inputs already resident on the device; asynchronous on ``stream``.  Returns device
        tensors.  ``validate=True`` first runs the device bounds check (synchronous)."""
        import torch

        pk = dp.packed
        n = pk.n_items
        if validate:
            self.validate_device(dp, stream)
        if logits2 is None:
            logits2 = torch.empty((n, 2), dtype=torch.float32, device=self.device)
        if p_yes is None:
            p_yes = torch.empty((n,), dtype=torch.float32, device=self.device)
        ws, ws_bytes = workspace if workspace is not None else self.workspace(pk.T, n, stream)
        if bad is None:
            bad = self._state(stream).bad
        if check:
            with torch.cuda.stream(self._torch_stream(stream)):
                bad.zero_()
        with self.device_guard():
            rc = self.lib.pf_score(self.handle, _ptr(dp.ids), _ptr(dp.pos), _ptr(dp.segs), len(pk.segs),
                                   _ptr(dp.work), len(pk.work), _ptr(dp.last_idx), n, pk.T,
                                   ws, ws_bytes, _ptr(logits2), _ptr(p_yes), _ptr(bad),
                                   self._stream(stream))
        _lib.check(rc)
        return logits2, p_yes

    def score_capture(self, dp: DevicePacked, rows, gains, stream=None, return_scores=False, out=None):
        """pf_score with the calibration capture (SPEC.md:200-203 capture flag): returns a device
        fp32 tensor [n_layers, len(rows), d_model] of rmsnorm(x_l[row]) * gains[l], the MLP input
        of every layer at the packed rows ``rows`` (device int32).  Synchronises ``stream``."""
        import torch

        cfg, pk = self.config, dp.packed
        n = pk.n_items
        rows = rows.to(device=self.device, dtype=torch.int32).contiguous()
        if rows.numel() and (int(rows.min()) < 0 or int(rows.max()) >= pk.T):
            raise ValueError("score_capture: capture rows outside [0, T)")
        gains = gains.to(device=self.device, dtype=torch.float32).contiguous()
        if tuple(gains.shape) != (cfg.n_layers, cfg.d_model):
            raise ValueError("score_capture: gains must be [n_layers, d_model]")
        shape = (cfg.n_layers, rows.numel(), cfg.d_model)
        if out is None:
            out = torch.empty(shape, dtype=torch.float32, device=self.device)
        elif (tuple(out.shape) != shape or out.dtype != torch.float32 or out.device.type != "cuda"
              or out.stride()[1:] != (cfg.d_model, 1)):
            raise ValueError("score_capture: out must be fp32 [n_layers, n_rows, d_model], rows dense")
        logits2 = torch.empty((n, 2), dtype=torch.float32, device=self.device)
        p_yes = torch.empty((n,), dtype=torch.float32, device=self.device)
        ws, ws_bytes = self.workspace(pk.T, n, stream)
        bad = self._state(stream).bad
        cap = _lib.PfCapture(rows=_ptr(rows), n_rows=rows.numel(), gains=_ptr(gains), out=_ptr(out),
                             out_layer_stride=out.stride(0))
        st = self._stream(stream)
        with self.device_guard():
            rc = self.lib.pf_score_capture(self.handle, _ptr(dp.ids), _ptr(dp.pos), _ptr(dp.segs), len(pk.segs),
                                           _ptr(dp.work), len(pk.work), _ptr(dp.last_idx), n, pk.T, ws, ws_bytes,
                                           _ptr(logits2), _ptr(p_yes), _ptr(bad), ctypes.byref(cap), st)
        _lib.check(rc)
        self._torch_stream(stream).synchronize()
        return (out, logits2, p_yes) if return_scores else out

    def graph_runner(self, dp: DevicePacked):
        """Capture one pf_score pass over ``dp`` into a CUDA graph (private workspace, output
        buffers and non-finite flag, so later calls cannot invalidate it).  Returns
        ``run() -> (logits2, p_yes)``; replay removes the ~150 host launches per pass.  The flag
        is not reset by replays: ``run.nonfinite()`` reads it (synchronising) and is non-zero once
        any replay since capture produced a non-finite logit; ``run.reset()`` clears it."""
        import torch

        pk = dp.packed
        n = pk.n_items
        need = int(self.lib.pf_workspace_bytes(self.handle, pk.T, n))
        ws_t = torch.empty(need + 4096, dtype=torch.uint8, device=self.device)
        base = _ptr(ws_t)
        ws = ((base + 1023) & ~1023, ws_t.numel() - (((base + 1023) & ~1023) - base))
        logits2 = torch.empty((n, 2), dtype=torch.float32, device=self.device)
        p_yes = torch.empty((n,), dtype=torch.float32, device=self.device)
        bad = torch.zeros(4, dtype=torch.int32, device=self.device)
        self.score_device(dp, logits2, p_yes, workspace=ws, bad=bad, check=False)   # sets kernel attributes
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.score_device(dp, logits2, p_yes, workspace=ws, bad=bad, check=False)

        def run():
            g.replay()
            return logits2, p_yes

        run.graph, run.keepalive = g, (ws_t, dp)
        run.nonfinite = lambda: int(bad[0].item())
        run.reset = lambda: bad.zero_()
        return run

    def score_host(self, pp: PinnedPacked, stream=None) -> ScoredBatch:
        """End-to-end through the C-ABI with host buffers (H2D + forward + D2H + sync)."""
        pk = pp.packed
        ws, ws_bytes = self.workspace(pk.T, pk.n_items, stream)
        with self.device_guard():
            rc = self.lib.pf_score_host(self.handle, _ptr(pp.ids), _ptr(pp.pos), _ptr(pp.segs),
                                        len(pk.segs), _ptr(pp.work), len(pk.work), _ptr(pp.last_idx),
                                        pk.n_items, pk.T, ws, ws_bytes, _ptr(pp.logits2), _ptr(pp.p_yes),
                                        self._stream(stream))
        _lib.check(rc)
        return ScoredBatch(pp.logits2.numpy().copy(), pp.p_yes.numpy().copy())

    def score_packed(self, packed: PackedBatch, stream=None) -> ScoredBatch:
        self.validate(packed)
        dp = DevicePacked(packed, self.device)
        logits2, p_yes = self.score_device(dp, stream=stream)
        self._torch_stream(stream).synchronize()
        if int(self.bad_flag(stream)[0].item()) != 0:
            raise ValueError("relevance_score: non-finite logits (SPEC.md:330)")
        return ScoredBatch(logits2.cpu().numpy(), p_yes.cpu().numpy())

    def validate(self, packed: PackedBatch) -> None:
        """Host-side bounds check of a packed batch (the same rules as pf_score_host's and the
        device check's): raises ValueError before any device work."""
        validate_packed(packed, self.config)

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.lib.pf_model_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def validate_packed(packed: PackedBatch, cfg: ModelConfig) -> None:
    """Bounds of every array pf_score reads (include/prefill_sm100.h packed-batch layout)."""
    T, n = packed.T, packed.n_items
    if T == 0 or n == 0:
        raise ValueError("empty batch")
    if packed.ids.shape != (T,) or packed.pos.shape != (T,):
        raise ValueError("ids/pos must have T entries")
    if packed.ids.min() < 0 or packed.ids.max() >= cfg.vocab_size:
        raise ValueError("token id outside the vocabulary")
    if packed.pos.min() < 0 or packed.pos.max() >= cfg.max_seq:
        raise ValueError(f"sequence exceeds max_seq={cfg.max_seq}")
    segs = np.asarray(packed.segs, dtype=np.int64).reshape(-1, 4)
    work = np.asarray(packed.work, dtype=np.int64).reshape(-1, 4)
    last = np.asarray(packed.last_idx, dtype=np.int64)
    if len(segs) < 1 or len(work) < 1 or len(segs) > T or len(work) > T or last.shape != (n,):
        raise ValueError("bad segment / work / last_idx counts")
    if ((segs[:, :3] < 0).any() or (segs[:, 3] < 1).any() or (segs[:, 0] + segs[:, 1] > T).any()
            or (segs[:, 2] + segs[:, 3] > T).any()):
        raise ValueError("segment outside [0, T)")
    if (segs[1:, 2] < segs[:-1, 2] + segs[:-1, 3]).any():
        # the packer's order; the last layer finds a last-token row's segment by its q offset
        raise ValueError("segments out of order (q ranges must increase and not overlap)")
    if (work[:, 0] < 0).any() or (work[:, 0] >= len(segs)).any() or (work[:, 1] < 0).any():
        raise ValueError("work tile names a missing segment")
    if (work[:, 1] * 128 >= segs[work[:, 0], 3]).any():
        raise ValueError("work tile outside its segment")
    if (last < 0).any() or (last >= T).any():
        raise ValueError("last_idx outside [0, T)")


def check_device_weights(w: DeviceWeights, device) -> None:
    """Shape discipline for the device layout pf_model_create builds tensor maps over:
    a list shorter than n_layers, or a tensor smaller than its config shape, would make the
    kernels read out of bounds, so both are rejected here."""
    import torch

    cfg = w.config
    L, d = cfg.n_layers, cfg.d_model
    qkv_n = (cfg.n_heads + 2 * cfg.n_kv_heads) * cfg.d_head
    want = {"w_qkv": (qkv_n, d), "w_o": (d, cfg.q_width), "w_gu": (2 * cfg.d_ff_pad, d),
            "w_down": (d, cfg.d_ff_pad)}
    for name, shape in want.items():
        ts = getattr(w, name)
        if len(ts) != L:
            raise ValueError(f"device weights: {name} has {len(ts)} layers, config has n_layers={L}")
        for l, t in enumerate(ts):
            if tuple(t.shape) != shape or t.dtype != torch.bfloat16 or not t.is_contiguous():
                raise ValueError(f"device weights: {name}[{l}] is {tuple(t.shape)} {t.dtype}, "
                                 f"expected contiguous bf16 {shape}")
    singles = {"embedding": ((cfg.vocab_size, d), torch.bfloat16), "ln_final": ((d,), torch.float32),
               "w_yes": ((d,), torch.float32), "w_no": ((d,), torch.float32),
               "rope_cos": ((cfg.max_seq, cfg.d_head // 2), torch.float32),
               "rope_sin": ((cfg.max_seq, cfg.d_head // 2), torch.float32)}
    for name, (shape, dt) in singles.items():
        t = getattr(w, name)
        if t is None or tuple(t.shape) != shape or t.dtype != dt or not t.is_contiguous():
            raise ValueError(f"device weights: {name} must be contiguous {dt} {shape}")
    for t in [w.embedding, *w.w_qkv, *w.w_o, *w.w_gu, *w.w_down, w.ln_final, w.w_yes, w.w_no]:
        if t.device != device:
            raise ValueError(f"device weights live on {t.device}, scorer device is {device}")


# ---------------------------------------------------------------------------- spec entry points
_SCORERS: dict = {}


def scorer_for(weights, device=None) -> PrefillScorer:
    """The replica that scores with ``weights`` on ``device``: a PrefillScorer is returned as is;
    host ``Weights`` and ``DeviceWeights`` get one cached scorer per (weights object, device), dropped
    when the weights object is collected.  Weights are immutable during inference, so
    the cache is keyed by identity."""
    import weakref

    import torch

    if isinstance(weights, PrefillScorer):
        return weights
    if not isinstance(weights, (Weights, DeviceWeights)):
        raise TypeError(f"expected Weights, DeviceWeights or PrefillScorer, got {type(weights).__name__}")
    if device is None:
        device = weights.embedding.device if isinstance(weights, DeviceWeights) else "cuda"
    dev = torch.device(device)
    if dev.type == "cuda" and dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (id(weights), str(dev))
    s = _SCORERS.get(key)
    if s is None:
        s = PrefillScorer(weights, dev)
        _SCORERS[key] = s
        weakref.finalize(weights, _SCORERS.pop, key, None)
    return s


def score_shared_batch(weights, shared: SharedBatch | Sequence[SharedBatch], device=None) -> ScoredBatch:
    """SPEC.md:273-281 on the device: ``score_shared_batch(weights, shared)`` with ``weights`` a
    ``Weights`` (the reference's type), ``DeviceWeights`` or ``PrefillScorer``.  One packed forward
    over [prefix | suffix_0 | ...] for one or several requests; results order-aligned with the input
    items.  Each result is the 2-logit view (logit_yes, logit_no) of the spec's last-token logits
    (north_star: the [vocab] row is never formed); ``relevance_score`` reads either form."""
    batches = [shared] if isinstance(shared, SharedBatch) else list(shared)
    if not batches or any(sb.n_items == 0 for sb in batches):
        raise ValueError("score_shared_batch: empty batch")
    cfg = _config_of(weights)
    for sb in batches:
        longest = len(sb.prefix_tokens) + max(len(x) for x in sb.suffixes)
        if longest > cfg.max_seq or min(len(x) for x in sb.suffixes) == 0:
            raise ValueError(f"score_shared_batch: prefix + suffix must be 1..max_seq={cfg.max_seq} tokens")
    model = scorer_for(weights, device)
    return model.score_packed(pack_requests(batches, model.config.max_seq))


@dataclass(frozen=True)
class KVCache:
    """The spec's KVCache on the B200 path: the prefix's tokens, not its K/V.

    north_star keeps no KV after a request, and a device launch recomputes a prefix's K/V inside
    the same packed pass that scores its suffixes (once per request, as score_shared_batch does),
    so the handle carries what that pass needs.  ``seq_len`` and ``n_layers`` keep the spec's
    invariants and errors (seq_len <= max_seq; layer-count mismatch)."""

    tokens: tuple
    n_layers: int

    @property
    def seq_len(self) -> int:
        return len(self.tokens)


def _config_of(weights) -> ModelConfig:
    cfg = getattr(weights, "config", None)
    if not isinstance(cfg, ModelConfig):
        raise TypeError(f"expected Weights, DeviceWeights or PrefillScorer, got {type(weights).__name__}")
    return cfg


def _one_item(weights, prefix: Sequence[int], suffix: Sequence[int], device):
    model = scorer_for(weights, device)
    res = model.score_packed(pack_requests([SharedBatch(list(prefix), [list(suffix)])], model.config.max_seq))
    return model, res.logits2[0].copy()


def forward_prefill(weights, tokens: Sequence[int], capture=None, device=None):
    """SPEC.md:200-208 ``forward_prefill(weights, tokens, capture)`` -> (last-token logits,
    KVCache, captured MLP inputs or None).  Logits are the (logit_yes, logit_no) view.  ``capture``
    truthy records every position's MLP input per layer (rmsnorm(x_l)·g_mlp, fp32
    [n_layers, len(tokens), d_model], the pruning module's calibration rows).
    Errors: empty or over-length sequence (ValueError)."""
    tokens = [int(t) for t in tokens]
    cfg = _config_of(weights)
    if not 1 <= len(tokens) <= cfg.max_seq:
        raise ValueError(f"forward_prefill: need 1 <= len(tokens) <= max_seq={cfg.max_seq}, got {len(tokens)}")
    model = scorer_for(weights, device)
    kv = KVCache(tuple(tokens), cfg.n_layers)
    if not capture:
        _, logits = _one_item(model, tokens[:-1], tokens[-1:], device)
        return logits, kv, None
    import torch

    packed = pack_requests([SharedBatch(tokens[:-1], [tokens[-1:]])], cfg.max_seq)
    model.validate(packed)
    dp = DevicePacked(packed, model.device)
    gains = torch.stack([g.float() for g in model.weights.ln_mlp])
    rows = torch.arange(len(tokens), dtype=torch.int32, device=model.device)   # packed row t = position t
    out, logits2, _ = model.score_capture(dp, rows, gains, return_scores=True)
    return logits2[0].cpu().numpy(), kv, out.cpu().numpy()


def forward_with_prefix(weights, prefix_cache: KVCache, suffix_tokens: Sequence[int], device=None):
    """SPEC.md:209-217 ``forward_with_prefix(weights, prefix_cache, suffix_tokens)`` -> (last-token
    logits, extended cache).  Suffix positions continue from the prefix length.  Errors (ValueError):
    empty suffix, prefix + suffix over max_seq, layer-count mismatch."""
    suffix = [int(t) for t in suffix_tokens]
    cfg = _config_of(weights)
    if not isinstance(prefix_cache, KVCache):
        raise TypeError("forward_with_prefix: prefix_cache must be the KVCache forward_prefill returned")
    if prefix_cache.n_layers != cfg.n_layers:
        raise ValueError(f"forward_with_prefix: cache has {prefix_cache.n_layers} layers, model has {cfg.n_layers}")
    if not suffix:
        raise ValueError("forward_with_prefix: empty suffix")
    if prefix_cache.seq_len + len(suffix) > cfg.max_seq:
        raise ValueError(f"forward_with_prefix: {prefix_cache.seq_len} + {len(suffix)} tokens exceed "
                         f"max_seq={cfg.max_seq}")
    _, logits = _one_item(weights, prefix_cache.tokens, suffix, device)
    return logits, KVCache(prefix_cache.tokens + tuple(suffix), cfg.n_layers)
