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


class PrefillScorer:
    """Model replica on one GPU: device weights + pf_model handle + growable workspace."""

    def __init__(self, weights: DeviceWeights | Weights, device="cuda"):
        import torch

        self.lib = _lib.load()
        if isinstance(weights, Weights):
            weights = to_device(weights, device)
        self.weights = weights
        self.config: ModelConfig = weights.config
        self.device = torch.device(device)
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
        _lib.check(self.lib.pf_model_create(ctypes.byref(desc), ctypes.byref(handle)))
        self.handle = handle
        self._ws = None
        self._bad = torch.zeros(4, dtype=torch.int32, device=self.device)

    # ------------------------------------------------------------------ workspace
    def workspace(self, T: int, n_items: int):
        import torch

        need = int(self.lib.pf_workspace_bytes(self.handle, T, n_items))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need + 4096, dtype=torch.uint8, device=self.device)
        base = _ptr(self._ws)
        aligned = (base + 1023) & ~1023
        return aligned, self._ws.numel() - (aligned - base)

    def _stream(self, stream):
        import torch

        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return ctypes.c_void_p(s.cuda_stream)

    # ------------------------------------------------------------------ scoring
    def score_device(self, dp: DevicePacked, logits2=None, p_yes=None, stream=None, check=True,
                     workspace=None):
        """Inputs already resident on the device; asynchronous.  Returns device tensors."""
        import torch

        pk = dp.packed
        n = pk.n_items
        if logits2 is None:
            logits2 = torch.empty((n, 2), dtype=torch.float32, device=self.device)
        if p_yes is None:
            p_yes = torch.empty((n,), dtype=torch.float32, device=self.device)
        ws, ws_bytes = workspace if workspace is not None else self.workspace(pk.T, n)
        if check:
            self._bad.zero_()
        rc = self.lib.pf_score(self.handle, _ptr(dp.ids), _ptr(dp.pos), _ptr(dp.segs), len(pk.segs),
                               _ptr(dp.work), len(pk.work), _ptr(dp.last_idx), n, pk.T,
                               ws, ws_bytes, _ptr(logits2), _ptr(p_yes), _ptr(self._bad),
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
        ws, ws_bytes = self.workspace(pk.T, n)
        cap = _lib.PfCapture(rows=_ptr(rows), n_rows=rows.numel(), gains=_ptr(gains), out=_ptr(out),
                             out_layer_stride=out.stride(0))
        st = self._stream(stream)
        rc = self.lib.pf_score_capture(self.handle, _ptr(dp.ids), _ptr(dp.pos), _ptr(dp.segs), len(pk.segs),
                                       _ptr(dp.work), len(pk.work), _ptr(dp.last_idx), n, pk.T, ws, ws_bytes,
                                       _ptr(logits2), _ptr(p_yes), _ptr(self._bad), ctypes.byref(cap), st)
        _lib.check(rc)
        (stream if stream is not None else torch.cuda.current_stream(self.device)).synchronize()
        return (out, logits2, p_yes) if return_scores else out

    def graph_runner(self, dp: DevicePacked):
        """Capture one pf_score pass over ``dp`` into a CUDA graph (private workspace and output
        buffers, so later calls cannot invalidate it).  Returns ``run() -> (logits2, p_yes)``;
        replay removes the ~200 host launches per pass."""
        import torch

        pk = dp.packed
        n = pk.n_items
        need = int(self.lib.pf_workspace_bytes(self.handle, pk.T, n))
        ws_t = torch.empty(need + 4096, dtype=torch.uint8, device=self.device)
        base = _ptr(ws_t)
        ws = ((base + 1023) & ~1023, ws_t.numel() - (((base + 1023) & ~1023) - base))
        logits2 = torch.empty((n, 2), dtype=torch.float32, device=self.device)
        p_yes = torch.empty((n,), dtype=torch.float32, device=self.device)
        self.score_device(dp, logits2, p_yes, workspace=ws)   # first launch sets kernel attributes
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.score_device(dp, logits2, p_yes, workspace=ws)

        def run():
            g.replay()
            return logits2, p_yes

        run.graph, run.keepalive = g, (ws_t, dp)
        return run

    def score_host(self, pp: PinnedPacked, stream=None) -> ScoredBatch:
        """End-to-end through the C-ABI with host buffers (H2D + forward + D2H + sync)."""
        pk = pp.packed
        ws, ws_bytes = self.workspace(pk.T, pk.n_items)
        rc = self.lib.pf_score_host(self.handle, _ptr(pp.ids), _ptr(pp.pos), _ptr(pp.segs),
                                    len(pk.segs), _ptr(pp.work), len(pk.work), _ptr(pp.last_idx),
                                    pk.n_items, pk.T, ws, ws_bytes, _ptr(pp.logits2), _ptr(pp.p_yes),
                                    self._stream(stream))
        _lib.check(rc)
        return ScoredBatch(pp.logits2.numpy().copy(), pp.p_yes.numpy().copy())

    def score_packed(self, packed: PackedBatch) -> ScoredBatch:
        import torch

        self.validate(packed)
        dp = DevicePacked(packed, self.device)
        logits2, p_yes = self.score_device(dp)
        torch.cuda.current_stream(self.device).synchronize()
        if int(self._bad[0].item()) != 0:
            raise ValueError("relevance_score: non-finite logits (SPEC.md:330)")
        return ScoredBatch(logits2.cpu().numpy(), p_yes.cpu().numpy())

    def validate(self, packed: PackedBatch) -> None:
        cfg = self.config
        if packed.T == 0 or packed.n_items == 0:
            raise ValueError("empty batch")
        if packed.ids.min() < 0 or packed.ids.max() >= cfg.vocab_size:
            raise ValueError("token id outside the vocabulary")
        if packed.pos.max() >= cfg.max_seq:
            raise ValueError(f"sequence exceeds max_seq={cfg.max_seq}")

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.lib.pf_model_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def score_shared_batch(model: PrefillScorer, shared: SharedBatch | Sequence[SharedBatch]) -> ScoredBatch:
    """SPEC.md:273-281 on the device: one packed forward over [prefix | suffix_0 | ...] for one
    or several requests; results order-aligned with the input items."""
    batches = [shared] if isinstance(shared, SharedBatch) else list(shared)
    return model.score_packed(pack_requests(batches, model.config.max_seq))
