"""Weights, seeded initialisation and the device-resident (B200) weight layout.

Reference: ``Weights`` / ``init_weights``.  The spec fixes
"seeded Gaussian init scaled by 1/sqrt(fan_in); deterministic per seed" and leaves the RNG and
draw order open; this module pins them (DESIGN.md §"pinned choices"):

* RNG: ``numpy.random.default_rng(seed)`` (PCG64), ``standard_normal(shape, dtype=float32)``.
* Draw order: token_embedding, then per layer W_q, W_k, W_v, W_o, W_gate, W_up, W_down, then
  the output head.  RMSNorm scales are 1.0 (not drawn).
* Scale: 1/sqrt(fan_in) with fan_in = rows of the ``x @ W`` matrix; the embedding is a one-hot
  lookup, fan_in = 1 (unit normal rows).
* Every matrix is rounded to bf16 (round-to-nearest-even), so the fp32 CPU oracle and the bf16
  device path use the *same* weight values and only activation precision differs
  (SURVEY.md §8c "parity weights").

Matrices follow the spec's row-vector convention ``y = x @ W`` ([in x out]).  ``DeviceWeights``
holds the K-major ([out x in]) bf16 copies the tcgen05 GEMMs consume (include/prefill_sm100.h).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterator

import numpy as np

from .config import ModelConfig

LAYER_FIELDS = ("W_q", "W_k", "W_v", "W_o", "W_gate", "W_up", "W_down")


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (ties to even); returns fp32 holding bf16 values."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32)
    lsb = (u >> np.uint32(16)) & np.uint32(1)
    r = (u + np.uint32(0x7FFF) + lsb) & np.uint32(0xFFFF0000)
    nan = np.isnan(x)
    out = r.view(np.float32).copy()
    if nan.any():
        out[nan] = np.nan
    return out


def layer_shapes(cfg: ModelConfig) -> dict[str, tuple[int, int]]:
    d, qw, kw, f = cfg.d_model, cfg.q_width, cfg.kv_width, cfg.d_ff
    return {"W_q": (d, qw), "W_k": (d, kw), "W_v": (d, kw), "W_o": (qw, d),
            "W_gate": (d, f), "W_up": (d, f), "W_down": (f, d)}


def draw_stream(cfg: ModelConfig, seed: int) -> Iterator[tuple[str, int, np.ndarray]]:
    """Yield (name, layer, bf16-rounded fp32 array) in the pinned draw order."""
    rng = np.random.default_rng(seed)
    emb = rng.standard_normal((cfg.vocab_size, cfg.d_model), dtype=np.float32)
    yield "token_embedding", -1, bf16_round(emb)
    del emb
    shapes = layer_shapes(cfg)
    for layer in range(cfg.n_layers):
        for name in LAYER_FIELDS:
            rows, cols = shapes[name]
            w = rng.standard_normal((rows, cols), dtype=np.float32)
            w *= np.float32(1.0 / np.sqrt(rows))
            yield name, layer, bf16_round(w)
    head = rng.standard_normal((cfg.d_model, cfg.vocab_size), dtype=np.float32)
    head *= np.float32(1.0 / np.sqrt(cfg.d_model))
    yield "head", -1, bf16_round(head)


@dataclass
class LayerWeights:
    W_q: np.ndarray
    W_k: np.ndarray
    W_v: np.ndarray
    W_o: np.ndarray
    W_gate: np.ndarray
    W_up: np.ndarray
    W_down: np.ndarray
    rms_attn: np.ndarray
    rms_mlp: np.ndarray


@dataclass
class Weights:
    """Host weights, spec layout.  Immutable by convention."""

    config: ModelConfig
    token_embedding: np.ndarray
    layers: list[LayerWeights]
    final_norm: np.ndarray
    head: np.ndarray  # [d_model x vocab]

    def param_count(self) -> int:
        n = self.token_embedding.size + self.final_norm.size + self.head.size
        for lw in self.layers:
            n += sum(getattr(lw, f).size for f in LAYER_FIELDS) + lw.rms_attn.size + lw.rms_mlp.size
        return n


def init_weights(config: ModelConfig, seed: int) -> Weights:
    """Seeded Gaussian init, bf16-representable values, host-resident."""
    layers: list[dict] = [dict() for _ in range(config.n_layers)]
    emb = head = None
    for name, layer, arr in draw_stream(config, seed):
        if name == "token_embedding":
            emb = arr
        elif name == "head":
            head = arr
        else:
            layers[layer][name] = arr
    ones = np.ones(config.d_model, dtype=np.float32)
    lws = [LayerWeights(rms_attn=ones.copy(), rms_mlp=ones.copy(), **lw) for lw in layers]
    return Weights(config, emb, lws, ones.copy(), head)


def rope_tables(cfg: ModelConfig) -> tuple[np.ndarray, np.ndarray]:
    """cos/sin [max_seq x d_head/2] for rotate-half RoPE, computed in float64 then cast to fp32:
    angle(p, i) = p * theta^(-2i/d_head)."""
    half = cfg.d_head // 2
    inv = cfg.rope_theta ** (-np.arange(half, dtype=np.float64) * 2.0 / cfg.d_head)
    ang = np.arange(cfg.max_seq, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


# ---------------------------------------------------------------------------- device layout
def interleave_gate_up(w_gate_t: "np.ndarray", w_up_t: "np.ndarray", d_ff_pad: int):
    """[F x d] gate/up (K-major) -> [2*F_pad x d] with per-128-neuron blocks [gate_j ; up_j].
    Works on numpy arrays or torch tensors (torch path used for large models)."""
    f, d = w_gate_t.shape
    nb = d_ff_pad // 128
    if hasattr(w_gate_t, "new_zeros"):
        out = w_gate_t.new_zeros((nb, 2, 128, d))
        g = w_gate_t.new_zeros((d_ff_pad, d)); g[:f] = w_gate_t
        u = w_up_t.new_zeros((d_ff_pad, d)); u[:f] = w_up_t
    else:
        out = np.zeros((nb, 2, 128, d), dtype=w_gate_t.dtype)
        g = np.zeros((d_ff_pad, d), dtype=w_gate_t.dtype); g[:f] = w_gate_t
        u = np.zeros((d_ff_pad, d), dtype=w_up_t.dtype); u[:f] = w_up_t
    out[:, 0] = g.reshape(nb, 128, d)
    out[:, 1] = u.reshape(nb, 128, d)
    return out.reshape(2 * d_ff_pad, d)


@dataclass
class DeviceWeights:
    """bf16 K-major device copies (torch tensors) + fp32 norm scales / head columns."""

    config: ModelConfig
    embedding: object
    w_qkv: list
    w_o: list
    w_gu: list
    w_down: list
    ln_attn: list
    ln_mlp: list
    ln_final: object
    w_yes: object
    w_no: object
    rope_cos: object
    rope_sin: object
    keepalive: list = field(default_factory=list)

    def nbytes(self) -> int:
        tot = 0
        for t in [self.embedding, *self.w_qkv, *self.w_o, *self.w_gu, *self.w_down]:
            tot += t.numel() * t.element_size()
        return tot


def _to_device_layer(cfg: ModelConfig, lw: dict, device, g_attn=None, g_mlp=None):
    """RMSNorm is fused into the GEMM epilogues on the device, so the norm gains are folded into
    the input rows of W_q/W_k/W_v and W_gate/W_up (fp32 product, then bf16).  Gains of 1.0 (the
    pinned init) leave the weights bit-identical."""
    import torch

    def dev(a, g=None):
        a = np.ascontiguousarray(a, dtype=np.float32)
        if g is not None and not np.all(g == 1.0):
            a = a * np.asarray(g, dtype=np.float32)[:, None]
        return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=torch.bfloat16)

    wq, wk, wv = dev(lw["W_q"], g_attn), dev(lw["W_k"], g_attn), dev(lw["W_v"], g_attn)
    w_qkv = torch.cat([wq, wk, wv], dim=1).t().contiguous()
    w_o = dev(lw["W_o"]).t().contiguous()
    w_gu = interleave_gate_up(dev(lw["W_gate"], g_mlp).t(), dev(lw["W_up"], g_mlp).t(),
                              cfg.d_ff_pad).contiguous()
    wd = dev(lw["W_down"]).t()
    w_down = torch.zeros((cfg.d_model, cfg.d_ff_pad), dtype=torch.bfloat16, device=device)
    w_down[:, : cfg.d_ff] = wd
    return w_qkv, w_o, w_gu, w_down


def to_device(weights: Weights, device="cuda") -> DeviceWeights:
    """Lay out host ``Weights`` for the device (transpose to K-major, fuse QKV, interleave
    gate/up, zero-pad d_ff to a multiple of 128)."""
    import torch

    cfg = weights.config
    dw = DeviceWeights(cfg, None, [], [], [], [], [], [], None, None, None, None, None)
    dw.embedding = torch.from_numpy(weights.token_embedding).to(device=device, dtype=torch.bfloat16)
    for lw in weights.layers:
        d = {f: getattr(lw, f) for f in LAYER_FIELDS}
        a, b, c, e = _to_device_layer(cfg, d, device, lw.rms_attn, lw.rms_mlp)
        dw.w_qkv.append(a); dw.w_o.append(b); dw.w_gu.append(c); dw.w_down.append(e)
        dw.ln_attn.append(torch.from_numpy(lw.rms_attn).to(device))
        dw.ln_mlp.append(torch.from_numpy(lw.rms_mlp).to(device))
    _finish(dw, cfg, weights.final_norm, weights.head, device)
    return dw


def init_device_weights(config: ModelConfig, seed: int, device="cuda") -> DeviceWeights:
    """Same values as ``to_device(init_weights(config, seed))`` but streamed tensor by tensor,
    so multi-GB models never sit in host memory at once."""
    import torch

    cfg = config
    dw = DeviceWeights(cfg, None, [], [], [], [], [], [], None, None, None, None, None)
    ones = np.ones(cfg.d_model, dtype=np.float32)
    cur: dict = {}
    for name, layer, arr in draw_stream(cfg, seed):
        if name == "token_embedding":
            dw.embedding = torch.from_numpy(arr).to(device=device, dtype=torch.bfloat16)
        elif name == "head":
            _finish(dw, cfg, ones, arr, device)
        else:
            cur[name] = arr
            if name == LAYER_FIELDS[-1]:
                a, b, c, e = _to_device_layer(cfg, cur, device)
                dw.w_qkv.append(a); dw.w_o.append(b); dw.w_gu.append(c); dw.w_down.append(e)
                dw.ln_attn.append(torch.from_numpy(ones).to(device))
                dw.ln_mlp.append(torch.from_numpy(ones).to(device))
                cur = {}
    return dw


def _finish(dw: DeviceWeights, cfg: ModelConfig, final_norm, head, device):
    import torch

    dw.ln_final = torch.from_numpy(np.ascontiguousarray(final_norm, dtype=np.float32)).to(device)
    dw.w_yes = torch.from_numpy(np.ascontiguousarray(head[:, cfg.yes_id])).to(device)
    dw.w_no = torch.from_numpy(np.ascontiguousarray(head[:, cfg.no_id])).to(device)
    cos, sin = rope_tables(cfg)
    dw.rope_cos = torch.from_numpy(cos).to(device)
    dw.rope_sin = torch.from_numpy(sin).to(device)
