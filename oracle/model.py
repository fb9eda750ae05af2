"""Oracle restatement of the reference ``model`` module.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  numpy, precision f32 or f64.

Architecture: decoder-only, pre-norm blocks
    x += Wo . attn(RoPE(Wq n1(x)), RoPE(Wk n1(x)), Wv n1(x))        (GQA, causal)
    x += Wdown . (silu(Wgate n2(x)) * Wup n2(x))                      (SwiGLU)
final RMSNorm on the last position only, untied head -> full [vocab] logits.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

LAYER_FIELDS = ("W_q", "W_k", "W_v", "W_o", "W_gate", "W_up", "W_down")


# ----------------------------------------------------------------------------- init
def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as fp32 (restated independently of the product)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    bits = x.view(np.uint32).astype(np.uint64)
    rounded = (bits + 0x7FFF + ((bits >> 16) & 1)) & 0xFFFF0000
    return rounded.astype(np.uint32).view(np.float32)


@dataclass
class OracleWeights:
    cfg: object
    token_embedding: np.ndarray
    layers: list
    final_norm: np.ndarray
    head: np.ndarray

    def astype(self, dtype) -> "OracleWeights":
        cast = lambda a: a.astype(dtype, copy=False)
        layers = [{k: cast(v) for k, v in lw.items()} for lw in self.layers]
        return OracleWeights(self.cfg, cast(self.token_embedding), layers, cast(self.final_norm),
                             cast(self.head))


def dims(cfg):
    d_head = cfg.d_head if getattr(cfg, "d_head", None) else cfg.d_model // cfg.n_heads
    return cfg.d_model, cfg.n_heads, cfg.n_kv_heads, d_head, cfg.d_ff


def init_weights(cfg, seed: int) -> OracleWeights:
    """seeded Gaussian, 1/sqrt(fan_in).  Pinned: PCG64 default_rng(seed);
    float32 standard normals drawn in the order embedding, per layer (W_q, W_k, W_v, W_o, W_gate,
    W_up, W_down), head; embedding fan_in = 1; RMSNorm scales = 1; all matrices bf16-rounded."""
    d, H, Hkv, dh, f = dims(cfg)
    rng = np.random.default_rng(seed)
    emb = bf16_round(rng.standard_normal((cfg.vocab_size, d), dtype=np.float32))
    shapes = {"W_q": (d, H * dh), "W_k": (d, Hkv * dh), "W_v": (d, Hkv * dh), "W_o": (H * dh, d),
              "W_gate": (d, f), "W_up": (d, f), "W_down": (f, d)}
    layers = []
    for _ in range(cfg.n_layers):
        lw = {}
        for name in LAYER_FIELDS:
            r, c = shapes[name]
            w = rng.standard_normal((r, c), dtype=np.float32) * np.float32(1.0 / np.sqrt(r))
            lw[name] = bf16_round(w)
        lw["rms_attn"] = np.ones(d, dtype=np.float32)
        lw["rms_mlp"] = np.ones(d, dtype=np.float32)
        layers.append(lw)
    head = bf16_round(rng.standard_normal((d, cfg.vocab_size), dtype=np.float32)
                      * np.float32(1.0 / np.sqrt(d)))
    return OracleWeights(cfg, emb, layers, np.ones(d, dtype=np.float32), head)


def param_count(cfg) -> int:
    d, H, Hkv, dh, f = dims(cfg)
    per_layer = d * H * dh + 2 * d * Hkv * dh + H * dh * d + 3 * d * f + 2 * d
    return cfg.vocab_size * d + cfg.n_layers * per_layer + d + d * cfg.vocab_size


# ----------------------------------------------------------------------------- ops
def rmsnorm(x: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    ms = np.mean(x * x, axis=-1, keepdims=True)
    return x / np.sqrt(ms + x.dtype.type(eps)) * g


def rope_tables(cfg, dtype):
    _, _, _, dh, _ = dims(cfg)
    half = dh // 2
    inv = cfg.rope_theta ** (-np.arange(half, dtype=np.float64) * 2.0 / dh)
    ang = np.arange(cfg.max_seq, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(dtype), np.sin(ang).astype(dtype)


def apply_rope(x: np.ndarray, pos: np.ndarray, cos: np.ndarray, sin: np.ndarray) -> np.ndarray:
    """Rotate-half: (x1, x2) -> (x1 c - x2 s, x2 c + x1 s) per head; x [S, nh, dh]."""
    half = x.shape[-1] // 2
    c = cos[pos][:, None, :]
    s = sin[pos][:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def silu(x):
    return x / (1.0 + np.exp(-x))


@dataclass
class AttentionPartial:
    output: np.ndarray  # [H, S, dh]
    lse: np.ndarray     # [H, S]


def attention_partial(q, k, v, causal: bool, n_rep: int) -> AttentionPartial:
    """Softmax attention of q [S,H,dh] over k,v [N,Hkv,dh] with max-subtraction.
    ``causal``: query i sees keys j <= i (requires N == S)."""
    S, H, dh = q.shape
    N = k.shape[0]
    kk = np.repeat(k, n_rep, axis=1).transpose(1, 2, 0)  # [H, dh, N]
    vv = np.repeat(v, n_rep, axis=1).transpose(1, 0, 2)  # [H, N, dh]
    s = np.matmul(q.transpose(1, 0, 2), kk) * q.dtype.type(1.0 / np.sqrt(dh))  # [H, S, N]
    if causal:
        mask = np.triu(np.ones((S, N), dtype=bool), k=1)
        s = np.where(mask[None], -np.inf, s)
    m = np.max(s, axis=-1, keepdims=True)
    p = np.exp(s - m)
    l = np.sum(p, axis=-1, keepdims=True)
    out = np.matmul(p, vv) / l
    lse = (m + np.log(l))[..., 0]
    return AttentionPartial(out, lse)


def merge_attention(a: AttentionPartial, b: AttentionPartial) -> np.ndarray:
    """(e^{lse_a} o_a + e^{lse_b} o_b)/(e^{lse_a}+e^{lse_b}), max-subtracted."""
    m = np.maximum(a.lse, b.lse)
    wa = np.exp(a.lse - m)[..., None]
    wb = np.exp(b.lse - m)[..., None]
    return (wa * a.output + wb * b.output) / (wa + wb)


# ----------------------------------------------------------------------------- forward
@dataclass
class KVCache:
    """per layer K, V [n_kv_heads x seq_len x d_head] (stored [S, Hkv, dh])."""

    k: list = field(default_factory=list)
    v: list = field(default_factory=list)

    @property
    def seq_len(self) -> int:
        return 0 if not self.k else int(self.k[0].shape[0])


def _forward(W: OracleWeights, tokens, prefix: KVCache | None, eps: float, capture: bool = False):
    cfg = W.cfg
    d, H, Hkv, dh, f = dims(cfg)
    dt = W.token_embedding.dtype
    tokens = np.asarray(tokens, dtype=np.int64)
    S = len(tokens)
    P = prefix.seq_len if prefix is not None else 0
    if S < 1:
        raise ValueError("forward: empty token sequence")
    if P + S > cfg.max_seq:
        raise ValueError(f"forward: length {P + S} exceeds max_seq {cfg.max_seq}")
    if prefix is not None and prefix.seq_len > 0 and len(prefix.k) != cfg.n_layers:
        raise ValueError("forward_with_prefix: layer-count mismatch")
    cos, sin = rope_tables(cfg, dt)
    pos = np.arange(P, P + S)
    x = W.token_embedding[tokens].astype(dt)
    cache = KVCache()
    captured = []
    n_rep = H // Hkv
    for l, lw in enumerate(W.layers):
        h = rmsnorm(x, lw["rms_attn"], eps)
        q = apply_rope((h @ lw["W_q"]).reshape(S, H, dh), pos, cos, sin)
        k = apply_rope((h @ lw["W_k"]).reshape(S, Hkv, dh), pos, cos, sin)
        v = (h @ lw["W_v"]).reshape(S, Hkv, dh)
        part = attention_partial(q, k, v, causal=True, n_rep=n_rep)
        if P > 0:
            pre = attention_partial(q, prefix.k[l], prefix.v[l], causal=False, n_rep=n_rep)
            o = merge_attention(pre, part)
        else:
            o = part.output
        x = x + o.transpose(1, 0, 2).reshape(S, H * dh) @ lw["W_o"]
        h2 = rmsnorm(x, lw["rms_mlp"], eps)
        if capture:
            captured.append(h2.copy())
        x = x + (silu(h2 @ lw["W_gate"]) * (h2 @ lw["W_up"])) @ lw["W_down"]
        cache.k.append(k)
        cache.v.append(v)
    last = rmsnorm(x[-1:], W.final_norm, eps)[0]
    logits = last @ W.head
    if capture:
        return logits, cache, captured
    return logits, cache


def forward_prefill(W: OracleWeights, tokens, eps: float = 1e-6, capture: bool = False):
    """SPEC.md:200-208 -> (last-token logits [vocab], KVCache); with ``capture`` also the per-layer
    MLP inputs rmsnorm(x_l) * g_l [S x d] ("capture flag records MLP inputs")."""
    return _forward(W, tokens, None, eps, capture)


def forward_with_prefix(W: OracleWeights, prefix_cache: KVCache, suffix_tokens, eps: float = 1e-6):
    """suffix positions continue at the prefix length."""
    if len(suffix_tokens) == 0:
        raise ValueError("forward_with_prefix: empty suffix")
    return _forward(W, suffix_tokens, prefix_cache, eps)
