"""Cross-check of the oracle's transformer arithmetic against an independent implementation:
Hugging Face transformers' LlamaForCausalLM, loaded with the oracle's weights, in float64.

The reference ships no model code, so no reference-executed logits exist.  The
oracle's open choices (pre-norm RMSNorm, rotate-half RoPE with angle p*theta^(-2i/dh),
GQA head h -> kv head h // (H/Hkv), scale 1/sqrt(dh), SwiGLU, untied head) are exactly Llama's, so
HF Llama computes the same function; this script records its last-token logits as golden vectors.

    python tests/golden/make_hf_llama_golden.py      (writes tests/golden/hf_llama_logits.json)

HF computes its RoPE tables, RMSNorm statistics and attention softmax in float32 on purpose; those three
are replaced by the same formulas in float64, so the comparison runs the HF attention / GQA / MLP /
residual code at float64 precision.

Recorded per (config, sequence): token ids, HF float64 logits at yes/no and at 256 fixed vocabulary
indices, plus the sum and the sum of squares of all logits (pins the full vector).  The CPU test
tests/test_oracle_hf.py checks the oracle against these values (and against HF live when transformers
is importable).
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "hf_llama_logits.json")

# (name, n_layers, d_model, n_heads, n_kv_heads, d_head, d_ff): C1 (BASELINE configs[0] shape),
# a GQA model with n_heads*d_head != d_model, and a C4-like pruned head/FFN ratio (10/5 heads).
CONFIGS = [("C1", 2, 256, 4, 2, 64, 1024), ("GQA_DH128", 3, 384, 4, 2, 128, 600),
           ("PRUNED_10_5", 2, 640, 10, 5, 128, 370)]
SEQ_LENS = (1, 37, 300)
SAMPLE = np.linspace(0, 32767, 256).astype(np.int64)


class Cfg:
    def __init__(self, L, d, H, Hkv, dh, f):
        self.n_layers, self.d_model, self.n_heads, self.n_kv_heads, self.d_head, self.d_ff = L, d, H, Hkv, dh, f
        self.vocab_size, self.rope_theta, self.max_seq = 32768, 10000.0, 2048


def hf_model(cfg, W):
    import torch
    from transformers import LlamaConfig, LlamaForCausalLM

    hc = LlamaConfig(vocab_size=cfg.vocab_size, hidden_size=cfg.d_model, intermediate_size=cfg.d_ff,
                     num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.n_heads,
                     num_key_value_heads=cfg.n_kv_heads, head_dim=cfg.d_head, hidden_act="silu",
                     max_position_embeddings=cfg.max_seq, rms_norm_eps=1e-6,
                     rope_parameters={"rope_theta": cfg.rope_theta, "rope_type": "default"},
                     attention_bias=False, mlp_bias=False, tie_word_embeddings=False)
    hc._attn_implementation = "eager"
    m = LlamaForCausalLM(hc).to(torch.float64).eval()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(t(W.token_embedding))
        for l, lw in enumerate(W.layers):
            blk = m.model.layers[l]
            blk.self_attn.q_proj.weight.copy_(t(lw["W_q"].T))
            blk.self_attn.k_proj.weight.copy_(t(lw["W_k"].T))
            blk.self_attn.v_proj.weight.copy_(t(lw["W_v"].T))
            blk.self_attn.o_proj.weight.copy_(t(lw["W_o"].T))
            blk.mlp.gate_proj.weight.copy_(t(lw["W_gate"].T))
            blk.mlp.up_proj.weight.copy_(t(lw["W_up"].T))
            blk.mlp.down_proj.weight.copy_(t(lw["W_down"].T))
            blk.input_layernorm.weight.copy_(t(lw["rms_attn"]))
            blk.post_attention_layernorm.weight.copy_(t(lw["rms_mlp"]))
        m.model.norm.weight.copy_(t(W.final_norm))
        m.lm_head.weight.copy_(t(W.head.T))
    # HF builds its RoPE tables in float32 on purpose (LlamaRotaryEmbedding.forward forces it); the
    # oracle tabulates in float64.  Same formula, float64 tables, so that only the
    # attention / MLP / norm code paths are compared at float64 precision.
    theta, dh = cfg.rope_theta, cfg.d_head
    inv = torch.from_numpy(theta ** (-np.arange(0, dh, 2, dtype=np.float64) / dh))

    def rope64(x, position_ids):
        ang = position_ids[..., None].to(torch.float64) * inv
        emb = torch.cat([ang, ang], dim=-1)
        return emb.cos().to(x.dtype), emb.sin().to(x.dtype)

    m.model.rotary_emb.forward = rope64

    # LlamaRMSNorm also computes in float32 internally; same formula, float64
    def rms64(mod):
        def fwd(h):
            return mod.weight * (h * torch.rsqrt(h.pow(2).mean(-1, keepdim=True) + mod.variance_epsilon))
        return fwd

    for mod in m.modules():
        if type(mod).__name__ == "LlamaRMSNorm":
            mod.forward = rms64(mod)

    # eager attention takes its softmax with dtype=float32; keep float64 inputs in float64
    import transformers.models.llama.modeling_llama as ML

    class _F:
        def __getattr__(self, name):
            return getattr(torch.nn.functional, name)

        @staticmethod
        def softmax(x, dim=-1, dtype=None):
            return torch.nn.functional.softmax(x, dim=dim, dtype=torch.float64 if x.dtype == torch.float64 else dtype)

    class _NN:
        def __getattr__(self, name):
            return getattr(torch.nn, name)

        functional = _F()

    ML.nn = _NN()
    return m


def hf_last_logits(m, tokens):
    import torch

    with torch.no_grad():
        out = m(input_ids=torch.tensor([tokens], dtype=torch.long), use_cache=False)
    return out.logits[0, -1].numpy()


def build_weights(name):
    """Oracle weights of config ``name`` (init_weights seed 3) with non-unit RMSNorm gains drawn from
    default_rng(11), so the norm weights are exercised too.  Returns (cfg, weights, rng) - the rng
    continues into the token draws."""
    import oracle.model as OM

    _, L, d, H, Hkv, dh, f = next(c for c in CONFIGS if c[0] == name)
    cfg = Cfg(L, d, H, Hkv, dh, f)
    W = OM.init_weights(cfg, seed=3)
    rng = np.random.default_rng(11)
    for lw in W.layers:
        lw["rms_attn"] = (1.0 + 0.25 * rng.standard_normal(d)).astype(np.float32)
        lw["rms_mlp"] = (1.0 + 0.25 * rng.standard_normal(d)).astype(np.float32)
    W.final_norm = (1.0 + 0.25 * rng.standard_normal(d)).astype(np.float32)
    return cfg, W, rng


def main():
    import oracle.model as OM

    rec = []
    for name, L, d, H, Hkv, dh, f in CONFIGS:
        cfg, W, rng = build_weights(name)
        m = hf_model(cfg, W)
        W64 = W.astype(np.float64)
        for S in SEQ_LENS:
            toks = [3] + [int(x) for x in rng.integers(16, cfg.vocab_size, S - 1)] if S > 1 else [11]
            ref = hf_last_logits(m, toks)
            mine, _ = OM.forward_prefill(W64, toks)
            err = float(np.max(np.abs(mine - ref)))
            print(f"{name} S={S}: max |oracle f64 - HF Llama f64| = {err:.3e}")
            rec.append({"config": name, "dims": [L, d, H, Hkv, dh, f], "weight_seed": 3, "gain_seed": 11,
                        "tokens": toks, "yes": float(ref[1]), "no": float(ref[2]),
                        "sample_idx": SAMPLE.tolist(), "sample": [float(v) for v in ref[SAMPLE]],
                        "sum": float(ref.sum()), "sumsq": float((ref * ref).sum()),
                        "oracle_max_abs_err": err})
    with open(OUT, "w") as fh:
        json.dump({"generator": "tests/golden/make_hf_llama_golden.py", "hf_model": "LlamaForCausalLM float64",
                   "records": rec}, fh)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
