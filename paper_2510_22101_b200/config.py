"""Model configuration — mirrors ``ModelConfig`` of the reference spec.

Reference: /root/reference/SPEC.md:177-180 (fields, defaults, invariants) and :222 (shape
discipline).  Two deliberate extensions for the B200 path:

* ``d_head`` is explicit.  The spec derives it as ``d_model / n_heads`` but the Qwen3-shaped
  configs have ``n_heads * d_head != d_model`` and GQA-group pruning (config C4) breaks the
  formula.  ``None`` keeps the spec default.
* ``precision`` adds ``"bf16"`` (the device arithmetic).  ``"f32"``/``"f64"`` remain the spec's
  CPU-oracle precisions.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field, replace


@dataclass(frozen=True)
class ModelConfig:
    n_layers: int = 8
    d_model: int = 64
    n_heads: int = 4
    n_kv_heads: int = 2
    d_ff: int = 256
    vocab_size: int = 32768
    rope_theta: float = 10000.0
    max_seq: int = 2048
    precision: str = "bf16"
    d_head: int | None = None
    rms_eps: float = 1e-6
    yes_id: int = 1
    no_id: int = 2

    def __post_init__(self):
        if self.d_head is None:
            if self.n_heads <= 0 or self.d_model % self.n_heads != 0:
                raise ValueError("d_model must be divisible by n_heads (SPEC.md:179)")
            object.__setattr__(self, "d_head", self.d_model // self.n_heads)
        for name in ("n_layers", "d_model", "n_heads", "n_kv_heads", "d_ff", "vocab_size",
                     "max_seq", "d_head"):
            if int(getattr(self, name)) < 1:
                raise ValueError(f"{name} must be >= 1")
        if self.n_heads % self.n_kv_heads != 0:
            raise ValueError("n_heads must be divisible by n_kv_heads (SPEC.md:179)")
        if self.d_head % 2 != 0:
            raise ValueError("d_head must be even (rotate-half RoPE)")
        if self.precision not in ("bf16", "f32", "f64"):
            raise ValueError(f"unknown precision {self.precision!r}")
        if not (0 <= self.yes_id < self.vocab_size and 0 <= self.no_id < self.vocab_size) \
                or self.yes_id == self.no_id:
            raise ValueError("yes_id/no_id must be distinct ids inside the vocabulary")

    # ------------------------------------------------------------------ derived shapes
    @property
    def q_width(self) -> int:
        return self.n_heads * self.d_head

    @property
    def kv_width(self) -> int:
        return self.n_kv_heads * self.d_head

    @property
    def d_ff_pad(self) -> int:
        """FFN width padded to a multiple of 128 for 16-byte TMA strides."""
        return -(-self.d_ff // 128) * 128

    def params_per_layer(self) -> int:
        d = self.d_model
        return (d * self.q_width + 2 * d * self.kv_width + self.q_width * d
                + 3 * d * self.d_ff + 2 * d)

    def param_count(self) -> int:
        """Closed-form parameter count: embedding + blocks + final norm + head."""
        return (self.vocab_size * self.d_model + self.n_layers * self.params_per_layer()
                + self.d_model + self.d_model * self.vocab_size)

    def linear_flops_per_token(self) -> int:
        """2*MACs of the QKV, O, gate/up and down GEMMs per token at true widths."""
        d = self.d_model
        return 2 * (d * (self.q_width + 2 * self.kv_width) + self.q_width * d + 3 * d * self.d_ff)

    def with_(self, **kw) -> "ModelConfig":
        return replace(self, **kw)

    def to_json(self) -> str:
        return json.dumps(asdict(self), sort_keys=True)

    @classmethod
    def from_json(cls, s: str) -> "ModelConfig":
        return cls(**json.loads(s))


@dataclass(frozen=True)
class RequestShape:
    """Synthetic request shape: one query prefix of ``prefix_len`` tokens shared by ``n_items``
    item suffixes of ``suffix_len`` tokens."""

    prefix_len: int
    n_items: int
    suffix_len: int
    n_requests: int = 1

    @property
    def tokens(self) -> int:
        return self.n_requests * (self.prefix_len + self.n_items * self.suffix_len)


# Config table of SURVEY.md §8 / BASELINE.md §2 (d_head explicit; † choices declared there).
C1 = ModelConfig(n_layers=2, d_model=256, n_heads=4, n_kv_heads=2, d_ff=1024, d_head=64)
C2 = ModelConfig(n_layers=28, d_model=1024, n_heads=16, n_kv_heads=8, d_ff=3072, d_head=128)
C3 = ModelConfig(n_layers=28, d_model=2048, n_heads=16, n_kv_heads=8, d_ff=6144, d_head=128)
C4 = ModelConfig(n_layers=28, d_model=2048, n_heads=10, n_kv_heads=5, d_ff=3686, d_head=128)
# Tiny configs with the device head width (d_head = 128) for fast GPU parity tests.
TINY = ModelConfig(n_layers=2, d_model=256, n_heads=2, n_kv_heads=1, d_ff=1024, d_head=128)
TINY_GQA = ModelConfig(n_layers=3, d_model=384, n_heads=4, n_kv_heads=2, d_ff=600, d_head=128)

CONFIGS = {"C1": C1, "C2": C2, "C3": C3, "C4": C4, "TINY": TINY, "TINY_GQA": TINY_GQA}

REQUESTS = {
    "C1": RequestShape(prefix_len=64, n_items=32, suffix_len=128),
    "C2": RequestShape(prefix_len=64, n_items=256, suffix_len=128),
    "C3": RequestShape(prefix_len=64, n_items=64, suffix_len=1024),
    "C4": RequestShape(prefix_len=64, n_items=256, suffix_len=100),
}
