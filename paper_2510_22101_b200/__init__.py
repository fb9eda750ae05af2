"""B200-native (sm_100a) prefill-only shared-prefix relevance scoring.

Drop-in for the scoring hot path of the reference package ``prefrank`` (arxiv 2510.22101):
``ModelConfig``, ``init_weights``, ``split_shared_prefix``, ``score_shared_batch``,
``relevance_score``, ``rank_items``, ``throughput_gain`` and the pruning shape contract keep the
reference spec's names and meanings.  The arithmetic
runs in libprefill_sm100.so (hand-written tcgen05/TMA kernels) behind a C-ABI.
"""

from .calibration import CalibrationSet, capture_calibration, prune_mlp_neurons_calibrated, sample_positions
from .config import CONFIGS, REQUESTS, ModelConfig, RequestShape
from .prefixcache import (AttentionPartial, PackedBatch, SharedBatch, concat_packed, merge_attention,
                          pack_requests, pack_token_lists, split_shared_prefix, throughput_gain)
from .scoring import RankedList, RelevanceScore, rank_items, relevance_score, top_k
from .weights import DeviceWeights, Weights, init_device_weights, init_weights, to_device

__all__ = [
    "CONFIGS", "REQUESTS", "ModelConfig", "RequestShape", "AttentionPartial", "PackedBatch",
    "SharedBatch", "concat_packed", "merge_attention", "pack_requests", "pack_token_lists", "split_shared_prefix",
    "throughput_gain", "RankedList", "RelevanceScore", "rank_items", "relevance_score", "top_k",
    "DeviceWeights", "Weights", "init_device_weights", "init_weights", "to_device",
    "PrefillScorer", "score_shared_batch", "forward_prefill", "forward_with_prefix", "KVCache", "scorer_for",
    "CalibrationSet", "capture_calibration", "prune_mlp_neurons_calibrated", "sample_positions",
]


def __getattr__(name):
    # engine imports torch lazily; keep `import paper_2510_22101_b200` light for CPU tooling
    if name in ("PrefillScorer", "score_shared_batch", "ScoredBatch", "DevicePacked", "PinnedPacked",
                "forward_prefill", "forward_with_prefix", "KVCache", "scorer_for"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)
