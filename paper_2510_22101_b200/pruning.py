"""Structured-pruning shape contract consumed by the B200 kernels.

Reference: pruning module.  The offline search (OSSCAR stand-in,
calibration capture, sensitivity sweeps, SFT) is out of scope; what the hot path needs is the
*result*: compacted dense weights at the pruned widths, described by per-layer keep-sets.

* ``PruneRecipe`` — SPEC.md:462-465.
* ``prune_mlp_neurons(weights, keep)`` — SPEC.md:477-485 output contract: per layer a keep-set S
  of size k = round((1 - sparsity) * d_ff), uniform across layers; a SwiGLU neuron
  j = (W_gate col j, W_up col j, W_down row j); new config d_ff = k.  The refit of
  W_down (least squares) belongs to the offline search; pass refit rows via ``w_down_rows``.
* ``remove_layers(weights, indices)`` — SPEC.md:486-494: blocks deleted, the rest renumbered.
* ``prune_kv_groups(weights, keep_groups)`` — extension for config C4 (SURVEY.md §7 "Head pruning
  is not in the spec"): whole GQA groups (one kv head + its H/Hkv query heads) are removed so
  n_heads % n_kv_heads == 0 still holds.
* ``select_keep_by_norm`` — a deterministic magnitude heuristic to produce keep-sets for tests
  and benchmarks (NOT the paper's OSSCAR; named as such).
Kernels receive compacted weights only (no runtime masking); the device layout zero-pads d_ff to
a multiple of 128 at load (exact: silu(0)*0 = 0 and zero W_down rows add nothing).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Sequence

import numpy as np

from .weights import LayerWeights, Weights


@dataclass(frozen=True)
class PruneRecipe:
    mlp_sparsity: float = 0.0
    layers_to_remove: tuple = ()
    sft_after_each_stage: bool = False
    kv_groups_to_keep: int | None = None   # extension: GQA-group pruning (C4)

    def __post_init__(self):
        if not (0.0 <= self.mlp_sparsity < 1.0):
            raise ValueError("mlp_sparsity must be in [0, 1)")


def kept_width(d_ff: int, sparsity: float) -> int:
    k = int(round((1.0 - sparsity) * d_ff))
    if k < 1:
        raise ValueError("pruned d_ff must be >= 1")
    return k


def _check_keep(keep: Sequence[int], n: int, what: str) -> np.ndarray:
    k = np.asarray(sorted(set(int(i) for i in keep)), dtype=np.int64)
    if len(k) != len(keep) or k.size == 0 or k[0] < 0 or k[-1] >= n:
        raise ValueError(f"{what}: keep-set must be distinct indices in [0, {n})")
    return k


def prune_mlp_neurons(weights: Weights, keep, w_down_rows=None) -> Weights:
    """Two call forms:
    * ``prune_mlp_neurons(weights, calib: CalibrationSet, sparsity)`` -- the reference signature
      (SPEC.md:477): calibrated keep-sets + W_down refit (``calibration.py``, OSSCAR stand-in);
    * ``prune_mlp_neurons(weights, keep_sets, w_down_rows=None)`` -- apply given per-layer keep-sets
      (and optional refit rows): the shape contract the kernels consume."""
    from .calibration import CalibrationSet, prune_mlp_neurons_calibrated

    if isinstance(keep, CalibrationSet):
        if w_down_rows is None:
            raise ValueError("prune_mlp_neurons(weights, calib, sparsity): sparsity required")
        return prune_mlp_neurons_calibrated(weights, keep, float(w_down_rows))
    cfg = weights.config
    if len(keep) != cfg.n_layers:
        raise ValueError("one keep-set per layer")
    sizes = {len(k) for k in keep}
    if len(sizes) != 1:
        raise ValueError("uniform per-layer sparsity (SPEC.md:523): keep-sets must have equal size")
    k = sizes.pop()
    layers = []
    for l, lw in enumerate(weights.layers):
        idx = _check_keep(keep[l], cfg.d_ff, f"layer {l}")
        if w_down_rows is None:
            down = lw.W_down[idx]
        else:
            # refit rows are aligned with the caller's keep-set order; neurons are taken in ascending
            # index order, so reorder the rows by the same permutation
            down = np.asarray(w_down_rows[l], dtype=np.float32)
            if down.shape != (k, cfg.d_model):
                raise ValueError("refit W_down rows must be [k x d_model]")
            down = down[np.argsort(np.asarray(keep[l], dtype=np.int64), kind="stable")]
        layers.append(replace(lw, W_gate=lw.W_gate[:, idx].copy(), W_up=lw.W_up[:, idx].copy(),
                              W_down=down.copy()))
    return Weights(replace(cfg, d_ff=k), weights.token_embedding, layers, weights.final_norm,
                   weights.head)


def remove_layers(weights: Weights, indices: Sequence[int]) -> Weights:
    cfg = weights.config
    drop = set(int(i) for i in indices)
    if any(i < 0 or i >= cfg.n_layers for i in drop):
        raise ValueError("layer index out of range")
    if len(drop) >= cfg.n_layers:
        raise ValueError("at least one layer must remain (SPEC.md:488)")
    layers = [lw for i, lw in enumerate(weights.layers) if i not in drop]
    return Weights(replace(cfg, n_layers=len(layers)), weights.token_embedding, layers,
                   weights.final_norm, weights.head)


def prune_kv_groups(weights: Weights, keep_groups: Sequence[int]) -> Weights:
    cfg = weights.config
    keep = _check_keep(keep_groups, cfg.n_kv_heads, "kv groups")
    r, dh = cfg.n_heads // cfg.n_kv_heads, cfg.d_head
    q_cols = np.concatenate([np.arange((g * r + i) * dh, (g * r + i + 1) * dh) for g in keep for i in range(r)])
    kv_cols = np.concatenate([np.arange(g * dh, (g + 1) * dh) for g in keep])
    layers = [replace(lw, W_q=lw.W_q[:, q_cols].copy(), W_k=lw.W_k[:, kv_cols].copy(),
                      W_v=lw.W_v[:, kv_cols].copy(), W_o=lw.W_o[q_cols].copy())
              for lw in weights.layers]
    cfg2 = replace(cfg, n_heads=len(keep) * r, n_kv_heads=len(keep))
    return Weights(cfg2, weights.token_embedding, layers, weights.final_norm, weights.head)


def select_keep_by_norm(weights: Weights, sparsity: float) -> list[np.ndarray]:
    """Magnitude heuristic (not OSSCAR): keep the k neurons with the largest
    ||W_gate[:, j]|| * ||W_up[:, j]|| * ||W_down[j, :]|| per layer; ties by index."""
    k = kept_width(weights.config.d_ff, sparsity)
    out = []
    for lw in weights.layers:
        score = (np.linalg.norm(lw.W_gate, axis=0) * np.linalg.norm(lw.W_up, axis=0)
                 * np.linalg.norm(lw.W_down, axis=1))
        order = np.lexsort((np.arange(score.size), -score))
        out.append(np.sort(order[:k]))
    return out


def apply_recipe(weights: Weights, recipe: PruneRecipe) -> Weights:
    """prune_mlp (norm heuristic keep-sets) -> remove_layers -> optional GQA-group pruning."""
    w = weights
    if recipe.mlp_sparsity > 0:
        w = prune_mlp_neurons(w, select_keep_by_norm(w, recipe.mlp_sparsity))
    if recipe.layers_to_remove:
        w = remove_layers(w, recipe.layers_to_remove)
    if recipe.kv_groups_to_keep is not None and recipe.kv_groups_to_keep < w.config.n_kv_heads:
        w = prune_kv_groups(w, range(recipe.kv_groups_to_keep))
    return w
