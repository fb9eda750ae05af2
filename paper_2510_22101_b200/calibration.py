"""Calibration capture and calibrated MLP-neuron pruning.

Reference: the pruning module of /root/reference/SPEC.md:453-533.
* ``CalibrationSet``: per-layer matrices of captured MLP inputs, rows = sampled
  token positions, columns = d_model; all layers have the same row count.
* ``capture_calibration(model, prompts, position_budget, seed)``: positions are
  subsampled uniformly without replacement over all tokens of all prompts (seeded PCG64), and
  their MLP inputs ``rmsnorm(x_l) * g_l`` are captured on the GPU by ``pf_score_capture``.  That is
  the reference ``forward_prefill`` capture flag, running the product kernels.
* ``prune_mlp_neurons_calibrated(weights, calib, sparsity)`` is the OSSCAR
  stand-in the spec names.  Per layer it takes the hidden activations ``H = silu(X W_gate) *
  (X W_up)`` of the captured inputs and picks a keep-set S of size k = round((1 - s) d_ff) by
  greedy backward elimination.  Each step minimises ``||H W_down - H_S W~_S||_F`` with a
  least-squares refit ``W~_S``.  The refit rows replace W_down.  A singular Gram matrix falls back
  to ridge ``lambda = 1e-6 trace/n`` with a warning.

The greedy step uses the closed form of the refit objective (an optimal-brain-surgeon downdate):
with ``G = H^T H``, ``A = G W``, ``M = G_SS^-1`` and ``B = M A_S`` (the current refit), removing
neuron j raises the error by ``||B_j||^2 / M_jj``, and ``M``, ``B`` are downdated in rank-1 form.
One step costs O(n^2 + n d) instead of a refit per candidate.  Both it and the search are host
math (float64 torch, on the GPU when available).  ``oracle/calibration.py`` restates them by
direct least squares and exhaustive search (test infrastructure).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .pruning import kept_width, prune_mlp_neurons
from .weights import Weights


@dataclass
class CalibrationSet:
    layers: list            # per layer: float32 [n_rows x d_model] captured MLP inputs
    n_tokens: int           # positions actually captured (= rows per layer)
    sources: np.ndarray     # int64 [n_rows, 2]: (prompt index, position) of each row

    def __post_init__(self):   # layers: numpy arrays, or device torch tensors (to_host=False)
        if len({int(x.shape[0]) for x in self.layers}) > 1:
            raise ValueError("CalibrationSet: per-layer row counts must be equal (SPEC.md:460)")


def sample_positions(prompt_lens: Sequence[int], budget: int, seed: int = 0) -> np.ndarray:
    """Uniform subsample of ``min(budget, total)`` positions, without replacement, over the
    concatenation of all prompts (PCG64 ``default_rng(seed).choice``), returned sorted as
    (prompt, position) pairs."""
    if budget < 1:
        raise ValueError("capture_calibration: budget must be >= 1 (SPEC.md:470)")
    lens = np.asarray(prompt_lens, dtype=np.int64)
    if lens.size == 0 or lens.sum() == 0:
        raise ValueError("capture_calibration: empty prompt set (SPEC.md:472)")
    total = int(lens.sum())
    n = min(int(budget), total)
    flat = np.sort(np.random.default_rng(seed).choice(total, size=n, replace=False))
    starts = np.cumsum(lens) - lens
    prompt = np.searchsorted(starts, flat, side="right") - 1
    return np.stack([prompt, flat - starts[prompt]], axis=1).astype(np.int64)


def capture_calibration(model, prompts: Sequence[Sequence[int]], position_budget: int, seed: int = 0,
                        max_tokens_per_launch: int = 65536, to_host: bool = True) -> CalibrationSet:
    """capture the MLP inputs of ``position_budget`` uniformly sampled positions.

    ``model`` is an ``engine.PrefillScorer``.  Each prompt runs as its own request (prefix = all
    but its last token), so packed row = request base + position; prompts are batched
    into launches of at most ``max_tokens_per_launch`` tokens.  The captured rows land in one device
    tensor [L, n, d]; ``to_host`` copies it once to (pinned) host memory as numpy, otherwise the
    layers stay on the device as torch views (``prune_mlp_neurons`` accepts either)."""
    import torch

    from .engine import DevicePacked
    from .prefixcache import pack_requests, split_shared_prefix

    prompts = [list(map(int, p)) for p in prompts]
    if any(len(p) == 0 for p in prompts):
        raise ValueError("capture_calibration: empty prompt")
    cfg = model.config
    src = sample_positions([len(p) for p in prompts], position_budget, seed)
    d, L = cfg.d_model, cfg.n_layers
    out = torch.empty((L, len(src), d), dtype=torch.float32, device=model.device)
    gains = torch.stack([g.float() for g in model.weights.ln_mlp]).contiguous().to(model.device)
    # launches: consecutive prompts up to the token cap (a longer prompt runs alone)
    groups, cur, cur_t = [], [], 0
    for i, p in enumerate(prompts):
        if cur and cur_t + len(p) > max_tokens_per_launch:
            groups.append(cur)
            cur, cur_t = [], 0
        cur.append(i)
        cur_t += len(p)
    if cur:
        groups.append(cur)
    row0 = 0
    for g in groups:
        sel = (src[:, 0] >= g[0]) & (src[:, 0] <= g[-1])
        n_sel = int(sel.sum())
        if n_sel == 0:
            continue
        packed = pack_requests([split_shared_prefix([prompts[i]]) for i in g], cfg.max_seq)
        base = np.zeros(len(prompts), dtype=np.int64)
        off = 0
        for i in g:
            base[i] = off
            off += len(prompts[i])
        rows = (base[src[sel, 0]] + src[sel, 1]).astype(np.int32)
        dp = DevicePacked(packed, model.device)
        model.score_capture(dp, torch.from_numpy(rows).to(model.device), gains, out=out[:, row0:row0 + n_sel])
        row0 += n_sel
    if to_host:
        host = torch.empty(out.shape, dtype=torch.float32, pin_memory=True)
        host.copy_(out)
        arr = host.numpy()
        return CalibrationSet([arr[l] for l in range(L)], int(len(src)), src)
    return CalibrationSet([out[l] for l in range(L)], int(len(src)), src)


# ----------------------------------------------------------------------------- OSSCAR stand-in
def _torch_device(device):
    import torch

    if device is not None:
        return torch.device(device)
    return torch.device("cuda" if torch.cuda.is_available() else "cpu")


def mlp_hidden(X, W_gate, W_up):
    """H = silu(X W_gate) * (X W_up) in float64 (torch tensors)."""
    import torch

    g = X @ W_gate
    return torch.nn.functional.silu(g) * (X @ W_up)


def greedy_backward_elimination(H, W_down, k: int):
    """Keep-set (sorted int64 numpy) and refit rows [k x d] minimising ||H W - H_S W~||_F by
    greedy backward elimination (ties -> lowest neuron index).  H [n x f], W_down [f x d] float64
    torch tensors on one device."""
    import torch

    f = H.shape[1]
    if not (1 <= k <= f):
        raise ValueError("greedy_backward_elimination: need 1 <= k <= d_ff")
    G = H.T @ H
    A = G @ W_down
    # singular: Cholesky fails, or a pivot is negligible against the largest diagonal entry
    Lc, info = torch.linalg.cholesky_ex(G)
    scale = float(torch.diagonal(G).max()) if f else 0.0
    if int(info) != 0 or scale <= 0.0 or float(torch.diagonal(Lc).square().min()) <= 1e-10 * scale:
        lam = 1e-6 * float(torch.trace(G)) / f
        warnings.warn(f"prune_mlp_neurons: singular least-squares system, ridge fallback lambda={lam:.3e}",
                      RuntimeWarning, stacklevel=2)
        G = G + lam * torch.eye(f, dtype=G.dtype, device=G.device)
        Lc = torch.linalg.cholesky(G)
    M = torch.cholesky_inverse(Lc)
    B = M @ A
    active = torch.ones(f, dtype=torch.bool, device=H.device)
    for _ in range(f - k):
        cost = (B * B).sum(dim=1) / torch.diagonal(M)
        cost = torch.where(active, cost, torch.full_like(cost, float("inf")))
        j = int(torch.argmin(cost))
        m = M[:, j].clone()
        mjj = m[j].clone()
        B -= torch.outer(m, B[j]) / mjj
        M -= torch.outer(m, m) / mjj
        active[j] = False
        M[j, :] = 0.0
        M[:, j] = 0.0
        M[j, j] = 1.0           # keeps the diagonal finite for the masked cost
        B[j] = 0.0
    keep = torch.nonzero(active).flatten()
    return keep.cpu().numpy().astype(np.int64), B[keep]


def prune_mlp_neurons_calibrated(weights: Weights, calib: CalibrationSet, sparsity: float, device=None) -> Weights:
    """per-layer calibrated keep-sets + W_down refit, then the shape contract of
    ``pruning.prune_mlp_neurons`` (uniform k, W_gate/W_up columns deleted)."""
    import torch

    cfg = weights.config
    if len(calib.layers) != cfg.n_layers:
        raise ValueError("prune_mlp_neurons: calibration set has a different layer count")
    k = kept_width(cfg.d_ff, sparsity)
    dev = _torch_device(device)
    keeps, rows = [], []
    for l, lw in enumerate(weights.layers):
        t = lambda a: (a if torch.is_tensor(a) else torch.as_tensor(np.asarray(a))).to(dev, torch.float64)
        H = mlp_hidden(t(calib.layers[l]), t(lw.W_gate), t(lw.W_up))
        keep, refit = greedy_backward_elimination(H, t(lw.W_down), k)
        keeps.append(keep)
        rows.append(refit.cpu().numpy().astype(np.float32))
    return prune_mlp_neurons(weights, keeps, rows)
