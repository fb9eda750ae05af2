"""Oracle restatement of the pruning module's calibration path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  numpy float64, direct formulas:
* ``sample_positions`` -- SPEC.md:468-476: uniform subsample of positions over all prompts
  (pinned rule: PCG64 ``default_rng(seed).choice(total, min(budget, total), replace=False)`` over
  the concatenated token positions, sorted).
* ``capture_calibration`` -- the same rows' MLP inputs from ``model.forward_prefill(capture=True)``
  (SPEC.md:200-203).
* ``refit_error(H, W, S)`` -- min over W~ of ||H W - H_S W~||_F^2 by least squares.
* ``greedy_backward`` -- SPEC.md:480 greedy backward elimination, each step re-solving the least
  squares for every candidate (O(f^2) solves; small layers only).  Ties -> lowest index.
* ``exhaustive_best`` -- the optimum over all C(f, k) subsets (SPEC.md:484's oracle).
"""

from __future__ import annotations

import itertools

import numpy as np

from . import model as M


def sample_positions(prompt_lens, budget: int, seed: int = 0) -> np.ndarray:
    if budget < 1:
        raise ValueError("budget must be >= 1")
    lens = [int(n) for n in prompt_lens]
    if not lens or sum(lens) == 0:
        raise ValueError("empty prompt set")
    owner = [(p, t) for p, n in enumerate(lens) for t in range(n)]
    pick = np.random.default_rng(seed).choice(len(owner), size=min(budget, len(owner)), replace=False)
    return np.array([owner[i] for i in sorted(pick.tolist())], dtype=np.int64).reshape(-1, 2)


def capture_calibration(W, prompts, budget: int, seed: int = 0, eps: float = 1e-6):
    src = sample_positions([len(p) for p in prompts], budget, seed)
    per_prompt = {}
    for p in sorted(set(src[:, 0].tolist())):
        per_prompt[p] = M.forward_prefill(W, prompts[p], eps, capture=True)[2]
    L = len(W.layers)
    return [np.stack([per_prompt[p][l][t] for p, t in src]) for l in range(L)], src


def hidden(X, W_gate, W_up):
    X = np.asarray(X, np.float64)
    g = X @ np.asarray(W_gate, np.float64)
    return g / (1.0 + np.exp(-g)) * (X @ np.asarray(W_up, np.float64))


def refit_error(H, W, S):
    S = list(S)
    target = H @ W
    Wt, *_ = np.linalg.lstsq(H[:, S], target, rcond=None)
    r = target - H[:, S] @ Wt
    return float(np.sum(r * r)), Wt


def greedy_backward(H, W, k):
    S = list(range(H.shape[1]))
    while len(S) > k:
        errs = [refit_error(H, W, [i for i in S if i != j])[0] for j in S]
        S.remove(S[int(np.argmin(errs))])
    return S, refit_error(H, W, S)


def exhaustive_best(H, W, k):
    best = None
    for S in itertools.combinations(range(H.shape[1]), k):
        e = refit_error(H, W, S)[0]
        if best is None or e < best[0]:
            best = (e, list(S))
    return best
