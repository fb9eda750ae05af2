"""Calibration capture + calibrated MLP pruning, CPU side.

The sampler, the fast greedy (closed-form OBS downdates) and the shape/refit contract are checked
against oracle/calibration.py: direct least squares per candidate and exhaustive subset search.
The GPU capture itself is in tests/test_calibration_gpu.py."""

import warnings

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle.calibration as OC  # noqa: E402
import oracle.model as OM  # noqa: E402
from paper_2510_22101_b200 import CONFIGS, init_weights  # noqa: E402
from paper_2510_22101_b200.calibration import (CalibrationSet, greedy_backward_elimination,  # noqa: E402
                                               mlp_hidden, sample_positions)
from paper_2510_22101_b200.pruning import prune_mlp_neurons  # noqa: E402


def test_sampler_matches_oracle_and_spec_examples():
    rng = np.random.default_rng(0)
    for seed in range(20):
        lens = rng.integers(1, 60, int(rng.integers(1, 12))).tolist()
        budget = int(rng.integers(1, 400))
        np.testing.assert_array_equal(sample_positions(lens, budget, seed), OC.sample_positions(lens, budget, seed))
    lens = [37] * 10
    src = sample_positions(lens, 100, 3)
    assert src.shape == (100, 2)                                             # SPEC.md:473 budget accounting
    np.testing.assert_array_equal(src, sample_positions(lens, 100, 3))       # SPEC.md:474 same seed
    assert len(np.unique(src, axis=0)) == 100                                 # without replacement
    for seed in range(10):                                                    # SPEC.md:475 coverage
        s = sample_positions(rng.integers(20, 200, 10).tolist(), 100, seed)
        assert len(set(s[:, 0].tolist())) >= 8
    assert sample_positions([3, 2], 999, 0).shape == (5, 2)                   # budget > total -> all
    with pytest.raises(ValueError):
        sample_positions([3], 0, 0)
    with pytest.raises(ValueError):
        sample_positions([], 5, 0)


def test_oracle_capture_is_the_mlp_input():
    cfg = CONFIGS["TINY"]
    ow = OM.init_weights(cfg, 0)
    toks = np.random.default_rng(1).integers(16, cfg.vocab_size, 23).tolist()
    logits, _, cap = OM.forward_prefill(ow, toks, capture=True)
    np.testing.assert_array_equal(logits, OM.forward_prefill(ow, toks)[0])
    assert len(cap) == cfg.n_layers and cap[0].shape == (23, cfg.d_model)
    ms = np.sqrt(np.mean(cap[0] ** 2, axis=-1))            # unit gains -> unit RMS rows
    np.testing.assert_allclose(ms, 1.0, rtol=1e-3)


def _toy(rng, n=200, d=8, f=10):
    X = rng.standard_normal((n, d))
    Wg, Wu = rng.standard_normal((d, f)) / np.sqrt(d), rng.standard_normal((d, f)) / np.sqrt(d)
    Wd = rng.standard_normal((f, d)) / np.sqrt(f)
    H = OC.hidden(X, Wg, Wu)
    return X, Wg, Wu, Wd, H


def test_fast_greedy_equals_direct_greedy():
    rng = np.random.default_rng(5)
    for _ in range(10):
        X, Wg, Wu, Wd, H = _toy(rng)
        t = lambda a: torch.as_tensor(a, dtype=torch.float64)
        Ht = mlp_hidden(t(X), t(Wg), t(Wu))
        np.testing.assert_allclose(Ht.numpy(), H, rtol=1e-12, atol=1e-12)
        keep, refit = greedy_backward_elimination(Ht, t(Wd), 5)
        S, (err, Wt) = OC.greedy_backward(H, Wd, 5)
        assert keep.tolist() == sorted(S)
        np.testing.assert_allclose(refit.numpy(), Wt[np.argsort(S)], rtol=1e-8, atol=1e-10)


def test_greedy_within_1p1_of_exhaustive_optimum():
    """d_ff=10, keep 5, 50 random instances -> greedy+refit error <= 1.1x optimum."""
    rng = np.random.default_rng(11)
    worst = 0.0
    for _ in range(50):
        X, Wg, Wu, Wd, H = _toy(rng)
        keep, _ = greedy_backward_elimination(torch.as_tensor(H), torch.as_tensor(Wd), 5)
        e_greedy = OC.refit_error(H, Wd, keep.tolist())[0]
        e_best = OC.exhaustive_best(H, Wd, 5)[0]
        worst = max(worst, e_greedy / e_best)
    assert worst <= 1.1, worst


def _calib_for(w, n=600, seed=0):
    rng = np.random.default_rng(seed)
    d = w.config.d_model
    return CalibrationSet([rng.standard_normal((n, d)).astype(np.float32) for _ in w.layers], n,
                          np.zeros((n, 2), dtype=np.int64))


def test_sparsity_zero_is_a_noop_refit():
    """sparsity 0 -> weights unchanged except the no-op refit (within 1e-10)."""
    w = init_weights(CONFIGS["TINY"], 0)
    calib = _calib_for(w, n=3000)   # n >= d_ff: a well-posed least-squares system
    p = prune_mlp_neurons(w, calib, 0.0)
    assert p.config.d_ff == w.config.d_ff
    for a, b in zip(w.layers, p.layers):
        np.testing.assert_array_equal(a.W_gate, b.W_gate)
        np.testing.assert_array_equal(a.W_up, b.W_up)
        assert np.max(np.abs(a.W_down.astype(np.float64) - b.W_down)) <= 1e-10 * max(1.0, np.abs(a.W_down).max())


def test_param_count_reduction_closed_form():
    """sparsity 0.5 -> parameter drop = L * 3 * d * (d_ff - k)."""
    w = init_weights(CONFIGS["TINY"], 0)
    cfg = w.config
    p = prune_mlp_neurons(w, _calib_for(w, n=3000), 0.5)
    k = int(round(0.5 * cfg.d_ff))
    assert p.config.d_ff == k
    assert w.param_count() - p.param_count() == cfg.n_layers * 3 * cfg.d_model * (cfg.d_ff - k)
    for lw in p.layers:
        assert lw.W_gate.shape == (cfg.d_model, k) and lw.W_down.shape == (k, cfg.d_model)


def test_calibrated_keep_beats_magnitude_on_reconstruction():
    """The calibrated keep-set reconstructs the layer output better than the magnitude heuristic."""
    from paper_2510_22101_b200.pruning import select_keep_by_norm

    w = init_weights(CONFIGS["TINY"], 0)
    calib = _calib_for(w, n=3000, seed=2)
    lw = w.layers[0]
    H = OC.hidden(calib.layers[0], lw.W_gate, lw.W_up)
    k = int(round(0.5 * w.config.d_ff))
    keep, _ = greedy_backward_elimination(torch.as_tensor(H), torch.as_tensor(lw.W_down.astype(np.float64)), k)
    mag = select_keep_by_norm(w, 0.5)[0]
    e_cal = OC.refit_error(H, lw.W_down.astype(np.float64), keep.tolist())[0]
    e_mag = OC.refit_error(H, lw.W_down.astype(np.float64), mag.tolist())[0]
    assert e_cal < e_mag


def test_singular_system_ridge_fallback():
    rng = np.random.default_rng(3)
    X, Wg, Wu, Wd, H = _toy(rng, n=200)
    H[:, 3] = H[:, 7]                       # duplicate neuron -> singular Gram matrix
    with warnings.catch_warnings(record=True) as rec:
        warnings.simplefilter("always")
        keep, refit = greedy_backward_elimination(torch.as_tensor(H), torch.as_tensor(Wd), 5)
    assert any("ridge" in str(r.message) for r in rec)
    assert len(keep) == 5 and np.all(np.isfinite(refit.numpy()))


def test_calibration_set_row_invariant():
    with pytest.raises(ValueError):
        CalibrationSet([np.zeros((3, 4)), np.zeros((4, 4))], 3, np.zeros((3, 2)))
