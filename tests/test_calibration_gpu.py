"""GPU calibration capture (pf_score_capture).

* captured MLP inputs vs the oracle's forward_prefill(capture=True) on the same sampled rows
  (bf16 activations vs fp32: relative Frobenius error per layer <= 2e-2, written here);
* capture is deterministic and leaves the scores unchanged;
* capture -> calibrated prune (OSSCAR stand-in) -> score on the GPU matches the oracle on the same
  pruned weights (|dp| <= 1e-2).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import oracle.calibration as OC  # noqa: E402
import oracle.model as OM  # noqa: E402
from paper_2510_22101_b200 import CONFIGS, init_weights, pack_requests  # noqa: E402
from paper_2510_22101_b200.calibration import capture_calibration  # noqa: E402
from paper_2510_22101_b200.engine import DevicePacked, PrefillScorer, score_shared_batch  # noqa: E402
from paper_2510_22101_b200.pruning import prune_mlp_neurons  # noqa: E402
from paper_2510_22101_b200.weights import bf16_round  # noqa: E402
from tests.synth import make_prompts, make_shared  # noqa: E402

TOL_CAPTURE = 2e-2
TOL_P = 1e-2


def oracle_weights(w):
    return OM.OracleWeights(w.config, w.token_embedding,
                            [{**{f: getattr(lw, f) for f in OM.LAYER_FIELDS},
                              "rms_attn": lw.rms_attn, "rms_mlp": lw.rms_mlp} for lw in w.layers],
                            w.final_norm, w.head)


def prompts_for(seed, n, lo=20, hi=160):
    rng = np.random.default_rng(seed)
    return [make_prompts(rng, 0, [int(rng.integers(lo, hi))], "spread")[0] for _ in range(n)]


@pytest.mark.parametrize("name", ["TINY", "TINY_GQA", "C1"])
def test_capture_matches_oracle(name):
    cfg = CONFIGS[name]
    w = init_weights(cfg, 0)
    rng = np.random.default_rng(4)
    for lw in w.layers:                      # non-unit MLP gains: capture must apply them
        lw.rms_mlp = bf16_round(rng.uniform(0.5, 1.5, cfg.d_model).astype(np.float32))
    prompts = prompts_for(1, 12)
    calib = capture_calibration(PrefillScorer(w), prompts, 300, seed=7, max_tokens_per_launch=700)
    ref, src = OC.capture_calibration(oracle_weights(w), prompts, 300, seed=7)
    np.testing.assert_array_equal(calib.sources, src)
    assert calib.n_tokens == 300 and len(calib.layers) == cfg.n_layers
    for l in range(cfg.n_layers):
        err = np.linalg.norm(calib.layers[l] - ref[l]) / np.linalg.norm(ref[l])
        print(f"{name} layer {l}: rel err {err:.2e}")
        assert err <= TOL_CAPTURE


def test_capture_deterministic_and_scores_unchanged(monkeypatch):
    """Captured rows are deterministic and independent of the launch split; a capturing pass runs
    every row through every layer, so its scores equal the uncompacted forward bit for bit (and the
    default forward, whose last layer runs on the last-token rows only, within 2e-3)."""
    cfg = CONFIGS["TINY_GQA"]
    scorer = PrefillScorer(init_weights(cfg, 0))
    prompts = prompts_for(2, 8)
    a = capture_calibration(scorer, prompts, 200, seed=1)
    b = capture_calibration(scorer, prompts, 200, seed=1, max_tokens_per_launch=300)
    c = capture_calibration(scorer, prompts, 200, seed=1, to_host=False)      # device-resident rows
    for x, y, z in zip(a.layers, b.layers, c.layers):
        np.testing.assert_array_equal(x, y)
        np.testing.assert_array_equal(x, z.cpu().numpy())
    packed = pack_requests([make_shared(np.random.default_rng(3), 30, [40, 50, 60], "spread")])
    plain = scorer.score_packed(packed)
    dp = DevicePacked(packed, scorer.device)
    rows = torch.arange(packed.T, dtype=torch.int32, device=scorer.device)
    gains = torch.stack([g.float() for g in scorer.weights.ln_mlp])
    out, logits2, _ = scorer.score_capture(dp, rows, gains, return_scores=True)
    assert out.shape == (cfg.n_layers, packed.T, cfg.d_model)
    monkeypatch.setenv("PF_NO_LAST_LAYER_COMPACT", "1")
    full = PrefillScorer(scorer.weights).score_packed(packed)
    np.testing.assert_array_equal(logits2.cpu().numpy(), full.logits2)
    p_cap = 1.0 / (1.0 + np.exp(-(logits2.cpu().numpy()[:, 0] - logits2.cpu().numpy()[:, 1])))
    assert np.max(np.abs(p_cap - plain.p_yes)) <= 2e-3


def test_capture_then_calibrated_prune_parity():
    cfg = CONFIGS["TINY"]                                   # d_ff 1024 -> keep 512
    w = init_weights(cfg, 0)
    calib = capture_calibration(PrefillScorer(w), prompts_for(5, 40, 60, 200), 3000, seed=0)
    assert calib.n_tokens == 3000
    pw = prune_mlp_neurons(w, calib, 0.5)
    assert pw.config.d_ff == 512
    for lw in pw.layers:                                    # device weights are bf16
        lw.W_down = bf16_round(lw.W_down)
    batches = [make_shared(np.random.default_rng(9), 48, list(np.random.default_rng(9).integers(1, 150, 20)),
                           "spread")]
    res = score_shared_batch(PrefillScorer(pw), batches)
    ow = oracle_weights(pw)
    p_ref = []
    for sb in batches:
        import oracle.prefixcache as OP
        import oracle.scoring as OS

        osb = OP.SharedBatch(list(sb.prefix_tokens), [list(s) for s in sb.suffixes])
        p_ref += [OS.relevance_score(lg)[0] for lg in OP.score_shared_batch(ow, osb)]
    assert np.max(np.abs(res.p_yes - np.asarray(p_ref))) <= TOL_P
