"""Calibration-path measurement: GPU capture throughput and the calibrated
prune (OSSCAR stand-in) cost at the unpruned 1.7B shape (C3 dims: L28 d2048 16/8 heads d_ff 6144),
the model C4 is pruned from (d_ff 6144 -> 3686 = 40% sparsity).

    python tools/calib_bench.py [--prompts 64] [--len 1024] [--budget 65536] [--json out.json]

capture: prompts of `len` synthetic tokens, `budget` sampled positions; timed = the whole
capture_calibration call (packing, H2D, forward with capture, D2H of the captured rows), and the
same forward without capture (pf_score) for the overhead.  prune: one layer's greedy backward
elimination + refit on `budget` rows (float64 torch on the GPU), extrapolated x L."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_22101_b200 import CONFIGS, init_device_weights, pack_requests, split_shared_prefix  # noqa: E402
from paper_2510_22101_b200.calibration import (capture_calibration, greedy_backward_elimination,  # noqa: E402
                                               mlp_hidden)
from paper_2510_22101_b200.engine import DevicePacked, PrefillScorer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--prompts", type=int, default=64)
    ap.add_argument("--len", type=int, default=1024)
    ap.add_argument("--budget", type=int, default=16384)
    ap.add_argument("--sparsity", type=float, default=0.4)
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    scorer = PrefillScorer(init_device_weights(cfg, 0, "cuda"))
    rng = np.random.default_rng(0)
    prompts = [[3] + rng.integers(16, cfg.vocab_size, a.len - 1).tolist() for _ in range(a.prompts)]
    tokens = a.prompts * a.len

    capture_calibration(scorer, prompts[:2], 64, seed=0)          # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    calib_h = capture_calibration(scorer, prompts, a.budget, seed=0)
    torch.cuda.synchronize()
    t_cap = time.perf_counter() - t0
    t0 = time.perf_counter()
    calib = capture_calibration(scorer, prompts, a.budget, seed=0, to_host=False)
    torch.cuda.synchronize()
    t_cap_dev = time.perf_counter() - t0
    assert np.array_equal(calib_h.layers[3], calib.layers[3].cpu().numpy())

    packed = pack_requests([split_shared_prefix([p]) for p in prompts], cfg.max_seq)
    dp = DevicePacked(packed, "cuda")
    scorer.score_device(dp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    scorer.score_device(dp)
    e1.record()
    torch.cuda.synchronize()
    t_fwd = e0.elapsed_time(e1) / 1e3

    # one layer of the calibrated prune (the captured rows are real MLP inputs of layer 0)
    w = scorer.weights
    k = int(round((1 - a.sparsity) * cfg.d_ff))
    d_ff = cfg.d_ff
    gu = w.w_gu[0].float()          # device layout: interleaved [gate_j | up_j] per 128-neuron block
    blocks = gu.view(-1, 2, 128, cfg.d_model)
    Wg = blocks[:, 0].reshape(-1, cfg.d_model)[:d_ff].T.double()
    Wu = blocks[:, 1].reshape(-1, cfg.d_model)[:d_ff].T.double()
    Wd = w.w_down[0].float()[:, :d_ff].T.double().contiguous()
    X = calib.layers[0].double()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    H = mlp_hidden(X, Wg, Wu)
    keep, refit = greedy_backward_elimination(H, Wd, k)
    torch.cuda.synchronize()
    t_prune = time.perf_counter() - t0

    res = {
        "config": a.config, "prompts": a.prompts, "prompt_len": a.len, "tokens": tokens,
        "budget_rows": calib.n_tokens,
        "capture_s": t_cap, "capture_tok_per_s": tokens / t_cap,
        "capture_device_resident_s": t_cap_dev, "capture_device_resident_tok_per_s": tokens / t_cap_dev,
        "forward_only_s": t_fwd, "forward_tok_per_s": tokens / t_fwd,
        "prune_layer_s": t_prune, "prune_model_s_est": t_prune * cfg.n_layers,
        "d_ff": d_ff, "k": k, "kept": int(len(keep)),
        "notes": "capture_s is end to end (pack + H2D + forward with capture + one pinned D2H of L x rows x d "
                 "fp32); capture_device_resident_s keeps the rows on the device (to_host=False); "
                 "forward_only_s is the device time of pf_score on the same packed batch",
    }
    print(json.dumps(res))
    if a.json:
        json.dump(res, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
