"""Run exactly `--warmup` + `--steps` packed scoring passes (pf_score) for ncu capture.

    ncu --metrics gpu__time_duration.sum --clock-control none -s <warmup*launches> -c <launches> \
        --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --config C4
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_22101_b200 import CONFIGS, REQUESTS, init_device_weights  # noqa: E402
from paper_2510_22101_b200.engine import DevicePacked, PrefillScorer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    a = ap.parse_args()
    cfg, shape = CONFIGS[a.config], REQUESTS[a.config]
    scorer = PrefillScorer(init_device_weights(cfg, 0, "cuda"))
    _, packed = bench.make_request(cfg, shape, 1000)
    dp = DevicePacked(packed)
    for _ in range(a.warmup + a.steps):
        scorer.score_device(dp)
    torch.cuda.synchronize()
    print("launches per step:", 5 * cfg.n_layers + 4)


if __name__ == "__main__":
    main()
