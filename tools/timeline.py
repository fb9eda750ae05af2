"""In-situ kernel timeline of pf_score steps via CUPTI (torch.profiler): per-kernel durations
under sustained load and the idle gaps between consecutive kernels.

    python tools/timeline.py --config C4 [--graph]
"""
import argparse
import collections
import json
import os
import re
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_22101_b200 import CONFIGS, REQUESTS, init_device_weights  # noqa: E402
from paper_2510_22101_b200.engine import DevicePacked, PrefillScorer  # noqa: E402

EPI = {"0": "bf16", "1": "qkv+rope", "2": "gate/up+swiglu", "3": "resid-add", "4": "resid-add+norm"}


def key(name):
    m = re.search(r"gemm_bf16_kernel<(?:\(int\))?(\d)", name)
    if m:
        return f"gemm<{EPI[m.group(1)]}>"
    return re.sub(r"^void |pf::|\(.*", "", name).split("<")[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--graph", action="store_true")
    ap.add_argument("--out", default="gpurun_out/timeline.json")
    a = ap.parse_args()
    cfg, shape = CONFIGS[a.config], REQUESTS[a.config]
    scorer = PrefillScorer(init_device_weights(cfg, 0, "cuda"))
    _, packed = bench.make_request(cfg, shape, 1000)
    dp = DevicePacked(packed)
    run = scorer.graph_runner(dp) if a.graph else (lambda: scorer.score_device(dp, check=False))
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.steps):
            run()
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    agg = collections.defaultdict(lambda: [0, 0.0])
    gaps = 0.0
    for i, e in enumerate(ev):
        agg[key(e["name"])][0] += 1
        agg[key(e["name"])][1] += e["dur"]
        if i:
            gaps += max(0.0, e["ts"] - (ev[i - 1]["ts"] + ev[i - 1]["dur"]))
    span = ev[-1]["ts"] + ev[-1]["dur"] - ev[0]["ts"]
    busy = sum(v[1] for v in agg.values())
    out = {"config": a.config, "graph": a.graph, "steps": a.steps, "span_us_per_step": span / a.steps,
           "busy_us_per_step": busy / a.steps, "gap_us_per_step": gaps / a.steps,
           "kernels": {k: {"n_per_step": n / a.steps, "avg_us": t / n, "share": t / busy}
                       for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])}}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
