"""Step time of one config under different launch modes, same process (same clocks/box):
graph replay (PDL on), eager (PDL on), eager with per-launch events (pf_profile), and the
per-class kernel sums.  Run twice: as is and with PF_NO_PDL=1.
    python tools/step_modes.py --config C4"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_22101_b200 import CONFIGS, REQUESTS, _lib, init_device_weights  # noqa: E402
from paper_2510_22101_b200.engine import DevicePacked, PrefillScorer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    cfg, shape = CONFIGS[a.config], REQUESTS[a.config]
    dev = torch.device("cuda", 0)
    scorer = PrefillScorer(init_device_weights(cfg, seed=0, device=dev), device=dev)
    _, packed = bench.make_request(cfg, shape, seed=1000)
    dp = DevicePacked(packed, dev)
    lib = _lib.load()
    graph = scorer.graph_runner(dp)
    eager = lambda: scorer.score_device(dp, check=False)

    def timed(fn, n):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    out = {"config": a.config, "pdl": os.environ.get("PF_NO_PDL", "0") != "1"}
    for rep in range(2):
        out[f"graph_ms_{rep}"] = timed(graph, a.steps)
        out[f"eager_ms_{rep}"] = timed(eager, a.steps)
        _lib.check(lib.pf_profile_enable(1))
        out[f"eager_events_ms_{rep}"] = timed(eager, a.steps)
        ms, nl = (ctypes.c_double * 7)(), (ctypes.c_int * 7)()
        _lib.check(lib.pf_profile_read(ms, nl, 7))
        _lib.check(lib.pf_profile_enable(0))
        n_pass = a.steps + 3
        out[f"kernel_sum_ms_{rep}"] = sum(ms) / n_pass
        out[f"classes_{rep}"] = {lib.pf_profile_class_name(c).decode(): round(ms[c] / n_pass, 3) for c in range(7)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
