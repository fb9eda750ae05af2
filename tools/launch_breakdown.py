"""Per-kernel share of one step from an ncu launch list (gpu__time_duration.sum CSV).
    python tools/launch_breakdown.py gpurun_out/launches_c4.csv"""
import collections
import csv
import re
import sys

EPI = {"0": "bf16", "1": "qkv+rope", "2": "gate/up+swiglu", "3": "resid-add", "4": "resid-add+norm",
       "100": "resid-add+norm, deep ring (O)"}


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])   # launches, ns, DRAM bytes
    for r in data:
        name = r[ki]
        m = re.search(r"gemm_bf16_kernel<(?:\(int\))?(\d+)", name)
        key = f"gemm<{EPI.get(m.group(1), m.group(1))}>" if m else re.sub(r"^void |pf::|\(.*", "", name).split("<")[0]
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            agg[key][0] += 1
            agg[key][1] += v * (1e3 if r[ui] == "usecond" else 1.0)
        elif r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1.0)
            agg[key][2] += v * scale
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':28s} {'share':>7s} {'n':>5s} {'avg us':>9s} {'total us':>10s} {'DRAM MB/launch':>15s} {'DRAM GB/s':>10s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:28s} {t / tot * 100:6.2f}% {n:5d} {t / n / 1e3:9.1f} {t / 1e3:10.1f} {b / n / 1e6:15.1f} {b / t:10.1f}")
    print(f"{'TOTAL':28s} {'':7s} {sum(v[0] for v in agg.values()):5d} {'':9s} {tot / 1e3:10.1f}")
    print("(ncu per-launch times: cold-cache, serialized, --clock-control none; shares, not absolutes)")


if __name__ == "__main__":
    main(sys.argv[1])
