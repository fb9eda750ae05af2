r"""Top SASS instructions by warp-stall samples for one kernel of an ncu report (needs -lineinfo
and --import-source on).    python tools/ncu_source_hot.py report.ncu-rep 'gemm_bf16_kernel<\(int\)2' [N]"""
import csv
import io
import re
import subprocess
import sys


def main(path, pattern, n=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'(?m)^"Kernel Name",', out)
    for b in blocks[1:]:
        name = b.split("\n", 1)[0]
        if not re.search(pattern, name):
            continue
        rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
        h = rows[0]
        si, ai, ss = h.index("Source"), h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
        stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
        tot = sum(float(r[ss] or 0) for r in rows[1:] if len(r) > ss)
        print(f"== {name[:90]}  total samples {tot:.0f}")
        agg = {}
        for r in rows[1:]:
            if len(r) <= ss:
                continue
            for i in stall_cols:
                agg[h[i]] = agg.get(h[i], 0) + float(r[i] or 0)
        print("   stall totals:", ", ".join(f"{k[6:]}={v / tot * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
        top = sorted(rows[1:], key=lambda r: -float(r[ss] or 0) if len(r) > ss else 0)[:n]
        for r in top:
            reasons = sorted(((h[i][6:], float(r[i] or 0)) for i in stall_cols), key=lambda x: -x[1])[:2]
            print(f"   {float(r[ss] or 0) / tot * 100:5.1f}%  {r[ai]}  {r[si][:70]:70s} {reasons}")
        break


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
