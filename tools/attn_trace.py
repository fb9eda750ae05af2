"""Per-event timeline of attention CTA 0 in one C4 layer (debug hook pf_debug_set_trace).
    python tools/attn_trace.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2510_22101_b200 import CONFIGS, REQUESTS, _lib, init_weights
from paper_2510_22101_b200.engine import DevicePacked, PrefillScorer

NAMES = {1: "QFULL", 2: "KVFULL", 3: "S_ISSUED", 4: "PREADY", 5: "PV_ISSUED", 6: "SFULL", 7: "PARRIVE",
         8: "ODONE", 9: "EPI_DONE", 10: "UNIT_START", 12: "EPI_WAITED", 13: "EPI_STAGED"}
import os
name = os.environ.get("PF_CFG", "C4")
cfg = CONFIGS[name].with_(n_layers=1)
shape = REQUESTS[name]
scorer = PrefillScorer(init_weights(cfg, 0))
_, packed = bench.make_request(cfg, shape, 1000)
dp = DevicePacked(packed)
scorer.score_device(dp)
torch.cuda.synchronize()
lib = _lib.load()
buf = torch.zeros(4 * 64 * 8 * 16, dtype=torch.int64, device="cuda")
_lib.check(lib.pf_debug_set_trace(buf.data_ptr(), buf.numel()))
scorer.score_device(dp)
torch.cuda.synchronize()
_lib.check(lib.pf_debug_set_trace(None, 0))
raw = buf.cpu().tolist()
ph = [int(x) for x in raw[-64:-53]]
if any(ph):   # -DPF_ATT_PHASES build: clock64 sums over every softmax warp of every CTA
    names = ["s_full wait", "softmax math", "pv_done wait", "rescale", "P st wait+arrive", "o_done wait",
             "epilogue: fence+TMA", "units", "epilogue: store wait", "epilogue: TMEM ld", "epilogue: cvt+STS"]
    idx = [0, 1, 2, 3, 4, 5, 8, 9, 10, 6]
    tot = sum(ph[i] for i in idx)
    print("softmax-warp cycles by phase (all CTAs):")
    for i in idx:
        print(f"  {names[i]:22s} {ph[i] / tot * 100:5.1f}%   {ph[i] / max(ph[7], 1):9.0f} cycles/unit")
    print(f"  units (x warps)   {ph[7]}")
recs = [int(x) & 0xFFFFFFFFFFFFFFFF for x in raw[:-64] if x != 0]
rows = []
for r in recs:
    ev, who, unit, blk, t = r >> 56, (r >> 48) & 0xff, (r >> 40) & 0xff, (r >> 32) & 0xff, r & 0xffffffff
    rows.append((t, ev, who, unit, blk))
rows.sort()
t0 = rows[0][0]
for t, ev, who, unit, blk in rows[:400]:
    print(f"{(t - t0) / 1000:8.2f} us  {NAMES.get(ev, ev):10s} role={who:3d} unit={unit:2d} blk={blk}")
print("total", (rows[-1][0] - t0) / 1000, "us,", len(rows), "records")
