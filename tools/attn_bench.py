"""Shared-prefix attention kernel alone at the BASELINE request shapes: CUDA-event time per launch,
algorithmic TFLOP/s (4*H*dh per unmasked (q, k) pair) and a parity check against a
torch fp32 reference on the first request's rows.

    python tools/attn_bench.py [C2 C3 C4 ...]        (PF_LIB_PATH selects a variant .so)
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_22101_b200 import CONFIGS, REQUESTS, _lib  # noqa: E402


def ref_rows(qkv, packed, H, Hkv, dh, n_segs):
    T = qkv.shape[0]
    q = qkv[:, : H * dh].float().view(T, H, dh)
    k = qkv[:, H * dh: (H + Hkv) * dh].float().view(T, Hkv, dh)
    v = qkv[:, (H + Hkv) * dh:].float().view(T, Hkv, dh)
    outs = []
    for kv_off, kv_len, q_off, q_len in packed.segs.tolist()[:n_segs]:
        rows = torch.arange(q_off, q_off + q_len, device=qkv.device)
        keys = torch.cat([torch.arange(kv_off, kv_off + kv_len, device=qkv.device), rows])
        kk = k[keys].repeat_interleave(H // Hkv, dim=1)
        vv = v[keys].repeat_interleave(H // Hkv, dim=1)
        s = torch.einsum("qhd,khd->hqk", q[rows], kk) / dh ** 0.5
        mask = torch.ones(q_len, kv_len + q_len, dtype=torch.bool, device=qkv.device)
        mask[:, kv_len:] = torch.tril(torch.ones(q_len, q_len, dtype=torch.bool, device=qkv.device))
        s = s.masked_fill(~mask, float("-inf"))
        outs.append((rows, torch.einsum("hqk,khd->qhd", torch.softmax(s, dim=-1), vv).reshape(q_len, H * dh)))
    return outs


def main():
    names = sys.argv[1:] or ["C2", "C4", "C3"]
    lib = _lib.load()
    res = {}
    for name in names:
        cfg, shape = CONFIGS[name], REQUESTS[name]
        _, packed = bench.make_request(cfg, shape, 1000)
        H, Hkv, dh, T = cfg.n_heads, cfg.n_kv_heads, cfg.d_head, packed.T
        g = torch.Generator(device="cuda").manual_seed(0)
        qkv = (torch.randn(T, (H + 2 * Hkv) * dh, device="cuda", generator=g) * 1.5).to(torch.bfloat16)
        out = torch.zeros(T, H * dh, device="cuda", dtype=torch.bfloat16)
        segs = torch.from_numpy(packed.segs).cuda()
        wk = packed.work.copy()
        if os.environ.get("PF_ATTN_L2") == "1":
            # timing probe: every work tile re-reads one of 16 items (footprint L2-resident)
            items = wk[:, 0] != 0
            wk[items, 0] = 1 + (wk[items, 0] - 1) % 16
        work = torch.from_numpy(wk).cuda()
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        P = lambda t: ctypes.c_void_p(t.data_ptr())
        run = lambda: _lib.check(lib.pf_prefix_attention(P(qkv), P(out), T, H, Hkv, dh, P(segs), P(work),
                                                         len(packed.work), st))
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        err = 0.0
        for rows, ref in ref_rows(qkv, packed, H, Hkv, dh, 4):
            err = max(err, float((out[rows].float() - ref).abs().max()))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = int(os.environ.get("PF_ATTN_REPS", "50"))
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        Pn, S = shape.prefix_len, np.asarray([shape.suffix_len] * shape.n_items, dtype=np.float64)
        pairs = Pn * (Pn + 1) / 2 + np.sum(S * Pn + S * (S + 1) / 2)
        fl = 4 * H * dh * pairs
        res[name] = {"us": us, "tflops": fl / us / 1e6, "max_abs_err": err, "T": T, "n_work": len(packed.work)}
        print(f"{name}: {us:8.1f} us  {fl / us / 1e6:7.1f} TFLOP/s  max|err| {err:.2e}  T={T} work={len(packed.work)}",
              flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    tag = os.environ.get("PF_TAG", "base")
    json.dump(res, open(f"gpurun_out/attn_bench_{tag}.json", "w"), indent=1)


if __name__ == "__main__":
    main()
