import ctypes, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2510_22101_b200 import CONFIGS, REQUESTS, _lib
lib = _lib.load()
for name in ["C4", "C3", "C2"]:
    cfg, shape = CONFIGS[name], REQUESTS[name]
    _, packed = bench.make_request(cfg, shape, 1000)
    H, Hkv, dh, T = cfg.n_heads, cfg.n_kv_heads, cfg.d_head, packed.T
    qkv = (torch.randn(T, (H + 2 * Hkv) * dh, device="cuda") * 1.5).to(torch.bfloat16)
    last = torch.from_numpy(packed.last_idx.astype(np.int32)).cuda()
    n = len(packed.last_idx)
    q = qkv[last.long(), : H * dh].contiguous()
    out = torch.empty(n, H * dh, device="cuda", dtype=torch.bfloat16)
    segs = torch.from_numpy(packed.segs).cuda()
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    run = lambda: _lib.check(lib.pf_attention_last_rows(P(q), P(qkv), H, Hkv, dh, P(segs), len(packed.segs), P(last), n, cfg.max_seq, P(out), st))
    for _ in range(3): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): run()
    e1.record(); torch.cuda.synchronize()
    print(name, f"last-row attention {e0.elapsed_time(e1) / 50 * 1e3:.1f} us  (n={n}, T={T})")
