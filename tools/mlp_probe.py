"""Fused layer tail (mlp.cu) alone at a config's full-T shape: launch time, per-wait-site stall
statistics (pf_debug_set_mlp_stats) and the three-GEMM sequence it replaces, under schedule lags /
no-dependency debug mode.   python tools/mlp_probe.py [C4] """

import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_22101_b200 import CONFIGS, REQUESTS, _lib, init_device_weights  # noqa: E402
from paper_2510_22101_b200.engine import PrefillScorer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = CONFIGS[name].with_(n_layers=1)
T = REQUESTS[name].tokens
lib = _lib.load()
sc = PrefillScorer(init_device_weights(cfg, 0, "cuda"))
w = sc.weights
d, kq, fp = cfg.d_model, cfg.q_width, cfg.d_ff_pad
dev = "cuda"
attn = (torch.randn(T, kq, device=dev) * 0.5).to(torch.bfloat16)
xb = torch.randn(T, d, device=dev).to(torch.bfloat16)
rlo = torch.full((T, d), 128, dtype=torch.uint8, device=dev)
hb = torch.empty(T, fp, device=dev, dtype=torch.bfloat16)
parts = (d + 255) // 256
ssm = torch.zeros(parts, T, device=dev)
ssa = torch.zeros(parts, T, device=dev)
ctr = torch.empty(8 * ((T + 255) // 256), dtype=torch.uint8, device=dev)
stats = torch.zeros(16, dtype=torch.int64, device=dev)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: t.data_ptr()


def tail():
    _lib.check(lib.pf_layer_tail(sc.handle, 0, P(attn), P(xb), P(rlo), P(hb), P(ssm), P(ssa), T, P(ctr),
                                 ctr.numel(), st))


def gex(**kw):
    a = _lib.PfGemmArgs()
    for k, v in kw.items():
        setattr(a, k, v.data_ptr() if hasattr(v, "data_ptr") else v)
    _lib.check(lib.pf_gemm_bf16_ex(ctypes.byref(a), st))


def three():
    gex(A=attn, lda=kq, B=w.w_o[0], ldb=kq, C=rlo, ldc=d, M=T, N=d, K=kq, epilogue=_lib.EPI_RESID_ADD_NORM,
        xb=xb, ldxb=d, ss_out=ssm, ss_ld=T)
    gex(A=xb, lda=d, B=w.w_gu[0], ldb=d, C=hb, ldc=fp, M=T, N=2 * fp, K=d, epilogue=_lib.EPI_SWIGLU,
        row_ss=ssm, ss_ld=T, inv_d=1.0 / d, eps=cfg.rms_eps)
    gex(A=hb, lda=fp, B=w.w_down[0], ldb=fp, C=rlo, ldc=d, M=T, N=d, K=fp, epilogue=_lib.EPI_RESID_ADD_NORM,
        xb=xb, ldxb=d, ss_out=ssa, ss_ld=T)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def kind_ab():
    """Each GEMM alone next to the fused kernel restricted to that tile kind (no dependencies)."""
    one = {
        "O": lambda: gex(A=attn, lda=kq, B=w.w_o[0], ldb=kq, C=rlo, ldc=d, M=T, N=d, K=kq,
                         epilogue=_lib.EPI_RESID_ADD_NORM, xb=xb, ldxb=d, ss_out=ssm, ss_ld=T),
        "GU": lambda: gex(A=xb, lda=d, B=w.w_gu[0], ldb=d, C=hb, ldc=fp, M=T, N=2 * fp, K=d, epilogue=_lib.EPI_SWIGLU,
                          row_ss=ssm, ss_ld=T, inv_d=1.0 / d, eps=cfg.rms_eps),
        "DN": lambda: gex(A=hb, lda=fp, B=w.w_down[0], ldb=fp, C=rlo, ldc=d, M=T, N=d, K=fp,
                          epilogue=_lib.EPI_RESID_ADD_NORM, xb=xb, ldxb=d, ss_out=ssa, ss_ld=T),
    }
    os.environ.update(PF_MLP_NODEP="1", PF_MLP_LAG_GU="4", PF_MLP_LAG_DN="8", PF_MLP_ROWS="1")
    for k, bit in (("O", 1), ("GU", 2), ("DN", 4)):
        os.environ["PF_MLP_KINDS"] = str(bit)
        a, b, a2, b2 = timeit(one[k]), timeit(tail), timeit(one[k]), timeit(tail)
        print(f"{k}: standalone {min(a, a2) * 1e3:.1f} us   fused-kind-only {min(b, b2) * 1e3:.1f} us")
    os.environ.update(PF_MLP_NODEP="0", PF_MLP_KINDS="7")


if os.environ.get("PF_MLP_KIND_AB") == "1":
    kind_ab()
    sys.exit(0)
if os.environ.get("PF_MLP_ONCE") == "1":
    for _ in range(3):
        tail()
    for _ in range(3):
        three()
    torch.cuda.synchronize()
    sys.exit(0)
print(f"{name}: T={T} three-GEMM sequence {timeit(three) * 1e3:.1f} us")
settings = [(1, 2, 3), (1, 4, 8), (2, 1, 2), (2, 2, 2), (2, 2, 4), (4, 1, 1), (4, 1, 2), (4, 2, 2), (8, 1, 1)]
if len(sys.argv) > 2:
    settings = [tuple(int(x) for x in a.split(",")) for a in sys.argv[2:]]
nodep = os.environ.get("PF_MLP_NODEP", "0")
for rows, gu, dn in settings:
    os.environ.update(PF_MLP_LAG_GU=str(gu), PF_MLP_LAG_DN=str(dn), PF_MLP_ROWS=str(rows))
    t = timeit(tail)
    stats.zero_()
    _lib.check(lib.pf_debug_set_mlp_stats(P(stats)))
    tail()
    torch.cuda.synchronize()
    _lib.check(lib.pf_debug_set_mlp_stats(None))
    s = stats.cpu().tolist()
    site = lambda i: f"{s[i] / 1e3:.0f}us/{s[i + 1]}"
    print(f"rows={rows} lag_gu={gu} lag_dn={dn} nodep={nodep}: {t * 1e3:.1f} us | stalls (sum over CTAs, us/count): "
          f"prod GU {site(0)} prod DN {site(2)} epi DN-ring {site(4)} epi GU-ss {site(6)} publish {site(8)}")
