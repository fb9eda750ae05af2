"""Epilogue pacing sweep: time the plain bf16 epilogue vs a fused one over K, so T(K) ~
max(T_mma(K), T_epi) exposes the fused epilogue's per-tile cost (B300_MICROARCH pacing law).
    python tools/epi_sweep.py [--epi resid|rope|swiglu] [--n N] [--ks 64,1280]"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_22101_b200 import _lib
from tools.gemm_bench import time_it

EPIS = {"resid": _lib.EPI_RESID_ADD_NORM, "rope": _lib.EPI_ROPE_BF16, "swiglu": _lib.EPI_SWIGLU}
ap = argparse.ArgumentParser()
ap.add_argument("--epi", default="resid", choices=list(EPIS))
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--m", type=int, default=25664)
ap.add_argument("--ks", default="64,128,256,512,768,1024,1280,2048,3712")
a = ap.parse_args()
lib = _lib.load()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
M, N, fused = a.m, a.n, EPIS[a.epi]
xb = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
ss = torch.ones(32, M, device="cuda")   # partial sums [part][M], parts = ceil(N or K / 256)
pos = torch.randint(0, 2048, (M,), device="cuda", dtype=torch.int32)
cs = torch.rand(2048, 64, device="cuda")
for K in [int(k) for k in a.ks.split(",")]:
    A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    row = []
    for epi in (_lib.EPI_BF16, fused):
        resid = epi == _lib.EPI_RESID_ADD_NORM
        ncol = N // 2 if epi == _lib.EPI_SWIGLU else N
        g = _lib.PfGemmArgs(A=A.data_ptr(), lda=K, B=B.data_ptr(), ldb=K, C=out.data_ptr(), ldc=ncol, M=M, N=N, K=K,
                            epilogue=epi, ss_out=ss.data_ptr() if resid else None,
                            xb=xb.data_ptr() if resid else None, ldxb=N, inv_d=1.0 / K, eps=1e-6,
                            row_ss=ss.data_ptr() if epi in (_lib.EPI_ROPE_BF16, _lib.EPI_SWIGLU) else None,
                            pos=pos.data_ptr(), rope_cos=cs.data_ptr(), rope_sin=cs.data_ptr(),
                            rope_heads=(N // 128) * 3 // 4 if epi == _lib.EPI_ROPE_BF16 else 0, rope_dh=128)
        row.append(time_it(lambda: _lib.check(lib.pf_gemm_bf16_ex(ctypes.byref(g), st))) * 1e3)
    print(f"K={K:5d}  plain {row[0]:7.1f} us   {a.epi} {row[1]:7.1f} us   mma-floor@1.5PF "
          f"{2*M*N*K/1.5e15*1e6:7.1f} us", flush=True)
