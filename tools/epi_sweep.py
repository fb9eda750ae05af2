"""Epilogue pacing sweep: time plain vs resid+norm GEMMs at M=25664 N=2048 over K, so T(K) ~
max(T_mma(K), T_epi) exposes the epilogue's per-tile cost (B300_MICROARCH pacing law).
    python tools/epi_sweep.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_22101_b200 import _lib
from tools.gemm_bench import time_it

lib = _lib.load()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
M, N = 25664, 2048
xb = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
lo = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
ss = torch.ones(M, device="cuda")
for K in [int(k) for k in os.environ.get("KS", "64,128,256,512,768,1024,1280,2048,3712").split(",")]:
    A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    row = []
    for epi in (_lib.EPI_BF16, _lib.EPI_RESID_ADD_NORM):
        norm = epi == _lib.EPI_RESID_ADD_NORM
        a = _lib.PfGemmArgs(A=A.data_ptr(), lda=K, B=B.data_ptr(), ldb=K, C=lo.data_ptr(), ldc=N, M=M, N=N, K=K,
                            epilogue=epi, ss_out=ss.data_ptr() if norm else None,
                            xb=xb.data_ptr() if norm else None, ldxb=N, inv_d=1.0 / N, eps=1e-6)
        row.append(time_it(lambda: _lib.check(lib.pf_gemm_bf16_ex(ctypes.byref(a), st))) * 1e3)
    print(f"K={K:5d}  plain {row[0]:7.1f} us   resid+norm {row[1]:7.1f} us   mma-floor@1.5PF "
          f"{2*M*N*K/1.5e15*1e6:7.1f} us", flush=True)
