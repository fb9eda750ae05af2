"""Run one fused GEMM variant a few times (for ncu).  python tools/gemm_one.py o+resid+norm"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_22101_b200 import _lib
import tools.gemm_bench as gb

name = sys.argv[1]
lib = _lib.load()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for n, M, N, K, epi, _ in gb.SHAPES:
    if n != name:
        continue
    A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    ncol = N // 2 if epi == _lib.EPI_SWIGLU else N
    C = torch.zeros(M, ncol, device="cuda", dtype=torch.float32 if epi == 3 else torch.bfloat16)
    xb = torch.empty(M, ncol, device="cuda", dtype=torch.bfloat16)
    ss = torch.ones(32, M, device="cuda")   # partial sums [part][M]
    pos = torch.zeros(M, device="cuda", dtype=torch.int32)
    cs = torch.ones(2048, 64, device="cuda")
    a = _lib.PfGemmArgs(A=A.data_ptr(), lda=K, B=B.data_ptr(), ldb=K, C=C.data_ptr(), ldc=ncol, M=M, N=N, K=K,
                        epilogue=epi, pos=pos.data_ptr(), rope_cos=cs.data_ptr(), rope_sin=cs.data_ptr(),
                        rope_heads=15 if epi == 1 else 0, row_ss=ss.data_ptr() if epi in (1, 2) else None,
                        ss_out=ss.data_ptr() if epi == 4 else None, xb=xb.data_ptr(), ldxb=ncol,
                        inv_d=1.0 / K, eps=1e-6)
    for _ in range(4):
        _lib.check(lib.pf_gemm_bf16_ex(ctypes.byref(a), st))
    torch.cuda.synchronize()
