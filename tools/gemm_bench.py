"""GEMM microbenchmark: libprefill_sm100 tcgen05 GEMM vs cuBLAS (torch.matmul) at the C4 layer
shapes and 8192^3.  CUDA-event timing, 5 warm-up + 20 timed launches, inputs > L2 rotated.

    python tools/gemm_bench.py [--cg 1|2] [--json out.json]
"""
import argparse
import ctypes
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2510_22101_b200 import _lib  # noqa: E402

T = 25664
T2 = 32832
SHAPES = [  # name, M, N (B rows), K, epilogue, useful flops (true widths)
    ("C2 qkv+rope", T2, 4096, 1024, _lib.EPI_ROPE_BF16, 2 * T2 * 4096 * 1024),
    ("C2 gate/up+swiglu", T2, 6144, 1024, _lib.EPI_SWIGLU, 2 * T2 * 1024 * 6144),
    ("C2 gate/up plain", T2, 6144, 1024, _lib.EPI_BF16, 2 * T2 * 1024 * 6144),
    ("C2 o+resid+norm", T2, 1024, 2048, _lib.EPI_RESID_ADD_NORM, 2 * T2 * 1024 * 2048),
    ("qkv+rope", T, 2560, 2048, _lib.EPI_ROPE_BF16, 2 * T * 2560 * 2048),
    ("qkv plain", T, 2560, 2048, _lib.EPI_BF16, 2 * T * 2560 * 2048),
    ("C2 qkv plain", T2, 4096, 1024, _lib.EPI_BF16, 2 * T2 * 4096 * 1024),
    ("o plain", T, 2048, 1280, _lib.EPI_BF16, 2 * T * 2048 * 1280),
    ("down plain", T, 2048, 3712, _lib.EPI_BF16, 2 * T * 3686 * 2048),
    ("o+resid", T, 2048, 1280, _lib.EPI_RESID_ADD, 2 * T * 2048 * 1280),
    ("gate/up+swiglu", T, 7424, 2048, _lib.EPI_SWIGLU, 2 * T * 2048 * 2 * 3686),
    ("down+resid", T, 2048, 3712, _lib.EPI_RESID_ADD, 2 * T * 3686 * 2048),
    ("o+resid+norm", T, 2048, 1280, _lib.EPI_RESID_ADD_NORM, 2 * T * 2048 * 1280),
    ("down+resid+norm", T, 2048, 3712, _lib.EPI_RESID_ADD_NORM, 2 * T * 3686 * 2048),
    ("square bf16", 8192, 8192, 8192, _lib.EPI_BF16, 2 * 8192 ** 3),
]


def time_it(fn, reps=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=None)
    ap.add_argument("--only", default=None, help="regex on shape names")
    ap.add_argument("--no-cublas", action="store_true")
    a = ap.parse_args()
    lib = _lib.load()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    cos = torch.rand(2048, 64, device="cuda")
    sin = torch.rand(2048, 64, device="cuda")
    pos = torch.randint(0, 2048, (max(T, T2),), device="cuda", dtype=torch.int32)
    res = []
    for name, M, N, K, epi, flops in SHAPES:
        if a.only and not re.search(a.only, name):
            continue
        A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
        ncol = N // 2 if epi == _lib.EPI_SWIGLU else N
        C = torch.zeros(M, ncol, device="cuda", dtype=torch.float32 if epi == _lib.EPI_RESID_ADD else torch.bfloat16)

        xb = torch.empty(M, ncol, device="cuda", dtype=torch.bfloat16) if epi == _lib.EPI_RESID_ADD_NORM else None
        ss = torch.ones(32, M, device="cuda")   # partial sums [part][M]
        # gathered cos/sin in the epilogue's layout (as pf_score builds it with rope_gather_kernel)
        cs_g = torch.rand(((M + 31) // 32) * 32 * 2 * 64, device="cuda")
        args = _lib.PfGemmArgs(A=A.data_ptr(), lda=K, B=B.data_ptr(), ldb=K, C=C.data_ptr(), ldc=ncol, M=M, N=N,
                               K=K, epilogue=epi, pos=pos.data_ptr() if epi == 1 else None,
                               rope_cos=cos.data_ptr(), rope_sin=sin.data_ptr(), rope_heads=(N // 128) * 3 // 4 if epi == 1 else 0,
                               row_ss=ss.data_ptr() if epi in (1, 2) else None,
                               ss_out=ss.data_ptr() if xb is not None else None,
                               xb=xb.data_ptr() if xb is not None else None, ldxb=ncol, inv_d=1.0 / K, eps=1e-6,
                               rope_cs=cs_g.data_ptr() if epi == 1 else None)

        def ours():
            _lib.check(lib.pf_gemm_bf16_ex(ctypes.byref(args), stream))

        Cb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        cublas = lambda: torch.matmul(A, B.t(), out=Cb)
        t_ours = time_it(ours)
        t_cub = float("nan") if a.no_cublas else time_it(cublas)
        mm_flops = 2.0 * M * N * K
        r = {"name": name, "M": M, "N": N, "K": K, "ours_us": t_ours * 1e3, "cublas_us": t_cub * 1e3,
             "ours_tflops_useful": flops / t_ours / 1e9, "ours_tflops_issued": mm_flops / t_ours / 1e9,
             "cublas_tflops": mm_flops / t_cub / 1e9}
        res.append(r)
        print(f"{name:16s} M{M} N{N} K{K}: ours {t_ours*1e3:8.1f} us ({r['ours_tflops_issued']:7.1f} TF issued) | "
              f"cuBLAS {t_cub*1e3:8.1f} us ({r['cublas_tflops']:7.1f} TF)", flush=True)
        del A, B, C, Cb
    if a.json:
        json.dump({"cta_group": os.environ.get("PF_GEMM_CTAS", "2"), "results": res}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
