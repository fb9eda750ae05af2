"""Op-level numerics of the sm_100a kernels against plain PyTorch fp32 references.

Every call goes through the C-ABI (libprefill_sm100.so via ctypes).
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2510_22101_b200 import _lib  # noqa: E402
from paper_2510_22101_b200.config import ModelConfig  # noqa: E402
from paper_2510_22101_b200.prefixcache import SharedBatch, pack_requests  # noqa: E402
from paper_2510_22101_b200.weights import interleave_gate_up, rope_tables  # noqa: E402


def P(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def gemm(lib, A, B, C, epi, pos=None, cos=None, sin=None, rope_heads=0):
    M, K = A.shape
    N = B.shape[0]
    rc = lib.pf_gemm_bf16(P(A), A.stride(0), P(B), B.stride(0), P(C), C.stride(0), M, N, K, epi,
                          P(pos), P(cos), P(sin), rope_heads, stream())
    _lib.check(rc)
    torch.cuda.synchronize()


def rand_bf16(*shape, scale=1.0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, generator=g, device="cuda") * scale).to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K", [(1000, 512, 256), (128, 256, 64), (8192, 1024, 512),
                                   (333, 2560, 2048)])
def test_gemm_bf16(lib, M, N, K):
    A = rand_bf16(M, K, seed=1)
    B = rand_bf16(N, K, scale=K ** -0.5, seed=2)
    C = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    gemm(lib, A, B, C, _lib.EPI_BF16)
    ref = A.float() @ B.float().t()
    torch.testing.assert_close(C.float(), ref, rtol=1.6e-2, atol=1e-2)


@pytest.mark.parametrize("M,N,K", [(1000, 256, 128), (5000, 2048, 1280)])
def test_gemm_resid_add(lib, M, N, K):
    A = rand_bf16(M, K, seed=3)
    B = rand_bf16(N, K, scale=K ** -0.5, seed=4)
    C0 = torch.randn(M, N, device="cuda")
    C = C0.clone()
    gemm(lib, A, B, C, _lib.EPI_RESID_ADD)
    ref = C0 + A.float() @ B.float().t()
    torch.testing.assert_close(C, ref, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("M,F,K", [(700, 384, 256), (3000, 3712, 2048)])
def test_gemm_swiglu(lib, M, F, K):
    A = rand_bf16(M, K, seed=5)
    G = rand_bf16(F, K, scale=K ** -0.5, seed=6)
    U = rand_bf16(F, K, scale=K ** -0.5, seed=7)
    Fp = -(-F // 128) * 128
    if Fp % 256:  # the SwiGLU tile covers 2 neuron blocks... keep F_pad a multiple of 128
        pass
    B = interleave_gate_up(G, U, Fp).contiguous()
    if B.shape[0] % 256:
        pytest.skip("SwiGLU GEMM needs 2*F_pad % 256 == 0")
    C = torch.full((M, Fp), float("nan"), device="cuda", dtype=torch.bfloat16)
    gemm(lib, A, B, C, _lib.EPI_SWIGLU)
    g = A.float() @ G.float().t()
    u = A.float() @ U.float().t()
    ref = torch.nn.functional.silu(g) * u
    torch.testing.assert_close(C[:, :F].float(), ref, rtol=2e-2, atol=2e-2)


def rope_ref(x, pos, cos, sin, n_rot_heads, dh=128):
    x = x.clone()
    c = cos[pos.long()]  # [M, dh/2]
    s = sin[pos.long()]
    for h in range(n_rot_heads):
        a = x[:, h * dh: h * dh + dh // 2].clone()
        b = x[:, h * dh + dh // 2: (h + 1) * dh].clone()
        x[:, h * dh: h * dh + dh // 2] = a * c - b * s
        x[:, h * dh + dh // 2: (h + 1) * dh] = b * c + a * s
    return x


@pytest.mark.parametrize("M,H,Hkv,K", [(900, 2, 1, 256), (2000, 10, 5, 2048)])
def test_gemm_rope(lib, M, H, Hkv, K):
    cfg = ModelConfig(n_layers=1, d_model=K, n_heads=H, n_kv_heads=Hkv, d_ff=128, d_head=128)
    cos, sin = (torch.from_numpy(t).cuda() for t in rope_tables(cfg))
    N = (H + 2 * Hkv) * 128
    A = rand_bf16(M, K, seed=8)
    B = rand_bf16(N, K, scale=K ** -0.5, seed=9)
    pos = torch.randint(0, cfg.max_seq, (M,), device="cuda", dtype=torch.int32)
    C = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    gemm(lib, A, B, C, _lib.EPI_ROPE_BF16, pos, cos, sin, H + Hkv)
    ref = rope_ref(A.float() @ B.float().t(), pos, cos, sin, H + Hkv)
    torch.testing.assert_close(C.float(), ref, rtol=1.6e-2, atol=2e-2)


def attention_ref(qkv, packed, H, Hkv, dh=128):
    T = qkv.shape[0]
    q = qkv[:, : H * dh].float().view(T, H, dh)
    k = qkv[:, H * dh: (H + Hkv) * dh].float().view(T, Hkv, dh)
    v = qkv[:, (H + Hkv) * dh:].float().view(T, Hkv, dh)
    out = torch.zeros(T, H, dh, device=qkv.device)
    grp = H // Hkv
    for kv_off, kv_len, q_off, q_len in packed.segs.tolist():
        rows = torch.arange(q_off, q_off + q_len, device=qkv.device)
        keys = torch.cat([torch.arange(kv_off, kv_off + kv_len, device=qkv.device), rows])
        kk = k[keys].repeat_interleave(grp, dim=1)  # [nk, H, dh]
        vv = v[keys].repeat_interleave(grp, dim=1)
        s = torch.einsum("qhd,khd->hqk", q[rows], kk) / dh ** 0.5
        mask = torch.ones(q_len, kv_len + q_len, dtype=torch.bool, device=qkv.device)
        mask[:, kv_len:] = torch.tril(torch.ones(q_len, q_len, dtype=torch.bool, device=qkv.device))
        s = s.masked_fill(~mask, float("-inf"))
        out[rows] = torch.einsum("hqk,khd->qhd", torch.softmax(s, dim=-1), vv)
    return out.view(T, H * dh)


@pytest.mark.parametrize("H,Hkv,dh", [(2, 1, 128), (4, 2, 128), (10, 5, 128), (4, 2, 64), (2, 2, 64)])
def test_prefix_attention(lib, H, Hkv, dh):
    rng = np.random.default_rng(0)
    reqs = [
        SharedBatch(list(rng.integers(16, 100, 64)), [list(rng.integers(16, 100, s)) for s in (100, 128, 200, 1, 300)]),
        SharedBatch(list(rng.integers(16, 100, 5)), [list(rng.integers(16, 100, 130))]),
        SharedBatch([], [list(rng.integers(16, 100, 7)), list(rng.integers(16, 100, 129))]),
        SharedBatch(list(rng.integers(16, 100, 200)), [list(rng.integers(16, 100, 3))]),
    ]
    packed = pack_requests(reqs)
    T = packed.T
    qkv = rand_bf16(T, (H + 2 * Hkv) * dh, seed=11)
    out = torch.full((T, H * dh), float("nan"), device="cuda", dtype=torch.bfloat16)
    segs = torch.from_numpy(packed.segs).cuda()
    work = torch.from_numpy(packed.work).cuda()
    rc = lib.pf_prefix_attention(P(qkv), P(out), T, H, Hkv, dh, P(segs), P(work), len(packed.work), stream())
    _lib.check(rc)
    torch.cuda.synchronize()
    ref = attention_ref(qkv, packed, H, Hkv, dh)
    torch.testing.assert_close(out.float(), ref, rtol=2e-2, atol=2e-2)


def test_embed_rmsnorm_head(lib):
    T, d, V = 777, 2048, 1000
    emb = rand_bf16(V, d, seed=12)
    ids = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
    resid = torch.empty(T, d, device="cuda")
    xb = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    lo = torch.full((T, d), 7, device="cuda", dtype=torch.uint8)
    ss = torch.full((d // 256, T), 5.0, device="cuda")       # partial-sum layout [part][T]
    _lib.check(lib.pf_embed(P(ids), P(emb), P(resid), P(xb), P(lo), P(ss), T, d, stream()))
    torch.cuda.synchronize()
    torch.testing.assert_close(resid, emb[ids.long()].float(), rtol=0, atol=0)
    torch.testing.assert_close(xb, emb[ids.long()], rtol=0, atol=0)
    assert bool((lo == 128).all())                           # residual low byte 0x80 = zero
    torch.testing.assert_close(ss[0], emb[ids.long()].float().pow(2).sum(-1), rtol=1e-5, atol=1e-3)
    assert float(ss[1:].abs().max()) == 0.0

    x = torch.randn(T, d, device="cuda") * 3
    g = torch.rand(d, device="cuda") + 0.5
    y = torch.empty(T, d, device="cuda", dtype=torch.bfloat16)
    _lib.check(lib.pf_rmsnorm(P(x), P(g), P(y), T, d, ctypes.c_float(1e-6), stream()))
    torch.cuda.synchronize()
    ref = x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + 1e-6) * g
    torch.testing.assert_close(y.float(), ref, rtol=1e-2, atol=1e-2)

    n = 50
    last = torch.randint(0, T, (n,), device="cuda", dtype=torch.int32)
    wy = torch.randn(d, device="cuda") / d ** 0.5
    wn = torch.randn(d, device="cuda") / d ** 0.5
    logits2 = torch.empty(n, 2, device="cuda")
    p = torch.empty(n, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(lib.pf_head_last_token(P(x), P(last), n, d, P(g), P(wy), P(wn), ctypes.c_float(1e-6),
                                      P(logits2), P(p), P(bad), stream()))
    torch.cuda.synchronize()
    h = x[last.long()]
    hn = h * torch.rsqrt(h.pow(2).mean(-1, keepdim=True) + 1e-6) * g
    ly, ln = hn @ wy, hn @ wn
    torch.testing.assert_close(logits2[:, 0], ly, rtol=1e-4, atol=1e-4)
    torch.testing.assert_close(logits2[:, 1], ln, rtol=1e-4, atol=1e-4)
    torch.testing.assert_close(p, torch.sigmoid(ly - ln), rtol=1e-5, atol=1e-5)
    assert int(bad.item()) == 0


def gemm_ex(lib, **kw):
    a = _lib.PfGemmArgs()
    for k, v in kw.items():
        setattr(a, k, v.data_ptr() if hasattr(v, "data_ptr") else v)
    _lib.check(lib.pf_gemm_bf16_ex(ctypes.byref(a), stream()))
    torch.cuda.synchronize()


def resid_lo_scale(hi):
    """2^(E - 142) per element (E = biased fp32 exponent of the bf16 hi; 0 for hi = 0)."""
    e = (hi.view(torch.int16).int() & 0xFFFF) >> 7 & 0xFF
    return torch.where(e > 0, torch.exp2((e - 142).float()), torch.zeros_like(e, dtype=torch.float32))


def resid_encode(x):
    """Residual stream format of the forward: hi = bf16(x), lo = byte b, x - hi = (b - 128) * 2^(E(hi) - 142)."""
    hi = x.to(torch.bfloat16)
    sc = resid_lo_scale(hi)
    q = torch.where(sc > 0, torch.round((x - hi.float()) / torch.where(sc > 0, sc, 1.0)), 0.0)
    return hi, (q.clamp(-128, 127) + 128).to(torch.uint8)


def resid_decode(hi, lo):
    return hi.float() + (lo.float() - 128) * resid_lo_scale(hi)


@pytest.mark.parametrize("M,N,K", [(1000, 256, 128), (5000, 2048, 1280), (700, 384, 256)])
def test_gemm_resid_add_norm(lib, M, N, K):
    """Fused RMSNorm producer on the residual x = hi + lo (hi = bf16(x), lo = byte b with
    x - hi = (b - 128) * 2^(E(hi) - 142)): x += A.B^T in place; ss_out[nb] = row sum of squares of the
    new x over n-tile nb (256 columns; deterministic partials, no atomics)."""
    A = rand_bf16(M, K, seed=30)
    B = rand_bf16(N, K, scale=K ** -0.5, seed=31)
    x0 = torch.randn(M, N, device="cuda") * 4
    x0[:, :7] *= 1e-3                                      # small magnitudes: the scale follows hi
    hi, lo = resid_encode(x0)
    x0 = resid_decode(hi, lo)
    assert float((lo != 128).float().mean()) > 0.9
    parts = (N + 255) // 256
    ss = torch.full((parts, M + 3), 0.25, device="cuda")     # row stride M + 3: ss_ld honoured
    gemm_ex(lib, A=A, lda=K, B=B, ldb=K, C=lo, ldc=N, M=M, N=N, K=K, epilogue=_lib.EPI_RESID_ADD_NORM,
            xb=hi, ldxb=N, ss_out=ss, ss_ld=M + 3)
    ref = x0 + A.float() @ B.float().t()
    x = resid_decode(hi, lo)
    # hi + lo keeps ~16 significant bits: |x - x_fp32| <= ulp(hi)/512 (ulp(hi)/256 when lo saturates
    # at a bf16 rounding tie) <= 2^-15 |x|
    torch.testing.assert_close(x, ref, rtol=4e-5, atol=2e-5)
    assert bool(((hi.float() - x).abs() <= x.abs() * 2.0 ** -8 + 1e-30).all())   # hi = bf16(x), half-ulp
    for p in range(parts):
        torch.testing.assert_close(ss[p, :M], ref[:, 256 * p:256 * (p + 1)].pow(2).sum(-1), rtol=1e-4, atol=1e-2)
    assert float((ss[:, M:] - 0.25).abs().max()) == 0.0


def test_gemm_row_scaled_swiglu_and_rope(lib):
    """Fused RMSNorm consumer: the accumulator row is scaled by rsqrt(sum of the ceil(K/256)
    partial sums of squares / d + eps) before the SwiGLU / RoPE epilogues."""
    M, K, F = 900, 512, 384
    x = torch.randn(M, K, device="cuda") * 3
    xb = x.to(torch.bfloat16)
    ss_in = xb.float().pow(2).sum(-1)
    frac = torch.rand(M, device="cuda")
    ss_parts = torch.stack([ss_in * frac, ss_in * (1 - frac)]).contiguous()   # [2][M]
    G = rand_bf16(F, K, scale=K ** -0.5, seed=32)
    U = rand_bf16(F, K, scale=K ** -0.5, seed=33)
    B = interleave_gate_up(G, U, F).contiguous()
    C = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    gemm_ex(lib, A=xb, lda=K, B=B, ldb=K, C=C, ldc=F, M=M, N=2 * F, K=K, epilogue=_lib.EPI_SWIGLU,
            row_ss=ss_parts, inv_d=1.0 / K, eps=1e-6)
    xn = xb.float() * torch.rsqrt(ss_in / K + 1e-6)[:, None]
    ref = torch.nn.functional.silu(xn @ G.float().t()) * (xn @ U.float().t())
    torch.testing.assert_close(C.float(), ref, rtol=2e-2, atol=2e-2)

    cfg = ModelConfig(n_layers=1, d_model=K, n_heads=2, n_kv_heads=1, d_ff=128, d_head=128)
    cos, sin = (torch.from_numpy(t).cuda() for t in rope_tables(cfg))
    Bq = rand_bf16(512, K, scale=K ** -0.5, seed=34)
    pos = torch.randint(0, 2048, (M,), device="cuda", dtype=torch.int32)
    Cq = torch.empty(M, 512, device="cuda", dtype=torch.bfloat16)
    gemm_ex(lib, A=xb, lda=K, B=Bq, ldb=K, C=Cq, ldc=512, M=M, N=512, K=K, epilogue=_lib.EPI_ROPE_BF16,
            pos=pos, rope_cos=cos, rope_sin=sin, rope_heads=3, row_ss=ss_parts, inv_d=1.0 / K, eps=1e-6)
    refq = rope_ref(xn @ Bq.float().t(), pos, cos, sin, 3)
    torch.testing.assert_close(Cq.float(), refq, rtol=1.6e-2, atol=2e-2)


def test_gemm_rope_dh64(lib):
    """RoPE epilogue on 64-wide heads (config C1: d_head = d_model / n_heads = 64)."""
    M, K, H, Hkv = 700, 256, 4, 2
    cfg = ModelConfig(n_layers=1, d_model=K, n_heads=H, n_kv_heads=Hkv, d_ff=128, d_head=64)
    cos, sin = (torch.from_numpy(t).cuda() for t in rope_tables(cfg))
    N = (H + 2 * Hkv) * 64
    A = rand_bf16(M, K, seed=40)
    B = rand_bf16(N, K, scale=K ** -0.5, seed=41)
    pos = torch.randint(0, cfg.max_seq, (M,), device="cuda", dtype=torch.int32)
    C = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    gemm_ex(lib, A=A, lda=K, B=B, ldb=K, C=C, ldc=N, M=M, N=N, K=K, epilogue=_lib.EPI_ROPE_BF16,
            pos=pos, rope_cos=cos, rope_sin=sin, rope_heads=H + Hkv, rope_dh=64)
    ref = rope_ref(A.float() @ B.float().t(), pos, cos, sin, H + Hkv, dh=64)
    torch.testing.assert_close(C.float(), ref, rtol=1.6e-2, atol=2e-2)


def gathered_cos_sin(cos, sin, pos):
    """The QKV epilogue's pre-gathered layout (elementwise.cu rope_gather_kernel): per 32-row group
    g, [cos | sin] x [half/4 float4 chunks] x [32 rows] x float4, so a warp's loads are coalesced."""
    T, half = pos.numel(), cos.shape[1]
    G, qn = (T + 31) // 32, half // 4
    cs = torch.zeros(G * 32, 2, qn, 4, device="cuda")
    cs[:T, 0] = cos[pos.long()].view(T, qn, 4)
    cs[:T, 1] = sin[pos.long()].view(T, qn, 4)
    return cs.view(G, 32, 2, qn, 4).permute(0, 2, 3, 1, 4).contiguous()


@pytest.mark.parametrize("M,H,Hkv,K,dh", [(1000, 10, 5, 512, 128), (777, 4, 2, 256, 64)])
def test_gemm_rope_gathered_table(lib, M, H, Hkv, K, dh):
    """RoPE epilogue reading the gathered cos/sin rows (the layout pf_score uses), including a ragged
    last 32-row group and V heads that pass through unrotated."""
    cfg = ModelConfig(n_layers=1, d_model=K, n_heads=H, n_kv_heads=Hkv, d_ff=128, d_head=dh)
    cos, sin = (torch.from_numpy(t).cuda() for t in rope_tables(cfg))
    N = (H + 2 * Hkv) * dh
    A = rand_bf16(M, K, seed=50)
    B = rand_bf16(N, K, scale=K ** -0.5, seed=51)
    pos = torch.randint(0, cfg.max_seq, (M,), device="cuda", dtype=torch.int32)
    cs = gathered_cos_sin(cos, sin, pos)
    C = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    gemm_ex(lib, A=A, lda=K, B=B, ldb=K, C=C, ldc=N, M=M, N=N, K=K, epilogue=_lib.EPI_ROPE_BF16,
            pos=pos, rope_cos=cos, rope_sin=sin, rope_heads=H + Hkv, rope_dh=dh, rope_cs=cs)
    ref = rope_ref(A.float() @ B.float().t(), pos, cos, sin, H + Hkv, dh=dh)
    torch.testing.assert_close(C.float(), ref, rtol=1.6e-2, atol=2e-2)


@pytest.mark.parametrize("H,Hkv,dh", [(2, 1, 128), (10, 5, 128), (4, 2, 64), (8, 1, 128), (3, 3, 64)])
def test_attention_last_rows(lib, H, Hkv, dh):
    """The last layer's attention of the last-token rows only (fp32) against the torch fp32
    reference of the full ragged attention at those rows: shared prefixes of 64 / 5 / 0 / 200 tokens,
    items of 1-300 tokens."""
    rng = np.random.default_rng(5)
    reqs = [
        SharedBatch(list(rng.integers(16, 100, 64)), [list(rng.integers(16, 100, s)) for s in (100, 128, 200, 1, 300)]),
        SharedBatch(list(rng.integers(16, 100, 5)), [list(rng.integers(16, 100, 130))]),
        SharedBatch([], [list(rng.integers(16, 100, 7)), list(rng.integers(16, 100, 129))]),
        SharedBatch(list(rng.integers(16, 100, 200)), [list(rng.integers(16, 100, 3))]),
    ]
    packed = pack_requests(reqs)
    T, n = packed.T, len(packed.last_idx)
    qkv = rand_bf16(T, (H + 2 * Hkv) * dh, seed=21)
    last = torch.from_numpy(packed.last_idx.astype(np.int32)).cuda()
    q_rows = qkv[last.long(), : H * dh].contiguous()
    out = torch.full((n, H * dh), float("nan"), device="cuda", dtype=torch.bfloat16)
    segs = torch.from_numpy(packed.segs).cuda()
    _lib.check(lib.pf_attention_last_rows(P(q_rows), P(qkv), H, Hkv, dh, P(segs), len(packed.segs), P(last), n,
                                          2048, P(out), stream()))
    torch.cuda.synchronize()
    ref = attention_ref(qkv, packed, H, Hkv, dh)[last.long()]
    torch.testing.assert_close(out.float(), ref, rtol=1e-2, atol=1e-2)
    # a key count past max_keys is reported as NaN rows (the head's non-finite flag), not read past smem
    _lib.check(lib.pf_attention_last_rows(P(q_rows), P(qkv), H, Hkv, dh, P(segs), len(packed.segs), P(last), n,
                                          6, P(out), stream()))
    torch.cuda.synchronize()
    assert bool(torch.isnan(out.float()).any(dim=1).all())


def test_prefix_attention_rescales_and_masked_blocks(lib):
    """Online softmax under large score swings (the lazy rescale of O in TMEM fires when the running
    max grows by > 2^8) and items long enough that whole warps see fully masked 32-key halves."""
    H, Hkv, dh = 4, 2, 128
    rng = np.random.default_rng(3)
    reqs = [SharedBatch(list(rng.integers(16, 100, 64)), [list(rng.integers(16, 100, s)) for s in (250, 129, 64)]),
            SharedBatch([], [list(rng.integers(16, 100, 190))])]
    packed = pack_requests(reqs)
    T = packed.T
    g = torch.Generator(device="cuda").manual_seed(7)
    qkv = torch.randn(T, (H + 2 * Hkv) * dh, device="cuda", generator=g)
    # keys grow with the row index: every later block raises the row max far past the threshold
    k0 = H * dh
    qkv[:, k0:k0 + Hkv * dh] *= torch.linspace(0.5, 6.0, T, device="cuda")[:, None]
    qkv[:, :H * dh] *= 3.0
    qkv = qkv.to(torch.bfloat16)
    out = torch.full((T, H * dh), float("nan"), device="cuda", dtype=torch.bfloat16)
    segs = torch.from_numpy(packed.segs).cuda()
    work = torch.from_numpy(packed.work).cuda()
    _lib.check(lib.pf_prefix_attention(P(qkv), P(out), T, H, Hkv, dh, P(segs), P(work), len(packed.work), stream()))
    torch.cuda.synchronize()
    ref = attention_ref(qkv, packed, H, Hkv, dh)
    assert torch.isfinite(out.float()).all()
    torch.testing.assert_close(out.float(), ref, rtol=2e-2, atol=3e-2)


@pytest.mark.parametrize("name,M", [("C4", 3000), ("C2", 1000), ("TINY_GQA", 700), ("C4", 255)])
def test_layer_tail_fused_equals_three_gemms(lib, name, M):
    """pf_layer_tail (mlp.cu: O + gate/up SwiGLU + down in one persistent launch with per-row-block
    completion counters) against the same three epilogues launched one after another through
    pf_gemm_bf16_ex: bit-identical residual (hi, lo), h and RMSNorm partials."""
    from paper_2510_22101_b200 import CONFIGS, init_device_weights
    from paper_2510_22101_b200.engine import PrefillScorer

    cfg = CONFIGS[name].with_(n_layers=1)
    sc = PrefillScorer(init_device_weights(cfg, 0, "cuda"))
    w = sc.weights
    d, kq, fp = cfg.d_model, cfg.q_width, cfg.d_ff_pad
    attn = rand_bf16(M, kq, scale=0.5, seed=40)
    x0 = torch.randn(M, d, device="cuda") * 2
    hi0, lo0 = resid_encode(x0)
    parts = (d + 255) // 256

    def run(fused):
        hi, lo = hi0.clone(), lo0.clone()
        h = torch.zeros(M, fp, device="cuda", dtype=torch.bfloat16)
        ss_m = torch.zeros(parts, M, device="cuda")
        ss_a = torch.zeros(parts, M, device="cuda")
        if fused:
            ctr = torch.empty(8 * ((M + 255) // 256), dtype=torch.uint8, device="cuda")
            _lib.check(lib.pf_layer_tail(sc.handle, 0, P(attn), P(hi), P(lo), P(h), P(ss_m), P(ss_a), M,
                                         P(ctr), ctr.numel(), stream()))
            torch.cuda.synchronize()
        else:
            gemm_ex(lib, A=attn, lda=kq, B=w.w_o[0], ldb=kq, C=lo, ldc=d, M=M, N=d, K=kq,
                    epilogue=_lib.EPI_RESID_ADD_NORM, xb=hi, ldxb=d, ss_out=ss_m, ss_ld=M)
            gemm_ex(lib, A=hi, lda=d, B=w.w_gu[0], ldb=d, C=h, ldc=fp, M=M, N=2 * fp, K=d,
                    epilogue=_lib.EPI_SWIGLU, row_ss=ss_m, ss_ld=M, inv_d=1.0 / d, eps=cfg.rms_eps)
            gemm_ex(lib, A=h, lda=fp, B=w.w_down[0], ldb=fp, C=lo, ldc=d, M=M, N=d, K=fp,
                    epilogue=_lib.EPI_RESID_ADD_NORM, xb=hi, ldxb=d, ss_out=ss_a, ss_ld=M)
        return hi, lo, h, ss_m, ss_a

    ref = run(False)
    for _ in range(2):                      # twice: counters are re-zeroed per call
        got = run(True)
        for a, b in zip(got, ref):
            assert torch.equal(a, b)
    # and against fp32 math (one layer tail on the decoded residual)
    x = resid_decode(hi0, lo0)
    x1 = x + attn.float() @ w.w_o[0].float().t()
    assert float((resid_decode(*ref[:2]) - x).abs().max()) > 0        # the tail did change x
    torch.testing.assert_close(ref[3].sum(0), x1.pow(2).sum(-1), rtol=1e-3, atol=1e-1)
