"""The residual stream's storage format: x = hi + (b - 128) * 2^(E(hi) - 142), hi =
bf16(x), b one byte.  A bit-level numpy restatement of the device helpers in csrc/ptx.cuh
(resid_decode, resid_lo_encode, pack_lo4), run on the CPU: it pins the format's precision and the
float tricks it relies on (exponent-field scales, the 1.5 * 2^23 rounding trick, byte packing), which
the GPU tests then check the kernels against (tests/test_ops_gpu.py::test_gemm_resid_add_norm)."""

import numpy as np

MAGIC = np.float32(12583040.0)          # 1.5 * 2^23 + 128
MAGIC_MAX = np.float32(12583167.0)      # byte 255


def f32(u):
    return np.asarray(u, dtype=np.uint32).view(np.float32)


def u32(x):
    return np.asarray(x, dtype=np.float32).view(np.uint32)


def bf16_rne(x):
    b = u32(x).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return f32(r.astype(np.uint32))


def lo_encode(x, hi):
    """resid_lo_encode: the byte of x against hi (as the low byte of a float)."""
    inv = f32(np.uint32(0x86800000) - (u32(hi) & np.uint32(0x7F800000)))   # 2^(142 - E)
    with np.errstate(over="ignore", invalid="ignore"):
        t = np.minimum(np.float32(x - hi) * inv + MAGIC, MAGIC_MAX).astype(np.float32)
    return (u32(t) & 0xFF).astype(np.uint8)


def lo_decode(hi, b):
    """resid_decode: hi + (b - 128) * 2^(E - 142) via the byte placed under 1.5 * 2^23."""
    q = f32(np.uint32(0x4B400000) | b.astype(np.uint32)) - MAGIC
    scale = f32(u32(hi) & np.uint32(0x7F800000)) * np.float32(2.0 ** -15)
    return (q * scale + hi).astype(np.float32)


def test_round_trip_precision():
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(200_000) * np.exp(rng.uniform(-12, 12, 200_000))).astype(np.float32)
    hi = bf16_rne(x)
    y = lo_decode(hi, lo_encode(x, hi))
    rel = np.abs(y.astype(np.float64) - x) / np.abs(x.astype(np.float64))
    # quantum ulp(hi)/256 <= 2^-15 |x|; half a quantum off except where b saturates at a bf16 tie
    assert rel.max() <= 2.0 ** -15
    assert np.median(rel) < 2.0 ** -17                   # ~quantum/4 on average: 2^-17.6 relative
    # against plain bf16 (8 significant bits) the low byte buys 8 bits
    rel_bf16 = np.abs(hi.astype(np.float64) - x) / np.abs(x.astype(np.float64))
    assert np.median(rel_bf16) > 100 * np.median(rel)


def test_zero_and_exact_bf16_values():
    x = np.array([0.0, -0.0, 1.0, -2.5, 3.0e-30, 65280.0], dtype=np.float32)
    hi = bf16_rne(x)
    b = lo_encode(x, hi)
    assert (b[hi == x] == 128).all()                       # exact bf16 values: lo byte 0x80 = zero
    np.testing.assert_array_equal(lo_decode(hi, np.full(len(x), 128, np.uint8)), hi)


def test_rounding_is_nearest():
    # the FMA into 1.5 * 2^23 rounds v = (x - hi) * 2^(142 - E) to the nearest integer
    hi = np.float32(1.0)                                    # E = 127: quantum 2^-15
    for k in range(-120, 121, 7):
        for frac in (0.25, 0.49, 0.51, 0.75):
            x = np.float32(1.0 + (k + frac) * 2.0 ** -15)
            b = int(lo_encode(np.array([x]), np.array([hi]))[0])
            assert b - 128 == int(np.rint(k + frac))


def test_pack_lo4_byte_order():
    """pack_lo4 = byte_perm(byte_perm(t0, t1, 0x0040), byte_perm(t2, t3, 0x0040), 0x5410): byte i of
    the packed word is the low byte of t_i (column 4w + i of the 64-byte lo row)."""
    def byte_perm(x, y, s):
        by = [(x >> (8 * i)) & 0xFF for i in range(4)] + [(y >> (8 * i)) & 0xFF for i in range(4)]
        return sum(by[(s >> (4 * n)) & 7] << (8 * n) for n in range(4))

    t = [0x4B400000 | v for v in (0x11, 0x22, 0x33, 0x44)]
    w = byte_perm(byte_perm(t[0], t[1], 0x0040), byte_perm(t[2], t[3], 0x0040), 0x5410)
    assert w == 0x44332211
    # decode's byte_perm(lo4, 0x4B400000, 0x7650 | k) puts byte k under 1.5 * 2^23
    for k in range(4):
        assert byte_perm(w, 0x4B400000, 0x7650 | k) == 0x4B400000 | (0x11 * (k + 1))
