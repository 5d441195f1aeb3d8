"""Exhaustive proof of the fused u8 epilogue used by every u8 kernel.

The reference rounds a blend result v to u8 as floor(RN(RN(v*255) + 0.5))
(service/app.py:75-77 via tensor.py:273-276, all f32). The kernels compute
floor(RN(fma(v, K, 0.5))) instead -- one FFMA (fv_common.cuh:
scale_to_u8_bits). This test checks the two agree for EVERY f32 v in the
range a blend can produce: [0, 1.0625] for K = 255 and [0, 4.25] for the
2:1 fast path's K = 63.75 (sum of four unit values, /4 folded into K).

fma(v, K, 0.5) is evaluated exactly in f64 (v has 24 significant bits, K at
most 8, so v*K + 0.5 fits in 53 bits for v >= 2^-20) and rounded once to f32.
Below 2^-20 both forms are floor(0.5 + tiny) = 0.
"""
import numpy as np
import pytest


def _mismatches(K, hi):
    k32 = np.float32(K)
    top = int(np.array([hi], dtype=np.float32).view(np.uint32)[0])
    step = 1 << 24
    bad = 0
    for lo in range(0, top + 1, step):
        x = np.arange(lo, min(lo + step, top + 1), dtype=np.uint32).view(np.float32)
        ref = np.floor((x * k32) + np.float32(0.5))  # two f32 roundings
        fused = np.floor((x.astype(np.float64) * float(K) + 0.5).astype(np.float32))
        m = (ref != fused) & (x >= np.float32(2.0 ** -20))
        bad += int(m.sum())
    return bad


@pytest.mark.parametrize("K,hi", [(255.0, 1.0625), (63.75, 4.25)])
def test_fused_epilogue_exhaustive(K, hi):
    assert _mismatches(K, hi) == 0


def test_tiny_inputs_round_to_zero():
    x = np.array([0.0, 2.0 ** -149, 2.0 ** -30, 2.0 ** -21], dtype=np.float32)
    for K in (255.0, 63.75):
        ref = np.floor(x * np.float32(K) + np.float32(0.5))
        assert (ref == 0).all()
        fused = np.floor((x.astype(np.float64) * K + 0.5).astype(np.float32))
        assert (fused == 0).all()


def test_gray_quotient_and_tie_from_one_product():
    """fv_gray.cu:gray_u8_quad: for every S + 500 the kernel can form
    (500 .. 255 * 1000 + 500) the high word of (S + 500) * M, M = ceil(2^32 /
    1000), is (S + 500) // 1000 and the low word is below M exactly when
    (S + 500) % 1000 == 0 (the decimal ties that re-run the f64 path); and
    S + 500 = 256 (r + 2 g) + (43 r + 75 g + 114 b + 500), the two byte dot
    products, for the extreme triples."""
    M = np.uint64(4294968)
    assert int(M) == -(-(1 << 32) // 1000)
    s = np.arange(500, 255 * 1000 + 501, dtype=np.uint64)
    p = s * M
    hi, lo = p >> np.uint64(32), p & np.uint64(0xFFFFFFFF)
    assert np.array_equal(hi, s // np.uint64(1000))
    assert np.array_equal(lo < M, s % np.uint64(1000) == 0)
    for r, g, b in [(0, 0, 0), (255, 255, 255), (255, 0, 0), (0, 255, 0), (0, 0, 255), (1, 2, 3)]:
        assert 256 * (r + 2 * g) + (43 * r + 75 * g + 114 * b + 500) == 299 * r + 587 * g + 114 * b + 500
