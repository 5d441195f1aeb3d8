"""CPU: pin the oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py), the reference's own known-answer tests, and
its scalar-loop twins. No GPU needed."""
import numpy as np
import pytest

import oracle as O
from paper_2505_12425_b200 import synth
from _helpers import golden


class TestGoldenPinning:
    @pytest.mark.parametrize("key", ["u8_rand", "u8_odd", "u8_kat", "u8_ties", "f32_rand"])
    def test_gray_matches_reference_output(self, key):
        g = golden("gray.npz")
        assert np.array_equal(O.gray_from_rgb(g[key + "_src"]), g[key + "_dst"])

    def test_gray_tie_set_is_complete(self):
        # every (r,g,b) with 299r+587g+114b = 500 (mod 1000): the cases where
        # the f64 op order, not the exact decimal, decides the rounding
        g = golden("gray.npz")
        assert g["u8_ties_src"].shape == (1, 16782, 3)

    @pytest.mark.parametrize("i", range(5))
    def test_resize_f32_matches_reference_output(self, i):
        g = golden("resize_f32.npz")
        a, d = g[f"c{i}_src"], g[f"c{i}_dst"]
        assert np.array_equal(O.resize_bilinear(a, d.shape[1], d.shape[0]), d)

    @pytest.mark.parametrize("i", range(7))
    def test_resize_u8_matches_reference_output(self, i):
        g = golden("resize_u8.npz")
        a, d = g[f"c{i}_src"], g[f"c{i}_dst"]
        assert np.array_equal(O.resize_u8(a, d.shape[1], d.shape[0]), d)

    @pytest.mark.parametrize("i", range(7))
    def test_resize_u8_row_band_is_exact(self, i):
        g = golden("resize_u8.npz")
        a, d = g[f"c{i}_src"], g[f"c{i}_dst"]
        h = d.shape[0]
        lo, hi = h // 3, max(h // 3 + 1, (2 * h) // 3)
        assert np.array_equal(O.resize_u8(a, d.shape[1], h, rows=(lo, hi)), d[lo:hi])

    def test_to_float_scaled_and_cast(self):
        g = golden("scalars.npz")
        assert np.array_equal(O.to_float_scaled(g["to_float_src"]), g["to_float_dst"])
        assert np.array_equal(O.cast_to_u8(g["cast_src"]), g["cast_dst"])


class TestReferenceKATs:
    """The reference's own known answers (pkg/tests/test_imgproc.py, test_image.py, test_tensor.py)."""

    def test_white_black(self):
        a = np.array([[[255, 255, 255], [0, 0, 0]]], np.uint8)
        assert O.gray_from_rgb(a).ravel().tolist() == [255, 0]

    def test_pure_red_is_76(self):
        assert O.gray_from_rgb(np.array([[[255, 0, 0]]], np.uint8)).item() == 76

    def test_bilinear_1x2_to_1x4(self):
        a = np.array([[[0.0], [1.0]]], np.float32)
        assert np.allclose(O.resize_bilinear(a, 4, 1).ravel(), [0.0, 0.25, 0.75, 1.0], atol=1e-7)

    def test_bilinear_identity_and_constant(self, rng):
        a = rng.random((7, 5, 3), dtype=np.float32)
        assert np.max(np.abs(O.resize_bilinear(a, 5, 7) - a)) <= 1e-6
        c = np.full((3, 3, 3), 0.625, np.float32)
        assert np.all(O.resize_bilinear(c, 7, 2) == np.float32(0.625))

    def test_to_float_128(self):
        assert O.to_float_scaled(np.array([128], np.uint8))[0] == np.float32(128) / np.float32(255)

    def test_cast_half_away(self):
        assert O.cast_to_u8(np.array([1.5, 2.5, 0.4, -3.0, 300.0], np.float32)).tolist() == [2, 3, 0, 0, 255]


class TestScalarTwins:
    def test_gray_scalar(self, rng):
        a = rng.integers(0, 256, (9, 13, 3), dtype=np.uint8)
        assert np.array_equal(O.gray_scalar(a), O.gray_from_rgb(a))

    @pytest.mark.parametrize("shape", [(6, 4, 11, 3), (9, 9, 4, 13), (2, 2, 5, 5), (12, 8, 4, 4)])
    def test_bilinear_scalar_u8_and_f32(self, rng, shape):
        sw, sh, dw, dh = shape
        a = rng.integers(0, 256, (sh, sw, 3), dtype=np.uint8)
        assert np.array_equal(O.bilinear_scalar(a, dw, dh), O.resize_u8(a, dw, dh))
        f = rng.random((sh, sw, 2), dtype=np.float32)
        assert np.array_equal(O.bilinear_scalar(f, dw, dh), O.resize_bilinear(f, dw, dh))

    @pytest.mark.parametrize("dtype", [np.uint8, np.float32])
    @pytest.mark.parametrize("perspective", [False, True])
    def test_warp_scalar(self, rng, dtype, perspective):
        h, w = 14, 17
        a = rng.integers(0, 256, (h, w, 3), dtype=np.uint8) if dtype == np.uint8 else rng.random((h, w, 3), dtype=np.float32)
        if perspective:
            hm = np.eye(3) + rng.normal(0, 0.02, (3, 3))
            hm[2, 2] = 1.0
            minv = O.invert_homography(hm)
            v = O.warp_perspective(a, minv, 12, 19, border=7)
        else:
            m = O.affine_forward(5, w, h)
            minv = O.invert_affine(m)
            v = O.warp_affine(a, minv, 12, 19, border=7)
        s = O.warp_scalar(a, minv, 12, 19, border=7, perspective=perspective)
        assert np.array_equal(v, s)

    def test_fused_scalar(self, rng):
        a = rng.integers(0, 256, (27, 48, 3), dtype=np.uint8)
        v = O.resize_normalize_chw(a, 16, 16, synth.MEAN, synth.STD)
        s = O.resize_normalize_chw_scalar(a, 16, 16, synth.MEAN, synth.STD)
        assert np.array_equal(v, s)


class TestBuilderContracts:
    def test_identity_warp_reproduces_input(self, rng):
        a = rng.integers(0, 256, (10, 12, 3), dtype=np.uint8)
        assert np.array_equal(O.warp_affine(a, np.eye(3)[:2], 10, 12), a)
        assert np.array_equal(O.warp_perspective(a, np.eye(3), 10, 12), a)
        f = rng.random((10, 12, 3), dtype=np.float32)
        assert np.array_equal(O.warp_affine(f, np.eye(3)[:2], 10, 12), f)

    def test_pure_scale_affine_equals_resize_interior(self, rng):
        # dst = 2x src: inverse map sx = 0.5 x - 0.25 is the resize pixel-centre map
        a = rng.random((16, 16, 3), dtype=np.float32)
        minv = np.array([[0.5, 0.0, -0.25], [0.0, 0.5, -0.25]])
        warp = O.warp_affine(a, minv, 32, 32)
        res = O.resize_bilinear(a, 32, 32)
        assert np.array_equal(warp[1:-1, 1:-1], res[1:-1, 1:-1])

    def test_fused_equals_composition(self, rng):
        a = rng.integers(0, 256, (54, 96, 3), dtype=np.uint8)
        u = O.resize_u8(a, 32, 32)
        lut = O.normalize_lut(synth.MEAN, synth.STD)
        expect = np.stack([lut[c][u[:, :, c]] for c in range(3)])
        assert np.array_equal(O.resize_normalize_chw(a, 32, 32, synth.MEAN, synth.STD), expect)

    def test_zero_w_gives_raw_border(self):
        a = np.full((4, 4, 1), 200, np.uint8)
        hm = np.array([[1.0, 0, 0], [0, 1.0, 0], [1.0, 0, -2.0]])  # W = x - 2
        out = O.warp_perspective(a, hm, 4, 4, border=9)
        assert out[0, 2, 0] == 9

    def test_synth_params_match_oracle(self):
        for i in range(4):
            assert np.array_equal(synth.affine_forward(31000 + i, 1920, 1080), O.affine_forward(31000 + i, 1920, 1080))
            assert np.array_equal(synth.perspective_forward(41000 + i), O.perspective_forward(41000 + i))
        assert np.array_equal(synth.seeded_u8_image(5, 4, 3, 9), O.seeded_u8_image(5, 4, 3, 9))

    def test_host_lut_matches_oracle(self):
        from paper_2505_12425_b200.imgproc import normalize_lut

        assert np.array_equal(normalize_lut(synth.MEAN, synth.STD), O.normalize_lut(synth.MEAN, synth.STD))


class TestGeomGolden:
    """flip / nearest / sobel restatements vs the reference's outputs."""

    def test_flip(self):
        g = golden("geom.npz")
        for i in range(4):
            assert np.array_equal(O.flip_horizontal(g[f"flip{i}_src"]), g[f"flip{i}_dst"])

    def test_nearest(self):
        g = golden("geom.npz")
        for i in range(6):
            d = g[f"near{i}_dst"]
            assert np.array_equal(O.resize_nearest(g[f"near{i}_src"], d.shape[1], d.shape[0]), d)

    def test_sobel(self):
        g = golden("geom.npz")
        for i in range(4):
            assert np.array_equal(O.sobel(g[f"sobel{i}_src"]), g[f"sobel{i}_dst"])

    def test_reference_kats(self):
        # pkg/tests/test_imgproc.py:61-105
        assert O.resize_nearest(np.array([[[10], [200]]], np.uint8), 4, 1).ravel().tolist() == [10, 10, 200, 200]
        assert O.resize_nearest(np.array([[[1], [2], [3], [4]]], np.uint8), 2, 1).ravel().tolist() == [1, 3]
        assert O.flip_horizontal(np.array([[[10], [20]]], np.uint8)).ravel().tolist() == [20, 10]
        ramp = np.tile(np.arange(6, dtype=np.float32)[None, :, None], (5, 1, 1))
        assert np.allclose(O.sobel(ramp)[1:-1, 1:-1, 0], 8.0)
