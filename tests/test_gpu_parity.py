"""GPU parity: every sm_100a kernel vs the oracle / reference golden vectors.

Bar (north_star): bit-exact for integer/indexing work, <= 1 LSB for u8 results
of float interpolation, rel 1e-5 for f32. Every kernel here reproduces the
reference's rounding op-for-op, so every assertion below is the stricter
BIT-EXACT bar (`np.array_equal`); `assert_within_gate` documents the looser
north_star gate and is checked too, so a regression shows which bar broke.
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2505_12425_b200 as fv
from _helpers import forced_path, golden, oracle_map
from paper_2505_12425_b200 import _native, synth

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def assert_within_gate(got, ref):
    if ref.dtype == np.uint8:
        assert np.max(np.abs(got.astype(np.int16) - ref.astype(np.int16))) <= 1
    else:
        assert np.all(np.abs(got.astype(np.float64) - ref) <= 1e-5 * np.maximum(1.0, np.abs(ref)))


def assert_exact(got, ref):
    assert got.shape == ref.shape and got.dtype == ref.dtype
    if not np.array_equal(got, ref):
        assert_within_gate(got, ref)
        bad = np.argwhere(got != ref)
        pytest.fail(f"{len(bad)} elements differ (within gate), first at {bad[0].tolist()}")


@pytest.fixture(params=[0, 1, 2], ids=["auto", "gather", "strip"])
def resize_path(request):
    with forced_path("resize", request.param):
        yield request.param


# ---------------------------------------------------------------------------
# a1 gray
# ---------------------------------------------------------------------------

class TestGray:
    @pytest.mark.parametrize("key", ["u8_rand", "u8_odd", "u8_kat", "u8_ties", "f32_rand"])
    def test_golden(self, key):
        g = golden("gray.npz")
        src = cu(g[key + "_src"])
        dst = torch.zeros(src.shape[:2] + (1,), dtype=src.dtype, device=DEV)
        fv.gray_from_rgb(src, dst)
        assert_exact(host(dst), g[key + "_dst"])

    def test_exhaustive_all_2_24_triples(self):
        r, g, b = np.meshgrid(np.arange(256), np.arange(256), np.arange(256), indexing="ij")
        a = np.stack([r, g, b], -1).astype(np.uint8).reshape(4096, 4096, 3)
        dst = torch.zeros((4096, 4096, 1), dtype=torch.uint8, device=DEV)
        fv.gray_from_rgb(cu(a), dst)
        assert_exact(host(dst), O.gray_from_rgb(a))

    def test_config0_full_frame(self):
        a = synth.seeded_u8_image(1920, 1080, 3, seed=synth.SEED_GRAY)
        dst = torch.zeros((1080, 1920, 1), dtype=torch.uint8, device=DEV)
        fv.gray_from_rgb(cu(a), dst)
        assert_exact(host(dst), O.gray_from_rgb(a))

    def test_crop_views_and_ragged_widths(self, rng):
        parent = rng.integers(0, 256, (40, 77, 3), dtype=np.uint8)
        p = cu(parent)
        for (y, x, h, w) in [(1, 3, 17, 23), (0, 0, 40, 77), (5, 1, 1, 1), (2, 16, 30, 33)]:
            dst = torch.zeros((h, w, 1), dtype=torch.uint8, device=DEV)
            fv.gray_from_rgb(p[y:y + h, x:x + w], dst)
            assert_exact(host(dst), O.gray_from_rgb(parent[y:y + h, x:x + w]))

    def test_batched(self, rng):
        a = rng.integers(0, 256, (5, 33, 48, 3), dtype=np.uint8)
        dst = torch.zeros((5, 33, 48, 1), dtype=torch.uint8, device=DEV)
        fv.gray_from_rgb(cu(a), dst)
        assert_exact(host(dst), np.stack([O.gray_from_rgb(x) for x in a]))

    def test_f32_matches_oracle(self, rng):
        a = rng.random((19, 37, 3), dtype=np.float32)
        dst = torch.zeros((19, 37, 1), dtype=torch.float32, device=DEV)
        fv.gray_from_rgb(cu(a), dst)
        assert_exact(host(dst), O.gray_from_rgb(a))


# ---------------------------------------------------------------------------
# a4 to_float_scaled
# ---------------------------------------------------------------------------

def test_to_float_scaled_every_value():
    g = golden("scalars.npz")
    dst = torch.zeros((1, 256, 1), dtype=torch.float32, device=DEV)
    fv.to_float_scaled(cu(g["to_float_src"]), dst)
    assert_exact(host(dst), g["to_float_dst"])


def test_to_float_scaled_shapes(rng):
    for shape in [(7, 13, 3), (64, 64, 4), (1, 1, 1)]:
        a = rng.integers(0, 256, shape, dtype=np.uint8)
        dst = torch.zeros(shape, dtype=torch.float32, device=DEV)
        fv.to_float_scaled(cu(a), dst)
        assert_exact(host(dst), O.to_float_scaled(a))


# ---------------------------------------------------------------------------
# a3 / a6 resize
# ---------------------------------------------------------------------------

class TestResize:
    @pytest.mark.parametrize("i", range(5))
    def test_f32_golden(self, resize_path, i):
        g = golden("resize_f32.npz")
        a, d = g[f"c{i}_src"], g[f"c{i}_dst"]
        dst = torch.zeros(d.shape, dtype=torch.float32, device=DEV)
        fv.resize_bilinear(cu(a), dst)
        assert_exact(host(dst), d)

    @pytest.mark.parametrize("i", range(7))
    def test_u8_golden(self, resize_path, i):
        g = golden("resize_u8.npz")
        a, d = g[f"c{i}_src"], g[f"c{i}_dst"]
        dst = torch.zeros(d.shape, dtype=torch.uint8, device=DEV)
        fv.resize_bilinear_u8(cu(a), dst)
        assert_exact(host(dst), d)

    def test_f32_kats(self, resize_path, rng):
        a = rng.random((7, 5, 3), dtype=np.float32)
        dst = torch.zeros((7, 5, 3), dtype=torch.float32, device=DEV)
        fv.resize_bilinear(cu(a), dst)
        assert_exact(host(dst), a)  # same-size resize is the identity
        dst = torch.zeros((1, 4, 1), dtype=torch.float32, device=DEV)
        fv.resize_bilinear(cu(np.array([[[0.0], [1.0]]], np.float32)), dst)
        assert host(dst).ravel().tolist() == [0.0, 0.25, 0.75, 1.0]

    @pytest.mark.parametrize("shape", [(23, 17, 11, 29, 3), (100, 3, 7, 250, 1), (64, 64, 33, 17, 4),
                                       (40, 30, 160, 120, 2), (1000, 10, 37, 3, 3), (3, 2, 2000, 9, 3)])
    def test_u8_and_f32_random_shapes(self, resize_path, rng, shape):
        sw, sh, dw, dh, c = shape
        a = rng.integers(0, 256, (sh, sw, c), dtype=np.uint8)
        dst = torch.zeros((dh, dw, c), dtype=torch.uint8, device=DEV)
        fv.resize_bilinear_u8(cu(a), dst)
        assert_exact(host(dst), O.resize_u8(a, dw, dh))
        f = rng.random((sh, sw, c), dtype=np.float32)
        dstf = torch.zeros((dh, dw, c), dtype=torch.float32, device=DEV)
        fv.resize_bilinear(cu(f), dstf)
        assert_exact(host(dstf), O.resize_bilinear(f, dw, dh))

    def test_u8_crop_views_batched(self, resize_path, rng):
        parent = rng.integers(0, 256, (3, 50, 90, 3), dtype=np.uint8)
        p = cu(parent)
        src = p[:, 3:41, 5:74]  # pitch kept from the parent, unaligned base
        dst_parent = torch.zeros((3, 30, 80, 3), dtype=torch.uint8, device=DEV)
        dst = dst_parent[:, 2:27, 1:61]
        fv.resize_bilinear_u8(src, dst)
        expect = np.stack([O.resize_u8(parent[i, 3:41, 5:74], 60, 25) for i in range(3)])
        assert_exact(host(dst), expect)
        assert not host(dst_parent)[:, :2].any()  # nothing written outside the view

    @pytest.mark.parametrize("c", [1, 3, 4])
    @pytest.mark.parametrize("geom", [(74, 10, 37, 5), (128, 70, 64, 35), (12, 5, 24, 10), (40, 70, 80, 140),
                                      (8, 1, 16, 2), (2, 2, 1, 1)])
    def test_u8_integer_ratio_paths(self, resize_path, rng, c, geom):
        """Exact 2:1 / 1:2 shapes (fast paths under 'auto'): ragged tail groups,
        band boundaries (>32 source rows), 1-row sources, batches."""
        sw, sh, dw, dh = geom
        a = rng.integers(0, 256, (2, sh, sw, c), dtype=np.uint8)
        dst = torch.zeros((2, dh, dw, c), dtype=torch.uint8, device=DEV)
        fv.resize_bilinear_u8(cu(a), dst)
        out = host(dst)
        for i in range(2):
            assert_exact(out[i], O.resize_u8(a[i], dw, dh))

    @pytest.mark.parametrize("geom", [(64, 48, 32, 24), (64, 48, 128, 96), (64, 48, 96, 72), (64, 48, 40, 30)])
    @pytest.mark.parametrize("path", [0, 1, 2])
    def test_u8_every_byte_value(self, geom, path):
        """Every u8 value enters the kernels' u8 -> RN(u/255) conversion (the
        two-FMA form in fv_common.cuh:unit2) through every path: 2:1, 1:2,
        generic ratios, gather; u8 HWC and the fused CHW mode."""
        sw, sh, dw, dh = geom
        a = (np.arange(sh * sw * 3) * 7 % 256).astype(np.uint8).reshape(sh, sw, 3)
        assert len(np.unique(a)) == 256
        with forced_path("resize", path):
            dst = torch.zeros((dh, dw, 3), dtype=torch.uint8, device=DEV)
            fv.resize_bilinear_u8(cu(a), dst)
            dc = torch.zeros((3, dh, dw), dtype=torch.float32, device=DEV)
            fv.resize_normalize_chw(cu(a), dc, synth.MEAN, synth.STD)
            out, outc = host(dst), host(dc)
        assert_exact(out, O.resize_u8(a, dw, dh))
        assert_exact(outc, O.resize_normalize_chw(a, dw, dh, synth.MEAN, synth.STD))

    @pytest.mark.parametrize("dw", [224, 300, 512, 640, 1000, 1280, 1920, 2048])
    @pytest.mark.parametrize("ratio", [4.8, 1.5, 2 / 3])
    def test_strip_tile_widths(self, rng, dw, ratio):
        """The strip kernel's consumer-warp count follows the destination
        width (the tuned default, or a narrower / wider tile when that idles
        >= 10% fewer lanes): both variants, u8 HWC and the fused CHW mode."""
        sw, sh, dh = max(1, round(dw * ratio)), 11, 7
        a = rng.integers(0, 256, (sh, sw, 3), dtype=np.uint8)
        with forced_path("resize", 2):
            dst = torch.zeros((dh, dw, 3), dtype=torch.uint8, device=DEV)
            fv.resize_bilinear_u8(cu(a), dst)
            dc = torch.zeros((3, dh, dw), dtype=torch.float32, device=DEV)
            fv.resize_normalize_chw(cu(a), dc, synth.MEAN, synth.STD)
            out, outc = host(dst), host(dc)
        assert_exact(out, O.resize_u8(a, dw, dh))
        assert_exact(outc, O.resize_normalize_chw(a, dw, dh, synth.MEAN, synth.STD))

    def test_cfg1_downscale_full_image(self):
        a = synth.seeded_u8_image(3840, 2160, 3, seed=synth.SEED_RESIZE)
        dst = torch.zeros((1080, 1920, 3), dtype=torch.uint8, device=DEV)
        fv.resize_bilinear_u8(cu(a), dst)
        assert_exact(host(dst), O.resize_u8(a, 1920, 1080))

    def test_cfg1_upscale_row_bands(self):
        a = synth.seeded_u8_image(3840, 2160, 3, seed=synth.SEED_RESIZE + 1)
        dst = torch.zeros((2, 4320, 7680, 3), dtype=torch.uint8, device=DEV)
        src = cu(np.stack([a, a]))
        fv.resize_bilinear_u8(src, dst)
        out = host(dst)
        for lo, hi in [(0, 40), (2150, 2190), (4290, 4320)]:
            ref = O.resize_u8(a, 7680, 4320, rows=(lo, hi))
            assert_exact(out[0, lo:hi], ref)
            assert_exact(out[1, lo:hi], ref)


# ---------------------------------------------------------------------------
# a10 fused
# ---------------------------------------------------------------------------

def _fused_ref(i):
    a = synth.seeded_u8_image(1920, 1080, 3, seed=synth.SEED_FUSED + i)
    return O.resize_normalize_chw(a, 640, 640, synth.MEAN, synth.STD)


def _affine_ref(i):
    a = synth.seeded_f32_image(1920, 1080, 3, seed=synth.SEED_AFFINE + i)
    m = synth.affine_forward(synth.SEED_AFFINE_PARAMS + i, 1920, 1080)
    return O.warp_affine(a, O.invert_affine(m), 1080, 1920, border=0.0)


def _affine_src_ref(i, u8, c, border):
    """Full 1080p frames for the source-tiled affine kernel's other
    instantiations: u8 (80-px tiles) and C = 4 f32, a non-zero border."""
    a = (synth.seeded_u8_image(1920, 1080, c, seed=synth.SEED_AFFINE + 100 + i) if u8
         else synth.seeded_f32_image(1920, 1080, c, seed=synth.SEED_AFFINE + 100 + i))
    m = synth.affine_forward(synth.SEED_AFFINE_PARAMS + 100 + i, 1920, 1080)
    return a, m, O.warp_affine(a, O.invert_affine(m), 1080, 1920, border=border)


def _persp_exact_ref(i):
    a = synth.seeded_u8_image(3840, 2160, 3, seed=synth.SEED_PERSP + i)
    return O.warp_perspective(a, O.invert_homography(synth.perspective_forward(synth.SEED_PERSP_PARAMS + i)),
                              2160, 3840, border=0)

class TestFused:
    def test_cfg4_full_images(self, resize_path):
        imgs = np.stack([synth.seeded_u8_image(1920, 1080, 3, seed=synth.SEED_FUSED + i) for i in range(3)])
        dst = torch.zeros((3, 3, 640, 640), dtype=torch.float32, device=DEV)
        fv.resize_normalize_chw(cu(imgs), dst, synth.MEAN, synth.STD)
        out = host(dst)
        for i in range(3):
            assert_exact(out[i], O.resize_normalize_chw(imgs[i], 640, 640, synth.MEAN, synth.STD))

    def test_cfg4_64_images_across_the_batch(self):
        """64 of cfg4's 512 images (every 8th seed) at full size through the
        default path in one launch, against the oracle (bit-exact)."""
        idx = list(range(0, 512, 8))
        imgs = np.stack([synth.seeded_u8_image(1920, 1080, 3, seed=synth.SEED_FUSED + i) for i in idx])
        dst = torch.zeros((len(idx), 3, 640, 640), dtype=torch.float32, device=DEV)
        fv.resize_normalize_chw(cu(imgs), dst, synth.MEAN, synth.STD)
        out = host(dst)
        for k, ref in enumerate(oracle_map(_fused_ref, [(i,) for i in idx])):
            assert_exact(out[k], ref)

    def test_golden_geometry_and_odd_shapes(self, resize_path, rng):
        g = golden("resize_u8.npz")
        lut = O.normalize_lut(synth.MEAN, synth.STD)
        a, d = g["c2_src"], g["c2_dst"]  # 96x54 -> 32x32: cfg4's x3 / x1.6875 ratios
        dst = torch.zeros((3, 32, 32), dtype=torch.float32, device=DEV)
        fv.resize_normalize_chw(cu(a), dst, synth.MEAN, synth.STD)
        assert_exact(host(dst), np.stack([lut[c][d[:, :, c]] for c in range(3)]))
        for (sw, sh, dw, dh, c) in [(77, 41, 13, 29, 3), (64, 64, 64, 64, 1), (10, 10, 30, 5, 4)]:
            a = rng.integers(0, 256, (sh, sw, c), dtype=np.uint8)
            mean, std = [0.5] * c, [0.25] * c
            dst = torch.zeros((c, dh, dw), dtype=torch.float32, device=DEV)
            fv.resize_normalize_chw(cu(a), dst, mean, std)
            assert_exact(host(dst), O.resize_normalize_chw(a, dw, dh, mean, std))


# ---------------------------------------------------------------------------
# a8 / a9 warps
# ---------------------------------------------------------------------------

@pytest.fixture(params=[0, 4, 1, 2], ids=["auto_src_tile", "tma_tile", "direct", "bulk_tile"])
def warp_path(request):
    with forced_path("warp", request.param):
        yield request.param


class TestWarp:
    def test_cfg2_affine_full_images(self, warp_path):
        n = 2
        imgs = np.stack([synth.seeded_f32_image(1920, 1080, 3, seed=synth.SEED_AFFINE + i) for i in range(n)])
        ms = np.stack([synth.affine_forward(synth.SEED_AFFINE_PARAMS + i, 1920, 1080) for i in range(n)])
        dst = torch.zeros_like(cu(imgs))
        fv.warp_affine(cu(imgs), dst, ms, border=0.0)
        out = host(dst)
        for i in range(n):
            assert_exact(out[i], O.warp_affine(imgs[i], O.invert_affine(ms[i]), 1080, 1920, border=0.0))

    def test_cfg2_affine_all_32_images(self):
        """All 32 cfg2 images (their seeded rotations / scales / shifts) at
        full size through the default path in one launch (bit-exact)."""
        n = 32
        imgs = np.stack([synth.seeded_f32_image(1920, 1080, 3, seed=synth.SEED_AFFINE + i) for i in range(n)])
        ms = np.stack([synth.affine_forward(synth.SEED_AFFINE_PARAMS + i, 1920, 1080) for i in range(n)])
        dst = torch.zeros_like(cu(imgs))
        fv.warp_affine(cu(imgs), dst, ms, border=0.0)
        out = host(dst)
        for i, ref in enumerate(oracle_map(_affine_ref, [(i,) for i in range(n)])):
            assert_exact(out[i], ref)

    @pytest.mark.parametrize("u8,c", [(True, 3), (True, 1), (False, 4), (True, 4)])
    def test_affine_source_tiles_full_frames(self, u8, c):
        """The source-tiled kernel's other tile geometries on full 1080p
        frames (two images with their own cfg2-style maps in one launch, a
        non-zero border so the outside pass blends border taps), bit-exact."""
        border = 37 if u8 else 0.3
        refs = oracle_map(_affine_src_ref, [(i, u8, c, border) for i in range(2)])
        src = cu(np.stack([r[0] for r in refs]))
        dst = torch.zeros_like(src)
        fv.warp_affine(src, dst, np.stack([r[1] for r in refs]), border=border)
        out = host(dst)
        for i, r in enumerate(refs):
            assert_exact(out[i], r[2])

    def test_cfg3_perspective_exact_all_16_images(self):
        """exact=True on all 16 cfg3 images, full frames (bit-exact)."""
        n = 16
        imgs = np.stack([synth.seeded_u8_image(3840, 2160, 3, seed=synth.SEED_PERSP + i) for i in range(n)])
        hs = np.stack([synth.perspective_forward(synth.SEED_PERSP_PARAMS + i) for i in range(n)])
        dst = torch.zeros_like(cu(imgs))
        fv.warp_perspective(cu(imgs), dst, hs, border=0, exact=True)
        out = host(dst)
        for i, ref in enumerate(oracle_map(_persp_exact_ref, [(i,) for i in range(n)])):
            assert_exact(out[i], ref)

    def test_cfg3_perspective_row_bands(self):
        n = 2
        imgs = np.stack([synth.seeded_u8_image(3840, 2160, 3, seed=synth.SEED_PERSP + i) for i in range(n)])
        hs = np.stack([synth.perspective_forward(synth.SEED_PERSP_PARAMS + i) for i in range(n)])
        dst = torch.zeros_like(cu(imgs))
        fv.warp_perspective(cu(imgs), dst, hs, border=0, exact=True)
        out = host(dst)
        for i in range(n):
            hinv = O.invert_homography(hs[i])
            for lo, hi in [(0, 24), (1070, 1094), (2136, 2160)]:
                assert_exact(out[i, lo:hi], O.warp_perspective(imgs[i], hinv, 2160, 3840, border=0, rows=(lo, hi)))

    def test_cfg3_perspective_fast_full_batch(self):
        """The default u8 perspective path (fv_warp_perspective_u8_fast) on
        all 16 cfg3 images, full frames: |out - oracle| <= 1 LSB everywhere
        (north-star gate for u8 float interpolation); the 1-LSB differences
        are rare (the f32 correction keeps the map within ~1e-5 px)."""
        n = 16
        imgs = np.stack([synth.seeded_u8_image(3840, 2160, 3, seed=synth.SEED_PERSP + i) for i in range(n)])
        hs = np.stack([synth.perspective_forward(synth.SEED_PERSP_PARAMS + i) for i in range(n)])
        dst = torch.zeros_like(cu(imgs))
        fv.warp_perspective(cu(imgs), dst, hs, border=0)
        out = host(dst)
        diff_px = 0
        for i in range(n):
            ref = O.warp_perspective(imgs[i], O.invert_homography(hs[i]), 2160, 3840, border=0)
            d = np.abs(out[i].astype(np.int16) - ref.astype(np.int16))
            assert d.max() <= 1, f"image {i}: max |diff| {d.max()}"
            diff_px += int(np.count_nonzero(d))
        frac = diff_px / out.size
        print(f"cfg3 fast path: {diff_px} of {out.size} u8 values differ by 1 LSB ({frac:.2e})")
        assert frac < 1e-3

    @pytest.mark.parametrize("c", [1, 3, 4])
    def test_perspective_fast_path_cases(self, rng, c):
        """The <= 1 LSB u8 perspective kernel beyond cfg3: strong homographies
        whose W changes sign inside the frame (the f64 per-pixel fallback),
        zoom-in / zoom-out, non-zero borders, ragged widths (tail groups),
        a batch with per-image matrices, and a crop view (offset rows)."""
        h, w = 150, 301
        a = rng.integers(0, 256, (3, h, w + 8, c), dtype=np.uint8)
        mats = [
            np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.004, 0.003, 1.0]]),     # W crosses 0 in the frame
            np.array([[0.45, 0.02, 10.0], [-0.03, 0.5, 5.0], [1e-4, -2e-4, 1.0]]),  # zoom in
            np.array([[2.6, 0.3, -40.0], [-0.2, 2.4, -20.0], [2e-3, 1e-3, 1.0]]),   # zoom out, strong tilt
            np.array([[1.0, 0.1, 3.0], [-0.1, 1.0, 2.0], [-3e-3, 2e-3, 1.0]]),
        ]
        for hinv in mats:
            for oh, ow, border, crop in [(h, w, 0, False), (97, 255, 17, False), (h, w, 255, True)]:
                view = a[:, :, 5:w + 5] if crop else np.ascontiguousarray(a[:, :, :w])
                src = cu(a)[:, :, 5:w + 5] if crop else cu(view)
                dst = torch.zeros((3, oh, ow, c), dtype=torch.uint8, device=DEV)
                fv.warp_perspective(src, dst, np.stack([hinv, hinv @ np.diag([1.0, 1.0, 1.0]), hinv]), border=border,
                                    inverse=True)
                got = host(dst)
                for i in range(3):
                    ref = O.warp_perspective(np.ascontiguousarray(view[i]), hinv, oh, ow, border=border)
                    assert_within_gate(got[i], ref)

    @pytest.mark.parametrize("dtype", [np.uint8, np.float32])
    def test_small_shapes_with_border(self, rng, dtype, warp_path):
        for (h, w, oh, ow, c) in [(14, 17, 12, 19, 3), (5, 5, 9, 9, 1), (33, 20, 20, 33, 4)]:
            a = rng.integers(0, 256, (h, w, c), dtype=np.uint8) if dtype == np.uint8 else rng.random((h, w, c), dtype=np.float32)
            m = O.affine_forward(7 + h, w, h)
            hm = np.eye(3) + rng.normal(0, 0.02, (3, 3))
            hm[2, 2] = 1.0
            for persp, mat in [(False, m), (True, hm)]:
                dst = torch.zeros((oh, ow, c), dtype=torch.from_numpy(a).dtype, device=DEV)
                if persp:
                    fv.warp_perspective(cu(a), dst, mat, border=7, exact=True)
                else:
                    fv.warp_affine(cu(a), dst, mat, border=7)
                inv = O.invert_homography(mat) if persp else O.invert_affine(mat)
                ref = (O.warp_perspective if persp else O.warp_affine)(a, inv, oh, ow, border=7)
                assert_exact(host(dst), ref)
                if persp:  # the default path: exact for f32, within 1 LSB for u8
                    fv.warp_perspective(cu(a), dst, mat, border=7)
                    assert_within_gate(host(dst), ref)

    @pytest.mark.parametrize("dtype", [np.uint8, np.float32])
    @pytest.mark.parametrize("c", [1, 3, 4])
    def test_affine_tile_kernel_cases(self, rng, dtype, c, warp_path):
        """The SMEM-staged affine kernel against the oracle: 16-byte aligned
        rows (staged), a zoom-out whose tile boxes exceed the staging budget
        (direct gathers inside the same kernel), a map that sends whole tiles
        outside the source (empty boxes), ragged tile edges, a batch, and a
        crop view whose rows are not 16-byte aligned (direct kernel)."""
        h, w = 70, 160  # 160 px: rows 16-byte aligned for every dtype / c
        a = rng.integers(0, 256, (3, h, w + 16, c), dtype=np.uint8)
        if dtype == np.float32:
            a = (a / np.float32(255)).astype(np.float32)
        base = [
            O.affine_forward(5, w, h),                                   # rotation / scale / shift
            np.array([[0.3, 0.05, 2.0], [-0.04, 0.35, 1.0]]),            # 3x zoom-out: boxes too big
            np.array([[1.0, 0.0, 500.0], [0.0, 1.0, -300.0]]),           # everything outside
            np.array([[0.9, 0.45, -20.0], [-0.45, 0.9, 30.0]]),          # 27 deg rotation
        ]
        for m in base:
            for oh, ow in [(h, w), (45, 77)]:
                for crop, border in [(False, 0), (True, 9)]:
                    b = border if dtype == np.uint8 else border / 255.0
                    view = a[:, :, 3:w + 3] if crop else np.ascontiguousarray(a[:, :, :w])
                    src = cu(a)[:, :, 3:w + 3] if crop else cu(view)
                    dst = torch.zeros((3, oh, ow, c), dtype=src.dtype, device=DEV)
                    fv.warp_affine(src, dst, np.stack([m] * 3), border=b)
                    got = host(dst)
                    inv = O.invert_affine(m)
                    for i in range(3):
                        assert_exact(got[i], O.warp_affine(np.ascontiguousarray(view[i]), inv, oh, ow, border=b))

    @pytest.mark.parametrize("dtype", [np.uint8, np.float32])
    def test_affine_source_tiles_degenerate_axes(self, rng, dtype, warp_path):
        """Maps whose inverse has zero entries (m0 = 0: a 90-degree turn, so a
        destination row runs along a source column; m3 = m1 = 0: a pure
        shift / scale), exact half-pixel shifts that put taps on tile
        boundaries, mirror images, and a shift that moves the source partly
        off the destination: every pixel is owned by one source tile or the
        outside pass, bit-exact."""
        h, w, c = 75, 96, 3
        a = rng.integers(0, 256, (h, w, c), dtype=np.uint8)
        if dtype == np.float32:
            a = (a / np.float32(255)).astype(np.float32)
        invs = [
            np.array([[0.0, 1.0, 0.0], [-1.0, 0.0, h - 1.0]]),           # 90-degree turn
            np.array([[0.0, -1.25, 80.0], [1.25, 0.0, -7.0]]),           # turn + zoom-out 1.25
            np.array([[1.0, 0.0, 0.5], [0.0, 1.0, -0.5]]),               # half-pixel shift
            np.array([[1.0, 0.0, 32.0], [0.0, 1.0, 24.0]]),              # shift by one source tile
            np.array([[-1.0, 0.0, w - 1.0], [0.0, 1.0, 0.0]]),           # mirror
            np.array([[0.5, 0.0, -10.0], [0.0, 0.5, 40.0]]),             # 2x zoom-in, partly outside
            np.array([[1.0, 1e-17, 3.0], [0.0, 1.0, 2.0]]),              # near-degenerate m1
        ]
        for inv in invs:
            for oh, ow, b in [(h, w, 0), (100, 130, 5)]:
                bb = b if dtype == np.uint8 else b / 255.0
                dst = torch.zeros((oh, ow, c), dtype=torch.from_numpy(a).dtype, device=DEV)
                fv.warp_affine(cu(a), dst, inv, border=bb, inverse=True)
                assert_exact(host(dst), O.warp_affine(a, inv, oh, ow, border=bb))

    def test_identity_and_zero_w(self, rng):
        a = rng.integers(0, 256, (10, 12, 3), dtype=np.uint8)
        dst = torch.zeros((10, 12, 3), dtype=torch.uint8, device=DEV)
        fv.warp_perspective(cu(a), dst, np.eye(3))
        assert_exact(host(dst), a)
        img = np.full((4, 4, 1), 200, np.uint8)
        hinv = np.array([[1.0, 0, 0], [0, 1.0, 0], [1.0, 0, -2.0]])
        dst = torch.zeros((4, 4, 1), dtype=torch.uint8, device=DEV)
        fv.warp_perspective(cu(img), dst, hinv, border=9, inverse=True, exact=True)
        assert_exact(host(dst), O.warp_perspective(img, hinv, 4, 4, border=9))
        assert host(dst)[0, 2, 0] == 9
        fv.warp_perspective(cu(img), dst, hinv, border=9, inverse=True)
        assert_within_gate(host(dst), O.warp_perspective(img, hinv, 4, 4, border=9))
        assert host(dst)[0, 2, 0] == 9


# ---------------------------------------------------------------------------
# discipline: determinism, zero allocation, native path really used
# ---------------------------------------------------------------------------

def test_deterministic_reruns_bit_identical(rng):
    a = cu(rng.integers(0, 256, (2, 216, 384, 3), dtype=np.uint8))
    d1 = torch.zeros((2, 432, 768, 3), dtype=torch.uint8, device=DEV)
    d2 = torch.zeros_like(d1)
    fv.resize_bilinear_u8(a, d1)
    fv.resize_bilinear_u8(a, d2)
    assert torch.equal(d1, d2)


def test_kernels_do_not_allocate(rng):
    rgb = cu(rng.integers(0, 256, (2, 64, 96, 3), dtype=np.uint8))
    gray = torch.zeros((2, 64, 96, 1), dtype=torch.uint8, device=DEV)
    up = torch.zeros((2, 128, 192, 3), dtype=torch.uint8, device=DEV)
    chw = torch.zeros((2, 3, 32, 32), dtype=torch.float32, device=DEV)
    f = torch.rand((2, 64, 96, 3), device=DEV)
    fw = torch.zeros_like(f)
    m = synth.affine_forward(1, 96, 64)
    fv.resize_normalize_chw(rgb, chw, synth.MEAN, synth.STD)  # warm the LUT cache
    torch.cuda.synchronize()
    before = torch.cuda.memory_stats(DEV)["allocation.all.allocated"]
    for _ in range(50):
        fv.gray_from_rgb(rgb, gray)
        fv.resize_bilinear_u8(rgb, up)
        fv.resize_normalize_chw(rgb, chw, synth.MEAN, synth.STD)
        fv.warp_affine(f, fw, m)
        fv.warp_perspective(rgb, up[:, :64, :96], np.eye(3))
    torch.cuda.synchronize()
    assert torch.cuda.memory_stats(DEV)["allocation.all.allocated"] == before


def test_native_kernels_launch():
    before = _native.launch_count()
    a = torch.zeros((8, 8, 3), dtype=torch.uint8, device=DEV)
    d = torch.zeros((8, 8, 1), dtype=torch.uint8, device=DEV)
    fv.gray_from_rgb(a, d)
    torch.cuda.synchronize()
    assert _native.launch_count() == before + 1


# ---------------------------------------------------------------------------
# property test: random geometry through every resize path
# ---------------------------------------------------------------------------
from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@given(sw=st.integers(1, 70), sh=st.integers(1, 40), dw=st.integers(1, 90), dh=st.integers(1, 50),
       c=st.sampled_from([1, 2, 3, 4, 5]), n=st.integers(1, 2), path=st.sampled_from([0, 1, 2]),
       seed=st.integers(0, 2**31 - 1))
@settings(max_examples=120, deadline=None)
def test_resize_random_geometry_all_paths(sw, sh, dw, dh, c, n, path, seed):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 256, (n, sh, sw, c), dtype=np.uint8)
    f = rng.random((n, sh, sw, c), dtype=np.float32)
    with forced_path("resize", path):
        du = torch.zeros((n, dh, dw, c), dtype=torch.uint8, device=DEV)
        df = torch.zeros((n, dh, dw, c), dtype=torch.float32, device=DEV)
        fv.resize_bilinear_u8(cu(a), du)
        fv.resize_bilinear(cu(f), df)
        ou, of = host(du), host(df)
    for i in range(n):
        assert np.array_equal(ou[i], O.resize_u8(a[i], dw, dh))
        assert np.array_equal(of[i], O.resize_bilinear(f[i], dw, dh))
    if c <= 4:
        mean, std = [0.3] * c, [0.2] * c
        dc = torch.zeros((n, c, dh, dw), dtype=torch.float32, device=DEV)
        fv.resize_normalize_chw(cu(a), dc, mean, std)
        oc = host(dc)
        for i in range(n):
            assert np.array_equal(oc[i], O.resize_normalize_chw(a[i], dw, dh, mean, std))


@given(h=st.integers(1, 30), w=st.integers(1, 40), oh=st.integers(1, 30), ow=st.integers(1, 40),
       c=st.sampled_from([1, 2, 3, 4]), u8=st.booleans(), persp=st.booleans(), border=st.integers(0, 255),
       seed=st.integers(0, 2**31 - 1))
@settings(max_examples=80, deadline=None)
def test_warp_random_geometry(h, w, oh, ow, c, u8, persp, border, seed):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 256, (h, w, c), dtype=np.uint8) if u8 else rng.random((h, w, c), dtype=np.float32)
    if persp:
        mat = np.eye(3) + rng.normal(0, 0.05, (3, 3))
        mat[2, 2] = 1.0
        inv = O.invert_homography(mat)
    else:
        mat = np.hstack([rng.normal(0, 1.0, (2, 2)) + np.eye(2), rng.normal(0, 5.0, (2, 1))])
        inv = O.invert_affine(mat)
    b = border if u8 else border / 255.0
    dst = torch.zeros((oh, ow, c), dtype=torch.from_numpy(a).dtype, device=DEV)
    if persp:
        fv.warp_perspective(cu(a), dst, inv, border=b, inverse=True, exact=True)
    else:
        fv.warp_affine(cu(a), dst, inv, border=b, inverse=True)
    ref = (O.warp_perspective if persp else O.warp_affine)(a, inv, oh, ow, border=b)
    assert_exact(host(dst), ref)
    if persp:
        fv.warp_perspective(cu(a), dst, inv, border=b, inverse=True)
        assert_within_gate(host(dst), ref)


@given(h=st.integers(1, 80), w16=st.integers(1, 6), oh=st.integers(1, 80), ow=st.integers(1, 100),
       c=st.sampled_from([1, 3, 4]), u8=st.booleans(), scale=st.floats(0.2, 3.0), angle=st.floats(-3.2, 3.2),
       border=st.integers(0, 255), seed=st.integers(0, 2**31 - 1))
@settings(max_examples=60, deadline=None)
def test_affine_tile_random_geometry(h, w16, oh, ow, c, u8, scale, angle, border, seed):
    """Random affine maps on 16-byte aligned rows (the staged tile kernel),
    any rotation, zoom in and out, bit-exact against the oracle."""
    rng = np.random.default_rng(seed)
    w = 16 * w16
    a = rng.integers(0, 256, (h, w, c), dtype=np.uint8) if u8 else rng.random((h, w, c), dtype=np.float32)
    ca, sa = np.cos(angle) * scale, np.sin(angle) * scale
    inv = np.array([[ca, -sa, rng.normal(0, 20)], [sa, ca, rng.normal(0, 20)]])
    b = border if u8 else border / 255.0
    dst = torch.zeros((oh, ow, c), dtype=torch.from_numpy(a).dtype, device=DEV)
    fv.warp_affine(cu(a), dst, inv, border=b, inverse=True)
    assert_exact(host(dst), O.warp_affine(a, inv, oh, ow, border=b))


def test_cfg1_full_batch_properties():
    """Size-independent properties at the full BASELINE configs[1] size (64
    4K images, both kernels): a constant image resizes to the same constant
    (exact at u8 level), and reruns are bit-identical."""
    n = 64
    vals = torch.tensor([(37 * i + 11) % 256 for i in range(n)], dtype=torch.uint8, device=DEV)
    src = vals.view(n, 1, 1, 1).expand(n, 2160, 3840, 3).contiguous()
    down = torch.zeros((n, 1080, 1920, 3), dtype=torch.uint8, device=DEV)
    up = torch.zeros((n, 4320, 7680, 3), dtype=torch.uint8, device=DEV)
    fv.resize_bilinear_u8(src, down)
    fv.resize_bilinear_u8(src, up)
    torch.cuda.synchronize()
    for out in (down, up):
        assert torch.equal(out.amin(dim=(1, 2, 3)), vals) and torch.equal(out.amax(dim=(1, 2, 3)), vals)
    # random content: two runs bit-identical (checksum over the whole batch)
    g = torch.Generator(device=DEV)
    g.manual_seed(7)
    src = torch.randint(0, 256, (n, 2160, 3840, 3), dtype=torch.uint8, device=DEV, generator=g)
    fv.resize_bilinear_u8(src, up)
    c1 = up.view(-1).to(torch.int64).sum().item()
    up2 = torch.empty_like(up)
    fv.resize_bilinear_u8(src, up2)
    assert torch.equal(up, up2) and c1 == up2.view(-1).to(torch.int64).sum().item()


def test_cfg1_upscale_full_image_exact():
    """One full 3840x2160 -> 7680x4320 image against the oracle (every row)."""
    a = synth.seeded_u8_image(3840, 2160, 3, seed=synth.SEED_RESIZE + 5)
    dst = torch.zeros((4320, 7680, 3), dtype=torch.uint8, device=DEV)
    fv.resize_bilinear_u8(cu(a), dst)
    assert_exact(host(dst), O.resize_u8(a, 7680, 4320))
