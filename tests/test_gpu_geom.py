"""GPU parity of SURVEY §8(f) kernels (flip, nearest, sobel) and an
out-of-bounds-write guard for every op: destinations are views inside a
canary-filled parent buffer, and nothing outside the view may change."""
import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle as O
import paper_2505_12425_b200 as fv
from _helpers import forced_path, golden
from paper_2505_12425_b200 import _native, synth

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


class TestGeom:
    def test_flip_golden_and_involution(self, rng):
        g = golden("geom.npz")
        for i in range(4):
            a, d = g[f"flip{i}_src"], g[f"flip{i}_dst"]
            dst = torch.zeros(d.shape, dtype=cu(a).dtype, device=DEV)
            fv.flip_horizontal(cu(a), dst)
            assert np.array_equal(host(dst), d)
        a = cu(rng.integers(0, 256, (3, 13, 7, 3), dtype=np.uint8))
        once, twice = torch.zeros_like(a), torch.zeros_like(a)
        fv.flip_horizontal(a, once)
        fv.flip_horizontal(once, twice)
        assert torch.equal(twice, a)

    def test_nearest_golden(self):
        g = golden("geom.npz")
        for i in range(6):
            a, d = g[f"near{i}_src"], g[f"near{i}_dst"]
            dst = torch.zeros(d.shape, dtype=cu(a).dtype, device=DEV)
            fv.resize_nearest(cu(a), dst)
            assert np.array_equal(host(dst), d)

    @given(k=st.integers(2, 5), w=st.integers(1, 9), h=st.integers(1, 9))
    @settings(max_examples=30, deadline=None)
    def test_nearest_integer_upscale_repeats_each_pixel(self, k, w, h):
        """pkg/tests/test_imgproc.py:107-115 as a GPU property."""
        a = np.random.default_rng(99).integers(0, 256, (h, w, 1), dtype=np.uint8)
        dst = torch.zeros((h * k, w * k, 1), dtype=torch.uint8, device=DEV)
        fv.resize_nearest(cu(a), dst)
        assert np.array_equal(host(dst), np.repeat(np.repeat(a, k, axis=0), k, axis=1))

    def test_nearest_config_size(self):
        a = synth.seeded_u8_image(3840, 2160, 3, seed=13)
        dst = torch.zeros((1080, 1920, 3), dtype=torch.uint8, device=DEV)
        fv.resize_nearest(cu(a), dst)
        assert np.array_equal(host(dst), O.resize_nearest(a, 1920, 1080))

    def test_sobel_golden_and_properties(self, rng):
        g = golden("geom.npz")
        for i in range(4):
            a, d = g[f"sobel{i}_src"], g[f"sobel{i}_dst"]
            dst = torch.zeros(d.shape, dtype=torch.float32, device=DEV)
            fv.sobel(cu(a), dst, 3)
            assert np.array_equal(host(dst), d)
        base = rng.random((2, 64, 80, 3), dtype=np.float32)
        d1 = torch.zeros(base.shape, dtype=torch.float32, device=DEV)
        fv.sobel(cu(base), d1, 3)
        out = host(d1)
        for i in range(2):
            assert np.array_equal(out[i], O.sobel(base[i]))
        with pytest.raises(fv.UnsupportedKernelSize):
            fv.sobel(cu(base[0]), d1[0], 5)


# ---------------------------------------------------------------------------
# out-of-bounds write guard
# ---------------------------------------------------------------------------

CANARY = 0xA5


def guarded(shape, dtype, pad=(3, 5, 7)):
    """A destination view strictly inside a canary-filled parent."""
    n, h, w, c = shape
    ph, pw = h + 2 * pad[0], w + 2 * pad[1]
    parent = torch.full((n + 2, ph, pw, c), 0, dtype=dtype, device=DEV)
    parent.view(torch.uint8).fill_(CANARY)
    view = parent[1:1 + n, pad[0]:pad[0] + h, pad[1]:pad[1] + w]
    return parent, view


def check_canaries(parent, shape, pad=(3, 5, 7)):
    n, h, w, c = shape
    es = parent.element_size()
    p = host(parent.view(torch.uint8)).reshape(parent.shape[0], parent.shape[1], -1)
    mask = np.ones(p.shape, bool)
    mask[1:1 + n, pad[0]:pad[0] + h, pad[1] * c * es:(pad[1] + w) * c * es] = False
    assert np.all(p[mask] == CANARY), "write outside the destination view"


@pytest.mark.parametrize("path", [0, 1, 2])
def test_no_writes_outside_destination(rng, path):
    with forced_path("resize", path):
        n, c = 2, 3
        src = cu(rng.integers(0, 256, (n, 37, 53, c), dtype=np.uint8))
        srcf = cu(rng.random((n, 37, 53, c), dtype=np.float32))
        cases = [
            ("resize_u8", (n, 23, 71, c), torch.uint8, lambda d: fv.resize_bilinear_u8(src, d)),
            ("resize_u8_up2", (n, 74, 106, c), torch.uint8, lambda d: fv.resize_bilinear_u8(src[:, :36, :52], d)),
            ("resize_f32", (n, 29, 17, c), torch.float32, lambda d: fv.resize_bilinear(srcf, d)),
            ("gray", (n, 37, 53, 1), torch.uint8, lambda d: fv.gray_from_rgb(src, d)),
            ("affine", (n, 40, 50, c), torch.float32, lambda d: fv.warp_affine(srcf, d, synth.affine_forward(3, 53, 37))),
            ("persp", (n, 40, 50, c), torch.uint8, lambda d: fv.warp_perspective(src, d, synth.perspective_forward(4))),
            ("persp_exact", (n, 40, 50, c), torch.uint8,
             lambda d: fv.warp_perspective(src, d, synth.perspective_forward(4), exact=True)),
            ("nearest", (n, 19, 90, c), torch.uint8, lambda d: fv.resize_nearest(src, d)),
            ("flip", (n, 37, 53, c), torch.uint8, lambda d: fv.flip_horizontal(src, d)),
        ]
        for name, shape, dt, call in cases:
            parent, view = guarded(shape, dt)
            call(view)
            check_canaries(parent, shape)
        # fused: planar destination inside a padded planar parent
        parent = torch.zeros((n + 2, c, 40, 48), dtype=torch.float32, device=DEV)
        parent.view(torch.uint8).fill_(CANARY)
        view = parent[1:1 + n, :, 3:35, 5:37]
        fv.resize_normalize_chw(src, view, synth.MEAN, synth.STD)
        p = host(parent.view(torch.uint8)).reshape(n + 2, c, 40, 48, 4)
        mask = np.ones(p.shape, bool)
        mask[1:1 + n, :, 3:35, 5:37] = False
        assert np.all(p[mask] == CANARY)


def test_empty_batch_is_a_no_op():
    src = torch.zeros((0, 8, 8, 3), dtype=torch.uint8, device=DEV)
    dst = torch.zeros((0, 16, 16, 3), dtype=torch.uint8, device=DEV)
    fv.resize_bilinear_u8(src, dst)
    fv.flip_horizontal(src, torch.zeros_like(src))
    torch.cuda.synchronize()


@pytest.mark.parametrize("dtype,c", [(np.uint8, 1), (np.uint8, 3), (np.uint8, 4), (np.float32, 3), (np.float32, 1),
                                     (np.uint16, 3)])
def test_flip_and_nearest_vector_paths(rng, dtype, c):
    """16-pixel vectorised kernels (width % 16 == 0) and the generic ones
    (ragged widths), batched, vs the oracle."""
    for (h, w, dh, dw) in [(9, 64, 18, 128), (5, 48, 7, 32), (6, 37, 11, 21)]:
        a = (rng.integers(0, 60000, (2, h, w, c)).astype(dtype) if dtype != np.float32
             else rng.random((2, h, w, c), dtype=np.float32))
        t = cu(a)
        f = torch.zeros_like(t)
        fv.flip_horizontal(t, f)
        nn = torch.zeros((2, dh, dw, c), dtype=t.dtype, device=DEV)
        fv.resize_nearest(t, nn)
        fo, no = host(f), host(nn)
        for i in range(2):
            assert np.array_equal(fo[i], O.flip_horizontal(a[i]))
            assert np.array_equal(no[i], O.resize_nearest(a[i], dw, dh))
