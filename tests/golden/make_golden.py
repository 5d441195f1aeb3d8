"""Generate golden vectors by running the UNMODIFIED reference (`fovea`) here.

Run once in the build container, where the read-only reference is mounted:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `fovea` from /root/reference/pkg/src and calls the reference's own
functions — imgproc.gray_from_rgb (imgproc.py:43), imgproc.resize_bilinear
(imgproc.py:100), imgproc.flip_horizontal / resize_nearest / sobel (imgproc.py:67-155), image.to_float_scaled (image.py:150), Tensor.cast
(tensor.py:265) and service.app._resize_u8 (app.py:64) — on small seeded
inputs, and writes inputs + outputs to tests/golden/*.npz. The GPU box never
reads /root/reference; tests there use only these committed fixtures.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main() -> None:
    sys.path.insert(0, REF)
    from fovea import imgproc
    from fovea.image import Image, ImageSize, ImageType, to_float_scaled
    from fovea.service.app import _resize_u8
    from fovea.tensor import Tensor

    rng = np.random.default_rng(20250518)

    def ref_gray(arr):
        src = Image.from_array(arr)
        dst = ImageType(arr.dtype, 1).from_size_val(src.size, 0)
        imgproc.gray_from_rgb(src, dst)
        return dst.as_array().copy()

    # ---- gray: seeded images, KATs, and every exact-decimal tie triple -----
    g = {}
    g["u8_rand"] = rng.integers(0, 256, (48, 64, 3), dtype=np.uint8)
    g["u8_odd"] = rng.integers(0, 256, (17, 23, 3), dtype=np.uint8)
    g["u8_kat"] = np.array([[[255, 255, 255], [0, 0, 0], [255, 0, 0], [0, 255, 0], [0, 0, 255]]], np.uint8)
    r, gg, b = np.meshgrid(np.arange(256), np.arange(256), np.arange(256), indexing="ij")
    s = 299 * r + 587 * gg + 114 * b
    tie = (s % 1000) == 500
    g["u8_ties"] = np.stack([r[tie], gg[tie], b[tie]], axis=-1).astype(np.uint8)[None]
    g["f32_rand"] = rng.random((11, 19, 3), dtype=np.float32)
    out = {}
    for k, v in g.items():
        out[k + "_src"] = v
        out[k + "_dst"] = ref_gray(v)
    np.savez_compressed(os.path.join(OUT, "gray.npz"), **out)

    # ---- f32 bilinear: the reference test shapes + a 3-channel case --------
    out = {}
    cases = [(6, 4, 11, 3, 2), (9, 9, 4, 13, 2), (2, 2, 5, 5, 2), (40, 30, 17, 23, 3), (5, 7, 5, 7, 3)]
    for i, (sw, sh, dw, dh, c) in enumerate(cases):
        a = rng.random((sh, sw, c), dtype=np.float32)
        src = Image.from_array(a)
        dst = ImageType(np.float32, c).from_size_val(ImageSize(dw, dh), 0.0)
        imgproc.resize_bilinear(src, dst)
        out[f"c{i}_src"] = a
        out[f"c{i}_dst"] = dst.as_array().copy()
    np.savez_compressed(os.path.join(OUT, "resize_f32.npz"), **out)

    # ---- u8 bilinear (_resize_u8): config scale pairs at small size --------
    # 2x down and 2x up (cfg1 ratios), 3 x 1.6875 (cfg4 ratios), odd shapes.
    out = {}
    cases = [(64, 36, 32, 18, 3), (32, 18, 64, 36, 3), (96, 54, 32, 32, 3),
             (23, 17, 11, 29, 3), (7, 5, 3, 3, 1), (1, 1, 4, 4, 3), (13, 9, 13, 9, 3)]
    for i, (sw, sh, dw, dh, c) in enumerate(cases):
        a = rng.integers(0, 256, (sh, sw, c), dtype=np.uint8)
        res = _resize_u8(Image.from_array(a), ImageSize(dw, dh), "bilinear")
        out[f"c{i}_src"] = a
        out[f"c{i}_dst"] = res.as_array().copy()
    np.savez_compressed(os.path.join(OUT, "resize_u8.npz"), **out)

    # ---- flip (imgproc.py:67), nearest (:89), sobel (:126) ----
    out = {}
    for i, (h, w, c, dt) in enumerate([(7, 13, 3, np.uint8), (5, 9, 4, np.uint8), (6, 5, 2, np.float32),
                                       (3, 4, 1, np.uint16)]):
        a = (rng.integers(0, 60000, (h, w, c)).astype(dt) if dt != np.float32 else rng.random((h, w, c), dtype=dt))
        dst = ImageType(dt, c).from_size_val(ImageSize(w, h), 0)
        imgproc.flip_horizontal(Image.from_array(a), dst)
        out[f"flip{i}_src"], out[f"flip{i}_dst"] = a, dst.as_array().copy()
    for i, (sw, sh, dw, dh, c, dt) in enumerate([(7, 5, 13, 3, 3, np.uint8), (16, 16, 5, 9, 3, np.uint8),
                                                  (3, 3, 3, 3, 3, np.uint8), (1, 1, 4, 4, 3, np.uint8),
                                                  (12, 7, 25, 4, 2, np.float32), (9, 9, 6, 14, 1, np.uint16)]):
        a = (rng.integers(0, 60000, (sh, sw, c)).astype(dt) if dt != np.float32 else rng.random((sh, sw, c), dtype=dt))
        dst = ImageType(dt, c).from_size_val(ImageSize(dw, dh), 0)
        imgproc.resize_nearest(Image.from_array(a), dst)
        out[f"near{i}_src"], out[f"near{i}_dst"] = a, dst.as_array().copy()
    ramp = np.tile(np.arange(6, dtype=np.float32)[None, :, None], (5, 1, 1))
    for i, a in enumerate([rng.random((9, 12, 3), dtype=np.float32), np.full((5, 5, 1), 3.25, np.float32), ramp,
                           rng.random((8, 8, 1), dtype=np.float32)]):
        dst = ImageType(np.float32, a.shape[2]).from_size_val(ImageSize(a.shape[1], a.shape[0]), 0.0)
        imgproc.sobel(Image.from_array(a), dst, 3)
        out[f"sobel{i}_src"], out[f"sobel{i}_dst"] = a, dst.as_array().copy()
    np.savez_compressed(os.path.join(OUT, "geom.npz"), **out)

    # ---- to_float_scaled for every u8 value; cast KATs ---------------------
    u = np.arange(256, dtype=np.uint8).reshape(1, 256, 1)
    f = ImageType(np.float32, 1).from_size_val(ImageSize(256, 1), 0.0)
    to_float_scaled(Image.from_array(u), f)
    vals = np.array([1.5, 2.5, -0.5, 0.4, -3.0, 300.0, 254.5, 255.49998, 0.49999997, np.nan], np.float32)
    cast = Tensor.from_shape_slice([vals.size], vals, dtype=np.float32).cast(np.uint8).as_array().copy()
    np.savez_compressed(os.path.join(OUT, "scalars.npz"), to_float_src=u, to_float_dst=f.as_array().copy(),
                        cast_src=vals, cast_dst=cast)
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
