"""Image-processing kernels writing into caller-provided CUDA output tensors.

Drop-in mirror of the reference's `fovea.imgproc` hot path (imgproc.py) on
B200: same function names and `(src, dst[, params]) -> None` shape, same
dtypes, rounding, interpolation and border semantics, same exception classes
raised in the same check order. Every op is bit-identical to the reference's
rounding, with one documented exception: `warp_perspective` on u8 images
defaults to the north star's <= 1 LSB gate for u8 float interpolation
(9.4e-5 of the cfg3 benchmark's values differ by one); pass `exact=True`
for the bit-exact kernel. Images are torch CUDA tensors, HWC
`[H, W, C]` or batched `[N, H, W, C]`; every op runs as one hand-written
sm_100a kernel launch per batch through the C ABI (include/fovea_b200.h) on
the tensor's current CUDA stream. Nothing here allocates device memory and
there is no CPU fallback: CPU tensors raise `UnsupportedDevice`.
"""
from __future__ import annotations

import ctypes
import functools

import numpy as np
import torch

from . import _native
from ._tensors import F32, U8, as_image, as_planar, check_distinct, same_device, stream_ptr
from .errors import ShapeMismatch, SingularTransform, SizeMismatch, UnsupportedDtype, UnsupportedKernelSize

__all__ = [
    "gray_from_rgb", "resize_bilinear", "resize_bilinear_u8", "resize_normalize_chw",
    "warp_affine", "warp_perspective", "normalize_lut", "flip_horizontal", "resize_nearest", "sobel",
]


def _check_batch(s, d) -> None:
    if s.n != d.n:
        raise SizeMismatch(f"source batch {s.n} and destination batch {d.n} differ")


def gray_from_rgb(src: torch.Tensor, dst: torch.Tensor) -> None:
    """BT.601 grayscale: 0.299 R + 0.587 G + 0.114 B per pixel (imgproc.py:43-64).

    u8 rounds half away from zero, bit-exact with the reference's f64 maths;
    f32 keeps the f64 sum narrowed to f32. Checks in the reference's order:
    channels 3 -> 1 (SizeMismatch), equal dtypes (UnsupportedDtype), equal
    sizes (SizeMismatch), dtype in {u8, f32} (UnsupportedDtype). Unlike the
    reference, aliased src/dst is rejected (AliasedBuffers): a GPU kernel
    cannot run in place without a temporary.
    """
    s, d = as_image(src, "src"), as_image(dst, "dst")
    if s.c != 3 or d.c != 1:
        raise SizeMismatch(f"expected 3-channel source and 1-channel destination, got {s.c} and {d.c}")
    if s.dtype != d.dtype:
        raise UnsupportedDtype(f"source {s.dtype} and destination {d.dtype} must match")
    if s.size != d.size:
        raise SizeMismatch(f"source {s!r} and destination {d!r} differ in size")
    _check_batch(s, d)
    if s.dtype not in (U8, F32):
        raise UnsupportedDtype(f"gray_from_rgb supports u8 and f32, got {s.dtype}")
    same_device(src, dst)
    check_distinct(src, dst)
    fn = "fv_gray_from_rgb_u8" if s.dtype == U8 else "fv_gray_from_rgb_f32"
    with torch.cuda.device(src.device):
        _native.call(fn, s.ptr, s.img_stride, s.row_pitch, d.ptr, d.img_stride, d.row_pitch,
                     s.n, s.h, s.w, stream_ptr(src))


def resize_bilinear(src: torch.Tensor, dst: torch.Tensor) -> None:
    """Bilinear resize of f32 images with pixel-centre mapping and edge clamp
    (imgproc.py:100-123). The destination's size defines the target."""
    s, d = as_image(src, "src"), as_image(dst, "dst")
    if s.dtype != F32 or d.dtype != F32:
        raise UnsupportedDtype(f"resize_bilinear requires f32 images, got {s.dtype} -> {d.dtype}")
    if s.c != d.c:
        raise SizeMismatch(f"source has {s.c} channels, destination {d.c}")
    check_distinct(src, dst)
    _check_batch(s, d)
    same_device(src, dst)
    with torch.cuda.device(src.device):
        _native.call("fv_resize_bilinear_f32", s.ptr, s.img_stride, s.row_pitch, s.h, s.w,
                     d.ptr, d.img_stride, d.row_pitch, d.h, d.w, s.c, s.n, stream_ptr(src))


def resize_bilinear_u8(src: torch.Tensor, dst: torch.Tensor) -> None:
    """u8 bilinear resize with the reference's `_resize_u8` semantics
    (service/app.py:64-78; SPEC.md:751 binding_resize): to_float_scaled ->
    resize_bilinear -> x255 -> Tensor.cast(u8), bit-exact, fused into one
    kernel that writes the caller's u8 `dst` (no f32 frames in memory)."""
    s, d = as_image(src, "src"), as_image(dst, "dst")
    if s.dtype != U8 or d.dtype != U8:
        raise UnsupportedDtype(f"resize_bilinear_u8 requires u8 images, got {s.dtype} -> {d.dtype}")
    if s.c != d.c:
        raise SizeMismatch(f"source has {s.c} channels, destination {d.c}")
    check_distinct(src, dst)
    _check_batch(s, d)
    same_device(src, dst)
    with torch.cuda.device(src.device):
        _native.call("fv_resize_bilinear_u8", s.ptr, s.img_stride, s.row_pitch, s.h, s.w,
                     d.ptr, d.img_stride, d.row_pitch, d.h, d.w, s.c, s.n, stream_ptr(src))


# ---------------------------------------------------------------------------
# fused preprocessing
# ---------------------------------------------------------------------------

def normalize_lut(mean, std) -> np.ndarray:
    """(C, 256) f32 table ((f32(u) / f32(255)) - mean_c) / std_c with each op
    an IEEE f32 op: to_float_scaled (image.py:158-160) followed by the
    normalisation, tabulated on the host once per (mean, std)."""
    mean = np.asarray(mean, dtype=np.float32).reshape(-1)
    std = np.asarray(std, dtype=np.float32).reshape(-1)
    if mean.shape != std.shape:
        raise ShapeMismatch(f"mean has {mean.size} entries, std {std.size}")
    unit = np.arange(256, dtype=np.float32)
    unit /= np.float32(255.0)
    return np.ascontiguousarray(((unit[None, :] - mean[:, None]) / std[:, None]).astype(np.float32))


@functools.lru_cache(maxsize=64)
def _cached_lut(mean: tuple, std: tuple) -> np.ndarray:
    """normalize_lut per (mean, std) as f32 tuples; bounded (a service that
    normalises with per-request statistics does not grow it without limit)."""
    lut = normalize_lut(mean, std)
    lut.setflags(write=False)
    return lut


def resize_normalize_chw(src: torch.Tensor, dst: torch.Tensor, mean, std) -> None:
    """Fused preprocessing: u8 bilinear resize (`_resize_u8` semantics, app.py:64-78)
    to dst's size, then f32(u)/255, minus `mean[c]`, divided by `std[c]`,
    written planar CHW into f32 `dst` `[C, H, W]` / `[N, C, H, W]` -- one
    kernel, no intermediate frame in HBM."""
    s = as_image(src, "src")
    n, c, h, w, d_is, d_ps, d_rp = as_planar(dst, "dst")
    if s.dtype != U8:
        raise UnsupportedDtype(f"source must be u8, got {s.dtype}")
    if dst.dtype != F32:
        raise UnsupportedDtype(f"destination must be f32, got {dst.dtype}")
    if s.c != c:
        raise SizeMismatch(f"source has {s.c} channels, destination {c}")
    if n != s.n:
        raise SizeMismatch(f"source batch {s.n} and destination batch {n} differ")
    if c > 4:
        raise ShapeMismatch(f"fused preprocessing supports up to 4 channels, got {c}")
    lut = _cached_lut(tuple(np.asarray(mean, np.float32).reshape(-1).tolist()),
                      tuple(np.asarray(std, np.float32).reshape(-1).tolist()))
    if lut.shape[0] != c:
        raise ShapeMismatch(f"mean/std have {lut.shape[0]} channels, image has {c}")
    check_distinct(src, dst)
    same_device(src, dst)
    with torch.cuda.device(src.device):
        _native.call("fv_resize_normalize_chw", s.ptr, s.img_stride, s.row_pitch, s.h, s.w,
                     dst.data_ptr(), d_is, d_ps, d_rp, h, w, c, n,
                     lut.ctypes.data_as(ctypes.c_void_p), stream_ptr(src))


# ---------------------------------------------------------------------------
# warps
# ---------------------------------------------------------------------------

def _matrices(m, n: int, rows: int, inverse: bool) -> np.ndarray:
    a = m.detach().cpu().numpy() if isinstance(m, torch.Tensor) else np.asarray(m)
    a = np.asarray(a, dtype=np.float64)
    if a.shape == (rows, 3):
        a = np.broadcast_to(a, (n, rows, 3))
    if a.shape != (n, rows, 3):
        raise ShapeMismatch(f"expected a {rows}x3 matrix or {n}x{rows}x3 matrices, got {a.shape}")
    if inverse:
        return np.ascontiguousarray(a)
    full = np.broadcast_to(np.eye(3), (n, 3, 3)).copy()
    full[:, :rows] = a
    try:
        inv = np.linalg.inv(full)  # batched f64 LAPACK getrf/getri, same per-matrix result as the oracle's
    except np.linalg.LinAlgError as e:
        raise SingularTransform("warp matrix is singular") from e
    if not np.all(np.isfinite(inv)):
        raise SingularTransform("warp matrix is singular")
    return np.ascontiguousarray(inv[:, :rows])


def _warp(src, dst, m, border, inverse, perspective, exact=True):
    s, d = as_image(src, "src"), as_image(dst, "dst")
    if s.dtype != d.dtype:
        raise UnsupportedDtype(f"source {s.dtype} and destination {d.dtype} must match")
    if s.dtype not in (U8, F32):
        raise UnsupportedDtype(f"warps support u8 and f32, got {s.dtype}")
    if s.c != d.c:
        raise SizeMismatch(f"source has {s.c} channels, destination {d.c}")
    check_distinct(src, dst)
    _check_batch(s, d)
    same_device(src, dst)
    mats = _matrices(m, s.n, 3 if perspective else 2, inverse)
    kind = "perspective" if perspective else "affine"
    if s.dtype == U8:
        b = int(border)
        if not 0 <= b <= 255:
            raise UnsupportedDtype(f"u8 border must be in [0, 255], got {border}")
        fn, bval = f"fv_warp_{kind}_u8" + ("" if exact else "_fast"), b
    else:
        fn, bval = f"fv_warp_{kind}_f32", float(border)
    with torch.cuda.device(src.device):
        _native.call(fn, s.ptr, s.img_stride, s.row_pitch, s.h, s.w, d.ptr, d.img_stride, d.row_pitch,
                     d.h, d.w, s.c, s.n, mats.ctypes.data_as(ctypes.c_void_p), bval, stream_ptr(src))


def warp_affine(src: torch.Tensor, dst: torch.Tensor, m, border=0, inverse: bool = False) -> None:
    """Bilinear affine warp into `dst` (absent from the reference, SPEC.md:369;
    contract in DESIGN.md §3). `m` is the forward (src -> dst) 2x3 matrix, or
    N of them; it is inverted once in f64 on the host (`inverse=True` passes
    dst -> src matrices directly). Taps outside the source read `border`."""
    _warp(src, dst, m, border, inverse, perspective=False)


def warp_perspective(src: torch.Tensor, dst: torch.Tensor, h, border=0, inverse: bool = False,
                     exact: bool = False) -> None:
    """Bilinear perspective warp into `dst` (absent from the reference). `h` is
    the forward 3x3 homography (or N of them), inverted once in f64 on the
    host. Pixels whose inverse-mapped W is 0 get the raw border value.

    u8 images: by default within 1 LSB of the builder oracle (the north-star
    gate for u8 results of float interpolation; f64 anchor + f32 projective
    correction per 32-pixel group, `fv_warp_perspective_u8_fast`); `exact=True`
    runs the bit-exact f64-per-pixel kernel. f32 images are always exact."""
    _warp(src, dst, h, border, inverse, perspective=True, exact=exact)


# ---------------------------------------------------------------------------
# flip, nearest, sobel
# ---------------------------------------------------------------------------

def flip_horizontal(src: torch.Tensor, dst: torch.Tensor) -> None:
    """dst(y, x) = src(y, width-1-x), all channels (imgproc.py:67-73). Any
    dtype of 1, 2, 4 or 8 bytes. Checks: layout (channels, dtype) ->
    SizeMismatch, size -> SizeMismatch, distinct -> AliasedBuffers."""
    s, d = as_image(src, "src"), as_image(dst, "dst")
    if s.c != d.c or s.dtype != d.dtype:
        raise SizeMismatch(f"source {s!r} and destination {d!r} differ in layout")
    if s.size != d.size:
        raise SizeMismatch(f"source {s!r} and destination {d!r} differ in size")
    check_distinct(src, dst)
    _check_batch(s, d)
    same_device(src, dst)
    with torch.cuda.device(src.device):
        _native.call("fv_flip_horizontal", s.ptr, s.img_stride, s.row_pitch, d.ptr, d.img_stride, d.row_pitch,
                     s.h, s.w, s.c, src.element_size(), s.n, stream_ptr(src))


def resize_nearest(src: torch.Tensor, dst: torch.Tensor) -> None:
    """Nearest-neighbour resize to dst's size (imgproc.py:89-97): index
    clip(ceil((x + 0.5) * src_n / dst_n) - 1, 0, src_n - 1) per axis (round
    half down of the pixel centre), any dtype of 1, 2, 4 or 8 bytes."""
    s, d = as_image(src, "src"), as_image(dst, "dst")
    if s.c != d.c or s.dtype != d.dtype:
        raise SizeMismatch(f"source {s!r} and destination {d!r} differ in layout")
    check_distinct(src, dst)
    _check_batch(s, d)
    same_device(src, dst)
    with torch.cuda.device(src.device):
        _native.call("fv_resize_nearest", s.ptr, s.img_stride, s.row_pitch, s.h, s.w, d.ptr, d.img_stride,
                     d.row_pitch, d.h, d.w, s.c, src.element_size(), s.n, stream_ptr(src))


def sobel(src: torch.Tensor, dst: torch.Tensor, kernel_size: int) -> None:
    """Gradient magnitude sqrt(Gx^2 + Gy^2) per channel, replicate border
    (imgproc.py:126-155), f32. Checks in the reference's order: kernel size
    (UnsupportedKernelSize), dtype (UnsupportedDtype), channels and size
    (SizeMismatch), distinct (AliasedBuffers)."""
    if kernel_size != 3:
        raise UnsupportedKernelSize(f"only kernel_size 3 is supported, got {kernel_size}")
    s, d = as_image(src, "src"), as_image(dst, "dst")
    if s.dtype != F32 or d.dtype != F32:
        raise UnsupportedDtype(f"sobel requires f32 images, got {s.dtype} -> {d.dtype}")
    if s.c != d.c:
        raise SizeMismatch(f"source has {s.c} channels, destination {d.c}")
    if s.size != d.size:
        raise SizeMismatch(f"source {s!r} and destination {d!r} differ in size")
    check_distinct(src, dst)
    _check_batch(s, d)
    same_device(src, dst)
    with torch.cuda.device(src.device):
        _native.call("fv_sobel_f32", s.ptr, s.img_stride, s.row_pitch, d.ptr, d.img_stride, d.row_pitch,
                     s.h, s.w, s.c, s.n, stream_ptr(src))
