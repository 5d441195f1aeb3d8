"""`to_float_scaled` (image.py:150-160) on B200."""
from __future__ import annotations

import torch

from . import _native
from ._tensors import F32, U8, as_image, check_distinct, same_device, stream_ptr
from .errors import SizeMismatch, UnsupportedDtype


def to_float_scaled(src: torch.Tensor, dst: torch.Tensor) -> None:
    """Write src / 255 into a caller-provided f32 image; no allocations.

    Checks in the reference's order (image.py:152-157): src u8, dst f32
    (UnsupportedDtype), then size and channels (SizeMismatch)."""
    s, d = as_image(src, "src"), as_image(dst, "dst")
    if s.dtype != U8:
        raise UnsupportedDtype(f"source must be u8, got {s.dtype}")
    if d.dtype != F32:
        raise UnsupportedDtype(f"destination must be f32, got {d.dtype}")
    if s.size != d.size or s.c != d.c or s.n != d.n:
        raise SizeMismatch(f"source {s!r} and destination {d!r} differ")
    same_device(src, dst)
    check_distinct(src, dst)
    with torch.cuda.device(src.device):
        _native.call("fv_to_float_scaled", s.ptr, s.img_stride, s.row_pitch, d.ptr, d.img_stride, d.row_pitch,
                     s.n, s.h, s.w, s.c, stream_ptr(src))
