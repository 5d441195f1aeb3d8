"""Torch tensor -> C-ABI image descriptors, and the reference's checks.

Images are torch CUDA tensors in HWC `[H, W, C]` or batched `[N, H, W, C]`
layout, the reference's interleaved layout (image.py:1-6). Crop views are
allowed: pixels must be interleaved (channel stride 1, pixel stride C) but
rows may have any pitch, like `ImageView` (image.py:66-75, 118-125).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from .errors import AliasedBuffers, NonContiguous, ShapeMismatch, UnsupportedDevice

U8 = torch.uint8
F32 = torch.float32


@dataclass(frozen=True)
class Img:
    t: torch.Tensor
    n: int
    h: int
    w: int
    c: int
    img_stride: int  # bytes
    row_pitch: int   # bytes

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    @property
    def dtype(self):
        return self.t.dtype

    @property
    def size(self):
        return (self.w, self.h)

    def __repr__(self) -> str:
        return f"Image({self.n}x{self.w}x{self.h}x{self.c}, {self.dtype})"


def as_image(t, name: str) -> Img:
    if not isinstance(t, torch.Tensor):
        raise ShapeMismatch(f"{name} must be a torch tensor, got {type(t).__name__}")
    if t.dim() not in (3, 4):
        raise ShapeMismatch(f"{name} must be [H, W, C] or [N, H, W, C], got shape {tuple(t.shape)}")
    es = t.element_size()
    st = t.stride()
    if t.dim() == 3:
        n, (h, w, c) = 1, t.shape
        img_stride = 0
    else:
        n, h, w, c = t.shape
        img_stride = st[0] * es
    if h < 1 or w < 1 or c < 1:
        raise ShapeMismatch(f"{name} has an empty image dimension: {tuple(t.shape)}")
    if (st[-1] != 1 and c > 1) or (st[-2] != c and w > 1):
        raise NonContiguous(f"{name} must have interleaved pixels (strides {st})")
    row_pitch = st[-3] * es if h > 1 else w * c * es
    return Img(t, n, h, w, c, img_stride, row_pitch)


def as_planar(t, name: str):
    """Planar CHW `[C, H, W]` / `[N, C, H, W]` f32 destination of the fused op.
    Returns (n, c, h, w, img_stride, plane_stride, row_pitch) in bytes."""
    if not isinstance(t, torch.Tensor) or t.dim() not in (3, 4):
        raise ShapeMismatch(f"{name} must be [C, H, W] or [N, C, H, W]")
    es = t.element_size()
    st = t.stride()
    if t.dim() == 3:
        n, (c, h, w) = 1, t.shape
        img_stride = 0
    else:
        n, c, h, w = t.shape
        img_stride = st[0] * es
    if st[-1] != 1 and w > 1:
        raise NonContiguous(f"{name} rows must be contiguous (strides {st})")
    return n, c, h, w, img_stride, st[-3] * es, st[-2] * es


def _extent(t: torch.Tensor):
    lo = t.data_ptr()
    span = sum((s - 1) * abs(st) for s, st in zip(t.shape, t.stride())) + 1
    return lo, lo + span * t.element_size()


def _runs(t: torch.Tensor):
    """Byte intervals [start, end) of `t`'s contiguous runs (the trailing
    dimensions merged while they are contiguous), sorted, or None when they
    are not disjoint and increasing (then the caller stays conservative)."""
    import numpy as np

    shape, stride = list(t.shape), list(t.stride())
    if any(s == 0 for s in shape):
        return np.empty(0, np.int64), np.empty(0, np.int64)
    run, k = 1, len(shape) - 1
    while k >= 0 and (shape[k] == 1 or stride[k] == run):
        run *= shape[k]
        k -= 1
    offs = np.zeros(1, np.int64)
    for d in range(k + 1):
        offs = (offs[:, None] + np.arange(shape[d], dtype=np.int64)[None, :] * stride[d]).reshape(-1)
    es = t.element_size()
    starts = np.sort(offs) * es + t.data_ptr()
    ends = starts + run * es
    if starts.size > 1 and np.any(starts[1:] < ends[:-1]):
        return None
    return starts, ends


def check_distinct(a: torch.Tensor, b: torch.Tensor) -> None:
    """imgproc.py:38-40 (`np.shares_memory`): AliasedBuffers when the two
    tensors share any byte. Disjoint address ranges pass at once; otherwise
    the exact test compares the tensors' contiguous runs (image rows), so
    interleaved views that share no element -- e.g. the left and right halves
    of one image -- are accepted, as NumPy accepts them."""
    if a.device != b.device:
        return
    a0, a1 = _extent(a)
    b0, b1 = _extent(b)
    if not (a0 < b1 and b0 < a1):
        return
    import numpy as np

    ra, rb = _runs(a), _runs(b)
    if ra is not None and rb is not None:
        (as_, ae), (bs, be) = ra, rb
        # for every run of b, the last run of a starting before b's end
        j = np.searchsorted(as_, be, side="left") - 1
        ok = j >= 0
        if not np.any(ae[j[ok]] > bs[ok]):
            return
    raise AliasedBuffers("source and destination must not share storage")


def same_device(*ts) -> None:
    """No CPU path: every operand must be a CUDA tensor on one device. Runs
    after the reference's own checks so their order is preserved."""
    dev = ts[0].device
    for t in ts:
        if not t.is_cuda:
            raise UnsupportedDevice(f"tensor on {t.device}: this library runs on CUDA only (no CPU fallback)")
    for t in ts[1:]:
        if t.device != dev:
            raise UnsupportedDevice(f"tensors on different devices: {dev} and {t.device}")


def stream_ptr(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream
