"""decode -> preprocess: the reference's `fovea.io.decode_jpeg` on the GPU.

`decode_jpeg(data) -> torch.Tensor` mirrors `fovea.io.jpeg.decode_jpeg(data)
-> Image` (io/jpeg.py:605-806): same stream subset, same errors
(`CorruptStream`, `UnsupportedJpegFeature`), bit-identical samples; the
result is an (H, W, C) u8 CUDA tensor (C = 3 for YCbCr streams, 1 for gray)
ready for `resize_normalize_chw`.

Work split (include/fovea_b200.h, "decode -> preprocess"): header parsing and
Huffman entropy decoding run on the host in the C ABI library -- serial per
restart segment by the format, so `decode_jpeg_batch` spreads images over
host threads (ctypes releases the GIL) -- and the dense stages (dequantise,
islow IDCT, chroma upsampling, YCbCr -> RGB) run as sm_100a kernels after one
H2D copy of the coefficients from pinned memory.
"""
from __future__ import annotations

import ctypes
import os
from concurrent.futures import ThreadPoolExecutor
from typing import Sequence

import torch

from . import _native
from .errors import CorruptStream, NativeError, UnsupportedDevice, UnsupportedJpegFeature

_ERRORS = {_native.FV_ECORRUPT: CorruptStream, _native.FV_EUNSUPPORTED: UnsupportedJpegFeature}


def _raise(rc: int, what: str) -> None:
    msg = _native.lib().fv_last_error().decode(errors="replace")
    cls = _ERRORS.get(rc)
    if cls is not None:
        raise cls(msg)
    raise NativeError(f"{what} failed ({rc}): {msg}")


def _bytes(data) -> bytes:
    if isinstance(data, (bytes, bytearray, memoryview)):
        return bytes(data)
    raise CorruptStream(f"expected a bytes-like JPEG stream, got {type(data).__name__}")


def jpeg_info(data) -> _native.FvJpegInfo:
    """Parsed header and buffer sizes (no entropy decoding)."""
    buf = _bytes(data)
    info = _native.FvJpegInfo()
    rc = _native.lib().fv_jpeg_info(buf, len(buf), ctypes.byref(info))
    if rc:
        _raise(rc, "fv_jpeg_info")
    return info


def _decode_coeffs(buf: bytes, info, pinned: bool):
    """Host entropy decoding into an int16 buffer (int64 when a DC value
    does not fit int16). Returns (tensor, coef_bytes)."""
    for dtype, width in ((torch.int16, 2), (torch.int64, 8)):
        t = torch.empty(max(int(info.coef_count), 1), dtype=dtype, pin_memory=pinned)
        rc = _native.lib().fv_jpeg_decode_coeffs(buf, len(buf), t.data_ptr(), t.numel(), width)
        if rc == 0:
            return t, width
        if rc != _native.FV_ERANGE:
            _raise(rc, "fv_jpeg_decode_coeffs")
    raise NativeError("fv_jpeg_decode_coeffs: coefficient range")  # unreachable: int64 always fits


def decode_coefficients(data):
    """Host-only step (no GPU): (info, quantised coefficients as an int64
    NumPy array in the library's layout). Used by the CPU parity tests."""
    buf = _bytes(data)
    info = jpeg_info(buf)
    t, _ = _decode_coeffs(buf, info, pinned=False)
    return info, t.to(torch.int64).numpy()


def _device(device) -> torch.device:
    if not torch.cuda.is_available():
        raise UnsupportedDevice("decode_jpeg runs its reconstruction on CUDA only (no CPU fallback)")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise UnsupportedDevice(f"device {dev}: this library runs on CUDA only (no CPU fallback)")
    return dev


def _reconstruct(info, coef_host: torch.Tensor, width: int, dev: torch.device, out=None) -> torch.Tensor:
    stream = torch.cuda.current_stream(dev)
    coef = coef_host.to(dev, non_blocking=True)
    planes = torch.empty(max(int(info.plane_bytes), 8), dtype=torch.uint8, device=dev)
    if out is None:
        out = torch.empty((info.height, info.width, info.ncomp), dtype=torch.uint8, device=dev)
    rc = _native.lib().fv_jpeg_reconstruct(ctypes.byref(info), coef.data_ptr(), width, planes.data_ptr(),
                                           out.data_ptr(), out.stride(0), stream.cuda_stream)
    if rc:
        _raise(rc, "fv_jpeg_reconstruct")
    return out


def decode_jpeg(data, device=None) -> torch.Tensor:
    """io/jpeg.py:605-806 -> (H, W, C) u8 tensor on `device` (default: the
    current CUDA device). Asynchronous on the current stream after the host
    entropy decoding returns."""
    buf = _bytes(data)
    dev = _device(device)
    info = jpeg_info(buf)
    coef, width = _decode_coeffs(buf, info, pinned=True)
    return _reconstruct(info, coef, width, dev)


def decode_jpeg_batch(streams: Sequence, device=None, threads: int | None = None) -> list:
    """Decode many streams: host entropy decoding on `threads` host threads
    (default: the usable cores), reconstruction kernels on the current stream.
    Raises the first stream's error, in input order."""
    dev = _device(device)
    bufs = [_bytes(d) for d in streams]
    threads = threads or max(1, len(os.sched_getaffinity(0)))

    def host(buf):
        info = jpeg_info(buf)
        coef, width = _decode_coeffs(buf, info, pinned=True)
        return info, coef, width

    with ThreadPoolExecutor(max_workers=min(threads, max(1, len(bufs)))) as ex:
        parts = list(ex.map(host, bufs))
    return [_reconstruct(info, coef, width, dev) for info, coef, width in parts]


def decoded_shape(data) -> tuple:
    info = jpeg_info(data)
    return (info.height, info.width, info.ncomp)


__all__ = ["decode_jpeg", "decode_jpeg_batch", "decode_coefficients", "jpeg_info", "decoded_shape"]
