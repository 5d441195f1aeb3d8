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
import threading
from typing import Sequence

import torch

from . import _native
from .errors import CorruptStream, NativeError, ShapeMismatch, UnsupportedDevice, UnsupportedJpegFeature

_ERRORS = {_native.FV_ECORRUPT: CorruptStream, _native.FV_EUNSUPPORTED: UnsupportedJpegFeature}

# images decoded per entropy path by decode_jpeg_batch (introspection for the
# tests and the bench: the GPU path must be the one that runs)
stats = {"gpu_entropy": 0, "host_entropy": 0}


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
    with torch.cuda.device(dev):  # the library launches on the current device's stream
        return _reconstruct(info, coef, width, dev)


class _Staging:
    """Pinned host staging for the batched decode, reused across calls. The
    library copies from it with its own cudaMemcpyAsync (invisible to torch's
    host allocator), so reuse waits on the event recorded after the last
    batch's copies."""

    lock = threading.Lock()
    buf = None
    event = None

    @classmethod
    def get(cls, nbytes: int) -> torch.Tensor:
        if cls.event is not None:
            cls.event.synchronize()
        if cls.buf is None or cls.buf.numel() < nbytes:
            cls.buf = None
            cls.buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, pin_memory=True)
        return cls.buf


def _host_batch(bufs, infos, outs, planes, plane_off, threads, stream, dev):
    """Host entropy decoding (native batch runtime) of `bufs` into `outs`:
    raises the first failing stream's error, in order."""
    n = len(bufs)
    lib = _native.lib()
    data = (ctypes.c_char_p * n)(*bufs)
    lens = (ctypes.c_int64 * n)(*[len(b) for b in bufs])
    info_arr = (_native.FvJpegInfo * n)(*infos)
    status = (ctypes.c_int32 * n)()
    word_off = []
    c = 0
    for f in infos:
        word_off.append(c)
        c += (int(f.coef_count) // 64 + int(f.sparse_words) + 31) // 32 * 32
    words_dev = torch.empty(max(c, 1), dtype=torch.int32, device=dev)
    with _Staging.lock:
        host = _Staging.get(4 * c)
        rc = lib.fv_jpeg_decode_batch(
            data, lens, n, info_arr, host.data_ptr(), (ctypes.c_int64 * n)(*word_off), words_dev.data_ptr(),
            planes.data_ptr(), (ctypes.c_int64 * n)(*plane_off), (ctypes.c_void_p * n)(*[o.data_ptr() for o in outs]),
            (ctypes.c_int64 * n)(*[o.stride(0) for o in outs]), status, threads, stream.cuda_stream)
        _Staging.event = torch.cuda.Event()
        _Staging.event.record(stream)
    if rc:
        i = next(k for k in range(n) if status[k])
        if status[i] != _native.FV_ERANGE:
            decode_jpeg(bufs[i], dev)  # raises with the message
            _raise(status[i], "fv_jpeg_decode_batch")
        # a DC coefficient beyond int16: this image with int64 coefficients, then the rest
        outs[i].copy_(decode_jpeg(bufs[i], dev))
        if i + 1 < n:
            _host_batch(bufs[i + 1:], infos[i + 1:], outs[i + 1:], planes, plane_off[i + 1:], threads, stream, dev)


def decode_jpeg_batch(streams: Sequence, device=None, threads: int | None = None, entropy: str = "gpu",
                      out: torch.Tensor | None = None) -> list:
    """Decode many streams. entropy="gpu" (default): headers parsed and
    segments unstuffed on `threads` host threads, Huffman decoding on the GPU
    (`fv_jpeg_decode_batch_gpu`); streams outside its coverage or with a
    corrupt entropy segment go through the host decoder. entropy="host": the
    native host batch runtime (threaded entropy decoding, each image's H2D +
    kernels issued as soon as it is ready). Either way the output is
    bit-identical to `decode_jpeg`, and the first failing stream's error (in
    input order) is raised, as a loop of `decode_jpeg` calls would.
    out: optional (N, H, W, C) u8 CUDA tensor receiving image i in out[i]
    (every stream must decode to (H, W, C)), e.g. to preprocess the whole
    batch with one `resize_normalize_chw` launch; the returned list then
    holds the views out[i]."""
    if entropy not in ("gpu", "host"):
        raise ValueError(f"entropy must be 'gpu' or 'host', got {entropy!r}")
    dev = _device(device)
    # every native call below allocates / launches on the current device
    # (pinned staging, streams): make it `dev` even when it is not current
    with torch.cuda.device(dev):
        return _decode_batch(streams, dev, threads, entropy, out)


def _decode_batch(streams, dev, threads, entropy, out):
    bufs = [_bytes(d) for d in streams]
    n = len(bufs)
    if n == 0:
        return []
    threads = threads or max(1, len(os.sched_getaffinity(0)))
    lib = _native.lib()
    data = (ctypes.c_char_p * n)(*bufs)
    lens = (ctypes.c_int64 * n)(*[len(b) for b in bufs])
    infos = (_native.FvJpegInfo * n)()
    status = (ctypes.c_int32 * n)()
    handle = ctypes.c_void_p()
    if entropy == "gpu":  # one parse: the plan also stages the GPU path's inputs
        rc = lib.fv_jpeg_batch_plan(data, lens, n, infos, status, threads, ctypes.byref(handle))
        if rc:
            _raise(rc, "fv_jpeg_batch_plan")
    else:
        lib.fv_jpeg_info_batch(data, lens, n, infos, status, threads)
    try:
        k = next((i for i in range(n) if status[i]), n)  # images before the first header error
        if out is not None:
            if (out.device != dev or out.dtype != torch.uint8 or out.dim() != 4 or out.shape[0] != n
                    or out.stride(3) != 1 or out.stride(2) != out.shape[3]):
                raise ShapeMismatch(f"out must be a ({n}, H, W, C) u8 tensor on {dev} with interleaved rows")
            for i, f in enumerate(infos[:k]):
                if tuple(out.shape[1:]) != (f.height, f.width, f.ncomp):
                    raise ShapeMismatch(f"stream {i} decodes to {(f.height, f.width, f.ncomp)}, out holds "
                                        f"{tuple(out.shape[1:])}")
        outs, plane_off = [], []
        p = 0
        for i in range(n):
            f = infos[i]
            ok = i < k
            outs.append((out[i] if out is not None else
                         torch.empty((f.height, f.width, f.ncomp), dtype=torch.uint8, device=dev)) if ok else None)
            plane_off.append(p)
            p += (int(f.plane_bytes) + 255) // 256 * 256 if ok else 0
        planes = torch.empty(max(p, 256), dtype=torch.uint8, device=dev)
        stream = torch.cuda.current_stream(dev)
        rest = list(range(k))
        if entropy == "gpu" and k:
            st = (ctypes.c_int32 * n)()
            # images from the first header error on: no target (NULL), not reconstructed
            dst = [o.data_ptr() if o is not None else None for o in outs]
            rc = lib.fv_jpeg_batch_run_gpu(
                handle, planes.data_ptr(), (ctypes.c_int64 * n)(*plane_off), (ctypes.c_void_p * n)(*dst),
                (ctypes.c_int64 * n)(*[o.stride(0) if o is not None else 0 for o in outs]), st,
                stream.cuda_stream)
            if rc:
                _raise(rc, "fv_jpeg_batch_run_gpu")
            rest = [i for i in range(k) if st[i] != 0]
            stats["gpu_entropy"] += k - len(rest)
        stats["host_entropy"] += len(rest)
        if rest:
            _host_batch([bufs[i] for i in rest], [infos[i] for i in rest], [outs[i] for i in rest], planes,
                        [plane_off[i] for i in rest], threads, stream, dev)
    finally:
        if handle.value:
            lib.fv_jpeg_batch_free(handle)
    outs = outs[:k]
    if k < n:
        jpeg_info(bufs[k])  # raises the header error of stream k
    return outs


def decoded_shape(data) -> tuple:
    info = jpeg_info(data)
    return (info.height, info.width, info.ncomp)


__all__ = ["decode_jpeg", "decode_jpeg_batch", "decode_coefficients", "jpeg_info", "decoded_shape"]
