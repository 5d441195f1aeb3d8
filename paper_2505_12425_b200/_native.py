"""ctypes binding of the C ABI declared in include/fovea_b200.h.

The library is the product: there is no CPU fallback. Loading fails loudly
(`NativeError`) when `lib/libfovea_b200.so` is missing; build it with
`python -m paper_2505_12425_b200._build` (or `__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import NativeError

# FOVEA_B200_LIB overrides the in-tree library (A/B builds of the same ABI)
LIB_PATH = os.environ.get("FOVEA_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "lib", "libfovea_b200.so")
# test build (-DFV_TEST_KNOBS): the same kernels plus the path-selection knobs
KNOBS_PATH = os.environ.get("FOVEA_B200_KNOBS_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "lib", "libfovea_b200_knobs.so")

_c = ctypes
_I64, _I32, _P, _D = _c.c_int64, _c.c_int32, _c.c_void_p, _c.c_double

# symbol -> argtypes; mirrors include/fovea_b200.h one to one
_IMG2 = [_P, _I64, _I64, _P, _I64, _I64]
SIGNATURES = {
    "fv_version": ([], _c.c_int),
    "fv_last_error": ([], _c.c_char_p),
    "fv_launch_count": ([], _c.c_uint64),
    "fv_gray_from_rgb_u8": (_IMG2 + [_I32, _I32, _I32, _P], _c.c_int),
    "fv_gray_from_rgb_f32": (_IMG2 + [_I32, _I32, _I32, _P], _c.c_int),
    "fv_to_float_scaled": (_IMG2 + [_I32, _I32, _I32, _I32, _P], _c.c_int),
    "fv_resize_bilinear_f32": ([_P, _I64, _I64, _I32, _I32, _P, _I64, _I64, _I32, _I32, _I32, _I32, _P], _c.c_int),
    "fv_resize_bilinear_u8": ([_P, _I64, _I64, _I32, _I32, _P, _I64, _I64, _I32, _I32, _I32, _I32, _P], _c.c_int),
    "fv_resize_normalize_chw": ([_P, _I64, _I64, _I32, _I32, _P, _I64, _I64, _I64, _I32, _I32, _I32, _I32, _P, _P],
                                _c.c_int),
    "fv_warp_affine_f32": ([_P, _I64, _I64, _I32, _I32, _P, _I64, _I64, _I32, _I32, _I32, _I32, _P, _c.c_float, _P],
                           _c.c_int),
    "fv_warp_affine_u8": ([_P, _I64, _I64, _I32, _I32, _P, _I64, _I64, _I32, _I32, _I32, _I32, _P, _c.c_uint8, _P],
                          _c.c_int),
    "fv_warp_perspective_u8": ([_P, _I64, _I64, _I32, _I32, _P, _I64, _I64, _I32, _I32, _I32, _I32, _P, _c.c_uint8,
                                _P], _c.c_int),
    "fv_warp_perspective_u8_fast": ([_P, _I64, _I64, _I32, _I32, _P, _I64, _I64, _I32, _I32, _I32, _I32, _P,
                                     _c.c_uint8, _P], _c.c_int),
    "fv_warp_perspective_f32": ([_P, _I64, _I64, _I32, _I32, _P, _I64, _I64, _I32, _I32, _I32, _I32, _P, _c.c_float,
                                 _P], _c.c_int),
    "fv_resize_nearest": ([_P, _I64, _I64, _I32, _I32, _P, _I64, _I64, _I32, _I32, _I32, _I32, _I32, _P], _c.c_int),
    "fv_flip_horizontal": (_IMG2 + [_I32, _I32, _I32, _I32, _I32, _P], _c.c_int),
    "fv_sobel_f32": (_IMG2 + [_I32, _I32, _I32, _I32, _P], _c.c_int),
}



class FvJpegInfo(_c.Structure):
    """Mirror of `FvJpegInfo` (include/fovea_b200.h)."""

    _fields_ = [
        ("width", _I32), ("height", _I32), ("ncomp", _I32),
        ("hmax", _I32), ("vmax", _I32), ("mcus_x", _I32), ("mcus_y", _I32),
        ("restart_interval", _I32),
        ("h", _I32 * 3), ("v", _I32 * 3), ("bw", _I32 * 3), ("bh", _I32 * 3), ("cw", _I32 * 3), ("ch", _I32 * 3),
        ("coef_offset", _I64 * 3), ("coef_count", _I64),
        ("plane_offset", _I64 * 3), ("plane_bytes", _I64), ("sparse_words", _I64),
        ("qt", (_c.c_uint16 * 64) * 3),
    ]


SIGNATURES.update({
    "fv_jpeg_info": ([_P, _I64, _c.POINTER(FvJpegInfo)], _c.c_int),
    "fv_jpeg_decode_coeffs": ([_P, _I64, _P, _I64, _I32], _c.c_int),
    "fv_jpeg_reconstruct": ([_c.POINTER(FvJpegInfo), _P, _I32, _P, _P, _I64, _P], _c.c_int),
    "fv_jpeg_info_batch": ([_P, _P, _I32, _c.POINTER(FvJpegInfo), _P, _I32], _c.c_int),
    "fv_jpeg_decode_batch": ([_P, _P, _I32, _c.POINTER(FvJpegInfo), _P, _P, _P, _P, _P, _P, _P, _P, _I32, _P],
                             _c.c_int),
    "fv_jpeg_decode_batch_gpu": ([_P, _P, _I32, _c.POINTER(FvJpegInfo), _P, _P, _P, _P, _P, _I32, _P], _c.c_int),
    "fv_jpeg_batch_plan": ([_P, _P, _I32, _c.POINTER(FvJpegInfo), _P, _I32, _c.POINTER(_c.c_void_p)], _c.c_int),
    "fv_jpeg_batch_run_gpu": ([_c.c_void_p, _P, _P, _P, _P, _P, _P], _c.c_int),
    "fv_jpeg_batch_free": ([_c.c_void_p], None),
})

FV_ECORRUPT, FV_EUNSUPPORTED, FV_ERANGE, FV_EFALLBACK = -3, -4, -5, -6

KNOB_SIGNATURES = {"fv_set_resize_path": ([_I32], None), "fv_set_warp_path": ([_I32], None)}

_libs = {}
_use_knobs = False
_lock = threading.Lock()


def _load(path, knobs):
    if not os.path.exists(path):
        raise NativeError(
            f"CUDA library not built: {path} is missing "
            "(run `python -m paper_2505_12425_b200._build`); there is no CPU fallback")
    import torch  # noqa: F401  -- loads the shared libcudart the library binds to
    handle = ctypes.CDLL(path)
    for name, (args, res) in {**SIGNATURES, **(KNOB_SIGNATURES if knobs else {})}.items():
        fn = getattr(handle, name)
        fn.argtypes = args
        fn.restype = res
    return handle


def lib():
    """The loaded library (loaded on first use): the product build, or the
    test build while `use_test_build(True)` is in effect."""
    key = "knobs" if _use_knobs else "product"
    h = _libs.get(key)
    if h is not None:
        return h
    with _lock:
        if key not in _libs:
            _libs[key] = _load(KNOBS_PATH if _use_knobs else LIB_PATH, _use_knobs)
    return _libs[key]


def use_test_build(on: bool) -> None:
    """Tests and A/B tools only: route every call through the test build
    (lib/libfovea_b200_knobs.so, -DFV_TEST_KNOBS), whose fv_set_resize_path /
    fv_set_warp_path force a particular kernel. Process-global."""
    global _use_knobs
    _use_knobs = bool(on)


def call(name: str, *args) -> None:
    """Call an ABI entry point and raise `NativeError` on a non-zero return."""
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().fv_last_error().decode(errors="replace")
        raise NativeError(f"{name} failed ({rc}): {msg}")


def launch_count() -> int:
    return int(lib().fv_launch_count())
