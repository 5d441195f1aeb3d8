"""CPU: the C-ABI library loads and exports every symbol include/fovea_b200.h
declares; the Python mirror raises the reference's exception classes in the
reference's check order and refuses CPU tensors (no CPU fallback)."""
import os
import re

import numpy as np
import pytest
import torch

import paper_2505_12425_b200 as fv
from paper_2505_12425_b200 import _native
from paper_2505_12425_b200.errors import (
    AliasedBuffers,
    FoveaError,
    NonContiguous,
    ShapeMismatch,
    SizeMismatch,
    UnsupportedDevice,
    UnsupportedDtype,
)

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "fovea_b200.h")


def header_symbols(test_build=False):
    """Entry points the header declares; those inside `#ifdef FV_TEST_KNOBS`
    only for the test build."""
    text = open(HEADER).read()
    knob_blocks = re.findall(r"#ifdef FV_TEST_KNOBS(.*?)#endif", text, flags=re.S)
    knobs = set(re.findall(r"\b(fv_[a-z0-9_]+)\s*\(", "".join(knob_blocks)))
    every = set(re.findall(r"\b(fv_[a-z0-9_]+)\s*\(", text))
    return sorted(every if test_build else every - knobs)


class TestAbi:
    def test_header_declares_the_hot_path(self):
        syms = header_symbols()
        for s in ["fv_gray_from_rgb_u8", "fv_resize_bilinear_u8", "fv_resize_bilinear_f32", "fv_warp_affine_f32",
                  "fv_warp_perspective_u8", "fv_resize_normalize_chw", "fv_to_float_scaled"]:
            assert s in syms

    def test_library_loads_and_exports_every_symbol(self):
        lib = _native.lib()
        for s in header_symbols():
            assert hasattr(lib, s), s
        assert lib.fv_version() == 100

    def test_binding_table_matches_header(self):
        assert sorted(_native.SIGNATURES) == header_symbols()
        assert sorted({**_native.SIGNATURES, **_native.KNOB_SIGNATURES}) == header_symbols(test_build=True)

    def test_path_knobs_only_in_the_test_build(self):
        """fv_set_resize_path / fv_set_warp_path are process-global test
        switches: absent from the product library, present in the test build."""
        import ctypes

        prod = ctypes.CDLL(_native.LIB_PATH)
        knobs = ctypes.CDLL(_native.KNOBS_PATH)
        for s in ("fv_set_resize_path", "fv_set_warp_path"):
            assert not hasattr(prod, s)
            assert hasattr(knobs, s)
        for s in header_symbols():
            assert hasattr(knobs, s), s

    def test_bad_arguments_rejected_before_launch(self):
        # EINVAL paths return before touching the device, so they run on CPU
        lib = _native.lib()
        rc = lib.fv_gray_from_rgb_u8(None, 0, 0, None, 0, 0, 1, 0, 4, None)
        assert rc == -1
        assert b"bad shape" in lib.fv_last_error()
        rc = lib.fv_resize_bilinear_u8(None, 0, 0, 4, 4, None, 0, 0, 4, 4, 3, 1, None)
        assert rc == -1 and b"null pointer" in lib.fv_last_error()

    def test_empty_batch_is_a_no_op(self):
        lib = _native.lib()
        assert lib.fv_gray_from_rgb_u8(None, 0, 0, None, 0, 0, 0, 4, 4, None) == 0
        assert lib.fv_resize_bilinear_u8(None, 0, 0, 4, 4, None, 0, 0, 8, 8, 3, 0, None) == 0
        assert lib.fv_warp_perspective_u8(None, 0, 0, 4, 4, None, 0, 0, 4, 4, 3, 0, None, 0, None) == 0


def u8(*shape):
    return torch.zeros(shape, dtype=torch.uint8)


def f32(*shape):
    return torch.zeros(shape, dtype=torch.float32)


class TestCheckOrder:
    """imgproc.py:48-52 / :102-106 / image.py:152-157 check order, on CPU tensors:
    the reference's checks fire first, the device check last."""

    def test_gray_channels_first(self):
        with pytest.raises(SizeMismatch):
            fv.gray_from_rgb(u8(2, 2, 4), f32(2, 2, 1))  # channel error wins over dtype error

    def test_gray_dtype_before_size(self):
        with pytest.raises(UnsupportedDtype):
            fv.gray_from_rgb(u8(2, 2, 3), f32(2, 3, 1))

    def test_gray_size(self):
        with pytest.raises(SizeMismatch):
            fv.gray_from_rgb(u8(2, 2, 3), u8(2, 3, 1))

    def test_gray_unsupported_dtype(self):
        with pytest.raises(UnsupportedDtype):
            fv.gray_from_rgb(torch.zeros(2, 2, 3, dtype=torch.int16), torch.zeros(2, 2, 1, dtype=torch.int16))

    def test_resize_rejects_u8_like_the_reference(self):
        with pytest.raises(UnsupportedDtype):
            fv.resize_bilinear(u8(4, 4, 3), u8(8, 8, 3))

    def test_resize_channels_then_alias(self):
        with pytest.raises(SizeMismatch):
            fv.resize_bilinear(f32(4, 4, 3), f32(8, 8, 2))
        t = f32(4, 4, 3)
        with pytest.raises(AliasedBuffers):
            fv.resize_bilinear(t, t)
        # overlapping crop views of one parent are rejected
        p = f32(8, 8, 3)
        with pytest.raises(AliasedBuffers):
            fv.resize_bilinear(p[:4], p[2:6])

    def test_alias_test_is_exact_like_np_shares_memory(self):
        """imgproc.py:38-40 uses np.shares_memory: interleaved views of one
        parent that share no element pass, any shared element is rejected."""
        import numpy as np

        from paper_2505_12425_b200._tensors import check_distinct

        p = f32(6, 10, 3)
        cases = [(p[:, :5], p[:, 5:]), (p[:, :6], p[:, 5:]), (p[:3], p[3:]), (p[:4], p[3:]),
                 (p[::2], p[1::2]), (p[:, ::2], p[:, 1::2]), (p[1:3, 2:7], p[2:5, 6:9]), (p[1:3, 2:6], p[2:5, 6:9])]
        for a, b in cases:
            shares = np.shares_memory(a.numpy(), b.numpy())
            if shares:
                with pytest.raises(AliasedBuffers):
                    check_distinct(a, b)
            else:
                check_distinct(a, b)

    def test_to_float_scaled_order(self):
        with pytest.raises(UnsupportedDtype):
            fv.to_float_scaled(f32(2, 2, 3), f32(2, 2, 3))
        with pytest.raises(UnsupportedDtype):
            fv.to_float_scaled(u8(2, 2, 3), u8(2, 2, 3))
        with pytest.raises(SizeMismatch):
            fv.to_float_scaled(u8(2, 2, 3), f32(2, 2, 1))

    def test_batch_mismatch(self):
        with pytest.raises(SizeMismatch):
            fv.resize_bilinear_u8(u8(2, 4, 4, 3), u8(3, 8, 8, 3))

    def test_layout_errors(self):
        with pytest.raises(ShapeMismatch):
            fv.resize_bilinear_u8(u8(4, 4), u8(8, 8))
        planar = u8(3, 4, 4).permute(1, 2, 0)  # channel stride != 1
        with pytest.raises(NonContiguous):
            fv.resize_bilinear_u8(planar, u8(8, 8, 3))

    def test_warp_checks(self):
        with pytest.raises(UnsupportedDtype):
            fv.warp_affine(u8(4, 4, 3), f32(4, 4, 3), np.eye(3)[:2])
        with pytest.raises(SizeMismatch):
            fv.warp_perspective(u8(4, 4, 3), u8(4, 4, 1), np.eye(3))

    def test_fused_checks(self):
        with pytest.raises(UnsupportedDtype):
            fv.resize_normalize_chw(f32(4, 4, 3), f32(3, 2, 2), (0, 0, 0), (1, 1, 1))
        with pytest.raises(SizeMismatch):
            fv.resize_normalize_chw(u8(4, 4, 3), f32(1, 2, 2), (0,), (1,))

    @pytest.mark.parametrize("call", [
        lambda: fv.gray_from_rgb(u8(2, 2, 3), u8(2, 2, 1)),
        lambda: fv.resize_bilinear(f32(4, 4, 3), f32(8, 8, 3)),
        lambda: fv.resize_bilinear_u8(u8(4, 4, 3), u8(8, 8, 3)),
        lambda: fv.to_float_scaled(u8(2, 2, 3), f32(2, 2, 3)),
        lambda: fv.warp_affine(f32(4, 4, 3), f32(4, 4, 3), np.eye(3)[:2]),
        lambda: fv.warp_perspective(u8(4, 4, 3), u8(4, 4, 3), np.eye(3)),
        lambda: fv.resize_normalize_chw(u8(4, 4, 3), f32(3, 2, 2), (0, 0, 0), (1, 1, 1)),
    ])
    def test_no_cpu_fallback(self, call):
        with pytest.raises(UnsupportedDevice):
            call()

    def test_errors_share_the_reference_base(self):
        for cls in (SizeMismatch, UnsupportedDtype, AliasedBuffers, UnsupportedDevice, NonContiguous, ShapeMismatch):
            assert issubclass(cls, FoveaError)


def test_normalize_lut_shape_and_values():
    from paper_2505_12425_b200 import synth

    lut = fv.normalize_lut(synth.MEAN, synth.STD)
    assert lut.shape == (3, 256) and lut.dtype == np.float32
    u = np.float32(128) / np.float32(255)
    assert lut[1, 128] == (u - np.float32(0.456)) / np.float32(0.224)
