"""fovea-b200: the kornia-rs / `fovea` image-transformation hot path on B200.

Public API (drop-in for the reference's `fovea.imgproc` / `fovea.image`
functions on torch CUDA tensors):

    gray_from_rgb(src, dst)                    imgproc.py:43-64
    resize_bilinear(src, dst)                  imgproc.py:100-123 (f32)
    resize_bilinear_u8(src, dst)               service/app.py:64-78 (_resize_u8)
    to_float_scaled(src, dst)                  image.py:150-160
    warp_affine(src, dst, m, border=0)         builder contract
    warp_perspective(src, dst, h, border=0)    builder contract
    resize_normalize_chw(src, dst, mean, std)  fused preprocessing
    resize_nearest(src, dst)                   imgproc.py:89-97
    flip_horizontal(src, dst)                  imgproc.py:67-73
    sobel(src, dst, 3)                         imgproc.py:126-155
    io.decode_jpeg(data) -> tensor             io/jpeg.py:605-806 (decode -> preprocess)

Every call is one sm_100a kernel launch through the C ABI in
include/fovea_b200.h; there is no CPU fallback.
"""
from .errors import (  # noqa: F401
    AliasedBuffers,
    CorruptStream,
    FoveaError,
    NativeError,
    NonContiguous,
    ShapeMismatch,
    SingularTransform,
    SizeMismatch,
    UnsupportedDevice,
    UnsupportedDtype,
    UnsupportedJpegFeature,
    UnsupportedKernelSize,
)
from . import io  # noqa: F401,E402
from .image import to_float_scaled  # noqa: F401
from .imgproc import (  # noqa: F401
    flip_horizontal,
    gray_from_rgb,
    normalize_lut,
    resize_bilinear,
    resize_bilinear_u8,
    resize_nearest,
    resize_normalize_chw,
    sobel,
    warp_affine,
    warp_perspective,
)

__version__ = "0.1.0"
