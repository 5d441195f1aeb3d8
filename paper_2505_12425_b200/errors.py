"""Exception types of the hot path, mirroring the reference's names.

Same class names and hierarchy as `fovea.errors` (errors.py:8-63) so that
callers catching the reference's exceptions catch these. Only the classes the
image-transformation path raises are mirrored; two are new for the GPU
boundary (`UnsupportedDevice`, `SingularTransform`) and one (`NativeError`)
wraps a failure reported by the C ABI.
"""


class FoveaError(Exception):
    """Base class for all library errors (errors.py:8-9)."""


class UnsupportedDtype(FoveaError):
    """Element type outside the supported set, or mismatched operand dtypes (errors.py:14-15)."""


class ShapeMismatch(FoveaError):
    """Operand shapes differ where equality is required (errors.py:38-39)."""


class NonContiguous(FoveaError):
    """Operation requires interleaved (pixel-contiguous) storage (errors.py:30-31)."""


class SizeMismatch(FoveaError):
    """Source and destination image sizes differ (errors.py:50-51)."""


class AliasedBuffers(FoveaError):
    """Source and destination share storage where they must be distinct (errors.py:58-59)."""


class UnsupportedKernelSize(FoveaError):
    """Filter kernel size outside the supported set (errors.py:62-63)."""


class CorruptStream(FoveaError):
    """Byte stream is not a well-formed instance of the expected format (errors.py:68-69)."""


class UnsupportedJpegFeature(FoveaError):
    """Valid JPEG using a feature outside the supported subset, e.g. progressive (errors.py:76-77)."""


class UnsupportedDevice(FoveaError):
    """Tensor is not resident on a CUDA device (there is no CPU path)."""


class SingularTransform(FoveaError):
    """Warp matrix cannot be inverted."""


class NativeError(FoveaError):
    """The CUDA library reported a failure (launch error or bad argument)."""
