"""CPU oracle for the image-transformation hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu-baseline /
`--impl reference` leg may import this package, and only as the checker (or
as the timed CPU reference arm). The product package
`paper_2505_12425_b200` never imports it: its path is the sm_100a CUDA
library, and it fails loudly when that library is missing.

Parity status:
  * gray_from_rgb, resize_bilinear (f32), to_float_scaled, cast→u8 and the
    `_resize_u8` composition are restatements of reference code and are
    PINNED against golden vectors produced by importing the reference itself
    (tests/golden/make_golden.py) and against the reference's own
    known-answer tests.
  * warp_affine, warp_perspective and the fused resize→normalise→CHW chain do
    not exist in the reference. Their contracts are
    builder-authored, consistent with the reference conventions; their
    golden vectors pin only the *components* they are composed from
    (bilinear blend order, u8 recipe, to_float_scaled). The composed ops are
    "parity unpinned" against any reference implementation.
"""
from .fovea_oracle import *  # noqa: F401,F403
