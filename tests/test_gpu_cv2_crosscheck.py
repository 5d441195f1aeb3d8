"""Independent cross-check of the warp contract against OpenCV.

The reference has no warps: the kernels and the oracle
share the builder's contract, so a convention error common to
both (matrix direction, pixel-centre origin, border rule) would pass the
parity tests. OpenCV's `warpAffine` / `warpPerspective` with WARP_INVERSE_MAP,
INTER_LINEAR and BORDER_CONSTANT implement the same convention (dst -> src
matrix, pixel centres at integer coordinates, per-tap constant border), but
quantise the sub-pixel position to 1/32 px (INTER_BITS = 5) and, for u8,
blend in fixed point. So the comparison is loose and runs on smooth images,
where a 1/64 px position error moves a value by far less than the tolerance:
u8 <= 2 LSB, f32 <= 5e-3 (values in [0, 1]; the oracle itself is within 1 LSB and
3.1e-3 of OpenCV on these cases), over the pixels whose four taps
are all inside the source (OpenCV's border handling of partially-outside
pixels differs only in that quantisation, but interior pixels are the
convention test).
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2505_12425_b200 as fv
import synth_fixtures
from paper_2505_12425_b200 import synth

cv2 = pytest.importorskip("cv2")
pytestmark = pytest.mark.gpu

H, W = 96, 128


def _smooth(seed, dtype):
    a = synth_fixtures.seeded_smooth_u8_image(W, H, 3, seed=seed)
    return a if dtype == np.uint8 else (a.astype(np.float32) / np.float32(255.0))


def _interior(inv, persp):
    y, x = np.mgrid[0:H, 0:W].astype(np.float64)
    if persp:
        w = inv[2, 0] * x + inv[2, 1] * y + inv[2, 2]
        sx = (inv[0, 0] * x + inv[0, 1] * y + inv[0, 2]) / w
        sy = (inv[1, 0] * x + inv[1, 1] * y + inv[1, 2]) / w
    else:
        sx = inv[0, 0] * x + inv[0, 1] * y + inv[0, 2]
        sy = inv[1, 0] * x + inv[1, 1] * y + inv[1, 2]
    return (sx >= 0.05) & (sx <= W - 1.05) & (sy >= 0.05) & (sy <= H - 1.05)


MATS = {
    "affine_rot_scale": (False, np.array([[0.95 * np.cos(0.3), -0.95 * np.sin(0.3), 12.0],
                                          [0.95 * np.sin(0.3), 0.95 * np.cos(0.3), -7.5]])),
    "affine_cfg2_like": (False, O.affine_forward(31003, W, H)),
    "persp_mild": (True, np.array([[1.02, 0.03, -4.0], [-0.02, 0.97, 3.0], [4e-4, -3e-4, 1.0]])),
    "persp_strong": (True, np.array([[0.9, 0.1, 6.0], [0.05, 1.1, -2.0], [2e-3, 1e-3, 1.0]])),
}


@pytest.mark.parametrize("dtype", [np.uint8, np.float32])
@pytest.mark.parametrize("name", sorted(MATS))
def test_warps_match_opencv_on_interior_pixels(name, dtype):
    persp, fwd = MATS[name]
    a = _smooth(7, dtype)
    full = np.eye(3)
    full[: 3 if persp else 2] = fwd
    inv = np.linalg.inv(full)
    dst = torch.zeros((H, W, 3), dtype=torch.uint8 if dtype == np.uint8 else torch.float32, device="cuda")
    src = torch.from_numpy(a).cuda()
    flags = cv2.INTER_LINEAR | cv2.WARP_INVERSE_MAP
    if persp:
        fv.warp_perspective(src, dst, fwd, border=0, exact=True)
        ref = cv2.warpPerspective(a, inv, (W, H), flags=flags, borderMode=cv2.BORDER_CONSTANT, borderValue=0)
    else:
        fv.warp_affine(src, dst, fwd, border=0)
        ref = cv2.warpAffine(a, inv[:2], (W, H), flags=flags, borderMode=cv2.BORDER_CONSTANT, borderValue=0)
    got = dst.cpu().numpy()
    mask = _interior(inv, persp)
    assert mask.mean() > 0.3  # the check covers a real share of the frame
    diff = np.abs(got.astype(np.float64) - ref.astype(np.float64))[mask]
    tol = 2.0 if dtype == np.uint8 else 5e-3
    assert diff.max() <= tol, f"{name} {dtype.__name__}: max |ours - OpenCV| = {diff.max()}"
    # and the default (<= 1 LSB) u8 perspective path agrees with OpenCV too
    if persp and dtype == np.uint8:
        fv.warp_perspective(src, dst, fwd, border=0)
        d2 = np.abs(dst.cpu().numpy().astype(np.float64) - ref.astype(np.float64))[mask]
        assert d2.max() <= tol + 1
