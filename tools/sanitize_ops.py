"""Small-shape launches of every staged (TMA / mbarrier) kernel for
compute-sanitizer (memcheck, racecheck, synccheck, initcheck), each checked
against the oracle so a sanitizer run also shows the results are right.

    compute-sanitizer --tool racecheck python tools/sanitize_ops.py

Kernels (shapes chosen to take each path): resize_down2_tma_kernel (2:1,
width multiple of 16), resize_up2_kernel (1:2), resize_strip_kernel HWC and
CHW (generic ratio, fused), warp_affine_tma_kernel (f32, u8), the
perspective tile kernel (border / staged / direct tiles), gray, flip,
nearest, sobel.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_12425_b200 as fv  # noqa: E402
from paper_2505_12425_b200 import synth  # noqa: E402


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check(name, got, ref, tol=0):
    torch.cuda.synchronize()
    d = np.abs(got.cpu().numpy().astype(np.float64) - ref.astype(np.float64)).max()
    status = "ok" if d <= tol else "MISMATCH"
    print(f"{status} {name} max|d|={d}")
    if d > tol:
        raise SystemExit(1)


def main():
    a = O.seeded_u8_image(128, 72, 3, seed=1)
    d = torch.zeros((36, 64, 3), dtype=torch.uint8, device="cuda")
    fv.resize_bilinear_u8(cu(a), d)
    check("resize_down2_tma", d, O.resize_u8(a, 64, 36))
    u = torch.zeros((144, 256, 3), dtype=torch.uint8, device="cuda")
    fv.resize_bilinear_u8(cu(a), u)
    check("resize_up2", u, O.resize_u8(a, 256, 144))
    g = torch.zeros((50, 90, 3), dtype=torch.uint8, device="cuda")
    fv.resize_bilinear_u8(cu(a), g)
    check("resize_strip u8 HWC", g, O.resize_u8(a, 90, 50))
    chw = torch.zeros((3, 40, 40), dtype=torch.float32, device="cuda")
    fv.resize_normalize_chw(cu(a), chw, synth.MEAN, synth.STD)
    check("resize_strip CHW (fused)", chw, O.resize_normalize_chw(a, 40, 40, synth.MEAN, synth.STD))
    f = O.seeded_f32_image(96, 64, 3, seed=2)
    m = O.affine_forward(3, 96, 64)
    wa = torch.zeros((64, 96, 3), dtype=torch.float32, device="cuda")
    fv.warp_affine(cu(f), wa, m)
    check("warp_affine_tma f32", wa, O.warp_affine(f, O.invert_affine(m), 64, 96))
    au = O.seeded_u8_image(96, 64, 3, seed=4)
    wu = torch.zeros((64, 96, 3), dtype=torch.uint8, device="cuda")
    fv.warp_affine(cu(au), wu, m)
    check("warp_affine_tma u8", wu, O.warp_affine(au, O.invert_affine(m), 64, 96))
    # perspective: a strong homography so border, staged and direct tiles all occur
    p = O.seeded_u8_image(320, 200, 3, seed=5)
    h = np.array([[1.0, 0.05, 5.0], [0.02, 0.9, -3.0], [0.0012, 0.0009, 1.0]])
    wp = torch.zeros((200, 320, 3), dtype=torch.uint8, device="cuda")
    fv.warp_perspective(cu(p), wp, h)
    check("warp_perspective tile kernel", wp, O.warp_perspective(p, O.invert_homography(h), 200, 320), tol=1)
    wpx = torch.zeros_like(wp)
    fv.warp_perspective(cu(p), wpx, h, exact=True)
    check("warp_perspective exact", wpx, O.warp_perspective(p, O.invert_homography(h), 200, 320))
    gr = torch.zeros((72, 128, 1), dtype=torch.uint8, device="cuda")
    fv.gray_from_rgb(cu(a), gr)
    check("gray", gr, O.gray_from_rgb(a))
    fl = torch.zeros_like(cu(a))
    fv.flip_horizontal(cu(a), fl)
    check("flip", fl, O.flip_horizontal(a))
    nn = torch.zeros((50, 90, 3), dtype=torch.uint8, device="cuda")
    fv.resize_nearest(cu(a), nn)
    check("nearest", nn, O.resize_nearest(a, 90, 50))
    so = torch.zeros((64, 96, 3), dtype=torch.float32, device="cuda")
    fv.sobel(cu(f), so, 3)
    check("sobel", so, O.sobel(f), tol=1e-5)
    print("all ok")


if __name__ == "__main__":
    main()
