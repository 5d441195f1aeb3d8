"""Run one BASELINE config's kernel(s) a few times at full size -- the short
command that `ncu` wraps (see profiles/README.md). Not a benchmark: no timing.

    python tools/profile_ops.py --op resize|down|up|gray|graybatch|affine|persp|fused|jpeg [--reps 2] [--images N]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_12425_b200 as fv  # noqa: E402
from paper_2505_12425_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", default="resize")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--images", type=int, default=0)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    runs = []
    if a.op in ("resize", "down", "up"):
        n = a.images or 64
        src = synth.device_u8_batch(n, 2160, 3840, 3, synth.SEED_RESIZE, dev)
        if a.op in ("resize", "down"):
            down = torch.zeros((n, 1080, 1920, 3), dtype=torch.uint8, device=dev)
            runs.append(lambda: fv.resize_bilinear_u8(src, down))
        if a.op in ("resize", "up"):
            up = torch.zeros((n, 4320, 7680, 3), dtype=torch.uint8, device=dev)
            runs.append(lambda: fv.resize_bilinear_u8(src, up))
    elif a.op == "gray":
        n = a.images or 32
        src = synth.device_u8_batch(n, 1080, 1920, 3, synth.SEED_GRAY, dev)
        dst = torch.zeros((n, 1080, 1920, 1), dtype=torch.uint8, device=dev)
        runs.append(lambda: [fv.gray_from_rgb(src[i], dst[i]) for i in range(n)])
    elif a.op in ("r720", "r1080"):  # generic ratios: 1080p -> 720p, 720p -> 1080p (strip kernel)
        n = a.images or 128
        (sh, sw), (dh, dw) = ((1080, 1920), (720, 1280)) if a.op == "r720" else ((720, 1280), (1080, 1920))
        src = synth.device_u8_batch(n, sh, sw, 3, 1, dev)
        dst = torch.zeros((n, dh, dw, 3), dtype=torch.uint8, device=dev)
        runs.append(lambda: fv.resize_bilinear_u8(src, dst))
    elif a.op == "graybatch":  # the same 32 frames in one launch
        n = a.images or 32
        src = synth.device_u8_batch(n, 1080, 1920, 3, synth.SEED_GRAY, dev)
        dst = torch.zeros((n, 1080, 1920, 1), dtype=torch.uint8, device=dev)
        runs.append(lambda: fv.gray_from_rgb(src, dst))
    elif a.op == "affine":
        n = a.images or 32
        src = synth.device_f32_batch(n, 1080, 1920, 3, synth.SEED_AFFINE, dev)
        dst = torch.zeros_like(src)
        ms = np.stack([synth.affine_forward(synth.SEED_AFFINE_PARAMS + i, 1920, 1080) for i in range(n)])
        runs.append(lambda: fv.warp_affine(src, dst, ms))
    elif a.op == "persp":
        n = a.images or 16
        src = synth.device_u8_batch(n, 2160, 3840, 3, synth.SEED_PERSP, dev)
        dst = torch.zeros_like(src)
        hs = np.stack([synth.perspective_forward(synth.SEED_PERSP_PARAMS + i) for i in range(n)])
        runs.append(lambda: fv.warp_perspective(src, dst, hs))
    elif a.op == "fused":
        n = a.images or 512
        src = synth.device_u8_batch(n, 1080, 1920, 3, synth.SEED_FUSED, dev)
        dst = torch.zeros((n, 3, 640, 640), dtype=torch.float32, device=dev)
        runs.append(lambda: fv.resize_normalize_chw(src, dst, synth.MEAN, synth.STD))
    elif a.op == "jpeg":  # decode -> preprocess: GPU entropy decoding + reconstruction of 64 1080p JPEGs
        import bench
        from paper_2505_12425_b200 import io as fio

        n = a.images or 64
        streams = bench.jpeg_streams(0, n)
        frames = torch.empty((n, 1080, 1920, 3), dtype=torch.uint8, device=dev)
        dst = torch.empty((n, 3, 640, 640), dtype=torch.float32, device=dev)
        runs.append(lambda: (fio.decode_jpeg_batch(streams, dev, out=frames),
                             fv.resize_normalize_chw(frames, dst, synth.MEAN, synth.STD)))
    else:
        raise SystemExit(f"unknown op {a.op}")
    for _ in range(a.reps):
        for r in runs:
            r()
    torch.cuda.synchronize()
    print("ok", a.op)


if __name__ == "__main__":
    main()
