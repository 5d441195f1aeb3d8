"""cfg2 affine: CUDA-event timing of the source-tiled kernel (default path)
and the destination-tiled TMA kernel (test build, warp path 4) on 32 x
1920x1080x3 f32 (inputs resident), plus their bit-equality.

    python tools/affine_perf.py [--reps 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_12425_b200 as fv  # noqa: E402
from paper_2505_12425_b200 import _native, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--u8", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = 32
    if a.u8:
        src = synth.device_u8_batch(n, 1080, 1920, 3, synth.SEED_AFFINE, dev)
    else:
        src = synth.device_f32_batch(n, 1080, 1920, 3, synth.SEED_AFFINE, dev)
    ms = np.stack([synth.affine_forward(synth.SEED_AFFINE_PARAMS + i, 1920, 1080) for i in range(n)])
    d_new, d_old = torch.zeros_like(src), torch.zeros_like(src)

    def old():
        _native.use_test_build(True)
        _native.lib().fv_set_warp_path(4)
        fv.warp_affine(src, d_old, ms)
        _native.lib().fv_set_warp_path(0)
        _native.use_test_build(False)

    runs = {"src_tiles": lambda: fv.warp_affine(src, d_new, ms), "dst_tiles_tma": old}
    for f in runs.values():
        for _ in range(3):
            f()
    torch.cuda.synchronize()
    for name, f in runs.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms_ = e0.elapsed_time(e1) / a.reps
        print(f"{name}: {ms_:.4f} ms / {n} images, {n * 1920 * 1080 / ms_ / 1e3:.0f} dst MP/s")
    same = torch.equal(d_new, d_old)
    print("bit-equal:", same)
    if not same:
        diff = (d_new.float() - d_old.float()).abs()
        print("max diff", float(diff.max()), "count", int((diff > 0).sum()))


if __name__ == "__main__":
    main()
