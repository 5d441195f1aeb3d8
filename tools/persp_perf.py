"""cfg3 perspective: CUDA-event timing of the exact and the <=1 LSB kernels
(16 x 3840x2160x3 u8, inputs resident), and the 1-LSB mismatch count of the
fast path against the exact kernel (which is bit-exact against the oracle).

    python tools/persp_perf.py [--reps 20]
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
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = 16
    src = synth.device_u8_batch(n, 2160, 3840, 3, synth.SEED_PERSP, dev)
    hs = np.stack([synth.perspective_forward(synth.SEED_PERSP_PARAMS + i) for i in range(n)])
    d_ex, d_fa, d_old = torch.zeros_like(src), torch.zeros_like(src), torch.zeros_like(src)
    from paper_2505_12425_b200 import _native

    def old():  # the round-1 kernel, through the test build's path knob
        _native.use_test_build(True)
        _native.lib().fv_set_warp_path(3)
        fv.warp_perspective(src, d_old, hs)
        _native.lib().fv_set_warp_path(0)
        _native.use_test_build(False)

    runs = {"exact": lambda: fv.warp_perspective(src, d_ex, hs, exact=True),
            "fast": lambda: fv.warp_perspective(src, d_fa, hs), "fast_r01": old}
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
        ms = e0.elapsed_time(e1) / a.reps
        print(f"{name}: {ms:.4f} ms / 16 images, {n * 3840 * 2160 / ms / 1e3:.0f} dst MP/s")
    for name, d in (("fast", d_fa), ("fast_r01", d_old)):
        diff = (d_ex.to(torch.int16) - d.to(torch.int16)).abs()
        print(f"{name} vs exact: max |diff| {int(diff.max())}, {int((diff > 0).sum())} of {diff.numel()} values differ")


if __name__ == "__main__":
    main()
