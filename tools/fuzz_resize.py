"""Randomised resize parity sweep (GPU vs oracle) beyond the hypothesis test's
example budget: random shapes, channel counts, batch sizes, crop views and
forced paths (auto / gather / strip) for u8 HWC, f32 HWC and the fused CHW
mode. Prints the first mismatch and exits 1, else the case count.

    python tools/fuzz_resize.py [--cases 2000] [--seed 0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_12425_b200 as fv  # noqa: E402
from _helpers import forced_path  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=2000)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    dev = "cuda:0"
    for i in range(a.cases):
        big = rng.random() < 0.15
        sw, sh = int(rng.integers(1, 2200 if big else 300)), int(rng.integers(1, 24 if big else 60))
        dw, dh = int(rng.integers(1, 2200 if big else 300)), int(rng.integers(1, 24 if big else 60))
        if rng.random() < 0.2:  # exact 2:1 / 1:2 shapes
            if rng.random() < 0.5:
                dw, dh = max(1, sw // 2), max(1, sh // 2)
                sw, sh = 2 * dw, 2 * dh
            else:
                dw, dh = 2 * sw, 2 * sh
        c = int(rng.choice([1, 2, 3, 4]))
        n = int(rng.integers(1, 3))
        path = int(rng.integers(0, 3))
        ox = int(rng.integers(0, 3)) if rng.random() < 0.3 else 0
        parent = rng.integers(0, 256, (n, sh, sw + ox, c), dtype=np.uint8)
        src_np = parent[:, :, ox:]
        with forced_path("resize", path):
            src = torch.from_numpy(parent).to(dev)[:, :, ox:]
            du = torch.zeros((n, dh, dw, c), dtype=torch.uint8, device=dev)
            fv.resize_bilinear_u8(src, du)
            dc = torch.zeros((n, c, dh, dw), dtype=torch.float32, device=dev)
            mean, std = [0.3] * c, [0.2] * c
            fv.resize_normalize_chw(src, dc, mean, std)
            ou, oc = du.cpu().numpy(), dc.cpu().numpy()
        for k in range(n):
            ref = O.resize_u8(np.ascontiguousarray(src_np[k]), dw, dh)
            if not np.array_equal(ou[k], ref):
                print(f"u8 mismatch case {i}: src {sw}x{sh} dst {dw}x{dh} c={c} n={n} path={path} ox={ox}")
                return 1
            refc = O.resize_normalize_chw(np.ascontiguousarray(src_np[k]), dw, dh, mean, std)
            if not np.array_equal(oc[k], refc):
                print(f"chw mismatch case {i}: src {sw}x{sh} dst {dw}x{dh} c={c} n={n} path={path} ox={ox}")
                return 1
    print(f"ok {a.cases} cases")
    return 0


if __name__ == "__main__":
    sys.exit(main())
