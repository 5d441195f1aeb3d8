"""Perspective tile kernel cost per tile class: a 16-image 4K batch where
every tile is border (map far outside), staged interior at scale 1
(identity + tiny tilt), staged zoom-out x0.25, and direct (zoom-in x2.5),
against cfg3's own homographies."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_12425_b200 as fv  # noqa: E402
from paper_2505_12425_b200 import synth  # noqa: E402

dev = torch.device("cuda", 0)
n = 16
src = synth.device_u8_batch(n, 2160, 3840, 3, synth.SEED_PERSP, dev)
dst = torch.zeros_like(src)
cases = {
    "cfg3": np.stack([synth.perspective_forward(synth.SEED_PERSP_PARAMS + i) for i in range(n)]),
    "border": np.stack([np.array([[1.0, 0, 1e5], [0, 1.0, 0], [0, 0, 1.0]])] * n),
    "staged_scale1": np.stack([np.array([[1.0, 1e-4, 0.3], [-1e-4, 1.0, 0.2], [1e-9, 1e-9, 1.0]])] * n),
    "zoomout_x0.25": np.stack([np.array([[4.0, 0, 0], [0, 4.0, 0], [1e-9, 1e-9, 1.0]])] * n),
    "zoomin_x2.5": np.stack([np.array([[0.4, 0, 0], [0, 0.4, 0], [1e-9, 1e-9, 1.0]])] * n),
}
t_end = time.time() + 2.0
while time.time() < t_end:
    fv.warp_perspective(src, dst, cases["cfg3"])
    torch.cuda.synchronize()
for name, hs in cases.items():
    for _ in range(3):
        fv.warp_perspective(src, dst, hs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fv.warp_perspective(src, dst, hs)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 20:.4f} ms")
