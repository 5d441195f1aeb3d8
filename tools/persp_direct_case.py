"""All-direct perspective case for profiling: 2x zoom-out (every 128x32 tile's
source box exceeds the staging window), 16 x 3840x2160x3 -> 1920x1080x3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_12425_b200 as fv  # noqa: E402
from paper_2505_12425_b200 import synth  # noqa: E402

dev = torch.device("cuda", 0)
src = synth.device_u8_batch(16, 2160, 3840, 3, synth.SEED_PERSP, dev)
dst = torch.zeros((16, 1080, 1920, 3), dtype=torch.uint8, device=dev)
hs = np.stack([np.array([[0.5, 0, 0], [0, 0.5, 0], [1e-10, 1e-10, 1.0]])] * 16)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for _ in range(2):
    fv.warp_perspective(src, dst, hs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    fv.warp_perspective(src, dst, hs)
e1.record()
torch.cuda.synchronize()
print(f"direct 2x zoom-out: {e0.elapsed_time(e1) / reps:.4f} ms")
