"""cfg3 perspective: per-image kernel time (one image per launch, after a 2 s soak)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2505_12425_b200 as fv
from paper_2505_12425_b200 import synth
dev = torch.device("cuda", 0)
n = 16
src = synth.device_u8_batch(n, 2160, 3840, 3, synth.SEED_PERSP, dev)
dst = torch.zeros_like(src)
hs = np.stack([synth.perspective_forward(synth.SEED_PERSP_PARAMS + i) for i in range(n)])
import time
t_end = time.time() + 2.0  # soak: clocks at their loaded state before timing
while time.time() < t_end:
    fv.warp_perspective(src, dst, hs)
    torch.cuda.synchronize()
for i in list(range(n)) * 2:
    for _ in range(3): fv.warp_perspective(src[i], dst[i], hs[i])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): fv.warp_perspective(src[i], dst[i], hs[i])
    e1.record(); torch.cuda.synchronize()
    print(i, round(e0.elapsed_time(e1) / 20, 4))
