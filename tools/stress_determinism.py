"""Run each TMA-ring kernel many times on the same input with other work
interleaved and report any run that differs from the first (race hunting)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_12425_b200 as fv
from paper_2505_12425_b200 import synth
dev = "cuda:0"
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g = torch.Generator(device=dev); g.manual_seed(7)
n = 16
src = torch.randint(0, 256, (n, 2160, 3840, 3), dtype=torch.uint8, device=dev, generator=g)
f_src = torch.randint(0, 256, (64, 1080, 1920, 3), dtype=torch.uint8, device=dev, generator=g)
junk = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
cases = {
  "up2": (lambda d: fv.resize_bilinear_u8(src, d), (n, 4320, 7680, 3), torch.uint8),
  "down2": (lambda d: fv.resize_bilinear_u8(src, d), (n, 1080, 1920, 3), torch.uint8),
  "fused": (lambda d: fv.resize_normalize_chw(f_src, d, synth.MEAN, synth.STD), (64, 3, 640, 640), torch.float32),
}
for name, (fn, shape, dt) in cases.items():
    ref = torch.zeros(shape, dtype=dt, device=dev)
    fn(ref)
    bad = 0
    for r in range(reps):
        out = torch.full(shape, 3, dtype=dt, device=dev)
        if r % 2:
            junk.random_(generator=g)   # vary timing / L2 state
        fn(out)
        torch.cuda.synchronize()
        m = int((out != ref).sum())
        if m:
            bad += 1
            print(name, "rep", r, "mismatches", m)
    print(name, "bad runs", bad, "of", reps)
