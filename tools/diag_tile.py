"""Quick check of the affine tile kernel: one small and one cfg2-size call,
timed, against the oracle on the small one (diagnostic, not a test)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_12425_b200 as fv
from paper_2505_12425_b200 import synth
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import fovea_oracle as O
dev = torch.device("cuda", 0)
a = np.random.default_rng(1).random((70, 160, 3), dtype=np.float32)
m = O.affine_forward(5, 160, 70)
d = torch.zeros((70, 160, 3), dtype=torch.float32, device=dev)
t = time.time(); fv.warp_affine(torch.from_numpy(a).to(dev), d, m); torch.cuda.synchronize(); print("small", time.time() - t, flush=True)
print("exact", np.array_equal(d.cpu().numpy(), O.warp_affine(a, O.invert_affine(m), 70, 160, border=0.0)), flush=True)
src = synth.device_f32_batch(32, 1080, 1920, 3, synth.SEED_AFFINE, dev)
dst = torch.zeros_like(src)
ms = np.stack([synth.affine_forward(synth.SEED_AFFINE_PARAMS + i, 1920, 1080) for i in range(32)])
for r in range(3):
    t = time.time(); fv.warp_affine(src, dst, ms); torch.cuda.synchronize(); print("cfg2", time.time() - t, flush=True)
