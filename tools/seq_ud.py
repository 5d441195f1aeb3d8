import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_12425_b200 as fv
from paper_2505_12425_b200 import synth
dev = torch.device("cuda", 0)
n = 64
src = synth.device_u8_batch(n, 2160, 3840, 3, 1, dev)
down = torch.zeros((n, 1080, 1920, 3), dtype=torch.uint8, device=dev)
up = torch.zeros((n, 4320, 7680, 3), dtype=torch.uint8, device=dev)
seq = sys.argv[1] if len(sys.argv) > 1 else "udud"
for c in seq:
    fv.resize_bilinear_u8(src, down if c == "d" else up)
torch.cuda.synchronize()
print("ok")
