import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_12425_b200 as fv
DEV = "cuda:0"
variant = sys.argv[1]
n = 64
g = torch.Generator(device=DEV); g.manual_seed(7)
up = torch.zeros((n, 4320, 7680, 3), dtype=torch.uint8, device=DEV)
if variant in ("const", "const_sync"):
    vals = torch.tensor([(37 * i + 11) % 256 for i in range(n)], dtype=torch.uint8, device=DEV)
    csrc = vals.view(n, 1, 1, 1).expand(n, 2160, 3840, 3).contiguous()
    fv.resize_bilinear_u8(csrc, up)
    if variant == "const_sync":
        torch.cuda.synchronize()
    del csrc
src = torch.randint(0, 256, (n, 2160, 3840, 3), dtype=torch.uint8, device=DEV, generator=g)
outs = []
for r in range(3):
    o = torch.full((n, 4320, 7680, 3), 9, dtype=torch.uint8, device=DEV) if r else up
    fv.resize_bilinear_u8(src, o)
    outs.append(o)
torch.cuda.synchronize()
print(variant, [int((outs[0] != o).sum()) for o in outs[1:]], int((outs[1] != outs[2]).sum()))
