import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2505_12425_b200 as fv
DEV="cuda:0"
n = 64
vals = torch.tensor([(37 * i + 11) % 256 for i in range(n)], dtype=torch.uint8, device=DEV)
src = vals.view(n, 1, 1, 1).expand(n, 2160, 3840, 3).contiguous()
down = torch.zeros((n, 1080, 1920, 3), dtype=torch.uint8, device=DEV)
up = torch.zeros((n, 4320, 7680, 3), dtype=torch.uint8, device=DEV)
fv.resize_bilinear_u8(src, down)
fv.resize_bilinear_u8(src, up)
torch.cuda.synchronize()
g = torch.Generator(device=DEV)
g.manual_seed(7)
src = torch.randint(0, 256, (n, 2160, 3840, 3), dtype=torch.uint8, device=DEV, generator=g)
fv.resize_bilinear_u8(src, up)
c1 = up.view(-1).to(torch.int64).sum().item()
up2 = torch.empty_like(up)
fv.resize_bilinear_u8(src, up2)
torch.cuda.synchronize()
d = (up != up2)
print("mismatch", int(d.sum()), "c1", c1, "c2", up2.view(-1).to(torch.int64).sum().item())
if d.any():
    idx = d.nonzero()
    print(idx[:5].tolist(), torch.unique(idx[:,0]).tolist()[:10], torch.unique(idx[:,1]).tolist()[:10], torch.unique(idx[:,2]).tolist()[:10])
if d.any():
    import numpy as np
    sys.path.insert(0, os.getcwd())
    import oracle as O
    img = int(idx[0, 0])
    rows = torch.unique(idx[idx[:, 0] == img][:, 1]).tolist()
    a = src[img].cpu().numpy()
    for r in rows[:6]:
        ref = O.resize_u8(a, 7680, 4320, rows=(r, r + 1))[0]
        u1 = up[img, r].cpu().numpy(); u2 = up2[img, r].cpu().numpy()
        cols = torch.unique(idx[(idx[:, 0] == img) & (idx[:, 1] == r)][:, 2]).tolist()
        print("row", r, "cols", cols[0], "..", cols[-1], len(cols), "run1 ok", bool((u1 == ref).all()), "run2 ok", bool((u2 == ref).all()))
