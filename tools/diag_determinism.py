import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_12425_b200 as fv
dev = "cuda:0"
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
mode = sys.argv[2] if len(sys.argv) > 2 else "up"
g = torch.Generator(device=dev); g.manual_seed(7)
src = torch.randint(0, 256, (n, 2160, 3840, 3), dtype=torch.uint8, device=dev, generator=g)
shape = (n, 4320, 7680, 3) if mode == "up" else (n, 1080, 1920, 3)
a = torch.zeros(shape, dtype=torch.uint8, device=dev)
b = torch.full(shape, 7, dtype=torch.uint8, device=dev)
fv.resize_bilinear_u8(src, a)
fv.resize_bilinear_u8(src, b)
torch.cuda.synchronize()
diff = (a != b)
print(mode, "n", n, "mismatches", int(diff.sum().item()))
if diff.any():
    idx = diff.nonzero()
    print("first", idx[:10].tolist())
    print("images", torch.unique(idx[:, 0]).tolist()[:20], "rows", torch.unique(idx[:, 1]).tolist()[:20])
    print("cols", torch.unique(idx[:, 2]).tolist()[:40])
    i = idx[0].tolist()
    print("a", a[i[0], i[1], i[2]].tolist(), "b", b[i[0], i[1], i[2]].tolist())
