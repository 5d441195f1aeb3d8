import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_12425_b200 as fv
dev = "cuda:0"
sh, sw, dh, dw, n = [int(v) for v in sys.argv[1:6]]
src = torch.randint(0, 256, (n, sh, sw, 3), dtype=torch.uint8, device=dev)
dst = torch.empty((n, dh, dw, 3), dtype=torch.uint8, device=dev)
fv.resize_bilinear_u8(src, dst)
torch.cuda.synchronize()
print("ok")
