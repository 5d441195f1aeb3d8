"""Throughput of the generic (strip) u8 resize path on common non-integer ratios."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_12425_b200 as fv
from paper_2505_12425_b200 import _native
dev = "cuda:0"
cases = [((2160, 3840), (1080, 1920), 64, 2), ((2160, 3840), (1080, 1920), 64, 0), ((1080, 1920), (720, 1280), 128, 0),
         ((720, 1280), (1080, 1920), 128, 0), ((1080, 1920), (640, 640), 256, 0), ((1080, 1920), (224, 224), 512, 0)]
for (sh, sw), (dh, dw), n, path in cases:
    _native.use_test_build(True)  # the path knob lives in the test build only
    _native.lib().fv_set_resize_path(path)
    src = torch.randint(0, 256, (n, sh, sw, 3), dtype=torch.uint8, device=dev)
    dst = torch.empty((n, dh, dw, 3), dtype=torch.uint8, device=dev)
    for _ in range(3): fv.resize_bilinear_u8(src, dst)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): fv.resize_bilinear_u8(src, dst)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    gb = (src.numel() + dst.numel()) / 1e9
    print(f"{sw}x{sh}->{dw}x{dh} n={n} path={path}: {ms:.3f} ms, {gb/ms*1e3:.0f} GB/s ({gb/ms*1e3/6538:.2f} of peak)")
_native.lib().fv_set_resize_path(0)
