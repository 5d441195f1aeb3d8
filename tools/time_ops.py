"""Quick CUDA-event timing of single kernels, alone and interleaved.

    python tools/time_ops.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_12425_b200 as fv  # noqa: E402
from paper_2505_12425_b200 import synth  # noqa: E402


def timeit(fns, reps=10):
    s = torch.cuda.current_stream()
    for f in fns:
        f()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in fns]
    tot = [0.0] * len(fns)
    for _ in range(reps):
        for i, f in enumerate(fns):
            evs[i][0].record(s)
            f()
            evs[i][1].record(s)
        torch.cuda.synchronize()
        for i in range(len(fns)):
            tot[i] += evs[i][0].elapsed_time(evs[i][1])
    return [t / reps for t in tot]


def main():
    dev = torch.device("cuda", 0)
    n = 64
    src = synth.device_u8_batch(n, 2160, 3840, 3, 1, dev)
    down = torch.zeros((n, 1080, 1920, 3), dtype=torch.uint8, device=dev)
    up = torch.zeros((n, 4320, 7680, 3), dtype=torch.uint8, device=dev)
    fd = lambda: fv.resize_bilinear_u8(src, down)  # noqa: E731
    fu = lambda: fv.resize_bilinear_u8(src, up)  # noqa: E731
    gb_d = (src.numel() + down.numel()) / 1e9
    gb_u = (src.numel() + up.numel()) / 1e9
    for name, fns in [("down alone", [fd]), ("up alone", [fu]), ("down,up", [fd, fu])]:
        t = timeit(fns)
        print(name, ["%.3f ms" % x for x in t], ["%.0f GB/s" % (g / (x / 1e3)) for g, x in zip([gb_d, gb_u] if name != "up alone" else [gb_u], t)])
    # host launch overhead: time 20 back-to-back launches of down
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(20):
        fd()
    e1.record(s)
    torch.cuda.synchronize()
    print("down back-to-back avg %.3f ms" % (e0.elapsed_time(e1) / 20))


if __name__ == "__main__":
    main()
