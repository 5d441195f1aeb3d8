"""Per-launch CUDA-event timing of the resize kernels in different
sequences (diagnostic for order effects)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_12425_b200 as fv  # noqa: E402
from paper_2505_12425_b200 import synth  # noqa: E402

dev = torch.device("cuda", 0)
n = 64
src = synth.device_u8_batch(n, 2160, 3840, 3, 1, dev)
down = torch.zeros((n, 1080, 1920, 3), dtype=torch.uint8, device=dev)
up = torch.zeros((n, 4320, 7680, 3), dtype=torch.uint8, device=dev)
junk = torch.zeros(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
F = {"d": lambda: fv.resize_bilinear_u8(src, down), "u": lambda: fv.resize_bilinear_u8(src, up),
     "z": lambda: junk.fill_(1), "r": lambda: junk.sum()}


def run(seq, label):
    s = torch.cuda.current_stream()
    for c in seq:
        F[c]()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in seq]
    for (a, b), c in zip(ev, seq):
        a.record(s)
        F[c]()
        b.record(s)
    torch.cuda.synchronize()
    print(label, " ".join(f"{c}:{a.elapsed_time(b):.3f}" for (a, b), c in zip(ev, seq)))


run("ddddd", "down x5      ")
run("ududud", "up/down      ")
run("zdzdzd", "fill256MB/down")
run("rdrdrd", "read256MB/down")
run("uuu", "up x3        ")
run("dudu", "down/up      ")
time.sleep(0.2)
run("d", "after sleep  ")


def outer(seq, label, marker=False):
    s = torch.cuda.current_stream()
    for c in seq:
        F[c]()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event() for _ in seq]
    e0.record(s)
    for c, m in zip(seq, marks):
        F[c]()
        if marker:
            m.record(s)
    e1.record(s)
    torch.cuda.synchronize()
    print(label, f"total {e0.elapsed_time(e1):.3f} ms for {seq}")


outer("ddddd", "outer only     ")
outer("ddddd", "outer + markers", marker=True)
outer("ududud", "outer u/d      ")
outer("uuu", "outer u        ")
run("ddddd", "per-launch ev  ")
