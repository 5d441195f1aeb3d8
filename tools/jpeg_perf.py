"""decode -> preprocess timing probe (not a benchmark): N seeded smooth
1080p frames encoded by Pillow (q90, 4:2:0) on the box, then
  host entropy decoding: one thread per image, T threads;
  H2D of the coefficients; the two GPU kernels; the whole decode_jpeg_batch;
  decode -> resize_normalize_chw (640x640).
    python tools/jpeg_perf.py [--n 64] [--threads 16]
"""
import argparse
import io as pyio
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from PIL import Image  # noqa: E402

import paper_2505_12425_b200 as fv
import synth_fixtures  # noqa: E402
from paper_2505_12425_b200 import io as fio, synth  # noqa: E402
from concurrent.futures import ThreadPoolExecutor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--w", type=int, default=1920)
    ap.add_argument("--h", type=int, default=1080)
    a = ap.parse_args()
    t = time.time()
    streams = []
    for i in range(a.n):
        b = pyio.BytesIO()
        Image.fromarray(synth_fixtures.seeded_smooth_u8_image(a.w, a.h, 3, seed=70000 + i)).save(b, "JPEG", quality=90, subsampling=2)
        streams.append(b.getvalue())
    print(f"encode {time.time() - t:.1f}s, mean stream {np.mean([len(s) for s in streams]) / 1e3:.0f} KB, cores {a.threads}")
    dev = torch.device("cuda", 0)
    fio.decode_jpeg(streams[0])
    torch.cuda.synchronize()
    # host entropy decoding
    infos = [fio.jpeg_info(s) for s in streams]
    bufs = [torch.empty(int(i.coef_count), dtype=torch.int16, pin_memory=True) for i in infos]
    lib = fv._native.lib()
    t = time.perf_counter()
    for s, i, b in zip(streams, infos, bufs):
        assert lib.fv_jpeg_decode_coeffs(s, len(s), b.data_ptr(), b.numel(), 2) == 0
    t1 = (time.perf_counter() - t) / a.n
    mb = np.mean([len(s) for s in streams]) / 1e6
    print(f"host entropy 1 thread: {t1 * 1e3:.2f} ms/img  ({mb / t1:.0f} MB/s compressed, {a.w * a.h / t1 / 1e6:.0f} MP/s)")
    with ThreadPoolExecutor(a.threads) as ex:
        t = time.perf_counter()
        list(ex.map(lambda z: lib.fv_jpeg_decode_coeffs(z[0], len(z[0]), z[2].data_ptr(), z[2].numel(), 2),
                    zip(streams, infos, bufs)))
        tT = (time.perf_counter() - t) / a.n
    print(f"host entropy {a.threads} threads: {tT * 1e3:.2f} ms/img  ({a.w * a.h / tT / 1e6:.0f} MP/s)")
    # device stages
    coef = [b.to(dev) for b in bufs]
    planes = [torch.empty(int(i.plane_bytes), dtype=torch.uint8, device=dev) for i in infos]
    outs = [torch.empty((i.height, i.width, 3), dtype=torch.uint8, device=dev) for i in infos]
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(2):
        e0.record(st)
        for i, c, p, o in zip(infos, coef, planes, outs):
            lib.fv_jpeg_reconstruct(torch.ctypes_ptr if False else __import__("ctypes").byref(i), c.data_ptr(), 2,
                                    p.data_ptr(), o.data_ptr(), o.stride(0), st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
    tk = e0.elapsed_time(e1) / a.n
    print(f"GPU IDCT+colour: {tk * 1e3:.1f} us/img  ({a.w * a.h / (tk / 1e3) / 1e6:.0f} MP/s)")
    e0.record(st)
    for b in bufs:
        b.to(dev, non_blocking=True)
    e1.record(st)
    torch.cuda.synchronize()
    th = e0.elapsed_time(e1) / a.n
    print(f"H2D coefficients: {th * 1e3:.1f} us/img ({bufs[0].numel() * 2 / 1e6:.1f} MB)")
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        imgs = fio.decode_jpeg_batch(streams, threads=a.threads)
        dst = torch.empty((a.n, 3, 640, 640), dtype=torch.float32, device=dev)
        for k, im in enumerate(imgs):
            fv.resize_normalize_chw(im, dst[k], synth.MEAN, synth.STD)
        torch.cuda.synchronize()
        tb = time.perf_counter() - t
    print(f"decode_jpeg_batch + preprocess: {tb * 1e3:.1f} ms for {a.n} ({a.n / tb:.0f} img/s, {a.n * a.w * a.h / tb / 1e6:.0f} MP/s)")


if __name__ == "__main__":
    main()
