"""GPU-entropy JPEG decoding under repetition: batches of Pillow-encoded
frames (mixed sizes, qualities, subsampling, gray and colour, smooth and
noisy content) decoded again and again through the GPU entropy path and
compared bit for bit with the host entropy path -- a check for rare races in
the speculative/round passes, not a benchmark.
    python tools/jpeg_stress.py [--batches 40] [--n 48] [--seed 1]
"""
import argparse
import io as pyio
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from PIL import Image, ImageFile  # noqa: E402

ImageFile.MAXBLOCK = 1 << 24  # optimize=True encodes in one block

from paper_2505_12425_b200 import io as fio, synth  # noqa: E402


def frame(rng):
    w, h = int(rng.integers(16, 1400)), int(rng.integers(16, 900))
    a = synth.seeded_smooth_u8_image(w, h, 3, seed=int(rng.integers(1 << 30)))
    if rng.random() < 0.3:  # noisier content: longer codes, more AC symbols
        a = np.clip(a.astype(np.int32) + rng.integers(-40, 41, a.shape), 0, 255).astype(np.uint8)
    img = Image.fromarray(a if rng.random() < 0.85 else a[:, :, 0])
    kw = dict(quality=int(rng.integers(40, 101)), subsampling=int(rng.integers(0, 3)),
              optimize=bool(rng.random() < 0.3))  # optimised = per-image Huffman tables
    buf = pyio.BytesIO()
    img.save(buf, format="JPEG", **kw)
    return buf.getvalue()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=40)
    ap.add_argument("--n", type=int, default=48)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--repeat", type=int, default=3)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    bad = 0
    total = 0
    for b in range(a.batches):
        streams = [frame(rng) for _ in range(a.n)]
        ref = [o.cpu().numpy() for o in fio.decode_jpeg_batch(streams, entropy="host")]
        for _ in range(a.repeat):
            got = fio.decode_jpeg_batch(streams, entropy="gpu")
            torch.cuda.synchronize()
            for i, (g, r) in enumerate(zip(got, ref)):
                total += 1
                if not np.array_equal(g.cpu().numpy(), r):
                    bad += 1
                    print(f"MISMATCH batch {b} image {i}", flush=True)
    print(f"jpeg_stress: {total} decodes, {bad} mismatches, gpu entropy {fio.stats}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
