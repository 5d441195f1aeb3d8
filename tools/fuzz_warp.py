"""Randomised warp parity sweep (GPU vs oracle): random affine / perspective
matrices (near-identity, rotations + scales, strong tilts with W sign
changes), shapes with 16-byte-aligned and ragged rows (the staged TMA tile
paths and the direct paths), C in {1, 3, 4}, u8 / f32, borders, batches.
Affine and `exact=True` perspective must be bit-exact; the default u8
perspective within 1 LSB (the north-star gate). Prints the first failure and
exits 1, else the case count and the default perspective's off-by-one rate.

    python tools/fuzz_warp.py [--cases 500] [--seed 0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_12425_b200 as fv  # noqa: E402


def rand_affine(rng, w, h):
    th = np.deg2rad(rng.uniform(-180, 180) if rng.random() < 0.3 else rng.uniform(-35, 35))
    s = np.exp(rng.uniform(np.log(0.3), np.log(3.0))) if rng.random() < 0.4 else rng.uniform(0.8, 1.25)
    a = s * np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    c = np.array([(w - 1) / 2.0, (h - 1) / 2.0])
    b = c + rng.normal(0, 0.1 * max(w, h), 2) - a @ c
    return np.hstack([a, b[:, None]])


def rand_homography(rng, w, h):
    m = np.eye(3)
    m[:2] = rand_affine(rng, w, h)
    scale = rng.choice([1e-5, 1e-4, 1e-3, 5e-3])
    m[2, :2] = rng.normal(0, scale, 2)
    return m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=500)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    dev = "cuda:0"
    off = tot = 0
    for i in range(a.cases):
        c = int(rng.choice([1, 3, 4]))
        u8 = bool(rng.random() < 0.6)
        persp = bool(rng.random() < 0.5)
        es = 1 if u8 else 4
        if rng.random() < 0.6:  # 16-byte aligned rows: the staged TMA paths
            w = 16 * int(rng.integers(1, 40)) // np.gcd(16, c * es) * 1
            w = max(1, w)
        else:
            w = int(rng.integers(1, 500))
        h = int(rng.integers(1, 200))
        oh, ow = int(rng.integers(1, 200)), int(rng.integers(1, 500))
        n = int(rng.integers(1, 3))
        border = int(rng.integers(0, 256))
        b = border if u8 else border / 255.0
        src = (rng.integers(0, 256, (n, h, w, c), dtype=np.uint8) if u8
               else rng.random((n, h, w, c), dtype=np.float32))
        fwd = [rand_homography(rng, w, h) if persp else rand_affine(rng, w, h) for _ in range(n)]
        inv = [O.invert_homography(m) if persp else O.invert_affine(m) for m in fwd]
        s_t = torch.from_numpy(src).to(dev)
        dst = torch.zeros((n, oh, ow, c), dtype=s_t.dtype, device=dev)
        if persp:
            fv.warp_perspective(s_t, dst, np.stack(inv), border=b, inverse=True, exact=True)
        else:
            fv.warp_affine(s_t, dst, np.stack(inv), border=b, inverse=True)
        got = dst.cpu().numpy()
        refs = [(O.warp_perspective if persp else O.warp_affine)(src[k], inv[k], oh, ow, border=b) for k in range(n)]
        for k in range(n):
            if not np.array_equal(got[k], refs[k]):
                print(f"exact mismatch case {i}: persp={persp} u8={u8} c={c} src {w}x{h} dst {ow}x{oh} n={n}")
                return 1
        if persp and u8:
            fv.warp_perspective(s_t, dst, np.stack(inv), border=b, inverse=True)
            got = dst.cpu().numpy().astype(np.int16)
            for k in range(n):
                d = np.abs(got[k] - refs[k].astype(np.int16))
                if d.max() > 1:
                    print(f"fast persp > 1 LSB case {i}: c={c} src {w}x{h} dst {ow}x{oh}")
                    return 1
                off += int((d == 1).sum())
                tot += d.size
    print(f"ok {a.cases} cases; default u8 perspective: {off} of {tot} values off by one ({off / max(tot, 1):.2e})")
    return 0


if __name__ == "__main__":
    sys.exit(main())
