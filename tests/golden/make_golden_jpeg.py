"""Generate tests/golden/jpeg.npz: JPEG streams and what the REFERENCE
decoder (fovea.io.jpeg.decode_jpeg, /root/reference) makes of them.

Runs in the build container only (it imports the reference and Pillow); the
fixture it writes is what the CPU and GPU tests read. Streams:
  * the reference encoder (4:4:4 RGB and gray);
  * Pillow: 4:4:4 / 4:2:2 / 4:2:0 at q60/85/95 (the reference's
    test_matches_reference_decoder grid), grayscale, restart markers, odd
    sizes down to 1x1, noise at q95/q100 (long codes, large coefficients),
    progressive (must be rejected);
  * a 4:4:0 stream (luma 1x2) and a 16-bit-DQT stream with restart markers,
    assembled here from the reference encoder's own building blocks (Pillow
    cannot write either);
  * error streams (PNG bytes, truncations) and seeded byte mutations of a
    small stream, recording the reference's outcome (image or exception).

    python tests/golden/make_golden_jpeg.py
"""
import io
import os
import struct
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from PIL import Image as PILImage  # noqa: E402

from fovea.image import Image  # noqa: E402
from fovea.io import decode_jpeg, encode_jpeg, encode_png  # noqa: E402
from fovea.io import jpeg as J  # noqa: E402
from fovea.synth import seeded_smooth_u8_image  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "jpeg.npz")


def pil(arr, quality=85, **kw):
    b = io.BytesIO()
    PILImage.fromarray(arr).save(b, format="JPEG", quality=quality, **kw)
    return b.getvalue()


def smooth(w, h, c, seed):
    return seeded_smooth_u8_image(w, h, c, seed=seed).as_array()


def assembled(arr, quality, luma_hv, restart=0, q16=False):
    """Baseline stream with luma sampling `luma_hv` = (h, v) and 1x1 chroma,
    built from the reference encoder's helpers (DCT, quantiser, Huffman
    writer, standard tables); chroma is box-downsampled."""
    H, W = arr.shape[:2]
    hs, vs = luma_hv
    ycc = J._rgb_to_ycbcr(arr)
    planes = [ycc[:, :, 0]]
    for c in (1, 2):
        p = ycc[:, :, c]
        ph, pw = -(-H // vs) * vs, -(-W // hs) * hs
        p = np.pad(p, ((0, ph - H), (0, pw - W)), mode="edge")
        planes.append(p.reshape(ph // vs, vs, pw // hs, hs).mean(axis=(1, 3)))
    qts = [J._scaled_qtable(J._QUANT_LUMA, quality), J._scaled_qtable(J._QUANT_CHROMA, quality)]
    mcux, mcuy = -(-W // (8 * hs)), -(-H // (8 * vs))
    samp = [(hs, vs), (1, 1), (1, 1)]
    comp_blocks = []
    for ci, p in enumerate(planes):
        h, v = samp[ci]
        bw, bh = mcux * h, mcuy * v
        p = np.pad(p, ((0, bh * 8 - p.shape[0]), (0, bw * 8 - p.shape[1])), mode="edge")
        blocks = p.reshape(bh, 8, bw, 8).transpose(0, 2, 1, 3).reshape(-1, 8, 8)
        q = qts[min(ci, 1)].astype(np.float64)
        zz = J._round_half_away(J._blocks_dct(blocks - 128.0) / q).astype(np.int64).reshape(-1, 64)[:, J._ZIGZAG]
        comp_blocks.append((zz.tolist(), bw))
    out = bytearray(b"\xff\xd8")
    for tid, t in enumerate(qts):
        zz = t.reshape(-1)[J._ZIGZAG]
        out += J._marker(0xFFDB, bytes([0x10 | tid]) + zz.astype(">u2").tobytes() if q16
                         else bytes([tid]) + zz.astype(np.uint8).tobytes())
    sof = struct.pack(">BHHB", 8, H, W, 3)
    for ci in range(3):
        h, v = samp[ci]
        sof += bytes([ci + 1, (h << 4) | v, min(ci, 1)])
    out += J._marker(0xFFC0, sof)
    for tc, tid, spec in [(0, 0, J._DC_LUMA_SPEC), (1, 0, J._AC_LUMA_SPEC), (0, 1, J._DC_CHROMA_SPEC),
                          (1, 1, J._AC_CHROMA_SPEC)]:
        out += J._marker(0xFFC4, J._dht_payload(tc, tid, spec))
    if restart:
        out += J._marker(0xFFDD, struct.pack(">H", restart))
    sos = bytes([3]) + b"".join(bytes([ci + 1, (min(ci, 1) << 4) | min(ci, 1)]) for ci in range(3)) + bytes([0, 63, 0])
    out += J._marker(0xFFDA, sos)
    codes = [(J._canonical_codes(*J._DC_LUMA_SPEC), J._canonical_codes(*J._AC_LUMA_SPEC))] + \
            [(J._canonical_codes(*J._DC_CHROMA_SPEC), J._canonical_codes(*J._AC_CHROMA_SPEC))] * 2
    w = J._BitWriter()
    preds = [0, 0, 0]
    for m in range(mcux * mcuy):
        if restart and m and m % restart == 0:
            w.flush()
            out += w.out + bytes([0xFF, 0xD0 + ((m // restart - 1) & 7)])
            w = J._BitWriter()
            preds = [0, 0, 0]
        my, mx = divmod(m, mcux)
        for ci in range(3):
            h, v = samp[ci]
            zz, bw = comp_blocks[ci]
            for by in range(v):
                for bx in range(h):
                    preds[ci] = J._encode_block(w, zz[(my * v + by) * bw + mx * h + bx], preds[ci], *codes[ci])
    w.flush()
    out += w.out + b"\xff\xd9"
    return bytes(out)


def gray_from_coefficients(zz_blocks, width, height, q16):
    """Single-component baseline stream whose quantised zigzag coefficients
    are given directly (one list of 64 per block, raster order): reaches
    values no encoder produces -- DC beyond int16, dequantised products far
    beyond int32 -- which the reference decodes with Python ints."""
    bw, bh = -(-width // 8), -(-height // 8)
    assert len(zz_blocks) == bw * bh
    out = bytearray(b"\xff\xd8")
    out += J._marker(0xFFDB, bytes([0x10]) + np.array(q16, dtype=">u2").tobytes())
    out += J._marker(0xFFC0, struct.pack(">BHHB", 8, height, width, 1) + bytes([1, 0x11, 0]))
    out += J._marker(0xFFC4, J._dht_payload(0, 0, J._DC_LUMA_SPEC))
    # AC table with every run/size symbol 0x00..0xFF so any value is codable
    ac_vals = list(range(256))
    ac_bits = [0] * 7 + [128, 128] + [0] * 7
    out += J._marker(0xFFC4, J._dht_payload(1, 0, (ac_bits, ac_vals)))
    out += J._marker(0xFFDA, bytes([1, 1, 0x00, 0, 63, 0]))
    dc = J._canonical_codes(*J._DC_LUMA_SPEC)
    ac = J._canonical_codes(ac_bits, ac_vals)
    w = J._BitWriter()
    pred = 0
    for zz in zz_blocks:
        pred = J._encode_block(w, zz, pred, dc, ac)
    w.flush()
    out += w.out + b"\xff\xd9"
    return bytes(out)


def main():
    cases = {}
    cases["ref444_q90"] = encode_jpeg(Image.from_array(smooth(64, 48, 3, 21)), 90)
    cases["ref_gray_q92"] = encode_jpeg(Image.from_array(smooth(25, 18, 1, 5)), 92)
    cases["ref444_q1"] = encode_jpeg(Image.from_array(smooth(8, 8, 3, 0)), 1)
    cases["ref444_q100"] = encode_jpeg(Image.from_array(smooth(8, 8, 3, 0)), 100)
    arr = smooth(129, 77, 3, 13)
    for ss in (0, 1, 2):
        for q in (60, 85, 95):
            cases[f"pil_ss{ss}_q{q}"] = pil(arr, q, subsampling=ss)
    cases["pil_photo_256"] = pil(smooth(256, 192, 3, 99), 85, subsampling=2)
    g = smooth(40, 30, 1, 3)[:, :, 0]
    b = io.BytesIO()
    PILImage.fromarray(g, mode="L").save(b, format="JPEG", quality=90)
    cases["pil_gray"] = b.getvalue()
    cases["pil_restart"] = pil(smooth(80, 64, 3, 17), 80, restart_marker_blocks=2)
    cases["pil_restart_420"] = pil(smooth(83, 61, 3, 18), 75, subsampling=2, restart_marker_blocks=3)
    for w, h in [(1, 1), (3, 5), (17, 9), (33, 31), (2, 40), (40, 2)]:
        cases[f"pil_odd_{w}x{h}"] = pil(smooth(w, h, 3, w * h), 90, subsampling=2)
    cases["pil_odd_422_5x7"] = pil(smooth(5, 7, 3, 35), 90, subsampling=1)
    noise = np.random.default_rng(7).integers(0, 256, (48, 72, 3), dtype=np.uint8)
    cases["pil_noise_q95_420"] = pil(noise, 95, subsampling=2)
    cases["pil_noise_q100_444"] = pil(noise, 100, subsampling=0)
    cases["asm_440_q85"] = assembled(smooth(45, 38, 3, 44), 85, (1, 2))
    cases["asm_440_2px"] = assembled(smooth(3, 2, 3, 45), 85, (1, 2))
    cases["asm_420_q16_rst"] = assembled(smooth(50, 34, 3, 46), 70, (2, 2), restart=3, q16=True)
    cases["asm_422_rst1"] = assembled(smooth(33, 17, 3, 47), 90, (2, 1), restart=1)
    # adversarial coefficients (what the int64 paths are for)
    blocks = []
    for k in range(24):  # DC ramps past int16 in steps of 2047 (the largest DC difference)
        zz = [0] * 64
        zz[0] = 2047 * k
        zz[1 + k % 5] = (-1) ** k * (1000 + 37 * k)
        blocks.append(zz)
    cases["asm_gray_dc_int16_overflow"] = gray_from_coefficients(blocks, 192, 8, [1] * 64)
    blocks = []
    rng_c = np.random.default_rng(11)
    for k in range(12):  # |AC| up to 32767 dequantised by 65535: IDCT products ~1e13
        zz = [int(v) for v in rng_c.integers(-32767, 32768, 64)]
        zz[0] = int(rng_c.integers(-1000, 1000))  # DC differences must stay codable (size <= 11)
        blocks.append(zz)
    cases["asm_gray_extreme_q16"] = gray_from_coefficients(blocks, 31, 20, [65535] * 64)
    # error streams
    cases["err_png"] = encode_png(Image.from_array(np.zeros((4, 4, 3), np.uint8)))
    cases["err_progressive"] = pil(smooth(32, 32, 3, 2), 85, progressive=True)
    base = pil(smooth(32, 32, 3, 2), 85)
    cases["err_truncated_half"] = base[: len(base) // 2]
    cases["err_empty"] = b""
    cases["err_soi_only"] = b"\xff\xd8"
    # seeded mutations / truncations of a small stream: whatever the reference does
    small = encode_jpeg(Image.from_array(smooth(24, 24, 3, 4)), 80)
    rng = np.random.default_rng(2024)
    for k in range(48):
        d = bytearray(small)
        for _ in range(int(rng.integers(1, 6))):
            d[int(rng.integers(0, len(d)))] = int(rng.integers(0, 256))
        cases[f"fuzz_mut_{k:02d}"] = bytes(d)
    for k, cut in enumerate(rng.integers(0, len(small), size=16)):
        cases[f"fuzz_cut_{k:02d}"] = small[: int(cut)]

    store = {}
    for name, data in cases.items():
        store[f"{name}__jpg"] = np.frombuffer(data, np.uint8)
        try:
            store[f"{name}__out"] = decode_jpeg(data).as_array()
        except Exception as e:  # noqa: BLE001 -- recording the reference's behaviour
            store[f"{name}__err"] = np.array(type(e).__name__)
    np.savez_compressed(OUT, **store)
    n_err = sum(1 for k in store if k.endswith("__err"))
    print(f"wrote {OUT}: {len(cases)} streams, {n_err} rejected")


if __name__ == "__main__":
    main()
