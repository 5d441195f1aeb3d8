"""CPU restatement of the reference's baseline JPEG decoder -- TEST
INFRASTRUCTURE ONLY (the checker for the GPU decode path; never imported by
the product).

Follows `fovea.io.jpeg.decode_jpeg` (/root/reference/pkg/src/fovea/io/
jpeg.py:605-806) step by step:

  * marker walk, table parsing and every error it raises (jpeg.py:605-735);
  * scan unstuffing and the split at restart markers (jpeg.py:574-602);
  * canonical Huffman decoding, DC prediction, AC run/size symbols (EOB for
    any size-0 symbol other than ZRL; ZRL may run past the block end
    silently) (jpeg.py:255-409), with the rule that a segment may not consume
    any bit past its real data (jpeg.py:777-780: `padded * 8 > nbits`);
  * dequantisation in natural order, the 13-bit fixed-point "islow" IDCT with
    its two descales and the final clip (jpeg.py:142-203, 783-790);
  * crop of each plane to its component size, the integer triangle chroma
    upsamplers (jpeg.py:809-841), crop to the image, and the 16-bit
    fixed-point YCbCr -> RGB (jpeg.py:226-235).

All arithmetic is Python/NumPy int64, like the reference. Parity pinned by
tests/golden/jpeg.npz: streams from the reference encoder and from Pillow,
decoded by the reference itself (tests/golden/make_golden_jpeg.py).

Divergence, deliberate: a DHT whose code counts overflow the code space is
CorruptStream here and in the C ABI. The reference (io/jpeg.py:274-296)
raises IndexError (not a FoveaError) when the overflow happens at a code
length <= 8, while filling its 8-bit lookup table; when it happens only at
lengths 9-16 it builds the table and decodes any stream that never uses the
unreachable codes. The C decoders' fast tables assume a valid code space, so
such tables are rejected up front (the reference's fuzz tests only require
"no crash other than FoveaError"; no encoder emits them).
"""
from __future__ import annotations

import struct

import numpy as np


class CorruptStream(Exception):
    pass


class UnsupportedJpegFeature(Exception):
    pass


# natural index of zigzag position k (jpeg.py:50-59, the JPEG standard order)
ZIGZAG = np.array([
    0, 1, 8, 16, 9, 2, 3, 10, 17, 24, 32, 25, 18, 11, 4, 5,
    12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6, 7, 14, 21, 28,
    35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
    58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63,
], dtype=np.int64)


# ---------------------------------------------------------------------------
# headers (jpeg.py:605-735)
# ---------------------------------------------------------------------------

def _huff_table(bits, values):
    """Canonical code tables (jpeg.py:269-296): per length L the first code,
    the last code (-1 if none) and the index of its first value."""
    if sum(bits) != len(values):
        raise CorruptStream("Huffman table size mismatch")
    mincode, maxcode, valptr = [0] * 17, [-1] * 17, [0] * 17
    code = idx = 0
    for length in range(1, 17):
        cnt = bits[length - 1]
        if cnt:
            if code + cnt > (1 << length):
                raise CorruptStream("Huffman code space overflow")
            valptr[length], mincode[length] = idx, code
            idx += cnt
            code += cnt
            maxcode[length] = code - 1
        code <<= 1
    return {"mincode": mincode, "maxcode": maxcode, "valptr": valptr, "values": list(values)}


def parse(data: bytes) -> dict:
    """Walk the markers up to the first SOS; returns the frame, tables, the
    scan's component order and its entropy-coded segments."""
    n = len(data)
    if n < 4 or data[0] != 0xFF or data[1] != 0xD8:
        raise CorruptStream("not a JPEG stream (bad SOI)")
    qt, dct, act = {}, {}, {}
    comps, height, width, dri = [], None, None, 0
    i = 2
    while True:
        if i + 2 > n:
            raise CorruptStream("stream ends without EOI")
        if data[i] != 0xFF:
            raise CorruptStream(f"expected marker at offset {i}")
        mk = data[i + 1]
        i += 2
        if mk == 0xD9:
            raise CorruptStream("EOI before scan data")
        if mk == 0x01 or 0xD0 <= mk <= 0xD7:
            continue
        if i + 2 > n:
            raise CorruptStream("truncated stream")
        (ln,) = struct.unpack_from(">H", data, i)
        if ln < 2:
            raise CorruptStream("bad segment length")
        if i + ln > n:
            raise CorruptStream("truncated stream")
        pl = data[i + 2:i + ln]
        i += ln
        if mk == 0xDB:  # DQT
            p = 0
            while p < len(pl):
                pq, tq = pl[p] >> 4, pl[p] & 15
                p += 1
                if pq not in (0, 1):
                    raise CorruptStream(f"bad DQT precision {pq}")
                cnt = 64 * (2 if pq else 1)
                if p + cnt > len(pl):
                    raise CorruptStream("truncated DQT")
                vals = (np.frombuffer(pl, ">u2", 64, p) if pq else np.frombuffer(pl, np.uint8, 64, p)).astype(np.int64)
                t = np.zeros(64, np.int64)
                t[ZIGZAG] = vals
                qt[tq] = t
                p += cnt
        elif mk in (0xC0, 0xC1):  # SOF0 / SOF1
            if len(pl) < 6:
                raise CorruptStream("truncated SOF")
            prec, height, width, nc = struct.unpack_from(">BHHB", pl, 0)
            if prec != 8:
                raise UnsupportedJpegFeature(f"sample precision {prec}")
            if height == 0 or width == 0:
                raise CorruptStream("zero dimension")
            if nc not in (1, 3):
                raise UnsupportedJpegFeature(f"{nc} components")
            if len(pl) != 6 + 3 * nc:
                raise CorruptStream("bad SOF length")
            comps = []
            for c in range(nc):
                cid, hv, tq = pl[6 + 3 * c:9 + 3 * c]
                h, v = hv >> 4, hv & 15
                if h not in (1, 2) or v not in (1, 2):
                    raise UnsupportedJpegFeature(f"sampling factors {h}x{v}")
                comps.append({"id": cid, "h": h, "v": v, "tq": tq})
            if nc == 1:
                comps[0]["h"] = comps[0]["v"] = 1
        elif mk == 0xC2:
            raise UnsupportedJpegFeature("progressive JPEG")
        elif mk in (0xC3, 0xC5, 0xC6, 0xC7, 0xC9, 0xCA, 0xCB, 0xCD, 0xCE, 0xCF):
            raise UnsupportedJpegFeature(f"SOF marker 0xFF{mk:02X}")
        elif mk == 0xCC:
            raise UnsupportedJpegFeature("arithmetic coding")
        elif mk == 0xC4:  # DHT
            p = 0
            while p < len(pl):
                if p + 17 > len(pl):
                    raise CorruptStream("truncated DHT")
                tc, th = pl[p] >> 4, pl[p] & 15
                bits = list(pl[p + 1:p + 17])
                cnt = sum(bits)
                if p + 17 + cnt > len(pl):
                    raise CorruptStream("truncated DHT values")
                (dct if tc == 0 else act)[th] = _huff_table(bits, pl[p + 17:p + 17 + cnt])
                p += 17 + cnt
        elif mk == 0xDD:  # DRI
            if len(pl) != 2:
                raise CorruptStream("bad DRI length")
            (dri,) = struct.unpack(">H", pl)
        elif mk == 0xDA:  # SOS
            if not comps:
                raise CorruptStream("SOS before SOF")
            if len(pl) < 1:
                raise CorruptStream("bad SOS length")
            ns = pl[0]
            if ns != len(comps):
                raise UnsupportedJpegFeature("multi-scan stream")
            if len(pl) != 1 + 2 * ns + 3:
                raise CorruptStream("bad SOS length")
            order = []
            for s in range(ns):
                cid, tbl = pl[1 + 2 * s], pl[2 + 2 * s]
                comp = next((c for c in comps if c["id"] == cid), None)
                if comp is None:
                    raise CorruptStream(f"scan references unknown component {cid}")
                td, ta = tbl >> 4, tbl & 15
                if td not in dct or ta not in act:
                    raise CorruptStream("scan references missing Huffman table")
                order.append(dict(comp, dc=dct[td], ac=act[ta]))
            segments = _split_scan(data, i)
            break
    if height is None:
        raise CorruptStream("no scan data")
    for c in order:
        if c["tq"] not in qt:
            raise CorruptStream(f"component references missing quant table {c['tq']}")
        c["q"] = qt[c["tq"]]
    return {"width": width, "height": height, "comps": order, "dri": dri, "segments": segments}


def _split_scan(data: bytes, i: int) -> list:
    """Unstuffed entropy-coded segments, split at RSTn (jpeg.py:574-602)."""
    segs, cur, n = [], bytearray(), len(data)
    while i < n:
        b = data[i]
        if b != 0xFF:
            cur.append(b)
            i += 1
            continue
        if i + 1 >= n:
            raise CorruptStream("scan ends mid-marker")
        nx = data[i + 1]
        if nx == 0x00:
            cur.append(0xFF)
            i += 2
        elif 0xD0 <= nx <= 0xD7:
            segs.append(bytes(cur))
            cur = bytearray()
            i += 2
        elif nx == 0xFF:
            i += 1
        else:
            segs.append(bytes(cur))
            return segs
    raise CorruptStream("scan ends without a terminating marker")


# ---------------------------------------------------------------------------
# entropy decoding (jpeg.py:299-409, 740-780)
# ---------------------------------------------------------------------------

class _Bits:
    """MSB-first reader over one segment, zero bits past its end; `over`
    says whether any of those was consumed."""

    def __init__(self, seg: bytes):
        self.seg, self.pos = seg, 0  # pos in bits

    def bit(self) -> int:
        p = self.pos
        self.pos += 1
        byte = p >> 3
        return (self.seg[byte] >> (7 - (p & 7))) & 1 if byte < len(self.seg) else 0

    def take(self, k: int) -> int:
        v = 0
        for _ in range(k):
            v = (v << 1) | self.bit()
        return v

    def over(self) -> bool:
        return self.pos > 8 * len(self.seg)


def _symbol(r: _Bits, t: dict) -> int:
    code = 0
    for length in range(1, 17):
        code = (code << 1) | r.bit()
        if t["maxcode"][length] >= 0 and code <= t["maxcode"][length] and code >= t["mincode"][length]:
            return t["values"][t["valptr"][length] + code - t["mincode"][length]]
    raise CorruptStream("invalid Huffman code")


def _extend(v: int, size: int) -> int:
    return v - (1 << size) + 1 if v < (1 << (size - 1)) else v


def decode_coefficients(info: dict) -> list:
    """Per scan component: int64 array (bh*bw, 64) of quantised coefficients
    in NATURAL order, blocks in raster order over the padded MCU grid."""
    comps = info["comps"]
    hmax = max(c["h"] for c in comps)
    vmax = max(c["v"] for c in comps)
    mx_n = -(-info["width"] // (8 * hmax))
    my_n = -(-info["height"] // (8 * vmax))
    total = mx_n * my_n
    out = []
    for c in comps:
        c["bw"], c["bh"] = mx_n * c["h"], my_n * c["v"]
        out.append(np.zeros((c["bw"] * c["bh"], 64), np.int64))
    dri = info["dri"]
    expected = [min(dri, total - s) for s in range(0, total, dri)] if dri else [total]
    if len(info["segments"]) < len(expected):
        raise CorruptStream(f"{len(info['segments'])} entropy segments, expected {len(expected)}")
    mcu = 0
    for si, cnt in enumerate(expected):
        r = _Bits(info["segments"][si])
        pred = [0] * len(comps)
        for _ in range(cnt):
            my, mx = divmod(mcu, mx_n)
            for ci, c in enumerate(comps):
                for by in range(c["v"]):
                    for bx in range(c["h"]):
                        blk = out[ci][(my * c["v"] + by) * c["bw"] + mx * c["h"] + bx]
                        size = _symbol(r, c["dc"])
                        if size:
                            if size > 11:
                                raise CorruptStream(f"bad DC size {size}")
                            pred[ci] += _extend(r.take(size), size)
                        blk[0] = pred[ci]
                        k = 1
                        while k < 64:
                            rs = _symbol(r, c["ac"])
                            size = rs & 15
                            if size == 0:
                                if rs == 0xF0:
                                    k += 16
                                    continue
                                break
                            k += rs >> 4
                            if k > 63:
                                raise CorruptStream("AC run past end of block")
                            blk[ZIGZAG[k]] = _extend(r.take(size), size)
                            k += 1
            mcu += 1
        if r.over():
            raise CorruptStream("entropy segment too short for its MCUs")
    return out


# ---------------------------------------------------------------------------
# reconstruction (jpeg.py:142-235, 783-841)
# ---------------------------------------------------------------------------

_K = {  # 13-bit fixed-point constants (jpeg.py:142-156)
    "c0298": 2446, "c0390": 3196, "c0541": 4433, "c0765": 6270, "c0899": 7373, "c1175": 9633,
    "c1501": 12299, "c1847": 15137, "c1961": 16069, "c2053": 16819, "c2562": 20995, "c3072": 25172,
}


def _idct_1d(s):
    """One 8-point pass (jpeg.py:163-191) on int64 arrays s[0..7]; outputs
    before descaling, in index order."""
    k = _K
    z1 = (s[2] + s[6]) * k["c0541"]
    e2 = z1 - s[6] * k["c1847"]
    e3 = z1 + s[2] * k["c0765"]
    e0 = (s[0] + s[4]) << 13
    e1 = (s[0] - s[4]) << 13
    a10, a13, a11, a12 = e0 + e3, e0 - e3, e1 + e2, e1 - e2
    z5 = (s[7] + s[3] + s[5] + s[1]) * k["c1175"]
    o0 = s[7] * k["c0298"]
    o1 = s[5] * k["c2053"]
    o2 = s[3] * k["c3072"]
    o3 = s[1] * k["c1501"]
    q1 = (s[7] + s[1]) * -k["c0899"]
    q2 = (s[5] + s[3]) * -k["c2562"]
    q3 = (s[7] + s[3]) * -k["c1961"] + z5
    q4 = (s[5] + s[1]) * -k["c0390"] + z5
    o0 = o0 + q1 + q3
    o1 = o1 + q2 + q4
    o2 = o2 + q2 + q3
    o3 = o3 + q1 + q4
    return [a10 + o3, a11 + o2, a12 + o1, a13 + o0, a13 - o0, a12 - o1, a11 - o2, a10 - o3]


def _descale(x, n):
    return (x + (1 << (n - 1))) >> n


def idct_islow(blocks: np.ndarray) -> np.ndarray:
    """(nb, 8, 8) dequantised int64 [row = vertical frequency] -> clipped
    samples (nb, 8, 8) with the +128 level shift (jpeg.py:194-203)."""
    cols = _idct_1d([blocks[:, k, :] for k in range(8)])          # along the columns
    ws = np.stack([_descale(v, 11) for v in cols], axis=1)
    rows = _idct_1d([ws[:, :, k] for k in range(8)])               # along the rows
    out = np.stack([_descale(v, 18) + 128 for v in rows], axis=2)
    return np.clip(out, 0, 255)


def upsample_h2(p: np.ndarray) -> np.ndarray:
    """jpeg.py:809-821: horizontal x2, near sample 3/4, far 1/4."""
    h, m = p.shape
    if m <= 2:
        return np.repeat(p, 2, axis=1)
    o = np.empty((h, 2 * m), np.int64)
    o[:, 0] = p[:, 0]
    o[:, 2::2] = (3 * p[:, 1:] + p[:, :-1] + 1) >> 2
    o[:, 1:-1:2] = (3 * p[:, :-1] + p[:, 1:] + 2) >> 2
    o[:, -1] = p[:, -1]
    return o


def upsample_h2v2(p: np.ndarray) -> np.ndarray:
    """jpeg.py:824-841: vertical 3:1 column sums, horizontal 3:1, one final
    rounding (+8 / +7 alternating)."""
    mh, m = p.shape
    if m <= 2:
        return np.repeat(np.repeat(p, 2, axis=0), 2, axis=1)
    up = np.concatenate([p[:1], p[:-1]], axis=0)
    dn = np.concatenate([p[1:], p[-1:]], axis=0)
    cs = np.empty((2 * mh, m), np.int64)
    cs[0::2] = 3 * p + up
    cs[1::2] = 3 * p + dn
    o = np.empty((2 * mh, 2 * m), np.int64)
    o[:, 0] = (cs[:, 0] * 4 + 8) >> 4
    o[:, 2::2] = (3 * cs[:, 1:] + cs[:, :-1] + 8) >> 4
    o[:, 1:-1:2] = (3 * cs[:, :-1] + cs[:, 1:] + 7) >> 4
    o[:, -1] = (cs[:, -1] * 4 + 7) >> 4
    return o


def ycbcr_to_rgb(y, cb, cr) -> np.ndarray:
    """jpeg.py:226-235."""
    xb, xr = cb - 128, cr - 128
    r = y + ((91881 * xr + 32768) >> 16)
    g = y + ((-22554 * xb + 32768 - 46802 * xr) >> 16)
    b = y + ((116130 * xb + 32768) >> 16)
    return np.clip(np.stack([r, g, b], axis=2), 0, 255).astype(np.uint8)


def component_planes(info: dict, coeffs: list) -> list:
    """IDCT samples of each component, cropped to its own size and upsampled
    to the image (jpeg.py:783-806)."""
    comps = info["comps"]
    hmax = max(c["h"] for c in comps)
    vmax = max(c["v"] for c in comps)
    W, H = info["width"], info["height"]
    planes = []
    for c, co in zip(comps, coeffs):
        sp = idct_islow((co * c["q"][None, :]).reshape(-1, 8, 8))
        plane = sp.reshape(c["bh"], c["bw"], 8, 8).transpose(0, 2, 1, 3).reshape(c["bh"] * 8, c["bw"] * 8)
        plane = plane[:-(-H * c["v"] // vmax), :-(-W * c["h"] // hmax)]
        fh, fv = hmax // c["h"], vmax // c["v"]
        if fh == 2 and fv == 2:
            plane = upsample_h2v2(plane)
        elif fh == 2:
            plane = upsample_h2(plane)
        elif fv == 2:
            plane = upsample_h2(plane.T).T
        planes.append(plane[:H, :W])
    return planes


def decode_jpeg(data: bytes) -> np.ndarray:
    """(H, W, 3) u8 for 3-component streams (planes in scan order as Y, Cb,
    Cr), (H, W, 1) for grayscale (jpeg.py:605-806)."""
    info = parse(data)
    planes = component_planes(info, decode_coefficients(info))
    if len(planes) == 1:
        return planes[0].astype(np.uint8)[:, :, None]
    return ycbcr_to_rgb(*planes)
