"""NumPy restatement of the reference (`fovea`) image-transformation path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Every function cites the
reference file:line it restates; paths are relative to the reference package
root `pkg/src/fovea/`. The arithmetic is written op-for-op in the same order
and the same precision as the reference so results are bit-identical:

  * IEEE f64 / f32 NumPy ufuncs, each op separately rounded (no FMA);
  * `uint8 * python-float` promotes to f64 (imgproc.py:56);
  * `f32 op python-float` stays f32 (NEP 50; tensor.py:273).

All images are HWC `np.ndarray`s; batched helpers loop over the leading axis.
Functions accept an optional `rows=(y_begin, y_end)` destination row range so
that large configurations can be checked (and timed as a CPU baseline) on a
bounded, seeded sample: bilinear sampling is row-separable, so a row band of
the output is computed exactly as the full-frame call would compute it.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "WR", "WG", "WB",
    "seeded_u8_image", "seeded_f32_image",
    "gray_from_rgb", "to_float_scaled", "cast_to_u8", "source_centers", "axis_taps",
    "resize_bilinear", "resize_u8", "normalize_lut", "resize_normalize_chw",
    "invert_affine", "invert_homography", "affine_forward", "perspective_forward",
    "warp_affine", "warp_perspective",
    "gray_scalar", "bilinear_scalar", "warp_scalar", "resize_normalize_chw_scalar",
    "flip_horizontal", "nearest_indices", "resize_nearest", "sobel",
]

# BT.601 luma weights -- imgproc.py:27
WR, WG, WB = 0.299, 0.587, 0.114


# --------------------------------------------------------------------------
# fixtures -- synth.py:14-23
# --------------------------------------------------------------------------

def seeded_u8_image(width: int, height: int, channels: int, seed: int = 0) -> np.ndarray:
    """synth.py:14-17: default_rng(seed).integers(0, 256, (H, W, C), u8)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, size=(height, width, channels), dtype=np.uint8)


def seeded_f32_image(width: int, height: int, channels: int, seed: int = 0) -> np.ndarray:
    """synth.py:20-23: default_rng(seed).random((H, W, C), f32)."""
    rng = np.random.default_rng(seed)
    return rng.random(size=(height, width, channels), dtype=np.float32)


# --------------------------------------------------------------------------
# a1: gray_from_rgb -- imgproc.py:43-64
# --------------------------------------------------------------------------

def gray_from_rgb(a: np.ndarray) -> np.ndarray:
    """imgproc.py:53-62. u8: f64 products/sums, floor(g+0.5), astype(u8).
    f32: widen to f64, same sum, narrow to f32. Returns (H, W, 1)."""
    if a.dtype == np.uint8:
        g = a[:, :, 0] * WR + a[:, :, 1] * WG + a[:, :, 2] * WB      # imgproc.py:56
        np.floor(g + 0.5, out=g)                                      # imgproc.py:57
        return g.astype(np.uint8)[:, :, None]                         # imgproc.py:58
    if a.dtype == np.float32:
        a64 = a.astype(np.float64)                                    # imgproc.py:60
        g = a64[:, :, 0] * WR + a64[:, :, 1] * WG + a64[:, :, 2] * WB
        return g.astype(np.float32)[:, :, None]                       # imgproc.py:62
    raise TypeError(f"gray_from_rgb supports u8 and f32, got {a.dtype}")


# --------------------------------------------------------------------------
# a4 / a5: to_float_scaled and Tensor.cast
# --------------------------------------------------------------------------

def to_float_scaled(a: np.ndarray) -> np.ndarray:
    """image.py:158-160: copy u8 into f32, then `/= f32(255)` (IEEE division)."""
    out = a.astype(np.float32)
    out /= np.float32(255.0)
    return out


def cast_to_u8(x: np.ndarray) -> np.ndarray:
    """tensor.py:272-276 float->u8: round half away from zero (f32 arithmetic),
    NaN->0, +-inf->limits, clip to [0, 255]."""
    rounded = np.where(x >= 0, np.floor(x + 0.5), np.ceil(x - 0.5))
    rounded = np.nan_to_num(rounded, nan=0.0, posinf=255.0, neginf=0.0)
    np.clip(rounded, 0, 255, out=rounded)
    return rounded.astype(np.uint8)


# --------------------------------------------------------------------------
# a2 / a3: coordinate tables and f32 bilinear resize -- imgproc.py:76-123
# --------------------------------------------------------------------------

def source_centers(dst_n: int, src_n: int) -> np.ndarray:
    """imgproc.py:76-78: (arange(dst_n) + 0.5) * (src_n / dst_n) - 0.5 in f64."""
    scale = src_n / dst_n
    return (np.arange(dst_n, dtype=np.float64) + 0.5) * scale - 0.5


def axis_taps(dst_n: int, src_n: int):
    """imgproc.py:109-116: clip before floor; i1 = min(i0+1, n-1); f = f32(s - i0)."""
    s = np.clip(source_centers(dst_n, src_n), 0.0, src_n - 1.0)
    i0 = np.floor(s).astype(np.int64)
    i1 = np.minimum(i0 + 1, src_n - 1)
    f = (s - i0).astype(np.float32)
    return i0, i1, f


def _blend(t00, t01, t10, t11, fx, fy, out=None):
    """imgproc.py:118-123 blend order: every product and sum is a separately
    rounded f32 op; `1 - f` is computed in f32."""
    top = t00 * (1 - fx) + t01 * fx
    bot = t10 * (1 - fx) + t11 * fx
    np.multiply(top, (1 - fy), out=top)
    np.multiply(bot, fy, out=bot)
    if out is None:
        return top + bot
    np.add(top, bot, out=out)
    return out


def resize_bilinear(a: np.ndarray, dst_w: int, dst_h: int, rows=None) -> np.ndarray:
    """imgproc.py:100-123 (f32 only). Returns dst rows [rows[0], rows[1])."""
    if a.dtype != np.float32:
        raise TypeError("resize_bilinear requires f32")
    h, w, _ = a.shape
    y_lo, y_hi = (0, dst_h) if rows is None else rows
    x0, x1, fx = axis_taps(dst_w, w)
    y0, y1, fy = axis_taps(dst_h, h)
    y0, y1, fy = y0[y_lo:y_hi], y1[y_lo:y_hi], fy[y_lo:y_hi]
    fx = fx[None, :, None]
    fy = fy[:, None, None]
    return _blend(a[y0[:, None], x0[None, :], :], a[y0[:, None], x1[None, :], :],
                  a[y1[:, None], x0[None, :], :], a[y1[:, None], x1[None, :], :], fx, fy)


# --------------------------------------------------------------------------
# a6: u8 bilinear resize -- service/app.py:64-78
# --------------------------------------------------------------------------

def resize_u8(a: np.ndarray, dst_w: int, dst_h: int, rows=None) -> np.ndarray:
    """app.py:70-78: to_float_scaled -> resize_bilinear -> x f32(255) -> cast(u8)."""
    if a.dtype != np.uint8:
        raise TypeError("resize_u8 requires u8")
    if rows is not None:
        # only the source rows the band touches need converting (same values)
        y0, y1, _ = axis_taps(dst_h, a.shape[0])
        lo, hi = int(y0[rows[0]]), int(y1[rows[1] - 1]) + 1
        src_f = np.zeros(a.shape, np.float32)
        src_f[lo:hi] = to_float_scaled(a[lo:hi])
    else:
        src_f = to_float_scaled(a)
    dst_f = resize_bilinear(src_f, dst_w, dst_h, rows)
    return cast_to_u8(dst_f * np.float32(255.0))                      # app.py:75-78


# --------------------------------------------------------------------------
# a10: fused resize -> normalise -> CHW (builder contract)
# --------------------------------------------------------------------------

def normalize_lut(mean, std) -> np.ndarray:
    """(C, 256) f32 table of ((f32(u) / f32(255)) - mean_c) / std_c, each op
    an f32 NumPy op: to_float_scaled (image.py:158-160) then normalisation."""
    mean = np.asarray(mean, dtype=np.float32)
    std = np.asarray(std, dtype=np.float32)
    u = to_float_scaled(np.arange(256, dtype=np.uint8))[None, :]
    return ((u - mean[:, None]) / std[:, None]).astype(np.float32)


def resize_normalize_chw(a: np.ndarray, dst_w: int, dst_h: int, mean, std, rows=None) -> np.ndarray:
    """a6 u8 resize, then (f32(u)/255 - mean)/std per channel, then HWC->CHW.
    Returns (C, rows, dst_w) f32."""
    u = resize_u8(a, dst_w, dst_h, rows)
    x = to_float_scaled(u)
    x = (x - np.asarray(mean, np.float32)) / np.asarray(std, np.float32)
    return np.ascontiguousarray(x.transpose(2, 0, 1))


# --------------------------------------------------------------------------
# a8 / a9: warps (builder contract)
# --------------------------------------------------------------------------

def invert_affine(m) -> np.ndarray:
    """Forward 2x3 (src->dst) -> inverse 2x3 (dst->src) via f64 np.linalg.inv
    of the 3x3 homogeneous matrix."""
    m = np.asarray(m, dtype=np.float64).reshape(2, 3)
    full = np.vstack([m, [0.0, 0.0, 1.0]])
    return np.linalg.inv(full)[:2].copy()


def invert_homography(hm) -> np.ndarray:
    """Forward 3x3 (src->dst) -> inverse 3x3 via f64 np.linalg.inv."""
    return np.linalg.inv(np.asarray(hm, dtype=np.float64).reshape(3, 3))


def affine_forward(seed: int, width: int, height: int) -> np.ndarray:
    """cfg2 parameters: theta~U(-30,30) deg, s~U(0.8,1.2), t~U(-50,50)^2 drawn
    in that order from default_rng(seed); rotation about the image centre
    c=((W-1)/2,(H-1)/2): A = s R(theta), b = c + t - A c."""
    rng = np.random.default_rng(seed)
    theta = np.deg2rad(rng.uniform(-30.0, 30.0))
    s = rng.uniform(0.8, 1.2)
    tx, ty = rng.uniform(-50.0, 50.0), rng.uniform(-50.0, 50.0)
    a = s * np.array([[np.cos(theta), -np.sin(theta)], [np.sin(theta), np.cos(theta)]])
    c = np.array([(width - 1) / 2.0, (height - 1) / 2.0])
    b = c + np.array([tx, ty]) - a @ c
    return np.hstack([a, b[:, None]])


def perspective_forward(seed: int) -> np.ndarray:
    """cfg3 parameters: H = I + eps, eps ~ N(0, 1e-3) iid on the 8 free
    entries (row-major), H[2,2] = 1, pixel coordinates."""
    eps = np.random.default_rng(seed).normal(0.0, 1e-3, 8)
    hm = np.eye(3).reshape(-1)
    hm[:8] += eps
    hm[8] = 1.0
    return hm.reshape(3, 3)


def _gather(img_f: np.ndarray, xi, yi, border_f):
    """Per-tap constant border: taps outside [0,W-1]x[0,H-1] read `border_f`."""
    h, w, c = img_f.shape
    inside = (xi >= 0) & (xi < w) & (yi >= 0) & (yi < h)
    vals = img_f[np.clip(yi, 0, h - 1), np.clip(xi, 0, w - 1)]
    return np.where(inside[..., None], vals, border_f)


def _warp(img_f: np.ndarray, sx, sy, border_f, finite):
    """Shared sampler. sx, sy: f64 (H, W) source coordinates."""
    h, w, _ = img_f.shape
    # guard the int conversion; clamping keeps every out-of-range tap out of range
    x0f = np.floor(np.where(finite, sx, 0.0))
    y0f = np.floor(np.where(finite, sy, 0.0))
    fx = (np.where(finite, sx, 0.0) - x0f).astype(np.float32)[..., None]
    fy = (np.where(finite, sy, 0.0) - y0f).astype(np.float32)[..., None]
    x0 = np.clip(x0f, -2.0, w + 1.0).astype(np.int64)
    y0 = np.clip(y0f, -2.0, h + 1.0).astype(np.int64)
    t00 = _gather(img_f, x0, y0, border_f)
    t01 = _gather(img_f, x0 + 1, y0, border_f)
    t10 = _gather(img_f, x0, y0 + 1, border_f)
    t11 = _gather(img_f, x0 + 1, y0 + 1, border_f)
    return _blend(t00.astype(np.float32), t01.astype(np.float32),
                  t10.astype(np.float32), t11.astype(np.float32), fx, fy)


def _grid(out_h, out_w, rows):
    y_lo, y_hi = (0, out_h) if rows is None else rows
    x = np.arange(out_w, dtype=np.float64)[None, :]
    y = np.arange(y_lo, y_hi, dtype=np.float64)[:, None]
    return x, y


def _finish(a: np.ndarray, out_f: np.ndarray, border, finite):
    """u8: the app.py:75-78 recipe (x255, round half away, clamp); f32: as is.
    Non-finite coordinates produce the raw border value."""
    if a.dtype == np.uint8:
        out = cast_to_u8(out_f * np.float32(255.0))
        return np.where(finite[..., None], out, np.uint8(border))
    return np.where(finite[..., None], out_f, np.float32(border))


def warp_affine(a: np.ndarray, m_inv, out_h: int, out_w: int, border=0, rows=None) -> np.ndarray:
    """Inverse-mapped bilinear warp. sx = m00*x + (m01*y + m02) and
    sy = m10*x + (m11*y + m12), f64, each op rounded; x0 = floor(sx),
    fx = f32(sx - x0); per-tap constant border; imgproc.py:118-123 blend.
    u8 images go through the _resize_u8 recipe (to_float_scaled -> blend ->
    x255 -> cast), f32 images are blended directly."""
    m = np.asarray(m_inv, np.float64).reshape(2, 3)
    x, y = _grid(out_h, out_w, rows)
    sx = m[0, 0] * x + (m[0, 1] * y + m[0, 2])
    sy = m[1, 0] * x + (m[1, 1] * y + m[1, 2])
    finite = np.isfinite(sx) & np.isfinite(sy)
    img_f, border_f = _as_float(a, border)
    return _finish(a, _warp(img_f, sx, sy, border_f, finite), border, finite)


def warp_perspective(a: np.ndarray, h_inv, out_h: int, out_w: int, border=0, rows=None) -> np.ndarray:
    """Projective inverse map: X = h00*x + (h01*y + h02), likewise Y, W (f64,
    each op rounded); W == 0 or a non-finite coordinate -> raw border; else
    r = 1/W, sx = X*r, sy = Y*r, then the warp_affine sampler."""
    hm = np.asarray(h_inv, np.float64).reshape(3, 3)
    x, y = _grid(out_h, out_w, rows)
    X = hm[0, 0] * x + (hm[0, 1] * y + hm[0, 2])
    Y = hm[1, 0] * x + (hm[1, 1] * y + hm[1, 2])
    W = hm[2, 0] * x + (hm[2, 1] * y + hm[2, 2])
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        r = 1.0 / W
        sx = X * r
        sy = Y * r
    finite = (W != 0) & np.isfinite(sx) & np.isfinite(sy)
    img_f, border_f = _as_float(a, border)
    return _finish(a, _warp(img_f, sx, sy, border_f, finite), border, finite)


def _as_float(a, border):
    if a.dtype == np.uint8:
        return to_float_scaled(a), to_float_scaled(np.array([border], np.uint8))[0]
    if a.dtype == np.float32:
        return a, np.float32(border)
    raise TypeError(f"warps support u8 and f32, got {a.dtype}")


# --------------------------------------------------------------------------
# scalar twins: naive per-pixel Python loops sharing no code with the above,
# in the style of the reference's pkg/tests/oracles.py:1-97
# --------------------------------------------------------------------------

def _f32(v):
    return float(np.float32(v))


def gray_scalar(arr: np.ndarray) -> np.ndarray:
    """pkg/tests/oracles.py:11-22."""
    h, w, _ = arr.shape
    px = arr.tolist()
    out = np.zeros((h, w, 1), np.uint8 if arr.dtype == np.uint8 else np.float32)
    for y in range(h):
        for x in range(w):
            r, g, b = px[y][x]
            v = r * 0.299 + g * 0.587 + b * 0.114
            out[y, x, 0] = math.floor(v + 0.5) if arr.dtype == np.uint8 else v
    return out


def _blend_scalar(t00, t01, t10, t11, fx, fy):
    # every intermediate rounded to f32, as the vectorised NumPy code does
    wx0, wy0 = _f32(1 - fx), _f32(1 - fy)
    top = _f32(_f32(t00 * wx0) + _f32(t01 * fx))
    bot = _f32(_f32(t10 * wx0) + _f32(t11 * fx))
    return _f32(_f32(top * wy0) + _f32(bot * fy))


def _u8_out(v):
    y = _f32(v * 255.0)
    t = _f32(y + 0.5)
    return min(max(math.floor(t), 0), 255)


def bilinear_scalar(arr: np.ndarray, dst_w: int, dst_h: int) -> np.ndarray:
    """pkg/tests/oracles.py:54-72 extended to u8 via the app.py:64-78 recipe."""
    h, w, c = arr.shape
    is_u8 = arr.dtype == np.uint8
    px = arr.tolist()
    out = np.zeros((dst_h, dst_w, c), arr.dtype)
    for y in range(dst_h):
        sy = min(max((y + 0.5) * (h / dst_h) - 0.5, 0.0), h - 1.0)
        y0 = math.floor(sy)
        y1 = min(y0 + 1, h - 1)
        fy = _f32(sy - y0)
        for x in range(dst_w):
            sx = min(max((x + 0.5) * (w / dst_w) - 0.5, 0.0), w - 1.0)
            x0 = math.floor(sx)
            x1 = min(x0 + 1, w - 1)
            fx = _f32(sx - x0)
            for ch in range(c):
                taps = [px[y0][x0][ch], px[y0][x1][ch], px[y1][x0][ch], px[y1][x1][ch]]
                if is_u8:
                    taps = [_f32(_f32(t) / _f32(255.0)) for t in taps]
                v = _blend_scalar(*taps, fx, fy)
                out[y, x, ch] = _u8_out(v) if is_u8 else v
    return out


def warp_scalar(arr: np.ndarray, m_inv, out_h: int, out_w: int, border=0, perspective=False) -> np.ndarray:
    """Per-pixel twin of warp_affine / warp_perspective."""
    h, w, c = arr.shape
    is_u8 = arr.dtype == np.uint8
    m = [float(v) for v in np.asarray(m_inv, np.float64).reshape(-1)]
    px = arr.tolist()
    bf = _f32(_f32(border) / _f32(255.0)) if is_u8 else _f32(border)
    out = np.zeros((out_h, out_w, c), arr.dtype)
    for y in range(out_h):
        for x in range(out_w):
            sx = m[0] * x + (m[1] * y + m[2])
            sy = m[3] * x + (m[4] * y + m[5])
            if perspective:
                wz = m[6] * x + (m[7] * y + m[8])
                if wz == 0.0:
                    out[y, x, :] = border
                    continue
                r = 1.0 / wz
                sx, sy = sx * r, sy * r
            if not (math.isfinite(sx) and math.isfinite(sy)):
                out[y, x, :] = border
                continue
            x0, y0 = math.floor(sx), math.floor(sy)
            fx, fy = _f32(sx - x0), _f32(sy - y0)
            for ch in range(c):
                taps = []
                for yy, xx in ((y0, x0), (y0, x0 + 1), (y0 + 1, x0), (y0 + 1, x0 + 1)):
                    if 0 <= xx < w and 0 <= yy < h:
                        t = px[yy][xx][ch]
                        taps.append(_f32(_f32(t) / _f32(255.0)) if is_u8 else t)
                    else:
                        taps.append(bf)
                v = _blend_scalar(*taps, fx, fy)
                out[y, x, ch] = _u8_out(v) if is_u8 else v
    return out


def resize_normalize_chw_scalar(arr: np.ndarray, dst_w: int, dst_h: int, mean, std) -> np.ndarray:
    u = bilinear_scalar(arr, dst_w, dst_h)
    c = arr.shape[2]
    out = np.zeros((c, dst_h, dst_w), np.float32)
    for ch in range(c):
        m, s = _f32(mean[ch]), _f32(std[ch])
        for y in range(dst_h):
            for x in range(dst_w):
                v = _f32(_f32(u[y, x, ch]) / _f32(255.0))
                out[ch, y, x] = _f32(_f32(v - m) / s)
    return out


# --------------------------------------------------------------------------
# flip, nearest, sobel -- imgproc.py:67-97, 126-155
# --------------------------------------------------------------------------

def flip_horizontal(a: np.ndarray) -> np.ndarray:
    """imgproc.py:73: dst = src[:, ::-1, :]."""
    return np.ascontiguousarray(a[:, ::-1, :])


def nearest_indices(dst_n: int, src_n: int) -> np.ndarray:
    """imgproc.py:81-86: ceil((i + 0.5) * scale) - 1, clipped (round half down)."""
    scale = src_n / dst_n
    z = (np.arange(dst_n, dtype=np.float64) + 0.5) * scale
    return np.clip(np.ceil(z).astype(np.int64) - 1, 0, src_n - 1)


def resize_nearest(a: np.ndarray, dst_w: int, dst_h: int) -> np.ndarray:
    """imgproc.py:94-97."""
    xi = nearest_indices(dst_w, a.shape[1])
    yi = nearest_indices(dst_h, a.shape[0])
    return np.ascontiguousarray(a[yi[:, None], xi[None, :], :])


def sobel(a: np.ndarray) -> np.ndarray:
    """imgproc.py:139-155: edge-padded 3x3 Sobel magnitude, f32 op order."""
    p = np.pad(a, ((1, 1), (1, 1), (0, 0)), mode="edge")
    left, right = p[1:-1, :-2, :], p[1:-1, 2:, :]
    up, down = p[:-2, 1:-1, :], p[2:, 1:-1, :]
    ul, ur = p[:-2, :-2, :], p[:-2, 2:, :]
    dl, dr = p[2:, :-2, :], p[2:, 2:, :]
    gx = (ur - ul) + 2.0 * (right - left) + (dr - dl)
    gy = (dl - ul) + 2.0 * (down - up) + (dr - ur)
    np.multiply(gx, gx, out=gx)
    np.multiply(gy, gy, out=gy)
    np.add(gx, gy, out=gx)
    return np.sqrt(gx).astype(np.float32)
