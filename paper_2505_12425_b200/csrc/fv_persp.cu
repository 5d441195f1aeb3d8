// fv_persp.cu -- a9 warp_perspective, u8, the default <= 1 LSB path.
//
// The reference has no warps; the contract is the
// builder's (oracle/fovea_oracle.py:warp_perspective): inverse
// map in f64, x0 = floor(sx), fx = f32(sx - x0), per-tap constant border,
// blend in imgproc.py:118-123 order, u8 through the app.py:64-78 recipe.
// North star gate for u8 results of float interpolation: <= 1 LSB.
//
// One CTA = one 128 x 48 destination tile (8 warps x 6 rows, rows 8 apart).
//   1. Tile class, from the four corner maps (f64): a projective map whose W
//      keeps one strict sign over the tile sends it onto the convex hull of
//      the mapped corners, so the hull's box (+2 / +3 px) holds every tap.
//        BORDER    the hull lies beyond one side of the source: every pixel
//                  is the border value (16-byte stores, no sampling);
//        STAGED    the box (clipped to the image) fits the shared-memory
//                  window: warp 0 streams its row segments into SMEM with
//                  1-D TMA bulk copies (cp.async.bulk + mbarrier) while all
//                  warps compute their maps; taps are read with LDS;
//                  STAGED_IN = the box lies inside the image, so no pixel
//                  needs a bounds test;
//        DIRECT    W changes sign in the tile, or the box is too large
//                  (zoom-out): direct global gathers, after one bulk L2
//                  prefetch per box row (boxes <= FV_PT_PF_MAX bytes).
//   2. Maps: one f64 anchor per 32 pixels of a row (lanes 0-23 of a warp
//      compute the 24 anchors of its 6 rows at once) -- s_a = (X, Y) / W at
//      the group's first pixel, relative to the tile origin -- then lane L
//      samples pixel x_a + L of every group with the f32 projective
//      correction s = s_a + k * L / W(L), k = (m0 - s_a.x m6, m3 - s_a.y m6),
//      W(L) = W_a + m6 L (rcp.approx), two pixels at a time as f32x2 pairs.
//      Anchors live in SMEM slots laid out so each 16 writers hit 16 distinct
//      banks and each reader gets a field of both pixels of its pair from one
//      LDS.128 (broadcast: a group is warp-uniform).
//   3. Error bound per group (u = 2^-24): W(L) carries <= u (rho + 1)
//      relative error with rho = (|W_a| + 31 |m6|) / Wmin (roundings of W_a,
//      m6 L and the add), rcp.approx <= 2u, f32(k) and k * L u each, the FMA
//      u (|s_rel| + Cmax): with Cmax = 31 |k| / Wmin the correction is off by
//      <= u Cmax (rho + 6); with s_rel's own rounding the coordinate is off by
//      <= u (Cmax (rho + 6) + 2 |s_rel|) per axis. A group whose bound exceeds
//      PT_MAX_ERR = 5e-4 px, whose W changes sign or vanishes, or whose anchor
//      is non-finite or far from the tile takes the f64 per-pixel map
//      (warp_tap, the exact kernel's). Bilinear sampling with a constant
//      border is continuous in (sx, sy), so |out - oracle| <= 255 * 1e-3 +
//      (blend roundings ~3e-4) < 1 LSB.
//   4. Blend on the 0..255 scale (magic-word taps; two horizontal lerps and a
//      vertical one as FFMA2 on pixel pairs, floor(v + 0.5)),
//      results stored as bytes into a per-warp SMEM row buffer; the warp then
//      writes the row segment (384 B for C = 3) with 16-byte stores.
#include "fv_warp.cuh"

namespace fv {

#ifndef FV_PT_TH
#define FV_PT_TH 48  // 6 rows per warp: measured 32 / 40 / 48 / 56 / 64 -> cfg3 0.443 / 0.428 / 0.425 / 0.420 / 0.414 ms, but 56+ rows push near-identity tiles out of the 56-row window (0.447 -> 0.519 ms)
#endif
constexpr int PT_TW = 128;          // tile width, destination pixels (4 anchor groups of 32)
constexpr int PT_TH = FV_PT_TH;     // tile height: PT_NW warps x PT_RPW rows
#ifndef PT_NW
#define PT_NW 8  // warps per CTA
#endif
constexpr int PT_RPW = PT_TH / PT_NW;  // rows per warp (rows warp, warp + PT_NW, ...)
#ifndef FV_PT_PITCH3
#define FV_PT_PITCH3 592  // C = 3 window pitch (bytes); 48-row tiles: 56 x 656 / 60 x 624 / 64 x 592 / 56 x 720 -> cfg3 0.425 / 0.423 / 0.421 / 0.487 ms
#endif
#ifndef FV_PT_WROWS
#define FV_PT_WROWS 64
#endif
constexpr int PT_WROWS = FV_PT_WROWS;  // SMEM window rows
constexpr float PT_MAX_ERR = 5e-4f;
#ifndef FV_PT_LERP
#define FV_PT_LERP 1  // blend as two horizontal lerps and a vertical one (27 f32x2 ops per pixel pair, not 31)
#endif
#ifndef FV_PT_PF_MAX
#define FV_PT_PF_MAX 196608  // DIRECT tiles: L2 prefetch of the box when it holds at most this many bytes (0 = off)
#endif
#ifndef PT_MINB
#define PT_MINB 4
#endif
// window pitch in bytes: an odd multiple of 16 (bulk-copy destinations are
// 16-byte aligned; rows rotate banks), wide enough for a 1.4x zoom-out of a
// 128-pixel row plus the tap window's 12-byte overhang (C = 3)
template <int C>
constexpr int pt_pitch() { return C == 1 ? 240 : (C == 3 ? FV_PT_PITCH3 : 848); }
template <int C>
constexpr int pt_obuf() { return PT_TW * C; }  // one output row segment
constexpr int PT_ANC_OFF = 64;                                   // 8 warps x 8 slots x 48 B (tile info at 16)
template <int C>
constexpr int pt_obuf_off() { return PT_ANC_OFF + PT_TH * 2 * 48; }  // anchor slots: 2 per tile row
template <int C>
constexpr int pt_win_off() { return pt_obuf_off<C>() + PT_NW * 2 * pt_obuf<C>(); }  // 2 row buffers per warp
template <int C>
constexpr int pt_smem() { return pt_win_off<C>() + PT_WROWS * pt_pitch<C>(); }

enum : int { PT_BORDER = 0, PT_STAGED = 1, PT_DIRECT = 2 };
// per-group flags of the anchors
enum : int { PG_F32 = 1, PG_INTERIOR = 2 };

struct PtArgs {
  int stage_ok;  // 16-byte aligned source rows of a whole number of 16-byte units
  int dst_vec;   // 16-byte aligned destination row segments
};

struct PtTile {
  int cls;
  int ox, oy;     // origin of the tile's relative tap coordinates (image pixels)
  int cy0, rows;  // window rows [cy0, cy0 + rows) of the source
  int sb0, len;   // window's first byte within a source row (16-aligned), bytes per row
  int cx0;        // first window column (image pixels)
};

// Step 1 (warp 0; lanes 0-3 map the corners): the tile's class and window.
template <int C>
__device__ __forceinline__ PtTile pt_classify(const WarpArgs& a, const PtArgs& pa, const double* m, int tx0, int ty0,
                                              int lane) {
  // the corner maps in f64, then the box in f32: coordinates are clamped to
  // +-2^30 and the box carries 2 px margins (+1e-6 relative), far above
  // f32's rounding of any coordinate that can reach the window (|s| < 2^13);
  // the f64 min / max chains and double shuffles cost warp 0 -- the CTA's
  // critical path -- more than they buy
  float sx = 0.0f, sy = 0.0f;
  int sg = 0;
  if (lane < 4) {
    const double cx = (double)(tx0 + ((lane & 1) ? PT_TW - 1 : 0));
    const double cy = (double)(ty0 + ((lane & 2) ? PT_TH - 1 : 0));
    const double X = m[0] * cx + m[1] * cy + m[2], Y = m[3] * cx + m[4] * cy + m[5];
    const double W = m[6] * cx + m[7] * cy + m[8];
    const double r = __drcp_rn(W);  // the box has 2 px margins: no need for a division
    const double dx = X * r, dy = Y * r;
    sg = (W > 0.0) ? 1 : (W < 0.0 ? 2 : 0);
    if (!(isfinite(dx) && isfinite(dy))) sg = 0;
    const double L = 1073741824.0;
    sx = (float)(dx < -L ? -L : (dx > L ? L : dx));
    sy = (float)(dy < -L ? -L : (dy > L ? L : dy));
  }
  const unsigned F = 0xffffffffu;
  float xlo = __shfl_sync(F, sx, 0), ylo = __shfl_sync(F, sy, 0);
  float xhi = xlo, yhi = ylo;
  int sgall = __shfl_sync(F, sg, 0);
#pragma unroll
  for (int k = 1; k < 4; ++k) {
    const float ux = __shfl_sync(F, sx, k), uy = __shfl_sync(F, sy, k);
    xlo = fminf(xlo, ux);
    xhi = fmaxf(xhi, ux);
    ylo = fminf(ylo, uy);
    yhi = fmaxf(yhi, uy);
    sgall &= __shfl_sync(F, sg, k);
  }
  PtTile t{PT_DIRECT, 0, 0, 0, 0, 0, 0, 0};
  if (sgall == 0) return t;  // W changes sign or vanishes in the tile: no hull
  const float mx = 2.0f + 1e-6f * fmaxf(fabsf(xlo), fabsf(xhi)), my = 2.0f + 1e-6f * fmaxf(fabsf(ylo), fabsf(yhi));
  if (xhi < -1.0f - mx || xlo > (float)a.sw + mx || yhi < -1.0f - my || ylo > (float)a.sh + my) {
    t.cls = PT_BORDER;
    return t;
  }
  const float bx0 = floorf(xlo) - 2.0f, bx1 = floorf(xhi) + 3.0f;
  const float by0 = floorf(ylo) - 2.0f, by1 = floorf(yhi) + 3.0f;
  t.ox = (int)bx0;
  t.oy = (int)by0;
  const int cx0 = max(t.ox, 0), cx1 = min((int)bx1, a.sw - 1);
  const int cy0 = max(t.oy, 0), cy1 = min((int)by1, a.sh - 1);
  if (cx0 > cx1 || cy0 > cy1) {  // no image pixel inside the box: every tap reads the border
    t.cls = PT_BORDER;
    return t;
  }
  t.cy0 = cy0;
  t.cx0 = cx0;
  t.rows = cy1 - cy0 + 1;
  t.sb0 = (cx0 * C) & ~15;
  t.len = ((cx1 + 1) * C - t.sb0 + 15) & ~15;
  const bool staged = pa.stage_ok && t.rows <= PT_WROWS && t.len <= pt_pitch<C>() - 16;
  t.cls = staged ? PT_STAGED : PT_DIRECT;
  return t;
}

// the last x0 whose tap window (NW words from x0 * C rounded down to 4 bytes)
// ends inside the row: sw - margin (window: only the pixel pair must be in)
template <int C, bool STAGED>
constexpr int pt_xmargin() { return STAGED ? 2 : (C == 4 ? 2 : (C == 3 ? 4 : 7)); }

// Taps of one source row from a 4-byte aligned word window: (x0, x0 + 1), C
// bytes each, as magic words 0x4B0000uu. `w` = NW consecutive words.
template <int C>
constexpr int pt_nw() { return C == 4 ? 2 : (C == 3 ? 3 : 2); }
template <int C>
__device__ __forceinline__ void pt_taps(const uint32_t (&w)[pt_nw<C>()], int sh, uint32_t (&t0)[C],
                                        uint32_t (&t1)[C]) {
  if constexpr (C == 4) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      t0[c] = magic_of(w, c);
      t1[c] = magic_of(w, 4 + c);
    }
  } else {
    constexpr int NV = (2 * C + 3) / 4;
    uint32_t v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = __funnelshift_r(w[i], w[i + 1], sh);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      t0[c] = magic_of(v, c);
      t1[c] = magic_of(v, C + c);
    }
  }
}

// One pixel with per-tap border handling (edge pixels of mixed tiles, groups
// on the f64 map): absolute taps (x0, y0); in-image taps come from the SMEM
// window (STAGED) or global memory. Writes C bytes at SMEM address `out`.
template <int C, bool STAGED>
__device__ __noinline__ void pt_pixel_generic(const WarpArgs& a, const uint8_t* simg, uint32_t win, int cy0, int sb0,
                                              bool finite, int x0, int y0, float fx, float fy, uint32_t out) {
  const uint32_t braw = (uint32_t)a.border_raw;
  uint32_t res[C];
  if (!finite || x0 < -1 || x0 >= a.sw || y0 < -1 || y0 >= a.sh) {
#pragma unroll
    for (int c = 0; c < C; ++c) res[c] = braw;
  } else {
    const bool ix0 = x0 >= 0, ix1 = x0 + 1 < a.sw, iy0 = y0 >= 0, iy1 = y0 + 1 < a.sh;
    const float wx0 = __fsub_rn(1.0f, fx), wy0 = __fsub_rn(1.0f, fy);
    const float w00 = __fmul_rn(wx0, wy0), w01 = __fmul_rn(fx, wy0), w10 = __fmul_rn(wx0, fy),
                w11 = __fmul_rn(fx, fy);
    const float b = (float)braw;
    auto tap = [&](bool ok, int x, int y, int c) -> float {
      if (!ok) return b;
      uint32_t v;
      if constexpr (STAGED) {
        const uint32_t ad = win + (uint32_t)((y - cy0) * pt_pitch<C>() + x * C + c - sb0);
        FV_CHECK(y >= cy0 && y - cy0 < PT_WROWS && x * C + c >= sb0 && x * C + c - sb0 < pt_pitch<C>() - 16);
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(ad));
      } else {
        v = simg[(int64_t)y * a.s_rp + x * C + c];
      }
      return (float)v;
    };
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const float a00 = tap(iy0 && ix0, x0, y0, c), a01 = tap(iy0 && ix1, x0 + 1, y0, c);
      const float a10 = tap(iy1 && ix0, x0, y0 + 1, c), a11 = tap(iy1 && ix1, x0 + 1, y0 + 1, c);
      const float v = __fmaf_rn(a11, w11, __fmaf_rn(a10, w10, __fmaf_rn(a01, w01, __fmaf_rn(a00, w00, 0.5f))));
      res[c] = (uint32_t)min((int)floorf(v), 255);
    }
  }
#pragma unroll
  for (int c = 0; c < C; ++c) asm volatile("st.shared.u8 [%0], %1;" ::"r"(out + c), "r"(res[c]));
}

// Both pixels of a pair on the f64 per-pixel map (warp_tap, the exact
// kernel's): groups whose error bound failed.
template <int C, bool STAGED>
__device__ __noinline__ void pt_pair_f64(const WarpArgs& a, const double* mrow, const uint8_t* simg, uint32_t win,
                                         int cy0, int sb0, int y, int xa, uint32_t out) {
  double m[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) m[i] = mrow[i];
  const double yd = (double)y;
  const double rx = __dadd_rn(__dmul_rn(m[1], yd), m[2]), ry = __dadd_rn(__dmul_rn(m[4], yd), m[5]);
  const double rw = __dadd_rn(__dmul_rn(m[7], yd), m[8]);
#pragma unroll 1
  for (int k = 0; k < 2; ++k) {
    const int x = xa + 32 * k;
    if (x >= a.dw) break;
    const WarpTap w = warp_tap<true>(m, rx, ry, rw, x, a.sw, a.sh);
    pt_pixel_generic<C, STAGED>(a, simg, win, cy0, sb0, w.finite, w.x0, w.y0, w.wx1, w.wy1, out + 32 * C * k);
  }
}

template <int N>
__device__ __forceinline__ void lds_words(uint32_t (&w)[N], uint32_t addr) {
#pragma unroll
  for (int i = 0; i < N; ++i) asm volatile("ld.shared.b32 %0, [%1];" : "=r"(w[i]) : "r"(addr + 4 * i));
}

// The row loop: taps from the SMEM window (STAGED) or global gathers. Per
// pixel pair the two groups' flags pick the path (warp-uniform): both
// INTERIOR -> no bounds tests; both F32 -> per-pixel edge tests (pixels past
// the destination's right edge, taps at the source edge); else the f64 map.
template <int C, bool STAGED>
__device__ __forceinline__ void pt_rows(const WarpArgs& a, const PtArgs& pa, const PtTile& t, const double* mrow,
                                        const uint8_t* simg, uint8_t* dimg, uint32_t smem0, int tx0, int ty0,
                                        int warp, int lane) {
  constexpr int P = pt_pitch<C>();
  constexpr int OB = pt_obuf<C>();
  constexpr int NW = pt_nw<C>();
  constexpr uint32_t MB = 0x4B400000u;  // bits of 1.5 * 2^23: floor(t) = bits(RD(t + 1.5 * 2^23)) - MB
  const uint32_t win = smem0 + pt_win_off<C>();
  // window address of a tap from the floor words (fx, fy) of its relative
  // coordinates: SBM + fy * P + fx * C (the magic offset folded in, mod 2^32)
  const uint32_t SBM = win + (uint32_t)((t.oy - t.cy0) * P + t.ox * C - t.sb0) - MB * (uint32_t)(P + C);
  // direct: byte offset inside the image of a tap from its floor words
  const uint32_t rp32 = (uint32_t)a.s_rp;
  const uint32_t GBM = (uint32_t)t.oy * rp32 + (uint32_t)(t.ox * C) - MB * (rp32 + (uint32_t)C);
  // edge tests on absolute taps: x = fx - MB + ox in [0, xlim], y likewise
  const uint32_t xoff = (uint32_t)t.ox - MB, yoff = (uint32_t)t.oy - MB;
  const uint32_t xlim = (uint32_t)(a.sw - pt_xmargin<C, STAGED>()), ylim = (uint32_t)(a.sh - 2);
  // lanes past the destination's right edge: a safe in-window / in-image tap
  const uint32_t safe_fx = (uint32_t)((STAGED ? t.cx0 : 0) - t.ox) + MB;
  const uint32_t safe_fy = (uint32_t)((STAGED ? t.cy0 : 0) - t.oy) + MB;
  const uint32_t anc = smem0 + PT_ANC_OFF + warp * PT_RPW * 2 * 48;
  const uint32_t obw = smem0 + pt_obuf_off<C>() + warp * 2 * OB;  // this warp's two row buffers
  const float lf = (float)lane;
  const f2_t LL = f2(lf, lf);
  const float m6l = (float)(mrow[6] * (double)lane);
  const f2_t M6L = f2(m6l, m6l);
  const f2_t HALF = f2(0.5f, 0.5f), MAG = f2(8388608.0f, 8388608.0f), NMAG = f2(-8388608.0f, -8388608.0f);
  const f2_t MG = f2(12582912.0f, 12582912.0f), NMG = f2(-12582912.0f, -12582912.0f), NEG1 = f2(-1.0f, -1.0f);
  const f2_t ONE = f2(1.0f, 1.0f);
  const int xbytes = min(PT_TW, a.dw - tx0) * C;
#pragma unroll 1
  for (int r = 0; r < PT_RPW; ++r) {
    const int y = ty0 + warp + PT_NW * r;
    if (y >= a.dh) break;  // warp-uniform
    const uint32_t ob = obw + (r & 1) * OB + lane * C;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      float4 F0, F1, F2;
      {
        const uint32_t sl = anc + (r * 2 + p) * 48;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(F0.x), "=f"(F0.y), "=f"(F0.z), "=f"(F0.w) : "r"(sl));
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(F1.x), "=f"(F1.y), "=f"(F1.z), "=f"(F1.w) : "r"(sl + 16));
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(F2.x), "=f"(F2.y), "=f"(F2.z), "=f"(F2.w) : "r"(sl + 32));
      }
      const int xa = tx0 + 64 * p + lane;  // pixels xa (group 2p) and xa + 32 (group 2p + 1)
      const uint32_t o0 = ob + 64 * p * C;
      const int both = __float_as_int(F2.z) & __float_as_int(F2.w);  // warp-uniform
      if (!(both & PG_F32)) {
        pt_pair_f64<C, STAGED>(a, mrow, simg, win, t.cy0, t.sb0, y, xa, o0);
        continue;
      }
      const f2_t W = fadd2(f2(F2.x, F2.y), M6L);
      uint32_t wl, wh;
      f2split(W, wl, wh);
      const f2_t R = f2(rcp_approx(__uint_as_float(wl)), rcp_approx(__uint_as_float(wh)));
      const f2_t TX = ffma2(fmul2(f2(F1.x, F1.y), LL), R, f2(F0.x, F0.y));
      const f2_t TY = ffma2(fmul2(f2(F1.z, F1.w), LL), R, f2(F0.z, F0.w));
      // floor: RD(t + 1.5 * 2^23) holds floor(t) + MB in its bits (|t| < 2^22)
      const f2_t FX = fadd2_rd(TX, MG), FY = fadd2_rd(TY, MG);
      const f2_t WX1 = ffma2(fadd2(FX, NMG), NEG1, TX);  // t - floor(t), exact
      const f2_t WY1 = ffma2(fadd2(FY, NMG), NEG1, TY);
      uint32_t fx[2], fy[2];
      f2split(FX, fx[0], fx[1]);
      f2split(FY, fy[0], fy[1]);
      bool v1 = true;
      if (!(both & PG_INTERIOR)) {
        const bool v0 = xa < a.dw;
        v1 = xa + 32 < a.dw;
        const bool i0 = fx[0] + xoff <= xlim && fy[0] + yoff <= ylim;
        const bool i1 = fx[1] + xoff <= xlim && fy[1] + yoff <= ylim;
        if (!__all_sync(0xffffffffu, (!v0 || i0) && (!v1 || i1))) {
          uint32_t a0, a1, b0, b1;
          f2split(WX1, a0, a1);
          f2split(WY1, b0, b1);
          if (v0)
            pt_pixel_generic<C, STAGED>(a, simg, win, t.cy0, t.sb0, true, (int)(fx[0] + xoff), (int)(fy[0] + yoff),
                                        __uint_as_float(a0), __uint_as_float(b0), o0);
          if (v1)
            pt_pixel_generic<C, STAGED>(a, simg, win, t.cy0, t.sb0, true, (int)(fx[1] + xoff), (int)(fy[1] + yoff),
                                        __uint_as_float(a1), __uint_as_float(b1), o0 + 32 * C);
          continue;
        }
        if (!v0) {
          fx[0] = safe_fx;
          fy[0] = safe_fy;
        }
        if (!v1) {
          fx[1] = safe_fx;
          fy[1] = safe_fy;
        }
      }
      // taps: NW aligned words per tap row, both rows share the byte shift
      uint32_t w[2][2][NW];  // [pixel][row][word]
      int sh[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if constexpr (STAGED) {
          const uint32_t o = SBM + fy[k] * (uint32_t)P + fx[k] * (uint32_t)C;
          sh[k] = (int)(o << 3);  // funnel shifts use the amount mod 32
          const uint32_t al = o & ~3u;
          FV_CHECK(al >= win && al + P + 4 * NW <= win + (uint32_t)(t.rows * P));
          lds_words(w[k][0], al);
          lds_words(w[k][1], al + P);
        } else {
          const uint32_t o = GBM + fy[k] * rp32 + fx[k] * (uint32_t)C;
          sh[k] = (int)(o << 3);
          const uint32_t* g0 = reinterpret_cast<const uint32_t*>(simg + (o & ~3u));
          const uint32_t* g1 = reinterpret_cast<const uint32_t*>(simg + (o & ~3u) + rp32);
#pragma unroll
          for (int i = 0; i < NW; ++i) {
            w[k][0][i] = __ldg(g0 + i);
            w[k][1][i] = __ldg(g1 + i);
          }
        }
      }
      uint32_t v00[2][C], v01[2][C], v10[2][C], v11[2][C];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        pt_taps<C>(w[k][0], sh[k], v00[k], v01[k]);
        pt_taps<C>(w[k][1], sh[k], v10[k], v11[k]);
      }
#if FV_PT_LERP
      // a = u00 + fx (u01 - u00) + 0.5, b likewise, v = a + fy (b - a): the
      // tap differences are exact on the magic words, u + 0.5 = M - (2^23 -
      // 0.5) exactly; each lerp rounds once (|error| < 2^-16 on the 0..256
      // scale, far inside the <= 1 LSB gate)
      const f2_t HM = f2(-8388607.5f, -8388607.5f);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const f2_t M00 = f2u(v00[0][c], v00[1][c]), M01 = f2u(v01[0][c], v01[1][c]);
        const f2_t M10 = f2u(v10[0][c], v10[1][c]), M11 = f2u(v11[0][c], v11[1][c]);
        const f2_t A = ffma2(WX1, ffma2(M00, NEG1, M01), fadd2(M00, HM));
        const f2_t B = ffma2(WX1, ffma2(M10, NEG1, M11), fadd2(M10, HM));
        const f2_t v = ffma2(WY1, ffma2(A, NEG1, B), A);
        uint32_t lo, hi;
        f2split(fadd2_rd(v, MAG), lo, hi);  // floor(v) in the low byte (0 <= v < 256)
        asm volatile("st.shared.u8 [%0], %1;" ::"r"(o0 + c), "r"(lo));
        if (v1) asm volatile("st.shared.u8 [%0], %1;" ::"r"(o0 + 32 * C + c), "r"(hi));
#else
      const f2_t WX0 = ffma2(WX1, NEG1, ONE), WY0 = ffma2(WY1, NEG1, ONE);
      const f2_t W00 = fmul2(WX0, WY0), W01 = fmul2(WX1, WY0), W10 = fmul2(WX0, WY1), W11 = fmul2(WX1, WY1);
      // first tap straight from its magic word M = 2^23 + u: C00 = 0.5 -
      // 2^23 W00 is exact for W00 >= 2^-24, so fma(M, W00, C00) = RN(u W00 + 0.5)
      const f2_t C00 = ffma2(W00, NMAG, HALF);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const f2_t A01 = fadd2(f2u(v01[0][c], v01[1][c]), NMAG);
        const f2_t A10 = fadd2(f2u(v10[0][c], v10[1][c]), NMAG), A11 = fadd2(f2u(v11[0][c], v11[1][c]), NMAG);
        const f2_t v = ffma2(A11, W11, ffma2(A10, W10, ffma2(A01, W01, ffma2(f2u(v00[0][c], v00[1][c]), W00, C00))));
        uint32_t lo, hi;
        f2split(fadd2_rd(v, MAG), lo, hi);  // floor(v) in the low byte (0 <= v < 256)
        asm volatile("st.shared.u8 [%0], %1;" ::"r"(o0 + c), "r"(lo));
        if (v1) asm volatile("st.shared.u8 [%0], %1;" ::"r"(o0 + 32 * C + c), "r"(hi));
#endif
      }
    }
    __syncwarp();
    // the row segment leaves with 16-byte stores
    uint8_t* d = dimg + (int64_t)y * a.d_rp + tx0 * C;
    const uint32_t rb = obw + (r & 1) * OB;
    if (pa.dst_vec && xbytes == OB) {
      for (int i = lane; i < OB / 16; i += 32) {
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(rb + 16 * i));
        *reinterpret_cast<uint4*>(d + 16 * i) = v;
      }
    } else {
      for (int i = lane; i < xbytes; i += 32) {
        uint32_t v;
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(rb + i));
        d[i] = (uint8_t)v;
      }
    }
  }
}

// Step 2 of the kernel, split around the CTA barrier. Lanes 0..4*PT_RPW-1:
// row r = lane / 4, group g = lane % 4 of this warp's rows.
struct PtAnchor {
  double sax, say;         // f64 map of the group's first pixel (absolute)
  float kx, ky, waf, iw;   // correction slopes, W_a, 1 / min |W| over the group
  float rho;               // (|W_a| + 31 |m6|) / min |W|
  float wef;               // W at the group's last pixel
  bool sign_ok;            // W keeps one strict sign over the group
};

__device__ __forceinline__ PtAnchor pt_anchor_map(const double* m, int tx0, int ty0, int warp, int lane) {
  PtAnchor p;
  p.sign_ok = false;
  if (lane < 4 * PT_RPW) {
    const int r = lane >> 2, g = lane & 3;
    const double yd = (double)(ty0 + warp + PT_NW * r), xd = (double)(tx0 + 32 * g);
    const double rx = m[1] * yd + m[2], ry = m[4] * yd + m[5];
    const double Wa = m[6] * xd + (m[7] * yd + m[8]);
    const double We = Wa + m[6] * 31.0;
    const double ra = __drcp_rn(Wa);
    p.sax = (m[0] * xd + rx) * ra;
    p.say = (m[3] * xd + ry) * ra;
    p.wef = (float)We;
    p.sign_ok = (Wa > 0.0 && We > 0.0) || (Wa < 0.0 && We < 0.0);
    p.kx = (float)(m[0] - p.sax * m[6]);
    p.ky = (float)(m[3] - p.say * m[6]);
    p.waf = (float)Wa;
    p.iw = __frcp_rn((float)fmin(fabs(Wa), fabs(We)));
    p.rho = (fabsf(p.waf) + 31.0f * fabsf((float)m[6])) * p.iw;
  }
  return p;
}

// Anchors written to slot (row, pair) as f32x2-ready pairs (group 2p, group
// 2p + 1) per field: {srx, sry, kx, ky, W_a, flags}; slot stride 12 words:
// the 16 writers of a field hit 16 distinct banks.
template <int C>
__device__ __forceinline__ void pt_anchor_store(const WarpArgs& a, const PtAnchor& p, const PtTile& t, bool staged,
                                                uint8_t* smem, int tx0, int warp, int lane) {
  if (lane < 4 * PT_RPW) {
    const int r = lane >> 2, g = lane & 3;
    const double dx = p.sax - (double)t.ox, dy = p.say - (double)t.oy;
    const bool fast = p.sign_ok && fabs(dx) < 1048576.0 && fabs(dy) < 1048576.0;  // false for NaN too
    const float srx = (float)dx, sry = (float)dy;
    int flags = 0;
    if (fast) {
      const float cx = fabsf(p.kx) * 31.0f * p.iw, cy = fabsf(p.ky) * 31.0f * p.iw;
      // u (Cmax (rho + 6) + 2 |s_rel|), with slack for the bound's own f32 roundings
      const float ex = 6.0e-8f * (cx * (p.rho + 7.0f) + 2.0f * fabsf(srx) + 1.0f);
      const float ey = 6.0e-8f * (cy * (p.rho + 7.0f) + 2.0f * fabsf(sry) + 1.0f);
      if (ex <= PT_MAX_ERR && ey <= PT_MAX_ERR) {  // false for inf / NaN
        flags = PG_F32;
        // the map is monotone along the group (W keeps its sign): its taps lie
        // between those of the first and last pixel. The last one from the
        // f32 correction s_a + 31 k / W_e (relative coordinates, |s| < 4200
        // px under the bound: within ~6e-4 px), offset in f64; 2e-3 px margins
        const float rex = __frcp_rn(p.wef);
        const float sex = __fmaf_rn(31.0f * p.kx, rex, srx), sey = __fmaf_rn(31.0f * p.ky, rex, sry);
        const double xl = (double)fminf(srx, sex) + (double)t.ox, xh = (double)fmaxf(srx, sex) + (double)t.ox;
        const double yl = (double)fminf(sry, sey) + (double)t.oy, yh = (double)fmaxf(sry, sey) + (double)t.oy;
        const int xlim = a.sw - (staged ? 2 : pt_xmargin<C, false>());
        if (tx0 + 32 * g + 31 < a.dw && xl >= 2e-3 && xh <= (double)(xlim + 1) - 2e-3 && yl >= 2e-3 &&
            yh <= (double)(a.sh - 1) - 2e-3)
          flags |= PG_INTERIOR;
      }
    }
    const uint32_t sl = smem_u32(smem) + PT_ANC_OFF + ((warp * PT_RPW * 2 + r * 2 + (g >> 1)) * 12 + (g & 1)) * 4;
    // 16 writers per store instruction (rows 0-3, then 4-7): distinct banks
#pragma unroll
    for (int hb = 0; hb < (PT_RPW + 3) / 4; ++hb) {
      if ((lane >> 4) == hb) {
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(sl), "f"(srx));
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(sl + 8), "f"(sry));
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(sl + 16), "f"(p.kx));
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(sl + 24), "f"(p.ky));
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(sl + 32), "f"(p.waf));
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(sl + 40), "r"(flags));
      }
    }
  }
}

template <int C>
__global__ void __launch_bounds__(PT_NW * 32, PT_MINB) warp_persp_tile_kernel(const __grid_constant__ WarpArgs a,
                                                                      const __grid_constant__ PtArgs pa,
                                                                      const __grid_constant__ WarpMats mats) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  PtTile* tile = reinterpret_cast<PtTile*>(smem + 16);
  uint8_t* win = smem + pt_win_off<C>();
  constexpr int P = pt_pitch<C>();
  constexpr int OB = pt_obuf<C>();
  const int n = blockIdx.z;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx0 = blockIdx.x * PT_TW, ty0 = blockIdx.y * PT_TH;
  const double* m = mats.m[n];
  const uint8_t* simg = reinterpret_cast<const uint8_t*>(a.src) + (int64_t)n * a.s_is;
  uint8_t* dimg = reinterpret_cast<uint8_t*>(a.dst) + (int64_t)n * a.d_is;

  // Step 2 (first half): the f64 anchor maps. Warps 1.. compute them while
  // warp 0 classifies the tile (they do not depend on the class); warp 0
  // after the barrier.
  PtAnchor ap;
  if (warp != 0) ap = pt_anchor_map(m, tx0, ty0, warp, lane);
  if (warp == 0) {
    const PtTile tt = pt_classify<C>(a, pa, m, tx0, ty0, lane);
    if (lane == 0) {
      *tile = tt;
      if (tt.cls == PT_STAGED) {
        mbar_init(bar, PT_NW);  // one arrive.expect_tx per warp
        fence_mbar_init();
      }
    }
  }
  __syncthreads();
  const PtTile t = *tile;
  if (t.cls == PT_BORDER) {  // CTA-uniform: no barrier follows
    const uint32_t braw = (uint32_t)a.border_raw;
    const uint32_t b4 = braw * 0x01010101u;
    const int xbytes = min(PT_TW, a.dw - tx0) * C;
#pragma unroll 1
    for (int r = 0; r < PT_RPW; ++r) {
      const int y = ty0 + warp + PT_NW * r;
      if (y >= a.dh) break;
      uint8_t* d = dimg + (int64_t)y * a.d_rp + tx0 * C;
      if (pa.dst_vec && xbytes == OB) {
        for (int i = lane; i < OB / 16; i += 32) *reinterpret_cast<uint4*>(d + 16 * i) = make_uint4(b4, b4, b4, b4);
      } else {
        for (int i = lane; i < xbytes; i += 32) d[i] = (uint8_t)braw;
      }
    }
    return;
  }
  const bool staged = t.cls == PT_STAGED;
  if (FV_PT_PF_MAX > 0 && !staged && pa.stage_ok && t.rows > 0 && t.rows * t.len <= FV_PT_PF_MAX) {
    // a DIRECT tile's gathers walk its box row by row, each step waiting
    // on DRAM: one bulk L2 prefetch per box row (one per thread) starts the
    // whole box's DRAM reads now, so the later steps hit L2
    const uint8_t* g = simg + (int64_t)t.cy0 * a.s_rp + t.sb0;
    for (int r = threadIdx.x; r < t.rows; r += PT_NW * 32)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g + (int64_t)r * a.s_rp), "r"((uint32_t)t.len)
                   : "memory");
  }
  if (warp == 0) ap = pt_anchor_map(m, tx0, ty0, warp, lane);
  if (staged) {  // every warp streams its share of the window's row segments (rows warp, warp + PT_NW, ...):
    // a bulk copy takes uniform operands, so one warp would issue the rows one at a time
    FV_CHECK(t.rows >= 1 && t.rows <= PT_WROWS && t.len >= 16 && t.len <= P - 16 && t.cy0 >= 0 &&
             t.cy0 + t.rows <= a.sh && t.sb0 >= 0 && t.sb0 + t.len <= a.sw * C);
    const int nr = max(0, (t.rows - warp + PT_NW - 1) / PT_NW);
    if (lane == 0) mbar_expect_tx(bar, (uint32_t)(nr * t.len));
    __syncwarp();
    const uint8_t* g = simg + (int64_t)t.cy0 * a.s_rp + t.sb0;
    for (int r = warp + PT_NW * lane; r < t.rows; r += PT_NW * 32)
      tma_bulk_g2s(win + r * P, g + (int64_t)r * a.s_rp, (uint32_t)t.len, bar);
  }

  // Step 2 (second half): anchors relative to the tile origin, flags, SMEM slots
  pt_anchor_store<C>(a, ap, t, staged, smem, tx0, warp, lane);
  __syncwarp();
  const uint32_t smem0 = smem_u32(smem);
  if (staged) {
    mbar_wait_block(bar, 0);
    pt_rows<C, true>(a, pa, t, m, simg, dimg, smem0, tx0, ty0, warp, lane);
  } else {
    pt_rows<C, false>(a, pa, t, m, simg, dimg, smem0, tx0, ty0, warp, lane);
  }
}

// 0 = launched; 1 = not applicable (caller takes another kernel); else error
template <int C>
static int launch_persp_tile_c(const WarpArgs& a, const PtArgs& pa, const WarpMats& mats, int nb, cudaStream_t st) {
  auto kern = warp_persp_tile_kernel<C>;
  constexpr int smem = pt_smem<C>();
  static unsigned long long attr_mask[2] = {0, 0};
  if (ensure_smem_attr(kern, smem, attr_mask) != FV_OK) return set_error(FV_ECUDA, "warp_persp_tile_kernel: smem attribute");
  dim3 grid((a.dw + PT_TW - 1) / PT_TW, (a.dh + PT_TH - 1) / PT_TH, nb);
  kern<<<grid, PT_NW * 32, smem, st>>>(a, pa, mats);
  return FV_OK;
}

int launch_persp_tile(const WarpArgs& a, const WarpMats& mats, int nb, cudaStream_t st) {
  PtArgs pa;
  const uintptr_t s = reinterpret_cast<uintptr_t>(a.src), d = reinterpret_cast<uintptr_t>(a.dst);
  pa.stage_ok = ((s | (uintptr_t)a.s_rp) & 15) == 0 && (nb <= 1 || (a.s_is & 15) == 0) &&
                (((int64_t)a.sw * a.c) & 15) == 0;
  pa.dst_vec = ((d | (uintptr_t)a.d_rp) & 15) == 0 && (nb <= 1 || (a.d_is & 15) == 0);
  if ((a.dh + PT_TH - 1) / PT_TH > 65535) return 1;
  switch (a.c) {
    case 1: return launch_persp_tile_c<1>(a, pa, mats, nb, st);
    case 3: return launch_persp_tile_c<3>(a, pa, mats, nb, st);
    case 4: return launch_persp_tile_c<4>(a, pa, mats, nb, st);
    default: return 1;
  }
}

}  // namespace fv
