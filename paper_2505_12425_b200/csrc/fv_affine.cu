// fv_affine.cu -- a8 warp_affine, SOURCE-tiled (round 2).
//
// Same contract and bits as the other affine kernels (fv_warp.cu header;
// oracle/fovea_oracle.py:warp_affine): sx = RN(RN(m0 x) + RN(RN(m1 y) + m2))
// in f64 (sy likewise), x0 = floor(sx), fx = f32(sx - x0), taps outside the
// source read the border, blend in imgproc.py:118-123 order.
//
// Why source tiles. A destination tile maps to a rotated parallelogram whose
// axis-aligned source box is 2-4x its footprint, and neighbouring tiles'
// boxes overlap: the round-1 kernel (32 x 16 destination tiles, a fixed 48 x
// 40 window) moved 3.1 GB of windows L2 -> SMEM for cfg2's 0.68 GB footprint
// and spent half its warp time waiting for them (profiles/r02c_ncu_affine).
// Here a CTA owns a SA_TW x 32 SOURCE tile instead (SA_TW = 60 for f32
// images): every destination pixel whose top-left tap (x0, y0) lies in the
// tile is sampled by this CTA, and its four taps lie in the (SA_TW + 1) x 33
// window -- one fixed-size 3-D TMA tensor copy (zero fill outside the image)
// -- so the source crosses L2 -> SMEM about once per byte.
//
// Ownership is decided per pixel by the exact f64 map: floor(sx) in
// [X0, X0 + SA_TW) and floor(sy) in [Y0, Y0 + 32). The tiles' ranges tile
// [-SA_TW, SA_TW (ntx - 1)) x [-32, 32 (nty - 1)), which holds every pixel
// with an in-image tap, so each destination pixel is owned by at most one
// tile; the rest (all taps outside the source) are written by the CTAs of
// grid column 0 (sa_outside_row) with the same test, in the same launch.
// Within a destination row the map is monotone (RN is), so the owned pixels
// of a row form an interval. The CTA finds its destination rows from the
// forward-mapped tile corners (+-1 row) and, one thread per row, each row's
// x interval from the inverse map (a superset: source-space margins of 1e-9
// relative dwarf the f64 roundings); a block scan compacts the non-empty
// rows into a table and the warps walk the flattened pixel list 64 indices
// at a time (full lanes however short the rows), each lane finding its row
// from one shared-memory load and two warp OR-reductions of the rows
// starting inside the step. The exact per-pixel test trims the intervals.
#include <cmath>

#include "fv_warp.cuh"

namespace fv {

// Window rows are a multiple of 128 bytes (32 banks): then a tap's bank
// depends on its column only, and the lanes of a warp -- consecutive
// destination pixels along a rotated source line -- collide only where two
// share a column (measured on cfg2's maps: 1.6 wavefronts per LDS against
// 2.3-3.4 for other pitches). Source tile: x0 range SA_TW (the window's
// (SA_TW + 1) pixels fit the row; X0 = SA_TW * k keeps the tensor copy's
// innermost start 16-byte aligned), y0 range SA_TH.
template <typename InT, int C>
constexpr int sa_box_elems() {  // window row in elements
  return sizeof(InT) == 4 ? (C == 1 ? 64 : (C == 3 ? 192 : 256)) : (C == 1 ? 128 : 256);
}
template <typename InT, int C>
constexpr int sa_tw() {
  return sizeof(InT) == 4 ? 60 : (C == 1 ? 112 : (C == 3 ? 80 : 60));
}
#ifndef FV_SA_TH
#define FV_SA_TH 32
#endif
constexpr int SA_TH = FV_SA_TH;  // A/B: 24 / 40 / 48
constexpr int SA_NW = 4;  // warps per CTA
#ifndef SA_MINB
#define SA_MINB 8
#endif
template <typename InT, int C>
constexpr bool sa_geometry_ok() {
  return (sa_tw<InT, C>() + 1) * C <= sa_box_elems<InT, C>() && (sa_tw<InT, C>() * C * (int)sizeof(InT)) % 16 == 0 &&
         (sa_box_elems<InT, C>() * (int)sizeof(InT)) % 128 == 0;
}
static_assert(sa_geometry_ok<float, 1>() && sa_geometry_ok<float, 3>() && sa_geometry_ok<float, 4>() &&
                  sa_geometry_ok<uint8_t, 1>() && sa_geometry_ok<uint8_t, 3>() && sa_geometry_ok<uint8_t, 4>(),
              "source-tile geometry");
template <typename InT, int C>
constexpr int sa_pitch() {
  return sa_box_elems<InT, C>() * (int)sizeof(InT);
}
constexpr int SA_WROWS = SA_TH + 1;

// Per-image constants from the host (f64): reciprocals of the inverse map's
// x coefficients (0 when the coefficient is 0) and the forward map's y row
// (destination y of a source point: f10 (sx - m2) + f11 (sy - m5)).
struct AffineAux {
  double r[MAXW][4];  // {1 / m0, 1 / m3, f10 = -m3 / det, f11 = m0 / det}
};

// x interval of destination row `y` (row terms rx, ry) whose pixels may map
// into [xlo, xhi) x [ylo, yhi) (source space): a superset (source-space
// margins of 1e-9 relative); empty when lo > hi. Integral doubles (may be
// +-inf); the caller clamps.
__device__ __forceinline__ void sa_row_span(double rm0, double rm3, double rx, double ry, double xlo, double xhi,
                                            double ylo, double yhi, double& lo, double& hi) {
  lo = -INFINITY;
  hi = INFINITY;
  const double ex = 1e-9 * (1.0 + fabs(xlo) + fabs(xhi) + fabs(rx));
  if (rm0 != 0.0) {
    const double a = (xlo - ex - rx) * rm0, b = (xhi + ex - rx) * rm0;
    lo = fmin(a, b);
    hi = fmax(a, b);
  } else if (!(rx >= xlo - ex && rx < xhi + ex)) {
    lo = INFINITY;
    hi = -INFINITY;
  }
  const double ey = 1e-9 * (1.0 + fabs(ylo) + fabs(yhi) + fabs(ry));
  if (rm3 != 0.0) {
    const double a = (ylo - ey - ry) * rm3, b = (yhi + ey - ry) * rm3;
    lo = fmax(lo, fmin(a, b));
    hi = fmin(hi, fmax(a, b));
  } else if (!(ry >= ylo - ey && ry < yhi + ey)) {
    lo = INFINITY;
    hi = -INFINITY;
  }
  // integer bounds: the margins ex, ey dwarf the roundings of the product
  // with the reciprocal (<= 2 ulp relative) and of the per-pixel map, so
  // every owned x lies in [ceil(lo), floor(hi)]
  lo = ceil(lo);
  hi = floor(hi);
}

// Bilinear blend of two pixels (pixel k -> d[k] when ok[k]) from raw taps,
// the imgproc.py:118-123 order with every product and sum rounded (sums as
// fma(q, runtime 1, p): fv_common.cuh's contraction note); u8 results take
// the app.py:75-77 epilogue.
template <typename InT, int C>
__device__ __forceinline__ void sa_blend_store(const WarpArgs& a, const float (&wx1)[2], const float (&wy1)[2],
                                               const uint32_t (&v00)[2][C], const uint32_t (&v01)[2][C],
                                               const uint32_t (&v10)[2][C], const uint32_t (&v11)[2][C],
                                               InT* d0, InT* d1, bool ok0, bool ok1) {
  const f2_t ONE = a.one2;
  const f2_t WX1 = f2(wx1[0], wx1[1]), WY1 = f2(wy1[0], wy1[1]);
  const f2_t WX0 = f2(__fsub_rn(1.0f, wx1[0]), __fsub_rn(1.0f, wx1[1]));
  const f2_t WY0 = f2(__fsub_rn(1.0f, wy1[0]), __fsub_rn(1.0f, wy1[1]));
#pragma unroll
  for (int c = 0; c < C; ++c) {
    f2_t t00, t01, t10, t11;
    if constexpr (sizeof(InT) == 1) {
      t00 = unit2(v00[0][c], v00[1][c]);
      t01 = unit2(v01[0][c], v01[1][c]);
      t10 = unit2(v10[0][c], v10[1][c]);
      t11 = unit2(v11[0][c], v11[1][c]);
    } else {
      t00 = f2u(v00[0][c], v00[1][c]);
      t01 = f2u(v01[0][c], v01[1][c]);
      t10 = f2u(v10[0][c], v10[1][c]);
      t11 = f2u(v11[0][c], v11[1][c]);
    }
    const f2_t top = ffma2(fmul2(t01, WX1), ONE, fmul2(t00, WX0));
    const f2_t bot = ffma2(fmul2(t11, WX1), ONE, fmul2(t10, WX0));
    const f2_t o = ffma2(fmul2(bot, WY1), ONE, fmul2(top, WY0));
    uint32_t lo, hi;
    if constexpr (sizeof(InT) == 1) {
      f2split(scale_to_u8_bits2(o, 255.0f), lo, hi);
      if (ok0) d0[c] = (InT)(lo & 0xFF);
      if (ok1) d1[c] = (InT)(hi & 0xFF);
    } else {
      f2split(o, lo, hi);
      if (ok0) d0[c] = __uint_as_float(lo);
      if (ok1) d1[c] = __uint_as_float(hi);
    }
  }
}

// raw tap at SMEM address `addr`: u8 -> magic word 0x4B0000uu, f32 -> bits
template <typename InT>
__device__ __forceinline__ uint32_t sa_lds(uint32_t addr) {
  uint32_t v;
  if constexpr (sizeof(InT) == 1) {
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return 0x4B000000u | v;
  } else {
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
  }
}

// The exact map of pixel (x, row terms rx, ry): f64 source coordinates.
__device__ __forceinline__ void sa_map(const double (&m)[9], int x, double rx, double ry, double& sx, double& sy) {
  const double xd = (double)x;
  sx = __dadd_rn(__dmul_rn(m[0], xd), rx);
  sy = __dadd_rn(__dmul_rn(m[3], xd), ry);
}

// Block-wide inclusive scan of two ints over the CTA's SA_NW warps.
__device__ __forceinline__ int2 sa_block_scan(int2 v, int lane, int warp, int2* wsum) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, v.x, d), b = __shfl_up_sync(0xffffffffu, v.y, d);
    if (lane >= d) {
      v.x += a;
      v.y += b;
    }
  }
  if (lane == 31) wsum[warp] = v;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < SA_NW - 1; ++w) {
    if (w < warp) {
      v.x += wsum[w].x;
      v.y += wsum[w].y;
    }
  }
  return v;
}

// Row of the CTA's flattened pixel index base + lane (lanes of one 32-index
// step). Rows are compacted (every row holds >= 1 pixel), so the rows that
// start inside the step start at distinct positions: one bit each in M.
// `r0` = the row holding index `base`; returns the lane's row and advances
// r0 to the row holding base + 32.
__device__ __forceinline__ int sa_row_of(const int* off, int nne, int base, int lane, int& r0) {
  const int j = r0 + 1 + lane;
  const int o = j <= nne ? off[j] : 0x7fffffff;
  const int p = o - base;  // >= 1
  const uint32_t bit = p < 32 ? (1u << p) : 0u;
  const uint32_t M = __reduce_or_sync(0xffffffffu, bit);
  const int row = r0 + __popc(M & ((2u << lane) - 1u));
  r0 += __popc(M) + (__any_sync(0xffffffffu, p == 32) ? 1 : 0);
  return row;
}
// The same for the 64 indices base + lane (row A) and base + 32 + lane (row
// B): up to 32 rows start inside a 64-index step only if each is short, so
// the lanes cover the next 32 row starts and a step holding more than 32
// starts (rows of 1-2 px) falls back to two 32-index lookups.
__device__ __forceinline__ void sa_rows_of64(const int* off, int nne, int base, int lane, int& r0, int& ra, int& rb) {
  const int j = r0 + 1 + lane;
  const int o = j <= nne ? off[j] : 0x7fffffff;
  const int p = o - base;  // >= 1
  if (__all_sync(0xffffffffu, p < 64)) {  // the 32nd next start is inside: > 32 may be (warp-uniform)
    ra = sa_row_of(off, nne, base, lane, r0);
    rb = sa_row_of(off, nne, base + 32, lane, r0);
    return;
  }
  const uint32_t lo = __reduce_or_sync(0xffffffffu, p < 32 ? (1u << p) : 0u);
  const uint32_t hi = __reduce_or_sync(0xffffffffu, (p >= 32 && p < 64) ? (1u << (p - 32)) : 0u);
  const uint32_t below = (2u << lane) - 1u;
  ra = r0 + __popc(lo & below);
  rb = r0 + __popc(lo) + __popc(hi & below);
  r0 += __popc(lo) + __popc(hi) + (__any_sync(0xffffffffu, p == 64) ? 1 : 0);
}

// SMEM layout of the source-tiled kernel
constexpr int SA_MAXR = SA_NW * 32;                 // destination rows per batch (one per thread)
constexpr int SA_OFF = 64;                          // int off[SA_MAXR + 1]
// row entries, 32 B: {x - index, byte offset of (row, x - index) in the image (64-bit), pad, rx, ry}
constexpr int SA_TAB = (SA_OFF + 4 * (SA_MAXR + 1) + 127) / 128 * 128;
constexpr int SA_WIN = SA_TAB + 32 * SA_MAXR;       // the window (128-byte aligned)
template <typename InT, int C>
constexpr int sa_smem2() {
  return SA_WIN + sa_pitch<InT, C>() * SA_WROWS;
}
static_assert(SA_WIN % 128 == 0, "window alignment");

// Destination pixels owned by no tile (every tap outside the source, or a
// non-finite map): the blend of four border taps (raw border when the map is
// not finite), exactly as the other kernels compute it. One warp per
// destination row: pixels outside the row's superset interval of the tile
// grid are unowned without a test (+0 stores for a +0 border); the interval's
// ends take the exact ownership test, chunk by chunk inwards until a chunk
// holds an owned pixel (the owned pixels of a row form an interval).
template <typename InT, int C>
__device__ __forceinline__ void sa_outside_chunk(const WarpArgs& a, const double (&m)[9], double rx, double ry,
                                                 double gx0, double gx1, double gy0, double gy1, InT* d, int x,
                                                 bool in_range, bool test, uint32_t bord, bool& any_owned) {
  double sx, sy;
  sa_map(m, x, rx, ry, sx, sy);
  const bool owned = test && sx >= gx0 && sx < gx1 && sy >= gy0 && sy < gy1;
  any_owned = __any_sync(0xffffffffu, in_range && owned);
  const bool out = in_range && !owned;
  if (a.zero_border) {
    if (out)
#pragma unroll
      for (int c = 0; c < C; ++c) d[x * C + c] = (InT)0;
    return;
  }
  const bool fin = isfinite(sx) && isfinite(sy);
  const double fx = floor(sx), fy = floor(sy);
  const float wx1[2] = {fin ? __double2float_rn(__dadd_rn(sx, -fx)) : 0.0f, 0.0f};
  const float wy1[2] = {fin ? __double2float_rn(__dadd_rn(sy, -fy)) : 0.0f, 0.0f};
  uint32_t v[2][C];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int c = 0; c < C; ++c) v[p][c] = bord;
  sa_blend_store<InT, C>(a, wx1, wy1, v, v, v, v, d + x * C, d, out && fin, false);
  if (out && !fin)
#pragma unroll
    for (int c = 0; c < C; ++c) d[x * C + c] = (InT)a.border_raw;
}

// bytes [b0, b1) of a row to 0: 16-byte stores in the aligned middle
__device__ __forceinline__ void sa_zero_bytes(char* row, int b0, int b1, int lane) {
  if (b0 >= b1) return;
  const int mis = (int)(reinterpret_cast<uintptr_t>(row) & 15);
  int a0 = ((b0 + mis + 15) & ~15) - mis, a1 = ((b1 + mis) & ~15) - mis;  // aligned middle [a0, a1)
  if (a0 > a1) a0 = a1 = b1;
  for (int b = b0 + lane; b < a0; b += 32) row[b] = 0;
  for (int b = a1 + lane; b < b1; b += 32) row[b] = 0;
  for (int b = a0 + 16 * lane; b < a1; b += 512) *reinterpret_cast<uint4*>(row + b) = make_uint4(0, 0, 0, 0);
}

template <typename InT, int C>
__device__ __forceinline__ void sa_outside_row(const WarpArgs& a, const double (&m)[9], double rm0, double rm3, int n,
                                               int y, int lane, double gx0, double gx1, double gy0, double gy1) {
  const double yd = (double)y;
  const double rx = __dadd_rn(__dmul_rn(m[1], yd), m[2]);
  const double ry = __dadd_rn(__dmul_rn(m[4], yd), m[5]);
  double lo, hi;
  sa_row_span(rm0, rm3, rx, ry, gx0, gx1, gy0, gy1, lo, hi);
  int xs = a.dw, xe = a.dw - 1;  // superset of the owned pixels (empty by default)
  if (lo <= hi && hi >= 0.0 && lo <= (double)(a.dw - 1)) {
    xs = (int)fmax(lo, 0.0);
    xe = (int)fmin(hi, (double)(a.dw - 1));
  }
  InT* d = reinterpret_cast<InT*>(reinterpret_cast<char*>(a.dst) + (int64_t)n * a.d_is + (int64_t)y * a.d_rp);
  const uint32_t bord = sizeof(InT) == 1 ? (0x4B000000u | (uint32_t)a.border_raw) : __float_as_uint(a.border_f);
  bool any;
  // outside the superset: unowned (a +0 border: +0 bytes, no map)
  if (a.zero_border) {
    constexpr int PB = C * (int)sizeof(InT);
    sa_zero_bytes(reinterpret_cast<char*>(d), 0, min(xs, a.dw) * PB, lane);
    sa_zero_bytes(reinterpret_cast<char*>(d), max(xe + 1, 0) * PB, a.dw * PB, lane);
  } else {
    // warp-uniform trip counts: sa_outside_chunk votes over the full warp
    const int xr = max(xe + 1, 0);
#pragma unroll 1
    for (int x0 = 0; x0 < xs; x0 += 32)
      sa_outside_chunk<InT, C>(a, m, rx, ry, gx0, gx1, gy0, gy1, d, x0 + lane, x0 + lane < xs, false, bord, any);
#pragma unroll 1
    for (int x0 = xr; x0 < a.dw; x0 += 32)
      sa_outside_chunk<InT, C>(a, m, rx, ry, gx0, gx1, gy0, gy1, d, x0 + lane, x0 + lane < a.dw, false, bord, any);
  }
  // the superset's ends, inwards until an owned pixel
#pragma unroll 1
  for (int x0 = xs; x0 <= xe; x0 += 32) {
    sa_outside_chunk<InT, C>(a, m, rx, ry, gx0, gx1, gy0, gy1, d, x0 + lane, x0 + lane <= xe, true, bord, any);
    if (any) break;
  }
#pragma unroll 1
  for (int x1 = xe; x1 >= xs; x1 -= 32) {
    sa_outside_chunk<InT, C>(a, m, rx, ry, gx0, gx1, gy0, gy1, d, x1 - lane, x1 - lane >= xs, true, bord, any);
    if (any) break;
  }
}

template <typename InT, int C>
__global__ void __launch_bounds__(SA_NW * 32, SA_MINB) warp_affine_src_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                       const __grid_constant__ WarpArgs a,
                                                                       const __grid_constant__ WarpMats mats,
                                                                       const __grid_constant__ AffineAux aux) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  int2* wsum = reinterpret_cast<int2*>(smem + 16);    // scan: warp totals
  int* shared_n = reinterpret_cast<int*>(smem + 48);  // {total, rows}
  int* off = reinterpret_cast<int*>(smem + SA_OFF);
  constexpr int ES = (int)sizeof(InT), PB = C * ES, P = sa_pitch<InT, C>();
  const int n = blockIdx.z;
  constexpr int SA_TW = sa_tw<InT, C>();
  const int X0 = SA_TW * ((int)blockIdx.x - 2), Y0 = SA_TH * ((int)blockIdx.y - 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double m[9];
#pragma unroll
  for (int i = 0; i < 6; ++i) m[i] = mats.m[n][i];
  m[6] = m[7] = m[8] = 0.0;
  if (blockIdx.x == 0) {  // grid column 0: the pixels no tile owns, rows [by * R, by * R + R)
    const double gx0 = -SA_TW, gx1 = (double)SA_TW * (gridDim.x - 2), gy0 = -SA_TH, gy1 = (double)SA_TH * (gridDim.y - 1);
    const int R = (a.dh + gridDim.y - 1) / gridDim.y;
    const int yend = min(a.dh, ((int)blockIdx.y + 1) * R);
#pragma unroll 1
    for (int y = (int)blockIdx.y * R + warp; y < yend; y += SA_NW)
      sa_outside_row<InT, C>(a, m, aux.r[n][0], aux.r[n][1], n, y, lane, gx0, gx1, gy0, gy1);
    return;
  }
  // destination rows of the tile: forward map (inverse of the 2x2) of the
  // source rectangle's corners, +-1 row
  const double rm0 = aux.r[n][0], rm3 = aux.r[n][1], i10 = aux.r[n][2], i11 = aux.r[n][3];
  const double xlo = (double)X0, xhi = (double)(X0 + SA_TW), ylo = (double)Y0, yhi = (double)(Y0 + SA_TH);
  // (linear in the corner: the extremes are the corner terms' signs)
  const double y00 = i10 * (xlo - m[2]) + i11 * (ylo - m[5]);
  const double ex = i10 * (double)SA_TW, ey = i11 * (double)SA_TH;
  const double dyl = y00 + (ex < 0.0 ? ex : 0.0) + (ey < 0.0 ? ey : 0.0);
  const double dyh = y00 + (ex > 0.0 ? ex : 0.0) + (ey > 0.0 ? ey : 0.0);
  double yl = floor(dyl) - 1.0, yh = ceil(dyh) + 1.0;
  yl = yl > 0.0 ? yl : 0.0;
  yh = yh < (double)(a.dh - 1) ? yh : (double)(a.dh - 1);
  if (!(yl <= yh)) return;  // CTA-uniform (also NaN)
  const int ry0 = (int)yl, ry1 = (int)yh;
  const bool inner = X0 >= 0 && X0 + SA_TW < a.sw && Y0 >= 0 && Y0 + SA_TH < a.sh;
  const uint32_t win = smem_u32(smem) + SA_WIN;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_expect_tx(bar, (uint32_t)(P * SA_WROWS));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(win),
        "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(X0 * C), "r"(Y0), "r"(n), "r"(smem_u32(bar))
        : "memory");
  }
  const uint32_t bord = sizeof(InT) == 1 ? (0x4B000000u | (uint32_t)a.border_raw) : __float_as_uint(a.border_f);
  char* dbase = reinterpret_cast<char*>(a.dst) + (int64_t)n * a.d_is;
  bool waited = false;
#pragma unroll 1
  for (int rb = ry0; rb <= ry1; rb += SA_MAXR) {
    // 1. this thread's destination row: its x interval (a superset of the
    //    owned pixels), compacted into the row table by a block scan
    const int y = rb + tid;
    int xs = 0, cnt = 0;
    double rx = 0.0, ry = 0.0;
    if (y <= ry1) {
      const double yd = (double)y;
      rx = __dadd_rn(__dmul_rn(m[1], yd), m[2]);
      ry = __dadd_rn(__dmul_rn(m[4], yd), m[5]);
      double lo, hi;
      sa_row_span(rm0, rm3, rx, ry, xlo, xhi, ylo, yhi, lo, hi);
      lo = fmax(lo, 0.0);
      hi = fmin(hi, (double)(a.dw - 1));
      if (lo <= hi) {
        xs = (int)lo;
        cnt = (int)hi - xs + 1;
      }
    }
    const int2 inc = sa_block_scan(make_int2(cnt, cnt > 0 ? 1 : 0), lane, warp, wsum);
    if (cnt > 0) {
      const int k = inc.y - 1, o = inc.x - cnt;
      off[k] = o;
      // {x - index, row's byte offset minus the index's (x = index: 0), rx, ry}
      const long long rbo = (long long)y * a.d_rp + (long long)(xs - o) * PB;
      int4* e = reinterpret_cast<int4*>(smem + SA_TAB + 32 * k);
      e[0] = make_int4(xs - o, (int)(unsigned long long)rbo, (int)((unsigned long long)rbo >> 32), 0);
      e[1] = make_int4(__double2loint(rx), __double2hiint(rx), __double2loint(ry), __double2hiint(ry));
    }
    if (tid == SA_MAXR - 1) {
      shared_n[0] = inc.x;
      shared_n[1] = inc.y;
      off[inc.y] = inc.x;
    }
    __syncthreads();
    const int total = shared_n[0], nne = shared_n[1];
    if (!waited) {
      mbar_wait_block(bar, 0);
      waited = true;
    }
    // 2. the flattened pixels: warp w takes a contiguous run of 64-index
    //    steps; lane l samples indices base + l (A) and base + 32 + l (B)
    const int nsteps = (total + 63) >> 6, per = (nsteps + SA_NW - 1) / SA_NW;
    const int s0 = warp * per, s1 = min(nsteps, s0 + per);
    int r0 = 0;
    if (s0 < s1) {  // the row holding index 64 * s0
      int le = 0;  // rows starting at or before the index (off[0] = 0)
#pragma unroll 1
      for (int j0 = 0; j0 < nne; j0 += 32) le += __popc(__ballot_sync(0xffffffffu, j0 + lane < nne && off[j0 + lane] <= 64 * s0));
      r0 = le - 1;
    }
#pragma unroll 1
    for (int s = s0; s < s1; ++s) {
      int x[2];
      long long dof[2];
      bool own[2];
      float wx1[2], wy1[2];
      int ox[2], oy[2];
      int rows[2];
      sa_rows_of64(off, nne, 64 * s, lane, r0, rows[0], rows[1]);
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int i = 64 * s + 32 * p + lane;
        const bool valid = i < total;
        const uint8_t* ep = smem + SA_TAB + 32 * (valid ? rows[p] : 0);
        const int4 e0 = *reinterpret_cast<const int4*>(ep);
        const int4 e1 = *reinterpret_cast<const int4*>(ep + 16);
        x[p] = i + e0.x;
        dof[p] = (long long)(((unsigned long long)(unsigned)e0.z << 32) | (unsigned)e0.y) + (long long)i * PB;
        const double rx_ = __hiloint2double(e1.y, e1.x), ry_ = __hiloint2double(e1.w, e1.z);
        double sx, sy;
        sa_map(m, x[p], rx_, ry_, sx, sy);
        // floor on the FP64 pipe instead of the conversion unit: RD(s + 1.5 *
        // 2^52) = 1.5 * 2^52 + floor(s) exactly for |s| < 2^51 (an enumerated
        // pixel's map lies within a few tile widths of the tile: its row
        // interval is a superset of the owned pixels by 1e-9 relative), its
        // low word is floor(s) as an int, and subtracting the magic back is
        // exact (cfg2: 0.303 -> 0.298 ms)
        const double MF = 6755399441055744.0;  // 1.5 * 2^52
        const double tx = __dadd_rd(sx, MF), ty = __dadd_rd(sy, MF);
        const int fxi = __double2loint(tx), fyi = __double2loint(ty);
        // owned: X0 <= sx < X0 + SA_TW and likewise y, i.e. floor(sx) in
        // [X0, X0 + SA_TW) (X0 integral)
        ox[p] = (int)((unsigned)fxi - (unsigned)X0);
        oy[p] = (int)((unsigned)fyi - (unsigned)Y0);
        own[p] = valid && (unsigned)ox[p] < (unsigned)SA_TW && (unsigned)oy[p] < (unsigned)SA_TH;
        wx1[p] = __double2float_rn(__dadd_rn(sx, -__dadd_rn(tx, -MF)));
        wy1[p] = __double2float_rn(__dadd_rn(sy, -__dadd_rn(ty, -MF)));
        if (!own[p]) {
          ox[p] = 0;
          oy[p] = 0;
        }
      }
      uint32_t v00[2][C], v01[2][C], v10[2][C], v11[2][C];
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const uint32_t o = win + (uint32_t)(oy[p] * P + ox[p] * PB);
        FV_CHECK(!own[p] || (ox[p] >= 0 && ox[p] < SA_TW && oy[p] >= 0 && oy[p] < SA_TH));
#pragma unroll
        for (int c = 0; c < C; ++c) {
          v00[p][c] = sa_lds<InT>(o + c * ES);
          v01[p][c] = sa_lds<InT>(o + PB + c * ES);
          v10[p][c] = sa_lds<InT>(o + P + c * ES);
          v11[p][c] = sa_lds<InT>(o + P + PB + c * ES);
        }
        if (!inner) {  // CTA-uniform: taps outside the source read the border
          const int tx = X0 + ox[p], ty = Y0 + oy[p];
          const bool ix0 = tx >= 0 && tx < a.sw, ix1 = tx + 1 >= 0 && tx + 1 < a.sw;
          const bool iy0 = ty >= 0 && ty < a.sh, iy1 = ty + 1 >= 0 && ty + 1 < a.sh;
#pragma unroll
          for (int c = 0; c < C; ++c) {
            v00[p][c] = (iy0 && ix0) ? v00[p][c] : bord;
            v01[p][c] = (iy0 && ix1) ? v01[p][c] : bord;
            v10[p][c] = (iy1 && ix0) ? v10[p][c] : bord;
            v11[p][c] = (iy1 && ix1) ? v11[p][c] : bord;
          }
        }
      }
      InT* d0 = reinterpret_cast<InT*>(dbase + dof[0]);
      InT* d1 = reinterpret_cast<InT*>(dbase + dof[1]);
      sa_blend_store<InT, C>(a, wx1, wy1, v00, v01, v10, v11, d0, d1, own[0], own[1]);
    }
    __syncthreads();  // the row table is rewritten by the next batch
  }
}

// 0 = launched, 1 = not applicable (caller takes another kernel), else error
template <typename InT, int C>
static int launch_affine_src_c(const WarpArgs& a, const WarpMats& mats, int nb, cudaStream_t st) {
  auto enc = tensor_map_encoder();
  if (!enc) return 1;
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)a.sw * C, (cuuint64_t)a.sh, (cuuint64_t)nb};
  const cuuint64_t strides[2] = {(cuuint64_t)a.s_rp, (cuuint64_t)(nb > 1 ? a.s_is : a.s_rp * a.sh)};
  constexpr int SA_TW = sa_tw<InT, C>();
  const cuuint32_t boxd[3] = {(cuuint32_t)sa_box_elems<InT, C>(), (cuuint32_t)SA_WROWS, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (enc(&tm, sizeof(InT) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
          const_cast<void*>(a.src), dims, strides, boxd, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 1;
  const int ntx = (a.sw + SA_TW - 1) / SA_TW + 1, nty = (a.sh + SA_TH - 1) / SA_TH + 1;
  if (nty > 65535 || (a.dh + 7) / 8 > 65535) return 1;
  AffineAux aux;
  for (int i = 0; i < nb; ++i) {
    const double* m = mats.m[i];
    const double det = m[0] * m[4] - m[1] * m[3];
    aux.r[i][0] = m[0] != 0.0 ? 1.0 / m[0] : 0.0;
    aux.r[i][1] = m[3] != 0.0 ? 1.0 / m[3] : 0.0;
    aux.r[i][2] = -m[3] / det;
    aux.r[i][3] = m[0] / det;
  }
  auto kern = warp_affine_src_kernel<InT, C>;
  constexpr int smem = sa_smem2<InT, C>();
  static unsigned long long attr_mask[2] = {0, 0};
  if (ensure_smem_attr(kern, smem, attr_mask) != FV_OK) return check_launch("warp_affine_src_kernel (smem attribute)");
  kern<<<dim3(ntx + 1, nty, nb), SA_NW * 32, smem, st>>>(tm, a, mats, aux);  // column 0: the outside pass
  return check_launch("warp_affine_src_kernel");
}

int launch_affine_src(const WarpArgs& a, const WarpMats& mats, int nb, int es, cudaStream_t st) {
  // finite maps with a bounded zoom-out only: a 32 x 32 source tile should
  // hold a few hundred destination pixels (|det| <= 4), else the
  // destination-tiled kernel wastes less of its window
  for (int i = 0; i < nb; ++i) {
    const double* m = mats.m[i];
    bool fin = true;
    for (int j = 0; j < 6; ++j) fin = fin && std::isfinite(m[j]);
    const double det = m[0] * m[4] - m[1] * m[3];
    if (!fin || !(std::fabs(det) <= 4.0 && std::fabs(det) >= 1e-6)) return 1;
    for (int j = 0; j < 6; ++j)
      if (std::fabs(m[j]) > 1e7) return 1;
  }
  if (es == 4) {
    switch (a.c) {
      case 1: return launch_affine_src_c<float, 1>(a, mats, nb, st);
      case 3: return launch_affine_src_c<float, 3>(a, mats, nb, st);
      case 4: return launch_affine_src_c<float, 4>(a, mats, nb, st);
    }
  } else {
    switch (a.c) {
      case 1: return launch_affine_src_c<uint8_t, 1>(a, mats, nb, st);
      case 3: return launch_affine_src_c<uint8_t, 3>(a, mats, nb, st);
      case 4: return launch_affine_src_c<uint8_t, 4>(a, mats, nb, st);
    }
  }
  return 1;
}

}  // namespace fv
