// fv_warp.cu -- a8 warp_affine / a9 warp_perspective, bilinear, constant
// border. The reference has neither; the contract is the
// builder's (oracle/fovea_oracle.py:warp_affine/_perspective),
// written in the reference's conventions:
//   * pixel (x, y) has its centre at integer (x, y) (imgproc.py:8-13);
//   * the host passes the per-image INVERSE matrix (dst -> src) in f64;
//   * sx = m0*x + (m1*y + m2) etc. in f64, each op rounded (__d*_rn: the
//     per-row term is hoisted, the per-pixel cost is one DMUL + one DADD per
//     coordinate); perspective: W == 0 or non-finite -> raw border, else
//     r = RN(1/W) (__drcp_rn), sx = X*r, sy = Y*r;
//   * x0 = floor(sx), fx = f32(sx - x0); each of the four taps outside the
//     source reads the border value; blend in imgproc.py:118-123 order;
//   * u8 images use the _resize_u8 recipe (app.py:64-78).
// Output is bit-identical to the oracle.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>

#include "fv_warp.cuh"

namespace fv {

constexpr int WARP_ROWS = 4;  // rows per thread in warp_kernel
#ifndef WK_MINB
#define WK_MINB 4  // warp_kernel: resident CTAs per SM the register budget is sized for
#endif

template <typename T>
__device__ __forceinline__ T to_out(float v);
template <>
__device__ __forceinline__ float to_out<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ uint8_t to_out<uint8_t>(float v) {
  return (uint8_t)unit_to_u8(v);
}

// every tap of the pixel outside the source, or a non-finite map: the
// gather's all-border case (gather_raw)
__device__ __forceinline__ bool tap_outside(const WarpTap& t, int sw, int sh) {
  return !t.finite || t.x0 < -1 || t.x0 >= sw || t.y0 < -1 || t.y0 >= sh;
}

// Raw taps of the two source pixels (x0, x0+1) of one row, all C channels:
// u8 -> magic words 0x4B0000uu (converted later, two at a time), f32 -> bits.
// u8, C = 3: three aligned 32-bit loads + two funnel shifts instead of six
// byte loads.
// SAFE: the caller guarantees x0 <= sw - kPairSafe<InT, C> (the wide window
// ends inside the row), so the in-row test and its per-element fallback --
// which ptxas if-converts into every gather -- are left out.
template <typename InT, int C>
constexpr int kPairSafe = (C == 3) ? (sizeof(InT) == 1 ? 4 : 3) : 2;  // generic: x0 + 1 < sw

template <typename InT, int C, bool SAFE = false>
__device__ __forceinline__ void load_pair_raw(const InT* row, int x0, int row_elems, uint32_t (&t0)[C],
                                              uint32_t (&t1)[C]) {
  if constexpr (sizeof(InT) == 1 && C == 3) {
    const uintptr_t p = reinterpret_cast<uintptr_t>(row) + 3 * x0;
    const uintptr_t al = p & ~(uintptr_t)3;
    if (SAFE || al + 12 <= reinterpret_cast<uintptr_t>(row) + row_elems) {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(al);
      const uint32_t w0 = __ldg(w), w1 = __ldg(w + 1), w2 = __ldg(w + 2);
      const int sh = (int)(p & 3) * 8;
      uint32_t v[2];
      v[0] = __funnelshift_r(w0, w1, sh);
      v[1] = __funnelshift_r(w1, w2, sh);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        t0[c] = magic_of(v, c);
        t1[c] = magic_of(v, 3 + c);
      }
      return;
    }
  }
  if constexpr (sizeof(InT) == 4 && C == 3) {
    // six consecutive floats at byte 12*x0: four aligned 8-byte loads cover
    // them for either 8-byte phase (4 LSU requests instead of 6)
    const uintptr_t p = reinterpret_cast<uintptr_t>(row) + 12 * x0;
    const uintptr_t al = p & ~(uintptr_t)7;
    if (SAFE || al + 32 <= reinterpret_cast<uintptr_t>(row) + 4 * row_elems) {
      const uint2* w = reinterpret_cast<const uint2*>(al);
      const uint2 q0 = __ldg(w), q1 = __ldg(w + 1), q2 = __ldg(w + 2), q3 = __ldg(w + 3);
      const uint32_t v[8] = {q0.x, q0.y, q1.x, q1.y, q2.x, q2.y, q3.x, q3.y};
      const bool odd = (p & 7) != 0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        t0[c] = odd ? v[c + 1] : v[c];
        t1[c] = odd ? v[c + 4] : v[c + 3];
      }
      return;
    }
  }
#pragma unroll
  for (int c = 0; c < C; ++c) {
    if constexpr (sizeof(InT) == 1) {
      t0[c] = 0x4B000000u | __ldg(row + x0 * C + c);
      t1[c] = 0x4B000000u | __ldg(row + (x0 + 1) * C + c);
    } else {
      t0[c] = __float_as_uint(__ldg(row + x0 * C + c));
      t1[c] = __float_as_uint(__ldg(row + (x0 + 1) * C + c));
    }
  }
}

template <typename InT, int C>
__device__ __forceinline__ void gather_raw(const WarpArgs& a, int n, const WarpTap& t, uint32_t bord,
                                           uint32_t (&t00)[C], uint32_t (&t01)[C], uint32_t (&t10)[C],
                                           uint32_t (&t11)[C]) {
  const bool inx = t.x0 >= 0 && t.x0 + 1 < a.sw, iny = t.y0 >= 0 && t.y0 + 1 < a.sh;
  const bool outside = tap_outside(t, a.sw, a.sh);
  if (inx && iny) {
    const InT* r0 = row_ptr<InT>(a.src, a.s_is, a.s_rp, n, t.y0);
    const InT* r1 = row_ptr<InT>(a.src, a.s_is, a.s_rp, n, t.y0 + 1);
    load_pair_raw<InT, C>(r0, t.x0, a.sw * C, t00, t01);
    load_pair_raw<InT, C>(r1, t.x0, a.sw * C, t10, t11);
  } else if (outside) {  // every tap reads the border
#pragma unroll
    for (int c = 0; c < C; ++c) t00[c] = t01[c] = t10[c] = t11[c] = bord;
  } else {
    const bool ix0 = t.x0 >= 0 && t.x0 < a.sw, ix1 = t.x0 + 1 >= 0 && t.x0 + 1 < a.sw;
    const bool iy0 = t.y0 >= 0 && t.y0 < a.sh, iy1 = t.y0 + 1 >= 0 && t.y0 + 1 < a.sh;
    const InT* r0 = row_ptr<InT>(a.src, a.s_is, a.s_rp, n, iy0 ? t.y0 : 0);
    const InT* r1 = row_ptr<InT>(a.src, a.s_is, a.s_rp, n, iy1 ? t.y0 + 1 : 0);
    auto raw = [&](const InT* r, int i) -> uint32_t {
      if constexpr (sizeof(InT) == 1) return 0x4B000000u | __ldg(r + i);
      else return __float_as_uint(__ldg(r + i));
    };
#pragma unroll
    for (int c = 0; c < C; ++c) {
      t00[c] = (iy0 && ix0) ? raw(r0, t.x0 * C + c) : bord;
      t01[c] = (iy0 && ix1) ? raw(r0, (t.x0 + 1) * C + c) : bord;
      t10[c] = (iy1 && ix0) ? raw(r1, t.x0 * C + c) : bord;
      t11[c] = (iy1 && ix1) ? raw(r1, (t.x0 + 1) * C + c) : bord;
    }
  }
}

// blend operands from two raw taps (one per pixel of the thread's pair)
template <typename InT>
__device__ __forceinline__ f2_t tap2(uint32_t r0, uint32_t r1) {
  if constexpr (sizeof(InT) == 1) return unit2(r0, r1);
  else return f2u(r0, r1);
}

// Bilinear blend of the two pixels of a thread (t[0] -> d0, t[1] -> d1 when
// ok1) from their raw taps, in imgproc.py:118-123 order with every product
// and sum rounded (each sum is fma(q, runtime 1, p): see the f32x2 note in
// fv_common.cuh); u8 results take the app.py:75-77 epilogue. Non-finite maps
// store the raw border.
template <typename InT, int C>
__device__ __forceinline__ void blend_store(const WarpArgs& a, const WarpTap (&t)[2], const uint32_t (&v00)[2][C],
                                            const uint32_t (&v01)[2][C], const uint32_t (&v10)[2][C],
                                            const uint32_t (&v11)[2][C], InT* d0, InT* d1, bool ok1) {
  const f2_t ONE = a.one2;
  const f2_t WX0 = f2(t[0].wx0, t[1].wx0), WX1 = f2(t[0].wx1, t[1].wx1);
  const f2_t WY0 = f2(t[0].wy0, t[1].wy0), WY1 = f2(t[0].wy1, t[1].wy1);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const f2_t top = ffma2(fmul2(tap2<InT>(v01[0][c], v01[1][c]), WX1), ONE, fmul2(tap2<InT>(v00[0][c], v00[1][c]), WX0));
    const f2_t bot = ffma2(fmul2(tap2<InT>(v11[0][c], v11[1][c]), WX1), ONE, fmul2(tap2<InT>(v10[0][c], v10[1][c]), WX0));
    const f2_t o = ffma2(fmul2(bot, WY1), ONE, fmul2(top, WY0));
    uint32_t lo, hi;
    if constexpr (sizeof(InT) == 1) {
      f2split(scale_to_u8_bits2(o, 255.0f), lo, hi);
      d0[c] = t[0].finite ? (InT)(lo & 0xFF) : (InT)a.border_raw;
      if (ok1) d1[c] = t[1].finite ? (InT)(hi & 0xFF) : (InT)a.border_raw;
    } else {
      f2split(o, lo, hi);
      d0[c] = t[0].finite ? __uint_as_float(lo) : a.border_raw;
      if (ok1) d1[c] = t[1].finite ? __uint_as_float(hi) : a.border_raw;
    }
  }
}

// Fixed-C kernel (C = 1, 3, 4): a 64 x 8 tile of destination pixels per CTA;
// each thread samples pixels x and x + 32 (a warp covers 64 consecutive
// pixels, lanes stay contiguous for the gathers). The matrix and the row
// terms m1*y + m2 etc. are loaded / computed once per thread; tap
// conversion, blend and the u8 epilogue of the two pixels run as packed
// f32x2 pairs. Interior pixels take unguarded loads, pixels whose four taps
// are all outside skip the loads.
template <typename InT, bool PERSP, int C>
__global__ void __launch_bounds__(256, WK_MINB) warp_kernel(const __grid_constant__ WarpArgs a,
                                                   const __grid_constant__ WarpMats mats) {
  const int n = blockIdx.z;
  const int x = blockIdx.x * 64 + threadIdx.x;
  if (x >= a.dw) return;
  const bool two = x + 32 < a.dw;
  double m[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) m[i] = mats.m[n][i];
  const uint32_t bord = sizeof(InT) == 1 ? (0x4B000000u | (uint32_t)a.border_raw) : __float_as_uint(a.border_f);
  // WARP_ROWS rows per thread (stride 8): the per-warp setup (matrix, params,
  // indices) is amortised over 64 x WARP_ROWS pixels
  const int y_end = min(blockIdx.y * 8 * WARP_ROWS + 8 * WARP_ROWS, a.dh);
  const int y_first = blockIdx.y * 8 * WARP_ROWS + threadIdx.y;
  if (PERSP && a.zero_border && y_first < y_end) {
    // Whole-warp early out: lanes 0-3 map the corners of the warp's region
    // (64 columns x its rows). With W of one strict sign at all four corners
    // (W is linear: no zero inside) the region maps onto the convex
    // quadrilateral of the mapped corners; if all four lie beyond the same
    // side of the source (margin 2 px + 1e-6 relative, far above the f64
    // rounding of the per-pixel map), every tap of every pixel is outside and
    // the output is exactly +0 -- no per-pixel coordinate work.
    const unsigned am = __activemask();
    const int lane = threadIdx.x;
    const int y_last = y_first + 8 * ((y_end - 1 - y_first) / 8);
    int bits = 0;
    if (lane < 4) {
      const double cx = (double)((lane & 1) ? min((int)blockIdx.x * 64 + 63, a.dw - 1) : (int)blockIdx.x * 64);
      const double cy = (double)((lane & 2) ? y_last : y_first);
      const double X = m[0] * cx + m[1] * cy + m[2], Y = m[3] * cx + m[4] * cy + m[5];
      const double W = m[6] * cx + m[7] * cy + m[8];
      const double sx = X / W, sy = Y / W;
      const double mx = 2.0 + 1e-6 * fabs(sx), my = 2.0 + 1e-6 * fabs(sy);
      if (isfinite(sx) && isfinite(sy)) {
        bits |= (sx < -1.0 - mx) ? 1 : 0;
        bits |= (sx > (double)a.sw + mx) ? 2 : 0;
        bits |= (sy < -1.0 - my) ? 4 : 0;
        bits |= (sy > (double)a.sh + my) ? 8 : 0;
      }
      bits |= W > 0.0 ? 16 : (W < 0.0 ? 32 : 0);
    }
    const int all = __shfl_sync(am, bits, 0) & __shfl_sync(am, bits, 1) & __shfl_sync(am, bits, 2) &
                    __shfl_sync(am, bits, 3);
    if ((all & 48) && (all & 15)) {
#pragma unroll 1
      for (int y = y_first; y < y_end; y += 8) {
        InT* d = row_ptr_mut<InT>(a.dst, a.d_is, a.d_rp, n, y) + x * C;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          d[c] = (InT)0;
          if (two) d[32 * C + c] = (InT)0;
        }
      }
      return;
    }
  }
#pragma unroll 1
  for (int y = y_first; y < y_end; y += 8) {
    const double yd = (double)y;
    const double rx = __dadd_rn(__dmul_rn(m[1], yd), m[2]);
    const double ry = __dadd_rn(__dmul_rn(m[4], yd), m[5]);
    const double rw = PERSP ? __dadd_rn(__dmul_rn(m[7], yd), m[8]) : 0.0;
    InT* d = row_ptr_mut<InT>(a.dst, a.d_is, a.d_rp, n, y) + x * C;
    WarpTap t[2];
    t[0] = warp_tap<PERSP>(m, rx, ry, rw, x, a.sw, a.sh);
    t[1] = warp_tap<PERSP>(m, rx, ry, rw, two ? x + 32 : x, a.sw, a.sh);
    // With a +0 border, a pixel whose four taps all lie outside the source
    // (or whose map is non-finite) is exactly +0: a blend of four +0
    // operands, or the raw border. Warps made only of such pixels skip the
    // gathers and the blend (the vote is warp-uniform: rows are). Affine
    // maps have too few such warps to pay for the vote (measured).
    if (PERSP && a.zero_border && __all_sync(__activemask(), tap_outside(t[0], a.sw, a.sh) && tap_outside(t[1], a.sw, a.sh))) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        d[c] = (InT)0;
        if (two) d[32 * C + c] = (InT)0;
      }
      continue;
    }
    uint32_t v00[2][C], v01[2][C], v10[2][C], v11[2][C];
    // warp-uniform fast path: every lane's taps interior with the wide load
    // window inside the row (no per-thread fallback code in the common case)
    bool easy = true;
#pragma unroll
    for (int k = 0; k < 2; ++k)
      easy &= t[k].finite && t[k].x0 >= 0 && t[k].x0 <= a.sw - kPairSafe<InT, C> && t[k].y0 >= 0 &&
              t[k].y0 + 1 < a.sh;
    if (__all_sync(__activemask(), easy)) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const InT* r0 = row_ptr<InT>(a.src, a.s_is, a.s_rp, n, t[k].y0);
        const InT* r1 = row_ptr<InT>(a.src, a.s_is, a.s_rp, n, t[k].y0 + 1);
        load_pair_raw<InT, C, true>(r0, t[k].x0, a.sw * C, v00[k], v01[k]);
        load_pair_raw<InT, C, true>(r1, t[k].x0, a.sw * C, v10[k], v11[k]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 2; ++k) gather_raw<InT, C>(a, n, t[k], bord, v00[k], v01[k], v10[k], v11[k]);
    }

    blend_store<InT, C>(a, t, v00, v01, v10, v11, d, d + 32 * C, two);
  }
}

// ---------------------------------------------------------------------------
// Affine, staged: a 32 x 32 destination tile per CTA. An affine map sends the
// tile to a parallelogram, so the source box spanned by the mapped corners
// (+2 px: per-pixel rounding and the x0+1 / y0+1 taps) holds every in-image
// tap of the tile. Warp 0 streams the box's row segments into shared memory
// with 1-D bulk copies (each source sector crosses L2 -> SMEM once per tile);
// the gathers then read SMEM. The direct kernel's limiter is L1 wavefronts
// (a warp-wide LDG touches one line per source row its 32 slanted pixels
// span, ~16 at 30 degrees, and each pixel needs 4 LDG.64 per tap row); an
// LDS costs only its bank-conflict degree. Tiles whose box exceeds the
// staging budget (strong zoom-out) take the direct gathers in the same
// kernel. Same maps, taps and blend as warp_kernel: bit-identical output.
// ---------------------------------------------------------------------------
constexpr int AT = 32;  // tile width, destination pixels

template <typename InT, int C>
__device__ __forceinline__ uint32_t smem_raw(const uint8_t* p) {
  if constexpr (sizeof(InT) == 1) return 0x4B000000u | *p;
  else return *reinterpret_cast<const uint32_t*>(p);
}

// raw tap of channel c of the source pixel at SMEM byte offset o
template <typename InT>
__device__ __forceinline__ uint32_t lds_raw(uint32_t addr) {
  uint32_t v;
  if constexpr (sizeof(InT) == 1) {
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return 0x4B000000u | v;
  } else {
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
  }
}

struct TileBox {
  int bx0, bx1, by0, by1, off, rowbytes, pitch, staged;
};

// Plan one tile (thread 0): its source box from the mapped corners (floor
// -2 / +3), and when the box fits the staging buffer, arm the barrier with
// the bytes the row copies will deliver.
template <int PB, int TH>
__device__ __forceinline__ TileBox plan_tile(const WarpArgs& a, const double* m, int tx0, int ty0, int stage_bytes,
                                             uint64_t* bar) {
  double xlo = 0, xhi = 0, ylo = 0, yhi = 0;
  bool fin = true;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double cx = (double)((k & 1) ? min(tx0 + AT, a.dw) - 1 : tx0);
    const double cy = (double)((k & 2) ? min(ty0 + TH, a.dh) - 1 : ty0);
    const double sx = __dadd_rn(__dmul_rn(m[0], cx), __dadd_rn(__dmul_rn(m[1], cy), m[2]));
    const double sy = __dadd_rn(__dmul_rn(m[3], cx), __dadd_rn(__dmul_rn(m[4], cy), m[5]));
    fin = fin && isfinite(sx) && isfinite(sy);
    xlo = k ? fmin(xlo, sx) : sx;
    xhi = k ? fmax(xhi, sx) : sx;
    ylo = k ? fmin(ylo, sy) : sy;
    yhi = k ? fmax(yhi, sy) : sy;
  }
  TileBox b{0, -1, 0, -1, 0, 0, 0, 0};
  if (fin) {
    b.bx0 = (int)fmax(floor(xlo) - 2.0, 0.0);
    b.bx1 = (int)fmin(floor(xhi) + 3.0, (double)(a.sw - 1));
    b.by0 = (int)fmax(floor(ylo) - 2.0, 0.0);
    b.by1 = (int)fmin(floor(yhi) + 3.0, (double)(a.sh - 1));
  }
  if (fin && b.bx0 <= b.bx1 && b.by0 <= b.by1) {
    b.off = (PB * b.bx0) & 15;  // rows are 16-byte aligned (host-checked)
    b.rowbytes = (b.off + (b.bx1 - b.bx0 + 1) * PB + 15) & ~15;
    b.pitch = b.rowbytes + (((b.rowbytes >> 4) & 1) ? 0 : 16);  // odd multiple of 16 B: rows rotate banks
    const int rows = b.by1 - b.by0 + 1;
    b.staged = (int64_t)rows * b.pitch <= stage_bytes;
    if (b.staged) {
      mbar_init(bar, 1);
      fence_mbar_init();
      mbar_expect_tx(bar, (uint32_t)(rows * b.rowbytes));
    }
  }
  return b;
}

// One AT x TH destination tile per CTA (32 x TH/4 threads, 4 pixels each:
// rows ly + {0, TH/4} and ly + {TH/2, 3TH/4} as two f32x2 pairs). Thread 0
// plans the box, warp 0 issues the row copies, all wait on the barrier; the
// other CTAs resident on the SM (8 for TH = 16) overlap the fill.
template <typename InT, int C, int TH>
__global__ void __launch_bounds__(8 * TH, 128 / TH) warp_affine_tile_kernel(const __grid_constant__ WarpArgs a,
                                                                             const __grid_constant__ WarpMats mats) {
  constexpr int PB = C * (int)sizeof(InT);  // bytes per pixel
  constexpr int ES = (int)sizeof(InT);
  constexpr int RS = TH / 4;                // row step between a thread's pixels
  constexpr int STAGE = TH == 32 ? 48 * 1024 : 24 * 1024;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  TileBox* box = reinterpret_cast<TileBox*>(smem + 16);
  uint8_t* stage = smem + 64;
  const int n = blockIdx.z;
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int tx0 = blockIdx.x * AT, ty0 = blockIdx.y * TH;
  double m[9];
#pragma unroll
  for (int i = 0; i < 6; ++i) m[i] = mats.m[n][i];
  m[6] = m[7] = m[8] = 0.0;

  if (lx == 0 && ly == 0) *box = plan_tile<PB, TH>(a, m, tx0, ty0, STAGE, bar);
  __syncthreads();
  const TileBox b = *box;
  if (b.staged && ly == 0) {  // warp 0 streams the box's row segments
    const uint8_t* base = reinterpret_cast<const uint8_t*>(a.src) + n * a.s_is + (int64_t)b.by0 * a.s_rp +
                          (int64_t)PB * b.bx0 - b.off;
    for (int r = lx; r <= b.by1 - b.by0; r += 32)
      tma_bulk_g2s(stage + r * b.pitch, base + (int64_t)r * a.s_rp, (uint32_t)b.rowbytes, bar);
  }
  const int x = tx0 + lx;
  const uint32_t bord = sizeof(InT) == 1 ? (0x4B000000u | (uint32_t)a.border_raw) : __float_as_uint(a.border_f);
  // SMEM address of source pixel (0, by0): (x, y) at sb + (y - by0) * pitch + x * PB
  const uint32_t sb = smem_u32(stage) + (uint32_t)(b.off - b.bx0 * PB);
  if (b.staged) mbar_wait_block(bar, 0);
  if (x >= a.dw) return;  // (no CTA-wide barrier follows)
#pragma unroll 1
  for (int half = 0; half < 2; ++half) {
    const int ya = ty0 + ly + 2 * RS * half, yb = ya + RS;
    if (ya >= a.dh) break;
    const bool okb = yb < a.dh;
    WarpTap t[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double yd = (double)((k && okb) ? yb : ya);
      const double rx = __dadd_rn(__dmul_rn(m[1], yd), m[2]);
      const double ry = __dadd_rn(__dmul_rn(m[4], yd), m[5]);
      t[k] = warp_tap<false>(m, rx, ry, 0.0, x, a.sw, a.sh);
    }
    uint32_t v00[2][C], v01[2][C], v10[2][C], v11[2][C];
    if (b.staged) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const WarpTap& q = t[k];
        const bool inx = q.x0 >= 0 && q.x0 + 1 < a.sw, iny = q.y0 >= 0 && q.y0 + 1 < a.sh;
        if (inx && iny) {  // interior: in-image taps lie inside the box
          const uint32_t o = sb + (uint32_t)((q.y0 - b.by0) * b.pitch + q.x0 * PB);
#pragma unroll
          for (int c = 0; c < C; ++c) {
            v00[k][c] = lds_raw<InT>(o + c * ES);
            v01[k][c] = lds_raw<InT>(o + PB + c * ES);
            v10[k][c] = lds_raw<InT>(o + b.pitch + c * ES);
            v11[k][c] = lds_raw<InT>(o + b.pitch + PB + c * ES);
          }
        } else if (tap_outside(q, a.sw, a.sh)) {
#pragma unroll
          for (int c = 0; c < C; ++c) v00[k][c] = v01[k][c] = v10[k][c] = v11[k][c] = bord;
        } else {  // straddles the image edge: per-tap test (clamps keep reads in the box)
          const bool ix0 = q.x0 >= 0 && q.x0 < a.sw, ix1 = q.x0 + 1 >= 0 && q.x0 + 1 < a.sw;
          const bool iy0 = q.y0 >= 0 && q.y0 < a.sh, iy1 = q.y0 + 1 >= 0 && q.y0 + 1 < a.sh;
          const int cx0 = min(max(q.x0, b.bx0), b.bx1), cx1 = min(max(q.x0 + 1, b.bx0), b.bx1);
          const int cy0 = min(max(q.y0, b.by0), b.by1) - b.by0, cy1 = min(max(q.y0 + 1, b.by0), b.by1) - b.by0;
          const uint32_t r0 = sb + (uint32_t)(cy0 * b.pitch), r1 = sb + (uint32_t)(cy1 * b.pitch);
#pragma unroll
          for (int c = 0; c < C; ++c) {
            v00[k][c] = (iy0 && ix0) ? lds_raw<InT>(r0 + cx0 * PB + c * ES) : bord;
            v01[k][c] = (iy0 && ix1) ? lds_raw<InT>(r0 + cx1 * PB + c * ES) : bord;
            v10[k][c] = (iy1 && ix0) ? lds_raw<InT>(r1 + cx0 * PB + c * ES) : bord;
            v11[k][c] = (iy1 && ix1) ? lds_raw<InT>(r1 + cx1 * PB + c * ES) : bord;
          }
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < 2; ++k) gather_raw<InT, C>(a, n, t[k], bord, v00[k], v01[k], v10[k], v11[k]);
    }
    InT* da = row_ptr_mut<InT>(a.dst, a.d_is, a.d_rp, n, ya) + x * C;
    InT* db = row_ptr_mut<InT>(a.dst, a.d_is, a.d_rp, n, okb ? yb : ya) + x * C;
    blend_store<InT, C>(a, t, v00, v01, v10, v11, da, db, okb);
  }
}

// ---------------------------------------------------------------------------
// Affine, TMA-tensor staged: the same 32 x 16 tiles and gathers as
// warp_affine_tile_kernel, but the source box is a FIXED 48 x 40 pixel
// window loaded by ONE 3-D tensor copy (image, row, element) issued by thread
// 0 -- no per-row copies serialised on warp 0 -- with the TMA's zero fill for
// coordinates outside the image (taps there read the border anyway). Tiles
// whose box exceeds the window take the direct gathers.
// ---------------------------------------------------------------------------
constexpr int TBH = 40;  // window rows
// window width in ELEMENTS (a 16-byte multiple, <= 256); the window starts at
// the box's first element rounded down to 16 bytes (the TMA faults on an
// unaligned innermost start coordinate: tools/probe/tma_probe.cu)
template <typename InT, int C>
constexpr int tma_win_elems() {
  return sizeof(InT) == 4 ? 48 * C : (C == 3 ? 192 : (C == 4 ? 256 : 64));
}

// Thread 0's part of a staged tile: the source box spanned by the mapped
// corners (every in-image tap of the tile lies in [floor(lo) - 2,
// floor(hi) + 3]) and, when it fits the window, ONE 3-D tensor copy of the
// window into `stage`, completing on `bar`. Returns {ex0, by0, staged}.
template <typename InT, int C>
__device__ __forceinline__ int3 affine_tma_issue(const CUtensorMap* tmap, const WarpArgs& a, const double (&m)[9], int n,
                                                 int tx0, int ty0, uint8_t* stage, uint64_t* bar) {
  constexpr int ES = (int)sizeof(InT);
  constexpr int TH = 16;
  constexpr int TBE = tma_win_elems<InT, C>();
  constexpr int AL = 16 / ES;
  double xlo = 0, xhi = 0, ylo = 0, yhi = 0;
  bool fin = true;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double cx = (double)((k & 1) ? min(tx0 + AT, a.dw) - 1 : tx0);
    const double cy = (double)((k & 2) ? min(ty0 + TH, a.dh) - 1 : ty0);
    const double sx = __dadd_rn(__dmul_rn(m[0], cx), __dadd_rn(__dmul_rn(m[1], cy), m[2]));
    const double sy = __dadd_rn(__dmul_rn(m[3], cx), __dadd_rn(__dmul_rn(m[4], cy), m[5]));
    fin = fin && isfinite(sx) && isfinite(sy);
    xlo = k ? fmin(xlo, sx) : sx;
    xhi = k ? fmax(xhi, sx) : sx;
    ylo = k ? fmin(ylo, sy) : sy;
    yhi = k ? fmax(yhi, sy) : sy;
  }
  fin = fin && xlo > -1e9 && xhi < 1e9 && ylo > -1e9 && yhi < 1e9;
  const int bx0 = fin ? (int)floor(xlo) - 2 : 0, by0 = fin ? (int)floor(ylo) - 2 : 0;
  const int e0 = bx0 * C;
  const int ex0 = (e0 >= 0 ? e0 : e0 - (AL - 1)) / AL * AL;  // floor to the alignment
  const bool staged = fin && ((int)floor(xhi) + 4) * C - ex0 <= TBE && (int)floor(yhi) + 3 - by0 < TBH;
  if (staged) {
    FV_CHECK(in_dyn_smem(smem_u32(stage), (uint32_t)(TBE * TBH * ES)));
    mbar_expect_tx(bar, (uint32_t)(TBE * TBH * ES));
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(stage)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(ex0), "r"(by0), "r"(n), "r"(smem_u32(bar))
        : "memory");
  }
  return make_int3(ex0, by0, staged ? 1 : 0);
}

// The threads' part of one 32 x 16 tile: 4 pixels each (rows ly, ly + 4,
// ly + 8, ly + 12). The f64 maps of all four pixels (affine_tile_maps) are
// computed BEFORE waiting for the window (`bar`, when staged) -- and before
// the CTA barrier that publishes the box -- so that work overlaps the box
// and the tensor copy (0.398 -> 0.358 ms for cfg2; also precomputing the window
// offsets, or mapping the box corners on four lanes, measured slower); then
// taps come from the window at `stage` (window element (ex0, by0) first)
// when staged, else from direct gathers; blend and store.
template <typename InT, int C>
__device__ __forceinline__ void affine_tile_maps(const WarpArgs& a, const double (&m)[9], int tx0, int ty0, int lx,
                                                 int ly, WarpTap (&t)[2][2]) {
  constexpr int RS = 4;
  const int x = tx0 + lx;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int ya = ty0 + ly + 2 * RS * half, yb = ya + RS;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double yd = (double)((k && yb < a.dh) ? yb : ya);
      const double rx = __dadd_rn(__dmul_rn(m[1], yd), m[2]);
      const double ry = __dadd_rn(__dmul_rn(m[4], yd), m[5]);
      t[half][k] = warp_tap<false>(m, rx, ry, 0.0, x, a.sw, a.sh);
    }
  }
}

template <typename InT, int C>
__device__ __forceinline__ void affine_tma_tile(const WarpArgs& a, const WarpTap (&t)[2][2], int n, int tx0, int ty0,
                                                int ex0, int by0, bool staged, const uint8_t* stage, uint64_t* bar,
                                                int lx, int ly) {
  constexpr int PB = C * (int)sizeof(InT);
  constexpr int ES = (int)sizeof(InT);
  constexpr int TH = 16, RS = TH / 4;
  constexpr int TBE = tma_win_elems<InT, C>();
  const int x = tx0 + lx;
  if (staged) mbar_wait_block(bar, 0);
  if (x >= a.dw) return;
  const uint32_t bord = sizeof(InT) == 1 ? (0x4B000000u | (uint32_t)a.border_raw) : __float_as_uint(a.border_f);
  // element e of row y at sb + (y * TBE + e) * ES
  const uint32_t sb = smem_u32(stage) - (uint32_t)((by0 * TBE + ex0) * ES);
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int ya = ty0 + ly + 2 * RS * half, yb = ya + RS;
    if (ya >= a.dh) break;
    const bool okb = yb < a.dh;
    uint32_t v00[2][C], v01[2][C], v10[2][C], v11[2][C];
    if (staged) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const WarpTap& q = t[half][k];
        const bool ix0 = q.x0 >= 0 && q.x0 < a.sw, ix1 = q.x0 + 1 >= 0 && q.x0 + 1 < a.sw;
        const bool iy0 = q.y0 >= 0 && q.y0 < a.sh, iy1 = q.y0 + 1 >= 0 && q.y0 + 1 < a.sh;
        // in-image taps lie in the window; others read the border (never the SMEM)
        const uint32_t o = sb + (uint32_t)((q.y0 * TBE + q.x0 * C) * ES);
        FV_CHECK(!(q.finite && iy0 && ix0 && iy1 && ix1) ||
                 (o >= smem_u32(stage) && o + TBE * ES + PB * 2 <= smem_u32(stage) + TBE * TBH * ES + PB));
#pragma unroll
        for (int c = 0; c < C; ++c) {
          v00[k][c] = (q.finite && iy0 && ix0) ? lds_raw<InT>(o + c * ES) : bord;
          v01[k][c] = (q.finite && iy0 && ix1) ? lds_raw<InT>(o + PB + c * ES) : bord;
          v10[k][c] = (q.finite && iy1 && ix0) ? lds_raw<InT>(o + TBE * ES + c * ES) : bord;
          v11[k][c] = (q.finite && iy1 && ix1) ? lds_raw<InT>(o + TBE * ES + PB + c * ES) : bord;
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < 2; ++k) gather_raw<InT, C>(a, n, t[half][k], bord, v00[k], v01[k], v10[k], v11[k]);
    }
    InT* da = row_ptr_mut<InT>(a.dst, a.d_is, a.d_rp, n, ya) + x * C;
    InT* db = row_ptr_mut<InT>(a.dst, a.d_is, a.d_rp, n, okb ? yb : ya) + x * C;
    blend_store<InT, C>(a, t[half], v00, v01, v10, v11, da, db, okb);
  }
}

template <typename InT, int C>
#ifndef FV_AFFINE_MINB
#define FV_AFFINE_MINB 8  // 8 x 23 KB windows per SM: 64 registers hold the four maps computed before the wait
#endif
__global__ void __launch_bounds__(128, FV_AFFINE_MINB) warp_affine_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                 const __grid_constant__ WarpArgs a,
                                                                 const __grid_constant__ WarpMats mats) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
  int* box = reinterpret_cast<int*>(smem + 16);  // ex0 (window's first element), by0, staged
  uint8_t* stage = smem + 128;
  const int n = blockIdx.z;
  const int tx0 = blockIdx.x * AT, ty0 = blockIdx.y * 16;
  double m[9];
#pragma unroll
  for (int i = 0; i < 6; ++i) m[i] = mats.m[n][i];
  m[6] = m[7] = m[8] = 0.0;
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    const int3 b = affine_tma_issue<InT, C>(&tmap, a, m, n, tx0, ty0, stage, bar);
    box[0] = b.x;
    box[1] = b.y;
    box[2] = b.z;
  }
  WarpTap t[2][2];
  affine_tile_maps<InT, C>(a, m, tx0, ty0, threadIdx.x, threadIdx.y, t);
  __syncthreads();
  affine_tma_tile<InT, C>(a, t, n, tx0, ty0, box[0], box[1], box[2] != 0, stage, bar, threadIdx.x, threadIdx.y);
}

// Any channel count: same sampler, channel loop at run time.
template <typename InT, bool PERSP>
__global__ void __launch_bounds__(256) warp_kernel_any(const __grid_constant__ WarpArgs a,
                                                       const __grid_constant__ WarpMats mats) {
  const int n = blockIdx.z;
  const int x = blockIdx.x * 32 + threadIdx.x;
  const int y = blockIdx.y * 8 + threadIdx.y;
  if (x >= a.dw || y >= a.dh) return;
  double m[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) m[i] = mats.m[n][i];
  const double yd = (double)y;
  const double rx = __dadd_rn(__dmul_rn(m[1], yd), m[2]);
  const double ry = __dadd_rn(__dmul_rn(m[4], yd), m[5]);
  const double rw = PERSP ? __dadd_rn(__dmul_rn(m[7], yd), m[8]) : 0.0;
  const WarpTap t = warp_tap<PERSP>(m, rx, ry, rw, x, a.sw, a.sh);
  InT* d = row_ptr_mut<InT>(a.dst, a.d_is, a.d_rp, n, y) + x * a.c;
  if (!t.finite) {
    for (int c = 0; c < a.c; ++c) d[c] = (InT)a.border_raw;
    return;
  }
  const bool ix0 = t.x0 >= 0 && t.x0 < a.sw, ix1 = t.x0 + 1 >= 0 && t.x0 + 1 < a.sw;
  const bool iy0 = t.y0 >= 0 && t.y0 < a.sh, iy1 = t.y0 + 1 >= 0 && t.y0 + 1 < a.sh;
  const InT* r0 = row_ptr<InT>(a.src, a.s_is, a.s_rp, n, iy0 ? t.y0 : 0);
  const InT* r1 = row_ptr<InT>(a.src, a.s_is, a.s_rp, n, iy1 ? t.y0 + 1 : 0);
  for (int c = 0; c < a.c; ++c) {
    const float t00 = (iy0 && ix0) ? tap_value(__ldg(r0 + t.x0 * a.c + c)) : a.border_f;
    const float t01 = (iy0 && ix1) ? tap_value(__ldg(r0 + (t.x0 + 1) * a.c + c)) : a.border_f;
    const float t10 = (iy1 && ix0) ? tap_value(__ldg(r1 + t.x0 * a.c + c)) : a.border_f;
    const float t11 = (iy1 && ix1) ? tap_value(__ldg(r1 + (t.x0 + 1) * a.c + c)) : a.border_f;
    const float top = lerp_ref(t00, t01, t.wx0, t.wx1);
    const float bot = lerp_ref(t10, t11, t.wx0, t.wx1);
    d[c] = to_out<InT>(lerp_ref(top, bot, t.wy0, t.wy1));
  }
}

// ---------------------------------------------------------------------------
// u8 perspective, <= 1 LSB (the north-star gate for u8 results of float
// interpolation; SURVEY §7 hard part 2 asks for f32 / mixed coordinates
// here). A warp covers 32 * PF_PX pixels of a row in groups of PF_PX:
//   * one f64 anchor per group, computed by one lane and shared through
//     SMEM: s_a = (X, Y)(x_a) / W(x_a); lane L then samples pixels
//     x_w + L + 32 j (contiguous lanes: coalesced gathers and stores);
//   * per pixel d = 0..7, exactly s(d) = s_a + k * d / W(d) with
//     k = (m0 - s_a.x * m6, m3 - s_a.y * m6) and W(d) = W_a + m6 * d: the f32
//     correction carries ~1e-7 RELATIVE error of a term of a few pixels, so
//     the coordinates stay within ~1e-5 px of the f64 map (bound below);
//   * the blend runs on the 0..255 scale (one rounding per FMA) and is
//     rounded half up: sum_ij u_ij * w_ij + 0.5, floor.
// Error budget against the exact recipe: |v_fast - v_exact| <= 255 * (Ex + Ey)
// + ~3e-4 with Ex, Ey <= PF_MAX_ERR px, checked per group in f32 from the
// anchor. With u = 2^-24, Cmax = |k| * 7 / Wmin (the largest correction)
// and rho = (|W_a| + 7 |m6|) / Wmin: W(d) carries <= u * (rho + 1) relative
// error (the f32 roundings of W_a and m6 and the FMA), rcp.approx <= 2u, k
// and the two products u each, so the correction is off by <= Cmax * u *
// (rho + 6) <= Cmax * 2^-23 * (rho + 4); the sum s_frac + c adds <= u * (1 +
// Cmax) and s_frac's own rounding 2^-25, both inside the 2^-22 term. The
// f64 per-pixel map (warp_tap) takes over when the bound fails, W changes
// sign or vanishes within the group, or the anchor is non-finite or beyond
// 2^22 px. Bilinear sampling with a constant border is continuous in
// (sx, sy) (a tap's weight reaches 0 exactly where it switches between the
// image and the border), so a shift of the integer tap across a boundary
// changes nothing beyond the same bound: |out - oracle| <= 1 LSB.
// ---------------------------------------------------------------------------
constexpr int PF_PX = 8;          // consecutive pixels per thread
#ifndef FV_PF_ROWS
#define FV_PF_ROWS 8  // measured: 2 -> 0.586, 4 -> 0.560, 8 -> 0.552, 16 -> 0.571 ms (cfg3)
#endif
constexpr int PF_ROWS = FV_PF_ROWS;  // rows per thread (stride 8)
constexpr float PF_MAX_ERR = 5e-4f;
#ifndef PF_JUNROLL
#define PF_JUNROLL 1
#endif
constexpr int kPfJUnroll = PF_JUNROLL;  // pixel pairs per sampling-loop iteration
#ifndef PF_MINB
#define PF_MINB 4  // resident CTAs per SM the register budget is sized for
#endif


// Window of the two taps (x0, x0 + 1) of one source row, C bytes each, from
// NWIN aligned 32-bit loads at byte offset `off` of a 4-byte aligned image;
// the caller guarantees x0 <= sw - pf_safe<C>() so the window ends inside
// the row. Returns magic words 0x4B0000uu.
template <int C>
constexpr int pf_nwin() { return (2 * C + 3 + 3) / 4; }
template <int C>
constexpr int pf_safe() { return (4 * pf_nwin<C>() + C - 1) / C; }
template <int C>
__device__ __forceinline__ void pf_row_taps(const uint8_t* img, uint32_t al, int sh, uint32_t (&t0)[C],
                                            uint32_t (&t1)[C]) {
  constexpr int NW = pf_nwin<C>(), NV = (2 * C + 3) / 4;
  const uint32_t* w = reinterpret_cast<const uint32_t*>(img + al);
  uint32_t win[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) win[i] = __ldg(w + i);
  uint32_t v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = __funnelshift_r(win[i], win[i + 1], sh);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    t0[c] = magic_of(v, c);
    t1[c] = magic_of(v, C + c);
  }
}

// One pixel of the <= 1 LSB perspective path with per-tap border handling
// (taps at the source edge, all-outside pixels, rows near the buffer end).
// The fast kernel calls it only from warps that hold such a pixel (a
// warp-uniform branch), so its guarded loads never take issue slots in the
// common path.
template <int C>
__device__ __forceinline__ void pf_pixel_generic(const WarpArgs& a, int n, int x0, int y0, float fx, float fy,
                                              uint8_t* d) {
  const uint32_t braw = (uint32_t)a.border_raw;
  if (x0 < -1 || x0 >= a.sw || y0 < -1 || y0 >= a.sh) {
    for (int c = 0; c < C; ++c) d[c] = (uint8_t)braw;
    return;
  }
  const bool ix0 = x0 >= 0, ix1 = x0 + 1 < a.sw, iy0 = y0 >= 0, iy1 = y0 + 1 < a.sh;
  const uint8_t* r0 = row_ptr<uint8_t>(a.src, a.s_is, a.s_rp, n, iy0 ? y0 : 0);
  const uint8_t* r1 = row_ptr<uint8_t>(a.src, a.s_is, a.s_rp, n, iy1 ? y0 + 1 : 0);
  const float wx0 = __fsub_rn(1.0f, fx), wy0 = __fsub_rn(1.0f, fy);
  const float w00 = __fmul_rn(wx0, wy0), w01 = __fmul_rn(fx, wy0), w10 = __fmul_rn(wx0, fy), w11 = __fmul_rn(fx, fy);
  const float b = (float)braw;
  for (int c = 0; c < C; ++c) {
    const float a00 = (iy0 && ix0) ? (float)__ldg(r0 + x0 * C + c) : b;
    const float a01 = (iy0 && ix1) ? (float)__ldg(r0 + (x0 + 1) * C + c) : b;
    const float a10 = (iy1 && ix0) ? (float)__ldg(r1 + x0 * C + c) : b;
    const float a11 = (iy1 && ix1) ? (float)__ldg(r1 + (x0 + 1) * C + c) : b;
    const float v = __fmaf_rn(a11, w11, __fmaf_rn(a10, w10, __fmaf_rn(a01, w01, __fmaf_rn(a00, w00, 0.5f))));
    d[c] = (uint8_t)min((int)floorf(v), 255);
  }
}

template <int C>
__global__ void __launch_bounds__(256, PF_MINB) warp_persp_fast_kernel(const __grid_constant__ WarpArgs a,
                                                              const __grid_constant__ WarpMats mats) {
  // anchors of the warp's 32 groups: {sxf, syf, kx, ky}, {W_a, ix_a, iy_a, fast}
  // anchors of the warp's 32 groups, stored by group PAIR (g, g + 4) --
  // the two groups a lane samples in one iteration -- so one LDS.128 yields
  // a field of both as f32x2 operands: {sxf, syf}, {kx, ky}, {W_a, ix_a},
  // {iy_a, fast}, each as (group g, group g + 4)
  __shared__ float4 anc[8][16][4];
  const int n = blockIdx.z;
  const int lane = threadIdx.x;
  const int xw = blockIdx.x * (32 * PF_PX);
  double m[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) m[i] = mats.m[n][i];
  const uint32_t braw = (uint32_t)a.border_raw;
  const int y_end = min((int)blockIdx.y * 8 * PF_ROWS + 8 * PF_ROWS, a.dh);
  const int y_first = blockIdx.y * 8 * PF_ROWS + threadIdx.y;
  if (y_first >= y_end || xw >= a.dw) return;  // warp-uniform
  // Whole-warp early out (as warp_kernel): the warp's region (32 * PF_PX
  // columns x its rows) maps, W of one sign at its corners, onto the convex
  // quadrilateral of the mapped corners; beyond one side of the source (2 px
  // + 1e-6 relative margin) every tap is outside and every pixel is exactly
  // the border (the weights sum to within 2^-21 of 1).
  {
    const int y_last = y_first + 8 * ((y_end - 1 - y_first) / 8);
    int bits = 0;
    if (lane < 4) {
      const double cx = (double)((lane & 1) ? min(xw + 32 * PF_PX - 1, a.dw - 1) : xw);
      const double cy = (double)((lane & 2) ? y_last : y_first);
      const double X = m[0] * cx + m[1] * cy + m[2], Y = m[3] * cx + m[4] * cy + m[5];
      const double W = m[6] * cx + m[7] * cy + m[8];
      const double sx = X / W, sy = Y / W;
      const double mx = 2.0 + 1e-6 * fabs(sx), my = 2.0 + 1e-6 * fabs(sy);
      if (isfinite(sx) && isfinite(sy)) {
        bits |= (sx < -1.0 - mx) ? 1 : 0;
        bits |= (sx > (double)a.sw + mx) ? 2 : 0;
        bits |= (sy < -1.0 - my) ? 4 : 0;
        bits |= (sy > (double)a.sh + my) ? 8 : 0;
      }
      bits |= W > 0.0 ? 16 : (W < 0.0 ? 32 : 0);
    }
    const int all = __shfl_sync(0xffffffffu, bits, 0) & __shfl_sync(0xffffffffu, bits, 1) &
                    __shfl_sync(0xffffffffu, bits, 2) & __shfl_sync(0xffffffffu, bits, 3);
    if ((all & 48) && (all & 15)) {
#pragma unroll 1
      for (int y = y_first; y < y_end; y += 8) {
        uint8_t* d = row_ptr_mut<uint8_t>(a.dst, a.d_is, a.d_rp, n, y);
#pragma unroll
        for (int j = 0; j < PF_PX; ++j) {
          const int x = xw + lane + 32 * j;
          if (x < a.dw) {
#pragma unroll
            for (int c = 0; c < C; ++c) d[x * C + c] = (uint8_t)braw;
          }
        }
      }
      return;
    }
  }
  const float m6f = (float)m[6];
  const float dlt = (float)(lane & (PF_PX - 1));
  const uint8_t* simg = reinterpret_cast<const uint8_t*>(a.src) + (int64_t)n * a.s_is;
  const uint32_t rp32 = (uint32_t)a.s_rp;
  const unsigned xlim = (unsigned)(a.sw - pf_safe<C>()), ylim = (unsigned)(a.sh - 1);
  const f2_t HALF = f2(0.5f, 0.5f), MAG = f2(8388608.0f, 8388608.0f), NMAG = f2(-8388608.0f, -8388608.0f);
  float4(&A)[16][4] = anc[threadIdx.y];
#pragma unroll 1
  for (int y = y_first; y < y_end; y += 8) {
    const double yd = (double)y;
    const double rx = m[1] * yd + m[2], ry = m[4] * yd + m[5], rw = m[7] * yd + m[8];
    {
      // this lane's anchor: group `lane`, pixels xg .. xg + PF_PX - 1
      const double xd = (double)(xw + PF_PX * lane);
      const double Wa = m[6] * xd + rw;
      const double We = Wa + m[6] * (double)(PF_PX - 1);
      const double ra = 1.0 / Wa;  // s_a only needs ~1e-10 px: one reciprocal for both axes
      const double sa_x = (m[0] * xd + rx) * ra, sa_y = (m[3] * xd + ry) * ra;
      bool fast = ((Wa > 0.0 && We > 0.0) || (Wa < 0.0 && We < 0.0)) && fabs(sa_x) < 4194304.0 &&
                  fabs(sa_y) < 4194304.0;  // false for NaN too
      const float kx = (float)(m[0] - sa_x * m[6]), ky = (float)(m[3] - sa_y * m[6]);
      const float waf = (float)Wa;
      if (fast) {
        // per-axis bound (block comment): Cmax * 2^-23 * ((|Wa| + 7|m6|) / Wmin + 4) + 2^-22
        const float iw = 1.0f / (float)fmin(fabs(Wa), fabs(We));
        const float rho = (fabsf(waf) + (float)(PF_PX - 1) * fabsf(m6f)) * iw + 4.0f;
        const float cx = fabsf(kx) * (float)(PF_PX - 1) * iw, cy = fabsf(ky) * (float)(PF_PX - 1) * iw;
        const float ex = cx * rho * 1.1920929e-7f + 2.3841858e-7f, ey = cy * rho * 1.1920929e-7f + 2.3841858e-7f;
        fast = ex <= PF_MAX_ERR && ey <= PF_MAX_ERR;  // false for inf / NaN
      }
      const double fxa = floor(sa_x), fya = floor(sa_y);
      float* q = reinterpret_cast<float*>(&A[(lane >> 3) * 4 + (lane & 3)][0]) + ((lane >> 2) & 1);
      q[0] = (float)(sa_x - fxa);
      q[2] = (float)(sa_y - fya);
      q[4] = kx;
      q[6] = ky;
      q[8] = waf;
      q[10] = __int_as_float(fast ? (int)fxa : 0);
      q[12] = __int_as_float(fast ? (int)fya : 0);
      q[14] = __int_as_float(fast ? 1 : 0);
    }
    __syncwarp();
    uint8_t* drow = row_ptr_mut<uint8_t>(a.dst, a.d_is, a.d_rp, n, y);
#pragma unroll kPfJUnroll
    for (int j = 0; j < PF_PX; j += 2) {
      // pixels x_k = xw + lane + 32 * (j + k): lanes stay contiguous for the
      // gathers; group (x_k - xw) / PF_PX holds the anchor, offset lane % 8
      int tx0[2], ty0[2];
      float tfx[2], tfy[2];
      const int pp = (j >> 1) * 4 + (lane >> 3);  // groups 4j + lane/8 and 4j + 4 + lane/8
      const float4 F0 = A[pp][0], F1 = A[pp][1], F2 = A[pp][2], F3 = A[pp][3];
      if (__float_as_int(F3.z) & __float_as_int(F3.w)) {
        // both pixels on the f32 correction: the two maps as f32x2 pairs
        const f2_t D = f2(dlt, dlt);
        const f2_t W = ffma2(f2(m6f, m6f), D, f2(F2.x, F2.y));
        uint32_t wl, wh;
        f2split(W, wl, wh);
        const f2_t R = f2(rcp_approx(__uint_as_float(wl)), rcp_approx(__uint_as_float(wh)));
        const f2_t TX = fadd2(f2(F0.x, F0.y), fmul2(fmul2(f2(F1.x, F1.y), D), R));
        const f2_t TY = fadd2(f2(F0.z, F0.w), fmul2(fmul2(f2(F1.z, F1.w), D), R));
        // floor: RD(t + 1.5 * 2^23) holds floor(t) in its low bits for |t| < 2^22
        const f2_t MG = f2(12582912.0f, 12582912.0f), NMG = f2(-12582912.0f, -12582912.0f);
        const f2_t FX = fadd2_rd(TX, MG), FY = fadd2_rd(TY, MG);
        uint32_t fxl, fxh, fyl, fyh, rxl, rxh, ryl, ryh;
        f2split(FX, fxl, fxh);
        f2split(FY, fyl, fyh);
        f2split(fadd2(TX, fadd2(NMG, FX) ^ 0x8000000080000000ull), rxl, rxh);  // t - floor(t)
        f2split(fadd2(TY, fadd2(NMG, FY) ^ 0x8000000080000000ull), ryl, ryh);
        tfx[0] = __uint_as_float(rxl);
        tfx[1] = __uint_as_float(rxh);
        tfy[0] = __uint_as_float(ryl);
        tfy[1] = __uint_as_float(ryh);
        tx0[0] = (int)(fxl - 0x4B400000u) + __float_as_int(F2.z);
        tx0[1] = (int)(fxh - 0x4B400000u) + __float_as_int(F2.w);
        ty0[0] = (int)(fyl - 0x4B400000u) + __float_as_int(F3.x);
        ty0[1] = (int)(fyh - 0x4B400000u) + __float_as_int(F3.y);
      } else {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          if (__float_as_int(k ? F3.w : F3.z)) {
            const float r = rcp_approx(__fmaf_rn(m6f, dlt, k ? F2.y : F2.x));  // <= 1 ulp (bound term 2^-23)
            const float tx = __fadd_rn(k ? F0.y : F0.x, __fmul_rn(__fmul_rn(k ? F1.y : F1.x, dlt), r));
            const float ty = __fadd_rn(k ? F0.w : F0.z, __fmul_rn(__fmul_rn(k ? F1.w : F1.z, dlt), r));
            const float flx = floorf(tx), fly = floorf(ty);
            tfx[k] = __fsub_rn(tx, flx);
            tfy[k] = __fsub_rn(ty, fly);
            tx0[k] = __float_as_int(k ? F2.w : F2.z) + (int)flx;  // |.| < 2^23: no clamp needed
            ty0[k] = __float_as_int(k ? F3.y : F3.x) + (int)fly;
          } else {
            // the f64 per-pixel map (warp_tap); non-finite -> every tap outside
            const WarpTap w = warp_tap<true>(m, rx, ry, rw, min(xw + lane + 32 * (j + k), a.dw - 1), a.sw, a.sh);
            tfx[k] = w.wx1;
            tfy[k] = w.wy1;
            tx0[k] = w.finite ? w.x0 : -2;
            ty0[k] = w.finite ? w.y0 : -2;
          }
        }
      }
      const int xa = xw + lane + 32 * j, xb = xa + 32;
      const bool va = xa < a.dw, vb = xb < a.dw;
      // interior: all four taps inside and the load window inside the row
      const bool easy = (!va || ((unsigned)tx0[0] <= xlim && (unsigned)ty0[0] < ylim)) &&
                        (!vb || ((unsigned)tx0[1] <= xlim && (unsigned)ty0[1] < ylim));
      if (!__all_sync(0xffffffffu, easy)) {
        const bool ina = va && (unsigned)(tx0[0] + 1) <= (unsigned)a.sw && (unsigned)(ty0[0] + 1) <= (unsigned)a.sh;
        const bool inb = vb && (unsigned)(tx0[1] + 1) <= (unsigned)a.sw && (unsigned)(ty0[1] + 1) <= (unsigned)a.sh;
        if (!__any_sync(0xffffffffu, ina || inb)) {  // the warp's 64 pixels are all border
#pragma unroll
          for (int c = 0; c < C; ++c) {
            if (va) drow[xa * C + c] = (uint8_t)braw;
            if (vb) drow[xb * C + c] = (uint8_t)braw;
          }
        } else {
          if (va) pf_pixel_generic<C>(a, n, tx0[0], ty0[0], tfx[0], tfy[0], drow + xa * C);
          if (vb) pf_pixel_generic<C>(a, n, tx0[1], ty0[1], tfx[1], tfy[1], drow + xb * C);
        }
        continue;
      }
      uint32_t v00[2][C], v01[2][C], v10[2][C], v11[2][C];
      {
        // 32-bit offsets inside the image (host-checked: < 2^31), 4-byte
        // aligned rows (host-checked): lanes past the edge load row 0
        const uint32_t oa = va ? (uint32_t)ty0[0] * rp32 + (uint32_t)(tx0[0] * C) : 0u;
        const uint32_t ob = vb ? (uint32_t)ty0[1] * rp32 + (uint32_t)(tx0[1] * C) : 0u;
        // rows are 4-byte aligned: both tap rows share the byte shift
        const int sha = (int)(oa & 3u) * 8, shb = (int)(ob & 3u) * 8;
        pf_row_taps<C>(simg, oa & ~3u, sha, v00[0], v01[0]);
        pf_row_taps<C>(simg, (oa & ~3u) + rp32, sha, v10[0], v11[0]);
        pf_row_taps<C>(simg, ob & ~3u, shb, v00[1], v01[1]);
        pf_row_taps<C>(simg, (ob & ~3u) + rp32, shb, v10[1], v11[1]);
      }
      const f2_t WX1 = f2(tfx[0], tfx[1]), WY1 = f2(tfy[0], tfy[1]);
      const f2_t WX0 = fadd2(f2(1.0f, 1.0f), fmul2(WX1, f2(-1.0f, -1.0f)));
      const f2_t WY0 = fadd2(f2(1.0f, 1.0f), fmul2(WY1, f2(-1.0f, -1.0f)));
      const f2_t W00 = fmul2(WX0, WY0), W01 = fmul2(WX1, WY0), W10 = fmul2(WX0, WY1), W11 = fmul2(WX1, WY1);
      // first tap straight from its magic word M = 2^23 + u: C00 = 0.5 -
      // 2^23 * W00 is exact for W00 >= 2^-24 (at most 24 significant bits
      // from 2^-1 down to W00's last bit times 2^23; below, off by <= 2^-25),
      // so fma(M, W00, C00) = RN(u * W00 + 0.5)
      const f2_t C00 = ffma2(W00, NMAG, HALF);
      uint8_t* pa = drow + xa * C;
      uint8_t* pb = drow + xb * C;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const f2_t A01 = fadd2(f2u(v01[0][c], v01[1][c]), NMAG);
        const f2_t A10 = fadd2(f2u(v10[0][c], v10[1][c]), NMAG), A11 = fadd2(f2u(v11[0][c], v11[1][c]), NMAG);
        const f2_t v = ffma2(A11, W11, ffma2(A10, W10, ffma2(A01, W01, ffma2(f2u(v00[0][c], v00[1][c]), W00, C00))));
        uint32_t lo, hi;
        f2split(fadd2_rd(v, MAG), lo, hi);  // floor(v) in the low byte (0 <= v < 256)
        if (va) pa[c] = (uint8_t)(lo & 0xFF);
        if (vb) pb[c] = (uint8_t)(hi & 0xFF);
      }
    }
    __syncwarp();
  }
}

#ifdef FV_TEST_KNOBS
static int g_warp_path = 0;  // 0 auto, 1 direct gathers only, 2 bulk-copy tiles, 3 round-1 perspective kernel
static int g_warp_tma = 1;   // TMA-tensor tiles when available (path 0)
static int g_warp_src = 1;   // source-tiled affine kernel when applicable (path 0)
#else
constexpr int g_warp_src = 1;
constexpr int g_warp_path = 0;  // product build: always the automatic selection
constexpr int g_warp_tma = 1;
#endif

constexpr int AT_H = 16;  // tile height of the staged affine kernel (16: 24 KB stage, 8 CTAs / SM)

template <typename InT, int C>
static int launch_tile(int dw, int dh, int nb, cudaStream_t st, const WarpArgs& a, const WarpMats& mats) {
  auto kern = warp_affine_tile_kernel<InT, C, AT_H>;
  const int smem = 64 + (AT_H == 32 ? 48 * 1024 : 24 * 1024);
  static unsigned long long attr_mask[2] = {0, 0};  // per instantiation
  if (ensure_smem_attr(kern, smem, attr_mask) != FV_OK) return check_launch("warp_affine_tile_kernel (smem attribute)");
  dim3 grid((dw + AT - 1) / AT, (dh + AT_H - 1) / AT_H, nb);
  kern<<<grid, dim3(32, AT_H / 4), smem, st>>>(a, mats);
  return FV_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// libcuda link); null when unavailable (then the bulk-copy tile kernel runs)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static std::once_flag once;
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 0 = launched, 1 = no tensor map (caller falls back), else error
template <typename InT, int C>
static int launch_tma(int dw, int dh, int nb, cudaStream_t st, const WarpArgs& a, const WarpMats& mats) {
  auto enc = tensor_map_encoder();
  if (!enc) return 1;
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)a.sw * C, (cuuint64_t)a.sh, (cuuint64_t)nb};
  const cuuint64_t strides[2] = {(cuuint64_t)a.s_rp, (cuuint64_t)(nb > 1 ? a.s_is : a.s_rp * a.sh)};
  const cuuint32_t boxd[3] = {(cuuint32_t)tma_win_elems<InT, C>(), (cuuint32_t)TBH, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  if (enc(&tm, sizeof(InT) == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
          const_cast<void*>(a.src), dims, strides, boxd, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 1;
  const int tiles_x = (dw + AT - 1) / AT, tiles_y = (dh + 15) / 16;
  auto kern = warp_affine_tma_kernel<InT, C>;
  const int smem = 128 + tma_win_elems<InT, C>() * TBH * (int)sizeof(InT);
  static unsigned long long attr_mask[2] = {0, 0};  // per instantiation
  if (ensure_smem_attr(kern, smem, attr_mask) != FV_OK) return check_launch("warp_affine_tma_kernel (smem attribute)");
  dim3 grid(tiles_x, tiles_y, nb);
  kern<<<grid, dim3(32, 4), smem, st>>>(tm, a, mats);  // the tensor map first: 64-byte aligned at offset 0
  return FV_OK;
}

template <typename InT, bool PERSP>
static int launch_warp(const InT* src, int64_t s_is, int64_t s_rp, int sh, int sw, InT* dst, int64_t d_is,
                       int64_t d_rp, int dh, int dw, int c, int n, const double* mats_host, int mat_len,
                       float border_f, float border_raw, cudaStream_t st, const char* fn);

// u8 perspective, <= 1 LSB path (warp_persp_fast_kernel); C outside {1, 3, 4}
// takes the exact kernel (which meets the same gate trivially)
static int launch_persp_fast(const uint8_t* src, int64_t s_is, int64_t s_rp, int sh, int sw, uint8_t* dst,
                             int64_t d_is, int64_t d_rp, int dh, int dw, int c, int n, const double* mats_host,
                             uint8_t border, cudaStream_t st, const char* fn) {
  const float bf = (float)border / 255.0f;
  // the fast kernel's 32-bit window loads want 4-byte aligned rows, offsets
  // inside an image below 2^31 and rows at least one load window wide
  const bool fits = (c == 1 || c == 3 || c == 4) && ((reinterpret_cast<uintptr_t>(src) | (uintptr_t)s_rp) & 3) == 0 &&
                    (n <= 1 || (s_is & 3) == 0) && s_rp > 0 && (int64_t)sh * s_rp < ((int64_t)1 << 31) &&
                    sw > 4 * 3 + 1 && sh >= 2;
  if (!fits)
    return launch_warp<uint8_t, true>(src, s_is, s_rp, sh, sw, dst, d_is, d_rp, dh, dw, c, n, mats_host, 9, bf,
                                      (float)border, st, fn);
  if (n < 0 || sh < 1 || sw < 1 || dh < 1 || dw < 1)
    return set_error(FV_EINVAL, "%s: bad shape n=%d src=%dx%d dst=%dx%d c=%d", fn, n, sh, sw, dh, dw, c);
  if ((int64_t)(dh + 8 * PF_ROWS - 1) / (8 * PF_ROWS) > 65535)
    return set_error(FV_EINVAL, "%s: destination height %d too large", fn, dh);
  if (n == 0) return FV_OK;
  if (!src || !dst || !mats_host) return set_error(FV_EINVAL, "%s: null pointer", fn);
  WarpArgs a{};
  a.s_is = s_is;
  a.s_rp = s_rp;
  a.sh = sh;
  a.sw = sw;
  a.d_is = d_is;
  a.d_rp = d_rp;
  a.dh = dh;
  a.dw = dw;
  a.c = c;
  a.border_f = bf;
  a.border_raw = (float)border;
  a.one2 = kOne2Bits;
  a.zero_border = border == 0;
  WarpMats mats;
  for (int b = 0; b < n; b += MAXW) {
    const int nb = (n - b) < MAXW ? (n - b) : MAXW;
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < 9; ++j) mats.m[i][j] = mats_host[(int64_t)(b + i) * 9 + j];
    a.src = reinterpret_cast<const char*>(src) + (int64_t)b * s_is;
    a.dst = reinterpret_cast<char*>(dst) + (int64_t)b * d_is;
    dim3 grid((dw + 32 * PF_PX - 1) / (32 * PF_PX), (dh + 8 * PF_ROWS - 1) / (8 * PF_ROWS), nb);
    int rc = g_warp_path == 3 ? 1 : launch_persp_tile(a, mats, nb, st);
    if (rc > 1 || rc < 0) return rc;
    if (rc == 1) {
      switch (c) {
        case 1: warp_persp_fast_kernel<1><<<grid, dim3(32, 8), 0, st>>>(a, mats); break;
        case 3: warp_persp_fast_kernel<3><<<grid, dim3(32, 8), 0, st>>>(a, mats); break;
        default: warp_persp_fast_kernel<4><<<grid, dim3(32, 8), 0, st>>>(a, mats); break;
      }
    }
    rc = check_launch(fn);
    if (rc) return rc;
  }
  return FV_OK;
}

template <typename InT, bool PERSP>
static int launch_warp(const InT* src, int64_t s_is, int64_t s_rp, int sh, int sw, InT* dst, int64_t d_is,
                       int64_t d_rp, int dh, int dw, int c, int n, const double* mats_host, int mat_len,
                       float border_f, float border_raw, cudaStream_t st, const char* fn) {
  if (n < 0 || sh < 1 || sw < 1 || dh < 1 || dw < 1 || c < 1)
    return set_error(FV_EINVAL, "%s: bad shape n=%d src=%dx%d dst=%dx%d c=%d", fn, n, sh, sw, dh, dw, c);
  if ((int64_t)(dh + 7) / 8 > 65535) return set_error(FV_EINVAL, "%s: destination height %d too large", fn, dh);
  if (n == 0) return FV_OK;
  if (!src || !dst || !mats_host) return set_error(FV_EINVAL, "%s: null pointer", fn);
  if (sizeof(InT) == 4 && ((s_is | s_rp | d_is | d_rp) & 3))
    return set_error(FV_EINVAL, "%s: strides not f32-aligned", fn);
  WarpArgs a{};
  a.s_is = s_is;
  a.s_rp = s_rp;
  a.sh = sh;
  a.sw = sw;
  a.d_is = d_is;
  a.d_rp = d_rp;
  a.dh = dh;
  a.dw = dw;
  a.c = c;
  a.border_f = border_f;
  a.border_raw = border_raw;
  a.one2 = kOne2Bits;
  a.zero_border = (__builtin_bit_cast(uint32_t, border_f) == 0u && __builtin_bit_cast(uint32_t, border_raw) == 0u) ? 1 : 0;
  WarpMats mats;
  for (int b = 0; b < n; b += MAXW) {
    const int nb = (n - b) < MAXW ? (n - b) : MAXW;
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < 9; ++j) mats.m[i][j] = j < mat_len ? mats_host[(int64_t)(b + i) * mat_len + j] : 0.0;
    a.src = reinterpret_cast<const char*>(src) + (int64_t)b * s_is;
    a.dst = reinterpret_cast<char*>(dst) + (int64_t)b * d_is;
    dim3 block(32, 8);
    dim3 grid2((dw + 63) / 64, (dh + 8 * WARP_ROWS - 1) / (8 * WARP_ROWS), nb);  // 2 px x WARP_ROWS rows per thread
    dim3 grid1((dw + 31) / 32, (dh + 7) / 8, nb);
    // affine, 16-byte aligned rows: the SMEM-staged tile kernel
    const int64_t pb = (int64_t)c * (int64_t)sizeof(InT);
    const bool rows16 = (reinterpret_cast<uintptr_t>(a.src) & 15) == 0 && (s_rp & 15) == 0 &&
                        (nb == 1 || (s_is & 15) == 0) && ((pb * sw) & 15) == 0;
    if (!PERSP && g_warp_path == 0 && rows16 && (c == 1 || c == 3 || c == 4)) {
      int rc = g_warp_src ? launch_affine_src(a, mats, nb, (int)sizeof(InT), st) : 1;
      if (rc == 0) continue;
      if (rc != 1) return rc;
      if (g_warp_tma) {
        switch (c) {
          case 1: rc = launch_tma<InT, 1>(dw, dh, nb, st, a, mats); break;
          case 3: rc = launch_tma<InT, 3>(dw, dh, nb, st, a, mats); break;
          default: rc = launch_tma<InT, 4>(dw, dh, nb, st, a, mats); break;
        }
      }
      if (rc == 1) {  // no tensor map: the bulk-copy staged kernel
        switch (c) {
          case 1: rc = launch_tile<InT, 1>(dw, dh, nb, st, a, mats); break;
          case 3: rc = launch_tile<InT, 3>(dw, dh, nb, st, a, mats); break;
          default: rc = launch_tile<InT, 4>(dw, dh, nb, st, a, mats); break;
        }
      }
      if (rc) return rc;
      rc = check_launch(fn);
      if (rc) return rc;
      continue;
    }
    switch (c) {
      case 1: warp_kernel<InT, PERSP, 1><<<grid2, block, 0, st>>>(a, mats); break;
      case 3: warp_kernel<InT, PERSP, 3><<<grid2, block, 0, st>>>(a, mats); break;
      case 4: warp_kernel<InT, PERSP, 4><<<grid2, block, 0, st>>>(a, mats); break;
      default: warp_kernel_any<InT, PERSP><<<grid1, block, 0, st>>>(a, mats); break;
    }
    int rc = check_launch(fn);
    if (rc) return rc;
  }
  return FV_OK;
}

}  // namespace fv

using namespace fv;

extern "C" {

#ifdef FV_TEST_KNOBS
void fv_set_warp_path(int32_t mode) {
  // 2: affine without TMA tensor maps; 3: the round-1 perspective kernel (A/B);
  // 4: affine on the destination-tiled TMA kernel (no source tiles)
  g_warp_path = (mode == 2 || mode == 4) ? 0 : mode;
  g_warp_tma = mode == 2 ? 0 : 1;
  g_warp_src = (mode == 2 || mode == 4) ? 0 : 1;
}
#endif

int fv_warp_affine_f32(const float* src, int64_t s_is, int64_t s_rp, int32_t sh, int32_t sw, float* dst,
                       int64_t d_is, int64_t d_rp, int32_t dh, int32_t dw, int32_t c, int32_t n,
                       const double* minv_host, float border, void* stream) {
  return launch_warp<float, false>(src, s_is, s_rp, sh, sw, dst, d_is, d_rp, dh, dw, c, n, minv_host, 6, border,
                                   border, static_cast<cudaStream_t>(stream), "fv_warp_affine_f32");
}

int fv_warp_affine_u8(const uint8_t* src, int64_t s_is, int64_t s_rp, int32_t sh, int32_t sw, uint8_t* dst,
                      int64_t d_is, int64_t d_rp, int32_t dh, int32_t dw, int32_t c, int32_t n,
                      const double* minv_host, uint8_t border, void* stream) {
  const float bf = (float)border / 255.0f;  // IEEE division == to_float_scaled
  return launch_warp<uint8_t, false>(src, s_is, s_rp, sh, sw, dst, d_is, d_rp, dh, dw, c, n, minv_host, 6, bf,
                                     (float)border, static_cast<cudaStream_t>(stream), "fv_warp_affine_u8");
}

int fv_warp_perspective_u8(const uint8_t* src, int64_t s_is, int64_t s_rp, int32_t sh, int32_t sw, uint8_t* dst,
                           int64_t d_is, int64_t d_rp, int32_t dh, int32_t dw, int32_t c, int32_t n,
                           const double* hinv_host, uint8_t border, void* stream) {
  const float bf = (float)border / 255.0f;
  return launch_warp<uint8_t, true>(src, s_is, s_rp, sh, sw, dst, d_is, d_rp, dh, dw, c, n, hinv_host, 9, bf,
                                    (float)border, static_cast<cudaStream_t>(stream), "fv_warp_perspective_u8");
}

int fv_warp_perspective_u8_fast(const uint8_t* src, int64_t s_is, int64_t s_rp, int32_t sh, int32_t sw,
                                uint8_t* dst, int64_t d_is, int64_t d_rp, int32_t dh, int32_t dw, int32_t c,
                                int32_t n, const double* hinv_host, uint8_t border, void* stream) {
  return launch_persp_fast(src, s_is, s_rp, sh, sw, dst, d_is, d_rp, dh, dw, c, n, hinv_host, border,
                           static_cast<cudaStream_t>(stream), "fv_warp_perspective_u8_fast");
}

int fv_warp_perspective_f32(const float* src, int64_t s_is, int64_t s_rp, int32_t sh, int32_t sw, float* dst,
                            int64_t d_is, int64_t d_rp, int32_t dh, int32_t dw, int32_t c, int32_t n,
                            const double* hinv_host, float border, void* stream) {
  return launch_warp<float, true>(src, s_is, s_rp, sh, sw, dst, d_is, d_rp, dh, dw, c, n, hinv_host, 9, border,
                                  border, static_cast<cudaStream_t>(stream), "fv_warp_perspective_f32");
}

}  // extern "C"
