// fv_resize_fast.cu -- exact integer-ratio fast paths of the u8 bilinear
// resize (a6: service.app._resize_u8, app.py:64-78), selected by the host
// when dst = src/2 or dst = 2*src in BOTH axes (BASELINE configs[1]).
//
// They compute the same bits as the generic path: for these ratios the
// reference's f64 coordinate map gives the same fractional weight pattern for
// every pixel, and the weights are powers of two or 0.75, so the reference's
// separately-rounded f32 blend (imgproc.py:118-123) has a shorter exact form:
//
//  2:1 down  sx = 2x + 0.5 (never clamped): w0 = w1 = 0.5 on both axes, so
//            out = RN(top/2 + bot/2) with top = RN(v00/2 + v01/2) equals
//            RN(RN(v00 + v01) + RN(v10 + v11)) / 4 (halving is exact, no
//            subnormals), and RN(out * 255) == RN(S * 63.75). 4 taps, 3 adds.
//  1:2 up    dst px 2m   : sx = m - 0.25 -> RN(0.25 v[m-1] + RN(0.75 v[m]))
//            dst px 2m+1 : sx = m + 0.25 -> RN(RN(0.75 v[m]) + 0.25 v[m+1])
//            The 0.25 product is exact, so each is one FMA around the shared
//            P[m] = RN(0.75 v[m]); edge pixels clamp to fx = 0 (copy).
//            Rows use the same identity with Q[k] = RN(0.75 h[k]) shared by
//            destination rows 2k and 2k+1.
// Bit-exactness against the oracle is covered by tests/test_gpu_parity.py at
// the full config sizes.
//
// Memory pattern: every thread moves whole 16-byte (down) / 4-byte (up)
// aligned chunks; a warp's loads and stores cover contiguous row segments.
#include "fv_common.cuh"

namespace fv {

struct FastArgs {
  const uint8_t* src;
  int64_t s_is, s_rp;
  int sh, sw;
  uint8_t* dst;
  int64_t d_is, d_rp;
  int dh, dw;
  int n;
  int groups;  // column groups per row
  int band;    // up2: source rows per band
  int bands;
};

// ---------------------------------------------------------------------------
// 2:1 downscale. Thread = 16 destination pixels of one row (16*C bytes out,
// 2 x 32*C bytes in, all 16-byte vectors).
// ---------------------------------------------------------------------------
template <int C>
__global__ void __launch_bounds__(128) resize_down2_kernel(const __grid_constant__ FastArgs a) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)a.n * a.dh * a.groups;
  if (gid >= total) return;
  const int g = (int)(gid % a.groups);
  const int64_t t = gid / a.groups;
  const int y = (int)(t % a.dh);
  const int n = (int)(t / a.dh);
  const uint8_t* r0 = a.src + n * a.s_is + (int64_t)(2 * y) * a.s_rp;
  const uint8_t* r1 = r0 + a.s_rp;
  uint8_t* d = a.dst + n * a.d_is + (int64_t)y * a.d_rp;
  const int px0 = g * 16;
  const float K = 63.75f;  // 255 / 4

  if (px0 + 16 <= a.dw) {
    uint32_t w0[8 * C], w1[8 * C];
    const uint4* s0 = reinterpret_cast<const uint4*>(r0 + px0 * 2 * C);
    const uint4* s1 = reinterpret_cast<const uint4*>(r1 + px0 * 2 * C);
#pragma unroll
    for (int i = 0; i < 2 * C; ++i) {
      // default caching, not evict-first: neighbouring lanes' 16-byte pieces
      // share 32-byte sectors across the unrolled loads, and an evict-first
      // line can leave L2 between them (2x DRAM reads when L2 is dirty)
      const uint4 u = __ldg(s0 + i);
      w0[4 * i] = u.x, w0[4 * i + 1] = u.y, w0[4 * i + 2] = u.z, w0[4 * i + 3] = u.w;
      const uint4 v = __ldg(s1 + i);
      w1[4 * i] = v.x, w1[4 * i + 1] = v.y, w1[4 * i + 2] = v.z, w1[4 * i + 3] = v.w;
    }
    uint32_t out[4 * C];
#pragma unroll
    for (int q = 0; q < 4 * C; ++q) {
      uint32_t b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int e = 4 * q + j;            // destination byte in the group
        const int p = e / C, c = e % C;     // pixel, channel
        const int o = 2 * p * C + c;        // first tap byte in the window
        const float top = __fadd_rn(unit_of(w0, o), unit_of(w0, o + C));
        const float bot = __fadd_rn(unit_of(w1, o), unit_of(w1, o + C));
        b[j] = scaled_to_u8_bits(__fmul_rn(__fadd_rn(top, bot), K));
      }
      out[q] = pack4(b[0], b[1], b[2], b[3]);
    }
    uint4* dv = reinterpret_cast<uint4*>(d + px0 * C);
#pragma unroll
    for (int i = 0; i < C; ++i) __stcs(dv + i, make_uint4(out[4 * i], out[4 * i + 1], out[4 * i + 2], out[4 * i + 3]));
  } else {
    for (int p = px0; p < a.dw; ++p)
      for (int c = 0; c < C; ++c) {
        const int o = 2 * p * C + c;
        const float top = __fadd_rn(u8_to_unit(r0[o]), u8_to_unit(r0[o + C]));
        const float bot = __fadd_rn(u8_to_unit(r1[o]), u8_to_unit(r1[o + C]));
        d[p * C + c] = (uint8_t)(scaled_to_u8_bits(__fmul_rn(__fadd_rn(top, bot), K)) & 0xFF);
      }
  }
}

// ---------------------------------------------------------------------------
// 1:2 upscale. Thread = 4 source pixels (8 destination pixels, 8*C bytes per
// destination row) of a band of source rows; walks the band top to bottom
// keeping the horizontal results h of the previous source row and
// Q = RN(0.75 h) in registers.
// ---------------------------------------------------------------------------
template <int C>
struct Up2 {
  static constexpr int E = 8 * C;                  // destination elements per thread per row
  static constexpr int NW = (4 + 5 * C + 3) / 4;   // source words per row window [4Ct-4, ...)
};

// the thread's source window of one row: bytes [4Ct - 4, 4Ct + 5C) as words
template <int C>
__device__ __forceinline__ void up2_load(const uint8_t* row, int t, int sw, uint32_t (&w)[Up2<C>::NW]) {
  constexpr int NW = Up2<C>::NW;
  const int ws = 4 * C * t - 4;  // window start byte (4-aligned)
  const uint32_t* rw = reinterpret_cast<const uint32_t*>(row + ws);
  const int row_bytes = sw * C;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    const int b = ws + 4 * i;
    w[i] = (b >= 0 && b < row_bytes) ? __ldg(rw + i) : 0u;
  }
}

// h for the thread's 8 destination pixels from one source row's window
template <int C>
__device__ __forceinline__ void up2_h(const uint32_t (&w)[Up2<C>::NW], int t, int last_t, float (&h)[8 * C]) {
  // v[m] for source pixels m = -1..4 relative to 4t, byte offset 4 + C*m in the window
  float P[4 * C];
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int c = 0; c < C; ++c) P[m * C + c] = __fmul_rn(unit_of(w, 4 + C * m + c), 0.75f);
#pragma unroll
  for (int m = 0; m < 4; ++m)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      h[(2 * m) * C + c] = __fmaf_rn(unit_of(w, 4 + C * (m - 1) + c), 0.25f, P[m * C + c]);
      h[(2 * m + 1) * C + c] = __fmaf_rn(unit_of(w, 4 + C * (m + 1) + c), 0.25f, P[m * C + c]);
    }
  if (t == 0) {  // destination pixel 0: clamped, fx = 0 -> copy
#pragma unroll
    for (int c = 0; c < C; ++c) h[c] = unit_of(w, 4 + c);
  }
  if (t == last_t) {  // destination pixel 2W-1: clamped, fx = 0 -> copy
#pragma unroll
    for (int c = 0; c < C; ++c) h[7 * C + c] = unit_of(w, 4 + 3 * C + c);
  }
}

// one destination row from two h rows: o = fma(hb, 0.25, qa) per element,
// packed 4 bytes at a time and written as 8-byte stores (8*C bytes)
template <int C>
__device__ __forceinline__ void up2_emit(uint8_t* drow, const float (&hb)[8 * C], const float (&qa)[8 * C]) {
#pragma unroll
  for (int i = 0; i < C; ++i) {
    uint32_t w[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int e = 8 * i + 4 * j;
      w[j] = pack4(unit_to_u8_bits(__fmaf_rn(hb[e], 0.25f, qa[e])), unit_to_u8_bits(__fmaf_rn(hb[e + 1], 0.25f, qa[e + 1])),
                   unit_to_u8_bits(__fmaf_rn(hb[e + 2], 0.25f, qa[e + 2])),
                   unit_to_u8_bits(__fmaf_rn(hb[e + 3], 0.25f, qa[e + 3])));
    }
    __stcs(reinterpret_cast<uint2*>(drow) + i, make_uint2(w[0], w[1]));
  }
}
// a row that is a plain copy of h (clamped rows 0 and 2H-1, fy = 0)
template <int C>
__device__ __forceinline__ void up2_emit_copy(uint8_t* drow, const float (&h)[8 * C]) {
#pragma unroll
  for (int i = 0; i < C; ++i) {
    uint32_t w[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int e = 8 * i + 4 * j;
      w[j] = pack4(unit_to_u8_bits(h[e]), unit_to_u8_bits(h[e + 1]), unit_to_u8_bits(h[e + 2]),
                   unit_to_u8_bits(h[e + 3]));
    }
    __stcs(reinterpret_cast<uint2*>(drow) + i, make_uint2(w[0], w[1]));
  }
}

// Source row k (window wc already loaded): hn = h_k, prefetch row k+1 into
// wn, then destination rows
//   2k-1 = fma(h_k, 0.25, Q_{k-1})   (rows k-1 @ 0.75, k @ 0.25)
//   2k   = fma(h_{k-1}, 0.25, Q_k)   (rows k-1 @ 0.25, k @ 0.75)
// q holds Q_{k-1} on entry and Q_k on exit; hp = h_{k-1}.
template <int C>
__device__ __forceinline__ void up2_step(const uint8_t* img, uint8_t* dimg, const FastArgs& a, int t, int k, int k1,
                                         const uint32_t (&wc)[Up2<C>::NW], uint32_t (&wn)[Up2<C>::NW],
                                         const float (&hp)[8 * C], float (&q)[8 * C], float (&hn)[8 * C]) {
  up2_h<C>(wc, t, a.groups - 1, hn);
  if (k + 1 < k1) up2_load<C>(img + (int64_t)(k + 1) * a.s_rp, t, a.sw, wn);
  if (k == 0) {
    up2_emit_copy<C>(dimg, hn);
  } else {
    up2_emit<C>(dimg + (int64_t)(2 * k - 1) * a.d_rp, hn, q);
  }
#pragma unroll
  for (int e = 0; e < 8 * C; ++e) q[e] = __fmul_rn(hn[e], 0.75f);
  if (k > 0) up2_emit<C>(dimg + (int64_t)(2 * k) * a.d_rp, hp, q);
}

template <int C>
__global__ void __launch_bounds__(128, 4) resize_up2_kernel(const __grid_constant__ FastArgs a) {
  constexpr int E = Up2<C>::E, NW = Up2<C>::NW;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)a.n * a.bands * a.groups;
  if (gid >= total) return;
  const int t = (int)(gid % a.groups);
  const int64_t r = gid / a.groups;
  const int band = (int)(r % a.bands);
  const int n = (int)(r / a.bands);
  const int k0 = band * a.band;
  const int k1 = min(k0 + a.band, a.sh);
  const uint8_t* img = a.src + n * a.s_is;
  uint8_t* dimg = a.dst + n * a.d_is + t * 8 * C;

  // two h buffers and two source windows used alternately (no register copies)
  float h0[E], h1[E], q[E];
  uint32_t w0[NW], w1[NW];
  if (k0 > 0) {
    up2_load<C>(img + (int64_t)(k0 - 1) * a.s_rp, t, a.sw, w1);
    up2_load<C>(img + (int64_t)k0 * a.s_rp, t, a.sw, w0);
    up2_h<C>(w1, t, a.groups - 1, h0);
#pragma unroll
    for (int e = 0; e < E; ++e) q[e] = __fmul_rn(h0[e], 0.75f);
  } else {
    up2_load<C>(img, t, a.sw, w0);
  }
  int k = k0;
#pragma unroll 1
  for (; k + 1 < k1; k += 2) {
    up2_step<C>(img, dimg, a, t, k, k1, w0, w1, h0, q, h1);
    up2_step<C>(img, dimg, a, t, k + 1, k1, w1, w0, h1, q, h0);
  }
  if (k < k1) {
    up2_step<C>(img, dimg, a, t, k, k1, w0, w1, h0, q, h1);
    if (k1 == a.sh) up2_emit_copy<C>(dimg + (int64_t)(2 * a.sh - 1) * a.d_rp, h1);
  } else if (k1 == a.sh) {
    up2_emit_copy<C>(dimg + (int64_t)(2 * a.sh - 1) * a.d_rp, h0);
  }
}

// ---------------------------------------------------------------------------
// host side: returns true when a fast path took the call
// ---------------------------------------------------------------------------
static inline bool aligned(const void* p, int m) { return (reinterpret_cast<uintptr_t>(p) % m) == 0; }

template <int C>
static int launch_fast_c(const FastArgs& a0, bool down, cudaStream_t st) {
  FastArgs a = a0;
  if (down) {
    a.groups = (a.dw + 15) / 16;
    const int64_t total = (int64_t)a.n * a.dh * a.groups;
    resize_down2_kernel<C><<<(unsigned)((total + 127) / 128), 128, 0, st>>>(a);
  } else {
    a.groups = a.sw / 4;
    a.band = 32;
    a.bands = (a.sh + a.band - 1) / a.band;
    const int64_t total = (int64_t)a.n * a.bands * a.groups;
    resize_up2_kernel<C><<<(unsigned)((total + 127) / 128), 128, 0, st>>>(a);
  }
  return check_launch(down ? "resize_down2_kernel" : "resize_up2_kernel");
}

// Called by fv_resize_bilinear_u8 before the generic paths. *taken = false
// leaves the call to them.
int resize_u8_fast(const uint8_t* src, int64_t s_is, int64_t s_rp, int sh, int sw, uint8_t* dst, int64_t d_is,
                   int64_t d_rp, int dh, int dw, int c, int n, cudaStream_t st, bool* taken) {
  *taken = false;
  if (c != 1 && c != 3 && c != 4) return FV_OK;
  const bool down = (sw == 2 * dw && sh == 2 * dh);
  const bool up = (dw == 2 * sw && dh == 2 * sh);
  if (!down && !up) return FV_OK;
  if (n == 1) s_is = d_is = 0;
  if (down) {
    if (!aligned(src, 16) || !aligned(dst, 16) || (s_is | s_rp | d_is | d_rp) & 15) return FV_OK;
  } else {
    if (sw % 4 != 0 || sh < 2 || !aligned(src, 4) || !aligned(dst, 8) || (s_is | s_rp) & 3 || (d_is | d_rp) & 7)
      return FV_OK;
  }
  FastArgs a{src, s_is, s_rp, sh, sw, dst, d_is, d_rp, dh, dw, n, 0, 0, 0};
  *taken = true;
  switch (c) {
    case 1: return launch_fast_c<1>(a, down, st);
    case 3: return launch_fast_c<3>(a, down, st);
    default: return launch_fast_c<4>(a, down, st);
  }
}

}  // namespace fv
