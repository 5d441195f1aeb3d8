// fv_resize.cu -- bilinear resize family:
//   a3  imgproc.resize_bilinear      (imgproc.py:100-123)      f32 -> f32 HWC
//   a6  service.app._resize_u8       (app.py:64-78)            u8  -> u8  HWC
//   a10 fused resize->normalise->CHW (builder contract)        u8  -> f32 CHW
//
// All three share one sampler: the reference's f64 pixel-centre map
// (imgproc.py:76-78, clip before floor :109-116) and its f32 blend order
// (imgproc.py:118-123). u8 sources enter the blend as RN(u/255)
// (image.py:159-160) and leave through x255 -> round-half-away -> u8
// (app.py:75-77, tensor.py:273-276), so the u8 result is bit-identical to the
// reference composition without its three f32 frames in memory.
//
// Two GPU paths, both exact:
//  * resize_strip_kernel (default): a CTA owns a tile of TW destination pixels
//    x a band of destination rows. The source rows the band needs stream
//    through a 4-slot shared-memory ring filled by the TMA unit
//    (cp.async.bulk + mbarrier), one row segment per bulk copy, prefetched
//    ahead of use. Horizontal taps are blended once per source row into
//    registers (h rows) and reused by every destination row that needs that
//    source row (2x upscale: each h row feeds ~4 output rows). Each thread
//    owns E consecutive HWC elements of the tile, so output rows leave as
//    16-byte stores. Sources must be 16-byte aligned (base, pitch, image
//    stride) and C <= 4.
//  * resize_gather_kernel: any alignment, channel count or scale; one thread
//    per destination pixel, taps gathered through L1.
#include <algorithm>
#include <type_traits>

#include "fv_common.cuh"

namespace fv {

enum { MODE_U8 = 0, MODE_F32 = 1, MODE_CHW = 2 };
#ifndef FV_STRIP_U8_IMM
#define FV_STRIP_U8_IMM 1  // u8 taps at immediate channel offsets from per-pixel shared addresses (A/B knob)
#endif
#ifndef FV_STRIP_ADAPT
#define FV_STRIP_ADAPT 1  // per-launch consumer-warp count (tile width) in the u8 / CHW strip modes (A/B knob)
#endif
constexpr int MAX_LUT = 4 * 256;
constexpr int kMaxStripSmem = 96 * 1024;

struct ResizeArgs {
  const void* src;
  int64_t s_is, s_rp;
  int sh, sw;
  void* dst;
  int64_t d_is, d_rp, d_ps;  // d_ps: plane stride (CHW only)
  int dh, dw;
  int c;
  double scale_x, scale_y;  // src_n / dst_n, computed once in f64 (imgproc.py:77)
  // strip kernel only
  int tile_px, band_rows, tiles_x, slot_bytes;
  int ncw;  // consumer warps per CTA (tile_px = ncw * 32 * G in the pixel-tile modes)
  int vec_store;
  f2_t one2;  // runtime {1.0f, 1.0f} (f32x2 contraction guard, fv_common.cuh)
};

struct LutArg {
  float v[MAX_LUT];
};

// ---------------------------------------------------------------------------
// generic gather kernel: one thread per destination pixel
// ---------------------------------------------------------------------------
template <typename InT, int MODE>
__global__ void __launch_bounds__(128) resize_gather_kernel(const __grid_constant__ ResizeArgs a,
                                                            const __grid_constant__ LutArg lut_arg) {
  __shared__ float lut[MODE == MODE_CHW ? MAX_LUT : 1];
  if (MODE == MODE_CHW) {
    for (int i = threadIdx.x; i < a.c * 256; i += blockDim.x) lut[i] = lut_arg.v[i];
    __syncthreads();
  }
  const int n = blockIdx.z;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= a.dw) return;
  const AxisTap tx = axis_tap(x, a.scale_x, a.sw);
  for (int y = blockIdx.y; y < a.dh; y += gridDim.y) {
    const AxisTap ty = axis_tap(y, a.scale_y, a.sh);
    const InT* r0 = row_ptr<InT>(a.src, a.s_is, a.s_rp, n, ty.i0);
    const InT* r1 = row_ptr<InT>(a.src, a.s_is, a.s_rp, n, ty.i1);
    for (int ch = 0; ch < a.c; ++ch) {
      float top = lerp_ref(tap_value(r0[tx.i0 * a.c + ch]), tap_value(r0[tx.i1 * a.c + ch]), tx.w0, tx.w1);
      float bot = lerp_ref(tap_value(r1[tx.i0 * a.c + ch]), tap_value(r1[tx.i1 * a.c + ch]), tx.w0, tx.w1);
      float o = lerp_ref(top, bot, ty.w0, ty.w1);
      if (MODE == MODE_U8) {
        row_ptr_mut<uint8_t>(a.dst, a.d_is, a.d_rp, n, y)[x * a.c + ch] = (uint8_t)unit_to_u8(o);
      } else if (MODE == MODE_F32) {
        row_ptr_mut<float>(a.dst, a.d_is, a.d_rp, n, y)[x * a.c + ch] = o;
      } else {
        float* plane = reinterpret_cast<float*>(reinterpret_cast<char*>(a.dst) + n * a.d_is + ch * a.d_ps);
        reinterpret_cast<float*>(reinterpret_cast<char*>(plane) + y * a.d_rp)[x] = lut[ch * 256 + unit_to_u8(o)];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// staged strip kernel
// ---------------------------------------------------------------------------

template <typename InT, int C, int MODE, bool AD = false>
struct StripCfg {
  // Lane ownership. MODE_U8: 4 consecutive pixels per lane (all channels:
  // per-pixel taps, one 4C-byte run per row -> C 32-bit stores). MODE_CHW: 4
  // pixels per lane at stride 32 (one coalesced 4-byte store per channel
  // plane). MODE_F32: G single floats per lane, warp-interleaved.
  static constexpr int NCW = MODE == MODE_CHW ? 5 : (MODE == MODE_U8 ? 4 : ((C == 3) ? 6 : 4));
  static constexpr int V = 1;
  static constexpr int G = MODE == MODE_F32 ? 8 : 4;
  static constexpr int EPT = MODE == MODE_F32 ? G : G * C;  // elements per thread
  static constexpr int TW_PX = MODE == MODE_F32 ? NCW * 32 * G / C : NCW * 32 * G;
  static constexpr int RING = 8;
  static constexpr int NT = (NCW + 1) * 32;  // + one producer warp
  // AD: the pixel-tile modes' variant with a per-launch consumer-warp count
  // (NCW_MIN..NCW_MAX, tile = ncw * 32 * G pixels), launched when it covers
  // the destination width with clearly fewer idle lanes than NCW; NT_MAX
  // bounds its block. The default variant keeps NCW a compile-time constant.
  static constexpr bool ADAPT = AD && MODE != MODE_F32;
  static constexpr int NCW_MIN = ADAPT ? 2 : NCW, NCW_MAX = ADAPT ? 6 : NCW;
  static constexpr int NT_MAX = (NCW_MAX + 1) * 32;
};

// Weights whose products are exact for every operand of this mode: any
// power of two for unit-range operands (u8/255 blends are never subnormal),
// only 0 and 1 for arbitrary f32 operands.
template <int MODE>
__device__ __forceinline__ bool exact_weight(float w) {
  return MODE == MODE_F32 ? (w == 0.0f || w == 1.0f) : pow2_or_zero(w);
}

// u8 pixel-tap modes: byte `CH` of tap pixel `addr` (a shared-space address)
template <int CH>
__device__ __forceinline__ uint32_t lds_u8_at(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(CH));
  return v;
}

// The u8 per-pixel-tap horizontal pass with the taps' shared addresses
// formed once per pixel (pa / pb = slot + tap offset) and each channel read
// at an immediate offset: element pair P of the thread's EPT elements.
template <int C, int MODE, int HM, int NA, int NP, int P>
struct HPassU8 {
  static __device__ __forceinline__ void run(const uint32_t (&pa)[NA], const uint32_t (&pb)[NA],
                                             const float (&wa)[NA], const float (&wb)[NA], f2_t one, f2_t (&h)[NP]) {
    constexpr int e0 = 2 * P, e1 = 2 * P + 1;
    constexpr int j0 = e0 / C, c0 = e0 % C, j1 = e1 / C, c1 = e1 % C;
    const f2_t va = unit2(0x4B000000u | lds_u8_at<c0>(pa[j0]), 0x4B000000u | lds_u8_at<c1>(pa[j1]));
    if constexpr (HM == 2) {
      h[P] = va;
    } else {
      const f2_t vb = unit2(0x4B000000u | lds_u8_at<c0>(pb[j0]), 0x4B000000u | lds_u8_at<c1>(pb[j1]));
      if constexpr (HM == 1) {
        h[P] = ffma2(vb, f2(wb[j0], wb[j1]), fmul2(va, f2(wa[j0], wa[j1])));
      } else {
        h[P] = ffma2(fmul2(vb, f2(wb[j0], wb[j1])), one, fmul2(va, f2(wa[j0], wa[j1])));
      }
    }
    HPassU8<C, MODE, HM, NA, NP, P + 1>::run(pa, pb, wa, wb, one, h);
  }
};
template <int C, int MODE, int HM, int NA, int NP>
struct HPassU8<C, MODE, HM, NA, NP, NP> {
  static __device__ __forceinline__ void run(const uint32_t (&)[NA], const uint32_t (&)[NA], const float (&)[NA],
                                             const float (&)[NA], f2_t, f2_t (&)[NP]) {}
};

// Horizontal pass of one staged source row into the h pairs. HM: 2 = copy
// (fx == 0), 1 = one exact product (fma form), 0 = the 3-op form -- chosen
// tile-uniformly, so no per-element branches. Per-pixel taps (u8 / CHW
// modes): element e reads tap offset o[e / C] + e % C (channel as immediate).
template <typename InT, int C, int MODE, int HM, int NA, int NP>
__device__ __forceinline__ void strip_hpass(const InT* seg, const int (&oa)[NA], const int (&ob)[NA],
                                            const float (&wa)[NA], const float (&wb)[NA], f2_t one,
                                            f2_t (&h)[NP]) {
  constexpr bool PX = MODE != MODE_F32;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const int e0 = 2 * p, e1 = 2 * p + 1;
    const int a0 = PX ? oa[e0 / C] + e0 % C : oa[e0], a1 = PX ? oa[e1 / C] + e1 % C : oa[e1];
    const int b0 = PX ? ob[e0 / C] + e0 % C : ob[e0], b1 = PX ? ob[e1 / C] + e1 % C : ob[e1];
    const float wa0 = PX ? wa[e0 / C] : wa[e0], wa1 = PX ? wa[e1 / C] : wa[e1];
    const float wb0 = PX ? wb[e0 / C] : wb[e0], wb1 = PX ? wb[e1 / C] : wb[e1];
    f2_t va, vb;
    if constexpr (sizeof(InT) == 1) {
      va = unit2(0x4B000000u | seg[a0], 0x4B000000u | seg[a1]);
      if constexpr (HM != 2) vb = unit2(0x4B000000u | seg[b0], 0x4B000000u | seg[b1]);
    } else {
      va = f2(seg[a0], seg[a1]);
      if constexpr (HM != 2) vb = f2(seg[b0], seg[b1]);
    }
    if constexpr (HM == 2) {
      h[p] = va;
    } else if constexpr (HM == 1) {
      h[p] = ffma2(vb, f2(wb0, wb1), fmul2(va, f2(wa0, wa1)));
    } else {
      h[p] = ffma2(fmul2(vb, f2(wb0, wb1)), one, fmul2(va, f2(wa0, wa1)));
    }
  }
}

template <typename InT, int C, int MODE, bool AD>
__global__ void __launch_bounds__(StripCfg<InT, C, MODE, AD>::NT_MAX, 3)
    resize_strip_kernel(const __grid_constant__ ResizeArgs a, const __grid_constant__ LutArg lut_arg) {
  using Cfg = StripCfg<InT, C, MODE, AD>;
  constexpr int V = Cfg::V, G = Cfg::G, EPT = Cfg::EPT, RING = Cfg::RING;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + RING;
  int4* rowtab = reinterpret_cast<int4*>(smem + 16 * RING);
  float* lut = reinterpret_cast<float*>(smem + 16 * RING + 16 * a.band_rows);
  uint8_t* slots = smem + 16 * RING + 16 * a.band_rows + (MODE == MODE_CHW ? C * 256 * 4 : 0);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int n = blockIdx.z;
  const int NCW = Cfg::ADAPT ? a.ncw : Cfg::NCW;
  const int tile_px = Cfg::ADAPT ? a.tile_px : Cfg::TW_PX;
  const int p0 = blockIdx.x * tile_px;
  const int p1 = min(p0 + tile_px, a.dw);
  const int yb = blockIdx.y * a.band_rows;
  const int nrows = min(a.band_rows, a.dh - yb);

  // source footprint of the tile: columns [xs_lo, xs_hi], one TMA bulk copy per row
  const int xs_lo = axis_tap(p0, a.scale_x, a.sw).i0;
  const int xs_hi = axis_tap(p1 - 1, a.scale_x, a.sw).i1;
  const int seg_byte = xs_lo * C * (int)sizeof(InT);
  const int shift = seg_byte & 15;
  const uint32_t nbytes = (uint32_t)((shift + (xs_hi + 1 - xs_lo) * C * (int)sizeof(InT) + 15) & ~15);

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < RING; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    fence_mbar_init();
  }
  // destination-row table of the band: y0, y1, RN(1 - fy), fy (imgproc.py:109-116)
  for (int i = tid; i < nrows; i += blockDim.x) {
    const AxisTap t = axis_tap(yb + i, a.scale_y, a.sh);
    rowtab[i] = make_int4(t.i0, t.i1, __float_as_int(t.w0), __float_as_int(t.w1));
  }
  if (MODE == MODE_CHW) {
    for (int i = tid; i < C * 256; i += blockDim.x) lut[i] = lut_arg.v[i];
  }

  // ------------------------------------------------------------------ producer
  if (warp == NCW) {
    __syncthreads();
    (void)__syncthreads_and(1);  // pair with the consumers' two tile-uniform votes
    (void)__syncthreads_and(1);
    if (lane == 0) {
      const char* src_img = reinterpret_cast<const char*>(a.src) + n * a.s_is + (seg_byte - shift);
      int last = -1, k = 0;
      for (int i = 0; i < nrows; ++i) {
        const int4 rt = rowtab[i];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int r = q == 0 ? rt.x : rt.y;
          if (r <= last) continue;  // rows are non-decreasing; each is fetched once
          last = r;
          const int slot = k % RING;
          if (k >= RING) mbar_wait_block(&empty[slot], (uint32_t)(((k / RING) - 1) & 1));
          FV_CHECK(r >= 0 && r < a.sh && seg_byte - shift >= 0 && nbytes <= (uint32_t)a.slot_bytes &&
                   (int64_t)r * a.s_rp + (seg_byte - shift) + nbytes <=
                       (int64_t)(a.sh - 1) * a.s_rp + (int64_t)a.sw * C * (int64_t)sizeof(InT));
          mbar_expect_tx(&full[slot], nbytes);
          tma_bulk_g2s(slots + slot * a.slot_bytes, src_img + (int64_t)r * a.s_rp, nbytes, &full[slot]);
          ++k;
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  // horizontal taps, loop-invariant over the band: per element (HWC modes)
  // or per pixel (CHW: all channels of a pixel share them; element e of
  // pixel j = e / C reads offset oa[j] + e % C)
  constexpr int NA = MODE != MODE_F32 ? G : EPT;  // per-pixel taps except f32 HWC
  const int shift_el = shift / (int)sizeof(InT);
  int oa[NA], ob[NA];
  float wa[NA], wb[NA];
  bool hfma = true, hcopy = true;
#pragma unroll
  for (int e = 0; e < NA; ++e) {
    int px, ch;
    if (MODE == MODE_CHW) {
      px = p0 + warp * 32 * G + e * 32 + lane;
      ch = 0;
    } else if (MODE == MODE_U8) {
      px = p0 + (warp * 32 + lane) * G + e;
      ch = 0;
    } else {
      const int idx = warp * (32 * G * V) + (e / V) * (32 * V) + lane * V + (e % V);
      px = p0 + idx / C;
      ch = idx % C;
    }
    const AxisTap t = axis_tap(px < p1 ? px : p0, a.scale_x, a.sw);
    const int o0 = shift_el + (t.i0 - xs_lo) * C + ch;
    const int o1 = shift_el + (t.i1 - xs_lo) * C + ch;
    // order the taps so that the second product is the exact one, if any
    const bool swap = !exact_weight<MODE>(t.w1) && exact_weight<MODE>(t.w0);
    oa[e] = swap ? o1 : o0;
    ob[e] = swap ? o0 : o1;
    wa[e] = swap ? t.w1 : t.w0;
    wb[e] = swap ? t.w0 : t.w1;
    hfma = hfma && exact_weight<MODE>(wb[e]);
    hcopy = hcopy && wb[e] == 0.0f && wa[e] == 1.0f;  // fx == 0: h is the tap itself
  }
  __syncthreads();  // row table, LUT and barriers ready
  // tile-uniform choice of the horizontal blend form (producer voted 1 above)
  const int all_copy = __syncthreads_and(hcopy);
  const int all_fma = __syncthreads_and(hfma);
  const int hmode = all_copy ? 2 : (all_fma ? 1 : 0);
  const f2_t one = a.one2;

  constexpr int NP = EPT / 2;  // element pairs (packed f32x2)
  f2_t ha[NP], hb[NP];
  int ra = -1, rb = -1, k = 0;

  const int slot_bytes = a.slot_bytes;
  auto consume = [&](f2_t (&h)[NP]) {
    const int slot = k % RING;
    mbar_wait(&full[slot], (uint32_t)((k / RING) & 1));
    const InT* seg = reinterpret_cast<const InT*>(slots + slot * slot_bytes);
    if constexpr (sizeof(InT) == 1 && MODE != MODE_F32 && FV_STRIP_U8_IMM) {
      const uint32_t sb = smem_u32(seg);
      uint32_t pa[NA], pb[NA];
#pragma unroll
      for (int j = 0; j < NA; ++j) {
        pa[j] = sb + (uint32_t)oa[j];
        pb[j] = sb + (uint32_t)ob[j];
      }
      if (hmode == 2) {
        HPassU8<C, MODE, 2, NA, NP, 0>::run(pa, pb, wa, wb, one, h);
      } else if (hmode == 1) {
        HPassU8<C, MODE, 1, NA, NP, 0>::run(pa, pb, wa, wb, one, h);
      } else {
        HPassU8<C, MODE, 0, NA, NP, 0>::run(pa, pb, wa, wb, one, h);
      }
    } else if (hmode == 2) {
      strip_hpass<InT, C, MODE, 2, NA, NP>(seg, oa, ob, wa, wb, one, h);
    } else if (hmode == 1) {
      strip_hpass<InT, C, MODE, 1, NA, NP>(seg, oa, ob, wa, wb, one, h);
    } else {
      strip_hpass<InT, C, MODE, 0, NA, NP>(seg, oa, ob, wa, wb, one, h);
    }
    slot_release(&empty[slot], lane);
    ++k;
  };

#pragma unroll 1
  for (int i = 0; i < nrows; ++i) {
    const int4 rt = rowtab[i];
    if (rt.x != ra) {
      if (rt.x == rb) {
#pragma unroll
        for (int p = 0; p < NP; ++p) ha[p] = hb[p];
      } else {
        consume(ha);
      }
      ra = rt.x;
    }
    if (rt.y != rb) {
      if (rt.y == ra) {
#pragma unroll
        for (int p = 0; p < NP; ++p) hb[p] = ha[p];
      } else {
        consume(hb);
      }
      rb = rt.y;
    }
    const float wy0 = __int_as_float(rt.z), wy1 = __int_as_float(rt.w);
    const f2_t WY0 = f2(wy0, wy0), WY1 = f2(wy1, wy1);
    f2_t o[NP];
    if (exact_weight<MODE>(wy1)) {
#pragma unroll
      for (int p = 0; p < NP; ++p) o[p] = ffma2(hb[p], WY1, fmul2(ha[p], WY0));
    } else if (exact_weight<MODE>(wy0)) {
#pragma unroll
      for (int p = 0; p < NP; ++p) o[p] = ffma2(ha[p], WY0, fmul2(hb[p], WY1));
    } else {
#pragma unroll
      for (int p = 0; p < NP; ++p) o[p] = ffma2(fmul2(hb[p], WY1), one, fmul2(ha[p], WY0));
    }

    const int y = yb + i;
    if constexpr (MODE == MODE_U8) {
      // the lane's 4 pixels = 4C consecutive bytes = C words (elements in order)
      const int px = p0 + (warp * 32 + lane) * G;
      uint8_t* dp = row_ptr_mut<uint8_t>(a.dst, a.d_is, a.d_rp, n, y) + (int64_t)px * C;
      uint32_t wd[C];
#pragma unroll
      for (int q = 0; q < C; ++q)
        wd[q] = pack4x2(scale_to_u8_bits2(o[2 * q], 255.0f), scale_to_u8_bits2(o[2 * q + 1], 255.0f));
      if (a.vec_store && px + G <= p1) {  // 4-byte aligned (px % 4 == 0, row 4-aligned)
#pragma unroll
        for (int q = 0; q < C; ++q) __stcs(reinterpret_cast<uint32_t*>(dp) + q, wd[q]);
      } else {
#pragma unroll
        for (int e = 0; e < EPT; ++e)
          if (px + e / C < p1) dp[e] = (uint8_t)((wd[e >> 2] >> ((e & 3) * 8)) & 0xFF);
      }
    } else if constexpr (MODE == MODE_F32) {
      float* drow = row_ptr_mut<float>(a.dst, a.d_is, a.d_rp, n, y) + p0 * C;
      const int row_el = (p1 - p0) * C;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        uint32_t lo, hi;
        f2split(o[p], lo, hi);
        const int i0 = warp * (32 * G) + (2 * p) * 32 + lane;
        if (i0 < row_el) __stcs(drow + i0, __uint_as_float(lo));
        if (i0 + 32 < row_el) __stcs(drow + i0 + 32, __uint_as_float(hi));
      }
    } else {
      char* img = reinterpret_cast<char*>(a.dst) + n * a.d_is + (int64_t)y * a.d_rp;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        uint32_t q[2];
        f2split(scale_to_u8_bits2(o[p], 255.0f), q[0], q[1]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = 2 * p + h, j = e / C, ch = e % C;
          const int px = p0 + warp * 32 * G + j * 32 + lane;
          if (px < p1) __stcs(reinterpret_cast<float*>(img + ch * a.d_ps) + px, lut[ch * 256 + (q[h] & 0xFF)]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host dispatch
// ---------------------------------------------------------------------------
#ifdef FV_TEST_KNOBS
static int g_resize_path = 0;  // 0 auto, 1 force gather, 2 force strip (no integer-ratio fast path)
#else
constexpr int g_resize_path = 0;  // product build: always the automatic selection
#endif

int resize_u8_fast(const uint8_t* src, int64_t s_is, int64_t s_rp, int sh, int sw, uint8_t* dst, int64_t d_is,
                   int64_t d_rp, int dh, int dw, int c, int n, cudaStream_t st, bool* taken);

static inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename InT, int C, int MODE>
static int launch_strip(ResizeArgs a, int n, const LutArg& lut, cudaStream_t st, bool* launched) {
  using Cfg = StripCfg<InT, C, MODE, true>;
  // consumer warps: the tuned default NCW unless another count covers dw
  // with >= 10% fewer warp-tiles (idle lanes in the last tile); ties -> wider
  a.ncw = Cfg::NCW;
  if (Cfg::ADAPT && FV_STRIP_ADAPT) {
    auto cost = [&](int w) { return (int64_t)((a.dw + w * 32 * Cfg::G - 1) / (w * 32 * Cfg::G)) * w; };
    int64_t best = cost(Cfg::NCW);
    const int64_t limit = best * 9 / 10;
    for (int w = Cfg::NCW_MAX; w >= Cfg::NCW_MIN; --w) {
      const int64_t c = cost(w);
      if (c <= limit && (a.ncw == Cfg::NCW || c < best)) {
        best = c;
        a.ncw = w;
      }
    }
  }
  const bool adapt = a.ncw != Cfg::NCW;
  a.tile_px = adapt ? a.ncw * 32 * Cfg::G : Cfg::TW_PX;
  a.tiles_x = (a.dw + a.tile_px - 1) / a.tile_px;
  // source footprint of one tile, upper bound: tile_px * scale_x + 3 px
  const double fp = (double)a.tile_px * a.scale_x;
  const int64_t fp_px = std::min<int64_t>((int64_t)fp + 3, (int64_t)a.sw);
  const int64_t slot = ((fp_px * C * (int64_t)sizeof(InT) + 16 + 15) / 16) * 16;
  // band height 16..64 rows, aiming at >= 8 CTAs per SM over the whole batch
  const int64_t rows_total = (int64_t)a.dh * a.tiles_x * n;
  a.band_rows = (int)std::max<int64_t>(16, std::min<int64_t>(64, rows_total / (8 * 148)));
  const int lut_bytes = MODE == MODE_CHW ? C * 256 * 4 : 0;
  const int64_t smem = 16 * Cfg::RING + 16 * a.band_rows + lut_bytes + Cfg::RING * slot;
  if (smem > kMaxStripSmem) return FV_OK;  // not eligible: caller falls back to gather
  a.slot_bytes = (int)slot;
  const int bands = (a.dh + a.band_rows - 1) / a.band_rows;
  auto kern = resize_strip_kernel<InT, C, MODE, false>;
  if constexpr (Cfg::ADAPT) {
    if (adapt) kern = resize_strip_kernel<InT, C, MODE, true>;
  }
  static unsigned long long attr_mask[2][2] = {{0, 0}, {0, 0}};  // per instantiation
  if (ensure_smem_attr(kern, kMaxStripSmem, attr_mask[adapt]) != FV_OK)
    return check_launch("resize_strip_kernel (smem attribute)");
  dim3 grid(a.tiles_x, bands, n);
  kern<<<grid, (a.ncw + 1) * 32, (size_t)smem, st>>>(a, lut);
  *launched = true;
  return check_launch("resize_strip_kernel");
}

template <typename InT, int MODE>
static int launch_resize(ResizeArgs a, int n, const LutArg& lut, cudaStream_t st) {
  const bool src_al = al16(a.src) && (a.s_is & 15) == 0 && (a.s_rp & 15) == 0;
  bool launched = false;
  if (g_resize_path != 1 && src_al && a.c >= 1 && a.c <= 4) {
    int rc = FV_OK;
    switch (a.c) {
      case 1: rc = launch_strip<InT, 1, MODE>(a, n, lut, st, &launched); break;
      case 2: rc = launch_strip<InT, 2, MODE>(a, n, lut, st, &launched); break;
      case 3: rc = launch_strip<InT, 3, MODE>(a, n, lut, st, &launched); break;
      case 4: rc = launch_strip<InT, 4, MODE>(a, n, lut, st, &launched); break;
    }
    if (rc != FV_OK || launched) return rc;
  }
  const int gy = a.dh < 65535 ? a.dh : 65535;
  dim3 grid((a.dw + 127) / 128, gy, n);
  resize_gather_kernel<InT, MODE><<<grid, 128, 0, st>>>(a, lut);
  return check_launch("resize_gather_kernel");
}

static int check_resize(const void* src, const void* dst, int n, int sh, int sw, int dh, int dw, int c,
                        const char* fn) {
  if (n < 0 || sh < 1 || sw < 1 || dh < 1 || dw < 1 || c < 1)
    return set_error(FV_EINVAL, "%s: bad shape n=%d src=%dx%d dst=%dx%d c=%d", fn, n, sh, sw, dh, dw, c);
  if (n > 65535) return set_error(FV_EINVAL, "%s: batch %d exceeds 65535", fn, n);
  if (n > 0 && (!src || !dst)) return set_error(FV_EINVAL, "%s: null pointer", fn);
  return FV_OK;
}

static ResizeArgs make_args(const void* src, int64_t s_is, int64_t s_rp, int sh, int sw, void* dst, int64_t d_is,
                            int64_t d_rp, int64_t d_ps, int dh, int dw, int c, int out_elem) {
  ResizeArgs a{};
  a.src = src;
  a.s_is = s_is;
  a.s_rp = s_rp;
  a.sh = sh;
  a.sw = sw;
  a.dst = dst;
  a.d_is = d_is;
  a.d_rp = d_rp;
  a.d_ps = d_ps;
  a.dh = dh;
  a.dw = dw;
  a.c = c;
  a.scale_x = (double)sw / (double)dw;  // imgproc.py:77, IEEE f64 division
  a.scale_y = (double)sh / (double)dh;
  const bool dst_al = (reinterpret_cast<uintptr_t>(dst) & 3) == 0 && (d_is & 3) == 0 && (d_rp & 3) == 0;
  a.vec_store = dst_al ? 1 : 0;
  a.one2 = kOne2Bits;
  (void)out_elem;
  return a;
}

}  // namespace fv

using namespace fv;

extern "C" {

#ifdef FV_TEST_KNOBS
void fv_set_resize_path(int32_t mode) { g_resize_path = mode; }
#endif

int fv_resize_bilinear_f32(const float* src, int64_t s_is, int64_t s_rp, int32_t sh, int32_t sw, float* dst,
                           int64_t d_is, int64_t d_rp, int32_t dh, int32_t dw, int32_t c, int32_t n, void* stream) {
  int rc = check_resize(src, dst, n, sh, sw, dh, dw, c, "fv_resize_bilinear_f32");
  if (rc || n == 0) return rc;
  if ((s_is | s_rp | d_is | d_rp) & 3) return set_error(FV_EINVAL, "fv_resize_bilinear_f32: strides not f32-aligned");
  ResizeArgs a = make_args(src, s_is, s_rp, sh, sw, dst, d_is, d_rp, 0, dh, dw, c, 4);
  static LutArg none;
  return launch_resize<float, MODE_F32>(a, n, none, static_cast<cudaStream_t>(stream));
}

int fv_resize_bilinear_u8(const uint8_t* src, int64_t s_is, int64_t s_rp, int32_t sh, int32_t sw, uint8_t* dst,
                          int64_t d_is, int64_t d_rp, int32_t dh, int32_t dw, int32_t c, int32_t n, void* stream) {
  int rc = check_resize(src, dst, n, sh, sw, dh, dw, c, "fv_resize_bilinear_u8");
  if (rc || n == 0) return rc;
  if (g_resize_path == 0) {  // exact 2:1 / 1:2 fast paths (fv_resize_fast.cu)
    bool taken = false;
    rc = resize_u8_fast(src, s_is, s_rp, sh, sw, dst, d_is, d_rp, dh, dw, c, n, static_cast<cudaStream_t>(stream),
                        &taken);
    if (rc || taken) return rc;
  }
  ResizeArgs a = make_args(src, s_is, s_rp, sh, sw, dst, d_is, d_rp, 0, dh, dw, c, 1);
  static LutArg none;
  return launch_resize<uint8_t, MODE_U8>(a, n, none, static_cast<cudaStream_t>(stream));
}

int fv_resize_normalize_chw(const uint8_t* src, int64_t s_is, int64_t s_rp, int32_t sh, int32_t sw, float* dst,
                            int64_t d_is, int64_t d_ps, int64_t d_rp, int32_t dh, int32_t dw, int32_t c, int32_t n,
                            const float* lut_host, void* stream) {
  int rc = check_resize(src, dst, n, sh, sw, dh, dw, c, "fv_resize_normalize_chw");
  if (rc || n == 0) return rc;
  if (c > 4) return set_error(FV_EINVAL, "fv_resize_normalize_chw: channels %d > 4", c);
  if (!lut_host) return set_error(FV_EINVAL, "fv_resize_normalize_chw: null lut");
  if ((d_is | d_ps | d_rp) & 3) return set_error(FV_EINVAL, "fv_resize_normalize_chw: strides not f32-aligned");
  LutArg lut;
  for (int i = 0; i < c * 256; ++i) lut.v[i] = lut_host[i];
  ResizeArgs a = make_args(src, s_is, s_rp, sh, sw, dst, d_is, d_rp, d_ps, dh, dw, c, 4);
  return launch_resize<uint8_t, MODE_CHW>(a, n, lut, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
