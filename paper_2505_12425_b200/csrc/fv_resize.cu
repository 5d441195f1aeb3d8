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

#include "fv_common.cuh"

namespace fv {

enum { MODE_U8 = 0, MODE_F32 = 1, MODE_CHW = 2 };
constexpr int RING = 4;
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
  int vec_store;
};

struct LutArg {
  float v[MAX_LUT];
};

// ---------------------------------------------------------------------------
// output stage
// ---------------------------------------------------------------------------
template <typename InT, int MODE>
struct OutT;
template <>
struct OutT<uint8_t, MODE_U8> {
  using T = uint8_t;
};
template <>
struct OutT<float, MODE_F32> {
  using T = float;
};
template <>
struct OutT<uint8_t, MODE_CHW> {
  using T = float;
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

// Sorted distinct source rows a band needs: the union of y0(y), y1(y) over
// the band's destination rows. Both are non-decreasing in y and y1 <= y0 + 1,
// so a row not yet seen is always above every row seen so far. Consumer and
// producer walk the same sequence.
struct RowSeq {
  int y, k, last;
};
__device__ __forceinline__ int next_row(RowSeq& s, int ye, double scale_y, int sh) {
  while (s.y < ye) {
    const AxisTap t = axis_tap(s.y, scale_y, sh);
    const int r = s.k == 0 ? t.i0 : t.i1;
    if (s.k == 1) {
      s.k = 0;
      ++s.y;
    } else {
      s.k = 1;
    }
    if (r > s.last) {  // y0(y+1) may be below y1(y): emit each row once, in order
      s.last = r;
      return r;
    }
  }
  return -1;
}

template <typename InT, int C, int E, int MODE, int NT>
__global__ void __launch_bounds__(NT, 2) resize_strip_kernel(const __grid_constant__ ResizeArgs a,
                                                             const __grid_constant__ LutArg lut_arg) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  float* lut = reinterpret_cast<float*>(smem + 64);
  uint8_t* slots = smem + 64 + (MODE == MODE_CHW ? C * 256 * 4 : 0);

  const int tid = threadIdx.x;
  const int n = blockIdx.z;
  const int tile = blockIdx.x;
  const int p0 = tile * a.tile_px;
  const int p1 = min(p0 + a.tile_px, a.dw);
  const int yb = blockIdx.y * a.band_rows;
  const int ye = min(yb + a.band_rows, a.dh);

  // source footprint of the tile: columns [xs_lo, xs_hi]
  const int xs_lo = axis_tap(p0, a.scale_x, a.sw).i0;
  const int xs_hi = axis_tap(p1 - 1, a.scale_x, a.sw).i1;
  const int seg_byte = xs_lo * C * (int)sizeof(InT);
  const int shift = seg_byte & 15;
  const int gstart = seg_byte - shift;
  const uint32_t nbytes = (uint32_t)((shift + (xs_hi + 1 - xs_lo) * C * (int)sizeof(InT) + 15) & ~15);
  const char* src_img = reinterpret_cast<const char*>(a.src) + n * a.s_is + gstart;

  RowSeq ps = {yb, 0, -1};
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < RING; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  if (MODE == MODE_CHW) {
    for (int i = tid; i < C * 256; i += NT) lut[i] = lut_arg.v[i];
  }
  __syncthreads();
  if (tid == 0) {
#pragma unroll 1
    for (int s = 0; s < RING; ++s) {
      const int r = next_row(ps, ye, a.scale_y, a.sh);
      if (r < 0) break;
      mbar_expect_tx(&full[s], nbytes);
      tma_bulk_g2s(slots + s * a.slot_bytes, src_img + r * a.s_rp, nbytes, &full[s]);
    }
  }

  // per-element horizontal taps (loop-invariant over the band)
  const int shift_el = shift / (int)sizeof(InT);
  int o0[E], o1[E];
  float w0[E], w1[E];
  bool valid[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int idx = tid * E + e;
    const int px = p0 + idx / C;
    const int ch = idx % C;
    valid[e] = px < p1;
    const AxisTap t = axis_tap(valid[e] ? px : p0, a.scale_x, a.sw);
    o0[e] = shift_el + (t.i0 - xs_lo) * C + ch;
    o1[e] = shift_el + (t.i1 - xs_lo) * C + ch;
    w0[e] = t.w0;
    w1[e] = t.w1;
  }

  float ha[E], hb[E];
  int ra = -1, rb = -1;
  int k = 0;  // source rows consumed

  auto consume = [&](float (&h)[E]) {
    const int slot = k % RING;
    mbar_wait(&full[slot], (uint32_t)((k / RING) & 1));
    const InT* seg = reinterpret_cast<const InT*>(slots + slot * a.slot_bytes);
#pragma unroll
    for (int e = 0; e < E; ++e) h[e] = lerp_ref(tap_value(seg[o0[e]]), tap_value(seg[o1[e]]), w0[e], w1[e]);
    __syncthreads();  // every thread is done with this slot
    if (tid == 0) {
      const int r = next_row(ps, ye, a.scale_y, a.sh);
      if (r >= 0) {
        fence_proxy_async();
        mbar_expect_tx(&full[slot], nbytes);
        tma_bulk_g2s(slots + slot * a.slot_bytes, src_img + r * a.s_rp, nbytes, &full[slot]);
      }
    }
    ++k;
  };

  using OT = typename OutT<InT, MODE>::T;
#pragma unroll 1
  for (int y = yb; y < ye; ++y) {
    const AxisTap ty = axis_tap(y, a.scale_y, a.sh);
    if (ty.i0 != ra) {
      if (ty.i0 == rb) {
#pragma unroll
        for (int e = 0; e < E; ++e) ha[e] = hb[e];
      } else {
        consume(ha);
      }
      ra = ty.i0;
    }
    if (ty.i1 != rb) {
      if (ty.i1 == ra) {
#pragma unroll
        for (int e = 0; e < E; ++e) hb[e] = ha[e];
      } else {
        consume(hb);
      }
      rb = ty.i1;
    }

    if constexpr (MODE == MODE_U8) {
      uint8_t* drow = row_ptr_mut<uint8_t>(a.dst, a.d_is, a.d_rp, n, y) + p0 * C + tid * E;
      uint32_t q[E];
#pragma unroll
      for (int e = 0; e < E; ++e) q[e] = unit_to_u8(lerp_ref(ha[e], hb[e], ty.w0, ty.w1));
      if (a.vec_store && valid[E - 1]) {
        static_assert(E % 16 == 0, "u8 strip stores 16-byte vectors");
#pragma unroll
        for (int v = 0; v < E / 16; ++v) {
          uint32_t wd[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int b = v * 16 + j * 4;
            wd[j] = __byte_perm(__byte_perm(q[b], q[b + 1], 0x0040), __byte_perm(q[b + 2], q[b + 3], 0x0040),
                                0x5410);
          }
          __stcs(reinterpret_cast<uint4*>(drow) + v, make_uint4(wd[0], wd[1], wd[2], wd[3]));
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (valid[e]) drow[e] = (uint8_t)q[e];
      }
    } else if constexpr (MODE == MODE_F32) {
      float* drow = row_ptr_mut<float>(a.dst, a.d_is, a.d_rp, n, y) + p0 * C + tid * E;
      float o[E];
#pragma unroll
      for (int e = 0; e < E; ++e) o[e] = lerp_ref(ha[e], hb[e], ty.w0, ty.w1);
      if (a.vec_store && valid[E - 1]) {
        static_assert(E % 4 == 0, "f32 strip stores 16-byte vectors");
#pragma unroll
        for (int v = 0; v < E / 4; ++v)
          __stcs(reinterpret_cast<float4*>(drow) + v, make_float4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]));
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (valid[e]) drow[e] = o[e];
      }
    } else {  // MODE_CHW: thread owns pixels [p0 + 4*tid, +4), all C channels
      static_assert(E == 4 * C, "CHW strip: 4 pixels per thread");
      char* img = reinterpret_cast<char*>(a.dst) + n * a.d_is + y * a.d_rp;
      const int px = p0 + tid * 4;
#pragma unroll
      for (int ch = 0; ch < C; ++ch) {
        float o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int e = j * C + ch;
          o[j] = lut[ch * 256 + unit_to_u8(lerp_ref(ha[e], hb[e], ty.w0, ty.w1))];
        }
        float* dp = reinterpret_cast<float*>(img + ch * a.d_ps) + px;
        if (a.vec_store && valid[E - 1]) {
          __stcs(reinterpret_cast<float4*>(dp), make_float4(o[0], o[1], o[2], o[3]));
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (valid[j * C]) dp[j] = o[j];
        }
      }
    }
  }
  (void)sizeof(OT);
}

// ---------------------------------------------------------------------------
// host dispatch
// ---------------------------------------------------------------------------
static int g_resize_path = 0;  // 0 auto, 1 force gather

template <typename InT, int C, int MODE>
struct StripCfg;
// u8 HWC: 16 bytes per thread
template <int C>
struct StripCfg<uint8_t, C, MODE_U8> {
  static constexpr int NT = (C == 3) ? 192 : 128;
  static constexpr int E = 16;
};
template <int C>
struct StripCfg<float, C, MODE_F32> {
  static constexpr int NT = (C == 3) ? 192 : 128;
  static constexpr int E = 4;
};
template <int C>
struct StripCfg<uint8_t, C, MODE_CHW> {
  static constexpr int NT = (C == 3) ? 192 : 128;
  static constexpr int E = 4 * C;
};

static inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <typename InT, int C, int MODE>
static int launch_strip(ResizeArgs a, int n, const LutArg& lut, cudaStream_t st, bool* launched) {
  using Cfg = StripCfg<InT, C, MODE>;
  constexpr int NT = Cfg::NT, E = Cfg::E;
  a.tile_px = NT * E / C;
  a.tiles_x = (a.dw + a.tile_px - 1) / a.tile_px;
  // source footprint of one tile, upper bound: tile_px * scale_x + 3 px
  const double fp = (double)a.tile_px * a.scale_x;
  const int64_t fp_px = std::min<int64_t>((int64_t)fp + 3, (int64_t)a.sw);
  const int64_t slot = ((fp_px * C * (int64_t)sizeof(InT) + 16 + 15) / 16) * 16;
  const int lut_bytes = MODE == MODE_CHW ? C * 256 * 4 : 0;
  const int64_t smem = 64 + lut_bytes + RING * slot;
  if (smem > kMaxStripSmem) return FV_OK;  // not eligible: caller falls back to gather
  a.slot_bytes = (int)slot;
  // band height 8..64 rows, aiming at >= 8 CTAs per SM over the whole batch
  const int64_t rows_total = (int64_t)a.dh * a.tiles_x * n;
  a.band_rows = (int)std::max<int64_t>(8, std::min<int64_t>(64, rows_total / (8 * 148)));
  const int bands = (a.dh + a.band_rows - 1) / a.band_rows;
  auto kern = resize_strip_kernel<InT, C, E, MODE, NT>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxStripSmem);
    attr_set = true;
  }
  dim3 grid(a.tiles_x, bands, n);
  kern<<<grid, NT, (size_t)smem, st>>>(a, lut);
  *launched = true;
  return check_launch("resize_strip_kernel");
}

template <typename InT, int MODE>
static int launch_resize(ResizeArgs a, int n, const LutArg& lut, cudaStream_t st) {
  const bool src_al = al16(a.src) && (a.s_is & 15) == 0 && (a.s_rp & 15) == 0;
  bool launched = false;
  if (g_resize_path == 0 && src_al && a.c >= 1 && a.c <= 4) {
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
  const bool dst_al = al16(dst) && (d_is & 15) == 0 && (d_rp & 15) == 0 && (d_ps & 15) == 0;
  a.vec_store = dst_al ? 1 : 0;
  (void)out_elem;
  return a;
}

}  // namespace fv

using namespace fv;

extern "C" {

void fv_set_resize_path(int32_t mode) { g_resize_path = mode; }

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
