// fv_gray.cu -- a1: imgproc.gray_from_rgb (imgproc.py:43-64) and
// a4: image.to_float_scaled (image.py:150-160).
//
// gray u8 is exact integer work. The reference computes
//   g = (f64(r)*0.299 + f64(g)*0.587) + f64(b)*0.114;  out = floor(g + 0.5)
// With S = 299r + 587g + 114b the exact value is S/1000 and the f64 error is
// < 1e-12, so floor(g + 0.5) == (S + 500) / 1000 unless S % 1000 == 500 (an
// exact decimal tie, 16,782 of 2^24 triples). Ties re-run the reference's f64
// op order (__dmul_rn/__dadd_rn, never contracted): 3,464 of them round down.
// Exhaustively verified against the oracle over all 2^24 triples
// (tests/test_gpu_parity.py::test_gray_exhaustive).
//
// Memory: 3 B in + 1 B out per pixel, HBM-bound. The vector path moves 16
// pixels per thread as 3 x 16 B loads and one 16 B store.
#include "fv_common.cuh"

#ifndef FV_GRAY_DP4A
#define FV_GRAY_DP4A 1  // vec kernel: luma by two IDP4A per pixel (A/B knob: 0 = per-byte extraction)
#endif

namespace fv {

__device__ __forceinline__ uint32_t gray_u8_px(uint32_t r, uint32_t g, uint32_t b) {
  uint32_t s = 299u * r + 587u * g + 114u * b + 500u;
  uint32_t q = __umulhi(s, 274877907u) >> 6;  // s / 1000 for s <= 255500
  if (s == q * 1000u) {
    double v = __dadd_rn(__dadd_rn(__dmul_rn((double)r, 0.299), __dmul_rn((double)g, 0.587)),
                         __dmul_rn((double)b, 0.114));
    q = (uint32_t)floor(__dadd_rn(v, 0.5));
  }
  return q;
}

// The same from a word holding (r, g, b) in its low three bytes: S + 500 =
// 256 (r + 2g) + (43r + 75g + 114b + 500) as two byte dot products (IDP4A).
__device__ __forceinline__ uint32_t gray_u8_word(uint32_t v) {
  const uint32_t lo = __dp4a(v, 0x00724B2Bu, 500u);  // 43 r + 75 g + 114 b + 500
  const uint32_t hi = __dp4a(v, 0x00000201u, 0u);    // r + 2 g
  const uint32_t s = (hi << 8) + lo;
  uint32_t q = __umulhi(s, 274877907u) >> 6;  // s / 1000 for s <= 255500
  if (s == q * 1000u) {
    const uint32_t r = v & 0xFF, g = (v >> 8) & 0xFF, b = (v >> 16) & 0xFF;
    const double x = __dadd_rn(__dadd_rn(__dmul_rn((double)r, 0.299), __dmul_rn((double)g, 0.587)),
                               __dmul_rn((double)b, 0.114));
    q = (uint32_t)floor(__dadd_rn(x, 0.5));
  }
  return q;
}

// Four pixels from their 12 bytes (three words) to one output word. Per pixel
// the 64-bit product (S + 500) * M, M = ceil(2^32 / 1000) = 4294968, gives the
// quotient in its high word (M * 1000 - 2^32 = 704, and 704 S / (1000 * 2^32) <
// 1 / 1000 for S + 500 <= 255500) and the tie test in its low one: with S + 500 =
// 1000 q + t the low word is 704 q + t M < 2^32, below M exactly when t = 0.
// The four tie flags OR into one predicate, so the rare f64 re-run costs one
// branch per output word instead of one per pixel (FV_GRAY_QUAD_TIE 0: the
// per-pixel branch, the A/B baseline).
#ifndef FV_GRAY_QUAD_TIE
#define FV_GRAY_QUAD_TIE 1
#endif
__device__ __forceinline__ uint32_t gray_u8_quad(const uint32_t* wd) {
  uint32_t w3[4] = {wd[0], __funnelshift_r(wd[0], wd[1], 24), __funnelshift_r(wd[1], wd[2], 16), wd[2] >> 8};
  uint32_t q[4];
#if FV_GRAY_QUAD_TIE
  bool tie = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t lo = __dp4a(w3[i], 0x00724B2Bu, 500u);  // 43 r + 75 g + 114 b + 500
    const uint32_t hi = __dp4a(w3[i], 0x00000201u, 0u);    // r + 2 g
    const uint64_t p = (uint64_t)((hi << 8) + lo) * 4294968u;
    q[i] = (uint32_t)(p >> 32);
    tie |= (uint32_t)p < 4294968u;
  }
  if (tie) {  // 12% of warps per word on uniform random input; re-running only the tie pixels from the kept low
              // words measured slower (0.0477 vs 0.0456 ms for 32 frames), as did 2 or 4 rows per thread on top
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = gray_u8_word(w3[i]);
  }
#else
#pragma unroll
  for (int i = 0; i < 4; ++i) q[i] = gray_u8_word(w3[i]);
#endif
  return pack4(q[0], q[1], q[2], q[3]);
}

// 16 pixels per thread; all of src/dst base, pitch and image stride are
// 16-byte aligned (checked on the host). Luma by two IDP4A per pixel
// (gray_u8_word): 0.058 -> 0.050 ms for 32 1080p frames in one launch (the
// per-byte extraction made this kernel issue-bound); loading two or four
// rows per thread before the arithmetic measured slower (0.060 / 0.064 ms).
// One tie branch per output word (gray_u8_quad): 0.050 -> 0.0456 ms.
__global__ void __launch_bounds__(128) gray_u8_vec_kernel(const uint8_t* __restrict__ src, int64_t s_is,
                                                          int64_t s_rp, uint8_t* __restrict__ dst,
                                                          int64_t d_is, int64_t d_rp, int h, int w) {
  const int n = blockIdx.z;
  const int groups = (w + 15) >> 4;
  const int gx = blockIdx.x * blockDim.x + threadIdx.x;
  if (gx >= groups) return;
  for (int y = blockIdx.y; y < h; y += gridDim.y) {
    const uint8_t* s = row_ptr<uint8_t>(src, s_is, s_rp, n, y) + gx * 48;
    uint8_t* d = row_ptr_mut<uint8_t>(dst, d_is, d_rp, n, y) + gx * 16;
    const int x0 = gx * 16;
    if (x0 + 16 <= w) {
      uint4 v[3];
      const uint4* s4 = reinterpret_cast<const uint4*>(s);
      v[0] = __ldg(s4);
      v[1] = __ldg(s4 + 1);
      v[2] = __ldg(s4 + 2);
      const uint32_t* wd = reinterpret_cast<const uint32_t*>(v);
      uint32_t out[4] = {0, 0, 0, 0};
#if FV_GRAY_DP4A
#pragma unroll
      for (int j = 0; j < 4; ++j) out[j] = gray_u8_quad(wd + 3 * j);
#else
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int k = 3 * i;
        uint32_t r = (wd[k >> 2] >> ((k & 3) * 8)) & 0xFF;
        uint32_t g = (wd[(k + 1) >> 2] >> (((k + 1) & 3) * 8)) & 0xFF;
        uint32_t b = (wd[(k + 2) >> 2] >> (((k + 2) & 3) * 8)) & 0xFF;
        out[i >> 2] |= gray_u8_px(r, g, b) << ((i & 3) * 8);
      }
#endif
      __stcs(reinterpret_cast<uint4*>(d), make_uint4(out[0], out[1], out[2], out[3]));
    } else {
      for (int i = 0; x0 + i < w; ++i) d[i] = (uint8_t)gray_u8_px(s[3 * i], s[3 * i + 1], s[3 * i + 2]);
    }
  }
}

// Same work as gray_u8_vec_kernel with a flat (image, row, group) index and
// 512-thread CTAs: with 8 pixels per thread a 1080p frame is ~260K groups,
// ~510 CTAs -- one wave, few CTA launches (launch latency dominates such
// small frames; 16 pixels per thread left the wave too short of warps).
#ifndef FV_GRAY_THREADS
#define FV_GRAY_THREADS 512
#endif
constexpr int kFlatThreads = FV_GRAY_THREADS;
#ifndef FV_GRAY_GY
#define FV_GRAY_GY 65535  // vec kernel: grid rows (each thread loops over h / FV_GRAY_GY rows)
#endif
#ifndef FV_GRAY_FLAT_MAX
#define FV_GRAY_FLAT_MAX (148 * 2048 * 4)  // 16-pixel groups up to which the flat kernel runs
#endif
#ifndef FV_GRAY_PX
#define FV_GRAY_PX 8  // measured: 16 -> 8 pixels per thread 3.3 -> 2.9 us per 1080p frame; 4 is slower
#endif
template <int PX>  // pixels per thread: 16 / 8 / 4 (three 16- / 8- / 4-byte loads)
__global__ void __launch_bounds__(kFlatThreads) gray_u8_flat_kernel(const uint8_t* __restrict__ src, int64_t s_is,
                                                           int64_t s_rp, uint8_t* __restrict__ dst, int64_t d_is,
                                                           int64_t d_rp, int h, int w, int64_t total) {
  // Programmatic dependent launch: wait for the previous grid in the stream
  // (its writes visible) before reading, then let the next grid launch -- its
  // CTA launch overlaps this grid's run instead of following its completion.
  // Before waiting, pull this thread's source sectors into L2: a prefetch has
  // no memory-order effect and L2 is the point of coherence, so a previous
  // grid still writing this input cannot make the later loads stale -- the
  // prefetch only overlaps this frame's DRAM ramp with that grid's tail.
  const int groups = (w + PX - 1) / PX;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = gid < total;
  const int gx = live ? (int)(gid % groups) : 0;
  const int64_t r = live ? gid / groups : 0;
  const int y = (int)(r % h);
  const int n = (int)(r / h);
  const uint8_t* s = row_ptr<uint8_t>(src, s_is, s_rp, n, y) + gx * 3 * PX;
  if (live) {
    const int last = min(3 * PX, 3 * (w - gx * PX)) - 1;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(s));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(s + last));
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");  // (earlier trigger measured slower)
  if (!live) return;
  uint8_t* d = row_ptr_mut<uint8_t>(dst, d_is, d_rp, n, y) + gx * PX;
  const int x0 = gx * PX;
  if (x0 + PX <= w) {
    uint32_t wd[3 * PX / 4];
    if (PX == 16) {
      const uint4* s4 = reinterpret_cast<const uint4*>(s);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const uint4 v = __ldg(s4 + k);
        wd[4 * k] = v.x, wd[4 * k + 1] = v.y, wd[4 * k + 2] = v.z, wd[4 * k + 3] = v.w;
      }
    } else if (PX == 8) {
      const uint2* s2 = reinterpret_cast<const uint2*>(s);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const uint2 v = __ldg(s2 + k);
        wd[2 * k] = v.x, wd[2 * k + 1] = v.y;
      }
    } else {
      const uint32_t* s1 = reinterpret_cast<const uint32_t*>(s);
#pragma unroll
      for (int k = 0; k < 3; ++k) wd[k] = __ldg(s1 + k);
    }
    uint32_t out[PX / 4];
#if FV_GRAY_DP4A
#pragma unroll
    for (int j = 0; j < PX / 4; ++j) out[j] = gray_u8_quad(wd + 3 * j);
#else
#pragma unroll
    for (int i = 0; i < PX / 4; ++i) out[i] = 0;
#pragma unroll
    for (int i = 0; i < PX; ++i) {
      const int k = 3 * i;
      uint32_t rr = (wd[k >> 2] >> ((k & 3) * 8)) & 0xFF;
      uint32_t g = (wd[(k + 1) >> 2] >> (((k + 1) & 3) * 8)) & 0xFF;
      uint32_t b = (wd[(k + 2) >> 2] >> (((k + 2) & 3) * 8)) & 0xFF;
      out[i >> 2] |= gray_u8_px(rr, g, b) << ((i & 3) * 8);
    }
#endif
    if (PX == 16) __stcs(reinterpret_cast<uint4*>(d), make_uint4(out[0], out[1], out[2], out[3]));
    else if (PX == 8) __stcs(reinterpret_cast<uint2*>(d), make_uint2(out[0], out[1]));
    else __stcs(reinterpret_cast<unsigned int*>(d), out[0]);
  } else {
    for (int i = 0; x0 + i < w; ++i) d[i] = (uint8_t)gray_u8_px(s[3 * i], s[3 * i + 1], s[3 * i + 2]);
  }
}

// any alignment / pitch: one pixel per thread
__global__ void gray_u8_px_kernel(const uint8_t* __restrict__ src, int64_t s_is, int64_t s_rp,
                                  uint8_t* __restrict__ dst, int64_t d_is, int64_t d_rp, int h, int w) {
  const int n = blockIdx.z;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= w) return;
  for (int y = blockIdx.y; y < h; y += gridDim.y) {
    const uint8_t* s = row_ptr<uint8_t>(src, s_is, s_rp, n, y) + 3 * x;
    row_ptr_mut<uint8_t>(dst, d_is, d_rp, n, y)[x] = (uint8_t)gray_u8_px(s[0], s[1], s[2]);
  }
}

// f32: imgproc.py:59-62 -- widen to f64, same sum order, narrow with RN.
__global__ void gray_f32_kernel(const float* __restrict__ src, int64_t s_is, int64_t s_rp,
                                float* __restrict__ dst, int64_t d_is, int64_t d_rp, int h, int w) {
  const int n = blockIdx.z;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= w) return;
  for (int y = blockIdx.y; y < h; y += gridDim.y) {
    const float* s = row_ptr<float>(src, s_is, s_rp, n, y) + 3 * x;
    double v = __dadd_rn(__dadd_rn(__dmul_rn((double)s[0], 0.299), __dmul_rn((double)s[1], 0.587)),
                         __dmul_rn((double)s[2], 0.114));
    row_ptr_mut<float>(dst, d_is, d_rp, n, y)[x] = __double2float_rn(v);
  }
}

// image.py:159-160: f32(u) / f32(255); 16 elements per thread when aligned.
__global__ void to_float_scaled_kernel(const uint8_t* __restrict__ src, int64_t s_is, int64_t s_rp,
                                       float* __restrict__ dst, int64_t d_is, int64_t d_rp, int h,
                                       int row_elems, bool vec) {
  const int n = blockIdx.z;
  const int gx = blockIdx.x * blockDim.x + threadIdx.x;
  const int e0 = gx * 16;
  if (e0 >= row_elems) return;
  for (int y = blockIdx.y; y < h; y += gridDim.y) {
    const uint8_t* s = row_ptr<uint8_t>(src, s_is, s_rp, n, y) + e0;
    float* d = row_ptr_mut<float>(dst, d_is, d_rp, n, y) + e0;
    if (vec && e0 + 16 <= row_elems) {
      uint4 v = __ldcs(reinterpret_cast<const uint4*>(s));
      const uint32_t* wd = reinterpret_cast<const uint32_t*>(&v);
      float f[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) f[i] = u8_to_unit((wd[i >> 2] >> ((i & 3) * 8)) & 0xFF);
      float4* d4 = reinterpret_cast<float4*>(d);
#pragma unroll
      for (int i = 0; i < 4; ++i) __stcs(d4 + i, make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]));
    } else {
      for (int i = 0; i < 16 && e0 + i < row_elems; ++i) d[i] = u8_to_unit(s[i]);
    }
  }
}

static inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static inline bool al16(int64_t v) { return (v & 15) == 0; }

static int check_common(const void* src, const void* dst, int32_t n, int32_t h, int32_t w, const char* fn) {
  if (n < 0 || h < 1 || w < 1) return set_error(FV_EINVAL, "%s: bad shape n=%d h=%d w=%d", fn, n, h, w);
  if (n > 0 && (!src || !dst)) return set_error(FV_EINVAL, "%s: null pointer", fn);
  if (n > 65535) return set_error(FV_EINVAL, "%s: batch %d exceeds 65535", fn, n);
  return FV_OK;
}

}  // namespace fv

using namespace fv;

extern "C" {

int fv_gray_from_rgb_u8(const uint8_t* src, int64_t s_is, int64_t s_rp, uint8_t* dst, int64_t d_is,
                        int64_t d_rp, int32_t n, int32_t h, int32_t w, void* stream) {
  int rc = check_common(src, dst, n, h, w, "fv_gray_from_rgb_u8");
  if (rc || n == 0) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int gy = h < FV_GRAY_GY ? h : FV_GRAY_GY;
  if (al16(src) && al16(dst) && al16(s_is) && al16(s_rp) && al16(d_is) && al16(d_rp)) {
    const int groups = (w + 15) / 16;
    const int64_t total16 = (int64_t)n * h * groups;
    const int64_t total = (int64_t)n * h * ((w + FV_GRAY_PX - 1) / FV_GRAY_PX);
    if (total16 <= (int64_t)FV_GRAY_FLAT_MAX) {  // small batches: one flat wave of large CTAs
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)((total + kFlatThreads - 1) / kFlatThreads));
      cfg.blockDim = dim3(kFlatThreads);
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, gray_u8_flat_kernel<FV_GRAY_PX>, src, s_is, s_rp, dst, d_is, d_rp, (int)h, (int)w, total);
    } else {
      dim3 grid((groups + 127) / 128, gy, n);
      gray_u8_vec_kernel<<<grid, 128, 0, st>>>(src, s_is, s_rp, dst, d_is, d_rp, h, w);
    }
  } else {
    dim3 grid((w + 127) / 128, gy, n);
    gray_u8_px_kernel<<<grid, 128, 0, st>>>(src, s_is, s_rp, dst, d_is, d_rp, h, w);
  }
  return check_launch("fv_gray_from_rgb_u8");
}

int fv_gray_from_rgb_f32(const float* src, int64_t s_is, int64_t s_rp, float* dst, int64_t d_is, int64_t d_rp,
                         int32_t n, int32_t h, int32_t w, void* stream) {
  int rc = check_common(src, dst, n, h, w, "fv_gray_from_rgb_f32");
  if (rc || n == 0) return rc;
  if ((s_is | s_rp | d_is | d_rp) & 3) return set_error(FV_EINVAL, "fv_gray_from_rgb_f32: strides not f32-aligned");
  const int gy = h < 65535 ? h : 65535;
  dim3 grid((w + 127) / 128, gy, n);
  gray_f32_kernel<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(src, s_is, s_rp, dst, d_is, d_rp, h, w);
  return check_launch("fv_gray_from_rgb_f32");
}

int fv_to_float_scaled(const uint8_t* src, int64_t s_is, int64_t s_rp, float* dst, int64_t d_is, int64_t d_rp,
                       int32_t n, int32_t h, int32_t w, int32_t c, void* stream) {
  int rc = check_common(src, dst, n, h, w, "fv_to_float_scaled");
  if (rc || n == 0) return rc;
  if (c < 1) return set_error(FV_EINVAL, "fv_to_float_scaled: channels %d", c);
  if ((d_is | d_rp) & 3) return set_error(FV_EINVAL, "fv_to_float_scaled: dst strides not f32-aligned");
  const int row_elems = w * c;
  const bool vec = al16(src) && al16(dst) && al16(s_is) && al16(s_rp) && al16(d_is) && al16(d_rp);
  const int gy = h < 65535 ? h : 65535;
  const int groups = (row_elems + 15) / 16;
  dim3 grid((groups + 127) / 128, gy, n);
  to_float_scaled_kernel<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(src, s_is, s_rp, dst, d_is, d_rp,
                                                                              h, row_elems, vec);
  return check_launch("fv_to_float_scaled");
}

}  // extern "C"
