// fv_geom.cu -- SURVEY §8(f) rank 1 and 3: the rest of the reference's
// imgproc kernels on the same boundary.
//   imgproc.flip_horizontal  (imgproc.py:67-73)   any dtype, pure indexing
//   imgproc.resize_nearest   (imgproc.py:81-97)   any dtype, pure indexing
//   imgproc.sobel            (imgproc.py:126-155) f32, 3x3, replicate border
// Indexing work is bit-exact by construction; sobel reproduces the NumPy op
// order (each f32 op separately rounded, correctly rounded sqrt).
#include "fv_common.cuh"

namespace fv {

// _nearest_indices (imgproc.py:81-86): z = (i + 0.5) * (src_n / dst_n) in f64,
// idx = clip(ceil(z) - 1, 0, src_n - 1)  (round-half-down of the centre)
__device__ __forceinline__ int nearest_index(int i, double scale, int src_n) {
  const double z = __dmul_rn(__dadd_rn((double)i, 0.5), scale);
  const int idx = (int)ceil(z) - 1;
  return min(max(idx, 0), src_n - 1);
}

template <typename T>
__device__ __forceinline__ void copy_px(T* d, const T* s, int c) {
  for (int k = 0; k < c; ++k) d[k] = s[k];
}

// one destination pixel per thread; T is the element type (1/2/4/8 bytes)
template <typename T>
__global__ void nearest_kernel(const char* __restrict__ src, int64_t s_is, int64_t s_rp, int sh, int sw,
                               char* __restrict__ dst, int64_t d_is, int64_t d_rp, int dh, int dw, int c,
                               double scale_x, double scale_y) {
  const int n = blockIdx.z;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= dw) return;
  const int sx = nearest_index(x, scale_x, sw);
  for (int y = blockIdx.y; y < dh; y += gridDim.y) {
    const int sy = nearest_index(y, scale_y, sh);
    const T* s = reinterpret_cast<const T*>(src + n * s_is + (int64_t)sy * s_rp) + (int64_t)sx * c;
    T* d = reinterpret_cast<T*>(dst + n * d_is + (int64_t)y * d_rp) + (int64_t)x * c;
    copy_px(d, s, c);
  }
}

template <typename T>
__global__ void flip_kernel(const char* __restrict__ src, int64_t s_is, int64_t s_rp, char* __restrict__ dst,
                            int64_t d_is, int64_t d_rp, int h, int w, int c) {
  const int n = blockIdx.z;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= w) return;
  for (int y = blockIdx.y; y < h; y += gridDim.y) {
    const T* s = reinterpret_cast<const T*>(src + n * s_is + (int64_t)y * s_rp) + (int64_t)(w - 1 - x) * c;
    T* d = reinterpret_cast<T*>(dst + n * d_is + (int64_t)y * d_rp) + (int64_t)x * c;
    copy_px(d, s, c);
  }
}

// ---------------------------------------------------------------------------
// vectorised paths: a thread owns 16 destination pixels of S bytes (16*S bytes,
// S 16-byte stores) and walks a band of rows with its column indices fixed.
// ---------------------------------------------------------------------------
template <int S>
struct Px16 {
  uint32_t w[4 * S];  // 16 pixels x S bytes
};

// byte i of the 16-pixel block, compile-time i after unrolling
template <int S>
__device__ __forceinline__ uint32_t blk_byte(const Px16<S>& b, int i) {
  return (b.w[i >> 2] >> ((i & 3) * 8)) & 0xFFu;
}

// flip: destination block g of a row is the reverse of source block
// (w/16 - 1 - g); pixel order reversed in registers (w % 16 == 0, aligned rows)
template <int S>
__global__ void __launch_bounds__(128) flip16_kernel(const char* __restrict__ src, int64_t s_is, int64_t s_rp,
                                                     char* __restrict__ dst, int64_t d_is, int64_t d_rp, int h,
                                                     int w) {
  const int n = blockIdx.z;
  const int groups = w / 16;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  for (int y = blockIdx.y; y < h; y += gridDim.y) {
    const uint4* s4 = reinterpret_cast<const uint4*>(src + n * s_is + (int64_t)y * s_rp + (int64_t)(groups - 1 - g) * 16 * S);
    uint4* d4 = reinterpret_cast<uint4*>(dst + n * d_is + (int64_t)y * d_rp + (int64_t)g * 16 * S);
    Px16<S> in;
#pragma unroll
    for (int i = 0; i < S; ++i) {
      const uint4 v = __ldg(s4 + i);
      in.w[4 * i] = v.x, in.w[4 * i + 1] = v.y, in.w[4 * i + 2] = v.z, in.w[4 * i + 3] = v.w;
    }
    uint32_t out[4 * S];
#pragma unroll
    for (int q = 0; q < 4 * S; ++q) {
      uint32_t b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int o = 4 * q + j, p = o / S, k = o % S;
        b[j] = blk_byte(in, (15 - p) * S + k);
      }
      out[q] = b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24);
    }
#pragma unroll
    for (int i = 0; i < S; ++i) __stcs(d4 + i, make_uint4(out[4 * i], out[4 * i + 1], out[4 * i + 2], out[4 * i + 3]));
  }
}

// pixel of S bytes at byte offset `off` of a row (S = 3: three byte loads)
template <int S>
__device__ __forceinline__ void load_px(const char* p, uint8_t (&v)[S]) {
#pragma unroll
  for (int k = 0; k < S; ++k) v[k] = __ldg(reinterpret_cast<const uint8_t*>(p) + k);
}

// nearest: the thread's 16 source column indices are computed once (f64,
// imgproc.py:81-86); each row gathers 16 pixels through L1 and writes S
// 16-byte vectors (dw % 16 == 0, aligned destination rows)
template <int S>
__global__ void __launch_bounds__(128) nearest16_kernel(const char* __restrict__ src, int64_t s_is, int64_t s_rp,
                                                        int sh, int sw, char* __restrict__ dst, int64_t d_is,
                                                        int64_t d_rp, int dh, int dw, double scale_x,
                                                        double scale_y, int rows_per_cta) {
  const int n = blockIdx.z;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= dw / 16) return;
  int sx[16];
#pragma unroll
  for (int p = 0; p < 16; ++p) sx[p] = nearest_index(g * 16 + p, scale_x, sw) * S;
  const int y0 = blockIdx.y * rows_per_cta, y1 = min(y0 + rows_per_cta, dh);
  for (int y = y0; y < y1; ++y) {
    const char* srow = src + n * s_is + (int64_t)nearest_index(y, scale_y, sh) * s_rp;
    uint8_t px[16][S];
#pragma unroll
    for (int p = 0; p < 16; ++p) load_px<S>(srow + sx[p], px[p]);
    uint32_t out[4 * S];
#pragma unroll
    for (int q = 0; q < 4 * S; ++q) {
      uint32_t b[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int o = 4 * q + j;
        b[j] = px[o / S][o % S];
      }
      out[q] = b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24);
    }
    uint4* d4 = reinterpret_cast<uint4*>(dst + n * d_is + (int64_t)y * d_rp + (int64_t)g * 16 * S);
#pragma unroll
    for (int i = 0; i < S; ++i) __stcs(d4 + i, make_uint4(out[4 * i], out[4 * i + 1], out[4 * i + 2], out[4 * i + 3]));
  }
}

static inline bool al16v(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// imgproc.py:139-155. p = edge-padded source; for each pixel and channel
//   gx = ((ur - ul) + 2*(right - left)) + (dr - dl)
//   gy = ((dl - ul) + 2*(down - up)) + (dr - ur)
//   out = sqrt(RN(gx*gx) + RN(gy*gy))          (f32, each op rounded)
__global__ void sobel_kernel(const char* __restrict__ src, int64_t s_is, int64_t s_rp, char* __restrict__ dst,
                             int64_t d_is, int64_t d_rp, int h, int w, int c) {
  const int n = blockIdx.z;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= w) return;
  const int xl = max(x - 1, 0), xr = min(x + 1, w - 1);
  for (int y = blockIdx.y; y < h; y += gridDim.y) {
    const int yu = max(y - 1, 0), yd = min(y + 1, h - 1);
    const float* ru = reinterpret_cast<const float*>(src + n * s_is + (int64_t)yu * s_rp);
    const float* rm = reinterpret_cast<const float*>(src + n * s_is + (int64_t)y * s_rp);
    const float* rd = reinterpret_cast<const float*>(src + n * s_is + (int64_t)yd * s_rp);
    float* d = reinterpret_cast<float*>(dst + n * d_is + (int64_t)y * d_rp) + (int64_t)x * c;
    for (int k = 0; k < c; ++k) {
      const float ul = __ldg(ru + xl * c + k), up = __ldg(ru + x * c + k), ur = __ldg(ru + xr * c + k);
      const float left = __ldg(rm + xl * c + k), right = __ldg(rm + xr * c + k);
      const float dl = __ldg(rd + xl * c + k), down = __ldg(rd + x * c + k), dr = __ldg(rd + xr * c + k);
      const float gx = __fadd_rn(__fadd_rn(__fsub_rn(ur, ul), __fmul_rn(2.0f, __fsub_rn(right, left))), __fsub_rn(dr, dl));
      const float gy = __fadd_rn(__fadd_rn(__fsub_rn(dl, ul), __fmul_rn(2.0f, __fsub_rn(down, up))), __fsub_rn(dr, ur));
      d[k] = __fsqrt_rn(__fadd_rn(__fmul_rn(gx, gx), __fmul_rn(gy, gy)));
    }
  }
}

static int check_geom(const void* src, const void* dst, int n, int sh, int sw, int dh, int dw, int c, int es,
                      const char* fn) {
  if (n < 0 || sh < 1 || sw < 1 || dh < 1 || dw < 1 || c < 1)
    return set_error(FV_EINVAL, "%s: bad shape n=%d src=%dx%d dst=%dx%d c=%d", fn, n, sh, sw, dh, dw, c);
  if (es != 1 && es != 2 && es != 4 && es != 8) return set_error(FV_EINVAL, "%s: element size %d", fn, es);
  if (n > 65535) return set_error(FV_EINVAL, "%s: batch %d exceeds 65535", fn, n);
  if (n > 0 && (!src || !dst)) return set_error(FV_EINVAL, "%s: null pointer", fn);
  return FV_OK;
}

}  // namespace fv

using namespace fv;

extern "C" {

int fv_resize_nearest(const void* src, int64_t s_is, int64_t s_rp, int32_t sh, int32_t sw, void* dst, int64_t d_is,
                      int64_t d_rp, int32_t dh, int32_t dw, int32_t c, int32_t elem_size, int32_t n, void* stream) {
  int rc = check_geom(src, dst, n, sh, sw, dh, dw, c, elem_size, "fv_resize_nearest");
  if (rc || n == 0) return rc;
  const double sx = (double)sw / (double)dw, sy = (double)sh / (double)dh;  // imgproc.py:83
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  const int S = c * elem_size;
  if ((S == 3 || S == 4) && dw % 16 == 0 && al16v(dst) && ((d_is | d_rp) & 15) == 0) {
    const int rows = 16;
    dim3 g16((dw / 16 + 127) / 128, (dh + rows - 1) / rows, n);
    if (S == 3)
      nearest16_kernel<3><<<g16, 128, 0, st>>>(s, s_is, s_rp, sh, sw, d, d_is, d_rp, dh, dw, sx, sy, rows);
    else
      nearest16_kernel<4><<<g16, 128, 0, st>>>(s, s_is, s_rp, sh, sw, d, d_is, d_rp, dh, dw, sx, sy, rows);
    return check_launch("fv_resize_nearest");
  }
  dim3 grid((dw + 127) / 128, dh < 65535 ? dh : 65535, n);
  switch (elem_size) {
    case 1: nearest_kernel<uint8_t><<<grid, 128, 0, st>>>(s, s_is, s_rp, sh, sw, d, d_is, d_rp, dh, dw, c, sx, sy); break;
    case 2: nearest_kernel<uint16_t><<<grid, 128, 0, st>>>(s, s_is, s_rp, sh, sw, d, d_is, d_rp, dh, dw, c, sx, sy); break;
    case 4: nearest_kernel<uint32_t><<<grid, 128, 0, st>>>(s, s_is, s_rp, sh, sw, d, d_is, d_rp, dh, dw, c, sx, sy); break;
    default: nearest_kernel<uint64_t><<<grid, 128, 0, st>>>(s, s_is, s_rp, sh, sw, d, d_is, d_rp, dh, dw, c, sx, sy); break;
  }
  return check_launch("fv_resize_nearest");
}

int fv_flip_horizontal(const void* src, int64_t s_is, int64_t s_rp, void* dst, int64_t d_is, int64_t d_rp,
                       int32_t h, int32_t w, int32_t c, int32_t elem_size, int32_t n, void* stream) {
  int rc = check_geom(src, dst, n, h, w, h, w, c, elem_size, "fv_flip_horizontal");
  if (rc || n == 0) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  const int S = c * elem_size;
  if ((S == 1 || S == 3 || S == 4 || S == 12) && w % 16 == 0 && al16v(src) && al16v(dst) &&
      ((s_is | s_rp | d_is | d_rp) & 15) == 0) {
    dim3 g16((w / 16 + 127) / 128, h < 65535 ? h : 65535, n);
    switch (S) {
      case 1: flip16_kernel<1><<<g16, 128, 0, st>>>(s, s_is, s_rp, d, d_is, d_rp, h, w); break;
      case 3: flip16_kernel<3><<<g16, 128, 0, st>>>(s, s_is, s_rp, d, d_is, d_rp, h, w); break;
      case 4: flip16_kernel<4><<<g16, 128, 0, st>>>(s, s_is, s_rp, d, d_is, d_rp, h, w); break;
      default: flip16_kernel<12><<<g16, 128, 0, st>>>(s, s_is, s_rp, d, d_is, d_rp, h, w); break;
    }
    return check_launch("fv_flip_horizontal");
  }
  dim3 grid((w + 127) / 128, h < 65535 ? h : 65535, n);
  switch (elem_size) {
    case 1: flip_kernel<uint8_t><<<grid, 128, 0, st>>>(s, s_is, s_rp, d, d_is, d_rp, h, w, c); break;
    case 2: flip_kernel<uint16_t><<<grid, 128, 0, st>>>(s, s_is, s_rp, d, d_is, d_rp, h, w, c); break;
    case 4: flip_kernel<uint32_t><<<grid, 128, 0, st>>>(s, s_is, s_rp, d, d_is, d_rp, h, w, c); break;
    default: flip_kernel<uint64_t><<<grid, 128, 0, st>>>(s, s_is, s_rp, d, d_is, d_rp, h, w, c); break;
  }
  return check_launch("fv_flip_horizontal");
}

int fv_sobel_f32(const float* src, int64_t s_is, int64_t s_rp, float* dst, int64_t d_is, int64_t d_rp, int32_t h,
                 int32_t w, int32_t c, int32_t n, void* stream) {
  int rc = check_geom(src, dst, n, h, w, h, w, c, 4, "fv_sobel_f32");
  if (rc || n == 0) return rc;
  if ((s_is | s_rp | d_is | d_rp) & 3) return set_error(FV_EINVAL, "fv_sobel_f32: strides not f32-aligned");
  dim3 grid((w + 127) / 128, h < 65535 ? h : 65535, n);
  sobel_kernel<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(reinterpret_cast<const char*>(src), s_is, s_rp,
                                                                    reinterpret_cast<char*>(dst), d_is, d_rp, h, w, c);
  return check_launch("fv_sobel_f32");
}

}  // extern "C"
