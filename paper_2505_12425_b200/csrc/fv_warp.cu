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
#include "fv_common.cuh"

namespace fv {

constexpr int MAXW = 256;  // images per launch (matrices live in the param block)

struct WarpArgs {
  const void* src;
  int64_t s_is, s_rp;
  int sh, sw;
  void* dst;
  int64_t d_is, d_rp;
  int dh, dw;
  int c;
  float border_f;     // border as a blend operand (u8: RN(b/255))
  float border_raw;   // border as stored for non-finite coordinates
};

struct WarpMats {
  double m[MAXW][9];
};

template <typename T>
__device__ __forceinline__ void store_out(T* p, float v);
template <>
__device__ __forceinline__ void store_out<float>(float* p, float v) {
  *p = v;
}
template <>
__device__ __forceinline__ void store_out<uint8_t>(uint8_t* p, float v) {
  *p = (uint8_t)unit_to_u8(v);
}

template <typename InT, bool PERSP>
__global__ void __launch_bounds__(128) warp_kernel(const __grid_constant__ WarpArgs a,
                                                   const __grid_constant__ WarpMats mats) {
  const int n = blockIdx.z;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= a.dw) return;
  const double* m = mats.m[n];
  const double xd = (double)x;
  for (int y = blockIdx.y; y < a.dh; y += gridDim.y) {
    const double yd = (double)y;
    double sx = __dadd_rn(__dmul_rn(m[0], xd), __dadd_rn(__dmul_rn(m[1], yd), m[2]));
    double sy = __dadd_rn(__dmul_rn(m[3], xd), __dadd_rn(__dmul_rn(m[4], yd), m[5]));
    bool finite = true;
    if (PERSP) {
      const double w = __dadd_rn(__dmul_rn(m[6], xd), __dadd_rn(__dmul_rn(m[7], yd), m[8]));
      if (w == 0.0) {
        finite = false;
      } else {
        const double r = __drcp_rn(w);
        sx = __dmul_rn(sx, r);
        sy = __dmul_rn(sy, r);
      }
    }
    finite = finite && isfinite(sx) && isfinite(sy);
    InT* d = row_ptr_mut<InT>(a.dst, a.d_is, a.d_rp, n, y) + x * a.c;
    if (!finite) {
      for (int ch = 0; ch < a.c; ++ch) d[ch] = (InT)a.border_raw;
      continue;
    }
    const double x0f = floor(sx), y0f = floor(sy);
    const float wx1 = __double2float_rn(__dadd_rn(sx, -x0f));
    const float wy1 = __double2float_rn(__dadd_rn(sy, -y0f));
    const float wx0 = __fsub_rn(1.0f, wx1), wy0 = __fsub_rn(1.0f, wy1);
    const int x0 = (int)fmin(fmax(x0f, -2.0), (double)a.sw + 1.0);
    const int y0 = (int)fmin(fmax(y0f, -2.0), (double)a.sh + 1.0);
    const bool ix0 = x0 >= 0 && x0 < a.sw, ix1 = x0 + 1 >= 0 && x0 + 1 < a.sw;
    const bool iy0 = y0 >= 0 && y0 < a.sh, iy1 = y0 + 1 >= 0 && y0 + 1 < a.sh;
    const InT* r0 = iy0 ? row_ptr<InT>(a.src, a.s_is, a.s_rp, n, y0) : nullptr;
    const InT* r1 = iy1 ? row_ptr<InT>(a.src, a.s_is, a.s_rp, n, y0 + 1) : nullptr;
    for (int ch = 0; ch < a.c; ++ch) {
      const float t00 = (iy0 && ix0) ? tap_value(__ldg(r0 + x0 * a.c + ch)) : a.border_f;
      const float t01 = (iy0 && ix1) ? tap_value(__ldg(r0 + (x0 + 1) * a.c + ch)) : a.border_f;
      const float t10 = (iy1 && ix0) ? tap_value(__ldg(r1 + x0 * a.c + ch)) : a.border_f;
      const float t11 = (iy1 && ix1) ? tap_value(__ldg(r1 + (x0 + 1) * a.c + ch)) : a.border_f;
      const float top = lerp_ref(t00, t01, wx0, wx1);
      const float bot = lerp_ref(t10, t11, wx0, wx1);
      store_out<InT>(d + ch, lerp_ref(top, bot, wy0, wy1));
    }
  }
}

template <typename InT, bool PERSP>
static int launch_warp(const InT* src, int64_t s_is, int64_t s_rp, int sh, int sw, InT* dst, int64_t d_is,
                       int64_t d_rp, int dh, int dw, int c, int n, const double* mats_host, int mat_len,
                       float border_f, float border_raw, cudaStream_t st, const char* fn) {
  if (n < 0 || sh < 1 || sw < 1 || dh < 1 || dw < 1 || c < 1)
    return set_error(FV_EINVAL, "%s: bad shape n=%d src=%dx%d dst=%dx%d c=%d", fn, n, sh, sw, dh, dw, c);
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
  WarpMats mats;
  for (int b = 0; b < n; b += MAXW) {
    const int nb = (n - b) < MAXW ? (n - b) : MAXW;
    for (int i = 0; i < nb; ++i)
      for (int j = 0; j < 9; ++j) mats.m[i][j] = j < mat_len ? mats_host[(int64_t)(b + i) * mat_len + j] : 0.0;
    a.src = reinterpret_cast<const char*>(src) + (int64_t)b * s_is;
    a.dst = reinterpret_cast<char*>(dst) + (int64_t)b * d_is;
    const int gy = dh < 65535 ? dh : 65535;
    dim3 grid((dw + 127) / 128, gy, nb);
    warp_kernel<InT, PERSP><<<grid, 128, 0, st>>>(a, mats);
    int rc = check_launch(fn);
    if (rc) return rc;
  }
  return FV_OK;
}

}  // namespace fv

using namespace fv;

extern "C" {

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

int fv_warp_perspective_f32(const float* src, int64_t s_is, int64_t s_rp, int32_t sh, int32_t sw, float* dst,
                            int64_t d_is, int64_t d_rp, int32_t dh, int32_t dw, int32_t c, int32_t n,
                            const double* hinv_host, float border, void* stream) {
  return launch_warp<float, true>(src, s_is, s_rp, sh, sw, dst, d_is, d_rp, dh, dw, c, n, hinv_host, 9, border,
                                  border, static_cast<cudaStream_t>(stream), "fv_warp_perspective_f32");
}

}  // extern "C"
