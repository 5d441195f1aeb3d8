// fv_warp.cuh -- shared pieces of the warp kernels (fv_warp.cu, fv_persp.cu):
// kernel arguments, the per-image inverse matrices and the exact f64
// per-pixel map of the builder contract.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

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
  f2_t one2;          // runtime {1.0f, 1.0f} (f32x2 contraction guard)
  int zero_border;    // border is +0: fully-outside pixels are exactly 0
};

struct WarpMats {
  double m[MAXW][9];
};

// Inverse map of destination pixel (x, y) and its bilinear taps.
struct WarpTap {
  int x0, y0;
  float wx0, wx1, wy0, wy1;
  bool finite;
};

template <bool PERSP>
__device__ __forceinline__ WarpTap warp_tap(const double (&m)[9], double rx, double ry, double rw, int x, int sw,
                                            int sh) {
  WarpTap t;
  const double xd = (double)x;
  double sx = __dadd_rn(__dmul_rn(m[0], xd), rx);
  double sy = __dadd_rn(__dmul_rn(m[3], xd), ry);
  t.finite = true;
  if (PERSP) {
    const double w = __dadd_rn(__dmul_rn(m[6], xd), rw);
    if (w == 0.0) {
      t.finite = false;
    } else {
      const double r = __drcp_rn(w);
      sx = __dmul_rn(sx, r);
      sy = __dmul_rn(sy, r);
    }
  }
  t.finite = t.finite && isfinite(sx) && isfinite(sy);
  if (!t.finite) {
    sx = 0.0;
    sy = 0.0;
  }
  const double fx = floor(sx), fy = floor(sy);
  t.wx1 = __double2float_rn(__dadd_rn(sx, -fx));
  t.wy1 = __double2float_rn(__dadd_rn(sy, -fy));
  t.wx0 = __fsub_rn(1.0f, t.wx1);
  t.wy0 = __fsub_rn(1.0f, t.wy1);
  // cvt.rmi saturates out-of-range values; clamping keeps every out-of-range
  // tap out of range (the oracle clips the float the same way)
  t.x0 = min(max(__double2int_rd(sx), -2), sw + 1);
  t.y0 = min(max(__double2int_rd(sy), -2), sh + 1);
  return t;
}

// fv_persp.cu: the tile-classified u8 perspective kernel (<= 1 LSB); 0 =
// launched, 1 = not applicable (channel count / grid), else an error code
int launch_persp_tile(const WarpArgs& a, const WarpMats& mats, int nb, cudaStream_t st);

// fv_affine.cu: the source-tiled affine kernel (+ its outside-pixel pass) for
// 16-byte aligned rows, C in {1, 3, 4}, es = element size (1 or 4); 0 =
// launched, 1 = not applicable, else an error code
int launch_affine_src(const WarpArgs& a, const WarpMats& mats, int nb, int es, cudaStream_t st);

// cuTensorMapEncodeTiled through the runtime's driver entry point (fv_warp.cu)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

}  // namespace fv
