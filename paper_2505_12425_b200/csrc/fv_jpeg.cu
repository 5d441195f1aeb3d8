// fv_jpeg.cu -- decode -> preprocess: the reference's
// baseline JPEG decoder (io/jpeg.py:605-806), bit-identical.
//
// Host (C++, fv_jpeg_host.cuh): marker walk, table parsing and the scan
// split with the reference's checks and error classes, and the host
// canonical-Huffman entropy decoder (natural-order coefficients) used by the
// single-image path, the host batch path and the GPU path's fallback. The
// GPU entropy decoder is fv_jpeg_gpu.cu.
// Device (sm_100a): dequantisation + the 13-bit fixed-point "islow" IDCT
// with the reference's NumPy int64 integers (int32 where no intermediate can
// overflow, decided per warp), so any stream -- including adversarial
// coefficient magnitudes -- gives the same samples; then one kernel that
// upsamples the chroma planes with the reference's integer triangle filters
// and converts YCbCr -> RGB (16-bit fixed point), writing the HWC u8 image.
// The batch kernels (one launch each for a whole batch) serve the GPU path
// and every dense int16 input; the per-image kernels below serve int32/int64
// and the host batch runtime's sparse stream.
#include <atomic>
#include <thread>

#include "fv_jpeg_host.cuh"

namespace fv {
namespace jpg {

// ---------------------------------------------------------------------------
// device
// ---------------------------------------------------------------------------

struct IdctArgs {
  const void* coeffs;
  uint8_t* planes;
  int ncomp;                // distinct components
  int64_t first_block[4];   // prefix sums of block counts
  int64_t coef_offset[3];
  int64_t plane_offset[3];
  int bw[3];
  alignas(16) uint16_t qt[3][64];  // rows are read as 16-byte vectors by the batch kernel
};

// One 8-point pass of the islow IDCT (jpeg.py:163-191), outputs before
// descaling in index order. The reference computes in int64 (NumPy); T =
// int32 gives the same integers whenever nothing overflows: every
// intermediate is a signed sum of input multiples with total gain <= 178219
// (triangle bound over the butterfly's terms; the outputs' exact L1 gain is
// 61214), so |inputs| <= kIdct32Max keeps all of them below 2^31 - 2^17.
constexpr int64_t kIdct32Max = 12000;

template <typename T>
__device__ __forceinline__ void idct8(const T (&s)[8], T (&o)[8]) {
  const T z1 = (s[2] + s[6]) * 4433;
  const T e2 = z1 - s[6] * 15137, e3 = z1 + s[2] * 6270;
  const T e0 = (s[0] + s[4]) * 8192, e1 = (s[0] - s[4]) * 8192;
  const T a10 = e0 + e3, a13 = e0 - e3, a11 = e1 + e2, a12 = e1 - e2;
  const T z5 = (s[7] + s[3] + s[5] + s[1]) * 9633;
  const T q1 = (s[7] + s[1]) * -7373, q2 = (s[5] + s[3]) * -20995;
  const T q3 = (s[7] + s[3]) * -16069 + z5, q4 = (s[5] + s[1]) * -3196 + z5;
  const T o0 = s[7] * 2446 + q1 + q3, o1 = s[5] * 16819 + q2 + q4;
  const T o2 = s[3] * 25172 + q2 + q3, o3 = s[1] * 12299 + q1 + q4;
  o[0] = a10 + o3;
  o[1] = a11 + o2;
  o[2] = a12 + o1;
  o[3] = a13 + o0;
  o[4] = a13 - o0;
  o[5] = a12 - o1;
  o[6] = a11 - o2;
  o[7] = a10 - o3;
}

// the pass in int32 when this thread's inputs allow it, else in int64
__device__ __forceinline__ void idct8_exact(const int64_t (&s)[8], int64_t (&o)[8]) {
  bool small = true;
#pragma unroll
  for (int k = 0; k < 8; ++k) small = small && s[k] >= -kIdct32Max && s[k] <= kIdct32Max;
  if (small) {
    int32_t a[8], b[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = (int32_t)s[k];
    idct8<int32_t>(a, b);
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = b[k];
  } else {
    idct8<int64_t>(s, o);
  }
}

// Second half of a block's IDCT, shared by the dense and sparse kernels:
// s = the dequantised column j (vertical frequencies 0..7) of block g.
__device__ __forceinline__ void idct_rows_store(int64_t (&s)[8], int64_t (&ws)[16][8][9], int g, int j, uint32_t mask,
                                                uint8_t* dst) {
  int64_t o[8];
  idct8_exact(s, o);
#pragma unroll
  for (int k = 0; k < 8; ++k) ws[g][k][j] = (o[k] + (1 << 10)) >> 11;
  __syncwarp(mask);
#pragma unroll
  for (int k = 0; k < 8; ++k) s[k] = ws[g][j][k];
  idct8_exact(s, o);
  uint32_t w[2] = {0, 0};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int64_t v = ((o[k] + (1 << 17)) >> 18) + 128;
    v = v < 0 ? 0 : (v > 255 ? 255 : v);
    w[k >> 2] |= (uint32_t)v << (8 * (k & 3));
  }
  *reinterpret_cast<uint2*>(dst) = make_uint2(w[0], w[1]);
}

// 16 JPEG blocks per CTA, 8 threads per block: thread j runs the vertical
// pass on column j, then the horizontal pass on row j, and stores row j
// (8 samples, one 8-byte store) into the component plane.
template <typename T>
__global__ void __launch_bounds__(128) jpeg_idct_kernel(const __grid_constant__ IdctArgs a) {
  __shared__ int64_t ws[16][8][9];
  const int g = threadIdx.x >> 3, j = threadIdx.x & 7;
  const int64_t blk = (int64_t)blockIdx.x * 16 + g;
  if (blk >= a.first_block[a.ncomp]) return;  // whole 8-thread groups exit together
  int c = 0;
  while (c + 1 < a.ncomp && blk >= a.first_block[c + 1]) ++c;
  const int64_t lb = blk - a.first_block[c];
  const T* co = reinterpret_cast<const T*>(a.coeffs) + a.coef_offset[c] + 64 * lb;
  int64_t s[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) s[k] = (int64_t)co[8 * k + j] * (int64_t)a.qt[c][8 * k + j];
  const int64_t by = lb / a.bw[c], bx = lb - by * a.bw[c];
  uint8_t* dst = a.planes + a.plane_offset[c] + (by * 8 + j) * (int64_t)a.bw[c] * 8 + bx * 8;
  idct_rows_store(s, ws, g, j, 0xFFu << (threadIdx.x & 24), dst);
}

// Same, from the batch runtime's sparse stream: the block's 8 threads zero
// a SMEM block, scatter its stored coefficients, then run the IDCT.
__global__ void __launch_bounds__(128) jpeg_idct_sparse_kernel(const __grid_constant__ IdctArgs a, const uint32_t* words,
                                                               int64_t nblk) {
  __shared__ int64_t ws[16][8][9];
  __shared__ int32_t cb[16][64];
  const int g = threadIdx.x >> 3, j = threadIdx.x & 7;
  const uint32_t mask = 0xFFu << (threadIdx.x & 24);
  const int64_t blk = (int64_t)blockIdx.x * 16 + g;
  if (blk >= a.first_block[a.ncomp]) return;
  int c = 0;
  while (c + 1 < a.ncomp && blk >= a.first_block[c + 1]) ++c;
  const int64_t lb = blk - a.first_block[c];
  const uint32_t* ent = words + nblk + words[blk];
  const uint32_t n = ent[0];
#pragma unroll
  for (int z = j; z < 64; z += 8) cb[g][z] = 0;
  __syncwarp(mask);
  for (uint32_t i = j; i < n; i += 8) {
    const uint32_t w = ent[1 + i];
    cb[g][w & 63] = (int32_t)(int16_t)(w >> 16);
  }
  __syncwarp(mask);
  int64_t s[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) s[k] = (int64_t)cb[g][8 * k + j] * (int64_t)a.qt[c][8 * k + j];
  const int64_t by = lb / a.bw[c], bx = lb - by * a.bw[c];
  uint8_t* dst = a.planes + a.plane_offset[c] + (by * 8 + j) * (int64_t)a.bw[c] * 8 + bx * 8;
  idct_rows_store(s, ws, g, j, mask, dst);
}

struct ColorArgs {
  const uint8_t* plane[3];
  int64_t pitch[3];
  int cw[3], ch[3], fh[3], fv[3];
  int ncomp, width, height;
  uint8_t* dst;
  int64_t d_rp;
};


__device__ __forceinline__ uint8_t clamp255(int v) { return (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v)); }

// Four consecutive samples (output columns x0..x0+3, x0 % 4 == 0) of
// component e at output row y, upsampled as the reference does: the needed
// plane samples are loaded once (indices clamped: a clamped value is only
// ever used by the edge formulas, which do not read it), then each output
// column takes its own formula (jpeg.py:809-841).
__device__ __forceinline__ void samples4(const ColorArgs& a, int e, int x0, int y, int (&s)[4]) {
  const uint8_t* p = a.plane[e];
  const int64_t pt = a.pitch[e];
  const int fh = a.fh[e], fv = a.fv[e], mw = a.cw[e], mh = a.ch[e];
  auto at = [&](int r, int c) { return (int)p[(int64_t)r * pt + min(max(c, 0), mw - 1)]; };
  if (fh == 1 && fv == 1) {
    const uint8_t* q = p + (int64_t)y * pt + x0;
    if (x0 + 3 < mw) {  // plane rows are 8-byte aligned, x0 % 4 == 0
      const uint32_t w = *reinterpret_cast<const uint32_t*>(q);
#pragma unroll
      for (int k = 0; k < 4; ++k) s[k] = (w >> (8 * k)) & 0xFF;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) s[k] = at(y, x0 + k);
    }
    return;
  }
  if (fh == 1) {  // vertical x2 only (4:4:0): the h2 filter along the columns
    const int m = mh, jj = y >> 1;
    if (m <= 2) {
#pragma unroll
      for (int k = 0; k < 4; ++k) s[k] = at(jj, x0 + k);
      return;
    }
    const int rn = (y == 0 || y == 2 * m - 1) ? jj : ((y & 1) ? jj + 1 : jj - 1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = at(jj, x0 + k), o = at(rn, x0 + k);
      s[k] = (y == 0 || y == 2 * m - 1) ? c : (y & 1) ? (3 * c + o + 2) >> 2 : (3 * c + o + 1) >> 2;
    }
    return;
  }
  // horizontal x2 (4:2:2) or 2x2 (4:2:0): columns j0-1 .. j0+2, j0 = x0 / 2
  const int j0 = x0 >> 1;
  int v[4];
  if (fv == 2) {
    const int r = y >> 1;
    if (mw <= 2) {  // replicate (the width decides, jpeg.py:831-832)
#pragma unroll
      for (int k = 0; k < 4; ++k) s[k] = at(r, (x0 + k) >> 1);
      return;
    }
    const int r2 = (y & 1) ? min(r + 1, mh - 1) : max(r - 1, 0);
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = 3 * at(r, j0 - 1 + k) + at(r2, j0 - 1 + k);  // column sums
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int X = x0 + k, jk = X >> 1, c = jk - j0 + 1;  // v[c] = colsum(jk)
      if (X == 0) s[k] = (v[c] * 4 + 8) >> 4;
      else if (X == 2 * mw - 1) s[k] = (v[c] * 4 + 7) >> 4;
      else if ((X & 1) == 0) s[k] = (3 * v[c] + v[c - 1] + 8) >> 4;
      else s[k] = (3 * v[c] + v[c + 1] + 7) >> 4;
    }
    return;
  }
  if (mw <= 2) {
#pragma unroll
    for (int k = 0; k < 4; ++k) s[k] = at(y, (x0 + k) >> 1);
    return;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = at(y, j0 - 1 + k);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int X = x0 + k, jk = X >> 1, c = jk - j0 + 1;
    if (X == 0) s[k] = v[c];
    else if (X == 2 * mw - 1) s[k] = v[c];
    else if ((X & 1) == 0) s[k] = (3 * v[c] + v[c - 1] + 1) >> 2;
    else s[k] = (3 * v[c] + v[c + 1] + 2) >> 2;
  }
}

// 4:2:0 chroma away from every edge: output columns x0..x0+3 need the
// column sums of chroma columns j0-1 .. j0+2 (j0 = x0/2), read from each of
// the two rows as one unaligned 4-byte window (two aligned words + a funnel
// shift); no clamping, no edge formulas. Returns false when not interior.
__device__ __forceinline__ bool chroma420_fast(const ColorArgs& a, int e, int x0, int y, int (&s)[4]) {
  const int mw = a.cw[e], mh = a.ch[e];
  const int j0 = x0 >> 1;
  const int64_t pt = a.pitch[e];
  if (mw <= 2 || x0 < 2 || j0 + 2 > mw - 1 || ((j0 - 1) & ~3) + 8 > pt) return false;
  const int r = y >> 1, r2 = (y & 1) ? min(r + 1, mh - 1) : max(r - 1, 0);
  const int base = (j0 - 1) & ~3, sh = 8 * ((j0 - 1) & 3);
  const uint32_t* p0 = reinterpret_cast<const uint32_t*>(a.plane[e] + (int64_t)r * pt + base);
  const uint32_t* p1 = reinterpret_cast<const uint32_t*>(a.plane[e] + (int64_t)r2 * pt + base);
  const uint32_t w0 = __funnelshift_r(__ldg(p0), __ldg(p0 + 1), sh);
  const uint32_t w1 = __funnelshift_r(__ldg(p1), __ldg(p1 + 1), sh);
  int v[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = 3 * (int)((w0 >> (8 * k)) & 0xFF) + (int)((w1 >> (8 * k)) & 0xFF);
  s[0] = (3 * v[1] + v[0] + 8) >> 4;  // X = x0     (even, column j0)
  s[1] = (3 * v[1] + v[2] + 7) >> 4;  // X = x0 + 1 (odd,  column j0)
  s[2] = (3 * v[2] + v[1] + 8) >> 4;  // X = x0 + 2 (even, column j0 + 1)
  s[3] = (3 * v[2] + v[3] + 7) >> 4;  // X = x0 + 3 (odd,  column j0 + 1)
  return true;
}

// Upsample + YCbCr -> RGB (jpeg.py:226-235, 783-806) of output pixels
// x0..x0+3 of row y; 12-byte groups stored as words when the row allows it.
__device__ __forceinline__ void color4(const ColorArgs& a, int x0, int y) {
  const int nk = min(4, a.width - x0);
  uint8_t* d = a.dst + (int64_t)y * a.d_rp;
  int Y[4];
  samples4(a, 0, x0, y, Y);
  if (a.ncomp == 1) {
    if (nk == 4 && ((reinterpret_cast<uintptr_t>(d + x0) & 3) == 0)) {
      *reinterpret_cast<uint32_t*>(d + x0) = (uint32_t)Y[0] | (Y[1] << 8) | (Y[2] << 16) | ((uint32_t)Y[3] << 24);
    } else {
      for (int k = 0; k < nk; ++k) d[x0 + k] = (uint8_t)Y[k];
    }
    return;
  }
  int B[4], R[4];
  const bool h2v2 = a.fh[1] == 2 && a.fv[1] == 2 && a.fh[2] == 2 && a.fv[2] == 2;
  if (!(h2v2 && nk == 4 && chroma420_fast(a, 1, x0, y, B) && chroma420_fast(a, 2, x0, y, R))) {
    samples4(a, 1, x0, y, B);
    samples4(a, 2, x0, y, R);
  }
  uint8_t o[12];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int xb = B[k] - 128, xr = R[k] - 128;
    o[3 * k] = clamp255(Y[k] + ((91881 * xr + 32768) >> 16));
    o[3 * k + 1] = clamp255(Y[k] + ((-22554 * xb + 32768 - 46802 * xr) >> 16));
    o[3 * k + 2] = clamp255(Y[k] + ((116130 * xb + 32768) >> 16));
  }
  uint8_t* q = d + 3 * x0;
  if (nk == 4 && (reinterpret_cast<uintptr_t>(q) & 3) == 0) {
    uint32_t* w = reinterpret_cast<uint32_t*>(q);
#pragma unroll
    for (int k = 0; k < 3; ++k)
      w[k] = (uint32_t)o[4 * k] | (o[4 * k + 1] << 8) | (o[4 * k + 2] << 16) | ((uint32_t)o[4 * k + 3] << 24);
  } else {
    for (int k = 0; k < 3 * nk; ++k) q[k] = o[k];
  }
}

__global__ void __launch_bounds__(256) jpeg_color_kernel(const __grid_constant__ ColorArgs a) {
  const int x0 = (blockIdx.x * 256 + threadIdx.x) * 4;
  if (x0 < a.width) color4(a, x0, blockIdx.y);
}

// Batched reconstruction (the GPU entropy path): one launch of each kernel
// for a whole batch; a group / CTA finds its image by binary search over the
// images' first block / row.
struct IdctImg {
  IdctArgs a;
  int64_t base;  // first block of the image in the batch
};
static_assert(alignof(IdctArgs) >= 16 && sizeof(IdctImg) % 16 == 0, "16-byte quant rows");
struct ColorImg {
  ColorArgs a;
  int64_t base;  // first row of the image in the batch
};
template <typename I>
__device__ __forceinline__ int find_img(const I* imgs, int n, int64_t k) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (imgs[mid].base <= k) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// One thread per JPEG block: the block's 64 coefficients come in as eight
// 16-byte loads (a warp reads 32 consecutive blocks, 4 KB contiguous), are
// dequantised in int32 (|coef| < 2^15, q < 2^16: exact) and stay in
// registers for both passes; row r of the samples leaves as one 8-byte store
// (a warp's stores of row r cover 32 consecutive blocks of a block row).
// Each pass runs in int32 when every input of the WARP is within kIdct32Max
// (a warp-uniform vote: no divergence), else in int64 -- the same integers
// either way (see idct8). After an int32 first pass the intermediates fit
// int32 (|o| <= 61214 * 12000 < 2^30), so the generic path only widens.
__device__ __forceinline__ bool warp_all_small(const int32_t (&b)[64]) {
  uint32_t bad = 0;
#pragma unroll
  for (int k = 0; k < 64; ++k) bad |= (uint32_t)(b[k] + (int32_t)kIdct32Max) > (uint32_t)(2 * kIdct32Max);
  return __all_sync(0xFFFFFFFFu, bad == 0);
}

__device__ __forceinline__ uint32_t pack4_u8(int32_t a, int32_t b, int32_t c, int32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// the rare path (crafted magnitudes): both passes in int64, column/row at a time
__device__ __noinline__ void idct_block_int64(const int16_t* co, const uint16_t* qt, uint8_t* dst, int64_t pitch) {
  int64_t ws[64];
#pragma unroll 1
  for (int j = 0; j < 8; ++j) {
    int64_t s[8], o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) s[k] = (int64_t)co[8 * k + j] * qt[8 * k + j];
    idct8<int64_t>(s, o);
#pragma unroll
    for (int k = 0; k < 8; ++k) ws[8 * k + j] = (o[k] + (1 << 10)) >> 11;
  }
#pragma unroll 1
  for (int r = 0; r < 8; ++r) {
    int64_t s[8], o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) s[k] = ws[8 * r + k];
    idct8<int64_t>(s, o);
    int32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t x = ((o[k] + (1 << 17)) >> 18) + 128;
      v[k] = (int32_t)(x < 0 ? 0 : (x > 255 ? 255 : x));
    }
    *reinterpret_cast<uint2*>(dst + r * pitch) = make_uint2(pack4_u8(v[0], v[1], v[2], v[3]), pack4_u8(v[4], v[5], v[6], v[7]));
  }
}

__global__ void __launch_bounds__(128) jpeg_idct_batch_kernel(const IdctImg* imgs, const int64_t* bases, int nimg,
                                                              int64_t total) {
  const int64_t gb0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = gb0 < total;
  const int64_t gb = live ? gb0 : total - 1;  // the whole warp stays for the votes; dead lanes do not store
  int lo = 0, hi = nimg - 1;
  while (lo < hi) {
    const int m = (lo + hi + 1) >> 1;
    if (__ldg(bases + m) <= gb) lo = m;
    else hi = m - 1;
  }
  const IdctArgs& a = imgs[lo].a;
  const int64_t blk = gb - __ldg(bases + lo);
  int c = 0;
  while (c + 1 < a.ncomp && blk >= a.first_block[c + 1]) ++c;
  const uint32_t lb = (uint32_t)(blk - a.first_block[c]);  // < 2^31 blocks per image
  const uint4* co = reinterpret_cast<const uint4*>(reinterpret_cast<const int16_t*>(a.coeffs) + a.coef_offset[c] +
                                                   64 * (int64_t)lb);
  const uint4* qt = reinterpret_cast<const uint4*>(&a.qt[c][0]);
  int32_t b[64];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const uint4 cr = __ldg(co + r), qr = qt[r];
    const uint32_t cw[4] = {cr.x, cr.y, cr.z, cr.w}, qw[4] = {qr.x, qr.y, qr.z, qr.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      b[8 * r + 2 * k] = (int32_t)(int16_t)(cw[k] & 0xFFFF) * (int32_t)(qw[k] & 0xFFFF);
      b[8 * r + 2 * k + 1] = ((int32_t)cw[k] >> 16) * (int32_t)(qw[k] >> 16);
    }
  }
  const uint32_t bw = (uint32_t)a.bw[c], by = lb / bw, bx = lb - by * bw;
  const int64_t pitch = (int64_t)bw * 8;
  uint8_t* dst = a.planes + a.plane_offset[c] + (int64_t)by * 8 * pitch + (int64_t)bx * 8;
  if (!warp_all_small(b)) {
    if (live) idct_block_int64(reinterpret_cast<const int16_t*>(co), &a.qt[c][0], dst, pitch);
    return;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {  // columns (vertical frequencies)
    int32_t s[8], o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) s[k] = b[8 * k + j];
    idct8<int32_t>(s, o);
#pragma unroll
    for (int k = 0; k < 8; ++k) b[8 * k + j] = (o[k] + (1 << 10)) >> 11;
  }
  const bool small2 = warp_all_small(b);
#pragma unroll
  for (int r = 0; r < 8; ++r) {  // rows
    int32_t v[8];
    if (small2) {
      int32_t s[8], o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) s[k] = b[8 * r + k];
      idct8<int32_t>(s, o);
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = min(max(((o[k] + (1 << 17)) >> 18) + 128, 0), 255);
    } else {
      int64_t s[8], o[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) s[k] = b[8 * r + k];
      idct8<int64_t>(s, o);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t x = ((o[k] + (1 << 17)) >> 18) + 128;
        v[k] = (int32_t)(x < 0 ? 0 : (x > 255 ? 255 : x));
      }
    }
    if (live)
      *reinterpret_cast<uint2*>(dst + r * pitch) =
          make_uint2(pack4_u8(v[0], v[1], v[2], v[3]), pack4_u8(v[4], v[5], v[6], v[7]));
  }
}

// Chroma columns 4i-1 .. 4i+4 of one chroma row (the 8 output columns
// 8i..8i+7 need them), column indices clamped to the plane: clamping is
// exactly the reference's edge rule -- its first/last output column formulas
// (jpeg.py:833-841) are the interior formula with the missing neighbour
// replaced by the edge column itself. Interior groups read three aligned
// words; edge groups read the six bytes one by one.
__device__ __forceinline__ void chroma6(const uint8_t* row, int i, int mw, bool interior, int (&c)[6]) {
  if (interior) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(row) + i;
    const uint32_t w0 = __ldg(p - 1), w1 = __ldg(p), w2 = __ldg(p + 1);
    c[0] = (int)(w0 >> 24);
#pragma unroll
    for (int t = 1; t < 5; ++t) c[t] = (int)((w1 >> (8 * (t - 1))) & 0xFF);
    c[5] = (int)(w2 & 0xFF);
  } else {
#pragma unroll
    for (int t = 0; t < 6; ++t) c[t] = (int)__ldg(row + min(max(4 * i - 1 + t, 0), mw - 1));
  }
}

// 4:2:0: the 8 upsampled samples of output columns 8i..8i+7 of one output
// row from its two chroma rows (near = the row's own, far = the one above
// for an even row, below for an odd row): column sums 3*near + far, then the
// horizontal 3:1 filter with +8 / +7 (jpeg.py:824-841).
__device__ __forceinline__ void upsample420_8(const int (&nr)[6], const int (&fr)[6], int (&s)[8]) {
  int v[6];
#pragma unroll
  for (int t = 0; t < 6; ++t) v[t] = 3 * nr[t] + fr[t];
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    const int t = (k >> 1) + 1;
    s[k] = (3 * v[t] + v[t - 1] + 8) >> 4;
    s[k + 1] = (3 * v[t] + v[t + 1] + 7) >> 4;
  }
}

// YCbCr -> RGB of 8 pixels (jpeg.py:226-235), stored as 3*n bytes (n <= 8)
__device__ __forceinline__ void store_rgb8(uint8_t* q, uint2 yv, const int (&cb)[8], const int (&cr)[8], int n) {
  int o[24];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int y = (int)(((k < 4 ? yv.x : yv.y) >> (8 * (k & 3))) & 0xFF);
    const int xb = cb[k] - 128, xr = cr[k] - 128;
    o[3 * k] = min(max(y + ((91881 * xr + 32768) >> 16), 0), 255);
    o[3 * k + 1] = min(max(y + ((-22554 * xb + 32768 - 46802 * xr) >> 16), 0), 255);
    o[3 * k + 2] = min(max(y + ((116130 * xb + 32768) >> 16), 0), 255);
  }
  uint32_t w[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) w[k] = pack4_u8(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]);
  const uintptr_t al = reinterpret_cast<uintptr_t>(q);
  if (n == 8 && (al & 7) == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) reinterpret_cast<uint2*>(q)[k] = make_uint2(w[2 * k], w[2 * k + 1]);
  } else if (n == 8 && (al & 3) == 0) {
#pragma unroll
    for (int k = 0; k < 6; ++k) reinterpret_cast<uint32_t*>(q)[k] = w[k];
  } else {
#pragma unroll
    for (int k = 0; k < 24; ++k)
      if (k < 3 * n) q[k] = (uint8_t)(w[k >> 2] >> (8 * (k & 3)));
  }
}

// Output rows 2m and 2m+1 (when present), columns 8i..8i+7 (those present),
// of a 4:2:0 image with chroma width > 2: the three chroma rows m-1, m, m+1
// (clamped: the reference's row replication) are read once for both rows.
// The Y plane's rows are padded to whole blocks, so its 8-byte load never
// leaves the row.
__device__ __forceinline__ void color420_16(const ColorArgs& a, int i, int m) {
  const int mw = a.cw[1], mh = a.ch[1];
  const int x0 = 8 * i, n = min(8, a.width - x0);
  const bool interior = i >= 1 && 4 * i + 4 <= mw - 1 && 4 * i + 8 <= a.pitch[1];
  const int ru = max(m - 1, 0), rd = min(m + 1, mh - 1);
  int b0[6], b1[6], b2[6], r0[6], r1[6], r2[6];
  chroma6(a.plane[1] + (int64_t)ru * a.pitch[1], i, mw, interior, b0);
  chroma6(a.plane[1] + (int64_t)m * a.pitch[1], i, mw, interior, b1);
  chroma6(a.plane[1] + (int64_t)rd * a.pitch[1], i, mw, interior, b2);
  chroma6(a.plane[2] + (int64_t)ru * a.pitch[2], i, mw, interior, r0);
  chroma6(a.plane[2] + (int64_t)m * a.pitch[2], i, mw, interior, r1);
  chroma6(a.plane[2] + (int64_t)rd * a.pitch[2], i, mw, interior, r2);
  const int y0 = 2 * m;
  {
    int cb[8], cr[8];
    upsample420_8(b1, b0, cb);
    upsample420_8(r1, r0, cr);
    const uint2 yv = __ldg(reinterpret_cast<const uint2*>(a.plane[0] + (int64_t)y0 * a.pitch[0] + x0));
    store_rgb8(a.dst + (int64_t)y0 * a.d_rp + 3 * x0, yv, cb, cr, n);
  }
  if (y0 + 1 < a.height) {
    int cb[8], cr[8];
    upsample420_8(b1, b2, cb);
    upsample420_8(r1, r2, cr);
    const uint2 yv = __ldg(reinterpret_cast<const uint2*>(a.plane[0] + (int64_t)(y0 + 1) * a.pitch[0] + x0));
    store_rgb8(a.dst + (int64_t)(y0 + 1) * a.d_rp + 3 * x0, yv, cb, cr, n);
  }
}

// One CTA per 8 output rows (4 row pairs) of an image of the batch; thread
// -> 8 columns of a row pair. The CTA's image and its arguments are looked
// up once (thread 0) and shared.
constexpr int kColorRows = 8;
__global__ void __launch_bounds__(256) jpeg_color_batch_kernel(const ColorImg* imgs, int nimg) {
  __shared__ ColorArgs sa;
  __shared__ int s_row0;
  if (threadIdx.x == 0) {
    const int im = find_img(imgs, nimg, (int64_t)blockIdx.x);
    sa = imgs[im].a;
    s_row0 = (int)(blockIdx.x - imgs[im].base) * kColorRows;
  }
  __syncthreads();
  const ColorArgs& a = sa;
  const int row0 = s_row0, row1 = min(row0 + kColorRows, a.height);
  const bool h2v2 = a.ncomp == 3 && a.fh[0] == 1 && a.fv[0] == 1 && a.fh[1] == 2 && a.fv[1] == 2 && a.fh[2] == 2 &&
                    a.fv[2] == 2 && a.cw[1] == a.cw[2] && a.ch[1] == a.ch[2] && a.cw[1] > 2;
  if (h2v2) {
    const int groups = (a.width + 7) >> 3;
    for (int y = row0; y < row1; y += 2)
      for (int i = threadIdx.x; i < groups; i += blockDim.x) color420_16(a, i, y >> 1);
    return;
  }
  for (int y = row0; y < row1; ++y)
    for (int x0 = threadIdx.x * 4; x0 < a.width; x0 += 4 * blockDim.x) color4(a, x0, y);
}

}  // namespace jpg
}  // namespace fv

using namespace fv;
using namespace fv::jpg;

extern "C" {

int fv_jpeg_info(const uint8_t* data, int64_t len, FvJpegInfo* info) {
  if (!info) return set_error(FV_EINVAL, "fv_jpeg_info: null info");
  std::unique_ptr<Stream> s(new Stream());
  const int rc = parse(data, len, *s);
  if (rc) return rc;
  fill_info(*s, *info);
  return FV_OK;
}

int fv_jpeg_decode_coeffs(const uint8_t* data, int64_t len, void* coeffs, int64_t coef_count, int32_t coef_bytes) {
  if (!coeffs || (coef_bytes != 2 && coef_bytes != 8))
    return set_error(FV_EINVAL, "fv_jpeg_decode_coeffs: coef_bytes must be 2 or 8");
  std::unique_ptr<Stream> s(new Stream());
  int rc = parse(data, len, *s);
  if (rc) return rc;
  FvJpegInfo f;
  fill_info(*s, f);
  if (coef_count < f.coef_count)
    return set_error(FV_EINVAL, "fv_jpeg_decode_coeffs: buffer holds %lld coefficients, stream needs %lld",
                     (long long)coef_count, (long long)f.coef_count);
  if (coef_bytes == 2) {
    Dense<int16_t> sink{static_cast<int16_t*>(coeffs)};
    return decode_scan(*s, f, sink);
  }
  Dense<int64_t> sink{static_cast<int64_t*>(coeffs)};
  return decode_scan(*s, f, sink);
}


}  // extern "C"

namespace fv {
namespace jpg {
// coef_bytes 2 / 4 / 8: dense int16 / int32 / int64 coefficients; 1: the
// sparse word stream of the host batch runtime
static int64_t make_idct_args(const FvJpegInfo& f, const void* coeffs, uint8_t* planes, IdctArgs& ia) {
  ia = IdctArgs{};
  ia.coeffs = coeffs;
  ia.planes = planes;
  int nd = 0;
  int64_t nb = 0;
  for (int e = 0; e < f.ncomp; ++e) {  // distinct components (duplicated scan entries share them)
    bool dup = false;
    for (int q = 0; q < nd; ++q) dup = dup || ia.coef_offset[q] == f.coef_offset[e];
    if (dup) continue;
    ia.first_block[nd] = nb;
    ia.coef_offset[nd] = f.coef_offset[e];
    ia.plane_offset[nd] = f.plane_offset[e];
    ia.bw[nd] = f.bw[e];
    memcpy(ia.qt[nd], f.qt[e], sizeof(ia.qt[nd]));
    nb += (int64_t)f.bw[e] * f.bh[e];
    ++nd;
  }
  ia.ncomp = nd;
  ia.first_block[nd] = nb;
  return nb;
}

static void make_color_args(const FvJpegInfo& f, uint8_t* planes, uint8_t* dst, int64_t dst_row_pitch, ColorArgs& ca) {
  ca = ColorArgs{};
  for (int e = 0; e < f.ncomp; ++e) {
    ca.plane[e] = planes + f.plane_offset[e];
    ca.pitch[e] = (int64_t)f.bw[e] * 8;
    ca.cw[e] = f.cw[e];
    ca.ch[e] = f.ch[e];
    ca.fh[e] = f.hmax / f.h[e];
    ca.fv[e] = f.vmax / f.v[e];
  }
  ca.ncomp = f.ncomp;
  ca.width = f.width;
  ca.height = f.height;
  ca.dst = dst;
  ca.d_rp = dst_row_pitch;
}

static int check_recon(const FvJpegInfo& f, uint8_t* planes, int64_t dst_row_pitch) {
  if (f.ncomp != 1 && f.ncomp != 3) return set_error(FV_EINVAL, "fv_jpeg_reconstruct: ncomp %d", f.ncomp);
  if (dst_row_pitch < (int64_t)f.width * f.ncomp) return set_error(FV_EINVAL, "fv_jpeg_reconstruct: row pitch too small");
  if ((reinterpret_cast<uintptr_t>(planes) & 7) != 0) return set_error(FV_EINVAL, "fv_jpeg_reconstruct: planes not 8-byte aligned");
  return FV_OK;
}

// coef_bytes 2 / 4 / 8: dense int16 / int32 / int64 coefficients; 1: the
// sparse word stream of the host batch runtime
int reconstruct(const FvJpegInfo& f, const void* coeffs, int32_t coef_bytes, uint8_t* planes, uint8_t* dst,
                int64_t dst_row_pitch, cudaStream_t st) {
  int rc = check_recon(f, planes, dst_row_pitch);
  if (rc) return rc;
  if (coef_bytes == 2 && (reinterpret_cast<uintptr_t>(coeffs) & 15) == 0) {  // the batch kernels, n = 1
    const FvJpegInfo* fs[1] = {&f};
    const int16_t* cs[1] = {static_cast<const int16_t*>(coeffs)};
    uint8_t* ps[1] = {planes};
    uint8_t* ds[1] = {dst};
    const int64_t dp[1] = {dst_row_pitch};
    return reconstruct_batch(1, fs, cs, ps, ds, dp, st);
  }
  IdctArgs ia;
  const int64_t nb = make_idct_args(f, coeffs, planes, ia);
  const int64_t grid = (nb + 15) / 16;
  if (grid > 0x7FFFFFFF) return set_error(FV_EINVAL, "fv_jpeg_reconstruct: too many blocks");
  if (coef_bytes == 2) jpeg_idct_kernel<int16_t><<<(unsigned)grid, 128, 0, st>>>(ia);
  else if (coef_bytes == 4) jpeg_idct_kernel<int32_t><<<(unsigned)grid, 128, 0, st>>>(ia);
  else if (coef_bytes == 8) jpeg_idct_kernel<int64_t><<<(unsigned)grid, 128, 0, st>>>(ia);
  else jpeg_idct_sparse_kernel<<<(unsigned)grid, 128, 0, st>>>(ia, static_cast<const uint32_t*>(coeffs), f.coef_count / 64);
  rc = check_launch("jpeg_idct_kernel");
  if (rc) return rc;
  ColorArgs ca;
  make_color_args(f, planes, dst, dst_row_pitch, ca);
  jpeg_color_kernel<<<dim3((f.width + 1023) / 1024, f.height), 256, 0, st>>>(ca);
  return check_launch("jpeg_color_kernel");
}

int reconstruct_batch(int n, const FvJpegInfo* const* fs, const int16_t* const* coeffs, uint8_t* const* planes,
                      uint8_t* const* dst, const int64_t* dst_pitch, cudaStream_t st) {
  if (n == 0) return FV_OK;
  std::vector<IdctImg> ii(n);
  std::vector<ColorImg> ci(n);
  int64_t blocks = 0, rows = 0;
  for (int i = 0; i < n; ++i) {
    int rc = check_recon(*fs[i], planes[i], dst_pitch[i]);
    if (rc) return rc;
    ii[i].base = blocks;
    blocks += make_idct_args(*fs[i], coeffs[i], planes[i], ii[i].a);
    ci[i].base = rows;
    make_color_args(*fs[i], planes[i], dst[i], dst_pitch[i], ci[i].a);
    rows += (fs[i]->height + kColorRows - 1) / kColorRows;  // the colour kernel's CTAs
  }
  if ((blocks + 15) / 16 > 0x7FFFFFFF || rows > 0x7FFFFFFF)
    return set_error(FV_EINVAL, "fv_jpeg_reconstruct: batch too large");
  std::vector<int64_t> bases(n);
  for (int i = 0; i < n; ++i) bases[i] = ii[i].base;
  IdctImg* di = nullptr;
  ColorImg* dc = nullptr;
  int64_t* db = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&di), n * sizeof(IdctImg), st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&dc), n * sizeof(ColorImg), st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&db), n * sizeof(int64_t), st) != cudaSuccess) {
    for (void* q : {(void*)di, (void*)dc, (void*)db})
      if (q) cudaFreeAsync(q, st);
    return set_error(FV_ECUDA, "fv_jpeg_reconstruct: argument buffers");
  }
  cudaMemcpyAsync(di, ii.data(), n * sizeof(IdctImg), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(dc, ci.data(), n * sizeof(ColorImg), cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(db, bases.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, st);
  jpeg_idct_batch_kernel<<<(unsigned)((blocks + 127) / 128), 128, 0, st>>>(di, db, n, blocks);
  int rc = check_launch("jpeg_idct_batch_kernel");
  if (!rc) {
    jpeg_color_batch_kernel<<<(unsigned)rows, 256, 0, st>>>(dc, n);
    rc = check_launch("jpeg_color_batch_kernel");
  }
  cudaFreeAsync(di, st);
  cudaFreeAsync(dc, st);
  cudaFreeAsync(db, st);
  return rc;
}

// Batch worker: parse + sparse entropy decoding into `words` (block header
// indices first, then the entries); *used = words written.
static int decode_one_sparse(const uint8_t* data, int64_t len, uint32_t* words, int64_t nwords, int64_t* used) {
  std::unique_ptr<Stream> s(new Stream());
  int rc = parse(data, len, *s);
  if (rc) return rc;
  FvJpegInfo f;
  fill_info(*s, f);
  const int64_t nblk = f.coef_count / 64;
  if (nwords < nblk + f.sparse_words) return set_error(FV_EINVAL, "fv_jpeg_decode_batch: sparse buffer too small");
  Sparse sink{words, words + nblk, f.sparse_words};
  rc = decode_scan(*s, f, sink);
  *used = nblk + sink.cur;
  return rc;
}
}  // namespace jpg
}  // namespace fv

extern "C" {

int fv_jpeg_reconstruct(const FvJpegInfo* info, const void* coeffs, int32_t coef_bytes, uint8_t* planes,
                        uint8_t* dst, int64_t dst_row_pitch, void* stream) {
  if (!info || !coeffs || !planes || !dst) return set_error(FV_EINVAL, "fv_jpeg_reconstruct: null pointer");
  if (coef_bytes != 2 && coef_bytes != 8) return set_error(FV_EINVAL, "fv_jpeg_reconstruct: coef_bytes must be 2 or 8");
  return reconstruct(*info, coeffs, coef_bytes, planes, dst, dst_row_pitch, static_cast<cudaStream_t>(stream));
}

int fv_jpeg_info_batch(const uint8_t* const* data, const int64_t* lens, int32_t n, FvJpegInfo* infos,
                       int32_t* status, int32_t threads) {
  if (n < 0 || (n > 0 && (!data || !lens || !infos || !status)))
    return set_error(FV_EINVAL, "fv_jpeg_info_batch: bad arguments");
  WorkPool::get().run(n, std::max(1, threads), [&](int32_t i) {
    std::unique_ptr<Stream> s(new Stream());
    status[i] = parse(data[i], lens[i], *s);
    if (status[i] == FV_OK) fill_info(*s, infos[i]);
  });
  return FV_OK;
}

int fv_jpeg_decode_batch(const uint8_t* const* data, const int64_t* lens, int32_t n, const FvJpegInfo* infos,
                         uint32_t* words_host, const int64_t* word_off, uint32_t* words_dev, uint8_t* planes,
                         const int64_t* plane_off, uint8_t* const* dst, const int64_t* dst_pitch, int32_t* status,
                         int32_t threads, void* stream) {
  if (n < 0 || (n > 0 && (!data || !lens || !infos || !words_host || !word_off || !words_dev || !planes ||
                          !plane_off || !dst || !dst_pitch || !status)))
    return set_error(FV_EINVAL, "fv_jpeg_decode_batch: bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  std::vector<std::atomic<int32_t>> done(n);
  std::vector<int64_t> used(n, 0);
  for (auto& d : done) d.store(1, std::memory_order_relaxed);  // 1 = pending
  // pool threads decode while this thread feeds the GPU (it finishes what
  // no pool thread took before returning)
  WorkPool& wp = WorkPool::get();
  WorkPool::Job job;
  job.fn = [&](int32_t i) {
    const int64_t cap = infos[i].coef_count / 64 + infos[i].sparse_words;
    const int rc = decode_one_sparse(data[i], lens[i], words_host + word_off[i], cap, &used[i]);
    if (rc == FV_OK) flush_lines(words_host + word_off[i], (size_t)used[i] * 4);  // DMA-friendly (see flush_lines)
    done[i].store(rc, std::memory_order_release);
  };
  job.n = n;
  job.want = std::max(1, std::min(std::min<int>(threads, n), wp.size()));
  wp.start(job);
  // in input order, as soon as an image's coefficients are ready: H2D of the
  // words it used, then its kernels
  int first = FV_OK;
  for (int32_t i = 0; i < n; ++i) {
    int32_t rc;
    while ((rc = done[i].load(std::memory_order_acquire)) == 1) std::this_thread::yield();
    status[i] = rc;
    if (rc != FV_OK || first != FV_OK) {
      if (first == FV_OK) first = rc;
      continue;
    }
    if (cudaMemcpyAsync(words_dev + word_off[i], words_host + word_off[i], used[i] * 4, cudaMemcpyHostToDevice, st) !=
        cudaSuccess) {
      first = set_error(FV_ECUDA, "fv_jpeg_decode_batch: H2D: %s", cudaGetErrorString(cudaGetLastError()));
      status[i] = first;
      continue;
    }
    rc = reconstruct(infos[i], words_dev + word_off[i], 1, planes + plane_off[i], dst[i], dst_pitch[i], st);
    if (rc) {
      first = rc;
      status[i] = rc;
    }
  }
  wp.wait(job);
  return first;
}

}  // extern "C"
