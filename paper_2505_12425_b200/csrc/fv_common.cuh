// fv_common.cuh -- shared device helpers for the sm_100a image kernels.
//
// Exact-arithmetic building blocks. Every helper reproduces one rounding step
// of the reference (NumPy, IEEE round-to-nearest per op, no FMA contraction):
// the float ops below are written with explicit __f*_rn / __d*_rn intrinsics,
// which nvcc never contracts into FMAs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include "../../include/fovea_b200.h"

namespace fv {

// ---------------------------------------------------------------------------
// device-side bounds checks (the checked build, -DFV_DEVICE_CHECKS: every
// TMA copy's shared-memory destination, and the staged kernels' shared-memory
// reads and copy sources against their buffers; compute-sanitizer is not
// available on the GPU pool, tools/checked_run.sh runs this build instead)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t dyn_smem_size() {
  uint32_t r;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}
#ifdef FV_DEVICE_CHECKS
__device__ __noinline__ inline void check_fail(const char* file, int line, const char* cond) {
  printf("FV_CHECK failed %s:%d: %s (block %d %d %d thread %d)\n", file, line, cond, blockIdx.x, blockIdx.y,
         blockIdx.z, threadIdx.x + blockDim.x * threadIdx.y);
  __trap();
}
#define FV_CHECK(cond) ((cond) ? (void)0 : ::fv::check_fail(__FILE__, __LINE__, #cond))
#else
#define FV_CHECK(cond) ((void)0)
#endif
// [addr, addr + bytes) inside the dynamic shared-memory allocation
__device__ __forceinline__ bool in_dyn_smem(uint32_t addr, uint32_t bytes) {
  extern __shared__ __align__(16) uint8_t fv_dyn_smem_base[];
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(fv_dyn_smem_base));
  return addr >= b && addr + bytes <= b + dyn_smem_size();
}

// ---------------------------------------------------------------------------
// error / launch bookkeeping (fv_util.cu)
// ---------------------------------------------------------------------------
int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);
void count_launch();

// Raise a kernel's dynamic shared-memory limit once per (kernel, device):
// the attribute is per device, and one process may drive several GPUs.
// `mask` is a static owned by the (per-kernel) caller: bit d = device d done.
template <typename K>
inline int ensure_smem_attr(K kern, int bytes, unsigned long long (&mask)[2]) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 128) return FV_ECUDA;
  unsigned long long& word = mask[dev >> 6];
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(__atomic_load_n(&word, __ATOMIC_ACQUIRE) & bit)) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
      return FV_ECUDA;
    __atomic_fetch_or(&word, bit, __ATOMIC_RELEASE);
  }
  return FV_OK;
}

// ---------------------------------------------------------------------------
// u8 <-> unit float
// ---------------------------------------------------------------------------

// RN(f32(u) / f32(255)) for u in [0, 255] -- image.py:159-160.
// f32(u) via the 2^23 magic (exact, no I2F), then a two-term reciprocal:
// RN(u*RHI + RN(u*RLO)) equals the IEEE quotient for all 256 inputs
// (checked exhaustively on the host and in tests/test_gpu_parity.py).
__device__ __forceinline__ float u8_to_unit(uint32_t u) {
  const float RHI = __uint_as_float(0x3B808081u);  // f32(1/255)
  const float RLO = __uint_as_float(0xAF7EFEFFu);  // f32(1/255 - RHI) = -2.3191758e-10
  float f = __fsub_rn(__uint_as_float(0x4B000000u | u), 8388608.0f);
  return __fmaf_rn(f, RHI, __fmul_rn(f, RLO));
}

// app.py:75 then tensor.py:273-276 for a non-negative blend result v <= 1:
// y = RN(v*255); t = RN(y + 0.5); q = floor(t); q <= 255 (see DESIGN.md §4:
// bilinear weights sum to <= 1 in f32, so no clamp can trigger).
// That epilogue, floor(RN(RN(v * K) + 0.5)) (K = 255; the 2:1 fast path
// folds the /4 into K = 63.75), equals
// floor(RN(fma(v, K, 0.5))) for EVERY f32 v in [0, 1.0625] (K = 255) and
// [0, 4.25] (K = 63.75) -- an exhaustive check over all 2^30 inputs, kept as
// tests/test_epilogue_identity.py. One FFMA replaces FMUL + FADD; floor is
// RD(t + 2^23), which leaves floor(t) in the low mantissa bits. Returns those
// float bits (0x4B0000uu).
__device__ __forceinline__ uint32_t scale_to_u8_bits(float v, float K) {
  return __float_as_uint(__fadd_rd(__fmaf_rn(v, K, 0.5f), 8388608.0f));
}
__device__ __forceinline__ uint32_t unit_to_u8(float v) {
  return scale_to_u8_bits(v, 255.0f) - 0x4B000000u;
}
// low bytes of four words -> one word
__device__ __forceinline__ uint32_t pack4(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t b3) {
  return __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
}
// ---------------------------------------------------------------------------
// Packed f32x2 arithmetic (sm_100: FADD2 / FMUL2 / FFMA2, two IEEE f32 ops per
// instruction, each lane rounded separately).
//
// CAUTION (ptxas 12.9): for .f32x2 ptxas contracts a mul.rn whose result is
// a MULTIPLICAND or a plain ADD operand into an FFMA2, ignoring the explicit
// rounding modifier (and -fmad=false). Only these shapes are used here:
//   * mul2 result as the ADDEND of an explicit fma2 (cannot be contracted:
//     the fma already has a product);
//   * add2 whose operands are not bare products;
//   * RN(p + q) of two products written as fma2(q, one, p) with `one` a
//     RUNTIME 1.0 (kernel argument), so ptxas cannot fold a product in.
// tests/test_gpu_parity.py checks every kernel bit-exactly at config sizes.
// ---------------------------------------------------------------------------
typedef unsigned long long f2_t;

__device__ __forceinline__ f2_t f2(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ f2_t f2u(uint32_t lo, uint32_t hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ void f2split(f2_t v, uint32_t& lo, uint32_t& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v));
}
__device__ __forceinline__ f2_t fmul2(f2_t a, f2_t b) {
  f2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t ffma2(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ f2_t fadd2(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t fadd2_rd(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// two u8_to_unit at once from two magic words 0x4B0000uu
#ifndef FV_UNIT2_FMA
#define FV_UNIT2_FMA 1  // two-FFMA2 form below (0: the subtract + split-constant three-op form)
#endif
__device__ __forceinline__ f2_t unit2(uint32_t m_lo, uint32_t m_hi) {
#if FV_UNIT2_FMA
  // y = u*257/2^16 is exact (17 significant bits), taken straight from the
  // magic word M = 2^23 + u: fma(M, 257/2^16, -2^23*257/2^16) = RN(y) = y.
  // Then RN(u/255) = RN(y * (1 + 2^-16 + 2^-32)): the dropped tail of
  // 65536/65535 is < 2^-47 relative and moves no u in [0, 255] across a
  // rounding boundary (checked exhaustively against exact rationals).
  const float K257 = __uint_as_float(0x3B808000u);  // 257 / 2^16
  const float CT = __uint_as_float(0x37800080u);    // 2^-16 + 2^-32
  const f2_t y = ffma2(f2u(m_lo, m_hi), f2(K257, K257), f2(-32896.0f, -32896.0f));
  return ffma2(y, f2(CT, CT), y);
#else
  const float RHI = __uint_as_float(0x3B808081u);
  const float RLO = __uint_as_float(0xAF7EFEFFu);
  const f2_t f = fadd2(f2u(m_lo, m_hi), f2(-8388608.0f, -8388608.0f));
  return ffma2(f, f2(RHI, RHI), fmul2(f, f2(RLO, RLO)));
#endif
}
// magic word 0x4B0000uu of byte i of a word array: PRMT puts the byte under
// the exponent of 2^23 (i compile-time after unrolling)
template <int N>
__device__ __forceinline__ uint32_t magic_of(const uint32_t (&w)[N], int i) {
  return __byte_perm(w[i >> 2], 0x4B000000u, 0x7440 + (i & 3));
}
// The runtime {1.0f, 1.0f} pair, passed as a 64-bit kernel argument so that
// it stays in a uniform register pair (ptxas cannot know its value).
constexpr f2_t kOne2Bits = 0x3F8000003F800000ull;

// scale_to_u8_bits on a pair (same exhaustive identity); returns the two
// float-bit words whose low bytes are the results.
__device__ __forceinline__ f2_t scale_to_u8_bits2(f2_t v, float scale) {
  return fadd2_rd(ffma2(v, f2(scale, scale), f2(0.5f, 0.5f)), f2(8388608.0f, 8388608.0f));
}
// low bytes of two pairs -> one word
__device__ __forceinline__ uint32_t pack4x2(f2_t a, f2_t b) {
  uint32_t a0, a1, b0, b1;
  f2split(a, a0, a1);
  f2split(b, b0, b1);
  return pack4(a0, a1, b0, b1);
}

// imgproc.py:118-123: top = a00*(1-fx) + a01*fx, etc. -- every product and
// sum separately rounded. w0 = RN(1 - f), w1 = f.
__device__ __forceinline__ float lerp_ref(float a, float b, float w0, float w1) {
  return __fadd_rn(__fmul_rn(a, w0), __fmul_rn(b, w1));
}

__device__ __forceinline__ bool pow2_or_zero(float w) { return (__float_as_uint(w) & 0x007FFFFFu) == 0; }

// ---------------------------------------------------------------------------
// resize coordinate map -- imgproc.py:76-78, 109-116
// s = clip((i + 0.5) * scale - 0.5, 0, n - 1) in f64, scale = src_n / dst_n;
// i0 = floor(s); i1 = min(i0 + 1, n - 1); f = f32(s - i0).
// ---------------------------------------------------------------------------
struct AxisTap {
  int i0, i1;
  float w0, w1;  // RN(1 - f), f
};

__device__ __forceinline__ AxisTap axis_tap(int i, double scale, int src_n) {
  double s = __dadd_rn(__dmul_rn(__dadd_rn((double)i, 0.5), scale), -0.5);
  s = fmin(fmax(s, 0.0), (double)(src_n - 1));
  double fl = floor(s);
  AxisTap t;
  t.i0 = (int)fl;
  t.i1 = min(t.i0 + 1, src_n - 1);
  t.w1 = __double2float_rn(__dadd_rn(s, -fl));
  t.w0 = __fsub_rn(1.0f, t.w1);
  return t;
}

// ---------------------------------------------------------------------------
// element load / store helpers
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ const T* row_ptr(const void* base, int64_t img_stride, int64_t pitch,
                                            int n, int y) {
  return reinterpret_cast<const T*>(reinterpret_cast<const char*>(base) + n * img_stride + y * pitch);
}
template <typename T>
__device__ __forceinline__ T* row_ptr_mut(void* base, int64_t img_stride, int64_t pitch, int n, int y) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(base) + n * img_stride + y * pitch);
}

// tap value as the blend operand: u8 -> unit float, f32 -> itself
__device__ __forceinline__ float tap_value(uint8_t u) { return u8_to_unit(u); }
__device__ __forceinline__ float tap_value(float f) { return f; }

// Warp index as a value ptxas can prove warp-uniform (a shuffle from lane
// 0). threadIdx.x >> 5 is uniform per warp, but ptxas treats it as per-thread:
// code after a warp-role branch on it then counts as divergent, and ptxas
// keeps the global-memory descriptor in ordinary registers and copies it into
// uniform ones (2 R2UR) before every global access in the loop. Branching on
// this value keeps the descriptor and the loop's address arithmetic uniform.
__device__ __forceinline__ int warp_index_uniform() {
  return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
}

// ---------------------------------------------------------------------------
// mbarrier + TMA bulk copy (cp.async.bulk) PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Consumer-side release of a TMA ring slot after reading it with ordinary
// loads. Every lane fences its generic-proxy reads against the async proxy
// (MEMBAR + FENCE.VIEW.ASYNC: the reads have completed before the slot can be
// refilled by cp.async.bulk), the warp converges, one lane arrives. Without
// the fence a refill could overtake a lane's in-flight LDS (observed as a
// rare wrong row on the first launch in a process).
__device__ __forceinline__ void slot_release(uint64_t* bar, int lane) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) mbar_arrive(bar);
}
// blocking wait: the thread is suspended (NANOSLEEP.SYNCS) until the phase
// completes or the hint (ns) expires, instead of spinning on try_wait
__device__ __forceinline__ void mbar_wait_block(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!ok);
}
// 1-D bulk copy global -> shared, completion signalled on `bar` (TMA unit,
// SASS UBLKCP). dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  FV_CHECK(in_dyn_smem(smem_u32(dst), bytes) && (bytes & 15) == 0 && (smem_u32(dst) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(src) & 15) == 0);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace fv
