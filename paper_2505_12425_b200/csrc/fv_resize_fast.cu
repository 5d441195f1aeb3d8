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
  f2_t one2;   // runtime {1.0f, 1.0f} (see fv_common.cuh: f32x2 contraction guard)
  int slot_bytes;
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
    // element pairs (e, e+1) in packed f32x2: 4 taps, 3 adds, epilogue
    uint32_t out[4 * C];
#pragma unroll
    for (int q = 0; q < 4 * C; ++q) {
      f2_t r[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int e0 = 4 * q + 2 * j, e1 = e0 + 1;  // destination bytes in the group
        const int o0 = 2 * (e0 / C) * C + e0 % C;   // first tap byte of each
        const int o1 = 2 * (e1 / C) * C + e1 % C;
        const f2_t top = fadd2(unit2(magic_of(w0, o0), magic_of(w0, o1)),
                               unit2(magic_of(w0, o0 + C), magic_of(w0, o1 + C)));
        const f2_t bot = fadd2(unit2(magic_of(w1, o0), magic_of(w1, o1)),
                               unit2(magic_of(w1, o0 + C), magic_of(w1, o1 + C)));
        r[j] = scale_to_u8_bits2(fadd2(top, bot), K);
      }
      out[q] = pack4x2(r[0], r[1]);
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
        d[p * C + c] = (uint8_t)(scale_to_u8_bits(__fadd_rn(top, bot), K) & 0xFF);
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

// h for the thread's 8 destination pixels from one source row's window, as
// 4C packed pairs laid out for FFMA2 (the destination element of each half is
// up2_elem below). Per channel, with v[m] the unit value of source pixel
// 4t + m (m = -1..4) and P[m] = RN(0.75 v[m]):
//   h[4c]     = {E0, E1}, h[4c + 1] = {E2, E3}   E[m] = fma(v[m-1], 0.25, P[m])  -> dst px 2m
//   h[4c + 2] = {O0, O1}, h[4c + 3] = {O2, O3}   O[m] = fma(v[m+1], 0.25, P[m])  -> dst px 2m+1
// The unit conversions are done in the pairs {v-1, v0}, {v1, v2}, {v3, v4};
// the P pairs {P0, P1}, {P2, P3} come from the two re-paired {v0, v1},
// {v2, v3} (register moves), so every product and sum is one f32x2 op.
template <int C>
__device__ __forceinline__ void up2_h(const uint32_t (&w)[Up2<C>::NW], int t, int last_t, f2_t (&h)[4 * C]) {
  const f2_t q4 = f2(0.25f, 0.25f), t4 = f2(0.75f, 0.75f);
#pragma unroll
  for (int c = 0; c < C; ++c) {
    // window byte of source pixel 4t + m, channel c: 4 + m*C + c
    const f2_t A = unit2(magic_of(w, 4 - C + c), magic_of(w, 4 + c));
    const f2_t B = unit2(magic_of(w, 4 + C + c), magic_of(w, 4 + 2 * C + c));
    const f2_t D = unit2(magic_of(w, 4 + 3 * C + c), magic_of(w, 4 + 4 * C + c));
    uint32_t a0, a1, b0, b1, d0, d1;
    f2split(A, a0, a1);
    f2split(B, b0, b1);
    f2split(D, d0, d1);
    // scalar products written straight into the two halves of a pair (an
    // f32x2 product of the re-paired {v0, v1} would first need two moves)
    const f2_t PX = f2(__fmul_rn(__uint_as_float(a1), 0.75f), __fmul_rn(__uint_as_float(b0), 0.75f));
    const f2_t PY = f2(__fmul_rn(__uint_as_float(b1), 0.75f), __fmul_rn(__uint_as_float(d0), 0.75f));
    f2_t E01 = ffma2(A, q4, PX);
    const f2_t E23 = ffma2(B, q4, PY), O01 = ffma2(B, q4, PX);
    f2_t O23 = ffma2(D, q4, PY);
    if (t == 0) {  // destination pixel 0: clamped, fx = 0 -> copy of v0
      uint32_t lo, hi;
      f2split(E01, lo, hi);
      E01 = f2u(a1, hi);
    }
    if (t == last_t) {  // destination pixel 2W-1: clamped, fx = 0 -> copy of v3
      uint32_t lo, hi;
      f2split(O23, lo, hi);
      O23 = f2u(lo, d0);
    }
    h[4 * c] = E01;
    h[4 * c + 1] = E23;
    h[4 * c + 2] = O01;
    h[4 * c + 3] = O23;
  }
}
// destination element (px * C + c) of half `hi` of pair p in up2_h's layout
template <int C>
__host__ __device__ constexpr int up2_elem(int p, int hi) {
  return (2 * (2 * ((p & 3) & 1) + hi) + ((p & 3) >> 1)) * C + p / 4;
}

#ifndef FV_UP2_CS
#define FV_UP2_CS 0  // 1: evict-first stores (st.global.cs); ptxas builds a cache-policy descriptor and
                     // moves it into uniform registers (2 R2UR) before every such store
#endif
__device__ __forceinline__ void up2_store(uint2* p, uint2 v) {
#if FV_UP2_CS
  __stcs(p, v);
#else
  *p = v;
#endif
}

// the 4C result pairs of one destination row (float-bit words, low byte =
// value) -> 2C words in memory order, written as C 8-byte stores
template <int C>
__device__ __forceinline__ void up2_pack_store(uint8_t* drow, const f2_t (&r)[4 * C]) {
  uint32_t e[8 * C];
#pragma unroll
  for (int p = 0; p < 4 * C; ++p) f2split(r[p], e[up2_elem<C>(p, 0)], e[up2_elem<C>(p, 1)]);
#pragma unroll
  for (int i = 0; i < C; ++i)
    up2_store(reinterpret_cast<uint2*>(drow) + i,
              make_uint2(pack4(e[8 * i], e[8 * i + 1], e[8 * i + 2], e[8 * i + 3]),
                         pack4(e[8 * i + 4], e[8 * i + 5], e[8 * i + 6], e[8 * i + 7])));
}
// one destination row from two h rows: o = fma(hb, 0.25, qa), epilogue in f32x2
template <int C>
__device__ __forceinline__ void up2_emit(uint8_t* drow, const f2_t (&hb)[4 * C], const f2_t (&qa)[4 * C]) {
  f2_t r[4 * C];
#pragma unroll
  for (int p = 0; p < 4 * C; ++p) r[p] = scale_to_u8_bits2(ffma2(hb[p], f2(0.25f, 0.25f), qa[p]), 255.0f);
  up2_pack_store<C>(drow, r);
}
// a row that is a plain copy of h (clamped rows 0 and 2H-1, fy = 0)
template <int C>
__device__ __forceinline__ void up2_emit_copy(uint8_t* drow, const f2_t (&h)[4 * C]) {
  f2_t r[4 * C];
#pragma unroll
  for (int p = 0; p < 4 * C; ++p) r[p] = scale_to_u8_bits2(h[p], 255.0f);
  up2_pack_store<C>(drow, r);
}

// TMA-staged variant: a CTA = 4 consumer warps (128 column groups = 512
// source pixels) + 1 producer warp. The producer streams the band's source
// row segments into an UP2_RING-slot shared-memory ring with 1-D bulk copies
// (cp.async.bulk, completion on the slot's "full" mbarrier); consumers read
// their 4-byte aligned windows with LDS (lane stride 12 B: conflict-free) and
// release the slot on its "empty" mbarrier.
constexpr int UP2_NCW = 3, UP2_GROUPS = UP2_NCW * 32, UP2_RING = 8;
#ifndef FV_UP2_CLAMP
#define FV_UP2_CLAMP 1  // 0: lanes past the tile's last group skip the row work (divergent stores)
#endif
#ifndef UP2_BAND
#define UP2_BAND 32  // source rows per CTA (one halo row re-read per band); 16 / 64 / 128 measured slower
#endif

template <int C>
__device__ __forceinline__ void up2_lds(const uint8_t* seg_row_base, int t, uint32_t (&w)[Up2<C>::NW]) {
  // seg_row_base points at source-row byte 0 inside the slot (may lie before
  // the slot for t = 0; those bytes feed only the clamped pixel and are unused)
  const uint32_t* rw = reinterpret_cast<const uint32_t*>(seg_row_base + 4 * C * t - 4);
  FV_CHECK(in_dyn_smem(smem_u32(rw), 4 * Up2<C>::NW));
#pragma unroll
  for (int i = 0; i < Up2<C>::NW; ++i) w[i] = rw[i];
}

// source row k: destination rows 2k-1 and 2k; dr points at row 2k
template <int C>
__device__ __forceinline__ void up2_step_s(uint8_t* dr, int64_t rp, int t, int last_t, bool first,
                                           const uint32_t (&w)[Up2<C>::NW], const f2_t (&hp)[4 * C],
                                           f2_t (&q)[4 * C], f2_t (&hn)[4 * C]) {
  up2_h<C>(w, t, last_t, hn);
  if (first) {
    up2_emit_copy<C>(dr, hn);
  } else {
    up2_emit<C>(dr - rp, hn, q);
  }
#pragma unroll
  for (int e = 0; e < 4 * C; ++e) q[e] = fmul2(hn[e], f2(0.75f, 0.75f));
  if (!first) up2_emit<C>(dr, hp, q);
}

template <int C>
__global__ void __launch_bounds__((UP2_NCW + 1) * 32, 4) resize_up2_kernel(const __grid_constant__ FastArgs a) {
  constexpr int NP = 4 * C, NW = Up2<C>::NW;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + UP2_RING;
  uint8_t* slots = smem + 16 * UP2_RING + 16;  // 16 bytes of slack before slot 0

  const int warp = warp_index_uniform(), lane = threadIdx.x & 31;
  const int n = blockIdx.z;
  const int k0 = blockIdx.y * a.band;
  const int k1 = min(k0 + a.band, a.sh);
  const int g0 = blockIdx.x * UP2_GROUPS;                 // first column group of the tile
  const int g1 = min(g0 + UP2_GROUPS, a.groups);
  // source bytes the tile reads: pixels [4*g0 - 1, 4*g1] clamped, 16-byte aligned superset
  const int b_lo = max(4 * g0 - 1, 0) * C;
  const int b_hi = min(4 * g1 + 1, a.sw) * C;
  const int gstart = b_lo & ~15;
  const uint32_t nbytes = (uint32_t)((b_hi - gstart + 15) & ~15);
  const int r_first = k0 > 0 ? k0 - 1 : 0;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < UP2_RING; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], UP2_NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == UP2_NCW) {  // producer
    if (lane == 0) {
      const uint8_t* src = a.src + n * a.s_is + gstart;
      for (int r = r_first, i = 0; r < k1; ++r, ++i) {
        const int slot = i % UP2_RING;
        if (i >= UP2_RING) mbar_wait_block(&empty[slot], (uint32_t)(((i / UP2_RING) - 1) & 1));
        FV_CHECK(r >= 0 && r < a.sh && gstart >= 0 &&
                 (int64_t)r * a.s_rp + gstart + nbytes <= (int64_t)(a.sh - 1) * a.s_rp + (int64_t)a.sw * C &&
                 nbytes <= (uint32_t)a.slot_bytes);
        mbar_expect_tx(&full[slot], nbytes);
        tma_bulk_g2s(slots + slot * a.slot_bytes, src + (int64_t)r * a.s_rp, nbytes, &full[slot]);
      }
    }
    return;
  }

#if FV_UP2_CLAMP
  // lanes past the tile's last group redo that group (same window, same
  // bytes to the same addresses): no divergent store region
  const int t = min(g0 + warp * 32 + lane, g1 - 1);
  constexpr bool active = true;
#else
  const int t = g0 + warp * 32 + lane;  // this thread's column group
  const bool active = t < g1;
#endif
  uint8_t* dimg = a.dst + n * a.d_is + (int64_t)t * 8 * C;
  const int64_t rp = a.d_rp;
  const int last_t = a.groups - 1;
  f2_t h0[NP], h1[NP], q[NP];
  uint32_t w[NW];
  int slot = 0;
  uint32_t phase = 0;
  auto take = [&]() {  // window of the next source row from the ring
    mbar_wait(&full[slot], phase);
    up2_lds<C>(slots + slot * a.slot_bytes - gstart, t, w);
    slot_release(&empty[slot], lane);
    if (++slot == UP2_RING) {
      slot = 0;
      phase ^= 1u;
    }
  };
  if (k0 > 0) {
    take();  // row k0 - 1
    up2_h<C>(w, t, last_t, h0);
#pragma unroll
    for (int e = 0; e < NP; ++e) q[e] = fmul2(h0[e], f2(0.75f, 0.75f));
  }
  int k = k0;
  uint8_t* dr = dimg + (int64_t)(2 * k0) * rp;  // destination row 2k
#pragma unroll 1
  for (; k + 1 < k1; k += 2) {
    take();
    if (active) up2_step_s<C>(dr, rp, t, last_t, k == 0, w, h0, q, h1);
    take();
    if (active) up2_step_s<C>(dr + 2 * rp, rp, t, last_t, false, w, h1, q, h0);
    dr += 4 * rp;
  }
  if (k < k1) {
    take();
    if (active) {
      up2_step_s<C>(dr, rp, t, last_t, k == 0, w, h0, q, h1);
      if (k1 == a.sh) up2_emit_copy<C>(dr + rp, h1);
    }
  } else if (k1 == a.sh && active) {
    up2_emit_copy<C>(dr - rp, h0);
  }
}

// 2:1 downscale, TMA-staged variant (dst width a multiple of 16 px): a CTA =
// D2_NCW consumer warps (one 16-pixel group per thread) + 1 producer warp
// streaming the tile's source row segments into a D2_RING-slot ring with
// 1-D bulk copies. Every source byte crosses L2 -> SMEM once (the direct
// kernel's 96-byte-strided 16-byte loads re-requested sectors from L2 2x),
// and consumers read their 96-byte windows with LDS.128.
constexpr int D2_NCW = 4, D2_GROUPS = D2_NCW * 32, D2_RING = 6;

template <int C>
__global__ void __launch_bounds__((D2_NCW + 1) * 32) resize_down2_tma_kernel(const __grid_constant__ FastArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + D2_RING;
  uint8_t* slots = smem + 16 * D2_RING;

  const int warp = warp_index_uniform(), lane = threadIdx.x & 31;
  const int n = blockIdx.z;
  const int y0 = blockIdx.y * a.band, y1 = min(y0 + a.band, a.dh);
  const int g0 = blockIdx.x * D2_GROUPS, g1 = min(g0 + D2_GROUPS, a.groups);
  const uint32_t nbytes = (uint32_t)((g1 - g0) * 32 * C);  // multiple of 16
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < D2_RING; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], D2_NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == D2_NCW) {  // producer: source rows 2*y0 .. 2*y1-1 in order
    if (lane == 0) {
      const uint8_t* src = a.src + n * a.s_is + (int64_t)g0 * 32 * C;
      for (int r = 2 * y0, i = 0; r < 2 * y1; ++r, ++i) {
        const int slot = i % D2_RING;
        if (i >= D2_RING) mbar_wait_block(&empty[slot], (uint32_t)(((i / D2_RING) - 1) & 1));
        FV_CHECK(r >= 0 && r < a.sh && (int64_t)g0 * 32 * C + nbytes <= (int64_t)a.sw * C &&
                 nbytes <= (uint32_t)a.slot_bytes);
        mbar_expect_tx(&full[slot], nbytes);
        tma_bulk_g2s(slots + slot * a.slot_bytes, src + (int64_t)r * a.s_rp, nbytes, &full[slot]);
      }
    }
    return;
  }

  const int t = g0 + warp * 32 + lane;
  const bool active = t < g1;
  const float K = 63.75f;  // 255 / 4
  int i = 0;
#pragma unroll 1
  for (int y = y0; y < y1; ++y, i += 2) {
    const int sa = i % D2_RING, sb = (i + 1) % D2_RING;
    mbar_wait(&full[sa], (uint32_t)((i / D2_RING) & 1));
    mbar_wait(&full[sb], (uint32_t)(((i + 1) / D2_RING) & 1));
    uint32_t w0[8 * C], w1[8 * C];
    if (active) {
      const uint4* s0 = reinterpret_cast<const uint4*>(slots + sa * a.slot_bytes + (t - g0) * 32 * C);
      const uint4* s1 = reinterpret_cast<const uint4*>(slots + sb * a.slot_bytes + (t - g0) * 32 * C);
#pragma unroll
      for (int k = 0; k < 2 * C; ++k) {
        const uint4 u = s0[k], v = s1[k];
        w0[4 * k] = u.x, w0[4 * k + 1] = u.y, w0[4 * k + 2] = u.z, w0[4 * k + 3] = u.w;
        w1[4 * k] = v.x, w1[4 * k + 1] = v.y, w1[4 * k + 2] = v.z, w1[4 * k + 3] = v.w;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // see slot_release
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&empty[sa]);
      mbar_arrive(&empty[sb]);
    }
    if (!active) continue;
    uint32_t out[4 * C];
#pragma unroll
    for (int q = 0; q < 4 * C; ++q) {
      f2_t r[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int e0 = 4 * q + 2 * j, e1 = e0 + 1;
        const int o0 = 2 * (e0 / C) * C + e0 % C;
        const int o1 = 2 * (e1 / C) * C + e1 % C;
        const f2_t top = fadd2(unit2(magic_of(w0, o0), magic_of(w0, o1)),
                               unit2(magic_of(w0, o0 + C), magic_of(w0, o1 + C)));
        const f2_t bot = fadd2(unit2(magic_of(w1, o0), magic_of(w1, o1)),
                               unit2(magic_of(w1, o0 + C), magic_of(w1, o1 + C)));
        r[j] = scale_to_u8_bits2(fadd2(top, bot), K);
      }
      out[q] = pack4x2(r[0], r[1]);
    }
    uint4* dv = reinterpret_cast<uint4*>(a.dst + n * a.d_is + (int64_t)y * a.d_rp + (int64_t)t * 16 * C);
#pragma unroll
    for (int k = 0; k < C; ++k) __stcs(dv + k, make_uint4(out[4 * k], out[4 * k + 1], out[4 * k + 2], out[4 * k + 3]));
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
    if (a.dw % 16 == 0) {  // TMA-staged kernel
      a.band = 16;
      a.bands = (a.dh + a.band - 1) / a.band;
      a.slot_bytes = D2_GROUPS * 32 * C;
      const size_t smem = 16 * D2_RING + (size_t)D2_RING * a.slot_bytes;
      auto kern = resize_down2_tma_kernel<C>;
      static unsigned long long attr_mask[2] = {0, 0};  // per instantiation
      if (ensure_smem_attr(kern, (int)smem, attr_mask) != FV_OK)
        return check_launch("resize_down2_tma_kernel (smem attribute)");
      dim3 grid((a.groups + D2_GROUPS - 1) / D2_GROUPS, a.bands, a.n);
      kern<<<grid, (D2_NCW + 1) * 32, smem, st>>>(a);
      return check_launch("resize_down2_tma_kernel");
    }
    const int64_t total = (int64_t)a.n * a.dh * a.groups;
    resize_down2_kernel<C><<<(unsigned)((total + 127) / 128), 128, 0, st>>>(a);
  } else {
    a.groups = a.sw / 4;
    a.band = UP2_BAND;
    a.bands = (a.sh + a.band - 1) / a.band;
    // ring slot: the tile's source bytes (+ halo, + alignment), 16-byte padded
    // on both sides for the unused halo words of the edge groups
    a.slot_bytes = ((UP2_GROUPS * 4 + 2) * C + 16 + 15) / 16 * 16 + 32;
    const size_t smem = 16 * UP2_RING + 16 + (size_t)UP2_RING * a.slot_bytes;
    auto kern = resize_up2_kernel<C>;
    static unsigned long long attr_mask[2] = {0, 0};  // per instantiation
  if (ensure_smem_attr(kern, (int)smem, attr_mask) != FV_OK) return check_launch("resize_up2_kernel (smem attribute)");
    dim3 grid((a.groups + UP2_GROUPS - 1) / UP2_GROUPS, a.bands, a.n);
    kern<<<grid, (UP2_NCW + 1) * 32, smem, st>>>(a);
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
    if (sw % 4 != 0 || sh < 2 || !aligned(src, 16) || !aligned(dst, 8) || (s_is | s_rp) & 15 || (d_is | d_rp) & 7)
      return FV_OK;
  }
  FastArgs a{src, s_is, s_rp, sh, sw, dst, d_is, d_rp, dh, dw, n, 0, 0, 0, kOne2Bits, 0};
  *taken = true;
  switch (c) {
    case 1: return launch_fast_c<1>(a, down, st);
    case 3: return launch_fast_c<3>(a, down, st);
    default: return launch_fast_c<4>(a, down, st);
  }
}

}  // namespace fv
