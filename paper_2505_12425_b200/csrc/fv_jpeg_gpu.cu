// fv_jpeg_gpu.cu -- GPU entropy decoding for the batched JPEG path
// (decode -> preprocess).
//
// Huffman decoding is serial along a segment, but the code is
// self-synchronising: a decoder started at an arbitrary bit soon falls into
// step with the true decode. Each restart segment's (unstuffed) bits are cut
// into kSubBits subsequences, one thread each:
//   1. speculative pass: thread t warms up on subsequence t-1 from a guessed
//      context (block slot 0, coefficient 0), then decodes its own bits and
//      records its exit state (bit position, slot, coefficient index), its
//      tally (blocks started, DC-difference sums per component) and, every
//      kCpBits, checkpoints of its state -- of its own decode and of its
//      warm-up over t-1 (two independent trajectories through each range);
//   2. sync rounds: E_t = decode(E_{t-1}, subsequence t) until no state
//      changes -- a fixed point is the true decode by induction (subsequence
//      0 of a segment starts exact). A round decode stops as soon as it
//      meets a recorded checkpoint state (the rest follows from the record),
//      and a thread whose state changed carries it on through up to kChain
//      following subsequences; unconverged images fall back;
//   3. scan: per segment, exclusive sums of the tallies -> the first block
//      and the DC predictions every subsequence starts from;
//   4. write pass: every block is written whole (zeros included, DC
//      prediction applied) by the thread it starts in, assembled in shared
//      memory -- the coefficient buffer needs no clearing and no second pass.
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <thread>

#include "fv_jpeg_host.cuh"

namespace fv {
namespace jpg {

#ifndef FV_JPEG_SUB_BITS
#define FV_JPEG_SUB_BITS 1024
#endif
constexpr int kSubBits = FV_JPEG_SUB_BITS;
// Device-only fast entry: an AC table's end-of-block code (<= 10 bits) as a
// "full" entry with this flag, so the decoder's common path covers
// coefficients and EOBs alike (86% of the symbols of typical q90 frames).
constexpr int32_t kEob = 1 << 14;
constexpr int kMaxSlots = 12;
constexpr int kSyncRounds = 6;    // rounds per chunk (one 4-byte readback per chunk)
constexpr int kSyncChunks = 32;   // cap: images still changing after this fall back
// tuning constants (overridable with -D for A/B builds)
#ifndef FV_JPEG_CHAIN
#define FV_JPEG_CHAIN 8
#endif
#ifndef FV_JPEG_CHAIN0
#define FV_JPEG_CHAIN0 8
#endif
#ifndef FV_JPEG_WARM_BITS
#define FV_JPEG_WARM_BITS 1024
#endif
#ifndef FV_JPEG_CP_BITS
#define FV_JPEG_CP_BITS 128
#endif
constexpr int kChain = FV_JPEG_CHAIN;    // subsequences one thread may carry a changed state through per round
constexpr int kChain0 = FV_JPEG_CHAIN0;  // ... in the first (full) round
constexpr int kWarmBits = FV_JPEG_WARM_BITS;  // speculative pass: bits decoded before a thread's own, to synchronise

__constant__ int kZigzagDev[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                                   12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                                   35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                                   58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

struct DevHuff {
  int32_t fast[1 << 10];
  int32_t maxcode[18];
  int32_t mincode[17];
  int32_t valptr[17];
  uint8_t values[256];
};

struct DevImg {
  int32_t dc_t[3], ac_t[3];  // per scan entry: index into the batch's (deduplicated) Huffman tables
  int8_t slot_e[kMaxSlots], slot_bx[kMaxSlots], slot_by[kMaxSlots];
  uint32_t slot_e2;  // slot_e packed, 2 bits per slot
  int64_t slot_off[kMaxSlots];  // coefficient offset of each slot's block within its MCU (component region included)
  int64_t mcu_row[3], mcu_col[3];  // coefficient strides of an MCU row / column per scan entry
  int32_t nslots, mcus_x;
  int32_t h[3], v[3], bw[3];
  int64_t coef_offset[3];  // within the image's dense int32 region
  int64_t coef_base;       // the region's start in the batch buffer
};

struct DevSeg {
  int32_t img;
  int32_t first_sub, nsub;
  int64_t byte_off;     // unstuffed bytes in the batch stream buffer
  int64_t bits;         // 8 * unstuffed length
  int64_t first_block;  // decode-order index of the segment's first block in its image
  int64_t nblocks;
  int64_t first_mcu, nmcu;
};

__device__ __forceinline__ uint64_t pack_state(int64_t pos, int slot, int z) {
  return ((uint64_t)pos << 16) | ((uint64_t)slot << 8) | (uint64_t)z;
}
__device__ __forceinline__ void unpack_state(uint64_t s, int64_t& pos, int& slot, int& z) {
  pos = (int64_t)(s >> 16);
  slot = (int)((s >> 8) & 0xFF);
  z = (int)(s & 0xFF);
}

// MSB-first reader over one unstuffed segment (16-byte aligned, zero padded
// to a multiple of 16 bytes in the batch buffer): refills 32 bits at a time
// from aligned words; words past the segment read as zero. The next word is
// loaded one refill ahead, so its latency overlaps the symbols decoded from
// the current ones (a lone thread's decode in the sync rounds is
// latency-bound).
struct DBits {
  const uint32_t* w;  // the segment's words
  int nw;             // words holding data (the rest of the segment's padding reads as zero too)
  int cur;            // index of `nxt` (segments stay below 2^27 bytes: gpu_eligible)
  uint64_t acc;
  uint32_t nxt;
  int nb;
  __device__ __forceinline__ void init(const uint8_t* seg, int64_t nbytes) {
    w = reinterpret_cast<const uint32_t*>(seg);
    nw = (int)((nbytes + 3) >> 2);
  }
  __device__ __forceinline__ uint32_t word(int i) const {
    return i < nw ? __byte_perm(__ldg(w + i), 0, 0x0123) : 0u;
  }
  // after fill(): at least 33 bits buffered (a symbol takes at most 16 + 15)
  __device__ __forceinline__ void fill() {
    if (nb <= 32) {
      acc |= (uint64_t)nxt << (32 - nb);
      nb += 32;
      nxt = word(++cur);
    }
  }
  __device__ __forceinline__ void start(int64_t bit) {
    const int c = (int)(bit >> 5);
    const int off = (int)(bit & 31);
    if (c + 32 < nw) asm volatile("prefetch.global.L1 [%0];" ::"l"(w + c + 32));  // the next line's words
    acc = (((uint64_t)word(c) << 32) | word(c + 1)) << off;
    nb = 64 - off;
    cur = c + 2;
    nxt = word(cur);
  }
  __device__ __forceinline__ uint32_t peek(int k) const { return (uint32_t)(acc >> (64 - k)); }
  __device__ __forceinline__ void skip(int k) {
    acc <<= k;
    nb -= k;
  }
  __device__ __forceinline__ int pos() const { return cur * 32 - nb; }
};

// one Huffman symbol; -1 = no code matches
__device__ __forceinline__ int dsym(DBits& b, const DevHuff& t, int32_t f) {
  if (f & (kFull | kSym)) {
    b.skip(f & 31);
    return (f >> 16) & 0xFF;
  }
  for (int len = 11; len <= 16; ++len) {
    const int32_t code = (int32_t)b.peek(len);
    if (t.maxcode[len] >= 0 && code <= t.maxcode[len]) {
      b.skip(len);
      return t.values[t.valptr[len] + code - t.mincode[len]];
    }
  }
  return -1;
}

__device__ __forceinline__ int32_t dextend(uint32_t v, int size) {
  return v < (1u << (size - 1)) ? (int32_t)v - (1 << size) + 1 : (int32_t)v;
}

enum { kModeSync = 0, kModeCount = 1, kModeWrite = 2 };

// Checkpoints of the speculative decode: its state (and the blocks it started
// so far) at the first symbol boundary at or past each mark start + k*kCpBits
// of its own subsequence. A later decode of the same subsequence that reaches
// a mark in exactly a recorded state has merged with the speculative
// trajectory -- the decoder state is (bit position, slot, coefficient index)
// and nothing else -- so its exit state and block count follow from the
// speculative ones without decoding further. k = 0 is the subsequence entry:
// a synchronised subsequence costs one compare in the rounds.
constexpr int kCpBits = FV_JPEG_CP_BITS;
constexpr int kCp = kSubBits / kCpBits;
constexpr uint64_t kNoState = ~0ull;  // an unrecorded checkpoint (never equals a real state)
enum { kCpNone = 0, kCpRecord = 1, kCpMatch = 2 };

// What a subsequence contributes to the scan: the blocks that start in it
// and the sums of their DC differences per scan entry. (In write mode the d
// fields carry the running DC predictions instead.)
struct Tally {
  int32_t n = 0, d0 = 0, d1 = 0, d2 = 0;
  __device__ __forceinline__ int32_t add_dc(int e, int32_t diff) {
    d0 += e == 0 ? diff : 0;
    d1 += e == 1 ? diff : 0;
    d2 += e == 2 ? diff : 0;
    return e == 0 ? d0 : (e == 1 ? d1 : d2);
  }
  __device__ __forceinline__ int4 v() const { return make_int4(n, d0, d1, d2); }
  __device__ __forceinline__ void add(int4 a, int4 b) {  // += a - b
    n += a.x - b.x;
    d0 += a.y - b.y;
    d1 += a.z - b.z;
    d2 += a.w - b.w;
  }
};

// The speculative pass's records for subsequence t, of two trajectories
// through t's bits: 0 = t's own decode, 1 = the warm-up decode of thread t+1
// (which starts at t's first bit with a guessed context, so it is an
// independent second chance to be in step). A round decode of t that meets
// either at a checkpoint is done: exit state and tally follow from that
// trajectory's records. Meeting trajectory 1 also ends a propagation chain
// at once: its exit state is where t+1's own decode started.
struct SpecRec {
  uint64_t* st[2];    // [kCp][nsub] states at the checkpoints (kNoState: none)
  int4* tal[2];       // [kCp][nsub] tallies from the range's start to the checkpoint
  uint64_t* exit[2];  // [nsub] states at the range's end
  int4* tot[2];       // [nsub] tallies over the range
};
constexpr bool kDual = kWarmBits == kSubBits;  // the warm-up covers exactly the preceding subsequence

struct Ckpt {
  uint64_t* st0;   // record: the trajectory's states; match: trajectory 0's
  uint64_t* st1;   // match: trajectory 1's states
  int4* tal;       // record: the trajectory's tallies
  int64_t nsub, t;
  int64_t mark;    // next mark (bit position)
  int k;           // next checkpoint index
  int hit;         // match mode: the checkpoint matched, or -1
  int traj;        // match mode: the trajectory matched
};

// Write mode's block addressing: the MCU position (mx, my) of the current
// block is derived once from its decode-order index (block indices of an
// image stay below 2^31: 65535^2 / 64 * 3) and then stepped as the decoder
// wraps its slot; a block's coefficients start at
//   coef_base + slot_off[slot] + my * mcu_row[e] + mx * mcu_col[e].
struct BlockPos {
  uint32_t mx, my, mcus_x;
  int64_t first, limit;  // the segment's blocks (decode order)
  int16_t* base;         // the image's coefficient region
  // (register copies: the block stores to global memory would otherwise make
  // the compiler reload the segment / image fields after each block)
  __device__ __forceinline__ void init(const DevImg& im, const DevSeg& sg, int64_t cb, int16_t* coef) {
    mcus_x = (uint32_t)im.mcus_x;
    first = sg.first_block;
    limit = sg.first_block + sg.nblocks;
    base = coef + im.coef_base;
    const uint32_t mcu = (uint32_t)cb / (uint32_t)im.nslots;
    my = mcu / mcus_x;
    mx = mcu - my * mcus_x;
  }
  __device__ __forceinline__ void next_mcu() {
    if (++mx == mcus_x) {
      mx = 0;
      ++my;
    }
  }
  // block `cb` in slot `slot`, or nullptr outside the segment (a
  // desynchronised decode can run past it)
  __device__ __forceinline__ int16_t* dst(const DevImg& im, int64_t cb, int slot, int e) const {
    if (cb < first || cb >= limit) return nullptr;
    return base + __ldg(&im.slot_off[slot]) + (int64_t)my * __ldg(&im.mcu_row[e]) + (int64_t)mx * __ldg(&im.mcu_col[e]);
  }
};

// Decode symbols starting before `end_bit` (write mode on the segment's last
// subsequence: until the segment's last block is complete). Anomalies on the
// true path (write mode, blocks of the segment) set *bad; elsewhere the
// decoder steps on deterministically (skip a bit / end the block).
// Write mode: each block is written whole -- zeros included, so the
// coefficient buffer needs no clearing -- by the thread whose range it
// STARTS in: that thread decodes on past its end bit to finish its last
// block, and a thread entering mid-block decodes the remainder without
// writing. The block is assembled in the thread's shared-memory buffer `sb`
// (64 int16, zero on entry and on exit) in natural order through `zz` (the
// zigzag table, shared memory) and leaves as eight 16-byte stores.
template <int MODE, int CPM = kCpNone>
__device__ uint64_t decode_run(const DevHuff* tabs, const DevImg& im, DBits& b, int slot, int z, int64_t end_bit, bool last_sub,
                               int64_t blk, const DevSeg& sg, int16_t* coef, Tally* tal, int* bad,
                               Ckpt* ck = nullptr, const uint8_t* zz = nullptr, int16_t* sb = nullptr) {
  const int64_t limit = sg.first_block + sg.nblocks, seg_bits = sg.bits;
  const uint32_t slot_e = im.slot_e2;  // 2 bits per slot
  const int nslots = im.nslots;
  int16_t* dst = nullptr;  // the current block's destination when this thread writes it
  const DevHuff* tac = tabs + im.ac_t[(slot_e >> (2 * slot)) & 3];  // the current block's AC table
  BlockPos bp;
  if (MODE == kModeWrite) bp.init(im, sg, z != 0 ? blk - 1 : blk, coef);
  // sync modes: the next position at which something happens (the range's
  // end or the next checkpoint mark) -- one compare per symbol
  const int end32 = (int)end_bit;
  int ev = end32;
  if (CPM != kCpNone) ev = ck->k < kCp ? min(end32, (int)ck->mark) : end32;
  for (;;) {
    const int pos = b.pos();
    if (MODE == kModeWrite && last_sub) {
      if (blk >= limit && z == 0) break;              // the segment's blocks are done
      if (pos > seg_bits + 64 * 16) { *bad = 1; break; }  // decoding deep into padding: corrupt
    } else if (MODE == kModeWrite) {
      if (pos >= end32 && z == 0) break;  // past the range and between blocks
    } else if (pos >= ev) {
      if (pos >= end32) break;
    }
    if (CPM != kCpNone && pos >= ev) {  // (not the end: a checkpoint mark)
      const uint64_t st = pack_state(pos, slot, z);
      if (CPM == kCpMatch) {
        const int64_t idx = ck->k * ck->nsub + ck->t;
        if (ck->st0[idx] == st || ck->st1[idx] == st) {
          ck->hit = ck->k;
          ck->traj = ck->st0[idx] == st ? 0 : 1;
          break;
        }
      }
      do {  // every mark this boundary is the first at or past
        if (CPM == kCpRecord) {
          ck->st0[ck->k * ck->nsub + ck->t] = st;
          ck->tal[ck->k * ck->nsub + ck->t] = tal->v();
        }
        ++ck->k;
        ck->mark += kCpBits;
      } while (ck->k < kCp && pos >= ck->mark);
      ev = ck->k < kCp ? min(end32, (int)ck->mark) : end32;
    }
    b.fill();
    const int e = (slot_e >> (2 * slot)) & 3;
    if (z == 0) {  // DC of a new block
      if (MODE != kModeWrite && tal) ++tal->n;
      if (MODE == kModeWrite) dst = bp.dst(im, blk++, slot, e);
      const DevHuff& t = tabs[im.dc_t[e]];
      tac = tabs + im.ac_t[e];
      const int32_t f = t.fast[b.peek(10)];
      int32_t diff;
      if (f & kFull) {
        b.skip(f & 31);
        diff = f >> 16;
      } else {
        const int size = dsym(b, t, f);
        if (size < 0 || size > 11) {
          if (MODE == kModeWrite && dst) *bad = 1;
          if (size < 0) b.skip(1);
          diff = 0;
        } else if (size) {
          diff = dextend(b.peek(size), size);
          b.skip(size);
        } else {
          diff = 0;
        }
      }
      if (MODE == kModeWrite) {
        if (dst) {  // the DC prediction: the running sum from the segment's prefix (k_scan)
          const int32_t dc = tal->add_dc(e, diff);
          if (dc < -32768 || dc > 32767) *bad = 1;  // beyond int16 (crafted streams): host decoder
          sb[0] = (int16_t)dc;
        }
      } else if (tal) {
        tal->add_dc(e, diff);
      }
      z = 1;
    } else {
      const DevHuff& t = *tac;
      const int32_t f = t.fast[b.peek(10)];
      if (f & kFull) {  // a coefficient (run + value in one lookup) or an EOB: one branch-free path
        b.skip(f & 31);
        const int zr = z + ((f >> 8) & 15);
        const bool eob = (f & kEob) != 0;
        const bool past = !eob && zr > 63;  // AC run past the block
        if (MODE == kModeWrite && dst) {
          if (past) *bad = 1;
          if (!eob && !past) sb[zz[zr]] = (int16_t)(f >> 16);
        }
        z = (eob || past) ? 64 : zr + 1;
      } else {
        const int rs = dsym(b, t, f);
        if (rs < 0) {
          if (MODE == kModeWrite && dst) *bad = 1;
          b.skip(1);
          z = 64;
        } else {
          const int sz = rs & 15;
          if (sz == 0) {
            z = rs == 0xF0 ? z + 16 : 64;
          } else {
            z += rs >> 4;
            if (z > 63) {
              if (MODE == kModeWrite && dst) *bad = 1;
              z = 64;
            } else {
              const int32_t v = dextend(b.peek(sz), sz);
              b.skip(sz);
              if (MODE == kModeWrite && dst) sb[zz[z]] = (int16_t)v;  // |v| < 2^15
              ++z;
            }
          }
        }
      }
    }
    if (z >= 64) {  // block complete
      z = 0;
      slot = slot + 1 == nslots ? 0 : slot + 1;
      if (MODE == kModeWrite) {
        if (dst) {  // the finished block leaves whole; the buffer is cleared for the next one
          uint4* sv = reinterpret_cast<uint4*>(sb);
          uint4* dv = reinterpret_cast<uint4*>(dst);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            dv[k] = sv[k];
            sv[k] = make_uint4(0, 0, 0, 0);
          }
          dst = nullptr;
        }
        if (slot == 0) bp.next_mcu();
        if (blk == limit && b.pos() > seg_bits) *bad = 1;  // consumed padding
      }
    }
  }
  return pack_state(b.pos(), slot, z);
}


// ---------------------------------------------------------------------------
// passes (one thread per subsequence)
// ---------------------------------------------------------------------------

struct Pass {
  const DevHuff* huff;  // the batch's distinct Huffman tables
  const DevImg* imgs;
  const DevSeg* segs;
  const int32_t* sub_seg;
  const uint8_t* stream;
  int64_t nsub;
};

__device__ __forceinline__ void sub_range(const Pass& P, int64_t t, const DevSeg*& sg, int64_t& local, int64_t& start,
                                          int64_t& end) {
  sg = &P.segs[P.sub_seg[t]];
  local = t - sg->first_sub;
  start = local * kSubBits;
  end = min(start + (int64_t)kSubBits, sg->bits);
}

__global__ void __launch_bounds__(128) k_spec(const __grid_constant__ Pass P, uint64_t* E, int4* tally,
                                              const __grid_constant__ SpecRec R) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.nsub) return;
  const DevSeg* sg;
  int64_t local, start, end;
  sub_range(P, t, sg, local, start, end);
  DBits b;
  b.init(P.stream + sg->byte_off, sg->bits >> 3);
  int slot = 0, z = 0;
  int64_t pos = start;
  if (local + 1 == sg->nsub)  // no thread warms up over this subsequence: no trajectory 1
    for (int k = 0; k < kCp; ++k) R.st[1][k * P.nsub + t] = kNoState;
  if (kWarmBits > 0 && local > 0) {  // warm up on the preceding bits: enter this subsequence (likely) in step
    const int64_t w0 = start > (int64_t)kWarmBits ? start - (int64_t)kWarmBits : 0;
    b.start(w0);
    Tally wt;
    Ckpt wk{R.st[1], nullptr, R.tal[1], P.nsub, t - 1, w0, 0, -1, 0};  // trajectory 1 of subsequence t-1
    const uint64_t e = kDual ? decode_run<kModeSync, kCpRecord>(P.huff, P.imgs[sg->img], b, 0, 0, start, false, 0, *sg,
                                                                nullptr, &wt, nullptr, &wk)
                             : decode_run<kModeSync>(P.huff, P.imgs[sg->img], b, 0, 0, start, false, 0, *sg, nullptr,
                                                     nullptr, nullptr);
    for (int k = kDual ? wk.k : 0; k < kCp; ++k) R.st[1][k * P.nsub + t - 1] = kNoState;
    R.exit[1][t - 1] = e;
    R.tot[1][t - 1] = wt.v();
    unpack_state(e, pos, slot, z);
  }
  b.start(pos);
  Tally tl;
  Ckpt ck{R.st[0], nullptr, R.tal[0], P.nsub, t, start, 0, -1, 0};
  const uint64_t e =
      decode_run<kModeSync, kCpRecord>(P.huff, P.imgs[sg->img], b, slot, z, end, false, 0, *sg, nullptr, &tl, nullptr, &ck);
  for (int k = ck.k; k < kCp; ++k) R.st[0][k * P.nsub + t] = kNoState;
  E[t] = e;
  R.exit[0][t] = e;
  tally[t] = tl.v();  // exact for each segment's first subsequence; the others are re-derived in the rounds
  R.tot[0][t] = tl.v();
}

// One propagation round over a work queue: for each queued subsequence t,
// E[t] = decode(E[t-1]). E is updated in place (64-bit stores are atomic, and
// reading a predecessor's old or new state is a valid iteration step). The
// invariant that makes the final state the fixed point: EVERY change of E[t]
// queues t+1 for the next round (deduplicated by a per-subsequence round
// mark), so t+1 is re-derived from E[t]'s final value; rounds run until one
// changes nothing. As an accelerator, a thread that changed E[t] also carries
// the new state on through up to kChain following subsequences itself (a
// desynchronised stretch would otherwise advance one subsequence per round).
// all_subs: the first round takes every subsequence (implicit queue).
__device__ __forceinline__ void enqueue(int32_t* qout, int* nout, int* mark, int64_t t, int round) {
  if (atomicExch(&mark[t], round) != round) qout[atomicAdd(nout, 1)] = (int32_t)t;
}

__global__ void __launch_bounds__(128) k_round(const __grid_constant__ Pass P, uint64_t* E, int4* tally,
                                               const int32_t* qin, const int* nin, int32_t* qout, int* nout, int* mark,
                                               int round, int all_subs, int chain, const __grid_constant__ SpecRec R) {
  const int64_t n = all_subs ? P.nsub : *nin;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = all_subs ? i : qin[i];
    const DevSeg* sg;
    int64_t local, start, end;
    sub_range(P, t, sg, local, start, end);
    if (local == 0) continue;
    uint64_t in = E[t - 1];
    for (int step = 0;; ++step) {
      uint64_t e;
      Tally tl;
      if (in == R.st[0][t]) {  // entered in the speculative decode's own entry state
        e = R.exit[0][t];
        tl.add(R.tot[0][t], make_int4(0, 0, 0, 0));
      } else {
        int64_t pos;
        int slot, z;
        unpack_state(in, pos, slot, z);
        DBits b;
        b.init(P.stream + sg->byte_off, sg->bits >> 3);
        b.start(pos);
        Ckpt ck{R.st[0], R.st[1], nullptr, P.nsub, t, start, 0, -1, 0};
        e = decode_run<kModeSync, kCpMatch>(P.huff, P.imgs[sg->img], b, slot, z, end, false, 0, *sg, nullptr, &tl, nullptr,
                                            &ck);
        if (ck.hit >= 0) {  // merged with a speculative trajectory: its exit, the rest of its tally
          e = R.exit[ck.traj][t];
          tl.add(R.tot[ck.traj][t], R.tal[ck.traj][ck.hit * P.nsub + t]);
        }
      }
      // this subsequence's tally: the LAST processing of t used its
      // predecessor's final state (see the invariant above), so at the fixed
      // point these are the true ones -- no separate count pass
      tally[t] = tl.v();
      if (e == E[t]) break;
      E[t] = e;
      if (local + 1 >= sg->nsub) break;
      enqueue(qout, nout, mark, t + 1, round);  // re-derive t+1 next round, whatever happens below
      if (step + 1 == chain) break;
      in = e;
      ++t;
      ++local;
      start = local * kSubBits;
      end = min(start + (int64_t)kSubBits, sg->bits);
    }
  }
}

// After the rounds: any subsequence whose state still disagrees with its
// predecessor's decode marks its image (not converged -> host decoder).
__global__ void __launch_bounds__(128) k_verify(const __grid_constant__ Pass P, const uint64_t* E, const int32_t* q,
                                                const int* nq, int* img_bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < *nq; i += (int64_t)gridDim.x * blockDim.x)
    img_bad[P.segs[P.sub_seg[q[i]]].img] = 1;
}

__device__ __forceinline__ void entry_state(const Pass& P, const uint64_t* E, int64_t t, int64_t local, int64_t start,
                                            int64_t& pos, int& slot, int& z) {
  if (local == 0) {
    pos = start;
    slot = 0;
    z = 0;
  } else {
    unpack_state(E[t - 1], pos, slot, z);
  }
}

// exclusive scan of the tallies of each segment's subsequences: the first
// block of every subsequence and the DC predictions it starts from
__global__ void __launch_bounds__(256) k_scan(const DevSeg* segs, int32_t nseg, const int4* tally, int64_t* base,
                                              int4* dcb) {
  __shared__ int64_t warp_n[8];
  __shared__ int32_t warp_d[3][8];
  const int sgi = blockIdx.x;
  if (sgi >= nseg) return;
  const DevSeg& sg = segs[sgi];
  int64_t carry = sg.first_block;
  int32_t c0d = 0, c1d = 0, c2d = 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t c0 = 0; c0 < sg.nsub; c0 += 256) {
    const int64_t i = c0 + threadIdx.x;
    const int4 v = i < sg.nsub ? tally[sg.first_sub + i] : make_int4(0, 0, 0, 0);
    int64_t x = v.x;
    int32_t y0 = v.y, y1 = v.z, y2 = v.w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t a = __shfl_up_sync(0xffffffffu, x, o);
      const int32_t b0 = __shfl_up_sync(0xffffffffu, y0, o), b1 = __shfl_up_sync(0xffffffffu, y1, o),
                    b2 = __shfl_up_sync(0xffffffffu, y2, o);
      if (lane >= o) {
        x += a;
        y0 += b0;
        y1 += b1;
        y2 += b2;
      }
    }
    if (lane == 31) {
      warp_n[w] = x;
      warp_d[0][w] = y0;
      warp_d[1][w] = y1;
      warp_d[2][w] = y2;
    }
    __syncthreads();
    int64_t pre = 0, tot = 0;
    int32_t p0 = 0, p1 = 0, p2 = 0, t0 = 0, t1 = 0, t2 = 0;
    for (int k = 0; k < 8; ++k) {
      if (k < w) {
        pre += warp_n[k];
        p0 += warp_d[0][k];
        p1 += warp_d[1][k];
        p2 += warp_d[2][k];
      }
      tot += warp_n[k];
      t0 += warp_d[0][k];
      t1 += warp_d[1][k];
      t2 += warp_d[2][k];
    }
    if (i < sg.nsub) {
      base[sg.first_sub + i] = carry + pre + x - v.x;
      dcb[sg.first_sub + i] = make_int4(0, c0d + p0 + y0 - v.y, c1d + p1 + y1 - v.z, c2d + p2 + y2 - v.w);
    }
    carry += tot;
    c0d += t0;
    c1d += t1;
    c2d += t2;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(128) k_write(const __grid_constant__ Pass P, const uint64_t* E, const int64_t* base,
                                               const int4* dcb, int16_t* coef, int* img_bad) {
  __shared__ uint8_t zz[64];
  // per-thread block buffers, 144-byte stride: a warp's 16-byte accesses to
  // them spread over all banks
  __shared__ __align__(16) int16_t bufs[128][72];
  if (threadIdx.x < 64) zz[threadIdx.x] = (uint8_t)kZigzagDev[threadIdx.x];
  uint4* mine = reinterpret_cast<uint4*>(bufs[threadIdx.x]);
#pragma unroll
  for (int k = 0; k < 8; ++k) mine[k] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.nsub) return;
  const DevSeg* sg;
  int64_t local, start, end, pos;
  int slot, z, bad = 0;
  sub_range(P, t, sg, local, start, end);
  entry_state(P, E, t, local, start, pos, slot, z);
  DBits b;
  b.init(P.stream + sg->byte_off, sg->bits >> 3);
  b.start(pos);
  const int4 d = dcb[t];
  Tally run;
  run.d0 = d.y;
  run.d1 = d.z;
  run.d2 = d.w;
  decode_run<kModeWrite>(P.huff, P.imgs[sg->img], b, slot, z, end, local == sg->nsub - 1, base[t], *sg, coef, &run, &bad,
                         nullptr, zz, bufs[threadIdx.x]);
  if (bad) img_bad[sg->img] = 1;
}

// ---------------------------------------------------------------------------
// host planning
// ---------------------------------------------------------------------------

inline void to_dev_huff(const Huff& h, DevHuff& d, bool dc) {
  memcpy(d.fast, h.fast, sizeof(d.fast));
  if (!dc)
    for (int x = 0; x < (1 << 10); ++x)
      if ((d.fast[x] & kSym) && ((d.fast[x] >> 16) & 0xFF) == 0x00) d.fast[x] = kFull | kEob | (d.fast[x] & 31);
  for (int l = 0; l < 17; ++l) {
    d.maxcode[l] = h.maxcode[l];
    d.mincode[l] = h.mincode[l];
    d.valptr[l] = h.valptr[l];
  }
  d.maxcode[17] = -1;
  memcpy(d.values, h.values, 256);
}

struct Plan {
  std::unique_ptr<Stream> s;
  int rc = FV_OK;
  bool gpu = false;
  int64_t nseg = 0, nsub = 0, bytes = 0, coefs = 0;
  uint64_t hkey[6] = {};  // Huffman table hashes: DC, AC per scan entry
  int32_t tab[6] = {};    // their indices among the batch's distinct tables
};

// Huffman tables are deduplicated across a batch (most encoders emit the
// standard tables): one copy per distinct table keeps the decoders' table
// lookups in L1. A table is defined by its codes and symbols (mincode,
// maxcode, valptr, values) and its class (the fast entries differ for DC).
inline uint64_t huff_key(const Huff& h, bool dc) {
  uint64_t x = dc ? 0x9E3779B97F4A7C15ull : 0xC2B2AE3D27D4EB4Full;
  auto mix = [&](const void* p, size_t n) {
    const uint8_t* c = static_cast<const uint8_t*>(p);
    for (size_t i = 0; i < n; ++i) x = (x ^ c[i]) * 0x100000001B3ull;
  };
  mix(h.mincode, sizeof(h.mincode));
  mix(h.maxcode, sizeof(h.maxcode));
  mix(h.valptr, sizeof(h.valptr));
  mix(h.values, 256);
  return x;
}
inline bool huff_same(const Huff& a, const Huff& b) {
  return memcmp(a.mincode, b.mincode, sizeof(a.mincode)) == 0 && memcmp(a.maxcode, b.maxcode, sizeof(a.maxcode)) == 0 &&
         memcmp(a.valptr, b.valptr, sizeof(a.valptr)) == 0 && memcmp(a.values, b.values, 256) == 0;
}

// Can the GPU path decode this stream exactly? (else: the host decoder)
inline bool gpu_eligible(const Stream& s, const FvJpegInfo& f) {
  int seen = 0;
  for (int e = 0; e < s.nscan; ++e) {
    const int k = s.scan_comp[e];
    if (seen & (1 << k)) return false;  // a component named twice by the scan
    seen |= 1 << k;
    const Comp& c = s.sof[k];
    int nv = 0;
    for (int l = 1; l <= 16; ++l) nv += s.dc[c.td].maxcode[l] >= 0 ? s.dc[c.td].maxcode[l] - s.dc[c.td].mincode[l] + 1 : 0;
    if (nv > 256) return false;
    nv = 0;
    for (int l = 1; l <= 16; ++l) nv += s.ac[c.ta].maxcode[l] >= 0 ? s.ac[c.ta].maxcode[l] - s.ac[c.ta].mincode[l] + 1 : 0;
    if (nv > 256) return false;
    // DC values of a segment stay within int32 (|diff| <= 2047 per block)
    const int64_t per_seg = (int64_t)(s.dri ? s.dri : (int64_t)s.mcus_x * s.mcus_y) * c.h * c.v;
    if (per_seg * 2047 >= (1ll << 31)) return false;
  }
  for (int64_t k = 0; k < (int64_t)s.seg_len.size(); ++k)
    if (s.seg_len[k] >= (int64_t(1) << 27)) return false;  // the bit reader's positions are 32-bit
  int64_t per_mcu = 0;
  for (int e = 0; e < s.nscan; ++e) per_mcu += s.sof[s.scan_comp[e]].h * s.sof[s.scan_comp[e]].v;
  if (per_mcu > kMaxSlots) return false;
  return f.coef_count > 0;
}

// Pinned host staging for the uploads and its device copy, kept across
// calls (one caller at a time: the lock is held from the plan until the batch
// is freed, and a call synchronises after the last pass that reads the device
// copy, so both are free again when the next call takes the lock). The upload
// runs on a per-device copy stream, so it can overlap whatever the caller's
// stream is still executing (e.g. the previous batch's reconstruction).
struct PinnedStage {
  static constexpr int kMaxDev = 64;
  struct Dev {
    uint8_t* p = nullptr;
    size_t cap = 0;
    cudaStream_t copy = nullptr;
    cudaEvent_t done = nullptr;
  };
  std::mutex lock;
  uint8_t* p = nullptr;
  size_t cap = 0;
  Dev dev[kMaxDev];
  uint8_t* get(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFreeHost(p);
      cap = std::max(bytes, cap * 2);
      if (cudaHostAlloc(reinterpret_cast<void**>(&p), cap, cudaHostAllocDefault) != cudaSuccess) {
        p = nullptr;
        cap = 0;
      }
    }
    return p;
  }
  // the current device's copy (grown to `bytes`), or nullptr
  Dev* device(size_t bytes) {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDev) return nullptr;
    Dev& x = dev[d];
    if (!x.copy && cudaStreamCreateWithFlags(&x.copy, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    if (!x.done && cudaEventCreateWithFlags(&x.done, cudaEventDisableTiming) != cudaSuccess) return nullptr;
    if (bytes > x.cap) {
      if (x.p) cudaFree(x.p);
      x.cap = std::max(bytes, x.cap * 2);
      if (cudaMalloc(reinterpret_cast<void**>(&x.p), x.cap) != cudaSuccess) {
        x.p = nullptr;
        x.cap = 0;
        return nullptr;
      }
    }
    return &x;
  }
};
inline PinnedStage& pinned_stage() {
  static PinnedStage s;
  return s;
}

// The scratch comes from the device's default stream-ordered pool; by
// default the pool returns freed memory to the OS at every synchronisation,
// which would re-map ~1 GB per batch. Keep it (once per device).
inline void keep_pool_memory() {
  static std::mutex m;
  static unsigned long long done[2] = {0, 0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 128) return;
  std::lock_guard<std::mutex> g(m);
  if (done[dev >> 6] & (1ull << (dev & 63))) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev >> 6] |= 1ull << (dev & 63);
}

// Stream-ordered scratch, returned to the pool (on the allocating stream)
// when it goes out of scope.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t st = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  int alloc(size_t count, cudaStream_t stream) {
    release();
    n = count;
    st = stream;
    return cudaMallocAsync(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(T), st) == cudaSuccess
               ? FV_OK
               : set_error(FV_ECUDA, "fv_jpeg_decode_batch_gpu: device allocation of %zu bytes", count * sizeof(T));
  }
  void release() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
  }
};

}  // namespace jpg
}  // namespace fv

using namespace fv;
using namespace fv::jpg;

namespace {
struct PhaseTimer {  // FV_JPEG_TIMING=1: host phase times (and GPU phase times) to stderr
  bool on = getenv("FV_JPEG_TIMING") != nullptr;
  std::vector<std::pair<const char*, cudaEvent_t>> ev;
  void gpu(const char* what, cudaStream_t st) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    ev.emplace_back(what, e);
  }
  void gpu_report() {
    if (!on || ev.size() < 2) return;
    cudaEventSynchronize(ev.back().second);
    for (size_t k = 1; k < ev.size(); ++k) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[k - 1].second, ev[k].second);
      fprintf(stderr, "[fv_jpeg_gpu]   gpu %-22s %8.3f ms\n", ev[k].first, ms);
    }
    for (auto& x : ev) cudaEventDestroy(x.second);
    ev.clear();
  }
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[fv_jpeg_gpu] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
    t0 = t;
  }
};
}  // namespace

// A planned batch: parsed streams, the GPU path's host staging (images,
// segments, unstuffed bytes in pinned memory, whose lock it holds) and the
// offsets; run_gpu() uploads and decodes it. Between plan and run the
// caller allocates the outputs from the parsed headers.
struct GpuBatch {
  int32_t n = 0;
  int nt = 1;
  std::vector<Plan> plan;
  std::vector<int64_t> seg_off, sub_off, byte_off, coef_off, img_idx;
  int64_t nseg = 0, nsub = 0, nbytes = 0, ncoef = 0;
  int32_t nimg = 0;
  std::unique_lock<std::mutex> stage_lock;
  uint8_t* stage_base = nullptr;
  size_t o_huff = 0, o_img = 0, o_seg = 0, o_sub = 0, o_bytes = 0, stage_bytes = 0;  // one contiguous upload
  DevImg* himg = nullptr;
  DevSeg* hseg = nullptr;
  int32_t* hsub = nullptr;
  uint8_t* hbytes = nullptr;
  PhaseTimer timer;

  template <class F>
  void parallel(F&& fn) {
    WorkPool::get().run(n, nt, std::forward<F>(fn));
  }

  int make(const uint8_t* const* data, const int64_t* lens, FvJpegInfo* infos, int32_t* status) {
  // 1. parse, eligibility, sizes
  plan.resize(n);
  parallel([&](int32_t i) {
    Plan& p = plan[i];
    p.s.reset(new Stream());
    p.rc = parse(data[i], lens[i], *p.s);
    if (p.rc) return;
    FvJpegInfo f;
    fill_info(*p.s, f);
    p.gpu = gpu_eligible(*p.s, f);
    if (!p.gpu) return;
    const Stream& s = *p.s;
    const int64_t total = (int64_t)s.mcus_x * s.mcus_y;
    p.nseg = s.dri ? (total + s.dri - 1) / s.dri : 1;
    for (int64_t k = 0; k < p.nseg; ++k) {
      p.bytes += (s.seg_len[k] + 15) / 16 * 16;
      p.nsub += std::max<int64_t>(1, (8 * s.seg_len[k] + kSubBits - 1) / kSubBits);
    }
    p.coefs = f.coef_count;
    for (int e = 0; e < s.nscan; ++e) {
      const Comp& c = s.sof[s.scan_comp[e]];
      p.hkey[2 * e] = huff_key(s.dc[c.td], true);
      p.hkey[2 * e + 1] = huff_key(s.ac[c.ta], false);
    }
  });
  timer.mark("parse + plan");
  // 2. offsets
  seg_off.assign(n, 0);
  sub_off.assign(n, 0);
  byte_off.assign(n, 0);
  coef_off.assign(n, 0);
  img_idx.assign(n, -1);
  for (int32_t i = 0; i < n; ++i) {
    status[i] = plan[i].rc;
    if (plan[i].rc == FV_OK) fill_info(*plan[i].s, infos[i]);
    if (!plan[i].gpu) continue;
    img_idx[i] = nimg++;
    seg_off[i] = nseg;
    sub_off[i] = nsub;
    byte_off[i] = nbytes;
    coef_off[i] = ncoef;
    nseg += plan[i].nseg;
    nsub += plan[i].nsub;
    nbytes += (plan[i].bytes + 15) / 16 * 16;
    ncoef += plan[i].coefs;
  }
  if (nimg == 0) return FV_OK;
  // distinct Huffman tables
  struct Uniq {
    uint64_t key;
    const Huff* h;
    bool dc;
  };
  std::vector<Uniq> uniq;
  for (int32_t i = 0; i < n; ++i) {
    if (!plan[i].gpu) continue;
    const Stream& s = *plan[i].s;
    for (int e = 0; e < s.nscan; ++e)
      for (int cls = 0; cls < 2; ++cls) {
        const Comp& c = s.sof[s.scan_comp[e]];
        const Huff& h = cls ? s.ac[c.ta] : s.dc[c.td];
        const uint64_t key = plan[i].hkey[2 * e + cls];
        size_t u = 0;
        while (u < uniq.size() && !(uniq[u].key == key && huff_same(*uniq[u].h, h))) ++u;
        if (u == uniq.size()) uniq.push_back({key, &h, cls == 0});
        plan[i].tab[2 * e + cls] = (int32_t)u;
      }
  }
  // 3. host staging: tables, images, segments, subsequence -> segment, unstuffed bytes
  PinnedStage& stage = pinned_stage();
  stage_lock = std::unique_lock<std::mutex>(stage.lock);  // held until the batch is freed
  o_huff = 0;
  o_img = o_huff + ((uniq.size() * sizeof(DevHuff) + 255) & ~size_t(255));
  o_seg = o_img + ((nimg * sizeof(DevImg) + 255) & ~size_t(255));
  o_sub = o_seg + ((nseg * sizeof(DevSeg) + 255) & ~size_t(255));
  o_bytes = o_sub + ((nsub * sizeof(int32_t) + 255) & ~size_t(255));
  stage_bytes = o_bytes + nbytes + 16;
  uint8_t* sbase = stage.get(stage_bytes);
  if (!sbase) return set_error(FV_ECUDA, "fv_jpeg_batch_plan: pinned staging of %zu bytes", stage_bytes);
  stage_base = sbase;
  {
    DevHuff* hh = reinterpret_cast<DevHuff*>(sbase + o_huff);
    std::unique_ptr<DevHuff> tmp(new DevHuff());
    for (size_t u = 0; u < uniq.size(); ++u) {  // class: the first use's (the key includes it)
      memset(tmp.get(), 0, sizeof(DevHuff));
      to_dev_huff(*uniq[u].h, *tmp, uniq[u].dc);
      memcpy(&hh[u], tmp.get(), sizeof(DevHuff));
    }
    flush_lines(hh, uniq.size() * sizeof(DevHuff));
  }
  himg = reinterpret_cast<DevImg*>(sbase + o_img);
  hseg = reinterpret_cast<DevSeg*>(sbase + o_seg);
  hsub = reinterpret_cast<int32_t*>(sbase + o_sub);
  hbytes = sbase + o_bytes;
    timer.mark("tables + staging layout");
    return FV_OK;
  }

  // image i's staging: its DevImg, segments, subsequence map and unstuffed
  // bytes (worker threads; the upload of finished images runs meanwhile)
  void stage_image(int32_t i) {
    if (!plan[i].gpu) return;
    const Stream& s = *plan[i].s;
    FvJpegInfo f;
    fill_info(s, f);
    // built locally, then written to the staging in one go (the staging is
    // written sequentially and never read back by the host)
    std::unique_ptr<DevImg> dp(new DevImg());
    DevImg& d = *dp;
    memset(&d, 0, sizeof(d));
    int slot = 0;
    for (int e = 0; e < s.nscan; ++e) {
      const Comp& c = s.sof[s.scan_comp[e]];
      d.dc_t[e] = plan[i].tab[2 * e];
      d.ac_t[e] = plan[i].tab[2 * e + 1];
      d.h[e] = c.h;
      d.v[e] = c.v;
      d.bw[e] = f.bw[e];
      d.coef_offset[e] = f.coef_offset[e];
      for (int by = 0; by < c.v; ++by)
        for (int bx = 0; bx < c.h; ++bx, ++slot) {
          d.slot_e[slot] = (int8_t)e;
          d.slot_e2 |= (uint32_t)e << (2 * slot);
          d.slot_bx[slot] = (int8_t)bx;
          d.slot_by[slot] = (int8_t)by;
        }
    }
    d.nslots = slot;
    d.mcus_x = s.mcus_x;
    for (int k = 0; k < slot; ++k) {
      const int e = d.slot_e[k];
      d.slot_off[k] = d.coef_offset[e] + 64 * ((int64_t)d.slot_by[k] * d.bw[e] + d.slot_bx[k]);
    }
    for (int e = 0; e < s.nscan; ++e) {
      d.mcu_row[e] = 64 * (int64_t)d.v[e] * d.bw[e];
      d.mcu_col[e] = 64 * (int64_t)d.h[e];
    }
    d.coef_base = coef_off[i];
    memcpy(&himg[img_idx[i]], &d, sizeof(d));
    flush_lines(&himg[img_idx[i]], sizeof(d));
    const int64_t total = (int64_t)s.mcus_x * s.mcus_y;
    int64_t bo = byte_off[i], so = sub_off[i];
    for (int64_t k = 0; k < plan[i].nseg; ++k) {
      DevSeg g{};
      g.img = (int32_t)img_idx[i];
      g.byte_off = bo;
      g.bits = 8 * s.seg_len[k];
      g.first_mcu = s.dri ? k * s.dri : 0;
      g.nmcu = s.dri ? std::min<int64_t>(s.dri, total - k * s.dri) : total;
      g.first_block = g.first_mcu * slot;
      g.nblocks = g.nmcu * slot;
      g.first_sub = (int32_t)so;
      g.nsub = (int32_t)std::max<int64_t>(1, (g.bits + kSubBits - 1) / kSubBits);
      hseg[seg_off[i] + k] = g;
      flush_lines(&hseg[seg_off[i] + k], sizeof(g));
      for (int32_t q = 0; q < g.nsub; ++q) hsub[so + q] = (int32_t)(seg_off[i] + k);
      flush_lines(&hsub[so], sizeof(int32_t) * (size_t)g.nsub);
      so += g.nsub;
      // unstuff the segment: copy runs between 0xFF bytes, FF 00 -> FF, drop fill FFs
      uint8_t* out = hbytes + bo;
      for (int64_t r = s.seg_raw[k]; r < s.seg_end[k];) {
        const uint8_t* f = static_cast<const uint8_t*>(memchr(s.data + r, 0xFF, (size_t)(s.seg_end[k] - r)));
        const int64_t run = f ? (f - (s.data + r)) : (s.seg_end[k] - r);
        memcpy(out, s.data + r, (size_t)run);
        out += run;
        r += run;
        if (r >= s.seg_end[k]) break;
        if (s.data[r + 1] == 0x00) {
          *out++ = 0xFF;
          r += 2;
        } else {
          ++r;  // fill byte
        }
      }
      memset(out, 0, (size_t)((s.seg_len[k] + 15) / 16 * 16 - s.seg_len[k]));  // zero padding
      flush_lines(hbytes + bo, (size_t)((s.seg_len[k] + 15) / 16 * 16));
      bo += (s.seg_len[k] + 15) / 16 * 16;  // 16-byte aligned, zero padded (DBits reads whole words)
    }
  }


  int run(uint8_t* planes, const int64_t* plane_off, uint8_t* const* dst, const int64_t* dst_pitch, int32_t* status,
          cudaStream_t st) {
    for (int32_t i = 0; i < n; ++i) status[i] = FV_EFALLBACK;
    if (nimg == 0) return FV_OK;
  // 4. staging + upload: worker threads unstuff the images while this thread
  // uploads each finished run of images (in input order) on the copy stream
  PinnedStage::Dev* ds = pinned_stage().device(stage_bytes);
  if (!ds) return set_error(FV_ECUDA, "fv_jpeg_decode_batch_gpu: device staging of %zu bytes", stage_bytes);
  int rc = FV_OK;
  {
    std::unique_ptr<std::atomic<int32_t>[]> staged(new std::atomic<int32_t>[n]);
    for (int32_t i = 0; i < n; ++i) staged[i].store(0, std::memory_order_relaxed);
    WorkPool& wp = WorkPool::get();
    WorkPool::Job job;
    job.fn = [&](int32_t i) {
      stage_image(i);
      staged[i].store(1, std::memory_order_release);
    };
    job.n = n;
    job.want = std::max(1, std::min(std::min<int>(nt, n), wp.size()));
    wp.start(job);
    size_t lo = o_bytes, hi = o_bytes;  // the pending byte run
    auto flush = [&](bool last) {
      if (hi > lo && (last || hi - lo >= (size_t(2) << 20))) {
        if (cudaMemcpyAsync(ds->p + lo, stage_base + lo, hi - lo, cudaMemcpyHostToDevice, ds->copy) != cudaSuccess)
          rc = rc ? rc : set_error(FV_ECUDA, "fv_jpeg_decode_batch_gpu: upload: %s", cudaGetErrorString(cudaGetLastError()));
        lo = hi;
      }
    };
    for (int32_t i = 0; i < n; ++i) {
      while (!staged[i].load(std::memory_order_acquire)) std::this_thread::yield();
      if (!plan[i].gpu) continue;
      hi = o_bytes + (size_t)byte_off[i] + (size_t)((plan[i].bytes + 15) / 16 * 16);
      flush(false);
    }
    flush(true);
    wp.wait(job);
    // tables, images, segments, subsequence map (written by the workers too)
    if (cudaMemcpyAsync(ds->p, stage_base, o_bytes, cudaMemcpyHostToDevice, ds->copy) != cudaSuccess ||
        cudaEventRecord(ds->done, ds->copy) != cudaSuccess || cudaStreamWaitEvent(st, ds->done, 0) != cudaSuccess)
      rc = rc ? rc : set_error(FV_ECUDA, "fv_jpeg_decode_batch_gpu: upload: %s", cudaGetErrorString(cudaGetLastError()));
  }
  timer.mark("unstuff + upload");
  // 5. device scratch (one stream-ordered allocation) and passes
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const int nrounds = kSyncRounds * kSyncChunks;
  const size_t o_tally = carve(sizeof(int4) * nsub), o_tot0 = carve(sizeof(int4) * nsub),
               o_tot1 = carve(sizeof(int4) * nsub), o_dcb = carve(sizeof(int4) * nsub),
               o_cpt0 = carve(sizeof(int4) * nsub * kCp), o_cpt1 = carve(sizeof(int4) * nsub * kCp),
               o_E0 = carve(sizeof(uint64_t) * nsub), o_Es0 = carve(sizeof(uint64_t) * nsub),
               o_Es1 = carve(sizeof(uint64_t) * nsub), o_cp0 = carve(sizeof(uint64_t) * nsub * kCp),
               o_cp1 = carve(sizeof(uint64_t) * nsub * kCp), o_q0 = carve(sizeof(int32_t) * nsub),
               o_q1 = carve(sizeof(int32_t) * nsub), o_mark = carve(sizeof(int32_t) * nsub),
               o_base = carve(sizeof(int64_t) * nsub), o_flags = carve(sizeof(int32_t) * (nimg + nrounds + 2));
  DevBuf<uint8_t> scratch;
  DevBuf<int16_t> dcoef;
  rc = rc ? rc : scratch.alloc(off, st);
  rc = rc ? rc : dcoef.alloc(ncoef, st);
  auto at = [&](size_t o) { return scratch.p + o; };
  int4* const tally_p = reinterpret_cast<int4*>(at(o_tally));
  int4* const dcb_p = reinterpret_cast<int4*>(at(o_dcb));
  uint64_t* const E0_p = reinterpret_cast<uint64_t*>(at(o_E0));
  int32_t* const q0_p = reinterpret_cast<int32_t*>(at(o_q0));
  int32_t* const q1_p = reinterpret_cast<int32_t*>(at(o_q1));
  int32_t* const mark_p = reinterpret_cast<int32_t*>(at(o_mark));
  int64_t* const base_p = reinterpret_cast<int64_t*>(at(o_base));
  int32_t* const flags_p = reinterpret_cast<int32_t*>(at(o_flags));
  std::vector<int32_t> hflags(nimg, 0);
  if (!rc) {
    timer.gpu("start (after the upload)", st);
    DevImg* const dimg_p = reinterpret_cast<DevImg*>(ds->p + o_img);
    DevSeg* const dseg_p = reinterpret_cast<DevSeg*>(ds->p + o_seg);
    const int32_t* const dsub_p = reinterpret_cast<const int32_t*>(ds->p + o_sub);
    const uint8_t* const dbytes_p = ds->p + o_bytes;
    // img_bad[nimg] = 0, then the per-round queue lengths (all 0); the round marks
    cudaMemsetAsync(flags_p, 0, sizeof(int32_t) * (nimg + nrounds + 2), st);
    cudaMemsetAsync(mark_p, 0, nsub * sizeof(int32_t), st);
    // (no clearing of dcoef: the write pass stores every block whole)
    Pass P{reinterpret_cast<const DevHuff*>(ds->p + o_huff), dimg_p, dseg_p, dsub_p, dbytes_p, nsub};
    const unsigned grid = (unsigned)((nsub + 127) / 128);
    int* img_bad = flags_p;
    int* changed = flags_p + nimg;  // changed[r], r = 0 .. kSyncRounds
    timer.gpu("flags + memsets", st);
    const SpecRec R{{reinterpret_cast<uint64_t*>(at(o_cp0)), reinterpret_cast<uint64_t*>(at(o_cp1))},
                     {reinterpret_cast<int4*>(at(o_cpt0)), reinterpret_cast<int4*>(at(o_cpt1))},
                     {reinterpret_cast<uint64_t*>(at(o_Es0)), reinterpret_cast<uint64_t*>(at(o_Es1))},
                     {reinterpret_cast<int4*>(at(o_tot0)), reinterpret_cast<int4*>(at(o_tot1))}};
    k_spec<<<grid, 128, 0, st>>>(P, E0_p, tally_p, R);
    timer.gpu("speculative pass", st);
    count_launch();
    uint64_t* Ein = E0_p;
    // rounds: the first over every subsequence, then over the queue of those
    // whose predecessor changed; after a chunk of rounds, one 4-byte readback
    // of the queue length decides whether another chunk is needed
    int32_t* qa = q0_p;
    int32_t* qb = q1_p;
    int* cnt = changed;  // cnt[r]: queue length produced by round r
    const unsigned qgrid = (unsigned)std::min<int64_t>((nsub + 127) / 128, 148 * 8);
    int r = 0;
    for (int chunk = 0; chunk < kSyncChunks && !rc; ++chunk) {
      for (int k = 0; k < kSyncRounds; ++k, ++r) {
        k_round<<<r == 0 ? grid : qgrid, 128, 0, st>>>(P, Ein, tally_p, qa, cnt + r, qb, cnt + r + 1, mark_p, r + 1,
                                                       r == 0, r == 0 ? kChain0 : kChain, R);
        if (timer.on) timer.gpu(r == 0 ? "round 0 (all)" : "round k (queue)", st);
        count_launch();
        std::swap(qa, qb);
      }
      int32_t last = 0;
      cudaMemcpyAsync(&last, cnt + r, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
      if (cudaStreamSynchronize(st) != cudaSuccess) {
        rc = set_error(FV_ECUDA, "fv_jpeg_decode_batch_gpu: %s", cudaGetErrorString(cudaGetLastError()));
        break;
      }
      if (last == 0) break;
      if (chunk + 1 == kSyncChunks) {  // still changing: those images go to the host decoder
        k_verify<<<qgrid, 128, 0, st>>>(P, Ein, qa, cnt + r, img_bad);
        count_launch();
      }
    }
    timer.gpu("sync rounds", st);
    timer.mark("speculative + sync rounds");
    if (timer.on) {
      std::vector<int32_t> ch(r + 1);
      cudaMemcpy(ch.data(), changed, (r + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost);
      fprintf(stderr, "[fv_jpeg_gpu] %lld subsequences, changed per round:", (long long)nsub);
      for (int q = 1; q <= r; ++q) fprintf(stderr, " %d", ch[q]);
      fprintf(stderr, "\n");
    }
    k_scan<<<(unsigned)nseg, 256, 0, st>>>(dseg_p, (int32_t)nseg, tally_p, base_p, dcb_p);
    k_write<<<grid, 128, 0, st>>>(P, Ein, base_p, dcb_p, dcoef.p, img_bad);
    timer.gpu("scan + write", st);
    rc = check_launch("fv_jpeg_decode_batch_gpu passes");
    count_launch();
    count_launch();
  }
  timer.mark("scan + write");
  if (!rc) {
    // which images decoded cleanly (a second sync)
    cudaMemcpyAsync(hflags.data(), flags_p, nimg * sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess)
      rc = set_error(FV_ECUDA, "fv_jpeg_decode_batch_gpu: %s", cudaGetErrorString(cudaGetLastError()));
  }
  if (!rc) {  // one batched reconstruction of the cleanly decoded images
    std::vector<FvJpegInfo> fi(n);
    std::vector<const FvJpegInfo*> fs;
    std::vector<const int16_t*> cs;
    std::vector<uint8_t*> ps, ds;
    std::vector<int64_t> dp;
    for (int32_t i = 0; i < n; ++i) {
      if (!plan[i].gpu || hflags[img_idx[i]] || !dst[i]) continue;  // NULL dst: not wanted
      fill_info(*plan[i].s, fi[i]);
      fs.push_back(&fi[i]);
      cs.push_back(dcoef.p + coef_off[i]);
      ps.push_back(planes + plane_off[i]);
      ds.push_back(dst[i]);
      dp.push_back(dst_pitch[i]);
    }
    timer.gpu("flags readback", st);
    rc = reconstruct_batch((int)fs.size(), fs.data(), cs.data(), ps.data(), ds.data(), dp.data(), st);
    timer.gpu("idct + colour", st);
    if (!rc)
      for (int32_t i = 0; i < n; ++i)
        if (plan[i].gpu && !hflags[img_idx[i]] && dst[i]) status[i] = FV_OK;
  }
  timer.mark("flags + reconstruct launch");
  timer.gpu_report();
    return rc;  // the DevBufs return to the pool here
  }
};

extern "C" {

int fv_jpeg_batch_plan(const uint8_t* const* data, const int64_t* lens, int32_t n, FvJpegInfo* infos, int32_t* status,
                       int32_t threads, void** handle) {
  if (!handle || n < 0 || (n > 0 && (!data || !lens || !infos || !status)))
    return set_error(FV_EINVAL, "fv_jpeg_batch_plan: bad arguments");
  keep_pool_memory();
  std::unique_ptr<GpuBatch> b(new GpuBatch());
  b->n = n;
  b->nt = std::max(1, std::min<int>(threads, n));
  const int rc = n ? b->make(data, lens, infos, status) : FV_OK;
  if (rc) return rc;
  *handle = b.release();
  return FV_OK;
}

int fv_jpeg_batch_run_gpu(void* handle, uint8_t* planes, const int64_t* plane_off, uint8_t* const* dst,
                          const int64_t* dst_pitch, int32_t* status, void* stream) {
  GpuBatch* b = static_cast<GpuBatch*>(handle);
  if (!b || (b->n > 0 && (!planes || !plane_off || !dst || !dst_pitch || !status)))
    return set_error(FV_EINVAL, "fv_jpeg_batch_run_gpu: bad arguments");
  return b->n ? b->run(planes, plane_off, dst, dst_pitch, status, static_cast<cudaStream_t>(stream)) : FV_OK;
}

void fv_jpeg_batch_free(void* handle) { delete static_cast<GpuBatch*>(handle); }

int fv_jpeg_decode_batch_gpu(const uint8_t* const* data, const int64_t* lens, int32_t n, const FvJpegInfo* infos,
                             uint8_t* planes, const int64_t* plane_off, uint8_t* const* dst, const int64_t* dst_pitch,
                             int32_t* status, int32_t threads, void* stream) {
  if (n < 0 || (n > 0 && (!data || !lens || !infos || !planes || !plane_off || !dst || !dst_pitch || !status)))
    return set_error(FV_EINVAL, "fv_jpeg_decode_batch_gpu: bad arguments");
  std::vector<FvJpegInfo> fi(n);
  void* h = nullptr;
  int rc = fv_jpeg_batch_plan(data, lens, n, fi.data(), status, threads, &h);
  if (!rc) rc = fv_jpeg_batch_run_gpu(h, planes, plane_off, dst, dst_pitch, status, stream);
  fv_jpeg_batch_free(h);
  return rc;
}

}  // extern "C"
