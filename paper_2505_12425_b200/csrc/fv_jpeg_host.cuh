// fv_jpeg_host.cuh -- host side of the JPEG decoder (io/jpeg.py:605-806):
// marker walk and table parsing with the reference's checks and error
// classes, the scan split, and canonical-Huffman entropy decoding into dense
// or sparse coefficient sinks. Shared by fv_jpeg.cu (host entropy path and
// GPU reconstruction) and fv_jpeg_gpu.cu (GPU entropy path planning).
#pragma once
#include <sched.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdarg>
#include <functional>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstring>
#include <memory>
#include <vector>

#include "fv_common.cuh"
#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace fv {
namespace jpg {

// natural index of zigzag position k (jpeg.py:50-59)
inline const int kZigzag[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                                12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                                35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                                58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

// Canonical Huffman table (jpeg.py:269-296): 8-bit lookup for short codes,
// per-length ranges for the rest.
// Fast table entries, indexed by the next 10 bits: kFull = code and its
// magnitude bits both fit: total length (bits 0-4), zero run (8-11), signed
// value (16-31); kSym = the code fits: its length (0-4) and symbol (16-23).
constexpr int32_t kFull = 1 << 12, kSym = 1 << 13;

struct Huff {
  bool present = false;
  int32_t fast[1 << 10];
  uint8_t lut_len[256];  // 0 = no code of <= 8 bits has this prefix
  uint8_t lut_val[256];
  int32_t mincode[17], maxcode[17], valptr[17];
  uint8_t values[16 * 255];
};

struct Comp {
  int id, h, v, tq;
  int td, ta;  // Huffman tables (the last scan entry naming the component wins, as in the reference)
};

struct Stream {
  int width = 0, height = 0, ncomp = 0;  // SOF
  bool have_sof = false;
  Comp sof[3];
  int nscan = 0;
  int scan_comp[3];  // scan entry -> SOF component (duplicates share state, jpeg.py:721-729)
  uint16_t qt[16][64];
  bool qt_ok[16] = {};
  Huff dc[16], ac[16];
  int dri = 0;
  // entropy-coded segments as raw byte ranges of the stream (stuffing and
  // fill bytes still in place) and their unstuffed lengths
  std::vector<int64_t> seg_raw;  // nseg + 1 boundaries: segment k is [seg_raw[k], seg_end[k])
  std::vector<int64_t> seg_end;
  std::vector<int64_t> seg_len;  // unstuffed bytes
  // geometry (after SOS)
  int hmax = 1, vmax = 1, mcus_x = 0, mcus_y = 0;
  const uint8_t* data = nullptr;  // the stream (segments point into it)
};

inline int corrupt(const char* fmt, ...) {
  char msg[256];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(msg, sizeof(msg), fmt, ap);
  va_end(ap);
  return set_error(FV_ECORRUPT, "%s", msg);
}
inline int unsupported(const char* fmt, ...) {
  char msg[256];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(msg, sizeof(msg), fmt, ap);
  va_end(ap);
  return set_error(FV_EUNSUPPORTED, "%s", msg);
}

inline int64_t extend(uint32_t v, int size);

inline int build_huff(Huff& t, const uint8_t* bits, const uint8_t* vals, int count, bool dc) {
  memset(t.lut_len, 0, sizeof(t.lut_len));
  memcpy(t.values, vals, count);
  int code = 0, idx = 0;
  for (int len = 1; len <= 16; ++len) {
    const int cnt = bits[len - 1];
    t.mincode[len] = 0;
    t.maxcode[len] = -1;
    t.valptr[len] = 0;
    if (cnt) {
      if (code + cnt > (1 << len)) return corrupt("Huffman code space overflow");
      t.valptr[len] = idx;
      t.mincode[len] = code;
      for (int k = 0; k < cnt; ++k, ++idx, ++code) {
        if (len <= 8) {
          const int lo = code << (8 - len);
          for (int j = lo; j < lo + (1 << (8 - len)); ++j) {
            t.lut_len[j] = (uint8_t)len;
            t.lut_val[j] = vals[idx];
          }
        }
      }
      t.maxcode[len] = code - 1;
    }
    code <<= 1;
  }
  for (int x = 0; x < (1 << 10); ++x) {
    t.fast[x] = 0;
    for (int len = 1; len <= 10; ++len) {
      const int code = x >> (10 - len);
      if (t.maxcode[len] < 0 || code > t.maxcode[len]) continue;
      const int sym = t.values[t.valptr[len] + code - t.mincode[len]];
      const int size = dc ? sym : (sym & 15);
      const bool valid = dc ? size <= 11 : size > 0;  // DC: the size check stays on the slow path
      if (valid && len + size <= 10) {
        const int64_t v = size ? extend((uint32_t)(x >> (10 - len - size)) & ((1u << size) - 1), size) : 0;
        t.fast[x] = kFull | (len + size) | ((dc ? 0 : sym >> 4) << 8) | (int32_t)((uint32_t)(v & 0xFFFF) << 16);
      } else {
        t.fast[x] = kSym | len | (sym << 16);
      }
      break;
    }
  }
  t.present = true;
  return FV_OK;
}

// Segments split at RSTn (jpeg.py:574-602), recorded as raw ranges plus
// their unstuffed lengths (the bit reader unstuffs on the fly: no copy).
inline int split_scan(const uint8_t* d, int64_t n, int64_t i, Stream& s) {
  s.seg_raw.assign(1, i);
  s.seg_end.clear();
  s.seg_len.clear();
  int64_t len = 0;
  while (i < n) {
    const uint8_t* f = static_cast<const uint8_t*>(memchr(d + i, 0xFF, (size_t)(n - i)));
    if (!f) break;
    len += (f - (d + i));
    i = f - d;
    if (i + 1 >= n) return corrupt("scan ends mid-marker");
    const uint8_t nx = d[i + 1];
    if (nx == 0x00) {
      ++len;
      i += 2;
    } else if (nx >= 0xD0 && nx <= 0xD7) {
      s.seg_end.push_back(i);
      s.seg_len.push_back(len);
      len = 0;
      i += 2;
      s.seg_raw.push_back(i);
    } else if (nx == 0xFF) {
      i += 1;  // fill byte
    } else {
      s.seg_end.push_back(i);
      s.seg_len.push_back(len);
      return FV_OK;
    }
  }
  return corrupt("scan ends without a terminating marker");
}

// Marker walk up to the first SOS and the scan split (jpeg.py:605-735),
// then the post-header checks and the MCU geometry (jpeg.py:737-768).
inline int parse(const uint8_t* d, int64_t n, Stream& s) {
  if (!d || n < 4 || d[0] != 0xFF || d[1] != 0xD8) return corrupt("not a JPEG stream (bad SOI)");
  s.data = d;
  int64_t i = 2;
  for (;;) {
    if (i + 2 > n) return corrupt("stream ends without EOI");
    if (d[i] != 0xFF) return corrupt("expected marker at offset %lld", (long long)i);
    const int mk = d[i + 1];
    i += 2;
    if (mk == 0xD9) return corrupt("EOI before scan data");
    if (mk == 0x01 || (mk >= 0xD0 && mk <= 0xD7)) continue;
    if (i + 2 > n) return corrupt("truncated stream");
    const int ln = (d[i] << 8) | d[i + 1];
    if (ln < 2) return corrupt("bad segment length");
    if (i + ln > n) return corrupt("truncated stream");
    const uint8_t* pl = d + i + 2;
    const int pn = ln - 2;
    i += ln;
    if (mk == 0xDB) {  // DQT
      int p = 0;
      while (p < pn) {
        const int pq = pl[p] >> 4, tq = pl[p] & 15;
        ++p;
        if (pq != 0 && pq != 1) return corrupt("bad DQT precision %d", pq);
        const int cnt = 64 * (pq ? 2 : 1);
        if (p + cnt > pn) return corrupt("truncated DQT");
        for (int k = 0; k < 64; ++k)
          s.qt[tq][kZigzag[k]] = pq ? (uint16_t)((pl[p + 2 * k] << 8) | pl[p + 2 * k + 1]) : pl[p + k];
        s.qt_ok[tq] = true;
        p += cnt;
      }
    } else if (mk == 0xC0 || mk == 0xC1) {  // SOF0 / SOF1
      if (pn < 6) return corrupt("truncated SOF");
      const int prec = pl[0], h = (pl[1] << 8) | pl[2], w = (pl[3] << 8) | pl[4], nc = pl[5];
      s.height = h;
      s.width = w;
      s.have_sof = true;
      if (prec != 8) return unsupported("sample precision %d", prec);
      if (h == 0 || w == 0) return corrupt("zero dimension");
      if (nc != 1 && nc != 3) return unsupported("%d components", nc);
      if (pn != 6 + 3 * nc) return corrupt("bad SOF length");
      s.ncomp = 0;
      for (int c = 0; c < nc; ++c) {
        Comp& cp = s.sof[c];
        cp.id = pl[6 + 3 * c];
        cp.h = pl[7 + 3 * c] >> 4;
        cp.v = pl[7 + 3 * c] & 15;
        cp.tq = pl[8 + 3 * c];
        cp.td = cp.ta = -1;
        if ((cp.h != 1 && cp.h != 2) || (cp.v != 1 && cp.v != 2))
          return unsupported("sampling factors %dx%d", cp.h, cp.v);
        s.ncomp = c + 1;
      }
      if (nc == 1) s.sof[0].h = s.sof[0].v = 1;
    } else if (mk == 0xC2) {
      return unsupported("progressive JPEG");
    } else if (mk == 0xC3 || mk == 0xC5 || mk == 0xC6 || mk == 0xC7 || mk == 0xC9 || mk == 0xCA || mk == 0xCB ||
               mk == 0xCD || mk == 0xCE || mk == 0xCF) {
      return unsupported("SOF marker 0xFF%02X", mk);
    } else if (mk == 0xCC) {
      return unsupported("arithmetic coding");
    } else if (mk == 0xC4) {  // DHT
      int p = 0;
      while (p < pn) {
        if (p + 17 > pn) return corrupt("truncated DHT");
        const int tc = pl[p] >> 4, th = pl[p] & 15;
        int cnt = 0;
        for (int k = 1; k <= 16; ++k) cnt += pl[p + k];
        if (p + 17 + cnt > pn) return corrupt("truncated DHT values");
        const int rc = build_huff(tc == 0 ? s.dc[th] : s.ac[th], pl + p + 1, pl + p + 17, cnt, tc == 0);
        if (rc) return rc;
        p += 17 + cnt;
      }
    } else if (mk == 0xDD) {  // DRI
      if (pn != 2) return corrupt("bad DRI length");
      s.dri = (pl[0] << 8) | pl[1];
    } else if (mk == 0xDA) {  // SOS
      if (s.ncomp == 0) return corrupt("SOS before SOF");
      if (pn < 1) return corrupt("bad SOS length");
      const int ns = pl[0];
      if (ns != s.ncomp) return unsupported("multi-scan stream");
      if (pn != 1 + 2 * ns + 3) return corrupt("bad SOS length");
      for (int e = 0; e < ns; ++e) {
        const int cid = pl[1 + 2 * e], tb = pl[2 + 2 * e];
        int k = 0;
        while (k < s.ncomp && s.sof[k].id != cid) ++k;
        if (k == s.ncomp) return corrupt("scan references unknown component %d", cid);
        const int td = tb >> 4, ta = tb & 15;
        if (!s.dc[td].present || !s.ac[ta].present) return corrupt("scan references missing Huffman table");
        s.sof[k].td = td;
        s.sof[k].ta = ta;
        s.scan_comp[e] = k;
      }
      s.nscan = ns;
      const int rc = split_scan(d, n, i, s);
      if (rc) return rc;
      break;
    }
    // other APPn / COM / unknown segments are skipped
  }
  if (!s.have_sof) return corrupt("no scan data");
  for (int e = 0; e < s.nscan; ++e) {
    const int tq = s.sof[s.scan_comp[e]].tq;  // a full byte; tables are numbered 0-15
    if (tq > 15 || !s.qt_ok[tq]) return corrupt("component references missing quant table %d", tq);
  }
  s.hmax = s.vmax = 1;
  for (int e = 0; e < s.nscan; ++e) {
    s.hmax = std::max(s.hmax, s.sof[s.scan_comp[e]].h);
    s.vmax = std::max(s.vmax, s.sof[s.scan_comp[e]].v);
  }
  s.mcus_x = (s.width + 8 * s.hmax - 1) / (8 * s.hmax);
  s.mcus_y = (s.height + 8 * s.vmax - 1) / (8 * s.vmax);
  const int64_t total = (int64_t)s.mcus_x * s.mcus_y;
  const int64_t nexp = s.dri ? (total + s.dri - 1) / s.dri : 1;
  const int64_t nseg = (int64_t)s.seg_len.size();
  if (nseg < nexp) return corrupt("%lld entropy segments, expected %lld", (long long)nseg, (long long)nexp);
  // Every block consumes at least two bits (a DC and an AC symbol), and a
  // segment may not consume bits past its data: a header claiming more
  // blocks than the used segments can hold is corrupt whatever the symbols
  // (checked here, before any allocation, instead of after decoding).
  int64_t per_mcu = 0;
  for (int e = 0; e < s.nscan; ++e) per_mcu += s.sof[s.scan_comp[e]].h * s.sof[s.scan_comp[e]].v;
  int64_t bits = 0;
  for (int64_t k = 0; k < nexp; ++k) bits += 8 * s.seg_len[k];
  if (2 * per_mcu * total > bits) return corrupt("entropy segment too short for its MCUs");
  return FV_OK;
}

// distinct SOF components referenced by the scan, in first-appearance order
inline int distinct(const Stream& s, int (&slot)[3]) {
  int nd = 0;
  int seen[3] = {-1, -1, -1};
  for (int e = 0; e < s.nscan; ++e) {
    const int k = s.scan_comp[e];
    int j = 0;
    while (j < nd && seen[j] != k) ++j;
    if (j == nd) seen[nd++] = k;
    slot[e] = j;
  }
  return nd;
}

inline int64_t sparse_cap(const Stream& s);

inline void fill_info(const Stream& s, FvJpegInfo& f) {
  memset(&f, 0, sizeof(f));
  f.width = s.width;
  f.height = s.height;
  f.ncomp = s.nscan;
  f.hmax = s.hmax;
  f.vmax = s.vmax;
  f.mcus_x = s.mcus_x;
  f.mcus_y = s.mcus_y;
  f.restart_interval = s.dri;
  int slot[3];
  const int nd = distinct(s, slot);
  int64_t coff[3], poff[3], c = 0, p = 0;
  for (int j = 0; j < nd; ++j) {
    int e = 0;
    while (slot[e] != j) ++e;
    const Comp& cp = s.sof[s.scan_comp[e]];
    const int64_t blocks = (int64_t)s.mcus_x * cp.h * s.mcus_y * cp.v;
    coff[j] = c;
    poff[j] = p;
    c += 64 * blocks;
    p += 64 * blocks;
  }
  for (int e = 0; e < s.nscan; ++e) {
    const Comp& cp = s.sof[s.scan_comp[e]];
    f.h[e] = cp.h;
    f.v[e] = cp.v;
    f.bw[e] = s.mcus_x * cp.h;
    f.bh[e] = s.mcus_y * cp.v;
    f.cw[e] = (int32_t)(((int64_t)s.width * cp.h + s.hmax - 1) / s.hmax);
    f.ch[e] = (int32_t)(((int64_t)s.height * cp.v + s.vmax - 1) / s.vmax);
    f.coef_offset[e] = coff[slot[e]];
    f.plane_offset[e] = poff[slot[e]];
    memcpy(f.qt[e], s.qt[cp.tq], sizeof(f.qt[e]));
  }
  f.coef_count = c;
  f.plane_bytes = p;
  f.sparse_words = sparse_cap(s);
}

// MSB-first bit reader over one segment: unstuffs the raw bytes on the fly
// (FF 00 -> FF, a fill FF is skipped), zero bits past the segment's data.
struct Bits {
  const uint8_t* p;
  int64_t pos, end;      // raw cursor and the segment's terminating marker
  int64_t fed = 0;       // bytes fed into acc (data or zero padding)
  int64_t n;             // unstuffed data bytes
  uint64_t acc = 0;
  int nb = 0;            // valid bits at the top of acc
  void fill() {
    if (nb > 56) return;
    // fast path: the next 8 raw bytes are data and hold no 0xFF (SWAR test
    // for a zero byte in ~w): append the k = (64 - nb) / 8 bytes at once
    if (pos + 8 <= end && fed + 8 <= n) {
      uint64_t w;
      memcpy(&w, p + pos, 8);
      const uint64_t x = ~w;
      if (((x - 0x0101010101010101ull) & ~x & 0x8080808080808080ull) == 0) {
        const int k = (64 - nb) >> 3;
        uint64_t be = __builtin_bswap64(w);
        if (k < 8) be &= ~((1ull << (64 - 8 * k)) - 1);
        acc |= be >> nb;
        pos += k;
        fed += k;
        nb += 8 * k;
        return;
      }
    }
    while (nb <= 56) {
      uint32_t b = 0;
      while (pos < end) {
        b = p[pos];
        if (b != 0xFF) {
          ++pos;
          break;
        }
        if (p[pos + 1] == 0x00) {  // stuffed FF (pos + 1 < end: the segment ends at a marker)
          pos += 2;
          break;
        }
        ++pos;  // fill FF
        b = 0;
      }
      if (fed >= n) b = 0;  // past the data: zero padding
      acc |= (uint64_t)b << (56 - nb);
      ++fed;
      nb += 8;
    }
  }
  uint32_t peek(int k) const { return (uint32_t)(acc >> (64 - k)); }
  void skip(int k) {
    acc <<= k;
    nb -= k;
  }
  bool over() const { return fed * 8 - nb > n * 8; }  // consumed bits past the data
};

inline int symbol(Bits& b, const Huff& t) {
  const uint32_t top = b.peek(8);
  if (t.lut_len[top]) {
    b.skip(t.lut_len[top]);
    return t.lut_val[top];
  }
  for (int len = 9; len <= 16; ++len) {
    const int32_t code = (int32_t)b.peek(len);
    if (t.maxcode[len] >= 0 && code <= t.maxcode[len]) {
      b.skip(len);
      return t.values[t.valptr[len] + code - t.mincode[len]];
    }
  }
  return -1;
}

inline int64_t extend(uint32_t v, int size) {
  return v < (1u << (size - 1)) ? (int64_t)v - (1 << size) + 1 : (int64_t)v;
}

// Entropy decoding (jpeg.py:326-409, 770-780) into `coeffs`.
// Where decoded blocks go. Dense<T>: 64 coefficients per block in natural
// order (the standalone ABI and the int64 path). Sparse: per block a header
// word (count) plus one word per stored coefficient, (int16 value << 16) |
// natural position, and the block's header index in `ptr` -- what the batch
// runtime ships to the GPU (no host zero-fill, ~3x fewer H2D bytes).
template <typename T>
struct Dense {
  T* coeffs;
  T* blk = nullptr;
  bool begin(const FvJpegInfo& f, int e, int64_t rb) {
    blk = coeffs + f.coef_offset[e] + 64 * rb;
    for (int z = 0; z < 64; ++z) blk[z] = 0;
    return true;
  }
  void put(int pos, int64_t v) { blk[pos] = (T)v; }
  void end() {}
  static constexpr bool kInt16 = sizeof(T) == 2;
};

struct Sparse {
  uint32_t* ptr;  // header index of each block (component blocks concatenated)
  uint32_t* ent;
  int64_t cap, cur = 0, hdr = 0;
  uint32_t cnt = 0;
  bool begin(const FvJpegInfo& f, int e, int64_t rb) {
    if (cur + 65 > cap) return false;
    ptr[f.coef_offset[e] / 64 + rb] = (uint32_t)cur;
    hdr = cur++;
    cnt = 0;
    return true;
  }
  void put(int pos, int64_t v) {
    ent[cur++] = ((uint32_t)(uint16_t)(int16_t)v << 16) | (uint32_t)pos;
    ++cnt;
  }
  void end() { ent[hdr] = cnt; }
  static constexpr bool kInt16 = true;
};

// Upper bound of the sparse entry words of a well-formed scan: a header and
// a DC word per decoded block, and each further word costs >= 2 bits (an AC
// symbol and its magnitude). Exceeding it means padding bits were consumed,
// i.e. the stream is corrupt (the reference's end-of-segment check).
inline int64_t sparse_cap(const Stream& s) {
  int64_t per_mcu = 0, bits = 0;
  for (int e = 0; e < s.nscan; ++e) per_mcu += s.sof[s.scan_comp[e]].h * s.sof[s.scan_comp[e]].v;
  const int64_t total = (int64_t)s.mcus_x * s.mcus_y;
  const int64_t nexp = s.dri ? (total + s.dri - 1) / s.dri : 1;
  for (int64_t k = 0; k < nexp; ++k) bits += 8 * s.seg_len[k];
  return 2 * per_mcu * total + bits / 2 + 65;
}

// Entropy decoding (jpeg.py:326-409, 770-780).
template <class Sink>
inline int decode_scan(const Stream& s, const FvJpegInfo& f, Sink& sink) {
  int64_t pred[3] = {0, 0, 0};  // per SOF component (duplicated scan entries share it)
  const int64_t total = (int64_t)s.mcus_x * s.mcus_y;
  const int64_t nexp = s.dri ? (total + s.dri - 1) / s.dri : 1;
  int64_t mcu = 0;
  for (int64_t sg = 0; sg < nexp; ++sg) {
    const int64_t cnt = s.dri ? std::min<int64_t>(s.dri, total - sg * s.dri) : total;
    Bits b;
    b.p = s.data;
    b.pos = s.seg_raw[sg];
    b.end = s.seg_end[sg];
    b.n = s.seg_len[sg];
    pred[0] = pred[1] = pred[2] = 0;
    for (int64_t m = 0; m < cnt; ++m, ++mcu) {
      const int64_t my = mcu / s.mcus_x, mx = mcu - my * s.mcus_x;
      for (int e = 0; e < s.nscan; ++e) {
        const int k = s.scan_comp[e];
        const Comp& cp = s.sof[k];
        const Huff& dct = s.dc[cp.td];
        const Huff& act = s.ac[cp.ta];
        for (int by = 0; by < cp.v; ++by)
          for (int bx = 0; bx < cp.h; ++bx) {
            if (!sink.begin(f, e, (my * cp.v + by) * (int64_t)f.bw[e] + mx * cp.h + bx))
              return corrupt("entropy segment too short for its MCUs");
            b.fill();
            const int32_t fd = dct.fast[b.peek(10)];
            if (fd & kFull) {
              b.skip(fd & 31);
              pred[k] += fd >> 16;
            } else {
              int size;
              if (fd & kSym) {
                b.skip(fd & 31);
                size = (fd >> 16) & 0xFF;
              } else {
                size = symbol(b, dct);
              }
              if (size < 0) return corrupt("invalid Huffman code");
              if (size) {
                if (size > 11) return corrupt("bad DC size %d", size);
                const uint32_t v = b.peek(size);
                b.skip(size);
                pred[k] += extend(v, size);
              }
            }
            if (Sink::kInt16 && (pred[k] < -32768 || pred[k] > 32767))
              return set_error(FV_ERANGE, "DC coefficient %lld does not fit int16", (long long)pred[k]);
            sink.put(0, pred[k]);
            for (int z = 1; z < 64;) {
              b.fill();
              const int32_t fa = act.fast[b.peek(10)];
              if (fa & kFull) {  // code + magnitude in one lookup
                b.skip(fa & 31);
                z += (fa >> 8) & 15;
                if (z > 63) return corrupt("AC run past end of block");
                sink.put(kZigzag[z], fa >> 16);
                ++z;
                continue;
              }
              int rs;
              if (fa & kSym) {
                b.skip(fa & 31);
                rs = (fa >> 16) & 0xFF;
              } else {
                rs = symbol(b, act);
              }
              if (rs < 0) return corrupt("invalid Huffman code");
              const int sz = rs & 15;
              if (sz == 0) {
                if (rs == 0xF0) {
                  z += 16;
                  continue;
                }
                break;  // EOB
              }
              z += rs >> 4;
              if (z > 63) return corrupt("AC run past end of block");
              const uint32_t v = b.peek(sz);
              b.skip(sz);
              sink.put(kZigzag[z], extend(v, sz));  // |v| < 2^15: fits int16
              ++z;
            }
            sink.end();
          }
      }
    }
    if (b.over()) return corrupt("entropy segment too short for its MCUs");
  }
  return FV_OK;
}

// Write back and evict a host range that worker threads just wrote to
// pinned staging. Measured on the GPU boxes: H2D DMA from pinned memory whose
// lines sit dirty in many cores' private caches runs at 6-8 GB/s (every line
// is snooped), against 54 GB/s once the writers flush them
// (tools/probe/h2d_probe3.cu).
#if defined(__x86_64__)
__attribute__((target("clflushopt"))) inline void flush_lines_opt(const void* p, size_t n) {
  char* c = static_cast<char*>(const_cast<void*>(p));
  for (size_t i = 0; i < n; i += 64) _mm_clflushopt(c + i);
  if (n) _mm_clflushopt(c + n - 1);
  _mm_sfence();
}
inline void flush_lines(const void* p, size_t n) {
  static const bool opt = __builtin_cpu_supports("clflushopt");
  if (opt) {
    flush_lines_opt(p, n);
    return;
  }
  const char* c = static_cast<const char*>(p);
  for (size_t i = 0; i < n; i += 64) _mm_clflush(c + i);
  if (n) _mm_clflush(c + n - 1);
  _mm_mfence();
}
#else
inline void flush_lines(const void*, size_t) {}
#endif

// ---------------------------------------------------------------------------
// host worker pool: the batch entry points run their per-image work (parse,
// unstuff, entropy decoding) on persistent threads -- spawning and joining
// a thread per worker costs tens of microseconds each, per call.
// ---------------------------------------------------------------------------

class WorkPool {
 public:
  // fn(i) for i in [0, n); `want` pool threads join (the caller may help)
  struct Job {
    std::function<void(int32_t)> fn;
    int32_t n = 0;
    int want = 0;
    std::atomic<int32_t> next{0};
    int joined = 0, running = 0;  // guarded by the pool mutex
    void work() {
      for (int32_t i; (i = next.fetch_add(1)) < n;) fn(i);
    }
  };

  // the process's pool (re-created in a forked child, whose threads are gone)
  static WorkPool& get() {
    static std::mutex m;
    static WorkPool* pool = nullptr;
    std::lock_guard<std::mutex> g(m);
    if (!pool || pool->pid_ != getpid()) pool = new WorkPool();  // never destroyed: no exit-time joins
    return *pool;
  }
  int size() const { return (int)threads_.size(); }

  void start(Job& j) {
    if (j.want <= 0) return;
    std::lock_guard<std::mutex> g(m_);
    queue_.push_back(&j);
    cv_.notify_all();
  }
  // all of j's iterations done and no pool thread still inside it (the
  // caller finishes what no thread took)
  void wait(Job& j) {
    {
      std::lock_guard<std::mutex> g(m_);
      unqueue(&j);
    }
    j.work();
    std::unique_lock<std::mutex> g(m_);
    done_.wait(g, [&] { return j.running == 0; });
  }
  // run fn over [0, n) on `threads` threads (the caller is one of them)
  void run(int32_t n, int threads, std::function<void(int32_t)> fn) {
    Job j;
    j.fn = std::move(fn);
    j.n = n;
    j.want = std::max(0, std::min(std::min(threads, (int)n) - 1, size()));
    start(j);
    j.work();
    wait(j);
  }

 private:
  WorkPool() : pid_(getpid()) {
    // one thread per CPU this process may run on
    int n = (int)std::thread::hardware_concurrency();
    cpu_set_t cs;
    if (sched_getaffinity(0, sizeof(cs), &cs) == 0) n = CPU_COUNT(&cs);
    n = std::max(1, n);
    for (int t = 0; t < n; ++t) threads_.emplace_back([this] { loop(); });
    for (auto& t : threads_) t.detach();
  }
  void unqueue(Job* j) {
    for (size_t k = 0; k < queue_.size(); ++k)
      if (queue_[k] == j) {
        queue_.erase(queue_.begin() + (long)k);
        return;
      }
  }
  void loop() {
    for (;;) {
      Job* j;
      {
        std::unique_lock<std::mutex> g(m_);
        cv_.wait(g, [&] { return !queue_.empty(); });
        j = queue_.front();
        ++j->running;
        if (++j->joined >= j->want) unqueue(j);
      }
      j->work();
      {
        std::lock_guard<std::mutex> g(m_);
        if (--j->running == 0) done_.notify_all();
      }
    }
  }
  pid_t pid_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  std::vector<Job*> queue_;
  std::vector<std::thread> threads_;
};

// GPU reconstruction (fv_jpeg.cu): dequantise + IDCT + upsample + colour of
// one image's coefficients (coef_bytes 2/4/8 dense int16/int32/int64, 1 the
// sparse word stream) into dst.
int reconstruct(const FvJpegInfo& f, const void* coeffs, int32_t coef_bytes, uint8_t* planes, uint8_t* dst,
                int64_t dst_row_pitch, cudaStream_t st);
// the same for n images with dense int16 coefficients: one launch per kernel
int reconstruct_batch(int n, const FvJpegInfo* const* fs, const int16_t* const* coeffs, uint8_t* const* planes,
                      uint8_t* const* dst, const int64_t* dst_pitch, cudaStream_t st);

}  // namespace jpg
}  // namespace fv
