// fv_jpeg.cu -- decode -> preprocess: the reference's
// baseline JPEG decoder (io/jpeg.py:605-806), bit-identical.
//
// Host (C++): marker walk, table parsing and the scan split with the
// reference's checks and error classes, then canonical-Huffman entropy
// decoding into quantised coefficients (natural order). This part is serial
// per restart segment by the format; it runs on the CPU, thread-safe, one
// image per thread in the batched Python wrapper.
// Device (sm_100a): dequantisation + the 13-bit fixed-point "islow" IDCT
// (8 threads per block, int64 like the reference's NumPy arithmetic, so any
// stream -- including adversarial coefficient magnitudes -- gives the same
// samples), then one kernel that upsamples the chroma planes with the
// reference's integer triangle filters and converts YCbCr -> RGB (16-bit
// fixed point), writing the HWC u8 image.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "fv_common.cuh"

namespace fv {
namespace jpg {

// natural index of zigzag position k (jpeg.py:50-59)
static const int kZigzag[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
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

static int corrupt(const char* fmt, ...) {
  char msg[256];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(msg, sizeof(msg), fmt, ap);
  va_end(ap);
  return set_error(FV_ECORRUPT, "%s", msg);
}
static int unsupported(const char* fmt, ...) {
  char msg[256];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(msg, sizeof(msg), fmt, ap);
  va_end(ap);
  return set_error(FV_EUNSUPPORTED, "%s", msg);
}

static inline int64_t extend(uint32_t v, int size);

static int build_huff(Huff& t, const uint8_t* bits, const uint8_t* vals, int count, bool dc) {
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
static int split_scan(const uint8_t* d, int64_t n, int64_t i, Stream& s) {
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
static int parse(const uint8_t* d, int64_t n, Stream& s) {
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
static int distinct(const Stream& s, int (&slot)[3]) {
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

static int64_t sparse_cap(const Stream& s);

static void fill_info(const Stream& s, FvJpegInfo& f) {
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

static inline int symbol(Bits& b, const Huff& t) {
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

static inline int64_t extend(uint32_t v, int size) {
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
static int64_t sparse_cap(const Stream& s) {
  int64_t per_mcu = 0, bits = 0;
  for (int e = 0; e < s.nscan; ++e) per_mcu += s.sof[s.scan_comp[e]].h * s.sof[s.scan_comp[e]].v;
  const int64_t total = (int64_t)s.mcus_x * s.mcus_y;
  const int64_t nexp = s.dri ? (total + s.dri - 1) / s.dri : 1;
  for (int64_t k = 0; k < nexp; ++k) bits += 8 * s.seg_len[k];
  return 2 * per_mcu * total + bits / 2 + 65;
}

// Entropy decoding (jpeg.py:326-409, 770-780).
template <class Sink>
static int decode_scan(const Stream& s, const FvJpegInfo& f, Sink& sink) {
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
  uint16_t qt[3][64];
};

// One 8-point pass of the islow IDCT (jpeg.py:163-191), int64, outputs
// before descaling in index order.
__device__ __forceinline__ void idct8(const int64_t (&s)[8], int64_t (&o)[8]) {
  const int64_t z1 = (s[2] + s[6]) * 4433;
  const int64_t e2 = z1 - s[6] * 15137, e3 = z1 + s[2] * 6270;
  const int64_t e0 = (s[0] + s[4]) * 8192, e1 = (s[0] - s[4]) * 8192;
  const int64_t a10 = e0 + e3, a13 = e0 - e3, a11 = e1 + e2, a12 = e1 - e2;
  const int64_t z5 = (s[7] + s[3] + s[5] + s[1]) * 9633;
  const int64_t q1 = (s[7] + s[1]) * -7373, q2 = (s[5] + s[3]) * -20995;
  const int64_t q3 = (s[7] + s[3]) * -16069 + z5, q4 = (s[5] + s[1]) * -3196 + z5;
  const int64_t o0 = s[7] * 2446 + q1 + q3, o1 = s[5] * 16819 + q2 + q4;
  const int64_t o2 = s[3] * 25172 + q2 + q3, o3 = s[1] * 12299 + q1 + q4;
  o[0] = a10 + o3;
  o[1] = a11 + o2;
  o[2] = a12 + o1;
  o[3] = a13 + o0;
  o[4] = a13 - o0;
  o[5] = a12 - o1;
  o[6] = a11 - o2;
  o[7] = a10 - o3;
}

// Second half of a block's IDCT, shared by the dense and sparse kernels:
// s = the dequantised column j (vertical frequencies 0..7) of block g.
__device__ __forceinline__ void idct_rows_store(int64_t (&s)[8], int64_t (&ws)[16][8][9], int g, int j, uint32_t mask,
                                                uint8_t* dst) {
  int64_t o[8];
  idct8(s, o);
#pragma unroll
  for (int k = 0; k < 8; ++k) ws[g][k][j] = (o[k] + (1 << 10)) >> 11;
  __syncwarp(mask);
#pragma unroll
  for (int k = 0; k < 8; ++k) s[k] = ws[g][j][k];
  idct8(s, o);
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

__device__ __forceinline__ int px(const uint8_t* p, int64_t pitch, int r, int c) { return p[r * pitch + c]; }

// Horizontal x2 triangle (jpeg.py:809-821) at output column X of row r
__device__ __forceinline__ int up_h2(const uint8_t* p, int64_t pitch, int r, int X, int m) {
  if (m <= 2) return px(p, pitch, r, X >> 1);
  const int jj = X >> 1;
  if (X == 0) return px(p, pitch, r, 0);
  if (X == 2 * m - 1) return px(p, pitch, r, m - 1);
  if ((X & 1) == 0) return (3 * px(p, pitch, r, jj) + px(p, pitch, r, jj - 1) + 1) >> 2;
  return (3 * px(p, pitch, r, jj) + px(p, pitch, r, jj + 1) + 2) >> 2;
}
// Vertical x2 (the reference transposes and reuses h2)
__device__ __forceinline__ int up_v2(const uint8_t* p, int64_t pitch, int Y, int c, int m) {
  if (m <= 2) return px(p, pitch, Y >> 1, c);
  const int jj = Y >> 1;
  if (Y == 0) return px(p, pitch, 0, c);
  if (Y == 2 * m - 1) return px(p, pitch, m - 1, c);
  if ((Y & 1) == 0) return (3 * px(p, pitch, jj, c) + px(p, pitch, jj - 1, c) + 1) >> 2;
  return (3 * px(p, pitch, jj, c) + px(p, pitch, jj + 1, c) + 2) >> 2;
}
// 2x2 triangle (jpeg.py:824-841): 3:1 column sums, then 3:1 across, +8/+7
__device__ __forceinline__ int up_h2v2(const uint8_t* p, int64_t pitch, int Y, int X, int mw, int mh) {
  if (mw <= 2) return px(p, pitch, Y >> 1, X >> 1);
  const int r = Y >> 1;
  const int r2 = (Y & 1) ? min(r + 1, mh - 1) : max(r - 1, 0);
  auto cs = [&](int c) { return 3 * px(p, pitch, r, c) + px(p, pitch, r2, c); };
  const int jj = X >> 1;
  if (X == 0) return (cs(0) * 4 + 8) >> 4;
  if (X == 2 * mw - 1) return (cs(mw - 1) * 4 + 7) >> 4;
  if ((X & 1) == 0) return (3 * cs(jj) + cs(jj - 1) + 8) >> 4;
  return (3 * cs(jj) + cs(jj + 1) + 7) >> 4;
}

__device__ __forceinline__ int sample(const ColorArgs& a, int e, int x, int y) {
  const uint8_t* p = a.plane[e];
  const int64_t pt = a.pitch[e];
  if (a.fh[e] == 2 && a.fv[e] == 2) return up_h2v2(p, pt, y, x, a.cw[e], a.ch[e]);
  if (a.fh[e] == 2) return up_h2(p, pt, y, x, a.cw[e]);
  if (a.fv[e] == 2) return up_v2(p, pt, y, x, a.ch[e]);
  return px(p, pt, y, x);
}

__device__ __forceinline__ uint8_t clamp255(int v) { return (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v)); }

// Upsample + YCbCr -> RGB (jpeg.py:226-235, 783-806), one pixel per thread.
__global__ void __launch_bounds__(256) jpeg_color_kernel(const __grid_constant__ ColorArgs a) {
  const int x = blockIdx.x * 256 + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= a.width) return;
  uint8_t* d = a.dst + (int64_t)y * a.d_rp;
  if (a.ncomp == 1) {
    d[x] = (uint8_t)px(a.plane[0], a.pitch[0], y, x);
    return;
  }
  const int Y = sample(a, 0, x, y), xb = sample(a, 1, x, y) - 128, xr = sample(a, 2, x, y) - 128;
  d[3 * x] = clamp255(Y + ((91881 * xr + 32768) >> 16));
  d[3 * x + 1] = clamp255(Y + ((-22554 * xb + 32768 - 46802 * xr) >> 16));
  d[3 * x + 2] = clamp255(Y + ((116130 * xb + 32768) >> 16));
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
// coef_bytes 2 / 8: dense int16 / int64 coefficients; 4: the sparse word
// stream of the batch runtime
static int reconstruct(const FvJpegInfo& f, const void* coeffs, int32_t coef_bytes, uint8_t* planes, uint8_t* dst,
                       int64_t dst_row_pitch, cudaStream_t st) {
  if (f.ncomp != 1 && f.ncomp != 3) return set_error(FV_EINVAL, "fv_jpeg_reconstruct: ncomp %d", f.ncomp);
  if (dst_row_pitch < (int64_t)f.width * f.ncomp) return set_error(FV_EINVAL, "fv_jpeg_reconstruct: row pitch too small");
  if ((reinterpret_cast<uintptr_t>(planes) & 7) != 0) return set_error(FV_EINVAL, "fv_jpeg_reconstruct: planes not 8-byte aligned");
  // distinct components (duplicated scan entries share coefficients and plane)
  IdctArgs ia{};
  ia.coeffs = coeffs;
  ia.planes = planes;
  int nd = 0;
  int64_t nb = 0;
  for (int e = 0; e < f.ncomp; ++e) {
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
  const int64_t grid = (nb + 15) / 16;
  if (grid > 0x7FFFFFFF) return set_error(FV_EINVAL, "fv_jpeg_reconstruct: too many blocks");
  if (coef_bytes == 2) jpeg_idct_kernel<int16_t><<<(unsigned)grid, 128, 0, st>>>(ia);
  else if (coef_bytes == 8) jpeg_idct_kernel<int64_t><<<(unsigned)grid, 128, 0, st>>>(ia);
  else jpeg_idct_sparse_kernel<<<(unsigned)grid, 128, 0, st>>>(ia, static_cast<const uint32_t*>(coeffs), f.coef_count / 64);
  int rc = check_launch("jpeg_idct_kernel");
  if (rc) return rc;
  ColorArgs ca{};
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
  jpeg_color_kernel<<<dim3((f.width + 255) / 256, f.height), 256, 0, st>>>(ca);
  return check_launch("jpeg_color_kernel");
}

static int decode_one(const uint8_t* data, int64_t len, void* coeffs, int64_t coef_count, int32_t coef_bytes,
                      FvJpegInfo* info_out) {
  std::unique_ptr<Stream> s(new Stream());
  int rc = parse(data, len, *s);
  if (rc) return rc;
  FvJpegInfo f;
  fill_info(*s, f);
  if (info_out) *info_out = f;
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
  std::atomic<int32_t> next{0};
  auto work = [&]() {
    for (int32_t i; (i = next.fetch_add(1)) < n;) {
      std::unique_ptr<Stream> s(new Stream());
      status[i] = parse(data[i], lens[i], *s);
      if (status[i] == FV_OK) fill_info(*s, infos[i]);
    }
  };
  const int nt = std::max(1, std::min<int>(threads, n));
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
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
  std::atomic<int32_t> next{0};
  auto work = [&]() {
    for (int32_t i; (i = next.fetch_add(1)) < n;) {
      const int64_t cap = infos[i].coef_count / 64 + infos[i].sparse_words;
      const int rc = decode_one_sparse(data[i], lens[i], words_host + word_off[i], cap, &used[i]);
      done[i].store(rc, std::memory_order_release);
    }
  };
  const int nt = std::max(1, std::min<int>(threads, n));
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) pool.emplace_back(work);
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
    rc = reconstruct(infos[i], words_dev + word_off[i], 4, planes + plane_off[i], dst[i], dst_pitch[i], st);
    if (rc) {
      first = rc;
      status[i] = rc;
    }
  }
  for (auto& t : pool) t.join();
  return first;
}

}  // extern "C"
