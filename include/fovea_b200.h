/*
 * fovea_b200.h -- C ABI of the B200 (sm_100a) image-transformation path.
 *
 * Drop-in boundary for the reference's hot path (`fovea`, a Python/NumPy
 * package; paths below are relative to /root/reference/pkg/src/fovea/):
 * every entry point replaces one reference function and keeps its semantics
 * (HWC interleaved images, same dtypes, rounding, interpolation and border).
 * The Python mirror `paper_2505_12425_b200` binds these with ctypes
 * (INTEGRATION.md shows the binding).
 *
 * Conventions shared by every entry point
 *   - All image pointers are caller-owned DEVICE memory; nothing is allocated
 *     or freed inside (the reference's preallocated-dst discipline,
 *     imgproc.py:1-6, bench.py:139-148).
 *   - Images are batches of N HWC images. Strides are in BYTES:
 *       *_img_stride  distance between consecutive images,
 *       *_row_pitch   distance between consecutive rows (>= width*C*elem;
 *                     crop views keep their parent's pitch, image.py:66-75).
 *     Pixels are C interleaved elements; channel stride is one element.
 *   - Small per-call parameters (warp matrices, normalisation LUT) are HOST
 *     pointers; they are copied into the kernel parameter block, so no device
 *     allocation or H2D copy happens per call.
 *   - `stream` is a cudaStream_t (0 = legacy default stream). Calls are
 *     asynchronous on that stream and deterministic (bit-identical reruns).
 *   - Return: FV_OK (0) on success; FV_EINVAL for a bad argument (checked
 *     before any launch; message in fv_last_error()); FV_ECUDA when the
 *     launch failed (cudaGetLastError text in fv_last_error()).
 *   - n == 0 is a valid no-op (empty batch).
 *   - Argument *validation in the reference's order* (SizeMismatch,
 *     UnsupportedDtype, AliasedBuffers) is done by the host mirror before it
 *     calls here; the ABI checks only what it needs to be memory-safe.
 */
#ifndef FOVEA_B200_H
#define FOVEA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FV_OK 0
#define FV_EINVAL (-1)
#define FV_ECUDA (-2)
#define FV_ECORRUPT (-3)     /* JPEG: malformed stream (errors.py CorruptStream) */
#define FV_EUNSUPPORTED (-4) /* JPEG: valid but outside the subset (UnsupportedJpegFeature) */
#define FV_ERANGE (-5)       /* JPEG: a coefficient does not fit the chosen width; retry wider */
#define FV_EFALLBACK (-6)    /* JPEG, GPU entropy path: this image needs the host decoder (not an error) */

/* ABI version (major*100 + minor). */
int fv_version(void);

/* Thread-local text of the last failure ("" if none). */
const char* fv_last_error(void);

/* Number of kernel launches issued by this library since load (all threads).
 * Used by bench.py to report `gpu_launches`. */
uint64_t fv_launch_count(void);

/* ---- a1: imgproc.gray_from_rgb (imgproc.py:43-64) ------------------------
 * u8: floor((f64(r)*0.299 + f64(g)*0.587) + f64(b)*0.114 + 0.5), exact.
 * f32: the same f64 sum narrowed to f32. src has 3 channels, dst 1. */
int fv_gray_from_rgb_u8(const uint8_t* src, int64_t src_img_stride, int64_t src_row_pitch,
                        uint8_t* dst, int64_t dst_img_stride, int64_t dst_row_pitch,
                        int32_t n, int32_t height, int32_t width, void* stream);
int fv_gray_from_rgb_f32(const float* src, int64_t src_img_stride, int64_t src_row_pitch,
                         float* dst, int64_t dst_img_stride, int64_t dst_row_pitch,
                         int32_t n, int32_t height, int32_t width, void* stream);

/* ---- a4: image.to_float_scaled (image.py:150-160) -------------------------
 * dst = f32(src) / f32(255), IEEE division, any channel count. */
int fv_to_float_scaled(const uint8_t* src, int64_t src_img_stride, int64_t src_row_pitch,
                       float* dst, int64_t dst_img_stride, int64_t dst_row_pitch,
                       int32_t n, int32_t height, int32_t width, int32_t channels, void* stream);

/* ---- a3: imgproc.resize_bilinear (imgproc.py:100-123) ---------------------
 * f32 bilinear, pixel-centre mapping sx=(x+0.5)*(src_w/dst_w)-0.5 in f64,
 * clamp before floor, blend in the reference's f32 op order (no FMA). */
int fv_resize_bilinear_f32(const float* src, int64_t src_img_stride, int64_t src_row_pitch,
                           int32_t src_height, int32_t src_width,
                           float* dst, int64_t dst_img_stride, int64_t dst_row_pitch,
                           int32_t dst_height, int32_t dst_width,
                           int32_t channels, int32_t n, void* stream);

/* ---- a6: service.app._resize_u8 bilinear (app.py:64-78) -----
 * to_float_scaled -> resize_bilinear -> x f32(255) -> Tensor.cast(u8)
 * (tensor.py:265-282: round half away from zero, saturate), bit-exact,
 * fused in one pass (no f32 intermediate in HBM). */
int fv_resize_bilinear_u8(const uint8_t* src, int64_t src_img_stride, int64_t src_row_pitch,
                          int32_t src_height, int32_t src_width,
                          uint8_t* dst, int64_t dst_img_stride, int64_t dst_row_pitch,
                          int32_t dst_height, int32_t dst_width,
                          int32_t channels, int32_t n, void* stream);

/* ---- a10: fused resize -> normalise -> HWC-to-CHW (builder contract) -----
 * The a6 u8 result u at (dst_height, dst_width), then
 * lut[c*256 + u] = ((f32(u)/f32(255)) - mean[c]) / std[c] (host-built table,
 * C*256 floats, channels <= 4), written planar: dst + n*dst_img_stride +
 * c*dst_plane_stride + y*dst_row_pitch + x*4. Replaces the composition
 * _resize_u8 (app.py:64-78) + to_float_scaled (image.py:150-160). */
int fv_resize_normalize_chw(const uint8_t* src, int64_t src_img_stride, int64_t src_row_pitch,
                            int32_t src_height, int32_t src_width,
                            float* dst, int64_t dst_img_stride, int64_t dst_plane_stride,
                            int64_t dst_row_pitch, int32_t dst_height, int32_t dst_width,
                            int32_t channels, int32_t n, const float* lut_host, void* stream);

/* ---- a8: warp_affine (absent from the reference) -------------
 * Inverse-mapped bilinear warp. minv_host: n * 6 doubles, the per-image
 * INVERSE (dst->src) 2x3 matrix, row-major. sx = m0*x + (m1*y + m2),
 * sy = m3*x + (m4*y + m5) in f64; per-tap constant border; blend as a3;
 * u8 images use the a6 recipe. */
int fv_warp_affine_f32(const float* src, int64_t src_img_stride, int64_t src_row_pitch,
                       int32_t src_height, int32_t src_width,
                       float* dst, int64_t dst_img_stride, int64_t dst_row_pitch,
                       int32_t dst_height, int32_t dst_width, int32_t channels, int32_t n,
                       const double* minv_host, float border, void* stream);
int fv_warp_affine_u8(const uint8_t* src, int64_t src_img_stride, int64_t src_row_pitch,
                      int32_t src_height, int32_t src_width,
                      uint8_t* dst, int64_t dst_img_stride, int64_t dst_row_pitch,
                      int32_t dst_height, int32_t dst_width, int32_t channels, int32_t n,
                      const double* minv_host, uint8_t border, void* stream);

/* ---- a9: warp_perspective (absent from the reference) --------
 * hinv_host: n * 9 doubles, per-image INVERSE homography, row-major.
 * X = h0*x + (h1*y + h2), Y = h3*x + (h4*y + h5), W = h6*x + (h7*y + h8);
 * W == 0 or non-finite coordinate -> raw border; else r = 1/W,
 * sx = X*r, sy = Y*r and the warp_affine sampler. */
int fv_warp_perspective_u8(const uint8_t* src, int64_t src_img_stride, int64_t src_row_pitch,
                           int32_t src_height, int32_t src_width,
                           uint8_t* dst, int64_t dst_img_stride, int64_t dst_row_pitch,
                           int32_t dst_height, int32_t dst_width, int32_t channels, int32_t n,
                           const double* hinv_host, uint8_t border, void* stream);
/* u8 perspective within the north-star gate for u8 results of float
 * interpolation: |out - exact| <= 1 LSB (same arguments and map). Per-thread
 * f64 anchor + f32 projective correction (<= 5e-4 px per axis, checked per
 * thread; the f64 per-pixel map where the bound fails), blend on the 0..255
 * scale rounded half up. The headline cfg3 path. */
int fv_warp_perspective_u8_fast(const uint8_t* src, int64_t src_img_stride, int64_t src_row_pitch,
                                int32_t src_height, int32_t src_width,
                                uint8_t* dst, int64_t dst_img_stride, int64_t dst_row_pitch,
                                int32_t dst_height, int32_t dst_width, int32_t channels, int32_t n,
                                const double* hinv_host, uint8_t border, void* stream);
int fv_warp_perspective_f32(const float* src, int64_t src_img_stride, int64_t src_row_pitch,
                            int32_t src_height, int32_t src_width,
                            float* dst, int64_t dst_img_stride, int64_t dst_row_pitch,
                            int32_t dst_height, int32_t dst_width, int32_t channels, int32_t n,
                            const double* hinv_host, float border, void* stream);

/* ---- the remaining imgproc kernels ---------------------------
 * imgproc.flip_horizontal (imgproc.py:67-73) and imgproc.resize_nearest
 * (imgproc.py:81-97, round-half-down pixel-centre index in f64): any element
 * type of elem_size 1, 2, 4 or 8 bytes, pure indexing (bit-exact).
 * imgproc.sobel (imgproc.py:126-155): f32, 3x3, replicate border, unnormalised
 * magnitude, NumPy's f32 op order. */
int fv_resize_nearest(const void* src, int64_t src_img_stride, int64_t src_row_pitch,
                      int32_t src_height, int32_t src_width,
                      void* dst, int64_t dst_img_stride, int64_t dst_row_pitch,
                      int32_t dst_height, int32_t dst_width,
                      int32_t channels, int32_t elem_size, int32_t n, void* stream);
int fv_flip_horizontal(const void* src, int64_t src_img_stride, int64_t src_row_pitch,
                       void* dst, int64_t dst_img_stride, int64_t dst_row_pitch,
                       int32_t height, int32_t width, int32_t channels, int32_t elem_size, int32_t n,
                       void* stream);
int fv_sobel_f32(const float* src, int64_t src_img_stride, int64_t src_row_pitch,
                 float* dst, int64_t dst_img_stride, int64_t dst_row_pitch,
                 int32_t height, int32_t width, int32_t channels, int32_t n, void* stream);

/* ---- decode -> preprocess: io.jpeg.decode_jpeg (io/jpeg.py:605-806) -----
 * Baseline / extended-sequential Huffman JPEG, 1 or 3 components, sampling
 * factors up to 2x2, restart markers, 8/16-bit quantisation tables --
 * bit-identical to the reference decoder (integer "islow" IDCT, integer
 * triangle chroma upsampling, 16-bit fixed-point YCbCr -> RGB).
 * Three steps (the output size is only known after the header):
 *   1. fv_jpeg_info       host: parse the headers and split the scan; sizes of
 *                         the coefficient buffer and the plane scratch.
 *   2. fv_jpeg_decode_coeffs  host, pure CPU, thread-safe: entropy-decode the
 *                         scan into quantised coefficients (natural order,
 *                         int16 or int64; FV_ERANGE asks for int64).
 *   3. fv_jpeg_reconstruct    device, async on `stream`: dequantise + IDCT into
 *                         the u8 component planes, then upsample + colour
 *                         convert into dst (H x W x ncomp u8, row pitch in
 *                         bytes).
 * Errors carry the reference's classes: FV_ECORRUPT / FV_EUNSUPPORTED, with
 * the message in fv_last_error(). Stream data is a HOST pointer. */
typedef struct FvJpegInfo {
  int32_t width, height, ncomp;        /* image size; 1 (gray) or 3 components */
  int32_t hmax, vmax, mcus_x, mcus_y;  /* MCU grid */
  int32_t restart_interval;            /* MCUs per restart segment, 0 = none */
  int32_t h[3], v[3];                  /* sampling factors, scan order */
  int32_t bw[3], bh[3];                /* blocks per component row / column */
  int32_t cw[3], ch[3];                /* component plane size before upsampling */
  int64_t coef_offset[3];              /* first coefficient of each component */
  int64_t coef_count;                  /* coefficients in the buffer (64 per block) */
  int64_t plane_offset[3];             /* byte offset of each u8 plane (pitch bw*8) */
  int64_t plane_bytes;                 /* plane scratch bytes */
  int64_t sparse_words;                /* batch runtime: bound of the sparse coefficient words */
  uint16_t qt[3][64];                  /* quantisation table per component, natural order */
} FvJpegInfo;

int fv_jpeg_info(const uint8_t* data, int64_t len, FvJpegInfo* info);
int fv_jpeg_decode_coeffs(const uint8_t* data, int64_t len, void* coeffs, int64_t coef_count, int32_t coef_bytes);
int fv_jpeg_reconstruct(const FvJpegInfo* info, const void* coeffs, int32_t coef_bytes, uint8_t* planes,
                        uint8_t* dst, int64_t dst_row_pitch, void* stream);

/* Batched form (the runtime around the kernels, native): parse n streams on
 * `threads` host threads (per-image status in `status`, FV_OK or the error
 * code; messages via a single-image fv_jpeg_info call), then decode them:
 * worker threads entropy-decode each image into a SPARSE coefficient stream
 * in the PINNED host buffer `words_host` (image i at word_off[i], capacity
 * coef_count/64 + sparse_words words: one header index per block, then per
 * block a count word and one (int16 value << 16 | natural position) word per
 * stored coefficient) while the calling thread, in input order, copies each
 * ready image's used words to words_dev + word_off[i] and launches its
 * reconstruction (planes + plane_off[i] -> dst[i], row pitch dst_pitch[i])
 * on `stream`. Returns the first failing image's code (later images are not
 * launched; FV_ERANGE: decode that image singly with int64 coefficients). */
int fv_jpeg_info_batch(const uint8_t* const* data, const int64_t* lens, int32_t n, FvJpegInfo* infos,
                       int32_t* status, int32_t threads);
int fv_jpeg_decode_batch(const uint8_t* const* data, const int64_t* lens, int32_t n, const FvJpegInfo* infos,
                         uint32_t* words_host, const int64_t* word_off, uint32_t* words_dev, uint8_t* planes,
                         const int64_t* plane_off, uint8_t* const* dst, const int64_t* dst_pitch, int32_t* status,
                         int32_t threads, void* stream);

/* GPU entropy decoding (batch): headers are parsed and the entropy-coded
 * segments unstuffed on `threads` host threads; the Huffman decoding itself
 * runs on the GPU (speculative, self-synchronising subsequence decoding: see
 * csrc/fv_jpeg_gpu.cu), followed by the same reconstruction kernels. One
 * stream synchronisation per call. status[i] = FV_OK when image i was decoded
 * into dst[i]; FV_EFALLBACK when it needs the host decoder (stream outside
 * the GPU path's coverage, or an anomaly on its decode path -- a corrupt
 * stream); the caller decodes those with fv_jpeg_decode_batch, which also
 * yields the exact error. Device scratch is stream-ordered (cudaMallocAsync). */
int fv_jpeg_decode_batch_gpu(const uint8_t* const* data, const int64_t* lens, int32_t n, const FvJpegInfo* infos,
                             uint8_t* planes, const int64_t* plane_off, uint8_t* const* dst, const int64_t* dst_pitch,
                             int32_t* status, int32_t threads, void* stream);

/* The same in two steps, so each stream is parsed once: fv_jpeg_batch_plan
 * parses the n streams (status[i] = FV_OK or the header error, infos[i] the
 * header when OK), lays out the GPU path's staging and returns a handle; the
 * caller allocates the outputs from `infos`; fv_jpeg_batch_run_gpu unstuffs
 * the streams on the library's worker threads while uploading each finished
 * run of images on an internal per-device copy stream (ordered before the
 * passes on `stream` by an event, so the upload may overlap work already
 * queued on `stream`), then decodes (status[i] = FV_OK or FV_EFALLBACK as
 * above; a NULL dst[i] skips image i, e.g. the images from the first header
 * error on); it returns once the statuses are known, with the reconstruction
 * still queued on `stream`. fv_jpeg_batch_free releases the handle (it holds
 * the library's pinned and device staging until then: one batch at a time
 * per process). The stream bytes must stay alive until the handle is freed. */
int fv_jpeg_batch_plan(const uint8_t* const* data, const int64_t* lens, int32_t n, FvJpegInfo* infos, int32_t* status,
                       int32_t threads, void** handle);
int fv_jpeg_batch_run_gpu(void* handle, uint8_t* planes, const int64_t* plane_off, uint8_t* const* dst,
                          const int64_t* dst_pitch, int32_t* status, void* stream);
void fv_jpeg_batch_free(void* handle);

/* ---- test-only kernel selection -------------------------------------------
 * Present only in the test build of the library (-DFV_TEST_KNOBS:
 * lib/libfovea_b200_knobs.so); the product library always selects
 * automatically and exports neither symbol. Process-global, not
 * thread-safe: for the parity tests that cover every GPU path.
 * Resize kernel selection: 0 = auto (default: exact 2:1 / 1:2 fast paths,
 * else the staged TMA strip kernel, else the direct-gather kernel),
 * 1 = always the direct-gather kernel, 2 = never the integer-ratio fast
 * paths. Exposed so the parity tests cover every GPU path. */
#ifdef FV_TEST_KNOBS
void fv_set_resize_path(int32_t mode);
#endif

/* Affine warp kernel selection: 0 = auto (default: the SMEM-staged tile
 * kernel when rows are 16-byte aligned -- the source window loaded by one
 * TMA tensor copy per tile, or by per-row bulk copies when no tensor map can
 * be encoded -- with direct gathers for tiles whose source box exceeds the
 * window), 1 = always the direct-gather kernel, 2 = the bulk-copy tile
 * kernel, 3 = the round-1 u8 perspective kernel (A/B reference for the
 * tile kernel). */
#ifdef FV_TEST_KNOBS
void fv_set_warp_path(int32_t mode);
#endif

#ifdef __cplusplus
}
#endif

#endif /* FOVEA_B200_H */
