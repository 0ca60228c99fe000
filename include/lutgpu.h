/*
 * lutgpu — C ABI of the B200 (sm_100a) LUT-layer inference path.
 *
 * The reference (`lutkit`, /root/reference/pkg/src/lutkit) is a pure Python /
 * NumPy package with no FFI; its drop-in boundary is the Python function API
 * (SURVEY.md §8(b)).  This header is the native boundary underneath the
 * Python mirror in `paper_2302_03213_b200/`: each entry replaces one reference
 * function, cited as file:line below.  A ctypes / cffi / C++ host binds these
 * directly (INTEGRATION.md shows the bindings).
 *
 * Conventions
 *  - All array pointers are caller-owned DEVICE memory unless the name says
 *    `_host`.  Layouts are row-major (C order) like the reference:
 *      A      (n, d) f32            rows of the layer input (as_matrix, tensor.py:28-33)
 *      books  (c, k, v) f32         codebooks (validate_codebooks, pq.py:44-50)
 *      codes  (n, c) u8             one index per (row, codebook)      [code_bits = 8]
 *             (n, ceil(c/2)) u8     two 4-bit indices per byte, low nibble = even c
 *                                                                      [code_bits = 4, k <= 16]
 *      table  (c, k, m) f32         T[c,k,m] (build_table, pq.py:177-193)
 *      q      (c, k, m) i8          quantized table, |q| <= 127 (quant.py:22-57)
 *      out    (n, m) f32            or NCHW when out_hw > 0 (see gathers)
 *  - Every call is stream-ordered and asynchronous on `stream` (a cudaStream_t;
 *    NULL = legacy default stream).  No call allocates device memory on the hot
 *    path; scratch is passed in.  There is no global mutable state: calls are
 *    reentrant across streams and threads.
 *  - Return value: LUT_OK or an error status (mirrors lutkit/errors.py:8-33):
 *      LUT_ERR_CONFIG     2  ConfigError / ShapeError (bad shape, bad option)
 *      LUT_ERR_DATA       3  DataError (NaN table; non-positive scale)
 *      LUT_ERR_CORRUPTION 5  CorruptionError (code index >= k)
 *      LUT_ERR_CUDA       6  CUDA runtime failure (lut_last_error() has text)
 *    Shape/option errors are detected on the host before any launch.  Data
 *    errors that need the data (index >= k, NaN) are raised on the device into
 *    `err_flag` (a device int32, may be NULL to skip the check) and surface at
 *    the next lut_read_status() on that flag.
 */
#ifndef LUTGPU_H
#define LUTGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define LUT_API __attribute__((visibility("default")))
#else
#define LUT_API
#endif

typedef struct CUstream_st* lut_stream_t; /* identical to cudaStream_t */

enum lut_status {
  LUT_OK = 0,
  LUT_ERR_CONFIG = 2,
  LUT_ERR_DATA = 3,
  LUT_ERR_CORRUPTION = 5,
  LUT_ERR_CUDA = 6,
};

enum lut_act { LUT_ACT_NONE = 0, LUT_ACT_RELU = 1, LUT_ACT_GELU = 2 };

/* ABI version (major*100 + minor). */
LUT_API int lut_version(void);

/* Text of the last error raised on the calling thread ("" if none). */
LUT_API const char* lut_last_error(void);

/* Bytes of the prepared-codebook buffer for lut_prepare_books(). */
LUT_API size_t lut_books_prep_bytes(int32_t c, int32_t k, int32_t v);

/*
 * Precompute what encode needs from the codebooks, once per layer:
 * per codebook the centroids, ||p_k||^2 (f64-accurate, rounded to f32) and
 * max_k ||p_k||^2, packed for bulk copies; for V = 32, K = 16 also the
 * centroids as a 128B-swizzled tf32 MMA operand tile and ||p_k|| rounded up
 * (tensor-core candidate screening, csrc/encode_tc.cu).  Replaces the per-call
 * `p_norm = einsum(...)` of centroid_search_fast (kernels.py:72-74).
 */
LUT_API int lut_prepare_books(const float* books, int32_t c, int32_t k, int32_t v,
                      void* books_prep, lut_stream_t stream);

/*
 * Nearest-centroid encode.  Replaces centroid_search_fast (kernels.py:62-102);
 * indices are identical to encode_hard (pq.py:171-174): argmin of the squared
 * L2 distance, ties to the lowest k.  fp32 FFMA evaluates ||p||^2 - 2 a.p; a
 * (row, codebook) whose best/second-best gap is inside the fp32 error bound is
 * re-decided in fp64 from literal differences and counted in
 * *near_tie_count (device int32, accumulated; may be NULL).
 * code_bits = 8 (u8) or 4 (packed nibbles, k <= 16); code_stride = bytes per
 * code row (0 = dense: c for u8, ceil(c/2) for u4; the one-hot gather wants
 * lut_code_stride(c)).
 */
LUT_API int lut_encode_f32(const float* a, int64_t n, int32_t d, const void* books_prep,
                   int32_t c, int32_t k, int32_t v, uint8_t* codes, int32_t code_bits,
                   int64_t code_stride, int32_t* near_tie_count, lut_stream_t stream);

/*
 * Encode with im2col fused into the row loader: reads the NCHW batch directly;
 * row = (b, oy, ox), column = (ci, dy, dx) channel-major exactly as
 * im2col (tensor.py:36-79) + Conv._lower (model.py:105-111).  d = cin*kh*kw.
 */
LUT_API int lut_encode_conv_f32(const float* x, int32_t batch, int32_t cin, int32_t h, int32_t w,
                        int32_t kh, int32_t kw, int32_t stride, int32_t pad,
                        const void* books_prep, int32_t c, int32_t k, int32_t v,
                        uint8_t* codes, int32_t code_bits, int32_t* near_tie_count,
                        lut_stream_t stream);

/*
 * Hash encode (hashing.encode_hash, hashing.py:171-196): one depth-L tree per
 * codebook, level-major thresholds, left on <=.  dims (c, L) int32 indices
 * into the sub-vector (< v), thresholds (c, 2^L - 1) f32, leaves (c, 2^L) u8.
 * u8 codes with row stride code_stride (0 = c).  1 <= L <= 16.
 */
LUT_API int lut_encode_hash(const float* a, int64_t n, int32_t d, const int32_t* dims, const float* thresholds,
                            const uint8_t* leaves, int32_t c, int32_t levels, int32_t v, uint8_t* codes,
                            int64_t code_stride, lut_stream_t stream);

/* Explicit im2col (tensor.py:36-79): cols (batch*ho*wo, cin*kh*kw). */
LUT_API int lut_im2col_f32(const float* x, int32_t batch, int32_t cin, int32_t h, int32_t w,
                   int32_t kh, int32_t kw, int32_t stride, int32_t pad, float* cols,
                   lut_stream_t stream);

/*
 * fp32 lookup-aggregate.  Replaces lut_gather_f32 / lut_matmul_ref
 * (kernels.py:138-140, pq.py:196-214) plus the bias add of lut_layer_infer
 * (kernels.py:176-177): out[n,m] = act(fl(sum_c T[c, code[n,c], m]) + bias[m]),
 * the sum in f32 in ascending c from +0.0 — bitwise equal to the reference.
 * bias may be NULL (no add).  out_hw > 0 writes NCHW: row n = (b, p) with
 * p < out_hw goes to out[(b*m + col)*out_hw + p] (Conv._raise, model.py:113-114).
 */
LUT_API int lut_gather_f32(const uint8_t* codes, int32_t code_bits, int64_t n, int32_t c, int32_t k,
                   int32_t m, const float* table, const float* bias, int32_t act, float* out,
                   int64_t out_hw, int32_t* err_flag, lut_stream_t stream);

/*
 * int8 lookup-aggregate.  Replaces lut_gather_i32 + lut_gather_accumulate
 * (kernels.py:105-135): exact int32 sums of int8 entries; out_i32 (may be NULL)
 * receives them; out (may be NULL) receives fl(f32(acc) * scale) [+ bias, act]
 * with no FMA contraction (bitwise equal to the reference).
 * scales: device f32; scale_mtile == 0 -> one scale (reference, quant.py:22-27);
 * scale_mtile > 0 -> scales[col / scale_mtile] (BASELINE config 2 extension).
 */
LUT_API int lut_gather_i8(const uint8_t* codes, int32_t code_bits, int64_t n, int32_t c, int32_t k,
                  int32_t m, const int8_t* q, const float* scales, int32_t scale_mtile,
                  const float* bias, int32_t act, float* out, int32_t* out_i32, int64_t out_hw,
                  int32_t* err_flag, lut_stream_t stream);

/* Table build (pq.py:177-193): f32 multiply then f32 add, j ascending. */
LUT_API int lut_build_table_f32(const float* b, int32_t m, const float* books, int32_t c, int32_t k,
                        int32_t v, float* table, lut_stream_t stream);

/*
 * Dense reference product (tensor.py:110-125, matmul_ref): out (n, m) =
 * a (n, d) @ b (d, m), each product rounded to f32 and added in ascending k
 * from +0.0 (no FMA) -- bitwise equal to the reference.  The dense baseline of
 * bench_kernel (kernels.py:288-349), not part of the LUT path.
 */
LUT_API int lut_matmul_ref_f32(const float* a, const float* b, int64_t n, int32_t d, int32_t m, float* out,
                               lut_stream_t stream);

/* Bytes of scratch for lut_quantize_table(). */
LUT_API size_t lut_quantize_scratch_bytes(int32_t c, int32_t k, int32_t m, int32_t scale_mtile);

/*
 * Symmetric int8 quantization (quant.py:40-57): scale = f32(f64(max|T|)/127)
 * (1.0 for an all-zero table), q = clip(rint_half_even(f64 T / f64 scale), +-127).
 * scale_mtile > 0 quantizes each m-tile with its own scale (extension).
 * A non-finite entry raises LUT_ERR_DATA through err_flag.
 */
LUT_API int lut_quantize_table(const float* table, int32_t c, int32_t k, int32_t m, int32_t scale_mtile,
                       int8_t* q, float* scales, void* scratch, int32_t* err_flag,
                       lut_stream_t stream);

/*
 * Tensor-core lookup-aggregate (Eq. 4: out = onehot(codes) . T as a
 * tcgen05 kind::i8 GEMM with inner dim c*k; power-of-two k <= 128).
 * The table is first laid out once per layer as a swizzled "B image":
 *   digits == 1: from the int8 table q — the int32 sums are EXACT, so the
 *                result is bitwise equal to lut_gather_i8 (kernels.py:105-135);
 *   digits == 2 or 4: from an f32 table, as balanced int8 digit planes of
 *                s_m * t (per-column scale s_m, |t| <= 2^(8*digits-2)); sums are
 *                exact integers rounded once to f32 (|error| <= c * s_m / 2;
 *                4 digits: c * max|T[:,:,m]| * 2^-31), within the fp32 contract.
 * lut_onehot_image_bytes() returns 0 when the shape is not supported.
 * codes rows must be 16-byte aligned: code_stride % 16 == 0 (use the padded
 * stride lut_code_stride()); codes are not range-checked on this path
 * (use it on codes produced by lut_encode_f32).
 */
LUT_API size_t lut_onehot_image_bytes(int32_t c, int32_t k, int32_t m, int32_t digits);
LUT_API int lut_onehot_prepare_i8(const int8_t* q, int32_t c, int32_t k, int32_t m, void* image,
                                  lut_stream_t stream);
LUT_API int lut_onehot_prepare_f32(const float* table, int32_t c, int32_t k, int32_t m, int32_t digits,
                                   void* image, int32_t* err_flag, lut_stream_t stream);
LUT_API int lut_gather_onehot(const uint8_t* codes, int64_t code_stride, int64_t n, int32_t c, int32_t k,
                              int32_t m, int32_t digits, const void* image, const float* scales,
                              int32_t scale_mtile, const float* bias, int32_t act, float* out,
                              int32_t* out_i32, int64_t out_hw, lut_stream_t stream);

/* Padded u8 code row stride (bytes) used by the layer path: round_up(c, 16). */
LUT_API int64_t lut_code_stride(int32_t c);

/*
 * Synchronize `stream`, read and clear the device error flag; returns the
 * status it held (LUT_OK, LUT_ERR_DATA or LUT_ERR_CORRUPTION) or LUT_ERR_CUDA.
 */
LUT_API int lut_read_status(int32_t* err_flag, lut_stream_t stream);

/* ---------------------------------------------------------------- layers */

/* A LUT layer as the device sees it (LutLayer, softpq.py:82-172). */
typedef struct lut_layer_desc {
  int32_t c, k, v, m;
  const void* books_prep;  /* from lut_prepare_books */
  const float* table;      /* (c,k,m) f32, or NULL */
  const int8_t* q;         /* (c,k,m) i8, or NULL */
  const float* scales;     /* device f32 */
  int32_t scale_mtile;     /* 0 = one scale */
  const float* bias;       /* (m) or NULL */
  int32_t act;             /* lut_act */
  int32_t integer;         /* 1 -> int8 path (needs q), 0 -> f32 path (needs table) */
  const void* onehot_image; /* optional tensor-core B image for the selected path, or NULL */
  int32_t onehot_digits;   /* 1 for the int8 path; 2 or 4 for the f32 path */
} lut_layer_desc;

/*
 * Full layer: encode -> lookup-aggregate -> bias/act.  Replaces
 * lut_layer_infer (kernels.py:143-178) with encoder="dist".  With an
 * onehot_image the lookup runs on the tensor cores, else on the CUDA cores.
 * codes_scratch: n * lut_code_stride(c) bytes (device, 16-byte aligned).
 */
LUT_API int lut_layer_forward(const lut_layer_desc* layer, const float* a, int64_t n, float* out,
                      uint8_t* codes_scratch, int32_t* near_tie_count, lut_stream_t stream);

/*
 * Full conv layer (LutConv.forward, model.py:199-203 with Conv._lower/_raise,
 * model.py:105-114): NCHW input x (batch, cin, h, w) -> encode of every
 * kh x kw patch (im2col fused, tensor.py:36-79) -> lookup-aggregate -> bias/act
 * -> NCHW output (batch, m, ho, wo).  codes_scratch: batch*ho*wo *
 * lut_code_stride(c) bytes.  The lookup is launched as a programmatic dependent
 * of the encode (it stages its table slice while the encode finishes).
 */
LUT_API int lut_conv_layer_forward(const lut_layer_desc* layer, const float* x, int32_t batch, int32_t cin,
                                   int32_t h, int32_t w, int32_t kh, int32_t kw, int32_t stride, int32_t pad,
                                   float* out, uint8_t* codes_scratch, int32_t* near_tie_count, lut_stream_t stream);

/*
 * Host-memory executor: the same layer over HOST rows.  Streams row chunks
 * host->device, runs lut_layer_forward, and streams results device->host, with
 * copies and compute overlapped on three streams (copy-in, compute, copy-out)
 * and double-buffered device chunks.  Pinned host buffers reach full PCIe
 * bandwidth; pageable ones work but are staged by the driver.
 */
typedef struct lut_pipeline lut_pipeline;

LUT_API int lut_pipeline_create(int32_t device, int64_t chunk_rows, int32_t d, int32_t m, int32_t c,
                        lut_pipeline** out);
LUT_API int lut_pipeline_run(lut_pipeline* p, const lut_layer_desc* layer, const float* a_host,
                     int64_t n, float* out_host, int32_t* near_tie_count_host);
LUT_API int lut_pipeline_destroy(lut_pipeline* p);

#ifdef __cplusplus
}
#endif
#endif /* LUTGPU_H */
