// extern "C" boundary (include/lutgpu.h): host-side validation mirroring the
// reference's exceptions, dispatch to the kernels, the layer composition
// (lutkit/kernels.py:143-178) and the host-memory executor.

#include <cuda.h>
#include <cuda_runtime.h>

#include <nvtx3/nvToolsExt.h>

#include <map>
#include <mutex>
#include <tuple>
#include <utility>
#include <string>

#include "common.cuh"

namespace {
// NVTX range around the host side of a launch (header-only nvtx3: a no-op
// unless a profiler is attached)
struct NvtxRange {
  bool open = true;
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  void pop() {
    if (open) nvtxRangePop();
    open = false;
  }
  ~NvtxRange() { pop(); }
};
}  // namespace

namespace lutgpu {

// kernels (encode.cu / gather.cu / table.cu)
int prepare_books(const float* books, int C, int K, int V, float* prep, cudaStream_t stream);
int encode_dense(const float* a, int64_t n, int d, const float* prep, int C, int K, int V, uint8_t* codes,
                 int code_bits, int64_t code_stride, int* near_tie, cudaStream_t stream, int force_generic);
int onehot_supported(int C, int K, int M, int digits);
size_t onehot_image_bytes(int C, int K, int M, int digits);
int onehot_prepare_i8(const int8_t* q, int C, int K, int M, void* image, cudaStream_t stream);
int onehot_prepare_f32(const float* t, int C, int K, int M, int digits, void* image, int* err, cudaStream_t stream);
int onehot_gather(const uint8_t* codes, int64_t code_stride, int64_t n, int C, int K, int M, int digits,
                  const void* image, const float* scales, int scale_mtile, const float* bias, int act, float* out,
                  int32_t* out_i32, int64_t out_hw, cudaStream_t stream, int pdl = 0);
int encode_conv_strided(const float* x, int batch, int cin, int h, int w, int kh, int kw, int stride, int pad,
                        const float* prep, int C, int K, int V, uint8_t* codes, int64_t code_stride, int* near_tie,
                        cudaStream_t stream);
int encode_conv(const float* x, int batch, int cin, int h, int w, int kh, int kw, int stride, int pad,
                const float* prep, int C, int K, int V, uint8_t* codes, int code_bits, int* near_tie,
                cudaStream_t stream);
int encode_hash(const float* a, int64_t n, int d, const int* dims, const float* thr, const uint8_t* leaves, int C,
                int L, int V, uint8_t* codes, int64_t code_stride, cudaStream_t stream);
int im2col(const float* x, int batch, int cin, int h, int w, int kh, int kw, int stride, int pad, float* cols,
           cudaStream_t stream);
int gather_f32(const uint8_t* codes, int code_bits, int64_t n, int C, int K, int M, const float* table,
               const float* bias, int act, float* out, int64_t out_hw, int* err, cudaStream_t stream,
               int force_generic);
int gather_i8(const uint8_t* codes, int code_bits, int64_t n, int C, int K, int M, const int8_t* q,
              const float* scales, int scale_mtile, const float* bias, int act, float* out, int32_t* out_i32,
              int64_t out_hw, int* err, cudaStream_t stream, int force_generic);
int gather_f32_strided(const uint8_t* codes, int code_bits, int64_t code_stride, int64_t n, int C, int K, int M,
                       const float* table, const float* bias, int act, float* out, int64_t out_hw, int* err,
                       cudaStream_t stream, int force_generic, int pdl = 0);
int gather_i8_strided(const uint8_t* codes, int code_bits, int64_t code_stride, int64_t n, int C, int K, int M,
                      const int8_t* q, const float* scales, int scale_mtile, const float* bias, int act, float* out,
                      int32_t* out_i32, int64_t out_hw, int* err, cudaStream_t stream, int force_generic, int pdl = 0);
int build_table(const float* b, int M, const float* books, int C, int K, int V, float* table,
                cudaStream_t stream);

size_t quantize_scratch_bytes(int C, int K, int M, int mtile);
int matmul_ref(const float* a, const float* b, int64_t n, int d, int m, float* out, cudaStream_t stream);
int quantize_table(const float* t, int C, int K, int M, int mtile, int8_t* q, float* scales, void* scratch,
                   int* err, cudaStream_t stream);

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return LUT_ERR_CUDA;
}

static int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  return dev;
}

int num_sms() {
  static int cache[64] = {};
  const int dev = current_device();
  if (!cache[dev]) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

size_t max_smem_optin() {
  static int cache[64] = {};
  const int dev = current_device();
  if (!cache[dev]) {
    int n = 227 * 1024;
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cache[dev] = n;
  }
  return (size_t)cache[dev];
}

// Per-(kernel, device) launch setup, done once: the dynamic shared-memory limit
// is raised to the device maximum, and occupancies are cached per (threads,
// smem).  Both driver calls cost microseconds, which small LUT layers (tens of
// microseconds of GPU time) would otherwise pay on every call.
namespace {
std::mutex g_kernel_mu;
std::map<std::pair<const void*, int>, bool> g_smem_set;
std::map<std::tuple<const void*, int, int, size_t>, int> g_occ;
}  // namespace

cudaError_t kernel_smem_attr(const void* func) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(g_kernel_mu);
  auto key = std::make_pair(func, dev);
  if (g_smem_set.count(key)) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem_optin());
  if (e == cudaSuccess) g_smem_set[key] = true;
  return e;
}

int kernel_occupancy(const void* func, int threads, size_t smem) {
  const int dev = current_device();
  {
    std::lock_guard<std::mutex> lk(g_kernel_mu);
    auto it = g_occ.find(std::make_tuple(func, dev, threads, smem));
    if (it != g_occ.end()) return it->second;
  }
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, threads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  std::lock_guard<std::mutex> lk(g_kernel_mu);
  g_occ[std::make_tuple(func, dev, threads, smem)] = per_sm;
  return per_sm;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

static bool make_tmap_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t cols,
                         uint64_t rows, uint64_t row_stride_bytes, uint32_t box_cols, uint32_t box_rows,
                         bool swizzle128, CUtensorMapSwizzle swz_override = CU_TENSOR_MAP_SWIZZLE_NONE) {
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t elem[2] = {1, 1};
  CUresult r = fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : swz_override,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_2d_f32(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint32_t box_cols,
                      uint32_t box_rows, bool swizzle128) {
  if ((cols * 4) % 16 != 0) return false;
  return make_tmap_2d(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, base, cols, rows, cols * 4, box_cols, box_rows,
                      swizzle128);
}

bool make_tmap_2d_f32_box(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint32_t box_cols,
                          uint32_t box_rows) {
  if ((cols * 4) % 16 != 0) return false;
  CUtensorMapSwizzle swz = box_cols == 32   ? CU_TENSOR_MAP_SWIZZLE_128B
                           : box_cols == 16 ? CU_TENSOR_MAP_SWIZZLE_64B
                           : box_cols == 8  ? CU_TENSOR_MAP_SWIZZLE_32B
                                            : CU_TENSOR_MAP_SWIZZLE_NONE;
  return make_tmap_2d(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, base, cols, rows, cols * 4, box_cols, box_rows, false, swz);
}

bool make_tmap_2d_u8(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t row_stride_bytes,
                     uint32_t box_cols, uint32_t box_rows, bool swizzle128) {
  if (row_stride_bytes % 16 != 0) return false;
  return make_tmap_2d(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, base, cols, rows, row_stride_bytes, box_cols, box_rows,
                      swizzle128);
}

// ---------------------------------------------------------------- checks

static int check_geometry(int C, int K, int V) {
  if (C < 0) return fail(LUT_ERR_CONFIG, "codebook count must be >= 0");
  if (V < 1) return fail(LUT_ERR_CONFIG, "sub-vector length must be >= 1");
  if (K < 1 || K > 256) return fail(LUT_ERR_CONFIG, "centroid count must be in [1, 256]");
  return LUT_OK;
}

static int check_codes(int code_bits, int K) {
  if (code_bits != 8 && code_bits != 4) return fail(LUT_ERR_CONFIG, "code_bits must be 8 or 4");
  if (code_bits == 4 && K > 16) return fail(LUT_ERR_CONFIG, "4-bit codes need K <= 16");
  return LUT_OK;
}

static int check_act(int act) {
  if (act != LUT_ACT_NONE && act != LUT_ACT_RELU && act != LUT_ACT_GELU)
    return fail(LUT_ERR_CONFIG, "unknown activation");
  return LUT_OK;
}

static int force_generic_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = probe_env("LUTGPU_FORCE_GENERIC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v;
}

#define LUT_TRY(expr)              \
  do {                             \
    int _s = (expr);               \
    if (_s != LUT_OK) return _s;   \
  } while (0)

}  // namespace lutgpu

using namespace lutgpu;

extern "C" {

int lut_version(void) { return 100; }

const char* lut_last_error(void) { return g_last_error.c_str(); }

size_t lut_books_prep_bytes(int32_t c, int32_t k, int32_t v) {
  if (c < 0 || k < 1 || v < 1) return 0;
  return (size_t)c * prep_stride(k, v) * sizeof(float);
}

int lut_prepare_books(const float* books, int32_t c, int32_t k, int32_t v, void* books_prep,
                      lut_stream_t stream) {
  LUT_TRY(check_geometry(c, k, v));
  if (c > 0 && (!books || !books_prep)) return fail(LUT_ERR_CONFIG, "null pointer");
  return prepare_books(books, c, k, v, static_cast<float*>(books_prep), (cudaStream_t)stream);
}

int lut_encode_f32(const float* a, int64_t n, int32_t d, const void* books_prep, int32_t c, int32_t k, int32_t v,
                   uint8_t* codes, int32_t code_bits, int64_t code_stride, int32_t* near_tie_count,
                   lut_stream_t stream) {
  LUT_TRY(check_geometry(c, k, v));
  LUT_TRY(check_codes(code_bits, k));
  if (n < 0) return fail(LUT_ERR_CONFIG, "row count must be >= 0");
  if ((int64_t)c * v != d) return fail(LUT_ERR_CONFIG, "input cols != C*V");
  if (n > 0 && c > 0 && (!a || !books_prep || !codes)) return fail(LUT_ERR_CONFIG, "null pointer");
  const int64_t dense = code_bits == 4 ? (c + 1) / 2 : c;
  if (code_stride != 0 && code_stride < dense) return fail(LUT_ERR_CONFIG, "code_stride smaller than a code row");
  const int64_t stride = code_stride ? code_stride : dense;
  return encode_dense(a, n, d, static_cast<const float*>(books_prep), c, k, v, codes, code_bits, stride,
                      near_tie_count, (cudaStream_t)stream, force_generic_env());
}

static int conv_dims(int32_t batch, int32_t cin, int32_t h, int32_t w, int32_t kh, int32_t kw, int32_t stride,
                     int32_t pad) {
  if (batch < 0 || cin < 1 || h < 1 || w < 1) return fail(LUT_ERR_CONFIG, "bad NCHW shape");
  if (stride < 1) return fail(LUT_ERR_CONFIG, "stride must be >= 1");
  if (pad < 0) return fail(LUT_ERR_CONFIG, "pad must be >= 0");
  if (kh < 1 || kw < 1 || kh > h + 2 * pad || kw > w + 2 * pad)
    return fail(LUT_ERR_CONFIG, "kernel does not fit padded input");
  return LUT_OK;
}

int lut_encode_conv_f32(const float* x, int32_t batch, int32_t cin, int32_t h, int32_t w, int32_t kh, int32_t kw,
                        int32_t stride, int32_t pad, const void* books_prep, int32_t c, int32_t k, int32_t v,
                        uint8_t* codes, int32_t code_bits, int32_t* near_tie_count, lut_stream_t stream) {
  LUT_TRY(conv_dims(batch, cin, h, w, kh, kw, stride, pad));
  LUT_TRY(check_geometry(c, k, v));
  LUT_TRY(check_codes(code_bits, k));
  if ((int64_t)c * v != (int64_t)cin * kh * kw) return fail(LUT_ERR_CONFIG, "patch cols != C*V");
  if (batch > 0 && (!x || !books_prep || !codes)) return fail(LUT_ERR_CONFIG, "null pointer");
  return encode_conv(x, batch, cin, h, w, kh, kw, stride, pad, static_cast<const float*>(books_prep), c, k, v,
                     codes, code_bits, near_tie_count, (cudaStream_t)stream);
}

int lut_encode_hash(const float* a, int64_t n, int32_t d, const int32_t* dims, const float* thresholds,
                    const uint8_t* leaves, int32_t c, int32_t levels, int32_t v, uint8_t* codes, int64_t code_stride,
                    lut_stream_t stream) {
  if (n < 0 || c < 0 || v < 1) return fail(LUT_ERR_CONFIG, "bad hash-encode geometry");
  if (levels < 1 || levels > 16) return fail(LUT_ERR_CONFIG, "tree depth must be in [1, 16]");
  if ((int64_t)c * v != d) return fail(LUT_ERR_CONFIG, "input cols not divisible into the trees");
  if (code_stride != 0 && code_stride < c) return fail(LUT_ERR_CONFIG, "code_stride smaller than a code row");
  if (n > 0 && c > 0 && (!a || !dims || !thresholds || !leaves || !codes)) return fail(LUT_ERR_CONFIG, "null pointer");
  return encode_hash(a, n, d, dims, thresholds, leaves, c, levels, v, codes, code_stride ? code_stride : c,
                     (cudaStream_t)stream);
}

int lut_im2col_f32(const float* x, int32_t batch, int32_t cin, int32_t h, int32_t w, int32_t kh, int32_t kw,
                   int32_t stride, int32_t pad, float* cols, lut_stream_t stream) {
  LUT_TRY(conv_dims(batch, cin, h, w, kh, kw, stride, pad));
  if (batch > 0 && (!x || !cols)) return fail(LUT_ERR_CONFIG, "null pointer");
  return im2col(x, batch, cin, h, w, kh, kw, stride, pad, cols, (cudaStream_t)stream);
}

int lut_gather_f32(const uint8_t* codes, int32_t code_bits, int64_t n, int32_t c, int32_t k, int32_t m,
                   const float* table, const float* bias, int32_t act, float* out, int64_t out_hw,
                   int32_t* err_flag, lut_stream_t stream) {
  LUT_TRY(check_geometry(c, k, 1));
  LUT_TRY(check_codes(code_bits, k));
  LUT_TRY(check_act(act));
  if (n < 0 || m < 0 || out_hw < 0) return fail(LUT_ERR_CONFIG, "negative size");
  if (out_hw > 0 && n % out_hw != 0) return fail(LUT_ERR_CONFIG, "rows not a multiple of out_hw");
  if (n > 0 && m > 0 && (!codes && c > 0)) return fail(LUT_ERR_CONFIG, "null codes");
  if (n > 0 && m > 0 && (!out || (c > 0 && !table))) return fail(LUT_ERR_CONFIG, "null pointer");
  return gather_f32(codes, code_bits, n, c, k, m, table, bias, act, out, out_hw, err_flag, (cudaStream_t)stream,
                    force_generic_env());
}

int lut_gather_i8(const uint8_t* codes, int32_t code_bits, int64_t n, int32_t c, int32_t k, int32_t m,
                  const int8_t* q, const float* scales, int32_t scale_mtile, const float* bias, int32_t act,
                  float* out, int32_t* out_i32, int64_t out_hw, int32_t* err_flag, lut_stream_t stream) {
  LUT_TRY(check_geometry(c, k, 1));
  LUT_TRY(check_codes(code_bits, k));
  LUT_TRY(check_act(act));
  if (n < 0 || m < 0 || out_hw < 0 || scale_mtile < 0) return fail(LUT_ERR_CONFIG, "negative size");
  if (out_hw > 0 && n % out_hw != 0) return fail(LUT_ERR_CONFIG, "rows not a multiple of out_hw");
  if (n > 0 && m > 0) {
    if (!out && !out_i32) return fail(LUT_ERR_CONFIG, "no output requested");
    if (c > 0 && (!codes || !q)) return fail(LUT_ERR_CONFIG, "null pointer");
    if (out && !scales) return fail(LUT_ERR_CONFIG, "null scales");
  }
  return gather_i8(codes, code_bits, n, c, k, m, q, scales, scale_mtile, bias, act, out, out_i32, out_hw, err_flag,
                   (cudaStream_t)stream, force_generic_env());
}

int lut_build_table_f32(const float* b, int32_t m, const float* books, int32_t c, int32_t k, int32_t v, float* table,
                        lut_stream_t stream) {
  LUT_TRY(check_geometry(c, k, v));
  if (m < 0) return fail(LUT_ERR_CONFIG, "negative m");
  if ((int64_t)c * k * m > 0 && (!b || !books || !table)) return fail(LUT_ERR_CONFIG, "null pointer");
  return build_table(b, m, books, c, k, v, table, (cudaStream_t)stream);
}

int lut_matmul_ref_f32(const float* a, const float* b, int64_t n, int32_t d, int32_t m, float* out,
                       lut_stream_t stream) {
  if (n < 0 || d < 0 || m < 0) return fail(LUT_ERR_CONFIG, "negative size");
  if (n > 0 && m > 0 && (!out || (d > 0 && (!a || !b)))) return fail(LUT_ERR_CONFIG, "null pointer");
  return matmul_ref(a, b, n, d, m, out, (cudaStream_t)stream);
}

size_t lut_quantize_scratch_bytes(int32_t c, int32_t k, int32_t m, int32_t scale_mtile) {
  return quantize_scratch_bytes(c, k, m, scale_mtile);
}

int lut_quantize_table(const float* table, int32_t c, int32_t k, int32_t m, int32_t scale_mtile, int8_t* q,
                       float* scales, void* scratch, int32_t* err_flag, lut_stream_t stream) {
  if (c < 0 || k < 0 || m < 0 || scale_mtile < 0) return fail(LUT_ERR_CONFIG, "negative size");
  if (!scales || !scratch || ((int64_t)c * k * m > 0 && (!table || !q))) return fail(LUT_ERR_CONFIG, "null pointer");
  return quantize_table(table, c, k, m, scale_mtile, q, scales, scratch, err_flag, (cudaStream_t)stream);
}

size_t lut_onehot_image_bytes(int32_t c, int32_t k, int32_t m, int32_t digits) {
  if (c < 1 || k < 1 || m < 1) return 0;
  if (!onehot_supported(c, k, m, digits)) return 0;
  return onehot_image_bytes(c, k, m, digits);
}

int lut_onehot_prepare_i8(const int8_t* q, int32_t c, int32_t k, int32_t m, void* image, lut_stream_t stream) {
  if (!lut_onehot_image_bytes(c, k, m, 1)) return fail(LUT_ERR_CONFIG, "shape not supported by the one-hot gather");
  if (!q || !image) return fail(LUT_ERR_CONFIG, "null pointer");
  return onehot_prepare_i8(q, c, k, m, image, (cudaStream_t)stream);
}

int lut_onehot_prepare_f32(const float* table, int32_t c, int32_t k, int32_t m, int32_t digits, void* image,
                           int32_t* err_flag, lut_stream_t stream) {
  if (digits < 2 || !lut_onehot_image_bytes(c, k, m, digits))
    return fail(LUT_ERR_CONFIG, "shape/digits not supported by the one-hot gather");
  if (!table || !image) return fail(LUT_ERR_CONFIG, "null pointer");
  return onehot_prepare_f32(table, c, k, m, digits, image, err_flag, (cudaStream_t)stream);
}

int lut_gather_onehot(const uint8_t* codes, int64_t code_stride, int64_t n, int32_t c, int32_t k, int32_t m,
                      int32_t digits, const void* image, const float* scales, int32_t scale_mtile, const float* bias,
                      int32_t act, float* out, int32_t* out_i32, int64_t out_hw, lut_stream_t stream) {
  LUT_TRY(check_act(act));
  if (n < 0 || m < 0 || out_hw < 0 || scale_mtile < 0) return fail(LUT_ERR_CONFIG, "negative size");
  if (out_hw > 0 && n % out_hw != 0) return fail(LUT_ERR_CONFIG, "rows not a multiple of out_hw");
  if (!lut_onehot_image_bytes(c, k, m, digits)) return fail(LUT_ERR_CONFIG, "shape not supported by the one-hot gather");
  if (n > 0 && (!codes || !image || (!out && !out_i32))) return fail(LUT_ERR_CONFIG, "null pointer");
  if (digits == 1 && out && !scales) return fail(LUT_ERR_CONFIG, "null scales");
  if (digits > 1 && out_i32) return fail(LUT_ERR_CONFIG, "int32 output only exists for digits == 1");
  return onehot_gather(codes, code_stride, n, c, k, m, digits, image, scales, scale_mtile, bias, act, out, out_i32,
                       out_hw, (cudaStream_t)stream);
}

int64_t lut_code_stride(int32_t c) { return c <= 0 ? 16 : ((int64_t)c + 15) / 16 * 16; }

int lut_read_status(int32_t* err_flag, lut_stream_t stream) {
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  if (!err_flag) return LUT_OK;
  int32_t h = 0;
  e = cudaMemcpy(&h, err_flag, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(err_flag)");
  if (h != 0) {
    e = cudaMemset(err_flag, 0, sizeof(int32_t));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(err_flag)");
    if (h == LUT_ERR_CORRUPTION) return fail(h, "encoding index >= K");
    if (h == LUT_ERR_DATA) return fail(h, "table contains NaN or infinity");
    return fail(h, "device error flag set");
  }
  return LUT_OK;
}

// ----------------------------------------------------------------- layers

static int check_layer(const lut_layer_desc* L) {
  if (!L) return fail(LUT_ERR_CONFIG, "null layer");
  LUT_TRY(check_geometry(L->c, L->k, L->v));
  LUT_TRY(check_act(L->act));
  if (L->m < 0) return fail(LUT_ERR_CONFIG, "negative m");
  if (!L->books_prep && L->c > 0) return fail(LUT_ERR_CONFIG, "layer has no prepared codebooks");
  if (L->integer) {
    if (!L->q || !L->scales) return fail(LUT_ERR_CONFIG, "integer path requested but the layer has no quantized table");
  } else if (!L->table && L->c > 0) {
    return fail(LUT_ERR_CONFIG, "float path requested but the layer has no table");
  }
  return LUT_OK;
}

int lut_layer_forward(const lut_layer_desc* L, const float* a, int64_t n, float* out, uint8_t* codes_scratch,
                      int32_t* near_tie_count, lut_stream_t stream) {
  LUT_TRY(check_layer(L));
  if (n < 0) return fail(LUT_ERR_CONFIG, "row count must be >= 0");
  if (n == 0 || L->m == 0) return LUT_OK;
  if (!out || (L->c > 0 && (!a || !codes_scratch))) return fail(LUT_ERR_CONFIG, "null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const int d = L->c * L->v;
  const int64_t stride = lut_code_stride(L->c);
  NvtxRange r_enc("lut.encode");
  LUT_TRY(encode_dense(a, n, d, static_cast<const float*>(L->books_prep), L->c, L->k, L->v, codes_scratch, 8, stride,
                       near_tie_count, s, force_generic_env()));
  r_enc.pop();
  NvtxRange r_gat("lut.gather");
  if (L->onehot_image) {
    const int digits = L->integer ? 1 : L->onehot_digits;
    return onehot_gather(codes_scratch, stride, n, L->c, L->k, L->m, digits, L->onehot_image, L->scales,
                         L->scale_mtile, L->bias, L->act, out, nullptr, 0, s, /*pdl=*/1);
  }
  if (L->integer)
    return gather_i8_strided(codes_scratch, 8, stride, n, L->c, L->k, L->m, L->q, L->scales, L->scale_mtile, L->bias,
                             L->act, out, nullptr, 0, nullptr, s, force_generic_env(), /*pdl=*/1);
  return gather_f32_strided(codes_scratch, 8, stride, n, L->c, L->k, L->m, L->table, L->bias, L->act, out, 0, nullptr,
                            s, force_generic_env(), /*pdl=*/1);
}

int lut_conv_layer_forward(const lut_layer_desc* L, const float* x, int32_t batch, int32_t cin, int32_t h, int32_t w,
                           int32_t kh, int32_t kw, int32_t stride, int32_t pad, float* out, uint8_t* codes_scratch,
                           int32_t* near_tie_count, lut_stream_t stream) {
  LUT_TRY(check_layer(L));
  LUT_TRY(conv_dims(batch, cin, h, w, kh, kw, stride, pad));
  if ((int64_t)L->c * L->v != (int64_t)cin * kh * kw) return fail(LUT_ERR_CONFIG, "patch cols != C*V");
  const int ho = (h + 2 * pad - kh) / stride + 1, wo = (w + 2 * pad - kw) / stride + 1;
  const int64_t n = (int64_t)batch * ho * wo;
  if (n == 0 || L->m == 0) return LUT_OK;
  if (!x || !out || !codes_scratch) return fail(LUT_ERR_CONFIG, "null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t stride_c = lut_code_stride(L->c);
  NvtxRange r_enc("lut.conv.encode");
  LUT_TRY(encode_conv_strided(x, batch, cin, h, w, kh, kw, stride, pad, static_cast<const float*>(L->books_prep),
                              L->c, L->k, L->v, codes_scratch, stride_c, near_tie_count, s));
  r_enc.pop();
  NvtxRange r_gat("lut.conv.gather");
  if (L->onehot_image) {
    const int digits = L->integer ? 1 : L->onehot_digits;
    return onehot_gather(codes_scratch, stride_c, n, L->c, L->k, L->m, digits, L->onehot_image, L->scales,
                         L->scale_mtile, L->bias, L->act, out, nullptr, (int64_t)ho * wo, s, /*pdl=*/1);
  }
  if (L->integer)
    return gather_i8_strided(codes_scratch, 8, stride_c, n, L->c, L->k, L->m, L->q, L->scales, L->scale_mtile, L->bias,
                             L->act, out, nullptr, (int64_t)ho * wo, nullptr, s, force_generic_env(), /*pdl=*/1);
  return gather_f32_strided(codes_scratch, 8, stride_c, n, L->c, L->k, L->m, L->table, L->bias, L->act, out,
                            (int64_t)ho * wo, nullptr, s, force_generic_env(), /*pdl=*/1);
}

// --------------------------------------------------------- host executor

struct lut_pipeline {
  int device;
  int64_t chunk_rows;
  int d, m, c;
  float* dA[2];
  float* dOut[2];
  uint8_t* dCodes[2];
  int32_t* dNear;
  cudaStream_t s_in, s_comp, s_out;
  cudaEvent_t ev_in[2], ev_comp[2], ev_out[2];
};

int lut_pipeline_destroy(lut_pipeline* p) {
  if (!p) return LUT_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  for (int i = 0; i < 2; ++i) {
    cudaFree(p->dA[i]);
    cudaFree(p->dOut[i]);
    cudaFree(p->dCodes[i]);
    if (p->ev_in[i]) cudaEventDestroy(p->ev_in[i]);
    if (p->ev_comp[i]) cudaEventDestroy(p->ev_comp[i]);
    if (p->ev_out[i]) cudaEventDestroy(p->ev_out[i]);
  }
  cudaFree(p->dNear);
  if (p->s_in) cudaStreamDestroy(p->s_in);
  if (p->s_comp) cudaStreamDestroy(p->s_comp);
  if (p->s_out) cudaStreamDestroy(p->s_out);
  delete p;
  cudaSetDevice(prev);
  return LUT_OK;
}

int lut_pipeline_create(int32_t device, int64_t chunk_rows, int32_t d, int32_t m, int32_t c, lut_pipeline** out) {
  if (!out) return fail(LUT_ERR_CONFIG, "null out");
  *out = nullptr;
  if (chunk_rows < 1 || d < 0 || m < 0 || c < 0) return fail(LUT_ERR_CONFIG, "bad pipeline geometry");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  lut_pipeline* p = new lut_pipeline();
  p->device = device;
  p->chunk_rows = chunk_rows;
  p->d = d;
  p->m = m;
  p->c = c;
  bool ok = true;
  for (int i = 0; i < 2 && ok; ++i) {
    ok &= cudaMalloc(&p->dA[i], (size_t)chunk_rows * (d > 0 ? d : 1) * sizeof(float)) == cudaSuccess;
    ok &= cudaMalloc(&p->dOut[i], (size_t)chunk_rows * (m > 0 ? m : 1) * sizeof(float)) == cudaSuccess;
    ok &= cudaMalloc(&p->dCodes[i], (size_t)chunk_rows * lut_code_stride(c)) == cudaSuccess;
    ok &= cudaEventCreateWithFlags(&p->ev_in[i], cudaEventDisableTiming) == cudaSuccess;
    ok &= cudaEventCreateWithFlags(&p->ev_comp[i], cudaEventDisableTiming) == cudaSuccess;
    ok &= cudaEventCreateWithFlags(&p->ev_out[i], cudaEventDisableTiming) == cudaSuccess;
  }
  ok = ok && cudaMalloc(&p->dNear, sizeof(int32_t)) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&p->s_comp, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking) == cudaSuccess;
  cudaSetDevice(prev);
  if (!ok) {
    lut_pipeline_destroy(p);
    return fail(LUT_ERR_CUDA, "pipeline allocation failed");
  }
  *out = p;
  return LUT_OK;
}

int lut_pipeline_run(lut_pipeline* p, const lut_layer_desc* L, const float* a_host, int64_t n, float* out_host,
                     int32_t* near_tie_count_host) {
  if (!p) return fail(LUT_ERR_CONFIG, "null pipeline");
  LUT_TRY(check_layer(L));
  if (L->c * L->v != p->d || L->m != p->m || L->c != p->c) return fail(LUT_ERR_CONFIG, "layer/pipeline mismatch");
  if (n < 0) return fail(LUT_ERR_CONFIG, "row count must be >= 0");
  if (n > 0 && (!a_host || !out_host)) return fail(LUT_ERR_CONFIG, "null host pointer");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  int status = LUT_OK;
  cudaError_t e = cudaMemsetAsync(p->dNear, 0, sizeof(int32_t), p->s_comp);
  const int64_t nchunks = (n + p->chunk_rows - 1) / p->chunk_rows;
  for (int64_t i = 0; i < nchunks && e == cudaSuccess && status == LUT_OK; ++i) {
    const int b = (int)(i & 1);
    const int64_t r0 = i * p->chunk_rows;
    const int64_t rows = (n - r0) < p->chunk_rows ? (n - r0) : p->chunk_rows;
    // copy-in may reuse dA[b] once compute of chunk i-2 has consumed it
    e = cudaStreamWaitEvent(p->s_in, p->ev_comp[b], 0);
    if (e == cudaSuccess && p->d > 0)
      e = cudaMemcpyAsync(p->dA[b], a_host + r0 * p->d, (size_t)rows * p->d * sizeof(float), cudaMemcpyHostToDevice,
                          p->s_in);
    if (e == cudaSuccess) e = cudaEventRecord(p->ev_in[b], p->s_in);
    // compute waits for its input and for copy-out of chunk i-2 (same out buffer)
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_comp, p->ev_in[b], 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_comp, p->ev_out[b], 0);
    if (e != cudaSuccess) break;
    NvtxRange r_chunk("lut.pipeline.chunk");
    status = lut_layer_forward(L, p->dA[b], rows, p->dOut[b], p->dCodes[b], p->dNear, (lut_stream_t)p->s_comp);
    if (status != LUT_OK) break;
    e = cudaEventRecord(p->ev_comp[b], p->s_comp);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_out, p->ev_comp[b], 0);
    if (e == cudaSuccess && p->m > 0)
      e = cudaMemcpyAsync(out_host + r0 * p->m, p->dOut[b], (size_t)rows * p->m * sizeof(float),
                          cudaMemcpyDeviceToHost, p->s_out);
    if (e == cudaSuccess) e = cudaEventRecord(p->ev_out[b], p->s_out);
  }
  if (e == cudaSuccess && status == LUT_OK) {
    int32_t near = 0;
    e = cudaMemcpyAsync(&near, p->dNear, sizeof(int32_t), cudaMemcpyDeviceToHost, p->s_comp);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->s_comp);
    if (e == cudaSuccess) e = cudaStreamSynchronize(p->s_out);
    if (e == cudaSuccess && near_tie_count_host) *near_tie_count_host = near;
  }
  cudaSetDevice(prev);
  if (status != LUT_OK) return status;
  if (e != cudaSuccess) return cuda_fail(e, "lut_pipeline_run");
  return LUT_OK;
}

}  // extern "C"
