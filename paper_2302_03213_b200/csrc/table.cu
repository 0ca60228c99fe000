// Offline table construction on the device (bit-exact restatements).
//   build_table     pq.py:177-193   T[c,k,m] = sum_j P[c,k,j]*B[cV+j,m], f32 multiply
//                                   then f32 add, j ascending from +0.0 (no FMA).
//   quantize_table  quant.py:40-57  scale = f32(f64 max|T| / 127), 1.0 if all zero;
//                                   q = clip(rint_half_even(f64 T / f64 scale), +-127).
// The m-tile variant (one scale per m-tile shared by all codebooks) is the
// BASELINE config-2 extension; with one tile covering M it is the reference.

#include "common.cuh"

namespace lutgpu {

__global__ void build_table_kernel(const float* __restrict__ b, int M, const float* __restrict__ books, int C,
                                   int K, int V, float* __restrict__ table) {
  const int64_t total = (int64_t)C * K * M;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ck = i / M;
    const int m = (int)(i - ck * M);
    const int c = (int)(ck / K);
    const float* p = books + ck * V;
    const float* bcol = b + (int64_t)c * V * M + m;
    float acc = 0.0f;
    for (int j = 0; j < V; ++j) acc = __fadd_rn(acc, __fmul_rn(__ldg(p + j), __ldg(bcol + (int64_t)j * M)));
    table[i] = acc;
  }
}

// pass 1: per-tile max |T| (as ordered uint bits) and non-finite detection
__global__ void table_maxabs_kernel(const float* __restrict__ t, int64_t CK, int M, int mtile,
                                    unsigned* __restrict__ maxbits, int* err) {
  const int64_t total = CK * M;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float x = t[i];
    if (!isfinite(x)) {
      if (err) atomicMax(err, (int)LUT_ERR_DATA);
      continue;
    }
    const int m = (int)(i % M);
    const int tile = mtile > 0 ? m / mtile : 0;
    atomicMax(maxbits + tile, __float_as_uint(fabsf(x)));
  }
}

__device__ __forceinline__ float tile_scale(unsigned bits) {
  const float maxabs = __uint_as_float(bits);
  if (maxabs == 0.0f) return 1.0f;
  return (float)((double)maxabs / 127.0);
}

// pass 2: scales and codes
__global__ void table_quantize_kernel(const float* __restrict__ t, int64_t CK, int M, int mtile,
                                      const unsigned* __restrict__ maxbits, int ntiles, int8_t* __restrict__ q,
                                      float* __restrict__ scales) {
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < ntiles; i += blockDim.x) scales[i] = tile_scale(maxbits[i]);
  const int64_t total = CK * M;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i % M);
    const int tile = mtile > 0 ? m / mtile : 0;
    const double s = (double)tile_scale(maxbits[tile]);
    double v = rint((double)t[i] / s);
    v = fmin(fmax(v, -127.0), 127.0);
    q[i] = isfinite(t[i]) ? (int8_t)(int)v : (int8_t)0;
  }
}

static int grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 32;
  if (b < 1) b = 1;
  return (int)(b < cap ? b : cap);
}

int build_table(const float* b, int M, const float* books, int C, int K, int V, float* table,
                cudaStream_t stream) {
  const int64_t total = (int64_t)C * K * M;
  if (total == 0) return LUT_OK;
  build_table_kernel<<<grid_for(total), 256, 0, stream>>>(b, M, books, C, K, V, table);
  LUT_CHECK_LAUNCH("build_table_kernel");
  return LUT_OK;
}

size_t quantize_scratch_bytes(int C, int K, int M, int mtile) {
  (void)C;
  (void)K;
  const int ntiles = mtile > 0 ? (M + mtile - 1) / mtile : 1;
  return (size_t)(ntiles > 0 ? ntiles : 1) * sizeof(unsigned);
}

int quantize_table(const float* t, int C, int K, int M, int mtile, int8_t* q, float* scales, void* scratch,
                   int* err, cudaStream_t stream) {
  const int ntiles = mtile > 0 ? (M + mtile - 1) / mtile : 1;
  unsigned* maxbits = static_cast<unsigned*>(scratch);
  cudaError_t e = cudaMemsetAsync(maxbits, 0, (size_t)ntiles * sizeof(unsigned), stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(quantize scratch)");
  const int64_t CK = (int64_t)C * K;
  const int64_t total = CK * M;
  if (total > 0) {
    table_maxabs_kernel<<<grid_for(total), 256, 0, stream>>>(t, CK, M, mtile, maxbits, err);
    LUT_CHECK_LAUNCH("table_maxabs_kernel");
  }
  table_quantize_kernel<<<grid_for(total), 256, 0, stream>>>(t, CK, M, mtile, maxbits, ntiles, q, scales);
  LUT_CHECK_LAUNCH("table_quantize_kernel");
  return LUT_OK;
}

}  // namespace lutgpu
