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

// Dense reference product (tensor.py:110-125, matmul_ref): out[n,m] =
// sum_k a[n,k]*b[k,m] with each product rounded to f32 and added in ascending
// k from +0.0 (numpy's `out += a[:, k:k+1] * b[k:k+1, :]`, no FMA).  Not on the
// LUT path: it is the dense baseline bench_kernel times the LUT layer against.
// 64 x 64 output tile per CTA, 256 threads x (4 rows x 4 cols), k staged
// through SMEM 16 at a time.
__global__ void __launch_bounds__(256) matmul_ref_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                         int N, int D, int M, float* __restrict__ out) {
  __shared__ float as[16][64 + 1];
  __shared__ float bs[16][64];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t row0 = (int64_t)blockIdx.y * 64, col0 = (int64_t)blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < D; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      const int kk = i & 15, r = i >> 4;  // a tile: 64 rows x 16 k
      const int64_t gr = row0 + r;
      as[kk][r] = (gr < N && k0 + kk < D) ? __ldg(a + gr * D + k0 + kk) : 0.0f;
      const int cc = i & 63, kb = i >> 6;  // b tile: 16 k x 64 cols
      const int64_t gc = col0 + cc;
      bs[kb][cc] = (gc < M && k0 + kb < D) ? __ldg(b + (int64_t)(k0 + kb) * M + gc) : 0.0f;
    }
    __syncthreads();
    const int kn = min(16, D - k0);
    for (int kk = 0; kk < kn; ++kk) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float av = as[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fadd_rn(acc[i][j], __fmul_rn(av, bs[kk][tx * 4 + j]));
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = row0 + ty * 4 + i;
    if (r >= N) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = col0 + tx * 4 + j;
      if (c < M) out[r * M + c] = acc[i][j];
    }
  }
}

int matmul_ref(const float* a, const float* b, int64_t n, int d, int m, float* out, cudaStream_t stream) {
  if (n == 0 || m == 0) return LUT_OK;
  const dim3 grid((unsigned)((m + 63) / 64), (unsigned)((n + 63) / 64));
  if (grid.y > 65535u) return fail(LUT_ERR_CONFIG, "matmul_ref: too many rows for one launch");
  matmul_ref_kernel<<<grid, 256, 0, stream>>>(a, b, (int)n, d, m, out);
  LUT_CHECK_LAUNCH("matmul_ref_kernel");
  return LUT_OK;
}

}  // namespace lutgpu
