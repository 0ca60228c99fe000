// Lookup-aggregate on sm_100a CUDA cores (the bitwise-exact paths).
//
//   f32:  out[n,m] = act(fl(sum_c T[c, code[n,c], m]) + bias[m])
//         sum in f32, c ascending from +0.0 — bitwise equal to lut_matmul_ref
//         (lutkit/pq.py:196-214) and lut_layer_infer's bias add (kernels.py:176-177).
//   i8:   acc[n,m] = sum_c q[c, code[n,c], m] exactly (int32), then
//         out = act(fl(fl(f32(acc) * scale) + bias)) — bitwise equal to
//         lut_gather_i32 + lut_gather_accumulate (kernels.py:105-135).
//
// Tiled kernels are table-stationary: a persistent CTA owns an m-tile, stages
// the (C, K, MT) table slice in shared memory once, and streams rows through
// it.  fp32: each lane owns 4 consecutive outputs (LDS.128 per lookup).
// int8: the slice is stored biased (q + 128, 1..255) so four int8 lookups
// are summed with two 32-bit adds into u16 pairs (<= 256 codebooks per pair
// group: 256 * 255 < 65536), widened to int32 after every 256 codebooks —
// the reference's int16-partials idea (kernels.py:105-127) on 32-bit ALUs.
// Generic kernels cover shapes whose table slice does not fit.

#include "common.cuh"

namespace lutgpu {

struct GatherArgs {
  const uint8_t* codes;
  int code_bits;
  int64_t code_stride;
  int64_t n;
  int C, K, M;
  const float* bias;
  int act;
  float* out;
  int32_t* out_i32;
  int64_t out_hw;
  int* err;
  // i8
  const float* scales;
  int scale_mtile;
};

// Row base and column stride of the output: row-major (N, M) or NCHW (one 32-bit
// division per row instead of a 64-bit one per element).
__device__ __forceinline__ void out_row(const GatherArgs& g, int64_t row, int64_t& base, int64_t& cstride) {
  if (g.out_hw > 0) {
    const uint32_t hw = (uint32_t)g.out_hw;
    const uint64_t b = row < 0xFFFFFFFFll ? (uint64_t)((uint32_t)row / hw) : (uint64_t)row / hw;
    const int64_t pix = row - (int64_t)b * g.out_hw;
    base = (int64_t)b * g.M * g.out_hw + pix;
    cstride = g.out_hw;
  } else {
    base = row * g.M;
    cstride = 1;
  }
}

__device__ __forceinline__ int64_t out_index(const GatherArgs& g, int64_t row, int col) {
  if (g.out_hw > 0) {
    const int64_t b = row / g.out_hw;
    const int64_t p = row - b * g.out_hw;
    return (b * g.M + col) * g.out_hw + p;
  }
  return row * g.M + col;
}

__device__ __forceinline__ int read_code(const GatherArgs& g, int64_t row, int c) {
  const uint8_t* r = g.codes + row * g.code_stride;
  if (g.code_bits == 8) return __ldg(r + c);
  const int byte = __ldg(r + (c >> 1));
  return (c & 1) ? (byte >> 4) : (byte & 15);
}

__device__ __forceinline__ int checked(const GatherArgs& g, int code) {
  if (code >= g.K) {
    if (g.err) atomicMax(g.err, (int)LUT_ERR_CORRUPTION);
    return g.K - 1;
  }
  return code;
}

__device__ __forceinline__ float scale_of(const GatherArgs& g, int col) {
  return g.scale_mtile > 0 ? __ldg(g.scales + col / g.scale_mtile) : __ldg(g.scales);
}

__device__ __forceinline__ float f32_epilogue(const GatherArgs& g, float acc, int col) {
  if (g.bias) acc = __fadd_rn(acc, __ldg(g.bias + col));
  return apply_act(acc, g.act);
}

// ------------------------------------------------------------ generic f32/i8

__global__ void gather_f32_generic(GatherArgs g, const float* __restrict__ table) {
  const int64_t total = g.n * g.M;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / g.M;
    const int col = (int)(i - row * g.M);
    float acc = 0.0f;
    for (int c = 0; c < g.C; ++c) {
      const int code = checked(g, read_code(g, row, c));
      acc = __fadd_rn(acc, __ldg(table + ((int64_t)c * g.K + code) * g.M + col));
    }
    g.out[out_index(g, row, col)] = f32_epilogue(g, acc, col);
  }
}

__global__ void gather_i8_generic(GatherArgs g, const int8_t* __restrict__ q) {
  const int64_t total = g.n * g.M;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / g.M;
    const int col = (int)(i - row * g.M);
    int acc = 0;
    for (int c = 0; c < g.C; ++c) {
      const int code = checked(g, read_code(g, row, c));
      acc += (int)__ldg(q + ((int64_t)c * g.K + code) * g.M + col);
    }
    const int64_t o = out_index(g, row, col);
    if (g.out_i32) g.out_i32[o] = acc;
    if (g.out) {
      float f = __fmul_rn(__int2float_rn(acc), scale_of(g, col));
      g.out[o] = f32_epilogue(g, f, col);
    }
  }
}

// ------------------------------------------------------------ tiled f32

constexpr int kGatherThreads = 256;

template <int MT>
__global__ void __launch_bounds__(kGatherThreads)
    gather_f32_tiled(GatherArgs g, const float* __restrict__ table) {
  constexpr int LPR = MT / 4;             // lanes per row
  constexpr int RPW = 32 / LPR;           // rows per warp
  constexpr int RPT = 4;                  // rows per thread per pass
  constexpr int ROWS = RPW * (kGatherThreads / 32) * RPT;
  extern __shared__ float4 tsm4[];
  float* tsm = reinterpret_cast<float*>(tsm4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane % LPR, rsub = lane / LPR;
  const int nmt = (g.M + MT - 1) / MT;
  const int64_t nrb = (g.n + ROWS - 1) / ROWS;
  const int cpm = gridDim.x >= (unsigned)nmt ? gridDim.x / nmt : 1;  // CTAs per m-tile
  const int first_mt = blockIdx.x % nmt;
  const int split = gridDim.x >= (unsigned)nmt ? blockIdx.x / nmt : 0;
  if (split >= cpm) return;
  const int64_t rb_per = (nrb + cpm - 1) / cpm;
  const int64_t rb0 = split * rb_per, rb1 = min(nrb, rb0 + rb_per);
  const int mt_step = gridDim.x >= (unsigned)nmt ? nmt : gridDim.x;
  const bool words = g.code_bits == 8 ? ((g.code_stride & 3) == 0 && (reinterpret_cast<uintptr_t>(g.codes) & 3) == 0)
                                      : ((g.code_stride & 3) == 0 && (reinterpret_cast<uintptr_t>(g.codes) & 3) == 0);
  const int span = g.code_bits == 8 ? 4 : 8;

  for (int mt = first_mt; mt < nmt; mt += mt_step) {
    const int m0 = mt * MT;
    __syncthreads();
    const bool vec = (g.M & 3) == 0 && (reinterpret_cast<uintptr_t>(table) & 15) == 0;
    for (int i = threadIdx.x; i < g.C * g.K * LPR; i += blockDim.x) {
      const int ck = i / LPR, qq = i - ck * LPR;
      const int col = m0 + 4 * qq;
      const float* src = table + (int64_t)ck * g.M + col;
      float4 v;
      if (vec && col + 3 < g.M) {
        v = __ldg(reinterpret_cast<const float4*>(src));  // one 16-byte load per 4 columns
      } else {
        v.x = col + 0 < g.M ? __ldg(src + 0) : 0.0f;
        v.y = col + 1 < g.M ? __ldg(src + 1) : 0.0f;
        v.z = col + 2 < g.M ? __ldg(src + 2) : 0.0f;
        v.w = col + 3 < g.M ? __ldg(src + 3) : 0.0f;
      }
      tsm4[i] = v;
    }
    __syncthreads();
    const int col0 = m0 + 4 * q;
    for (int64_t rb = rb0; rb < rb1; ++rb) {
      int64_t rows[RPT];
      float4 acc[RPT];
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        rows[r] = rb * ROWS + (int64_t)r * (RPW * (kGatherThreads / 32)) + warp * RPW + rsub;
        acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      int c = 0;
      if (words) {
        const int cfull = (g.C / span) * span;
        for (; c < cfull; c += span) {
          uint32_t w[RPT];
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const int64_t rr = rows[r] < g.n ? rows[r] : g.n - 1;
            w[r] = __ldg(reinterpret_cast<const uint32_t*>(g.codes + rr * g.code_stride +
                                                          (g.code_bits == 8 ? c : (c >> 1))));
          }
          for (int s = 0; s < span; ++s) {
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
              int code = g.code_bits == 8 ? (int)((w[r] >> (8 * s)) & 255u) : (int)((w[r] >> (4 * s)) & 15u);
              code = checked(g, code);
              const float4 t = tsm4[((c + s) * g.K + code) * LPR + q];
              acc[r].x = __fadd_rn(acc[r].x, t.x);
              acc[r].y = __fadd_rn(acc[r].y, t.y);
              acc[r].z = __fadd_rn(acc[r].z, t.z);
              acc[r].w = __fadd_rn(acc[r].w, t.w);
            }
          }
        }
      }
      for (; c < g.C; ++c) {
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const int64_t rr = rows[r] < g.n ? rows[r] : g.n - 1;
          const int code = checked(g, read_code(g, rr, c));
          const float4 t = tsm4[(c * g.K + code) * LPR + q];
          acc[r].x = __fadd_rn(acc[r].x, t.x);
          acc[r].y = __fadd_rn(acc[r].y, t.y);
          acc[r].z = __fadd_rn(acc[r].z, t.z);
          acc[r].w = __fadd_rn(acc[r].w, t.w);
        }
      }
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        if (rows[r] >= g.n) continue;
        float v[4] = {acc[r].x, acc[r].y, acc[r].z, acc[r].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (col0 + e < g.M) ? f32_epilogue(g, v[e], col0 + e) : 0.f;
        if (g.out_hw == 0 && col0 + 3 < g.M && (g.M & 3) == 0 &&
            (reinterpret_cast<uintptr_t>(g.out) & 15) == 0) {
          *reinterpret_cast<float4*>(g.out + rows[r] * g.M + col0) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
          int64_t base, cs;
          out_row(g, rows[r], base, cs);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (col0 + e < g.M) g.out[base + (int64_t)(col0 + e) * cs] = v[e];
        }
      }
    }
  }
}

// ------------------------------------------------------------ tiled int8

template <int MT>
__global__ void __launch_bounds__(kGatherThreads)
    gather_i8_tiled(GatherArgs g, const int8_t* __restrict__ q8) {
  constexpr int LPR = MT / 16;            // lanes per row, 16 columns each
  constexpr int RPW = 32 / LPR;
  constexpr int RPT = 2;
  constexpr int ROWS = RPW * (kGatherThreads / 32) * RPT;
  extern __shared__ uint4 qsm4[];
  uint8_t* qsm = reinterpret_cast<uint8_t*>(qsm4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ql = lane % LPR, rsub = lane / LPR;
  const int nmt = (g.M + MT - 1) / MT;
  const int64_t nrb = (g.n + ROWS - 1) / ROWS;
  const int cpm = gridDim.x >= (unsigned)nmt ? gridDim.x / nmt : 1;
  const int first_mt = blockIdx.x % nmt;
  const int split = gridDim.x >= (unsigned)nmt ? blockIdx.x / nmt : 0;
  if (split >= cpm) return;
  const int64_t rb_per = (nrb + cpm - 1) / cpm;
  const int64_t rb0 = split * rb_per, rb1 = min(nrb, rb0 + rb_per);
  const int mt_step = gridDim.x >= (unsigned)nmt ? nmt : gridDim.x;
  const bool words = (g.code_stride & 3) == 0 && (reinterpret_cast<uintptr_t>(g.codes) & 3) == 0;
  const int span = g.code_bits == 8 ? 4 : 8;
  uint32_t cw[RPT];
  int have = 0;

  for (int mt = first_mt; mt < nmt; mt += mt_step) {
    const int m0 = mt * MT;
    __syncthreads();
    for (int i = threadIdx.x; i < g.C * g.K * MT; i += blockDim.x) {
      const int ck = i / MT, cc = i - ck * MT;
      const int col = m0 + cc;
      const int v = col < g.M ? (int)__ldg(q8 + (int64_t)ck * g.M + col) : 0;
      qsm[i] = (uint8_t)(v + 128);
    }
    __syncthreads();
    const int col0 = m0 + 16 * ql;
    for (int64_t rb = rb0; rb < rb1; ++rb) {
      int64_t rows[RPT];
      int tot[RPT][16];
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        rows[r] = rb * ROWS + (int64_t)r * (RPW * (kGatherThreads / 32)) + warp * RPW + rsub;
#pragma unroll
        for (int e = 0; e < 16; ++e) tot[r][e] = 0;
      }
      for (int c0 = 0; c0 < g.C; c0 += 256) {
        const int c1 = min(g.C, c0 + 256);
        uint32_t lo[RPT][4], hi[RPT][4];
#pragma unroll
        for (int r = 0; r < RPT; ++r)
#pragma unroll
          for (int i = 0; i < 4; ++i) lo[r][i] = hi[r][i] = 0u;
        for (int c = c0; c < c1; ++c) {
          if (words && (c & (span - 1)) == 0 && c + span <= c1) {
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
              const int64_t rr = rows[r] < g.n ? rows[r] : g.n - 1;
              cw[r] = __ldg(reinterpret_cast<const uint32_t*>(g.codes + rr * g.code_stride +
                                                             (g.code_bits == 8 ? c : (c >> 1))));
            }
            have = span;
          }
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            int code;
            if (have > 0) {
              code = g.code_bits == 8 ? (int)(cw[r] & 255u) : (int)(cw[r] & 15u);
              cw[r] = g.code_bits == 8 ? (cw[r] >> 8) : (cw[r] >> 4);
            } else {
              const int64_t rr = rows[r] < g.n ? rows[r] : g.n - 1;
              code = read_code(g, rr, c);
            }
            code = checked(g, code);
            const uint4 t = qsm4[((c * g.K + code) * MT >> 4) + ql];
            lo[r][0] += t.x & 0x00FF00FFu;
            hi[r][0] += (t.x >> 8) & 0x00FF00FFu;
            lo[r][1] += t.y & 0x00FF00FFu;
            hi[r][1] += (t.y >> 8) & 0x00FF00FFu;
            lo[r][2] += t.z & 0x00FF00FFu;
            hi[r][2] += (t.z >> 8) & 0x00FF00FFu;
            lo[r][3] += t.w & 0x00FF00FFu;
            hi[r][3] += (t.w >> 8) & 0x00FF00FFu;
          }
          if (have > 0) --have;
        }
        const int bias128 = 128 * (c1 - c0);
#pragma unroll
        for (int r = 0; r < RPT; ++r)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            tot[r][4 * i + 0] += (int)(lo[r][i] & 0xFFFFu) - bias128;
            tot[r][4 * i + 2] += (int)(lo[r][i] >> 16) - bias128;
            tot[r][4 * i + 1] += (int)(hi[r][i] & 0xFFFFu) - bias128;
            tot[r][4 * i + 3] += (int)(hi[r][i] >> 16) - bias128;
          }
      }
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        if (rows[r] >= g.n) continue;
        int64_t base, cs;
        out_row(g, rows[r], base, cs);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int col = col0 + e;
          if (col >= g.M) continue;
          const int64_t o = base + (int64_t)col * cs;
          if (g.out_i32) g.out_i32[o] = tot[r][e];
          if (g.out) {
            float f = __fmul_rn(__int2float_rn(tot[r][e]), scale_of(g, col));
            g.out[o] = f32_epilogue(g, f, col);
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------ host launch

static GatherArgs make_args(const uint8_t* codes, int code_bits, int64_t n, int C, int K, int M,
                            const float* bias, int act, float* out, int32_t* out_i32, int64_t out_hw,
                            int* err) {
  GatherArgs g;
  g.codes = codes;
  g.code_bits = code_bits;
  g.code_stride = code_bits == 4 ? (C + 1) / 2 : C;
  g.n = n;
  g.C = C;
  g.K = K;
  g.M = M;
  g.bias = bias;
  g.act = act;
  g.out = out;
  g.out_i32 = out_i32;
  g.out_hw = out_hw;
  g.err = err;
  g.scales = nullptr;
  g.scale_mtile = 0;
  return g;
}

static int generic_grid(int64_t total) {
  int64_t b = (total + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)(b < cap ? (b > 0 ? b : 1) : cap);
}

template <class T>
static int launch_tiled(void (*kern)(GatherArgs, const T*), int nmt, size_t smem, const GatherArgs& g,
                        const T* table, cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(gather)");
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kGatherThreads, smem);
  if (per_sm < 1) per_sm = 1;
  const int slots = num_sms() * per_sm;
  // CTAs per m-tile: each re-stages its m-tile's table slice, so with few rows cap
  // the split at ~min_rows rows per CTA (LUTGPU_GATHER_MINROWS; 0 = no cap)
  int64_t min_rows = 256;
  if (const char* e = probe_env("LUTGPU_GATHER_MINROWS")) min_rows = atoll(e);
  int cpm = nmt >= slots ? 1 : slots / nmt;
  if (min_rows > 0) {
    const int64_t cap = (g.n + min_rows - 1) / min_rows;
    if (cap < cpm) cpm = (int)(cap > 0 ? cap : 1);
  }
  int grid = nmt >= slots ? slots : cpm * nmt;
  kern<<<grid, kGatherThreads, smem, stream>>>(g, table);
  return LUT_OK;
}

int gather_f32_strided(const uint8_t* codes, int code_bits, int64_t code_stride, int64_t n, int C, int K, int M,
                       const float* table, const float* bias, int act, float* out, int64_t out_hw, int* err,
                       cudaStream_t stream, int force_generic) {
  if (n == 0 || M == 0) return LUT_OK;
  GatherArgs g = make_args(codes, code_bits, n, C, K, M, bias, act, out, nullptr, out_hw, err);
  g.code_stride = code_stride;
  const size_t budget = 200 * 1024;
  const size_t per_col = (size_t)C * K * sizeof(float);
  int MT = 0;
  // m-tile width: the widest slice that fits; with few rows prefer narrower
  // slices (more m-tiles, each CTA stages less) until the m-tiles fill the chip
  int mt_cap = 64;
  if (const char* e = probe_env("LUTGPU_GATHER_MT")) mt_cap = atoi(e);
  else if (n < 65536) {
    const int floor_mt = n < 16384 ? 8 : 16;
    while (mt_cap > floor_mt && (M + mt_cap - 1) / mt_cap < num_sms()) mt_cap /= 2;
  }
  if (!force_generic && C > 0) {
    for (int cand : {64, 32, 16, 8, 4}) {
      if (cand <= mt_cap && per_col * cand <= budget && (cand <= 4 || (M + 3) / 4 * 4 >= cand)) {
        MT = cand;
        break;
      }
    }
  }
  if (MT == 0) {
    gather_f32_generic<<<generic_grid(n * M), 256, 0, stream>>>(g, table);
    LUT_CHECK_LAUNCH("gather_f32_generic");
    return LUT_OK;
  }
  const int nmt = (M + MT - 1) / MT;
  const size_t smem = per_col * MT;
  int st = LUT_OK;
  switch (MT) {
    case 64: st = launch_tiled(gather_f32_tiled<64>, nmt, smem, g, table, stream); break;
    case 32: st = launch_tiled(gather_f32_tiled<32>, nmt, smem, g, table, stream); break;
    case 16: st = launch_tiled(gather_f32_tiled<16>, nmt, smem, g, table, stream); break;
    case 8: st = launch_tiled(gather_f32_tiled<8>, nmt, smem, g, table, stream); break;
    default: st = launch_tiled(gather_f32_tiled<4>, nmt, smem, g, table, stream); break;
  }
  if (st != LUT_OK) return st;
  LUT_CHECK_LAUNCH("gather_f32_tiled");
  return LUT_OK;
}

int gather_i8_strided(const uint8_t* codes, int code_bits, int64_t code_stride, int64_t n, int C, int K, int M,
                      const int8_t* q, const float* scales, int scale_mtile, const float* bias, int act, float* out,
                      int32_t* out_i32, int64_t out_hw, int* err, cudaStream_t stream, int force_generic) {
  if (n == 0 || M == 0) return LUT_OK;
  GatherArgs g = make_args(codes, code_bits, n, C, K, M, bias, act, out, out_i32, out_hw, err);
  g.code_stride = code_stride;
  g.scales = scales;
  g.scale_mtile = scale_mtile;
  const size_t budget = 200 * 1024;
  const size_t per_col = (size_t)C * K;
  int MT = 0;
  if (!force_generic && C > 0) {
    for (int cand : {128, 64, 32, 16}) {
      if (per_col * cand <= budget && (cand <= 16 || (M + 15) / 16 * 16 >= cand)) {
        MT = cand;
        break;
      }
    }
  }
  if (MT == 0) {
    gather_i8_generic<<<generic_grid(n * M), 256, 0, stream>>>(g, q);
    LUT_CHECK_LAUNCH("gather_i8_generic");
    return LUT_OK;
  }
  const int nmt = (M + MT - 1) / MT;
  const size_t smem = per_col * MT;
  int st = LUT_OK;
  switch (MT) {
    case 128: st = launch_tiled(gather_i8_tiled<128>, nmt, smem, g, q, stream); break;
    case 64: st = launch_tiled(gather_i8_tiled<64>, nmt, smem, g, q, stream); break;
    case 32: st = launch_tiled(gather_i8_tiled<32>, nmt, smem, g, q, stream); break;
    default: st = launch_tiled(gather_i8_tiled<16>, nmt, smem, g, q, stream); break;
  }
  if (st != LUT_OK) return st;
  LUT_CHECK_LAUNCH("gather_i8_tiled");
  return LUT_OK;
}

}  // namespace lutgpu

namespace lutgpu {

int gather_f32(const uint8_t* codes, int code_bits, int64_t n, int C, int K, int M, const float* table,
               const float* bias, int act, float* out, int64_t out_hw, int* err, cudaStream_t stream,
               int force_generic) {
  return gather_f32_strided(codes, code_bits, code_bits == 4 ? (C + 1) / 2 : C, n, C, K, M, table, bias, act, out,
                            out_hw, err, stream, force_generic);
}

int gather_i8(const uint8_t* codes, int code_bits, int64_t n, int C, int K, int M, const int8_t* q,
              const float* scales, int scale_mtile, const float* bias, int act, float* out, int32_t* out_i32,
              int64_t out_hw, int* err, cudaStream_t stream, int force_generic) {
  return gather_i8_strided(codes, code_bits, code_bits == 4 ? (C + 1) / 2 : C, n, C, K, M, q, scales, scale_mtile,
                           bias, act, out, out_i32, out_hw, err, stream, force_generic);
}

}  // namespace lutgpu
