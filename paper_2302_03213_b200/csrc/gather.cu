// Lookup-aggregate on sm_100a CUDA cores (the bitwise-exact paths).
//
//   f32:  out[n,m] = act(fl(sum_c T[c, code[n,c], m]) + bias[m])
//         sum in f32, c ascending from +0.0 — bitwise equal to lut_matmul_ref
//         (lutkit/pq.py:196-214) and lut_layer_infer's bias add (kernels.py:176-177).
//   i8:   acc[n,m] = sum_c q[c, code[n,c], m] exactly (int32), then
//         out = act(fl(fl(f32(acc) * scale) + bias)) — bitwise equal to
//         lut_gather_i32 + lut_gather_accumulate (kernels.py:105-135).
//
// The tiled kernels are table-stationary and row-parallel (thread = row): a CTA
// owns an m-tile, stages its (C, K, MT) table slice in shared memory in a
// chunk-major layout that lets the LSU broadcast repeated lookups, and streams
// row blocks through it.  fp32 sums with packed add.rn.f32x2 (two IEEE adds).
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
  int pdl;  // launched as a programmatic dependent of the encode (lut_layer_forward)
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

// ------------------------------------------------------------ row-parallel tiled
//
// Thread = one row.  A CTA owns an m-tile (MT output columns) and stages the
// table slice for it in SMEM as [c][chunk][k][8 B] (f32: a chunk = 2 columns;
// int8: 8 columns).  For a given (c, chunk) a half-warp's 16 lanes read at most
// K distinct 8-byte chunks of one K*8-byte region: for K <= 16 that region is
// one 128-byte bank row, so every LDS.64 is conflict-free (equal codes are
// broadcast) and a warp's lookup costs exactly 2 wavefronts — the SMEM
// roofline of 128 B/clk/SM, where the column-parallel layout [c][k][m] loses
// ~40% to bank conflicts between rows.
// Units = (m-tile, row block), walked in row bands so the band's codes stay
// in L2 while every CTA re-stages its slice only when its m-tile changes.

struct RowWalk {
  int64_t nrb, band_rb, band, nbands, left, rbl, brb;
  int nmt, mt, slot, nslots;
  __device__ void init(int64_t nrb_, int nmt_, int64_t band_rb_) {
    nrb = nrb_;
    nmt = nmt_;
    band_rb = band_rb_;
    slot = (int)blockIdx.x;
    nslots = (int)gridDim.x;
    nbands = (nrb + band_rb - 1) / band_rb;
    band = -1;
    left = 0;
  }
  __device__ bool next(int& mt_out, int64_t& rb_out) {
    while (left == 0) {
      if (++band >= nbands) return false;
      brb = min(band_rb, nrb - band * band_rb);
      const int64_t ub = (int64_t)nmt * brb;
      const int64_t lo = ub * slot / nslots, hi = ub * (slot + 1) / nslots;
      left = hi - lo;
      mt = (int)(lo / brb);
      rbl = lo - (int64_t)mt * brb;
    }
    mt_out = mt;
    rb_out = band * band_rb + rbl;
    --left;
    if (++rbl == brb) {
      rbl = 0;
      ++mt;
    }
    return true;
  }
};

// Codes of one row, 16 at a time when the rows are 16-byte aligned.
struct RowCodes {
  const uint8_t* p;
  bool v16;
  __device__ __forceinline__ uint4 load16(int c0) const {
    if (v16) return __ldg(reinterpret_cast<const uint4*>(p + c0));
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      w[i] = (uint32_t)__ldg(p + c0 + 4 * i) | ((uint32_t)__ldg(p + c0 + 4 * i + 1) << 8) |
             ((uint32_t)__ldg(p + c0 + 4 * i + 2) << 16) | ((uint32_t)__ldg(p + c0 + 4 * i + 3) << 24);
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};

__device__ __forceinline__ uint32_t code_byte(const uint4& w, int s) {
  const uint32_t x = s < 4 ? w.x : s < 8 ? w.y : s < 12 ? w.z : w.w;
  return (x >> (8 * (s & 3))) & 255u;
}

// Range check of 16 codes (any code >= K raises CorruptionError through the
// error flag; the lookup then reads a clamped entry, the result is discarded).
__device__ __forceinline__ bool codes_bad(const uint4& w, int K, int pow2) {
  if (pow2) {
    const uint32_t hi = 0x01010101u * (uint32_t)(0xFF & ~(K - 1));
    return ((w.x | w.y | w.z | w.w) & hi) != 0u;
  }
  bool bad = false;
#pragma unroll
  for (int s = 0; s < 16; ++s) bad |= code_byte(w, s) >= (uint32_t)K;
  return bad;
}

__device__ __forceinline__ uint64_t lds64(uint32_t saddr) {
  uint64_t v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(saddr));
  return v;
}

__device__ __forceinline__ void fadd2(uint64_t& a, uint64_t t) {
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(a) : "l"(t));  // two IEEE fp32 adds
}

// Stage the m-tile's table slice: 8 loads in flight per thread (the slice is
// read once per m-tile change; a load-then-store loop is latency-bound on a
// cold L2).  f32 chunk = 2 columns, the (c, k) row segment read as float2.
template <int NP, int T>
__device__ __forceinline__ void stage_f32_slice(uint2* tsm, const float* __restrict__ table, int M, int C, int K,
                                                int m0) {
  const int total = C * K * NP;
  const bool vec = (M & 1) == 0 && (reinterpret_cast<uintptr_t>(table) & 7) == 0;
  const int lk = (K & (K - 1)) == 0 ? __ffs(K) - 1 : -1;
  if (vec && m0 + 2 * NP <= M) {
    // every 8-byte pair in flight at once (cp.async, no register staging): the
    // slice costs one L2 / HBM round trip instead of one per load batch
    const uint32_t sbase = smem_u32(tsm);
    for (int i = threadIdx.x; i < total; i += T) {
      const int ck = i / NP, j = i - ck * NP;
      const int c = lk >= 0 ? ck >> lk : ck / K, k = ck - c * K;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sbase + (uint32_t)(((c * NP + j) * K + k) * 8)),
                   "l"(table + (int64_t)ck * M + m0 + 2 * j)
                   : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  for (int base = threadIdx.x; base < total; base += 8 * T) {
    uint2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + u * T;
      if (i < total) {
        const int ck = i / NP, j = i - ck * NP;
        const int col = m0 + 2 * j;
        const float* src = table + (int64_t)ck * M + col;
        if (vec && col + 1 < M) {
          v[u] = __ldg(reinterpret_cast<const uint2*>(src));
        } else {
          v[u].x = col < M ? __float_as_uint(__ldg(src)) : 0u;
          v[u].y = col + 1 < M ? __float_as_uint(__ldg(src + 1)) : 0u;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + u * T;
      if (i < total) {
        const int ck = i / NP, j = i - ck * NP;
        const int c = lk >= 0 ? ck >> lk : ck / K, k = ck - c * K;
        tsm[(c * NP + j) * K + k] = v[u];
      }
    }
  }
}

// int8 chunk = 8 columns, stored biased (q + 128 = q ^ 0x80 per byte).
template <int NO, int T>
__device__ __forceinline__ void stage_i8_slice(uint2* qsm, const int8_t* __restrict__ q8, int M, int C, int K,
                                               int m0) {
  const int total = C * K * NO;
  const bool vec = (M & 7) == 0 && (reinterpret_cast<uintptr_t>(q8) & 7) == 0;
  const int lk = (K & (K - 1)) == 0 ? __ffs(K) - 1 : -1;
  if (vec && m0 + 8 * NO <= M) {
    // all 8-byte chunks in flight (cp.async), then bias them in place
    const uint32_t sbase = smem_u32(qsm);
    for (int i = threadIdx.x; i < total; i += T) {
      const int ck = i / NO, j = i - ck * NO;
      const int c = lk >= 0 ? ck >> lk : ck / K, k = ck - c * K;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sbase + (uint32_t)(((c * NO + j) * K + k) * 8)),
                   "l"(q8 + (int64_t)ck * M + m0 + 8 * j)
                   : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    for (int i = threadIdx.x; i < total; i += T) {
      const uint2 w = qsm[i];
      qsm[i] = make_uint2(w.x ^ 0x80808080u, w.y ^ 0x80808080u);
    }
    return;
  }
  for (int base = threadIdx.x; base < total; base += 8 * T) {
    uint2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + u * T;
      if (i < total) {
        const int ck = i / NO, j = i - ck * NO;
        const int col = m0 + 8 * j;
        const int8_t* src = q8 + (int64_t)ck * M + col;
        if (vec && col + 7 < M) {
          v[u] = __ldg(reinterpret_cast<const uint2*>(src));
        } else {
          uint32_t w[2] = {0u, 0u};
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (col + e < M) w[e >> 2] |= (uint32_t)(uint8_t)__ldg(src + e) << (8 * (e & 3));
          v[u] = make_uint2(w[0], w[1]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = base + u * T;
      if (i < total) {
        const int ck = i / NO, j = i - ck * NO;
        const int c = lk >= 0 ? ck >> lk : ck / K, k = ck - c * K;
        // columns beyond M stay 0 + 128 (their sums are never stored)
        qsm[(c * NO + j) * K + k] = make_uint2(v[u].x ^ 0x80808080u, v[u].y ^ 0x80808080u);
      }
    }
  }
}

// One unit of the row-parallel f32 gather: T rows (thread = row) x 2*NP columns
// starting at m0, the m-tile's table slice staged at sbase ([c][chunk][k] pairs).
// KC = K when it is a compile-time constant (16: every BASELINE shape), so the
// NP lookups of a codebook are one address and NP immediate offsets; 0 = runtime K.
template <int NP, int T, int KC>
__device__ __forceinline__ void f32_rows_unit(const GatherArgs& g, uint32_t sbase, int m0, int64_t rb, bool v16,
                                              int pow2, bool& bad) {
  const int K = KC > 0 ? KC : g.K, C = g.C;
  const uint32_t cstep = (uint32_t)(NP * K * 8);  // bytes per codebook
  const int64_t row = rb * T + threadIdx.x;
  const bool live = row < g.n;
  const int64_t rr = live ? row : g.n - 1;
  uint64_t acc[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) acc[j] = 0ull;  // (+0.0f, +0.0f)
  auto clamp = [&](uint32_t code) -> uint32_t {
    if constexpr (KC > 0 && (KC & (KC - 1)) == 0) return code & (uint32_t)(KC - 1);
    return pow2 ? (code & (uint32_t)(K - 1)) : min(code, (uint32_t)(K - 1));
  };
  if (g.code_bits == 8) {
    RowCodes rc{g.codes + rr * g.code_stride, v16};
    int c0 = 0;
    // the next 16 codes are loaded while the current 16 are looked up (a
    // load-then-use loop serialises one global latency per 16 codebooks)
    uint4 wn = C >= 16 ? rc.load16(0) : make_uint4(0u, 0u, 0u, 0u);
    for (; c0 + 16 <= C; c0 += 16) {
      const uint4 w = wn;
      if (c0 + 32 <= C) wn = rc.load16(c0 + 16);
      bad |= codes_bad(w, K, pow2);
      const uint32_t cb = sbase + (uint32_t)c0 * cstep;
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        const uint32_t a = cb + (uint32_t)s * cstep + clamp(code_byte(w, s)) * 8u;
#pragma unroll
        for (int j = 0; j < NP; ++j) fadd2(acc[j], lds64(a + (uint32_t)(j * K * 8)));
      }
    }
    for (; c0 < C; ++c0) {
      uint32_t code = __ldg(rc.p + c0);
      bad |= code >= (uint32_t)K;
      code = min(code, (uint32_t)(K - 1));
      const uint32_t a = sbase + (uint32_t)c0 * cstep + code * 8u;
#pragma unroll
      for (int j = 0; j < NP; ++j) fadd2(acc[j], lds64(a + (uint32_t)(j * K * 8)));
    }
  } else {
    for (int c = 0; c < C; ++c) {
      uint32_t code = (uint32_t)read_code(g, rr, c);
      bad |= code >= (uint32_t)K;
      code = min(code, (uint32_t)(K - 1));
      const uint32_t a = sbase + (uint32_t)c * cstep + code * 8u;
#pragma unroll
      for (int j = 0; j < NP; ++j) fadd2(acc[j], lds64(a + (uint32_t)(j * K * 8)));
    }
  }
  if (!live) return;
  int64_t obase, ocs;
  out_row(g, row, obase, ocs);
  float v[2 * NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) asm("mov.b64 {%0, %1}, %2;" : "=f"(v[2 * j]), "=f"(v[2 * j + 1]) : "l"(acc[j]));
  if (m0 + 2 * NP <= g.M) {
    // full tile: the bias / activation branches are uniform and taken once per tile
    if (g.bias) {
      if ((reinterpret_cast<uintptr_t>(g.bias) & 7) == 0) {
#pragma unroll
        for (int j = 0; j < NP; ++j) {
          const float2 b = __ldg(reinterpret_cast<const float2*>(g.bias + m0) + j);
          v[2 * j] = __fadd_rn(v[2 * j], b.x);
          v[2 * j + 1] = __fadd_rn(v[2 * j + 1], b.y);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 2 * NP; ++e) v[e] = __fadd_rn(v[e], __ldg(g.bias + m0 + e));
      }
    }
    if (g.act == LUT_ACT_RELU) {
#pragma unroll
      for (int e = 0; e < 2 * NP; ++e) v[e] = fmaxf(v[e], 0.0f);
    } else if (g.act == LUT_ACT_GELU) {
#pragma unroll
      for (int e = 0; e < 2 * NP; ++e) v[e] = gelu_erf(v[e]);
    }
    float* o = g.out + obase + (int64_t)m0 * ocs;
    if (ocs == 1 && NP >= 2 && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
#pragma unroll
      for (int e = 0; e + 3 < 2 * NP; e += 4) *reinterpret_cast<float4*>(o + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
    } else if (ocs == 1 && ((reinterpret_cast<uintptr_t>(o) & 7) == 0)) {
#pragma unroll
      for (int e = 0; e < 2 * NP; e += 2) *reinterpret_cast<float2*>(o + e) = make_float2(v[e], v[e + 1]);
    } else {
#pragma unroll
      for (int e = 0; e < 2 * NP; ++e) o[(int64_t)e * ocs] = v[e];
    }
    return;
  }
#pragma unroll
  for (int e = 0; e < 2 * NP; ++e)
    if (m0 + e < g.M) g.out[obase + (int64_t)(m0 + e) * ocs] = f32_epilogue(g, v[e], m0 + e);
}

// Thread block of T threads; NP chunks of 2 f32 columns per thread (MT = 2 * NP).
template <int NP, int T, int KC>
__global__ void __launch_bounds__(T, T <= 128 ? 4 : 1)
    gather_f32_rows(GatherArgs g, const float* __restrict__ table, int64_t band_rb) {
  extern __shared__ uint2 tsm[];  // [C][NP][K] float pairs
  constexpr int MT = 2 * NP;
  const int nmt = (g.M + MT - 1) / MT;
  const int64_t nrb = (g.n + T - 1) / T;
  const int K = KC > 0 ? KC : g.K, C = g.C;
  const int pow2 = (K & (K - 1)) == 0;
  const bool v16 = g.code_bits == 8 && (g.code_stride & 15) == 0 && (reinterpret_cast<uintptr_t>(g.codes) & 15) == 0;
  const uint32_t sbase = smem_u32(tsm);
  RowWalk walk;
  walk.init(nrb, nmt, band_rb);
  int cur = -1;
  int mt;
  int64_t rb;
  bool bad = false;
  while (walk.next(mt, rb)) {
    const int m0 = mt * MT;
    if (mt != cur) {
      __syncthreads();
      stage_f32_slice<NP, T>(tsm, table, g.M, C, K, m0);
      __syncthreads();
      if (cur < 0) grid_dependency_wait();  // the table slice is staged while the encode finishes
      cur = mt;
    }
    f32_rows_unit<NP, T, KC>(g, sbase, m0, rb, v16, pow2, bad);
  }
  if (bad && g.err) atomicMax(g.err, (int)LUT_ERR_CORRUPTION);
}

// Per 8-column chunk the accumulators hold sx = sum of the raw words of bytes
// 0-3, ox = sum of their odd bytes {1, 3} as u16 lanes, and sy / oy for bytes
// 4-7.  Since w = even(w) + (odd(w) << 8) as integers, the even-byte sums
// follow exactly (mod 2^32, every lane < 2^16) as sx - (ox << 8) once per
// 256-codebook block (i8_even): one PRMT per word instead of two.
template <int NO>
__device__ __forceinline__ void i8_lookup(uint32_t (&acc)[NO][4], uint32_t cbase, uint32_t code, int K) {
  const uint32_t a = cbase + code * 8u;
#pragma unroll
  for (int j = 0; j < NO; ++j) {
    const uint64_t t = lds64(a + (uint32_t)(j * K * 8));
    const uint32_t w0 = (uint32_t)t, w1 = (uint32_t)(t >> 32);
    acc[j][0] += w0;
    acc[j][1] += __byte_perm(w0, 0, 0x4341);  // biased bytes 1, 3 -> u16 lanes
    acc[j][2] += w1;
    acc[j][3] += __byte_perm(w1, 0, 0x4341);
  }
}

// Two codebooks at once: their contributions meet in one IADD3 per accumulator.
template <int NO>
__device__ __forceinline__ void i8_lookup2(uint32_t (&acc)[NO][4], uint32_t cbase0, uint32_t code0, uint32_t cbase1,
                                           uint32_t code1, int K) {
  const uint32_t a0 = cbase0 + code0 * 8u, a1 = cbase1 + code1 * 8u;
#pragma unroll
  for (int j = 0; j < NO; ++j) {
    const uint64_t t0 = lds64(a0 + (uint32_t)(j * K * 8));
    const uint64_t t1 = lds64(a1 + (uint32_t)(j * K * 8));
    const uint32_t x0 = (uint32_t)t0, y0 = (uint32_t)(t0 >> 32), x1 = (uint32_t)t1, y1 = (uint32_t)(t1 >> 32);
    acc[j][0] += x0 + x1;
    acc[j][1] += __byte_perm(x0, 0, 0x4341) + __byte_perm(x1, 0, 0x4341);
    acc[j][2] += y0 + y1;
    acc[j][3] += __byte_perm(y0, 0, 0x4341) + __byte_perm(y1, 0, 0x4341);
  }
}

// raw word sums -> even-byte u16 lanes: acc = {bytes {0,2}, {1,3}, {4,6}, {5,7}}
template <int NO>
__device__ __forceinline__ void i8_even(uint32_t (&acc)[NO][4]) {
#pragma unroll
  for (int j = 0; j < NO; ++j) {
    acc[j][0] -= acc[j][1] << 8;
    acc[j][2] -= acc[j][3] << 8;
  }
}

// int8: NO chunks of 8 columns per thread (MT = 8 * NO); biased bytes (q + 128)
// summed as u16 pairs, widened every 256 codebooks when WIDE.
template <int NO, bool WIDE, int T, int KC>
__global__ void __launch_bounds__(T, T <= 128 ? 4 : 1)
    gather_i8_rows(GatherArgs g, const int8_t* __restrict__ q8, int64_t band_rb) {
  extern __shared__ uint2 qsm[];  // [C][NO][K] x 8 biased bytes
  constexpr int MT = 8 * NO;
  const int nmt = (g.M + MT - 1) / MT;
  const int64_t nrb = (g.n + T - 1) / T;
  const int K = KC > 0 ? KC : g.K, C = g.C;  // KC: compile-time K (immediate lookup offsets)
  const int pow2 = (K & (K - 1)) == 0;
  const bool v16 = g.code_bits == 8 && (g.code_stride & 15) == 0 && (reinterpret_cast<uintptr_t>(g.codes) & 15) == 0;
  const uint32_t sbase = smem_u32(qsm);
  const uint32_t cstep = (uint32_t)(NO * K * 8);
  RowWalk walk;
  walk.init(nrb, nmt, band_rb);
  int cur = -1;
  int mt;
  int64_t rb;
  bool bad = false;
  while (walk.next(mt, rb)) {
    const int m0 = mt * MT;
    if (mt != cur) {
      __syncthreads();
      stage_i8_slice<NO, T>(qsm, q8, g.M, C, K, m0);
      __syncthreads();
      if (cur < 0) grid_dependency_wait();
      cur = mt;
    }
    const int64_t row = rb * T + threadIdx.x;
    const bool live = row < g.n;
    const int64_t rr = live ? row : g.n - 1;
    int tot[WIDE ? NO * 8 : 1];
    if constexpr (WIDE) {
#pragma unroll
      for (int e = 0; e < NO * 8; ++e) tot[e] = 0;
    }
    uint32_t acc[NO][4];  // per 8 columns: bytes {0,2}, {1,3}, {4,6}, {5,7} as u16 pairs
    RowCodes rc{g.codes + rr * g.code_stride, v16};
    for (int cb = 0; cb < C; cb += 256) {  // a u16 lane holds <= 256 biased bytes (256 * 255 < 65536)
      const int ce = min(C, cb + 256);
#pragma unroll
      for (int j = 0; j < NO; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[j][i] = 0u;
      int c0 = cb;
      if (g.code_bits == 8) {
        uint4 wn = c0 + 16 <= ce ? rc.load16(c0) : make_uint4(0u, 0u, 0u, 0u);
        for (; c0 + 16 <= ce; c0 += 16) {
          const uint4 w = wn;  // next 16 codes in flight during these lookups
          if (c0 + 32 <= ce) wn = rc.load16(c0 + 16);
          bad |= codes_bad(w, K, pow2);
#pragma unroll
          for (int s = 0; s < 16; s += 2) {
            uint32_t k0 = code_byte(w, s), k1 = code_byte(w, s + 1);
            k0 = pow2 ? (k0 & (uint32_t)(K - 1)) : min(k0, (uint32_t)(K - 1));
            k1 = pow2 ? (k1 & (uint32_t)(K - 1)) : min(k1, (uint32_t)(K - 1));
            i8_lookup2<NO>(acc, sbase + (uint32_t)(c0 + s) * cstep, k0, sbase + (uint32_t)(c0 + s + 1) * cstep, k1, K);
          }
        }
      }
      for (; c0 < ce; ++c0) {
        const uint32_t code = (uint32_t)read_code(g, rr, c0);
        bad |= code >= (uint32_t)K;
        i8_lookup<NO>(acc, sbase + (uint32_t)c0 * cstep, min(code, (uint32_t)(K - 1)), K);
      }
      i8_even<NO>(acc);
      if constexpr (WIDE) {
        const int b128 = 128 * (ce - cb);
#pragma unroll
        for (int j = 0; j < NO; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            tot[j * 8 + 4 * h + 0] += (int)(acc[j][2 * h] & 0xFFFFu) - b128;
            tot[j * 8 + 4 * h + 2] += (int)(acc[j][2 * h] >> 16) - b128;
            tot[j * 8 + 4 * h + 1] += (int)(acc[j][2 * h + 1] & 0xFFFFu) - b128;
            tot[j * 8 + 4 * h + 3] += (int)(acc[j][2 * h + 1] >> 16) - b128;
          }
      }
    }
    if (!live) continue;
    int64_t obase, ocs;
    out_row(g, row, obase, ocs);
    const int b_all = 128 * C;
    const bool vrow = ocs == 1 && (g.M & 3) == 0;
#pragma unroll
    for (int j = 0; j < NO; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // 4 columns at a time
        const int col = m0 + 8 * j + 4 * h;
        int a[4];
        if constexpr (WIDE) {
#pragma unroll
          for (int e = 0; e < 4; ++e) a[e] = tot[j * 8 + 4 * h + e];
        } else {
          a[0] = (int)(acc[j][2 * h] & 0xFFFFu) - b_all;
          a[1] = (int)(acc[j][2 * h + 1] & 0xFFFFu) - b_all;
          a[2] = (int)(acc[j][2 * h] >> 16) - b_all;
          a[3] = (int)(acc[j][2 * h + 1] >> 16) - b_all;
        }
        const bool vec = vrow && col + 3 < g.M;
        if (g.out_i32) {
          if (vec && (reinterpret_cast<uintptr_t>(g.out_i32) & 15) == 0)
            *reinterpret_cast<int4*>(g.out_i32 + obase + col) = make_int4(a[0], a[1], a[2], a[3]);
          else
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (col + e < g.M) g.out_i32[obase + (int64_t)(col + e) * ocs] = a[e];
        }
        if (g.out) {
          float v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            v[e] = col + e < g.M ? f32_epilogue(g, __fmul_rn(__int2float_rn(a[e]), scale_of(g, col + e)), col + e)
                                 : 0.f;
          if (vec && (reinterpret_cast<uintptr_t>(g.out) & 15) == 0)
            *reinterpret_cast<float4*>(g.out + obase + col) = make_float4(v[0], v[1], v[2], v[3]);
          else
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (col + e < g.M) g.out[obase + (int64_t)(col + e) * ocs] = v[e];
        }
      }
    }
  }
  if (bad && g.err) atomicMax(g.err, (int)LUT_ERR_CORRUPTION);
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
  g.pdl = 0;
  return g;
}

static int generic_grid(int64_t total) {
  int64_t b = (total + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)(b < cap ? (b > 0 ? b : 1) : cap);
}

// Grid and band for the row-parallel kernels: as many CTAs as fit (SMEM slice
// per CTA), at most one per unit; a band of row blocks keeps its codes in L2
// while each CTA walks ~64 consecutive units of it (so it spans ~2 m-tiles and
// re-stages its slice ~2-3 times per band).
template <class T, int TH>
static int launch_rows(void (*kern)(GatherArgs, const T*, int64_t), int nmt, size_t smem, const GatherArgs& g,
                       const T* table, cudaStream_t stream) {
  cudaError_t e = kernel_smem_attr(reinterpret_cast<const void*>(kern));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(gather)");
  const int per_sm = kernel_occupancy(reinterpret_cast<const void*>(kern), TH, smem);
  const int64_t nrb = (g.n + TH - 1) / TH;
  const int64_t units = nrb * nmt;
  const int64_t slots = (int64_t)num_sms() * per_sm;
  const int grid = (int)(units < slots ? units : slots);
  int64_t band_rb = (64 * (int64_t)grid + nmt - 1) / nmt;
  const int64_t code_row_bytes = g.code_stride > 0 ? g.code_stride : g.C;
  const int64_t max_band = ((int64_t)32 << 20) / (TH * code_row_bytes + 1);
  if (band_rb > max_band) band_rb = max_band;
  if (band_rb < 1) band_rb = 1;
  if (band_rb > nrb) band_rb = nrb;
  if (g.pdl) {
    // programmatic dependent launch: CTAs start on the SMs the encode leaves free
    // and stage their table slices before griddepcontrol.wait (the codes)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(TH);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, g, table, band_rb);
    if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernelEx(gather, PDL)");
    return LUT_OK;
  }
  kern<<<grid, TH, smem, stream>>>(g, table, band_rb);
  return LUT_OK;
}

// Rows per CTA: 512 (16 warps hide the LDS latency) unless that leaves SMs idle.
static bool small_rows(int64_t n, int nmt) { return (n + 511) / 512 * (int64_t)nmt < 2 * (int64_t)num_sms(); }

template <int NP, int KC>
static int launch_f32_k(int nmt, size_t smem, const GatherArgs& g, const float* table, cudaStream_t stream, int th) {
#ifdef LUTGPU_PROBES
  if (th == 128) return launch_rows<float, 128>(gather_f32_rows<NP, 128, KC>, nmt, smem, g, table, stream);
  if (th == 256) return launch_rows<float, 256>(gather_f32_rows<NP, 256, KC>, nmt, smem, g, table, stream);
  if (th == 1024) return launch_rows<float, 1024>(gather_f32_rows<NP, 1024, KC>, nmt, smem, g, table, stream);
#else
  (void)th;
#endif
  return launch_rows<float, 512>(gather_f32_rows<NP, 512, KC>, nmt, smem, g, table, stream);
}

template <int NP>
static int launch_f32(int nmt, size_t smem, const GatherArgs& g, const float* table, cudaStream_t stream, int th) {
  return g.K == 16 ? launch_f32_k<NP, 16>(nmt, smem, g, table, stream, th)
                   : launch_f32_k<NP, 0>(nmt, smem, g, table, stream, th);
}

int gather_f32_strided(const uint8_t* codes, int code_bits, int64_t code_stride, int64_t n, int C, int K, int M,
                       const float* table, const float* bias, int act, float* out, int64_t out_hw, int* err,
                       cudaStream_t stream, int force_generic, int pdl) {
  if (n == 0 || M == 0) return LUT_OK;
  GatherArgs g = make_args(codes, code_bits, n, C, K, M, bias, act, out, nullptr, out_hw, err);
  g.code_stride = code_stride;
  g.pdl = pdl;
  const size_t budget = 200 * 1024;
  const size_t per_chunk = (size_t)C * K * 8;  // SMEM bytes per 2-column chunk
  int NP = 0;
  if (!force_generic && C > 0) {
    for (int cand : {8, 4, 2, 1})
      if (per_chunk * cand <= budget) {
        NP = cand;
        break;
      }
    while (NP > 1 && 2 * (NP / 2) >= M) NP /= 2;  // do not stage columns beyond M
  }
  if (NP == 0) {
    gather_f32_generic<<<generic_grid(n * M), 256, 0, stream>>>(g, table);
    LUT_CHECK_LAUNCH("gather_f32_generic");
    return LUT_OK;
  }
  int nmt = (M + 2 * NP - 1) / (2 * NP);
  // 512-row CTAs (16 warps hide the LDS latency); few rows: narrower slices until
  // there are >= 1.5 units per SM, or >= 4 when a unit is heavy (C * NP > 512:
  // the last wave's imbalance) — tools/f32_sweep.py, graph-timed on B200:
  // configs[0] 21.1 -> 11.7 us, the configs[2] convs 16-19 -> 15-16 us,
  // configs[1] FFN2 59 -> 55 us
  while (NP > 1 && (n + 511) / 512 * (int64_t)nmt * 2 < (C * NP > 512 ? 8 : 3) * (int64_t)num_sms()) {
    NP /= 2;
    nmt = (M + 2 * NP - 1) / (2 * NP);
  }
  int th = 512;
  if (const char* e = probe_env("LUTGPU_F32_NP")) {
    NP = atoi(e);
    nmt = (M + 2 * NP - 1) / (2 * NP);
  }
  if (const char* e = probe_env("LUTGPU_F32_T")) th = atoi(e);
  const size_t smem = per_chunk * NP;
  int st = LUT_OK;
  switch (NP) {
    case 8: st = launch_f32<8>(nmt, smem, g, table, stream, th); break;
    case 4: st = launch_f32<4>(nmt, smem, g, table, stream, th); break;
    case 2: st = launch_f32<2>(nmt, smem, g, table, stream, th); break;
    default: st = launch_f32<1>(nmt, smem, g, table, stream, th); break;
  }
  if (st != LUT_OK) return st;
  LUT_CHECK_LAUNCH("gather_f32_rows");
  return LUT_OK;
}

template <int NO, bool WIDE, int KC>
static int launch_i8_k(int nmt, size_t smem, const GatherArgs& g, const int8_t* q, cudaStream_t stream, bool small) {
  return small ? launch_rows<int8_t, 128>(gather_i8_rows<NO, WIDE, 128, KC>, nmt, smem, g, q, stream)
               : launch_rows<int8_t, 512>(gather_i8_rows<NO, WIDE, 512, KC>, nmt, smem, g, q, stream);
}

template <int NO, bool WIDE>
static int launch_i8(int nmt, size_t smem, const GatherArgs& g, const int8_t* q, cudaStream_t stream, bool small) {
  return g.K == 16 ? launch_i8_k<NO, WIDE, 16>(nmt, smem, g, q, stream, small)
                   : launch_i8_k<NO, WIDE, 0>(nmt, smem, g, q, stream, small);
}

int gather_i8_strided(const uint8_t* codes, int code_bits, int64_t code_stride, int64_t n, int C, int K, int M,
                      const int8_t* q, const float* scales, int scale_mtile, const float* bias, int act, float* out,
                      int32_t* out_i32, int64_t out_hw, int* err, cudaStream_t stream, int force_generic, int pdl) {
  if (n == 0 || M == 0) return LUT_OK;
  GatherArgs g = make_args(codes, code_bits, n, C, K, M, bias, act, out, out_i32, out_hw, err);
  g.code_stride = code_stride;
  g.pdl = pdl;
  g.scales = scales;
  g.scale_mtile = scale_mtile;
  const size_t budget = 200 * 1024;
  const size_t per_chunk = (size_t)C * K * 8;  // SMEM bytes per 8-column chunk
  const bool wide = C > 256;
  int NO = 0;
  if (!force_generic && C > 0) {
    for (int cand : {4, 2, 1})
      if (per_chunk * cand <= budget && !(wide && cand > 2)) {
        NO = cand;
        break;
      }
    while (NO > 1 && 8 * (NO / 2) >= M) NO /= 2;  // do not stage columns beyond M
  }
  if (NO == 0) {
    gather_i8_generic<<<generic_grid(n * M), 256, 0, stream>>>(g, q);
    LUT_CHECK_LAUNCH("gather_i8_generic");
    return LUT_OK;
  }
  int nmt = (M + 8 * NO - 1) / (8 * NO);
  bool small = small_rows(n, nmt);
  while (small && NO > 1 && (n + 127) / 128 * (int64_t)nmt < 4 * (int64_t)num_sms()) {
    NO /= 2;
    nmt = (M + 8 * NO - 1) / (8 * NO);
  }
  const size_t smem = per_chunk * NO;
  int st = LUT_OK;
  if (wide) {
    st = NO == 2 ? launch_i8<2, true>(nmt, smem, g, q, stream, small) : launch_i8<1, true>(nmt, smem, g, q, stream, small);
  } else {
    switch (NO) {
      case 4: st = launch_i8<4, false>(nmt, smem, g, q, stream, small); break;
      case 2: st = launch_i8<2, false>(nmt, smem, g, q, stream, small); break;
      default: st = launch_i8<1, false>(nmt, smem, g, q, stream, small); break;
    }
  }
  if (st != LUT_OK) return st;
  LUT_CHECK_LAUNCH("gather_i8_rows");
  return LUT_OK;
}

}  // namespace lutgpu

namespace lutgpu {

int gather_f32(const uint8_t* codes, int code_bits, int64_t n, int C, int K, int M, const float* table,
               const float* bias, int act, float* out, int64_t out_hw, int* err, cudaStream_t stream,
               int force_generic) {
  return gather_f32_strided(codes, code_bits, code_bits == 4 ? (C + 1) / 2 : C, n, C, K, M, table, bias, act, out,
                            out_hw, err, stream, force_generic, 0);
}

int gather_i8(const uint8_t* codes, int code_bits, int64_t n, int C, int K, int M, const int8_t* q,
              const float* scales, int scale_mtile, const float* bias, int act, float* out, int32_t* out_i32,
              int64_t out_hw, int* err, cudaStream_t stream, int force_generic) {
  return gather_i8_strided(codes, code_bits, code_bits == 4 ? (C + 1) / 2 : C, n, C, K, M, q, scales, scale_mtile,
                           bias, act, out, out_i32, out_hw, err, stream, force_generic, 0);
}

}  // namespace lutgpu
