// Nearest-centroid encode on sm_100a.
//
// Semantics: indices identical to the reference's encode_hard
// (lutkit/pq.py:171-174; literal f64 squared distances, ties -> lowest k),
// which centroid_search_fast (lutkit/kernels.py:62-102) reproduces with the
// expansion ||p||^2 - 2 a.p.
//
// Arithmetic: fp32 FFMA evaluates d_k = ||p_k||^2 - 2 a.p_k (two interleaved
// chains, the -2 folded exactly into a), tracking best and second-best.  The
// fp32 error of any d_k is < 2(V+3) u (||a||^2 + max_k ||p_k||^2), u = 2^-24
// (||p||^2 exact to 1 ulp, 2|a.p| <= ||a||^2 + ||p||^2).  If the gap between the
// best and second-best fp32 distance is within TAU = 4(V+4) u (||a||^2 + pmax)
// — twice the sum of the two bounds — the fp32 winner may differ from the
// exact one, so that (row, codebook) is re-decided from literal f64
// differences exactly like encode_hard, and counted as a near tie.  Outside
// the bound the fp32 winner is provably the exact argmin.
//
// Kernels
//  encode_tma_kernel<V>   V in {4, 8, 16, 32}: persistent, warp-specialised.
//    One producer warp streams 32-column x 512-row tiles of A with TMA
//    (cp.async.bulk.tensor, 128B swizzle) plus the prepared codebooks of those
//    columns (cp.async.bulk) into a 3-stage mbarrier ring; 8 consumer warps,
//    2 rows per lane, read their row's sub-vector conflict-free from the
//    swizzled tile and the centroids as warp-broadcast LDS.128.  Codes are
//    packed in registers and stored as 16-byte vectors per row group.
//  encode_rows_kernel<VT> generic (any V <= 256, any K <= 256), one thread per
//    (row, codebook-pair), templated row loader: dense rows or on-the-fly
//    im2col patches from an NCHW batch (conv fusion, tensor.py:36-79).

#include <float.h>

#include "common.cuh"
#include "encode_dev.cuh"

namespace lutgpu {


__global__ void prepare_books_kernel(const float* __restrict__ books, int C, int K, int V,
                                     float* __restrict__ prep) {
  const int c = blockIdx.x;
  const int S = prep_stride(K, V);
  float* rec = prep + (size_t)c * S;
  const float* src = books + (size_t)c * K * V;
  for (int i = threadIdx.x; i < K * V; i += blockDim.x) rec[i] = src[i];
  if (prep_has_tc(K, V)) {  // swizzled tf32 operand tile + |p_k| rounded up (encode_tc.cu)
    float* tc = rec + prep_base(K, V);
    for (int i = threadIdx.x; i < K * V; i += blockDim.x) {
      const int k = i / V, j = i - (i / V) * V;
      tc[k * 32 + 4 * ((j >> 2) ^ (k & 7)) + (j & 3)] = src[i];
    }
    if (threadIdx.x == 0) {  // 2^-7 max_k |p_k|, rounded up (screening half-width)
      double mx = 0.0;
      for (int k = 0; k < K; ++k) {
        double s = 0.0;
        for (int j = 0; j < V; ++j) s = fma((double)src[k * V + j], (double)src[k * V + j], s);
        mx = fmax(mx, s);
      }
      tc[K * V] = __double2float_ru(sqrt(mx) * (1.0 + 1e-15) * 0.0078125);
      for (int k = 1; k < K; ++k) tc[K * V + k] = 0.0f;
    }
  }
  __shared__ float smax[32];
  float local = 0.0f;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < V; ++j) {
      double x = (double)src[k * V + j];
      s = fma(x, x, s);
    }
    float f = (float)s;
    rec[K * V + k] = f;
    local = fmaxf(local, f);
  }
  for (int o = 16; o > 0; o >>= 1) local = fmaxf(local, __shfl_xor_sync(0xffffffffu, local, o));
  if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.0f;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) m = fmaxf(m, smax[w]);
    rec[K * V + K] = m;
    for (int i = K * V + K + 1; i < prep_base(K, V); ++i) rec[i] = 0.0f;
  }
}

// packed-pair FP32 (sm_100 FFMA2 / FADD2): two lanes of math per issue slot
__device__ __forceinline__ uint64_t pack_f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack_f2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}


// --------------------------------------------------------------- TMA path

// Consumer geometry: W consumer warps x RPL rows per lane = one 512-row tile.
// A broadcast LDS.128 of a centroid costs 4 SMEM wavefronts whatever the
// address pattern, so the centroid traffic per (row, k) is 1/RPL of a
// wavefront per lane: RPL = 4 (4 warps) halves it against RPL = 2 (8 warps).
constexpr int kBoxRows = 256;                 // TMA box rows
constexpr int kTileRows = 512;
constexpr int kTileBoxes = kTileRows / kBoxRows;  // A boxes per stage
constexpr int kBoxBytes = kBoxRows * 128;     // 32 KB (32 f32 columns)

struct EncTmaParams {
  const float* prep;
  int S;          // prepared record stride (floats)
  int64_t n;
  int C, K;
  int G;          // codebooks per output group (flush granularity)
  int ngroups;
  int64_t ntiles;
  uint8_t* codes;
  int code_bits;
  int64_t code_stride;  // bytes per row of codes
  int* near_tie;
  int stages;
  int stage_bytes;
  int debug;  // LUTGPU_ENC_DEBUG: 1 = consumers skip the distance math (TMA streaming only)
};

__device__ __forceinline__ void store_code_group(uint8_t* dst, uint32_t w0, uint32_t w1,
                                                 uint32_t w2, uint32_t w3, int nbytes) {
  if (nbytes == 16 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
    *reinterpret_cast<uint4*>(dst) = make_uint4(w0, w1, w2, w3);
    return;
  }
  if (nbytes == 8 && ((reinterpret_cast<uintptr_t>(dst) & 7) == 0)) {
    *reinterpret_cast<uint2*>(dst) = make_uint2(w0, w1);
    return;
  }
  if (nbytes == 4 && ((reinterpret_cast<uintptr_t>(dst) & 3) == 0)) {
    *reinterpret_cast<uint32_t*>(dst) = w0;
    return;
  }
  uint32_t w[4] = {w0, w1, w2, w3};
  for (int i = 0; i < nbytes; ++i) dst[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
}

// CHAIN = 1: one packed accumulator chain per (row, k) over raw a (the -2 is
// applied once, d = fma(-2, a.p, |p|^2)): no per-element FMUL and no per-k
// FADD2 merge; CHAIN = 0: |p|^2 seeded, two chains over -2a.  Both are sums of
// V+1 rounded terms, inside the same error bound (TAU).
template <int V, int kEncWarps, int kRPL, int CHAIN = 0>
__global__ void __launch_bounds__((kEncWarps + 1) * 32, 1)
    encode_tma_kernel(const __grid_constant__ CUtensorMap tmap, const EncTmaParams p) {
  grid_launch_dependents();  // a programmatic dependent (the gather) may start staging
  constexpr int kRowsPerPass = kEncWarps * 32;  // rows covered by one pass of all consumer lanes
  static_assert(kRowsPerPass * kRPL == kTileRows, "tile geometry");
  constexpr int NB = 32 / V;   // codebooks per 32-column box
  constexpr int NJ = V / 4;    // 16-byte chunks per sub-vector
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window (LDS, not generic LD)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)p.stages * p.stage_bytes);
  uint64_t* empty = full + p.stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kEncWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int64_t nunits = p.ntiles * p.ngroups;
  const int boxes_per_group = p.G / NB;
  const int nboxes = (p.C + NB - 1) / NB;

  if (warp == kEncWarps) {
    // ---------------- producer
    if (lane == 0) {
      prefetch_tmap(&tmap);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int64_t tile = u / p.ngroups;
        const int grp = (int)(u % p.ngroups);
        const int b0 = grp * boxes_per_group;
        const int b1 = min(nboxes, b0 + boxes_per_group);
        for (int b = b0; b < b1; ++b) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + (size_t)stage * p.stage_bytes;
          const int nsub = min(NB, p.C - b * NB);
          const uint32_t book_bytes = (uint32_t)nsub * p.S * 4;
          mbar_arrive_expect_tx(&full[stage], kTileBoxes * kBoxBytes + book_bytes);
#pragma unroll
          for (int r = 0; r < kTileBoxes; ++r)
            tma_load_2d(st + r * kBoxBytes, &tmap, b * 32, (int32_t)(tile * kTileRows + r * kBoxRows),
                        &full[stage]);
          bulk_load(st + kTileBoxes * kBoxBytes, p.prep + (size_t)b * NB * p.S, book_bytes, &full[stage]);
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers
  int stage = 0;
  uint32_t phase = 0;
  const int rr = warp * 32 + lane;  // this lane's first row in the tile (then + kRowsPerPass)
  const int sw = rr & 7;            // 128B swizzle phase of this row
  const float tau_c = tau_coef(V);
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t tile = u / p.ngroups;
    const int grp = (int)(u % p.ngroups);
    const int c_begin = grp * p.G;
    const int c_end = min(p.C, c_begin + p.G);
    const int b0 = c_begin / NB;
    const int b1 = (c_end + NB - 1) / NB;
    uint32_t pk[kRPL][4];
#pragma unroll
    for (int r = 0; r < kRPL; ++r) pk[r][0] = pk[r][1] = pk[r][2] = pk[r][3] = 0u;
    int ncodes = 0;

    for (int b = b0; b < b1; ++b) {
      mbar_wait(&full[stage], phase);
      const uint8_t* st = smem + (size_t)stage * p.stage_bytes;
      const float* cent_all = reinterpret_cast<const float*>(st + kTileBoxes * kBoxBytes);
#pragma unroll
      for (int sb = 0; sb < NB; ++sb) {
        const int c = b * NB + sb;
        if (c >= c_end || (p.debug & 1)) break;
        const float* cb = cent_all + sb * p.S;
        // packed pairs (-2 a_j, -2 a_j+1): FFMA2 does two FMAs per issue slot
        uint64_t a2[kRPL][V / 2];
        float asq[kRPL];
#pragma unroll
        for (int r = 0; r < kRPL; ++r) {
          const int q_ = rr + r * kRowsPerPass;
          const float* rowp = reinterpret_cast<const float*>(st + (q_ >> 8) * kBoxBytes + (q_ & 255) * 128);
          asq[r] = 0.0f;
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            const float4 x = *reinterpret_cast<const float4*>(rowp + (((sb * NJ + j) ^ sw) << 2));
            asq[r] = fmaf(x.x, x.x, asq[r]);
            asq[r] = fmaf(x.y, x.y, asq[r]);
            asq[r] = fmaf(x.z, x.z, asq[r]);
            asq[r] = fmaf(x.w, x.w, asq[r]);
            if constexpr (CHAIN == 1) {
              a2[r][2 * j + 0] = pack_f2(x.x, x.y);
              a2[r][2 * j + 1] = pack_f2(x.z, x.w);
            } else {
              a2[r][2 * j + 0] = pack_f2(-2.0f * x.x, -2.0f * x.y);
              a2[r][2 * j + 1] = pack_f2(-2.0f * x.z, -2.0f * x.w);
            }
          }
        }
        float best[kRPL], second[kRPL];
        int bi[kRPL];
#pragma unroll
        for (int r = 0; r < kRPL; ++r) {
          best[r] = FLT_MAX;
          second[r] = FLT_MAX;
          bi[r] = 0;
        }
        const float* norms = cb + p.K * V;
        const uint32_t cb_s = smem_u32(cb);
#pragma unroll 2
        for (int k = 0; k < p.K; ++k) {
          const float pn = norms[k];
          uint64_t acc0[kRPL], acc1[kRPL];
#pragma unroll
          for (int r = 0; r < kRPL; ++r) {
            acc0[r] = CHAIN == 1 ? 0ull : pack_f2(pn, 0.0f);
            acc1[r] = 0ull;
          }
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            uint64_t q01, q23;
            asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];"
                         : "=l"(q01), "=l"(q23)
                         : "r"(cb_s + (uint32_t)((k * V + 4 * j) * 4)));
#pragma unroll
            for (int r = 0; r < kRPL; ++r) {
              if constexpr (CHAIN == 1) {
                acc0[r] = ffma2(a2[r][2 * j + 0], q01, acc0[r]);
                acc0[r] = ffma2(a2[r][2 * j + 1], q23, acc0[r]);
              } else {
                acc0[r] = ffma2(a2[r][2 * j + 0], q01, acc0[r]);
                acc1[r] = ffma2(a2[r][2 * j + 1], q23, acc1[r]);
              }
            }
          }
#pragma unroll
          for (int r = 0; r < kRPL; ++r) {
            float lo, hi;
            float d;
            if constexpr (CHAIN == 1) {
              unpack_f2(acc0[r], lo, hi);
              d = fmaf(-2.0f, lo + hi, pn);
            } else {
              unpack_f2(fadd2(acc0[r], acc1[r]), lo, hi);
              d = lo + hi;
            }
            second[r] = fminf(second[r], fmaxf(best[r], d));
            bi[r] = (d < best[r]) ? k : bi[r];
            best[r] = fminf(best[r], d);
          }
        }
        const float pmax = norms[p.K];
#pragma unroll
        for (int r = 0; r < kRPL; ++r) {
          const float tau = tau_c * (asq[r] + pmax);
          if (!(second[r] - best[r] > tau)) {
            // near tie (or NaN): exact f64 decision from the staged tile
            const int q_ = rr + r * kRowsPerPass;
          const float* rowp = reinterpret_cast<const float*>(st + (q_ >> 8) * kBoxBytes + (q_ & 255) * 128);
            auto get_a = [&](int j) {
              const int q = sb * NJ + (j >> 2);
              return rowp[((q ^ sw) << 2) + (j & 3)];
            };
            bi[r] = exact_argmin(get_a, cb, p.K, V);
            const int64_t row = tile * kTileRows + r * kRowsPerPass + rr;
            if (p.near_tie && row < p.n) atomicAdd(p.near_tie, 1);
          }
          // shift the code into the 128-bit per-row register
          const uint32_t code = (uint32_t)bi[r];
          if (p.code_bits == 8) {
            pk[r][0] = __funnelshift_r(pk[r][0], pk[r][1], 8);
            pk[r][1] = __funnelshift_r(pk[r][1], pk[r][2], 8);
            pk[r][2] = __funnelshift_r(pk[r][2], pk[r][3], 8);
            pk[r][3] = (pk[r][3] >> 8) | (code << 24);
          } else {
            pk[r][0] = __funnelshift_r(pk[r][0], pk[r][1], 4);
            pk[r][1] = __funnelshift_r(pk[r][1], pk[r][2], 4);
            pk[r][2] = __funnelshift_r(pk[r][2], pk[r][3], 4);
            pk[r][3] = (pk[r][3] >> 4) | (code << 28);
          }
        }
        ++ncodes;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == p.stages) {
        stage = 0;
        phase ^= 1;
      }
    }

    // flush this group's codes: right-align the shift register first
    const int bits = p.code_bits;
    const int slots = 128 / bits;
    for (int s = ncodes; s < slots; ++s) {
#pragma unroll
      for (int r = 0; r < kRPL; ++r) {
        pk[r][0] = __funnelshift_r(pk[r][0], pk[r][1], bits);
        pk[r][1] = __funnelshift_r(pk[r][1], pk[r][2], bits);
        pk[r][2] = __funnelshift_r(pk[r][2], pk[r][3], bits);
        pk[r][3] = pk[r][3] >> bits;
      }
    }
    const int nbytes = (ncodes * bits + 7) / 8;
    const int64_t off = (int64_t)c_begin * bits / 8;
#pragma unroll
    for (int r = 0; r < kRPL; ++r) {
      const int64_t row = tile * kTileRows + r * kRowsPerPass + rr;
      if (row < p.n)
        store_code_group(p.codes + row * p.code_stride + off, pk[r][0], pk[r][1], pk[r][2], pk[r][3],
                         nbytes);
    }
  }
}

// ------------------------------------------------------------ generic path

struct DenseRows {
  const float* a;
  int64_t lda;
  __device__ __forceinline__ float operator()(int64_t row, int col) const {
    return __ldg(a + row * lda + col);
  }
};

struct ConvRows {  // im2col on the fly; col = (ci, dy, dx) channel-major
  const float* x;
  int cin, h, w, kh, kw, stride, pad, ho, wo;
  __device__ __forceinline__ float operator()(int64_t row, int col) const {
    const int hw = ho * wo;
    const int64_t b = row / hw;
    const int pix = (int)(row - b * hw);
    const int oy = pix / wo, ox = pix - (pix / wo) * wo;
    const int kk = kh * kw;
    const int ci = col / kk;
    const int r = col - ci * kk;
    const int dy = r / kw, dx = r - (r / kw) * kw;
    const int iy = oy * stride + dy - pad, ix = ox * stride + dx - pad;
    if (iy < 0 || iy >= h || ix < 0 || ix >= w) return 0.0f;
    return __ldg(x + ((b * cin + ci) * (int64_t)h + iy) * w + ix);
  }
};

// VT: compile-time register capacity for the sub-vector (0 = stream from memory)
template <int VT, class Rows>
__global__ void __launch_bounds__(256) encode_rows_kernel(Rows rows, int64_t n, const float* __restrict__ prep,
                                                          int S, int C, int K, int V, uint8_t* __restrict__ codes,
                                                          int code_bits, int64_t code_stride, int* near_tie) {
  grid_launch_dependents();  // a programmatic dependent (the gather) may start staging
  extern __shared__ float sh[];  // up to 2 prepared codebook records
  const int cpt = (code_bits == 4) ? 2 : 1;  // codebooks per thread (nibble pairs share a byte)
  const int c0 = blockIdx.y * cpt;
  const int ncb = min(cpt, C - c0);
  for (int i = threadIdx.x; i < ncb * S; i += blockDim.x) sh[i] = prep[(size_t)c0 * S + i];
  __syncthreads();
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const float tau_c = tau_coef(V);
  uint32_t packed = 0;
  for (int s = 0; s < ncb; ++s) {
    const int c = c0 + s;
    const float* cb = sh + s * S;
    const float* norms = cb + K * V;
    float best = FLT_MAX, second = FLT_MAX, asq = 0.0f;
    int bi = 0;
    if constexpr (VT > 0) {
      float a[VT];
#pragma unroll
      for (int j = 0; j < VT; ++j) {
        float x = (j < V) ? rows(row, c * V + j) : 0.0f;
        asq = fmaf(x, x, asq);
        a[j] = -2.0f * x;
      }
      for (int k = 0; k < K; ++k) {
        float acc0 = norms[k], acc1 = 0.0f;
        const float* pkv = cb + k * V;
#pragma unroll
        for (int j = 0; j < VT; ++j) {
          if (j < V) {
            if (j & 1) acc1 = fmaf(a[j], pkv[j], acc1);
            else acc0 = fmaf(a[j], pkv[j], acc0);
          }
        }
        const float d = acc0 + acc1;
        second = fminf(second, fmaxf(best, d));
        bi = (d < best) ? k : bi;
        best = fminf(best, d);
      }
    } else {
      for (int j = 0; j < V; ++j) {
        float x = rows(row, c * V + j);
        asq = fmaf(x, x, asq);
      }
      for (int k = 0; k < K; ++k) {
        float acc0 = norms[k], acc1 = 0.0f;
        const float* pkv = cb + k * V;
        for (int j = 0; j < V; ++j) {
          const float x = -2.0f * rows(row, c * V + j);
          if (j & 1) acc1 = fmaf(x, pkv[j], acc1);
          else acc0 = fmaf(x, pkv[j], acc0);
        }
        const float d = acc0 + acc1;
        second = fminf(second, fmaxf(best, d));
        bi = (d < best) ? k : bi;
        best = fminf(best, d);
      }
    }
    if (!(second - best > tau_c * (asq + norms[K]))) {
      auto get_a = [&](int j) { return rows(row, c * V + j); };
      bi = exact_argmin(get_a, cb, K, V);
      if (near_tie) atomicAdd(near_tie, 1);
    }
    if (code_bits == 8) {
      codes[row * code_stride + c] = (uint8_t)bi;
    } else {
      packed |= (uint32_t)bi << (4 * s);
    }
  }
  if (code_bits == 4) codes[row * code_stride + c0 / 2] = (uint8_t)packed;
}

// ------------------------------------------------------- conv plane path
// A LutConv whose codebook is one input channel's kh x kw patch (V = kh*kw,
// C = Cin: configs[2]) encodes each (image, channel) plane independently.
// Unit = (plane group g of 8 channels, image b); units are g-major so a
// persistent CTA keeps its centroids in registers across consecutive units.
// The group's 8 planes (contiguous in NCHW) arrive by one cp.async.bulk into
// a double-buffered SMEM slot while the previous unit computes; warp w owns
// plane w: its K x V centroids live in registers as (k, k+1) pairs and every
// distance is FFMA2.  Padding is a predicate on the SMEM read, no halo copy.
// Codes are staged per unit and stored 8 channels (8 bytes) per pixel.

constexpr int kConvWarps = 8;

struct ConvPlaneParams {
  const float* x;
  const float* prep;
  int S;
  int batch, cin, h, w, stride, pad, ho, wo;
  int ngroups;
  int64_t nunits;
  uint8_t* codes;
  int64_t code_stride;
  int* near_tie;
  uint32_t plane_bytes;  // h*w*4
  uint32_t slot_bytes;   // 8 planes, 128-aligned
};

// Best / second-best / lowest-index argmin of 2*KP distances held as
// (2k, 2k+1) pairs, as a log-depth tree: a sequential scan is a 3-op dependent
// chain per centroid, which with 8 warps per SM left the kernel latency-bound.
// Ties keep the lower index (strict < when the higher-index half wins), the
// reference's np.argmin rule; equal best values give second == best, i.e. an
// exact tie that the caller re-decides in f64.
template <int KP>
__device__ __forceinline__ void argmin_tree(const uint64_t (&acc)[KP], float& best_out, float& second_out,
                                            int& idx_out) {
  float b[KP], s2[KP];
  int ix[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    float d0, d1;
    unpack_f2(acc[k], d0, d1);
    const bool pk = d1 < d0;
    b[k] = fminf(d0, d1);
    s2[k] = fmaxf(d0, d1);
    ix[k] = pk ? 2 * k + 1 : 2 * k;
  }
#pragma unroll
  for (int w = 1; w < KP; w *= 2) {
#pragma unroll
    for (int k = 0; k + w < KP; k += 2 * w) {
      const bool pk = b[k + w] < b[k];  // right (higher indices) wins only strictly
      const float hi = fmaxf(b[k], b[k + w]);
      s2[k] = fminf(hi, pk ? s2[k + w] : s2[k]);
      b[k] = fminf(b[k], b[k + w]);
      ix[k] = pk ? ix[k + w] : ix[k];
    }
  }
  best_out = b[0];
  second_out = s2[0];
  idx_out = ix[0];
}

template <int K, int KH>
__global__ void __launch_bounds__(kConvWarps * 32, 1) encode_conv_plane_kernel(ConvPlaneParams p) {
  grid_launch_dependents();  // a programmatic dependent (the gather) may start staging
  constexpr int V = KH * KH;
  constexpr int KP = K / 2;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  float* slot[2] = {reinterpret_cast<float*>(smem), reinterpret_cast<float*>(smem + p.slot_bytes)};
  uint8_t* cst = smem + 2 * p.slot_bytes;  // ho*wo x 8 code bytes
  uint64_t* bar = reinterpret_cast<uint64_t*>(cst + (((size_t)p.ho * p.wo * 8 + 15) & ~(size_t)15));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hw_out = p.ho * p.wo;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int64_t u, int s) {
    const int g = (int)(u / p.batch), b = (int)(u - (int64_t)g * p.batch);
    const int nplanes = min(kConvWarps, p.cin - g * kConvWarps);
    const uint32_t bytes = (uint32_t)nplanes * p.plane_bytes;
    mbar_arrive_expect_tx(&bar[s], bytes);
    bulk_load(slot[s], p.x + ((int64_t)b * p.cin + (int64_t)g * kConvWarps) * p.h * p.w, bytes, &bar[s]);
  };
  int64_t u = blockIdx.x;
  if (threadIdx.x == 0 && u < p.nunits) issue(u, 0);

  uint64_t cp[KP][V];  // centroid pairs (k even, k odd) per coordinate
  uint64_t np[KP];     // norm pairs
  float pmax = 0.0f;
  int cur_c = -1;
  const float tau_c = tau_coef(V);
  for (int it = 0; u < p.nunits; u += gridDim.x, ++it) {
    const int s = it & 1;
    const int g = (int)(u / p.batch), b = (int)(u - (int64_t)g * p.batch);
    if (threadIdx.x == 0 && u + gridDim.x < p.nunits) {
      fence_proxy_async_smem();
      issue(u + gridDim.x, s ^ 1);
    }
    const int c = g * kConvWarps + warp;
    if (c < p.cin && c != cur_c) {
      const float* rec = p.prep + (size_t)c * p.S;
#pragma unroll
      for (int k = 0; k < KP; ++k) {
#pragma unroll
        for (int j = 0; j < V; ++j) cp[k][j] = pack_f2(__ldg(rec + (2 * k) * V + j), __ldg(rec + (2 * k + 1) * V + j));
        np[k] = pack_f2(__ldg(rec + K * V + 2 * k), __ldg(rec + K * V + 2 * k + 1));
      }
      pmax = __ldg(rec + K * V + K);
      cur_c = c;
    }
    mbar_wait(&bar[s], (uint32_t)(it >> 1) & 1u);
    if (c < p.cin) {
      const float* plane = slot[s] + (size_t)warp * (p.plane_bytes / 4);
      // two pixels per lane per pass: independent FFMA2 / argmin chains for ILP
      constexpr int R = 2;
      const float inv_wo = 1.0f / (float)p.wo;
      for (int base = 0; base < hw_out; base += 32 * R) {
        int pixr[R], y0[R], x0[R];
        float a[R][V], asq[R];
        uint64_t acc[R][KP];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int pix = min(base + r * 32 + lane, hw_out - 1);  // clamped lanes recompute a valid pixel
          const int oy = __float2int_rz(((float)pix + 0.5f) * inv_wo), ox = pix - oy * p.wo;
          pixr[r] = base + r * 32 + lane;
          y0[r] = oy * p.stride - p.pad;
          x0[r] = ox * p.stride - p.pad;
          asq[r] = 0.0f;
#pragma unroll
          for (int dy = 0; dy < KH; ++dy) {
#pragma unroll
            for (int dx = 0; dx < KH; ++dx) {
              const int iy = y0[r] + dy, ix = x0[r] + dx;
              const bool in = (unsigned)iy < (unsigned)p.h && (unsigned)ix < (unsigned)p.w;
              const float v = in ? plane[iy * p.w + ix] : 0.0f;
              a[r][dy * KH + dx] = v;
              asq[r] = fmaf(v, v, asq[r]);
            }
          }
#pragma unroll
          for (int k = 0; k < KP; ++k) acc[r][k] = np[k];
        }
#pragma unroll
        for (int j = 0; j < V; ++j) {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const float m2 = -2.0f * a[r][j];
            const uint64_t a2 = pack_f2(m2, m2);
#pragma unroll
            for (int k = 0; k < KP; ++k) acc[r][k] = ffma2(a2, cp[k][j], acc[r][k]);
          }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float best, second;
          int bi;
          argmin_tree<KP>(acc[r], best, second, bi);
          if (pixr[r] < hw_out) {
            if (!(second - best > tau_c * (asq[r] + pmax))) {
              const int H = p.h, W = p.w, yy = y0[r], xx = x0[r];
              auto get_a = [plane, yy, xx, H, W](int j) {
                const int iy = yy + j / KH, ix = xx + j % KH;
                return ((unsigned)iy < (unsigned)H && (unsigned)ix < (unsigned)W) ? plane[iy * W + ix] : 0.0f;
              };
              bi = exact_argmin(get_a, p.prep + (size_t)c * p.S, K, V);
              if (p.near_tie) atomicAdd(p.near_tie, 1);
            }
            cst[pixr[r] * 8 + warp] = (uint8_t)bi;
          }
        }
      }
    }
    __syncthreads();  // codes staged; slot s fully consumed
    {
      const int nplanes = min(kConvWarps, p.cin - g * kConvWarps);
      uint8_t* dst0 = p.codes + ((int64_t)b * hw_out) * p.code_stride + g * kConvWarps;
      if (nplanes == kConvWarps && (p.code_stride & 7) == 0 && (reinterpret_cast<uintptr_t>(p.codes) & 7) == 0) {
        for (int pix = threadIdx.x; pix < hw_out; pix += blockDim.x)
          *reinterpret_cast<uint2*>(dst0 + (int64_t)pix * p.code_stride) = *reinterpret_cast<const uint2*>(cst + pix * 8);
      } else {
        for (int i = threadIdx.x; i < hw_out * nplanes; i += blockDim.x) {
          const int pix = i / nplanes, q = i - pix * nplanes;
          dst0[(int64_t)pix * p.code_stride + q] = cst[pix * 8 + q];
        }
      }
    }
    __syncthreads();  // code staging reusable
  }
}

template <int K, int KH>
static int launch_conv_plane(const float* x, int batch, int cin, int h, int w, int stride, int pad, int ho, int wo,
                             const float* prep, uint8_t* codes, int64_t code_stride, int* near_tie,
                             cudaStream_t stream, bool* used) {
  *used = false;
  ConvPlaneParams p;
  p.plane_bytes = (uint32_t)h * w * 4;
  if ((p.plane_bytes & 15) || (reinterpret_cast<uintptr_t>(x) & 15)) return LUT_OK;
  p.slot_bytes = (p.plane_bytes * kConvWarps + 127) & ~127u;
  const size_t smem = 2 * (size_t)p.slot_bytes + (((size_t)ho * wo * 8 + 15) & ~(size_t)15) + 16 + 128;
  if (smem > max_smem_optin()) return LUT_OK;
  p.x = x;
  p.prep = prep;
  p.S = prep_stride(K, KH * KH);
  p.batch = batch;
  p.cin = cin;
  p.h = h;
  p.w = w;
  p.stride = stride;
  p.pad = pad;
  p.ho = ho;
  p.wo = wo;
  p.ngroups = (cin + kConvWarps - 1) / kConvWarps;
  p.nunits = (int64_t)p.ngroups * batch;
  p.codes = codes;
  p.code_stride = code_stride;
  p.near_tie = near_tie;
  auto kern = encode_conv_plane_kernel<K, KH>;
  cudaError_t e = kernel_smem_attr(reinterpret_cast<const void*>(kern));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(encode_conv_plane)");
  const int nsm = num_sms();
  const int grid = (int)(p.nunits < nsm ? p.nunits : nsm);
  kern<<<grid, kConvWarps * 32, smem, stream>>>(p);
  LUT_CHECK_LAUNCH("encode_conv_plane_kernel");
  *used = true;
  return LUT_OK;
}

// ---------------------------------------------------------------- hash encode
// Depth-L tree traversal per (row, codebook) — hashing.encode_hash
// (lutkit/hashing.py:171-196): at level l go right iff value[dims[l]] > thr
// (left on <=), thresholds level-major, emit the reached leaf's index.
// L compares and no multiplications per sub-vector.

__global__ void encode_hash_kernel(const float* __restrict__ a, int64_t n, int d, const int* __restrict__ dims,
                                   const float* __restrict__ thr, const uint8_t* __restrict__ leaves, int C, int L,
                                   int V, uint8_t* __restrict__ codes, int64_t code_stride) {
  const int c = blockIdx.y;
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const float* sub = a + row * d + (int64_t)c * V;
  const int* dm = dims + c * L;
  const float* th = thr + (int64_t)c * ((1 << L) - 1);
  int node = 0, off = 0;
  for (int l = 0; l < L; ++l) {
    const float x = __ldg(sub + __ldg(dm + l));
    node = 2 * node + (x > __ldg(th + off + node) ? 1 : 0);
    off += 1 << l;
  }
  codes[row * code_stride + c] = __ldg(leaves + (int64_t)c * (1 << L) + node);
}

int encode_hash(const float* a, int64_t n, int d, const int* dims, const float* thr, const uint8_t* leaves, int C,
                int L, int V, uint8_t* codes, int64_t code_stride, cudaStream_t stream) {
  if (n == 0 || C == 0) return LUT_OK;
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)C);
  encode_hash_kernel<<<grid, 256, 0, stream>>>(a, n, d, dims, thr, leaves, C, L, V, codes, code_stride);
  LUT_CHECK_LAUNCH("encode_hash_kernel");
  return LUT_OK;
}

// ---------------------------------------------------------------- im2col

__global__ void im2col_kernel(ConvRows rows, int64_t n, int d, float* __restrict__ cols) {
  const int64_t total = n * d;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / d;
    const int col = (int)(i - row * d);
    cols[i] = rows(row, col);
  }
}

// ------------------------------------------------------------ host launch

static int launch_rows(const DenseRows* dense, const ConvRows* conv, int64_t n, const float* prep, int C,
                       int K, int V, uint8_t* codes, int code_bits, int64_t code_stride, int* near_tie,
                       cudaStream_t stream) {
  const int S = prep_stride(K, V);
  const int cpt = code_bits == 4 ? 2 : 1;
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)((C + cpt - 1) / cpt));
  const size_t smem = (size_t)cpt * S * sizeof(float);
#define LUT_ROWS_LAUNCH(VT)                                                                            \
  do {                                                                                                 \
    if (dense) {                                                                                       \
      auto kern = encode_rows_kernel<VT, DenseRows>;                                                   \
      if (smem > 48 * 1024) kernel_smem_attr(reinterpret_cast<const void*>(kern)); \
      kern<<<grid, 256, smem, stream>>>(*dense, n, prep, S, C, K, V, codes, code_bits, code_stride, near_tie); \
    } else {                                                                                           \
      auto kern = encode_rows_kernel<VT, ConvRows>;                                                    \
      if (smem > 48 * 1024) kernel_smem_attr(reinterpret_cast<const void*>(kern)); \
      kern<<<grid, 256, smem, stream>>>(*conv, n, prep, S, C, K, V, codes, code_bits, code_stride, near_tie); \
    }                                                                                                  \
  } while (0)
  if (V <= 1) LUT_ROWS_LAUNCH(1);
  else if (V <= 2) LUT_ROWS_LAUNCH(2);
  else if (V <= 3) LUT_ROWS_LAUNCH(3);
  else if (V <= 4) LUT_ROWS_LAUNCH(4);
  else if (V <= 8) LUT_ROWS_LAUNCH(8);
  else if (V <= 9) LUT_ROWS_LAUNCH(9);
  else if (V <= 16) LUT_ROWS_LAUNCH(16);
  else if (V <= 32) LUT_ROWS_LAUNCH(32);
  else if (V <= 64) LUT_ROWS_LAUNCH(64);
  else LUT_ROWS_LAUNCH(0);
#undef LUT_ROWS_LAUNCH
  LUT_CHECK_LAUNCH("encode_rows_kernel");
  return LUT_OK;
}

template <int V>
static int launch_tma(const float* a, int64_t n, int d, const float* prep, int C, int K, uint8_t* codes,
                      int code_bits, int64_t code_stride, int* near_tie, cudaStream_t stream, bool* used) {
  *used = false;
  const int S = prep_stride(K, V);
  constexpr int NB = 32 / V;
  const int book_bytes = NB * S * 4;
  const int stage_bytes = ((kTileBoxes * kBoxBytes + book_bytes) + 1023) & ~1023;
  const size_t budget = max_smem_optin();
  int stages = (int)((budget - 1024 - 256) / stage_bytes);
  if (stages > 4) stages = 4;
  if (stages < 2) return LUT_OK;  // does not fit: caller falls back
  CUtensorMap tmap;
  if (!make_tmap_2d_f32(&tmap, a, (uint64_t)d, (uint64_t)n, 32, kBoxRows, true)) return LUT_OK;

  EncTmaParams p;
  p.prep = prep;
  p.S = S;
  p.n = n;
  p.C = C;
  p.K = K;
  p.code_bits = code_bits;
  p.code_stride = code_stride;
  p.codes = codes;
  p.near_tie = near_tie;
  p.stages = stages;
  p.stage_bytes = stage_bytes;
  {
    const char* e = probe_env("LUTGPU_ENC_DEBUG");
    p.debug = e ? atoi(e) : 0;
    const char* st = probe_env("LUTGPU_ENC_STAGES");
    if (st && atoi(st) >= 2 && atoi(st) <= stages) p.stages = stages = atoi(st);
  }
  p.ntiles = (n + kTileRows - 1) / kTileRows;
  const int nsm = num_sms();
  // group = flush granularity: 16 B of codes per row, shrunk until the grid fills the chip
  // (powers of two >= NB, so a box never straddles groups; even for nibble pairs)
  int G = code_bits == 8 ? 16 : 32;
  const int gmin = (code_bits == 4 && NB < 2) ? 2 : NB;
  while (G > gmin && p.ntiles * ((C + G - 1) / G) < 2LL * nsm) G /= 2;
  p.G = G;
  p.ngroups = (C + G - 1) / G;
  const int64_t nunits = p.ntiles * p.ngroups;
  const int grid = (int)(nunits < nsm ? nunits : nsm);
  const size_t smem = (size_t)stages * stage_bytes + 2 * stages * sizeof(uint64_t) + 1024;
  // rows per lane (LUTGPU_ENC_RPL = 2 or 4; default 2), accumulator form (LUTGPU_ENC_CHAIN = 0 or 1)
  int rpl = 2, chain = 1;
  if (const char* r = probe_env("LUTGPU_ENC_RPL")) rpl = atoi(r) == 4 ? 4 : 2;
  if (const char* c = probe_env("LUTGPU_ENC_CHAIN")) chain = atoi(c) == 0 ? 0 : 1;
  auto kern = rpl == 2 ? (chain ? encode_tma_kernel<V, 8, 2, 1> : encode_tma_kernel<V, 8, 2, 0>)
                       : (chain ? encode_tma_kernel<V, 4, 4, 1> : encode_tma_kernel<V, 4, 4, 0>);
  const int threads = rpl == 2 ? 9 * 32 : 5 * 32;
  cudaError_t e = kernel_smem_attr(reinterpret_cast<const void*>(kern));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(encode_tma)");
  kern<<<grid, threads, smem, stream>>>(tmap, p);
  LUT_CHECK_LAUNCH("encode_tma_kernel");
  *used = true;
  return LUT_OK;
}

int encode_dense_tc(const float* a, int64_t n, int d, const float* prep, int C, int K, int V, uint8_t* codes,
                    int code_bits, int64_t code_stride, int* near_tie, cudaStream_t stream, bool* used);

int encode_dense(const float* a, int64_t n, int d, const float* prep, int C, int K, int V, uint8_t* codes,
                 int code_bits, int64_t code_stride, int* near_tie, cudaStream_t stream, int force_generic) {
  if (n == 0 || C == 0) return LUT_OK;
  const bool aligned = (reinterpret_cast<uintptr_t>(a) & 15) == 0 && (reinterpret_cast<uintptr_t>(prep) & 15) == 0;
  if (!force_generic && aligned && !(probe_env("LUTGPU_ENC_TC") && probe_env("LUTGPU_ENC_TC")[0] == '0')) {
    bool used = false;
    const int st = encode_dense_tc(a, n, d, prep, C, K, V, codes, code_bits, code_stride, near_tie, stream, &used);
    if (st != LUT_OK) return st;
    if (used) return LUT_OK;
  }
  if (!force_generic && aligned && K <= 128 && n >= kTileRows / 2) {
    bool used = false;
    int st = LUT_OK;
    switch (V) {
      case 4: st = launch_tma<4>(a, n, d, prep, C, K, codes, code_bits, code_stride, near_tie, stream, &used); break;
      case 8: st = launch_tma<8>(a, n, d, prep, C, K, codes, code_bits, code_stride, near_tie, stream, &used); break;
      case 16: st = launch_tma<16>(a, n, d, prep, C, K, codes, code_bits, code_stride, near_tie, stream, &used); break;
      case 32: st = launch_tma<32>(a, n, d, prep, C, K, codes, code_bits, code_stride, near_tie, stream, &used); break;
      default: break;
    }
    if (st != LUT_OK) return st;
    if (used) return LUT_OK;
  }
  DenseRows rows{a, d};
  return launch_rows(&rows, nullptr, n, prep, C, K, V, codes, code_bits, code_stride, near_tie, stream);
}

int launch_conv_tc(const float* x, int batch, int cin, int h, int w, int stride, int pad, int ho, int wo,
                   const float* prep, int K, uint8_t* codes, int64_t code_stride, int* near_tie, cudaStream_t stream,
                   bool* used);

int launch_conv_strip(const float* x, int batch, int cin, int h, int w, int stride, int pad, int ho, int wo,
                      const float* prep, int K, uint8_t* codes, int64_t code_stride, int* near_tie,
                      cudaStream_t stream, bool* used);

int encode_conv_strided(const float* x, int batch, int cin, int h, int w, int kh, int kw, int stride, int pad,
                        const float* prep, int C, int K, int V, uint8_t* codes, int64_t code_stride, int* near_tie,
                        cudaStream_t stream) {
  const int ho = (h + 2 * pad - kh) / stride + 1, wo = (w + 2 * pad - kw) / stride + 1;
  const int64_t n = (int64_t)batch * ho * wo;
  if (n == 0 || C == 0) return LUT_OK;
  ConvRows rows{x, cin, h, w, kh, kw, stride, pad, ho, wo};
  const char* force = probe_env("LUTGPU_CONV_GENERIC");
  if (kh == 3 && kw == 3 && V == 9 && C == cin && !(force && atoi(force))) {
    bool used = false;
    int st = LUT_OK;
    const char* strip_env = probe_env("LUTGPU_CONV_STRIP");
    if (K == 16 && !(strip_env && strip_env[0] == '0')) {
      // register-tiled pixel strips on the FP32 pipe (encode_conv_strip.cu)
      st = launch_conv_strip(x, batch, cin, h, w, stride, pad, ho, wo, prep, K, codes, code_stride, near_tie, stream,
                             &used);
      if (st != LUT_OK) return st;
      if (used) return LUT_OK;
    }
    const char* tc_env = probe_env("LUTGPU_CONV_TC");
    if (K == 16 && !(tc_env && tc_env[0] == '0')) {
      // tensor-core screening (encode_conv_tc.cu)
      st = launch_conv_tc(x, batch, cin, h, w, stride, pad, ho, wo, prep, K, codes, code_stride, near_tie, stream,
                          &used);
      if (st != LUT_OK) return st;
      if (used) return LUT_OK;
    }
    if (K == 16)
      st = launch_conv_plane<16, 3>(x, batch, cin, h, w, stride, pad, ho, wo, prep, codes, code_stride, near_tie,
                                    stream, &used);
    else if (K == 8)
      st = launch_conv_plane<8, 3>(x, batch, cin, h, w, stride, pad, ho, wo, prep, codes, code_stride, near_tie,
                                   stream, &used);
    if (st != LUT_OK) return st;
    if (used) return LUT_OK;
  }
  return launch_rows(nullptr, &rows, n, prep, C, K, V, codes, 8, code_stride, near_tie, stream);
}

int encode_conv(const float* x, int batch, int cin, int h, int w, int kh, int kw, int stride, int pad,
                const float* prep, int C, int K, int V, uint8_t* codes, int code_bits, int* near_tie,
                cudaStream_t stream) {
  if (code_bits == 8)
    return encode_conv_strided(x, batch, cin, h, w, kh, kw, stride, pad, prep, C, K, V, codes, C, near_tie, stream);
  const int ho = (h + 2 * pad - kh) / stride + 1, wo = (w + 2 * pad - kw) / stride + 1;
  const int64_t n = (int64_t)batch * ho * wo;
  if (n == 0 || C == 0) return LUT_OK;
  ConvRows rows{x, cin, h, w, kh, kw, stride, pad, ho, wo};
  return launch_rows(nullptr, &rows, n, prep, C, K, V, codes, code_bits, (C + 1) / 2, near_tie, stream);
}

int im2col(const float* x, int batch, int cin, int h, int w, int kh, int kw, int stride, int pad, float* cols,
           cudaStream_t stream) {
  const int ho = (h + 2 * pad - kh) / stride + 1, wo = (w + 2 * pad - kw) / stride + 1;
  const int64_t n = (int64_t)batch * ho * wo;
  const int d = cin * kh * kw;
  if (n == 0 || d == 0) return LUT_OK;
  ConvRows rows{x, cin, h, w, kh, kw, stride, pad, ho, wo};
  const int64_t total = n * d;
  const int blocks = (int)((total + 255) / 256 < 65535 * 8 ? (total + 255) / 256 : 65535 * 8);
  im2col_kernel<<<blocks, 256, 0, stream>>>(rows, n, d, cols);
  LUT_CHECK_LAUNCH("im2col_kernel");
  return LUT_OK;
}

int prepare_books(const float* books, int C, int K, int V, float* prep, cudaStream_t stream) {
  if (C == 0) return LUT_OK;
  prepare_books_kernel<<<C, 128, 0, stream>>>(books, C, K, V, prep);
  LUT_CHECK_LAUNCH("prepare_books_kernel");
  return LUT_OK;
}

}  // namespace lutgpu
