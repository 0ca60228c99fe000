// 3x3 conv LUT encode on the FP32 pipe, register-tiled over pixel strips
// (configs[2]: V = 9, C = Cin, K = 16, stride 1).
//
// Indices are identical to encode_hard (lutkit/pq.py:171-174: literal f64
// distances, ties -> lowest k) by the CUDA-core encoders' two exact steps
// (encode_dev.cuh): fp32 distances d_k = fma-chain(|p_k|^2, -2 a_j p_kj, j
// ascending); when the runner-up lies within tau_coef(9) (|a|^2 + max|p|^2) of the
// best the pair is re-decided from literal f64 differences.
//
// Geometry.  A pixel-channel costs 144 FMAs; the FP32 pipe (125 FMA/clk/SM
// measured, FFMA2 = FFMA in flops but half the issue slots) is the roofline
// SURVEY 8(d) names for this config.  The round-2 kernels sat far from it:
// the plane kernel (encode.cu) holds a channel's centroids in registers (255
// registers, 2 warps per scheduler, 48% issue) and the tensor-core screen
// (encode_conv_tc.cu) spends ~280 instructions per pixel-channel on the patch
// gather, the 3xTF32 split and the screen.  Here:
//   * warp = one input channel (its centroids are read as broadcast LDS.128 of
//     (-2 p_kj) for 4 centroids, no centroid registers), lane = a strip of P = 4
//     consecutive output pixels of one row: the 3 x 6 input window is loaded once
//     (4.5 LDS per pixel instead of 9) and each centroid load feeds 4 pixels
//     (2 FFMA2 per pixel per LDS.128);
//   * 64 distance accumulators + the window fit 128 registers: 16 warps per SM;
//   * the argmin is one min tree plus a 16-bit candidate mask (d_k <= best +
//     bound): a lone candidate is the answer, no second-best bookkeeping.
// ~170 issue slots and ~1.25 SMEM wavefronts per pixel-channel.
//
// Work: unit = (block of IB images, group of 8 channels), IB * Ho * Wo ~ 1024
// pixels; the unit's planes (8 channels of one image are contiguous in NCHW)
// arrive by bulk copy into a double-buffered slot while the previous unit
// computes.  Units are group-major: a CTA restages its 8 centroid records only
// when the group changes.  Codes are staged per unit and stored 8 channels
// (8 bytes) per pixel.  Padding is a predicate on the window loads.

#include <float.h>

#include "common.cuh"
#include "encode_dev.cuh"

namespace lutgpu {

namespace {

constexpr int kCsWarps = 8;                       // channels per unit = warps per CTA
constexpr int kCsK = 16, kCsV = 9;
constexpr int kCsRec = kCsV * kCsK + kCsK + 4;    // floats per staged channel: [j][k] (-2 p), |p_k|^2 x16, max|p|^2, pad

struct ConvStripParams {
  const float* x;
  const float* prep;
  int S;
  int batch, cin, h, w, pad, ho, wo;
  int ib;       // images per unit
  int nblk;     // ceil(batch / ib)
  int64_t nunits;
  int spr;      // strips per output row
  int spi;      // strips per image
  uint8_t* codes;
  int64_t code_stride;
  int* near_tie;
  uint32_t plane_floats;
  uint32_t slot_bytes;  // ib x 8 planes, 128-aligned
};

__device__ __forceinline__ uint64_t cs_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void cs_unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t cs_ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int P>
__global__ void __launch_bounds__(kCsWarps * 32, 2) encode_conv_strip_kernel(const ConvStripParams p) {
  grid_launch_dependents();  // a programmatic dependent (the gather) may start staging
  constexpr int K = kCsK, V = kCsV, KH = 3, W6 = P + 2;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  float* slot0 = reinterpret_cast<float*>(smem);  // slot s at slot0 + s * slot_floats (shared-space arithmetic: LDS, not LD)
  const uint32_t slot_floats = p.slot_bytes / 4;
  float* cent = reinterpret_cast<float*>(smem + 2 * p.slot_bytes);
  uint8_t* cst = reinterpret_cast<uint8_t*>(cent + kCsWarps * kCsRec);
  const int hw_out = p.ho * p.wo;
  const int npx = p.ib * hw_out;  // staged code bytes per channel
  uint64_t* bar = reinterpret_cast<uint64_t*>(cst + (((size_t)p.ib * hw_out * 8 + 15) & ~(size_t)15));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // it-th unit of this CTA.  When the grid is a multiple of the channel groups a CTA
  // stays on one group (its centroid records are staged once); otherwise units are
  // walked group-major with a grid stride.
  const int ngroups = (p.cin + kCsWarps - 1) / kCsWarps;
  const bool pinned = gridDim.x % ngroups == 0;
  const int bstep = pinned ? gridDim.x / ngroups : 0;
  auto unit_at = [&](int it, int& g, int& bb) -> bool {
    if (pinned) {
      g = blockIdx.x % ngroups;
      bb = blockIdx.x / ngroups + it * bstep;
      return bb < p.nblk;
    }
    const int64_t u = blockIdx.x + (int64_t)it * gridDim.x;
    g = (int)(u / p.nblk);
    bb = (int)(u - (int64_t)g * p.nblk);
    return u < p.nunits;
  };
  auto issue = [&](int g, int bb, int s) {
    const int b0 = bb * p.ib;
    const int nimg = min(p.ib, p.batch - b0);
    const int nplanes = min(kCsWarps, p.cin - g * kCsWarps);
    const uint32_t bytes = (uint32_t)nplanes * p.plane_floats * 4u;
    mbar_arrive_expect_tx(&bar[s], bytes * (uint32_t)nimg);
    for (int i = 0; i < nimg; ++i)
      bulk_load(slot0 + (size_t)s * slot_floats + (size_t)i * kCsWarps * p.plane_floats,
                p.x + ((int64_t)(b0 + i) * p.cin + (int64_t)g * kCsWarps) * p.plane_floats, bytes, &bar[s]);
  };
  int g, bb;
  bool live = unit_at(0, g, bb);
  if (threadIdx.x == 0 && live) issue(g, bb, 0);

  const float tau_c = tau_coef(V);
  const float inv_ho = 1.0f / (float)p.ho, inv_spr = 1.0f / (float)p.spr;
  int cur_g = -1;
  for (int it = 0; live; ++it) {
    const int s = it & 1;
    const int b0 = bb * p.ib;
    const int nimg = min(p.ib, p.batch - b0);
    const int rlo = 0, rhi = nimg * p.ho;  // the unit's rows (image-major)
    int g_next, bb_next;
    const bool live_next = unit_at(it + 1, g_next, bb_next);
    if (threadIdx.x == 0 && live_next) {
      fence_proxy_async_smem();
      issue(g_next, bb_next, s ^ 1);
    }
    if (g != cur_g) {
      // stage the group's centroid records: [j][k] of -2 p_kj (exact scaling), norms, max norm
      for (int i = threadIdx.x; i < kCsWarps * (K * V + K + 1); i += blockDim.x) {
        const int ch = i / (K * V + K + 1), r = i - ch * (K * V + K + 1);
        const int c = g * kCsWarps + ch;
        float val = 0.0f;
        if (c < p.cin) {
          const float* rec = p.prep + (size_t)c * p.S;
          if (r < K * V) {
            const int j = r / K, k = r - j * K;
            val = -2.0f * __ldg(rec + k * V + j);
          } else {
            val = __ldg(rec + r);  // norms at K*V .. K*V+K-1, max norm at K*V+K
          }
        }
        cent[ch * kCsRec + r] = val;
      }
      cur_g = g;
      __syncthreads();
    }
    mbar_wait(&bar[s], (uint32_t)(it >> 1) & 1u);
    const int c = g * kCsWarps + warp;
    if (c < p.cin) {
      const float* cw = cent + warp * kCsRec;
      const float pmax = cw[K * V + K];
      for (int st = rlo * p.spr + lane; st < rhi * p.spr; st += 32) {
        // strip -> (unit row = image * Ho + output row, first output column); exact for these small integers
        const int row = __float2int_rz(((float)st + 0.5f) * inv_spr);
        const int xs = (st - row * p.spr) * P;
        const int img = __float2int_rz(((float)row + 0.5f) * inv_ho);
        const int oy = row - img * p.ho;
        const float* plane = slot0 + (uint32_t)s * slot_floats + (uint32_t)(img * kCsWarps + warp) * p.plane_floats;
        const int y0 = oy - p.pad, x0 = xs - p.pad;
        float v[KH][W6];
        // pad <= 1 and stride 1: only the window's first and last column can fall outside the row
        const bool cl = (unsigned)x0 < (unsigned)p.w, cr = (unsigned)(x0 + P + 1) < (unsigned)p.w;
#pragma unroll
        for (int dy = 0; dy < KH; ++dy) {
          const int iy = y0 + dy;
          const bool rok = (unsigned)iy < (unsigned)p.h;
          const float* rp = plane + iy * p.w + x0;
          v[dy][0] = (rok && cl) ? rp[0] : 0.0f;
#pragma unroll
          for (int xx = 1; xx <= P; ++xx) v[dy][xx] = rok ? rp[xx] : 0.0f;
          v[dy][P + 1] = (rok && cr) ? rp[P + 1] : 0.0f;
        }
        uint64_t acc[P][K / 2];
        {
          const float4 n0 = *reinterpret_cast<const float4*>(cw + K * V + 0);
          const float4 n1 = *reinterpret_cast<const float4*>(cw + K * V + 4);
          const float4 n2 = *reinterpret_cast<const float4*>(cw + K * V + 8);
          const float4 n3 = *reinterpret_cast<const float4*>(cw + K * V + 12);
          const uint64_t np[K / 2] = {cs_pack(n0.x, n0.y), cs_pack(n0.z, n0.w), cs_pack(n1.x, n1.y),
                                      cs_pack(n1.z, n1.w), cs_pack(n2.x, n2.y), cs_pack(n2.z, n2.w),
                                      cs_pack(n3.x, n3.y), cs_pack(n3.z, n3.w)};
#pragma unroll
          for (int i = 0; i < P; ++i)
#pragma unroll
            for (int q = 0; q < K / 2; ++q) acc[i][q] = np[q];
        }
#pragma unroll
        for (int dy = 0; dy < KH; ++dy) {
#pragma unroll
          for (int dx = 0; dx < KH; ++dx) {
            const float* cj = cw + (dy * KH + dx) * K;
            const float4 c0 = *reinterpret_cast<const float4*>(cj + 0);
            const float4 c1 = *reinterpret_cast<const float4*>(cj + 4);
            const float4 c2 = *reinterpret_cast<const float4*>(cj + 8);
            const float4 c3 = *reinterpret_cast<const float4*>(cj + 12);
            const uint64_t cp[K / 2] = {cs_pack(c0.x, c0.y), cs_pack(c0.z, c0.w), cs_pack(c1.x, c1.y),
                                        cs_pack(c1.z, c1.w), cs_pack(c2.x, c2.y), cs_pack(c2.z, c2.w),
                                        cs_pack(c3.x, c3.y), cs_pack(c3.z, c3.w)};
#pragma unroll
            for (int i = 0; i < P; ++i) {
              const float a = v[dy][i + dx];
              const uint64_t a2 = cs_pack(a, a);
#pragma unroll
              for (int q = 0; q < K / 2; ++q) acc[i][q] = cs_ffma2(a2, cp[q], acc[i][q]);
            }
          }
        }
        // |a|^2 per pixel from column sums (only scales the near-tie bound)
        float csq[W6];
#pragma unroll
        for (int xx = 0; xx < W6; ++xx) csq[xx] = fmaf(v[2][xx], v[2][xx], fmaf(v[1][xx], v[1][xx], v[0][xx] * v[0][xx]));
        const int pl0 = img * hw_out + oy * p.wo + xs;
        uint32_t cpk = 0u;
#pragma unroll
        for (int i = 0; i < P; ++i) {
          float d[K];
#pragma unroll
          for (int q = 0; q < K / 2; ++q) cs_unpack(acc[i][q], d[2 * q], d[2 * q + 1]);
          float m4[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) m4[q] = fminf(fminf(d[4 * q], d[4 * q + 1]), fminf(d[4 * q + 2], d[4 * q + 3]));
          const float best = fminf(fminf(m4[0], m4[1]), fminf(m4[2], m4[3]));
          const float asq = (csq[i] + csq[i + 1] + csq[i + 2]) * 1.000001f;
          const float lim = __fadd_ru(best, __fmul_ru(tau_c, asq + pmax));
          uint32_t mask = 0u;
#pragma unroll
          for (int k = 0; k < K; ++k) mask |= (d[k] <= lim) ? (1u << k) : 0u;
          int bi = __ffs((int)mask) - 1;
          if (mask == 0u || (mask & (mask - 1u)) != 0u) {
            // near tie (or NaN): literal f64 re-decision over all K (encode_hard semantics)
            const int H = p.h, Wd = p.w, yy = y0, xx0 = x0 + i;
            auto get_a = [plane, yy, xx0, H, Wd](int j) {
              const int iy = yy + j / KH, ix = xx0 + j % KH;
              return ((unsigned)iy < (unsigned)H && (unsigned)ix < (unsigned)Wd) ? plane[iy * Wd + ix] : 0.0f;
            };
            bi = exact_argmin(get_a, p.prep + (size_t)c * p.S, K, V);
            if (p.near_tie) atomicAdd(p.near_tie, 1);
          }
          cpk |= (uint32_t)bi << (8 * i);
        }
        // channel-major staging: the strip's P codes are one conflict-free store
        if (P == 4) *reinterpret_cast<uint32_t*>(cst + warp * npx + pl0) = cpk;
        else *reinterpret_cast<uint16_t*>(cst + warp * npx + pl0) = (uint16_t)cpk;
      }
    }
    __syncthreads();  // codes staged; slot s fully consumed
    {
      const int nplanes = min(kCsWarps, p.cin - g * kCsWarps);
      const int pix0 = rlo * p.wo, npix = rhi * p.wo;  // the range's pixels of this unit
      uint8_t* dst0 = p.codes + ((int64_t)b0 * hw_out) * p.code_stride + g * kCsWarps;
      if (nplanes == kCsWarps && (p.code_stride & 7) == 0 && (reinterpret_cast<uintptr_t>(p.codes) & 7) == 0 &&
          ((pix0 | npix | npx) & 3) == 0) {
        // 4 pixels per thread: one word per channel, transposed to 8 code bytes per pixel
        for (int pix = pix0 + 4 * threadIdx.x; pix < npix; pix += 4 * blockDim.x) {
          uint32_t wq[kCsWarps];
#pragma unroll
          for (int q = 0; q < kCsWarps; ++q) wq[q] = *reinterpret_cast<const uint32_t*>(cst + q * npx + pix);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint32_t sel = (uint32_t)i | ((uint32_t)(4 + i) << 4);  // byte i of each word
            const uint32_t t01 = __byte_perm(wq[0], wq[1], sel), t23 = __byte_perm(wq[2], wq[3], sel);
            const uint32_t t45 = __byte_perm(wq[4], wq[5], sel), t67 = __byte_perm(wq[6], wq[7], sel);
            uint2 o;
            o.x = __byte_perm(t01, t23, 0x5410);
            o.y = __byte_perm(t45, t67, 0x5410);
            *reinterpret_cast<uint2*>(dst0 + (int64_t)(pix + i) * p.code_stride) = o;
          }
        }
      } else {
        for (int i = pix0 * nplanes + threadIdx.x; i < npix * nplanes; i += blockDim.x) {
          const int pix = i / nplanes, q = i - pix * nplanes;
          dst0[(int64_t)pix * p.code_stride + q] = cst[q * npx + pix];
        }
      }
    }
    __syncthreads();  // code staging reusable
    live = live_next;
    g = g_next;
    bb = bb_next;
  }
}

template <int P>
int launch_strip(ConvStripParams& p, size_t smem, cudaStream_t stream) {
  auto kern = encode_conv_strip_kernel<P>;
  cudaError_t e = kernel_smem_attr(reinterpret_cast<const void*>(kern));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(encode_conv_strip)");
  const int64_t cap = 2 * (int64_t)num_sms();
  const int grid = (int)(p.nunits < cap ? p.nunits : cap);
  kern<<<grid, kCsWarps * 32, smem, stream>>>(p);
  LUT_CHECK_LAUNCH("encode_conv_strip_kernel");
  return LUT_OK;
}

}  // namespace

// Returns LUT_OK with *used = false when the shape is not this kernel's (the
// caller falls back to the tensor-core / plane kernels).
int launch_conv_strip(const float* x, int batch, int cin, int h, int w, int stride, int pad, int ho, int wo,
                      const float* prep, int K, uint8_t* codes, int64_t code_stride, int* near_tie,
                      cudaStream_t stream, bool* used) {
  *used = false;
  if (K != kCsK || stride != 1 || pad > 1 || (wo & 1)) return LUT_OK;
  const int64_t plane_bytes = (int64_t)h * w * 4;
  if ((plane_bytes & 15) || (reinterpret_cast<uintptr_t>(x) & 15)) return LUT_OK;
  const int hw_out = ho * wo;
  if (hw_out <= 0 || hw_out > 4096) return LUT_OK;
  ConvStripParams p;
  const int P = (wo & 3) == 0 ? 4 : 2;
  // ~1024 output pixels per unit (512 and 256 measured slower: more per-unit staging / syncs)
  constexpr int kUnitPx = 1024;
  p.ib = hw_out >= kUnitPx ? 1 : (kUnitPx / hw_out < batch ? kUnitPx / hw_out : batch);
  p.plane_floats = (uint32_t)(h * w);
  p.slot_bytes = (uint32_t)(((int64_t)p.ib * kCsWarps * plane_bytes + 127) & ~(int64_t)127);
  const size_t smem = 2 * (size_t)p.slot_bytes + kCsWarps * kCsRec * 4 + (((size_t)p.ib * hw_out * 8 + 15) & ~(size_t)15) +
                      16 + 128;
  if (smem > 110 * 1024) return LUT_OK;  // two CTAs per SM
  p.x = x;
  p.prep = prep;
  p.S = prep_stride(kCsK, kCsV);
  p.batch = batch;
  p.cin = cin;
  p.h = h;
  p.w = w;
  p.pad = pad;
  p.ho = ho;
  p.wo = wo;
  p.nblk = (batch + p.ib - 1) / p.ib;
  p.nunits = (int64_t)((cin + kCsWarps - 1) / kCsWarps) * p.nblk;
  p.spr = wo / P;
  p.spi = ho * p.spr;
  p.codes = codes;
  p.code_stride = code_stride;
  p.near_tie = near_tie;
  const int st = P == 4 ? launch_strip<4>(p, smem, stream) : launch_strip<2>(p, smem, stream);
  if (st != LUT_OK) return st;
  *used = true;
  return LUT_OK;
}

}  // namespace lutgpu
