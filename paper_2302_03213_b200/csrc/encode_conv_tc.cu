// 3x3 conv LUT encode with tensor-core candidate screening (configs[2]).
//
// A LutConv whose codebook is one input channel's 3x3 patch (V = 9, C = Cin,
// model.py:179-218) encodes every output pixel against each channel's K = 16
// centroids.  Indices are identical to encode_hard (lutkit/pq.py:171-174:
// literal f64 distances, ties -> lowest k), by the same two exact steps as
// encode_tc.cu:
//   1. Screen: per (128-pixel tile, channel) 3xTF32 tcgen05.mma.kind::tf32
//      (M = 128 pixels, N = 16 centroids, K = 16: the 9 patch values + zeros,
//      two K = 8 steps x {a_hi.p_hi, a_hi.p_lo, a_lo.p_hi}) computes every a.p_k
//      to ~2^-19 relative.  With D = 2^-15 |a| max|p_k| + 2^-21 (|a|^2 +
//      max|p_k|^2) (>= 2x the error bound) every k with d~_k > min d~ + 2D is
//      provably not the argmin; a lone candidate is it.  (Plain tf32 — 2^-7
//      instead of 2^-15 — left >= 2 candidates in most 32-pixel warps at V = 9,
//      and the divergent refinement cost more than the FFMA kernel.)
//   2. Refine the rest in fp32 (d = fma(-2, a.p, |p|^2)) and, within TAU,
//      re-decide from literal f64 differences over the candidates.
// The patches never exist in HBM (no im2col): each thread (= pixel = TMEM
// lane) gathers its 9 values from the channel plane in SMEM (padding is a
// predicate) and writes them straight into TMEM as the MMA's A operand.
// Versus the FFMA plane kernel (encode.cu, 144 FMAs + a 16-way argmin per
// pixel-channel, 255 registers, 2 warps per scheduler) a pixel-channel costs
// 9 LDS + one TMEM store + one TMEM load + the screen.
//
// Work: a unit = (512 consecutive output pixels, 16-channel group); units are
// group-major so a CTA rebuilds its centroid tiles only when the group changes.
// CTA = 4 groups of 4 warps (one 128-pixel tile each) + 1 producer warp.  The
// unit's input planes (the images its pixels belong to, the group's 16
// channels: contiguous in NCHW) arrive by bulk copy into a double-buffered slot.
// Per group a 2-deep pipeline over channels: gather + TMEM store of channel c
// and its MMA, then the screen of channel c - 1 while the MMA runs.

#include <float.h>

#include "common.cuh"

namespace lutgpu {

constexpr int kCtGroups = 4;                    // 128-pixel tiles per unit
constexpr int kCtRows = 128 * kCtGroups;        // output pixels per unit
constexpr int kCtCh = 16;                       // channels per unit
constexpr int kCtThreads = (4 * kCtGroups + 1) * 32;
constexpr int kCtBTile = 16 * 128;              // 16 centroids x 32 tf32 (K padded), 128B swizzle

struct ConvTcParams {
  const float* x;
  const float* prep;
  int S;  // prep record stride (floats)
  int batch, cin, h, w, stride, pad, ho, wo;
  int64_t nrows;      // batch * ho * wo
  int64_t nchunks;    // ceil(nrows / 512)
  int ngroups;        // ceil(cin / 16)
  int64_t nunits;
  int imgs;           // images per chunk (slot capacity)
  uint32_t slot_bytes;
  uint8_t* codes;
  int64_t code_stride;
  int* near_tie;
};

__device__ __forceinline__ uint64_t ct_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;  // 8-row atoms 1 KB apart
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}

// kind::tf32, D f32, A (TMEM) / B (SMEM, K-major) tf32, M = 128, N = 16
constexpr uint32_t kCtIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (2u << 17) | (8u << 24);

__device__ __forceinline__ void ct_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void ct_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}

// Screen one (pixel, channel): dv = the 16 3xTF32 values D_k = a.p_k - |p_k|^2/2
// from TMEM (the MMA's K column 9 holds A = 1 against B = -|p_k|^2/2, so
// D_k = -d~_k / 2), a = the fp32 patch, asq = |a|^2, ax = [|p_k|^2 x16, max|p|^2,
// 2^-15 max|p| (up)], cp = the channel's fp32 centroids.  Returns the encode_hard index.
__device__ __forceinline__ int conv_screen(const uint32_t (&dv)[16], const float (&a)[9], float asq, const float* ax,
                                          const float* cp, float tau_c, int* near_tie, bool live) {
  constexpr int V = 9, K = 16;
  // |D_k + d_k / 2| <= hwd / 2 with hwd = 2^-15 |a| max|p_k| + 2^-19 (|a|^2 + max|p_k|^2):
  // the 3xTF32 dot error <= 3 * 2^-20 sum|a_j p_j| (the dropped a_lo.p_lo and the
  // truncations of the low parts), |p_k|^2 / 2 split hi + lo (the lo part truncated:
  // 2^-21 |p_k|^2) and the fp32 accumulation over 6 chained MMAs, with a 2x margin;
  // every k with D_k < max D - hwd is provably not the argmin.  The absolute floor
  // keeps the bound positive for vanishing operands.
  const float al = __fmul_ru(__fsqrt_ru(asq), 1.0000002f);
  const float hwd = fmaf(al, ax[K + 1], fmaf(1.9073486e-6f, asq + ax[K], 1e-30f));
  float dt[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) dt[k] = __uint_as_float(dv[k]);
  float mx = fmaxf(fmaxf(dt[0], dt[1]), fmaxf(dt[2], dt[3]));
#pragma unroll
  for (int k = 4; k < 16; k += 4) mx = fmaxf(mx, fmaxf(fmaxf(dt[k], dt[k + 1]), fmaxf(dt[k + 2], dt[k + 3])));
  const float thr = __fsub_rd(mx, hwd);
  uint32_t mask = 0u;
#pragma unroll
  for (int k = 0; k < 16; ++k) mask |= (dt[k] >= thr) ? (1u << k) : 0u;
  if (mask != 0u && (mask & (mask - 1u)) == 0u) return __ffs((int)mask) - 1;
  // refine the candidates in fp32 (d = fma(-2, a.p, |p|^2), encode.cu's formulation)
  float best = FLT_MAX, second = FLT_MAX;
  int bi = 0;
  uint32_t m = mask;
  while (m) {
    const int k = __ffs((int)m) - 1;
    m &= m - 1u;
    float dot = 0.0f;
#pragma unroll
    for (int j = 0; j < V; ++j) dot = fmaf(a[j], cp[k * V + j], dot);
    const float dk = fmaf(-2.0f, dot, ax[k]);
    second = fminf(second, fmaxf(best, dk));
    bi = (dk < best) ? k : bi;
    best = fminf(best, dk);
  }
  if (second - best > tau_c * (asq + ax[K])) return bi;
  // near tie (or NaN): literal f64 differences over the candidates (all K for NaN)
  double bd = 0.0;
  int bk = -1;
  uint32_t mm = mask ? mask : 0xFFFFu;
  while (mm) {
    const int k = __ffs((int)mm) - 1;
    mm &= mm - 1u;
    double sacc = 0.0;
    for (int j = 0; j < V; ++j) {
      const double diff = (double)a[j] - (double)cp[k * V + j];
      sacc = __dadd_rn(sacc, __dmul_rn(diff, diff));
    }
    if (bk < 0 || sacc < bd) {
      bd = sacc;
      bk = k;
    }
  }
  if (near_tie && live) atomicAdd(near_tie, 1);
  return bk;
}

__global__ void __launch_bounds__(kCtThreads, 1) encode_conv_tc_kernel(const ConvTcParams p) {
  grid_launch_dependents();  // a programmatic dependent (the gather) may start staging
  constexpr int V = 9, K = 16;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* btiles = smem;                                        // [16 ch][hi, lo][2 KB]
  float* aux = reinterpret_cast<float*>(btiles + 2 * kCtCh * kCtBTile);  // [16 ch][K norms, pmax, 2^-15 maxp, pad]
  float* cent = aux + kCtCh * 32;                                // [16 ch][K x V] fp32 centroids (refine / f64)
  uint8_t* slots = reinterpret_cast<uint8_t*>(cent + kCtCh * K * V);
  slots += (128u - (smem_u32(slots) & 127u)) & 127u;
  uint8_t* cst = slots + 2 * p.slot_bytes;                       // [512 rows][16 codes]
  uint64_t* bars = reinterpret_cast<uint64_t*>(cst + kCtRows * 16);
  uint64_t* slot_full = bars;                                    // [2]
  uint64_t* dfull = bars + 2;                                    // [groups][2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 + 2 * kCtGroups);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hw_out = p.ho * p.wo;
  const int plane = p.h * p.w;

  if (threadIdx.x == 0) {
    mbar_init(&slot_full[0], 1);
    mbar_init(&slot_full[1], 1);
    for (int i = 0; i < 2 * kCtGroups; ++i) mbar_init(&dfull[i], 1);
    fence_mbar_init();
  }
  if (warp == 4 * kCtGroups) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  auto unit_geom = [&](int64_t u, int& g, int64_t& r0, int& b0, int& nimg, int& nch) {
    g = (int)(u / p.nchunks);
    r0 = (u - (int64_t)g * p.nchunks) * kCtRows;
    b0 = (int)(r0 / hw_out);
    const int64_t r1 = min(p.nrows, r0 + kCtRows) - 1;
    nimg = (int)(r1 / hw_out) - b0 + 1;
    nch = min(kCtCh, p.cin - g * kCtCh);
  };

  if (warp == 4 * kCtGroups) {
    // ------------------------------------------------ producer: input planes of each unit
    // (the whole warp walks the units: bar.sync is warp-aligned; lane 0 issues the copies)
    int it = 0;
    for (int64_t u = blockIdx.x; u < p.nunits; u += gridDim.x, ++it) {
      int g, b0, nimg, nch;
      int64_t r0;
      unit_geom(u, g, r0, b0, nimg, nch);
      const int s = it & 1;
      // the slot is free once every compute thread has passed the unit that used it
      if (it >= 2) named_barrier_sync(1 + s, kCtThreads);
      if (lane == 0) {
        const uint32_t bytes = (uint32_t)(nch * plane * 4);
        mbar_arrive_expect_tx(&slot_full[s], bytes * (uint32_t)nimg);
        for (int i = 0; i < nimg; ++i)
          bulk_load(slots + s * p.slot_bytes + (size_t)i * kCtCh * plane * 4,
                    p.x + ((int64_t)(b0 + i) * p.cin + (int64_t)g * kCtCh) * plane, bytes, &slot_full[s]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------ compute groups
    const int grp = warp >> 2, q = warp & 3;
    const int r_local = grp * 128 + q * 32 + lane;  // pixel within the unit
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(grp * 128);
    const float tau_c = (4.0f * V + 16.0f) * 5.9604645e-8f;
    uint32_t dphase = 0u;  // bit b: parity of dfull[grp][b]
    int cur_g = -1;
    int it = 0;
    for (int64_t u = blockIdx.x; u < p.nunits; u += gridDim.x, ++it) {
      int g, b0, nimg, nch;
      int64_t r0;
      unit_geom(u, g, r0, b0, nimg, nch);
      const int s = it & 1;
      if (g != cur_g) {
        // centroid tiles of this channel group (all compute threads; the previous
        // unit's MMAs have completed: every group waited on its last D)
        named_barrier_sync(3, 4 * kCtGroups * 32);
        const int t = threadIdx.x;
        for (int i = t; i < kCtCh * kCtBTile / 4; i += 4 * kCtGroups * 32) {
          const int ch = i >> 9, rem = i & 511, k = rem >> 5, kk = rem & 31;  // 512 floats per tile
          const int c = g * kCtCh + ch;
          float v = 0.0f;
          if (c < p.cin && kk < V) v = __ldg(p.prep + (size_t)c * p.S + k * V + kk);
          if (c < p.cin && kk == V) v = -0.5f * __ldg(p.prep + (size_t)c * p.S + K * V + k);  // against A = 1
          const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);  // tf32(p), then p - tf32(p)
          const int off = k * 32 + ((((kk >> 2) ^ (k & 7)) << 2) | (kk & 3));
          reinterpret_cast<float*>(btiles + (2 * ch) * kCtBTile)[off] = hi;
          reinterpret_cast<float*>(btiles + (2 * ch + 1) * kCtBTile)[off] = v - hi;
        }
        for (int i = t; i < kCtCh * K * V; i += 4 * kCtGroups * 32) {
          const int ch = i / (K * V), rem = i - ch * (K * V);
          const int c = g * kCtCh + ch;
          cent[i] = c < p.cin ? __ldg(p.prep + (size_t)c * p.S + rem) : 0.0f;
        }
        for (int i = t; i < kCtCh * 32; i += 4 * kCtGroups * 32) {
          const int ch = i >> 5, j = i & 31;
          const int c = g * kCtCh + ch;
          float v = 0.0f;
          if (c < p.cin) {
            const float* rec = p.prep + (size_t)c * p.S;
            if (j < K) v = __ldg(rec + K * V + j);                              // |p_k|^2
            else if (j == K) v = __ldg(rec + K * V + K);                        // max |p_k|^2
            else if (j == K + 1) v = __fmul_ru(__fsqrt_ru(__ldg(rec + K * V + K)), 3.0517578e-05f);  // 2^-15 max|p_k| (up)
          }
          aux[i] = v;
        }
        fence_proxy_async_smem();  // generic-proxy writes of the B tiles -> the tensor core's async proxy
        named_barrier_sync(3, 4 * kCtGroups * 32);
        cur_g = g;
      }
      mbar_wait(&slot_full[s], (uint32_t)(it >> 1) & 1u);
      const float* pl = reinterpret_cast<const float*>(slots + s * p.slot_bytes);
      const int64_t row = r0 + r_local;
      const bool live = row < p.nrows;
      const int64_t rr = live ? row : p.nrows - 1;
      const int bl = (int)(rr / hw_out) - b0, pix = (int)(rr - (int64_t)(b0 + bl) * hw_out);
      const int oy = pix / p.wo, ox = pix - oy * p.wo;
      const int y0 = oy * p.stride - p.pad, x0 = ox * p.stride - p.pad;
      const float* img = pl + (size_t)bl * kCtCh * plane;
      // the patch's 9 plane offsets and padding mask are the same for every channel
      int poff[V];
      uint32_t pmask = 0u;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int iy = y0 + j / 3, ix = x0 + j % 3;
        const bool in = (unsigned)iy < (unsigned)p.h && (unsigned)ix < (unsigned)p.w;
        poff[j] = in ? iy * p.w + ix : 0;
        pmask |= in ? (1u << j) : 0u;
      }
      uint64_t codes_lo = 0ull, codes_hi = 0ull;  // this pixel's 16 codes, byte c at 8 * c
      // 2-slot TMEM ring per group (A_hi 16 | A_lo 16 | D 16 columns): the screen of
      // channel c - 1 runs while channel c's MMAs execute.
      float ap[V], asq_prev = 0.0f;
#pragma unroll 1
      for (int cl = 0; cl <= nch; ++cl) {
        float a[V], asq = 0.0f;
        const int bsel = cl & 1;
        if (cl < nch) {
          const float* pc = img + (size_t)cl * plane;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            const float v = ((pmask >> j) & 1u) ? pc[poff[j]] : 0.0f;
            a[j] = v;
            asq = fmaf(v, v, asq);
          }
          // 3xTF32: a = a_hi + a_lo with a_hi = tf32(a) (the MMA truncates its fp32 inputs)
          uint32_t ah[16], al2[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float v = j < V ? a[j] : (j == V ? 1.0f : 0.0f);  // column 9: the -|p_k|^2/2 term
            const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
            ah[j] = __float_as_uint(hi);
            al2[j] = __float_as_uint(v - hi);
          }
          const uint32_t sl = lane_base + (uint32_t)(bsel * 48);
          ct_st16(sl, ah);
          ct_st16(sl + 16, al2);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          named_barrier_sync(4 + grp, 128);
          if (q == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t bh = ct_desc(smem_u32(btiles + (2 * cl) * kCtBTile));      // p_hi
            const uint64_t bl = ct_desc(smem_u32(btiles + (2 * cl + 1) * kCtBTile));  // p_lo
            const uint32_t ta = tmem + (uint32_t)(grp * 128 + bsel * 48);            // lane 0: A_hi; +16 A_lo; +32 D
            asm volatile(
                "{\n\t.reg .pred e, f, t;\n\t.reg .b32 ah1, al0, al1, d;\n\t"
                "setp.ne.u32 f, %3, %3;\n\t"
                "setp.eq.u32 t, %3, %3;\n\t"
                "add.u32 ah1, %0, 8;\n\t"
                "add.u32 al0, %0, 16;\n\t"
                "add.u32 al1, %0, 24;\n\t"
                "add.u32 d, %0, 32;\n\t"
                "elect.sync _|e, 0xffffffff;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [%0], %1, %2, f;\n\t"   // a_hi.p_hi, K 0..7
                "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [%0], %4, %2, t;\n\t"   // a_hi.p_lo
                "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al0], %1, %2, t;\n\t"  // a_lo.p_hi
                "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah1], %5, %2, t;\n\t"  // K 8..15
                "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [ah1], %6, %2, t;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::tf32 [d], [al1], %5, %2, t;\n\t"
                "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t}" ::"r"(ta),
                "l"(bh), "r"(kCtIdesc), "r"(0u), "l"(bl), "l"(bh + 2), "l"(bl + 2),
                "r"(smem_u32(&dfull[grp * 2 + bsel]))
                : "memory");
          }
        }
        if (cl > 0) {
          const int pc = cl - 1, ps = pc & 1;
          mbar_wait(&dfull[grp * 2 + ps], (dphase >> ps) & 1u);
          dphase ^= 1u << ps;
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          uint32_t dv[16];
          ct_ld16(lane_base + (uint32_t)(ps * 48 + 32), dv);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          const int code = conv_screen(dv, ap, asq_prev, aux + pc * 32, cent + pc * K * V, tau_c, p.near_tie, live);
          if (pc < 8)
            codes_lo |= (uint64_t)code << (8 * pc);
          else
            codes_hi |= (uint64_t)code << (8 * (pc - 8));
        }
        if (cl < nch) {
#pragma unroll
          for (int j = 0; j < V; ++j) ap[j] = a[j];
          asq_prev = asq;
        }
      }
      // the unit's codes: 16 bytes per pixel at the group's channel offset
      if (live) {
        uint8_t* dst = p.codes + row * p.code_stride + (int64_t)g * kCtCh;
        if (nch == kCtCh && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
          *reinterpret_cast<uint4*>(dst) = make_uint4((uint32_t)codes_lo, (uint32_t)(codes_lo >> 32),
                                                      (uint32_t)codes_hi, (uint32_t)(codes_hi >> 32));
        } else {
          for (int i = 0; i < nch; ++i) dst[i] = (uint8_t)((i < 8 ? codes_lo >> (8 * i) : codes_hi >> (8 * (i - 8))) & 255u);
        }
      }
      // this thread is done with slot s: the producer may refill it (2 units later)
      asm volatile("bar.arrive %0, %1;" ::"r"(1 + s), "r"(kCtThreads) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4 * kCtGroups) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

// Returns LUT_OK with *used = false when the shape is not this kernel's (the
// caller falls back to the FFMA plane kernel).
int launch_conv_tc(const float* x, int batch, int cin, int h, int w, int stride, int pad, int ho, int wo,
                   const float* prep, int K, uint8_t* codes, int64_t code_stride, int* near_tie, cudaStream_t stream,
                   bool* used) {
  *used = false;
  if (K != 16) return LUT_OK;
  const int64_t hw_out = (int64_t)ho * wo;
  // a 512-pixel unit spans whole images or lies inside one
  if (!(hw_out % kCtRows == 0 || kCtRows % hw_out == 0)) return LUT_OK;
  if (((int64_t)h * w * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(x) & 15)) return LUT_OK;
  ConvTcParams p;
  p.x = x;
  p.prep = prep;
  p.S = prep_stride(16, 9);
  p.batch = batch;
  p.cin = cin;
  p.h = h;
  p.w = w;
  p.stride = stride;
  p.pad = pad;
  p.ho = ho;
  p.wo = wo;
  p.nrows = (int64_t)batch * hw_out;
  p.nchunks = (p.nrows + kCtRows - 1) / kCtRows;
  p.ngroups = (cin + kCtCh - 1) / kCtCh;
  p.nunits = p.nchunks * p.ngroups;
  p.imgs = hw_out >= kCtRows ? 1 : (int)(kCtRows / hw_out);
  p.slot_bytes = (uint32_t)((p.imgs * kCtCh * h * w * 4 + 127) & ~127);
  p.codes = codes;
  p.code_stride = code_stride;
  p.near_tie = near_tie;
  const size_t smem = 1024 + 2 * kCtCh * kCtBTile + kCtCh * 32 * 4 + kCtCh * 16 * 9 * 4 + 128 + 2 * (size_t)p.slot_bytes +
                      kCtRows * 16 + (2 + 2 * kCtGroups) * 8 + 16;
  if (smem > max_smem_optin()) return LUT_OK;
  cudaError_t e = kernel_smem_attr(reinterpret_cast<const void*>(encode_conv_tc_kernel));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(encode_conv_tc)");
  const int nsm = num_sms();
  const int grid = (int)(p.nunits < nsm ? p.nunits : nsm);
  encode_conv_tc_kernel<<<grid, kCtThreads, smem, stream>>>(p);
  LUT_CHECK_LAUNCH("encode_conv_tc_kernel");
  *used = true;
  return LUT_OK;
}

}  // namespace lutgpu
