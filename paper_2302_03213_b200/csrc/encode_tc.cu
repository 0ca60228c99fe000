// Nearest-centroid encode with tensor-core candidate screening (sm_100a),
// for sub-vectors of V = 32 floats and K = 16 or 64 centroids (configs[1,3,4]).
//
// Semantics are those of encode.cu (indices identical to the reference's
// encode_hard, lutkit/pq.py:171-174: literal f64 squared distances, ties ->
// lowest k).  The arithmetic is split in two exact-by-construction steps:
//
//  1. Screen.  One tcgen05.mma.kind::tf32 (M = 128 rows, N = 16 centroids,
//     K = 32 in four K = 8 steps) per (128-row tile, codebook) computes every
//     a.p_k with operands truncated to tf32 (10-bit mantissa; the probe in
//     tools/tf32_probe.cu confirms truncation and an fp32 accumulation error
//     <= 3 * 2^-23 * sum|a_j p_j|).  The screened distance
//     d~_k = |p_k|^2 - 2 a.p~_k then satisfies |d~_k - d_k| <= D with
//        D = 2^-7 |a| max_k|p_k| + 2^-21 (|a|^2 + max_k |p_k|^2)
//     (truncation of a and p: 2 * 2^-10 sum|a_j p_j|; products of the
//     truncation errors 2^-20; accumulation 2^-17; the factor 2 of -2 a.p; the
//     fp32 roundings of d~; |a| rounded up) — a 2x margin over the bound.
//     Every k with d~_k > min_j d~_j + 2D is provably not the argmin, so the
//     exact argmin is among the candidates; a lone candidate is it.
//  2. Refine (only rows with >= 2 candidates).  The candidates' distances are
//     re-evaluated in fp32 exactly as in encode.cu (packed FFMA over raw a,
//     d = fma(-2, a.p, |p|^2)); if the best two are within TAU the row is
//     re-decided from literal f64 differences over all K (encode_hard), and
//     counted as a near tie.
//
// Kernel anatomy (one persistent CTA per SM, 2 + 4*GR warps, GR = 3 (K = 16) or 4 (K = 64); NK = K):
//   warp 0     producer: per stage (one codebook of one 128-row tile) a TMA
//              box of A (32 columns x 128 rows, 128B swizzle, 16 KB) plus the
//              codebook's pre-swizzled tf32 B tile (2 KB) and norms by bulk copy.
//   warp 1     TMEM allocator + MMA issuer: 4 kind::tf32 MMAs per stage into
//              a 16-column TMEM slot, tcgen05.commit -> the stage's D barrier.
//   warps 2..  GR groups of 4 (thread = row = TMEM lane) taking every GR-th ring
//              stages: tcgen05.ld the 16 dots, screen, refine; a unit's 16 codes
//              per row meet in SMEM and leave as one 16-byte vector per row.
// The ring of kTcStages stages bounds both the SMEM (A, B) and the TMEM slots.

#include <float.h>

#include "common.cuh"

namespace lutgpu {

// Stage: A tile (16 KB) | B tile (NK x 128 B) | aux 1 KB: [NK |p|^2][pmax][pad] at 0,
// 2^-7 max|p| at byte 512.  GR consumer groups of 4 warps; the ring depth is a
// multiple of GR so that every slot is always consumed by the same group, and
// stages x NK TMEM columns fit the 512.
template <int NK> constexpr int tc_stage_bytes() { return 16384 + NK * 128 + 1024; }
template <int GR, int NK> struct TcGeom;
template <> struct TcGeom<2, 16> { static constexpr int stages = 10; };
template <> struct TcGeom<3, 16> { static constexpr int stages = 9; };
template <> struct TcGeom<4, 16> { static constexpr int stages = 8; };
template <> struct TcGeom<2, 64> { static constexpr int stages = 8; };
template <> struct TcGeom<3, 64> { static constexpr int stages = 6; };
template <> struct TcGeom<4, 64> { static constexpr int stages = 8; };
constexpr int kTcG = 16;                            // codebooks per unit (16 B of codes per row)

struct EncTcParams {
  const float* prep;  // prepared records (prep_stride floats each), TC section present
  int S;              // record stride (floats)
  int64_t n;
  int C;
  int ngroups;
  int64_t ntiles, nunits;
  uint8_t* codes;
  int64_t code_stride;
  int* near_tie;
};

__device__ __forceinline__ uint64_t tc_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;             // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO: 8-row atoms 1 KB apart
  d |= (uint64_t)1 << 46;             // sm100 descriptor version
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}

// kind::tf32, D f32, A/B tf32 (K-major), M = 128, N = NK
template <int NK>
constexpr uint32_t tc_idesc() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NK >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ uint64_t f2pk(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2up(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int NK> struct TcMask { using T = uint32_t; };
template <> struct TcMask<64> { using T = uint64_t; };
__device__ __forceinline__ int ffs_mask(uint32_t m) { return __ffs((int)m); }
__device__ __forceinline__ int ffs_mask(uint64_t m) { return __ffsll((long long)m); }

__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}

template <int GR, int NK>
__global__ void __launch_bounds__((2 + 4 * GR) * 32, 1)
    encode_tc_kernel(const __grid_constant__ CUtensorMap tmap, const EncTcParams p) {
  grid_launch_dependents();  // a programmatic dependent (the gather) may start staging
  constexpr int kTcStages = TcGeom<GR, NK>::stages;
  constexpr int kTcStageBytes = tc_stage_bytes<NK>();
  constexpr int kAux = 16384 + NK * 128;             // aux offset inside a stage
  constexpr uint32_t kTmemCols = NK == 16 ? 256 : 512;
  static_assert(kTcStages * NK <= (int)kTmemCols, "TMEM slots");
  using MaskT = typename TcMask<NK>::T;  // candidate set: one bit per centroid
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTcStages * kTcStageBytes);
  uint64_t* dfull = full + kTcStages;
  uint64_t* empty = dfull + kTcStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(empty + kTcStages);
  uint8_t* cbuf = smem + ((kTcStages * kTcStageBytes + 3 * kTcStages * 8 + 16 + 127) & ~127);  // [2][128 rows][16 codes]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&dfull[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      prefetch_tmap(&tmap);
      const uint64_t pol_a = l2_policy_evict_first();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = blockIdx.x; u < p.nunits; u += gridDim.x) {
        const int64_t tile = u / p.ngroups;
        const int c0 = (int)(u % p.ngroups) * kTcG;
        const int c1 = min(p.C, c0 + kTcG);
        for (int c = c0; c < c1; ++c) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * kTcStageBytes;
          const float* rec = p.prep + (size_t)c * p.S;
          mbar_arrive_expect_tx(&full[stage], 16384 + NK * 128 + (NK + 4) * 4 + 64);
          tma_load_2d_hint(st, &tmap, c * 32, (int32_t)(tile * 128), &full[stage], pol_a);  // A is read once
          bulk_load(st + 16384, rec + prep_base(NK, 32), NK * 128, &full[stage]);   // swizzled tf32 B tile
          bulk_load(st + kAux, rec + NK * 32, (NK + 4) * 4, &full[stage]);           // |p_k|^2, pmax, pad
          bulk_load(st + kAux + 512, rec + prep_base(NK, 32) + NK * 32, 64, &full[stage]);  // 2^-7 max|p_k| (up)
          if (++stage == kTcStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t u = blockIdx.x; u < p.nunits; u += gridDim.x) {
      const int c0 = (int)(u % p.ngroups) * kTcG;
      const int c1 = min(p.C, c0 + kTcG);
      for (int c = c0; c < c1; ++c) {
        mbar_wait(&full[stage], phase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sa = smem_u32(smem + stage * kTcStageBytes);
        const uint64_t adesc = tc_sw128_desc(sa);
        const uint64_t bdesc = tc_sw128_desc(sa + 16384);
        const uint32_t d = tmem + (uint32_t)(stage * NK);
        asm volatile(
            "{\n\t.reg .pred e, f, t;\n\t"
            "setp.ne.u32 f, %11, %11;\n\t"
            "setp.eq.u32 t, %11, %11;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, f;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %4, %5, %3, t;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %6, %7, %3, t;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %8, %9, %3, t;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%10];\n\t}" ::"r"(d),
            "l"(adesc), "l"(bdesc), "r"(tc_idesc<NK>()), "l"(adesc + 2), "l"(bdesc + 2), "l"(adesc + 4), "l"(bdesc + 4),
            "l"(adesc + 6), "l"(bdesc + 6), "r"(smem_u32(&dfull[stage])), "r"(0u)
            : "memory");
        if (++stage == kTcStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ screen + refine (two groups)
    // Group g takes the CTA's ring stages with index parity g: with an even ring
    // depth every slot is always consumed by the same group, so each group sees
    // all phases of its barriers in order.  Codes meet in a per-unit SMEM buffer.
    const int grp = (warp - 2) >> 2;
    const int q = warp & 3;  // TMEM lane quarter
    const int r = q * 32 + lane;
    const int sw = r & 7;
    const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
    const float tau_c = (4.0f * 32 + 16.0f) * 5.9604645e-8f;  // encode.cu TAU for V = 32
    // this group's ring slots are grp, grp + GR, ... (GR divides the ring depth), visited in order
    int stage = grp;
    uint32_t phase = 0;
    int umod = 0;  // (CTA ring stage index of the current unit's first stage) mod GR
    int ub = 0;    // code buffer of the current unit
    int lu = 0;    // this CTA's unit counter
    for (int64_t u = blockIdx.x; u < p.nunits; u += gridDim.x, ++lu) {
      const int c0 = (int)(u % p.ngroups) * kTcG;
      const int c1 = min(p.C, c0 + kTcG);
      const int nst = c1 - c0;
      const int64_t tile = u / p.ngroups;
      const int64_t row = tile * 128 + r;
      const int cc0 = (grp - umod + GR) % GR;
      umod = (umod + nst) % GR;
      for (int cc = cc0; cc < nst; cc += GR) {
        const int cur = stage;
        const uint32_t cph = phase;
        stage += GR;
        if (stage >= kTcStages) {
          stage -= kTcStages;
          phase ^= 1;
        }
        mbar_wait(&dfull[cur], cph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint8_t* st = smem + cur * kTcStageBytes;
        const uint32_t dslot = lane_addr + (uint32_t)(cur * NK);
        uint32_t dv[16];
        tc_ld16(dslot, dv);
        // this row's sub-vector (fp32, from the swizzled A tile) and |a|^2
        const uint32_t arow = smem_u32(st) + (uint32_t)(r * 128);
        float a[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(a[4 * j]), "=f"(a[4 * j + 1]), "=f"(a[4 * j + 2]), "=f"(a[4 * j + 3])
                       : "r"(arow + (uint32_t)((j ^ sw) << 4)));
        }
        uint64_t a2[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) a2[j] = f2pk(a[2 * j], a[2 * j + 1]);
        uint64_t sq = 0ull;
#pragma unroll
        for (int j = 0; j < 16; ++j) sq = f2fma(a2[j], a2[j], sq);
        float sq_lo, sq_hi;
        f2up(sq, sq_lo, sq_hi);
        const float asq = sq_lo + sq_hi;
        const float* aux = reinterpret_cast<const float*>(st + kAux);  // [NK |p|^2][pmax][pad] .. @512: 2^-7 max|p|
        const float* pn = aux;
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // screening half-width, one per row: D = 2^-7 |a| max_k|p_k| + 2^-21 (|a|^2 + max_k |p_k|^2)
        // (|a| and max|p| rounded up); candidates: d~_k <= min_j d~_j + 2D (rounded up)
        const float al = __fmul_ru(__fsqrt_ru(asq), 1.0000002f);
        const float hw = fmaf(al, aux[128], 4.7683716e-7f * (asq + aux[NK]));
        float dt[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) dt[k] = fmaf(-2.0f, __uint_as_float(dv[k]), pn[k]);
        float mn = fminf(fminf(dt[0], dt[1]), fminf(dt[2], dt[3]));
#pragma unroll
        for (int k = 4; k < 16; k += 4) mn = fminf(mn, fminf(fminf(dt[k], dt[k + 1]), fminf(dt[k + 2], dt[k + 3])));
#pragma unroll
        for (int kc = 16; kc < NK; kc += 16) {  // K = 64: the other 16-column chunks (minimum pass)
          uint32_t dw[16];
          tc_ld16(dslot + (uint32_t)kc, dw);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int k = 0; k < 16; k += 4) {
            const float e0 = fmaf(-2.0f, __uint_as_float(dw[k]), pn[kc + k]);
            const float e1 = fmaf(-2.0f, __uint_as_float(dw[k + 1]), pn[kc + k + 1]);
            const float e2 = fmaf(-2.0f, __uint_as_float(dw[k + 2]), pn[kc + k + 2]);
            const float e3 = fmaf(-2.0f, __uint_as_float(dw[k + 3]), pn[kc + k + 3]);
            mn = fminf(mn, fminf(fminf(e0, e1), fminf(e2, e3)));
          }
        }
        const float thr = __fadd_ru(mn, 2.0f * hw);
        // candidate bits per 16-column chunk in 32-bit registers (constant shifts:
        // the chunk loops are unrolled), merged into the K-bit mask once per chunk
        uint32_t m16 = 0u;
#pragma unroll
        for (int k = 0; k < 16; ++k) m16 |= (dt[k] <= thr) ? (1u << k) : 0u;
        MaskT mask = (MaskT)m16;
#pragma unroll
        for (int kc = 16; kc < NK; kc += 16) {  // K = 64: candidate pass (same fp32 expression)
          uint32_t dw[16];
          tc_ld16(dslot + (uint32_t)kc, dw);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          uint32_t mc = 0u;
#pragma unroll
          for (int k = 0; k < 16; ++k) mc |= (fmaf(-2.0f, __uint_as_float(dw[k]), pn[kc + k]) <= thr) ? (1u << k) : 0u;
          mask |= (MaskT)mc << kc;
        }
        int code;
        if ((mask & (mask - 1)) == 0 && mask != 0) {
          code = ffs_mask(mask) - 1;
        } else {
          // refine the candidates in fp32 (encode.cu formulation) from the swizzled B tile
          const uint32_t btile = smem_u32(st + 16384);
          float best = FLT_MAX, second = FLT_MAX;
          int bi = 0;
          MaskT m = mask;
          while (m) {
            const int k = ffs_mask(m) - 1;
            m &= m - 1;
            uint64_t acc = 0ull;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              uint64_t c01, c23;
              asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];"
                           : "=l"(c01), "=l"(c23)
                           : "r"(btile + (uint32_t)(k * 128 + ((j ^ (k & 7)) << 4))));
              acc = f2fma(a2[2 * j], c01, acc);
              acc = f2fma(a2[2 * j + 1], c23, acc);
            }
            float lo, hi;
            f2up(acc, lo, hi);
            const float dk = fmaf(-2.0f, lo + hi, pn[k]);
            second = fminf(second, fmaxf(best, dk));
            bi = (dk < best) ? k : bi;
            best = fminf(best, dk);
          }
          code = bi;
          if (!(second - best > tau_c * (asq + aux[NK]))) {
            // near tie (or NaN): literal f64 decision over all K (encode_hard)
            // over the candidates (every other k is provably farther), ascending k
            double bd = 0.0;
            int bk = -1;
            MaskT mm = mask ? mask : (MaskT)(NK == 64 ? ~0ull : 0xFFFFull);  // NaN rows: all K, as encode_hard
            while (mm) {
              const int k = ffs_mask(mm) - 1;
              mm &= mm - 1;
              const float* crow = reinterpret_cast<const float*>(st + 16384 + k * 128);
              double s = 0.0;
              for (int j = 0; j < 32; ++j) {
                const double diff = (double)a[j] - (double)crow[(((j >> 2) ^ (k & 7)) << 2) + (j & 3)];
                s = __dadd_rn(s, __dmul_rn(diff, diff));
              }
              if (bk < 0 || s < bd) {
                bd = s;
                bk = k;
              }
            }
            code = bk;
            if (p.near_tie && row < p.n) atomicAdd(p.near_tie, 1);
          }
        }
        // all reads of this stage (TMEM slot, A and B tiles) are done: release it
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[cur]);
        cbuf[(ub * 128 + r) * 16 + cc] = (uint8_t)code;
      }
      // all groups' codes of this unit are in cbuf[ub]: one group writes them out
      named_barrier_sync(1, 128 * GR);
      if (grp == lu % GR && row < p.n) {
        const uint8_t* src = cbuf + (ub * 128 + r) * 16;
        uint8_t* dst = p.codes + row * p.code_stride + c0;
        if (nst == 16 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
          *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
        } else {
          for (int i = 0; i < nst; ++i) dst[i] = src[i];
        }
      }
      ub ^= 1;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
}

// Returns LUT_OK with *used = false when the shape is not this kernel's.
int encode_dense_tc(const float* a, int64_t n, int d, const float* prep, int C, int K, int V, uint8_t* codes,
                    int code_bits, int64_t code_stride, int* near_tie, cudaStream_t stream, bool* used) {
  *used = false;
  if (V != 32 || (K != 16 && K != 64) || code_bits != 8 || n < 128 || !prep_has_tc(K, V)) return LUT_OK;
  if ((reinterpret_cast<uintptr_t>(a) & 15) || (reinterpret_cast<uintptr_t>(prep) & 15) || (d % 4)) return LUT_OK;
  CUtensorMap tmap;
  if (!make_tmap_2d_f32(&tmap, a, (uint64_t)d, (uint64_t)n, 32, 128, true)) return LUT_OK;
  EncTcParams p;
  p.prep = prep;
  p.S = prep_stride(K, V);
  p.n = n;
  p.C = C;
  p.ngroups = (C + kTcG - 1) / kTcG;
  p.ntiles = (n + 127) / 128;
  p.nunits = p.ntiles * p.ngroups;
  p.codes = codes;
  p.code_stride = code_stride;
  p.near_tie = near_tie;
  const int nsm = num_sms();
  const int grid = (int)(p.nunits < nsm ? p.nunits : nsm);
  int gr = K == 16 ? 3 : 4;  // consumer groups (LUTGPU_ENC_TC_GROUPS = 2, 3 or 4)
  if (const char* g = probe_env("LUTGPU_ENC_TC_GROUPS")) gr = atoi(g) == 2 ? 2 : atoi(g) == 3 ? 3 : 4;
  int stages;
  void (*kern)(const CUtensorMap, const EncTcParams);
  if (K == 16) {
    stages = gr == 2 ? TcGeom<2, 16>::stages : gr == 3 ? TcGeom<3, 16>::stages : TcGeom<4, 16>::stages;
    kern = gr == 2 ? encode_tc_kernel<2, 16> : gr == 3 ? encode_tc_kernel<3, 16> : encode_tc_kernel<4, 16>;
  } else {
    stages = gr == 2 ? TcGeom<2, 64>::stages : gr == 3 ? TcGeom<3, 64>::stages : TcGeom<4, 64>::stages;
    kern = gr == 2 ? encode_tc_kernel<2, 64> : gr == 3 ? encode_tc_kernel<3, 64> : encode_tc_kernel<4, 64>;
  }
  const size_t sb = K == 16 ? tc_stage_bytes<16>() : tc_stage_bytes<64>();
  const size_t smem = (((size_t)stages * sb + 3 * stages * sizeof(uint64_t) + 16 + 127) & ~size_t(127)) + 4096 + 1024;
  if (smem > max_smem_optin()) return LUT_OK;
  cudaError_t e = kernel_smem_attr(reinterpret_cast<const void*>(kern));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(encode_tc)");
  kern<<<grid, (2 + 4 * gr) * 32, smem, stream>>>(tmap, p);
  LUT_CHECK_LAUNCH("encode_tc_kernel");
  *used = true;
  return LUT_OK;
}

}  // namespace lutgpu
