// One-hot lookup-aggregate for tables whose B image does not fit in SMEM at
// 64 columns per SM (C*K > 2304 bytes per column, e.g. configs[4] K = 64:
// 8 KB per column).  The resident-B pair kernel (onehot.cu) would have to drop
// to 16 columns per SM (MMA N = 32, one-hot A regenerated every 32 output
// columns); here B is streamed instead and every MMA keeps N = 128.
//
//   acc[r, m] = sum_{c,k} [code[r,c] == k] * q[c, k, m]   (exact int32, the
//   same GEMM as onehot.cu; bitwise equal to lut_gather_i32, kernels.py:105-127)
//
// Geometry: a CTA pair (cluster of 2, tcgen05 cta_group::2, M = 256 rows per
// MMA) computes a unit of TWO 256-row tiles x 128 columns (64 per SM).  Per
// ring stage (2 K blocks = 256 bytes of logical K) the producer streams the
// stage's B slice (64 columns x 256 B = 16 KB per SM) from L2 by bulk copy,
// the generators write the 2:4-compressed one-hot of both row tiles into TMEM,
// and the MMA issuer applies the one B stage to both row tiles (2 x 4
// tcgen05.mma.sp) — each streamed B byte feeds 512 rows, so the B traffic is
// 64 cols x C*K bytes per 512 rows per SM (K = 64, C = 128: ~20 B/clk/SM).
// TMEM: two 128-column int32 accumulators (one per row tile, 256 columns) +
// a 3-slot A ring (80 columns per slot: per row tile 32 compressed A + 8
// metadata columns).  The accumulators are single-buffered: the next unit's
// MMAs wait until the epilogue has read them (4 tcgen05.ld passes, ~3% of a
// 256-MMA unit).
//
// Warp roles (19 warps, as the resident pair kernel):
//   0-7   generators: row tile = warp >> 2, TMEM lane quarter = warp & 3
//   8-15  epilogue: accumulator = (warp - 8) >> 2, lane quarter = warp & 3
//   16    producer: code boxes (per unit, double-buffered), B stages (6-deep ring)
//   17    TMEM allocator; leader: MMA issuer; peer: forwards its stage
//         readiness (A stored + B landed) to the leader
//   18    leader: watcher (a_full + b_full) handing stages to the issuer

#include "onehot_dev.cuh"

namespace lutgpu {

constexpr int kSNA = 3;             // A ring slots (TMEM)
constexpr int kSNB = 6;             // B ring slots (SMEM), a multiple of kSNA
constexpr int kSSlotCols = 80;      // TMEM columns per A slot (2 row tiles x (32 A + 8 metadata))
constexpr int kSBStage = 64 * 2 * kKB;  // B bytes per stage per SM: 64 columns x 2 K blocks
static_assert(kSNB % kSNA == 0, "stage barriers serve both rings");

template <int K, int FAST>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
    onehot_stream_kernel(const __grid_constant__ CUtensorMap codes_map, const __grid_constant__ CUtensorMap out_map,
                         const __grid_constant__ OneHotParams p) {
  static_assert(K >= 8, "stream kernel: K >= 8");
  static_assert(FAST == 0 || FAST == 4 || FAST == 6,
                "stream kernel epilogues: 4 (plain int8), 6 (bias, act, m-tile scales; TMA stores), 0 (generic)");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int code_box_bytes = kRowsPerTile * 128;                  // 128 rows x 128 codes
  const int code_unit_bytes = 2 * p.code_boxes * code_box_bytes;  // both row tiles
  uint8_t* b_ring = smem;                                         // kSNB x 16 KB
  uint8_t* code_smem = b_ring + kSNB * kSBStage;                  // 2 units
  uint8_t* stage_out = code_smem + 2 * code_unit_bytes;           // [acc 2][buf 2] x 16 KB
  constexpr int kBox = kRowsPerTile * 32 * 4;                     // 128 rows x 32 f32
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage_out + 4 * kBox);
  uint64_t* code_full = bars + 0;             // [2]
  uint64_t* code_empty = bars + 2;            // [2] 8 generator warps
  uint64_t* b_full = bars + 4;                // [kSNB] local, tx
  uint64_t* stage_done = bars + 4 + kSNB;     // [kSNB] multicast commit: A slot + B slot free
  uint64_t* a_full = bars + 4 + 2 * kSNB;     // [kSNA] leader: 8 + 1 peer forward; peer: 8
  uint64_t* acc_full = bars + 4 + 2 * kSNB + kSNA;   // multicast commit
  uint64_t* acc_empty = acc_full + 1;                // leader: 8 epilogue warps + 1 peer
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(acc_empty + 1);
  const int nst = (p.nkb + 1) >> 1;  // ring stages per unit

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&code_full[i], 1);
      mbar_init(&code_empty[i], kGenWarps);
    }
    for (int i = 0; i < kSNB; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&stage_done[i], 1);
    }
    for (int i = 0; i < kSNA; ++i) mbar_init(&a_full[i], leader ? kGenWarps + 1 : kGenWarps);
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, kGenWarps + 1);
    fence_mbar_init();
  }
  if (warp == kPMma) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_smem)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;
  if (tmem_base != 0) __trap();
  constexpr uint32_t kACol0 = 256;  // accumulators [0, 256), A ring after

  UnitWalk walk;
  walk.init(p, (int)(blockIdx.x >> 1), (int)(gridDim.x >> 1));
  const uint32_t a_full_l = map_to_rank(smem_u32(a_full), 0);
  const uint32_t acc_empty_l = map_to_rank(smem_u32(acc_empty), 0);

  if (warp == kPProd) {
    // ------------------------------------------------ producer (both CTAs)
    if (lane == 0) {
      prefetch_tmap(&codes_map);
      const uint64_t pol_codes = l2_policy_evict_last();  // re-read once per n-tile of the band
      uint32_t g = 0;  // global stage counter
      int unit = 0;
      int ntile;
      int64_t rt;
      while (walk.next(ntile, rt)) {
        const int cs = unit & 1;
        mbar_wait(&code_empty[cs], ((unit >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&code_full[cs], (uint32_t)code_unit_bytes);
        for (int j = 0; j < 2; ++j)
          for (int bx = 0; bx < p.code_boxes; ++bx)
            tma_load_2d_hint(code_smem + cs * code_unit_bytes + (j * p.code_boxes + bx) * code_box_bytes, &codes_map,
                             bx * 128, (int32_t)(rt * 4 * kRowsPerTile + j * 2 * kRowsPerTile + rank * kRowsPerTile),
                             &code_full[cs], pol_codes);
        const uint8_t* src = p.b_image + ((size_t)(2 * ntile + (int)rank) * p.nkb) * (64 * kKB);
        for (int st = 0; st < nst; ++st, ++g) {
          const uint32_t bs = g % kSNB;
          if (g >= (uint32_t)kSNB) mbar_wait(&stage_done[bs], ((g / kSNB) & 1) ^ 1);
          const int kb0 = 2 * st;
          const uint32_t bytes = (uint32_t)((kb0 + 1 < p.nkb ? 2 : 1) * 64 * kKB);
          mbar_arrive_expect_tx(&b_full[bs], bytes);
          bulk_load(b_ring + bs * kSBStage, src + (size_t)kb0 * 64 * kKB, bytes, &b_full[bs]);
        }
        ++unit;
      }
    }
  } else if (warp == kPWatch) {
    // ------------------------------------------------ watcher (leader)
    if (leader) {
      uint32_t g = 0;
      int unit = 0;
      int ntile;
      int64_t rt;
      while (walk.next(ntile, rt)) {
        if (unit > 0) mbar_wait_rlx(acc_empty, (unit - 1) & 1, 1);
        for (int st = 0; st < nst; ++st, ++g) {
          mbar_wait_rlx(&a_full[g % kSNA], (g / kSNA) & 1, 1);
          while (!mbar_try_wait(&b_full[g % kSNB], (g / kSNB) & 1)) {  // acquire: TMA-written B
          }
          named_barrier_sync(9, 64);
        }
        ++unit;
      }
    }
  } else if (warp == kPMma && !leader) {
    // ------------------------------------------------ peer: forward stage readiness
    uint32_t g = 0;
    int ntile;
    int64_t rt;
    while (walk.next(ntile, rt)) {
      for (int st = 0; st < nst; ++st, ++g) {
        mbar_wait_rlx(&a_full[g % kSNA], (g / kSNA) & 1, 1);
        mbar_wait_rlx(&b_full[g % kSNB], (g / kSNB) & 1, 1);
        tc_fence_after();
        tc_fence_before();
        if (lane == 0) mbar_arrive_cluster_rlx(a_full_l + (g % kSNA) * 8);
        __syncwarp();
      }
    }
  } else if (warp == kPMma) {
    // ------------------------------------------------ MMA issuer (leader)
    const uint32_t idesc = idesc_i8(256, 128) | 4u;  // sparse A
    const uint64_t bstep = (uint64_t)((64 * kKB) >> 4);
    const int nkb = p.nkb;
    uint32_t g = 0;
    int ntile;
    int64_t rt;
    while (walk.next(ntile, rt)) {
      for (int st = 0; st < nst; ++st, ++g) {
        named_barrier_sync(9, 64);  // A slot stored in both CTAs, B stage landed in both
        tc_fence_after();
        const uint64_t bd = sw128_desc(b_ring + (g % kSNB) * kSBStage);
        const uint32_t ab = kACol0 + (g % kSNA) * kSSlotCols;
        const uint32_t two = 2 * st + 1 < nkb;
        issue_stage_sp<2>(0u, ab, bd, bstep, idesc, st != 0, two, ab + 32);          // row tile 0
        issue_stage_sp<2>(128u, ab + 40, bd, bstep, idesc, st != 0, two, ab + 72);   // row tile 1
        commit_elect(&stage_done[g % kSNB], true);
      }
      commit_elect(acc_full, true);
    }
  } else if (warp < kGenWarps) {
    // ------------------------------------------------ generators (both CTAs)
    const int sub = warp & 3, j = warp >> 2;
    const int row_in_tile = sub * 32 + lane;
    const int sw = row_in_tile & 7;
    const uint32_t lane_base = tmem_base + ((uint32_t)(sub * 32) << 16) + kACol0 + (uint32_t)(j * 40);
    uint32_t g = 0;
    int unit = 0;
    int ntile;
    int64_t rt;
    while (walk.next(ntile, rt)) {
      const int cs = unit & 1;
      mbar_wait(&code_full[cs], (unit >> 1) & 1);
      const uint32_t row_saddr =
          smem_u32(code_smem + cs * code_unit_bytes + j * p.code_boxes * code_box_bytes) + row_in_tile * 128;
      for (int st = 0; st < nst; ++st, ++g) {
        StageCodes<K, 2> cd;
        cd.load(row_saddr, sw, st);
        uint32_t w[32], we[8];
        build_sparse<K, 2>(cd, w, we);
        if (g >= (uint32_t)kSNA) mbar_wait_rlx(&stage_done[(g - kSNA) % kSNB], ((g - kSNA) / kSNB) & 1, 0);
        tc_fence_after();
        const uint32_t slot = lane_base + (g % kSNA) * kSSlotCols;
        tmem_st32(slot, w);
        tmem_st8(slot + 32, we);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[g % kSNA]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&code_empty[cs]);
      ++unit;
    }
  } else if (warp >= kPEpi0 && warp < kPEpi0 + 8) {
    // ------------------------------------------------ epilogue (both CTAs)
    const int sub = warp & 3, a = (warp - kPEpi0) >> 2;
    const int row_in_tile = sub * 32 + lane;
    const int swz = row_in_tile & 7;
    const bool grp_leader = sub == 0 && lane == 0;  // issues this accumulator's TMA stores
    const float scale0 = (p.scales && p.out) ? __ldg(p.scales) : 1.0f;
    const uint64_t scale2 = pk_f2(scale0, scale0);
    int unit = 0;
    int ntile;
    int64_t rt;
    while (walk.next(ntile, rt)) {
      mbar_wait(acc_full, unit & 1);
      tc_fence_after();
      const int64_t row0 = rt * 4 * kRowsPerTile + a * 2 * kRowsPerTile + rank * kRowsPerTile;
      const int m_base = ntile * 128;
      for (int ps = 0; ps < 4; ++ps) {
        uint32_t v[32];
        tmem_ld32(tmem_base + ((uint32_t)(sub * 32) << 16) + (uint32_t)(a * 128 + ps * 32), v);
        tmem_ld_wait();
        if (ps == 3) {  // both accumulators read by this CTA's 8 warps: release them
          tc_fence_before();
          if (leader) {
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty);
          } else {
            named_barrier_sync(4, 256);
            if (warp == kPEpi0 && lane == 0) mbar_arrive_cluster_rlx(acc_empty_l);
          }
        }
        if constexpr (FAST == 0) {
          // generic: direct stores (any M, int32 and / or NCHW output, per-m-tile scales)
          const int64_t row = row0 + row_in_tile;
          if (row < p.n) {
            const int mp = m_base + ps * 32;
            int64_t base = row * p.M, cstr = 1;
            if (p.out_hw > 0) {
              const int64_t b = row / p.out_hw;
              base = b * p.M * p.out_hw + (row - b * p.out_hw);
              cstr = p.out_hw;
            }
#pragma unroll 4
            for (int q = 0; q < 32; ++q) {
              const int m = mp + q;
              if (m >= p.M) break;
              const int64_t o = base + (int64_t)m * cstr;
              if (p.out_i32) p.out_i32[o] = (int)v[q];
              if (p.out) {
                const float s = p.scale_mtile > 0 ? __ldg(p.scales + m / p.scale_mtile) : scale0;
                float f = __fmul_rn(__int2float_rn((int)v[q]), s);
                if (p.bias) f = __fadd_rn(f, __ldg(p.bias + m));
                p.out[o] = apply_act(f, p.act);
              }
            }
          }
          continue;
        }
        // staging box (a, ps & 1): the store issued from it two passes ago has been read
        uint8_t* box = stage_out + (a * 2 + (ps & 1)) * kBox;
        if (sub == 0) {
          if (lane == 0) bulk_wait_read1();
          __syncwarp();
          asm volatile("bar.arrive %0, 128;" ::"r"(5 + 2 * a) : "memory");
        } else {
          named_barrier_sync(5 + 2 * a, 128);
        }
        const uint32_t dst = smem_u32(box) + row_in_tile * 128;
        const int mp = m_base + ps * 32;  // first column of this pass
        uint64_t sc2 = scale2;
        if constexpr (FAST == 6) {
          if (p.scale_mtile > 0) {
            const float s = mp < p.M ? __ldg(p.scales + mp / p.scale_mtile) : 1.0f;
            sc2 = pk_f2(s, s);
          }
#pragma unroll
          for (int hb = 0; hb < 32; hb += 16) {
            float f[16];
#pragma unroll
            for (int q = 0; q < 16; q += 2) {
              const uint64_t b = pk_f2(__int_as_float(0x4B400000 + (int)v[hb + q]),
                                       __int_as_float(0x4B400000 + (int)v[hb + q + 1]));
              up_f2(mul_f2(add_f2(b, kNegMagic2), sc2), f[q], f[q + 1]);
            }
            if (p.bias) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int m = mp + hb + 4 * q;
                if (m < p.M) {
                  const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + m));
                  f[4 * q] = __fadd_rn(f[4 * q], b4.x);
                  f[4 * q + 1] = __fadd_rn(f[4 * q + 1], b4.y);
                  f[4 * q + 2] = __fadd_rn(f[4 * q + 2], b4.z);
                  f[4 * q + 3] = __fadd_rn(f[4 * q + 3], b4.w);
                }
              }
            }
            if (p.act == LUT_ACT_GELU) {
#pragma unroll
              for (int q = 0; q < 16; ++q) f[q] = gelu_erf(f[q]);
            } else if (p.act) {
#pragma unroll
              for (int q = 0; q < 16; ++q) f[q] = apply_act(f[q], p.act);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
              sts_v4(dst + (uint32_t)(((hb / 4 + q) ^ swz) << 4), f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) {  // exact int -> f32 (|x| < 2^22), times the table scale
            float f0, f1, f2, f3;
            const uint64_t b01 = pk_f2(__int_as_float(0x4B400000 + (int)v[4 * q]),
                                       __int_as_float(0x4B400000 + (int)v[4 * q + 1]));
            const uint64_t b23 = pk_f2(__int_as_float(0x4B400000 + (int)v[4 * q + 2]),
                                       __int_as_float(0x4B400000 + (int)v[4 * q + 3]));
            up_f2(mul_f2(add_f2(b01, kNegMagic2), sc2), f0, f1);
            up_f2(mul_f2(add_f2(b23, kNegMagic2), sc2), f2, f3);
            sts_v4(dst + (uint32_t)((q ^ swz) << 4), f0, f1, f2, f3);
          }
        }
        fence_proxy_async_smem();
        if (sub != 0) {
          asm volatile("bar.arrive %0, 128;" ::"r"(6 + 2 * a) : "memory");
        } else {
          named_barrier_sync(6 + 2 * a, 128);
          if (grp_leader) {
            if (mp < p.M) tma_store_2d_hint(&out_map, box, mp, (int32_t)row0, l2_policy_evict_first());
            bulk_commit();
          }
        }
      }
      ++unit;
    }
    if (FAST != 0 && grp_leader) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == kPMma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
  }
}

size_t onehot_stream_smem(int code_boxes) {
  return (size_t)kSNB * kSBStage + 2 * (size_t)(2 * code_boxes * kRowsPerTile * 128) + 4 * (kRowsPerTile * 32 * 4) +
         (4 + 2 * kSNB + kSNA + 2) * 8 + 16 + 1024;
}

template <int K, int FAST>
static int launch_stream_k(const CUtensorMap& map, const CUtensorMap& omap, const OneHotParams& p, size_t smem,
                           int grid, cudaStream_t stream) {
  auto kern = onehot_stream_kernel<K, FAST>;
  cudaError_t e = kernel_smem_attr(reinterpret_cast<const void*>(kern));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(onehot_stream)");
  kern<<<grid, kPairThreads, smem, stream>>>(map, omap, p);
  LUT_CHECK_LAUNCH("onehot_stream_kernel");
  return LUT_OK;
}

// p: filled by onehot_gather (B image with NT = 64 per SM, pair tiles); here the
// unit geometry (512-row blocks) and the launch.
int onehot_stream_launch(const CUtensorMap& map, const CUtensorMap& omap, OneHotParams p, int fast,
                         cudaStream_t stream) {
  p.nrt = (p.n + 4 * kRowsPerTile - 1) / (4 * kRowsPerTile);  // 512-row blocks
  const int nsm = num_sms();
  const int64_t units = (int64_t)p.ntiles * p.nrt;
  const int pairs = (int)(units < nsm / 2 ? units : nsm / 2);
  // band of row blocks: every pair walks ~4 units of it, the band's codes stay in L2
  int64_t band = (4 * (int64_t)pairs + p.ntiles - 1) / p.ntiles;
  if (band < 1) band = 1;
  if (band > p.nrt) band = p.nrt;
  p.band_rt = band;
  const size_t smem = onehot_stream_smem(p.code_boxes);
  if (smem > max_smem_optin()) return fail(LUT_ERR_CONFIG, "one-hot stream gather: shared memory budget exceeded");
  const int grid = 2 * pairs;
  switch (p.K) {
#define LUT_STREAM_K(KK)                                                                                 \
  case KK:                                                                                               \
    return fast == 4   ? launch_stream_k<KK, 4>(map, omap, p, smem, grid, stream)                        \
           : fast == 6 ? launch_stream_k<KK, 6>(map, omap, p, smem, grid, stream)                        \
                       : launch_stream_k<KK, 0>(map, omap, p, smem, grid, stream);
    LUT_STREAM_K(16)
    LUT_STREAM_K(32)
    LUT_STREAM_K(64)
    LUT_STREAM_K(128)
#undef LUT_STREAM_K
    default:
      return fail(LUT_ERR_CONFIG, "one-hot stream gather: K must be 16, 32, 64 or 128");
  }
}

}  // namespace lutgpu
