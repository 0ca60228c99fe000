// Lookup-aggregate as a one-hot GEMM on the 5th-gen tensor cores (sm_100a).
//
// The paper writes the aggregation as onehot(idx) . T (Eq. 4):
//   acc[n, m] = sum_{c,k} [code[n,c] == k] * q[c, k, m]
// For int8 tables this is an exact int8 x int8 -> int32 GEMM with inner dim
// C*K, i.e. bit-exact against lut_gather_i32 (lutkit/kernels.py:105-127) —
// integer addition is associative, so the MMA's order does not matter.
//
// fp32 tables use DIGITS int8 planes: T[c,k,m] ~= s_m * t, t an integer with
// |t| <= 2^(8*DIGITS-2), written as balanced base-256 digits t = sum_i b_i 256^i.
// Each digit plane is one more group of B columns; the epilogue recombines
// the exact int32 digit sums in int64 and rounds once: out = f32(f64(sum) * s_m).
// Error vs the exact sum <= C * s_m / 2 (4 digits: C * max|T[:,:,m]| * 2^-31),
// far inside the fp32 contract (rtol/atol 1e-5, BASELINE north star); the
// bitwise ascending-c fp32 path remains in gather.cu.
//
// Kernel anatomy (one persistent CTA per SM, 12 warps):
//   warp 0      producer: bulk-copies the prepared B image of the current
//               n-tile (resident in SMEM, reloaded only when the n-tile
//               changes) and TMA-loads 128-row code tiles (128B swizzle).
//   warp 1      TMEM allocator + MMA issuer (one elected lane):
//               tcgen05.mma.cta_group::1.kind::i8, A from TMEM, B from SMEM.
//   warps 4-7   one-hot generators: thread = row = TMEM lane; builds the
//               row's one-hot bytes for a 128-byte K block in registers and
//               tcgen05.st's them into a 4-stage A ring in TMEM (the A
//               operand never touches shared memory).
//   warps 8-11  epilogue: tcgen05.ld the int32 accumulator (double
//               buffered in TMEM), scale (+digit recombination), bias, act,
//               128-bit stores.
// Work = (n-tile, 128-row tile) units, walked in row bands so every CTA works
// near the same rows (codes stay in L2) while each CTA keeps one n-tile's B
// image for many consecutive row tiles.

#include "common.cuh"

namespace lutgpu {

constexpr int kOhThreads = 12 * 32;
constexpr int kRowsPerTile = 128;
constexpr int kKB = 128;       // K bytes per A stage / B block
constexpr int kAStages = 4;

struct OneHotParams {
  const uint8_t* b_image;   // [ntiles][nkb][NT][128] swizzled
  int64_t n;
  int C, K, M;
  int NT;                   // B rows (MMA N) per tile
  int MT;                   // real output columns per tile = NT / digits
  int ntiles;
  int nkb;                  // K blocks of 128 bytes
  int64_t nrt;              // row tiles
  int64_t band_rt;          // row tiles per band
  int code_boxes;           // 128-byte TMA boxes per code row
  const float* scales;      // digits == 1: one scale or per m-tile
  int scale_mtile;
  const double* col_scale;  // digits > 1: per output column
  const float* bias;
  int act;
  float* out;
  int64_t out_hw;
  int32_t* out_i32;
  uint32_t tmem_cols;
};

// ------------------------------------------------------------ PTX helpers

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem]^T ; kind::i8, M=128
__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate), "r"(0), "r"(0), "r"(0), "r"(0)
      : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
      "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
      "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// SMEM matrix descriptor: K-major, 128B swizzle, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(const void* smem_ptr) {
  const uint64_t addr = smem_u32(smem_ptr);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;          // start address
  d |= (uint64_t)1 << 16;                 // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO = 1024 B
  d |= (uint64_t)1 << 46;                 // version (sm100)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

// kind::i8 instruction descriptor: A u8 (one-hot), B s8, D s32, K-major both.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4)            // D format s32
         | (0u << 7)          // A unsigned 8-bit
         | (1u << 10)         // B signed 8-bit
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// ------------------------------------------------------------ work walk

struct UnitWalk {
  int64_t band, nbands, lo, hi, cur;  // units [lo, hi) of the current band
  int64_t brt;
  const OneHotParams* p;
  __device__ void init(const OneHotParams& pp) {
    p = &pp;
    nbands = (pp.nrt + pp.band_rt - 1) / pp.band_rt;
    band = -1;
    lo = hi = cur = 0;
  }
  // next unit -> (ntile, rt); false at the end
  __device__ bool next(int& ntile, int64_t& rt) {
    while (cur >= hi) {
      if (++band >= nbands) return false;
      brt = min(p->band_rt, p->nrt - band * p->band_rt);
      const int64_t ub = (int64_t)p->ntiles * brt;
      lo = ub * blockIdx.x / gridDim.x;
      hi = ub * (blockIdx.x + 1) / gridDim.x;
      cur = lo;
    }
    ntile = (int)(cur / brt);
    rt = band * p->band_rt + cur % brt;
    ++cur;
    return true;
  }
};

// ------------------------------------------------------------ one-hot words

// 32 words = one 128-byte K block of this row's one-hot; codes for the block
// come from the swizzled code tile.  Power-of-two K only (host checks).
template <int K>
__device__ __forceinline__ void onehot_block(const uint8_t* code_row_sw, int sw, int kb, int C, bool valid,
                                             uint32_t (&w)[32]) {
  constexpr int CPB = kKB / K;  // codebooks per block (>= 1 for K <= 128)
  if constexpr (K >= 4) {
    constexpr int WPC = K / 4;  // words per codebook
    const int c0 = kb * CPB;
    constexpr int NW = (CPB + 3) / 4;
    uint32_t codes4[NW];
    // fetch the CPB code bytes from the swizzled tile (aligned words)
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const int byte = (c0 & ~3) + 4 * i;
      const int chunk = byte >> 4, within = byte & 15;
      codes4[i] = *reinterpret_cast<const uint32_t*>(code_row_sw + (((chunk & 7) ^ sw) << 4) + ((chunk >> 3) << 14) +
                                                     within);
    }
    if constexpr (CPB < 4) codes4[0] >>= 8 * (c0 & 3);
#pragma unroll
    for (int cb = 0; cb < CPB; ++cb) {
      const uint32_t code = (codes4[cb >> 2] >> (8 * (cb & 3))) & 255u;
      const bool live = valid && (c0 + cb < C);
      if constexpr (K == 16) {
        // one 64-bit shift places the byte; bit 3 of the code picks the half
        const uint64_t v = live ? (1ull << (8 * (code & 7))) : 0ull;
        const bool upper = (code & 8) != 0;
        w[cb * 4 + 0] = upper ? 0u : (uint32_t)v;
        w[cb * 4 + 1] = upper ? 0u : (uint32_t)(v >> 32);
        w[cb * 4 + 2] = upper ? (uint32_t)v : 0u;
        w[cb * 4 + 3] = upper ? (uint32_t)(v >> 32) : 0u;
      } else {
        const uint32_t bit = live ? (1u << (8 * (code & 3))) : 0u;
        const uint32_t wi = code >> 2;
#pragma unroll
        for (int j = 0; j < WPC; ++j) w[cb * WPC + j] = (wi == (uint32_t)j) ? bit : 0u;
      }
    }
  } else {
    // K in {1, 2}: several codebooks per word
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      uint32_t v = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int kbyte = kb * kKB + 4 * j + b;
        const int c = kbyte / K, kk = kbyte % K;
        if (valid && c < C) {
          const int chunk = c >> 4, within = c & 15;
          const uint32_t code =
              code_row_sw[(((chunk & 7) ^ sw) << 4) + ((chunk >> 3) << 14) + within];
          if ((int)code == kk) v |= 1u << (8 * b);
        }
      }
      w[j] = v;
    }
  }
}

// ------------------------------------------------------------ kernel

template <int K, int DIGITS>
__global__ void __launch_bounds__(kOhThreads, 1)
    onehot_gemm_kernel(const __grid_constant__ CUtensorMap codes_map, const __grid_constant__ OneHotParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b_bytes = p.NT * p.nkb * kKB;
  uint8_t* b_smem = smem;
  const int code_tile_bytes = p.code_boxes * kRowsPerTile * 128;
  uint8_t* code_smem = smem + ((b_bytes + 1023) & ~1023);  // 2 stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(code_smem + 2 * code_tile_bytes);
  uint64_t* b_full = bars + 0;
  uint64_t* b_empty = bars + 1;
  uint64_t* code_full = bars + 2;   // [2]
  uint64_t* code_empty = bars + 4;  // [2]
  uint64_t* a_full = bars + 6;      // [kAStages]
  uint64_t* a_empty = bars + 6 + kAStages;
  uint64_t* acc_full = bars + 6 + 2 * kAStages;   // [2]
  uint64_t* acc_empty = bars + 8 + 2 * kAStages;  // [2]
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(bars + 10 + 2 * kAStages);

  if (threadIdx.x == 0) {
    mbar_init(b_full, 1);
    mbar_init(b_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&code_full[i], 1);
      mbar_init(&code_empty[i], 4);
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);
    }
    for (int i = 0; i < kAStages; ++i) {
      mbar_init(&a_full[i], 4);
      mbar_init(&a_empty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_base_smem, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;
  const uint32_t acc_col0 = 0;                    // accumulators: [0, 2*NT)
  const uint32_t a_col0 = 2 * p.NT;               // A ring: kAStages x 32 columns

  UnitWalk walk;
  walk.init(p);

  if (warp == 0) {
    // ------------------------------------------------ producer
    if (lane == 0) {
      prefetch_tmap(&codes_map);
      int cur_ntile = -1;
      uint32_t b_phase = 0;
      int cs = 0;
      uint32_t cphase = 0;
      int ntile;
      int64_t rt;
      bool first_b = true;
      while (walk.next(ntile, rt)) {
        if (ntile != cur_ntile) {
          if (!first_b) {
            mbar_wait(b_empty, b_phase);
            b_phase ^= 1;
          }
          first_b = false;
          mbar_arrive_expect_tx(b_full, (uint32_t)b_bytes);
          const uint8_t* src = p.b_image + (size_t)ntile * b_bytes;
          for (int off = 0; off < b_bytes; off += 32768) {
            const int chunk = min(32768, b_bytes - off);
            bulk_load(b_smem + off, src + off, (uint32_t)chunk, b_full);
          }
          cur_ntile = ntile;
        }
        mbar_wait(&code_empty[cs], cphase ^ 1);
        mbar_arrive_expect_tx(&code_full[cs], (uint32_t)code_tile_bytes);
        for (int bx = 0; bx < p.code_boxes; ++bx)
          tma_load_2d(code_smem + cs * code_tile_bytes + bx * kRowsPerTile * 128, &codes_map, bx * 128,
                      (int32_t)(rt * kRowsPerTile), &code_full[cs]);
        if (++cs == 2) {
          cs = 0;
          cphase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    const uint32_t idesc = idesc_i8(128, p.NT);
    int cur_ntile = -1;
    uint32_t b_phase = 0;
    int as = 0;
    uint32_t aphase = 0;
    int acc = 0;
    uint32_t accphase = 0;
    int ntile;
    int64_t rt;
    UnitWalk look = walk;
    int nt_next;
    int64_t rt_next;
    bool has_next = look.next(nt_next, rt_next);
    while (has_next) {
      ntile = nt_next;
      rt = rt_next;
      has_next = look.next(nt_next, rt_next);
      if (ntile != cur_ntile) {
        mbar_wait(b_full, b_phase);
        b_phase ^= 1;
        cur_ntile = ntile;
      }
      mbar_wait(&acc_empty[acc], accphase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc_col0 + acc * p.NT;
      for (int kb = 0; kb < p.nkb; ++kb) {
        mbar_wait(&a_full[as], aphase);
        tc_fence_after();
        if (lane == 0) {
          const uint8_t* bblk = b_smem + (size_t)kb * p.NT * kKB;
#pragma unroll
          for (int j = 0; j < kKB / 32; ++j) {
            const uint32_t a_tmem = tmem_base + a_col0 + as * 32 + j * 8;
            mma_i8_ts(d_tmem, a_tmem, sw128_desc(bblk + j * 32), idesc, (kb | j) != 0);
          }
          tc_commit(&a_empty[as]);
        }
        __syncwarp();
        if (++as == kAStages) {
          as = 0;
          aphase ^= 1;
        }
      }
      if (lane == 0) {
        tc_commit(&acc_full[acc]);
        if (!has_next || nt_next != ntile) tc_commit(b_empty);
      }
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        accphase ^= 1;
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------ one-hot generators
    const int sub = warp & 3;
    const int row_in_tile = sub * 32 + lane;
    const int sw = row_in_tile & 7;
    int cs = 0;
    uint32_t cphase = 0;
    int as = 0;
    uint32_t aphase = 0;
    int ntile;
    int64_t rt;
    while (walk.next(ntile, rt)) {
      mbar_wait(&code_full[cs], cphase);
      const uint8_t* code_row = code_smem + cs * code_tile_bytes + row_in_tile * 128;
      const bool valid = rt * kRowsPerTile + row_in_tile < p.n;
      for (int kb = 0; kb < p.nkb; ++kb) {
        uint32_t w[32];
        onehot_block<K>(code_row, sw, kb, p.C, valid, w);
        mbar_wait(&a_empty[as], aphase ^ 1);
        tc_fence_after();
        tmem_st32(tmem_base + ((uint32_t)(sub * 32) << 16) + a_col0 + as * 32, w);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[as]);
        if (++as == kAStages) {
          as = 0;
          aphase ^= 1;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&code_empty[cs]);
      if (++cs == 2) {
        cs = 0;
        cphase ^= 1;
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------ epilogue
    const int sub = warp & 3;
    const int row_in_tile = sub * 32 + lane;
    int acc = 0;
    uint32_t accphase = 0;
    int ntile;
    int64_t rt;
    while (walk.next(ntile, rt)) {
      mbar_wait(&acc_full[acc], accphase);
      tc_fence_after();
      const int64_t row = rt * kRowsPerTile + row_in_tile;
      const bool live = row < p.n;
      const int m_base = ntile * p.MT;
      for (int ch = 0; ch < p.NT; ch += 16) {
        uint32_t v[16];
        tmem_ld16(tmem_base + ((uint32_t)(sub * 32) << 16) + acc_col0 + acc * p.NT + ch, v);
        tmem_ld_wait();
        if (!live) continue;
        constexpr int RC = 16 / DIGITS;  // real columns in this chunk
        float f[RC];
#pragma unroll
        for (int j = 0; j < RC; ++j) {
          const int m = m_base + (ch / DIGITS) + j;
          float x;
          if constexpr (DIGITS == 1) {
            const int acc_i = (int)v[j];
            if (p.out_i32 && m < p.M) {
              const int64_t o = p.out_hw > 0 ? ((row / p.out_hw) * p.M + m) * p.out_hw + row % p.out_hw
                                             : row * p.M + m;
              p.out_i32[o] = acc_i;
            }
            const float s = (m < p.M && p.scales)
                                ? (p.scale_mtile > 0 ? __ldg(p.scales + m / p.scale_mtile) : __ldg(p.scales))
                                : 1.0f;
            x = __fmul_rn(__int2float_rn(acc_i), s);
          } else {
            long long t = 0;
#pragma unroll
            for (int dg = DIGITS - 1; dg >= 0; --dg) t = t * 256 + (long long)(int)v[j * DIGITS + dg];
            const double s = m < p.M ? __ldg(p.col_scale + m) : 0.0;
            x = (float)((double)t * s);
          }
          if (p.bias && m < p.M) x = __fadd_rn(x, __ldg(p.bias + m));
          f[j] = apply_act(x, p.act);
        }
        if (p.out) {
          const int m0 = m_base + ch / DIGITS;
          if (p.out_hw == 0 && m0 + RC <= p.M && (p.M & 3) == 0 && (RC & 3) == 0) {
            float4* dst = reinterpret_cast<float4*>(p.out + row * p.M + m0);
#pragma unroll
            for (int j = 0; j < RC / 4; ++j) dst[j] = make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < RC; ++j) {
              const int m = m0 + j;
              if (m < p.M) {
                const int64_t o = p.out_hw > 0 ? ((row / p.out_hw) * p.M + m) * p.out_hw + row % p.out_hw
                                               : row * p.M + m;
                p.out[o] = f[j];
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
      if (++acc == 2) {
        acc = 0;
        accphase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// ------------------------------------------------------------ B image prep

// Swizzled K-major image of B for tile nt: byte (n_local, kbyte) at
// kb*NT*128 + n_local*128 + (((kk>>4) ^ (n_local&7))<<4) + (kk&15).
__device__ __forceinline__ size_t bimg_offset(int nt, int n_local, int kbyte, int NT, int nkb) {
  const int kb = kbyte >> 7, kk = kbyte & 127;
  return (size_t)nt * NT * nkb * kKB + (size_t)kb * NT * kKB + (size_t)n_local * kKB +
         ((((kk >> 4) ^ (n_local & 7)) << 4) | (kk & 15));
}

__global__ void bimg_i8_kernel(const int8_t* __restrict__ q, int C, int K, int M, int NT, int nkb, int ntiles,
                               uint8_t* __restrict__ img) {
  const int64_t total = (int64_t)ntiles * NT * nkb * kKB;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int kbyte = (int)(i % (nkb * kKB));
    const int64_t r = i / (nkb * kKB);
    const int n_local = (int)(r % NT), nt = (int)(r / NT);
    const int m = nt * NT + n_local;
    const int c = kbyte / K, kk = kbyte % K;
    int8_t v = 0;
    if (c < C && m < M) v = q[((int64_t)c * K + kk) * M + m];
    img[bimg_offset(nt, n_local, kbyte, NT, nkb)] = (uint8_t)v;
  }
}

__global__ void col_maxabs_kernel(const float* __restrict__ t, int64_t CK, int M, unsigned* __restrict__ maxbits,
                                  int* err) {
  const int64_t total = CK * M;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const float x = t[i];
    if (!isfinite(x)) {
      if (err) atomicMax(err, (int)LUT_ERR_DATA);
      continue;
    }
    atomicMax(maxbits + (i % M), __float_as_uint(fabsf(x)));
  }
}

__global__ void col_scale_kernel(const unsigned* __restrict__ maxbits, int M, int digits, double* __restrict__ s) {
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < M; m += gridDim.x * blockDim.x) {
    const double mx = (double)__uint_as_float(maxbits[m]);
    s[m] = mx > 0.0 ? mx / ldexp(1.0, 8 * digits - 2) : 1.0;
  }
}

__global__ void bimg_digits_kernel(const float* __restrict__ t, int C, int K, int M, int digits, int NT, int MT,
                                   int nkb, int ntiles, const double* __restrict__ s, uint8_t* __restrict__ img) {
  const int64_t total = (int64_t)ntiles * MT * nkb * kKB;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int kbyte = (int)(i % (nkb * kKB));
    const int64_t r = i / (nkb * kKB);
    const int m_local = (int)(r % MT), nt = (int)(r / MT);
    const int m = nt * MT + m_local;
    const int c = kbyte / K, kk = kbyte % K;
    long long tv = 0;
    if (c < C && m < M) {
      const float x = t[((int64_t)c * K + kk) * M + m];
      tv = isfinite(x) ? llrint((double)x / s[m]) : 0;
    }
    for (int dg = 0; dg < digits; ++dg) {
      long long b = ((tv + 128) & 255) - 128;  // balanced digit in [-128, 127]
      tv = (tv - b) / 256;
      img[bimg_offset(nt, m_local * digits + dg, kbyte, NT, nkb)] = (uint8_t)(int8_t)b;
    }
  }
}

// ------------------------------------------------------------ host

struct OneHotGeom {
  int NT, MT, ntiles, nkb;
  size_t img_bytes;
};

static bool pow2_k(int K) { return K >= 1 && K <= 128 && (K & (K - 1)) == 0; }

static OneHotGeom onehot_geom(int C, int K, int M, int digits) {
  OneHotGeom g{};
  g.nkb = (C * K + kKB - 1) / kKB;
  const size_t budget = 144 * 1024;
  int NT = 128;
  while (NT > 16 && (size_t)NT * g.nkb * kKB > budget) NT /= 2;
  // do not waste B rows on a small M
  while (NT > 16 && NT / 2 >= M * digits) NT /= 2;
  g.NT = NT;
  g.MT = NT / digits;
  g.ntiles = (M + g.MT - 1) / g.MT;
  g.img_bytes = (size_t)g.ntiles * NT * g.nkb * kKB;
  return g;
}

int onehot_supported(int C, int K, int M, int digits) {
  if (!pow2_k(K) || C < 1 || M < 1) return 0;
  if (digits != 1 && digits != 2 && digits != 4) return 0;
  OneHotGeom g = onehot_geom(C, K, M, digits);
  if ((size_t)g.NT * g.nkb * kKB > 144 * 1024) return 0;
  if (g.NT % digits) return 0;
  return 1;
}

size_t onehot_image_bytes(int C, int K, int M, int digits) {
  OneHotGeom g = onehot_geom(C, K, M, digits);
  return g.img_bytes + (digits > 1 ? (size_t)M * (sizeof(double) + sizeof(unsigned)) + 64 : 0);
}

static int grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 32;
  if (b < 1) b = 1;
  return (int)(b < cap ? b : cap);
}

int onehot_prepare_i8(const int8_t* q, int C, int K, int M, void* image, cudaStream_t stream) {
  OneHotGeom g = onehot_geom(C, K, M, 1);
  const int64_t total = (int64_t)g.ntiles * g.NT * g.nkb * kKB;
  bimg_i8_kernel<<<grid_for(total), 256, 0, stream>>>(q, C, K, M, g.NT, g.nkb, g.ntiles, static_cast<uint8_t*>(image));
  LUT_CHECK_LAUNCH("bimg_i8_kernel");
  return LUT_OK;
}

int onehot_prepare_f32(const float* t, int C, int K, int M, int digits, void* image, int* err, cudaStream_t stream) {
  OneHotGeom g = onehot_geom(C, K, M, digits);
  uint8_t* img = static_cast<uint8_t*>(image);
  double* s = reinterpret_cast<double*>(img + ((g.img_bytes + 15) & ~size_t(15)));
  unsigned* maxbits = reinterpret_cast<unsigned*>(s + M);
  cudaError_t e = cudaMemsetAsync(maxbits, 0, (size_t)M * sizeof(unsigned), stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(col max)");
  const int64_t CK = (int64_t)C * K;
  col_maxabs_kernel<<<grid_for(CK * M), 256, 0, stream>>>(t, CK, M, maxbits, err);
  col_scale_kernel<<<(M + 255) / 256, 256, 0, stream>>>(maxbits, M, digits, s);
  const int64_t total = (int64_t)g.ntiles * g.MT * g.nkb * kKB;
  bimg_digits_kernel<<<grid_for(total), 256, 0, stream>>>(t, C, K, M, digits, g.NT, g.MT, g.nkb, g.ntiles, s, img);
  LUT_CHECK_LAUNCH("bimg_digits_kernel");
  return LUT_OK;
}

const double* onehot_col_scale(const void* image, int C, int K, int M, int digits) {
  OneHotGeom g = onehot_geom(C, K, M, digits);
  return reinterpret_cast<const double*>(static_cast<const uint8_t*>(image) + ((g.img_bytes + 15) & ~size_t(15)));
}

template <int K, int DIGITS>
static int launch_onehot_k(const CUtensorMap& map, OneHotParams& p, size_t smem, int grid, cudaStream_t stream) {
  auto kern = onehot_gemm_kernel<K, DIGITS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(onehot)");
  kern<<<grid, kOhThreads, smem, stream>>>(map, p);
  LUT_CHECK_LAUNCH("onehot_gemm_kernel");
  return LUT_OK;
}

template <int DIGITS>
static int dispatch_k(int K, const CUtensorMap& map, OneHotParams& p, size_t smem, int grid, cudaStream_t stream) {
  switch (K) {
    case 1: return launch_onehot_k<1, DIGITS>(map, p, smem, grid, stream);
    case 2: return launch_onehot_k<2, DIGITS>(map, p, smem, grid, stream);
    case 4: return launch_onehot_k<4, DIGITS>(map, p, smem, grid, stream);
    case 8: return launch_onehot_k<8, DIGITS>(map, p, smem, grid, stream);
    case 16: return launch_onehot_k<16, DIGITS>(map, p, smem, grid, stream);
    case 32: return launch_onehot_k<32, DIGITS>(map, p, smem, grid, stream);
    case 64: return launch_onehot_k<64, DIGITS>(map, p, smem, grid, stream);
    case 128: return launch_onehot_k<128, DIGITS>(map, p, smem, grid, stream);
    default: return fail(LUT_ERR_CONFIG, "one-hot gather needs power-of-two K <= 128");
  }
}

// codes: (n, code_stride) u8 with code_stride % 16 == 0 (TMA row pitch)
int onehot_gather(const uint8_t* codes, int64_t code_stride, int64_t n, int C, int K, int M, int digits,
                  const void* image, const float* scales, int scale_mtile, const float* bias, int act, float* out,
                  int32_t* out_i32, int64_t out_hw, cudaStream_t stream) {
  if (n == 0 || M == 0) return LUT_OK;
  if (!onehot_supported(C, K, M, digits)) return fail(LUT_ERR_CONFIG, "shape not supported by the one-hot gather");
  if (code_stride % 16 != 0 || (reinterpret_cast<uintptr_t>(codes) & 15))
    return fail(LUT_ERR_CONFIG, "one-hot gather needs 16-byte aligned code rows");
  OneHotGeom g = onehot_geom(C, K, M, digits);
  CUtensorMap map;
  const int code_boxes = (C + 127) / 128;
  if (!make_tmap_2d_u8(&map, codes, (uint64_t)code_stride, (uint64_t)n, (uint64_t)code_stride, 128, kRowsPerTile,
                       true))
    return fail(LUT_ERR_CUDA, "cuTensorMapEncodeTiled(codes) failed");
  OneHotParams p{};
  p.b_image = static_cast<const uint8_t*>(image);
  p.n = n;
  p.C = C;
  p.K = K;
  p.M = M;
  p.NT = g.NT;
  p.MT = g.MT;
  p.ntiles = g.ntiles;
  p.nkb = g.nkb;
  p.nrt = (n + kRowsPerTile - 1) / kRowsPerTile;
  p.code_boxes = code_boxes;
  p.scales = scales;
  p.scale_mtile = scale_mtile;
  p.col_scale = digits > 1 ? onehot_col_scale(image, C, K, M, digits) : nullptr;
  p.bias = bias;
  p.act = act;
  p.out = out;
  p.out_hw = out_hw;
  p.out_i32 = out_i32;
  uint32_t cols = 2 * g.NT + kAStages * 32;
  uint32_t alloc = 32;
  while (alloc < cols) alloc <<= 1;
  p.tmem_cols = alloc;
  const int nsm = num_sms();
  const int64_t units = (int64_t)g.ntiles * p.nrt;
  const int grid = (int)(units < nsm ? units : nsm);
  // band = row tiles such that ntiles * band divides evenly over the grid
  int64_t a = grid, b = g.ntiles;
  while (b) {
    const int64_t t = a % b;
    a = b;
    b = t;
  }
  p.band_rt = grid / a;
  if (p.band_rt < 1) p.band_rt = 1;
  if (p.band_rt > p.nrt) p.band_rt = p.nrt;
  const size_t b_bytes = (size_t)g.NT * g.nkb * kKB;
  const size_t smem = ((b_bytes + 1023) & ~size_t(1023)) + 2 * (size_t)code_boxes * kRowsPerTile * 128 + 256 + 1024;
  if (smem > max_smem_optin()) return fail(LUT_ERR_CONFIG, "one-hot gather: shared memory budget exceeded");
  switch (digits) {
    case 1: return dispatch_k<1>(K, map, p, smem, grid, stream);
    case 2: return dispatch_k<2>(K, map, p, smem, grid, stream);
    case 4: return dispatch_k<4>(K, map, p, smem, grid, stream);
    default: return fail(LUT_ERR_CONFIG, "digits must be 1, 2 or 4");
  }
}

}  // namespace lutgpu
