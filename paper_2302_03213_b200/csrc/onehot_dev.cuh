// Device-side building blocks of the one-hot tensor-core gathers (onehot.cu,
// onehot_stream.cu): launch parameters, tcgen05 / TMEM / mbarrier / cluster PTX
// wrappers, the 2:4-sparse one-hot generator and the MMA issue blocks.
#pragma once

#include "common.cuh"

namespace lutgpu {


// Ablation bits and role counters exist only in probe builds (-DLUTGPU_PROBES,
// tools/build_probes.sh): in the product build they are compile-time zero, so
// no check of them reaches the issued code.
#ifdef LUTGPU_PROBES
#define OH_DEBUG(p) ((p).debug)
#define OH_TRACE(p) ((p).trace)
#else
#define OH_DEBUG(p) 0
#define OH_TRACE(p) static_cast<unsigned long long*>(nullptr)
#endif

constexpr int kOhThreads = 14 * 32;  // producer, MMA, 8 generators, 4 epilogue
constexpr int kRowsPerTile = 128;
constexpr int kKB = 128;       // K bytes per A stage / B block
constexpr int kMaxAStages = 24;  // A ring depth bound (barrier arrays)

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
  int a_stages;             // A ring depth (<= kMaxAStages)
  int n_acc;                // TMEM accumulator buffers (pair kernel: 1 or 2)
  int spin;                 // 1: latency-critical waits poll instead of sleeping
  int tma_out;              // 1: epilogue stages the tile in SMEM and TMA-stores it
  int stage_slab;           // pair kernel: SMEM staging slab allocated (TMA or transpose epilogue)
  int epi;                  // pair kernel epilogue variant (0 generic; plain int8: 1/4 TMA, 2 direct, 3 transpose)
  int watch;                // pair kernel: warp 18 polls the issuer's barriers and hands stages over (bar.sync)
  unsigned long long* trace;  // optional per-role cycle counters (LUTGPU_OH_TRACE), CTA 0 only
  unsigned long long* tl;     // optional event timeline (LUTGPU_OH_TL=<file>), CTAs 0 and 1 (one pair)
  int sparse;               // 2:4-compressed one-hot A (tcgen05.mma.sp), else dense
  int stage_kb;             // pair kernel, sparse: 128-byte K blocks per A ring stage (1 or 2)
  int pdl;                  // launched as a programmatic dependent of the layer's encode
  int debug;                // ablation bits (LUTGPU_OH_DEBUG): 1 no epilogue math/stores, 2 no MMA,
                            // 4 no TMEM A stores, 8 MMA only (no A handshake, generators idle)
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

__device__ __forceinline__ void tmem_ld16_lo(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}

template <int OFF>
__device__ __forceinline__ void tmem_ld32_at(uint32_t taddr, uint32_t (&v)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[OFF + 0]), "=r"(v[OFF + 1]), "=r"(v[OFF + 2]), "=r"(v[OFF + 3]), "=r"(v[OFF + 4]), "=r"(v[OFF + 5]),
        "=r"(v[OFF + 6]), "=r"(v[OFF + 7]), "=r"(v[OFF + 8]), "=r"(v[OFF + 9]), "=r"(v[OFF + 10]), "=r"(v[OFF + 11]),
        "=r"(v[OFF + 12]), "=r"(v[OFF + 13]), "=r"(v[OFF + 14]), "=r"(v[OFF + 15]), "=r"(v[OFF + 16]),
        "=r"(v[OFF + 17]), "=r"(v[OFF + 18]), "=r"(v[OFF + 19]), "=r"(v[OFF + 20]), "=r"(v[OFF + 21]),
        "=r"(v[OFF + 22]), "=r"(v[OFF + 23]), "=r"(v[OFF + 24]), "=r"(v[OFF + 25]), "=r"(v[OFF + 26]),
        "=r"(v[OFF + 27]), "=r"(v[OFF + 28]), "=r"(v[OFF + 29]), "=r"(v[OFF + 30]), "=r"(v[OFF + 31])
      : "r"(taddr)
      : "memory");
}

template <int OFF>
__device__ __forceinline__ void tmem_ld16_at(uint32_t taddr, uint32_t (&v)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[OFF + 0]), "=r"(v[OFF + 1]), "=r"(v[OFF + 2]), "=r"(v[OFF + 3]), "=r"(v[OFF + 4]), "=r"(v[OFF + 5]),
        "=r"(v[OFF + 6]), "=r"(v[OFF + 7]), "=r"(v[OFF + 8]), "=r"(v[OFF + 9]), "=r"(v[OFF + 10]), "=r"(v[OFF + 11]),
        "=r"(v[OFF + 12]), "=r"(v[OFF + 13]), "=r"(v[OFF + 14]), "=r"(v[OFF + 15])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ uint64_t pk_f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void up_f2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t add_f2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t mul_f2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
constexpr uint64_t kNegMagic2 = 0xCB400000CB400000ull;  // {-12582912.0f, -12582912.0f}

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
  // Units of a band are ordered n-tile-major; this CTA owns a contiguous
  // slice [lo, hi) of each band.  All state is 32-bit and updated
  // incrementally (no per-unit 64-bit division on the critical path).
  int band, nbands;
  int brt;            // row tiles in the current band
  int left;           // units left in this band's slice
  int ntile, rtl;     // current position (rtl = row tile inside the band)
  int nrt, band_rt, ntiles;
  int slot, nslots;   // this worker (CTA or CTA pair) among all workers
  __device__ void init(const OneHotParams& pp, int slot_ = -1, int nslots_ = -1) {
    nrt = (int)pp.nrt;
    band_rt = (int)pp.band_rt;
    ntiles = pp.ntiles;
    slot = slot_ < 0 ? (int)blockIdx.x : slot_;
    nslots = nslots_ < 0 ? (int)gridDim.x : nslots_;
    nbands = (nrt + band_rt - 1) / band_rt;
    band = -1;
    left = 0;
  }
  __device__ bool next(int& nt, int64_t& rt) {
    while (left == 0) {
      if (++band >= nbands) return false;
      brt = min(band_rt, nrt - band * band_rt);
      const int64_t ub = (int64_t)ntiles * brt;
      const int lo = (int)(ub * slot / nslots);
      const int hi = (int)(ub * (slot + 1) / nslots);
      left = hi - lo;
      ntile = lo / brt;
      rtl = lo - ntile * brt;
    }
    nt = ntile;
    rt = (int64_t)band * band_rt + rtl;
    --left;
    if (++rtl == brt) {
      rtl = 0;
      ++ntile;
    }
    return true;
  }
};

// ------------------------------------------------------------ kernel

__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}

__device__ __forceinline__ void sts_v4(uint32_t saddr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int32_t x, int32_t y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, const void* src, int32_t x, int32_t y,
                                                  uint64_t policy) {
#if LUTGPU_L2_HINTS
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src)), "l"(policy)
               : "memory");
#else
  (void)policy;
  tma_store_2d(map, src, x, y);
#endif
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Code bytes of one ring stage (two 128-byte K blocks) for this row, read
// from the 128B-swizzled code tile (16-byte chunk j of row r at
// ((j ^ (r & 7)) << 4), 16 KB per 128-column box).
template <int K, int KB = 2>
struct StageCodes {
  static constexpr int CPB = kKB / K;          // codebooks per K block
  static constexpr int CPS = KB * CPB;         // codebooks per stage
  static constexpr int NW = (CPS + 3) / 4;     // code words per stage
  uint32_t w[NW];
  __device__ __forceinline__ void load(uint32_t row_saddr, int sw, int st) {
    const int c0 = st * CPS;
    if constexpr (NW == 4) {  // 16 code bytes = one aligned chunk
      const int chunk = c0 >> 4;
      const uint32_t a = row_saddr + ((chunk >> 3) << 14) + (((chunk & 7) ^ sw) << 4);
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                   : "r"(a));
    } else {
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        const int byte = (c0 & ~3) + 4 * i;
        const int chunk = byte >> 4;
        w[i] = lds_u32(row_saddr + ((chunk >> 3) << 14) + (((chunk & 7) ^ sw) << 4) + (byte & 15));
      }
      if constexpr (CPS < 4) w[0] >>= 8 * (c0 & 3);
    }
  }
};

// 1 << s for a 64-bit value with PTX semantics: shift counts >= 64 give 0.
__device__ __forceinline__ uint64_t shl64(uint32_t s) {
  uint64_t r;
  asm("shl.b64 %0, 1, %1;" : "=l"(r) : "r"(s));
  return r;
}

// One-hot bytes of a stage: byte (cb*K + code) of the 2*128-byte row is 1.
// No validity masking: rows >= n are never stored and codebooks >= C meet
// zero rows of the B image.
template <int K>
__device__ __forceinline__ void build_onehot(const StageCodes<K>& cd, uint32_t (&w)[64]) {
  constexpr int CPS = StageCodes<K>::CPS;
  constexpr int WPC = K / 4;  // words per codebook
#pragma unroll
  for (int cb = 0; cb < CPS; ++cb) {
    const uint32_t code = __byte_perm(cd.w[cb >> 2], 0, 0x4440 + (cb & 3)) & (K - 1);
    if constexpr (K == 16) {
      const uint64_t lo = shl64(code << 3);          // bytes 0..7   (code < 8)
      const uint64_t hi = shl64((code << 3) - 64u);  // bytes 8..15  (code >= 8; wraps -> 0 otherwise)
      w[cb * 4 + 0] = (uint32_t)lo;
      w[cb * 4 + 1] = (uint32_t)(lo >> 32);
      w[cb * 4 + 2] = (uint32_t)hi;
      w[cb * 4 + 3] = (uint32_t)(hi >> 32);
    } else if constexpr (K == 8) {
      const uint64_t v = shl64(code << 3);
      w[cb * 2 + 0] = (uint32_t)v;
      w[cb * 2 + 1] = (uint32_t)(v >> 32);
    } else if constexpr (K == 4) {
      w[cb] = 1u << (code << 3);
    } else {
      const uint32_t bit = 1u << ((code & 3) << 3);
      const uint32_t wi = code >> 2;
#pragma unroll
      for (int j = 0; j < WPC; ++j) w[cb * WPC + j] = (wi == (uint32_t)j) ? bit : 0u;
    }
  }
}

// 2:4-compressed one-hot of a stage for tcgen05.mma.sp (kind::i8).  Logical
// position P = cb*K + code lies in group G = P/4 with hot slot h = code&3.
// Every group of a codebook uses the same position pair: (2,3) if code&2
// else (0,1) (cold groups carry zeros, so their pair is free), hence the
// compressed row holds byte 2*(code>>2) + (code&1) = 1 and zeros elsewhere,
// and the codebook's metadata nibbles (i0 | i1<<2, little-endian per group,
// 8 groups per 32-bit TMEM column) are all 0xE or all 0x4 (layout verified
// against dense results by tools/sparse_probe.cu).  Four codes are
// processed per 32-bit word with byte-parallel masks.
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t s) {  // PTX: s >= 32 gives 0
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
  return r;
}

template <int K, int KB = 2>
__device__ __forceinline__ void build_sparse(const StageCodes<K, KB>& cd, uint32_t (&a)[16 * KB],
                                             uint32_t (&e)[4 * KB]) {
  constexpr int CPS = StageCodes<K, KB>::CPS;
  if constexpr (K == 16 || K == 8) {
#pragma unroll
    for (int i = 0; i < CPS / 4; ++i) {
      const uint32_t W = cd.w[i] & (0x01010101u * (K - 1));
      const uint32_t bp8 = ((((W >> 1) & 0x06060606u) | (W & 0x01010101u)) << 3);  // 8 * compressed byte
      const uint32_t hb = (W >> 1) & 0x01010101u;                                    // pair (2,3) flag
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t sh = __byte_perm(bp8, 0, 0x4440 + j);
        if constexpr (K == 16) {  // 8 compressed bytes = 2 words; 4 groups = 16 metadata bits
          a[(4 * i + j) * 2 + 0] = shl_clamp(1u, sh);
          a[(4 * i + j) * 2 + 1] = shl_clamp(1u, sh - 32u);
        } else {  // 4 compressed bytes = 1 word; 2 groups = 8 metadata bits
          a[4 * i + j] = shl_clamp(1u, sh);
        }
      }
      if constexpr (K == 16) {  // metadata word = 2 codebooks: nibbles 0x4 + 0xA*flag (disjoint bits)
        e[2 * i + 0] = __byte_perm(hb, 0, 0x4140) * 0xAAAAu + 0x44444444u;
        e[2 * i + 1] = __byte_perm(hb, 0, 0x4342) * 0xAAAAu + 0x44444444u;
      } else {  // metadata word = 4 codebooks, one byte each
        e[i] = hb * 0xAAu + 0x44444444u;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4 * KB; ++i) e[i] = 0x44444444u;
#pragma unroll
    for (int cb = 0; cb < CPS; ++cb) {
      const uint32_t code = __byte_perm(cd.w[cb >> 2], 0, 0x4440 + (cb & 3)) & (K - 1);
      const uint32_t bytepos = 2u * (code >> 2) + (code & 1u);  // compressed byte inside the codebook
      const uint32_t flag = (code >> 1) & 1u;
      if constexpr (K == 4) {  // 2 bytes = half word; 1 group = 1 nibble
        if ((cb & 1) == 0) a[cb >> 1] = 0u;
        a[cb >> 1] |= 1u << (16 * (cb & 1) + (bytepos << 3));
        e[cb >> 3] ^= (flag * 0xAu) << (4 * (cb & 7));
      } else {  // K >= 32: K/8 words and K/32 metadata words (all 0xE or all 0x4) per codebook
        constexpr int WPC = K / 8;
        constexpr int EPC = K / 32;
        const uint32_t wi = bytepos >> 2, bit = 1u << ((bytepos & 3) << 3);
#pragma unroll
        for (int j = 0; j < WPC; ++j) a[cb * WPC + j] = (wi == (uint32_t)j) ? bit : 0u;
#pragma unroll
        for (int j = 0; j < EPC; ++j) e[cb * EPC + j] = flag ? 0xEEEEEEEEu : 0x44444444u;
      }
    }
  }
}

__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

__device__ __forceinline__ void tmem_st64(uint32_t taddr, const uint32_t (&v)[64]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, "
      "%36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, "
      "%57, %58, %59, %60, %61, %62, %63, %64};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
      "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
      "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]), "r"(v[32]), "r"(v[33]), "r"(v[34]), "r"(v[35]),
      "r"(v[36]), "r"(v[37]), "r"(v[38]), "r"(v[39]), "r"(v[40]), "r"(v[41]), "r"(v[42]), "r"(v[43]), "r"(v[44]),
      "r"(v[45]), "r"(v[46]), "r"(v[47]), "r"(v[48]), "r"(v[49]), "r"(v[50]), "r"(v[51]), "r"(v[52]), "r"(v[53]),
      "r"(v[54]), "r"(v[55]), "r"(v[56]), "r"(v[57]), "r"(v[58]), "r"(v[59]), "r"(v[60]), "r"(v[61]), "r"(v[62]),
      "r"(v[63])
      : "memory");
}

// One ring stage (up to two 128-byte K blocks = 8 MMAs) issued from a single
// asm block executed by the whole warp, predicated on elect.sync: operands stay
// warp-uniform (no per-MMA R2UR/ELECT loop in SASS) and the 8 address offsets
// are immediates.  acc0 = accumulate flag of the stage's first MMA.
#define OH_MMA_G(G, AOFF, BOFF, PRED)       \
  "add.u32 ta, %1, " #AOFF ";\n\t"        \
  "add.u64 tb, %2, " #BOFF ";\n\t"        \
  "@e tcgen05.mma.cta_group::" #G ".kind::i8 [%0], [ta], tb, %4, " #PRED ";\n\t"
#define OH_MMA_H(G, AOFF, BOFF)             \
  "add.u32 ta, %1, " #AOFF ";\n\t"        \
  "add.u64 tb, tb2, " #BOFF ";\n\t"       \
  "@e tcgen05.mma.cta_group::" #G ".kind::i8 [%0], [ta], tb, %4, pt2;\n\t"
#define OH_STAGE_ASM(G)                                                                      \
  "{\n\t.reg .pred e, p0, pt2, e2;\n\t.reg .b32 ta;\n\t.reg .b64 tb, tb2;\n\t"            \
  "elect.sync _|e, 0xffffffff;\n\t"                                                         \
  "setp.ne.u32 p0, %5, 0;\n\t"                                                              \
  "setp.eq.u32 pt2, %4, %4;\n\t"                                                            \
  OH_MMA_G(G, 0, 0, p0) OH_MMA_G(G, 8, 2, pt2) OH_MMA_G(G, 16, 4, pt2) OH_MMA_G(G, 24, 6, pt2) \
  "setp.ne.u32 e2, %6, 0;\n\t"                                                              \
  "and.pred e, e, e2;\n\t"                                                                  \
  "add.u64 tb2, %2, %3;\n\t"                                                                \
  OH_MMA_H(G, 32, 0) OH_MMA_H(G, 40, 2) OH_MMA_H(G, 48, 4) OH_MMA_H(G, 56, 6) "}"

// Sparse stage: 4 tcgen05.mma.sp (K = 64 logical each): compressed A 8 TMEM
// columns and metadata 2 columns per MMA, B advanced 64 bytes per MMA.
#define OH_SP_G(G, AOFF, BOFF, EOFF, PRED) \
  "add.u32 ta, %1, " #AOFF ";\n\t"       \
  "add.u64 tb, %2, " #BOFF ";\n\t"       \
  "add.u32 te, %7, " #EOFF ";\n\t"       \
  "@e tcgen05.mma.sp.cta_group::" #G ".kind::i8 [%0], [ta], tb, [te], %4, " #PRED ";\n\t"
#define OH_SP_H(G, AOFF, BOFF, EOFF)       \
  "add.u32 ta, %1, " #AOFF ";\n\t"       \
  "add.u64 tb, tb2, " #BOFF ";\n\t"      \
  "add.u32 te, %7, " #EOFF ";\n\t"       \
  "@e tcgen05.mma.sp.cta_group::" #G ".kind::i8 [%0], [ta], tb, [te], %4, pt2;\n\t"
#define OH_SP_STAGE_ASM(G)                                                   \
  "{\n\t.reg .pred e, p0, pt2, e2;\n\t.reg .b32 ta, te;\n\t.reg .b64 tb, tb2;\n\t" \
  "elect.sync _|e, 0xffffffff;\n\t"                                        \
  "setp.ne.u32 p0, %5, 0;\n\t"                                             \
  "setp.eq.u32 pt2, %4, %4;\n\t"                                           \
  OH_SP_G(G, 0, 0, 0, p0) OH_SP_G(G, 8, 4, 2, pt2)                          \
  "setp.ne.u32 e2, %6, 0;\n\t"                                             \
  "and.pred e, e, e2;\n\t"                                                 \
  "add.u64 tb2, %2, %3;\n\t"                                               \
  OH_SP_H(G, 16, 0, 4) OH_SP_H(G, 24, 4, 6) "}"

#define OH_SP1_STAGE_ASM(G)                                                  \
  "{\n\t.reg .pred e, p0, pt2;\n\t.reg .b32 ta, te;\n\t.reg .b64 tb;\n\t"      \
  "elect.sync _|e, 0xffffffff;\n\t"                                        \
  "setp.ne.u32 p0, %4, 0;\n\t"                                             \
  "setp.eq.u32 pt2, %3, %3;\n\t"                                           \
  "add.u32 ta, %1, 0;\n\tadd.u64 tb, %2, 0;\n\tadd.u32 te, %5, 0;\n\t"    \
  "@e tcgen05.mma.sp.cta_group::" #G ".kind::i8 [%0], [ta], tb, [te], %3, p0;\n\t" \
  "add.u32 ta, %1, 8;\n\tadd.u64 tb, %2, 4;\n\tadd.u32 te, %5, 2;\n\t"    \
  "@e tcgen05.mma.sp.cta_group::" #G ".kind::i8 [%0], [ta], tb, [te], %3, pt2;\n\t}"

// one-K-block sparse stage: 2 tcgen05.mma.sp
template <int CG>
__device__ __forceinline__ void issue_stage_sp1(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc0,
                                                uint32_t meta) {
  if constexpr (CG == 2) {
    asm volatile(OH_SP1_STAGE_ASM(2)::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc0), "r"(meta) : "memory");
  } else {
    asm volatile(OH_SP1_STAGE_ASM(1)::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc0), "r"(meta) : "memory");
  }
}

template <int CG>
__device__ __forceinline__ void issue_stage_sp(uint32_t d, uint32_t a, uint64_t b, uint64_t bstep, uint32_t idesc,
                                               uint32_t acc0, uint32_t two, uint32_t meta) {
  if constexpr (CG == 2) {
    asm volatile(OH_SP_STAGE_ASM(2)::"r"(d), "r"(a), "l"(b), "l"(bstep), "r"(idesc), "r"(acc0), "r"(two), "r"(meta)
                 : "memory");
  } else {
    asm volatile(OH_SP_STAGE_ASM(1)::"r"(d), "r"(a), "l"(b), "l"(bstep), "r"(idesc), "r"(acc0), "r"(two), "r"(meta)
                 : "memory");
  }
}

// One ring stage (up to two 128-byte K blocks = 8 MMAs) issued from a single
// asm block executed by the whole warp, predicated on elect.sync: operands stay
// warp-uniform (no per-MMA R2UR/ELECT loop in SASS) and the 8 address offsets
// are immediates.  acc0 = accumulate flag of the stage's first MMA; two = the
// stage holds a second K block.
template <int CG>
__device__ __forceinline__ void issue_stage(uint32_t d, uint32_t a, uint64_t b, uint64_t bstep, uint32_t idesc,
                                            uint32_t acc0, uint32_t two) {
  if constexpr (CG == 2) {
    asm volatile(OH_STAGE_ASM(2)::"r"(d), "r"(a), "l"(b), "l"(bstep), "r"(idesc), "r"(acc0), "r"(two) : "memory");
  } else {
    asm volatile(OH_STAGE_ASM(1)::"r"(d), "r"(a), "l"(b), "l"(bstep), "r"(idesc), "r"(acc0), "r"(two) : "memory");
  }
}

// tcgen05.commit from an elected lane (whole warp executes it)
__device__ __forceinline__ void commit_elect(uint64_t* bar, bool pair) {
  if (pair)
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

// cycle accounting for the LUTGPU_OH_TRACE diagnostic (CTA 0, one lane per role)
// Timeline probe (LUTGPU_OH_TL): %globaltimer stamps of pipeline events of the
// first pair, indexed by global ring stage (generators / MMA) or unit (epilogue).
constexpr int kTlN = 192, kTlEv = 20;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// The probes compile in only with -DLUTGPU_PROBES (tools/build_probes.sh): their
// parameter checks and clock reads otherwise sit on the MMA issuer's critical path.
#ifdef LUTGPU_PROBES
#define TL(ev, idx)                                                                                  \
  do {                                                                                               \
    if (p.tl && blockIdx.x < 2 && (int)(idx) >= 0 && (int)(idx) < kTlN)                             \
      p.tl[((int)blockIdx.x * kTlEv + (ev)) * kTlN + (int)(idx)] = gtime();                          \
  } while (0)
#define OH_T0(var) long long var = (OH_TRACE(p) && blockIdx.x == 0) ? clock64() : 0
#define OH_ACC(slot, var) \
  do {                    \
    if (OH_TRACE(p) && blockIdx.x == 0 && lane == 0) atomicAdd(OH_TRACE(p) + (slot), (unsigned long long)(clock64() - var)); \
  } while (0)
#else
#define TL(ev, idx) \
  do {              \
  } while (0)
#define OH_T0(var) \
  do {             \
  } while (0)
#define OH_ACC(slot, var) \
  do {                    \
  } while (0)
#endif

// Role warps.  A warp may only touch the TMEM lane quarter warp % 4, so each
// group of 4 consecutive warps covers all 128 rows whatever its first index.
constexpr int kGenWarp0 = 2;   // warps 2..9: generators (parity = (warp-2)>>2)
constexpr int kEpiWarp0 = 10;  // warps 10..13: epilogue (pair kernel: 10..17, one accumulator half each)
constexpr int kPairThreads = 19 * 32;  // + warp 18: the leader's barrier watcher
constexpr int kGenWarps = 8;
constexpr int kStageCols = 64;  // TMEM columns per A stage (2 K blocks x 128 B / 4 B)
constexpr int kSparseStageCols = 40;  // 2:4 sparse stage: 32 compressed A + 8 metadata columns

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// arrive on an mbarrier given by its shared::cluster address (may be the peer's)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Relaxed remote arrive / waits for the per-stage and per-unit handshakes.
// No generic memory crosses the pair on these paths: the A stages and
// accumulators live in TMEM and are ordered by tcgen05.wait::st/ld plus the
// tcgen05 thread-sync fences around the arrive/wait.  A release.cluster arrive
// compiles to MEMBAR.ALL.GPU (~1 us under the output stream) and an
// acquire.cluster wait to CCTL.IVALL; the relaxed forms compile to neither.
__device__ __forceinline__ void mbar_arrive_cluster_rlx(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool mbar_test_rlx(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.relaxed.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_try_wait_rlx(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
// spin as in mbar_wait_crit (1: poll; else sleep-wait)
__device__ __forceinline__ void mbar_wait_rlx(uint64_t* bar, uint32_t parity, int spin) {
  if (spin == 1) {
    while (!mbar_test_rlx(bar, parity)) {
    }
  } else {
    while (!mbar_try_wait_rlx(bar, parity)) {
    }
  }
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_cluster(bar, parity)) {
  }
}
__device__ __forceinline__ bool mbar_test_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// latency-critical wait: poll (test_wait) when spin, else sleep in try_wait
__device__ __forceinline__ bool mbar_try_wait_cluster_nohint(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// spin: 0 = try_wait with a long suspend hint, 1 = test_wait polling,
// 2 = try_wait with the hardware's default time slice
__device__ __forceinline__ void mbar_wait_crit(uint64_t* bar, uint32_t parity, int spin) {
  if (spin == 1) {
    while (!mbar_test_cluster(bar, parity)) {
    }
  } else if (spin == 2) {
    while (!mbar_try_wait_cluster_nohint(bar, parity)) {
    }
  } else {
    mbar_wait_cluster(bar, parity);
  }
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  // arrive on the barrier at this offset in both CTAs of the pair
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mma_i8_ts_pair(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}




// Pair-kernel warp roles.  The SMSP arbiter issues from the highest warp id
// first, so the latency-critical single-thread roles (MMA issuer, producer)
// take the top ids; generators and epilogue keep warp % 4 == TMEM lane quarter.
constexpr int kPGen0 = 0;    // warps 0..7: one-hot generators (parity = warp >> 2)
constexpr int kPEpi0 = 8;    // warps 8..15: epilogue (accumulator half = (warp - 8) >> 2)
constexpr int kPProd = 16;   // producer (B image, code tiles)
constexpr int kPMma = 17;    // TMEM allocator + MMA issuer (leader) / peer signaler
constexpr int kPWatch = 18;  // leader: barrier watcher for the MMA issuer

}  // namespace lutgpu
