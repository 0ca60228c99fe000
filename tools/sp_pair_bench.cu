// Microbenchmark: issue/execute rate of 2:4-sparse kind::i8 MMAs (A + metadata in TMEM)
// as the pair gather issues them (elect.sync asm blocks of 4 MMAs), cta_group::1 vs ::2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sp_pair_bench.bin tools/sp_pair_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
#define SP_G(G, AOFF, BOFF, EOFF)                                                       \
  "add.u32 ta, %1, " #AOFF ";\n\tadd.u64 tb, %2, " #BOFF ";\n\tadd.u32 te, %5, " #EOFF ";\n\t" \
  "@e tcgen05.mma.sp.cta_group::" #G ".kind::i8 [%0], [ta], tb, [te], %3, p0;\n\t"
#define SP_GS(G, AOFF, BOFF, EOFF)                                                      \
  "add.u64 tas, %6, " #AOFF ";\n\tadd.u64 tb, %2, " #BOFF ";\n\tadd.u32 te, %5, " #EOFF ";\n\t" \
  "@e tcgen05.mma.sp.cta_group::" #G ".kind::i8 [%0], tas, tb, [te], %3, p0;\n\t"
// A operand from SMEM (descriptor %6) instead of TMEM; metadata still in TMEM
#define SP_STAGE_AS(G)                                                                    \
  "{\n\t.reg .pred e, p0;\n\t.reg .b32 te;\n\t.reg .b64 tb, tas;\n\t"                 \
  "elect.sync _|e, 0xffffffff;\n\tsetp.ne.u32 p0, %4, 0;\n\t"                          \
  SP_GS(G, 0, 0, 0) SP_GS(G, 2, 4, 2) SP_GS(G, 4, 8, 4) SP_GS(G, 6, 12, 6) "}"
#define SP_STAGE(G)                                                                       \
  "{\n\t.reg .pred e, p0;\n\t.reg .b32 ta, te;\n\t.reg .b64 tb;\n\t"                     \
  "elect.sync _|e, 0xffffffff;\n\tsetp.ne.u32 p0, %4, 0;\n\t"                          \
  SP_G(G, 0, 0, 0) SP_G(G, 8, 4, 2) SP_G(G, 16, 8, 4) SP_G(G, 24, 12, 6) "}"

template <int G>
__global__ void __cluster_dims__(2, 1, 1) bench(int N, int iters, long long* out, int mode) {
  __shared__ volatile int stop;
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2;
  __shared__ __align__(8) uint64_t bar3;
  __shared__ uint32_t flag;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 100000000;" ::"r"(smem_u32(&bar2)));
    flag = 1;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar3)));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar3)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    if (G == 2)
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    else
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tbase;
  if (warp == 1 && (rank == 0 || G == 1)) {
    const uint32_t idesc = idesc_i8(G == 2 ? 256 : 128, N) | 4u;
    const uint64_t b = sw128_desc(smem_u32(sm + 32768));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint32_t a = 256 + (uint32_t)(i & 3) * 40;
      uint64_t bb = b;
      uint32_t dd = t;
      if (mode & 512) {
        const int st = (i >> 1) & 3;                 // stage within the unit (2 asm blocks per stage)
        const int half = i & 1;
        const int unit = i >> 3;
        a = 256 + (uint32_t)((i >> 1) % 3) * 80 + (uint32_t)half * 32;
        bb = b + (uint64_t)(((4 * st + 2 * half) * 64 * 128) >> 4);
        dd = t + (uint32_t)(unit & 1) * 128;
        if (mode & 8192) dd = t;
        if (mode & 16384) bb = b;
        if (mode & 32768) a = 256 + (uint32_t)(i & 3) * 40;
        if (mode & 4096) {  // A ring in columns 0..239, accumulators at 256 / 384
          a -= 256;
          dd += 256;
        }
      }
      if ((mode & 256) && (!(i & 1) || (mode & 1048576))) asm volatile("bar.sync 1, 64;" ::: "memory");  // hand-off from the watcher warp (1048576: every 4 MMAs)
      if ((mode & 8) && ((mode & 64) ? !(i & 3) : !(i & 1))) {  // poll a completed barrier every 8 (or 16) MMAs
        uint32_t ok = 0;
        if (mode & 128) {  // poll a plain SMEM flag word (LSU path) instead of an mbarrier
          while (!ok) asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(ok) : "r"(smem_u32(&flag)) : "memory");
        } else if (mode & 32)
          while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar3)) : "memory");
        else
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.relaxed.cluster.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                       : "=r"(ok) : "r"(smem_u32(&bar3)) : "memory");
        if (!(mode & 16)) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      if constexpr (G == 2) {
        if ((mode & 65536) && !(i & 1)) {  // stage A (80 cols) from SMEM into TMEM with 10 tcgen05.cp 128x256b
          const uint64_t src = sw128_desc(smem_u32(sm) + (uint32_t)((i >> 1) & 1) * 40960);
#pragma unroll
          for (int j = 0; j < 10; ++j)
            asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                         "@e tcgen05.cp.cta_group::2.128x256b [%0], %1;\n\t}" ::"r"(t + a + 8 * j),
                         "l"(src + (uint64_t)((j * 4096) >> 4)) : "memory");
        }
        if (mode & 262144)
          asm volatile(SP_STAGE_AS(2)::"r"(dd), "r"(t + a), "l"(bb), "r"(idesc), "r"((uint32_t)((i & 7) != 0)),
                       "r"(t + a + 64 - 32 * (uint32_t)(i & 1) + 8 * (uint32_t)(i & 1)),
                       "l"(sw128_desc(smem_u32(sm) + (uint32_t)(i & 3) * 8192)) : "memory");
        else
        asm volatile(SP_STAGE(2)::"r"(dd), "r"(t + a), "l"(bb), "r"(idesc), "r"((uint32_t)((i & 7) != 0)),
                     "r"(t + a + 64 - 32 * (uint32_t)(i & 1) + 8 * (uint32_t)(i & 1))
                     : "memory");
        if ((mode & 4) && ((i & 1) || (mode & 1048576))) {  // commit every 8 MMAs (1048576: every 4) (multicast to both CTAs' barrier 2)
          asm volatile(
              "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
              ::"r"(smem_u32(&bar2)), "h"((uint16_t)3) : "memory");
        }
      }
      else
        asm volatile(SP_STAGE(1)::"r"(t), "r"(t + a), "l"(b), "r"(idesc), "r"((uint32_t)(i != 0)), "r"(t + a + 32)
                     : "memory");
    }
    if (threadIdx.x == 32) {
      if (G == 2)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"((uint16_t)3));
      else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar)));
    }
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    if (threadIdx.x == 32) out[blockIdx.x] = clock64() - t0;
    stop = 1;
  } else if (warp == 2 && (mode & 256) && (rank == 0 || G == 1)) {
    // watcher: polls the (completed) barrier, then releases the issuer through a named barrier
    for (int i = 0; i < iters; i += (mode & 1048576) ? 1 : 2) {
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.relaxed.cluster.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar3)) : "memory");
      asm volatile("bar.sync 1, 64;" ::: "memory");
    }
  } else if (warp >= 4 && warp < 12 && (mode & 1)) {
    // generator-like: tcgen05.st x32 into A-ring columns of this warp's lane quarter
    const uint32_t a = t + ((uint32_t)((warp & 3) * 32) << 16) + ((mode & 4096) ? 0u : 256u) + (uint32_t)((warp >> 2) & 1) * 128;
    long long n = 0;
    if (mode & 131072) {  // same bytes as STS into the SMEM A image (4 KB per warp iteration)
      const uint32_t base = smem_u32(sm) + (uint32_t)(warp - 4) * 4096 + (threadIdx.x & 31) * 16;
      while (!stop && n < 200000) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(base + j * 512), "r"((uint32_t)n) : "memory");
        asm volatile("bar.sync %0, 32;" ::"r"(2 + warp - 4) : "memory");
        ++n;
      }
    } else
    while (!stop && n < 200000) {
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
          "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(a + (uint32_t)(n & 3) * 32),
          "r"((uint32_t)n));
      asm volatile("tcgen05.wait::st.sync.aligned;");
      ++n;
    }
  } else if (warp >= 12 && warp < 16 && (mode & 2)) {
    // epilogue-like: tcgen05.ld x32 from accumulator columns
    const uint32_t a = t + ((uint32_t)((warp & 3) * 32) << 16) + ((mode & 4096) ? 384u : 128u);
    uint32_t s = 0;
    long long n = 0;
    while (!stop && n < 200000) {
      uint32_t v[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
          "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(a + (uint32_t)(n & 3) * 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      s += v[0] + v[31];
      ++n;
    }
    if (s == 12345) out[0] = 0;
  }
  if (G == 2 && rank == 1 && warp == 1) {  // peer: wait for the multicast commit too
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  if (warp == 0) {
    if (G == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(t));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
  }
}

template <int G>
static void run(int N, int blocks, int mode = 0) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * blocks);
  cudaMemset(d, 0, sizeof(long long) * blocks);
  const int iters = 2048;
  cudaFuncSetAttribute(bench<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  bench<G><<<blocks, 512, 200 * 1024>>>(N, iters, d, mode);
  bench<G><<<blocks, 512, 200 * 1024>>>(N, iters, d, mode);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0;
  int cnt = 0;
  for (int i = 0; i < blocks; ++i)
    if (h[i]) avg += h[i], ++cnt;
  avg /= cnt;
  const double mmas = 4.0 * iters;
  printf("sparse i8 cta_group::%d N=%3d blocks=%3d mode=%d: %6.1f clk/mma (per-SM rows 128, K=64 logical) %s\n", G, N, blocks, mode,
         avg / mmas, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  // 772: no generators (MMA-bound floor); 773: tcgen05.st generators (the shipped layout);
  // +65536: A staged SMEM->TMEM by tcgen05.cp; +131072: generators write SMEM (STS) instead;
  // +262144: A read by the MMA straight from SMEM (descriptor), metadata still in TMEM.
  for (int mode : {0, 4, 260, 516, 772 + 8192, 772 + 16384, 772 + 32768, 772 + 8192 + 16384 + 32768, 772, 773, 772 + 65536, 773 + 65536, 773 + 131072, 773 + 65536 + 131072, 772 + 262144,
                   773 + 262144 + 131072, 775 + 65536 + 131072, 775 + 262144 + 131072, 775})
    run<2>(128, 148, mode);
  for (int n : {128, 160, 192, 224, 256})  // one accumulator at column 256, A ring at 0..239
    for (int mode : {4, 772 + 4096 + 8192, 773 + 4096 + 8192, 775 + 4096 + 8192}) run<2>(n, 148, mode);
  // 4-MMA ring stages (commit + watcher hand-off every 4 MMAs): the N = 192 design's 2-K-block stages
  for (int n : {128, 192})
    for (int mode : {772 + 4096 + 8192 + 1048576, 773 + 4096 + 8192 + 1048576, 775 + 4096 + 8192 + 1048576}) run<2>(n, 148, mode);
  return 0;
}
