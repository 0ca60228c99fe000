// Microbenchmark: tcgen05.mma.cta_group::2.kind::i8 (M=256, A from TMEM) issue
// rate on a CTA pair, alone and while other warps stream tcgen05.st / .ld
// traffic through the same TMEM (the one-hot gather's generator / epilogue).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_pair_bench.bin tools/mma_pair_bench.cu
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

__global__ void __cluster_dims__(2, 1, 1) bench(int N, int iters, int mode, int cta_group2, int aspan, int ss, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int stop;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    if (cta_group2)
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    else
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tbase;
  if (warp == 1 && (rank == 0 || !cta_group2)) {
    if ((threadIdx.x & 31) == 0) {
      const uint32_t idesc = idesc_i8(cta_group2 ? 256 : 128, N);
      const uint64_t b = sw128_desc(smem_u32(sm + 32768));
      const uint64_t adesc = sw128_desc(smem_u32(sm));
      long long t0 = clock64();
      for (int i = 0; i < iters; ++i) {
        const uint32_t acc = (i & 7) != 0;
        const uint32_t aoff = (uint32_t)(i % aspan);
        if (ss) {
          // A from SMEM: aspan distinct 32-byte K slices over 8 x 1024B-atoms blocks of 16 KB
          const uint64_t ad = adesc + (uint64_t)(((aoff >> 2) * 16384 + (aoff & 3) * 32) >> 4);
          if (cta_group2)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(t),
                         "l"(ad), "l"(b + (uint64_t)((i & 3) * 2)), "r"(idesc), "r"(acc));
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(t),
                         "l"(ad), "l"(b + (uint64_t)((i & 3) * 2)), "r"(idesc), "r"(acc));
        } else if (cta_group2)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(t),
                       "r"(t + 256 + aoff * 8), "l"(b + (uint64_t)((i & 3) * 2)), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(t),
                       "r"(t + 256 + aoff * 8), "l"(b + (uint64_t)((i & 3) * 2)), "r"(idesc), "r"(acc));
      }
      if (cta_group2)
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"((uint16_t)3));
      else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar)));
      out[blockIdx.x] = clock64() - t0;
      stop = 1;
    }
  } else if (warp >= 4 && warp < 12 && (mode & 1)) {
    // generator-like: tcgen05.st x64 into columns [384, 448) of this warp's lane quarter
    const uint32_t a = t + ((uint32_t)((warp & 3) * 32) << 16) + 384;
    uint32_t v[64];
    for (int i = 0; i < 64; ++i) v[i] = i;
    long long n = 0;
    while (!stop && n < 100000) {
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
          "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, "
          "%36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, "
          "%57, %58, %59, %60, %61, %62, %63, %64};" ::"r"(a),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
          "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
          "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
          "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]), "r"(v[32]), "r"(v[33]), "r"(v[34]), "r"(v[35]),
          "r"(v[36]), "r"(v[37]), "r"(v[38]), "r"(v[39]), "r"(v[40]), "r"(v[41]), "r"(v[42]), "r"(v[43]), "r"(v[44]),
          "r"(v[45]), "r"(v[46]), "r"(v[47]), "r"(v[48]), "r"(v[49]), "r"(v[50]), "r"(v[51]), "r"(v[52]), "r"(v[53]),
          "r"(v[54]), "r"(v[55]), "r"(v[56]), "r"(v[57]), "r"(v[58]), "r"(v[59]), "r"(v[60]), "r"(v[61]), "r"(v[62]),
          "r"(v[63]));
      asm volatile("tcgen05.wait::st.sync.aligned;");
      ++n;
    }
  } else if (warp >= 12 && warp < 16 && (mode & 2)) {
    // epilogue-like: tcgen05.ld x16 from the accumulator columns
    const uint32_t a = t + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t s = 0;
    long long n = 0;
    while (!stop && n < 100000) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
          "%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(a + (uint32_t)((n & 7) * 16)));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      s += v[0] + v[15];
      ++n;
    }
    if (s == 12345) out[0] = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;");
  if (warp == 0) {
    if (cta_group2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(t));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 296);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 4096;
  for (int ss : {0, 1})
  for (int cg2 : {0, 1})
    for (int N : {128, 256})
      for (int aspan : {1, 2, 4, 8, 16})
      for (int mode : {0}) {
        if (ss && aspan > 8) continue;
        bench<<<2, 512, 100 * 1024>>>(N, iters, mode, cg2, aspan, ss, d);
        bench<<<2, 512, 100 * 1024>>>(N, iters, mode, cg2, aspan, ss, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[2];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        const double clk = (double)h[0] / iters;
        const double macs = (cg2 ? 128.0 : 128.0) * N * 32;  // per SM
        printf("%s cta_group::%d N=%3d aspan=%2d mode=%d: %6.1f clk/mma  %6.0f MAC/clk/SM %s\n", ss ? "SS" : "TS",
               cg2 ? 2 : 1, N, aspan, mode, clk, macs / clk, e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
