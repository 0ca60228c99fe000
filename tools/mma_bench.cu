// Microbenchmark: cycles per tcgen05.mma on one SM for the shapes the one-hot
// gather can use (kind::i8, M=128, A from TMEM or SMEM, several N) plus a
// kind::f16 reference.  Data are zeros; only the issue/execute rate matters.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
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
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {  // bf16 x bf16 -> f32
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int MODE>  // 0: i8 TS, 1: i8 SS, 2: f16 SS, 3: i8 TS with disable-output-lane mask
__global__ void bench(int N, int iters, long long* out, int extra) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2[8];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tbase;
  if (threadIdx.x == 0) {
    const uint32_t idesc = MODE == 2 ? idesc_f16(128, N) : idesc_i8(128, N);
    const uint64_t a = sw128_desc(smem_u32(sm));
    const uint64_t b = sw128_desc(smem_u32(sm + 32768));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t acc = (i & 3) != 0;
      if (MODE == 0) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(t),
                     "r"(t + 256 + (i & 3) * 8), "l"(b + (uint64_t)((i & 3) * 2)), "r"(idesc), "r"(acc));
      } else if (MODE == 3) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(t),
                     "r"(t + 256 + (i & 3) * 8), "l"(b + (uint64_t)((i & 3) * 2)), "r"(idesc), "r"(acc), "r"(0),
                     "r"(0), "r"(0), "r"(0));
      } else if (MODE == 1) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(t),
                     "l"(a + (uint64_t)((i & 3) * 2)), "l"(b + (uint64_t)((i & 3) * 2)), "r"(idesc), "r"(acc));
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(t),
                     "l"(a + (uint64_t)((i & 3) * 2)), "l"(b + (uint64_t)((i & 3) * 2)), "r"(idesc), "r"(acc));
      }
      if ((i & 7) == 7) {
        if (extra & 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_u32(&bar2[(i >> 3) & 7])));
        if (extra & 2) asm volatile("tcgen05.fence::after_thread_sync;");
        if (extra & 4) asm volatile("tcgen05.fence::before_thread_sync;");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    }
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
}

template <int MODE>
static void run(const char* name, int N, int blocks, int extra = 0) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * blocks);
  const int iters = 4096;
  cudaFuncSetAttribute(bench<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  bench<MODE><<<blocks, 128, 100 * 1024>>>(N, iters, d, extra);  // warm
  bench<MODE><<<blocks, 128, 100 * 1024>>>(N, iters, d, extra);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < blocks; ++i) avg += h[i];
  avg /= blocks;
  const double macs = 128.0 * N * (MODE == 2 ? 16 : 32);
  printf("%-10s N=%3d blocks=%3d extra=%d: %7.1f clk/mma  %7.0f MAC/clk/SM  %s\n", name, N, blocks, extra, avg / iters,
         macs * iters / avg, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main(int argc, char** argv) {
  if (argc > 1) {
    for (int extra = 0; extra < 8; ++extra) run<0>("i8 TS", 64, 1, extra);
    for (int extra : {0, 1, 3}) run<0>("i8 TS", 128, 1, extra);
    for (int extra : {0, 1, 3}) run<0>("i8 TS", 256, 1, extra);
    return 0;
  }
  for (int blocks : {1, 148}) {
    for (int N : {16, 32, 64, 128, 256}) run<0>("i8 TS", N, blocks);
    for (int N : {16, 64, 256}) run<3>("i8 TSmask", N, blocks);
    for (int N : {64, 128, 256}) run<1>("i8 SS", N, blocks);
    for (int N : {64, 256}) run<2>("bf16 SS", N, blocks);
  }
  return 0;
}
