// Prints the register <-> (lane, column) mapping of tcgen05.ld.16x256b.x2 on sm_100a:
// every TMEM cell is first written with lane * 1000 + column through 32x32b stores.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_ld_probe.bin tools/tmem_ld_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(uint32_t* out) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tbase;
  // thread = TMEM lane (warp w owns lanes 32w..32w+31): columns 0..15 <- lane*1000 + col
  const uint32_t row = warp * 32 + lane;
  uint32_t v[16];
  for (int c = 0; c < 16; ++c) v[c] = row * 1000 + c;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          t + ((uint32_t)(warp * 32) << 16)),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // each warp reads 16 lanes x 16 columns of its quarter, lane halves 0 and 1
  for (int lh = 0; lh < 2; ++lh) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(t + ((uint32_t)(warp * 32 + lh * 16) << 16))
                 : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) out[((warp * 2 + lh) * 32 + lane) * 8 + i] = r[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(t));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 4 * 2 * 32 * 8 * 4);
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  static uint32_t h[4 * 2 * 32 * 8];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int w : {0, 2})
    for (int lh = 0; lh < 2; ++lh)
      for (int t : {0, 1, 2, 3, 4, 5, 31}) {
        printf("warp %d lh %d thread %2d:", w, lh, t);
        for (int i = 0; i < 8; ++i) {
          const uint32_t x = h[((w * 2 + lh) * 32 + t) * 8 + i];
          printf("  r%d=(L%u,c%u)", i, x / 1000, x % 1000);
        }
        printf("\n");
      }
  return 0;
}
