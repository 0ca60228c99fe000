// Probe: tcgen05.mma.sp kind::i8 with A (2:4-compressed) and metadata in TMEM.
// Establishes the metadata encoding for a one-hot A empirically and times the
// sparse MMA issue rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sparse_probe.bin tools/sparse_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
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
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int sparse) {
  return (sparse ? 4u : 0u) | (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

constexpr int KL = 128;  // logical K (one 128-byte B K block)

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]));
}

// mode: metadata hypothesis.  0: nibble per group (lo 2 bits = first index), pair
// (h&2, h&2+1), value in slot h&1.  1: same but nibbles in reverse group order.
template <int N>
__global__ void probe(const int8_t* bsrc, const int* kstar, int* out, int mode, int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = threadIdx.x;
  // B: N rows x 128 bytes, SW128 K-major: chunk j of row n at chunk j ^ (n & 7)
  for (int i = threadIdx.x; i < N * KL; i += blockDim.x) {
    const int n = i / KL, k = i % KL;
    const int chunk = (k >> 4) ^ (n & 7);
    sm[n * 128 + chunk * 16 + (k & 15)] = (uint8_t)bsrc[n * KL + k];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
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
  // compressed A (64 bytes = 16 words) and metadata (128 logical / 8 per byte = 16 bytes = 4 words)
  uint32_t a[16] = {0}, e[4] = {0};
  const int ks = kstar[m];
  for (int g = 0; g < KL / 4; ++g) {
    uint32_t nib = 0x4;  // (0, 1)
    if (g == ks / 4) {
      const int h = ks & 3;
      const int i0 = h & 2, i1 = i0 + 1;
      nib = (uint32_t)(i0 | (i1 << 2));
      const int byte = 2 * g + (h & 1);
      a[byte >> 2] |= 1u << (8 * (byte & 3));
    }
    const int gg = mode == 1 ? ((g & ~7) | (7 - (g & 7))) : g;
    e[gg >> 3] |= nib << (4 * (gg & 7));
  }
  const uint32_t lane_base = t + ((uint32_t)(warp * 32) << 16);
  tmem_st16(lane_base + 256, a);
  tmem_st4(lane_base + 300, e);
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_i8(128, N, 1);
    const uint64_t b = sw128_desc(smem_u32(sm));
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t acc = (q != 0);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], [%1], %2, [%5], %3, p;\n\t}" ::"r"(t),
                     "r"(t + 256 + q * 8), "l"(b + (uint64_t)(q * 4)), "r"(idesc), "r"(acc), "r"(t + 300 + q * 2));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar)));
    }
    *cycles = clock64() - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[N];
#pragma unroll
  for (int c = 0; c < N; c += 16) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[c + 0]), "=r"(v[c + 1]), "=r"(v[c + 2]), "=r"(v[c + 3]), "=r"(v[c + 4]), "=r"(v[c + 5]),
          "=r"(v[c + 6]), "=r"(v[c + 7]), "=r"(v[c + 8]), "=r"(v[c + 9]), "=r"(v[c + 10]), "=r"(v[c + 11]),
          "=r"(v[c + 12]), "=r"(v[c + 13]), "=r"(v[c + 14]), "=r"(v[c + 15])
        : "r"(lane_base + c));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int c = 0; c < N; ++c) out[m * N + c] = (int)v[c];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t));
  (void)lane;
}

template <int N>
static int run_n() {
  static int8_t hb[N * KL];
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < KL; ++k)
      hb[n * KL + k] = n == 0 ? (int8_t)k : n == 1 ? (int8_t)1 : (int8_t)(((k * 7 + n * 13) % 200) - 100);
  int hk[128];
  for (int m = 0; m < 128; ++m) hk[m] = (m * 37 + 5) % KL;
  int8_t* db;
  int *dk, *dout;
  long long* dcyc;
  cudaMalloc(&db, sizeof(hb));
  cudaMalloc(&dk, sizeof(hk));
  cudaMalloc(&dout, 128 * N * sizeof(int));
  cudaMalloc(&dcyc, sizeof(long long));
  cudaMemcpy(db, hb, sizeof(hb), cudaMemcpyHostToDevice);
  cudaMemcpy(dk, hk, sizeof(hk), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  static int hout[128 * N];
  for (int mode = 0; mode < 1; ++mode) {
    probe<N><<<1, 128, 64 * 1024>>>(db, dk, dout, mode, 1, dcyc);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      printf("mode %d: %s\n", mode, cudaGetErrorString(err));
      return 1;
    }
    cudaMemcpy(hout, dout, sizeof(hout), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n)
        if (hout[m * N + n] != hb[n * KL + hk[m]]) ++bad;
    printf("mode %d: mismatches %d / %d\n", mode, bad, 128 * N);
    for (int m = 0; m < 2; ++m)
      printf("  row %d k*=%3d  D[0]=%4d D[1]=%4d D[2]=%4d (want %4d)\n", m, hk[m], hout[m * N], hout[m * N + 1],
             hout[m * N + 2], hb[2 * KL + hk[m]]);
  }
  for (int iters : {1024}) {
    probe<N><<<1, 128, 64 * 1024>>>(db, dk, dout, 0, iters, dcyc);
    cudaDeviceSynchronize();
    long long cyc;
    cudaMemcpy(&cyc, dcyc, sizeof(cyc), cudaMemcpyDeviceToHost);
    printf("sparse i8 TS M=128 N=%d: %.1f clk per MMA (K=64 logical) = %.0f logical MAC/clk\n", N,
           (double)cyc / (2.0 * iters), 128.0 * N * 64 * 2.0 * iters / (double)cyc);
  }
  return 0;
}

int main() {
  run_n<64>();
  run_n<128>();
  run_n<256>();
  return 0;
}
