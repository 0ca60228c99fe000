// Probe for a tensor-core encode: tcgen05.mma kind::tf32, M=128, small N.
//  (1) numerics: how the MMA treats the low 13 bits of f32 operands (truncate /
//      round / keep) and the size of its accumulation error vs an f64 reference;
//  (2) rate: cycles per MMA for N in {16, 32, 64}, A from TMEM (TS) or SMEM (SS).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tf32_probe.bin tools/tf32_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// A: 128 x 32 f32 (row-major), B: N x 32 f32 (row-major), D: 128 x N f32.
// mode 0: A from TMEM; mode 1: A from SMEM.
__global__ void numerics(const float* A, const float* B, int N, float* D, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  uint8_t* sa = sm;            // 128 rows x 128 B
  uint8_t* sb = sm + 16384;    // N rows x 128 B
  for (int i = t; i < 128 * 8; i += blockDim.x) {
    const int r = i >> 3, j = i & 7;
    memcpy(sa + r * 128 + ((j ^ (r & 7)) << 4), A + r * 32 + 4 * j, 16);
  }
  for (int i = t; i < N * 8; i += blockDim.x) {
    const int r = i >> 3, j = i & 7;
    memcpy(sb + r * 128 + ((j ^ (r & 7)) << 4), B + r * 32 + 4 * j, 16);
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  // A row t -> TMEM lane t, columns 64..95
  {
    uint32_t v[32];
    for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(A[t * 32 + j]);
    const uint32_t addr = tm + ((uint32_t)(warp * 32) << 16) + 64;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(addr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
        "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
        "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (t == 0) {
    const uint32_t idesc = idesc_tf32(128, N);
    for (int k = 0; k < 4; ++k) {
      const uint64_t bd = sw128_desc(smem_u32(sb) + 32 * k);
      if (mode == 0)
        mma_ts(tm, tm + 64 + 8 * k, bd, idesc, k > 0);
      else
        mma_ss(tm, sw128_desc(smem_u32(sa) + 32 * k), bd, idesc, k > 0);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t addr = tm + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) D[t * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

// rate: one thread issues `iters` MMAs (K=8 each) into a rotating set of accumulators
__global__ void rate(int N, int iters, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (t == 0) {
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
  const uint32_t tm = tbase;
  if (t == 0) {
    const uint32_t idesc = idesc_tf32(128, N);
    const uint64_t b = sw128_desc(smem_u32(sm + 16384));
    const uint64_t a = sw128_desc(smem_u32(sm));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      // mode&2: one accumulator, always accumulate; mode&4: 8 independent accumulators (N<=16 apart)
      uint32_t d = tm + (uint32_t)((i >> 2) & 3) * 64;
      uint32_t acc = (i & 3) != 0;
      if (mode & 2) { d = tm; acc = i > 0; }
      if (mode & 4) { d = tm + (uint32_t)(i & 7) * 16; acc = 0; }
      if ((mode & 1) == 0)
        mma_ts(d, tm + 256 + (i & 3) * 8, b + (uint64_t)((i & 3) * 2), idesc, acc);
      else
        mma_ss(d, a + (uint64_t)((i & 3) * 2), b + (uint64_t)((i & 3) * 2), idesc, acc);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

static float trunc_tf32(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}
static float rna_tf32(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  const int N = 16;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, 128 * 32 * 4);
  cudaMalloc(&dB, 64 * 32 * 4);
  cudaMalloc(&dD, 128 * 64 * 4);
  cudaFuncSetAttribute(numerics, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  static float A[128 * 32], B[64 * 32], D[128 * 64];
  srand(1);
  auto rnd = [] { return (float)(((double)rand() / RAND_MAX) * 2.0 - 1.0) * 1.7f; };
  for (int mode = 0; mode < 2; ++mode) {
    for (int variant = 0; variant < 3; ++variant) {
      // variant 0: raw f32; 1: exact tf32 (masked) operands; 2: raw with products of mixed sign magnitudes
      for (int i = 0; i < 128 * 32; ++i) A[i] = variant == 1 ? trunc_tf32(rnd()) : rnd();
      for (int i = 0; i < N * 32; ++i) B[i] = variant == 1 ? trunc_tf32(rnd()) : rnd();
      if (variant == 2)
        for (int i = 0; i < 128 * 32; ++i) A[i] *= (i % 7 == 0) ? 1024.0f : 1.0f;
      cudaMemcpy(dA, A, sizeof(A), cudaMemcpyHostToDevice);
      cudaMemcpy(dB, B, N * 32 * 4, cudaMemcpyHostToDevice);
      numerics<<<1, 128, 64 * 1024>>>(dA, dB, N, dD, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("numerics mode %d: %s\n", mode, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(D, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
      double emax_raw = 0, emax_tr = 0, emax_rn = 0, rel_tr = 0;
      for (int r = 0; r < 128; ++r)
        for (int c = 0; c < N; ++c) {
          double sr = 0, st = 0, sn = 0, sabs = 0;
          for (int k = 0; k < 32; ++k) {
            sr += (double)A[r * 32 + k] * B[c * 32 + k];
            st += (double)trunc_tf32(A[r * 32 + k]) * trunc_tf32(B[c * 32 + k]);
            sn += (double)rna_tf32(A[r * 32 + k]) * rna_tf32(B[c * 32 + k]);
            sabs += fabs((double)trunc_tf32(A[r * 32 + k]) * trunc_tf32(B[c * 32 + k]));
          }
          const double g = D[r * N + c];
          emax_raw = fmax(emax_raw, fabs(g - sr));
          emax_tr = fmax(emax_tr, fabs(g - st));
          emax_rn = fmax(emax_rn, fabs(g - sn));
          rel_tr = fmax(rel_tr, fabs(g - st) / sabs);
        }
      printf("numerics mode=%s variant=%d: max|D-exact(raw)|=%.3e  max|D-exact(trunc)|=%.3e  max|D-exact(rna)|=%.3e  "
             "max err(trunc)/sum|t| = %.3e (= %.2f * 2^-23)\n",
             mode == 0 ? "TS" : "SS", variant, emax_raw, emax_tr, emax_rn, rel_tr, rel_tr / ldexp(1.0, -23));
    }
  }
  long long* dout;
  cudaMalloc(&dout, 148 * 8);
  for (int mode : {0, 1, 2, 3, 4, 5})
    for (int n : {16, 32, 64, 128}) {
      if ((mode & 4) && n > 16) continue;
      for (int rep = 0; rep < 2; ++rep) {
        const int iters = 4096;
        rate<<<148, 128, 64 * 1024>>>(n, iters, mode, dout);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("rate: %s\n", cudaGetErrorString(e));
          return 1;
        }
        long long h[148];
        cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost);
        double s = 0;
        for (int i = 0; i < 148; ++i) s += h[i];
        if (rep == 1)
          printf("rate %s mode=%d N=%3d: %.2f cycles per MMA (M=128,K=8) -> %.0f MAC/clk/SM\n", (mode & 1) == 0 ? "TS" : "SS", mode, n,
                 s / 148 / iters, 128.0 * n * 8 / (s / 148 / iters));
      }
    }
  return 0;
}
