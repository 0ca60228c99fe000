// FFMA2 operand-pattern throughput (sm_100a): the strip conv encode's inner loop
// acc[i][q] = fma2((a_i, a_i), cp[q], acc[i][q]) with 32 accumulators, 8 centroid
// pairs and 4 scalars, against variants of the multiplicand's form.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ffma2_pattern.bin tools/ffma2_pattern.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// MODE 0: scalar multiplicand packed (a, a) (compiler may use the .F32 broadcast form)
// MODE 1: multiplicand pair (a, a') with distinct halves (a true 64-bit register operand)
// MODE 2: pixels paired instead of centroids: (a_i, a_i+1) x (p, p) broadcast on the centroid side
// MODE 3: plain FFMA on 64 scalar accumulators (same flops)
template <int MODE>
__global__ void __launch_bounds__(256, 2) k(int iters, const float* in, float* out, long long* cyc) {
  float a[4], c[16];
  for (int i = 0; i < 4; ++i) a[i] = in[i + threadIdx.x % 3];
  for (int i = 0; i < 16; ++i) c[i] = in[8 + i + threadIdx.x % 5];
  long long t0 = clock64();
  float s = 0;
  if (MODE == 3) {
    float acc[4][16];
    for (int i = 0; i < 4; ++i)
      for (int q = 0; q < 16; ++q) acc[i][q] = (float)(i + q);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[i][q] = fmaf(a[i], c[q], acc[i][q]);
    }
    for (int i = 0; i < 4; ++i)
      for (int q = 0; q < 16; ++q) s += acc[i][q];
  } else {
    uint64_t acc[4][8];
    for (int i = 0; i < 4; ++i)
      for (int q = 0; q < 8; ++q) acc[i][q] = pack((float)i, (float)q);
    uint64_t cp[8], a2[4];
    for (int q = 0; q < 8; ++q) cp[q] = MODE == 2 ? pack(c[q], c[q]) : pack(c[2 * q], c[2 * q + 1]);
    for (int i = 0; i < 4; ++i) a2[i] = MODE == 0 ? pack(a[i], a[i]) : pack(a[i], a[(i + 1) & 3] * 1.5f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[i][q] = ffma2(a2[i], cp[q], acc[i][q]);
    }
    for (int i = 0; i < 4; ++i)
      for (int q = 0; q < 8; ++q) s += __uint_as_float((uint32_t)acc[i][q]) + __uint_as_float((uint32_t)(acc[i][q] >> 32));
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// MIX: every FFMA2 (or FFMA pair) is followed by NA independent integer ALU ops (LOP3 / IADD3 on
// 8 private chains): does an FFMA2 hold the issue port for its 2 pipe cycles, or can ALU
// instructions issue in its shadow?
template <int NA, bool PAIRED>
__global__ void __launch_bounds__(256, 2) kmix(int iters, const float* in, float* out, long long* cyc) {
  float a[4], c[16];
  for (int i = 0; i < 4; ++i) a[i] = in[i + threadIdx.x % 3];
  for (int i = 0; i < 16; ++i) c[i] = in[8 + i + threadIdx.x % 5];
  uint32_t z[8];
  for (int i = 0; i < 8; ++i) z[i] = threadIdx.x * 2654435761u + i;
  const uint32_t zk = __float_as_uint(in[40]), zk2 = __float_as_uint(in[41]);
  uint64_t acc[4][8], cp[8], a2[4];
  float fa[4][16];
  for (int i = 0; i < 4; ++i)
    for (int q = 0; q < 8; ++q) acc[i][q] = pack((float)i, (float)q);
  for (int i = 0; i < 4; ++i)
    for (int q = 0; q < 16; ++q) fa[i][q] = (float)(i + q);
  for (int q = 0; q < 8; ++q) cp[q] = pack(c[2 * q], c[2 * q + 1]);
  for (int i = 0; i < 4; ++i) a2[i] = pack(a[i], a[i]);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (PAIRED) acc[i][q] = ffma2(a2[i], cp[q], acc[i][q]);
        else {
          asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(fa[i][2 * q]) : "f"(a[i]), "f"(c[2 * q]));
          asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(fa[i][2 * q + 1]) : "f"(a[i]), "f"(c[2 * q + 1]));
        }
#pragma unroll
        for (int n = 0; n < NA; ++n)
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(z[(q + n) & 7]) : "r"(zk), "r"(zk2));
      }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 4; ++i)
    for (int q = 0; q < 8; ++q) s += __uint_as_float((uint32_t)acc[i][q]) + __uint_as_float((uint32_t)(acc[i][q] >> 32));
  for (int i = 0; i < 4; ++i)
    for (int q = 0; q < 16; ++q) s += fa[i][q];
  for (int i = 0; i < 8; ++i) s += (float)z[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int NA, bool PAIRED>
void runmix(const char* name) {
  float *in, *out;
  long long* cyc;
  cudaMalloc(&in, 64 * 4);
  cudaMalloc(&out, 296 * 256 * 4);
  cudaMalloc(&cyc, 296 * 8);
  float h[64];
  for (int i = 0; i < 64; ++i) h[i] = 1.0f + 1e-3f * i;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  const int iters = 2048;
  kmix<NA, PAIRED><<<296, 256>>>(iters, in, out, cyc);
  kmix<NA, PAIRED><<<296, 256>>>(iters, in, out, cyc);
  cudaDeviceSynchronize();
  long long hc[296];
  cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 296; ++i) avg += hc[i];
  avg /= 296;
  // per SMSP: 4 warps x iters x 32 (FFMA2 | FFMA pair) groups
  printf("%-44s %.2f clk per (64 FMA + %d ALU) per SMSP\n", name, avg / (4.0 * iters * 32), NA);
}

template <int MODE>
void run(const char* name) {
  float *in, *out;
  long long* cyc;
  cudaMalloc(&in, 64 * 4);
  cudaMalloc(&out, 296 * 256 * 4);
  cudaMalloc(&cyc, 296 * 8);
  float h[64];
  for (int i = 0; i < 64; ++i) h[i] = 1.0f + 1e-3f * i;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  const int iters = 2048;
  k<MODE><<<296, 256>>>(iters, in, out, cyc);
  k<MODE><<<296, 256>>>(iters, in, out, cyc);
  cudaDeviceSynchronize();
  long long hc[296];
  cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 296; ++i) avg += hc[i];
  avg /= 296;
  // 2 CTAs of 256 threads per SM: 512 threads x 64 FMAs per iteration
  printf("%-44s %.1f FMA/clk/SM\n", name, (double)iters * 64 * 512 / avg);
}

int main() {
  run<0>("FFMA2 (a,a) scalar-broadcast multiplicand");
  run<1>("FFMA2 (a,a') 64-bit multiplicand");
  run<2>("FFMA2 pixel pairs x (p,p)");
  run<3>("FFMA scalar");
  runmix<0, true>("FFMA2 alone");
  runmix<1, true>("FFMA2 + 1 LOP3");
  runmix<2, true>("FFMA2 + 2 LOP3");
  runmix<3, true>("FFMA2 + 3 LOP3");
  runmix<0, false>("2 FFMA alone");
  runmix<1, false>("2 FFMA + 1 LOP3");
  runmix<2, false>("2 FFMA + 2 LOP3");
  return 0;
}
