// FFMA vs FFMA2 (fma.rn.f32x2) throughput per SM: independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ffma2_bench.bin tools/ffma2_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

template <int CH, bool PAIR>
__global__ void k(int iters, float x, float* out, long long* cyc) {
  long long t0 = clock64();
  if (PAIR) {
    uint64_t acc[CH];
    uint64_t a = ((uint64_t)__float_as_uint(x) << 32) | __float_as_uint(x * 0.5f);
    for (int i = 0; i < CH; ++i) acc[i] = a + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < CH; ++i) acc[i] = ffma2(acc[i], a, a);
    float s = 0;
    for (int i = 0; i < CH; ++i) s += __uint_as_float((uint32_t)acc[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  } else {
    float acc[CH];
    for (int i = 0; i < CH; ++i) acc[i] = x + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < CH; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(acc[i]) : "f"(x), "f"(acc[CH - 1 - i]));
    float s = 0;
    for (int i = 0; i < CH; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int CH, bool PAIR>
void run(int threads) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  k<CH, PAIR><<<148, threads>>>(iters, 1.0001f, out, cyc);
  k<CH, PAIR><<<148, threads>>>(iters, 1.0001f, out, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double fma = (double)iters * CH * threads * (PAIR ? 2 : 1);
  printf("%s chains=%d threads=%4d: %.1f FMA/clk/SM\n", PAIR ? "FFMA2" : "FFMA ", CH, threads, fma / avg);
}

int main() {
  for (int t : {128, 256, 512, 1024}) {
    run<8, false>(t);
    run<8, true>(t);
  }
  run<4, true>(256);
  run<16, true>(256);
  return 0;
}
