// Shared device helpers for the sm_100a LUT kernels: status plumbing, PTX
// wrappers for mbarrier / TMA / bulk copies, and small numeric helpers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>

#include "../../include/lutgpu.h"

namespace lutgpu {

// ----------------------------------------------------------------- host side

void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
int num_sms();
size_t max_smem_optin();
// once per (kernel, device): dynamic SMEM limit raised to the device maximum
cudaError_t kernel_smem_attr(const void* func);
// cached cudaOccupancyMaxActiveBlocksPerMultiprocessor
int kernel_occupancy(const void* func, int threads, size_t smem);

// Tuning / ablation knobs (LUTGPU_OH_*, LUTGPU_ENC_*, ...) are read only in
// probe builds (-DLUTGPU_PROBES, tools/build_probes.sh); the product build never
// consults the environment on a call path.
inline const char* probe_env(const char* name) {
#ifdef LUTGPU_PROBES
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

#define LUT_CHECK_LAUNCH(where)                              \
  do {                                                       \
    cudaError_t _e = cudaGetLastError();                     \
    if (_e != cudaSuccess) return ::lutgpu::cuda_fail(_e, where); \
  } while (0)

// Encodes a 2-D row-major f32 tensor map (cols x rows, 128B swizzle) via the
// driver entry point, so the library needs no link-time libcuda dependency.
bool make_tmap_2d_f32(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                      uint32_t box_cols, uint32_t box_rows, bool swizzle128);
// f32 2-D map whose box inner size (floats) picks the matching swizzle:
// 32 -> 128B, 16 -> 64B, 8 -> 32B, 4 -> none (TMA-store epilogues).
bool make_tmap_2d_f32_box(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint32_t box_cols,
                          uint32_t box_rows);
bool make_tmap_2d_u8(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows,
                     uint64_t row_stride_bytes, uint32_t box_cols, uint32_t box_rows,
                     bool swizzle128);

// prepared codebook record (floats): [K*V centroids][K norms][pmax][pad to 4]
// and, for the tensor-core encode shapes (V = 32, K = 16 or 64), a tf32 operand tile
// of the centroids in the 128B-swizzled K-major layout (chunk j of centroid k
// at k*32 + 4*(j ^ (k & 7)) floats) followed by 2^-7 max_k |p_k| rounded up
// (and K-1 zero floats).
__host__ __device__ inline int prep_base(int k, int v) { return ((k * v + k + 1) + 3) & ~3; }
__host__ __device__ inline bool prep_has_tc(int k, int v) { return (k == 16 || k == 64) && v == 32; }
__host__ __device__ inline int prep_stride(int k, int v) { return prep_base(k, v) + (prep_has_tc(k, v) ? k * v + k : 0); }

// ---------------------------------------------------------------- device side

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// try_wait with a suspend-time hint: the waiting thread sleeps until the phase
// completes (or the hint elapses) instead of spinning on issue slots that the
// co-resident producer / generator / epilogue warps need.
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_sleep(bar, parity)) {
  }
}

// TMA 2-D tile load global -> shared, completion counted on `bar`.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t x,
                                            int32_t y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// L2 eviction-priority hints for the streaming operands of the configs[4] layer: the
// encode's input and the gather's output are touched once (evict_first), the code tiles
// are re-read once per n-tile of a band (evict_last), so the 17 GB streams do not push
// the band's codes and the table image out of the 126 MB L2.
#ifndef LUTGPU_L2_HINTS
#define LUTGPU_L2_HINTS 1
#endif
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int32_t x, int32_t y,
                                                 uint64_t* bar, uint64_t policy) {
#if LUTGPU_L2_HINTS
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
#else
  (void)policy;
  tma_load_2d(dst, map, x, y, bar);
#endif
}

// 1-D bulk copy global -> shared (16B-aligned, size multiple of 16).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_load_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                               uint64_t policy) {
#if LUTGPU_L2_HINTS
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
#else
  (void)policy;
  bulk_load(dst, src, bytes, bar);
#endif
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Programmatic dependent launch: the primary lets its dependent grid launch
// early; the dependent waits for the primary's completion (and memory) here.
// Both are no-ops for launches without a programmatic dependency.
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void named_barrier_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Exact-erf GELU in f32 (extension epilogue; the reference has ReLU only).
__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
}

__device__ __forceinline__ float apply_act(float x, int act) {
  if (act == LUT_ACT_RELU) return fmaxf(x, 0.0f);  // np.maximum(x, 0)
  if (act == LUT_ACT_GELU) return gelu_erf(x);
  return x;
}

}  // namespace lutgpu
