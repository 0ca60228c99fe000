// Exactness helpers shared by the CUDA-core encoders (encode.cu) and the fused
// small-layer kernel (gather.cu): the fp32 near-tie bound and the literal f64
// re-decision with encode_hard semantics (lutkit/pq.py:171-174).
#pragma once

#include <float.h>

#include "common.cuh"

namespace lutgpu {

__device__ __forceinline__ float tau_coef(int v) { return (4.0f * v + 16.0f) * 5.9604645e-8f; }

// Literal f64 re-decision (encode_hard semantics) for one (row, codebook).
template <class GetA>
__device__ __noinline__ int exact_argmin(GetA get_a, const float* __restrict__ cent, int K, int V) {
  double best = 0.0;
  int bi = 0;
  for (int k = 0; k < K; ++k) {
    double s = 0.0;
    for (int j = 0; j < V; ++j) {
      double diff = (double)get_a(j) - (double)cent[k * V + j];
      s = __dadd_rn(s, __dmul_rn(diff, diff));
    }
    if (k == 0 || s < best) {
      best = s;
      bi = k;
    }
  }
  return bi;
}

// Exact code of one (row, codebook) from fp32 distances d_k = |p_k|^2 - 2 a.p_k
// (a held in registers, VT >= V), re-decided in f64 when the best two are within
// the fp32 error bound tau_coef(V) * (|a|^2 + max|p|^2).  cb = the prepared
// record [K x V centroids][K norms][max norm] (SMEM).
template <int VT, class GetA>
__device__ __forceinline__ int encode_one(GetA get_a, const float* cb, int K, int V, int* near_tie, bool count) {
  const float* norms = cb + K * V;
  float a[VT];
  float asq = 0.0f;
#pragma unroll
  for (int j = 0; j < VT; ++j) {
    const float x = (j < V) ? get_a(j) : 0.0f;
    asq = fmaf(x, x, asq);
    a[j] = -2.0f * x;
  }
  float best = FLT_MAX, second = FLT_MAX;
  int bi = 0;
  for (int k = 0; k < K; ++k) {
    float acc0 = norms[k], acc1 = 0.0f;
    const float* pkv = cb + k * V;
#pragma unroll
    for (int j = 0; j < VT; ++j) {
      if (j < V) {
        if (j & 1) acc1 = fmaf(a[j], pkv[j], acc1);
        else acc0 = fmaf(a[j], pkv[j], acc0);
      }
    }
    const float d = acc0 + acc1;
    second = fminf(second, fmaxf(best, d));
    bi = (d < best) ? k : bi;
    best = fminf(best, d);
  }
  if (!(second - best > tau_coef(V) * (asq + norms[K]))) {
    bi = exact_argmin(get_a, cb, K, V);
    if (near_tie && count) atomicAdd(near_tie, 1);
  }
  return bi;
}

}  // namespace lutgpu
