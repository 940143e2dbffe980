// lse_merge.cuh — join n_parts normalised partial results of the same rows
// (each the attention of a row over a DISJOINT slice of its keys, with its
// natural-log LSE) into the attention over the union of the slices:
//   M = max_k lse_k,  w_k = e^(lse_k - M),
//   out = sum_k w_k out_k / sum_k w_k,   lse = M + ln sum_k w_k.
// This is the "+" of Eq. 4 (App. E.3 splits the softmax at mc,
// PAPER.md:1170-1181) applied across ranks: the cross-GPU context split of
// SURVEY §8(f) row f3 (each rank attends to an mc slice; TP FAQ PAPER.md:
// 701-702).  A part with lse = -inf (no keys) contributes nothing.
// One warp per row; d / 32 elements per lane; inputs in the problem dtype.
#pragma once
#include "common.cuh"

namespace ba {

BA_DEVINL float to_float(float x) { return x; }
BA_DEVINL float to_float(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T>
BA_DEVINL T from_float(float x);
template <>
BA_DEVINL float from_float<float>(float x) { return x; }
template <>
BA_DEVINL __nv_bfloat16 from_float<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

struct LseMergeParams {
  const void* out_parts;  // [n_parts][rows][d]
  const float* lse_parts; // [n_parts][rows]
  void* out;              // [rows][d]
  float* lse;             // [rows] or null
  int n_parts, rows, d;
};

template <typename T>
__global__ void __launch_bounds__(256) lse_merge_kernel(const LseMergeParams P) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= P.rows) return;
  float M = kNegInf;
  for (int k = 0; k < P.n_parts; ++k) M = fmaxf(M, P.lse_parts[(size_t)k * P.rows + row]);
  const float Ms = (M == kNegInf) ? 0.f : M;
  const T* op = reinterpret_cast<const T*>(P.out_parts);
  float Z = 0.f;
  float acc[8];  // d <= 256
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.f;
  for (int k = 0; k < P.n_parts; ++k) {
    const float w = expf(P.lse_parts[(size_t)k * P.rows + row] - Ms);
    Z += w;
    const T* src = op + ((size_t)k * P.rows + row) * P.d;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int x = e * 32 + lane;
      if (x < P.d) acc[e] = fmaf(w, to_float(src[x]), acc[e]);
    }
  }
  const float inv = 1.f / Z;
  T* dst = reinterpret_cast<T*>(P.out) + (size_t)row * P.d;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int x = e * 32 + lane;
    if (x < P.d) dst[x] = from_float<T>(acc[e] * inv);
  }
  if (P.lse && lane == 0) P.lse[row] = M + logf(Z);
}

}  // namespace ba
