// append.cuh — KV append of the decode step: write this
// step's K/V rows of the n query tokens into the per-sample decode caches at
// positions lens[i] .. lens[i] + n - 1 (the "+K_prev" rows of the per-step
// KV accounting, Table 5 :982-987), before the
// attention of the same step reads them.
//   k_new, v_new [b][g][n][d]  ->  Kd, Vd [b][g][md_cap][d]
// lens[i] is clamped to [0, md_cap] (as everywhere on the device); a row whose
// position would reach md_cap is dropped (the device cannot report errors).
// One 16-byte vector per thread and tensor: the copy is a few hundred KB and
// runs as the first launch of the append+attend call; the attention launch
// is programmatically dependent on it (PDL), so its prologue overlaps this.
#pragma once
#include "common.cuh"

namespace ba {

struct AppendParams {
  const void* k_new;
  const void* v_new;
  void* Kd;
  void* Vd;
  const int32_t* lens;
  int b, g, n, md_cap;
  int vec_per_row;  // 16-byte vectors per d-row = d * elem / 16
};

__global__ void __launch_bounds__(256) kv_append_kernel(const AppendParams P) {
  pdl_wait();  // the previous step (which may update lens) has completed
  const long long total = (long long)P.b * P.g * P.n * P.vec_per_row;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < total;
       v += (long long)gridDim.x * blockDim.x) {
    const long long row = v / P.vec_per_row;        // (i, c, k)
    const int e = (int)(v - row * P.vec_per_row);
    const int k = (int)(row % P.n);
    const long long ic = row / P.n;                 // i * g + c
    const int i = (int)(ic / P.g);
    int L = P.lens[i];
    L = L < 0 ? 0 : (L > P.md_cap ? P.md_cap : L);
    const int pos = L + k;
    if (pos >= P.md_cap) continue;
    const size_t dst = ((size_t)ic * P.md_cap + pos) * P.vec_per_row + e;
    reinterpret_cast<uint4*>(P.Kd)[dst] = reinterpret_cast<const uint4*>(P.k_new)[v];
    reinterpret_cast<uint4*>(P.Vd)[dst] = reinterpret_cast<const uint4*>(P.v_new)[v];
  }
  pdl_launch_dependents();
}

}  // namespace ba
