// append.cuh — KV append of the decode step, fused into
// the attention launch: this step's K/V rows of the n query tokens go into the
// per-sample decode caches at positions lens[i] .. lens[i] + n - 1 (the
// "+K_prev" rows of the per-step KV accounting, Table 5 :982-987;
// SPEC.md:214-222) by the SAME CTA that later reads the tile holding them:
//   * tensor-core kernels (TMA reads): the CTA owning the decode tile (fused
//     kernel) or the decode item (rows kernel) stores the rows with generic
//     stores, then fence.proxy.async.global, then issues its TMA loads;
//   * CUDA-core kernel (generic loads): items read the new rows straight from
//     k_new / v_new, and the row-block-0 item of the split holding a row
//     stores it for the next steps.
// No other CTA reads a written row in this step, so no grid-wide ordering is
// needed and the append costs no launch.  lens[i] is clamped to [0, md_cap]
// (as everywhere on the device); a row whose position would reach md_cap is
// dropped (the device cannot report errors).
#pragma once
#include "common.cuh"

namespace ba {

struct AppendSrc {
  const void* k_new;  // [b][g][n][d] (cache element type)
  const void* v_new;
  void* Kd;           // [b][g][dec_cap][d]
  void* Vd;
  int n;              // rows per (sample, group); 0 = no append in this call
  int row_bytes;      // d * element bytes (a multiple of 16)
  int dec_cap;        // md_cap = the position stride of Kd / Vd
  int g;
};

BA_DEVINL void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// One warp stores the appended rows of (sample i, group c) whose positions lie
// in [p0, p1); L0 = the clamped cache length before the step.  which: 1 = K,
// 2 = V, 3 = both.
BA_DEVINL void append_rows_warp(const AppendSrc& A, int i, int c, int L0, int p0, int p1, int lane,
                                int which = 3) {
  const int lo = max(L0, p0);
  const int hi = min(min(L0 + A.n, A.dec_cap), p1);
  const int vpr = A.row_bytes >> 4;  // 16-byte vectors per row
  for (int pos = lo; pos < hi; ++pos) {
    const size_t ic = (size_t)i * A.g + c;
    const size_t src = (ic * A.n + (pos - L0)) * vpr;
    const size_t dst = (ic * A.dec_cap + pos) * vpr;
    if (which & 1)
      for (int e = lane; e < vpr; e += 32)
        reinterpret_cast<uint4*>(A.Kd)[dst + e] = reinterpret_cast<const uint4*>(A.k_new)[src + e];
    if (which & 2)
      for (int e = lane; e < vpr; e += 32)
        reinterpret_cast<uint4*>(A.Vd)[dst + e] = reinterpret_cast<const uint4*>(A.v_new)[src + e];
  }
}

BA_DEVINL int clamp_len(const int32_t* lens, int i, int cap) {
  const int L = lens[i];
  return L < 0 ? 0 : (L > cap ? cap : L);
}

}  // namespace ba
