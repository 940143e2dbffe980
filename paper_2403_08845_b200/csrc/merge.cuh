// merge.cuh — join the per-split partials of one output row with one
// log-sum-exp and write the normalised result (SURVEY §8(a) a3 + a6).
//
// Partials k = (m_k, l_k, o_k) with m_k the running max in log2 units,
// l_k = sum 2^(s - m_k), o_k = sum 2^(s - m_k) v.  With M = max_k m_k:
//   L = sum_k 2^(m_k - M) l_k ;  out = (sum_k 2^(m_k - M) o_k) / L
//   lse = (M + log2 L) * ln 2
// which is softmax over the concatenation S_c ⊕ S_d,
// split at mc and summed (Eq. 4), in exact arithmetic.
// Empty partials carry m = -inf, l = 0, o = 0 and drop out.
#pragma once
#include "common.cuh"

namespace ba {

struct MergeParams {
  const float* ws_o;   // [rows][S][D]
  const float* ws_ml;  // [rows][S][2]
  int rows, S;
  int h, p;
  // context slots: mode 0 none, 1 fixed count nsc
  int ctx_mode, nsc;
  int dec_slot0, nsd;
  void* out;           // [rows][D] in T
  float* lse;          // [rows] or null
  int32_t* lens_out;   // append+attend: lens[i] <- min(clamp(lens[i]) + lens_add, dec_cap)
  int b, lens_add, dec_cap;
  float vscale;        // FP8 KV: partials are in V-code units, out = v_scale * o / L (else 1)
};

// Number of context partials written for output row gr.
BA_DEVINL int ctx_slots_of_row(const MergeParams& P, int gr) {
  (void)gr;
  return P.ctx_mode == 1 ? P.nsc : 0;
}

template <typename T, int D>
__global__ void __launch_bounds__(256) merge_kernel(const MergeParams P) {
  constexpr int EPL = (D + 31) / 32;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  pdl_wait();  // launched programmatically dependent on the partial kernel
  pdl_launch_dependents();
  // append+attend: the partial kernels (earlier launches) have read lens
  if (P.lens_out && blockIdx.x == 0)
    for (int i = threadIdx.x; i < P.b; i += blockDim.x) {
      int L = P.lens_out[i];
      L = L < 0 ? 0 : (L > P.dec_cap ? P.dec_cap : L);
      P.lens_out[i] = min(L + P.lens_add, P.dec_cap);
    }
  if (warp >= P.rows) return;
  const int nctx = ctx_slots_of_row(P, warp);
  const int ntot = nctx + P.nsd;
  // slot index of the k-th live partial
  auto slot_of = [&](int k) { return k < nctx ? k : P.dec_slot0 + (k - nctx); };
  const float* ml = P.ws_ml + (size_t)warp * P.S * 2;
  const float* o = P.ws_o + (size_t)warp * P.S * D;
  if constexpr (D == 128) {
    if (ntot <= 32) {
      // one load round trip: every lane's (m, l) of partial `lane` AND the
      // float4 slices (d = 4 lane ..) of the first 8 partials' rows go out
      // together; later batches of 8 (rare) follow
      const float2 mlk = lane < ntot ? __ldcg(reinterpret_cast<const float2*>(ml) + slot_of(lane))
                                     : make_float2(kNegInf, 0.f);
      float4 ov[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        ov[q] = q < ntot ? __ldcg(reinterpret_cast<const float4*>(o + (size_t)slot_of(q) * D) + lane)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      float M = mlk.x;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
      const float Ms = (M == kNegInf) ? 0.f : M;
      const float wl = lane < ntot ? ex2(mlk.x - Ms) : 0.f;
      float L = wl * mlk.y;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int k0 = 0; k0 < ntot; k0 += 8) {
        if (k0 > 0) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            ov[q] = k0 + q < ntot ? __ldcg(reinterpret_cast<const float4*>(o + (size_t)slot_of(k0 + q) * D) + lane)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float wq = __shfl_sync(0xffffffffu, wl, (k0 + q) & 31);
          if (k0 + q < ntot) {
            acc.x = fmaf(wq, ov[q].x, acc.x); acc.y = fmaf(wq, ov[q].y, acc.y);
            acc.z = fmaf(wq, ov[q].z, acc.z); acc.w = fmaf(wq, ov[q].w, acc.w);
          }
        }
      }
      const float invL = P.vscale / L;
      if constexpr (sizeof(T) == 2) {
        const uint2 packed = make_uint2(pack_bf16x2(acc.x * invL, acc.y * invL), pack_bf16x2(acc.z * invL, acc.w * invL));
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(P.out) + (size_t)warp * D + 4 * lane) = packed;
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(P.out) + (size_t)warp * D + 4 * lane) =
            make_float4(acc.x * invL, acc.y * invL, acc.z * invL, acc.w * invL);
      }
      if (P.lse && lane == 0) P.lse[warp] = (M + lg2(L)) * kLn2;
      return;
    }
  }
  // (m, l) of up to 32 partials per round, one per lane: the row max and the
  // weights take one load round trip instead of one per partial
  float M = kNegInf;
  for (int k0 = 0; k0 < ntot; k0 += 32) {
    const int k = k0 + lane;
    const float mk = k < ntot ? ml[2 * slot_of(k)] : kNegInf;
    M = fmaxf(M, mk);
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
  const float Ms = (M == kNegInf) ? 0.f : M;
  float acc[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) acc[e] = 0.f;
  float L = 0.f;
  for (int k0 = 0; k0 < ntot; k0 += 32) {
    const int kl = k0 + lane;
    float wl = 0.f;
    if (kl < ntot) {
      const int s = slot_of(kl);
      wl = ex2(ml[2 * s] - Ms);
      L = fmaf(wl, ml[2 * s + 1], L);
    }
    const int nk = min(32, ntot - k0);
    // value rows 4 partials at a time: all loads of a batch before any use
    for (int kb = 0; kb < nk; kb += 4) {
      float ov[4][EPL];
      float wk[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        wk[q] = __shfl_sync(0xffffffffu, wl, (kb + q) & 31);
        const int k = k0 + kb + q;
        const float* os = o + (size_t)slot_of(k < ntot ? k : k0) * D;
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const int x = e * 32 + lane;
          ov[q][e] = (kb + q < nk && x < D) ? __ldcg(os + x) : 0.f;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[e] = fmaf(kb + q < nk ? wk[q] : 0.f, ov[q][e], acc[e]);
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) L += __shfl_xor_sync(0xffffffffu, L, off);
  const float invL = P.vscale / L;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const int x = e * 32 + lane;
    if (x < D) {
      const float v = acc[e] * invL;
      if constexpr (sizeof(T) == 2) {
        reinterpret_cast<__nv_bfloat16*>(P.out)[(size_t)warp * D + x] = __float2bfloat16_rn(v);
      } else {
        reinterpret_cast<float*>(P.out)[(size_t)warp * D + x] = v;
      }
    }
  }
  if (P.lse && lane == 0) P.lse[warp] = (M + lg2(L)) * kLn2;
}

}  // namespace ba
