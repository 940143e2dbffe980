// fma_partial.cuh — CUDA-core (FMA) split-K partial attention kernel.
//
// Used where too few query rows share a KV tile to fill a tensor-core tile
// (SURVEY §8(d) "FMA vs tcgen05 rule"): the decode branch when p = h/g < 16
// (MHA, GQA), every branch of fp32 problems (kind::tf32 would break the 1e-5
// bound, reading R13), and bf16 context branches with b*p < 16 rows.
//
// A work item is (group c, a block of <= RB query rows that share one KV
// sequence, a key range [t0, t1) of that sequence, an output slot).  The
// context branch's sequence is Kc[c] (no batch axis, Eq. 3), the
// decode branch's is Kd[i][c].  The item's online-softmax
// partial (m, l, o) per row — m in log2 units, o unnormalised — goes to the
// fp32 workspace slot; merge.cuh joins the slots with one log-sum-exp, the
// exact form of the single softmax over S_c ⊕ S_d.
//
// Thread mapping: 16 lanes per key (lane j owns elements (c*16 + j)*LW .. +LW
// of each row, so each 16-lane load is one coalesced 16*LW-element segment);
// a warp processes 2 keys per step, U steps per iteration, 4 warps per CTA
// cover 8*U consecutive keys per iteration.  Each (warp, half-warp) keeps its
// own running (m, l, o) for its keys; the 8 streams are merged in shared
// memory at the end of the item.
#pragma once
#include "append.cuh"
#include "common.cuh"

namespace ba {

struct FmaParams {
  const void* q;
  const void* Kc;
  const void* Vc;
  const void* Kd;
  const void* Vd;
  const int32_t* lens;
  int b, h, g, p, mc;
  int dec_stride;   // position stride of Kd/Vd (md_cap, or mc+md_cap for the replicated baseline)
  int dec_cap;      // clamp for lens[i]
  int lens_offset;  // decode valid length = lens_offset + clamp(lens[i], 0, dec_cap)
  int lens_add;     // append+attend: valid decode length min(lens[i] + lens_add, dec_cap)
  int ntok;         // tokens per head (multi-token step): token k of a row group sees
                    // decode positions < max(L - (ntok - 1 - k), lens_offset)
  float scale_log2; // scale * log2(e)
  int nsc, nsd;     // context / decode splits per row (nsc = 0: no context branch)
  int ctx_chunk, dec_chunk;  // keys per split
  int nrb_c, nrb_d;          // row blocks per context group / per decode (sample, group)
  int n_ctx_items;           // g * nsc * nrb_c
  int S;                     // slots per output row (>= nsc + nsd; tc context may use more)
  int dec_slot0;             // first slot index of the decode splits
  float* ws_o;               // [b*h][S][D]
  float* ws_ml;              // [b*h][S][2]  (m in log2 units, l)
  AppendSrc app;             // append+attend (app.n > 0): decode items read positions >= the
                             // old length from k_new / v_new; row block 0 stores them
};

template <typename T>
struct Vec;  // per-element-type load helpers

template <>
struct Vec<__nv_bfloat16> {
  static constexpr int kVecElems = 8;
  // Load LW bf16 elements (LW in {1,2,4,8}) and widen to fp32.
  template <int LW>
  static BA_DEVINL void load(const __nv_bfloat16* p, float* out) {
    if constexpr (LW == 8) {
      uint4 r = ldg_stream(p);
      out[0] = bf16lo(r.x); out[1] = bf16hi(r.x); out[2] = bf16lo(r.y); out[3] = bf16hi(r.y);
      out[4] = bf16lo(r.z); out[5] = bf16hi(r.z); out[6] = bf16lo(r.w); out[7] = bf16hi(r.w);
    } else if constexpr (LW == 4) {
      uint2 r = ldg_stream8(p);
      out[0] = bf16lo(r.x); out[1] = bf16hi(r.x); out[2] = bf16lo(r.y); out[3] = bf16hi(r.y);
    } else if constexpr (LW == 2) {
      uint32_t r = ldg_stream4(p);
      out[0] = bf16lo(r); out[1] = bf16hi(r);
    } else {
      out[0] = __bfloat162float(*p);
    }
  }
};

template <>
struct Vec<float> {
  static constexpr int kVecElems = 4;
  template <int LW>
  static BA_DEVINL void load(const float* p, float* out) {
    if constexpr (LW == 4) {
      uint4 r = ldg_stream(p);
      out[0] = __uint_as_float(r.x); out[1] = __uint_as_float(r.y);
      out[2] = __uint_as_float(r.z); out[3] = __uint_as_float(r.w);
    } else if constexpr (LW == 2) {
      uint2 r = ldg_stream8(p);
      out[0] = __uint_as_float(r.x); out[1] = __uint_as_float(r.y);
    } else {
      out[0] = __uint_as_float(ldg_stream4(p));
    }
  }
};

// FP8 E4M3 cache codes (f4, reading R19): loads decode two codes per
// cvt.rn.f16x2.e4m3x2 (exact: every E4M3 value is an f16 normal or zero)
// and widen to fp32; the per-tensor scales are applied outside (k_scale in
// the logit scale, v_scale in the merge).
struct e4m3_t {
  uint8_t bits;
};

BA_DEVINL void e4m3x2_to_f32(uint32_t two_codes, float& lo, float& hi) {
  const uint32_t h2 = e4m3x2_to_f16x2(two_codes);
  lo = __half2float(__ushort_as_half((unsigned short)(h2 & 0xffffu)));
  hi = __half2float(__ushort_as_half((unsigned short)(h2 >> 16)));
}

template <>
struct Vec<e4m3_t> {
  static constexpr int kVecElems = 16;
  template <int LW>
  static BA_DEVINL void load(const e4m3_t* p, float* out) {
    if constexpr (LW == 8) {
      const uint2 r = ldg_stream8(p);
      e4m3x2_to_f32(r.x, out[0], out[1]);
      e4m3x2_to_f32(r.x >> 16, out[2], out[3]);
      e4m3x2_to_f32(r.y, out[4], out[5]);
      e4m3x2_to_f32(r.y >> 16, out[6], out[7]);
    } else if constexpr (LW == 4) {
      const uint32_t r = ldg_stream4(p);
      e4m3x2_to_f32(r, out[0], out[1]);
      e4m3x2_to_f32(r >> 16, out[2], out[3]);
    } else if constexpr (LW == 2) {
      const uint32_t r = *reinterpret_cast<const unsigned short*>(p);
      e4m3x2_to_f32(r, out[0], out[1]);
    } else {
      float unused;
      e4m3x2_to_f32(p->bits, out[0], unused);
    }
  }
};

// T: element type of q (and out); TK: element type of the KV cache.  Lane j
// owns elements (ch*16 + j)*LW .. +LW of a row in both, so LW is the smaller
// vector width of the two.
template <typename T, int D, int RB, typename TK = T>
struct FmaCfg {
  static constexpr int kThreads = 128;
  static constexpr int kEPL = D / 16;  // elements per lane per row
  static constexpr int kVW = Vec<T>::kVecElems < Vec<TK>::kVecElems ? Vec<T>::kVecElems
                                                                     : Vec<TK>::kVecElems;
  static constexpr int kLW = kVW < kEPL ? kVW : kEPL;
  static constexpr int kNCH = kEPL / kLW;  // loads per row per lane
  static constexpr int kU = 4;             // key steps per warp per iteration
  static constexpr int kKeysPerIter = 4 * 2 * kU;
  static_assert(D % 16 == 0, "D must be a multiple of 16");
};

template <typename T, int D, int RB, typename TK = T>
__global__ void __launch_bounds__(128) fma_partial_kernel(const FmaParams P) {
  using C = FmaCfg<T, D, RB, TK>;
  constexpr int EPL = C::kEPL, LW = C::kLW, NCH = C::kNCH, U = C::kU;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lg = lane >> 4, j = lane & 15;

  // ---- decode the work item --------------------------------------------
  int it = blockIdx.x;
  int c, r_begin, r_end, t0, t1, slot, row_base;  // rows r -> (r/p)*h + c*p + r%p
  int dec_L = -1, dec_r0 = 0;  // decode item: valid length, first row of the sample
  int app_L0 = 1 << 30;        // append+attend: keys >= app_L0 come from k_new / v_new
  const TK* Kn = nullptr;
  const TK* Vn = nullptr;
  const TK* Kb;
  const TK* Vb;
  if (it < P.n_ctx_items) {
    const int rb = it % P.nrb_c;
    const int s = (it / P.nrb_c) % P.nsc;
    c = it / (P.nrb_c * P.nsc);
    const int R = P.b * P.p;
    r_begin = rb * RB;
    r_end = min(R, r_begin + RB);
    t0 = s * P.ctx_chunk;
    t1 = min(P.mc, t0 + P.ctx_chunk);
    Kb = reinterpret_cast<const TK*>(P.Kc) + (size_t)c * P.mc * D;
    Vb = reinterpret_cast<const TK*>(P.Vc) + (size_t)c * P.mc * D;
    slot = s;
    row_base = 0;
  } else {
    it -= P.n_ctx_items;
    const int rb = it % P.nrb_d;
    const int s = (it / P.nrb_d) % P.nsd;
    const int ic = it / (P.nrb_d * P.nsd);
    c = ic % P.g;
    const int i = ic / P.g;
    int L = P.lens[i];
    L = L < 0 ? 0 : (L > P.dec_cap ? P.dec_cap : L);
    L = min(L + P.lens_add, P.dec_cap);
    L += P.lens_offset;
    dec_L = L;
    dec_r0 = i * P.p;
    r_begin = i * P.p + rb * RB;
    r_end = min(i * P.p + P.p, r_begin + RB);
    t0 = s * P.dec_chunk;
    t1 = min(L, t0 + P.dec_chunk);
    const size_t base = ((size_t)i * P.g + c) * P.dec_stride * D;
    Kb = reinterpret_cast<const TK*>(P.Kd) + base;
    Vb = reinterpret_cast<const TK*>(P.Vd) + base;
    slot = P.dec_slot0 + s;
    if (P.app.n > 0) {
      const int L0 = clamp_len(P.lens, i, P.dec_cap);
      app_L0 = P.lens_offset + L0;
      const size_t nb = ((size_t)i * P.g + c) * P.app.n * D;
      Kn = reinterpret_cast<const TK*>(P.app.k_new) + nb - (size_t)app_L0 * D;
      Vn = reinterpret_cast<const TK*>(P.app.v_new) + nb - (size_t)app_L0 * D;
      // the row-block-0 item of the split holding a new row stores it (for the
      // next steps; nobody reads it from Kd / Vd in this one)
      if (rb == 0 && warp == 0) append_rows_warp(P.app, i, c, L0, t0, t1, lane);
    }
    row_base = 0;
  }
  (void)row_base;
  const int nrows = r_end - r_begin;

  // ---- query rows to registers, pre-scaled into log2 units --------------
  float qr[RB][NCH][LW];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    const int rr = r_begin + r;
    if (r < nrows) {
      const int gr = (rr / P.p) * P.h + c * P.p + (rr % P.p);
      const T* qp = reinterpret_cast<const T*>(P.q) + (size_t)gr * D;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        Vec<T>::template load<LW>(qp + (ch * 16 + j) * LW, qr[r][ch]);
#pragma unroll
        for (int e = 0; e < LW; ++e) qr[r][ch][e] *= P.scale_log2;
      }
    } else {
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int e = 0; e < LW; ++e) qr[r][ch][e] = 0.f;
    }
  }

  // per-row end of the valid keys: t1, or for a decode row the intra-step
  // causal bound of its token (multi-token step; ntok = 1: t1)
  int lim[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    lim[r] = t1;
    if (dec_L >= 0 && P.ntok > 1) {
      const int k = (r_begin + r - dec_r0) % P.ntok;
      lim[r] = min(t1, max(dec_L - (P.ntok - 1 - k), P.lens_offset));
    }
  }
  float m[RB], l[RB], o[RB][NCH][LW];
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    m[r] = kNegInf;
    l[r] = 0.f;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
      for (int e = 0; e < LW; ++e) o[r][ch][e] = 0.f;
  }

  // ---- stream keys --------------------------------------------------------
  for (int base = t0; base < t1; base += C::kKeysPerIter) {
    float kv[U][NCH][LW], vv[U][NCH][LW];
    int tk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      tk[u] = base + warp * (2 * U) + u * 2 + lg;
      if (tk[u] < t1) {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
          Vec<TK>::template load<LW>((tk[u] >= app_L0 ? Kn : Kb) + (size_t)tk[u] * D + (ch * 16 + j) * LW,
                                     kv[u][ch]);
      } else {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
          for (int e = 0; e < LW; ++e) kv[u][ch][e] = 0.f;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (tk[u] < t1) {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
          Vec<TK>::template load<LW>((tk[u] >= app_L0 ? Vn : Vb) + (size_t)tk[u] * D + (ch * 16 + j) * LW,
                                     vv[u][ch]);
      } else {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
          for (int e = 0; e < LW; ++e) vv[u][ch][e] = 0.f;
      }
    }
    // logits (log2 units) for each key and row, reduced over the 16 lanes
    float s[U][RB];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        float acc = 0.f;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
          for (int e = 0; e < LW; ++e) acc = fmaf(qr[r][ch][e], kv[u][ch][e], acc);
        s[u][r] = acc;
      }
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1)
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int r = 0; r < RB; ++r) s[u][r] += __shfl_xor_sync(0xffffffffu, s[u][r], off);
    // online softmax update, once per U keys
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      float mx = m[r];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (tk[u] >= lim[r]) s[u][r] = kNegInf;
        mx = fmaxf(mx, s[u][r]);
      }
      const float ms = (mx == kNegInf) ? 0.f : mx;
      const float alpha = ex2(m[r] - ms);
      float pu[U];
      float lsum = 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        pu[u] = ex2(s[u][r] - ms);
        lsum += pu[u];
      }
      l[r] = fmaf(l[r], alpha, lsum);
      m[r] = mx;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int e = 0; e < LW; ++e) {
          float acc = o[r][ch][e] * alpha;
#pragma unroll
          for (int u = 0; u < U; ++u) acc = fmaf(pu[u], vv[u][ch][e], acc);
          o[r][ch][e] = acc;
        }
    }
  }

  // ---- merge the 8 (warp, half-warp) streams in shared memory ----------
  __shared__ float sm_m[8][RB], sm_l[8][RB];
  __shared__ float sm_o[8][RB][D];
  const int stream = warp * 2 + lg;
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    if (j == 0) {
      sm_m[stream][r] = m[r];
      sm_l[stream][r] = l[r];
    }
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
      for (int e = 0; e < LW; ++e) sm_o[stream][r][(ch * 16 + j) * LW + e] = o[r][ch][e];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < nrows * D; idx += C::kThreads) {
    const int r = idx / D, x = idx % D;
    float M = kNegInf;
#pragma unroll
    for (int k = 0; k < 8; ++k) M = fmaxf(M, sm_m[k][r]);
    const float Ms = (M == kNegInf) ? 0.f : M;
    float L = 0.f, acc = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float w = ex2(sm_m[k][r] - Ms);
      L = fmaf(w, sm_l[k][r], L);
      acc = fmaf(w, sm_o[k][r][x], acc);
    }
    const int rr = r_begin + r;
    const int gr = (rr / P.p) * P.h + c * P.p + (rr % P.p);
    const size_t sl = (size_t)gr * P.S + slot;
    P.ws_o[sl * D + x] = acc;
    if (x == 0) {
      P.ws_ml[sl * 2 + 0] = M;
      P.ws_ml[sl * 2 + 1] = L;
    }
  }
}

}  // namespace ba
