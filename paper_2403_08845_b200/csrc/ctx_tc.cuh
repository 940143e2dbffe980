// ctx_tc.cuh — context branch of the bifurcated decode step on the 5th-gen
// tensor cores (tcgen05 + TMEM + TMA), sm_100a.
//
// What it computes (Eq. 3-4 context rows): for every
// KV group c, the R = b*p query rows that share Kc[c] / Vc[c] ("the axis b does
// not appear") against the whole shared context, producing one
// online-softmax partial (m, l, o) per row and per CTA segment.  Kc/Vc are
// streamed from HBM exactly once for the whole batch.
//
// Swap-AB formulation (rows are few, positions are many):
//   S^T[128 pos x N rows]  = Kc_tile[128 x d] . q_chunk^T[d x N]   (M=128, K=d)
//   O^T[d x N rows]       += Vc_tile^T[d x 128] . P^T[128 x N]      (M=d=128, K=128)
// so N = rows per chunk (16..128) is a legal MMA N even for R = 16 or 32.
// Kc/Vc tiles arrive by TMA (128B swizzle) into a NST-stage ring; S^T (double
// buffered) and O^T live in TMEM; P goes through shared memory (MN-major).
//
// Warp roles (12 warps): 0 = TMA producer, 1 = MMA issuer (one lane),
// 2 = TMEM allocator, 3 = idle, 4..11 = softmax/epilogue.  Softmax warp w
// reads TMEM lanes 32*(w%4).. (= positions of the tile, = d in the epilogue)
// and columns [half*CPT, half*CPT+CPT) with half = (w-4)/4, CPT = N/2.
//
// Online softmax with a stale-max fast path: P = 2^(s*scale*log2e - m_run)
// with the running per-row max m_run; only when some logit exceeds m_run by
// more than kTh (CTA-wide vote via bar.red.or) do the warps compute the exact
// tile max, rescale l and O^T (in TMEM) and raise m_run.  The result is the
// same softmax (m_run is only a reference point); values stay <= 2^kTh.
//
// Work split: flat tile index f = (c*nrc + rc)*ntile + t over (group, row
// chunk, 128-position tile); CTA k of G takes [k*T/G, (k+1)*T/G) — balanced
// to one tile.  A maximal run with one (c, rc) is a segment; each segment
// writes one partial to workspace slot k - owner(first tile of (c, rc)).
#pragma once
#include "common.cuh"
#include "tc_ptx.cuh"

namespace ba {

struct CtxTcParams {
  CUtensorMap tmK;  // Kc as 3D (d, mc, g), box (64, 128, 1), SW128
  CUtensorMap tmV;  // Vc, same
  CUtensorMap tmQ;  // q as 3D (d, h, b), box (64, p, N/p), SW128
  int b, h, g, p, mc;
  int nrc;          // row chunks per group
  int ntile;        // ceil(mc / 128)
  long long T;      // total tiles g*nrc*ntile
  int G;            // CTAs (gridDim.x)
  int nst;          // pipeline stages
  float scale_log2;
  int S;            // slots per row in the workspace
  float* ws_o;      // [b*h][S][128]
  float* ws_ml;     // [b*h][S][2]
};

namespace ctx {
constexpr int kThreads = 384;
constexpr int kD = 128;
constexpr int kBM = 128;              // positions per tile (MMA M)
constexpr int kStageBytes = 65536;    // K tile 32 KB + V tile 32 KB
constexpr float kTh = 8.0f;           // fast-path slack (log2 units)

__host__ __device__ constexpr int p_atom(int N) { return (N % 64 == 0) ? 64 : ((N % 32 == 0) ? 32 : 16); }
__host__ __device__ constexpr int p_layout(int N) {
  return p_atom(N) == 64 ? tc::kSw128 : (p_atom(N) == 32 ? tc::kSw64 : tc::kSw32);
}
__host__ __device__ constexpr int tmem_cols(int N) {
  return 3 * N <= 32 ? 32 : 3 * N <= 64 ? 64 : 3 * N <= 128 ? 128 : 3 * N <= 256 ? 256 : 512;
}
// dynamic smem: stages + q (256N) + 2 P buffers (256N each) + reduction scratch + barriers
__host__ __device__ constexpr int smem_fixed(int N) { return 3 * 256 * N + 2 * 2048 + 1024 + 256 + 1024; }

// owner CTA of flat tile f when T tiles are split over G CTAs as [kT/G, (k+1)T/G)
__host__ __device__ inline int owner(long long f, long long T, int G) {
  return (int)(((f + 1) * (long long)G - 1) / T);
}
}  // namespace ctx

// Load CPT consecutive TMEM columns (CPT a multiple of 8) into r[].
template <int CPT>
BA_DEVINL void tmem_ld_cols(uint32_t taddr, uint32_t* r) {
  int c = 0;
#pragma unroll
  for (; c + 32 <= CPT; c += 32) tc::tmem_ld<32>(taddr + c, r + c);
#pragma unroll
  for (; c + 16 <= CPT; c += 16) tc::tmem_ld<16>(taddr + c, r + c);
#pragma unroll
  for (; c + 8 <= CPT; c += 8) tc::tmem_ld<8>(taddr + c, r + c);
}

template <int N>
__global__ void __launch_bounds__(ctx::kThreads, 1)
    ctx_tc_kernel(const __grid_constant__ CtxTcParams P) {
  using namespace ctx;
  constexpr int CPT = N / 2;                 // columns per softmax thread
  constexpr int W = p_atom(N);               // P swizzle atom width (elements)
  constexpr int PRB = 2 * W;                 // P row bytes
  constexpr int PLBO = kBM * PRB;            // P stride between atoms
  constexpr int PSWM = W == 64 ? 7 : (W == 32 ? 3 : 1);
  constexpr uint32_t IDESC_QK = tc::idesc_bf16(128, N, 0, 0);
  constexpr uint32_t IDESC_PV = tc::idesc_bf16(128, N, 1, 1);
  constexpr uint32_t TMEM_COLS = tmem_cols(N);
  static_assert(N % 16 == 0 && N >= 16 && N <= 128, "N");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int NST = P.nst;
  uint8_t* sm_stage = smem;
  uint8_t* sm_q = smem + NST * kStageBytes;
  uint8_t* sm_p = sm_q + 256 * N;                       // 2 buffers of 256N bytes
  float* sm_red = reinterpret_cast<float*>(sm_p + 2 * 256 * N);  // [4][128] slow-path col max
  float* sm_l = sm_red + 4 * 128;                       // [4][128] epilogue row sums
  float* sm_mrun = sm_l + 4 * 128;                      // [2][128] running max (log2 units)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm_mrun + 256);
  uint64_t* kv_full = bars;
  uint64_t* kv_empty = bars + 8;
  uint64_t* q_full = bars + 16;
  uint64_t* q_empty = bars + 17;
  uint64_t* s_full = bars + 18;   // [2]
  uint64_t* s_free = bars + 20;   // [2]
  uint64_t* p_full = bars + 22;   // [2]
  uint64_t* p_empty = bars + 24;  // [2]
  uint64_t* o_full = bars + 26;
  uint64_t* o_empty = bars + 27;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 28);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      tc::mbar_init(tc::smem_u32(&kv_full[s]), 1);
      tc::mbar_init(tc::smem_u32(&kv_empty[s]), 1);
    }
    tc::mbar_init(tc::smem_u32(q_full), 1);
    tc::mbar_init(tc::smem_u32(q_empty), 1);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(tc::smem_u32(&s_full[s]), 1);
      tc::mbar_init(tc::smem_u32(&s_free[s]), 8);
      tc::mbar_init(tc::smem_u32(&p_full[s]), 8);
      tc::mbar_init(tc::smem_u32(&p_empty[s]), 1);
    }
    tc::mbar_init(tc::smem_u32(o_full), 1);
    tc::mbar_init(tc::smem_u32(o_empty), 8);
    tc::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&P.tmK);
    tc::prefetch_tmap(&P.tmV);
    tc::prefetch_tmap(&P.tmQ);
  }
  if (warp == 2) {
    tc::tmem_alloc(tc::smem_u32(tmem_holder), TMEM_COLS);
    tc::tmem_relinquish();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const uint32_t tS = tmem;            // S slots at columns [0,N) and [N,2N)
  const uint32_t tO = tmem + 2 * N;    // O^T at [2N, 3N)

  // this CTA's tile range
  const long long T = P.T;
  const int G = P.G;
  const long long f0 = (long long)blockIdx.x * T / G;
  const long long f1 = (long long)(blockIdx.x + 1) * T / G;
  const int ntile = P.ntile;

  if (warp == 0) {
    // ========================= TMA producer =========================
    if (lane == 0) {
      uint32_t tt = 0, sg = 0;
      const uint64_t pol_kv = P.nrc == 1 ? tc::policy_evict_first() : tc::policy_evict_last();
      for (long long f = f0; f < f1; ++sg) {
        const int seg = (int)(f / ntile);
        const long long fend = f1 < (long long)(seg + 1) * ntile ? f1 : (long long)(seg + 1) * ntile;
        const int c = seg / P.nrc, rc = seg % P.nrc;
        tc::mbar_wait(tc::smem_u32(q_empty), (sg & 1) ^ 1);
        tc::mbar_arrive_expect_tx(tc::smem_u32(q_full), 2 * N * 128);
        tc::tma_load_3d(tc::smem_u32(sm_q), &P.tmQ, tc::smem_u32(q_full), 0, c * P.p, rc * (N / P.p));
        tc::tma_load_3d(tc::smem_u32(sm_q + N * 128), &P.tmQ, tc::smem_u32(q_full), 64, c * P.p,
                        rc * (N / P.p));
        for (; f < fend; ++f, ++tt) {
          const int t = (int)(f % ntile);
          const int s = tt % NST;
          tc::mbar_wait(tc::smem_u32(&kv_empty[s]), ((tt / NST) & 1) ^ 1);
          const uint32_t bar = tc::smem_u32(&kv_full[s]);
          tc::mbar_arrive_expect_tx(bar, kStageBytes);
          const uint32_t dst = tc::smem_u32(sm_stage + s * kStageBytes);
          tc::tma_load_3d_hint(dst, &P.tmK, bar, 0, t * kBM, c, pol_kv);
          tc::tma_load_3d_hint(dst + 16384, &P.tmK, bar, 64, t * kBM, c, pol_kv);
          tc::tma_load_3d_hint(dst + 32768, &P.tmV, bar, 0, t * kBM, c, pol_kv);
          tc::tma_load_3d_hint(dst + 49152, &P.tmV, bar, 64, t * kBM, c, pol_kv);
        }
      }
    }
  } else if (warp == 1) {
    // ========================= MMA issuer ===========================
    if (lane == 0) {
      uint32_t tt = 0, u = 0, sg = 0;
      const uint32_t q_addr = tc::smem_u32(sm_q);
      const uint32_t p_addr = tc::smem_u32(sm_p);
      auto issue_pv = [&](uint32_t v, uint32_t stg, bool first) {
        if (first) tc::mbar_wait(tc::smem_u32(o_empty), (sg & 1) ^ 1);
        tc::mbar_wait(tc::smem_u32(&p_full[v & 1]), (v >> 1) & 1);
        tc::tc_fence_after();
        const uint32_t vbase = tc::smem_u32(sm_stage + stg * kStageBytes + 32768);
        const uint32_t pbase = p_addr + (v & 1) * 256 * N;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t ad = tc::smem_desc(vbase + k * 2048, 16384, 1024, tc::kSw128);
          const uint64_t bd = tc::smem_desc(pbase + k * 16 * PRB, PLBO, 8 * PRB, p_layout(N));
          tc::mma_bf16(tO, ad, bd, IDESC_PV, (first && k == 0) ? 0u : 1u);
        }
        tc::mma_commit(tc::smem_u32(&p_empty[v & 1]));
        tc::mma_commit(tc::smem_u32(&kv_empty[stg]));
      };
      for (long long f = f0; f < f1; ++sg) {
        const int seg = (int)(f / ntile);
        const long long fend = f1 < (long long)(seg + 1) * ntile ? f1 : (long long)(seg + 1) * ntile;
        tc::mbar_wait(tc::smem_u32(q_full), sg & 1);
        tc::tc_fence_after();
        const long long fstart = f;
        uint32_t prev_stage = 0;
        for (; f < fend; ++f, ++tt, ++u) {
          const uint32_t s = tt % NST;
          tc::mbar_wait(tc::smem_u32(&kv_full[s]), (tt / NST) & 1);
          const uint32_t slot = u & 1;
          tc::mbar_wait(tc::smem_u32(&s_free[slot]), ((u >> 1) & 1) ^ 1);
          tc::tc_fence_after();
          const uint32_t kbase = tc::smem_u32(sm_stage + s * kStageBytes);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t ad = tc::smem_desc(kbase + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, tc::kSw128);
            const uint64_t bd = tc::smem_desc(q_addr + (k >> 2) * (N * 128) + (k & 3) * 32, 16, 1024, tc::kSw128);
            tc::mma_bf16(tS + slot * N, ad, bd, IDESC_QK, k > 0 ? 1u : 0u);
          }
          tc::mma_commit(tc::smem_u32(&s_full[slot]));
          if (f + 1 == fend) tc::mma_commit(tc::smem_u32(q_empty));
          if (f > fstart) issue_pv(u - 1, prev_stage, f - 1 == fstart);
          prev_stage = s;
        }
        issue_pv(u - 1, prev_stage, fend - 1 == fstart);
        tc::mma_commit(tc::smem_u32(o_full));
      }
    }
  } else if (warp >= 4) {
    // ==================== softmax + epilogue (8 warps) ===================
    const int sw = warp - 4;
    const int quad = warp & 3;       // TMEM lane quadrant
    const int half = sw >> 2;        // column half
    const int col0 = half * CPT;
    const int pos = quad * 32 + lane;          // position within tile / d in epilogue
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    const float sl2 = P.scale_log2;
    const int R = P.b * P.p;
    uint32_t u = 0, sg = 0, cur = 0;  // cur: which sm_mrun buffer holds m_run
    for (long long f = f0; f < f1; ++sg) {
      const int seg = (int)(f / ntile);
      const long long fend = f1 < (long long)(seg + 1) * ntile ? f1 : (long long)(seg + 1) * ntile;
      const int c = seg / P.nrc, rc = seg % P.nrc;
      const long long fstart = f;
      float l_part[CPT];
#pragma unroll
      for (int n = 0; n < CPT; ++n) l_part[n] = 0.f;
      for (; f < fend; ++f, ++u) {
        const int t = (int)(f % ntile);
        const uint32_t slot = u & 1;
        const bool first = (f == fstart);
        const float* mrun = sm_mrun + cur * 128 + col0;
        tc::mbar_wait(tc::smem_u32(&s_full[slot]), (u >> 1) & 1);
        tc::tc_fence_after();
        float x[CPT];
        tmem_ld_cols<CPT>(tS + slot * N + col0 + lane_addr, reinterpret_cast<uint32_t*>(x));
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_free[slot]));
        const bool valid = t * kBM + pos < P.mc;
        // x = s*scale*log2e - mref ; mref = m_run (0 on the segment's first tile)
        float excess = kNegInf;
#pragma unroll
        for (int n = 0; n < CPT; ++n) {
          const float mref = first ? 0.f : mrun[n];
          x[n] = valid ? fmaf(x[n], sl2, -mref) : kNegInf;
          excess = fmaxf(excess, x[n]);
        }
        if (tc::named_bar_or(1, 256, first || excess > kTh)) {
          // ---- slow path: exact column max over the tile, new m_run, rescale ----
#pragma unroll
          for (int n = 0; n < CPT; ++n) {
            float v = x[n];
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
            if (lane == (n & 31)) sm_red[quad * 128 + col0 + n] = v;
          }
          tc::named_bar_sync(2, 256);
          float* mnext = sm_mrun + (cur ^ 1) * 128 + col0;
#pragma unroll
          for (int n = 0; n < CPT; ++n) {
            const int col = col0 + n;
            const float mref = first ? 0.f : mrun[n];
            const float tmax = mref + fmaxf(fmaxf(sm_red[col], sm_red[128 + col]),
                                            fmaxf(sm_red[256 + col], sm_red[384 + col]));
            const float mnew = first ? tmax : fmaxf(mrun[n], tmax);
            const float alpha = first ? 0.f : ex2(mrun[n] - mnew);
            l_part[n] *= alpha;
            x[n] += mref - mnew;  // -inf stays -inf
            if (quad == 0 && lane == 0) mnext[n] = mnew;
          }
          if (!first) {
            // O^T holds earlier tiles of this segment: wait for PV(u-1), rescale columns
            const uint32_t pv = u - 1;
            tc::mbar_wait(tc::smem_u32(&p_empty[pv & 1]), (pv >> 1) & 1);
            tc::tc_fence_after();
#pragma unroll
            for (int n = 0; n < CPT; n += 8) {
              uint32_t orr[8];
              tc::tmem_ld<8>(tO + col0 + n + lane_addr, orr);
              tc::tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 8; ++e)
                orr[e] = __float_as_uint(__uint_as_float(orr[e]) * ex2(mrun[n + e] - mnext[n + e]));
              tc::tmem_st<8>(tO + col0 + n + lane_addr, orr);
            }
            tc::tmem_st_wait();
            tc::tc_fence_before();
          }
          tc::named_bar_sync(2, 256);  // m_run(next) visible; m_run(cur) reads done
          cur ^= 1;
        }
        // ---- P = 2^x (bf16), per-position partial row sums ----
        tc::mbar_wait(tc::smem_u32(&p_empty[slot]), ((u >> 1) & 1) ^ 1);
        uint8_t* pbuf = sm_p + slot * 256 * N;
#pragma unroll
        for (int n = 0; n < CPT; n += 8) {
          uint32_t pk[4];
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const float p0 = ex2(x[n + e]), p1 = ex2(x[n + e + 1]);
            l_part[n + e] += p0;
            l_part[n + e + 1] += p1;
            pk[e / 2] = pack_bf16x2(p0, p1);
          }
          const int col = col0 + n;
          uint32_t off = (uint32_t)((col / W) * PLBO + pos * PRB + (col % W) * 2);
          off ^= ((off >> 7) & PSWM) << 4;
          *reinterpret_cast<uint4*>(pbuf + off) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(tc::smem_u32(&p_full[slot]));
      }
      // ---------------- segment epilogue ----------------
      // l: reduce over the 32 positions of this warp, then over the 4 quadrants
#pragma unroll
      for (int n = 0; n < CPT; ++n) {
        float v = l_part[n];
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == (n & 31)) sm_l[quad * 128 + col0 + n] = v;
      }
      const int slot_idx = blockIdx.x - ctx::owner((long long)seg * ntile, T, G);
      tc::mbar_wait(tc::smem_u32(o_full), sg & 1);
      tc::tc_fence_after();
#pragma unroll
      for (int n = 0; n < CPT; n += 8) {
        uint32_t orr[8];
        tc::tmem_ld<8>(tO + col0 + n + lane_addr, orr);
        tc::tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int r = rc * N + col0 + n + e;
          if (r < R) {
            const int gr = (r / P.p) * P.h + c * P.p + (r % P.p);
            P.ws_o[((size_t)gr * P.S + slot_idx) * kD + pos] = __uint_as_float(orr[e]);
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(o_empty));
      tc::named_bar_sync(2, 256);
      if (sw < 4) {
        // 128 threads: column sw*32 + lane (N <= 128)
        const int col = sw * 32 + lane;
        const int r = rc * N + col;
        if (col < N && r < R) {
          const int gr = (r / P.p) * P.h + c * P.p + (r % P.p);
          const float L = sm_l[col] + sm_l[128 + col] + sm_l[256 + col] + sm_l[384 + col];
          float* ml = P.ws_ml + ((size_t)gr * P.S + slot_idx) * 2;
          ml[0] = sm_mrun[cur * 128 + col];
          ml[1] = L;
        }
      }
      tc::named_bar_sync(2, 256);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, TMEM_COLS);
  }
}

}  // namespace ba
