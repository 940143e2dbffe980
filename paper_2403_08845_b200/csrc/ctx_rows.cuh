// ctx_rows.cuh — the CONTEXT branch of the bifurcated step for wide row sets
// (R = b*p >= 64 query rows per KV group: C3, C4, C5, multi-token steps),
// rows on the MMA's M dimension (sm_100a tcgen05 + TMEM + TMA).
//
// What it computes (Eq. 3-4 context rows; "axis b does
// not appear", :259): for a block of 128 of the R rows of group c and a range
// of 128-position context tiles, the online-softmax partial
//   m = running max of s*scale*log2e,  l = sum 2^(x - m),  o = sum 2^(x - m) Vc
// written to the workspace context slot of the range; the fused kernel
// (bif_tc.cuh) streams the decode branch and joins these partials with its
// own in the LSE merge.  Each Kc/Vc tile is read once per 128-row block
// (ceil(R/128) times instead of ceil(R/32) times by the swap-AB kernel).
//
// Tile math (rows on M):
//   S[128 rows x 128 pos]  = Q_blk[128 x d] . K_tile^T       (A = Q, B = K, both K-major)
//   O[128 rows x d]       += P . V16_tile                     (A = P K-major, B = V MN-major)
// Two threads own a row (TMEM lane = row, one per half of the positions):
// the row max is a 2-way exchange, the stale-max test and the O rescale are
// per row — no vote across the rows of a column as in the swap-AB kernel.
// Round 2 (reading R23): the V tile is converted in place to f16 x 2^-8 by two
// converter warps once it lands, so P = 2^(x - m) enters the PV MMA as ONE
// f16 operand (11 significant bits; the bf16 pair P_hi + P_lo of round 1 cost
// twice the PV MMAs), stored to TMEM over its S slot and read from there as
// the A operand; the epilogue scales O back by 2^8 (exact).  TMEM: 3 S slots
// (P(u) overwrites S(u)) + O = 512 columns.
//
// Warps: 0 / 3 TMA producers of the K / V halves (one lane each), 1 MMA
// issuer (one lane), 2 TMEM allocator and (with 12) V converter, 4..11
// softmax/epilogue: two threads per row, each taking half of the tile's
// positions and of the O columns.
#pragma once
#include "append.cuh"
#include "common.cuh"
#include "tc_ptx.cuh"

namespace ba {

struct CtxRowsParams {
  CUtensorMap tmKc, tmVc;  // (d, mc, g), box (64, 128, 1), SW128
  CUtensorMap tmKd, tmVd;  // (d, md_cap, b*g), box (64, 128, 1): decode items (p >= 32)
  // Q block by TMA (round 3; the softmax threads' global loads cost ~4k cycles
  // per item): q_mode 1 = q as (d, h, b), box (64, p, 128/p) at (., c*p,
  // rb*128/p) (p divides 128); 2 = q as (d, b*h) rows, box (64, 128) at
  // (., rb*128) (g = 1: a block's rows are consecutive); 0 = thread loads
  CUtensorMap tmQ;
  int q_mode;
  int nrp;                 // ctx_rows2_kernel: row-block pairs per group (items pair blocks 2rp, 2rp+1)
  const int32_t* lens;     // decode items: valid length min(clamp(lens[i]) + lens_add, dec_cap)
  int dec_cap, lens_add;
  AppendSrc app;           // append+attend: this step's rows, stored by the decode item's CTA
  int ntok;                // multi-token step: decode row r (token r % ntok) sees
                           // positions < L - (ntok - 1 - r % ntok)
  int items_ctx;           // items [0, items_ctx) are context items, then b*g decode items
  int dec_slot;            // workspace slot of the decode partial
  unsigned long long* trace;  // BIFATTN_PROF builds: per-role cycle accounting [grid][1024]
  const void* q;           // [b][h][128] bf16 (rows of group c: (i, c*p + j))
  int b, h, g, p, mc;
  int R, nrb;              // rows per group, 128-row blocks per group
  int ntile, tps, nsplit;  // context tiles, tiles per split, splits per (c, rb)
  int items;               // g * nrb * nsplit
  float scale_log2;
  int S;                   // workspace slots per row (context slots [0, nsplit))
  float* ws_o;             // [b*h][S][128]
  float* ws_ml;            // [b*h][S][2]
};

// Experiment bits (CTXR_EXP, experiment builds only; wrong results): 1 skip
// the row-max exchange barrier, 2 skip the exp/pack work (P = 0), 4 skip the
// PV MMAs, 8 skip the QK MMAs.
#ifndef CTXR_EXP
#define CTXR_EXP 0
#endif
namespace ctxr {
constexpr int kStage = 65536;           // K tile 32 KB + V tile 32 KB
constexpr int kNst = 3;                 // K/V stages
constexpr int kS = 3;                   // S/P slots in TMEM (3 x 128 columns + O = 512)
constexpr int kQ = kNst * kStage;       // Q block (32 KB)
constexpr int kBar = kQ + 32768;        // barriers
constexpr int kXch = kBar + 256;        // row-max exchange [2 tiles][2 halves][128 rows] floats
constexpr int kLsx = kXch + 2048;       // item-end row-sum exchange [128 rows] floats (own slot)
constexpr int kSmem = kLsx + 512;       // 232192 <= 227 KB
constexpr float kTh = 8.0f;             // stale-max slack (log2 units), as bif_tc.cuh
constexpr int kThreads = 416;        // 13 warps: + warp 12, the second V converter
constexpr float kVScale = 0.00390625f;  // V is converted to f16 as V * 2^-8 (reading R23)


// byte offset of 16-byte chunk `ch` (0..15) of row r in a 128-row x 128-col
// bf16 K-major SW128 tile stored as two 64-column halves (the TMA box layout)
BA_DEVINL uint32_t sw128_off(int r, int ch) {
  return (uint32_t)((ch >> 3) * 16384 + r * 128 + (((ch & 7) ^ (r & 7)) << 4));
}
}  // namespace ctxr

__global__ void __launch_bounds__(ctxr::kThreads, 1)
    ctx_rows_kernel(const __grid_constant__ CtxRowsParams P) {
  using namespace ctxr;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBar);
  // K and V halves of a stage have their own barriers: K(u) is released by
  // QK(u), V(u) by PV(u), so the next K load does not wait for the PV
  uint64_t* k_full = bars;        // [kNst]
  uint64_t* k_empty = bars + 3;   // [kNst]
  uint64_t* s_full = bars + 6;    // [kS]
  uint64_t* s_free = bars + 9;    // [kS]
  uint64_t* q_full = bars + 12;
  uint64_t* q_empty = bars + 13;
  uint64_t* p_empty = bars + 14;  // PV(u) done (O quiescent for a rescale)
  uint64_t* o_full = bars + 15;
  uint64_t* o_empty = bars + 16;
  uint64_t* v_full = bars + 17;   // [kNst]
  uint64_t* v_empty = bars + 20;  // [kNst]
  uint64_t* p_full = bars + 23;   // [kS] P(u) stored over S(u)
  uint64_t* v_cvt = bars + 26;    // [kNst] V(u) converted to f16 in place
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 30);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kNst; ++s) {
      tc::mbar_init(tc::smem_u32(&k_full[s]), 1);
      tc::mbar_init(tc::smem_u32(&k_empty[s]), 1);
      tc::mbar_init(tc::smem_u32(&v_full[s]), 1);
      tc::mbar_init(tc::smem_u32(&v_empty[s]), 1);
    }
    for (int s = 0; s < kS; ++s) {
      tc::mbar_init(tc::smem_u32(&s_full[s]), 1);
      tc::mbar_init(tc::smem_u32(&s_free[s]), 1);  // PV(u) done: slot reusable
      tc::mbar_init(tc::smem_u32(&p_full[s]), 8);
    }
    tc::mbar_init(tc::smem_u32(q_full), P.q_mode ? 1 : 8);
    tc::mbar_init(tc::smem_u32(q_empty), 1);
    tc::mbar_init(tc::smem_u32(p_empty), 1);
    tc::mbar_init(tc::smem_u32(o_full), 1);
    tc::mbar_init(tc::smem_u32(o_empty), 8);
    for (int s = 0; s < kNst; ++s) tc::mbar_init(tc::smem_u32(&v_cvt[s]), 64);
    tc::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&P.tmKc);
    tc::prefetch_tmap(&P.tmVc);
    if (P.q_mode) tc::prefetch_tmap(&P.tmQ);
    if (P.items > P.items_ctx) {
      tc::prefetch_tmap(&P.tmKd);
      tc::prefetch_tmap(&P.tmVd);
    }
  }
  if (warp == 2) {
    tc::tmem_alloc(tc::smem_u32(tmem_holder), 512);
    tc::tmem_relinquish();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  pdl_wait();
  pdl_launch_dependents();
  const uint32_t tmem = *tmem_holder;
  const uint32_t tS = tmem;        // S buffers at columns [0,128), [128,256)
  const uint32_t tO = tmem + kS * 128;  // O after the kS S/P slots
  // P(u) = P_hi | P_lo as bf16 pairs is stored over S(u) (columns [0, 64) and
  // [64, 128) of its slot) once S(u) is in registers: the S slots double as a
  // double-buffered P, and a slot is free again when PV(u) completes

  // item k: a context item (group c, row block rb, split s, tiles [t0, t1) of
  // Kc[c]) or, for k >= items_ctx, the decode item of (sample i, group c):
  // the p query rows of sample i against the tiles of Kd[i][c] (p >= 32 rows
  // fill a useful share of the 128-row block).  L = valid
  // positions, z = the K/V tensor map's group coordinate.
  struct Item {
    bool dec;
    int c, rb, s, t0, t1, L, z, i;
  };
  auto item_of = [&](int k) {
    Item it;
    if (k < P.items_ctx) {
      it.dec = false;
      it.s = k % P.nsplit;
      const int cr = k / P.nsplit;
      it.rb = cr % P.nrb;
      it.c = cr / P.nrb;
      it.t0 = it.s * P.tps;
      it.t1 = min(P.ntile, it.t0 + P.tps);
      it.L = P.mc;
      it.z = it.c;
      it.i = 0;
    } else {
      const int j = k - P.items_ctx;
      it.dec = true;
      it.i = j / P.g;
      it.c = j - it.i * P.g;
      it.rb = 0;
      it.s = P.dec_slot;
      int L = P.lens[it.i];
      L = L < 0 ? 0 : (L > P.dec_cap ? P.dec_cap : L);
      it.L = min(L + P.lens_add, P.dec_cap);
      it.t0 = 0;
      it.t1 = (it.L + 127) >> 7;
      it.z = it.i * P.g + it.c;
    }
    return it;
  };

  if (warp == 0 || warp == 3) {
    // append+attend: the K (warp 0) / V (warp 3) rows of this CTA's decode items
    // before any TMA of them (same CTA: generic stores, then a proxy fence)
    if (P.app.n > 0) {
      for (int k = blockIdx.x; k < P.items; k += gridDim.x) {
        if (k < P.items_ctx) continue;
        const int j = k - P.items_ctx, i = j / P.g, c = j - (j / P.g) * P.g;
        append_rows_warp(P.app, i, c, clamp_len(P.lens, i, P.dec_cap), 0, P.dec_cap, lane,
                         warp == 0 ? 1 : 2);
      }
      fence_proxy_async_global();
      __syncwarp();
      fence_proxy_async_global();
    }
    // ============ TMA producers: K (warp 0), V (warp 3), Q (warp 0 lane 1) ============
    if (lane == 1 && warp == 0 && P.q_mode) {
      // the Q block of every non-empty item, as soon as the previous item's
      // last QK has read the single Q buffer
      uint32_t it = 0;
      for (int k = blockIdx.x; k < P.items; k += gridDim.x) {
        const Item I = item_of(k);
        if (I.t1 == I.t0) continue;
        tc::mbar_wait_sleep(tc::smem_u32(q_empty), (it & 1) ^ 1);
        const uint32_t bar = tc::smem_u32(q_full);
        tc::mbar_arrive_expect_tx(bar, 32768);
        const uint32_t dst = tc::smem_u32(smem + kQ);
        int y, z;
        if (P.q_mode == 1) {  // (head c*p + j, sample): rows of the block are (sample, j)
          y = I.c * P.p;
          z = I.dec ? I.i : I.rb * (128 / P.p);
        } else {              // g = 1: row gr = i*h + j = the row within the group
          y = I.dec ? I.i * P.h : I.rb * 128;
          z = 0;
        }
        tc::tma_load_3d(dst, &P.tmQ, bar, 0, y, z);
        tc::tma_load_3d(dst + 16384, &P.tmQ, bar, 64, y, z);
        ++it;
      }
    } else if (lane == 0) {
      const bool isk = warp == 0;
      uint64_t* full = isk ? k_full : v_full;
      uint64_t* empty = isk ? k_empty : v_empty;
      const uint64_t pol = tc::policy_evict_last();  // re-read by the other row blocks
      uint32_t u = 0;
      for (int k = blockIdx.x; k < P.items; k += gridDim.x) {
        const Item I = item_of(k);
        const CUtensorMap* map = I.dec ? (isk ? &P.tmKd : &P.tmVd) : (isk ? &P.tmKc : &P.tmVc);
        for (int t = I.t0; t < I.t1; ++t, ++u) {
          const int st = u % kNst;
          tc::mbar_wait_sleep(tc::smem_u32(&empty[st]), ((u / kNst) & 1) ^ 1);
          const uint32_t bar = tc::smem_u32(&full[st]);
          tc::mbar_arrive_expect_tx(bar, kStage / 2);
          const uint32_t dst = tc::smem_u32(smem + st * kStage + (isk ? 0 : 32768));
          tc::tma_load_3d_hint(dst, map, bar, 0, t * 128, I.z, pol);
          tc::tma_load_3d_hint(dst + 16384, map, bar, 64, t * 128, I.z, pol);
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    if (lane == 0) {
      constexpr uint32_t IDESC_QK = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t IDESC_PV = tc::idesc_f16(128, 128, 0, 1);  // f16 P (TMEM) x f16 V
      const uint32_t qbase = tc::smem_u32(smem + kQ);
      uint32_t u = 0, it = 0;
      // O += P(v) . V(v): both bf16 parts of P into the same accumulator
      Prof pf;  // 0 q_full, 1 k_full, 2 s_free, 3 QK issue, 4 v_full, 5 p_full, 6 PV issue, 7 o_empty
      auto pv = [&](uint32_t v, bool first) {
        pf.mark(3);
        tc::mbar_wait_sleep(tc::smem_u32(&v_cvt[v % kNst]), (v / kNst) & 1);
        pf.mark(4);
        tc::mbar_wait_sleep(tc::smem_u32(&p_full[v % kS]), (v / kS) & 1);
        pf.mark(5);
        tc::tc_fence_after();
        const uint32_t vb = tc::smem_u32(smem + (v % kNst) * kStage + 32768);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          // A = P from TMEM: 16 positions per step = 8 columns of f16 pairs
          const uint64_t bd = tc::smem_desc(vb + k * 2048, 16384, 1024, tc::kSw128);
          if (!(CTXR_EXP & 4))
            tc::mma_bf16_ts(tO, tS + (v % kS) * 128 + k * 8, bd, IDESC_PV,
                            (first && k == 0) ? 0u : 1u);
        }
        tc::mma_commit(tc::smem_u32(&s_free[v % kS]));
        tc::mma_commit(tc::smem_u32(&v_empty[v % kNst]));
        pf.mark(6);
      };
      for (int k = blockIdx.x; k < P.items; k += gridDim.x) {
        const Item I = item_of(k);
        if (I.t1 == I.t0) continue;  // empty decode item: the softmax threads write it
        const int t0 = I.t0, t1 = I.t1;
        pf.mark(3);
        tc::mbar_wait_sleep(tc::smem_u32(q_full), it & 1);
        pf.mark(0);
        const uint32_t u0 = u;
        for (int t = t0; t < t1; ++t, ++u) {
          tc::mbar_wait_sleep(tc::smem_u32(&k_full[u % kNst]), (u / kNst) & 1);
          pf.mark(1);
          tc::mbar_wait_sleep(tc::smem_u32(&s_free[u % kS]), ((u / kS) & 1) ^ 1);
          pf.mark(2);
          tc::tc_fence_after();
          const uint32_t kb = tc::smem_u32(smem + (u % kNst) * kStage);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t ad = tc::smem_desc(qbase + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024,
                                              tc::kSw128);
            const uint64_t bd = tc::smem_desc(kb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024,
                                              tc::kSw128);
            if (!(CTXR_EXP & 8)) tc::mma_bf16(tS + (u % kS) * 128, ad, bd, IDESC_QK, kk > 0 ? 1u : 0u);
          }
          tc::mma_commit(tc::smem_u32(&s_full[u % kS]));
          tc::mma_commit(tc::smem_u32(&k_empty[u % kNst]));  // K(u) reusable
          if (t == t1 - 1) tc::mma_commit(tc::smem_u32(q_empty));  // Q block reusable
          if (u > u0) pv(u - 1, u - 1 == u0);
          else {
            pf.mark(3);
            tc::mbar_wait_sleep(tc::smem_u32(o_empty), (it & 1) ^ 1);  // O drained
            pf.mark(7);
          }
        }
        pv(u - 1, u - 1 == u0);
        tc::mma_commit(tc::smem_u32(o_full));
        ++it;
      }
      pf.mark(3);
      pf.dump(P.trace ? P.trace + (size_t)blockIdx.x * 1024 : nullptr, 8);
    }
  } else if (warp == 2 || warp == 12) {
    // ============ V converters (warps 2 and 12): bf16 V tile -> f16 * 2^-8 in place ============
    // (element-wise and in place, so the TMA's SW128 layout is kept; each warp
    // takes half of the tile's 2048 16-byte chunks, consecutive lanes on
    // consecutive chunks: conflict-free)
    const int half = warp == 2 ? 0 : 1;
    uint32_t u = 0;
    for (int k = blockIdx.x; k < P.items; k += gridDim.x) {
      const Item I = item_of(k);
      for (int t = I.t0; t < I.t1; ++t, ++u) {
        const int st = u % kNst;
        tc::mbar_wait(tc::smem_u32(&v_full[st]), (u / kNst) & 1);
        uint8_t* const vt = smem + st * kStage + 32768;
#pragma unroll 4
        for (int ch = half * 1024 + lane; ch < half * 1024 + 1024; ch += 32) {
          uint4 v = lds128(vt + ch * 16);
          v.x = pack_f16x2(bf16lo(v.x) * kVScale, bf16hi(v.x) * kVScale);
          v.y = pack_f16x2(bf16lo(v.y) * kVScale, bf16hi(v.y) * kVScale);
          v.z = pack_f16x2(bf16lo(v.z) * kVScale, bf16hi(v.z) * kVScale);
          v.w = pack_f16x2(bf16lo(v.w) * kVScale, bf16hi(v.w) * kVScale);
          sts128(vt + ch * 16, v);
        }
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(tc::smem_u32(&v_cvt[st]));
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ============ softmax + epilogue: two threads per row (one per half) ============
    // warps 4..7 (hf = 0) take positions [0, 64) and O columns [0, 64) of their
    // rows, warps 8..11 (hf = 1) positions [64, 128) and O columns [64, 128);
    // the two halves of a row agree on its running max through one 256-thread
    // barrier per tile (double-buffered exchange slots).
    const int hf = (warp - 4) >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;                    // row in the block = TMEM lane
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    const float sl2 = P.scale_log2;
    uint8_t* const sq = smem + kQ;
    float* const sm_x = reinterpret_cast<float*>(smem + kXch);
    uint32_t u = 0, it = 0;
    Prof pf;  // 0 Q load, 1 s_full wait, 2 S load, 3 max, 4 exchange barrier, 5 rescale, 6 P, 7 epilogue
    for (int k = blockIdx.x; k < P.items; k += gridDim.x) {
      const Item I = item_of(k);
      const int c = I.c, s = I.s, t0 = I.t0, t1 = I.t1;
      const int rg = I.rb * 128 + r;                    // row within the group (context)
      const bool valid_row = I.dec ? r < P.p : rg < P.R;
      BA_CHECK(I.s >= 0 && I.s < P.S && I.c < P.g && (!I.dec || I.i < P.b));
      const int gr = !valid_row ? -1
                     : I.dec ? I.i * P.h + c * P.p + r
                             : (rg / P.p) * P.h + c * P.p + rg % P.p;
      if (t1 == t0) {
        // empty decode item (lens = 0): an empty partial (m = -inf, l = 0, o = 0)
        if (valid_row) {
          float* wo = P.ws_o + ((size_t)gr * P.S + s) * 128 + hf * 64;
#pragma unroll
          for (int e = 0; e < 64; e += 4) *reinterpret_cast<float4*>(wo + e) = make_float4(0.f, 0.f, 0.f, 0.f);
          if (hf == 0) reinterpret_cast<float2*>(P.ws_ml)[(size_t)gr * P.S + s] = make_float2(kNegInf, 0.f);
        }
        continue;
      }
      // ---- this half of the Q row -> shared memory (SW128, the TMA box layout) ----
      if (!P.q_mode) {
      tc::mbar_wait(tc::smem_u32(q_empty), (it & 1) ^ 1);
      {
        const uint4* src = reinterpret_cast<const uint4*>(P.q) + (size_t)(valid_row ? gr : 0) * 16;
#pragma unroll
        for (int ch = 8 * hf; ch < 8 * hf + 8; ++ch) {
          const uint4 v = valid_row ? __ldg(src + ch) : make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(sq + sw128_off(r, ch)) = v;
        }
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(q_full));
      // L2 prefetch of this thread's half Q row of the NEXT item (its load is
      // on the item-switch path; the item's tiles take microseconds)
      if (k + (int)gridDim.x < P.items) {
        const Item In = item_of(k + gridDim.x);
        const int rgn = In.rb * 128 + r;
        const bool vn = In.dec ? r < P.p : rgn < P.R;
        if (vn) {
          const int grn = In.dec ? In.i * P.h + In.c * P.p + r : (rgn / P.p) * P.h + In.c * P.p + rgn % P.p;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const uint4*>(P.q) + (size_t)grn * 16 + 8 * hf));
        }
      }
      }  // !q_mode
      float m = kNegInf, l = 0.f;  // l: this half's share of the row sum
      pf.mark(0);
      for (int t = t0; t < t1; ++t, ++u) {
        tc::mbar_wait(tc::smem_u32(&s_full[u % kS]), (u / kS) & 1);
        pf.mark(1);
        tc::tc_fence_after();
        float x[64];
        tc::tmem_ld<32>(tS + (u % kS) * 128 + hf * 64 + lane_addr, reinterpret_cast<uint32_t*>(x));
        tc::tmem_ld<32>(tS + (u % kS) * 128 + hf * 64 + 32 + lane_addr, reinterpret_cast<uint32_t*>(x) + 32);
        tc::tmem_ld_wait();
        pf.mark(2);
        // logits in log2 units; positions past mc masked (last tile only)
        const int Lrow = I.dec && P.ntok > 1 ? max(I.L - (P.ntok - 1 - r % P.ntok), 0) : I.L;
        const int nvalid = min(128, Lrow - t * 128) - hf * 64;
        // row max over this half's 64 positions: 8 independent chains (a
        // single running fmax was a 64-deep dependency chain, ~1k cycles/pass),
        // on the raw logits (the scale is positive: max commutes with it, and
        // the scaling folds into the exponent's FFMA2 below)
        float mq[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) mq[k] = kNegInf;
        if (nvalid >= 64) {
#pragma unroll
          for (int i = 0; i < 64; ++i) mq[i & 7] = fmaxf(mq[i & 7], x[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            x[i] = i < nvalid ? x[i] : kNegInf;
            mq[i & 7] = fmaxf(mq[i & 7], x[i]);
          }
        }
        const float mh = fmaxf(fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])),
                               fmaxf(fmaxf(mq[4], mq[5]), fmaxf(mq[6], mq[7]))) * sl2;
        pf.mark(3);
        float* const xs = sm_x + (u & 1) * 256;
        xs[hf * 128 + r] = mh;
        if (!(CTXR_EXP & 1)) tc::named_bar_sync(1, 256);
        const float mx = fmaxf(mh, xs[(hf ^ 1) * 128 + r]);
        pf.mark(4);
        if (m == kNegInf || mx > m + kTh) {
          // raise the reference to the exact max; rescale l and this half of the O row
          const float mn = mx;
          if (m != kNegInf && t > t0) {
            // PV(u-1) done (O quiescent): the commit that frees S slot (u-1) % kS
            tc::mbar_wait(tc::smem_u32(&s_free[(u - 1) % kS]), ((u - 1) / kS) & 1);
            const float a = ex2(m - mn);
            l *= a;
            tc::tc_fence_after();
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              uint32_t o[8];
              tc::tmem_ld<8>(tO + hf * 64 + q * 8 + lane_addr, o);
              tc::tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * a);
              tc::tmem_st<8>(tO + hf * 64 + q * 8 + lane_addr, o);
            }
            tc::tmem_st_wait();
            tc::tc_fence_before();
          }
          m = mn;
        }
        pf.mark(5);
        const float mref = m == kNegInf ? 0.f : m;  // a row with no valid position yet: P = 0
        // P = 2^(x - m) as ONE f16 operand (reading R23; V is f16 * 2^-8) into
        // TMEM over S: the PV's A operand
        // exponent x * scale - m as one FFMA2 per pair; partial row sums as FADD2
        const float2 sl2v = make_float2(sl2, sl2), nmv = make_float2(-mref, -mref);
        float2 lq[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};  // independent partial row sums
#pragma unroll
        for (int j = 0; j < ((CTXR_EXP & 2) ? 0 : 4); ++j) {
          uint32_t hk[8];
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            // (round 3 again moved 3 of 8 pairs to a packed degree-3 FMA-pipe
            // polynomial: C4 48.6 vs 45.9 us, C3 70.4 vs 68.1 us without it —
            // the pass is bound by issue and latency, not by MUFU)
            const float2 z = fma2(make_float2(x[j * 16 + e], x[j * 16 + e + 1]), sl2v, nmv);
            const float2 pz = make_float2(ex2(z.x), ex2(z.y));
            lq[(e >> 1) & 1] = add2(lq[(e >> 1) & 1], pz);
            hk[e / 2] = pack_f16x2(pz.x, pz.y);
          }
          tc::tmem_st<8>(tS + (u % kS) * 128 + hf * 32 + j * 8 + lane_addr, hk);
        }
        l += (lq[0].x + lq[0].y) + (lq[1].x + lq[1].y);
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(tc::smem_u32(&p_full[u % kS]));
        pf.mark(6);
      }
      // ---- the item's partial: O row (relative to 2^m), m, l ----
      tc::mbar_wait(tc::smem_u32(o_full), it & 1);
      tc::tc_fence_after();
      float* wo = valid_row ? P.ws_o + ((size_t)gr * P.S + s) * 128 + hf * 64 : nullptr;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        uint32_t o[32];
        tc::tmem_ld<32>(tO + hf * 64 + q * 32 + lane_addr, o);
        tc::tmem_ld_wait();
        if (valid_row) {
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(wo + q * 32 + e) =  // undo V * 2^-8 (exact)
                make_float4(__uint_as_float(o[e]) * 256.f, __uint_as_float(o[e + 1]) * 256.f,
                            __uint_as_float(o[e + 2]) * 256.f, __uint_as_float(o[e + 3]) * 256.f);
        }
      }
      // row sum = both halves' shares, through its own exchange slot (written
      // by the hf = 1 half, read by hf = 0 between this barrier and the next
      // item's first tile barrier)
      float* const ls = reinterpret_cast<float*>(smem + kLsx);
      if (hf == 1) ls[r] = l;
      tc::named_bar_sync(1, 256);
      if (hf == 0 && valid_row)
        reinterpret_cast<float2*>(P.ws_ml)[(size_t)gr * P.S + s] = make_float2(m, l + ls[r]);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(o_empty));
      ++it;
      pf.mark(7);
    }
    if (threadIdx.x == 128) pf.dump(P.trace ? P.trace + (size_t)blockIdx.x * 1024 : nullptr, 0);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

}  // namespace ba
