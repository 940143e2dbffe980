// ctx_rows2.cuh — the rows-on-M context kernel with TWO 128-row blocks per
// CTA item in ping-pong (round 3), sm_100a tcgen05 + TMEM + TMA.
//
// Same computation as ctx_rows_kernel (ctx_rows.cuh; Eq. 3-4 context rows,
// PAPER.md:254, :266, "axis b does not appear", :259): for row blocks A = 2rp
// and B = 2rp + 1 of group c and a range of 128-position context tiles, the
// online-softmax partial (m, l, o) of every row, written to the workspace
// context slot of the range (decode items: block A = the p rows of (i, c)).
//
// Why a second kernel: the one-block kernel's pass is bound by its softmax
// warps (both halves of a row meet in a per-tile barrier, so all 8 warps are
// in the same phase and the MUFU exponentials never overlap the max, TMEM
// traffic or the waits; ~2300 cycles per 128 x 128 pass against a 1024-cycle
// MUFU floor).  Here one warpgroup owns block A and one block B, ONE thread
// per row (the whole 128-position S row in registers, no exchange), and the
// MMA issuer interleaves the blocks —
//     QK_A(u), PV_B(u-1), QK_B(u), PV_A(u), QK_A(u+1), ...
// — so the tensor pipe runs one block's MMAs while the other block's
// warpgroup computes its exponentials: the two softmax phases alternate on
// the MUFU and each K/V tile serves 256 rows.
//
// TMEM: S_A | S_B | O_A | O_B (128 columns each; P(u) as f16 pairs over its
// S slot, the PV's A operand; V converted in place to f16 x 2^-8, reading
// R23).  Shared memory: 2 K/V stages + Q_A + Q_B (Q blocks by TMA only).
// Warps: 0 producers (lane 0 K, lane 1 V, lane 2 Q; the whole warp stores
// append rows first), 1 MMA issuer, 2 TMEM allocator + V converter, 3 V
// converter, 4-7 block A, 8-11 block B (softmax, then the item's epilogue).
#pragma once
#include "append.cuh"
#include "common.cuh"
#include "ctx_rows.cuh"
#include "tc_ptx.cuh"

namespace ba {
namespace ctxr2 {
constexpr int kStage = 65536;      // K tile 32 KB + V tile 32 KB
constexpr int kNst = 2;            // K/V stages
constexpr int kQ = kNst * kStage;  // Q_A at kQ, Q_B at kQ + 32 KB
constexpr int kBar = kQ + 65536;   // barriers
constexpr int kSmem = kBar + 256;  // 196864
constexpr int kThreads = 384;      // 12 warps
constexpr float kTh = 8.0f;        // stale-max slack (log2 units), as ctx_rows.cuh
constexpr float kVScale = 0.00390625f;
}  // namespace ctxr2

__global__ void __launch_bounds__(ctxr2::kThreads, 1)
    ctx_rows2_kernel(const __grid_constant__ CtxRowsParams P) {
  using namespace ctxr2;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBar);
  uint64_t* k_full = bars;          // [2]
  uint64_t* k_empty = bars + 2;     // [2]
  uint64_t* v_full = bars + 4;      // [2]
  uint64_t* v_empty = bars + 6;     // [2]
  uint64_t* v_cvt = bars + 8;       // [2]
  uint64_t* q_full = bars + 10;
  uint64_t* q_empty = bars + 11;
  uint64_t* s_full = bars + 12;     // [2] block A, B: QK(u) done
  uint64_t* p_full = bars + 14;     // [2] P(u) stored over S
  uint64_t* pv_done = bars + 16;    // [2] PV(u) done (S/P slot free, O quiescent)
  uint64_t* o_empty = bars + 18;    // [2] the block's O drained by its epilogue
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 20);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kNst; ++s) {
      tc::mbar_init(tc::smem_u32(&k_full[s]), 1);
      tc::mbar_init(tc::smem_u32(&k_empty[s]), 1);
      tc::mbar_init(tc::smem_u32(&v_full[s]), 1);
      tc::mbar_init(tc::smem_u32(&v_empty[s]), 1);
      tc::mbar_init(tc::smem_u32(&v_cvt[s]), 64);
    }
    tc::mbar_init(tc::smem_u32(q_full), 1);
    tc::mbar_init(tc::smem_u32(q_empty), 1);
    for (int x = 0; x < 2; ++x) {
      tc::mbar_init(tc::smem_u32(&s_full[x]), 1);
      tc::mbar_init(tc::smem_u32(&p_full[x]), 4);
      tc::mbar_init(tc::smem_u32(&pv_done[x]), 1);
      tc::mbar_init(tc::smem_u32(&o_empty[x]), 4);
    }
    tc::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&P.tmKc);
    tc::prefetch_tmap(&P.tmVc);
    tc::prefetch_tmap(&P.tmQ);
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
  const uint32_t tS = tmem;          // S_A at [0, 128), S_B at [128, 256)
  const uint32_t tO = tmem + 256;    // O_A at [256, 384), O_B at [384, 512)

  // item k < items_ctx: context rows blocks 2rp, 2rp+1 of group c, split s;
  // else the decode item of (sample i, group c): block A = its p rows
  struct Item {
    bool dec, hasB;
    int c, rp, s, t0, t1, L, z, i;
  };
  auto item_of = [&](int k) {
    Item it;
    if (k < P.items_ctx) {
      it.dec = false;
      it.s = k % P.nsplit;
      const int cr = k / P.nsplit;
      it.rp = cr % P.nrp;
      it.c = cr / P.nrp;
      it.hasB = 2 * it.rp + 1 < P.nrb;
      it.t0 = it.s * P.tps;
      it.t1 = min(P.ntile, it.t0 + P.tps);
      it.L = P.mc;
      it.z = it.c;
      it.i = 0;
    } else {
      const int j = k - P.items_ctx;
      it.dec = true;
      it.hasB = false;
      it.i = j / P.g;
      it.c = j - it.i * P.g;
      it.rp = 0;
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

  if (warp == 0) {
    // append+attend: this CTA's decode items' new rows before any TMA of them
    if (P.app.n > 0) {
      for (int k = blockIdx.x; k < P.items; k += gridDim.x) {
        if (k < P.items_ctx) continue;
        const int j = k - P.items_ctx, i = j / P.g, c = j - (j / P.g) * P.g;
        append_rows_warp(P.app, i, c, clamp_len(P.lens, i, P.dec_cap), 0, P.dec_cap, lane, 3);
      }
      fence_proxy_async_global();
      __syncwarp();
      fence_proxy_async_global();
    }
    if (lane == 0 || lane == 1) {
      // ============ K (lane 0) / V (lane 1) tiles, all items in order ============
      const bool isk = lane == 0;
      uint64_t* full = isk ? k_full : v_full;
      uint64_t* empty = isk ? k_empty : v_empty;
      const uint64_t pol = tc::policy_evict_last();  // re-read by the other row-block pairs
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
    } else if (lane == 2) {
      // ============ Q blocks A (and B) of every non-empty item ============
      uint32_t it = 0;
      for (int k = blockIdx.x; k < P.items; k += gridDim.x) {
        const Item I = item_of(k);
        if (I.t1 == I.t0) continue;
        tc::mbar_wait_sleep(tc::smem_u32(q_empty), (it & 1) ^ 1);
        const uint32_t bar = tc::smem_u32(q_full);
        tc::mbar_arrive_expect_tx(bar, I.hasB ? 65536 : 32768);
        for (int x = 0; x < (I.hasB ? 2 : 1); ++x) {
          const uint32_t dst = tc::smem_u32(smem + kQ + x * 32768);
          const int rb = 2 * I.rp + x;
          int y, z;
          if (P.q_mode == 1) {
            y = I.c * P.p;
            z = I.dec ? I.i : rb * (128 / P.p);
          } else {
            y = I.dec ? I.i * P.h : rb * 128;
            z = 0;
          }
          tc::tma_load_3d(dst, &P.tmQ, bar, 0, y, z);
          tc::tma_load_3d(dst + 16384, &P.tmQ, bar, 64, y, z);
        }
        ++it;
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    if (lane == 0) {
      constexpr uint32_t IDESC_QK = tc::idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t IDESC_PV = tc::idesc_f16(128, 128, 0, 1);  // f16 P (TMEM) x f16 V
      uint32_t u = 0, it = 0;
      uint32_t nP[2] = {0, 0};    // PVs issued per block
      uint32_t nIt[2] = {0, 0};   // items per block (O drains)
      // a PV of block x still to issue: (tile counter, stage, first tile of its item?)
      bool pendB = false;
      uint32_t pendB_u = 0;
      bool pendB_first = false;
      Prof pf;
      auto qk = [&](int x, uint32_t st) {
        pf.mark(6);
        if (nP[x] > 0) tc::mbar_wait_sleep(tc::smem_u32(&pv_done[x]), (nP[x] - 1) & 1);  // S/P slot free
        pf.mark(2);
        tc::tc_fence_after();
        const uint32_t qbase = tc::smem_u32(smem + kQ + x * 32768);
        const uint32_t kb = tc::smem_u32(smem + st * kStage);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t ad = tc::smem_desc(qbase + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, tc::kSw128);
          const uint64_t bd = tc::smem_desc(kb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, tc::kSw128);
          tc::mma_bf16(tS + x * 128, ad, bd, IDESC_QK, kk > 0 ? 1u : 0u);
        }
        tc::mma_commit(tc::smem_u32(&s_full[x]));
        pf.mark(3);
      };
      auto pv = [&](int x, uint32_t v, bool first, bool release_v) {
        pf.mark(6);
        if (first) tc::mbar_wait_sleep(tc::smem_u32(&o_empty[x]), (nIt[x] & 1) ^ 1);  // O drained
        pf.mark(7);
        tc::mbar_wait_sleep(tc::smem_u32(&v_cvt[v % kNst]), (v / kNst) & 1);
        pf.mark(4);
        tc::mbar_wait_sleep(tc::smem_u32(&p_full[x]), nP[x] & 1);
        pf.mark(5);
        tc::tc_fence_after();
        const uint32_t vb = tc::smem_u32(smem + (v % kNst) * kStage + 32768);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = tc::smem_desc(vb + kk * 2048, 16384, 1024, tc::kSw128);
          tc::mma_bf16_ts(tO + x * 128, tS + x * 128 + kk * 8, bd, IDESC_PV, (first && kk == 0) ? 0u : 1u);
        }
        tc::mma_commit(tc::smem_u32(&pv_done[x]));
        if (release_v) tc::mma_commit(tc::smem_u32(&v_empty[v % kNst]));
        ++nP[x];
      };
      for (int k = blockIdx.x; k < P.items; k += gridDim.x) {
        const Item I = item_of(k);
        if (I.t1 == I.t0) continue;
        pf.mark(6);
        tc::mbar_wait_sleep(tc::smem_u32(q_full), it & 1);
        pf.mark(0);
        for (int t = I.t0; t < I.t1; ++t, ++u) {
          const uint32_t st = u % kNst;
          pf.mark(6);
          tc::mbar_wait_sleep(tc::smem_u32(&k_full[st]), (u / kNst) & 1);
          pf.mark(1);
          qk(0, st);                                     // QK_A(u)
          if (pendB) {                                   // PV_B(u-1): releases V(u-1)
            pv(1, pendB_u, pendB_first, true);
            if (pendB_first) {}                          // (O_B drain tracked by nIt[1])
            pendB = false;
          }
          if (I.hasB) qk(1, st);                         // QK_B(u)
          tc::mma_commit(tc::smem_u32(&k_empty[st]));    // K(u) read by both QKs
          if (t == I.t1 - 1) tc::mma_commit(tc::smem_u32(q_empty));  // Q blocks reusable
          pv(0, u, t == I.t0, !I.hasB);                  // PV_A(u) (releases V(u) if no B)
          if (I.hasB) {
            pendB = true;
            pendB_u = u;
            pendB_first = t == I.t0;
          }
        }
        ++nIt[0];
        if (I.hasB) {
          // the item's last PV_B before the next item's first QK_A (its O_B drain
          // and the next item's Q both wait on it)
          pv(1, pendB_u, pendB_first, true);
          pendB = false;
          ++nIt[1];
        }
        ++it;
      }
      pf.mark(6);
      pf.dump(P.trace ? P.trace + (size_t)blockIdx.x * 1024 : nullptr, 520);  // (0..40: the fused kernel's)
    }
  } else if (warp == 2 || warp == 3) {
    // ============ V converters: bf16 V tile -> f16 * 2^-8 in place (R23) ============
    const int half = warp - 2;
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
    // ============ softmax + epilogue: block x, one thread per row ============
    const int x = (warp - 4) >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // row in the block = TMEM lane
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    const uint32_t tSx = tS + x * 128, tOx = tO + x * 128;
    const float sl2 = P.scale_log2;
    uint32_t n = 0, nit = 0;  // this block's tiles / items
    Prof pf;
    for (int k = blockIdx.x; k < P.items; k += gridDim.x) {
      const Item I = item_of(k);
      const int rb = 2 * I.rp + x;
      const int rg = rb * 128 + r;
      const bool valid_row = I.dec ? r < P.p : rg < P.R;
      BA_CHECK(I.s >= 0 && I.s < P.S && I.c < P.g && (!I.dec || I.i < P.b));
      const int gr = !valid_row ? -1
                     : I.dec ? I.i * P.h + I.c * P.p + r
                             : (rg / P.p) * P.h + I.c * P.p + rg % P.p;
      if (x == 1 && !I.hasB) continue;  // block B is not part of this item
      if (I.t1 == I.t0) {
        // empty decode item (lens = 0): an empty partial (m = -inf, l = 0, o = 0)
        if (valid_row) {
          float* wo = P.ws_o + ((size_t)gr * P.S + I.s) * 128;
#pragma unroll
          for (int e = 0; e < 128; e += 4) *reinterpret_cast<float4*>(wo + e) = make_float4(0.f, 0.f, 0.f, 0.f);
          reinterpret_cast<float2*>(P.ws_ml)[(size_t)gr * P.S + I.s] = make_float2(kNegInf, 0.f);
        }
        continue;
      }
      const int Lrow = I.dec && P.ntok > 1 ? max(I.L - (P.ntok - 1 - r % P.ntok), 0) : I.L;
      float m = kNegInf, l = 0.f;
      pf.mark(0);
      for (int t = I.t0; t < I.t1; ++t, ++n) {
        tc::mbar_wait(tc::smem_u32(&s_full[x]), n & 1);
        pf.mark(1);
        tc::tc_fence_after();
        float xs[128];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          tc::tmem_ld<32>(tSx + q * 32 + lane_addr, reinterpret_cast<uint32_t*>(xs) + q * 32);
        tc::tmem_ld_wait();
        pf.mark(2);
        // row max on the raw logits (the scale is positive), 8 chains
        const int nvalid = min(128, Lrow - t * 128);
        float mq[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) mq[e] = kNegInf;
        if (nvalid >= 128) {
#pragma unroll
          for (int i = 0; i < 128; ++i) mq[i & 7] = fmaxf(mq[i & 7], xs[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 128; ++i) {
            xs[i] = i < nvalid ? xs[i] : kNegInf;
            mq[i & 7] = fmaxf(mq[i & 7], xs[i]);
          }
        }
        const float mx = fmaxf(fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])),
                               fmaxf(fmaxf(mq[4], mq[5]), fmaxf(mq[6], mq[7]))) * sl2;
        pf.mark(3);
        if (m == kNegInf || mx > m + kTh) {
          // raise the reference to the exact max; rescale l and the O row (PV(u-1)
          // of this block completed before QK(u) was issued: O is quiescent)
          if (m != kNegInf && t > I.t0) {
            const float a = ex2(m - mx);
            l *= a;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              uint32_t o[8];
              tc::tmem_ld<8>(tOx + q * 8 + lane_addr, o);
              tc::tmem_ld_wait();
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * a);
              tc::tmem_st<8>(tOx + q * 8 + lane_addr, o);
            }
            tc::tmem_st_wait();
          }
          m = mx;
        }
        pf.mark(5);
        const float mref = m == kNegInf ? 0.f : m;
        const float2 sl2v = make_float2(sl2, sl2), nmv = make_float2(-mref, -mref);
        float2 lq[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint32_t hk[8];
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const float2 z = fma2(make_float2(xs[j * 16 + e], xs[j * 16 + e + 1]), sl2v, nmv);
            const float2 pz = make_float2(ex2(z.x), ex2(z.y));
            lq[(e >> 1) & 1] = add2(lq[(e >> 1) & 1], pz);
            hk[e / 2] = pack_f16x2(pz.x, pz.y);
          }
          tc::tmem_st<8>(tSx + j * 8 + lane_addr, hk);
        }
        l += (lq[0].x + lq[0].y) + (lq[1].x + lq[1].y);
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(tc::smem_u32(&p_full[x]));
        pf.mark(6);
      }
      // ---- the item's partial: O row (relative to 2^m), m, l ----
      tc::mbar_wait(tc::smem_u32(&pv_done[x]), (n - 1) & 1);  // this block's last PV
      tc::tc_fence_after();
      float* wo = valid_row ? P.ws_o + ((size_t)gr * P.S + I.s) * 128 : nullptr;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t o[32];
        tc::tmem_ld<32>(tOx + q * 32 + lane_addr, o);
        tc::tmem_ld_wait();
        if (valid_row) {
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            *reinterpret_cast<float4*>(wo + q * 32 + e) =  // undo V * 2^-8 (exact)
                make_float4(__uint_as_float(o[e]) * 256.f, __uint_as_float(o[e + 1]) * 256.f,
                            __uint_as_float(o[e + 2]) * 256.f, __uint_as_float(o[e + 3]) * 256.f);
        }
      }
      if (valid_row) reinterpret_cast<float2*>(P.ws_ml)[(size_t)gr * P.S + I.s] = make_float2(m, l);
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(&o_empty[x]));
      ++nit;
      pf.mark(7);
    }
    if (threadIdx.x == 128) pf.dump(P.trace ? P.trace + (size_t)blockIdx.x * 1024 : nullptr, 512);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

}  // namespace ba
