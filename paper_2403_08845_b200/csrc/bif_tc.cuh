// bif_tc.cuh — one incremental-decoding step of context-aware bifurcated
// attention on the 5th-gen tensor cores (tcgen05 + TMEM + TMA), sm_100a:
// ONE cooperative persistent kernel (bif_tc_kernel): stream + grid barrier +
// LSE merge.
//
// What it computes (Eq. 3-4; App. E.3):
//   context segments:  the R = b*p query rows of group c that share Kc[c] and
//                      Vc[c] (no batch axis) against a run
//                      of 128-position context tiles — each context tile is
//                      read from HBM once for all b samples;
//   decode segments:   the rows of sample i for a block of gpc = N/p groups
//                      against the 128-position tiles of Kd[i][c]/Vd[i][c]
//                      (PAPER.md:255, :267), group after group — i.e. in
//                      memory order of the [b][g][md][d] cache; a tile of
//                      group c only feeds the p columns of group c (others
//                      masked), positions masked at lens[i];
//   merge:             every row's partials (m, l, o) joined with one
//                      log-sum-exp — the single softmax over S_c ⊕ S_d
//                       split at mc and summed (Eq. 4).
//
// Tile math (swap-AB: query rows are few, positions many):
//   S^T[128 pos x N]  = K_tile[128 x d] . q_chunk^T[d x N]    (M=128, K=d=128)
//   O^T[d x N]       += V_tile^T[d x 128] . P^T[128 x N]       (M=d=128, K=128)
// K/V tiles arrive by TMA (128B swizzle) in an NST-stage ring; S^T (2 slots)
// and O^T (2 buffers) live in TMEM; P (bf16) goes through shared memory.
//
// Warp roles (1 CTA per SM):
//   warp 0            TMA producer (one lane)
//   warp 1            QK issuer (one lane): QK(u) when its K tile, q and an
//                     S slot are ready
//   warp 2            TMEM allocator
//   warp 3            PV issuer (one lane): PV(u) when P(u) is ready
//   warps 4..4+4W-1   softmax (W warpgroups): warp w reads TMEM lanes
//                     32*(w%4).. (= tile positions), CPT = N/W columns
//   last 4 warps      epilogue: drains O^T of a finished segment from TMEM to
//                     the workspace while the softmax warps run the next one
//
// Online softmax with a stale-max fast path: P = 2^(s*scale*log2e - m_run);
// only when a valid logit exceeds m_run by more than kTh, or a column sees its
// first valid logit (m_run unset), do the softmax warps (vote: bar.red.or)
// compute the exact tile max per column and raise m_run — rescaling l and
// O^T only for columns whose max actually grew.  Same softmax; P <= 2^kTh.
//
// Work split: flat tiles f in [0, Tc + Td): context tiles first, in units
// (c, band, rc) of bw tiles (ctx_unit; one band = f = (c*nrc + rc)*ntile_c + t
// when nrc = 1), then decode tiles in Kd memory order,
// f = Tc + (i*g + c)*ntile_d + t.  CTA k streams the contiguous range
// [cs[k], cs[k+1]) planned on the host (bifattn_api.cu, plan_split): equal
// 64 KB-tile counts, except that a range crossing into another chunk is
// charged a segment-switch penalty and boundaries snap to chunk ends when
// close.  A maximal run of tiles of one context chunk (c, rc) or one decode
// chunk (i, cb) is a segment and writes one partial (m, l, o) for every row
// of its chunk to its workspace slot (context slots [0, Sc), decode slots
// [Sc, S)).
#pragma once
#include "append.cuh"
#include "common.cuh"
#include "tc_ptx.cuh"

namespace ba {

constexpr int bif_max_ctas = 160;

struct BifTcParams {
  CUtensorMap tmKc, tmVc;  // Kc/Vc as 3D (d, mc, g), box (64, 128, 1), SW128
  CUtensorMap tmQc;        // q as 3D (d, h, b), box (64, p, N/p), SW128
  CUtensorMap tmKd, tmVd;  // Kd/Vd as 3D (d, dec_stride, b*g), box (64, 128, 1)
  CUtensorMap tmQd;        // q as 3D (d, h, b), box (64, min(N, h), 1), SW128
  CUtensorMap tmQ1;        // dyn: q as 3D (d, h, b), box (64, p, 1) — the p query rows of a column
  const int32_t* lens;
  // dyn = 1: the decode branch is NOT in the static tile ranges; after its
  // static (context) range every CTA takes decode columns (sample i, group c),
  // col = i*g + c < ncol = b*g, from the grid-wide counter *col_ctr and its
  // softmax warps compute them on the CUDA cores (p = 1, 2 or 4 query rows per
  // column — a GEMV, not an MMA tile).  One decode partial per row (slot Sc).
  int dyn, ncol;
  // a column's tiles are cut into dparts parts of dunit tiles (the queue hands
  // out (column, part) units, unit = col * dparts + part; part k writes decode
  // slot Sc + k, an empty partial when it starts past the column's length):
  // enough units to balance the CTAs when columns are few or long
  int dparts, dunit;
  unsigned* col_ctr;       // grid_ctr + 2 (reset to 0 by the grid barrier's last arriver)
  int b, h, g, p, mc;
  int dec_cap, lens_offset;  // decode length = lens_offset + clamp(lens[i], 0, dec_cap)
  int lens_add;              // append+attend: lens[i] counts the cache BEFORE this step's n
                             // appended rows; the step sees min(lens[i] + lens_add, dec_cap)
  int32_t* lens_out;         // append+attend: lens updated in place after the step (or null)
  AppendSrc app;             // append+attend: this step's K/V rows (app.n = 0: none), stored
                             // by the CTA owning the decode tile that holds them (append.cuh)
  int ntok;                  // tokens per head (multi-token step): in-group row k sees decode
                             // positions < max(L - (ntok - 1 - k % ntok), lens_offset)
  int N;                     // rows per chunk (== template N)
  int nrc, ntile_c, ntile_d;
  int bw, nband;             // context band width (tiles) and bands per group (see seg_at)
  int ext_ctx;               // > 0: the context branch ran in ctx_rows_kernel (ctx_rows.cuh),
                             // which wrote ext_ctx context partials per row (slots [0, ext_ctx))
  int spc;                   // samples per context row chunk = N / p
  int gpc, ndc;              // groups per decode chunk = N / p; decode chunks per sample
  int qd_rows;               // rows of the decode q box = min(N, h)
  long long Tc, Td;          // context tiles, decode tiles
  int G, nst;
  int npb;                   // P buffer slots (1 or 2; each a P_hi, P_lo pair)
  int pf_dist;               // L2 prefetch distance in tiles beyond the one being loaded (0: off)
  int rot;                   // context segments start at tile (blockIdx*rot) mod length (0: in order)
  int cs[bif_max_ctas + 1];  // CTA k streams flat tiles [cs[k], cs[k+1]) of [context | decode]
  // workspace slot (index among the CTAs sharing the chunk) of CTA k's FIRST
  // segment part; every later segment part of a CTA starts a chunk (slot 0).
  // Planned on the host: a binary search of cs[] in parameter space at the
  // start costs ~8 dependent constant-cache misses before the first TMA.
  int slot0[bif_max_ctas];
  float scale_log2;
  float vscale;              // FP8 KV: out = v_scale * o / l (partials in V-code units); else 1
  int S, Sc;                 // slots per row; decode slots start at Sc
  float* ws_o;               // [b*h][S][128]
  float* ws_ml;              // [b*h][S][2]
  unsigned* grid_ctr;        // grid barrier: 64-bit arrival count at [0, 1] (+256 per launch; zeroed once), [2] col_ctr
  void* out;                 // [b][h][128] bf16
  float* lse;                // [b][h] or null
  unsigned long long* trace; // optional [G][kTraceSlots] globaltimer stamps (instrumentation)
  int dbg;                   // experiment bits (wrong results): 1 skip softmax math,
                             // 4/8 general/narrow P write skips the PV(u-1) wait
};

namespace bif {
constexpr int kD = 128;
constexpr int kBM = 128;            // positions per tile (MMA M)
constexpr int kStageBytes = 65536;  // K tile 32 KB + V tile 32 KB
constexpr float kTh = 8.0f;         // fast-path slack (log2 units)
constexpr int kTraceSlots = 1024;  // per CTA: 4 roles x 256 stamps
constexpr int kNarrowP = 8;         // decode tiles with p <= 8 valid columns take the narrow path

// softmax warpgroups: keep columns per softmax thread <= 32
__host__ __device__ constexpr int softmax_wgs(int N) { return N > 0 ? 2 : 2; }  // measured: 2 beats 1 at N=16/32
__host__ __device__ constexpr int threads(int swg) { return 32 * (8 + 4 * swg); }

__host__ __device__ constexpr int p_atom(int N) { return (N % 64 == 0) ? 64 : ((N % 32 == 0) ? 32 : 16); }
__host__ __device__ constexpr int p_layout(int N) {
  return p_atom(N) == 64 ? tc::kSw128 : (p_atom(N) == 32 ? tc::kSw64 : tc::kSw32);
}
// TMEM: 2 S^T slots (N columns) + 2 O^T buffers (2N: the P_hi and P_lo halves)
__host__ __device__ constexpr int tmem_cols(int N) {
  return 6 * N <= 32 ? 32 : 6 * N <= 64 ? 64 : 6 * N <= 128 ? 128 : 6 * N <= 256 ? 256 : 512;
}
// FP8 KV (KV8): each tile lands by TMA as E4M3 codes (K 16 KB, V 16 KB, SW128
// rows of 128 codes) in the upper half of its own f16 stage region (K codes
// at +16 KB, V codes at +48 KB) and the converter warps expand it IN PLACE
// into the f16 layout the MMAs read: a stage holds codes, then f16.
// dynamic smem besides the stages: 2 q + npb P buffers (256N B per q buffer
// and per P part; P = P_hi | P_lo, or one f16 part with KV8), col-max scratch
// [4][N], row sums [2][4][N], m_run [2][N], final m [2][N] (floats), lengths
// [64] ints, barriers (512 B)
// + 128 B: the merge part counts of each warp's first output row
__host__ __device__ constexpr int smem_fixed(int N, int npb, bool kv8 = false) {
  return (2 + (kv8 ? 1 : 2) * npb) * 256 * N + 4 * (4 * N + 8 * N + 2 * N + 2 * N) + 256 + 512 + 128;
}

// CTA owning flat tile f (the CTA ranges [cs[k], cs[k+1]) are non-empty and
// cover [0, Tc + Td)): binary search of the start table.
__host__ __device__ inline int owner(const int* cs, int G, long long f) {
  int lo = 0, hi = G - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (cs[mid] <= f) lo = mid; else hi = mid - 1;
  }
  return lo;
}
// Number of CTAs that cover flat tiles [a, e) (e > a).
__host__ __device__ inline int parts_of(const int* cs, int G, long long a, long long e) {
  return owner(cs, G, e - 1) - owner(cs, G, a) + 1;
}

struct Seg {
  bool dec;        // decode segment?
  int c, rc;       // context: group, row chunk
  int i, cb;       // decode: sample, group block (groups [cb*gpc, (cb+1)*gpc))
  int t0, c0;      // first tile's position-tile index and (decode) group
  int ntiles;      // tiles in this CTA's part of the segment
  int slot;        // workspace slot of this CTA's partial
  long long next;  // work index (CTA work order) after this segment part
};

BA_DEVINL int dec_len(const BifTcParams& P, int i) {
  int L = P.lens[i];
  L = L < 0 ? 0 : (L > P.dec_cap ? P.dec_cap : L);
  L = min(L + P.lens_add, P.dec_cap);
  return P.lens_offset + L;
}

// This CTA's work: flat tiles [f0, f1) of [context tiles | decode tiles];
// work index w = f - f0.
struct Range {
  long long f0, f1;
  BA_DEVINL long long n() const { return f1 - f0; }
};
BA_DEVINL Range my_range(const BifTcParams& P) {
  Range r;
  r.f0 = P.cs[blockIdx.x];
  r.f1 = P.cs[blockIdx.x + 1];
  return r;
}

// First / one-past-last decode tile of chunk (i, cb).
__host__ __device__ inline long long dec_chunk_begin(long long g, long long gpc, long long ntd,
                                                     int i, int cb) {
  return ((long long)i * g + (long long)cb * gpc) * ntd;
}
__host__ __device__ inline long long dec_chunk_end(long long g, long long gpc, long long ntd, int i,
                                                   int cb) {
  const long long c1 = (long long)(cb + 1) * gpc < g ? (long long)(cb + 1) * gpc : g;
  return ((long long)i * g + c1) * ntd;
}

// Context unit of flat context tile f: the context tiles of group c are cut
// into bands of bw tiles (the last band may be narrower) and ordered
// (c, band, rc, tile): the nrc row chunks of a band follow each other, so a
// CTA re-reads a band's K/V while it is still in L2 (bw = ntile_c: one band,
// the plain (c, rc, tile) order).  Returns the unit's first flat tile and
// width; c, band, rc and the tile index within the group through the refs.
__host__ __device__ inline long long ctx_unit(int nrc, int ntc, int bw, long long f, int& c,
                                             int& band, int& rc, int& tg, int& wb) {
  const long long GT = (long long)nrc * ntc;
  c = (int)(f / GT);
  const long long r = f - (long long)c * GT;
  const int nfull = ntc / bw;
  const long long full = (long long)nfull * nrc * bw;
  long long base;
  int tb;
  if (r < full) {
    band = (int)(r / ((long long)nrc * bw));
    const long long rr = r - (long long)band * nrc * bw;
    wb = bw;
    rc = (int)(rr / bw);
    tb = (int)(rr - (long long)rc * bw);
    base = (long long)band * nrc * bw;
  } else {
    const long long r2 = r - full;
    band = nfull;
    wb = ntc - nfull * bw;
    rc = (int)(r2 / wb);
    tb = (int)(r2 - (long long)rc * wb);
    base = full;
  }
  tg = band * bw + tb;
  return (long long)c * GT + base + (long long)rc * wb;
}

BA_DEVINL Seg seg_at(const BifTcParams& P, const Range& rg, long long w) {
  Seg s;
  const long long f = rg.f0 + w;
  if (f < P.Tc && P.nband <= 1) {
    // one band: chunk (c, rc) = f / ntile_c (the common case, fewer divisions)
    const long long seg = f / P.ntile_c;
    const long long fend = min((seg + 1) * P.ntile_c, rg.f1);
    s.dec = false;
    s.c = (int)(seg / P.nrc);
    s.rc = (int)(seg - (long long)s.c * P.nrc);
    s.i = s.cb = 0;
    s.t0 = (int)(f - seg * P.ntile_c);
    s.c0 = s.c;
    s.ntiles = (int)(fend - f);
    s.slot = w == 0 ? P.slot0[blockIdx.x] : 0;
    s.next = w + (fend - f);
  } else if (f < P.Tc) {
    int c, band, rc, tg, wb;
    const long long u0 = ctx_unit(P.nrc, P.ntile_c, P.bw, f, c, band, rc, tg, wb);
    const long long fend = min(u0 + wb, rg.f1);
    s.dec = false;
    s.c = c;
    s.rc = rc;
    s.i = s.cb = 0;
    s.t0 = tg;
    s.c0 = s.c;
    s.ntiles = (int)(fend - f);
    // banded: the planner never splits a unit, slot = band; else the CTA's
    // index among the CTAs that share the chunk
    s.slot = P.nband > 1 ? band : (w == 0 ? P.slot0[blockIdx.x] : 0);
    s.next = w + (fend - f);
  } else {
    const long long fd = f - P.Tc;
    const long long ic = fd / P.ntile_d;  // i*g + c
    s.dec = true;
    s.i = (int)(ic / P.g);
    s.c0 = (int)(ic % P.g);
    s.cb = s.c0 / P.gpc;
    s.c = s.rc = 0;
    s.t0 = (int)(fd - ic * P.ntile_d);
    const long long fend = min(P.Tc + dec_chunk_end(P.g, P.gpc, P.ntile_d, s.i, s.cb), rg.f1);
    s.ntiles = (int)(fend - f);
    s.slot = P.Sc + (w == 0 ? P.slot0[blockIdx.x] : 0);
    s.next = w + (fend - f);
  }
  return s;
}

// Tile streamed at step j of a context segment: the CTAs' streams start at
// staggered offsets (rotation) so they do not walk the same DRAM pages in step.
BA_DEVINL int ctx_tile(const BifTcParams& P, const Seg& s, int j) {
  if (P.rot == 0 || s.ntiles <= 1) return s.t0 + j;
  return s.t0 + (int)(((unsigned)j + (unsigned)blockIdx.x * (unsigned)P.rot) % (unsigned)s.ntiles);
}

// K/V box coordinates of the CTA's w-th tile: decode?, TMA z, tile index t.
BA_DEVINL void tile_at(const BifTcParams& P, const Range& rg, long long w, bool& dec, int& z, int& t) {
  const long long f = rg.f0 + w;
  if (f < P.Tc) {
    int c, band, rc, tg, wb;
    ctx_unit(P.nrc, P.ntile_c, P.bw, f, c, band, rc, tg, wb);
    dec = false;
    z = c;
    t = tg;
  } else {
    const long long fd = f - P.Tc;
    const long long ic = fd / P.ntile_d;  // i*g + c = the Kd/Vd map's z
    dec = true;
    z = (int)ic;
    t = (int)(fd - ic * P.ntile_d);
  }
}

// Partials written for context chunk (c, rc) / decode chunk (i, cb).
__host__ __device__ inline int ctx_parts(const BifTcParams& P, int c, int rc) {
  if (P.ext_ctx > 0) return P.ext_ctx;
  if (P.Tc == 0) return 0;
  if (P.nband > 1) return P.nband;  // one partial per band (units are never split)
  const long long ff = ((long long)c * P.nrc + rc) * P.ntile_c;
  return parts_of(P.cs, P.G, ff, ff + P.ntile_c);
}
__host__ __device__ inline int dec_parts(const BifTcParams& P, int i, int cb) {
  if (P.dyn) return P.ncol > 0 ? P.dparts : 0;  // one partial per (column, part) unit
  if (P.Td == 0) return 0;
  const long long a = P.Tc + dec_chunk_begin(P.g, P.gpc, P.ntile_d, i, cb);
  const long long e = P.Tc + dec_chunk_end(P.g, P.gpc, P.ntile_d, i, cb);
  return parts_of(P.cs, P.G, a, e);
}

// output row of column col of a segment's chunk, or -1 for padding
BA_DEVINL int row_of(const BifTcParams& P, const Seg& s, int col) {
  if (s.dec) {
    const int j = s.cb * P.gpc * P.p + col;
    return j < P.h ? s.i * P.h + j : -1;
  }
  const int r = s.rc * P.N + col;
  if (r >= P.b * P.p) return -1;
  const int i = r / P.p;
  return i * P.h + s.c * P.p + (r - i * P.p);
}
}  // namespace bif

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

// two bf16 (lo, hi halves of a word) -> float2 (exact)
BA_DEVINL float2 bf16x2_f2(uint32_t w) { return make_float2(bf16lo(w), bf16hi(w)); }
// two f16 (lo, hi) -> float2 (exact)
BA_DEVINL float2 f16x2_f2(uint32_t w) {
  __half2 h;
  h = *reinterpret_cast<const __half2*>(&w);
  return __half22float2(h);
}

// ---------------------------------------------------------------------------
// Dynamic decode columns with PQ = p = 2 or 4 query rows (GQA), CUDA cores.
// Same division of a tile as the p = 1 path (warp sw: positions 16 sw ..
// 16 sw + 15; QK with 2 lanes per position, PV with lane l on d = 4l .. 4l+3),
// but the PQ query rows are read from shared memory as fp32 (converted from
// the column's bf16 q box once per column: broadcast reads, the two d halves
// 16 B apart in bank) and each position's PQ probabilities go through a
// per-warp shared-memory row to the PV lanes.  Per warp and row an exact
// online softmax; at the column's end warps 0..PQ-1 join the NSW partials of
// rows c*p .. c*p + PQ - 1 of sample i (workspace slot Sc).
// ---------------------------------------------------------------------------
namespace bif {
constexpr int kQHalf = 68;  // floats per (row, d half) of the fp32 q: 64 + 16 B of bank padding
__host__ __device__ constexpr int cc_extra_bytes(int pq) {
  return pq > 1 ? (2 * pq * kQHalf * 4 + 8 * 16 * pq * 4 + 127) / 128 * 128 : 0;
}
}  // namespace bif

struct DynSmem {
  uint8_t* stage;        // NST x 64 KB K/V stages
  const uint8_t* q;      // 2 bf16 q buffers of QB bytes (d halves at +0 and +Nq*128)
  int QB, Nq, nst;
  uint64_t *kv_full, *kv_empty, *q_full, *q_empty;
  const int2* ring;      // (column, length) per q buffer
  float* scr_o;          // [NSW][PQ][128] warp partials (the idle P buffer)
  float* scr_ml;         // [NSW][PQ][2]
  float* qf;             // [PQ][2][kQHalf] fp32 query rows
  float* pex;            // [NSW][16][PQ] probabilities of the warp's positions
};

template <int PQ, int NSW>
BA_DEVINL void dyn_cc_multi(const BifTcParams& P, const DynSmem& S, int sw, int lane, uint32_t& u,
                            uint32_t& sg) {
  constexpr int kD = bif::kD, kBM = bif::kBM;
  const int hf = lane >> 4;
  const int pp = 16 * sw + (lane & 15);
  const int vch = (lane & 15) >> 1, vsub = (lane & 1) * 8;
  const float sl2 = P.scale_log2;
  const int tid = sw * 32 + lane;  // 0 .. 32 NSW - 1
  for (;; ++sg) {
    const uint32_t qb = sg & 1;
    tc::mbar_wait(tc::smem_u32(&S.q_full[qb]), (sg >> 1) & 1);
    const int unit = reinterpret_cast<const volatile int*>(S.ring + qb)[0];
    if (unit < 0) break;
    const int Lc = reinterpret_cast<const volatile int*>(S.ring + qb)[1];
    const int col = unit / P.dparts, part = unit - col * P.dparts;
    const int t0 = part * P.dunit;
    // q rows (bf16, SW128 box rows) -> fp32 [r][half][kQHalf]: one 16-byte chunk per thread
    if (tid < PQ * 16) {
      const int r = tid >> 4, h2 = (tid >> 3) & 1, ch = tid & 7;
      const uint4 v = *reinterpret_cast<const uint4*>(S.q + qb * S.QB + h2 * (S.Nq * 128) + r * 128 +
                                                      ((ch ^ (r & 7)) << 4));
      float* const dst = S.qf + (r * 2 + h2) * bif::kQHalf + ch * 8;
      *reinterpret_cast<float4*>(dst) = make_float4(bf16lo(v.x), bf16hi(v.x), bf16lo(v.y), bf16hi(v.y));
      *reinterpret_cast<float4*>(dst + 4) = make_float4(bf16lo(v.z), bf16hi(v.z), bf16lo(v.w), bf16hi(v.w));
    }
    // (also orders the previous column's joins before this column's partial writes)
    tc::named_bar_sync(2, 32 * NSW);
    if (tid == 0) tc::mbar_arrive(tc::smem_u32(&S.q_empty[qb]));  // bf16 q no longer read
    float m_w[PQ], l_w[PQ];
    float4 o[PQ];
#pragma unroll
    for (int r = 0; r < PQ; ++r) {
      m_w[r] = kNegInf;
      l_w[r] = 0.f;
      o[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float* const pw = S.pex + sw * 16 * PQ;
    const int nt = min((Lc + kBM - 1) / kBM, t0 + P.dunit);
    for (int t = t0; t < nt; ++t, ++u) {
      const uint32_t st = u % S.nst;
      tc::mbar_wait(tc::smem_u32(&S.kv_full[st]), (u / S.nst) & 1);
      const uint8_t* const stage = S.stage + st * bif::kStageBytes;
      // ---- PQ logits of position pp (this lane's d half, then the other) ----
      const uint8_t* const krow = stage + hf * 16384 + pp * 128;
      float2 a[PQ];
#pragma unroll
      for (int r = 0; r < PQ; ++r) a[r] = make_float2(0.f, 0.f);
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const uint4 kv = *reinterpret_cast<const uint4*>(krow + ((ch ^ (pp & 7)) << 4));
        const float2 k0 = bf16x2_f2(kv.x), k1 = bf16x2_f2(kv.y), k2 = bf16x2_f2(kv.z), k3 = bf16x2_f2(kv.w);
#pragma unroll
        for (int r = 0; r < PQ; ++r) {
          const float* const qr = S.qf + (r * 2 + hf) * bif::kQHalf + ch * 8;
          const float4 qa = *reinterpret_cast<const float4*>(qr);
          const float4 qc = *reinterpret_cast<const float4*>(qr + 4);
          ffma2(a[r], k0, make_float2(qa.x, qa.y));
          ffma2(a[r], k1, make_float2(qa.z, qa.w));
          ffma2(a[r], k2, make_float2(qc.x, qc.y));
          ffma2(a[r], k3, make_float2(qc.z, qc.w));
        }
      }
      const bool valid = t * kBM + pp < Lc;
      float pe[PQ];
#pragma unroll
      for (int r = 0; r < PQ; ++r) {
        float sdot = a[r].x + a[r].y;
        sdot += __shfl_xor_sync(0xffffffffu, sdot, 16);
        const float x = valid ? sdot * sl2 : kNegInf;
        float mt = x;
#pragma unroll
        for (int off = 8; off >= 1; off >>= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, off));
        const float mn = fmaxf(m_w[r], mt);
        const float mref = (mn == kNegInf) ? 0.f : mn;
        const float alpha = ex2(m_w[r] - mref);
        l_w[r] *= alpha;
        o[r].x *= alpha; o[r].y *= alpha; o[r].z *= alpha; o[r].w *= alpha;
        m_w[r] = mn;
        pe[r] = ex2(x - mref);
        l_w[r] += hf ? 0.f : pe[r];
      }
      // this warp's probabilities [position][row] for the PV lanes
      if (hf == 0) {
        if constexpr (PQ == 4)
          *reinterpret_cast<float4*>(pw + (lane & 15) * 4) = make_float4(pe[0], pe[1], pe[2], pe[3]);
        else
          *reinterpret_cast<float2*>(pw + (lane & 15) * 2) = make_float2(pe[0], pe[1]);
      }
      __syncwarp();
      // ---- o[r] += p[r] . V over the warp's valid positions (lane: d = 4 lane ..) ----
      const uint8_t* const vb = stage + 32768 + hf * 16384 + vsub;
      const int nv = min(max(Lc - (t * kBM + 16 * sw), 0), 16);
      for (int k = 0; k < nv; ++k) {
        const int rr = 16 * sw + k;
        const uint2 v = *reinterpret_cast<const uint2*>(vb + rr * 128 + ((vch ^ (rr & 7)) << 4));
        const float2 v0 = bf16x2_f2(v.x), v1 = bf16x2_f2(v.y);
        float pk[PQ];
        if constexpr (PQ == 4) {
          const float4 p4 = *reinterpret_cast<const float4*>(pw + k * 4);
          pk[0] = p4.x; pk[1] = p4.y; pk[2] = p4.z; pk[3] = p4.w;
        } else {
          const float2 p2 = *reinterpret_cast<const float2*>(pw + k * 2);
          pk[0] = p2.x; pk[1] = p2.y;
        }
#pragma unroll
        for (int r = 0; r < PQ; ++r) {
          float2 lo = make_float2(o[r].x, o[r].y), hi = make_float2(o[r].z, o[r].w);
          ffma2(lo, v0, make_float2(pk[r], pk[r]));
          ffma2(hi, v1, make_float2(pk[r], pk[r]));
          o[r] = make_float4(lo.x, lo.y, hi.x, hi.y);
        }
      }
      __syncwarp();  // every lane's stage and pex reads are done
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(&S.kv_empty[st]));  // 1 of NSW
    }
    // ---- join the NSW warp partials of each of the PQ rows ----
#pragma unroll
    for (int r = 0; r < PQ; ++r) {
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) l_w[r] += __shfl_xor_sync(0xffffffffu, l_w[r], off);
      *reinterpret_cast<float4*>(S.scr_o + (sw * PQ + r) * kD + 4 * lane) = o[r];
      if (lane == 0) *reinterpret_cast<float2*>(S.scr_ml + (sw * PQ + r) * 2) = make_float2(m_w[r], l_w[r]);
    }
    tc::named_bar_sync(2, 32 * NSW);
    if (sw < PQ) {
      const int r = sw;
      float M = kNegInf;
#pragma unroll
      for (int w2 = 0; w2 < NSW; ++w2) M = fmaxf(M, S.scr_ml[(w2 * PQ + r) * 2]);
      const float Ms = (M == kNegInf) ? 0.f : M;
      float4 od = make_float4(0.f, 0.f, 0.f, 0.f);
      float ls = 0.f;
#pragma unroll
      for (int w2 = 0; w2 < NSW; ++w2) {
        const float wt = ex2(S.scr_ml[(w2 * PQ + r) * 2] - Ms);
        const float4 v = *reinterpret_cast<const float4*>(S.scr_o + (w2 * PQ + r) * kD + 4 * lane);
        od.x = fmaf(wt, v.x, od.x); od.y = fmaf(wt, v.y, od.y);
        od.z = fmaf(wt, v.z, od.z); od.w = fmaf(wt, v.w, od.w);
        ls = fmaf(wt, S.scr_ml[(w2 * PQ + r) * 2 + 1], ls);
      }
      const int i = col / P.g, c = col - i * P.g;
      const size_t gr = (size_t)i * P.h + c * PQ + r;
      BA_CHECK(gr < (size_t)P.b * P.h && P.Sc + part < P.S && (c + 1) * PQ <= P.h);
      *reinterpret_cast<float4*>(P.ws_o + (gr * P.S + P.Sc + part) * kD + 4 * lane) = od;
      if (lane == 0) reinterpret_cast<float2*>(P.ws_ml)[gr * P.S + P.Sc + part] = make_float2(M, ls);
    }
  }
}

BA_DEVINL unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

BA_DEVINL bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

// Butterfly transpose-reduce over the 32 lanes of a warp: v[CPT] per lane ->
// lane l holds in v[0] the max / sum of column (l % CPT) over all 32 lanes.
// CPT-1 (+ log2(32/CPT)) shuffles instead of 5*CPT.  CPT a power of two <= 32.
template <int CPT, bool kMax>
BA_DEVINL void warp_col_reduce_pow2(float* v, int lane) {
#pragma unroll
  for (int w = CPT / 2; w >= 1; w >>= 1) {
    const bool upper = lane & w;  // lanes with bit w set keep columns [w, 2w)
#pragma unroll
    for (int k = 0; k < w; ++k) {
      const float send = upper ? v[k] : v[k + w];
      const float keep = upper ? v[k + w] : v[k];
      const float got = __shfl_xor_sync(0xffffffffu, send, w);
      v[k] = kMax ? fmaxf(keep, got) : keep + got;
    }
  }
#pragma unroll
  for (int off = CPT; off < 32; off <<= 1) {
    const float got = __shfl_xor_sync(0xffffffffu, v[0], off);
    v[0] = kMax ? fmaxf(v[0], got) : v[0] + got;
  }
}
template <int CPT, bool kMax>
BA_DEVINL void warp_col_reduce(float* v, int lane) {
  if constexpr ((CPT & (CPT - 1)) == 0) {
    warp_col_reduce_pow2<CPT, kMax>(v, lane);
  } else {
    float keep = kMax ? kNegInf : 0.f;
#pragma unroll
    for (int n = 0; n < CPT; ++n) {
      float a = v[n];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        const float got = __shfl_xor_sync(0xffffffffu, a, off);
        a = kMax ? fmaxf(a, got) : a + got;
      }
      if (lane == n) keep = a;
    }
    v[0] = keep;
  }
}

// ----------------------------------------------------------------------------
// LSE merge of one output row gr (one warp): join its context partials
// [0, nctx) and decode partials [Sc, Sc + ndec) with one log-sum-exp.
// (m is in log2 units; l and o are relative to 2^m.)
// ----------------------------------------------------------------------------
BA_DEVINL void merge_row(const BifTcParams& P, int gr, int lane, int nctx, int ndec) {
  const int n = nctx + ndec;
  BA_CHECK(gr >= 0 && gr < P.b * P.h && nctx <= P.Sc && P.Sc + ndec <= P.S);
  const float2* ml = reinterpret_cast<const float2*>(P.ws_ml) + (size_t)gr * P.S;
  const float* obuf = P.ws_o + (size_t)gr * P.S * bif::kD;
  float M = kNegInf, Lsum = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  // running-max merge over batches of 8 partials; every load of a batch is
  // issued before any is used (one L2 round trip per batch)
  for (int q0 = 0; q0 < n; q0 += 8) {
    float2 mv[8];
    float4 ov[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int q = q0 + k;
      if (q < n) {
        const int sl = q < nctx ? q : P.Sc + q - nctx;
        mv[k] = __ldcg(ml + sl);
        ov[k] = __ldcg(reinterpret_cast<const float4*>(obuf + (size_t)sl * bif::kD) + lane);
      }
    }
    float Mb = M;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (q0 + k < n) Mb = fmaxf(Mb, mv[k].x);
    const float Ms = (Mb == kNegInf) ? 0.f : Mb;
    const float a = (M == kNegInf) ? 0.f : ex2(M - Ms);
    Lsum *= a;
    acc.x *= a; acc.y *= a; acc.z *= a; acc.w *= a;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (q0 + k < n) {
        const float wgt = ex2(mv[k].x - Ms);
        Lsum = fmaf(wgt, mv[k].y, Lsum);
        acc.x = fmaf(wgt, ov[k].x, acc.x);
        acc.y = fmaf(wgt, ov[k].y, acc.y);
        acc.z = fmaf(wgt, ov[k].z, acc.z);
        acc.w = fmaf(wgt, ov[k].w, acc.w);
      }
    }
    M = Mb;
  }
  const float inv = P.vscale / Lsum;
  const uint2 packed = make_uint2(pack_bf16x2(acc.x * inv, acc.y * inv),
                                  pack_bf16x2(acc.z * inv, acc.w * inv));
  *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(P.out) + (size_t)gr * bif::kD + lane * 4) = packed;
  if (P.lse && lane == 0) P.lse[gr] = (M + lg2(Lsum)) * kLn2;
}

// Cycle accounting for experiments (BIFATTN_PROF builds only): per-role
// accumulators of where time goes, dumped into the trace buffer at exit.
#ifdef BIFATTN_PROF
BA_DEVINL unsigned long long prof_clock() {
  unsigned long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
struct Prof {
  unsigned long long acc[8];
  unsigned long long last;
  __device__ Prof() : last(prof_clock()) {
    for (int k = 0; k < 8; ++k) acc[k] = 0;
  }
  BA_DEVINL void mark(int k) {
    const unsigned long long now = prof_clock();
    acc[k] += now - last;
    last = now;
  }
  BA_DEVINL void count(int k) { acc[k] += 1; }
  BA_DEVINL void dump(unsigned long long* tr, int base) {
    if (tr)
      for (int k = 0; k < 8; ++k) tr[base + k] = acc[k];
  }
};
constexpr bool kStamp = false;
#else
#ifdef BIFATTN_TRACE
constexpr bool kStamp = true;  // timeline stamps (experiment builds only)
#else
constexpr bool kStamp = false;
#endif
struct Prof {
  BA_DEVINL void mark(int) {}
  BA_DEVINL void count(int) {}
  BA_DEVINL void dump(unsigned long long*, int) {}
};
#endif

// Experiment bits (BifTcParams::dbg) exist only in BIFATTN_EXPERIMENTS builds;
// the product kernel sees a constant 0 and carries none of their branches.
#ifdef BIFATTN_EXPERIMENTS
#define BIF_DBG (P.dbg)
#else
#define BIF_DBG 0
#endif

// MT: multi-token step (P.ntok > 1) — the decode paths carry the per-column
// intra-step causal bound; compiled out of the single-token kernel (it cost
// ~1.5 us per C2b step in registers and issue slots).
// KV8: FP8 E4M3 KV cache (f4, reading R19) — the epilogue warps also expand
// each TMA-landed code tile into an f16 stage and convert q to f16 in place;
// P enters the PV MMA as ONE f16 operand (11 significant bits, the split is
// not needed), so O^T has N columns.
template <int N, int SWG, bool MT, bool KV8 = false>
__global__ void __launch_bounds__(32 * (8 + 4 * SWG), 1)
    bif_tc_kernel(const __grid_constant__ BifTcParams P) {
  using namespace bif;
  constexpr int NSW = 4 * SWG;               // softmax warps
  constexpr int CPT = N / SWG;               // columns per softmax thread
  constexpr int EPI0 = 4 + NSW;              // first epilogue warp
  constexpr int NP = KV8 ? N : 2 * N;        // P / O^T width: [P_hi | P_lo] columns (KV8: P)
  constexpr int W = p_atom(NP);
  constexpr int PRB = 2 * W;
  constexpr int PLBO = kBM * PRB;
  constexpr int PSWM = W == 64 ? 7 : (W == 32 ? 3 : 1);
  constexpr uint32_t IDESC_QK = KV8 ? tc::idesc_f16(128, N, 0, 0) : tc::idesc_bf16(128, N, 0, 0);
  constexpr uint32_t IDESC_PV = KV8 ? tc::idesc_f16(128, NP, 1, 1) : tc::idesc_bf16(128, NP, 1, 1);
  // KV8: + the f16 K tiles of the NST stages in TMEM (64 columns each), the
  // QK MMA's A operand
  constexpr uint32_t TMEM_COLS = KV8 ? 512 : tmem_cols(N);
  constexpr int QB = 256 * N;  // bytes of one q buffer / one P part
  constexpr int PB = KV8 ? QB : 2 * QB;  // bytes of one P slot
  static_assert(N % 16 == 0 && N >= 16 && N <= 64 && CPT % 8 == 0 && CPT <= 32, "N");

  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x == 0 && (reinterpret_cast<uintptr_t>(smem) & 1023)) __trap();  // SW128 needs 1 KB
  const int NST = P.nst;
  uint8_t* sm_stage = smem;
  uint8_t* sm_q = smem + NST * kStageBytes;  // 2 buffers
  uint8_t* sm_p = sm_q + 2 * QB;             // npb slots of (P_hi, P_lo) / P
  float* sm_red = reinterpret_cast<float*>(sm_p + P.npb * PB);  // [4][N] col max (slow path)
  float* sm_l = sm_red + 4 * N;                             // [2][4][N] row sums per O buffer
  float* sm_mold = sm_l + 8 * N;                            // [N] running max before a slow path
  float* sm_mfin = sm_mold + 2 * N;                         // [2][N] final max per O buffer
  int* sm_len = reinterpret_cast<int*>(sm_mfin + 2 * N);    // [64] decode lengths of the chunk
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm_len + 64);
  uint64_t* kv_full = bars;        // [8]
  uint64_t* kv_empty = bars + 8;   // [8]
  uint64_t* q_full = bars + 16;    // [2]
  uint64_t* q_empty = bars + 18;   // [2]
  uint64_t* s_full = bars + 20;    // [2]
  uint64_t* s_free = bars + 22;    // [2]
  uint64_t* p_full = bars + 24;    // [2]
  uint64_t* p_empty = bars + 26;   // [2]
  uint64_t* o_full = bars + 28;    // [2]  last PV of a segment done
  uint64_t* o_empty = bars + 30;   // [2]  epilogue drained the O buffer
  uint64_t* e_full = bars + 32;    // [2]  softmax wrote row sums / final max
  uint64_t* e_empty = bars + 34;   // [2]  epilogue consumed them
  uint64_t* k_cvt = bars + 36;     // [4]  KV8: K of the stage converted to f16
  uint64_t* v_cvt = bars + 40;     // [4]  KV8: V of the stage converted to f16
  uint64_t* q_cvt = bars + 44;     // [2]  KV8: q converted to f16
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 48);
  int* sm_mcnt = reinterpret_cast<int*>(bars + 64);  // [16 warps][2]: merge part counts

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // every shared-memory region this plan uses lies inside the launch's allocation
  BA_CHECK(threadIdx.x != 0 ||
           (uint32_t)(reinterpret_cast<uint8_t*>(bars + 64) + 128 - smem) +
                   (uint32_t)(P.dyn && P.p > 1 ? bif::cc_extra_bytes(P.p) : 0) <= dyn_smem_bytes());
  auto tstamp = [&](int slot, unsigned long long tag) {
    if (kStamp && P.trace) P.trace[(size_t)blockIdx.x * kTraceSlots + slot] = (gtimer() & 0x00ffffffffffffffull) | (tag << 56);
#ifdef BIFATTN_PROF
    if (P.trace) P.trace[(size_t)blockIdx.x * kTraceSlots + 48 + (slot - 250)] = prof_clock();
#endif
  };
  if (threadIdx.x == 0) tstamp(250, 50);
  const int rows = P.b * P.h;
  const int r0 = (int)((long long)blockIdx.x * rows / P.G);
  const int r1 = (int)((long long)(blockIdx.x + 1) * rows / P.G);

  if (threadIdx.x < 46) {
    // one mbarrier per thread (bars[t]; a serial init of ~40 barriers by one
    // thread cost ~0.5 us of the prologue): arrival counts by role
    const int t = threadIdx.x;
    uint32_t cnt = 0;
    if (t < 8) cnt = t < NST ? 1 : 0;                              // kv_full
    else if (t < 16) cnt = t - 8 < NST ? NSW : 0;                  // kv_empty: PV commit + NSW-1, or NSW warps (dyn)
    else if (t < 22) cnt = 1;                                      // q_full, q_empty, s_full
    else if (t < 26) cnt = NSW;                                    // s_free, p_full
    else if (t < 30) cnt = 1;                                      // p_empty, o_full
    else if (t < 32) cnt = 4;                                      // o_empty
    else if (t < 34) cnt = 32 * NSW;                               // e_full: every softmax thread
    else if (t < 36) cnt = 128;                                    // e_empty: every epilogue thread
    else if (t < 44) cnt = KV8 && ((t - 36) & 3) < NST ? 4 : 0;    // k_cvt, v_cvt
    else cnt = KV8 ? 4 : 0;                                        // q_cvt
    if (cnt) tc::mbar_init(tc::smem_u32(&bars[t]), cnt);
    tc::fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&P.tmKc);
    tc::prefetch_tmap(&P.tmVc);
    tc::prefetch_tmap(&P.tmQc);
    tc::prefetch_tmap(&P.tmKd);
    tc::prefetch_tmap(&P.tmVd);
    tc::prefetch_tmap(&P.tmQd);
    if (P.dyn) tc::prefetch_tmap(&P.tmQ1);
  }
  if (warp == 2) {
    tc::tmem_alloc(tc::smem_u32(tmem_holder), TMEM_COLS);
    tc::tmem_relinquish();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  // programmatic dependent launch: the prologue above overlapped the previous
  // kernel; wait for it before touching any global memory (the producer warp
  // first plans its first segment from the parameters while the previous
  // kernel drains; measured neutral), and let the next launch start its own
  // prologue
  // decode-only launch after the rows kernel (ext_ctx, no context tiles): it
  // reads nothing the rows kernel writes until the merge, and the rows kernel
  // waited for the previous step before letting this launch start, so its
  // CTAs stream decode columns on the SMs the rows kernel leaves free (a
  // non-cooperative launch) and wait for it only before the grid barrier
  const bool early = P.ext_ctx > 0 && P.Tc == 0;
  if (warp != 0 && !early) pdl_wait();
  pdl_launch_dependents();
  if (threadIdx.x == 0) tstamp(254, 54);
  const uint32_t tmem = *tmem_holder;
  const uint32_t tS = tmem;          // S^T slots at columns [0,N), [N,2N)
  const uint32_t tO = tmem + 2 * N;  // O^T buffers at [2N,4N), [4N,6N): O_hi | O_lo halves
  const uint32_t tK = tmem + 4 * N;  // KV8: f16 K tile of stage st at [tK + 64 st, +64)

  const Range rg = my_range(P);
  const long long nw = rg.n();

  if (warp == 0) {
    // parameter-only planning of the first segment, before the PDL wait
    Seg s_first;
    if (lane == 0 && nw > 0) s_first = seg_at(P, rg, 0);
    const uint64_t pol_c = P.nrc == 1 ? tc::policy_evict_first() : tc::policy_evict_last();
    const uint64_t pol_d = tc::policy_evict_first();
    if (!early) pdl_wait();
    // append+attend: store this step's K/V rows that fall in this CTA's decode
    // tiles before any TMA of them (same CTA: generic stores, then a proxy fence)
    if (P.app.n > 0 && P.Td > 0) {
      for (long long f = max(rg.f0, P.Tc); f < rg.f1; ++f) {
        const long long fd = f - P.Tc;
        const long long ic = fd / P.ntile_d;
        const int t = (int)(fd - ic * P.ntile_d);
        const int i = (int)(ic / P.g), c = (int)(ic - (long long)i * P.g);
        append_rows_warp(P.app, i, c, clamp_len(P.lens, i, P.dec_cap), t * kBM, t * kBM + kBM, lane);
      }
      fence_proxy_async_global();
      __syncwarp();
      fence_proxy_async_global();
    }
    // ============================ TMA producer ============================
    uint32_t p_tt = 0, p_sg = 0;  // tiles / segments issued by the static range
    if (lane == 0) {
      Prof pf;
      uint32_t tt = 0, sg = 0;
      tstamp(240, 60);
      for (long long w = 0; w < nw; ++sg) {
        const Seg s = w == 0 ? s_first : seg_at(P, rg, w);
        if (sg == 0) tstamp(241, 61);
        const uint32_t qbuf = sg & 1;
        if (BIF_DBG & 16384) tc::mbar_wait_sleep(tc::smem_u32(&q_empty[qbuf]), ((sg >> 1) & 1) ^ 1, BIF_DBG & 262144); else tc::mbar_wait(tc::smem_u32(&q_empty[qbuf]), ((sg >> 1) & 1) ^ 1);
        pf.mark(0);
        const uint32_t qb = tc::smem_u32(&q_full[qbuf]);
        const uint32_t qdst = tc::smem_u32(sm_q + qbuf * QB);
        if (!s.dec) {
          tc::mbar_arrive_expect_tx(qb, 2 * N * 128);
          tc::tma_load_3d(qdst, &P.tmQc, qb, 0, s.c * P.p, s.rc * P.spc);
          tc::tma_load_3d(qdst + N * 128, &P.tmQc, qb, 64, s.c * P.p, s.rc * P.spc);
        } else {
          tc::mbar_arrive_expect_tx(qb, 2 * P.qd_rows * 128);
          tc::tma_load_3d(qdst, &P.tmQd, qb, 0, s.cb * P.gpc * P.p, s.i);
          tc::tma_load_3d(qdst + N * 128, &P.tmQd, qb, 64, s.cb * P.gpc * P.p, s.i);
        }
        pf.mark(1);
        if (sg == 0) tstamp(242, 62);
        const CUtensorMap* mk = s.dec ? &P.tmKd : &P.tmKc;
        const CUtensorMap* mv = s.dec ? &P.tmVd : &P.tmVc;
        const uint64_t pol = s.dec ? pol_d : pol_c;
        const int ntl = s.dec ? P.ntile_d : P.ntile_c;
        int t = s.t0, cg = s.c0;
        for (int j = 0; j < s.ntiles; ++j, ++tt) {
          const int z = s.dec ? s.i * P.g + cg : s.c;  // TMA z: group, or sample*g + group
          const int tl = s.dec ? t : ctx_tile(P, s, j);
          if constexpr (KV8) {
            // E4M3 codes of the K and V tiles (128 positions x 128 B rows) into
            // the upper halves of the stage; the converter warps expand in place
            const int st = tt % NST;
            tc::mbar_wait_sleep(tc::smem_u32(&kv_empty[st]), ((tt / NST) & 1) ^ 1);
            const uint32_t bar = tc::smem_u32(&kv_full[st]);
            tc::mbar_arrive_expect_tx(bar, 32768);
            const uint32_t dst = tc::smem_u32(sm_stage + st * kStageBytes);
            tc::tma_load_3d_hint(dst + 16384, mk, bar, 0, tl * kBM, z, pol);
            tc::tma_load_3d_hint(dst + 49152, mv, bar, 0, tl * kBM, z, pol);
          } else {
          const int st = tt % NST;
          tc::mbar_wait_sleep(tc::smem_u32(&kv_empty[st]), ((tt / NST) & 1) ^ 1, BIF_DBG & 262144);
          pf.mark(2);
          if (kStamp && P.trace && tt < 128) P.trace[(size_t)blockIdx.x * kTraceSlots + 256 + tt] = (gtimer() & 0x00ffffffffffffffull) | (30ull << 56);
          const uint32_t bar = tc::smem_u32(&kv_full[st]);
          tc::mbar_arrive_expect_tx(bar, kStageBytes);
          const uint32_t dst = tc::smem_u32(sm_stage + st * kStageBytes);
          tc::tma_load_3d_hint(dst, mk, bar, 0, tl * kBM, z, pol);
          tc::tma_load_3d_hint(dst + 16384, mk, bar, 64, tl * kBM, z, pol);
          tc::tma_load_3d_hint(dst + 32768, mv, bar, 0, tl * kBM, z, pol);
          tc::tma_load_3d_hint(dst + 49152, mv, bar, 64, tl * kBM, z, pol);
          }
          // L2 prefetch pf_dist tiles ahead: more bytes in flight than the ring holds
          if (P.pf_dist > 0) {
            const long long wp = (long long)tt + P.pf_dist;
            if (wp < nw) {
              bool pd;
              int pz, pt;
              tile_at(P, rg, wp, pd, pz, pt);
              const CUtensorMap* pk = pd ? &P.tmKd : &P.tmKc;
              const CUtensorMap* pv = pd ? &P.tmVd : &P.tmVc;
              tc::tma_prefetch_3d(pk, 0, pt * kBM, pz);
              tc::tma_prefetch_3d(pk, 64, pt * kBM, pz);
              tc::tma_prefetch_3d(pv, 0, pt * kBM, pz);
              tc::tma_prefetch_3d(pv, 64, pt * kBM, pz);
            }
          }
          pf.mark(3);
          if (++t == ntl) {
            t = 0;
            ++cg;
          }
        }
        w = s.next;
      }
      pf.dump(P.trace ? P.trace + (size_t)blockIdx.x * kTraceSlots : nullptr, 16);
      p_tt = tt;
      p_sg = sg;
    }
    if constexpr (!MT && NSW == 8) {
      if (P.dyn) {
        // ===== dynamic decode columns (whole warp: lane 0 drives the TMA, the
        // warp stores this step's appended rows) =====
        uint32_t tt = __shfl_sync(0xffffffffu, p_tt, 0), sg = __shfl_sync(0xffffffffu, p_sg, 0);
        int2* const ring = reinterpret_cast<int2*>(bars + 56);  // [2] (column, length) per q buffer
        const unsigned ncol = (unsigned)P.ncol * (unsigned)P.dparts;  // units
        const unsigned gp = (unsigned)P.g * (unsigned)P.dparts;       // units per sample
        // the next unit's id and column length are fetched one unit ahead
        unsigned nxt = 0;
        int nxtL = 0;
        if (lane == 0) {
          nxt = atomicAdd(P.col_ctr, 1u);
          if (nxt < ncol) nxtL = dec_len(P, (int)(nxt / gp));
        }
        for (;; ++sg) {
          const unsigned col = __shfl_sync(0xffffffffu, nxt, 0);
          const int L = __shfl_sync(0xffffffffu, nxtL, 0);
          if (lane == 0 && col < ncol) nxt = atomicAdd(P.col_ctr, 1u);
          const uint32_t qbuf = sg & 1;
          if (lane == 0) tc::mbar_wait_sleep(tc::smem_u32(&q_empty[qbuf]), ((sg >> 1) & 1) ^ 1);
          if (col >= ncol) {  // queue drained: tell the softmax warps
            if (lane == 0) {
              ring[qbuf] = make_int2(-1, 0);
              tc::mbar_arrive(tc::smem_u32(&q_full[qbuf]));
            }
            break;
          }
          const int i = (int)(col / gp);
          const int cp = (int)(col - (unsigned)i * gp);  // c * dparts + part
          const int c = cp / P.dparts, part = cp - c * P.dparts;
          const int t0 = part * P.dunit;
          BA_CHECK(i < P.b && c < P.g && part < P.dparts && L >= 0 && L <= P.lens_offset + P.dec_cap);
          if (P.app.n > 0) {  // append+attend: this unit's new rows before its TMA
            append_rows_warp(P.app, i, c, clamp_len(P.lens, i, P.dec_cap), t0 * kBM,
                             (t0 + P.dunit) * kBM, lane);
            fence_proxy_async_global();
            __syncwarp();
            fence_proxy_async_global();
          }
          if (lane == 0) {
            ring[qbuf] = make_int2((int)col, L);
            const uint32_t qb = tc::smem_u32(&q_full[qbuf]);
            const uint32_t qdst = tc::smem_u32(sm_q + qbuf * QB);
            tc::mbar_arrive_expect_tx(qb, 256 * P.p);
            tc::tma_load_3d(qdst, &P.tmQ1, qb, 0, c * P.p, i);
            tc::tma_load_3d(qdst + N * 128, &P.tmQ1, qb, 64, c * P.p, i);
            const int z = i * P.g + c;
            const int nt = min((L + kBM - 1) / kBM, t0 + P.dunit);
            for (int t = t0; t < nt; ++t, ++tt) {
              const int st = tt % NST;
              tc::mbar_wait_sleep(tc::smem_u32(&kv_empty[st]), ((tt / NST) & 1) ^ 1);
              const uint32_t bar = tc::smem_u32(&kv_full[st]);
              const uint32_t dst = tc::smem_u32(sm_stage + st * kStageBytes);
              if constexpr (KV8) {  // code tiles into the stage's code slots (as the static path)
                tc::mbar_arrive_expect_tx(bar, 32768);
                tc::tma_load_3d_hint(dst + 16384, &P.tmKd, bar, 0, t * kBM, z, pol_d);
                tc::tma_load_3d_hint(dst + 49152, &P.tmVd, bar, 0, t * kBM, z, pol_d);
              } else {
                tc::mbar_arrive_expect_tx(bar, kStageBytes);
                tc::tma_load_3d_hint(dst, &P.tmKd, bar, 0, t * kBM, z, pol_d);
                tc::tma_load_3d_hint(dst + 16384, &P.tmKd, bar, 64, t * kBM, z, pol_d);
                tc::tma_load_3d_hint(dst + 32768, &P.tmVd, bar, 0, t * kBM, z, pol_d);
                tc::tma_load_3d_hint(dst + 49152, &P.tmVd, bar, 64, t * kBM, z, pol_d);
              }
            }
            if (nxt < ncol) nxtL = dec_len(P, (int)(nxt / gp));
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ========================== QK issuer (one lane) ==========================
    // S^T(u) = K_tile(u) . q^T once the tile has landed and the softmax has
    // released the S slot; blocking waits (no spinning on the SM's issue slots).
    if (lane == 0) {
      const uint32_t q_addr = tc::smem_u32(sm_q);
      Prof pf;
      uint32_t u = 0, sg = 0;
      for (long long w = 0; w < nw; ++sg) {
        const Seg s = seg_at(P, rg, w);
        const uint32_t qbase = q_addr + (sg & 1) * QB;
        if (KV8) tc::mbar_wait(tc::smem_u32(&q_cvt[sg & 1]), (sg >> 1) & 1);
        else if (BIF_DBG & 16384) tc::mbar_wait_sleep(tc::smem_u32(&q_full[sg & 1]), (sg >> 1) & 1, BIF_DBG & 262144); else tc::mbar_wait(tc::smem_u32(&q_full[sg & 1]), (sg >> 1) & 1);
        pf.mark(0);
        for (int j = 0; j < s.ntiles; ++j, ++u) {
          const uint32_t st = u % NST;
          const uint32_t slot = u & 1;
          tc::mbar_wait_sleep(tc::smem_u32(KV8 ? &k_cvt[st] : &kv_full[st]), (u / NST) & 1, BIF_DBG & 262144);
          pf.mark(1);
          if (kStamp && P.trace && u < 128)
            P.trace[(size_t)blockIdx.x * kTraceSlots + 256 + 128 + u] = (gtimer() & 0x00ffffffffffffffull) | (33ull << 56);
          if (BIF_DBG & 65536) tc::mbar_wait_sleep(tc::smem_u32(&s_free[slot]), ((u >> 1) & 1) ^ 1, BIF_DBG & 262144); else tc::mbar_wait(tc::smem_u32(&s_free[slot]), ((u >> 1) & 1) ^ 1);
          pf.mark(2);
          tc::tc_fence_after();
          const uint32_t kbase = tc::smem_u32(sm_stage + st * kStageBytes);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint64_t bd = tc::smem_desc(qbase + (k >> 2) * (N * 128) + (k & 3) * 32, 16, 1024, tc::kSw128);
            if constexpr (KV8) {  // A = the f16 K tile in TMEM (8 columns per K step)
              tc::mma_bf16_ts(tS + slot * N, tK + st * 64 + k * 8, bd, IDESC_QK, k > 0 ? 1u : 0u);
            } else {
              const uint64_t ad = tc::smem_desc(kbase + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024, tc::kSw128);
              tc::mma_bf16(tS + slot * N, ad, bd, IDESC_QK, k > 0 ? 1u : 0u);
            }
          }
          tc::mma_commit(tc::smem_u32(&s_full[slot]));
          if (BIF_DBG & 1024) tc::mma_commit(tc::smem_u32(&kv_empty[st]));  // experiment: release at QK
          pf.mark(3);
          if (kStamp && P.trace && u < 256)
            P.trace[(size_t)blockIdx.x * kTraceSlots + 512 + u] = (gtimer() & 0x00ffffffffffffffull) | (31ull << 56);
        }
        tc::mma_commit(tc::smem_u32(&q_empty[sg & 1]));  // q buffer reusable
        w = s.next;
      }
      pf.dump(P.trace ? P.trace + (size_t)blockIdx.x * kTraceSlots : nullptr, 24);
    }
  } else if (warp == 3) {
    // ========================== PV issuer (one lane) ==========================
    // O^T += V_tile^T . P^T once P(u) is in shared memory (and, for a
    // segment's first tile, the epilogue has drained this O buffer).  Its
    // commits release the P buffer and the K/V stage (QK(u) completed before
    // the softmax could produce P(u)).
    if (lane == 0) {
      const uint32_t p_addr = tc::smem_u32(sm_p);
      Prof pf;
      uint32_t u = 0, sg = 0;
      for (long long w = 0; w < nw; ++sg) {
        const Seg s = seg_at(P, rg, w);
        const uint32_t ob = sg & 1;
        if (BIF_DBG & 16384) tc::mbar_wait_sleep(tc::smem_u32(&o_empty[ob]), ((sg >> 1) & 1) ^ 1, BIF_DBG & 262144); else tc::mbar_wait(tc::smem_u32(&o_empty[ob]), ((sg >> 1) & 1) ^ 1);
        pf.mark(0);
        for (int j = 0; j < s.ntiles; ++j, ++u) {
          const uint32_t st = u % NST;
          const uint32_t ps = P.npb == 2 ? (u & 1) : 0, ph = P.npb == 2 ? (u >> 1) : u;
          tc::mbar_wait_sleep(tc::smem_u32(&p_full[ps]), ph & 1, BIF_DBG & 262144);
          if (KV8) tc::mbar_wait_sleep(tc::smem_u32(&v_cvt[st]), (u / NST) & 1);
          pf.mark(1);
          tc::tc_fence_after();
          const uint32_t vbase = tc::smem_u32(sm_stage + st * kStageBytes + 32768);
          // P = P_hi + P_lo (two bf16 parts side by side): one MMA per K step
          // gives [O_hi | O_lo]^T += V^T [P_hi | P_lo]^T, V read once
          const uint32_t pbase = p_addr + ps * PB;
#pragma unroll
          for (int k = 0; k < ((BIF_DBG & 32) ? 0 : 8); ++k) {
            const uint64_t ad = tc::smem_desc(vbase + k * 2048, 16384, 1024, tc::kSw128);
            const uint64_t bd = tc::smem_desc(pbase + k * 16 * PRB, PLBO, 8 * PRB, p_layout(NP));
            tc::mma_bf16(tO + ob * NP, ad, bd, IDESC_PV, (j == 0 && k == 0) ? 0u : 1u);
          }
          tc::mma_commit(tc::smem_u32(&p_empty[ps]));
          if (!(BIF_DBG & 1024)) tc::mma_commit(tc::smem_u32(&kv_empty[st]));
          tc::mbar_arrive_cnt(tc::smem_u32(&kv_empty[st]), NSW - 1);
          pf.mark(2);
          if (kStamp && P.trace && u < 256)
            P.trace[(size_t)blockIdx.x * kTraceSlots + 768 + u] = (gtimer() & 0x00ffffffffffffffull) | (32ull << 56);
        }
        tc::mma_commit(tc::smem_u32(&o_full[ob]));
        w = s.next;
      }
      pf.dump(P.trace ? P.trace + (size_t)blockIdx.x * kTraceSlots : nullptr, 32);
    }
  } else if (warp >= 4 && warp < EPI0) {
    // ========================= softmax (NSW warps) ==========================
    const int sw = warp - 4;
    const int quad = warp & 3;
    const int col0 = (sw >> 2) * CPT;
    const int pos = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    const float sl2 = P.scale_log2;
    uint32_t u = 0, sg = 0;
    unsigned long long* tr = P.trace ? P.trace + (size_t)blockIdx.x * kTraceSlots : nullptr;
    int ntr = 0;
    auto stamp = [&](unsigned long long tag) {
      if (kStamp && tr && threadIdx.x == 128 && ntr < 256) tr[ntr++] = (gtimer() & 0x00ffffffffffffffull) | (tag << 56);
    };
    stamp(1);
    Prof pf;
    // valid positions of a segment's sequence; decode lengths are prefetched one
    // segment ahead so no global-load latency sits on a segment boundary
    auto seg_len = [&](const Seg& q) { return q.dec ? dec_len(P, q.i) : P.mc; };
    int L = nw > 0 ? seg_len(seg_at(P, rg, 0)) : 0;
    for (long long w = 0; w < nw; ++sg) {
      const Seg s = seg_at(P, rg, w);
      const int Ln = s.next < nw ? seg_len(seg_at(P, rg, s.next)) : 0;  // used next segment
      const uint32_t ob = sg & 1;
      const uint32_t tOb = tO + ob * NP;
      int t = s.t0, cl = s.c0 - s.cb * P.gpc;  // tile index, group within the decode chunk
      const int ntl = s.dec ? P.ntile_d : P.ntile_c;
#ifdef BIFATTN_NO_NARROW
      if (false) {  // A/B variant: decode tiles through the general path
#else
      if (s.dec && P.p <= kNarrowP) {
#endif
        // ====== narrow decode path: a tile of group c feeds only its p columns ======
        // Half-0 warps (one per TMEM lane quadrant) handle the p valid columns
        // with an exact per-tile max; half-1 warps only keep the barriers.
        const bool h0 = sw < 4;
        float* nred = reinterpret_cast<float*>(sm_len);  // [2 slots][4 quads][kNarrowP]
        bool e_waited = false;
        const int cfirst = cl;
        // first column of the group whose P a slot holds (-1: arbitrary data,
        // e.g. from a context segment): the other columns of a slot stay zero
        // from tile to tile, so only a group switch re-zeroes p columns
        int pcol0 = -1, pcol1 = -1;
        float m_g[kNarrowP], l_g[kNarrowP];
#pragma unroll
        for (int k = 0; k < kNarrowP; ++k) {
          m_g[k] = kNegInf;
          l_g[k] = 0.f;
        }
        for (int j = 0; j < s.ntiles; ++j, ++u) {
          const int cv0 = cl * P.p;
          const uint32_t slot = u & 1;
          const uint32_t ps = P.npb == 2 ? (u & 1) : 0, ph = P.npb == 2 ? (u >> 1) : u;  // P slot, its phase
          pf.mark(6);
          if (BIF_DBG & 32768) tc::mbar_wait_sleep(tc::smem_u32(&s_full[slot]), (u >> 1) & 1, BIF_DBG & 262144);
          else tc::mbar_wait(tc::smem_u32(&s_full[slot]), (u >> 1) & 1);
          pf.mark(0);
          tc::tc_fence_after();
          if (j == 0) stamp(3);
          stamp(20);
          float xv[kNarrowP];
          if (h0) {
#pragma unroll
            for (int k = 0; k < kNarrowP; ++k)
              if (k < P.p) tc::tmem_ld<1>(tS + slot * N + cv0 + k + lane_addr, reinterpret_cast<uint32_t*>(&xv[k]));
            tc::tmem_ld_wait();
          }
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_free[slot]));
          pf.mark(1);
          if (BIF_DBG & 1) {
            tc::mbar_wait(tc::smem_u32(&p_empty[ps]), (ph & 1) ^ 1);
            tc::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&p_full[ps]));
            if (++t == ntl) { t = 0; ++cl; }
            continue;
          }
          const int tpos = t * kBM + pos;
          if (h0) {
#pragma unroll
            for (int k = 0; k < kNarrowP; ++k) {
              if (k < P.p) {
                // multi-token step: the intra-step causal bound of token k % ntok
                const int Lk = MT ? max(L - (P.ntok - 1 - k % P.ntok), P.lens_offset) : L;
                xv[k] = tpos < Lk ? xv[k] * sl2 : kNegInf;
                float v = xv[k];
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
                if (lane == 0) nred[(slot * 4 + quad) * kNarrowP + k] = v;
              }
            }
          }
          if (h0) tc::named_bar_sync(3, 128);  // the 4 half-0 warps (one per quadrant)
          pf.mark(2);
          stamp(21);
          if (h0) {
            float pv[kNarrowP], alpha[kNarrowP], tm[kNarrowP];
            bool resc = false;
#pragma unroll
            for (int k = 0; k < kNarrowP; ++k) {
              if (k < P.p) {
                const float* nr = nred + slot * 4 * kNarrowP + k;
                tm[k] = fmaxf(fmaxf(nr[0], nr[kNarrowP]), fmaxf(nr[2 * kNarrowP], nr[3 * kNarrowP]));
              }
            }
#pragma unroll
            for (int k = 0; k < kNarrowP; ++k) {
              if (k < P.p) {
                const float mo = m_g[k];
                float mn = mo;
                alpha[k] = 1.f;
                if (mo == kNegInf) {
                  mn = tm[k];  // first valid tile of this column: exact max
                } else if (tm[k] > mo + kTh) {
                  mn = tm[k];  // lazy rescale: only when P would exceed 2^kTh
                  alpha[k] = ex2(mo - mn);
                  l_g[k] *= alpha[k];
                  resc = true;
                }
                m_g[k] = mn;
                pv[k] = (mn == kNegInf) ? 0.f : ex2(xv[k] - mn);
              }
            }
            if (resc) {  // uniform over half-0 warps (same shared values)
              tc::mbar_wait(tc::smem_u32(&p_empty[(u - 1) % P.npb]), ((u - 1) / P.npb) & 1);  // PV(u-1) done
              tc::tc_fence_after();
#pragma unroll
              for (int k = 0; k < kNarrowP; ++k) {
                if (k < P.p && alpha[k] != 1.f) {
                  uint32_t o1, o2 = 0;
                  tc::tmem_ld<1>(tOb + cv0 + k + lane_addr, &o1);
                  if (!KV8) tc::tmem_ld<1>(tOb + N + cv0 + k + lane_addr, &o2);
                  tc::tmem_ld_wait();
                  o1 = __float_as_uint(__uint_as_float(o1) * alpha[k]);
                  o2 = __float_as_uint(__uint_as_float(o2) * alpha[k]);
                  tc::tmem_st<1>(tOb + cv0 + k + lane_addr, &o1);
                  if (!KV8) tc::tmem_st<1>(tOb + N + cv0 + k + lane_addr, &o2);
                }
              }
              tc::tmem_st_wait();
              tc::tc_fence_before();
            }
            // P row of this position (hi and lo parts): zeros except the p valid columns
            pf.mark(3);
            stamp(27);
            if (!(BIF_DBG & 8)) tc::mbar_wait(tc::smem_u32(&p_empty[ps]), (ph & 1) ^ 1);  // PV(u-npb) done
            stamp(28);
            uint8_t* const sm_pb = sm_p + ps * PB;
            pf.mark(4);
            const int pc = ps ? pcol1 : pcol0;
            if (pc < 0) {
#pragma unroll
              for (int n = 0; n < NP; n += 8) {
                uint32_t off = (uint32_t)((n / W) * PLBO + pos * PRB + (n % W) * 2);
                off ^= ((off >> 7) & PSWM) << 4;
                *reinterpret_cast<uint4*>(sm_pb + off) = make_uint4(0, 0, 0, 0);
              }
            } else if (pc != cv0) {
#pragma unroll
              for (int k = 0; k < kNarrowP; ++k) {
                if (k < P.p) {  // the previous group's columns (both parts) back to zero
                  const int col = pc + k;
                  uint32_t off = (uint32_t)((col / W) * PLBO + pos * PRB + (col % W) * 2);
                  off ^= ((off >> 7) & PSWM) << 4;
                  *reinterpret_cast<uint16_t*>(sm_pb + off) = 0;
                  if constexpr (!KV8) {
                    uint32_t offl = (uint32_t)(((N + col) / W) * PLBO + pos * PRB + ((N + col) % W) * 2);
                    offl ^= ((offl >> 7) & PSWM) << 4;
                    *reinterpret_cast<uint16_t*>(sm_pb + offl) = 0;
                  }
                }
              }
            }
            if (ps) pcol1 = cv0; else pcol0 = cv0;
#pragma unroll
            for (int k = 0; k < kNarrowP; ++k) {
              if (k < P.p) {
                const int col = cv0 + k;
                l_g[k] += pv[k];
                uint32_t off = (uint32_t)((col / W) * PLBO + pos * PRB + (col % W) * 2);
                off ^= ((off >> 7) & PSWM) << 4;
                if constexpr (KV8) {
                  *reinterpret_cast<__half*>(sm_pb + off) = __float2half_rn(pv[k]);
                } else {
                  const __nv_bfloat16 hi = __float2bfloat16_rn(pv[k]);
                  const __nv_bfloat16 lo = __float2bfloat16_rn(pv[k] - __bfloat162float(hi));
                  uint32_t offl = (uint32_t)(((N + col) / W) * PLBO + pos * PRB + ((N + col) % W) * 2);
                  offl ^= ((offl >> 7) & PSWM) << 4;
                  *reinterpret_cast<__nv_bfloat16*>(sm_pb + off) = hi;
                  *reinterpret_cast<__nv_bfloat16*>(sm_pb + offl) = lo;
                }
              }
            }
            tc::fence_proxy_async_smem();
          } else {
            // half-1 warps join no per-tile barrier: this wait keeps their
            // p_full arrival for tile u behind the completion of tile u - npb
            // on the same P slot, so their arrivals stay in the slot's phase
            tc::mbar_wait(tc::smem_u32(&p_empty[ps]), (ph & 1) ^ 1);
          }
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(tc::smem_u32(&p_full[ps]));
          pf.mark(5);
          stamp(23);
          // end of this group's tiles (or of this segment part): flush its row sums / max
          if (t == ntl - 1 || j == s.ntiles - 1) {
            if (!e_waited) {  // the epilogue has consumed this buffer's previous segment
              tc::mbar_wait(tc::smem_u32(&e_empty[ob]), ((sg >> 1) & 1) ^ 1);
              e_waited = true;
            }
            if (h0) {
#pragma unroll
              for (int k = 0; k < kNarrowP; ++k) {
                if (k < P.p) {
                  float v = l_g[k];
#pragma unroll
                  for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                  if (lane == 0) sm_l[(ob * 4 + quad) * N + cv0 + k] = v;
                  if (lane == 0 && quad == 0) sm_mfin[ob * N + cv0 + k] = m_g[k];
                  m_g[k] = kNegInf;
                  l_g[k] = 0.f;
                }
              }
            }
          }
          if (++t == ntl) {
            t = 0;
            ++cl;
          }
        }
        // columns of groups this segment part did not visit: no contribution
        if (!e_waited) tc::mbar_wait(tc::smem_u32(&e_empty[ob]), ((sg >> 1) & 1) ^ 1);
        {
          const int vlo = cfirst * P.p;
          const int vhi = (t == 0 ? cl : cl + 1) * P.p;  // one past the last visited column
          for (int k = sw * 32 + lane; k < N; k += 32 * NSW) {
            if (k < vlo || k >= vhi) {
              sm_l[(ob * 4 + 0) * N + k] = 0.f;
              sm_l[(ob * 4 + 1) * N + k] = 0.f;
              sm_l[(ob * 4 + 2) * N + k] = 0.f;
              sm_l[(ob * 4 + 3) * N + k] = 0.f;
              sm_mfin[ob * N + k] = kNegInf;
            }
          }
        }
        stamp(4);
        tc::mbar_arrive(tc::smem_u32(&e_full[ob]));
      } else {
        // ====== general path: every column of the tile may be valid ======
        float l_part[CPT], mr[CPT];  // per-position row sums; running max per column
#pragma unroll
        for (int n = 0; n < CPT; ++n) {
          l_part[n] = 0.f;
          mr[n] = kNegInf;
        }
        // every column of this thread has a running max (uniform: mr is common
        // to all positions); only a context segment gets there for all columns
        bool all_set = false;
        for (int j = 0; j < s.ntiles; ++j, ++u) {
          const int cv0 = s.dec ? cl * P.p : 0;
          const int cv1 = s.dec ? cv0 + P.p : N;
          const uint32_t slot = u & 1;
          const uint32_t ps = P.npb == 2 ? (u & 1) : 0, ph = P.npb == 2 ? (u >> 1) : u;  // P slot, its phase
          pf.mark(6);
          if (BIF_DBG & 32768) tc::mbar_wait_sleep(tc::smem_u32(&s_full[slot]), (u >> 1) & 1, BIF_DBG & 262144);
          else tc::mbar_wait(tc::smem_u32(&s_full[slot]), (u >> 1) & 1);
          pf.mark(0);
          tc::tc_fence_after();
          if (j == 0) stamp(s.dec ? 3 : 2);
          stamp(20);
          float x[CPT];
          tmem_ld_cols<CPT>(tS + slot * N + col0 + lane_addr, reinterpret_cast<uint32_t*>(x));
          tc::tmem_ld_wait();
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(tc::smem_u32(&s_free[slot]));
          pf.mark(1);
          if (BIF_DBG & 1) {
            tc::mbar_wait(tc::smem_u32(&p_empty[ps]), (ph & 1) ^ 1);
            tc::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&p_full[ps]));
            if (++t == ntl) { t = 0; ++cl; }
            continue;
          }
          bool need = false;
          const int tl = s.dec ? t : ctx_tile(P, s, j);
          if (all_set && (tl + 1) * kBM <= L) {
            // fast path (warp-uniform): every column of this thread has its
            // running max and every position of the tile is valid
#pragma unroll
            for (int n = 0; n < CPT; ++n) {
              x[n] = fmaf(x[n], sl2, -mr[n]);
              need |= x[n] > kTh;
            }
          } else {
            const int tpos = tl * kBM + pos;
            const bool vpos = tpos < L;
#pragma unroll
            for (int n = 0; n < CPT; ++n) {
              const int col = col0 + n;
              bool vc = vpos && col >= cv0 && col < cv1;
              if (MT && s.dec)  // intra-step causal bound of the column's token
                vc = vc && tpos < max(L - (P.ntok - 1 - (col - cv0) % P.ntok), P.lens_offset);
              const float mref = (mr[n] == kNegInf) ? 0.f : mr[n];
              x[n] = vc ? fmaf(x[n], sl2, -mref) : kNegInf;
              need |= vc && (mr[n] == kNegInf || x[n] > kTh);
            }
          }
          const bool slowp = (BIF_DBG & 4096) ? (bool)__any_sync(0xffffffffu, need) : tc::named_bar_or(1, 32 * NSW, need);
          pf.mark(2);
          stamp(slowp ? 22 : 21);
          if (slowp) pf.count(7);
          if (slowp) {
            // ---- slow path: exact max of the tile's valid columns, new running max ----
            if (quad == 0 && lane == 0) {
#pragma unroll
              for (int n = 0; n < CPT; ++n) sm_mold[col0 + n] = mr[n];
            }
            if (col0 < cv1 && col0 + CPT > cv0) {  // warp-uniform: this warp has valid columns
              if (cv1 - cv0 >= CPT) {
                float v[CPT];
#pragma unroll
                for (int n = 0; n < CPT; ++n) v[n] = x[n];
                warp_col_reduce<CPT, true>(v, lane);
                if (lane < CPT) sm_red[quad * N + col0 + lane] = v[0];
              } else {
#pragma unroll
                for (int n = 0; n < CPT; ++n) {
                  const int col = col0 + n;
                  if (col >= cv0 && col < cv1) {
                    float v = x[n];
#pragma unroll
                    for (int off = 16; off >= 1; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
                    if (lane == 0) sm_red[quad * N + col] = v;
                  }
                }
              }
            }
            stamp(24);
            tc::named_bar_sync(2, 32 * NSW);
            stamp(25);
            bool grew = false;
#pragma unroll
            for (int n = 0; n < CPT; ++n) {
              const int col = col0 + n;
              const float cm = (col >= cv0 && col < cv1)
                                   ? fmaxf(fmaxf(sm_red[col], sm_red[N + col]), fmaxf(sm_red[2 * N + col], sm_red[3 * N + col]))
                                   : kNegInf;
              const float mo = mr[n];
              const float mref = (mo == kNegInf) ? 0.f : mo;
              const float mn = fmaxf(mo, mref + cm);  // unchanged if the column had no valid logit
              // l and O of a column are exactly 0 while its max is unset
              l_part[n] *= (mo == kNegInf) ? 0.f : ex2(mo - mn);
              x[n] = (mn == kNegInf) ? kNegInf : x[n] + (mref - mn);
              grew |= (mo != kNegInf) && (mn > mo);
              mr[n] = mn;
            }
            all_set = !s.dec;
#pragma unroll
            for (int n = 0; n < CPT; ++n) all_set = all_set && mr[n] != kNegInf;
            // (the vote's barrier also orders these sm_red reads before later writes)
            stamp(26);
            if (tc::named_bar_or(1, 32 * NSW, grew)) {
              // O^T holds earlier tiles of this segment: wait for PV(u-1), rescale
              tc::mbar_wait(tc::smem_u32(&p_empty[(u - 1) % P.npb]), ((u - 1) / P.npb) & 1);  // PV(u-1) done
              tc::tc_fence_after();
#pragma unroll
              for (int n = 0; n < CPT; n += 8) {
                uint32_t orr[8], orl[8];
                tc::tmem_ld<8>(tOb + col0 + n + lane_addr, orr);
                if (!KV8) tc::tmem_ld<8>(tOb + N + col0 + n + lane_addr, orl);
                tc::tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  const float mo = sm_mold[col0 + n + e];
                  const float a = (mo == kNegInf) ? 1.f : ex2(mo - mr[n + e]);
                  orr[e] = __float_as_uint(__uint_as_float(orr[e]) * a);
                  if (!KV8) orl[e] = __float_as_uint(__uint_as_float(orl[e]) * a);
                }
                tc::tmem_st<8>(tOb + col0 + n + lane_addr, orr);
                if (!KV8) tc::tmem_st<8>(tOb + N + col0 + n + lane_addr, orl);
              }
              tc::tmem_st_wait();
              tc::tc_fence_before();
            }
          }
          // ---- P = 2^x as two bf16 parts (P_hi + P_lo carries ~16 mantissa
          //      bits) into shared memory; fp32 row sums ----
          pf.mark(3);
          stamp(27);
          if (!(BIF_DBG & 4)) tc::mbar_wait(tc::smem_u32(&p_empty[ps]), (ph & 1) ^ 1);  // PV(u-npb) done
          stamp(28);
          uint8_t* const sm_pb = sm_p + ps * PB;
          pf.mark(4);
#pragma unroll
          for (int n = 0; n < CPT; n += 8) {
            if constexpr (KV8) {  // one f16 part
              uint32_t hk[4];
#pragma unroll
              for (int e = 0; e < 8; e += 2) {
                const float p0 = ex2(x[n + e]), p1 = ex2(x[n + e + 1]);
                l_part[n + e] += p0;
                l_part[n + e + 1] += p1;
                hk[e / 2] = pack_f16x2(p0, p1);
              }
              const int col = col0 + n;
              uint32_t off = (uint32_t)((col / W) * PLBO + pos * PRB + (col % W) * 2);
              off ^= ((off >> 7) & PSWM) << 4;
              *reinterpret_cast<uint4*>(sm_pb + off) = make_uint4(hk[0], hk[1], hk[2], hk[3]);
            } else {
            uint32_t hk[4], lk[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              float p0 = ex2(x[n + e]), p1 = ex2(x[n + e + 1]);
              if (BIF_DBG & 131072) {  // experiment: twice the exp work
                p0 = ex2(p0 * 1e-30f + x[n + e]);
                p1 = ex2(p1 * 1e-30f + x[n + e + 1]);
              }
              l_part[n + e] += p0;
              l_part[n + e + 1] += p1;
              hk[e / 2] = pack_bf16x2_trunc(p0, p1);
              lk[e / 2] = pack_bf16x2_trunc(p0 - bf16lo(hk[e / 2]), p1 - bf16hi(hk[e / 2]));
            }
            const int col = col0 + n;
            uint32_t off = (uint32_t)((col / W) * PLBO + pos * PRB + (col % W) * 2);
            off ^= ((off >> 7) & PSWM) << 4;
            uint32_t offl = (uint32_t)(((N + col) / W) * PLBO + pos * PRB + ((N + col) % W) * 2);
            offl ^= ((offl >> 7) & PSWM) << 4;
            if (!(BIF_DBG & 2048)) {
              *reinterpret_cast<uint4*>(sm_pb + off) = make_uint4(hk[0], hk[1], hk[2], hk[3]);
              *reinterpret_cast<uint4*>(sm_pb + offl) = make_uint4(lk[0], lk[1], lk[2], lk[3]);
            }
            }
          }
          tc::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(tc::smem_u32(&p_full[ps]));
          pf.mark(5);
          stamp(23);
          if (++t == ntl) {
            t = 0;
            ++cl;
          }
        }
        // ---- hand the segment's row sums / max to the epilogue warps ----
        stamp(4);
        warp_col_reduce<CPT, false>(l_part, lane);  // lane l: column l of this warp, over 32 positions
        tc::mbar_wait(tc::smem_u32(&e_empty[ob]), ((sg >> 1) & 1) ^ 1);
        if (lane < CPT) sm_l[(ob * 4 + quad) * N + col0 + lane] = l_part[0];
        if (quad == 0 && lane == 0) {
#pragma unroll
          for (int n = 0; n < CPT; ++n) sm_mfin[ob * N + col0 + n] = mr[n];
        }
        tc::mbar_arrive(tc::smem_u32(&e_full[ob]));
      }
      w = s.next;
      L = Ln;
    }
    if constexpr (!MT && NSW == 8) {
      if (!KV8 && P.dyn && P.p > 1) {
        // ====== dynamic decode columns, p = 2 / 4 query rows (dyn_cc_multi) ======
        if (u > 0) tc::mbar_wait(tc::smem_u32(&p_empty[(u - 1) % P.npb]), ((u - 1) / P.npb) & 1);
        DynSmem S;
        S.stage = sm_stage;
        S.q = sm_q;
        S.QB = QB;
        S.Nq = N;
        S.nst = NST;
        S.kv_full = kv_full;
        S.kv_empty = kv_empty;
        S.q_full = q_full;
        S.q_empty = q_empty;
        S.ring = reinterpret_cast<const int2*>(bars + 56);
        S.scr_o = reinterpret_cast<float*>(sm_p);
        S.scr_ml = sm_red;
        S.qf = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars + 64) + 128);
        S.pex = S.qf + 2 * P.p * bif::kQHalf;
        // (planned only for N = 16, bf16 cache: compiled only there)
        if constexpr (N == 16 && !KV8) {
          if (P.p == 4) dyn_cc_multi<4, NSW>(P, S, sw, lane, u, sg);
          else dyn_cc_multi<2, NSW>(P, S, sw, lane, u, sg);
        }
      } else if (P.dyn) {
        // ====== dynamic decode columns on the CUDA cores (p = 1) ======
        // Column (i, c): one query row against Kd[i][c] / Vd[i][c], a GEMV.
        // Warp sw owns tile positions [16 sw, 16 sw + 16): QK with 2 lanes per
        // position (lane half hf = d half), then PV over the same positions with
        // lane l holding d = 4l .. 4l + 3.  Each warp keeps its own exact online
        // softmax (m, l, o) over the column's tiles; at the column's end the
        // NSW partials are joined through shared memory into ONE partial of row
        // i*h + c (workspace slot Sc).  fp32 throughout (bf16 products are exact).
        const int2* const ring = reinterpret_cast<const int2*>(bars + 56);
        float* const scr_o = reinterpret_cast<float*>(sm_p);  // [2][NSW][128] (the idle P buffer)
        float* const scr_ml = sm_red;                         // [2][NSW][2]
        // the last PV of the static range has read the P buffer
        if (u > 0) tc::mbar_wait(tc::smem_u32(&p_empty[(u - 1) % P.npb]), ((u - 1) / P.npb) & 1);
        const int hf = lane >> 4;
        const int pp = 16 * sw + (lane & 15);        // QK: this lane's tile position
        const int vch = (lane & 15) >> 1;            // PV: 16-byte chunk of d = 4 lane ..
        const int vsub = (lane & 1) * 8;             //     and the 8-byte half of it
        const float sl2 = P.scale_log2;
        int cb = 0;
        stamp(39);  // static range done
        for (;; ++sg) {
          const uint32_t qb = sg & 1;
          tc::mbar_wait(tc::smem_u32(&q_full[qb]), (sg >> 1) & 1);
          stamp(40);  // column's q (and id) in shared memory
          const int unit = reinterpret_cast<const volatile int*>(ring + qb)[0];
          if (unit < 0) break;
          const int Lc = reinterpret_cast<const volatile int*>(ring + qb)[1];
          const int col = unit / P.dparts, part = unit - col * P.dparts;
          const int t0 = part * P.dunit;
          // this lane's half of the query row, fp32 (row 0 of the SW128 q box: unswizzled)
          float qf[64];
          {
            const uint8_t* const qrow = sm_q + qb * QB + hf * (N * 128);
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
              const uint4 v = *reinterpret_cast<const uint4*>(qrow + ch * 16);
              qf[8 * ch + 0] = bf16lo(v.x); qf[8 * ch + 1] = bf16hi(v.x);
              qf[8 * ch + 2] = bf16lo(v.y); qf[8 * ch + 3] = bf16hi(v.y);
              qf[8 * ch + 4] = bf16lo(v.z); qf[8 * ch + 5] = bf16hi(v.z);
              qf[8 * ch + 6] = bf16lo(v.w); qf[8 * ch + 7] = bf16hi(v.w);
            }
          }
          float m_w = kNegInf, l_w = 0.f;
          float2 oa = make_float2(0.f, 0.f), ob2 = make_float2(0.f, 0.f);
          const int nt = min((Lc + kBM - 1) / kBM, t0 + P.dunit);
          for (int t = t0; t < nt; ++t, ++u) {
            const uint32_t st = u % NST;
            tc::mbar_wait(tc::smem_u32(&kv_full[st]), (u / NST) & 1);
            stamp(41);  // tile landed
            const uint8_t* const stage = sm_stage + st * kStageBytes;
            // ---- logit of position pp: this lane's 64 products, + the other half ----
            float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
            if constexpr (KV8) {
              // E4M3 codes of row pp (128 B, SW128 chunks of 16 codes; the stage's
              // K code slot at +16 KB): this lane's 64 codes = chunks 4 hf .. 4 hf + 3,
              // exact via f16 (R20); k_scale is in the logit scale
              const uint8_t* const krow = stage + 16384 + pp * 128;
#pragma unroll
              for (int cc = 0; cc < 4; ++cc) {
                const uint4 v = *reinterpret_cast<const uint4*>(krow + (((4 * hf + cc) ^ (pp & 7)) << 4));
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 k0 = f16x2_f2(e4m3x2_to_f16x2(w[e])), k1 = f16x2_f2(e4m3x2_to_f16x2(w[e] >> 16));
                  ffma2(a0, k0, make_float2(qf[16 * cc + 4 * e + 0], qf[16 * cc + 4 * e + 1]));
                  ffma2(a1, k1, make_float2(qf[16 * cc + 4 * e + 2], qf[16 * cc + 4 * e + 3]));
                }
              }
            } else {
              const uint8_t* const krow = stage + hf * 16384 + pp * 128;
#pragma unroll
              for (int ch = 0; ch < 8; ++ch) {
                const uint4 v = *reinterpret_cast<const uint4*>(krow + ((ch ^ (pp & 7)) << 4));
                ffma2(a0, bf16x2_f2(v.x), make_float2(qf[8 * ch + 0], qf[8 * ch + 1]));
                ffma2(a1, bf16x2_f2(v.y), make_float2(qf[8 * ch + 2], qf[8 * ch + 3]));
                ffma2(a0, bf16x2_f2(v.z), make_float2(qf[8 * ch + 4], qf[8 * ch + 5]));
                ffma2(a1, bf16x2_f2(v.w), make_float2(qf[8 * ch + 6], qf[8 * ch + 7]));
              }
            }
            float sdot = (a0.x + a0.y) + (a1.x + a1.y);
            sdot += __shfl_xor_sync(0xffffffffu, sdot, 16);
            const int tpos = t * kBM + pp;
            const float x = tpos < Lc ? sdot * sl2 : kNegInf;
            // ---- exact online softmax over this warp's positions ----
            float mt = x;
#pragma unroll
            for (int off = 8; off >= 1; off >>= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, off));
            const float mn = fmaxf(m_w, mt);
            const float mref = (mn == kNegInf) ? 0.f : mn;
            const float alpha = ex2(m_w - mref);  // 0 while m_w is unset (l, o are 0)
            l_w *= alpha;
            oa.x *= alpha; oa.y *= alpha; ob2.x *= alpha; ob2.y *= alpha;
            m_w = mn;
            const float pe = ex2(x - mref);  // 0 at masked positions
            l_w += hf ? 0.f : pe;
            // ---- o += p . V over the warp's valid positions (lane: d = 4 lane ..) ----
            const uint8_t* const vb = stage + 32768 + hf * 16384 + vsub;
            const int nv = min(max(Lc - (t * kBM + 16 * sw), 0), 16);
            if constexpr (KV8) {
              // V codes (the stage's V code slot at +48 KB): 4 codes = d 4 lane .. per row
              const uint8_t* const vc = stage + 49152 + (lane & 3) * 4;
              for (int k = 0; k < nv; ++k) {
                const float pk = __shfl_sync(0xffffffffu, pe, k);
                const int r = 16 * sw + k;
                const uint32_t w = *reinterpret_cast<const uint32_t*>(vc + r * 128 + (((lane >> 2) ^ (r & 7)) << 4));
                ffma2(oa, f16x2_f2(e4m3x2_to_f16x2(w)), make_float2(pk, pk));
                ffma2(ob2, f16x2_f2(e4m3x2_to_f16x2(w >> 16)), make_float2(pk, pk));
              }
            } else if (nv == 16) {
#pragma unroll
              for (int k = 0; k < 16; ++k) {
                const float pk = __shfl_sync(0xffffffffu, pe, k);
                const int r = 16 * sw + k;
                const uint2 v = *reinterpret_cast<const uint2*>(vb + r * 128 + ((vch ^ (r & 7)) << 4));
                ffma2(oa, bf16x2_f2(v.x), make_float2(pk, pk));
                ffma2(ob2, bf16x2_f2(v.y), make_float2(pk, pk));
              }
            } else {
              for (int k = 0; k < nv; ++k) {  // positions past the length are never read
                const float pk = __shfl_sync(0xffffffffu, pe, k);
                const int r = 16 * sw + k;
                const uint2 v = *reinterpret_cast<const uint2*>(vb + r * 128 + ((vch ^ (r & 7)) << 4));
                ffma2(oa, bf16x2_f2(v.x), make_float2(pk, pk));
                ffma2(ob2, bf16x2_f2(v.y), make_float2(pk, pk));
              }
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&kv_empty[st]));  // 1 of NSW
            stamp(42);  // tile done
          }
          // ---- join the NSW warp partials of the column: one (m, l, o) ----
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) l_w += __shfl_xor_sync(0xffffffffu, l_w, off);
          *reinterpret_cast<float4*>(scr_o + (cb * NSW + sw) * kD + 4 * lane) = make_float4(oa.x, oa.y, ob2.x, ob2.y);
          if (lane == 0) *reinterpret_cast<float2*>(scr_ml + (cb * NSW + sw) * 2) = make_float2(m_w, l_w);
          tc::named_bar_sync(2, 32 * NSW);
          if (sw < 4) {
            const int d = sw * 32 + lane;
            const float2* const ml = reinterpret_cast<const float2*>(scr_ml + cb * NSW * 2);
            float M = kNegInf;
#pragma unroll
            for (int w2 = 0; w2 < NSW; ++w2) M = fmaxf(M, ml[w2].x);
            const float Ms = (M == kNegInf) ? 0.f : M;
            float od = 0.f, ls = 0.f;
#pragma unroll
            for (int w2 = 0; w2 < NSW; ++w2) {
              const float wt = ex2(ml[w2].x - Ms);
              od = fmaf(wt, scr_o[(cb * NSW + w2) * kD + d], od);
              ls = fmaf(wt, ml[w2].y, ls);
            }
            const int i = col / P.g, c = col - i * P.g;
            const size_t gr = (size_t)i * P.h + c;  // p = 1
            BA_CHECK(gr < (size_t)P.b * P.h && P.Sc + part < P.S);
            P.ws_o[(gr * P.S + P.Sc + part) * kD + d] = od;
            if (d == 0) reinterpret_cast<float2*>(P.ws_ml)[gr * P.S + P.Sc + part] = make_float2(M, ls);
          }
          // every warp loaded q before the barrier: the buffer goes back
          if (sw == 0 && lane == 0) tc::mbar_arrive(tc::smem_u32(&q_empty[qb]));
          stamp(43);  // column joined and written
          cb ^= 1;
        }
      }
    }
    stamp(7);
    pf.mark(6);
    if (threadIdx.x == 128 || threadIdx.x == 256)
      pf.dump(P.trace ? P.trace + (size_t)blockIdx.x * kTraceSlots : nullptr, threadIdx.x == 128 ? 0 : 8);
  } else if (warp == 2) {
    // ===== merge bookkeeping, off the critical path (this warp is otherwise
    // idle after the TMEM allocation): part counts of every warp's first
    // merge row (binary searches of the CTA table) =====
    if (lane < (int)(blockDim.x >> 5)) {
      const int gr = r0 + lane;
      int nc = 0, nd = 0;
      if (gr < r1) {
        const int i = gr / P.h, j = gr - i * P.h;
        const int c = j / P.p;
        nc = ctx_parts(P, c, (i * P.p + (j - c * P.p)) / P.N);
        nd = dec_parts(P, i, c / P.gpc);
      }
      sm_mcnt[2 * lane] = nc;
      sm_mcnt[2 * lane + 1] = nd;
    }
  } else if (warp >= EPI0 && warp < EPI0 + 4) {
    // ===================== epilogue warpgroup (4 warps) =====================
    // O^T lanes are d = 32*(warp%4) + lane; columns are the chunk's rows.
    const int quad = warp & 3;
    const int d = quad * 32 + lane;
    const int et = threadIdx.x - 32 * EPI0;  // 0..127
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    // drain(s, sg): O^T of segment part s (the sg-th of this CTA) -> workspace
    auto drain = [&](const Seg& s, uint32_t sg) {
      const uint32_t ob = sg & 1;
      if (BIF_DBG & 8192) tc::mbar_wait_sleep(tc::smem_u32(&o_full[ob]), (sg >> 1) & 1, BIF_DBG & 262144);
      else tc::mbar_wait(tc::smem_u32(&o_full[ob]), (sg >> 1) & 1);
      tc::tc_fence_after();
      // output rows of the chunk's columns, stepped without divisions (row_of):
      // decode chunk: head j = j0 + col of sample i; context chunk: row r =
      // r0 + col of the (sample, head-in-group) grid, advanced (ri, rj)
      const int R = P.b * P.p;
      int ri = 0, rj = 0, jd = 0;
      if (s.dec) {
        jd = s.cb * P.gpc * P.p;
      } else {
        const int r0 = s.rc * N;
        ri = r0 / P.p;
        rj = r0 - ri * P.p;
      }
      BA_CHECK(s.slot >= 0 && s.slot < P.S);
      float* const wo = P.ws_o + (size_t)s.slot * kD + d;
      const size_t row_stride = (size_t)P.S * kD;
#pragma unroll
      for (int n = 0; n < ((BIF_DBG & 524288) ? 0 : N); n += 16) {
        uint32_t orr[16], orl[16];
        if (!(BIF_DBG & 2097152)) {
          tc::tmem_ld<16>(tO + ob * NP + n + lane_addr, orr);
          if (KV8) {
#pragma unroll
            for (int e = 0; e < 16; ++e) orl[e] = 0u;  // +0.0f
          } else {
            tc::tmem_ld<16>(tO + ob * NP + N + n + lane_addr, orl);
          }
          tc::tmem_ld_wait();
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) orr[e] = orl[e] = (uint32_t)e;
        }
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int col = n + e;
          int gr;
          if (s.dec) {
            gr = jd + col < P.h ? s.i * P.h + jd + col : -1;
          } else {
            gr = s.rc * N + col < R ? ri * P.h + s.c * P.p + rj : -1;
            if (++rj == P.p) {
              rj = 0;
              ++ri;
            }
          }
          if (gr >= 0 && !(BIF_DBG & 1048576)) wo[(size_t)gr * row_stride] = __uint_as_float(orr[e]) + __uint_as_float(orl[e]);
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(&o_empty[ob]));
      if (BIF_DBG & 8192) tc::mbar_wait_sleep(tc::smem_u32(&e_full[ob]), (sg >> 1) & 1, BIF_DBG & 262144);
      else tc::mbar_wait(tc::smem_u32(&e_full[ob]), (sg >> 1) & 1);
      if (et < N) {
        const int gr = row_of(P, s, et);
        if (gr >= 0) {
          const float* lb = sm_l + ob * 4 * N;
          const float Lr = lb[et] + lb[N + et] + lb[2 * N + et] + lb[3 * N + et];
          reinterpret_cast<float2*>(P.ws_ml)[(size_t)gr * P.S + s.slot] = make_float2(sm_mfin[ob * N + et], Lr);
        }
      }
      tc::mbar_arrive(tc::smem_u32(&e_empty[ob]));
    };
    if constexpr (!KV8) {
      uint32_t sg = 0;
      for (long long w = 0; w < nw; ++sg) {
        const Seg s = seg_at(P, rg, w);
        drain(s, sg);
        w = s.next;
      }
    } else {
      // ---- KV8: these warps are also the converters.  Per segment: q (bf16
      // -> f16 in place); per tile: the E4M3 codes of the raw ring -> the f16
      // stage in the layout the MMAs read (two 64-column SW128 halves).  The
      // previous segment is drained after this segment's first two tiles are
      // converted (the MMAs work on them meanwhile).  A warp instruction
      // covers 8 rows x 4 chunks of 16 codes: no bank conflicts. ----
      const int cw = quad;  // rows [32 cw, 32 cw + 32) of every tile
      uint32_t u = 0, sg = 0;
      Seg prev;
      bool pending = false;
      for (long long w = 0; w < nw; ++sg) {
        const Seg s = seg_at(P, rg, w);
        const uint32_t qbuf = sg & 1;
        tc::mbar_wait(tc::smem_u32(&q_full[qbuf]), (sg >> 1) & 1);
        uint4* qv = reinterpret_cast<uint4*>(sm_q + qbuf * QB);
        for (int i = et; i < QB / 16; i += 128) {
          uint4 v = qv[i];
          v.x = pack_f16x2(bf16lo(v.x), bf16hi(v.x));
          v.y = pack_f16x2(bf16lo(v.y), bf16hi(v.y));
          v.z = pack_f16x2(bf16lo(v.z), bf16hi(v.z));
          v.w = pack_f16x2(bf16lo(v.w), bf16hi(v.w));
          qv[i] = v;
        }
        tc::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(tc::smem_u32(&q_cvt[qbuf]));
        for (int j = 0; j < s.ntiles; ++j, ++u) {
          const int st = u % NST;
          tc::mbar_wait(tc::smem_u32(&kv_full[st]), (u / NST) & 1);
          uint8_t* const stage = sm_stage + st * kStageBytes;
          // K: each thread expands the 128 codes of ITS position row (its TMEM
          // lane, R = 32 cw + lane) into f16 pairs and stores them into the
          // stage's K slot in TMEM (64 columns, d = 2j, 2j + 1 in column j):
          // the QK MMA reads A from there, so the f16 K never touches smem.
          // An 8-lane phase reads 8 consecutive rows' chunks at distinct
          // swizzled positions: conflict-free.
          {
            const int R = 32 * cw + lane;
            const uint8_t* const krow = stage + 16384 + R * 128;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint32_t kv[32];
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4) {
                const int c = 4 * h + c4;
                const uint4 v = lds128(krow + ((c ^ (R & 7)) << 4));
                kv[8 * c4 + 0] = e4m3x2_to_f16x2(v.x);
                kv[8 * c4 + 1] = e4m3x2_to_f16x2(v.x >> 16);
                kv[8 * c4 + 2] = e4m3x2_to_f16x2(v.y);
                kv[8 * c4 + 3] = e4m3x2_to_f16x2(v.y >> 16);
                kv[8 * c4 + 4] = e4m3x2_to_f16x2(v.z);
                kv[8 * c4 + 5] = e4m3x2_to_f16x2(v.z >> 16);
                kv[8 * c4 + 6] = e4m3x2_to_f16x2(v.w);
                kv[8 * c4 + 7] = e4m3x2_to_f16x2(v.w >> 16);
              }
              tc::tmem_st<32>(tK + st * 64 + h * 32 + lane_addr, kv);
            }
            tc::tmem_st_wait();
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&k_cvt[st]));
          }
          // V: the codes of row R (region + 16 KB + R*128) expand in place to
          // f16 row R of both 64-column halves.  Lane: code chunks c0 and
          // c0 + 4 (-> half 0 and half 1) of row r8 of an 8-row block; an 8-lane
          // shared-memory phase covers rows k and k + 4, whose swizzled chunk
          // sets are complementary (conflict-free loads), and the second row
          // of a phase stores its odd f16 chunk first (the two rows then hit
          // even and odd chunk sets: conflict-free stores).  Half-1 rows
          // overwrite the code rows they come from: a block's stores follow a
          // __syncwarp after all its loads (and the next block's prefetch,
          // which reads other rows).
          const int r8 = ((lane >> 2) & 1) * 4 + (lane >> 3);
          const bool odd_first = (lane >> 2) & 1;
          {
            uint8_t* const reg = stage + 32768;
            const int c0 = lane & 3;
            auto code_at = [&](int blk, int c) {
              const int R = 32 * cw + 8 * blk + r8;
              return lds128(reg + 16384 + R * 128 + ((c ^ (R & 7)) << 4));
            };
            uint4 a0 = code_at(0, c0), a1 = code_at(0, c0 + 4);
#pragma unroll
            for (int blk = 0; blk < 4; ++blk) {
              uint4 n0, n1;
              if (blk < 3) {
                n0 = code_at(blk + 1, c0);
                n1 = code_at(blk + 1, c0 + 4);
              }
              uint4 h0a, h0b, h1a, h1b;
              h0a.x = e4m3x2_to_f16x2(a0.x); h0a.y = e4m3x2_to_f16x2(a0.x >> 16);
              h0a.z = e4m3x2_to_f16x2(a0.y); h0a.w = e4m3x2_to_f16x2(a0.y >> 16);
              h0b.x = e4m3x2_to_f16x2(a0.z); h0b.y = e4m3x2_to_f16x2(a0.z >> 16);
              h0b.z = e4m3x2_to_f16x2(a0.w); h0b.w = e4m3x2_to_f16x2(a0.w >> 16);
              h1a.x = e4m3x2_to_f16x2(a1.x); h1a.y = e4m3x2_to_f16x2(a1.x >> 16);
              h1a.z = e4m3x2_to_f16x2(a1.y); h1a.w = e4m3x2_to_f16x2(a1.y >> 16);
              h1b.x = e4m3x2_to_f16x2(a1.z); h1b.y = e4m3x2_to_f16x2(a1.z >> 16);
              h1b.z = e4m3x2_to_f16x2(a1.w); h1b.w = e4m3x2_to_f16x2(a1.w >> 16);
              const int R = 32 * cw + 8 * blk + r8;
              const int x = R & 7;
              const int ca = 2 * c0 + (odd_first ? 1 : 0), cb = 2 * c0 + (odd_first ? 0 : 1);
              __syncwarp();  // every lane's loads of this block precede the overwrite
              uint8_t* const d0 = reg + R * 128;
              uint8_t* const d1 = reg + 16384 + R * 128;
              sts128(d0 + ((ca ^ x) << 4), odd_first ? h0b : h0a);
              sts128(d0 + ((cb ^ x) << 4), odd_first ? h0a : h0b);
              sts128(d1 + ((ca ^ x) << 4), odd_first ? h1b : h1a);
              sts128(d1 + ((cb ^ x) << 4), odd_first ? h1a : h1b);
              if (blk < 3) {
                a0 = n0;
                a1 = n1;
              }
            }
            tc::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tc::smem_u32(&v_cvt[st]));
          }
          if (pending && (j == 1 || j == s.ntiles - 1)) {
            drain(prev, sg - 1);
            pending = false;
          }
        }
        if (pending) drain(prev, sg - 1);
        prev = s;
        pending = true;
        w = s.next;
      }
      if (pending) drain(prev, sg - 1);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) tstamp(251, 51);
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, TMEM_COLS);
  }
  // ---- grid-wide barrier (cooperative launch: all CTAs are resident), then
  //      every CTA joins the partials of its share of the output rows ----
  // part counts of this CTA's merge rows (computed while waiting)
  const int nwarps = (int)(blockDim.x >> 5);
  const int my_gr = r0 + warp;
  int my_nctx = sm_mcnt[2 * warp], my_ndec = sm_mcnt[2 * warp + 1];
  if (threadIdx.x == 0) {
    if (early) pdl_wait();  // the rows kernel's context partials are complete
    tstamp(249, 49);
    // monotonic barrier: the 64-bit word grid_ctr[0..1] grows by exactly
    // kLaunchStride per launch (G arrivals + the last arriver's pad), so a
    // launch starts at a multiple of the stride whatever G the plans on this
    // workspace use; the CTAs poll the counter itself — no reset and no
    // generation flip (one dependent round trip fewer after the last arrival
    // than round 2's count + generation pair)
    constexpr unsigned long long kLaunchStride = 256;  // > bif_max_ctas
    unsigned long long* const ctr = reinterpret_cast<unsigned long long*>(P.grid_ctr);
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(ctr) : "memory");
    tstamp(248, 48);
    const unsigned long long target = old / kLaunchStride * kLaunchStride + (unsigned long long)P.G;
    if (old + 1ull == target) {
      // the last arrival: every CTA has taken its last decode column — the
      // queue starts at 0 next launch; pad the count to the next stride (no
      // CTA of the next launch arrives before this grid has completed)
      if (P.dyn) asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(P.col_ctr) : "memory");
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(ctr), "l"(kLaunchStride - (unsigned long long)P.G) : "memory");
    } else {
      unsigned long long cur;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(ctr) : "memory");
      } while (cur < target);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) tstamp(252, 52);
  // append+attend: every CTA has read lens (before the barrier); advance it
  if (P.lens_out && blockIdx.x == 0)
    for (int i = threadIdx.x; i < P.b; i += blockDim.x) P.lens_out[i] = dec_len(P, i) - P.lens_offset;
  for (int gr = my_gr; gr < r1; gr += nwarps) {
    if (gr != my_gr) {
      const int i = gr / P.h, j = gr - i * P.h;
      const int c = j / P.p;
      my_nctx = ctx_parts(P, c, (i * P.p + (j - c * P.p)) / P.N);
      my_ndec = dec_parts(P, i, c / P.gpc);
    }
    merge_row(P, gr, lane, my_nctx, my_ndec);
  }
  __syncthreads();
  if (threadIdx.x == 0) tstamp(253, 53);
}

}  // namespace ba
