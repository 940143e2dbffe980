// bifattn_api.cu — host side of the C ABI declared in include/bifattn.h:
// validation, planning (splits, kernel choice), workspace layout, launches.
//
// Plans of one bifurcated step:
//   TC  (bf16, d = 128, b*p >= 16 rows share the context tile): ONE persistent
//       launch of bif_tc_kernel (bif_tc.cuh) — context tiles (Kc/Vc read once
//       for all b samples, Eq. 3-4 context rows) and decode
//       tiles (Kd/Vd per sample) stream through one
//       TMA/tcgen05 pipeline; the last partial of each (group, row chunk) merges.
//   FMA (fp32, other d, few rows): context FMA kernel + decode FMA kernel
//       (fma_partial.cuh) + merge kernel (merge.cuh): three launches.
// The replicated-KV baseline runs the same kernels with no context branch.
#include <algorithm>
#include <mutex>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/bifattn.h"
#include "common.cuh"
#include "bif_tc.cuh"
#include "ctx_rows2.cuh"
#include "fma_partial.cuh"
#include "merge.cuh"
#include "append.cuh"
#include "lse_merge.cuh"
#include "ctx_rows.cuh"
#include "stream_read.cuh"

namespace {

// Planner / experiment knobs.  Release builds compile every knob to its
// default (no environment-dependent behaviour on the product path); only
// BIFATTN_EXPERIMENTS builds (the round-1 sweeps) read the environment.
#ifdef BIFATTN_EXPERIMENTS
int knob_i(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
double knob_d(const char* name, double dflt) {
  const char* e = getenv(name);
  return e ? atof(e) : dflt;
}
#else
constexpr int knob_i(const char*, int dflt) { return dflt; }
constexpr double knob_d(const char*, double dflt) { return dflt; }
#endif

thread_local int g_last_cuda_error = 0;
thread_local char g_plan_buf[512];
thread_local void* g_trace = nullptr;
thread_local void* const* g_events = nullptr;
thread_local int g_nevents = 0;

// Brackets launch k with the caller's timing events (ba_set_launch_events).
struct LaunchRec {
  cudaStream_t st;
  int k = 0;
  explicit LaunchRec(cudaStream_t s) : st(s) {}
  void begin() {
    if (g_events && k < g_nevents) cudaEventRecord((cudaEvent_t)g_events[2 * k], st);
  }
  int end() {
    cudaError_t e = cudaGetLastError();
    if (g_events && k < g_nevents) cudaEventRecord((cudaEvent_t)g_events[2 * k + 1], st);
    ++k;
    if (e != cudaSuccess) {
      g_last_cuda_error = (int)e;
      return BA_ECUDA;
    }
    return BA_OK;
  }
};

struct DevInfo {
  int sms = 0;
  int major = 0;
  bool ok = false;
};

std::mutex g_mu;
DevInfo g_dev[64];
bool g_dev_init[64];

int device_info(DevInfo* out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return BA_ENODEV;
  }
  if (dev < 0 || dev >= 64) return BA_ENODEV;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_dev_init[dev]) {
    DevInfo di;
    int major = 0, sms = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      cudaGetLastError();
      return BA_ENODEV;
    }
    di.major = major;
    di.sms = sms;
    di.ok = (major == 10);
    g_dev[dev] = di;
    g_dev_init[dev] = true;
  }
  *out = g_dev[dev];
  return out->ok ? BA_OK : BA_ENODEV;
}

inline int cdiv(long a, long b) { return (int)((a + b - 1) / b); }

struct Plan {
  int D = 0;
  bool bf16 = false;
  int elem = 0;
  bool replicated = false;
  int ctx_mode = 0;  // 0 none (replicated baseline), 1 FMA kernel, 2 in the tcgen05 kernel
  bool tc = false;   // single-launch tcgen05 plan
  // tcgen05 plan
  int tc_N = 0, tc_nrc = 0, tc_ntile_c = 0, tc_ntile_d = 0, tc_G = 0, tc_nst = 0, tc_npb = 1;
  int tc_Sc = 0, tc_Sd = 0, tc_smem = 0;
  int tc_bw = 0, tc_nband = 0;  // context band width (tiles), bands per group
  // rows-on-M context kernel (ctx_rows.cuh) for R = b*p >= 64 rows per group
  bool ctx_rows = false;
  int cr_nrb = 0, cr_ntile = 0, cr_tps = 0, cr_nsplit = 0, cr_items = 0, cr_grid = 0;
  // decode branch also in the rows kernel (p >= 32 rows per sample and group);
  // the second launch is then the light merge kernel, not the fused kernel
  bool cr_dec = false;
  // two 128-row blocks per item in ping-pong (ctx_rows2.cuh; Q by TMA only)
  bool cr_v2 = false;
  int cr_nrp = 0;
  int cr_items_ctx = 0;
  long long tc_Tc = 0, tc_T = 0;
  int tc_cs[ba::bif_max_ctas + 1];
  int tc_slot0[ba::bif_max_ctas];  // slot of each CTA's first segment part (bif_tc.cuh)
  size_t off_cnt = 0;
  // FMA context branch
  int nsc = 0, ctx_chunk = 0, rb_c = 1, nrb_c = 0;
  // FMA decode branch
  int nsd = 0, dec_chunk = 0, rb_d = 1, nrb_d = 0;
  int dec_stride = 0, dec_cap = 0, lens_offset = 0;
  int S = 0, dec_slot0 = 0;
  size_t off_o = 0, off_ml = 0, ws_bytes = 0;
  int launches = 0;
  // decode columns taken dynamically by the fused kernel's CTAs after their
  // static (context) range and computed on the CUDA cores (p = 1, bf16,
  // single-token, no FP8): the static table covers the context tiles only
  bool dyn = false;
  int dparts = 1, dunit = 1;  // dyn: parts per column, tiles per part
  int ntok = 1;  // query tokens per (sample, head) row group (multi-token step)
  bool kv8 = false;  // FP8 E4M3 KV cache (f4)
  int kv_elem = 0;   // bytes per KV element
};

// bifurcated_attn_decode_append: this step's K/V rows and the lens update.
struct AppendArgs {
  const void* k_new;
  const void* v_new;
  int32_t* lens;  // updated in place after the step
  int n;          // rows appended per (sample, group)
};

// Split the flat tile sequence [0, T) (chunk ends `ends`, increasing, last =
// T) into G non-empty contiguous CTA ranges cs[0..G].  Each CTA gets about the
// same cost = tiles + kSegPenalty per extra chunk it enters; a range stops at
// a chunk end when the leftover budget could not pay for another segment.
void plan_split(const std::vector<long long>& ends, long long T, long long Tc, int G, int* cs,
                bool whole_ctx_units, double kDecCost) {
  static const double kSegPenalty = knob_d("BIFATTN_SEG_PENALTY", 2.0);
  // cost of tiles [a, b)
  auto cost = [&](long long a, long long b) {
    const long long c0 = std::min(b, Tc) - std::min(a, Tc);
    return (double)c0 + kDecCost * (double)((b - a) - c0);
  };
  long long cur = 0;
  size_t ci = 0;  // index of the chunk containing cur
  for (int k = 0; k < G; ++k) {
    cs[k] = (int)cur;
    const int left = G - k;
    if (left == 1) {
      cur = T;
      break;
    }
    // remaining virtual work: tile costs + a penalty per remaining chunk start
    const double vrem = cost(cur, T) + kSegPenalty * (double)(ends.size() - ci - 1);
    double budget = vrem / left;
    const long long max_end = T - (left - 1);  // leave >= 1 tile per remaining CTA
    long long start = cur;
    while (cur < T) {
      const double rc = cost(cur, ends[ci]);
      if (rc <= budget + 0.5) {
        budget -= rc;
        cur = ends[ci];
        ++ci;
        if (budget < kSegPenalty + 1.0) break;  // no room for another segment
        budget -= kSegPenalty;
      } else if (whole_ctx_units && cur < Tc) {
        // banded context: units are never split (one partial slot per band);
        // take the unit if at least half of it fits the budget
        if (cur == start || budget >= 0.5 * rc) {
          cur = ends[ci];
          ++ci;
        }
        break;
      } else {
        const double unit = cur < Tc ? 1.0 : kDecCost;
        long long take = (long long)(budget / unit + 0.5);
        if (take < 1 && cur == start) take = 1;
        cur += take;
        break;
      }
    }
    if (cur <= start) cur = start + 1;
    if (cur > max_end) cur = max_end;
    while (ci < ends.size() && ends[ci] <= cur) ++ci;
  }
  cs[G] = (int)T;
}

int pick_rb(int rows) { return rows >= 4 ? 4 : (rows >= 2 ? 2 : 1); }

int validate(const ba_problem_t* pr) {
  if (!pr) return BA_ENULL;
  if (pr->dtype != BA_BF16 && pr->dtype != BA_FP32) return BA_EDTYPE;
  // FP8 KV cache (f4, reading R19): q / out stay bf16
  if (pr->kv_dtype == BA_FP8_E4M3 && pr->dtype != BA_BF16) return BA_EDTYPE;
  if (pr->b < 1 || pr->h < 1 || pr->g < 1 || pr->mc < 1 || pr->md_cap < 0) return BA_EINVAL;
  if (pr->h % pr->g != 0) return BA_EINVAL;
  if (pr->n_tok < 0 || pr->n_tok > 128 || (long long)pr->h * (pr->n_tok > 1 ? pr->n_tok : 1) > (1 << 20))
    return BA_EINVAL;
  const int d = pr->d;
  if (d != 16 && d != 32 && d != 64 && d != 128 && d != 256) return BA_EINVAL;
  // int32 index safety for the per-tensor element counts used in the kernels
  const long long kd = (long long)pr->b * pr->g * ((long long)pr->md_cap + pr->mc) * d;
  if (kd > (1ll << 40)) return BA_EINVAL;
  return BA_OK;
}

// The kernels see a multi-token step (n_tok = n > 1) as h*n query rows per
// sample in g groups (q [b][h][n][d] is [b][h*n][d]; the n tokens of a head are
// adjacent rows of its group) plus the intra-step causal bound per row.
inline int ntok_of(const ba_problem_t* pr) { return pr->n_tok > 1 ? pr->n_tok : 1; }
inline ba_problem_t effective(const ba_problem_t* pr) {
  ba_problem_t e = *pr;
  e.h = pr->h * ntok_of(pr);
  return e;
}

// Plan for the bifurcated step (replicated == false) or the replicated baseline.
int make_plan(const ba_problem_t* pr_in, int sms, bool replicated, Plan* pl) {
  int rc = validate(pr_in);
  if (rc) return rc;
  const ba_problem_t E = effective(pr_in);
  const ba_problem_t* pr = &E;
  Plan P;
  P.ntok = ntok_of(pr_in);
  P.D = pr->d;
  P.bf16 = pr->dtype == BA_BF16;
  P.elem = P.bf16 ? 2 : 4;
  P.kv8 = pr->kv_dtype == BA_FP8_E4M3;
  P.kv_elem = P.kv8 ? 1 : P.elem;
  P.replicated = replicated;
  const int b = pr->b, h = pr->h, g = pr->g, p = h / g;
  const int target = 4 * sms;  // CTAs of 128 threads per launch (~4 per SM)
  const int R = b * p;
  int tcN = 0;
  if (P.bf16 && pr->d == 128 && R >= 16 && !(pr->flags & BA_FLAG_FORCE_FMA)) {
    // tcgen05 plan: N = rows per chunk, a multiple of 16 and of p, >= p
    // N = 48/64 spill softmax registers (128 per thread at 512 threads) and
    // leave 2 K/V stages: measured 2x slower per tile than N = 32 (round-1
    // N sweep), which beats them even with twice the context row chunks.  So
    // the smallest legal N that covers min(R, 32) rows.
    static const int cands[] = {16, 32, 48, 64};
    const int want = R < 32 ? R : 32;
    for (int N : cands) {
      if (N % p) continue;
      if (P.kv8 && (N > 32 || P.ntok > 1)) continue;  // FP8 tensor-core kernel: N = 16 / 32, n = 1
      if (!tcN) tcN = N;  // smallest legal
      if (N >= want) {
        tcN = N;
        break;
      }
    }
    static const int n_env = knob_i("BIFATTN_N", 0);  // experiment override: BIFATTN_N=16|32|48|64
    if (n_env && n_env % p == 0 && (n_env == 16 || n_env == 32 || n_env == 48 || n_env == 64)) tcN = n_env;
  }
  static const int ctx_rows_env = knob_i("BIFATTN_CTX_ROWS", 1);  // BIFATTN_CTX_ROWS=0 disables the rows-on-M kernel
  // Rows-on-M context kernel for R >= 64 rows per group: measured faster
  // than the fused kernel's 32-row context passes on every such shape (round
  // 1: C3 104 -> 90 us, C4 163 -> 86 us, C5 2.7 -> 1.8 ms, 4-token C2b 137 ->
  // 111 us, 2-token C2b 86 -> 81 us); at R = 32 (C2b) it is slower (78 vs
  // 58.7 us: a 128-row pass costs more than a 32-row swap-AB pass).  BA_FLAG_CTX_ROWS forces it (any R), BA_FLAG_NO_CTX_ROWS or
  // BIFATTN_CTX_ROWS=0 keep the single fused launch.
  const bool want_rows = ((pr->flags & BA_FLAG_CTX_ROWS) || R >= 64 || ctx_rows_env == 2) &&
                         !(pr->flags & BA_FLAG_NO_CTX_ROWS) && !P.kv8;
  if (tcN && !replicated && ctx_rows_env && want_rows) {
    // context branch on the rows-on-M kernel; the fused kernel streams only
    // the decode tiles, so its N just has to hold p (smallest legal)
    P.ctx_rows = true;
    for (int N : {16, 32, 48, 64})
      if (N % p == 0) {
        tcN = N;
        break;
      }
    P.cr_nrb = cdiv(R, 128);
    P.cr_ntile = cdiv(pr->mc, 128);
    // decode items in the rows kernel?  (see below; decided first: the
    // two-block kernel runs them one block at a time, slower than the
    // one-block kernel's two threads per row)
    static const int rows_dec_env = knob_i("BIFATTN_ROWS_DEC", 1);  // BIFATTN_ROWS_DEC=0: decode stays in the fused kernel
    const long long dec_tiles = (long long)b * g * cdiv(pr->md_cap, 128);
    // (round 3: p = 1 decode branches go to the fused launch's dynamic
    // CUDA-core columns instead (C5); for C3 (p = 4) that plan measured 78 us
    // against 70 us with decode items here: its decode launch also joins 9
    // context partials per row)
    const bool dyn_cand = p == 1 && P.ntok == 1 && !P.kv8;
    const bool will_cr_dec = rows_dec_env && (p >= 32 || dec_tiles <= 4096 || rows_dec_env == 2) &&
                             p <= 128 && pr->md_cap >= 1 && !(dyn_cand && rows_dec_env != 2);
    // two-block ping-pong kernel (ctx_rows2.cuh) for context-only launches
    // whose Q blocks are TMA boxes (g = 1, or p divides 128), >= 2 row blocks
    // per group: C5's context 432 -> 360 us; with decode items (C3, C4) the
    // one-block kernel stays faster (C4 46.2 vs 48.6, C3 69.5 vs 75.4 us)
#ifdef BIFATTN_ROWS1
    P.cr_v2 = false;  // A/B variant: the one-block rows kernel
#else
    P.cr_v2 = (g == 1 || 128 % p == 0) && P.cr_nrb >= 2 && !will_cr_dec;
#endif
    P.cr_nrp = P.cr_v2 ? cdiv(P.cr_nrb, 2) : P.cr_nrb;
    // one wave of long items: every item pays a Q load, a pipeline refill and
    // a 64 KB partial (written here, read by the merge)
    static const int ns_env = knob_i("BIFATTN_ROWS_SPLITS", 0);  // experiment override: BIFATTN_ROWS_SPLITS
    int ns = ns_env > 0 ? ns_env : std::max(1, sms / (g * P.cr_nrp));
    ns = std::max(1, std::min(ns, P.cr_ntile));
    P.cr_tps = cdiv(P.cr_ntile, ns);
    P.cr_nsplit = cdiv(P.cr_ntile, P.cr_tps);
    P.cr_items = g * P.cr_nrp * P.cr_nsplit;
    P.cr_items_ctx = P.cr_items;
    // decode items too when p >= 32 (they fill the row block) or when the
    // decode part is small (<= 4096 tiles: C3, multi-token C2b), where a second
    // persistent launch costs more than the half-empty row blocks (measured:
    // C3 88.8 -> 78 us; C5's 131072 decode tiles stay in the fused kernel)
    // decode items too when p >= 32 (they fill the row block) or when the
    // decode part is small (<= 4096 tiles: C3, multi-token C2b), where a second
    // persistent launch costs more than the half-empty row blocks (measured:
    // C3 88.8 -> 78 us; C5's 131072 decode tiles stay in the fused kernel).
    // (Round 2 measured a decode launch running CONCURRENTLY with the rows
    // kernel on the SMs it leaves free — PDL, griddepcontrol.wait only before
    // the merge: the cooperative decode launch does not start until the rows
    // kernel has drained, so C3 took 124 us and C5 3.3 ms; not used.)
    if (will_cr_dec) {
      P.cr_dec = true;
      P.cr_items += b * g;
    }
    P.cr_grid = std::min(P.cr_items, sms);
  }
  if (tcN) {
    P.tc = true;
    P.ctx_mode = replicated ? 0 : 2;
    P.tc_N = tcN;
    P.tc_nrc = cdiv(R, tcN);
    P.dec_stride = replicated ? pr->mc + pr->md_cap : pr->md_cap;
    P.dec_cap = pr->md_cap;
    P.lens_offset = replicated ? pr->mc : 0;
    P.tc_ntile_c = (replicated || P.ctx_rows) ? 0 : cdiv(pr->mc, 128);
    P.tc_ntile_d = cdiv(P.lens_offset + P.dec_cap, 128);
    P.tc_Tc = (long long)g * P.tc_nrc * P.tc_ntile_c;
    // p = 1 decode columns (one query row against Kd[i][c]: a GEMV) on the
    // CUDA cores, taken dynamically after the static context range (round 3:
    // the narrow tensor-core decode tile cost ~1.6 us against ~1.0 for a
    // context tile and set the tail; a CUDA-core column tile is well under the
    // per-SM HBM time of a 64 KB tile)
    // p = 2 / 4 (GQA) columns read q as fp32 from extra shared memory and use
    // the P buffer as the join scratch: only where that keeps 3 K/V stages
    // (N = 16; the N = 32 fused plans have no room)
    auto pq_fits = [&](int pq) {
      if (pq <= 1) return true;
      const int fx = ba::bif::smem_fixed(tcN, 2, false) + ba::bif::cc_extra_bytes(pq);
      return (227 * 1024 - fx) / ba::bif::kStageBytes >= 3 && 2 * 256 * tcN * 2 >= 8 * pq * 512;
    };
#ifdef BIFATTN_NO_DYN
    P.dyn = false;  // A/B variant build: decode tiles in the static ranges (narrow path)
#else
    // p = 4 columns measured slower than the narrow tensor-core path (48.1 vs
    // 45.4 us, b=4 h=32 g=8 mc=1k md=8k); p = 2 faster (36.3 vs 41.0 us)
    P.dyn = (p == 1 || (p == 2 && !P.kv8)) && P.ntok == 1 && !P.cr_dec && P.tc_ntile_d > 0 &&
            pq_fits(p);
#endif
    const int cc_x = P.dyn && p > 1 ? ba::bif::cc_extra_bytes(p) : 0;  // extra shared memory
    P.tc_T = P.tc_Tc + (P.dyn ? 0 : (long long)g * b * P.tc_ntile_d);
    const int gmax = sms < ba::bif_max_ctas ? sms : ba::bif_max_ctas;
    P.tc_G = (int)(P.tc_T < gmax ? P.tc_T : gmax);
    if (P.tc_T == 0 || P.dyn) P.tc_G = gmax;  // no tiles (ctx_rows, md_cap = 0): the merge only; dyn: every SM
    // P double-buffered when that keeps the K/V stage count (else one slot)
    P.tc_npb = 2;
    if ((227 * 1024 - ba::bif::smem_fixed(tcN, 2, P.kv8) - cc_x) / ba::bif::kStageBytes <
        (227 * 1024 - ba::bif::smem_fixed(tcN, 1, P.kv8) - cc_x) / ba::bif::kStageBytes)
      P.tc_npb = 1;
    static const int npb_env = knob_i("BIFATTN_NPB", 0);  // experiment override: BIFATTN_NPB=1|2
    if (npb_env == 1 || npb_env == 2) P.tc_npb = npb_env;
    if (cc_x) P.tc_npb = 2;  // the join scratch of p = 2 / 4 columns needs both P slots
    const int avail = 227 * 1024 - ba::bif::smem_fixed(tcN, P.tc_npb, P.kv8) - cc_x;  // dynamic smem is 1 KB aligned
    P.tc_nst = avail / ba::bif::kStageBytes;
    if (P.tc_nst > 4) P.tc_nst = 4;
    P.tc_smem = P.tc_nst * ba::bif::kStageBytes + ba::bif::smem_fixed(tcN, P.tc_npb, P.kv8) + cc_x;
    const int gpc = tcN / p;  // groups per decode chunk
    const int ndc = (g + gpc - 1) / gpc;
    // context bands (ctx_unit, bif_tc.cuh): with several row chunks per group
    // the context is cut into bands of bw tiles whose row-chunk passes follow
    // each other (L2 re-reads instead of HBM); one band when nrc = 1
    static const int bw_env = knob_i("BIFATTN_BAND", 0);  // experiment override: BIFATTN_BAND=<tiles>
    // Default: one band.  Measured (round 1, profiles/r01/band_sweep.txt): bands
    // of 8/16/32 tiles were SLOWER on C3, C4, C5 and the 4-token C2b step —
    // the re-reads already hit L2 where the context fits, and a multi-chunk
    // tile pass is bound by the per-tile softmax, not by HBM.
    int bw_try = P.tc_ntile_c;
    if (P.tc_nrc > 1 && P.tc_ntile_c > 0 && bw_env > 0 && bw_env < P.tc_ntile_c) bw_try = bw_env;
    // Cost of a decode tile relative to a context tile pass, for balancing
    // the CTA ranges.  Measured optima (round 1 sweeps, profiles/r01/
    // deccost_sweep.txt): 1.7 at N = 16 (C2a), 1.25 at N = 32 (C2b and C5,
    // whose 1 GB context is re-read from HBM by its 8 row chunks), 2.0 when
    // several row chunks pass an L2-resident context (C3, the 4-token C2b
    // step: the re-reads are L2 hits, cheaper than decode tiles from HBM),
    // more for MQA's 128 passes over a 4 MB context (C4).
    static const double dc_env = knob_d("BIFATTN_DEC_COST", 0.0);
    // The re-reads hit L2 when the whole context fits in it, or when a chunk
    // is about as long as a CTA's range, so that the nrc passes over a group
    // run concurrently on neighbouring CTAs (not one after another in one CTA).
    const double ctx_bytes = 2.0 * g * (double)pr->mc * pr->d * P.elem;
    const bool l2_rereads = P.tc_nrc > 1 && (ctx_bytes <= 64.0 * (1 << 20) ||
                                             1.5 * P.tc_ntile_c * P.tc_G >= (double)P.tc_T);
    // (round-2 per-CTA timelines, scripts/timeline.py: a decode tile costs
    // 1.4x a context tile pass at N = 32 and 1.65x with the FP8 cache)
    double dec_cost = tcN == 16 ? 1.7 : (P.kv8 ? 1.65 : 1.4);
    if (l2_rereads) dec_cost *= P.tc_nrc >= 32 ? 2.4 : 1.6;
    if (dc_env > 0) dec_cost = dc_env;
    int sc = 0, sd = 0;
    for (; P.tc_T == 0;) {  // nothing to stream: empty ranges, merge only
      for (int k = 0; k <= P.tc_G; ++k) P.tc_cs[k] = 0;
      P.tc_bw = 1;
      P.tc_nband = 0;
      break;
    }
    for (; P.tc_T > 0;) {
      P.tc_bw = bw_try;
      P.tc_nband = P.tc_ntile_c ? cdiv(P.tc_ntile_c, P.tc_bw) : 0;
      const bool banded = P.tc_nband > 1;
      // unit ends in the flat [context | decode] tile space
      std::vector<long long> ends;
      for (int c = 0; P.tc_ntile_c && c < g; ++c) {
        long long f = (long long)c * P.tc_nrc * P.tc_ntile_c;
        for (int band = 0; band < P.tc_nband; ++band) {
          const int wb = std::min(P.tc_bw, P.tc_ntile_c - band * P.tc_bw);
          for (int r = 0; r < P.tc_nrc; ++r) {
            f += wb;
            ends.push_back(f);
          }
        }
      }
      for (int i = 0; P.tc_ntile_d && !P.dyn && i < b; ++i)
        for (int cb = 0; cb < ndc; ++cb)
          ends.push_back(P.tc_Tc + ba::bif::dec_chunk_end(g, gpc, P.tc_ntile_d, i, cb));
      // fewer static tiles than CTAs (dyn, tiny context): one tile per CTA,
      // the remaining CTAs' static ranges empty (at the END of the table, so
      // owner() / parts_of() still count only CTAs that write partials)
      const int Gs = P.tc_T < P.tc_G ? (int)P.tc_T : P.tc_G;
      plan_split(ends, P.tc_T, P.tc_Tc, Gs, P.tc_cs, banded, dec_cost);
      for (int k = Gs + 1; k <= P.tc_G; ++k) P.tc_cs[k] = (int)P.tc_T;
      sc = sd = 0;
      bool whole = true;
      long long prev = 0;
      for (size_t k = 0; k < ends.size(); ++k) {
        const int n = ba::bif::parts_of(P.tc_cs, P.tc_G, prev, ends[k]);
        if (prev < P.tc_Tc) {
          whole = whole && n == 1;
          sc = std::max(sc, n);
        } else {
          sd = std::max(sd, n);
        }
        prev = ends[k];
      }
      if (!banded) break;
      if (whole) {
        sc = P.tc_nband;  // one partial per band
        break;
      }
      bw_try = P.tc_ntile_c;  // a unit got split (tiny problem): plain order
    }
    // slot of each CTA's first segment part: its index among the CTAs sharing
    // the chunk that holds its first tile (banded context: the band, set in-kernel)
    for (int k = 0; k < P.tc_G; ++k) {
      const long long f = P.tc_cs[k];
      long long a = 0;
      if (f >= P.tc_T || P.tc_cs[k + 1] <= f) {
        P.tc_slot0[k] = 0;  // empty range
        continue;
      }
      if (f < P.tc_Tc) {
        a = (f / P.tc_ntile_c) * P.tc_ntile_c;
      } else {
        const long long ic = (f - P.tc_Tc) / P.tc_ntile_d;
        const int i = (int)(ic / g), cb = (int)(ic % g) / gpc;
        a = P.tc_Tc + ba::bif::dec_chunk_begin(g, gpc, P.tc_ntile_d, i, cb);
      }
      P.tc_slot0[k] = k - ba::bif::owner(P.tc_cs, P.tc_G, a);
    }
    if (P.ctx_rows) sc = P.cr_nsplit;  // context partials written by ctx_rows_kernel
    if (P.cr_dec) sd = 1;              // one decode partial per row, also from ctx_rows_kernel
    if (P.dyn) {
      // (column, part) units: at least ~6 per CTA so the queue balances the
      // CTAs, parts of >= 2 tiles (each part pays a q load and a join)
      const long long ncol = (long long)b * g;
#ifndef BIFATTN_DYN_UNITS
#define BIFATTN_DYN_UNITS 6
#endif
#ifndef BIFATTN_DYN_MIN_TILES
#define BIFATTN_DYN_MIN_TILES 2
#endif
      long long parts = ((long long)BIFATTN_DYN_UNITS * P.tc_G + ncol - 1) / ncol;
      if (parts > (P.tc_ntile_d + BIFATTN_DYN_MIN_TILES - 1) / BIFATTN_DYN_MIN_TILES)
        parts = (P.tc_ntile_d + BIFATTN_DYN_MIN_TILES - 1) / BIFATTN_DYN_MIN_TILES;
      if (parts < 1) parts = 1;
      P.dunit = (int)((P.tc_ntile_d + parts - 1) / parts);
      P.dparts = (P.tc_ntile_d + P.dunit - 1) / P.dunit;
      sd = P.dparts;                   // one decode partial per (row, part)
    }
    P.tc_Sc = sc;
    P.tc_Sd = sd;
    P.S = sc + sd;
    if (P.S < 1) P.S = 1;
    const size_t rows = (size_t)b * h;
    P.off_cnt = 0;                         // grid-barrier counter
    P.off_o = 256;
    P.off_ml = P.off_o + rows * P.S * 128 * sizeof(float);
    P.ws_bytes = P.off_ml + rows * P.S * 2 * sizeof(float);
    P.ws_bytes = (P.ws_bytes + 255) & ~(size_t)255;
    P.launches = P.ctx_rows ? 2 : 1;
    *pl = P;
    return BA_OK;
  }
  if (!replicated) {
    // context branch, FMA kernel: rows R = b*p share each Kc tile
    P.ctx_mode = 1;
    P.rb_c = pick_rb(R);
    P.nrb_c = cdiv(R, P.rb_c);
    long items = (long)g * P.nrb_c;
    int nsc = cdiv(target, items);
    nsc = nsc < 1 ? 1 : nsc;
    const int max_nsc = cdiv(pr->mc, 64);
    if (nsc > max_nsc) nsc = max_nsc;
    P.ctx_chunk = cdiv(cdiv(pr->mc, nsc), 32) * 32;
    P.nsc = cdiv(pr->mc, P.ctx_chunk);
    P.dec_stride = pr->md_cap;
    P.dec_cap = pr->md_cap;
    P.lens_offset = 0;
  } else {
    P.ctx_mode = 0;
    P.nsc = 0;
    P.dec_stride = pr->mc + pr->md_cap;
    P.dec_cap = pr->md_cap;
    P.lens_offset = pr->mc;
  }
  const int maxlen = P.lens_offset + P.dec_cap;
  P.rb_d = pick_rb(p);
  P.nrb_d = cdiv(p, P.rb_d);
  if (maxlen > 0) {
    long items = (long)b * g * P.nrb_d;
    int nsd = cdiv(target, items);
    nsd = nsd < 1 ? 1 : nsd;
    const int max_nsd = cdiv(maxlen, 64);
    if (nsd > max_nsd) nsd = max_nsd;
    P.dec_chunk = cdiv(cdiv(maxlen, nsd), 32) * 32;
    P.nsd = cdiv(maxlen, P.dec_chunk);
  } else {
    P.nsd = 0;
    P.dec_chunk = 32;
  }
  P.dec_slot0 = P.nsc;
  P.S = P.nsc + P.nsd;
  if (P.S < 1) P.S = 1;
  const size_t rows = (size_t)b * h;
  // bytes [0, 256) stay reserved in EVERY plan: the tensor-core plans keep
  // their self-resetting grid-barrier words there, and one workspace may serve
  // FMA and tensor-core problems alternately (e.g. speculative steps of n = 1
  // and n = 4 sharing a workspace sized for the larger one)
  P.off_cnt = 0;
  P.off_o = 256;
  P.off_ml = P.off_o + rows * P.S * P.D * sizeof(float);
  P.ws_bytes = P.off_ml + rows * P.S * 2 * sizeof(float);
  P.ws_bytes = (P.ws_bytes + 255) & ~(size_t)255;
  P.launches = (P.ctx_mode != 0 ? 1 : 0) + (P.nsd > 0 ? 1 : 0) + 1;
  *pl = P;
  return BA_OK;
}

template <typename T, int D, typename TK = T>
int launch_fma_rb(int rb, int grid, const ba::FmaParams& fp, LaunchRec& rec) {
  if (grid <= 0) return BA_OK;
  cudaStream_t st = rec.st;
  rec.begin();
  switch (rb) {
    case 1: ba::fma_partial_kernel<T, D, 1, TK><<<grid, 128, 0, st>>>(fp); break;
    case 2: ba::fma_partial_kernel<T, D, 2, TK><<<grid, 128, 0, st>>>(fp); break;
    default: ba::fma_partial_kernel<T, D, 4, TK><<<grid, 128, 0, st>>>(fp); break;
  }
  return rec.end();
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    else
      cudaGetLastError();
  });
  return fn;
}

// 3D bf16 tensor map with a 128-byte-swizzled box of (64, box1, box2).
// Per-thread caches of plans and tensor maps: a decode loop calls with the
// same problem (and usually the same buffers) every step, so planning and
// cuTensorMapEncodeTiled are paid once (host cost per call, not GPU time).
struct PlanKey {
  ba_problem_t prob;
  int sms;
  bool replicated;
};
struct PlanEntry {
  PlanKey key;
  Plan plan;
  bool valid = false;
};
thread_local PlanEntry g_plan_cache[4];
thread_local int g_plan_next = 0;

int cached_plan(const ba_problem_t* pr, int sms, bool replicated, const Plan** out) {
  PlanKey k;
  memset(&k, 0, sizeof k);
  k.prob = *pr;
  k.sms = sms;
  k.replicated = replicated;
  for (auto& e : g_plan_cache)
    if (e.valid && memcmp(&e.key, &k, sizeof k) == 0) {
      *out = &e.plan;
      return BA_OK;
    }
  PlanEntry& e = g_plan_cache[g_plan_next];
  g_plan_next = (g_plan_next + 1) & 3;
  e.valid = false;
  const int rc = make_plan(pr, sms, replicated, &e.plan);
  if (rc) return rc;
  e.key = k;
  e.valid = true;
  *out = &e.plan;
  return BA_OK;
}

// bf16 maps: box (64, box1, box2) = 128-byte rows; u8 maps (FP8 codes):
// box (128, box1, box2), also 128-byte rows.  Both 128-byte swizzled.
int encode_tmap_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                 uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box1, uint32_t box2,
                 bool u8) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return BA_ECUDA;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {u8 ? 128u : 64u, box1, box2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, u8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                  const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    g_last_cuda_error = 1000 + (int)r;
    return BA_ECUDA;
  }
  return BA_OK;
}

struct TmapEntry {
  const void* base;
  uint64_t d0, d1, d2, s1, s2;
  uint32_t b1, b2;
  bool u8;
  CUtensorMap map;
};
thread_local TmapEntry g_tmap_cache[16];
thread_local int g_tmap_n = 0, g_tmap_next = 0;

int make_tmap_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                 uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box1, uint32_t box2,
                 bool u8 = false) {
  for (int k = 0; k < g_tmap_n; ++k) {
    const TmapEntry& e = g_tmap_cache[k];
    if (e.base == base && e.d0 == d0 && e.d1 == d1 && e.d2 == d2 && e.s1 == stride1_bytes &&
        e.s2 == stride2_bytes && e.b1 == box1 && e.b2 == box2 && e.u8 == u8) {
      *m = e.map;
      return BA_OK;
    }
  }
  const int rc = encode_tmap_3d(m, base, d0, d1, d2, stride1_bytes, stride2_bytes, box1, box2, u8);
  if (rc) return rc;
  TmapEntry& e = g_tmap_cache[g_tmap_next];
  g_tmap_next = (g_tmap_next + 1) & 15;
  if (g_tmap_n < 16) ++g_tmap_n;
  e = TmapEntry{base, d0, d1, d2, stride1_bytes, stride2_bytes, box1, box2, u8, *m};
  return BA_OK;
}

// The dynamic-shared-memory opt-in is a per-device attribute of a kernel:
// set it once per (kernel, device), under the library mutex.
template <typename Kern>
int ensure_smem_attr(Kern* fn, int bytes, bool* done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
    cudaGetLastError();
    return BA_ENODEV;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  if (done[dev]) return BA_OK;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) {
    g_last_cuda_error = (int)e;
    return BA_ECUDA;
  }
  done[dev] = true;
  return BA_OK;
}

template <int N, int SWG, bool MT, bool KV8 = false>
int launch_bif_tc_n(const ba::BifTcParams& bp, int smem, uint32_t flags, LaunchRec& rec) {
  // the decode-only launch after the rows kernel starts on the SMs the rows
  // kernel leaves free: not cooperative (its grid barrier still completes —
  // the rows kernel ends on its own and frees the rest); every other launch
  // is cooperative (all CTAs co-resident before the grid barrier)
#ifdef BIFATTN_NONCOOP
  const bool coop = false;  // experiment: every fused launch non-cooperative
#else
  const bool coop = !(bp.ext_ctx > 0 && bp.Tc == 0);
#endif
  static bool attr_done[64];
  if (int rc = ensure_smem_attr(ba::bif_tc_kernel<N, SWG, MT, KV8>, 227 * 1024, attr_done)) return rc;
  // one cooperative launch (all CTAs co-resident: the kernel ends with a grid
  // barrier and the LSE merge); programmatic stream serialisation lets its
  // prologue overlap the previous kernel on the stream
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(bp.G);
  cfg.blockDim = dim3(ba::bif::threads(SWG));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = rec.st;
  cudaLaunchAttribute attr[2];
  // cooperative unless this is the early-start decode launch (see coop above)
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = coop ? 1 : 0;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = (flags & BA_FLAG_NO_PDL) ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  rec.begin();
  cudaError_t e = cudaLaunchKernelEx(&cfg, ba::bif_tc_kernel<N, SWG, MT, KV8>, bp);
  if (e != cudaSuccess) {
    g_last_cuda_error = (int)e;
    rec.end();
    return BA_ECUDA;
  }
  return rec.end();
}

// The merge launch, programmatically dependent on the partial kernel before it
// (PDL: it launches while that kernel drains; merge_kernel waits with
// griddepcontrol.wait before reading the partials).  Already begun with rec.
template <typename T, int D>
int launch_merge(const ba::MergeParams& mp, uint32_t flags, LaunchRec& rec) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cdiv(mp.rows, 8));
  cfg.blockDim = dim3(256);
  cfg.stream = rec.st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = (flags & BA_FLAG_NO_PDL) ? 0 : 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, ba::merge_kernel<T, D>, mp);
  if (e != cudaSuccess) {
    g_last_cuda_error = (int)e;
    rec.end();
    return BA_ECUDA;
  }
  return rec.end();
}

// tcgen05 step: streaming kernel + PDL-chained merge.  Replicated baseline:
// Kc = Vc = nullptr, Kd/Vd are the replicated caches [b][g][mc+md_cap][d].
int run_tc(const ba_problem_t* pr, const Plan& P, const void* q, const void* Kc, const void* Vc,
           const void* Kd, const void* Vd, const int32_t* lens, void* out, float* lse, void* ws,
           float scale_log2, cudaStream_t st, const AppendArgs* ap, const ba::AppendSrc& app) {
  ba::BifTcParams bp;
  memset(&bp, 0, sizeof bp);
  const int p = pr->h / pr->g;
  const uint64_t d = 128;
  int rc = BA_OK;
  const uint64_t ek = P.kv8 ? 1 : 2;  // bytes per KV element
  if (P.tc_Tc > 0) {
    rc = make_tmap_3d(&bp.tmKc, Kc, d, pr->mc, pr->g, d * ek, (uint64_t)pr->mc * d * ek, 128, 1, P.kv8);
    if (!rc) rc = make_tmap_3d(&bp.tmVc, Vc, d, pr->mc, pr->g, d * ek, (uint64_t)pr->mc * d * ek, 128, 1, P.kv8);
    if (!rc) rc = make_tmap_3d(&bp.tmQc, q, d, pr->h, pr->b, d * 2, (uint64_t)pr->h * d * 2, p, P.tc_N / p);
  }
  if (!rc && (P.tc_T > P.tc_Tc || P.dyn)) {
    const uint64_t ds = (uint64_t)P.dec_stride;
    const uint64_t bg = (uint64_t)pr->b * pr->g;
    rc = make_tmap_3d(&bp.tmKd, Kd, d, ds, bg, d * ek, ds * d * ek, 128, 1, P.kv8);
    if (!rc) rc = make_tmap_3d(&bp.tmVd, Vd, d, ds, bg, d * ek, ds * d * ek, 128, 1, P.kv8);
    if (!rc)
      rc = make_tmap_3d(&bp.tmQd, q, d, pr->h, pr->b, d * 2, (uint64_t)pr->h * d * 2,
                        std::min(P.tc_N, pr->h), 1);
    if (!rc && P.dyn) rc = make_tmap_3d(&bp.tmQ1, q, d, pr->h, pr->b, d * 2, (uint64_t)pr->h * d * 2, p, 1);
  }
  if (!rc && P.tc_Tc == 0)  // replicated baseline: q map for the decode chunks
    rc = make_tmap_3d(&bp.tmQc, q, d, pr->h, pr->b, d * 2, (uint64_t)pr->h * d * 2, p, P.tc_N / p);
  if (rc) return rc;
  bp.lens = lens;
  bp.lens_add = ap ? ap->n : 0;
  bp.lens_out = ap ? ap->lens : nullptr;
  bp.app = app;
  bp.b = pr->b; bp.h = pr->h; bp.g = pr->g; bp.p = p; bp.mc = pr->mc;
  bp.dec_cap = P.dec_cap; bp.lens_offset = P.lens_offset; bp.ntok = P.ntok;
  bp.N = P.tc_N;
  bp.nrc = P.tc_nrc; bp.ntile_c = P.tc_ntile_c; bp.ntile_d = P.tc_ntile_d;
  bp.bw = P.tc_bw > 0 ? P.tc_bw : 1; bp.nband = P.tc_nband;
  bp.spc = P.tc_N / p;
  bp.gpc = P.tc_N / p;
  bp.ndc = (pr->g + bp.gpc - 1) / bp.gpc;
  bp.qd_rows = std::min(P.tc_N, pr->h);
  bp.Tc = P.tc_Tc; bp.Td = P.tc_T - P.tc_Tc; bp.G = P.tc_G; bp.nst = P.tc_nst; bp.npb = P.tc_npb;
  static const int pf_env = knob_i("BIFATTN_PF", 0);  // L2 prefetch distance (tiles; measured slower: off)
  bp.pf_dist = pf_env;
  static const int rot_env = knob_i("BIFATTN_ROT", 0);  // context stream stagger (tiles per CTA index)
  bp.rot = rot_env;
  memcpy(bp.cs, P.tc_cs, sizeof(int) * (P.tc_G + 1));
  memcpy(bp.slot0, P.tc_slot0, sizeof(int) * P.tc_G);
  bp.ext_ctx = P.ctx_rows ? P.cr_nsplit : 0;
  bp.scale_log2 = scale_log2;
  bp.vscale = (P.kv8 && pr->v_scale > 0.f) ? pr->v_scale : 1.f;
  bp.S = P.S; bp.Sc = P.tc_Sc;
  bp.ws_o = reinterpret_cast<float*>(static_cast<char*>(ws) + P.off_o);
  bp.ws_ml = reinterpret_cast<float*>(static_cast<char*>(ws) + P.off_ml);
  bp.grid_ctr = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + P.off_cnt);
  bp.dyn = P.dyn ? 1 : 0;
  bp.ncol = P.dyn ? pr->b * pr->g : 0;
  bp.dparts = P.dparts;
  bp.dunit = P.dunit;
  bp.col_ctr = bp.grid_ctr + 2;
  bp.out = out;
  bp.lse = lse;
  bp.trace = static_cast<unsigned long long*>(g_trace);
  static const int dbg_skip = knob_i("BIFATTN_DBG", 0);
  bp.dbg = dbg_skip;
  LaunchRec rec(st);
  if (P.ctx_rows) {
    // context branch, rows on M (ctx_rows.cuh); the fused launch below streams
    // the decode tiles and joins these partials in its merge
    ba::CtxRowsParams cp;
    memset(&cp, 0, sizeof cp);
    rc = make_tmap_3d(&cp.tmKc, Kc, d, pr->mc, pr->g, d * 2, (uint64_t)pr->mc * d * 2, 128, 1);
    if (!rc) rc = make_tmap_3d(&cp.tmVc, Vc, d, pr->mc, pr->g, d * 2, (uint64_t)pr->mc * d * 2, 128, 1);
    if (rc) return rc;
    cp.q = q;
    cp.b = pr->b; cp.h = pr->h; cp.g = pr->g; cp.p = p; cp.mc = pr->mc;
    // Q blocks by TMA where a block is one box (rows on M = (sample, head j))
#ifdef BIFATTN_NO_QTMA
    if (false) {  // A/B variant: the softmax threads load Q
#else
    if (pr->g == 1) {
#endif
      cp.q_mode = 2;
      rc = make_tmap_3d(&cp.tmQ, q, d, (uint64_t)pr->b * pr->h, 1, d * 2, (uint64_t)pr->b * pr->h * d * 2, 128, 1);
    } else if (128 % p == 0) {
      cp.q_mode = 1;
      rc = make_tmap_3d(&cp.tmQ, q, d, pr->h, pr->b, d * 2, (uint64_t)pr->h * d * 2, p, 128 / p);
    }
    if (rc) return rc;
    cp.R = pr->b * p; cp.nrb = P.cr_nrb; cp.nrp = P.cr_nrp;
    cp.ntile = P.cr_ntile; cp.tps = P.cr_tps; cp.nsplit = P.cr_nsplit; cp.items = P.cr_items;
    cp.scale_log2 = scale_log2;
    cp.S = P.S;
    cp.items_ctx = P.cr_items_ctx;
    cp.trace = static_cast<unsigned long long*>(g_trace);
    cp.dec_slot = P.cr_nsplit;
    cp.lens = lens;
    cp.dec_cap = P.dec_cap;
    cp.lens_add = ap ? ap->n : 0;
    cp.app = app;
    cp.ntok = P.ntok;
    if (P.cr_dec) {
      const uint64_t ds = (uint64_t)P.dec_stride, bg = (uint64_t)pr->b * pr->g;
      rc = make_tmap_3d(&cp.tmKd, Kd, d, ds, bg, d * 2, ds * d * 2, 128, 1);
      if (!rc) rc = make_tmap_3d(&cp.tmVd, Vd, d, ds, bg, d * 2, ds * d * 2, 128, 1);
      if (rc) return rc;
    }
    cp.ws_o = bp.ws_o;
    cp.ws_ml = bp.ws_ml;
    static bool attr_done[64], attr_done2[64];
    if (P.cr_v2) {
      if (int rc2 = ensure_smem_attr(ba::ctx_rows2_kernel, ba::ctxr2::kSmem, attr_done2)) return rc2;
    } else if (int rc2 = ensure_smem_attr(ba::ctx_rows_kernel, ba::ctxr::kSmem, attr_done)) {
      return rc2;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P.cr_grid);
    cfg.blockDim = dim3(P.cr_v2 ? ba::ctxr2::kThreads : ba::ctxr::kThreads);
    cfg.dynamicSmemBytes = P.cr_v2 ? ba::ctxr2::kSmem : ba::ctxr::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = (pr->flags & BA_FLAG_NO_PDL) ? 0 : 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    rec.begin();
    const cudaError_t e = P.cr_v2 ? cudaLaunchKernelEx(&cfg, ba::ctx_rows2_kernel, cp)
                                  : cudaLaunchKernelEx(&cfg, ba::ctx_rows_kernel, cp);
    if (e != cudaSuccess) {
      g_last_cuda_error = (int)e;
      rec.end();
      return BA_ECUDA;
    }
    rc = rec.end();
    if (rc) return rc;
    if (P.cr_dec) {
      // both branches' partials are in the workspace: the light LSE merge
      ba::MergeParams mp;
      memset(&mp, 0, sizeof mp);
      mp.ws_o = bp.ws_o;
      mp.ws_ml = bp.ws_ml;
      mp.rows = pr->b * pr->h;
      mp.S = P.S;
      mp.h = pr->h;
      mp.p = p;
      mp.ctx_mode = 1;
      mp.nsc = P.cr_nsplit;
      mp.dec_slot0 = P.cr_nsplit;
      mp.nsd = 1;
      mp.out = out;
      mp.lse = lse;
      mp.lens_out = ap ? ap->lens : nullptr;
      mp.b = pr->b;
      mp.lens_add = ap ? ap->n : 0;
      mp.dec_cap = P.dec_cap;
      mp.vscale = 1.f;
      rec.begin();
      return launch_merge<__nv_bfloat16, 128>(mp, pr->flags, rec);
    }
  }
  // softmax warpgroups (override for experiments: BIFATTN_SWG=1|2)
  static const int swg_env = knob_i("BIFATTN_SWG", 0);
  int swg = (swg_env == 1 || swg_env == 2 || (swg_env == 4 && P.tc_N == 32)) ? swg_env : ba::bif::softmax_wgs(P.tc_N);
  if (P.dyn) swg = 2;  // the CUDA-core decode columns are written for 8 softmax warps
  if (P.kv8) {  // FP8 KV cache (single-token step, N = 16 / 32)
    switch (P.tc_N) {
      case 16: return launch_bif_tc_n<16, 2, false, true>(bp, P.tc_smem, pr->flags, rec);
      case 32: return launch_bif_tc_n<32, 2, false, true>(bp, P.tc_smem, pr->flags, rec);
    }
    return BA_EINVAL;
  }
  if (P.ntok > 1) {  // multi-token kernels (MT): the default warpgroup split only
    switch (P.tc_N) {
      case 16: return launch_bif_tc_n<16, 2, true>(bp, P.tc_smem, pr->flags, rec);
      case 32: return launch_bif_tc_n<32, 2, true>(bp, P.tc_smem, pr->flags, rec);
      case 48: return launch_bif_tc_n<48, 2, true>(bp, P.tc_smem, pr->flags, rec);
      case 64: return launch_bif_tc_n<64, 2, true>(bp, P.tc_smem, pr->flags, rec);
    }
    return BA_EINVAL;
  }
  switch (P.tc_N * 4 + swg) {
    case 16 * 4 + 1: return launch_bif_tc_n<16, 1, false>(bp, P.tc_smem, pr->flags, rec);
    case 16 * 4 + 2: return launch_bif_tc_n<16, 2, false>(bp, P.tc_smem, pr->flags, rec);
    case 32 * 4 + 1: return launch_bif_tc_n<32, 1, false>(bp, P.tc_smem, pr->flags, rec);
    case 32 * 4 + 2: return launch_bif_tc_n<32, 2, false>(bp, P.tc_smem, pr->flags, rec);
    case 32 * 4 + 4: return launch_bif_tc_n<32, 4, false>(bp, P.tc_smem, pr->flags, rec);
    case 48 * 4 + 2: return launch_bif_tc_n<48, 2, false>(bp, P.tc_smem, pr->flags, rec);
    case 64 * 4 + 2: return launch_bif_tc_n<64, 2, false>(bp, P.tc_smem, pr->flags, rec);
  }
  return BA_EINVAL;
}

template <typename T, int D, typename TK = T>
int run_plan(const ba_problem_t* pr, const Plan& P, const void* q, const void* Kc,
             const void* Vc, const void* Kd, const void* Vd, const int32_t* lens, void* out,
             float* lse, void* ws, cudaStream_t st,
             const AppendArgs* ap) {
  const int b = pr->b, h = pr->h, g = pr->g, p = h / g;
  float scale = pr->scale > 0.f ? pr->scale : 1.0f / sqrtf((float)D);
  ba::FmaParams fp;
  memset(&fp, 0, sizeof fp);
  fp.q = q; fp.Kc = Kc; fp.Vc = Vc; fp.Kd = Kd; fp.Vd = Vd; fp.lens = lens;
  fp.b = b; fp.h = h; fp.g = g; fp.p = p; fp.mc = pr->mc;
  fp.dec_stride = P.dec_stride; fp.dec_cap = P.dec_cap; fp.lens_offset = P.lens_offset;
  fp.ntok = P.ntok;
  fp.lens_add = ap ? ap->n : 0;
  // append+attend: the rows are stored by the attention kernels themselves
  // (append.cuh), no separate launch
  if (ap) {
    fp.app.k_new = ap->k_new;
    fp.app.v_new = ap->v_new;
    fp.app.Kd = const_cast<void*>(Kd);
    fp.app.Vd = const_cast<void*>(Vd);
    fp.app.n = ap->n;
    fp.app.row_bytes = D * (int)sizeof(TK);
    fp.app.dec_cap = P.dec_cap;
    fp.app.g = g;
  }
  // FP8 KV: K = code * k_scale, folded into the logit scale (R19)
  const float kscale = (P.kv8 && pr->k_scale > 0.f) ? pr->k_scale : 1.f;
  fp.scale_log2 = scale * kscale * ba::kLog2e;
  fp.nsc = P.nsc; fp.nsd = P.nsd;
  fp.ctx_chunk = P.ctx_chunk; fp.dec_chunk = P.dec_chunk;
  fp.nrb_c = P.nrb_c; fp.nrb_d = P.nrb_d;
  fp.S = P.S; fp.dec_slot0 = P.dec_slot0;
  fp.ws_o = reinterpret_cast<float*>(static_cast<char*>(ws) + P.off_o);
  fp.ws_ml = reinterpret_cast<float*>(static_cast<char*>(ws) + P.off_ml);
  int rc;
  if (P.tc) {
    if constexpr (sizeof(T) == 2 && D == 128)
      return run_tc(pr, P, q, Kc, Vc, Kd, Vd, lens, out, lse, ws, fp.scale_log2, st, ap, fp.app);
    return BA_EINVAL;
  }
  LaunchRec rec(st);
  // 1. context branch (FMA)
  if (P.ctx_mode == 1 && P.nsc > 0) {
    ba::FmaParams f = fp;
    f.n_ctx_items = g * P.nsc * P.nrb_c;
    rc = launch_fma_rb<T, D, TK>(P.rb_c, f.n_ctx_items, f, rec);
    if (rc) return rc;
  }
  // 2. decode branch (FMA): items b * g * nsd * nrb_d
  if (P.nsd > 0) {
    ba::FmaParams f = fp;
    f.n_ctx_items = 0;
    rc = launch_fma_rb<T, D, TK>(P.rb_d, b * g * P.nsd * P.nrb_d, f, rec);
    if (rc) return rc;
  }
  // 3. merge
  ba::MergeParams mp;
  mp.ws_o = fp.ws_o;
  mp.ws_ml = fp.ws_ml;
  mp.rows = b * h;
  mp.S = P.S;
  mp.h = h;
  mp.p = p;
  mp.ctx_mode = P.ctx_mode;
  mp.nsc = P.nsc;
  mp.dec_slot0 = P.dec_slot0;
  mp.nsd = P.nsd;
  mp.out = out;
  mp.lse = lse;
  mp.lens_out = ap ? ap->lens : nullptr;
  mp.b = b;
  mp.lens_add = ap ? ap->n : 0;
  mp.dec_cap = P.dec_cap;
  mp.vscale = (P.kv8 && pr->v_scale > 0.f) ? pr->v_scale : 1.f;
  const int warps_per_block = 8;
  rec.begin();
  (void)warps_per_block;
  return launch_merge<T, D>(mp, pr->flags, rec);
}

template <typename T, typename TK = T>
int run_d(const ba_problem_t* pr, const Plan& P, const void* q, const void* Kc, const void* Vc,
          const void* Kd, const void* Vd, const int32_t* lens, void* out, float* lse, void* ws,
          cudaStream_t st,
          const AppendArgs* ap = nullptr) {
  switch (pr->d) {
    case 16: return run_plan<T, 16, TK>(pr, P, q, Kc, Vc, Kd, Vd, lens, out, lse, ws, st, ap);
    case 32: return run_plan<T, 32, TK>(pr, P, q, Kc, Vc, Kd, Vd, lens, out, lse, ws, st, ap);
    case 64: return run_plan<T, 64, TK>(pr, P, q, Kc, Vc, Kd, Vd, lens, out, lse, ws, st, ap);
    case 128: return run_plan<T, 128, TK>(pr, P, q, Kc, Vc, Kd, Vd, lens, out, lse, ws, st, ap);
    case 256: return run_plan<T, 256, TK>(pr, P, q, Kc, Vc, Kd, Vd, lens, out, lse, ws, st, ap);
  }
  return BA_EINVAL;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int common_checks(const ba_problem_t* pr, const void* const* ptrs, int nptr, void* ws,
                  size_t ws_bytes, size_t need) {
  for (int k = 0; k < nptr; ++k) {
    if (!ptrs[k]) return BA_ENULL;
    if (!aligned16(ptrs[k])) return BA_EALIGN;
  }
  if (!ws || ws_bytes < need) return BA_EWORKSPACE;
  if (!aligned16(ws)) return BA_EALIGN;
  (void)pr;
  return BA_OK;
}

// Packed serving-step layout: [q | k_new | v_new | lens] in, [out | lse] out,
// each part starting at a 256-byte boundary.
struct StepLayout {
  size_t q, k, v, lens, in_bytes, out, lse, out_bytes;
};
StepLayout step_layout(const ba_problem_t* pr) {
  auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t e = pr->dtype == BA_BF16 ? 2 : 4;
  const size_t ekv = pr->kv_dtype == BA_FP8_E4M3 ? 1 : e;
  const size_t n = ntok_of(pr), d = pr->d;
  StepLayout L;
  L.q = 0;
  L.k = up((size_t)pr->b * pr->h * n * d * e);
  L.v = L.k + up((size_t)pr->b * pr->g * n * d * ekv);
  L.lens = L.v + up((size_t)pr->b * pr->g * n * d * ekv);
  L.in_bytes = L.lens + up((size_t)pr->b * 4);
  L.out = 0;
  L.lse = up((size_t)pr->b * pr->h * n * d * e);
  L.out_bytes = L.lse + up((size_t)pr->b * pr->h * n * 4);
  return L;
}

}  // namespace

extern "C" {

size_t ba_workspace_bytes(const ba_problem_t* prob) {
  if (validate(prob) != BA_OK) return 0;
  DevInfo di;
  int sms = device_info(&di) == BA_OK ? di.sms : 148;
  const Plan *a, *r;
  if (cached_plan(prob, sms, false, &a) != BA_OK) return 0;
  if (cached_plan(prob, sms, true, &r) != BA_OK) return 0;
  return a->ws_bytes > r->ws_bytes ? a->ws_bytes : r->ws_bytes;
}

int bifurcated_attn_decode(const ba_problem_t* prob, const void* q, const void* Kc,
                           const void* Vc, const void* Kd, const void* Vd,
                           const int32_t* lens, void* out, float* lse, void* workspace,
                           size_t workspace_bytes, void* stream) {
  int rc = validate(prob);
  if (rc) return rc;
  DevInfo di;
  rc = device_info(&di);
  if (rc) return rc;
  const Plan* PP;
  rc = cached_plan(prob, di.sms, false, &PP);
  if (rc) return rc;
  const Plan P = *PP;  // copy: the cache may evict the entry below
  const void* ptrs[] = {q, Kc, Vc, out, lens};
  rc = common_checks(prob, ptrs, 5, workspace, workspace_bytes, ba_workspace_bytes(prob));
  if (rc) return rc;
  if (prob->md_cap > 0) {
    if (!Kd || !Vd) return BA_ENULL;
    if (!aligned16(Kd) || !aligned16(Vd)) return BA_EALIGN;
  }
  if (lse && (reinterpret_cast<uintptr_t>(lse) & 3u)) return BA_EALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const ba_problem_t E = effective(prob);  // h*n query rows per sample
  if (P.kv8)
    return run_d<__nv_bfloat16, ba::e4m3_t>(&E, P, q, Kc, Vc, Kd, Vd, lens, out, lse, workspace, st);
  if (P.bf16)
    return run_d<__nv_bfloat16>(&E, P, q, Kc, Vc, Kd, Vd, lens, out, lse, workspace, st);
  return run_d<float>(&E, P, q, Kc, Vc, Kd, Vd, lens, out, lse, workspace, st);
}

int bifurcated_attn_decode_append(const ba_problem_t* prob, const void* q, const void* k_new,
                                  const void* v_new, const void* Kc, const void* Vc, void* Kd,
                                  void* Vd, int32_t* lens, void* out, float* lse,
                                  void* workspace, size_t workspace_bytes, void* stream) {
  int rc = validate(prob);
  if (rc) return rc;
  if (prob->md_cap < 1) return BA_EINVAL;
  DevInfo di;
  rc = device_info(&di);
  if (rc) return rc;
  const Plan* PP;
  rc = cached_plan(prob, di.sms, false, &PP);
  if (rc) return rc;
  const Plan P = *PP;
  const void* ptrs[] = {q, Kc, Vc, Kd, Vd, out, lens, k_new, v_new};
  rc = common_checks(prob, ptrs, 9, workspace, workspace_bytes, ba_workspace_bytes(prob));
  if (rc) return rc;
  if (lse && (reinterpret_cast<uintptr_t>(lse) & 3u)) return BA_EALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const ba_problem_t E = effective(prob);
  const AppendArgs ap{k_new, v_new, lens, ntok_of(prob)};
  if (P.kv8)
    return run_d<__nv_bfloat16, ba::e4m3_t>(&E, P, q, Kc, Vc, Kd, Vd, lens, out, lse, workspace, st, &ap);
  if (P.bf16)
    return run_d<__nv_bfloat16>(&E, P, q, Kc, Vc, Kd, Vd, lens, out, lse, workspace, st, &ap);
  return run_d<float>(&E, P, q, Kc, Vc, Kd, Vd, lens, out, lse, workspace, st, &ap);
}

int bifurcated_attn_decode_append_host(const ba_problem_t* prob, const void* hq,
                                       const void* hk_new, const void* hv_new,
                                       const int32_t* hlens, void* hout, float* hlse, void* dq,
                                       void* dk_new, void* dv_new, const void* Kc, const void* Vc,
                                       void* Kd, void* Vd, int32_t* dlens, void* dout,
                                       float* dlse, void* workspace, size_t workspace_bytes,
                                       void* stream) {
  int rc = validate(prob);
  if (rc) return rc;
  if (!hq || !hk_new || !hv_new || !hout) return BA_ENULL;
  DevInfo di;
  rc = device_info(&di);
  if (rc) return rc;
  const size_t e = prob->dtype == BA_BF16 ? 2 : 4;
  const size_t ekv = prob->kv_dtype == BA_FP8_E4M3 ? 1 : e;
  const size_t d = prob->d, n = ntok_of(prob);
  const size_t nq = (size_t)prob->b * prob->h * n * d * e;
  const size_t nkv = (size_t)prob->b * prob->g * n * d * ekv;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto cp = [&](void* dst, const void* src, size_t bytes, cudaMemcpyKind k) -> int {
    if (bytes == 0) return BA_OK;
    if (!dst) return BA_ENULL;
    const cudaError_t ce = cudaMemcpyAsync(dst, src, bytes, k, st);
    if (ce != cudaSuccess) {
      g_last_cuda_error = (int)ce;
      return BA_ECUDA;
    }
    return BA_OK;
  };
  if ((rc = cp(dq, hq, nq, cudaMemcpyHostToDevice))) return rc;
  if ((rc = cp(dk_new, hk_new, nkv, cudaMemcpyHostToDevice))) return rc;
  if ((rc = cp(dv_new, hv_new, nkv, cudaMemcpyHostToDevice))) return rc;
  if (hlens && (rc = cp(dlens, hlens, (size_t)prob->b * sizeof(int32_t), cudaMemcpyHostToDevice)))
    return rc;
  rc = bifurcated_attn_decode_append(prob, dq, dk_new, dv_new, Kc, Vc, Kd, Vd, dlens, dout, dlse,
                                     workspace, workspace_bytes, stream);
  if (rc) return rc;
  if ((rc = cp(hout, dout, nq, cudaMemcpyDeviceToHost))) return rc;
  if (hlse && dlse)
    return cp(hlse, dlse, (size_t)prob->b * prob->h * n * sizeof(float), cudaMemcpyDeviceToHost);
  return BA_OK;
}

size_t ba_step_in_bytes(const ba_problem_t* prob) {
  return validate(prob) == BA_OK ? step_layout(prob).in_bytes : 0;
}
size_t ba_step_out_bytes(const ba_problem_t* prob) {
  return validate(prob) == BA_OK ? step_layout(prob).out_bytes : 0;
}

int bifurcated_attn_decode_step_packed(const ba_problem_t* prob, const void* h_in, void* h_out,
                                       void* d_in, void* d_out, int with_lse, const void* Kc,
                                       const void* Vc, void* Kd, void* Vd, void* workspace,
                                       size_t workspace_bytes, void* stream) {
  int rc = validate(prob);
  if (rc) return rc;
  if (!h_in || !h_out || !d_in || !d_out) return BA_ENULL;
  if (!aligned16(d_in) || !aligned16(d_out)) return BA_EALIGN;
  const StepLayout L = step_layout(prob);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t ce = cudaMemcpyAsync(d_in, h_in, L.in_bytes, cudaMemcpyHostToDevice, st);
  if (ce != cudaSuccess) {
    g_last_cuda_error = (int)ce;
    return BA_ECUDA;
  }
  char* di = static_cast<char*>(d_in);
  char* dout = static_cast<char*>(d_out);
  rc = bifurcated_attn_decode_append(prob, di + L.q, di + L.k, di + L.v, Kc, Vc, Kd, Vd,
                                     reinterpret_cast<int32_t*>(di + L.lens), dout + L.out,
                                     with_lse ? reinterpret_cast<float*>(dout + L.lse) : nullptr,
                                     workspace, workspace_bytes, stream);
  if (rc) return rc;
  ce = cudaMemcpyAsync(h_out, d_out, with_lse ? L.out_bytes : L.lse, cudaMemcpyDeviceToHost, st);
  if (ce != cudaSuccess) {
    g_last_cuda_error = (int)ce;
    return BA_ECUDA;
  }
  return BA_OK;
}

int replicated_attn_decode(const ba_problem_t* prob, const void* q, const void* K,
                           const void* V, const int32_t* lens, void* out, float* lse,
                           void* workspace, size_t workspace_bytes, void* stream) {
  int rc = validate(prob);
  if (rc) return rc;
  DevInfo di;
  rc = device_info(&di);
  if (rc) return rc;
  const Plan* PP;
  rc = cached_plan(prob, di.sms, true, &PP);
  if (rc) return rc;
  const Plan P = *PP;  // copy: the cache may evict the entry below
  const void* ptrs[] = {q, K, V, out, lens};
  rc = common_checks(prob, ptrs, 5, workspace, workspace_bytes, ba_workspace_bytes(prob));
  if (rc) return rc;
  if (lse && (reinterpret_cast<uintptr_t>(lse) & 3u)) return BA_EALIGN;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const ba_problem_t E = effective(prob);
  if (P.kv8)
    return run_d<__nv_bfloat16, ba::e4m3_t>(&E, P, q, nullptr, nullptr, K, V, lens, out, lse, workspace, st);
  if (P.bf16)
    return run_d<__nv_bfloat16>(&E, P, q, nullptr, nullptr, K, V, lens, out, lse, workspace, st);
  return run_d<float>(&E, P, q, nullptr, nullptr, K, V, lens, out, lse, workspace, st);
}

int bifurcated_attn_decode_host(const ba_problem_t* prob, const void* hq, const void* hKc,
                                const void* hVc, const void* hKd, const void* hVd,
                                const int32_t* hlens, void* hout, float* hlse, void* dq,
                                void* dKc, void* dVc, void* dKd, void* dVd, int32_t* dlens,
                                void* dout, float* dlse, void* workspace,
                                size_t workspace_bytes, void* stream) {
  int rc = validate(prob);
  if (rc) return rc;
  if (!hq || !hKc || !hVc || !hlens || !hout) return BA_ENULL;
  if (prob->md_cap > 0 && (!hKd || !hVd)) return BA_ENULL;
  DevInfo di;
  rc = device_info(&di);
  if (rc) return rc;
  const size_t e = prob->dtype == BA_BF16 ? 2 : 4;
  const size_t ekv = prob->kv_dtype == BA_FP8_E4M3 ? 1 : e;
  const size_t d = prob->d;
  const size_t nq = (size_t)prob->b * prob->h * ntok_of(prob) * d * e;
  const size_t nc = (size_t)prob->g * prob->mc * d * ekv;
  const size_t nd = (size_t)prob->b * prob->g * prob->md_cap * d * ekv;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto cp = [&](void* dst, const void* src, size_t n, cudaMemcpyKind k) -> int {
    if (n == 0) return BA_OK;
    if (!dst) return BA_ENULL;
    cudaError_t ce = cudaMemcpyAsync(dst, src, n, k, st);
    if (ce != cudaSuccess) {
      g_last_cuda_error = (int)ce;
      return BA_ECUDA;
    }
    return BA_OK;
  };
  if ((rc = cp(dq, hq, nq, cudaMemcpyHostToDevice))) return rc;
  if ((rc = cp(dKc, hKc, nc, cudaMemcpyHostToDevice))) return rc;
  if ((rc = cp(dVc, hVc, nc, cudaMemcpyHostToDevice))) return rc;
  if ((rc = cp(dKd, hKd, nd, cudaMemcpyHostToDevice))) return rc;
  if ((rc = cp(dVd, hVd, nd, cudaMemcpyHostToDevice))) return rc;
  if ((rc = cp(dlens, hlens, (size_t)prob->b * sizeof(int32_t), cudaMemcpyHostToDevice)))
    return rc;
  rc = bifurcated_attn_decode(prob, dq, dKc, dVc, dKd, dVd, dlens, dout, dlse, workspace,
                              workspace_bytes, stream);
  if (rc) return rc;
  if ((rc = cp(hout, dout, nq, cudaMemcpyDeviceToHost))) return rc;
  if (hlse && dlse) {
    if ((rc = cp(hlse, dlse, (size_t)prob->b * prob->h * ntok_of(prob) * sizeof(float),
                  cudaMemcpyDeviceToHost)))
      return rc;
  }
  return BA_OK;
}

int ba_lse_merge(int n_parts, int rows, int d, int dtype, const void* out_parts,
                 const float* lse_parts, void* out, float* lse, void* stream) {
  if (n_parts < 1 || rows < 0 || d < 1 || d > 256) return BA_EINVAL;
  if (dtype != BA_BF16 && dtype != BA_FP32) return BA_EDTYPE;
  if (!out_parts || !lse_parts || !out) return BA_ENULL;
  DevInfo di;
  int rc = device_info(&di);
  if (rc) return rc;
  if (rows == 0) return BA_OK;
  ba::LseMergeParams mp{out_parts, lse_parts, out, lse, n_parts, rows, d};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int blocks = cdiv(rows, 8);
  if (dtype == BA_BF16)
    ba::lse_merge_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(mp);
  else
    ba::lse_merge_kernel<float><<<blocks, 256, 0, st>>>(mp);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_last_cuda_error = (int)e;
    return BA_ECUDA;
  }
  return BA_OK;
}

int ba_launches_per_call(const ba_problem_t* prob) {
  DevInfo di;
  int sms = device_info(&di) == BA_OK ? di.sms : 148;
  Plan P;
  int rc = make_plan(prob, sms, false, &P);
  return rc ? rc : P.launches;
}

const char* ba_plan_string(const ba_problem_t* prob) {
  DevInfo di;
  int sms = device_info(&di) == BA_OK ? di.sms : 148;
  Plan P;
  int rc = make_plan(prob, sms, false, &P);
  if (rc) {
    snprintf(g_plan_buf, sizeof g_plan_buf, "invalid (%d)", rc);
    return g_plan_buf;
  }
  char dyn_tag[64] = "";
  if (P.dyn) snprintf(dyn_tag, sizeof dyn_tag, ",dec=cuda_core_dyn(parts=%d)", P.dparts);
  if (P.tc && P.cr_dec)
    snprintf(g_plan_buf, sizeof g_plan_buf,
             "ctx_rows%s(blocks=%d,splits=%d,tiles/split=%d,items=%d+%d dec,ctas=%d) + merge "
             "launches=2 ws=%zu",
             P.cr_v2 ? "2" : "", P.cr_nrb, P.cr_nsplit, P.cr_tps, P.cr_items_ctx, P.cr_items - P.cr_items_ctx,
             P.cr_grid, P.ws_bytes);
  else if (P.tc && P.ctx_rows)
    snprintf(g_plan_buf, sizeof g_plan_buf,
             "ctx_rows%s(blocks=%d,splits=%d,tiles/split=%d,items=%d,ctas=%d) + "
             "dec_tc(N=%d,dec_tiles=%lld%s,ctas=%d,stages=%d,slots=%d+%d) launches=2 ws=%zu",
             P.cr_v2 ? "2" : "", P.cr_nrb, P.cr_nsplit, P.cr_tps, P.cr_items, P.cr_grid, P.tc_N,
             P.dyn ? (long long)prob->b * prob->g * P.tc_ntile_d : P.tc_T, dyn_tag,
             P.tc_G, P.tc_nst, P.tc_Sc, P.tc_Sd, P.ws_bytes);
  else if (P.tc)
    snprintf(g_plan_buf, sizeof g_plan_buf,
             "fused_tc(N=%d,nrc=%d,band=%d,ctx_tiles=%lld,dec_tiles=%lld%s,ctas=%d,stages=%d,pbuf=%d,"
             "slots=%d+%d,smem=%d) launches=1 ws=%zu",
             P.tc_N, P.tc_nrc, P.tc_bw, P.tc_Tc,
             P.dyn ? (long long)prob->b * prob->g * P.tc_ntile_d : P.tc_T - P.tc_Tc,
             dyn_tag, P.tc_G, P.tc_nst, P.tc_npb, P.tc_Sc,
             P.tc_Sd, P.tc_smem, P.ws_bytes);
  else
    snprintf(g_plan_buf, sizeof g_plan_buf,
             "ctx=fma(nsc=%d,chunk=%d,rb=%d) dec=fma(nsd=%d,chunk=%d,rb=%d) S=%d launches=%d "
             "ws=%zu",
             P.nsc, P.ctx_chunk, P.rb_c, P.nsd, P.dec_chunk, P.rb_d, P.S, P.launches, P.ws_bytes);
  if (P.kv8) {
    const size_t n = strlen(g_plan_buf);
    snprintf(g_plan_buf + n, sizeof g_plan_buf - n, " kv=e4m3");
  }
  return g_plan_buf;
}

const char* ba_launch_name(const ba_problem_t* prob, int k) {
  DevInfo di;
  int sms = device_info(&di) == BA_OK ? di.sms : 148;
  Plan P;
  if (make_plan(prob, sms, false, &P) != BA_OK) return nullptr;
  const char* names[4];
  int n = 0;
  if (P.tc && P.cr_dec) {
    names[n++] = "fused_rows";
    names[n++] = "merge";
  } else if (P.tc && P.ctx_rows) {
    names[n++] = "ctx_rows";
    names[n++] = "dec_tc_merge";
  } else if (P.tc) {
    names[n++] = "fused_tc";
  } else {
    if (P.ctx_mode == 1) names[n++] = "ctx_fma";
    if (P.nsd > 0) names[n++] = "dec_fma";
    names[n++] = "merge";
  }
  return (k >= 0 && k < n) ? names[k] : nullptr;
}

void ba_set_trace_buffer(void* dev_buf) { g_trace = dev_buf; }

int ba_stream_read_bench(const void* buf, size_t bytes, void* sink, void* stream) {
  if (!buf || !sink) return BA_ENULL;
  if (!aligned16(buf) || (reinterpret_cast<uintptr_t>(sink) & 3u)) return BA_EALIGN;
  DevInfo di;
  const int rc = device_info(&di);
  if (rc) return rc;
  const size_t n16 = bytes / 16;
  if (n16 == 0) return BA_OK;
  const size_t want = (n16 + 4 * 512 - 1) / (4 * 512);
  const unsigned grid = (unsigned)std::min<size_t>(want, (size_t)di.sms * 4);
  ba::stream_read_kernel<<<grid, 512, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(buf), n16, static_cast<unsigned*>(sink));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    g_last_cuda_error = (int)e;
    return BA_ECUDA;
  }
  return BA_OK;
}

int ba_plan_ctas(const ba_problem_t* prob, int32_t* cs, int cap) {
  DevInfo di;
  int sms = device_info(&di) == BA_OK ? di.sms : 148;
  Plan P;
  int rc = make_plan(prob, sms, false, &P);
  if (rc) return rc;
  if (!P.tc) return 0;
  if (cs) {
    for (int k = 0; k <= P.tc_G && k < cap; ++k) cs[k] = P.tc_cs[k];
  }
  return P.tc_G;
}

void ba_set_launch_events(void* const* events, int n) {
  g_events = n > 0 ? events : nullptr;
  g_nevents = n > 0 ? n : 0;
}

int ba_select_path(const ba_problem_t* prob, int policy, long long threshold) {
  const int rc = validate(prob);
  if (rc) return rc;
  if (policy == BA_PATH_BIFURCATED || policy == BA_PATH_NAIVE) return policy;
  if (policy != BA_PATH_AUTO) return BA_EINVAL;
  const long long th = threshold > 0 ? threshold : BA_AUTO_THRESHOLD;
  return (long long)prob->b * prob->mc > th ? BA_PATH_BIFURCATED : BA_PATH_NAIVE;
}

const char* ba_strerror(int code) {
  switch (code) {
    case BA_OK: return "ok";
    case BA_EINVAL: return "invalid problem shape";
    case BA_ENULL: return "null pointer";
    case BA_EALIGN: return "pointer not 16-byte aligned";
    case BA_EWORKSPACE: return "workspace missing or too small";
    case BA_EDTYPE: return "unsupported dtype";
    case BA_ENODEV: return "no sm_100 CUDA device (there is no CPU fallback)";
    case BA_ECUDA: return "CUDA error";
  }
  return "unknown error";
}

int ba_last_cuda_error(void) { return g_last_cuda_error; }

int ba_version(void) { return 3; }

}  // extern "C"
