/*
 * bifattn.h — C ABI of libbifattn.so: one incremental-decoding step of
 * context-aware bifurcated attention (arXiv 2403.08845) on NVIDIA B200 (sm_100a).
 *
 * THE OPERATION (§4.2, Eq. 3-4; code App. E.3)
 *   b samples share one prefill context.  For sample i in [0,b) and query head
 *   j in [0,h), with group c = j / p, p = h / g (layout `bgpnk`):
 *     S_c[t] = scale * <q[i,j,:], Kc[c,t,:]>             t in [0, mc)
 *                 — "einsum(bgpnk, gm_ck)": Kc has no batch axis
 *     S_d[t] = scale * <q[i,j,:], Kd[i,c,t,:]>           t in [0, lens[i])
 *                 — "einsum(bgpnk, bgm_dk)"
 *     w      = softmax(S_c ⊕ S_d)   ONE softmax over the joined row
 *                 (cat, then softmax: PAPER.md:1159-1166)
 *     out[i,j,:] = <w_c, Vc[c]> + <w_d, Vd[i,c]>          (Eq. 4)
 *     lse[i,j]   = ln sum_t exp(S_t)                      (natural log)
 *   This equals ordinary generalized multi-query attention over the replicated
 *   cache K = Kc ⊕ Kd[i] (proof App. E.1).
 *   The device computes the joint softmax as a log-sum-exp merge of per-split
 *   partials (m, l, o), which is the same function in exact arithmetic.
 *
 * LAYOUT — all tensors row-major and contiguous, all in ONE dtype (prob->dtype):
 *   q    [b][h][d]             query of this step (n = 1 token per sample;
 *                               [b][h][n][d] for a multi-token step, below)
 *   Kc,Vc[g][mc][d]            the single shared context cache ("compact shape
 *                               1hm_ck or simply hm_ck")
 *   Kd,Vd[b][g][md_cap][d]     per-sample decode caches, preallocated to md_cap;
 *                               positions [0, lens[i]) of sample i are valid
 *   lens int32 [b]  (device)   valid decode length per sample; values are
 *                               clamped to [0, md_cap] on the device (a device
 *                               cannot report errors synchronously)
 *   out  [b][h][d]             result, rounded to nearest-even in the dtype
 *   lse  float32 [b][h]        optional (NULL = not written)
 *
 * OWNERSHIP — the caller owns every buffer (PyTorch allocates them) and keeps
 *   them alive until the work on `stream` has finished.  The library never
 *   allocates or frees device memory per call; it caches per-device attributes
 *   and kernel attributes under a mutex, and per host thread the last plans
 *   (keyed by the problem) and TMA descriptors (keyed by pointer and shape).
 *
 * EXECUTION — every call is asynchronous on `stream` (a cudaStream_t passed as
 *   void*; NULL = legacy default stream), reentrant, and CUDA-graph capturable
 *   (no host synchronisation, no allocation, lens read on the device).
 *
 * ERRORS — host-side checks only; a call returns BA_OK (0) or a negative code
 *   and launches nothing on error.  There is NO CPU fallback: without an sm_100
 *   device every compute call returns BA_ENODEV.
 */
#ifndef BIFATTN_H
#define BIFATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { BA_BF16 = 0, BA_FP32 = 1, BA_FP8_E4M3 = 2 } ba_dtype_t;

enum {
  BA_OK = 0,
  BA_EINVAL = -1,     /* bad shape: h % g != 0, b/h/g < 1, mc < 1, md_cap < 0, unsupported d */
  BA_ENULL = -2,      /* a required pointer is NULL                                          */
  BA_EALIGN = -3,     /* a tensor pointer is not 16-byte aligned                             */
  BA_EWORKSPACE = -4, /* workspace NULL or smaller than ba_workspace_bytes()                */
  BA_EDTYPE = -5,     /* dtype not BA_BF16 / BA_FP32, or an FP8 cache with a non-bf16 dtype */
  BA_ENODEV = -6,     /* no CUDA device of compute capability 10.x (sm_100a)                 */
  BA_ECUDA = -7       /* a CUDA runtime call or kernel launch failed (see ba_last_cuda_error) */
};

/* flags (ba_problem_t.flags) */
#define BA_FLAG_FORCE_FMA 0x1u /* route every branch through the CUDA-core FMA kernel
                                  (tests use it to cover both kernel families)       */
#define BA_FLAG_NO_PDL 0x2u    /* do not use programmatic dependent launch           */
#define BA_FLAG_CTX_ROWS 0x4u  /* bf16, d = 128: run the context branch on the rows-on-M
                                  kernel also for b*p < 64 (default: b*p >= 64)       */
#define BA_FLAG_NO_CTX_ROWS 0x8u /* bf16, d = 128: keep the single fused launch (context
                                  in 32-row passes) also for b*p >= 64 (tests cover 
                                  every path)                                         */

typedef struct {
  int32_t b;        /* samples sharing the context, >= 1                                */
  int32_t h;        /* query heads (rank-local when sharded), >= 1                      */
  int32_t g;        /* KV groups (rank-local), >= 1, h % g == 0                         */
  int32_t d;        /* head dim (k = v): 16, 32, 64, 128 or 256           */
  int32_t mc;       /* shared context length, >= 1                                      */
  int32_t md_cap;   /* decode-cache capacity = position stride of Kd/Vd, >= 0           */
  ba_dtype_t dtype; /* dtype of q, Kc, Vc, Kd, Vd and out                               */
  float scale;      /* logit scale; <= 0 means 1/sqrt(d) (the paper omits it: reading R1) */
  uint32_t flags;   /* BA_FLAG_*; 0 for the default (fastest) path                      */
  int32_t n_tok;    /* query tokens per sample in this step (multi-token / speculative
                       verification step, App. G PAPER.md:1219-1226 "with n_g replacing
                       n"); 0 or 1 = the single-token step.  See MULTI-TOKEN below.    */
  ba_dtype_t kv_dtype; /* storage of Kc, Vc, Kd, Vd: BA_FP8_E4M3 for an FP8 cache (see
                       FP8 KV below); any other value = stored in `dtype` (0 = default)  */
  float k_scale;    /* FP8 KV: K = E4M3 code value * k_scale; <= 0 means 1            */
  float v_scale;    /* FP8 KV: V = E4M3 code value * v_scale; <= 0 means 1            */
} ba_problem_t;

/* FP8 KV (kv_dtype = BA_FP8_E4M3, FAQ 5:
 * quantised attention "will effectively reduce the memory I/O for KV cache by
 * a factor of 2"; reading R19):
 *   Kc, Vc [g][mc][d] and Kd, Vd [b][g][md_cap][d] hold one-byte OCP FP8 E4M3
 *   codes (bias 7, no infinities); one fp32 scale per tensor kind, shared by
 *   the context and decode caches.  q and out stay bf16 (dtype must be
 *   BA_BF16).  The step is the same attention over the dequantised cache
 *   (code value x scale); the kernels convert codes to f16 exactly, fold
 *   k_scale into the logit scale and apply v_scale in the final merge.  The
 *   tensor-core path converts q to f16 (exact for bf16 values of magnitude in
 *   [2^-17, 65504]; the caller keeps |q| < 65504), so P enters the PV MMA as
 *   one f16 operand.  k_new / v_new of the append entry points are codes too.
 *   Algorithmic bytes: 2*1*d*g*(mc + sum lens) + 2*2*b*h*d. */

/* MULTI-TOKEN STEP (n_tok = n > 1):
 *   q, out [b][h][n][d], lse [b][h][n]: token k of head j of sample i.
 *   The n tokens' own K/V are the LAST n valid positions of the decode cache
 *   (already appended, like the single-token step's current token, reading
 *   R3), so token k sees every context position and the decode positions
 *     t < lens[i] - (n - 1 - k)        (intra-step causal mask; SPEC.md:441-449
 *                                       "mask offset m_c + m_d")
 *   and none when that bound is <= 0.  Kc/Vc and Kd/Vd are still read once
 *   per step for all n tokens (the I/O amortisation App. G describes).
 *   n = 1 is exactly the single-token step. */

/* Bytes of device workspace bifurcated_attn_decode() / replicated_attn_decode()
 * need: a 256-byte header (the fused kernel's grid barrier: a 64-bit arrival
 * count that grows by 256 per launch; the dynamic decode-unit queue counter,
 * left at 0 by every completed launch), then fp32 partials (m, l, o[d]) per
 * output row and split.  Returns 0 for an invalid problem.  The workspace must
 * be 16-byte aligned and ZEROED ONCE before its first use (cudaMemset); one
 * workspace then serves any number of back-to-back calls of any problems (and
 * CUDA graph replays) on one stream.  Calls that may run concurrently need
 * separate workspaces.
 * Concurrency note: the fused launch is cooperative (its grid barrier needs
 * every CTA resident); the decode-only launch that follows the rows kernel
 * (long contexts with many samples) is not, so that it can start on the SMs
 * the rows kernel leaves free — it needs every SM of the device to become
 * available to it eventually (no other kernel may occupy SMs indefinitely
 * while it runs, e.g. one waiting on this step's output). */
size_t ba_workspace_bytes(const ba_problem_t* prob);

/* One decode step of bifurcated attention (see above).  Kc/Vc are read from
 * HBM once for the whole batch; Kd/Vd once per sample.
 *   prob              problem descriptor (host pointer)
 *   q, Kc, Vc, Kd, Vd device pointers, layouts above, 16-byte aligned
 *   lens              device int32 [b]
 *   out               device [b][h][d]; must not alias any input
 *   lse               device float32 [b][h] or NULL
 *   workspace         device, >= ba_workspace_bytes(prob) bytes
 *   stream            cudaStream_t (as void*)
 * Returns BA_OK or a negative BA_E* code. */
int bifurcated_attn_decode(const ba_problem_t* prob, const void* q, const void* Kc,
                           const void* Vc, const void* Kd, const void* Vd,
                           const int32_t* lens, void* out, float* lse, void* workspace,
                           size_t workspace_bytes, void* stream);

/* KV append + attention of one decode step in one call (
 * the per-step "+K_prev / +V_prev" cache write of PAPER.md Table 5 :982-987,
 * SPEC.md:214-222).  With n = max(prob->n_tok, 1):
 *   1. writes k_new, v_new [b][g][n][d] (this step's keys/values of the n
 *      query tokens) into Kd, Vd at positions lens[i] .. lens[i] + n - 1
 *      (lens clamped to [0, md_cap]; rows at positions >= md_cap are dropped);
 *   2. runs the bifurcated step exactly as bifurcated_attn_decode with the
 *      valid decode length min(lens[i] + n, md_cap) (the appended tokens see
 *      themselves — reading R3 — and the multi-token causal bound applies);
 *   3. stores lens[i] <- min(lens[i] + n, md_cap) on the device after every
 *      read of lens, so the next step's call (or a CUDA-graph replay) needs
 *      no host work.
 * The append is FUSED into the attention launch(es): the CTA that will read
 * the tile (or decode item) holding a new row stores it first — generic
 * stores, then a proxy fence, then its TMA loads; the CUDA-core kernel reads
 * the new rows from k_new / v_new directly — so the call launches exactly
 * what bifurcated_attn_decode launches (ba_launches_per_call).  Kd, Vd and
 * lens are modified; k_new/v_new 16-byte aligned; md_cap >= 1.  Errors as
 * bifurcated_attn_decode. */
int bifurcated_attn_decode_append(const ba_problem_t* prob, const void* q, const void* k_new,
                                  const void* v_new, const void* Kc, const void* Vc, void* Kd,
                                  void* Vd, int32_t* lens, void* out, float* lse,
                                  void* workspace, size_t workspace_bytes, void* stream);

/* One serving step with HOST inputs and outputs, the caches resident on the
 * device: copies this step's q, k_new, v_new (and lens, if hlens != NULL;
 * otherwise the device lens carries on from the previous step) from host
 * memory (pinned for async behaviour) into dq, dk_new, dv_new, dlens, runs
 * bifurcated_attn_decode_append (appends the rows, attends, advances dlens),
 * and copies out (and lse if hlse and dlse) back.  All on `stream`; returns
 * after enqueueing. */
int bifurcated_attn_decode_append_host(const ba_problem_t* prob, const void* hq,
                                       const void* hk_new, const void* hv_new,
                                       const int32_t* hlens, void* hout, float* hlse, void* dq,
                                       void* dk_new, void* dv_new, const void* Kc, const void* Vc,
                                       void* Kd, void* Vd, int32_t* dlens, void* dout,
                                       float* dlse, void* workspace, size_t workspace_bytes,
                                       void* stream);

/* One serving step with ONE host->device and ONE device->host copy (SURVEY
 * §8(f) row f2; the decode loop of PAPER.md Table 5's per-step accounting):
 * the caches stay resident; the host packs this step's inputs into one pinned
 * buffer and gets the result back in one:
 *   h_in / d_in  [ q | k_new | v_new | lens ]   ba_step_in_bytes(prob) bytes
 *   h_out / d_out[ out | lse ]                   ba_step_out_bytes(prob) bytes
 * each part starting at a 256-byte boundary (q [b][h][n][d], k_new / v_new
 * [b][g][n][d] in the cache type, lens int32 [b] = each cache's length BEFORE
 * this step; out [b][h][n][d], lse float32 [b][h][n], copied back only when
 * with_lse != 0).  Runs H2D(in), bifurcated_attn_decode_append (rows appended
 * into Kd, Vd; lens advanced inside d_in), D2H(out) on `stream` and returns
 * after enqueueing — the whole step is CUDA-graph capturable.  d_in / d_out
 * are caller-owned device buffers (16-byte aligned), h_in / h_out pinned host
 * memory for asynchronous copies. */
size_t ba_step_in_bytes(const ba_problem_t* prob);
size_t ba_step_out_bytes(const ba_problem_t* prob);
int bifurcated_attn_decode_step_packed(const ba_problem_t* prob, const void* h_in, void* h_out,
                                       void* d_in, void* d_out, int with_lse, const void* Kc,
                                       const void* Vc, void* Kd, void* Vd, void* workspace,
                                       size_t workspace_bytes, void* stream);

/* The same step with HOST inputs and outputs (end-to-end entry point): copies
 * q, Kc, Vc, Kd, Vd, lens from host memory (pinned for async behaviour) into
 * the caller-owned device buffers dq..dlens, runs bifurcated_attn_decode, and
 * copies out (and lse if both hlse and dlse are non-NULL) back to host memory,
 * all on `stream`.  Returns after enqueueing; synchronise the stream before
 * reading hout. */
int bifurcated_attn_decode_host(const ba_problem_t* prob, const void* hq, const void* hKc,
                                const void* hVc, const void* hKd, const void* hVd,
                                const int32_t* hlens, void* hout, float* hlse, void* dq,
                                void* dKc, void* dVc, void* dKd, void* dVd, int32_t* dlens,
                                void* dout, float* dlse, void* workspace,
                                size_t workspace_bytes, void* stream);

/* Non-bifurcated baseline ("K_c tensor is loaded b times"):
 * ordinary generalized multi-query decode attention over a REPLICATED cache
 *   K, V [b][g][mc + md_cap][d]   (context copied into every sample's cache)
 * sample i attends to positions [0, mc + lens[i]).  Same kernels, no shared
 * context branch.  Workspace: ba_workspace_bytes(prob). */
int replicated_attn_decode(const ba_problem_t* prob, const void* q, const void* K,
                           const void* V, const int32_t* lens, void* out, float* lse,
                           void* workspace, size_t workspace_bytes, void* stream);

/* Log-sum-exp join of partial results (the cross-GPU
 * context split): out_parts [n_parts][rows][d] (dtype) and lse_parts float32
 * [n_parts][rows] are n_parts results of the SAME rows, each the attention of
 * a row over a disjoint slice of its keys (e.g. rank r's slice of the
 * context, one rank also holding the decode part), with their natural-log
 * LSE as written by bifurcated_attn_decode.  Writes the attention over the
 * union of the slices (Eq. 4 "+", applied across slices):
 *   M = max_k lse_k;  out = sum_k e^(lse_k - M) out_k / sum_k e^(lse_k - M);
 *   lse = M + ln sum_k e^(lse_k - M)   (lse nullable).
 * A part with lse = -inf contributes nothing.  Device pointers; d <= 256;
 * one launch on `stream`.  The parts are rounded to the dtype before the
 * join (bf16: one extra rounding per part). */
int ba_lse_merge(int n_parts, int rows, int d, int dtype, const void* out_parts,
                 const float* lse_parts, void* out, float* lse, void* stream);

/* Number of kernel launches one bifurcated_attn_decode() call makes for this
 * problem on the current device (for the benchmark's launch count): 1 for the
 * fused tensor-core plan (one cooperative launch, b*p < 64 rows per group), 2
 * for the rows-on-M plan (rows kernel + merge, or rows kernel + fused decode
 * launch), 3 for the CUDA-core plan.  bifurcated_attn_decode_append launches
 * the same kernels (the append is fused into them). */
int ba_launches_per_call(const ba_problem_t* prob);

/* Human-readable kernel plan for this problem (static string owned by the
 * library, valid until the next call from the same thread). */
const char* ba_plan_string(const ba_problem_t* prob);

/* Name of kernel launch k (0-based, in launch order) of one call for this
 * problem, e.g. "fused_tc", "fused_rows", "ctx_rows", "dec_tc_merge",
 * "ctx_fma", "dec_fma", "merge" (static string), or NULL. */
const char* ba_launch_name(const ba_problem_t* prob, int k);

/* Instrumentation for the benchmark's per-kernel CUDA-event timing.  While
 * set, launch k (< n) of every subsequent call made BY THIS THREAD is
 * bracketed by cudaEventRecord(events[2k]) / cudaEventRecord(events[2k+1]) on
 * the call's stream.  `events` are caller-created cudaEvent_t handles (as
 * void*); the array must stay valid while set.  (NULL, 0) disables.  Recording
 * events between launches serialises programmatic-dependent launches. */
void ba_set_launch_events(void* const* events, int n);

/* Instrumentation: while set, the fused tensor-core kernel launched by THIS
 * thread writes tagged %globaltimer stamps into dev_buf (device, uint64
 * [gridDim][1024], zeroed by the caller), each tag<<56 | time_ns.  Per CTA:
 * [0,256) softmax: 1 start, 2/3 first tile of a context/decode segment,
 * 20 S ready, 21/22 fast/slow path, 23 P handed to MMA, 4 segment end,
 * 7 done; [256,512) producer: 30 stage free (TMA issue) per tile;
 * [512,768) MMA: 31 QK issued per tile; [768,1024) MMA: 32 PV issued.
 * NULL disables. */
void ba_set_trace_buffer(void* dev_buf);

/* Measurement instrumentation (not part of the attention step): one launch
 * of a read-only streaming kernel over `bytes` of device memory at `buf`
 * (16-byte aligned): 128-bit non-caching loads, 4 per thread in flight,
 * 4 CTAs of 512 threads per SM, XOR-folded so the loads cannot be elided
 * (`sink`: device uint32, written only on a magic fold value).  bench.py
 * times it with CUDA events (best of 10 over 2 GiB) as the read-only HBM
 * peak of the run.  Returns BA_OK or a BA_E* code. */
int ba_stream_read_bench(const void* buf, size_t bytes, void* sink, void* stream);

/* Work split of the tensor-core plan for this problem (bf16, d = 128): CTA k
 * streams flat tiles [cs[k], cs[k+1]) of [context tiles | decode tiles]
 * (128 positions each).  Writes min(cap, G + 1) entries to cs (nullable) and
 * returns G, or 0 if the problem takes the CUDA-core plan, or a BA_E* code. */
int ba_plan_ctas(const ba_problem_t* prob, int32_t* cs, int cap);

/* Workload-based switch (PAPER.md FAQ 4 :688-689: "one
 * can get the best of both worlds ... by triggering bifurcated attention under
 * high workload scenarios and using normal attention otherwise"; SPEC.md:257-
 * 258, :284-287 select_path):
 *   policy BA_PATH_BIFURCATED / BA_PATH_NAIVE force the choice; BA_PATH_AUTO
 *   returns bifurcated iff b * mc > threshold (threshold <= 0: the library's
 *   measured default, BA_AUTO_THRESHOLD).  A caller keeps the
 *   replicated cache [b][g][mc + md_cap][d] and calls replicated_attn_decode
 *   for BA_PATH_NAIVE, the bifurcated cache and bifurcated_attn_decode
 *   otherwise.  Returns BA_PATH_BIFURCATED or BA_PATH_NAIVE, or a BA_E* code
 *   for an invalid problem / policy. */
enum { BA_PATH_AUTO = 0, BA_PATH_BIFURCATED = 1, BA_PATH_NAIVE = 2 };
#define BA_AUTO_THRESHOLD 16384LL /* b*mc elements (SPEC.md:303 placeholder 2^14) */
int ba_select_path(const ba_problem_t* prob, int policy, long long threshold);

/* Message for a BA_* code (static string). */
const char* ba_strerror(int code);

/* The cudaError_t of the last BA_ECUDA on this thread (0 if none). */
int ba_last_cuda_error(void);

/* ABI version: 3 (2 added ba_problem_t.n_tok, the multi-token step; 3 added
 * kv_dtype, k_scale, v_scale: the FP8 KV cache). */
int ba_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BIFATTN_H */
