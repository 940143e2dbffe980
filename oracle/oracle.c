/*
 * oracle.c — plain, slow, obviously-correct fp64 CPU oracle for one incremental
 * decoding step of generalized multi-query attention (arXiv 2403.08845).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2403_08845_b200/) never links, imports or calls it, and shares no code,
 * header, table or helper with it.
 *
 * What it computes (the plain definition, not the bifurcated algorithm):
 *   The paper states that bifurcated attention "yield[s] the exact same results
 *   <w,V> as the original attention in Equation 1 and 2" (§4.2;
 *   proof App. E.1).  So the oracle is Eq. 1-2
 *   (§3.3) with one softmax per row (the code listing's
 *   "softmax ... (omitted)" between the two einsums, App. E.3),
 *   evaluated over the key set K = Kc ⊕ Kd (§4.1), with the
 *   context KV replicated into every sample's cache ("naively ... K_c tensor is
 *   loaded b times").
 *
 *   For sample i, head j (group c = j / p, p = h / g, reading R2),
 *   M = mc + lens[i]:
 *     Kfull = [ Kc[c, 0..mc-1] ; Kd[i, c, 0..lens[i]-1] ]   (concat order R5)
 *     l_t   = s * sum_x q[i,j,x] * Kfull[t,x]                (Eq. 1; scale R1)
 *     mx    = max_t l_t ; w_t = exp(l_t - mx) ; Z = sum_t w_t
 *     out[i,j,x] = (sum_t w_t * Vfull[t,x]) / Z             (Eq. 2)
 *     lse[i,j]   = mx + log(Z)
 *   All sums run left to right in fp64.  Inputs are widened to fp64 exactly at
 *   use (bf16 bit patterns or fp32), so input quantisation is not error (R14).
 *
 * Second mode, oracle_bifurcated_f64: the paper's bifurcated algorithm step by
 * step (Eq. 3-4; code App. E.3): context
 * logits against the single Kc (no b axis), decode logits against Kd[i],
 * concatenated, ONE softmax, weights split at mc, two value products summed.
 * Logits and weights are computed in the replicated mode's order, so they agree
 * bit-for-bit; the value product is split at mc and summed (Eq. 4), so outputs
 * agree to fp64 rounding (bit-for-bit when lens[i] = 0).  That agreement is the
 * App. E.1 proof run as a test.
 *
 * Pins (tests/test_oracle_pins.py): torch fp64 SDPA over the replicated cache,
 * the App. E.3 listing in torch fp64, closed forms (single key, q = 0, planted
 * key, lens = 0), SPEC worked examples (tests/golden/), softmax invariants,
 * MQA/MHA limits, bifurcated == replicated (weights bit-exact), mutation tests.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_BF16 0
#define OR_FP32 1

/* Widen one stored element to fp64 exactly. bf16 = top 16 bits of an fp32. */
static double widen(const void *base, size_t idx, int dtype) {
  if (dtype == OR_BF16) {
    uint32_t u = ((uint32_t)((const uint16_t *)base)[idx]) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
  }
  return (double)((const float *)base)[idx];
}

/* Validate the problem; returns 0 or -1. */
static int check(int b, int h, int g, int d, int mc, int md_cap, int dtype) {
  if (b < 1 || h < 1 || g < 1 || d < 1 || mc < 0 || md_cap < 0) return -1;
  if (h % g != 0) return -1;
  if (dtype != OR_BF16 && dtype != OR_FP32) return -1;
  return 0;
}

/* Number of valid decode positions of sample i (clamped to [0, md_cap]). */
static int dec_len(const int32_t *lens, int i, int md_cap) {
  int L = lens ? lens[i] : md_cap;
  if (L < 0) L = 0;
  if (L > md_cap) L = md_cap;
  return L;
}

/*
 * Replicated (non-bifurcated) attention, Eq. 1-2.  Computes the rows listed in
 * `rows` (row = i*h + j), or all b*h rows if rows == NULL.
 *   out     : [nrows][d]   fp64 normalised output
 *   lse     : [nrows]      fp64 natural-log sum-exp of the scaled logits (nullable)
 *   weights : [nrows][mc+md_cap] fp64 softmax weights, zero-padded (nullable)
 * Returns 0, or -1 on a bad problem / allocation failure.
 */
int oracle_attn_decode_f64(int b, int h, int g, int d, int mc, int md_cap, int dtype,
                           double scale, const void *q, const void *Kc, const void *Vc,
                           const void *Kd, const void *Vd, const int32_t *lens,
                           const int32_t *rows, int nrows, double *out, double *lse,
                           double *weights, int nthreads) {
  if (check(b, h, g, d, mc, md_cap, dtype)) return -1;
  if (!rows) nrows = b * h;
  const int p = h / g;
  const int Mcap = mc + md_cap;
  int err = 0;
  (void)nthreads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
  for (int r = 0; r < nrows; ++r) {
    const int row = rows ? rows[r] : r;
    const int i = row / h, j = row % h, c = j / p;
    const int M = mc + dec_len(lens, i, md_cap);
    /* Step 1: materialise this sample's full cache Kfull/Vfull = Kc ⊕ Kd[i]
     * for group c (the context replicated into sample i's cache). */
    double *Kf = (double *)malloc(sizeof(double) * (size_t)(M > 0 ? M : 1) * d);
    double *Vf = (double *)malloc(sizeof(double) * (size_t)(M > 0 ? M : 1) * d);
    double *l = (double *)malloc(sizeof(double) * (size_t)(M > 0 ? M : 1));
    if (!Kf || !Vf || !l || M < 1) {
      free(Kf); free(Vf); free(l);
#pragma omp atomic write
      err = 1;
      continue;
    }
    for (int t = 0; t < M; ++t) {
      for (int x = 0; x < d; ++x) {
        size_t src;
        if (t < mc) {
          src = ((size_t)c * mc + t) * d + x;
          Kf[(size_t)t * d + x] = widen(Kc, src, dtype);
          Vf[(size_t)t * d + x] = widen(Vc, src, dtype);
        } else {
          src = (((size_t)i * g + c) * md_cap + (t - mc)) * d + x;
          Kf[(size_t)t * d + x] = widen(Kd, src, dtype);
          Vf[(size_t)t * d + x] = widen(Vd, src, dtype);
        }
      }
    }
    /* Step 2: logits l_t = s * <q, Kfull_t>  (Eq. 1). */
    for (int t = 0; t < M; ++t) {
      double acc = 0.0;
      for (int x = 0; x < d; ++x)
        acc += widen(q, ((size_t)i * h + j) * d + x, dtype) * Kf[(size_t)t * d + x];
      l[t] = scale * acc;
    }
    /* Step 3: one softmax over all M positions. */
    double mx = l[0];
    for (int t = 1; t < M; ++t)
      if (l[t] > mx) mx = l[t];
    double Z = 0.0;
    for (int t = 0; t < M; ++t) {
      l[t] = exp(l[t] - mx); /* l now holds the unnormalised weights w_t */
      Z += l[t];
    }
    /* Step 4: out = (sum_t w_t Vfull_t) / Z  (Eq. 2). */
    for (int x = 0; x < d; ++x) {
      double acc = 0.0;
      for (int t = 0; t < M; ++t) acc += l[t] * Vf[(size_t)t * d + x];
      out[(size_t)r * d + x] = acc / Z;
    }
    if (lse) lse[r] = mx + log(Z);
    if (weights) {
      for (int t = 0; t < Mcap; ++t) weights[(size_t)r * Mcap + t] = t < M ? l[t] / Z : 0.0;
    }
    free(Kf); free(Vf); free(l);
  }
  return err ? -1 : 0;
}

/*
 * Bifurcated attention in fp64, the paper's algorithm in its own order
 * (Eq. 3-4; App. E.3 listing).  Same outputs/arguments as above.
 *   <q,Kc> : einsum(bgpnk, gm_ck) — Kc has no batch axis
 *   <q,Kd> : einsum(bgpnk, bgm_dk)
 *   cat along m, one softmax
 *   w split at mc; <w_c,Vc> + <w_d,Vd>
 */
int oracle_bifurcated_f64(int b, int h, int g, int d, int mc, int md_cap, int dtype,
                          double scale, const void *q, const void *Kc, const void *Vc,
                          const void *Kd, const void *Vd, const int32_t *lens,
                          const int32_t *rows, int nrows, double *out, double *lse,
                          double *weights, int nthreads) {
  if (check(b, h, g, d, mc, md_cap, dtype)) return -1;
  if (!rows) nrows = b * h;
  const int p = h / g;
  int err = 0;
  (void)nthreads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
  for (int r = 0; r < nrows; ++r) {
    const int row = rows ? rows[r] : r;
    const int i = row / h, j = row % h, c = j / p;
    const int md = dec_len(lens, i, md_cap);
    const int M = mc + md;
    double *Sc = (double *)malloc(sizeof(double) * (size_t)(mc > 0 ? mc : 1));
    double *Sd = (double *)malloc(sizeof(double) * (size_t)(md > 0 ? md : 1));
    double *oc = (double *)malloc(sizeof(double) * (size_t)d);
    double *od = (double *)malloc(sizeof(double) * (size_t)d);
    if (!Sc || !Sd || !oc || !od || M < 1) {
      free(Sc); free(Sd); free(oc); free(od);
#pragma omp atomic write
      err = 1;
      continue;
    }
    /* <q, Kc>: the context key of group c, shared by every sample. */
    for (int t = 0; t < mc; ++t) {
      double acc = 0.0;
      for (int x = 0; x < d; ++x)
        acc += widen(q, ((size_t)i * h + j) * d + x, dtype) *
               widen(Kc, ((size_t)c * mc + t) * d + x, dtype);
      Sc[t] = scale * acc;
    }
    /* <q, Kd>: sample i's own decode key. */
    for (int t = 0; t < md; ++t) {
      double acc = 0.0;
      for (int x = 0; x < d; ++x)
        acc += widen(q, ((size_t)i * h + j) * d + x, dtype) *
               widen(Kd, (((size_t)i * g + c) * md_cap + t) * d + x, dtype);
      Sd[t] = scale * acc;
    }
    /* Concatenate (context first) and take ONE softmax over the joined row. */
    double mx = mc > 0 ? Sc[0] : Sd[0];
    for (int t = 0; t < mc; ++t) if (Sc[t] > mx) mx = Sc[t];
    for (int t = 0; t < md; ++t) if (Sd[t] > mx) mx = Sd[t];
    double Z = 0.0;
    for (int t = 0; t < mc; ++t) { Sc[t] = exp(Sc[t] - mx); Z += Sc[t]; }
    for (int t = 0; t < md; ++t) { Sd[t] = exp(Sd[t] - mx); Z += Sd[t]; }
    /* Split the weights at mc; <w_c, Vc> and <w_d, Vd> as two separate
     * products, joined by summation (Eq. 4).  The split changes the fp64
     * summation order of the value product only, so outputs agree with the
     * replicated mode to rounding, while the weights (same order) agree
     * bit-for-bit. */
    for (int x = 0; x < d; ++x) {
      double acc = 0.0;
      for (int t = 0; t < mc; ++t) acc += Sc[t] * widen(Vc, ((size_t)c * mc + t) * d + x, dtype);
      oc[x] = acc;
    }
    for (int x = 0; x < d; ++x) {
      double acc = 0.0;
      for (int t = 0; t < md; ++t)
        acc += Sd[t] * widen(Vd, (((size_t)i * g + c) * md_cap + t) * d + x, dtype);
      od[x] = acc;
    }
    for (int x = 0; x < d; ++x) od[x] = oc[x] + od[x];
    if (weights) {
      const int Mcap = mc + md_cap;
      for (int t = 0; t < Mcap; ++t)
        weights[(size_t)r * Mcap + t] = t < mc ? Sc[t] / Z : (t < M ? Sd[t - mc] / Z : 0.0);
    }
    for (int x = 0; x < d; ++x) out[(size_t)r * d + x] = od[x] / Z;
    if (lse) lse[r] = mx + log(Z);
    free(Sc); free(Sd); free(oc); free(od);
  }
  return err ? -1 : 0;
}

/*
 * Multi-token step (App. G: n_g draft tokens decoded in one
 * step, "with n_g replacing n"; SPEC.md:441-449 decode_multi: "intra-step causal
 * masking (mask offset m_c+m_d)").  Plain masked attention, Eq. 1-2 over the
 * replicated cache Kfull = Kc ⊕ Kd[i][0..L_i), L_i = clamp(lens[i], 0, md_cap),
 * where the n query tokens of sample i sit at the last n cache positions
 * P_k = mc + L_i - n + k (their K/V already appended, reading R3) and token k
 * attends to the cache positions t <= P_k (causal mask).  Context positions
 * (t < mc) are always visible.  q, out [b][h][n][d]; row = (i*h + j)*n + k.
 * With n = 1 this is oracle_attn_decode_f64 exactly.
 */
int oracle_attn_decode_multi_f64(int b, int h, int n, int g, int d, int mc, int md_cap,
                                 int dtype, double scale, const void *q, const void *Kc,
                                 const void *Vc, const void *Kd, const void *Vd,
                                 const int32_t *lens, const int32_t *rows, int nrows,
                                 double *out, double *lse, double *weights, int nthreads) {
  if (check(b, h, g, d, mc, md_cap, dtype) || n < 1) return -1;
  if (!rows) nrows = b * h * n;
  const int p = h / g;
  const int Mcap = mc + md_cap;
  int err = 0;
  (void)nthreads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
  for (int r = 0; r < nrows; ++r) {
    const int row = rows ? rows[r] : r;
    const int k = row % n, ij = row / n;
    const int i = ij / h, j = ij % h, c = j / p;
    const int Li = dec_len(lens, i, md_cap);
    const int M = mc + Li;
    const long Pk = (long)mc + Li - n + k; /* this token's own cache position */
    double *l = (double *)malloc(sizeof(double) * (size_t)(M > 0 ? M : 1));
    if (!l || M < 1) {
      free(l);
#pragma omp atomic write
      err = 1;
      continue;
    }
    /* Logits over Kfull = Kc ⊕ Kd[i]; masked (weight 0) past the causal bound. */
    int any = 0;
    double mx = 0.0;
    for (int t = 0; t < M; ++t) {
      const int vis = t < mc || t <= Pk;
      if (!vis) continue;
      double acc = 0.0;
      for (int x = 0; x < d; ++x) {
        const double kv = t < mc ? widen(Kc, ((size_t)c * mc + t) * d + x, dtype)
                                 : widen(Kd, (((size_t)i * g + c) * md_cap + (t - mc)) * d + x, dtype);
        acc += widen(q, (((size_t)i * h + j) * n + k) * d + x, dtype) * kv;
      }
      l[t] = scale * acc;
      if (!any || l[t] > mx) mx = l[t];
      any = 1;
    }
    double Z = 0.0;
    for (int t = 0; t < M; ++t) {
      const int vis = t < mc || t <= Pk;
      l[t] = vis ? exp(l[t] - mx) : 0.0;
      Z += l[t];
    }
    for (int x = 0; x < d; ++x) {
      double acc = 0.0;
      for (int t = 0; t < M; ++t) {
        if (l[t] == 0.0) continue;
        const double vv = t < mc ? widen(Vc, ((size_t)c * mc + t) * d + x, dtype)
                                 : widen(Vd, (((size_t)i * g + c) * md_cap + (t - mc)) * d + x, dtype);
        acc += l[t] * vv;
      }
      out[(size_t)r * d + x] = acc / Z;
    }
    if (lse) lse[r] = mx + log(Z);
    if (weights)
      for (int t = 0; t < Mcap; ++t) weights[(size_t)r * Mcap + t] = t < M ? l[t] / Z : 0.0;
    free(l);
  }
  return err ? -1 : 0;
}

/*
 * FP8 (E4M3) KV cache (FAQ 5: "the lower
 * memory on the attention tensor will effectively reduce the memory I/O for
 * KV cache by a factor of 2 in the case of int8 quantization"; reading R19):
 * Kc, Vc, Kd, Vd hold OCP FP8 E4M3 codes (1 sign, 4 exponent bits with bias 7,
 * 3 mantissa bits; no infinities; S.1111.111 is NaN) with one fp32 scale per
 * tensor kind shared by the context and decode caches: the cache value is
 *   K = e4m3(code) * k_scale,   V = e4m3(code) * v_scale.
 * q is bf16 or fp32 (q_dtype).  The attention is Eq. 1-2 over the replicated
 * cache exactly as oracle_attn_decode_f64, on those dequantised values
 * (widened exactly: a 4-bit significand times a 24-bit one fits in fp64), so
 * the quantisation is input, not error.
 */
static double e4m3_value(uint8_t code) {
  const int s = code >> 7, e = (code >> 3) & 15, m = code & 7;
  double v;
  if (e == 15 && m == 7) return NAN;
  if (e == 0)
    v = ldexp((double)m, -9); /* subnormal: (m / 8) * 2^-6 */
  else
    v = ldexp(1.0 + (double)m / 8.0, e - 7);
  return s ? -v : v;
}

/* The value of E4M3 code `code` (exported for the pins: the decode table). */
double oracle_e4m3_value(int code) { return e4m3_value((uint8_t)(code & 255)); }

int oracle_attn_decode_kv8_f64(int b, int h, int g, int d, int mc, int md_cap, int q_dtype,
                               double scale, double k_scale, double v_scale, const void *q,
                               const uint8_t *Kc, const uint8_t *Vc, const uint8_t *Kd,
                               const uint8_t *Vd, const int32_t *lens, const int32_t *rows,
                               int nrows, double *out, double *lse, double *weights,
                               int nthreads) {
  if (check(b, h, g, d, mc, md_cap, q_dtype)) return -1;
  if (!rows) nrows = b * h;
  const int p = h / g;
  const int Mcap = mc + md_cap;
  int err = 0;
  (void)nthreads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
  for (int r = 0; r < nrows; ++r) {
    const int row = rows ? rows[r] : r;
    const int i = row / h, j = row % h, c = j / p;
    const int M = mc + dec_len(lens, i, md_cap);
    double *Kf = (double *)malloc(sizeof(double) * (size_t)(M > 0 ? M : 1) * d);
    double *Vf = (double *)malloc(sizeof(double) * (size_t)(M > 0 ? M : 1) * d);
    double *l = (double *)malloc(sizeof(double) * (size_t)(M > 0 ? M : 1));
    if (!Kf || !Vf || !l || M < 1) {
      free(Kf); free(Vf); free(l);
#pragma omp atomic write
      err = 1;
      continue;
    }
    /* Step 1: this sample's full cache Kc ⊕ Kd[i] for group c, dequantised. */
    for (int t = 0; t < M; ++t) {
      for (int x = 0; x < d; ++x) {
        size_t src;
        if (t < mc) {
          src = ((size_t)c * mc + t) * d + x;
          Kf[(size_t)t * d + x] = e4m3_value(Kc[src]) * k_scale;
          Vf[(size_t)t * d + x] = e4m3_value(Vc[src]) * v_scale;
        } else {
          src = (((size_t)i * g + c) * md_cap + (t - mc)) * d + x;
          Kf[(size_t)t * d + x] = e4m3_value(Kd[src]) * k_scale;
          Vf[(size_t)t * d + x] = e4m3_value(Vd[src]) * v_scale;
        }
      }
    }
    /* Step 2: logits (Eq. 1). */
    for (int t = 0; t < M; ++t) {
      double acc = 0.0;
      for (int x = 0; x < d; ++x)
        acc += widen(q, ((size_t)i * h + j) * d + x, q_dtype) * Kf[(size_t)t * d + x];
      l[t] = scale * acc;
    }
    /* Step 3: one softmax over all M positions. */
    double mx = l[0];
    for (int t = 1; t < M; ++t)
      if (l[t] > mx) mx = l[t];
    double Z = 0.0;
    for (int t = 0; t < M; ++t) {
      l[t] = exp(l[t] - mx);
      Z += l[t];
    }
    /* Step 4: out = (sum_t w_t V_t) / Z (Eq. 2). */
    for (int x = 0; x < d; ++x) {
      double acc = 0.0;
      for (int t = 0; t < M; ++t) acc += l[t] * Vf[(size_t)t * d + x];
      out[(size_t)r * d + x] = acc / Z;
    }
    if (lse) lse[r] = mx + log(Z);
    if (weights)
      for (int t = 0; t < Mcap; ++t) weights[(size_t)r * Mcap + t] = t < M ? l[t] / Z : 0.0;
    free(Kf); free(Vf); free(l);
  }
  return err ? -1 : 0;
}

/*
 * KV-read element counts of Eq. 5-6 (§4.3), per K or V
 * tensor, per layer:  naive  g*k*b*(mc+md);  bifurcated  g*k*(mc+b*md).
 */
int64_t oracle_kv_read_elements(int64_t b, int64_t g, int64_t k, int64_t mc, int64_t md,
                                int bifurcated) {
  return bifurcated ? g * k * (mc + b * md) : g * k * b * (mc + md);
}
