/*
 * LouisKV CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * This file is the plain, slow, obviously-correct reference for every step of
 * the LouisKV retrieval hot path (arXiv 2510.11292). Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * leg may load it. The product library (paper_2510_11292_b200/) shares no code,
 * header, table or constant with this file and never calls it.
 *
 * Citation format: P:n = /root/reference/PAPER.md line n (section in brackets),
 * S:n = SPEC.md line n. Readings of silent/ambiguous passages are DESIGN.md
 * §Readings R-* (they follow SURVEY.md §8(c) AMB-*).
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (no SIMD
 * intrinsics, no FMA contraction: every fused multiply-add below is an
 * explicit fmaf() call that the recipe prescribes).
 *
 * Precision: fp64 wherever the paper fixes no precision; the bit-exact
 * "recipes" R1 (trigger, fp64) and R2/R3 (group scores, fp32) are written out
 * operation by operation so the GPU can reproduce them bit for bit.
 *
 * Parity status per function (pins live in tests/test_oracle_*.py):
 *   lko_cosine_r1 / lko_trigger_r1      pinned (symmetry)
 *   lko_exp_r3                          pinned (vs libm exp, relative 2e-7)
 *   lko_group_scores_r2 / _f64          pinned (S:339-342 closed forms, sum=1, g=1 argsort)
 *   lko_select_greedy                   pinned (brute force on <=12 units)
 *   lko_kmeans                          pinned (Lloyd monotone, partition, fixed point,
 *                                        planted recovery, sklearn Lloyd equality)
 *   lko_segment_centroid                pinned (S:152-154 closed form)
 *   lko_attention_f64                   pinned (S:402-414 closed forms, SDPA)
 *   lko_e4m3_round                      pinned (every finite bf16 value vs torch's float8_e4m3fn
 *                                        cast, hand-worked ties / subnormals / saturation)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* bf16 round-to-nearest-even (reading R-AMB18: all fp32->bf16 are RNE).      */
/* ------------------------------------------------------------------------ */
float lko_bf16_round(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) { /* inf / nan: truncate, keep nan quiet */
    if (u & 0x007FFFFFu) u |= 0x00400000u;
    u &= 0xFFFF0000u;
  } else {
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    u &= 0xFFFF0000u;
  }
  float y;
  memcpy(&y, &u, 4);
  return y;
}

/* ------------------------------------------------------------------------ */
/* R1: cosine similarity and the semantic-boundary trigger.                   */
/* P:101-106 [§4.1 eq. r_t = (1/H) Σ_h cosine(q_{t-1}^h, q_t^h)],             */
/* P:301 [Alg. 1: is_new_segment = (t==1) ∨ (CosineSimilarity < r)].          */
/* Recipe (fp64, fixed order, R1): the d elements are cut into 16   */
/* contiguous chunks of ceil(d/16); each chunk is summed sequentially         */
/* (multiply then add, no fma) for dot, ||a||², ||b||²; the 16 partial sums   */
/* are combined by a balanced pairwise tree s[l] += s[l+8], +4, +2, +1.        */
/* cos = dot / (sqrt(na)*sqrt(nb)), clamped to [-1,1]; zero norm -> 0. */
/* ------------------------------------------------------------------------ */
static double r1_tree16(double* s) {
  for (int off = 8; off >= 1; off >>= 1)
    for (int l = 0; l < off; ++l) s[l] = s[l] + s[l + off];
  return s[0];
}

double lko_cosine_r1(const float* a, const float* b, int d) {
  double pd[16], pa[16], pb[16];
  const int chunk = (d + 15) / 16;
  for (int l = 0; l < 16; ++l) {
    double dot = 0.0, na = 0.0, nb = 0.0;
    for (int e = l * chunk; e < (l + 1) * chunk && e < d; ++e) {
      double x = (double)a[e], y = (double)b[e];
      dot = dot + x * y;
      na = na + x * x;
      nb = nb + y * y;
    }
    pd[l] = dot;
    pa[l] = na;
    pb[l] = nb;
  }
  double dot = r1_tree16(pd), na = r1_tree16(pa), nb = r1_tree16(pb);
  if (na == 0.0 || nb == 0.0) return 0.0;
  double c = dot / (sqrt(na) * sqrt(nb));
  if (c > 1.0) c = 1.0;
  if (c < -1.0) c = -1.0;
  return c;
}

/* q_ref, q_cur: [H][d]. Returns flag; *r_out = r_t (fp64).  t is 1-based.   */
int lko_trigger_r1(const float* q_ref, const float* q_cur, int H, int d, int t,
                   double tau, double* r_out) {
  double s = 0.0;
  for (int h = 0; h < H; ++h) s = s + lko_cosine_r1(q_ref + (size_t)h * d, q_cur + (size_t)h * d, d);
  double r = s / (double)H;
  if (r_out) *r_out = r;
  if (t == 1) return 1;
  return r < tau ? 1 : 0;
}

/* ------------------------------------------------------------------------ */
/* R3: portable fp32 exp for x <= 0.                                          */
/* t = x*log2(e); n = rint(t); f = t - n; 2^f by degree-6 Horner in fmaf with */
/* Taylor coefficients c_i = ln2^i / i! (ln2^i by repeated fp64 products,     */
/* divided by i! in fp64, rounded to fp32); scale by 2^n via exponent bits;   */
/* t < -126 -> 0.                                                             */
/* ------------------------------------------------------------------------ */
static float r3_coef[7];
static int r3_init_done = 0;
static void r3_init(void) {
  const double ln2 = 0.6931471805599453094;
  double p = 1.0, fact = 1.0;
  for (int i = 0; i <= 6; ++i) {
    if (i > 0) { p = p * ln2; fact = fact * (double)i; }
    r3_coef[i] = (float)(p / fact);
  }
  r3_init_done = 1;
}

float lko_exp_r3(float x) {
  if (!r3_init_done) r3_init();
  const float log2e = (float)1.4426950408889634074;
  float t = x * log2e;
  if (t < -126.0f) return 0.0f;
  float n = rintf(t);
  float f = t - n;
  float p = r3_coef[6];
  for (int i = 5; i >= 0; --i) p = fmaf(p, f, r3_coef[i]);
  int ni = (int)n;
  uint32_t bits = (uint32_t)(ni + 127) << 23;
  float scale;
  memcpy(&scale, &bits, 4);
  return p * scale;
}

/* ------------------------------------------------------------------------ */
/* R2: group-consistent scores (P:243-247 [App. B eq. A_t^i]).                */
/*   l_{j,u} = fl32(fmaf-chain_e(q_{j,e}, c_{u,e})) * fl32(1/sqrt(d))         */
/*   m_j = max_u l_{j,u};  e_{j,u} = exp_R3(l_{j,u} - m_j)                    */
/*   Z_j = fl32(Σ_u floor(e_{j,u} 2^40)) * 2^-40   (exact integer sum)         */
/*   A_u = (Σ_{j ascending} e_{j,u} / Z_j) / g                                */
/* q: [g][d] fp32 (bf16 values); C: [n][d] fp32 (bf16 values). A: [n].        */
/* Softmax axis = units of this KV head, per query head (reading R-AMB5).     */
/* ------------------------------------------------------------------------ */
int lko_group_scores_r2(const float* q, int g, const float* C, int n, int d, float* A) {
  if (n <= 0 || g <= 0) return -1;
  const float inv_sqrt_d = (float)(1.0 / sqrt((double)d));
  float* l = (float*)malloc(sizeof(float) * (size_t)n);
  float* ev = (float*)malloc(sizeof(float) * (size_t)n);
  if (!l || !ev) { free(l); free(ev); return -2; }
  for (int u = 0; u < n; ++u) A[u] = 0.0f;
  for (int j = 0; j < g; ++j) {
    const float* qj = q + (size_t)j * d;
    float m = -INFINITY;
    for (int u = 0; u < n; ++u) {
      const float* cu = C + (size_t)u * d;
      float acc = 0.0f;
      for (int e = 0; e < d; ++e) acc = fmaf(qj[e], cu[e], acc);
      l[u] = acc * inv_sqrt_d;
      if (l[u] > m) m = l[u];
    }
    uint64_t zfix = 0;
    for (int u = 0; u < n; ++u) {
      ev[u] = lko_exp_r3(l[u] - m);
      zfix += (uint64_t)(ev[u] * 1099511627776.0f); /* 2^40, truncation */
    }
    float Z = (float)zfix * 9.094947017729282379e-13f; /* 2^-40 */
    for (int u = 0; u < n; ++u) A[u] = A[u] + ev[u] / Z;
  }
  for (int u = 0; u < n; ++u) A[u] = A[u] / (float)g;
  free(l);
  free(ev);
  return 0;
}

/* Textbook fp64 definition of A (for the definition pin, not for parity).   */
int lko_group_scores_f64(const float* q, int g, const float* C, int n, int d, double* A) {
  if (n <= 0 || g <= 0) return -1;
  double* l = (double*)malloc(sizeof(double) * (size_t)n);
  if (!l) return -2;
  for (int u = 0; u < n; ++u) A[u] = 0.0;
  for (int j = 0; j < g; ++j) {
    double m = -INFINITY;
    for (int u = 0; u < n; ++u) {
      double s = 0.0;
      for (int e = 0; e < d; ++e) s += (double)q[(size_t)j * d + e] * (double)C[(size_t)u * d + e];
      l[u] = s / sqrt((double)d);
      if (l[u] > m) m = l[u];
    }
    double Z = 0.0;
    for (int u = 0; u < n; ++u) Z += exp(l[u] - m);
    for (int u = 0; u < n; ++u) A[u] += exp(l[u] - m) / Z;
  }
  for (int u = 0; u < n; ++u) A[u] /= (double)g;
  free(l);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Budgeted selection (P:126, P:281 [Alg. 1 Retrieve]).            */
/* Order units by (A desc, id asc); greedy skip-and-continue: take u iff       */
/* size_u <= remaining budget. Output ids in ASCENDING id order.               */
/* Plain O(n^2) selection sort of the order — slow and obvious.               */
/* ------------------------------------------------------------------------ */
int lko_select_greedy(const float* A, const int* sizes, int n, long long B, int* out_ids) {
  char* used = (char*)calloc((size_t)(n > 0 ? n : 1), 1);
  char* taken = (char*)calloc((size_t)(n > 0 ? n : 1), 1);
  if (!used || !taken) { free(used); free(taken); return -1; }
  long long rem = B;
  for (int it = 0; it < n; ++it) {
    int best = -1;
    for (int u = 0; u < n; ++u) {
      if (used[u]) continue;
      if (best < 0 || A[u] > A[best]) best = u; /* strict > keeps the lower id on ties */
    }
    used[best] = 1;
    if ((long long)sizes[best] <= rem) {
      taken[best] = 1;
      rem -= sizes[best];
    }
  }
  int cnt = 0;
  for (int u = 0; u < n; ++u)
    if (taken[u]) out_ids[cnt++] = u;
  free(used);
  free(taken);
  return cnt;
}

/* ------------------------------------------------------------------------ */
/* k-means of prompt keys (P:120 [§4.2 Prefill], P:260-263 [Alg. 1]).          */
/* X: [N][d] fp32 (bf16 values). k clusters, iters Lloyd iterations.           */
/* Init: C0_j = x_{floor(j*N/k)}  (reading R-AMB8).                            */
/* Each iteration: (i) assign argmin_j dist(x_i, c_j), ties -> lower j;        */
/*   mode 0 (exact):  dist = Σ_e (x_e - c_e)^2 in fp64;                        */
/*   mode 1 (bf16 operand, mirrors the GPU's declared precision, R-AMB10):     */
/*          dist = ||x||^2 - 2 x·bf16(c) + ||c||^2 (fp64, ||c|| of fp32 c).    */
/* (ii) repair empty clusters (R-AMB9): E = empty ids ascending; for each      */
/*   E[r] in order pick the point with the largest max(dmin, 0) (ties -> lower */
/*   index)                                                                    */
/*   among points whose cluster has >= 2 members at pick time and that were   */
/*   not picked before; move it to E[r].                                       */
/* (iii) c_j = mean of members in fp64, stored fp32.                           */
/* (iv) J_it = Σ_i ||x_i - c_{a_i}||^2 (fp64, new centroids).                  */
/* Outputs: assign[N], C[k][d], counts[k], J[iters], dmin[N] (last assign).    */
/* ------------------------------------------------------------------------ */
static double sqdist_exact(const float* x, const float* c, int d) {
  double s = 0.0;
  for (int e = 0; e < d; ++e) {
    double t = (double)x[e] - (double)c[e];
    s += t * t;
  }
  return s;
}

int lko_kmeans(const float* X, int N, int d, int k, int iters, int mode, int* assign,
               float* C, int* counts, double* J, float* dmin_out) {
  if (N <= 0 || k <= 0 || k > N || d <= 0) return -1;
  double* dmin = (double*)malloc(sizeof(double) * (size_t)N);
  double* xnorm = (double*)malloc(sizeof(double) * (size_t)N);
  double* cnorm = (double*)malloc(sizeof(double) * (size_t)k);
  float* cb = (float*)malloc(sizeof(float) * (size_t)k * d);
  double* sum = (double*)malloc(sizeof(double) * (size_t)k * d);
  char* picked = (char*)malloc((size_t)N);
  if (!dmin || !xnorm || !cnorm || !cb || !sum || !picked) return -2;

  for (int j = 0; j < k; ++j) {
    long long src = ((long long)j * N) / k;
    memcpy(C + (size_t)j * d, X + (size_t)src * d, sizeof(float) * d);
  }
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
    for (int e = 0; e < d; ++e) s += (double)X[(size_t)i * d + e] * (double)X[(size_t)i * d + e];
    xnorm[i] = s;
  }

  for (int it = 0; it < iters; ++it) {
    /* (i) assignment */
    if (mode == 1) {
      for (int j = 0; j < k; ++j) {
        double s = 0.0;
        for (int e = 0; e < d; ++e) {
          float c = C[(size_t)j * d + e];
          s += (double)c * (double)c;
          cb[(size_t)j * d + e] = lko_bf16_round(c);
        }
        cnorm[j] = s;
      }
    }
    for (int i = 0; i < N; ++i) {
      const float* x = X + (size_t)i * d;
      int best = 0;
      double bd = INFINITY;
      for (int j = 0; j < k; ++j) {
        double dist;
        if (mode == 1) {
          double dot = 0.0;
          for (int e = 0; e < d; ++e) dot += (double)x[e] * (double)cb[(size_t)j * d + e];
          dist = xnorm[i] - 2.0 * dot + cnorm[j];
        } else {
          dist = sqdist_exact(x, C + (size_t)j * d, d);
        }
        if (dist < bd) { bd = dist; best = j; }
      }
      assign[i] = best;
      dmin[i] = bd;
    }
    /* (ii) repair */
    for (int j = 0; j < k; ++j) counts[j] = 0;
    for (int i = 0; i < N; ++i) counts[assign[i]]++;
    memset(picked, 0, (size_t)N);
    for (int j = 0; j < k; ++j) {
      if (counts[j] != 0) continue;
      int donor = -1;
      for (int i = 0; i < N; ++i) {
        if (picked[i] || counts[assign[i]] < 2) continue;
        /* donor key = max(dmin, 0): a squared distance is >= 0; a negative mode-1 value is a
           rounding artefact of the expanded form (reading R-AMB9) */
        if (donor < 0 || fmax(dmin[i], 0.0) > fmax(dmin[donor], 0.0)) donor = i;
      }
      if (donor < 0) break; /* cannot happen for k <= N */
      counts[assign[donor]]--;
      assign[donor] = j;
      counts[j] = 1;
      picked[donor] = 1;
      dmin[donor] = 0.0;
    }
    /* (iii) update */
    memset(sum, 0, sizeof(double) * (size_t)k * d);
    for (int i = 0; i < N; ++i)
      for (int e = 0; e < d; ++e) sum[(size_t)assign[i] * d + e] += (double)X[(size_t)i * d + e];
    for (int j = 0; j < k; ++j)
      for (int e = 0; e < d; ++e) C[(size_t)j * d + e] = (float)(sum[(size_t)j * d + e] / (double)counts[j]);
    /* (iv) objective */
    double Jit = 0.0;
    for (int i = 0; i < N; ++i) Jit += sqdist_exact(X + (size_t)i * d, C + (size_t)assign[i] * d, d);
    if (J) J[it] = Jit;
  }
  if (dmin_out)
    for (int i = 0; i < N; ++i) dmin_out[i] = (float)dmin[i];
  free(dmin); free(xnorm); free(cnorm); free(cb); free(sum); free(picked);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Segment centroid (P:123 [§4.2 Decode: "index vector derived from averaging */
/* its key vectors"], P:270 [Alg. 1]). fp32 sequential sum in time order then */
/* division by len (fp32 RN) — reading R-SEG (bit-exact replicable).          */
/* ------------------------------------------------------------------------ */
void lko_segment_centroid(const float* keys, int len, int d, float* out) {
  for (int e = 0; e < d; ++e) {
    float s = 0.0f;
    for (int i = 0; i < len; ++i) s = s + keys[(size_t)i * d + e];
    out[e] = s / (float)len;
  }
}

/* ------------------------------------------------------------------------ */
/* Attention o = softmax(q K^T / sqrt(d)) V, fp64 (P:63-65 [§3.1 eq.]).        */
/* q: [g][d]; K, V: [n][d]; out: [g][d] fp64.                                  */
/* ------------------------------------------------------------------------ */
int lko_attention_f64(const float* q, int g, const float* K, const float* V, int n, int d,
                      double* out) {
  if (n <= 0) return -1;
  double* s = (double*)malloc(sizeof(double) * (size_t)n);
  if (!s) return -2;
  for (int j = 0; j < g; ++j) {
    double m = -INFINITY;
    for (int r = 0; r < n; ++r) {
      double dot = 0.0;
      for (int e = 0; e < d; ++e) dot += (double)q[(size_t)j * d + e] * (double)K[(size_t)r * d + e];
      s[r] = dot / sqrt((double)d);
      if (s[r] > m) m = s[r];
    }
    double Z = 0.0;
    for (int r = 0; r < n; ++r) { s[r] = exp(s[r] - m); Z += s[r]; }
    for (int e = 0; e < d; ++e) {
      double acc = 0.0;
      for (int r = 0; r < n; ++r) acc += s[r] * (double)V[(size_t)r * d + e];
      out[(size_t)j * d + e] = acc / Z;
    }
  }
  free(s);
  return 0;
}

/* Array helpers (plain loops over the scalar definitions above). */
void lko_bf16_round_n(const float* x, float* y, long long n) {
  for (long long i = 0; i < n; ++i) y[i] = lko_bf16_round(x[i]);
}
void lko_exp_r3_n(const float* x, float* y, long long n) {
  for (long long i = 0; i < n; ++i) y[i] = lko_exp_r3(x[i]);
}

/* Centroids of a given clustering: C_j = mean of {x_i : a_i = j} in fp64, stored fp32
 * ("calculates the centroid C_i for each cluster by averaging all its key vectors";
 * the same update step as lko_kmeans (iii)). Returns -1 if a cluster is empty. */
int lko_centroids_of(const float* X, const int* assign, int N, int d, int k, float* C) {
  double* sum = (double*)calloc((size_t)k * d, sizeof(double));
  int* cnt = (int*)calloc((size_t)k, sizeof(int));
  if (!sum || !cnt) { free(sum); free(cnt); return -2; }
  for (int i = 0; i < N; ++i) {
    cnt[assign[i]]++;
    for (int e = 0; e < d; ++e) sum[(size_t)assign[i] * d + e] += (double)X[(size_t)i * d + e];
  }
  int rc = 0;
  for (int j = 0; j < k; ++j) {
    if (cnt[j] == 0) { rc = -1; continue; }
    for (int e = 0; e < d; ++e) C[(size_t)j * d + e] = (float)(sum[(size_t)j * d + e] / (double)cnt[j]);
  }
  free(sum); free(cnt);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* FP8 (E4M3) host pool — SURVEY §8(f) row 3 ("FP8 KV in the pool halves the  */
/* link bytes"); the paper keeps its pool in FP16 ("All KV cache is     */
/* stored in FP16"), so this is a variant, reading R-FP8: a pool  */
/* row holds e4m3(x) of every bf16 element x, round-to-nearest-even, values  */
/* beyond the largest finite E4M3 magnitude (448) saturate to +-448.          */
/* E4M3: 1 sign, 4 exponent bits (bias 7), 3 mantissa bits, no infinities;    */
/* normal magnitudes 2^-6 .. 448, subnormals m * 2^-9 (m = 1..7).             */
/* Written out from that definition: the quantum of |x| is 2^(e-3) for the    */
/* binade [2^e, 2^(e+1)) with e >= -6, else the subnormal quantum 2^-9;       */
/* x / quantum is exact in fp64, rint() rounds it half-to-even.               */
/* ------------------------------------------------------------------------ */
float lko_e4m3_round(float x) {
  if (x != x) return x;
  const double ax = fabs((double)x);
  if (ax == 0.0) return x;
  double y;
  if (ax >= 448.0) {
    y = 448.0;
  } else {
    int e;
    (void)frexp(ax, &e); /* ax = f * 2^e, f in [0.5, 1): binade [2^(e-1), 2^e) */
    int eb = e - 1;      /* ax in [2^eb, 2^(eb+1)) */
    if (eb < -6) eb = -6; /* subnormal range shares the quantum of the first normal binade */
    const double q = ldexp(1.0, eb - 3);
    y = rint(ax / q) * q; /* (a tie at the top of a binade rounds up into the next: still exact) */
    if (y > 448.0) y = 448.0;
  }
  return (float)(x < 0 ? -y : y);
}
void lko_e4m3_round_n(const float* x, float* y, long long n) {
  for (long long i = 0; i < n; ++i) y[i] = lko_e4m3_round(x[i]);
}
