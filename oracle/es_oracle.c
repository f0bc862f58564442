/*
 * es_oracle.c — CPU ORACLE (test infrastructure only; see es_oracle.h).
 *
 * Plain C99, one run at a time, sequential loops, every step written in the order of
 * NUMERICS.md (which cites PAPER.md). Built with -O2 -ffp-contract=off -fno-fast-math so that
 * every binary32 operation below is exactly one IEEE operation.
 *
 * Parity status per function (see DESIGN.md §Oracle pins):
 *   philox / uniforms / LN / SINCOS2PI / normals  — pinned (KAT, exhaustive vs libm, moments)
 *   init / ask                                      — pinned (antithetic closed forms, σ→0)
 *   eval (sphere/rosenbrock/rastrigin)               — pinned (S:655–657 hand values, optima)
 *   rank / centered rank / weights                   — pinned (brute force, Σ, ratios)
 *   reduce / tell (4 algorithms)                     — pinned (FD expectation on linear f,
 *                                                      S:290 quadratic, S:307–309, S:371–372,
 *                                                      S:438 zero-path, hand Adam recursion)
 */
#include "es_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* ---------------- N1 Philox4x32-10 (Salmon et al. 2011) ---------------- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ---------------- N3 uniforms ---------------- */
float orc_u_a(uint32_t o) { return 2.0f - u2f(0x3F800000u | (o >> 9)); }
float orc_u_b(uint32_t o) { return u2f(0x3F800000u | (o >> 9)) - 1.0f; }

/* ---------------- N4 LN ---------------- */
static const float LN2_HI = 0x1.62e400p-1f, LN2_LO = 0x1.7f7d1cp-20f, SQRT2_F = 0x1.6a09e6p+0f;
static const float L0 = -0x1.fffffap-2f, L1 = 0x1.5556f4p-2f, L2 = -0x1.00049ap-2f,
                   L3 = 0x1.98d2c0p-3f, L4 = -0x1.535d30p-3f, L5 = 0x1.318528p-3f,
                   L6 = -0x1.25049cp-3f, L7 = 0x1.65c768p-4f;

float orc_ln(float u) {
  uint32_t b = f2u(u);
  float E = (float)((int32_t)(b >> 23) - 127);
  float m = u2f((b & 0x007FFFFFu) | 0x3F800000u);
  if (m > SQRT2_F) {
    m = m * 0.5f;
    E = E + 1.0f;
  }
  float r = m - 1.0f;
  float Q = L7;
  Q = fmaf(Q, r, L6);
  Q = fmaf(Q, r, L5);
  Q = fmaf(Q, r, L4);
  Q = fmaf(Q, r, L3);
  Q = fmaf(Q, r, L2);
  Q = fmaf(Q, r, L1);
  Q = fmaf(Q, r, L0);
  float r2 = r * r;
  float p = fmaf(Q, r2, r);
  return fmaf(E, LN2_HI, fmaf(E, LN2_LO, p));
}

/* ---------------- N5 SINCOS2PI ---------------- */
static const float S0 = 0x1.921fb6p+0f, S1 = -0x1.4abbbap-1f, S2 = 0x1.465e92p-4f,
                   S3 = -0x1.2d930ep-8f;
static const float C1 = -0x1.3bd3ccp+0f, C2 = 0x1.03c1dep-2f, C3 = -0x1.55c5e0p-6f,
                   C4 = 0x1.d9d584p-11f;

void orc_sincos2pi(float u, float *c, float *s) {
  float t4 = 4.0f * u;
  float k = rintf(t4);
  float r = t4 - k;
  int q = ((int)k) & 3;
  float ss = r * r;
  float S = fmaf(fmaf(fmaf(S3, ss, S2), ss, S1), ss, S0);
  float sp = r * S;
  float C = fmaf(fmaf(fmaf(fmaf(C4, ss, C3), ss, C2), ss, C1), ss, 1.0f);
  switch (q) {
    case 0: *c = C; *s = sp; break;
    case 1: *c = -sp; *s = C; break;
    case 2: *c = -C; *s = -sp; break;
    default: *c = sp; *s = -C; break;
  }
}

/* ---------------- N2 normals ---------------- */
void orc_normals4(uint64_t seed, uint32_t q, uint32_t i, uint32_t t, uint32_t tag, float out[4]) {
  uint32_t ctr[4] = {q, i, t, tag};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t o[4];
  orc_philox4x32_10(ctr, key, o);
  float c, s;
  float rho0 = sqrtf(-2.0f * orc_ln(orc_u_a(o[0])));
  orc_sincos2pi(orc_u_b(o[1]), &c, &s);
  out[0] = rho0 * c;
  out[1] = rho0 * s;
  float rho2 = sqrtf(-2.0f * orc_ln(orc_u_a(o[2])));
  orc_sincos2pi(orc_u_b(o[3]), &c, &s);
  out[2] = rho2 * c;
  out[3] = rho2 * s;
}

void orc_direction(uint64_t seed, uint32_t i, uint32_t t, int64_t D, float *z) {
  float n[4];
  for (int64_t q = 0; 4 * q < D; ++q) {
    orc_normals4(seed, (uint32_t)q, i, t, 0u, n);
    for (int k = 0; k < 4 && 4 * q + k < D; ++k) z[4 * q + k] = n[k];
  }
}

/* z of direction i at generation t for the run's dimensions (global indices when r->dims). */
static void run_direction(const orc_run_t *r, uint32_t i, uint32_t t, float *z) {
  if (!r->dims) {
    orc_direction(r->p.seed, i, t, r->num_dims, z);
    return;
  }
  float n[4];
  int64_t cur = -1;
  for (int64_t d = 0; d < r->num_dims; ++d) {
    int64_t g = r->dims[d];
    if (g / 4 != cur) {
      cur = g / 4;
      orc_normals4(r->p.seed, (uint32_t)cur, i, t, 0u, n);
    }
    z[d] = n[g % 4];
  }
}

static int64_t gdim(const orc_run_t *r, int64_t d) { return r->dims ? r->dims[d] : d; }

/* ---------------- N6 init / ask ---------------- */
static int is_antithetic(int algo) {
  return algo == ORC_OPENAI_ES || algo == ORC_PGPE || algo == ORC_ARS;
}

int orc_num_directions(const orc_run_t *r) {
  return is_antithetic(r->algo) ? r->popsize / 2 : r->popsize;
}

static float *vf(const orc_run_t *r, int field) { return r->vec + (int64_t)field * r->num_dims; }

int orc_init(orc_run_t *r) {
  const int64_t D = r->num_dims;
  const int32_t N = r->popsize;
  if (N < 2 || D < 1) return 1;
  if (is_antithetic(r->algo) && (N % 2) != 0) return 1;
  if (r->algo < 0 || r->algo > 4) return 1;
  const orc_params_t *p = &r->p;
  uint32_t key[2] = {(uint32_t)p->seed, (uint32_t)(p->seed >> 32)};
  float *mean = vf(r, ORC_V_MEAN);
  for (int64_t d = 0; d < D; ++d) {
    int64_t g = gdim(r, d);
    uint32_t ctr[4] = {(uint32_t)(g / 4), 0u, 0u, 1u}, o[4];
    orc_philox4x32_10(ctr, key, o);
    mean[d] = fmaf(p->init_max - p->init_min, orc_u_b(o[g % 4]), p->init_min);
  }
  for (int64_t d = 0; d < D; ++d) {
    vf(r, ORC_V_SIGMA)[d] = p->sigma_init;
    vf(r, ORC_V_ADAM_M)[d] = 0.0f;
    vf(r, ORC_V_ADAM_V)[d] = 0.0f;
    vf(r, ORC_V_PSIGMA)[d] = 0.0f;
    vf(r, ORC_V_PC)[d] = 0.0f;
    vf(r, ORC_V_C)[d] = 1.0f;
    vf(r, ORC_V_BEST_X)[d] = mean[d];
  }
  r->t = 0;
  r->lr = p->lrate_init;
  r->sigma = p->sigma_init;
  r->b1pow = 1.0;
  r->b2pow = 1.0;
  r->best_f = INFINITY;
  r->mu = 0;
  r->mueff = r->c_sigma = r->d_sigma = r->c_c = r->c_1 = r->c_mu = r->chi_d = 0.0;
  r->eta_sigma = 0.0;
  if (!r->dims) r->full_dims = D;
  double Dd = (double)r->full_dims;
  if (r->algo == ORC_SNES) {
    /* N11 SNES utilities: w = softmax(beta * (rank/N - 0.5)), rank(best) = N-1 */
    double *u = (double *)malloc(sizeof(double) * (size_t)N);
    double z = 0.0;
    for (int32_t q = 0; q < N; ++q) u[q] = (double)p->temperature * ((double)(N - 1 - q) / N - 0.5);
    for (int32_t q = 0; q < N; ++q) z += exp(u[q] - u[0]);
    for (int32_t q = 0; q < N; ++q) r->wpos[q] = (float)(exp(u[q] - u[0]) / z);
    free(u);
    r->eta_sigma = (3.0 + log(Dd)) / (5.0 * sqrt(Dd));
  } else if (r->algo == ORC_SEP_CMA_ES) {
    int32_t mu = (int32_t)floor((double)p->elite_ratio * (double)N);
    if (mu < 1) return 1;
    double *w = (double *)malloc(sizeof(double) * (size_t)N);
    double sum = 0.0, sum2 = 0.0;
    for (int32_t q = 0; q < N; ++q) {
      w[q] = q < mu ? log((N + 1) / 2.0) - log((double)(q + 1)) : 0.0;
      sum += w[q];
    }
    for (int32_t q = 0; q < N; ++q) {
      w[q] /= sum;
      sum2 += w[q] * w[q];
      r->wpos[q] = (float)w[q];
    }
    free(w);
    double mueff = 1.0 / sum2;
    r->mu = mu;
    r->mueff = mueff;
    r->c_sigma = (mueff + 2.0) / (Dd + mueff + 5.0);
    double t0 = sqrt((mueff - 1.0) / (Dd + 1.0)) - 1.0;
    r->d_sigma = 1.0 + 2.0 * (t0 > 0.0 ? t0 : 0.0) + r->c_sigma;
    r->c_c = (4.0 + mueff / Dd) / (Dd + 4.0 + 2.0 * mueff / Dd);
    double c1 = 2.0 / ((Dd + 1.3) * (Dd + 1.3) + mueff);
    double cmu = 2.0 * (mueff - 2.0 + 1.0 / mueff) / ((Dd + 2.0) * (Dd + 2.0) + mueff);
    if (cmu > 1.0 - c1) cmu = 1.0 - c1;
    r->c_1 = c1 * (Dd + 2.0) / 3.0;   /* Ros & Hansen (2008) separable learning-rate boost */
    r->c_mu = cmu * (Dd + 2.0) / 3.0;
    r->chi_d = sqrt(Dd) * (1.0 - 1.0 / (4.0 * Dd) + 1.0 / (21.0 * Dd * Dd));
  }
  return 0;
}

/* x of member j under the current state (N6). */
void orc_member(const orc_run_t *r, int32_t j, float *x) {
  const int64_t D = r->num_dims;
  const float *mean = vf(r, ORC_V_MEAN);
  const float *sd = vf(r, ORC_V_SIGMA);
  const float *Cd = vf(r, ORC_V_C);
  int anti = is_antithetic(r->algo);
  uint32_t i = anti ? (uint32_t)(j / 2) : (uint32_t)j;
  int neg = anti && (j % 2 == 1);
  float *z = (float *)malloc(sizeof(float) * (size_t)D);
  run_direction(r, i, r->t, z);
  for (int64_t d = 0; d < D; ++d) {
    float s;
    switch (r->algo) {
      case ORC_OPENAI_ES: s = r->sigma; break;
      case ORC_ARS: s = r->sigma; break;
      case ORC_PGPE: s = sd[d]; break;
      case ORC_SNES: s = sd[d]; break;
      default: s = r->sigma * sqrtf(Cd[d]); break;
    }
    if (neg) s = -s;
    x[d] = fmaf(s, z[d], mean[d]);
    /* box bounds: only the asked member is clipped, the distribution is not truncated */
    x[d] = fminf(fmaxf(x[d], r->p.clip_min), r->p.clip_max);
  }
  free(z);
}

void orc_ask(const orc_run_t *r, float *x) {
  for (int32_t j = 0; j < r->popsize; ++j) orc_member(r, j, x + (int64_t)j * r->num_dims);
}

/* Weight-decay regularisation ("weight decay regularization"): the penalty
 * coef * ||x_j||_2^2 is added to the minimised fitness, ||x||^2 summed in binary64 in d order. */
void orc_weight_decay(const float *f, const float *x, int32_t n, int64_t D, float coef, float *out) {
  for (int32_t j = 0; j < n; ++j) {
    double s = 0.0;
    for (int64_t d = 0; d < D; ++d) s += (double)x[j * D + d] * (double)x[j * D + d];
    out[j] = (float)((double)f[j] + (double)coef * s);
  }
}

void orc_run_weight_decay(const orc_run_t *r, const float *f, float *out) {
  const int64_t D = r->num_dims;
  float *x = (float *)malloc(sizeof(float) * (size_t)D);
  for (int32_t j = 0; j < r->popsize; ++j) {
    orc_member(r, j, x);
    orc_weight_decay(f + j, x, 1, D, r->p.weight_decay, out + j);
  }
  free(x);
}

/* ---------------- N7 fitness ---------------- */
/* sin(pi b) for b in [0, 1/2]: b * P(b^2), P of degree 5 (NUMERICS N7, Rastrigin's S). */
static const float R0 = 0x1.921fb6p+1f, R1 = -0x1.4abc12p+2f, R2 = 0x1.467bc4p+1f,
                   R3 = -0x1.358390p-1f, R4 = 0x1.afe86cp-4f, R5 = -0x1.656ac0p-5f;

float orc_sinpi_half(float b) {
  float s = b * b;
  float P = R5;
  P = fmaf(P, s, R4);
  P = fmaf(P, s, R3);
  P = fmaf(P, s, R2);
  P = fmaf(P, s, R1);
  P = fmaf(P, s, R0);
  return b * P;
}

float orc_eval_one(int32_t fn, const float *x, int64_t D) {
  double acc = 0.0;
  if (fn == ORC_SPHERE) {
    for (int64_t d = 0; d < D; ++d) acc += (double)x[d] * (double)x[d];
  } else if (fn == ORC_ROSENBROCK) {
    for (int64_t d = 0; d + 1 < D; ++d) {
      double a = x[d], b = x[d + 1];
      double t1 = b - a * a;
      double t2 = 1.0 - a;
      acc += 100.0 * (t1 * t1) + t2 * t2;
    }
  } else {
    for (int64_t d = 0; d < D; ++d) {
      float a = fabsf(x[d]);
      float fr = a - floorf(a);
      float b = fminf(fr, 1.0f - fr);       /* sin(pi fr) = sin(pi min(fr, 1 - fr)), b exact */
      double S = orc_sinpi_half(b);
      acc += (double)x[d] * (double)x[d] + 20.0 * (S * S);
    }
  }
  return (float)acc;
}

void orc_eval(int32_t fn, const float *x, int32_t n, int64_t D, float *f) {
  for (int32_t j = 0; j < n; ++j) f[j] = orc_eval_one(fn, x + (int64_t)j * D, D);
}

/* ---------------- N9–N11 ranking ---------------- */
uint32_t orc_key(float f) {
  if (isnan(f)) return 0xFFFFFFFFu;
  if (f == 0.0f) return 0x80000000u;
  uint32_t b = f2u(f);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}

typedef struct { uint32_t key; int32_t j; } kj_t;
static int cmp_kj(const void *a, const void *b) {
  const kj_t *x = (const kj_t *)a, *y = (const kj_t *)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->j < y->j ? -1 : (x->j > y->j);
}

void orc_rank(const float *f, int32_t N, int32_t *s, int32_t *e, int32_t *perm) {
  kj_t *a = (kj_t *)malloc(sizeof(kj_t) * (size_t)N);
  for (int32_t j = 0; j < N; ++j) { a[j].key = orc_key(f[j]); a[j].j = j; }
  qsort(a, (size_t)N, sizeof(kj_t), cmp_kj);
  for (int32_t p = 0; p < N; ++p) {
    int32_t lo = p, hi = p;
    while (lo > 0 && a[lo - 1].key == a[p].key) --lo;
    while (hi + 1 < N && a[hi + 1].key == a[p].key) ++hi;
    if (perm) perm[p] = a[p].j;
    s[a[p].j] = lo;
    e[a[p].j] = hi;
  }
  free(a);
}

void orc_centered_rank(const float *f, int32_t N, float *c) {
  int32_t *s = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
  int32_t *e = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
  orc_rank(f, N, s, e, NULL);
  for (int32_t j = 0; j < N; ++j)
    c[j] = (float)(s[j] + e[j] - (N - 1)) / (float)(2 * (N - 1));
  free(s);
  free(e);
}

void orc_member_weights(const float *wpos, const float *f, int32_t N, float *w) {
  int32_t *s = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
  int32_t *e = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
  orc_rank(f, N, s, e, NULL);
  for (int32_t j = 0; j < N; ++j) {
    float sum = 0.0f;
    for (int32_t p = s[j]; p <= e[j]; ++p) sum = sum + wpos[p];
    w[j] = sum / (float)(e[j] - s[j] + 1);
  }
  free(s);
  free(e);
}

/* z-score shaping: (f - mean) / (std + 1e-8), population std, in double. */
void orc_zscore(const float *f, int32_t N, float *out) {
  double mu = 0.0, var = 0.0;
  for (int32_t j = 0; j < N; ++j) mu += (double)f[j];
  mu = mu / N;
  for (int32_t j = 0; j < N; ++j) var += ((double)f[j] - mu) * ((double)f[j] - mu);
  double sd = sqrt(var / N) + 1e-8;
  for (int32_t j = 0; j < N; ++j) out[j] = (float)(((double)f[j] - mu) / sd);
}

/* ---------------- N12 reductions ---------------- */
/* Number of tell entries: P directions (antithetic), N members (SNES), or Sep-CMA's weighted
 * sorted positions (through the end of the tie group containing position mu-1). */
/* ARS (Mania et al. 2018): k = max(1, round(elite_ratio * P)) directions with
 * the best min(f+, f-), ordered by (key(min), index). */
/* PGPE uses the same rule for its elite pairs (Q13: elite_ratio 1.0 keeps every pair). */
static int ars_k(const orc_run_t *r) {
  int P = r->popsize / 2;
  int k = (int)floor((double)r->p.elite_ratio * (double)P + 0.5);
  return k < 1 ? 1 : (k > P ? P : k);
}

static void ars_select(const orc_run_t *r, const float *f, int32_t *sel /* [k] */) {
  int P = r->popsize / 2;
  float *mn = (float *)malloc(sizeof(float) * (size_t)P);
  int32_t *s = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
  int32_t *e = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
  int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)P);
  for (int i = 0; i < P; ++i) mn[i] = fminf(f[2 * i], f[2 * i + 1]);
  orc_rank(mn, P, s, e, perm);
  for (int q = 0; q < ars_k(r); ++q) sel[q] = perm[q];
  free(mn); free(s); free(e); free(perm);
}

/* population std of the 2k fitness values of the selected pairs (double) */
static double ars_sigma_r(const orc_run_t *r, const float *f, const int32_t *sel, int k) {
  double m = 0.0, v = 0.0;
  for (int q = 0; q < k; ++q) m += (double)f[2 * sel[q]] + (double)f[2 * sel[q] + 1];
  m = m / (2.0 * k);
  for (int q = 0; q < k; ++q) {
    double a = (double)f[2 * sel[q]] - m, b = (double)f[2 * sel[q] + 1] - m;
    v += a * a + b * b;
  }
  return sqrt(v / (2.0 * k));
}

int orc_num_entries(const orc_run_t *r, const float *f) {
  if (r->algo == ORC_ARS || r->algo == ORC_PGPE) return ars_k(r);
  if (is_antithetic(r->algo)) return r->popsize / 2;
  if (r->algo == ORC_SNES) return r->popsize;
  int32_t N = r->popsize;
  int32_t *s = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
  int32_t *e = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
  int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
  orc_rank(f, N, s, e, perm);
  int ne = e[perm[r->mu - 1]] + 1;
  free(s); free(e); free(perm);
  return ne;
}

/* The direction sums of N12 restricted to tell entries [e0, e1): the share one rank of a
 * population-sharded run reduces before the all-reduce ("batch evolutionary gradients ...
 * aggregated via map-reduce"). orc_reduce is the full range. */
void orc_reduce_range(const orc_run_t *r, const float *f, int32_t e0, int32_t e1, double *G) {
  const int64_t D = r->num_dims;
  const int32_t N = r->popsize;
  double *G0 = G, *G1 = G + D;
  for (int64_t d = 0; d < 2 * D; ++d) G[d] = 0.0;
  float *sh = (float *)malloc(sizeof(float) * (size_t)N);
  float *z = (float *)malloc(sizeof(float) * (size_t)D);
  if (r->algo == ORC_ARS) {
    /* entries are the selected directions in selection order; coefficient f+ - f- (raw) */
    int k = ars_k(r);
    int32_t *sel = (int32_t *)malloc(sizeof(int32_t) * (size_t)k);
    ars_select(r, f, sel);
    for (int32_t q = e0; q < e1; ++q) {
      int i = sel[q];
      double a = (double)f[2 * i] - (double)f[2 * i + 1];
      run_direction(r, (uint32_t)i, r->t, z);
      for (int64_t d = 0; d < D; ++d) G0[d] += a * (double)z[d];
    }
    free(sel);
  } else if (is_antithetic(r->algo)) {
    if (r->p.shaping == 1) {
      memcpy(sh, f, sizeof(float) * (size_t)N);
    } else if (r->p.shaping == 2) {
      orc_zscore(f, N, sh);
    } else {
      orc_centered_rank(f, N, sh);
    }
    double bbar = 0.0;
    for (int32_t j = 0; j < N; ++j) bbar += (double)sh[j];
    bbar = bbar / N;
    /* PGPE elite pairs (reading Q13b): with k = round(elite_ratio P) < P the entries are the k
     * pairs ARS would select (by key(min(f+, f-)), then pair index), in that order; k = P keeps
     * every pair in index order. The shaping and the baseline use the whole population. */
    int32_t *sel = NULL;
    if (r->algo == ORC_PGPE && ars_k(r) < N / 2) {
      sel = (int32_t *)malloc(sizeof(int32_t) * (size_t)ars_k(r));
      ars_select(r, f, sel);
    }
    for (int32_t q = e0; q < e1; ++q) {
      int32_t i = sel ? sel[q] : q;
      double a = (double)sh[2 * i] - (double)sh[2 * i + 1];
      double h = ((double)sh[2 * i] + (double)sh[2 * i + 1]) * 0.5 - bbar;
      run_direction(r, (uint32_t)i, r->t, z);
      for (int64_t d = 0; d < D; ++d) {
        G0[d] += a * (double)z[d];
        if (r->algo == ORC_PGPE) G1[d] += h * ((double)z[d] * (double)z[d] - 1.0);
      }
    }
    free(sel);
  } else {
    int32_t *s = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
    int32_t *e = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
    int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
    orc_rank(f, N, s, e, perm);
    orc_member_weights(r->wpos, f, N, sh);
    for (int32_t q = e0; q < e1; ++q) {
      /* SNES entries are members in index order; Sep-CMA entries are sorted positions */
      int32_t j = r->algo == ORC_SNES ? q : perm[q];
      double w = (double)sh[j];
      if (sh[j] == 0.0f) continue; /* outside the elite: contributes exactly 0 */
      run_direction(r, (uint32_t)j, r->t, z);
      for (int64_t d = 0; d < D; ++d) {
        double zd = (double)z[d];
        G0[d] += w * zd;
        if (r->algo == ORC_SNES) G1[d] += w * (zd * zd - 1.0);
        else G1[d] += w * (zd * zd);
      }
    }
    free(s); free(e); free(perm);
  }
  free(sh);
  free(z);
}

void orc_reduce(const orc_run_t *r, const float *f, double *G) {
  orc_reduce_range(r, f, 0, orc_num_entries(r, f), G);
}

/* SGD with momentum: v' = fma(mu, v, g); mean' = mean - lr * v'. State in ADAM_M. */
static void sgd(orc_run_t *r, int64_t d, float g) {
  float *mean = vf(r, ORC_V_MEAN), *v = vf(r, ORC_V_ADAM_M);
  float vn = fmaf(r->p.momentum, v[d], g);
  v[d] = vn;
  mean[d] = mean[d] - r->lr * vn;
}

static void adam(orc_run_t *r, int64_t d, float g, float bc1, float bc2) {
  float *mean = vf(r, ORC_V_MEAN), *am = vf(r, ORC_V_ADAM_M), *av = vf(r, ORC_V_ADAM_V);
  const float b1 = r->p.beta1, b2 = r->p.beta2;
  float mn = fmaf(b1, am[d], (1.0f - b1) * g);
  float vn = fmaf(b2, av[d], (1.0f - b2) * (g * g));
  am[d] = mn;
  av[d] = vn;
  mean[d] = mean[d] - r->lr * ((mn / bc1) / (sqrtf(vn / bc2) + r->p.eps));
}

static int tell_impl(orc_run_t *r, const float *f);

/* Weight decay (when set) is the first step of tell: every later step — best tracking included
 * (reading R-WD) — sees f_j + weight_decay ||x_j||^2. */
int orc_tell(orc_run_t *r, const float *f) {
  if (r->p.weight_decay == 0.0f) return tell_impl(r, f);
  float *fw = (float *)malloc(sizeof(float) * (size_t)r->popsize);
  orc_run_weight_decay(r, f, fw);
  int rc = tell_impl(r, fw);
  free(fw);
  return rc;
}

static int tell_impl(orc_run_t *r, const float *f) {
  const int64_t D = r->num_dims;
  const int32_t N = r->popsize;
  /* best tracking with the pre-update state */
  int32_t *s = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
  int32_t *e = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
  int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
  orc_rank(f, N, s, e, perm);
  int32_t jb = perm[0];
  if (f[jb] < r->best_f) {
    r->best_f = f[jb];
    orc_member(r, jb, vf(r, ORC_V_BEST_X));
  }
  free(s);
  free(e);
  free(perm);

  double *G = (double *)malloc(sizeof(double) * 2 * (size_t)D);
  orc_reduce(r, f, G);
  int rc = orc_tell_apply(r, f, G);
  free(G);
  return rc;
}

/* The update of N12 from the direction sums G[2][D] (what orc_reduce, or the sum over ranks of
 * orc_reduce_range, produced), then t <- t+1. f is needed only by ARS (selection, sigma_R). */
int orc_tell_apply(orc_run_t *r, const float *f, const double *G) {
  const int64_t D = r->num_dims;
  const int32_t N = r->popsize;
  const double *G0 = G, *G1 = G + D;
  float *mean = vf(r, ORC_V_MEAN), *sd = vf(r, ORC_V_SIGMA);

  if (r->algo == ORC_ARS) {
    /* ARS update for minimisation (elite directions, sigma_R; no state normalisation):
     * mean -= alpha / (k sigma_R) * sum (f+ - f-) z_i */
    int k = ars_k(r);
    int32_t *sel = (int32_t *)malloc(sizeof(int32_t) * (size_t)k);
    ars_select(r, f, sel);
    double sr = ars_sigma_r(r, f, sel, k);
    free(sel);
    if (sr > 0.0) {
      float scale = (float)((double)r->lr / ((double)k * sr));
      for (int64_t d = 0; d < D; ++d) mean[d] = mean[d] - scale * (float)G0[d];
    }
    r->lr = fmaxf(r->lr * r->p.lrate_decay, r->p.lrate_limit);
    r->sigma = fmaxf(r->sigma * r->p.sigma_decay, r->p.sigma_limit);
  } else if (r->algo == ORC_OPENAI_ES || r->algo == ORC_PGPE) {
    r->b1pow = r->b1pow * (double)r->p.beta1;
    r->b2pow = r->b2pow * (double)r->p.beta2;
    float bc1 = (float)(1.0 - r->b1pow), bc2 = (float)(1.0 - r->b2pow);
    /* gradients of the mean (and PGPE's sigma step) first, so that ClipUp's global norms can be
     * formed before any mean moves */
    float *gm = (float *)malloc(sizeof(float) * (size_t)D);
    for (int64_t d = 0; d < D; ++d) {
      if (r->algo == ORC_OPENAI_ES) {
        gm[d] = (float)G0[d] / ((float)N * r->sigma);
      } else {
        /* PGPE normalises by the 2k members / k pairs it used (k = P: N and P) */
        float sig = sd[d];
        gm[d] = (sig * (float)G0[d]) / (float)(2 * ars_k(r));
        float gs = (sig * (float)G1[d]) / (float)ars_k(r);
        float mc = r->p.sigma_max_change;
        float st = sig - r->p.sigma_lrate * gs;
        float lo = (1.0f - mc) * sig, hi = (1.0f + mc) * sig;
        st = fminf(fmaxf(st, lo), hi);
        sd[d] = fmaxf(st * r->p.sigma_decay, r->p.sigma_limit);
      }
    }
    if (r->p.optimizer == ORC_ADAM) {
      for (int64_t d = 0; d < D; ++d) adam(r, d, gm[d], bc1, bc2);
    } else if (r->p.optimizer == ORC_SGD) {
      for (int64_t d = 0; d < D; ++d) sgd(r, d, gm[d]);
    } else {
      /* ClipUp (Toklu et al. 2020): g_hat = g / ||g||, v' = mu v + lr g_hat,
       * v' clipped to norm max_speed, mean' = mean - v'. Norms in double. */
      float *v = vf(r, ORC_V_ADAM_M);
      double n2 = 0.0;
      for (int64_t d = 0; d < D; ++d) n2 += (double)gm[d] * (double)gm[d];
      double gn = sqrt(n2);
      float inv = gn > 0.0 ? (float)(1.0 / gn) : 0.0f;
      double v2 = 0.0;
      for (int64_t d = 0; d < D; ++d) {
        v[d] = fmaf(r->p.momentum, v[d], r->lr * (gm[d] * inv));
        v2 += (double)v[d] * (double)v[d];
      }
      double vn = sqrt(v2);
      float clip = vn > (double)r->p.max_speed ? (float)((double)r->p.max_speed / vn) : 1.0f;
      for (int64_t d = 0; d < D; ++d) {
        v[d] = v[d] * clip;
        mean[d] = mean[d] - v[d];
      }
    }
    free(gm);
    r->lr = fmaxf(r->lr * r->p.lrate_decay, r->p.lrate_limit);
    if (r->algo == ORC_OPENAI_ES) r->sigma = fmaxf(r->sigma * r->p.sigma_decay, r->p.sigma_limit);
  } else if (r->algo == ORC_SNES) {
    for (int64_t d = 0; d < D; ++d) {
      float sig = sd[d];
      mean[d] = mean[d] + sig * (float)G0[d];
      sd[d] = sig * (float)exp(r->eta_sigma * 0.5 * G1[d]);
    }
  } else {
    float *ps = vf(r, ORC_V_PSIGMA), *pc = vf(r, ORC_V_PC), *Cd = vf(r, ORC_V_C);
    const float omcs = (float)(1.0 - r->c_sigma);
    const float ks = (float)sqrt(r->c_sigma * (2.0 - r->c_sigma) * r->mueff);
    double norm2 = 0.0;
    for (int64_t d = 0; d < D; ++d) {
      float Z = (float)G0[d];
      float y = sqrtf(Cd[d]) * Z;
      mean[d] = mean[d] + r->sigma * y;
      ps[d] = omcs * ps[d] + ks * Z;
      norm2 += (double)ps[d] * (double)ps[d];
    }
    double norm = sqrt(norm2);
    float sig_new = r->sigma * (float)exp((r->c_sigma / r->d_sigma) * (norm / r->chi_d - 1.0));
    double lhs = norm / sqrt(1.0 - pow(1.0 - r->c_sigma, 2.0 * (double)(r->t + 1)));
    int hs = lhs < (1.4 + 2.0 / ((double)r->full_dims + 1.0)) * r->chi_d;
    const float omcc = (float)(1.0 - r->c_c);
    const float kc = hs ? (float)sqrt(r->c_c * (2.0 - r->c_c) * r->mueff) : 0.0f;
    const float aC = (float)(1.0 - r->c_1 - r->c_mu +
                             (1.0 - (double)hs) * r->c_1 * r->c_c * (2.0 - r->c_c));
    const float c1f = (float)r->c_1, cmuf = (float)r->c_mu;
    for (int64_t d = 0; d < D; ++d) {
      float Z = (float)G0[d], Q = (float)G1[d];
      float C0 = Cd[d];
      float y = sqrtf(C0) * Z;
      float pcn = omcc * pc[d] + kc * y;
      pc[d] = pcn;
      Cd[d] = aC * C0 + c1f * (pcn * pcn) + cmuf * (C0 * Q);
    }
    r->sigma = sig_new;
  }
  r->t = r->t + 1;
  return 0;
}

/* ---------------- N15 synthetic fitness ---------------- */
void orc_synth_fitness(uint64_t seed, uint32_t t, int32_t N, float *f) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (int32_t j = 0; j < N; ++j) {
    uint32_t ctr[4] = {(uint32_t)(j / 4), 0u, t, 4u}, o[4];
    orc_philox4x32_10(ctr, key, o);
    f[j] = orc_u_b(o[j % 4]);
  }
}

/* ---------------- batch helpers (tests) ---------------- */
void orc_ln_n(const float *u, float *out, int64_t n) {
  for (int64_t k = 0; k < n; ++k) out[k] = orc_ln(u[k]);
}
void orc_sinpi_half_n(const float *b, float *out, int64_t n) {
  for (int64_t k = 0; k < n; ++k) out[k] = orc_sinpi_half(b[k]);
}
void orc_sincos2pi_n(const float *u, float *c, float *s, int64_t n) {
  for (int64_t k = 0; k < n; ++k) orc_sincos2pi(u[k], c + k, s + k);
}
/* n consecutive normals of stream (i, t, tag): index k uses counter (k/4, i, t, tag). */
void orc_normals_n(uint64_t seed, uint32_t i, uint32_t t, uint32_t tag, int64_t n, float *out) {
  float v[4];
  for (int64_t q = 0; 4 * q < n; ++q) {
    orc_normals4(seed, (uint32_t)q, i, t, tag, v);
    for (int k = 0; k < 4 && 4 * q + k < n; ++k) out[4 * q + k] = v[k];
  }
}

/* ---------------- N14 synthetic MLP fitness ---------------- */
/* IEEE binary16 round-to-nearest-even, returned widened to float (exact). */
float orc_fp16(float f) {
  if (isnan(f)) return f;
  uint32_t sign = f2u(f) & 0x80000000u;
  float a = fabsf(f);
  float r;
  if (a >= 65520.0f) {
    r = INFINITY;
  } else if (a < 0x1p-14f) {           /* binary16 subnormal range: quantum 2^-24 */
    r = rintf(a * 0x1p24f) * 0x1p-24f;
  } else {                             /* 11 significant bits: quantum 2^(e-10) */
    int e = (int)((f2u(a) >> 23) & 0xFF) - 127;
    float quantum = ldexpf(1.0f, e - 10);
    r = rintf(a / quantum) * quantum;
  }
  return u2f(sign | f2u(r));
}

struct orc_mlp {
  int32_t nw, batch;
  int32_t w[16];
  uint64_t seed;
  int64_t D;
  float *U;      /* [batch][w0] */
  double *Y;     /* [batch][wL] teacher outputs g_L(theta*) under the N14 definition */
  float *Y16;    /* [batch][wL] teacher outputs under the N14' fp16-image model */
};

int64_t orc_mlp_dims(const orc_mlp_t *p) { return p->D; }

static int64_t layer_off(const orc_mlp_t *p, int l) {   /* l = 1..L */
  int64_t off = 0;
  for (int q = 1; q < l; ++q) off += (int64_t)p->w[q - 1] * p->w[q] + p->w[q];
  return off;
}

void orc_mlp_teacher(const orc_mlp_t *p, float *theta) {
  for (int l = 1; l < p->nw; ++l) {
    const int in = p->w[l - 1], out = p->w[l];
    const float s = (float)(1.0 / sqrt((double)in));
    float *W = theta + layer_off(p, l);
    for (int n = 0; n < out; ++n)
      for (int k = 0; k < in; ++k) {
        float z[4];
        orc_normals4(p->seed, (uint32_t)(k / 4), (uint32_t)(4096 * l + n), 0u, 3u, z);
        W[(int64_t)n * in + k] = z[k % 4] * s;
      }
    for (int n = 0; n < out; ++n) W[(int64_t)out * in + n] = 0.0f;
  }
}

/* N14 (the definition; P:265-270 tanh MLP, fp32 parameters as the paper's JAX networks):
 * every layer a_l = h_{l-1} W_l^T + b_l and h_l = tanh(a_l) in binary64 from the fp32 inputs U and
 * the fp32 parameter vector x, nothing rounded in between; out [batch][wL]. */
static void mlp_forward(const orc_mlp_t *p, const float *x, double *out) {
  const int B = p->batch;
  int maxw = 0;
  for (int l = 0; l < p->nw; ++l) maxw = p->w[l] > maxw ? p->w[l] : maxw;
  double *h = (double *)malloc(sizeof(double) * (size_t)B * maxw);
  double *hn = (double *)malloc(sizeof(double) * (size_t)B * maxw);
  for (int b = 0; b < B; ++b)
    for (int k = 0; k < p->w[0]; ++k) h[(int64_t)b * p->w[0] + k] = (double)p->U[(int64_t)b * p->w[0] + k];
  for (int l = 1; l < p->nw; ++l) {
    const int in = p->w[l - 1], nout = p->w[l];
    const float *W = x + layer_off(p, l);
    const float *bias = W + (int64_t)nout * in;
    for (int b = 0; b < B; ++b)
      for (int n = 0; n < nout; ++n) {
        double acc = 0.0;
        for (int k = 0; k < in; ++k) acc += h[(int64_t)b * in + k] * (double)W[(int64_t)n * in + k];
        double g = tanh(acc + (double)bias[n]);
        if (l + 1 < p->nw) hn[(int64_t)b * nout + n] = g;
        else out[(int64_t)b * nout + n] = g;
      }
    double *t = h; h = hn; hn = t;
  }
  free(h); free(hn);
}

/* N14' (a labelled APPROXIMATION, not the definition): the model of what the fp16-image fast path
 * computes — every parameter (weights and biases) and the inputs rounded to binary16, products of
 * binary16 values summed (here in binary64), + fp16(b), tanh rounded to fp32, hidden activations
 * rounded to binary16. Its distance to N14 is measured member by member (orc_mlp_eval vs
 * orc_mlp_eval_f16), which is the fast path's derived error bound. */
static void mlp_forward_f16(const orc_mlp_t *p, const float *x, float *out) {
  const int B = p->batch;
  int maxw = 0;
  for (int l = 0; l < p->nw; ++l) maxw = p->w[l] > maxw ? p->w[l] : maxw;
  double *h = (double *)malloc(sizeof(double) * (size_t)B * maxw);
  double *hn = (double *)malloc(sizeof(double) * (size_t)B * maxw);
  double *Wd = (double *)malloc(sizeof(double) * (size_t)maxw * maxw);
  for (int b = 0; b < B; ++b)
    for (int k = 0; k < p->w[0]; ++k) h[(int64_t)b * p->w[0] + k] = orc_fp16(p->U[(int64_t)b * p->w[0] + k]);
  for (int l = 1; l < p->nw; ++l) {
    const int in = p->w[l - 1], nout = p->w[l];
    const float *W = x + layer_off(p, l);
    const float *bias = W + (int64_t)nout * in;
    for (int64_t e = 0; e < (int64_t)nout * in; ++e) Wd[e] = orc_fp16(W[e]);
    for (int b = 0; b < B; ++b)
      for (int n = 0; n < nout; ++n) {
        double acc = 0.0;
        for (int k = 0; k < in; ++k) acc += h[(int64_t)b * in + k] * Wd[(int64_t)n * in + k];
        float g = (float)tanh(acc + (double)orc_fp16(bias[n]));
        if (l + 1 < p->nw) hn[(int64_t)b * nout + n] = orc_fp16(g);
        else out[(int64_t)b * nout + n] = g;
      }
    double *t = h; h = hn; hn = t;
  }
  free(h); free(hn); free(Wd);
}

orc_mlp_t *orc_mlp_create(const int32_t *widths, int32_t nw, int32_t batch, uint64_t seed) {
  if (nw < 2 || nw > 16 || batch < 1) return NULL;
  orc_mlp_t *p = (orc_mlp_t *)calloc(1, sizeof(orc_mlp_t));
  p->nw = nw; p->batch = batch; p->seed = seed;
  for (int l = 0; l < nw; ++l) p->w[l] = widths[l];
  p->D = layer_off(p, nw);
  const int in0 = widths[0], outL = widths[nw - 1];
  p->U = (float *)malloc(sizeof(float) * (size_t)batch * in0);
  for (int b = 0; b < batch; ++b)
    for (int k = 0; k < in0; ++k) {
      float z[4];
      orc_normals4(seed, (uint32_t)(k / 4), (uint32_t)b, 0u, 2u, z);
      p->U[(int64_t)b * in0 + k] = z[k % 4];
    }
  float *theta = (float *)malloc(sizeof(float) * (size_t)p->D);
  orc_mlp_teacher(p, theta);
  p->Y = (double *)malloc(sizeof(double) * (size_t)batch * outL);
  p->Y16 = (float *)malloc(sizeof(float) * (size_t)batch * outL);
  mlp_forward(p, theta, p->Y);
  mlp_forward_f16(p, theta, p->Y16);
  free(theta);
  return p;
}

void orc_mlp_destroy(orc_mlp_t *p) {
  if (!p) return;
  free(p->U); free(p->Y); free(p->Y16); free(p);
}

/* f(x) = mean over (b, n) of (g_L(x) - g_L(theta*))^2, in binary64, rounded once (N14). */
void orc_mlp_eval(const orc_mlp_t *p, const float *x, int32_t n, float *f) {
  const int B = p->batch, outL = p->w[p->nw - 1];
  double *g = (double *)malloc(sizeof(double) * (size_t)B * outL);
  for (int32_t j = 0; j < n; ++j) {
    mlp_forward(p, x + (int64_t)j * p->D, g);
    double acc = 0.0;
    for (int64_t e = 0; e < (int64_t)B * outL; ++e) {
      double d = g[e] - p->Y[e];
      acc += d * d;
    }
    f[j] = (float)(acc / ((double)B * outL));
  }
  free(g);
}

/* The N14' approximation model's fitness (fp16 parameter image; teacher under the same model). */
void orc_mlp_eval_f16(const orc_mlp_t *p, const float *x, int32_t n, float *f) {
  const int B = p->batch, outL = p->w[p->nw - 1];
  float *g = (float *)malloc(sizeof(float) * (size_t)B * outL);
  for (int32_t j = 0; j < n; ++j) {
    mlp_forward_f16(p, x + (int64_t)j * p->D, g);
    double acc = 0.0;
    for (int64_t e = 0; e < (int64_t)B * outL; ++e) {
      double d = (double)g[e] - (double)p->Y16[e];
      acc += d * d;
    }
    f[j] = (float)(acc / ((double)B * outL));
  }
  free(g);
}

const double *orc_mlp_targets(const orc_mlp_t *p) { return p->Y; }
const float *orc_mlp_targets_f16(const orc_mlp_t *p) { return p->Y16; }
const float *orc_mlp_inputs(const orc_mlp_t *p) { return p->U; }
