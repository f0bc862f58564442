/*
 * es_oracle.h — CPU ORACLE for the evosax diagonal-Gaussian ES hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library. The product path (paper_2212_04180_b200) never
 * does, and shares no code, header or table with it.
 *
 * A plain, slow, obviously-correct transcription of NUMERICS.md (which restates PAPER.md's
 * ask–evaluate–tell loop, for OpenAI-ES / PGPE / SNES / Sep-CMA-ES).
 * One run at a time; vmap-style batching is the caller looping over runs.
 */
#ifndef ES_ORACLE_H
#define ES_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OPENAI_ES = 0, ORC_PGPE = 1, ORC_SNES = 2, ORC_SEP_CMA_ES = 3, ORC_ARS = 4 };
enum { ORC_ADAM = 0, ORC_SGD = 1, ORC_CLIPUP = 2 };
enum { ORC_SPHERE = 0, ORC_ROSENBROCK = 1, ORC_RASTRIGIN = 2 };

/* Per-run vector fields inside orc_run_t.vec, each [D] floats. */
enum { ORC_V_MEAN = 0, ORC_V_SIGMA = 1, ORC_V_ADAM_M = 2, ORC_V_ADAM_V = 3,
       ORC_V_PSIGMA = 4, ORC_V_PC = 5, ORC_V_C = 6, ORC_V_BEST_X = 7, ORC_NV = 8 };

typedef struct {
  uint64_t seed;
  float init_min, init_max;
  float sigma_init, sigma_decay, sigma_limit;
  float lrate_init, lrate_decay, lrate_limit;
  float beta1, beta2, eps;
  float sigma_lrate, sigma_max_change;
  float temperature;
  float elite_ratio;   /* Sep-CMA elite; ARS / PGPE fraction of pairs kept (PGPE 1.0 = all) */
  int32_t shaping; /* 0 centered rank, 1 raw fitness, 2 z-score (OpenAI-ES/PGPE) */
  int32_t optimizer;   /* 0 Adam, 1 SGD with momentum, 2 ClipUp (OpenAI-ES/PGPE) */
  float momentum;      /* SGD / ClipUp momentum */
  float max_speed;     /* ClipUp velocity clip */
  float weight_decay;  /* fitness += weight_decay * ||x_j||^2 at tell */
  float clip_min, clip_max; /* box bounds applied to the asked members */
} orc_params_t;

typedef struct {
  int32_t algo;
  int32_t popsize;
  int64_t num_dims;
  orc_params_t p;
  /* per-run scalars (NUMERICS N12) */
  uint32_t t;
  float lr;
  float sigma;       /* scalar sigma: OpenAI-ES, Sep-CMA-ES */
  double b1pow, b2pow;
  float best_f;
  int32_t mu;        /* Sep-CMA elite count */
  double mueff, c_sigma, d_sigma, c_c, c_1, c_mu, chi_d, eta_sigma;
  float *vec;        /* caller-owned [ORC_NV][D] */
  float *wpos;       /* caller-owned [N] position weights (SNES / Sep-CMA) */
  /* Optional dimension subset: when dims != NULL the run holds only the num_dims global dimensions
   * dims[0..num_dims) of a problem with full_dims dimensions (noise counters use the global
   * index; D-dependent constants use full_dims). Exact for every per-dimension quantity of
   * OpenAI-ES / PGPE / SNES (their updates are elementwise given the ranks); Sep-CMA-ES's global
   * ||p_sigma|| needs dims == NULL. Used to check full-size GPU runs on sampled dimensions. */
  const int64_t *dims;
  int64_t full_dims;
} orc_run_t;

/* N1–N5 primitives */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
float orc_u_a(uint32_t o);
float orc_u_b(uint32_t o);
float orc_ln(float u);
void orc_sincos2pi(float u, float *c, float *s);
/* 4 normals of counter (q, i, t, tag) under key(seed) (N2) */
void orc_normals4(uint64_t seed, uint32_t q, uint32_t i, uint32_t t, uint32_t tag, float out[4]);
/* z row of direction i at generation t, dims [0, D) (tag ASK) */
void orc_direction(uint64_t seed, uint32_t i, uint32_t t, int64_t D, float *z);

/* N6 init / ask */
int orc_init(orc_run_t *r);
int orc_num_directions(const orc_run_t *r);
void orc_ask(const orc_run_t *r, float *x /* [N][D] */);
void orc_member(const orc_run_t *r, int32_t j, float *x /* [D] */);
/* weight-decay regularisation: out_j = f_j + coef ||x_j||^2 for n rows x */
void orc_weight_decay(const float *f, const float *x, int32_t n, int64_t D, float coef, float *out);
/* the same for the run's current members (regenerated); out may alias f */
void orc_run_weight_decay(const orc_run_t *r, const float *f, float *out);

/* N7 fitness */
void orc_eval(int32_t fn, const float *x, int32_t n, int64_t D, float *f);
float orc_eval_one(int32_t fn, const float *x, int64_t D);
float orc_sinpi_half(float b);

/* N9–N11 ranking and shaping */
uint32_t orc_key(float f);
void orc_rank(const float *f, int32_t N, int32_t *s, int32_t *e, int32_t *perm);
void orc_centered_rank(const float *f, int32_t N, float *c);
void orc_member_weights(const float *wpos, const float *f, int32_t N, float *w);
void orc_zscore(const float *f, int32_t N, float *out);

/* N12 tell: reductions (double) G[k][D] from shaped values, then update. */
void orc_reduce(const orc_run_t *r, const float *f, double *G /* [2][D] */);
int orc_num_entries(const orc_run_t *r, const float *f);
void orc_reduce_range(const orc_run_t *r, const float *f, int32_t e0, int32_t e1, double *G);
int orc_tell(orc_run_t *r, const float *f);
/* the update half of orc_tell (no best tracking, no weight decay): N12 from G[2][D], then t+1 */
int orc_tell_apply(orc_run_t *r, const float *f, const double *G);

/* batch helpers for exhaustive / statistical tests */
void orc_ln_n(const float *u, float *out, int64_t n);
void orc_sincos2pi_n(const float *u, float *c, float *s, int64_t n);
void orc_sinpi_half_n(const float *b, float *out, int64_t n);
void orc_normals_n(uint64_t seed, uint32_t i, uint32_t t, uint32_t tag, int64_t n, float *out);

/* N14 synthetic MLP fitness: orc_mlp_eval is the definition (binary64 forward of the fp32
 * parameters); orc_mlp_eval_f16 is the N14' fp16-image approximation model (labelled, not the
 * definition) whose distance to N14 is the fp16 fast path's derived bound. */
typedef struct orc_mlp orc_mlp_t;
float orc_fp16(float f);
orc_mlp_t *orc_mlp_create(const int32_t *widths, int32_t nw, int32_t batch, uint64_t seed);
void orc_mlp_destroy(orc_mlp_t *p);
int64_t orc_mlp_dims(const orc_mlp_t *p);
void orc_mlp_teacher(const orc_mlp_t *p, float *theta);
void orc_mlp_eval(const orc_mlp_t *p, const float *x, int32_t n, float *f);
void orc_mlp_eval_f16(const orc_mlp_t *p, const float *x, int32_t n, float *f);
const double *orc_mlp_targets(const orc_mlp_t *p);
const float *orc_mlp_targets_f16(const orc_mlp_t *p);
const float *orc_mlp_inputs(const orc_mlp_t *p);

/* N15 synthetic fitness */
void orc_synth_fitness(uint64_t seed, uint32_t t, int32_t N, float *f);

#ifdef __cplusplus
}
#endif
#endif
