/* oracle_sanitize_main.c — drives the C oracle (oracle/es_oracle.c) through every algorithm,
 * optimizer, shaping and bound variant, the ranking primitives (ties, NaN, ±0) and the MLP
 * problem, for a build with -fsanitize=address,undefined (tests/test_oracle_sanitize.py).
 * Test infrastructure only; prints "ok" when every call returned. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "es_oracle.h"

static orc_params_t base_params(uint64_t seed) {
  orc_params_t p;
  memset(&p, 0, sizeof p);
  p.seed = seed;
  p.init_min = -2.0f; p.init_max = 2.0f;
  p.sigma_init = 0.05f; p.sigma_decay = 0.999f; p.sigma_limit = 0.01f;
  p.lrate_init = 0.01f; p.lrate_decay = 0.999f; p.lrate_limit = 0.001f;
  p.beta1 = 0.9f; p.beta2 = 0.999f; p.eps = 1e-8f;
  p.sigma_lrate = 0.2f; p.sigma_max_change = 0.2f;
  p.temperature = 12.0f; p.elite_ratio = 0.5f;
  p.momentum = 0.9f; p.max_speed = 0.05f;
  p.clip_min = -INFINITY; p.clip_max = INFINITY;
  return p;
}

static int run(int algo, int N, int64_t D, orc_params_t p, int gens, int fn) {
  orc_run_t r;
  memset(&r, 0, sizeof r);
  r.algo = algo; r.popsize = N; r.num_dims = D; r.p = p;
  r.vec = calloc((size_t)ORC_NV * D, sizeof(float));
  r.wpos = calloc((size_t)N, sizeof(float));
  float *x = malloc(sizeof(float) * N * D), *f = malloc(sizeof(float) * N);
  double *G = malloc(sizeof(double) * 2 * D);
  int rc = orc_init(&r);
  for (int g = 0; rc == 0 && g < gens; ++g) {
    orc_ask(&r, x);
    orc_eval(fn, x, N, D, f);
    orc_reduce(&r, f, G);
    rc = orc_tell(&r, f);
  }
  free(x); free(f); free(G); free(r.vec); free(r.wpos);
  return rc;
}

int main(void) {
  const int algos[5] = {ORC_OPENAI_ES, ORC_PGPE, ORC_SNES, ORC_SEP_CMA_ES, ORC_ARS};
  int bad = 0;
  for (int a = 0; a < 5; ++a)
    for (int fn = 0; fn < 3; ++fn) {
      orc_params_t p = base_params(100 + a);
      bad |= run(algos[a], 16, 37, p, 3, fn);
      p.weight_decay = 0.05f; p.clip_min = -1.0f; p.clip_max = 1.5f; p.shaping = a < 2 ? 2 : 0;
      p.elite_ratio = a == ORC_PGPE ? 0.25f : 0.4f;
      bad |= run(algos[a], 24, 5, p, 3, fn);
    }
  for (int opt = 1; opt <= 2; ++opt) {
    orc_params_t p = base_params(7);
    p.optimizer = opt;
    bad |= run(ORC_OPENAI_ES, 16, 37, p, 4, ORC_SPHERE);
    bad |= run(ORC_PGPE, 16, 37, p, 4, ORC_RASTRIGIN);
  }
  /* ranking corner cases: ties, NaN, ±0, one member */
  float f[9] = {1.0f, NAN, -0.0f, 0.0f, 1.0f, -INFINITY, INFINITY, 1.0f, NAN};
  int32_t s[9], e[9], perm[9];
  float c[9];
  orc_rank(f, 9, s, e, perm);
  orc_centered_rank(f, 9, c);
  orc_zscore(f, 1, c);
  orc_rank(f, 1, s, e, perm);
  /* MLP problem */
  const int32_t widths[4] = {8, 16, 16, 4};
  orc_mlp_t *m = orc_mlp_create(widths, 4, 32, 3);
  const int64_t Dm = orc_mlp_dims(m);
  float *theta = malloc(sizeof(float) * 2 * Dm), fm[2];
  orc_mlp_teacher(m, theta);
  for (int64_t d = 0; d < Dm; ++d) theta[Dm + d] = theta[d] + 0.01f;
  orc_mlp_eval(m, theta, 2, fm);
  free(theta);
  orc_mlp_destroy(m);
  float fs[16];
  orc_synth_fitness(5, 2, 16, fs);
  if (bad) { printf("init/tell failed\n"); return 1; }
  printf("ok\n");
  return 0;
}
