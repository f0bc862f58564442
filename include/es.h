/*
 * es.h — C ABI of the B200-native evosax hot path (libes_b200.so).
 *
 * One generation of the ask → evaluate → tell loop of PAPER.md §2.1 (Listing 1) for the
 * diagonal-Gaussian ES family of Table 1 — OpenAI-ES, PGPE, SNES and
 * Sep-CMA-ES — batched over R independent runs (the paper's vmap over seeds or
 * hyperparameters) and optionally population-sharded over W GPUs with NCCL (the paper's
 * Future Work), plus the SURVEY §8(f) rows: fused ask + evaluate and D-sharding (f1), the
 * peer-memory fused tell (f2), the variants ARS / z-score / weight decay / SGD / ClipUp / PGPE
 * elite pairs / box bounds (f3) and full-covariance CMA-ES (f4). The arithmetic is frozen in
 * NUMERICS.md (N1–N17).
 *
 * Conventions (all entry points):
 *   - Minimisation. Fitness is "lower is better".
 *   - Every call is asynchronous and stream-ordered on the cudaStream_t given (NULL = legacy
 *     default stream); no call synchronises the device unless it is handed host memory.
 *   - Buffer arguments may be DEVICE pointers (no copy) or HOST pointers (pinned or pageable; the
 *     library stages them through device scratch with cudaMemcpyAsync and, for host outputs,
 *     synchronises the stream before returning). Host fitness INPUTS of es_tell / es_tell_local /
 *     es_weight_decay are read before the call returns (copied into a pinned staging buffer), so
 *     the caller may refill them at once. Layouts are row-major and dense.
 *   - Arguments are validated before any launch or state change; on error nothing is modified.
 *   - No C++ exception crosses the ABI. One context is used by one host thread at a time.
 *   - Member j of run r on rank w is global member w*(N/W) + j (antithetic pairs never straddle
 *     ranks). Noise is a pure function of (seed_r, direction, generation, dim): results are
 *     independent of R, W and launch shape (NUMERICS N2).
 */
#ifndef ES_B200_H
#define ES_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *es_stream_t; /* == cudaStream_t */

typedef enum {
  ES_OPENAI_ES = 0,
  ES_PGPE = 1,
  ES_SNES = 2,
  ES_SEP_CMA_ES = 3,/* P:179 */
  ES_ARS = 4,       /* antithetic, top-k directions, sigma_R normalised */
  ES_CMA_ES = 5     /* full covariance, x = m + σ·A·z with A = chol(C)
                       (P:106), refreshed every k = max(1, ⌊1/(10·D·(c₁+c_μ))⌋) tells; D ≤ 4096.
                       Population sharding: every rank samples all N members and runs the
                       identical tell on the all-gathered fitness (replicated state, no gradient
                       collective); x / fitness cover this rank's N/W members. No D-sharding  */
} es_algo_t;

typedef enum { ES_OPT_ADAM = 0, ES_OPT_SGD = 1, ES_OPT_CLIPUP = 2 } es_optimizer_t;

typedef enum {
  ES_FIT_SPHERE = 0,     /* Σ x_d²                                  (P:212 BBOB)      */
  ES_FIT_ROSENBROCK = 1, /* Σ 100(x_{d+1} − x_d²)² + (1 − x_d)²                              */
  ES_FIT_RASTRIGIN = 2,  /* 10D + Σ (x_d² − 10 cos 2πx_d), cancellation-free form (N7)         */
  ES_FIT_MLP = 3,        /* synthetic tanh-MLP regression fitness (N14): the
                            MLP of the fp32 parameters, fp32-accurate (binary16 hi/lo split of
                            every operand, three-product tensor-core sums; parameters |x| < 255) */
  ES_FIT_MLP16 = 4       /* the same MLP at binary16 parameter and activation precision (N14′):
                            a labelled APPROXIMATION of ES_FIT_MLP (its distance to N14 is
                            measured per member in the tests), half the bytes per parameter   */
} es_fitness_t;

typedef enum {
  ES_SUCCESS = 0,
  ES_ERR_INVALID_ARG = 1, /* bad sizes / hyperparameters / NULL pointers                         */
  ES_ERR_BAD_STATE = 2,   /* call order violated (tell without ask, problem not set, ...)       */
  ES_ERR_CUDA = 3,        /* CUDA launch or runtime error; message in es_last_error            */
  ES_ERR_NCCL = 4,        /* NCCL error; the context is unusable afterwards                     */
  ES_ERR_OOM = 5,         /* device allocation failed                                           */
  ES_ERR_UNSUPPORTED = 6  /* valid request outside what this build implements                   */
} es_status_t;

/* Hyperparameters of one run. Defaults: PAPER.md App. B "Ant" column (P:285–286, P:301–308,
 * P:323–332). Fields an algorithm does not use are ignored. */
typedef struct {
  uint64_t seed;              /* Philox key of the run (N1, N2)                                */
  float init_min, init_max;   /* mean_0 ~ U[init_min, init_max] from the INIT stream (N6)       */
  float sigma_init;           /* σ_0: scalar (OpenAI-ES, Sep-CMA-ES) or every σ_d (PGPE, SNES) */
  float sigma_decay, sigma_limit; /* σ ← max(σ·decay, limit) per generation (OpenAI-ES, PGPE)  */
  float lrate_init, lrate_decay, lrate_limit; /* Adam learning-rate schedule (OpenAI-ES, PGPE)  */
  float beta1, beta2, eps;    /* Adam: 0.9, 0.999, 1e-8                                 */
  float sigma_lrate;          /* PGPE σ learning rate: 0.2                              */
  float sigma_max_change;     /* PGPE relative σ clip: 0.2                              */
  float temperature;          /* SNES β                                          */
  float elite_ratio;          /* Sep-CMA-ES μ = ⌊elite_ratio·N⌋; ARS / PGPE keep
                                 k = max(1, round(elite_ratio·N/2)) pairs of best min(f+, f−)
                                 (PGPE 1.0 = every pair, DESIGN reading Q13b), in (0, 1] */
  int32_t shaping;            /* 0 = centered rank; 1 = raw fitness; 2 = z-score
                                 (P:213). OpenAI-ES / PGPE only (ARS always uses raw fitness)    */
  int32_t optimizer;          /* es_optimizer_t for the mean of OpenAI-ES / PGPE: Adam,
                                 SGD with momentum, ClipUp                               */
  float momentum;             /* SGD / ClipUp momentum (0.9)                                     */
  float max_speed;            /* ClipUp velocity norm limit (2·lrate)                            */
  float weight_decay;         /* ≥ 0: tell ranks f_j + weight_decay·‖x_j‖² ("weight decay
                                 regularization"; every algorithm; best tracking included)      */
  float clip_min, clip_max;   /* box bounds: asked members are clipped into
                                 [clip_min, clip_max]; the distribution is not truncated (the
                                 tell regenerates the unclipped z). ±INFINITY = unbounded        */
} es_run_params_t;

/* Fields readable with es_get / writable with es_set (checkpoint / resume). Shapes per context. */
typedef enum {
  ES_FIELD_MEAN = 0,     /* float [R][D]                                                     */
  ES_FIELD_SIGMA_D = 1,  /* float [R][D]  per-dimension σ (PGPE, SNES)                       */
  ES_FIELD_ADAM_M = 2,   /* float [R][D]  Adam m / SGD / ClipUp velocity (OpenAI-ES, PGPE)    */
  ES_FIELD_ADAM_V = 3,   /* float [R][D]                                                     */
  ES_FIELD_P_SIGMA = 4,  /* float [R][D]  Sep-CMA-ES evolution path p_σ                      */
  ES_FIELD_P_C = 5,      /* float [R][D]  Sep-CMA-ES evolution path p_c                       */
  ES_FIELD_C = 6,        /* float [R][D]  Sep-CMA-ES diagonal covariance                      */
  ES_FIELD_BEST_X = 7,   /* float [R][D]  best member so far                           */
  ES_FIELD_BEST_F = 8,   /* float [R]     best fitness so far                          */
  ES_FIELD_SIGMA = 9,    /* float [R]     scalar σ (OpenAI-ES, Sep-CMA-ES)                    */
  ES_FIELD_LRATE = 10,   /* float [R]     current Adam learning rate                          */
  ES_FIELD_GEN = 11,     /* uint32 [R]    completed tells t                                   */
  ES_FIELD_SHAPED = 12,  /* float [R][N]  last tell's shaped fitness: c_j (N10) or ω_j (N11)  */
  ES_FIELD_RANK_S = 13,  /* int32 [R][N]  last tell's tie-group start s_j (N9)               */
  ES_FIELD_RANK_E = 14,  /* int32 [R][N]  last tell's tie-group end e_j (N9)                 */
  ES_FIELD_PERM = 15,    /* int32 [R][N]  member at each sorted position (N9)                */
  ES_FIELD_FITNESS = 16, /* float [R][N]  last tell's full (gathered) fitness                 */
  ES_FIELD_DIRSUM = 17,  /* double [2][R][D] this rank's (after es_tell_local) or the summed
                            (before es_tell_apply) binary64 direction sums of N12; OpenAI-ES
                            uses only the first R*D entries                                    */
  ES_FIELD_NORM2 = 18,   /* double [R] Sep-CMA-ES: a D-shard's share of ‖p_σ'‖² after
                            es_tell_local; the caller sets the rank sum before es_tell_apply     */
  ES_FIELD_COV = 19,     /* float [R][D][D] CMA-ES covariance C (symmetric, both triangles kept) */
  ES_FIELD_CHOL = 20,    /* float [R][D][D] CMA-ES sampling factor A (lower; upper = 0)       */
  ES_NUM_FIELDS = 21
} es_field_t;

typedef struct es_ctx es_ctx_t;

/* Create a context: allocates the R runs' state on the current device and initialises it
 * (Listing 1 `strategy.initialize`; N6). popsize N is the GLOBAL population; each rank
 * owns N/W members (= N/(2W) antithetic pairs or N/W directions). For world_size > 1,
 * nccl_unique_id points at the 128-byte ncclUniqueId that rank 0 created and broadcast
 * (e.g. via torch.distributed). world_size == 1 with an id (from es_nccl_get_unique_id) creates a
 * one-rank communicator and es_tell then runs the population-sharded data plane (fitness
 * all-gather, direction-sum all-reduce, separate update kernel) on one GPU; NULL: the fused tell.
 * world_size > 1 with nccl_unique_id == NULL creates a communicator-less shard (split-phase tell only).
 * Errors: ES_ERR_INVALID_ARG if N < 2, D < 1, R < 1, N odd (OpenAI-ES/PGPE), N mod W != 0,
 * N/W odd (OpenAI-ES/PGPE), ⌊elite_ratio·N⌋ < 1 (Sep-CMA-ES), negative σ_init, non-positive
 * lrate_init (OpenAI-ES/PGPE), world_rank outside [0, W); ES_ERR_UNSUPPORTED if N > 2^20;
 * ES_ERR_OOM / ES_ERR_CUDA / ES_ERR_NCCL on allocation / runtime failure. *out is NULL on error.
 * Ownership: the context owns every state buffer and the NCCL communicator. */
es_status_t es_init(es_ctx_t **out, es_algo_t algo, int32_t num_runs, int32_t popsize,
                    int64_t num_dims, const es_run_params_t *params /* host [num_runs] */,
                    int32_t world_rank, int32_t world_size, const void *nccl_unique_id,
                    es_stream_t stream);

/* ask: write this rank's population x = m + σ·z (N6), float [R][N/W][D]. Idempotent within
 * a generation. Errors: ES_ERR_INVALID_ARG for NULL x. */
es_status_t es_ask(es_ctx_t *ctx, float *x, es_stream_t stream);

/* Fused ask + evaluate ("sampling ... can become a burden", P:225
 * memory): forms this rank's population exactly as es_ask (bit-identical x, written to x
 * [R][N/W][D] unless x is NULL — then it is never materialised in fp32) and writes its fitness (as
 * es_eval_bbob) to fitness [R][N/W]. BBOB: one kernel that evaluates while sampling. ES_FIT_MLP:
 * the ask, then the fp32-accurate tensor-core MLP on the fp32 population (x NULL: an internal
 * [R][N/W][D] buffer holds it). ES_FIT_MLP16 (N14′): the ask kernel writes the fp16 parameter
 * image the fitness uses, which the tcgen05 MLP kernel streams with TMA. For both MLP fitnesses x,
 * if given, must be 16-byte aligned device memory. ES_CMA_ES: the tensor-core sampling, then
 * es_eval_bbob's kernels (BBOB or the MLP on fp32 x). Counts as the generation's ask. Errors:
 * ES_ERR_INVALID_ARG for NULL fitness or a misaligned / host x with an MLP fitness;
 * ES_ERR_BAD_STATE for an MLP fitness without es_set_mlp_problem. */
es_status_t es_ask_eval(es_ctx_t *ctx, es_fitness_t fn, float *x, float *fitness,
                        es_stream_t stream);

/* evaluate: fitness[n] = f(x[n]) for n rows of length D (N7; MLP: N14, N14′).
 * Context-free for the BBOB functions (ctx may be NULL); ES_FIT_MLP / ES_FIT_MLP16 need a context
 * on which es_set_mlp_problem was called and D equal to its parameter count. x float [n][D],
 * fitness float [n]; host pointers are staged through the context's buffers (temporaries only
 * beyond their size), and the call then synchronises the stream. Errors: ES_ERR_INVALID_ARG
 * (n < 0, D < 1, unknown fn), ES_ERR_BAD_STATE (MLP problem not set). */
es_status_t es_eval_bbob(es_ctx_t *ctx, es_fitness_t fn, const float *x, int64_t n, int64_t num_dims,
                    float *fitness, es_stream_t stream);

/* tell: update every run from this rank's fitness slice, float [R][N/W]. Performs the
 * all-gather of fitness (W>1), ranks/shapes (N9–N11), best tracking, the regenerating reduction
 * over directions (N12; z is never stored — x is NOT an input, a documented departure from
 * P:96's tell(x, fitness, ...)), the all-reduce of the direction sums (W>1), the update and
 * t ← t+1. Errors: ES_ERR_BAD_STATE if no es_ask since the last tell; ES_ERR_INVALID_ARG for
 * NULL fitness. */
es_status_t es_tell(es_ctx_t *ctx, const float *fitness, es_stream_t stream);

/* Split-phase tell, for callers that manage the communication themselves (es_tell is exactly
 * all-gather + es_tell_local + all-reduce(ES_FIELD_DIRSUM) + es_tell_apply):
 *   es_tell_local  ranks/shapes the GATHERED fitness fitness_all (float [W][R][N/W], the rank-major
 *                  result of all-gathering every rank's slice), tracks the best member and reduces
 *                  this rank's share of the tell entries (es_shard_plan) into ES_FIELD_DIRSUM.
 *   es_tell_apply  applies the update from ES_FIELD_DIRSUM, which the caller has replaced by its
 *                  sum over ranks (es_get / es_set), and advances t.
 * Contexts created with world_size > 1 and nccl_unique_id == NULL have no communicator and can
 * only tell this way (es_tell then returns ES_ERR_BAD_STATE). Errors: ES_ERR_BAD_STATE when called
 * out of order (ask → local → apply). */
es_status_t es_tell_local(es_ctx_t *ctx, const float *fitness_all, es_stream_t stream);
es_status_t es_tell_apply(es_ctx_t *ctx, es_stream_t stream);

/* D-sharded contexts ("D-sharded multi-GPU mode for separable fitness"):
 * instead of splitting the population, each of W ranks owns a quad-aligned range of
 * dimensions [d_begin, d_end) of every member (es_dshard_plan) for all N members and R runs. The
 * noise counter is the global quad index, so every rank's members are column slices of the
 * unsharded population, bit for bit. A separable BBOB fitness (Sphere, Rosenbrock,
 * Rastrigin) is a sum over dims, so the only data-path collective of a generation is an
 * all-reduce of R·N binary64 partial fitness values inside es_ask_eval (plus R doubles of
 * ‖p_σ'‖² for Sep-CMA-ES inside es_tell); the tell needs no gradient all-reduce at all because
 * each rank updates only its own dims. Rosenbrock's pair term across a boundary uses a halo dim
 * d_end whose state each rank updates redundantly (identical arithmetic, identical bits).
 *   es_init_dshard     as es_init, W = world size of the dimension split; nccl_unique_id as there
 *                      (NULL: a communicator-less shard, split phase only). Weight decay and
 *                      ClipUp take their global norms from the ranks' shares (below).
 *   es_dshard_plan     out = (d_begin, d_end, state end = min(d_end + 1, D)); ES_ERR_INVALID_ARG
 *                      if ceil(D/4) < W (a rank would own no dims).
 *   es_dshard_info     out = (d_begin, d_end, state end, D) of a context.
 *   es_ask_eval        with a communicator: fitness [R][N] of the WHOLE problem on every rank
 *                      (x, if given, is this rank's column slice [R][N][d_end − d_begin]).
 *   es_ask_eval_partial  this rank's binary64 partial fitness [R][N] (host or device) for callers
 *                      that sum over ranks themselves; fitness = (float)(Σ_ranks partial).
 *   es_tell            fitness [R][N] (the full population's); no gradient collective. Global
 *                      norms are sums of the ranks' shares, all-reduced with the communicator:
 *                      ‖p_σ'‖² (Sep-CMA-ES, R doubles), weight decay's ‖x_j‖² (R·N doubles,
 *                      P:213) and ClipUp's ‖g‖², ‖v'‖² (R doubles each).
 *   es_tell_local / es_tell_apply  (no communicator) as es_tell; the caller sums the ES_FIELD_NORM2
 *                      shares over the ranks and es_set's the sum before each es_tell_apply
 *                      call; es_tell_apply_phases(ctx) calls are needed (2 with ClipUp: after
 *                      the first, NORM2 holds the ‖v'‖² share; 1 otherwise).
 *   es_sqnorm_partial  this rank's binary64 Σ_{owned d} x_jd² [R][N] of the asked generation
 *                      (device memory); es_weight_decay_apply(f, Σ_ranks sqnorm, out) then gives
 *                      out = f + weight_decay·‖x_j‖² — the split-phase weight decay, whose result
 *                      goes to es_tell_local (which applies no weight decay itself).
 * State fields (es_get / es_set) have the context's state dims (d_end − d_begin + halo). */
es_status_t es_init_dshard(es_ctx_t **out, es_algo_t algo, int32_t num_runs, int32_t popsize,
                           int64_t num_dims, const es_run_params_t *params, int32_t world_rank,
                           int32_t world_size, const void *nccl_unique_id, es_stream_t stream);
es_status_t es_dshard_plan(int64_t num_dims, int32_t world_size, int32_t rank, int64_t out[3]);
es_status_t es_dshard_info(const es_ctx_t *ctx, int64_t out[4]);
es_status_t es_ask_eval_partial(es_ctx_t *ctx, es_fitness_t fn, float *x, double *partial,
                                es_stream_t stream);
int32_t es_tell_apply_phases(const es_ctx_t *ctx);   /* 1 or 2; −1 for a NULL context */
es_status_t es_sqnorm_partial(es_ctx_t *ctx, double *sqnorm, es_stream_t stream);
es_status_t es_weight_decay_apply(es_ctx_t *ctx, const float *fitness, const double *sqnorm,
                                  float *out, es_stream_t stream);

/* the population-sharded tell with its collective fused into one kernel over
 * peer memory ("batch evolutionary gradients ... aggregated via map-reduce", memory split
 * across devices). Each rank exports the device pointers of its direction-sum buffer
 * (ES_FIELD_DIRSUM layout) and of its state fields; after es_p2p_set_peers, es_tell_p2p_apply
 * runs ONE kernel in which rank w reads the W partial sums of its quad slice [Q·w/W, Q·(w+1)/W)
 * from the peers (NVLink loads, summed in rank order), applies the update to the slice (its
 * optimizer state — Adam m/v, SGD velocity — is the only copy: state memory is split across the
 * ranks), and writes the slice's mean, best_x and (PGPE, SNES) σ_d into every peer's state
 * (NVLink stores). No NCCL all-reduce of D doubles is involved. Supported: OpenAI-ES, PGPE, SNES,
 * ARS with Adam or SGD; Sep-CMA-ES and ClipUp need global norms, so they run
 * es_p2p_finish_phases(ctx) more phases, each an es_tell_p2p_finish after a barrier:
 *   Sep-CMA-ES (1 phase): sum the ranks' norm2 shares of ‖p_σ'‖² (rank order), update σ, h_σ and
 *     the slice's p_c and C, and store the C slice into every peer;
 *   ClipUp (2 phases, Toklu et al. 2020): the apply kernel parks g and leaves the slice's
 *     ‖g‖² share; phase 0 sums the shares → v' = μ v + lr g/‖g‖ on the slice and its ‖v'‖² share;
 *     phase 1 sums those → the max_speed clip, m −= v on the slice, mean slice stored into every
 *     peer (the velocity stays with its owner).
 *   es_p2p_export     fill *out with this context's pointers (fields it does not keep are NULL).
 *   es_p2p_set_peers  peers[v] = rank v's export as mapped in THIS process (v = 0..W−1, W the
 *                     context's world size, ≤ 8; peers[rank] is this context's own export).
 *   es_tell_p2p_apply after es_tell_local on every rank (and a barrier: the peers' sums must be
 *                     complete), the fused reduce-scatter → update → all-gather; the caller
 *                     orders a second barrier before any rank's next es_ask.
 *   es_p2p_ipc_export / es_p2p_ipc_open  for real multi-GPU runs: 10 cudaIpcMemHandle_t (64 B
 *                     each: dirsum, the 8 fields, norm2) per rank; es_p2p_ipc_open takes all W
 *                     ranks' blocks (rank-major), maps the peers' and calls es_p2p_set_peers.
 * With a communicator and peers set, es_tell uses this path (all-gather of fitness, local
 * reduction, 4-byte NCCL barrier, the fused kernel, barrier, then each finish phase and a
 * barrier). es_tell_p2p_finish is a no-op when es_p2p_finish_phases is 0. Errors:
 * ES_ERR_UNSUPPORTED for CMA-ES / D-shard contexts / W > 8; ES_ERR_BAD_STATE out of order or
 * without peers (also a finish phase with no es_tell_p2p_apply pending). */
typedef struct {
  const double *dirsum;   /* [2][R][D] binary64 direction sums (this rank's share after tell_local) */
  float *field[8];        /* es_field_t 0..7 base pointers, float [R][D]; NULL if not kept        */
  const double *norm2;    /* [2R] this rank's slice shares: Sep-CMA ‖p_σ'‖² at [0,R); ClipUp ‖g‖²
                             at [0,R) and ‖v'‖² at [R,2R)                                        */
} es_peer_t;
es_status_t es_p2p_export(const es_ctx_t *ctx, es_peer_t *out);
es_status_t es_p2p_set_peers(es_ctx_t *ctx, const es_peer_t *peers, int32_t world_size);
es_status_t es_tell_p2p_apply(es_ctx_t *ctx, es_stream_t stream);
es_status_t es_tell_p2p_finish(es_ctx_t *ctx, es_stream_t stream);
int32_t es_p2p_finish_phases(const es_ctx_t *ctx);   /* 0, 1 or 2; −1 for a NULL context */
es_status_t es_p2p_ipc_export(const es_ctx_t *ctx, void *handles /* 10 × 64 bytes */);
es_status_t es_p2p_ipc_open(es_ctx_t *ctx, const void *handles_all /* W × 10 × 64 bytes */);

/* f2, NVLS variant: the same fused tell with the reduction done INSIDE the NVSwitch. Every rank
 * binds one symmetric buffer (direction sums, mean, best_x, σ_d) to a multicast object; the kernel
 * reads Σ_ranks of its slice with multimem.ld_reduce.add.f64 and broadcasts the updated slice with
 * multimem.st. Setup (collective): one rank calls es_nvls_open(creator = 1), which writes the
 * 64-byte fabric handle of the multicast object to *handle; the others call it with creator = 0
 * and that handle; after a barrier every rank calls es_nvls_bind (which moves those fields into
 * the bound buffer); after another barrier es_tell uses this path (W > 1 with a communicator),
 * or callers run es_tell_local → barrier → es_tell_nvls_apply → barrier. The in-switch sum
 * order is the hardware's (results may differ from the rank-ordered paths in the last binary64
 * bits). Errors: ES_ERR_UNSUPPORTED without multicast / fabric-handle support or for other
 * algorithms; ES_ERR_BAD_STATE out of order. */
es_status_t es_nvls_open(es_ctx_t *ctx, void *handle /* 64 bytes */, int32_t creator);
es_status_t es_nvls_bind(es_ctx_t *ctx);
es_status_t es_tell_nvls_apply(es_ctx_t *ctx, es_stream_t stream);

/* Weight-decay regularisation of this rank's fitness slice:
 * out[r][j] = (float)((double)fitness[r][j] + (double)weight_decay_r · Σ_d (double)x_jd²) for the
 * members x_j of the current (asked, not yet told) generation, regenerated from the noise counter
 * (x is not an input); out = fitness where weight_decay_r = 0. es_tell applies it itself; callers
 * of the split-phase tell apply it to their slice BEFORE gathering. fitness / out: float [R][N/W],
 * host or device, may alias. Errors: ES_ERR_BAD_STATE outside ask → tell; ES_ERR_INVALID_ARG for
 * NULL pointers. */
es_status_t es_weight_decay(es_ctx_t *ctx, const float *fitness, float *out, es_stream_t stream);

/* Population-sharding plan: for a population of `popsize` over world_size ranks and
 * `entries` weighted tell entries (P directions, or Sep-CMA-ES's weighted positions), write
 * out[0..4) = (first member, end member, first entry, end entry) owned by `rank`. Host-only. */
es_status_t es_shard_plan(int32_t popsize, int32_t entries, int32_t world_size, int32_t rank,
                          int32_t out[4]);

/* Synthetic fitness for tell-only sweeps (N15): fitness[r][j], j over this rank's members. */
es_status_t es_synth_fitness(es_ctx_t *ctx, float *fitness, es_stream_t stream);

/* Copy a state field out (es_get) or in (es_set); dst/src may be host or device. Errors:
 * ES_ERR_INVALID_ARG for an unknown field or one this algorithm does not keep. */
es_status_t es_get(es_ctx_t *ctx, es_field_t field, void *dst, es_stream_t stream);
es_status_t es_set(es_ctx_t *ctx, es_field_t field, const void *src, es_stream_t stream);

/* MLP fitness problem (N14): widths[0..n_widths) layer widths (input first; every layer tanh,
 * P:268–269), `batch` inputs drawn from the DATA stream of data_seed, teacher θ* from the TEACHER
 * stream, targets Y* = MLP_θ*(U) computed on the device by the same kernels (one set per MLP
 * fitness, so f(θ*) = 0 exactly for each). Flattening of a
 * parameter vector: per layer W as [out][in] row-major (nn.Linear layout) then b[out], layers in
 * order. Synchronises the stream. Errors: ES_ERR_INVALID_ARG for n_widths outside 2..16;
 * ES_ERR_UNSUPPORTED for widths not multiples of 16 in [16, 512] or batch != 128. */
es_status_t es_set_mlp_problem(es_ctx_t *ctx, const int32_t *widths, int32_t n_widths,
                               int32_t batch, uint64_t data_seed, es_stream_t stream);

/* Number of parameters of an MLP with these widths (Σ in·out + out); -1 on bad input. */
int64_t es_mlp_num_params(const int32_t *widths, int32_t n_widths);

/* Sizes of the context: R, N (global), N/W (local), D, P (global directions), W, rank. */
es_status_t es_shape(const es_ctx_t *ctx, int64_t out[7]);

/* Number of kernels this library launched on behalf of the context since creation. */
int64_t es_kernel_launches(const es_ctx_t *ctx);

/* Kernel timing for the benchmark: while enabled, the library brackets every kernel it launches
 * for this context with a CUDA event pair on the launching stream. es_profile_read synchronises
 * on the last event, then writes up to max_kinds entries: names (NUL-terminated, 32 bytes each),
 * total milliseconds and launch counts per kernel kind, clears the record and returns the number
 * of kinds (or -1 on error). */
es_status_t es_profile_enable(es_ctx_t *ctx, int32_t on);
int32_t es_profile_read(es_ctx_t *ctx, char *names /* [max_kinds][32] */, double *ms,
                        int64_t *counts, int32_t max_kinds);

/* Diagnostics for the parity tests: evaluate one NUMERICS primitive elementwise on the device.
 *   which = 0  Philox4x32-10 (N1): in uint32 [n][6] = (c0, c1, c2, c3, k0, k1) → out uint32 [n][4]
 *   which = 1  LN (N4):            in float [n]                                 → out float [n]
 *   which = 2  SINCOS2PI (N5):     in float [n]                                 → out float [n][2]
 *   which = 3  normals (N2):       in uint32 [n][6] = (q, i, t, tag, k0, k1)    → out float [n][4]
 *   which = 4  ρ square root:      in float [n] (= −2·LN(u))                    → out float [n]
 *   which = 5  sin(πb), b ≤ 1/2 (N7): in float [n]                              → out float [n]
 *   which = 6  tanh of the MLP (N14): in float [n]                              → out float [n]
 *   which = 7  tanh of N14′'s hidden layers (rounded to binary16 next): float [n] → float [n]
 * in/out are device pointers. Errors: ES_ERR_INVALID_ARG for unknown `which` or n < 0. */
es_status_t es_debug_primitive(int32_t which, const void *in, void *out, int64_t n,
                               es_stream_t stream);

/* Out-of-bounds-write detection for every device buffer the library allocates (compute-sanitizer
 * is unavailable on the target pool). When the environment variable ES_GUARD_ALLOCS=1 is set at
 * es_init / es_init_dshard, each state / workspace allocation of the context (all but the MLP
 * problem's read-only data set) gets 256-byte guard zones before and after it, filled
 * with 0xA5; es_debug_check_guards synchronises the device and writes to *bad_bytes the number of
 * guard bytes that no longer hold 0xA5 (0 = no write outside any buffer so far). Guard mode
 * rejects es_p2p_ipc_export (an IPC handle maps the allocation base). Errors: ES_ERR_BAD_STATE
 * when the context was not created in guard mode. */
es_status_t es_debug_check_guards(es_ctx_t *ctx, int64_t *bad_bytes);

es_status_t es_destroy(es_ctx_t *ctx);

/* Last error message of the context (or of the calling thread when ctx is NULL). */
const char *es_last_error(const es_ctx_t *ctx);
const char *es_status_string(es_status_t s);

/* Size of ncclUniqueId and a helper creating one (rank 0), so that bindings need no NCCL. */
int32_t es_nccl_unique_id_size(void);
es_status_t es_nccl_get_unique_id(void *out /* host, es_nccl_unique_id_size() bytes */);

#ifdef __cplusplus
}
#endif
#endif /* ES_B200_H */
