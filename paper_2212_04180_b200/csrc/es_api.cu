// es_api.cu — the C ABI (include/es.h): context lifetime, argument validation, host-side constant
// tables (binary64, NUMERICS N11/N12), host↔device staging, NCCL plumbing and the launch sequence
// of one generation. No exception crosses the ABI; every CUDA/NCCL failure becomes a status code.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>

#include "es_ctx.h"

thread_local std::string g_err;

namespace esb {
bool pdl_on() {
  static const bool on = [] {
    const char* e = std::getenv("ES_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int sm_count() {
  static std::atomic<int> n[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int v = n[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    n[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}
}  // namespace esb

static bool antithetic(int algo) { return is_anti(algo); }

// ---- host constant tables (binary64; NUMERICS N11, N12) ------------------------------------
static void snes_weights(int N, double beta, std::vector<float>& out) {
  std::vector<double> u(N);
  for (int p = 0; p < N; ++p) u[p] = beta * ((double)(N - 1 - p) / N - 0.5);
  double z = 0.0;
  for (int p = 0; p < N; ++p) z += std::exp(u[p] - u[0]);
  for (int p = 0; p < N; ++p) out[p] = (float)(std::exp(u[p] - u[0]) / z);
}

static void sepcma_setup(int N, int64_t D, float elite, RunScal& rs, std::vector<float>& out) {
  const int mu = (int)std::floor((double)elite * (double)N);   // P:286 elite ratio
  std::vector<double> w(N, 0.0);
  double sum = 0.0, sum2 = 0.0;
  for (int p = 0; p < mu; ++p) {
    w[p] = std::log((N + 1) / 2.0) - std::log((double)(p + 1));
    sum += w[p];
  }
  for (int p = 0; p < N; ++p) {
    w[p] /= sum;
    sum2 += w[p] * w[p];
    out[p] = (float)w[p];
  }
  const double mueff = 1.0 / sum2, Dd = (double)D;
  rs.mu = mu;
  rs.mueff = mueff;
  rs.c_sigma = (mueff + 2.0) / (Dd + mueff + 5.0);
  rs.d_sigma = 1.0 + 2.0 * std::max(0.0, std::sqrt((mueff - 1.0) / (Dd + 1.0)) - 1.0) + rs.c_sigma;
  rs.c_c = (4.0 + mueff / Dd) / (Dd + 4.0 + 2.0 * mueff / Dd);
  const double c1 = 2.0 / ((Dd + 1.3) * (Dd + 1.3) + mueff);
  const double cmu = std::min(1.0 - c1, 2.0 * (mueff - 2.0 + 1.0 / mueff) /
                                            ((Dd + 2.0) * (Dd + 2.0) + mueff));
  rs.c_1 = c1 * (Dd + 2.0) / 3.0;      // Ros & Hansen (2008): separable learning-rate boost
  rs.c_mu = cmu * (Dd + 2.0) / 3.0;
  rs.chi_d = std::sqrt(Dd) * (1.0 - 1.0 / (4.0 * Dd) + 1.0 / (21.0 * Dd * Dd));
}

extern "C" {

const char* es_status_string(es_status_t s) {
  switch (s) {
    case ES_SUCCESS: return "success";
    case ES_ERR_INVALID_ARG: return "invalid argument";
    case ES_ERR_BAD_STATE: return "bad state";
    case ES_ERR_CUDA: return "CUDA error";
    case ES_ERR_NCCL: return "NCCL error";
    case ES_ERR_OOM: return "out of device memory";
    case ES_ERR_UNSUPPORTED: return "unsupported";
  }
  return "unknown status";
}

const char* es_last_error(const es_ctx_t* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

int32_t es_nccl_unique_id_size(void) { return (int32_t)sizeof(ncclUniqueId); }

es_status_t es_nccl_get_unique_id(void* out) {
  if (!out) return fail(nullptr, ES_ERR_INVALID_ARG, "out is NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, ES_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  std::memcpy(out, &id, sizeof id);
  return ES_SUCCESS;
}

int64_t es_kernel_launches(const es_ctx_t* ctx) { return ctx ? ctx->launches : -1; }

es_status_t es_shape(const es_ctx_t* c, int64_t out[7]) {
  if (!c || !out) return fail(nullptr, ES_ERR_INVALID_ARG, "NULL argument");
  out[0] = c->s.R; out[1] = c->s.N; out[2] = c->s.Nloc; out[3] = c->s.D; out[4] = c->s.P;
  out[5] = c->s.W; out[6] = c->s.rank;
  return ES_SUCCESS;
}

es_status_t es_destroy(es_ctx_t* c) {
  if (!c) return ES_SUCCESS;
  cudaDeviceSynchronize();
  if (c->comm) ncclCommDestroy(c->comm);
  for (auto& r : c->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : c->pool) cudaEventDestroy(e);
  if (c->nvls.stage) {
    cudaDeviceSynchronize();
    nvls_close(c->nvls);
  }
  for (void* p : c->ipc_open) cudaIpcCloseMemHandle(p);
  if (c->mlp) mlp_problem_destroy(c->mlp);
  for (int k = 0; k < 2; ++k) {
    if (c->hstage[k]) cudaFreeHost(c->hstage[k]);
    if (c->hstage_ev[k]) cudaEventDestroy(c->hstage_ev[k]);
  }
  for (void* p : c->allocs) cudaFree(p);
  delete c;
  return ES_SUCCESS;
}

// f1 D-sharding: quad-aligned contiguous dimension ranges (the Philox counter is the global quad).
static bool dshard_range(int64_t D, int32_t W, int32_t rank, int64_t& d0, int64_t& d1) {
  const int64_t Qg = (D + 3) / 4;                         // balanced: sizes differ by ≤ 1 quad
  const int64_t q0 = Qg * rank / W, q1 = Qg * (rank + 1) / W;
  d0 = 4 * q0;
  d1 = std::min<int64_t>(4 * q1, D);
  return d1 > d0;
}

es_status_t es_dshard_plan(int64_t D, int32_t W, int32_t rank, int64_t out[3]) {
  if (!out || D < 1 || W < 1 || rank < 0 || rank >= W)
    return fail(nullptr, ES_ERR_INVALID_ARG, "bad D-shard plan arguments");
  int64_t d0, d1;
  if (!dshard_range(D, W, rank, d0, d1))
    return fail(nullptr, ES_ERR_INVALID_ARG, "ceil(D/4) < world_size: rank %d owns no dims", rank);
  out[0] = d0; out[1] = d1; out[2] = std::min<int64_t>(d1 + 1, D);
  return ES_SUCCESS;
}

static es_status_t init_impl(es_ctx_t** out, es_algo_t algo, int32_t R, int32_t N, int64_t D,
                             const es_run_params_t* params, int32_t rank, int32_t W,
                             const void* uid, cudaStream_t st, bool dsh) {
  if (!out) return fail(nullptr, ES_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if ((int)algo < 0 || (int)algo > 5) return fail(nullptr, ES_ERR_INVALID_ARG, "unknown algo %d", algo);
  if (!params) return fail(nullptr, ES_ERR_INVALID_ARG, "params is NULL");
  if (R < 1) return fail(nullptr, ES_ERR_INVALID_ARG, "num_runs must be >= 1");
  if (N < 2) return fail(nullptr, ES_ERR_INVALID_ARG, "popsize must be >= 2");
  if (D < 1) return fail(nullptr, ES_ERR_INVALID_ARG, "num_dims must be >= 1");
  if (D >= (int64_t(1) << 34)) return fail(nullptr, ES_ERR_INVALID_ARG, "num_dims must be < 2^34");
  if (W < 1 || rank < 0 || rank >= W) return fail(nullptr, ES_ERR_INVALID_ARG, "bad rank/world_size");
  const int32_t pW = dsh ? 1 : W, prank = dsh ? 0 : rank;   // population sharding
  if (algo == ES_CMA_ES && dsh)
    return fail(nullptr, ES_ERR_UNSUPPORTED, "CMA-ES: D-sharding is not implemented");
  for (int r = 0; r < R && algo == ES_CMA_ES; ++r)
    if (params && params[r].weight_decay != 0.0f)
      return fail(nullptr, ES_ERR_UNSUPPORTED, "CMA-ES: weight decay is not implemented");
  if (algo == ES_CMA_ES && D > kCmaMaxDims)
    return fail(nullptr, ES_ERR_UNSUPPORTED, "CMA-ES: num_dims > %d is not implemented", kCmaMaxDims);
  int64_t d0 = 0, d1 = D;
  if (dsh && !dshard_range(D, W, rank, d0, d1))
    return fail(nullptr, ES_ERR_INVALID_ARG, "ceil(D/4) < world_size: rank %d owns no dims", rank);
  if (N % pW) return fail(nullptr, ES_ERR_INVALID_ARG, "popsize must be divisible by world_size");
  if (antithetic(algo) && ((N % 2) || ((N / pW) % 2)))
    return fail(nullptr, ES_ERR_INVALID_ARG, "antithetic strategies need an even popsize per rank");
  if (N > (1 << 20)) return fail(nullptr, ES_ERR_UNSUPPORTED, "popsize > 2^20 is not implemented");
  for (int r = 0; r < R; ++r) {
    const es_run_params_t& p = params[r];
    if (!(p.sigma_init >= 0.0f)) return fail(nullptr, ES_ERR_INVALID_ARG, "run %d: sigma_init < 0", r);
    if (antithetic(algo) && !(p.lrate_init > 0.0f))
      return fail(nullptr, ES_ERR_INVALID_ARG, "run %d: lrate_init must be > 0", r);
    const bool cmaish = algo == ES_SEP_CMA_ES || algo == ES_CMA_ES;
    if (cmaish && (int)std::floor((double)p.elite_ratio * N) < 1)
      return fail(nullptr, ES_ERR_INVALID_ARG, "run %d: floor(elite_ratio*N) < 1", r);
    if (cmaish && !(p.elite_ratio <= 1.0f))
      return fail(nullptr, ES_ERR_INVALID_ARG, "run %d: elite_ratio > 1", r);
    const bool adamish = algo == ES_OPENAI_ES || algo == ES_PGPE;
    if (p.shaping != 0 && !((p.shaping == 1 || p.shaping == 2) && adamish))
      return fail(nullptr, ES_ERR_INVALID_ARG, "run %d: raw/z-score shaping only for OpenAI-ES/PGPE", r);
    if (p.optimizer != ES_OPT_ADAM && !(adamish && (p.optimizer == ES_OPT_SGD || p.optimizer == ES_OPT_CLIPUP)))
      return fail(nullptr, ES_ERR_INVALID_ARG, "run %d: SGD/ClipUp only for OpenAI-ES/PGPE", r);
    if (p.optimizer == ES_OPT_CLIPUP && !(p.max_speed > 0.0f))
      return fail(nullptr, ES_ERR_INVALID_ARG, "run %d: ClipUp needs max_speed > 0", r);
    if ((algo == ES_ARS || algo == ES_PGPE) && !(p.elite_ratio > 0.0f && p.elite_ratio <= 1.0f))
      return fail(nullptr, ES_ERR_INVALID_ARG, "run %d: ARS/PGPE elite_ratio must be in (0, 1]", r);
    if (!(p.weight_decay >= 0.0f) || std::isinf(p.weight_decay))
      return fail(nullptr, ES_ERR_INVALID_ARG, "run %d: weight_decay must be finite and >= 0", r);
    if (!(p.clip_min <= p.clip_max))
      return fail(nullptr, ES_ERR_INVALID_ARG, "run %d: need clip_min <= clip_max", r);
  }
  es_ctx* c = new (std::nothrow) es_ctx();
  if (c) {
    const char* g = std::getenv("ES_GUARD_ALLOCS");
    c->guard = g && g[0] == '1';
  }
  if (!c) return fail(nullptr, ES_ERR_OOM, "host allocation failed");
  DevState& s = c->s;
  s.algo = algo; s.R = R; s.N = N; s.W = pW; s.rank = prank; s.Nloc = N / pW;
  s.any_clip = 0;
  // state dims: the owned [d0, d1) plus, for a D-shard that is not the last, the halo dim d1
  // (updated redundantly, bit-identically to its owner) that Rosenbrock's last pair term needs
  s.Dg = D;
  s.dshard = dsh ? 1 : 0;
  s.q0 = d0 / 4;
  s.Dx = d1 - d0;
  s.D = std::min<int64_t>(d1 + 1, D) - d0;
  s.Q = (s.D + 3) / 4;
  s.Qx = (s.Dx + 3) / 4;
  c->dW = dsh ? W : 1;
  c->drank = dsh ? rank : 0;
  c->d0 = d0;
  s.P = antithetic(algo) ? N / 2 : N;
  auto bail = [&](es_status_t e) { std::string m = c->err; es_destroy(c); g_err = m; return e; };
#define TRY(expr)                                                                              \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess) {                                                                  \
      fail(c, _e == cudaErrorMemoryAllocation ? ES_ERR_OOM : ES_ERR_CUDA, "%s: %s", #expr,     \
           cudaGetErrorString(_e));                                                           \
      return bail(_e == cudaErrorMemoryAllocation ? ES_ERR_OOM : ES_ERR_CUDA);               \
    }                                                                                         \
  } while (0)
  const size_t RD = (size_t)R * s.D, RN = (size_t)R * N;
  const int a = (int)algo;
  const bool cma = a == CMA_ES;
  bool need[NVEC] = {true, a == PGPE || a == SNES, antithetic(a), antithetic(a),
                     a == SEP_CMA_ES || cma, a == SEP_CMA_ES || cma, a == SEP_CMA_ES, true};
  for (int f = 0; f < NVEC; ++f) {
    s.vec[f] = nullptr;
    if (need[f]) TRY(dalloc(c, (void**)&s.vec[f], RD * sizeof(float)));
  }
  TRY(dalloc(c, (void**)&s.rs, R * sizeof(RunScal)));
  TRY(dalloc(c, (void**)&s.gs, R * sizeof(GenScal)));
  TRY(dalloc(c, (void**)&s.wpos, RN * sizeof(float)));
  TRY(dalloc(c, (void**)&s.fit, RN * sizeof(float)));
  TRY(dalloc(c, (void**)&s.shaped, RN * sizeof(float)));
  TRY(dalloc(c, (void**)&s.rs_s, RN * sizeof(int32_t)));
  TRY(dalloc(c, (void**)&s.rs_e, RN * sizeof(int32_t)));
  TRY(dalloc(c, (void**)&s.perm, RN * sizeof(int32_t)));
  TRY(dalloc(c, (void**)&s.pos, RN * sizeof(int32_t)));
  TRY(dalloc(c, (void**)&s.n2, 2 * (size_t)R * sizeof(double)));   // [0,R) shares, [R,2R) ClipUp ‖v'‖²
  s.cov = s.chol = s.cw = s.zbuf = s.ybuf = nullptr;
  s.chol_fail = nullptr;
  s.ut = s.vt = nullptr;
  s.kp = 0;
  if (cma) {
    const size_t RDD = (size_t)R * s.D * s.D, RND = (size_t)R * N * s.D;
    TRY(dalloc(c, (void**)&s.cov, RDD * sizeof(float)));
    TRY(dalloc(c, (void**)&s.chol, RDD * sizeof(float)));
    TRY(dalloc(c, (void**)&s.cw, RDD * sizeof(float)));
    TRY(dalloc(c, (void**)&s.zbuf, RND * sizeof(float)));
    TRY(dalloc(c, (void**)&s.ybuf, RND * sizeof(float)));
    TRY(dalloc(c, (void**)&s.chol_fail, R * sizeof(int32_t)));
    s.kp = (N + 31) / 32 * 32;
    TRY(dalloc(c, (void**)&s.ut, (size_t)R * s.D * s.kp * sizeof(float)));
    TRY(dalloc(c, (void**)&s.vt, (size_t)R * s.D * s.kp * sizeof(float)));
  }
  if (dsh) TRY(dalloc(c, (void**)&c->fpart, RN * sizeof(double)));
  TRY(dalloc(c, (void**)&s.dir, RN * sizeof(uint32_t)));
  TRY(dalloc(c, (void**)&s.coefA, RN * sizeof(double)));
  TRY(dalloc(c, (void**)&s.coefB, RN * sizeof(double)));
  TRY(dalloc(c, (void**)&s.G, 2 * RD * sizeof(double)));
  const int bpr = tell_blocks_per_run(s);
  TRY(dalloc(c, (void**)&s.arrive, (size_t)R * bpr * sizeof(uint32_t)));
  const size_t nparts = cma ? std::max<size_t>(bpr, (size_t)((s.D + 31) / 32)) : (size_t)bpr;
  TRY(dalloc(c, (void**)&s.normpart, (size_t)R * nparts * sizeof(double)));
  {
    int npad = 1;
    while (npad < N) npad <<= 1;
    s.gkeys = nullptr;
    if (npad > 16384) TRY(dalloc(c, (void**)&s.gkeys, (size_t)R * npad * sizeof(uint64_t)));
    // counting rank: [3][R][N] counters, [R][64] j-tile and [R] run arrivals, [R][2] slots
    const size_t nc = 3 * RN + (size_t)R * 64 + 3 * (size_t)R;
    TRY(dalloc(c, (void**)&s.rcnt, nc * sizeof(uint32_t)));
    TRY(cudaMemsetAsync(s.rcnt, 0, nc * sizeof(uint32_t), st));
    TRY(dalloc(c, (void**)&s.rbpart, (size_t)R * 64 * sizeof(double)));
    s.rrad = nullptr;
    s.rrad_bar = nullptr;
    if (R <= 16 && N <= 65536) {
      TRY(dalloc(c, (void**)&s.rrad, ((size_t)4 * R * N + (size_t)R * 256 * 32) * sizeof(uint32_t)));
      TRY(dalloc(c, (void**)&s.rrad_bar, 2 * sizeof(unsigned)));
      TRY(cudaMemsetAsync(s.rrad_bar, 0, 2 * sizeof(unsigned), st));
    }
  }
  // population sharding with a communicator — also a one-rank one (W = 1 with an id: the
  // collective data plane of es_tell executed on a single GPU)
  const bool pcoll = !dsh && (W > 1 || uid);
  if (pcoll) TRY(dalloc(c, (void**)&c->fgather, RN * sizeof(float)));
  // per-run scalars and weight tables, computed on the host in binary64
  c->host_rs.assign(R, RunScal{});
  std::vector<float> wpos(RN, 0.0f), wr(N);
  for (int r = 0; r < R; ++r) {
    const es_run_params_t& p = params[r];
    RunScal& rs = c->host_rs[r];
    rs.seed = p.seed; rs.t = 0; rs.lr = p.lrate_init; rs.sigma = p.sigma_init;
    rs.best_f = INFINITY; rs.shaping = p.shaping; rs.b1pow = 1.0; rs.b2pow = 1.0;
    rs.init_min = p.init_min; rs.init_max = p.init_max; rs.sigma_init = p.sigma_init;
    rs.sigma_decay = p.sigma_decay; rs.sigma_limit = p.sigma_limit;
    rs.lrate_decay = p.lrate_decay; rs.lrate_limit = p.lrate_limit;
    rs.beta1 = p.beta1; rs.beta2 = p.beta2; rs.eps = p.eps;
    rs.sigma_lrate = p.sigma_lrate; rs.sigma_max_change = p.sigma_max_change;
    rs.optimizer = p.optimizer; rs.momentum = p.momentum; rs.max_speed = p.max_speed;
    rs.weight_decay = p.weight_decay; rs.clip_lo = p.clip_min; rs.clip_hi = p.clip_max;
    rs.clip = std::isfinite(p.clip_min) || std::isfinite(p.clip_max);
    if (rs.clip) s.any_clip = 1;
    if (p.weight_decay != 0.0f) c->any_wd = true;
    if (algo == ES_ARS || algo == ES_PGPE) {   // k = max(1, round(elite_ratio · P)), P = N/2
      const int P = N / 2;
      rs.ars_k = std::max(1, std::min(P, (int)std::floor((double)p.elite_ratio * (double)P + 0.5)));
    }
    if (p.optimizer == ES_OPT_CLIPUP) c->any_clipup = true;
    std::fill(wr.begin(), wr.end(), 0.0f);
    if (algo == ES_SNES) {
      snes_weights(N, (double)p.temperature, wr);
      rs.eta_sigma = (3.0 + std::log((double)D)) / (5.0 * std::sqrt((double)D));
    } else if (algo == ES_SEP_CMA_ES) {
      sepcma_setup(N, D, p.elite_ratio, rs, wr);
    } else if (algo == ES_CMA_ES) {
      sepcma_setup(N, D, p.elite_ratio, rs, wr);
      // full CMA-ES: the tutorial rates without the separable (D+2)/3 boost, and the refresh
      // period k = max(1, ⌊1/(10·D·(c₁ + c_μ))⌋) of the Cholesky factor (R-CMA)
      const double Dd = (double)D, me = rs.mueff;
      rs.c_1 = 2.0 / ((Dd + 1.3) * (Dd + 1.3) + me);
      rs.c_mu = std::min(1.0 - rs.c_1, 2.0 * (me - 2.0 + 1.0 / me) / ((Dd + 2.0) * (Dd + 2.0) + me));
      rs.k_refresh = std::max(1, (int)std::floor(1.0 / (10.0 * Dd * (rs.c_1 + rs.c_mu))));
    }
    std::copy(wr.begin(), wr.end(), wpos.begin() + (size_t)r * N);
  }
  // the counting rank needs a shaping that is a per-member function of the ranks (no z-score,
  // no ARS / elite-pair selection)
  s.rank_par = algo != ES_ARS;
  for (int r = 0; r < R; ++r) {
    const RunScal& rs = c->host_rs[r];
    if ((antithetic(algo) && rs.shaping == 2) || (algo == ES_PGPE && rs.ars_k < N / 2))
      s.rank_par = 0;
  }
  {
    // tell entry split from each run's expected entry count on this rank (Sep-CMA-ES: μ_r)
    std::vector<int> ent(R);
    for (int r = 0; r < R; ++r) {
      int ne = algo == ES_SEP_CMA_ES ? c->host_rs[r].mu : (antithetic(algo) ? N / 2 : N);
      if (algo == ES_ARS || (algo == ES_PGPE && c->host_rs[r].ars_k < N / 2)) ne = c->host_rs[r].ars_k;
      int e0, e1;
      shard_range(ne, pW, prank, e0, e1);
      ent[r] = std::max(1, e1 - e0);
    }
    c->split = tell_pick_split(s, ent);
    if (c->split.nchunk > 1)
      TRY(dalloc(c, (void**)&s.Gchunk, (size_t)c->split.nchunk * 2 * RD * sizeof(double)));
    const std::vector<int4> items = tell_items(R, ent, c->split);
    if (items.size() > 65535) {
      fail(c, ES_ERR_UNSUPPORTED, "tell: %zu work items > 65535", items.size());
      return bail(ES_ERR_UNSUPPORTED);
    }
    int4* dit = nullptr;
    TRY(dalloc(c, (void**)&dit, items.size() * sizeof(int4)));
    TRY(cudaMemcpyAsync(dit, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
    c->split.items = dit;
    c->split.nitems = (int)items.size();
  }
  TRY(cudaMemcpyAsync(s.rs, c->host_rs.data(), R * sizeof(RunScal), cudaMemcpyHostToDevice, st));
  TRY(cudaMemcpyAsync(s.wpos, wpos.data(), RN * sizeof(float), cudaMemcpyHostToDevice, st));
  TRY(cudaMemsetAsync(s.arrive, 0, (size_t)R * bpr * sizeof(uint32_t), st));
  TRY(cudaMemsetAsync(s.G, 0, 2 * RD * sizeof(double), st));
  TRY(cudaMemsetAsync(s.coefB, 0, RN * sizeof(double), st));
  TRY(launch_init(s, st));
  c->launches += 1;
  if (cma) {
    TRY(launch_cma_init(s, st));
    c->launches += 1;
  }
  c->host_t.assign(R, 0u);
  TRY(cudaStreamSynchronize(st));   // host tables above are stack-owned
  if ((W > 1 || pcoll) && uid) {
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof id);
    ncclResult_t nr = ncclCommInitRank(&c->comm, W, id, rank);
    if (nr != ncclSuccess) {
      fail(c, ES_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(nr));
      return bail(ES_ERR_NCCL);
    }
    c->pcoll = pcoll;
  }
#undef TRY
  *out = c;
  return ES_SUCCESS;
}

es_status_t es_init(es_ctx_t** out, es_algo_t algo, int32_t R, int32_t N, int64_t D,
                    const es_run_params_t* params, int32_t rank, int32_t W, const void* uid,
                    es_stream_t stream) {
  return init_impl(out, algo, R, N, D, params, rank, W, uid, (cudaStream_t)stream, false);
}

es_status_t es_init_dshard(es_ctx_t** out, es_algo_t algo, int32_t R, int32_t N, int64_t D,
                           const es_run_params_t* params, int32_t rank, int32_t W,
                           const void* uid, es_stream_t stream) {
  return init_impl(out, algo, R, N, D, params, rank, W, uid, (cudaStream_t)stream, true);
}

es_status_t es_dshard_info(const es_ctx_t* c, int64_t out[4]) {
  if (!c || !out) return fail(nullptr, ES_ERR_INVALID_ARG, "NULL argument");
  out[0] = c->d0; out[1] = c->d0 + c->s.Dx; out[2] = c->d0 + c->s.D; out[3] = c->s.Dg;
  return ES_SUCCESS;
}

es_status_t es_ask(es_ctx_t* c, float* x, es_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!c || !x) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (c->broken) return fail(c, ES_ERR_BAD_STATE, "context unusable after an NCCL error");
  const DevState& s = c->s;
  const size_t bytes = (size_t)s.R * s.Nloc * s.Dx * sizeof(float);
  float* dst = x;
  const bool host = !is_device_ptr(x);
  if (host) {
    if (!c->xstage) CUDA_OR(c, dalloc(c, (void**)&c->xstage, bytes));
    dst = c->xstage;
  }
  if (s.algo == CMA_ES) {
    int nk = 0;
    ProfScope ps(c, "cma_ask", st);
    CUDA_OR(c, launch_cma_ask(s, dst, st, &nk));
    c->launches += nk;
  } else {
    ProfScope ps(c, "ask", st);
    CUDA_OR(c, launch_ask(s, dst, st));
    c->launches += 1;
  }
  if (host) {
    CUDA_OR(c, cudaMemcpyAsync(x, dst, bytes, cudaMemcpyDeviceToHost, st));
    CUDA_OR(c, cudaStreamSynchronize(st));
  }
  c->asked = true;
  return ES_SUCCESS;
}

static es_status_t ask_eval_bbob(es_ctx* c, es_fitness_t fn, float* x, float* f, double* fpo,
                                 cudaStream_t st);

es_status_t es_ask_eval(es_ctx_t* c, es_fitness_t fn, float* x, float* f, es_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!c || !f) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if ((int)fn < 0 || (int)fn > 4) return fail(c, ES_ERR_INVALID_ARG, "unknown fitness %d", fn);
  if (c->broken) return fail(c, ES_ERR_BAD_STATE, "context unusable after an NCCL error");
  const DevState& s = c->s;
  const size_t nloc = (size_t)s.R * s.Nloc;
  if (s.dshard && c->dW > 1 && !c->comm)
    return fail(c, ES_ERR_BAD_STATE, "D-shard without communicator: use es_ask_eval_partial");
  if (is_mlp(fn)) {
    if (s.dshard) return fail(c, ES_ERR_UNSUPPORTED, "the MLP fitness is not separable over dims");
    if (!c->mlp) return fail(c, ES_ERR_BAD_STATE, "es_set_mlp_problem was not called");
    if (mlp_problem_dims(c->mlp) != s.D) return fail(c, ES_ERR_INVALID_ARG, "D != MLP parameters");
    if (s.algo != CMA_ES && x && (!is_device_ptr(x) || (reinterpret_cast<uintptr_t>(x) & 15)))
      return fail(c, ES_ERR_INVALID_ARG, "x must be 16-byte aligned device memory (MLP fitness)");
  }
  if (s.algo == CMA_ES) {     // sample (tiled contraction) then evaluate (BBOB or the MLP)
    const bool xh = x && !is_device_ptr(x), fh = !is_device_ptr(f);
    float* xd = x;
    if (!x || xh) {
      if (!c->xstage) CUDA_OR(c, dalloc(c, (void**)&c->xstage, nloc * s.Dx * sizeof(float)));
      xd = c->xstage;
    }
    float* fd = f;
    if (fh) {
      if (!c->fstage) CUDA_OR(c, dalloc(c, (void**)&c->fstage, nloc * sizeof(float)));
      fd = c->fstage;
    }
    int nk = 0;
    {
      ProfScope ps(c, "cma_ask", st);
      CUDA_OR(c, launch_cma_ask(s, xd, st, &nk));
    }
    {
      ProfScope ps(c, fn == ES_FIT_MLP ? "eval_mlp" : fn == ES_FIT_MLP16 ? "eval_mlp16" : "eval_bbob", st);
      CUDA_OR(c, fn == ES_FIT_MLP ? launch_mlp_eval(c->mlp, xd, (int64_t)nloc, fd, st)
                 : fn == ES_FIT_MLP16 ? launch_mlp_eval_f16(c->mlp, xd, (int64_t)nloc, fd, st)
                                      : launch_eval_bbob((int)fn, xd, (int64_t)nloc, s.D, fd, st));
    }
    c->launches += nk + 1;
    if (xh) CUDA_OR(c, cudaMemcpyAsync(x, xd, nloc * s.Dx * sizeof(float), cudaMemcpyDeviceToHost, st));
    if (fh) CUDA_OR(c, cudaMemcpyAsync(f, fd, nloc * sizeof(float), cudaMemcpyDeviceToHost, st));
    if (xh || fh) CUDA_OR(c, cudaStreamSynchronize(st));
    c->asked = true;
    return ES_SUCCESS;
  }
  if (fn == ES_FIT_MLP) {
    // N14: the ask writes the split image (and x unless NULL); the fp32-accurate MLP streams the
    // image's two binary16 planes with TMA
    if (s.Dx % 4) return fail(c, ES_ERR_UNSUPPORTED, "MLP fitness needs D % 4 == 0");
    __half* img = mlp_problem_image(c->mlp, (int64_t)nloc, st);
    if (!img) return fail(c, ES_ERR_OOM, "MLP split image of %zu members", nloc);
    float* fd = f;
    const bool fh = !is_device_ptr(f);
    if (fh) {
      if (!c->fstage) CUDA_OR(c, dalloc(c, (void**)&c->fstage, nloc * sizeof(float)));
      fd = c->fstage;
    }
    {
      ProfScope ps(c, "ask32", st);
      CUDA_OR(c, launch_ask_split(s, x, img, st));
    }
    {
      ProfScope ps(c, "eval_mlp", st);
      CUDA_OR(c, launch_mlp_eval_img(c->mlp, (int64_t)nloc, fd, st));
    }
    c->launches += 2;
    if (fh) {
      CUDA_OR(c, cudaMemcpyAsync(f, fd, nloc * sizeof(float), cudaMemcpyDeviceToHost, st));
      CUDA_OR(c, cudaStreamSynchronize(st));
    }
    c->asked = true;
    return ES_SUCCESS;
  }
  if (fn == ES_FIT_MLP16) {
    // N14′: the ask writes fp16(x) (and x unless NULL); the MLP streams that image with TMA
    if (!c->x16) CUDA_OR(c, dalloc(c, (void**)&c->x16, nloc * s.D * sizeof(__half)));
    float* fd = f;
    const bool fh = !is_device_ptr(f);
    if (fh) {
      if (!c->fstage) CUDA_OR(c, dalloc(c, (void**)&c->fstage, nloc * sizeof(float)));
      fd = c->fstage;
    }
    {
      ProfScope ps(c, "ask16", st);
      CUDA_OR(c, launch_ask16(s, x, c->x16, st));
    }
    {
      ProfScope ps(c, "eval_mlp16", st);
      CUDA_OR(c, launch_mlp_eval16(c->mlp, c->x16, (int64_t)nloc, fd, st));
    }
    c->launches += 2;
    if (fh) {
      CUDA_OR(c, cudaMemcpyAsync(f, fd, nloc * sizeof(float), cudaMemcpyDeviceToHost, st));
      CUDA_OR(c, cudaStreamSynchronize(st));
    }
    c->asked = true;
    return ES_SUCCESS;
  }
  return ask_eval_bbob(c, fn, x, f, nullptr, st);
}

// BBOB fused ask + evaluate. f: fitness out (a D-shard sums the ranks' binary64 partials with
// NCCL first); fpo: a D-shard's own partials out instead (es_ask_eval_partial).
static es_status_t ask_eval_bbob(es_ctx* c, es_fitness_t fn, float* x, float* f, double* fpo,
                                 cudaStream_t st) {
  const DevState& s = c->s;
  const size_t nloc = (size_t)s.R * s.Nloc;
  if (!c->aepart)
    CUDA_OR(c, dalloc(c, (void**)&c->aepart, nloc * ask_eval_blocks_per_run(s) * sizeof(double)));
  float* xd = x;
  const bool xh = x && !is_device_ptr(x);
  if (xh) {
    if (!c->xstage) CUDA_OR(c, dalloc(c, (void**)&c->xstage, nloc * s.Dx * sizeof(float)));
    xd = c->xstage;
  }
  void* out = f ? (void*)f : (void*)fpo;
  const bool oh = !is_device_ptr(out);
  float* fd = f;
  if (f && oh) {
    if (!c->fstage) CUDA_OR(c, dalloc(c, (void**)&c->fstage, nloc * sizeof(float)));
    fd = c->fstage;
  }
  if (!s.dshard) {
    ProfScope ps(c, "ask_eval", st);
    CUDA_OR(c, launch_ask_eval(s, (int)fn, xd, c->aepart, fd, st));
    c->launches += 2;
  } else {
    {
      ProfScope ps(c, "ask_eval", st);
      CUDA_OR(c, launch_ask_eval_partial(s, (int)fn, xd, c->aepart, c->fpart, st));
      c->launches += 2;
    }
    if (f) {
      if (c->dW > 1) {     // the only data-path collective of a D-sharded generation: R·N doubles
        ProfScope ps(c, "allreduce", st);
        NCCL_OR(c, ncclAllReduce(c->fpart, c->fpart, nloc, ncclFloat64, ncclSum, c->comm, st));
      }
      CUDA_OR(c, launch_partial_to_fitness(c->fpart, (int64_t)nloc, fd, st));
      c->launches += 1;
    } else {
      CUDA_OR(c, cudaMemcpyAsync(fpo, c->fpart, nloc * sizeof(double), cudaMemcpyDefault, st));
    }
  }
  if (xh) CUDA_OR(c, cudaMemcpyAsync(x, xd, nloc * s.Dx * sizeof(float), cudaMemcpyDeviceToHost, st));
  if (f && oh) CUDA_OR(c, cudaMemcpyAsync(f, fd, nloc * sizeof(float), cudaMemcpyDeviceToHost, st));
  if (xh || oh) CUDA_OR(c, cudaStreamSynchronize(st));
  c->asked = true;
  return ES_SUCCESS;
}

es_status_t es_ask_eval_partial(es_ctx_t* c, es_fitness_t fn, float* x, double* fpart,
                                es_stream_t stream_) {
  if (!c || !fpart) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (!c->s.dshard) return fail(c, ES_ERR_BAD_STATE, "es_ask_eval_partial needs a D-sharded context");
  if ((int)fn < 0 || (int)fn > 2) return fail(c, ES_ERR_INVALID_ARG, "separable BBOB fitness only");
  return ask_eval_bbob(c, fn, x, nullptr, fpart, (cudaStream_t)stream_);
}

es_status_t es_synth_fitness(es_ctx_t* c, float* f, es_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!c || !f) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  const DevState& s = c->s;
  const size_t bytes = (size_t)s.R * s.Nloc * sizeof(float);
  float* dst = f;
  const bool host = !is_device_ptr(f);
  if (host) {
    if (!c->fstage) CUDA_OR(c, dalloc(c, (void**)&c->fstage, bytes));
    dst = c->fstage;
  }
  {
    ProfScope ps(c, "synth_fitness", st);
    CUDA_OR(c, launch_synth(s, dst, st));
  }
  c->launches += 1;
  if (host) {
    CUDA_OR(c, cudaMemcpyAsync(f, dst, bytes, cudaMemcpyDeviceToHost, st));
    CUDA_OR(c, cudaStreamSynchronize(st));
  }
  c->asked = true;   // synthetic fitness stands in for ask + evaluate of this generation
  return ES_SUCCESS;
}

es_status_t es_eval_bbob(es_ctx_t* c, es_fitness_t fn, const float* x, int64_t n, int64_t D,
                         float* f, es_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!x || !f) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (n < 0 || D < 1) return fail(c, ES_ERR_INVALID_ARG, "bad sizes n=%lld D=%lld", (long long)n, (long long)D);
  if ((int)fn < 0 || (int)fn > 4) return fail(c, ES_ERR_INVALID_ARG, "unknown fitness %d", fn);
  if (is_mlp(fn)) {
    if (!c || !c->mlp) return fail(c, ES_ERR_BAD_STATE, "es_set_mlp_problem was not called");
    if (mlp_problem_dims(c->mlp) != D)
      return fail(c, ES_ERR_INVALID_ARG, "D=%lld != MLP parameter count %lld", (long long)D,
                  (long long)mlp_problem_dims(c->mlp));
  }
  if (n == 0) return ES_SUCCESS;
  const bool xh = !is_device_ptr(x), fh = !is_device_ptr(f);
  const float* xd = x;
  float* fd = f;
  // host buffers are staged through the context's cached buffers when they fit (no cudaMalloc /
  // cudaFree per call, which would synchronise the device); temporaries beyond that are freed on
  // every exit path
  struct Tmp {
    void* p = nullptr;
    ~Tmp() { if (p) cudaFree(p); }
  } tmpx, tmpf;
  const size_t cap = c ? (size_t)c->s.R * c->s.Nloc : 0;
  if (xh) {
    if (c && (size_t)n <= cap && D == c->s.Dx) {
      if (!c->xstage) CUDA_OR(c, dalloc(c, (void**)&c->xstage, cap * c->s.Dx * sizeof(float)));
      xd = c->xstage;
    } else {
      CUDA_OR(c, cudaStreamSynchronize(st));
      CUDA_OR(c, cudaMalloc(&tmpx.p, (size_t)n * D * sizeof(float)));
      xd = (const float*)tmpx.p;
    }
    CUDA_OR(c, cudaMemcpyAsync(const_cast<float*>(xd), x, (size_t)n * D * sizeof(float),
                               cudaMemcpyHostToDevice, st));
  }
  if (fh) {
    if (c && (size_t)n <= cap) {
      if (!c->fstage) CUDA_OR(c, dalloc(c, (void**)&c->fstage, cap * sizeof(float)));
      fd = c->fstage;
    } else {
      CUDA_OR(c, cudaMalloc(&tmpf.p, (size_t)n * sizeof(float)));
      fd = (float*)tmpf.p;
    }
  }
  cudaError_t e;
  {
    ProfScope ps(c, fn == ES_FIT_MLP ? "eval_mlp" : fn == ES_FIT_MLP16 ? "eval_mlp16" : "eval_bbob", st);
    e = fn == ES_FIT_MLP ? launch_mlp_eval(c->mlp, xd, n, fd, st)
        : fn == ES_FIT_MLP16 ? launch_mlp_eval_f16(c->mlp, xd, n, fd, st)
                             : launch_eval_bbob((int)fn, xd, n, D, fd, st);
  }
  if (e != cudaSuccess) {
    cudaStreamSynchronize(st);
    return fail(c, ES_ERR_CUDA, "eval launch: %s", cudaGetErrorString(e));
  }
  if (c) c->launches += 1;
  if (fh) CUDA_OR(c, cudaMemcpyAsync(f, fd, (size_t)n * sizeof(float), cudaMemcpyDeviceToHost, st));
  // host x / fitness: the copies complete (and temporaries may be freed) before returning
  if (xh || fh || tmpx.p || tmpf.p) CUDA_OR(c, cudaStreamSynchronize(st));
  return ES_SUCCESS;
}

// a6 + a7 (+ a10 bookkeeping): ranks of the gathered fitness, then this rank's entry reduction.
static es_status_t tell_local_impl(es_ctx* c, const float* fsrc, bool fused, cudaStream_t st) {
  const DevState& s = c->s;
  {
    ProfScope ps(c, "rank", st);
    CUDA_OR(c, launch_rank(s, fsrc, st));
  }
  c->launches += rank_launches(s);
  if (s.algo == CMA_ES) {
    // refresh the Cholesky factor after this tell for the runs whose k divides t + 1. Every
    // refresh kernel re-checks that per run on the device (t is device state), so the host
    // counter only skips launches that would all be no-ops; once a generation has been captured
    // into a CUDA graph (replays do not run this host code) the launches are always issued.
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
      c->graph_seen = true;
    bool refresh = c->graph_seen;
    for (int r = 0; r < s.R; ++r) {
      c->host_t[r] += 1;
      if (c->host_t[r] % (uint32_t)c->host_rs[r].k_refresh == 0) refresh = true;
    }
    int nk = 0;
    ProfScope ps(c, "cma_tell", st);
    CUDA_OR(c, launch_cma_tell(s, refresh, st, &nk));
    c->launches += nk;
    return ES_SUCCESS;
  }
  ProfScope ps(c, fused ? "tell" : "tell_reduce", st);
  CUDA_OR(c, launch_tell_reduce(s, fused, c->split, st));
  c->launches += 1;
  return ES_SUCCESS;
}

// a9 from the summed direction sums (update kernel), then Sep-CMA's global-norm phases.
// n2_summed: a D-shard's ‖p_σ'‖² share was already summed over ranks by the caller (split phase).
static es_status_t tell_apply_impl(es_ctx* c, bool fused, cudaStream_t st, bool n2_summed = false) {
  const DevState& s = c->s;
  if (s.algo == CMA_ES) return ES_SUCCESS;          // launch_cma_tell did every phase
  if (!fused) {
    ProfScope ps(c, "tell_update", st);
    CUDA_OR(c, launch_tell_update(s, st));
    c->launches += 1;
  }
  if (s.algo == SEP_CMA_ES) {
    if (s.dshard && !n2_summed) {
      CUDA_OR(c, launch_sepcma_n2(s, st));
      c->launches += 1;
      if (c->dW > 1) {   // R doubles: the D-shard's second (tiny) collective
        ProfScope ps(c, "allreduce", st);
        NCCL_OR(c, ncclAllReduce(s.n2, s.n2, (size_t)s.R, ncclFloat64, ncclSum, c->comm, st));
      }
    }
    int nk = 0;
    ProfScope ps(c, "sepcma_finish", st);
    CUDA_OR(c, launch_sepcma_finish(s, st, &nk));
    c->launches += nk;
  }
  if (c->any_clipup) {
    int nk = 0;
    ProfScope ps(c, "clipup_finish", st);
    if (s.dshard && c->dW > 1) {
      // the two global norms of a D-shard: shares summed by NCCL here; in the split-phase API
      // (n2_summed) es_tell_apply drives the phases and the caller sums
      if (!n2_summed) {
        CUDA_OR(c, launch_sepcma_n2(s, st));                      // ‖g‖² share
        for (int ph = 0; ph < 2; ++ph) {
          NCCL_OR(c, ncclAllReduce(s.n2, s.n2, (size_t)s.R, ncclFloat64, ncclSum, c->comm, st));
          int k = 0;
          CUDA_OR(c, launch_clipup_dshard_phase(s, ph, st, &k));
          nk += k;
        }
        nk += 1;
      }
    } else {
      CUDA_OR(c, launch_clipup_finish(s, st, &nk));
    }
    c->launches += nk;
  }
  return ES_SUCCESS;
}

static const float* stage_fitness(es_ctx* c, const float* f, size_t n, cudaStream_t st,
                                  float** buf, es_status_t* err) {
  *err = ES_SUCCESS;
  if (is_device_ptr(f)) return f;
  if (!*buf) {
    cudaError_t e = dalloc(c, (void**)buf, n * sizeof(float));
    if (e != cudaSuccess) { *err = fail(c, ES_ERR_OOM, "staging: %s", cudaGetErrorString(e)); return nullptr; }
  }
  // the caller's host buffer is read synchronously (into a pinned staging buffer) so it may be
  // refilled as soon as this call returns; the asynchronous H2D copy reads the staging buffer
  cudaError_t e = cudaSuccess;
  if (c->hstage_n < n) {
    for (int k = 0; k < 2; ++k) {
      if (c->hstage_ev[k]) cudaEventSynchronize(c->hstage_ev[k]);
      if (c->hstage[k]) cudaFreeHost(c->hstage[k]);
      c->hstage[k] = nullptr;
    }
    c->hstage_n = 0;
    for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
      e = cudaMallocHost((void**)&c->hstage[k], n * sizeof(float));
      if (e == cudaSuccess && !c->hstage_ev[k])
        e = cudaEventCreateWithFlags(&c->hstage_ev[k], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) { *err = fail(c, ES_ERR_OOM, "host staging: %s", cudaGetErrorString(e)); return nullptr; }
    c->hstage_n = n;
  }
  const int k = c->hstage_k;
  c->hstage_k ^= 1;
  if ((e = cudaEventSynchronize(c->hstage_ev[k])) != cudaSuccess) {   // its previous copy is done
    *err = fail(c, ES_ERR_CUDA, "staging event: %s", cudaGetErrorString(e));
    return nullptr;
  }
  std::memcpy(c->hstage[k], f, n * sizeof(float));
  e = cudaMemcpyAsync(*buf, c->hstage[k], n * sizeof(float), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaEventRecord(c->hstage_ev[k], st);
  if (e != cudaSuccess) { *err = fail(c, ES_ERR_CUDA, "H2D fitness: %s", cudaGetErrorString(e)); return nullptr; }
  return *buf;
}

static es_status_t weight_decay_impl(es_ctx* c, const float* fd, float* out, cudaStream_t st);

es_status_t es_tell(es_ctx_t* c, const float* fitness, es_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!c || !fitness) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (c->broken) return fail(c, ES_ERR_BAD_STATE, "context unusable after an NCCL error");
  if (!c->asked) return fail(c, ES_ERR_BAD_STATE, "es_tell without a preceding es_ask");
  const DevState& s = c->s;
  if ((s.W > 1 || (c->dW > 1 && (s.algo == SEP_CMA_ES || c->any_clipup || c->any_wd))) && !c->comm)
    return fail(c, ES_ERR_BAD_STATE, "no communicator: use es_tell_local / es_tell_apply "
                "(and es_sqnorm_partial / es_weight_decay_apply for weight decay)");
  const size_t nloc = (size_t)s.R * s.Nloc;
  es_status_t err;
  const float* fl = stage_fitness(c, fitness, nloc, st, &c->fstage, &err);
  if (!fl) return err;
  if (c->any_wd) {   // weight decay on this rank's slice before anything sees it
    if ((err = weight_decay_impl(c, fl, nullptr, st)) != ES_SUCCESS) return err;
    fl = c->wdbuf;
  }
  // the collective path: W > 1, or a one-rank communicator (c->pcoll)
  const bool coll = s.W > 1 || c->pcoll;
  const bool fused = !coll;
  const float* fsrc = fl;
  if (coll) {   // a5: every rank obtains all N fitness values
    ProfScope ps(c, "allgather", st);
    NCCL_OR(c, ncclAllGather(fl, c->fgather, nloc, ncclFloat, c->comm, st));
    fsrc = c->fgather;
  }
  if (s.W > 1 && c->nvls.stage == 2) {
    // f2 NVLS: barrier → in-switch reduce-scatter / update / multicast all-gather → barrier
    if ((err = tell_local_impl(c, fsrc, false, st)) != ES_SUCCESS) return err;
    if (!c->bar) CUDA_OR(c, dalloc(c, (void**)&c->bar, sizeof(int)));
    NCCL_OR(c, ncclAllReduce(c->bar, c->bar, 1, ncclInt32, ncclSum, c->comm, st));
    c->told_local = true;
    if ((err = es_tell_nvls_apply(c, stream_)) != ES_SUCCESS) return err;
    NCCL_OR(c, ncclAllReduce(c->bar, c->bar, 1, ncclInt32, ncclSum, c->comm, st));
    return ES_SUCCESS;
  }
  if (s.W > 1 && c->peers.W == s.W) {
    // f2: barrier → fused peer-memory reduce-scatter / update / all-gather → barrier
    if ((err = tell_local_impl(c, fsrc, false, st)) != ES_SUCCESS) return err;
    if (!c->bar) CUDA_OR(c, dalloc(c, (void**)&c->bar, sizeof(int)));
    NCCL_OR(c, ncclAllReduce(c->bar, c->bar, 1, ncclInt32, ncclSum, c->comm, st));
    c->told_local = true;
    if ((err = es_tell_p2p_apply(c, stream_)) != ES_SUCCESS) return err;
    NCCL_OR(c, ncclAllReduce(c->bar, c->bar, 1, ncclInt32, ncclSum, c->comm, st));
    for (int ph = p2p_phases(c); ph > 0; --ph) {   // Sep-CMA σ / C, ClipUp's two norms
      if ((err = es_tell_p2p_finish(c, stream_)) != ES_SUCCESS) return err;
      NCCL_OR(c, ncclAllReduce(c->bar, c->bar, 1, ncclInt32, ncclSum, c->comm, st));
    }
    return ES_SUCCESS;
  }
  if ((err = tell_local_impl(c, fsrc, fused, st)) != ES_SUCCESS) return err;
  if (coll && s.algo != CMA_ES) {   // a8 (P:226 pmean): sum the binary64 direction sums over ranks
    const size_t cnt = (size_t)(s.algo == OPENAI_ES || s.algo == ARS ? 1 : 2) * s.R * s.D;
    ProfScope ps(c, "allreduce", st);
    NCCL_OR(c, ncclAllReduce(s.G, s.G, cnt, ncclFloat64, ncclSum, c->comm, st));
  }
  if ((err = tell_apply_impl(c, fused, st)) != ES_SUCCESS) return err;
  c->asked = false;
  return ES_SUCCESS;
}

// out == nullptr: into c->wdbuf.
static es_status_t weight_decay_impl(es_ctx* c, const float* fd, float* out, cudaStream_t st) {
  const DevState& s = c->s;
  const size_t nloc = (size_t)s.R * s.Nloc;
  if (!c->aepart)
    CUDA_OR(c, dalloc(c, (void**)&c->aepart, nloc * ask_eval_blocks_per_run(s) * sizeof(double)));
  if (!out) {
    if (!c->wdbuf) CUDA_OR(c, dalloc(c, (void**)&c->wdbuf, nloc * sizeof(float)));
    out = c->wdbuf;
  }
  ProfScope ps(c, "weight_decay", st);
  if (s.dshard && c->dW > 1) {
    // ‖x_j‖² is a sum over every rank's dims: this rank's binary64 share, summed by NCCL (R·N
    // doubles, the same collective as the partial fitness), then f + wd·‖x‖²
    if (!c->wdn2) CUDA_OR(c, dalloc(c, (void**)&c->wdn2, nloc * sizeof(double)));
    CUDA_OR(c, launch_ask_eval_partial(s, (int)ES_FIT_SPHERE, nullptr, c->aepart, c->wdn2, st));
    NCCL_OR(c, ncclAllReduce(c->wdn2, c->wdn2, nloc, ncclFloat64, ncclSum, c->comm, st));
    CUDA_OR(c, launch_wd_apply(s, c->wdn2, fd, out, st));
    c->launches += 3;
    return ES_SUCCESS;
  }
  CUDA_OR(c, launch_weight_decay(s, c->aepart, fd, out, st));
  c->launches += 2;
  return ES_SUCCESS;
}

es_status_t es_weight_decay(es_ctx_t* c, const float* fitness, float* out, es_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!c || !fitness || !out) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (!c->asked) return fail(c, ES_ERR_BAD_STATE, "es_weight_decay needs an asked generation");
  if (c->s.algo == CMA_ES) return fail(c, ES_ERR_UNSUPPORTED, "CMA-ES: weight decay is not implemented");
  if (c->s.dshard && c->dW > 1 && !c->comm)
    return fail(c, ES_ERR_BAD_STATE, "D-shard without communicator: sum es_sqnorm_partial over "
                "the ranks and use es_weight_decay_apply");
  const size_t nloc = (size_t)c->s.R * c->s.Nloc;
  es_status_t err;
  const float* fd = stage_fitness(c, fitness, nloc, st, &c->fstage, &err);
  if (!fd) return err;
  const bool oh = !is_device_ptr(out);
  if ((err = weight_decay_impl(c, fd, oh ? nullptr : out, st)) != ES_SUCCESS) return err;
  if (oh) {
    CUDA_OR(c, cudaMemcpyAsync(out, c->wdbuf, nloc * sizeof(float), cudaMemcpyDeviceToHost, st));
    CUDA_OR(c, cudaStreamSynchronize(st));
  }
  return ES_SUCCESS;
}

es_status_t es_tell_local(es_ctx_t* c, const float* fitness_all, es_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!c || !fitness_all) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (!c->asked || c->told_local) return fail(c, ES_ERR_BAD_STATE, "es_tell_local out of order");
  es_status_t err;
  const float* fsrc = stage_fitness(c, fitness_all, (size_t)c->s.R * c->s.N, st, &c->fgather_stage, &err);
  if (!fsrc) return err;
  if (c->s.dshard) {
    // D-shard: every rank ranks the full fitness and updates its own dims in place; only
    // Sep-CMA-ES leaves a share (ES_FIELD_NORM2) for the caller to sum before es_tell_apply
    if ((err = tell_local_impl(c, fsrc, true, st)) != ES_SUCCESS) return err;
    if (c->s.algo == SEP_CMA_ES || c->any_clipup) {   // ‖p_σ'‖² / ‖g‖² share → ES_FIELD_NORM2
      CUDA_OR(c, launch_sepcma_n2(c->s, st));
      c->launches += 1;
    }
    c->apply_phase = 0;
  } else if ((err = tell_local_impl(c, fsrc, false, st)) != ES_SUCCESS) {
    return err;
  }
  c->told_local = true;
  return ES_SUCCESS;
}

static int tell_apply_phases(const es_ctx* c) {
  return c->s.dshard && c->dW > 1 && c->any_clipup ? 2 : 1;
}

int32_t es_tell_apply_phases(const es_ctx_t* c) { return c ? tell_apply_phases(c) : -1; }

es_status_t es_tell_apply(es_ctx_t* c, es_stream_t stream_) {
  if (!c) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (!c->told_local) return fail(c, ES_ERR_BAD_STATE, "es_tell_apply without es_tell_local");
  cudaStream_t st = (cudaStream_t)stream_;
  if (tell_apply_phases(c) == 2) {
    // D-shard ClipUp: phase 0 reads the summed ‖g‖² and leaves the ‖v'‖² share in NORM2;
    // phase 1 reads its sum and finishes the step
    int nk = 0;
    {
      ProfScope ps(c, "clipup_finish", st);
      CUDA_OR(c, launch_clipup_dshard_phase(c->s, c->apply_phase, st, &nk));
    }
    c->launches += nk;
    if (c->apply_phase == 0) {
      c->apply_phase = 1;
      return ES_SUCCESS;
    }
    c->apply_phase = 0;
  } else {
    es_status_t err = tell_apply_impl(c, c->s.dshard != 0, st, true);
    if (err != ES_SUCCESS) return err;
  }
  c->told_local = false;
  c->asked = false;
  return ES_SUCCESS;
}

es_status_t es_sqnorm_partial(es_ctx_t* c, double* out, es_stream_t stream_) {
  if (!c || !out) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (!c->asked) return fail(c, ES_ERR_BAD_STATE, "es_sqnorm_partial needs an asked generation");
  if (c->s.algo == CMA_ES) return fail(c, ES_ERR_UNSUPPORTED, "not for CMA-ES");
  if (!is_device_ptr(out)) return fail(c, ES_ERR_INVALID_ARG, "out must be device memory");
  const DevState& s = c->s;
  if (!c->aepart)
    CUDA_OR(c, dalloc(c, (void**)&c->aepart,
                      (size_t)s.R * s.Nloc * ask_eval_blocks_per_run(s) * sizeof(double)));
  ProfScope ps(c, "sqnorm_partial", (cudaStream_t)stream_);
  CUDA_OR(c, launch_ask_eval_partial(s, (int)ES_FIT_SPHERE, nullptr, c->aepart, out, (cudaStream_t)stream_));
  c->launches += 2;
  return ES_SUCCESS;
}

es_status_t es_weight_decay_apply(es_ctx_t* c, const float* f, const double* sqnorm, float* out,
                                  es_stream_t stream_) {
  if (!c || !f || !sqnorm || !out) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (!is_device_ptr(f) || !is_device_ptr(sqnorm) || !is_device_ptr(out))
    return fail(c, ES_ERR_INVALID_ARG, "f, sqnorm and out must be device memory");
  ProfScope ps(c, "weight_decay", (cudaStream_t)stream_);
  CUDA_OR(c, launch_wd_apply(c->s, sqnorm, f, out, (cudaStream_t)stream_));
  c->launches += 1;
  return ES_SUCCESS;
}

es_status_t es_shard_plan(int32_t N, int32_t entries, int32_t W, int32_t rank, int32_t out[4]) {
  if (!out || N < 1 || entries < 0 || W < 1 || rank < 0 || rank >= W || N % W)
    return fail(nullptr, ES_ERR_INVALID_ARG, "bad shard plan arguments");
  out[0] = rank * (N / W);
  out[1] = (rank + 1) * (N / W);
  int e0, e1;
  shard_range(entries, W, rank, e0, e1);
  out[2] = e0;
  out[3] = e1;
  return ES_SUCCESS;
}

static bool field_ok(const es_ctx* c, int f, void** base, size_t* elem, size_t* count, bool* scal,
                     size_t* off) {
  const DevState& s = c->s;
  *scal = false;
  *elem = 4;
  if (f >= 0 && f < NVEC) {
    *base = s.vec[f];
    *count = (size_t)s.R * s.D;
    return s.vec[f] != nullptr;
  }
  const size_t RN = (size_t)s.R * s.N;
  switch (f) {
    case ES_FIELD_BEST_F: *scal = true; *off = offsetof(RunScal, best_f); return true;
    case ES_FIELD_SIGMA: *scal = true; *off = offsetof(RunScal, sigma); return !(s.algo == PGPE || s.algo == SNES);
    case ES_FIELD_LRATE: *scal = true; *off = offsetof(RunScal, lr); return antithetic(s.algo);
    case ES_FIELD_GEN: *scal = true; *off = offsetof(RunScal, t); return true;
    case ES_FIELD_SHAPED: *base = s.shaped; *count = RN; return true;
    case ES_FIELD_RANK_S: *base = s.rs_s; *count = RN; return true;
    case ES_FIELD_RANK_E: *base = s.rs_e; *count = RN; return true;
    case ES_FIELD_PERM: *base = s.perm; *count = RN; return true;
    case ES_FIELD_FITNESS: *base = s.fit; *count = RN; return true;
    case ES_FIELD_DIRSUM: *base = s.G; *count = 2 * (size_t)s.R * s.D; *elem = 8; return true;
    case ES_FIELD_NORM2: *base = s.n2; *count = (size_t)s.R; *elem = 8; return s.algo == SEP_CMA_ES || c->any_clipup;
    case ES_FIELD_COV: *base = s.cov; *count = (size_t)s.R * s.D * s.D; return s.cov != nullptr;
    case ES_FIELD_CHOL: *base = s.chol; *count = (size_t)s.R * s.D * s.D; return s.chol != nullptr;
  }
  return false;
}

es_status_t es_get(es_ctx_t* c, es_field_t field, void* dst, es_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!c || !dst) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  void* base = nullptr;
  size_t elem, count = 0, off = 0;
  bool scal;
  if (!field_ok(c, field, &base, &elem, &count, &scal, &off))
    return fail(c, ES_ERR_INVALID_ARG, "field %d not kept by this algorithm", field);
  if (scal)
    CUDA_OR(c, cudaMemcpy2DAsync(dst, 4, (char*)c->s.rs + off, sizeof(RunScal), 4, c->s.R,
                                 cudaMemcpyDefault, st));
  else
    CUDA_OR(c, cudaMemcpyAsync(dst, base, count * elem, cudaMemcpyDefault, st));
  if (!is_device_ptr(dst)) CUDA_OR(c, cudaStreamSynchronize(st));
  return ES_SUCCESS;
}

es_status_t es_set(es_ctx_t* c, es_field_t field, const void* src, es_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!c || !src) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (field >= ES_FIELD_SHAPED && field != ES_FIELD_DIRSUM && field != ES_FIELD_NORM2 &&
      field != ES_FIELD_COV && field != ES_FIELD_CHOL)
    return fail(c, ES_ERR_INVALID_ARG, "field %d is read-only", field);
  void* base = nullptr;
  size_t elem, count = 0, off = 0;
  bool scal;
  if (!field_ok(c, field, &base, &elem, &count, &scal, &off))
    return fail(c, ES_ERR_INVALID_ARG, "field %d not kept by this algorithm", field);
  if (scal)
    CUDA_OR(c, cudaMemcpy2DAsync((char*)c->s.rs + off, sizeof(RunScal), src, 4, 4, c->s.R,
                                 cudaMemcpyDefault, st));
  else
    CUDA_OR(c, cudaMemcpyAsync(base, src, count * elem, cudaMemcpyDefault, st));
  if (field == ES_FIELD_GEN) {
    // Adam's β^t products are a pure function of t (t exact double multiplications, N12): rebuild
    // them so that a resumed run continues bit-identically.
    std::vector<uint32_t> t(c->s.R);
    CUDA_OR(c, cudaStreamSynchronize(st));
    CUDA_OR(c, cudaMemcpy(t.data(), src, c->s.R * sizeof(uint32_t), cudaMemcpyDefault));
    c->host_t = t;                                 // CMA-ES refresh schedule follows t
    std::vector<double> p(2 * (size_t)c->s.R);
    for (int r = 0; r < c->s.R; ++r) {
      double b1 = 1.0, b2 = 1.0;
      for (uint32_t k = 0; k < t[r]; ++k) {
        b1 = b1 * (double)c->host_rs[r].beta1;
        b2 = b2 * (double)c->host_rs[r].beta2;
      }
      p[2 * r] = b1;
      p[2 * r + 1] = b2;
    }
    CUDA_OR(c, cudaMemcpy2DAsync((char*)c->s.rs + offsetof(RunScal, b1pow), sizeof(RunScal),
                                 p.data(), 16, 16, c->s.R, cudaMemcpyHostToDevice, st));
  }
  CUDA_OR(c, cudaStreamSynchronize(st));
  return ES_SUCCESS;
}

es_status_t es_debug_check_guards(es_ctx_t* c, int64_t* bad_bytes) {
  if (!c || !bad_bytes) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (!c->guard) return fail(c, ES_ERR_BAD_STATE, "context not created with ES_GUARD_ALLOCS=1");
  CUDA_OR(c, cudaDeviceSynchronize());
  std::vector<unsigned char> h(kGuard);
  int64_t bad = 0;
  for (const auto& z : c->zones) {
    CUDA_OR(c, cudaMemcpy(h.data(), z.p, z.bytes, cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < z.bytes; ++k) bad += h[k] != 0xA5;
  }
  *bad_bytes = bad;
  return ES_SUCCESS;
}

es_status_t es_profile_enable(es_ctx_t* c, int32_t on) {
  if (!c) return fail(nullptr, ES_ERR_INVALID_ARG, "NULL context");
  c->profiling = on != 0;
  return ES_SUCCESS;
}

int32_t es_profile_read(es_ctx_t* c, char* names, double* ms, int64_t* counts, int32_t max_k) {
  if (!c || !names || !ms || !counts || max_k < 1) return -1;
  std::vector<std::string> kinds;
  std::vector<double> tot;
  std::vector<int64_t> cnt;
  for (auto& r : c->recs) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return -1;
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    size_t k = 0;
    while (k < kinds.size() && kinds[k] != r.name) ++k;
    if (k == kinds.size()) { kinds.push_back(r.name); tot.push_back(0.0); cnt.push_back(0); }
    tot[k] += t;
    cnt[k] += 1;
    c->pool.push_back(r.a);
    c->pool.push_back(r.b);
  }
  c->recs.clear();
  const int n = std::min<int>((int)kinds.size(), max_k);
  for (int k = 0; k < n; ++k) {
    std::memset(names + 32 * k, 0, 32);
    std::strncpy(names + 32 * k, kinds[k].c_str(), 31);
    ms[k] = tot[k];
    counts[k] = cnt[k];
  }
  return n;
}

es_status_t es_debug_primitive(int32_t which, const void* in, void* out, int64_t n,
                               es_stream_t stream_) {
  if (which < 0 || which > 7 || n < 0) return fail(nullptr, ES_ERR_INVALID_ARG, "bad which/n");
  if (n > 0 && (!in || !out)) return fail(nullptr, ES_ERR_INVALID_ARG, "NULL argument");
  CUDA_OR(nullptr, launch_primitive(which, in, out, n, (cudaStream_t)stream_));
  return ES_SUCCESS;
}

int64_t es_mlp_num_params(const int32_t* widths, int32_t nw) {
  if (!widths || nw < 2) return -1;
  int64_t n = 0;
  for (int l = 0; l + 1 < nw; ++l) {
    if (widths[l] < 1 || widths[l + 1] < 1) return -1;
    n += (int64_t)widths[l] * widths[l + 1] + widths[l + 1];
  }
  return n;
}

es_status_t es_set_mlp_problem(es_ctx_t* c, const int32_t* widths, int32_t nw, int32_t batch,
                               uint64_t seed, es_stream_t stream_) {
  if (!c || !widths) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (nw < 2 || nw > 16) return fail(c, ES_ERR_INVALID_ARG, "need 2..16 layer widths");
  std::string err;
  void* p = mlp_problem_create(widths, nw, batch, seed, (cudaStream_t)stream_, &err);
  if (!p) return fail(c, err.rfind("unsupported", 0) == 0 ? ES_ERR_UNSUPPORTED : ES_ERR_INVALID_ARG,
                      "%s", err.c_str());
  // the fp32-accurate kernel's per-member scratch for a whole population, so that generations
  // can be graph-captured (the scratch only grows outside capture, for larger es_eval_bbob calls)
  if (cudaError_t e = mlp_problem_reserve(p, (int64_t)c->s.R * c->s.Nloc, (cudaStream_t)stream_)) {
    mlp_problem_destroy(p);
    return fail(c, ES_ERR_CUDA, "MLP scratch: %s", cudaGetErrorString(e));
  }
  if (c->mlp) mlp_problem_destroy(c->mlp);
  c->mlp = p;
  return ES_SUCCESS;
}

}  // extern "C"
