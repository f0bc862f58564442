// es_internal.h — device data layout and kernel entry points of libes_b200 (not part of the ABI).
//
// HBM layout (per context, all dense, 256-B aligned allocations):
//   vec[f]      float [R][D] for each state field f the algorithm keeps (mean, σ_d, Adam m/v,
//               p_σ, p_c, C, best_x) — structure-of-arrays so that every kernel streams float4.
//   rs          RunScal [R]   per-run scalars + hyperparameters (device-resident, so a captured
//               CUDA graph of a generation replays with no host round trip).
//   gs          GenScal [R]   this generation's scalars, written by the rank kernel.
//   wpos        float [R][N]  position weights w_p (SNES / Sep-CMA, N11).
//   shaped/s/e/perm [R][N]    ranking results of the last tell (N9–N11).
//   dir, coefA, coefB [R][N]  per-entry tell coefficients: direction index and its weights.
//   Gpart       double [R][2][D] (+ chunk partials) reduction workspace.
#pragma once
#include <atomic>
#include <cuda_runtime.h>

#include <cuda.h>

#include <cstdint>
#include <vector>

namespace esb {

enum Algo : int { OPENAI_ES = 0, PGPE = 1, SNES = 2, SEP_CMA_ES = 3, ARS = 4, CMA_ES = 5 };
static constexpr int64_t kCmaMaxDims = 4096;   // full CMA-ES: C is D×D per run (f4)
enum Optim : int { OPT_ADAM = 0, OPT_SGD = 1, OPT_CLIPUP = 2 };
__host__ __device__ constexpr bool is_anti(int a) { return a == OPENAI_ES || a == PGPE || a == ARS; }
enum Field : int {
  F_MEAN = 0, F_SIGMA_D = 1, F_ADAM_M = 2, F_ADAM_V = 3, F_PSIGMA = 4, F_PC = 5, F_C = 6,
  F_BEST_X = 7, NVEC = 8
};

struct alignas(16) RunScal {
  uint64_t seed;
  uint32_t t;
  int32_t mu;
  float lr, sigma, best_f;
  int32_t shaping;
  double b1pow, b2pow;
  float init_min, init_max, sigma_init, sigma_decay, sigma_limit, lrate_decay, lrate_limit;
  float beta1, beta2, eps, sigma_lrate, sigma_max_change;
  double c_sigma, d_sigma, c_c, c_1, c_mu, chi_d, mueff, eta_sigma;
  int32_t optimizer, ars_k;      // ars_k: elite pairs k of ARS / PGPE (P when every pair is kept)
  float momentum, max_speed;
  float weight_decay, clip_lo, clip_hi;
  int32_t clip;                   // clip_lo or clip_hi finite
  int32_t k_refresh;              // CMA-ES: Cholesky factor refreshed after every k-th tell
};

struct alignas(16) GenScal {
  uint32_t t;          // generation being told (pre-increment)
  int32_t jbest;       // member at sorted position 0
  int32_t improved;    // f[jbest] < best_f before this tell
  int32_t nentries;    // coefficient entries carrying weight (P, or Sep-CMA's weighted positions)
  float lr, sigma;     // pre-decay learning rate and scalar σ
  float bc1, bc2;      // Adam bias corrections 1 − β^{t+1}
  double bbar;         // PGPE baseline
  float sigma_new;     // Sep-CMA σ' (written by the norm kernel)
  int32_t hsig;        // Sep-CMA h_σ
  float ars_scale;     // ARS: α / (k·σ_R), or 0 when σ_R = 0
  float clip_inv;      // ClipUp: 1/‖g‖ (0 if ‖g‖ = 0), then the velocity clip factor
};

struct DevState {
  int algo, R, N, Nloc, W, rank;
  int any_clip;        // some run has box bounds (selects the clipping ask instances)
  int64_t D, Q;        // state dims of this context (incl. a D-shard's halo dim), Q = ceil(D/4)
  int64_t Dx, Qx;      // member row length written to x (= D unless D-sharded), Qx = ceil(Dx/4)
  int64_t q0;          // global quad of local dim 0 (D-shard: d_begin/4) — the noise counter
  int64_t Dg;          // global problem dimension (constants, Sep-CMA h_σ)
  int dshard;          // dimension-sharded context (f1): fitness partials are summed over ranks
  int P;               // global directions
  float* vec[NVEC];
  RunScal* rs;
  GenScal* gs;
  float* wpos;
  float* fit;          // [R][N] gathered fitness, run-major
  float* shaped;
  int32_t* rs_s;
  int32_t* rs_e;
  int32_t* perm;
  uint32_t* dir;       // [R][N]
  double* coefA;       // [R][N]
  double* coefB;       // [R][N]
  double* G;           // [2][R][D] reduced sums (W>1 path, and Sep-CMA Z/Q)
  double* Gchunk;      // [nchunk][R][2][D] partials when the direction range is split
  uint32_t* arrive;    // [R][blocks_per_run] last-block counters
  double* normpart;    // [R][blocks_per_run] Sep-CMA ‖p_σ‖² partials
  uint64_t* gkeys;     // [R][npad] sort keys in global memory (N > 16384 only)
  uint32_t* rcnt;      // counting rank (few runs): [3][R][N] counters + arrivals + slots, zero
                      // between tells (k_rank.cu)
  double* rbpart;     // [R][64] counting rank: PGPE baseline partials per j-tile
  unsigned* rrad_bar; // radix rank: grid-barrier counters [2] (zero between launches)
  uint32_t* rrad;     // radix rank (few runs, 4096 < N ≤ 65536): keys / indices ping-pong [4][R][N] + digit totals [R][256][32]
  int rank_par;       // every run's shaping is per-member in the ranks (counting rank allowed)
  int32_t* pos;        // [R][N] member → sorted position (ARS pair selection)
  double* n2;          // [R] D-shard Sep-CMA ‖p_σ'‖² share, summed over ranks before the finish
  // full-covariance CMA-ES (f4)
  float* cov;          // [R][D][D] C, symmetric (both triangles stored)
  float* chol;         // [R][D][D] A = chol(C) as of the last refresh, lower (upper = 0)
  float* cw;           // [R][D][D] factorisation workspace
  float* zbuf;         // [R][N][D] this generation's z
  float* ybuf;         // [R][N][D] y = A z
  int32_t* chol_fail;  // [R] the last refresh failed (A kept)
  float* ut;           // [R][D][kp] w_e·y_e transposed (tensor-core covariance update operand)
  float* vt;           // [R][D][kp] y_e transposed
  int kp;              // entry capacity of ut / vt (N rounded up to 32)
};

// full CMA-ES helpers shared by k_cma.cu and k_cma_syrk.cu
// the Cholesky factor is refreshed after this tell (rs.t already counts it)
__device__ __forceinline__ bool chol_due_rs(const RunScal& rs) {
  return rs.k_refresh > 0 && (rs.t % (uint32_t)rs.k_refresh) == 0u;
}
// lower tile index t → (I, J), I ≥ J
__device__ __forceinline__ void lower_tile(int t, int& I, int& J) {
  I = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
  while ((I + 1) * (I + 2) / 2 <= t) ++I;
  while (I * (I + 1) / 2 > t) --I;
  J = t - I * (I + 1) / 2;
}

// f2 peer-memory tell: every rank's direction-sum buffer and state fields, as device pointers
// valid in this process (peer mappings over NVLink, or plain pointers for ranks emulated on one GPU).
static constexpr int kMaxPeers = 8;
struct PeerTable {
  int W;
  const double* G[kMaxPeers];
  float* vec[kMaxPeers][NVEC];
  const double* n2[kMaxPeers];      // Sep-CMA-ES ‖p_σ'‖² share of each rank's slice
};

// f2 NVLS variant: one symmetric buffer per rank bound to a multicast object.
struct NvlsHost {
  CUdevice dev = 0;
  size_t gran = 0, bytes = 0, used = 0;
  size_t off_g = 0, off_mean = 0, off_best = 0, off_sig = (size_t)-1;
  CUmemGenericAllocationHandle phys = 0, mc = 0;
  CUdeviceptr uva = 0, mcva = 0;
  bool have_mc = false, have_phys = false;
  int stage = 0;                      // 1 opened (device added, memory mapped), 2 bound
};
struct NvlsView {                     // multicast addresses of the symmetric fields
  const double* G;
  float* mean;
  float* best;
  float* sig;                         // nullptr if σ_d is not kept
};
const char* nvls_open(const DevState& s, NvlsHost& h, void* handle, bool creator);
const char* nvls_bind(NvlsHost& h);
void nvls_close(NvlsHost& h);

// Population sharding: rank's contiguous share [e0, e1) of ne tell entries. Shared by the
// tell kernel and es_shard_plan so that host plan and device split cannot disagree.
__host__ __device__ __forceinline__ void shard_range(int ne, int W, int rank, int& e0, int& e1) {
  const int per = (ne + W - 1) / W;
  e0 = rank * per < ne ? rank * per : ne;
  e1 = e0 + per < ne ? e0 + per : ne;
}

// Launch helpers (return cudaGetLastError()).
cudaError_t launch_init(const DevState& s, cudaStream_t st);
cudaError_t launch_ask(const DevState& s, float* x, cudaStream_t st);
cudaError_t launch_eval_bbob(int fn, const float* x, int64_t n, int64_t D, float* f,
                             cudaStream_t st);
cudaError_t launch_rank(const DevState& s, const float* fsrc, cudaStream_t st);
int rank_launches(const DevState& s);
cudaError_t launch_synth(const DevState& s, float* f, cudaStream_t st);
// Tell: regenerate-and-reduce over this rank's entries. fused=true (W == 1) applies the update in
// the same kernel; otherwise the sums land in s.G for the all-reduce and launch_tell_update
// applies them. Sep-CMA-ES additionally needs launch_sepcma_finish (global ‖p_σ‖, σ, h_σ, p_c, C).
// Each returns the number of kernels it launched through *nk.
// grid.y = nchunk; run r's entries are cut into chunks of echunk (see tell_kernel)
// The tell grid: x = quad block of a run, y = work item (run, entry chunk, the run's chunk count)
// from a host-built table — runs with few entries get few items, so no CTA starts only to exit and
// no CTA divides blockIdx to find its run. echunk entries per chunk (the last chunk of a run also
// takes any tie-extended entries, Sep-CMA-ES N11).
struct TellSplit {
  int nchunk, echunk;    // largest chunk count of a run, entries per chunk
  int nitems = 0;        // work items (grid.y)
  const int4* items = nullptr;   // device [nitems] (run, chunk, chunks of the run, 0)
};
std::vector<int4> tell_items(int R, const std::vector<int>& ent, const TellSplit& sp);
cudaError_t launch_tell_reduce(const DevState& s, bool fused, TellSplit sp, cudaStream_t st);
cudaError_t launch_tell_update(const DevState& s, cudaStream_t st);
cudaError_t launch_sepcma_finish(const DevState& s, cudaStream_t st, int* nk);
cudaError_t launch_sepcma_n2(const DevState& s, cudaStream_t st);
cudaError_t launch_sepcma_norm(const DevState& s, cudaStream_t st);   // σ', h_σ only
// D-shard: per-member binary64 partial fitness of the owned dims (fused ask + evaluate), and the
// conversion of the rank-summed partials to fp32 fitness
cudaError_t launch_ask_eval_partial(const DevState& s, int fn, float* x, double* part,
                                    double* fpart, cudaStream_t st);
cudaError_t launch_partial_to_fitness(const double* fsum, int64_t n, float* f, cudaStream_t st);
cudaError_t launch_clipup_finish(const DevState& s, cudaStream_t st, int* nk);
// ClipUp phase 0 / 1 of a D-sharded context from the summed norms in s.n2 (k_tell.cu)
cudaError_t launch_clipup_dshard_phase(const DevState& s, int phase, cudaStream_t st, int* nk);
// weight decay from per-member squared norms summed over the D-shard ranks (k_ask_eval.cu)
cudaError_t launch_wd_apply(const DevState& s, const double* sqnorm, const float* f, float* out,
                            cudaStream_t st);
// f2: reduce-scatter (peer loads, rank order) → update of this rank's quad slice → all-gather
// (peer stores) in one kernel
cudaError_t launch_p2p_apply(const DevState& s, const PeerTable& pt, bool clipup, cudaStream_t st,
                             int* nk);
// the phases after a barrier each: Sep-CMA-ES one (σ, p_c, C), ClipUp two (‖g‖, ‖v'‖)
cudaError_t launch_p2p_finish(const DevState& s, const PeerTable& pt, int phase, cudaStream_t st,
                              int* nk);
// f2 NVLS: the same with multimem.ld_reduce (sum in the switch) and multimem.st (broadcast)
cudaError_t launch_nvls_apply(const DevState& s, const NvlsView& v, cudaStream_t st);
// f_out = f + weight_decay_r ‖x_j‖² for this rank's members (2 kernels; part as ask_eval's)
cudaError_t launch_weight_decay(const DevState& s, double* part, const float* f, float* out,
                                cudaStream_t st);
int tell_blocks_per_run(const DevState& s);
// CMA-ES (k_cma.cu)
cudaError_t launch_cma_init(const DevState& s, cudaStream_t st);
cudaError_t launch_cma_ask(const DevState& s, float* x, cudaStream_t st, int* nk);
cudaError_t launch_cma_tell(const DevState& s, bool refresh, cudaStream_t st, int* nk);
// the sampling contraction on tcgen05 (kind::tf32, 3-pass split); needs D % 4 == 0
bool cma_tc_supported(const DevState& s);
bool syrk_tc_supported(const DevState& s);
cudaError_t launch_chol_update_tc(const DevState& s, int kb, cudaStream_t st);
cudaError_t launch_cma_cov_tc(const DevState& s, cudaStream_t st);
cudaError_t launch_cma_sample_tc(const DevState& s, float* x, cudaStream_t st);
// ent[r]: expected tell entries of run r on this rank
TellSplit tell_pick_split(const DevState& s, const std::vector<int>& ent);
constexpr int kTellThreads = 128;
int sm_count();   // of the current device

// Programmatic dependent launch (PDL) for the generation's short kernels (ask → evaluate → rank →
// tell → finish): each is launched with programmatic stream serialization, so its CTAs are
// scheduled while its predecessor drains; its first statement waits for the predecessor grid's
// completion and memory flush (griddepcontrol.wait, a no-op without the attribute), then lets
// its own successor launch. Nothing is read or written before the wait, so stream order holds.
// ES_PDL=0 launches them plainly (A/B switch).
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_on();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Opt a kernel into `bytes` of dynamic shared memory once per device (the attribute is per device:
// a process driving several GPUs sets it on each). `done` is the call site's device bitmask.
inline cudaError_t smem_attr_once(const void* kernel, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = dev < 64 ? (1ull << dev) : 0ull;
  if (bit && (done.load(std::memory_order_relaxed) & bit)) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_relaxed);
  return e;
}

}  // namespace esb
