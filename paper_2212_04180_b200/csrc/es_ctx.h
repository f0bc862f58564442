// es_ctx.h — the host-side context behind the C ABI (es_api.cu, es_api_peer.cu): es_ctx, the
// status / error plumbing (fail, CUDA_OR, NCCL_OR), device allocation with the optional guard
// zones, the NVTX + event profiling scope, and the peer-memory tell's support predicates.
#pragma once
#include <nvtx3/nvToolsExt.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/es.h"
#include "es_internal.h"

namespace esb {
cudaError_t launch_mlp_eval(void* prob, const float* x, int64_t n, float* f, cudaStream_t st);
cudaError_t launch_mlp_eval_f16(void* prob, const float* x, int64_t n, float* f, cudaStream_t st);
cudaError_t mlp_problem_reserve(void* prob, int64_t n, cudaStream_t st);
__half* mlp_problem_image(void* prob, int64_t n, cudaStream_t st);
cudaError_t launch_mlp_eval_img(void* prob, int64_t n, float* f, cudaStream_t st);
cudaError_t launch_ask_split(const DevState& s, float* x, __half* img, cudaStream_t st);
inline bool is_mlp(int fn) { return fn == ES_FIT_MLP || fn == ES_FIT_MLP16; }
void* mlp_problem_create(const int32_t* widths, int32_t nw, int32_t batch, uint64_t seed,
                         cudaStream_t st, std::string* err);
void mlp_problem_destroy(void* prob);
int64_t mlp_problem_dims(const void* prob);
cudaError_t launch_primitive(int which, const void* in, void* out, int64_t n, cudaStream_t st);
cudaError_t launch_ask_eval(const DevState& s, int fn, float* x, double* part, float* f,
                            cudaStream_t st);
cudaError_t launch_ask16(const DevState& s, float* x, __half* x16, cudaStream_t st);
cudaError_t launch_mlp_eval16(void* prob, const __half* x16, int64_t n, float* f,
                              cudaStream_t st);
int ask_eval_blocks_per_run(const DevState& s);
}  // namespace esb

using namespace esb;

struct es_ctx {
  DevState s{};
  std::vector<RunScal> host_rs;
  PeerTable peers{};            // f2 peer-memory tell (peers.W = 0: not set)
  NvlsHost nvls;                // f2 NVLS multicast tell (stage 2: bound)
  std::vector<void*> ipc_open;  // peer mappings opened by es_p2p_ipc_open
  int* bar = nullptr;           // 4-byte NCCL barrier word
  int dW = 1, drank = 0;        // D-shard world (f1); population world is s.W
  std::vector<uint32_t> host_t; // completed tells per run (CMA-ES Cholesky refresh schedule)
  bool graph_seen = false;      // a tell was stream-captured: always launch the refresh kernels
  int64_t d0 = 0;               // first owned global dim
  double* fpart = nullptr;      // [R][N] D-shard binary64 partial fitness
  bool any_clipup = false;
  bool any_wd = false;
  float* wdbuf = nullptr;       // [R][Nloc] weight-decayed fitness
  ncclComm_t comm = nullptr;
  bool asked = false;
  bool told_local = false;
  int apply_phase = 0;          // D-shard ClipUp: next es_tell_apply phase (0 or 1)
  double* wdn2 = nullptr;       // [R][N] D-shard squared norms (weight decay)
  int p2p_phase = -1;           // next es_tell_p2p_finish phase (-1: no apply pending)
  bool broken = false;
  TellSplit split{1, 1};
  float* fgather = nullptr;     // [W][R][Nloc]
  bool pcoll = false;           // population-sharded with a communicator (also W = 1)
  float* fstage = nullptr;      // [R][Nloc] staging of host fitness
  float* fgather_stage = nullptr;  // [W][R][Nloc] staging of host gathered fitness (split phase)
  // host inputs are first copied (CPU memcpy) into one of two pinned host buffers, so the
  // caller may reuse its buffer as soon as the call returns; an event per buffer guards its reuse
  float* hstage[2] = {nullptr, nullptr};
  size_t hstage_n = 0;
  cudaEvent_t hstage_ev[2] = {nullptr, nullptr};
  int hstage_k = 0;
  float* xstage = nullptr;      // [R][Nloc][D] staging of a host population
  double* aepart = nullptr;     // [R][Nloc][blocks] fused ask+eval partial sums
  __half* x16 = nullptr;        // [R][Nloc][D] fp16 parameter image (MLP fused path, N14′)
  void* mlp = nullptr;
  int64_t launches = 0;
  bool profiling = false;
  struct Rec { const char* name; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  std::vector<void*> allocs;     // cudaMalloc bases
  bool guard = false;            // ES_GUARD_ALLOCS=1: 256-B 0xA5 zones around every allocation
  struct Zone { const unsigned char* p; size_t bytes; };
  std::vector<Zone> zones;
  std::string err;
};

extern thread_local std::string g_err;   // defined in es_api.cu

inline es_status_t fail(es_ctx* c, es_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  g_err = buf;
  return st;
}

#define CUDA_OR(c, expr)                                                                     \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess)                                                                  \
      return fail((c), _e == cudaErrorMemoryAllocation ? ES_ERR_OOM : ES_ERR_CUDA, "%s: %s", \
                  #expr, cudaGetErrorString(_e));                                           \
  } while (0)

#define NCCL_OR(c, expr)                                                                \
  do {                                                                                 \
    ncclResult_t _r = (expr);                                                          \
    if (_r != ncclSuccess) {                                                           \
      if (c) (c)->broken = true;                                                       \
      return fail((c), ES_ERR_NCCL, "%s: %s", #expr, ncclGetErrorString(_r));           \
    }                                                                                  \
  } while (0)

inline constexpr size_t kGuard = 256;   // keeps the 256-B alignment of the returned pointer

inline cudaError_t dalloc(es_ctx* c, void** p, size_t bytes) {
  bytes = std::max<size_t>(bytes, 256);
  if (!c->guard) {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaSuccess) c->allocs.push_back(*p);
    return e;
  }
  bytes = (bytes + kGuard - 1) / kGuard * kGuard;
  unsigned char* base = nullptr;
  cudaError_t e = cudaMalloc((void**)&base, bytes + 2 * kGuard);
  if (e != cudaSuccess) return e;
  c->allocs.push_back(base);
  if ((e = cudaMemset(base, 0xA5, kGuard)) != cudaSuccess) return e;
  if ((e = cudaMemset(base + kGuard + bytes, 0xA5, kGuard)) != cudaSuccess) return e;
  c->zones.push_back({base, kGuard});
  c->zones.push_back({base + kGuard + bytes, kGuard});
  *p = base + kGuard;
  return cudaSuccess;
}

// Profiling brackets: an NVTX range around each launch group (host side, for nsys / ncu --nvtx;
// header-only NVTX 3 — a no-op branch when no tool is attached) and, when profiling is enabled
// (bench), an event pair on the launching stream.
inline cudaEvent_t prof_event(es_ctx* c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
struct ProfScope {
  es_ctx* c;
  cudaStream_t st;
  size_t idx = (size_t)-1;
  ProfScope(es_ctx* c_, const char* name, cudaStream_t st_) : c(c_), st(st_) {
    nvtxRangePushA(name);
    if (c && c->profiling) {
      es_ctx::Rec r{name, prof_event(c), prof_event(c)};
      cudaEventRecord(r.a, st);
      c->recs.push_back(r);
      idx = c->recs.size() - 1;
    }
  }
  ~ProfScope() {
    if (idx != (size_t)-1) cudaEventRecord(c->recs[idx].b, st);
    nvtxRangePop();
  }
};

inline bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}


// f2 peer-memory tell: supported contexts, and the es_tell_p2p_finish calls (each after a
// barrier) one generation needs.
inline bool p2p_algo_ok(const es_ctx* c) {
  const int a = c->s.algo;
  return (a == OPENAI_ES || a == PGPE || a == SNES || a == ARS || a == SEP_CMA_ES) && !c->s.dshard;
}

inline int p2p_phases(const es_ctx* c) {
  return c->s.algo == SEP_CMA_ES ? 1 : (c->any_clipup ? 2 : 0);
}
