// es_api_peer.cu — the C ABI of the f2 fused peer-memory tell (include/es.h):
// peer pointer tables, CUDA IPC export / open, the NVLS multicast binding and the apply / finish
// launches. The collective-free data path itself is in k_tell.cu (p2p_*, nvls_apply_kernel) and
// the multicast object lifecycle in k_nvls.cu.
#include <cstring>

#include "es_ctx.h"

extern "C" {

static constexpr int kIpcHandles = 10;   // dirsum, the 8 fields, norm2

es_status_t es_p2p_export(const es_ctx_t* c, es_peer_t* out) {
  if (!c || !out) return fail(nullptr, ES_ERR_INVALID_ARG, "NULL argument");
  out->dirsum = c->s.G;
  for (int f = 0; f < 8; ++f) out->field[f] = c->s.vec[f];
  out->norm2 = c->s.n2;
  return ES_SUCCESS;
}

es_status_t es_p2p_set_peers(es_ctx_t* c, const es_peer_t* peers, int32_t W) {
  if (!c || !peers) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (W != c->s.W) return fail(c, ES_ERR_INVALID_ARG, "peers for %d ranks, context has %d", W, c->s.W);
  if (W > kMaxPeers) return fail(c, ES_ERR_UNSUPPORTED, "more than %d peers", kMaxPeers);
  if (!p2p_algo_ok(c)) return fail(c, ES_ERR_UNSUPPORTED, "peer-memory tell: not with CMA-ES / D-sharding");
  PeerTable pt{};
  pt.W = W;
  for (int v = 0; v < W; ++v) {
    if (!peers[v].dirsum) return fail(c, ES_ERR_INVALID_ARG, "peer %d: NULL dirsum", v);
    pt.G[v] = peers[v].dirsum;
    pt.n2[v] = peers[v].norm2;
    if (p2p_phases(c) && !pt.n2[v]) return fail(c, ES_ERR_INVALID_ARG, "peer %d: NULL norm2", v);
    for (int f = 0; f < NVEC; ++f) {
      pt.vec[v][f] = peers[v].field[f];
      if (c->s.vec[f] && (f == F_MEAN || f == F_BEST_X || f == F_SIGMA_D || f == F_C) && !pt.vec[v][f])
        return fail(c, ES_ERR_INVALID_ARG, "peer %d: field %d missing", v, f);
    }
  }
  c->peers = pt;
  return ES_SUCCESS;
}

es_status_t es_tell_p2p_apply(es_ctx_t* c, es_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!c) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (!c->told_local) return fail(c, ES_ERR_BAD_STATE, "es_tell_p2p_apply without es_tell_local");
  if (c->peers.W != c->s.W) return fail(c, ES_ERR_BAD_STATE, "es_p2p_set_peers was not called");
  int nk = 0;
  {
    ProfScope ps(c, "p2p_apply", st);
    CUDA_OR(c, launch_p2p_apply(c->s, c->peers, c->any_clipup, st, &nk));
  }
  c->launches += nk;
  c->told_local = false;
  c->asked = false;
  c->p2p_phase = p2p_phases(c) ? 0 : -1;
  return ES_SUCCESS;
}

es_status_t es_nvls_open(es_ctx_t* c, void* handle, int32_t creator) {
  if (!c || !handle) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (!p2p_algo_ok(c) || c->s.algo == SEP_CMA_ES || c->any_clipup)
    return fail(c, ES_ERR_UNSUPPORTED, "NVLS tell: OpenAI-ES/PGPE/SNES/ARS, Adam/SGD");
  if (c->nvls.stage) return fail(c, ES_ERR_BAD_STATE, "es_nvls_open called twice");
  if (const char* e = nvls_open(c->s, c->nvls, handle, creator != 0)) {
    nvls_close(c->nvls);
    return fail(c, ES_ERR_UNSUPPORTED, "NVLS: %s", e);
  }
  return ES_SUCCESS;
}

es_status_t es_nvls_bind(es_ctx_t* c) {
  if (!c) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (const char* e = nvls_bind(c->nvls)) return fail(c, ES_ERR_BAD_STATE, "NVLS: %s", e);
  // move the symmetric fields into the bound buffer (unicast alias) and repoint the state
  DevState& s = c->s;
  const size_t RD = (size_t)s.R * s.D;
  char* base = reinterpret_cast<char*>(c->nvls.uva);
  double* G = reinterpret_cast<double*>(base + c->nvls.off_g);
  CUDA_OR(c, cudaMemcpy(G, s.G, 2 * RD * sizeof(double), cudaMemcpyDeviceToDevice));
  s.G = G;
  const int f[3] = {F_MEAN, F_BEST_X, F_SIGMA_D};
  const size_t off[3] = {c->nvls.off_mean, c->nvls.off_best, c->nvls.off_sig};
  for (int i = 0; i < 3; ++i) {
    if (!s.vec[f[i]]) continue;
    float* dst = reinterpret_cast<float*>(base + off[i]);
    CUDA_OR(c, cudaMemcpy(dst, s.vec[f[i]], RD * sizeof(float), cudaMemcpyDeviceToDevice));
    s.vec[f[i]] = dst;
  }
  return ES_SUCCESS;
}

static NvlsView nvls_view(const es_ctx* c) {
  char* mc = reinterpret_cast<char*>(c->nvls.mcva);
  NvlsView v;
  v.G = reinterpret_cast<const double*>(mc + c->nvls.off_g);
  v.mean = reinterpret_cast<float*>(mc + c->nvls.off_mean);
  v.best = reinterpret_cast<float*>(mc + c->nvls.off_best);
  v.sig = c->nvls.off_sig == (size_t)-1 ? nullptr : reinterpret_cast<float*>(mc + c->nvls.off_sig);
  return v;
}

es_status_t es_tell_nvls_apply(es_ctx_t* c, es_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!c) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (!c->told_local) return fail(c, ES_ERR_BAD_STATE, "es_tell_nvls_apply without es_tell_local");
  if (c->nvls.stage != 2) return fail(c, ES_ERR_BAD_STATE, "NVLS buffer not bound");
  {
    ProfScope ps(c, "nvls_apply", st);
    CUDA_OR(c, launch_nvls_apply(c->s, nvls_view(c), st));
  }
  c->launches += 1;
  c->told_local = false;
  c->asked = false;
  return ES_SUCCESS;
}

es_status_t es_tell_p2p_finish(es_ctx_t* c, es_stream_t stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (!c) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  if (c->peers.W != c->s.W) return fail(c, ES_ERR_BAD_STATE, "es_p2p_set_peers was not called");
  if (!p2p_phases(c)) return ES_SUCCESS;             // nothing after the apply kernel
  if (c->p2p_phase < 0) return fail(c, ES_ERR_BAD_STATE, "es_tell_p2p_finish without es_tell_p2p_apply");
  int nk = 0;
  {
    ProfScope ps(c, "p2p_finish", st);
    CUDA_OR(c, launch_p2p_finish(c->s, c->peers, c->p2p_phase, st, &nk));
  }
  c->launches += nk;
  c->p2p_phase = c->p2p_phase + 1 < p2p_phases(c) ? c->p2p_phase + 1 : -1;
  return ES_SUCCESS;
}

int32_t es_p2p_finish_phases(const es_ctx_t* c) { return c ? p2p_phases(c) : -1;
}

es_status_t es_p2p_ipc_export(const es_ctx_t* c, void* handles) {
  if (!c || !handles) return fail(nullptr, ES_ERR_INVALID_ARG, "NULL argument");
  if (c->guard) return fail(nullptr, ES_ERR_UNSUPPORTED, "IPC export in guard mode (ES_GUARD_ALLOCS)");
  auto* h = static_cast<cudaIpcMemHandle_t*>(handles);
  std::memset(handles, 0, kIpcHandles * sizeof(cudaIpcMemHandle_t));
  cudaError_t e = cudaIpcGetMemHandle(&h[0], c->s.G);
  for (int f = 0; f < 8 && e == cudaSuccess; ++f)
    if (c->s.vec[f]) e = cudaIpcGetMemHandle(&h[1 + f], c->s.vec[f]);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h[9], c->s.n2);
  if (e != cudaSuccess) return fail(nullptr, ES_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  return ES_SUCCESS;
}

es_status_t es_p2p_ipc_open(es_ctx_t* c, const void* all) {
  if (!c || !all) return fail(c, ES_ERR_INVALID_ARG, "NULL argument");
  const int W = c->s.W;
  if (W > kMaxPeers) return fail(c, ES_ERR_UNSUPPORTED, "more than %d peers", kMaxPeers);
  const auto* h = static_cast<const cudaIpcMemHandle_t*>(all);
  static const cudaIpcMemHandle_t zero{};
  std::vector<es_peer_t> peers(W);
  for (int v = 0; v < W; ++v) {
    if (v == c->s.rank) {
      es_p2p_export(c, &peers[v]);
      continue;
    }
    const cudaIpcMemHandle_t* hv = h + kIpcHandles * v;
    void* p = nullptr;
    CUDA_OR(c, cudaIpcOpenMemHandle(&p, hv[0], cudaIpcMemLazyEnablePeerAccess));
    c->ipc_open.push_back(p);
    peers[v].dirsum = static_cast<const double*>(p);
    for (int f = 0; f < 8; ++f) {
      peers[v].field[f] = nullptr;
      if (std::memcmp(&hv[1 + f], &zero, sizeof zero) == 0) continue;
      CUDA_OR(c, cudaIpcOpenMemHandle(&p, hv[1 + f], cudaIpcMemLazyEnablePeerAccess));
      c->ipc_open.push_back(p);
      peers[v].field[f] = static_cast<float*>(p);
    }
    CUDA_OR(c, cudaIpcOpenMemHandle(&p, hv[9], cudaIpcMemLazyEnablePeerAccess));
    c->ipc_open.push_back(p);
    peers[v].norm2 = static_cast<const double*>(p);
  }
  return es_p2p_set_peers(c, peers.data(), W);
}

}  // extern "C"
