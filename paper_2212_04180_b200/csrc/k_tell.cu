// k_tell.cu — K6+K7: the fused tell. Regenerate z from the Philox counter (never stored, never
// re-read), reduce the weighted direction sums of NUMERICS N12 in binary64, and apply the OpenAI-ES
// + Adam, PGPE, SNES or Sep-CMA-ES update.
//
// Mapping: one thread owns (run r, quad q of 4 dims) and a contiguous range of tell entries
// (directions, or Sep-CMA's weighted sorted positions); the (direction index, coefficients) of a
// tile of entries are staged in shared memory and broadcast to all threads. Per entry: one Philox
// call → 4 normals → k DFMAs per normal. When the entry range is split across several CTAs (grid.y
// = nchunk, to fill 148 SMs), each CTA writes binary64 partials and the LAST CTA of its (run, quad
// tile) — elected with a threadfence + atomic counter — sums the partials in chunk order (so the
// result does not depend on scheduling) and runs the update epilogue in the same kernel.
// Bound: Philox + Box–Muller issue rate (ALU); the state traffic (16–32 B/dim) is ~0.1 % of time.
#include <algorithm>
#include <cstdlib>

#include "es_internal.h"
#include "noise.cuh"

namespace esb {

#ifndef ES_TELL_MINB
#define ES_TELL_MINB 8
#endif
static constexpr int TT = kTellThreads;

// s.G layout [2][R][D]: the first R·D doubles are the only ones OpenAI-ES all-reduces.
__device__ __forceinline__ int64_t gidx(const DevState& s, int k, int r, int64_t d) {
  return ((int64_t)k * s.R + r) * s.D + d;
}
static constexpr int kTile = 256;

struct Acc {
  double a[4], b[4];
  double wsum;   // Σ of the z²-term coefficients (PGPE h_i, SNES ω_j): Σ c(z²−1) = Σ c z² − Σ c
};

// Per normal: F2F + 1 DFMA (OpenAI-ES); F2F + DFMA + DMUL + DFMA (PGPE); F2F + DMUL + DADD + DFMA
// (SNES, Sep-CMA: u = ω z feeds both sums). The (z² − 1) of N12 is applied once per chunk through
// wsum — the same real-number sum, reassociated (binary64, ~1e-16 relative).
template <int ALGO>
__device__ __forceinline__ void accumulate(Acc& acc, const float4& z, double cA, double cB) {
  const float zz[4] = {z.x, z.y, z.z, z.w};
  if (ALGO == PGPE) acc.wsum = __dadd_rn(acc.wsum, cB);
  if (ALGO == SNES) acc.wsum = __dadd_rn(acc.wsum, cA);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double zd = (double)zz[k];
    if (ALGO == OPENAI_ES || ALGO == ARS) {
      acc.a[k] = __fma_rn(cA, zd, acc.a[k]);
    } else if (ALGO == PGPE) {
      acc.a[k] = __fma_rn(cA, zd, acc.a[k]);
      acc.b[k] = __fma_rn(cB, __dmul_rn(zd, zd), acc.b[k]);
    } else {
      const double u = __dmul_rn(cA, zd);
      acc.a[k] = __dadd_rn(acc.a[k], u);
      acc.b[k] = __fma_rn(u, zd, acc.b[k]);
    }
  }
}

__device__ __forceinline__ double block_sum_tt(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int k = 0; k < TT / 32; ++k) t = __dadd_rn(t, red[k]);
  return t;
}

__device__ __forceinline__ void adam_step(float& mean, float& am, float& av, float g,
                                          const RunScal& rs, const GenScal& gs) {
  const float b1 = rs.beta1, b2 = rs.beta2;
  const float mn = __fmaf_rn(b1, am, __fmul_rn(__fsub_rn(1.0f, b1), g));
  const float vn = __fmaf_rn(b2, av, __fmul_rn(__fsub_rn(1.0f, b2), __fmul_rn(g, g)));
  const float den = __fadd_rn(__fsqrt_rn(__fdiv_rn(vn, gs.bc2)), rs.eps);
  mean = __fsub_rn(mean, __fmul_rn(gs.lr, __fdiv_rn(__fdiv_rn(mn, gs.bc1), den)));
  am = mn;
  av = vn;
}

// The optimizer step of OpenAI-ES / PGPE for one dim. Adam and momentum SGD
// update in place; ClipUp needs two global norms, so here it only parks g (binary64 slot of s.G)
// and adds g² to the block's norm partial; launch_clipup_finish completes the step.
__device__ __forceinline__ void opt_step(const DevState& s, int r, int64_t d, int64_t idx,
                                         float& mean, float g, const RunScal& rs,
                                         const GenScal& gs, double& norm2) {
  if (rs.optimizer == OPT_ADAM) {
    adam_step(mean, s.vec[F_ADAM_M][idx], s.vec[F_ADAM_V][idx], g, rs, gs);
  } else if (rs.optimizer == OPT_SGD) {
    const float vn = __fmaf_rn(rs.momentum, s.vec[F_ADAM_M][idx], g);
    s.vec[F_ADAM_M][idx] = vn;
    mean = __fsub_rn(mean, __fmul_rn(gs.lr, vn));
  } else {
    s.G[gidx(s, 0, r, d)] = (double)g;
    if (d < s.Dx) norm2 = __dadd_rn(norm2, __dmul_rn((double)g, (double)g));
  }
}

// Update epilogue for the 4 dims of quad q of run r from the reduced sums G0, G1 (N12). Also
// regenerates best_x from the pre-update state when this generation improved.
// Sep-CMA: phase 1 only (mean, p_σ, Z/Q to s.G, ‖p_σ‖² partial of the block to normpart).
template <int ALGO>
__device__ void apply_update(const DevState& s, int r, int64_t q, bool active, const double* G0,
                             const double* G1, int qb, int bpr, double* red) {
  const RunScal& rs = s.rs[r];
  const GenScal& gs = s.gs[r];
  double norm2 = 0.0;
  if (active) {
    const Philox ph(rs.seed);
    float4 zb = make_float4(0.f, 0.f, 0.f, 0.f);
    float sgn = 1.0f;
    if (gs.improved) {
      constexpr bool kAnti = is_anti(ALGO);
      const int i = kAnti ? gs.jbest / 2 : gs.jbest;
      sgn = (kAnti && (gs.jbest & 1)) ? -1.0f : 1.0f;
      zb = normal4(ph, (uint32_t)(q + s.q0), (uint32_t)i, gs.t);
    }
    const float zbv[4] = {zb.x, zb.y, zb.z, zb.w};
    float omcs = 0.f, ks = 0.f;
    if (ALGO == SEP_CMA_ES) {
      omcs = (float)__dsub_rn(1.0, rs.c_sigma);
      ks = (float)sqrt(__dmul_rn(__dmul_rn(rs.c_sigma, __dsub_rn(2.0, rs.c_sigma)), rs.mueff));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t d = 4 * q + k;
      if (d >= s.D) break;
      const int64_t idx = (int64_t)r * s.D + d;
      float mean = s.vec[F_MEAN][idx];
      if (gs.improved) {
        float sc;
        if (ALGO == OPENAI_ES || ALGO == ARS) sc = gs.sigma;
        else if (ALGO == SEP_CMA_ES) sc = __fmul_rn(gs.sigma, __fsqrt_rn(s.vec[F_C][idx]));
        else sc = s.vec[F_SIGMA_D][idx];
        float xb = __fmaf_rn(sgn * sc, zbv[k], mean);
        if (rs.clip) xb = fminf(fmaxf(xb, rs.clip_lo), rs.clip_hi);   // the member as asked
        s.vec[F_BEST_X][idx] = xb;
      }
      if (ALGO == ARS) {
        // ARS: mean −= α/(k σ_R) · Σ_sel (f+ − f−) z; no step when σ_R = 0
        if (gs.ars_scale != 0.0f) mean = __fsub_rn(mean, __fmul_rn(gs.ars_scale, (float)G0[k]));
      } else if (ALGO == OPENAI_ES) {
        const float g = __fdiv_rn((float)G0[k], __fmul_rn((float)s.N, gs.sigma));
        opt_step(s, r, d, idx, mean, g, rs, gs, norm2);
      } else if (ALGO == PGPE) {
        const float sig = s.vec[F_SIGMA_D][idx];
        // normalised by the 2k members / k pairs used (k = N/2 unless elite pairs, Q13b)
        const float gm = __fdiv_rn(__fmul_rn(sig, (float)G0[k]), (float)(2 * gs.nentries));
        const float gsg = __fdiv_rn(__fmul_rn(sig, (float)G1[k]), (float)gs.nentries);
        opt_step(s, r, d, idx, mean, gm, rs, gs, norm2);
        const float mc = rs.sigma_max_change;
        float st = __fsub_rn(sig, __fmul_rn(rs.sigma_lrate, gsg));
        const float lo = __fmul_rn(__fsub_rn(1.0f, mc), sig);
        const float hi = __fmul_rn(__fadd_rn(1.0f, mc), sig);
        st = fminf(fmaxf(st, lo), hi);
        s.vec[F_SIGMA_D][idx] = fmaxf(__fmul_rn(st, rs.sigma_decay), rs.sigma_limit);
      } else if (ALGO == SNES) {
        const float sig = s.vec[F_SIGMA_D][idx];
        mean = __fadd_rn(mean, __fmul_rn(sig, (float)G0[k]));
        s.vec[F_SIGMA_D][idx] =
            __fmul_rn(sig, (float)exp(__dmul_rn(__dmul_rn(rs.eta_sigma, 0.5), G1[k])));
      } else {
        const float Z = (float)G0[k];
        const float y = __fmul_rn(__fsqrt_rn(s.vec[F_C][idx]), Z);
        mean = __fadd_rn(mean, __fmul_rn(gs.sigma, y));
        const float ps = __fadd_rn(__fmul_rn(omcs, s.vec[F_PSIGMA][idx]), __fmul_rn(ks, Z));
        s.vec[F_PSIGMA][idx] = ps;
        if (d < s.Dx) norm2 = __dadd_rn(norm2, __dmul_rn((double)ps, (double)ps));   // not the halo
        s.G[gidx(s, 0, r, d)] = G0[k];
        s.G[gidx(s, 1, r, d)] = G1[k];
      }
      s.vec[F_MEAN][idx] = mean;
    }
  }
  // block-uniform: one run per block
  if (ALGO == SEP_CMA_ES || ((ALGO == OPENAI_ES || ALGO == PGPE) && rs.optimizer == OPT_CLIPUP)) {
    const double tot = block_sum_tt(norm2, red);
    if (threadIdx.x == 0) s.normpart[(int64_t)r * bpr + qb] = tot;
  }
}

// grid.y = the largest per-run chunk count; run r's entries [e0, e1) are cut into chunks of
// `echunk` entries, nch_r = max(1, ⌈(e1 − e0)/echunk⌉) of them — so runs with few weighted entries
// (Sep-CMA-ES elite ratios vmapped over runs) occupy few CTAs and the block scheduler packs
// the SMs instead of one wave waiting on the longest runs. CTAs past nch_r exit at once.
template <int ALGO>
__global__ void __launch_bounds__(TT, ES_TELL_MINB) tell_kernel(DevState s,
                                                                 const int4* __restrict__ items,
                                                                 int echunk, int fused) {
  __shared__ uint32_t sdir[kTile];
  __shared__ double sA[kTile];
  __shared__ double sB[kTile];
  __shared__ double red[TT / 32];
  __shared__ int sh_last;
  pdl_enter();
  const int4 it = items[blockIdx.y];
  const int r = it.x, chunk = it.y, nchunk = it.z;
  const int qb = blockIdx.x, bpr = gridDim.x;
  const int64_t q = (int64_t)qb * TT + threadIdx.x;
  const bool active = q < s.Q;
  const GenScal& gs = s.gs[r];
  const int ne = gs.nentries;
  int e0 = 0, e1 = ne;
  if (s.W > 1) shard_range(ne, s.W, s.rank, e0, e1);
  const int c0 = min(e1, e0 + chunk * echunk);
  const int c1 = chunk == nchunk - 1 ? e1 : min(e1, c0 + echunk);
  const Philox ph(s.rs[r].seed);
  const uint32_t t = gs.t;
  const uint32_t* dir = s.dir + (int64_t)r * s.N;
  const double* cA = s.coefA + (int64_t)r * s.N;
  const double* cB = s.coefB + (int64_t)r * s.N;
  Acc acc;
  acc.wsum = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) acc.a[k] = acc.b[k] = 0.0;
  for (int b0 = c0; b0 < c1; b0 += kTile) {
    const int nb = min(kTile, c1 - b0);
    __syncthreads();
    for (int e = threadIdx.x; e < nb; e += TT) {
      sdir[e] = dir[b0 + e];
      sA[e] = cA[b0 + e];
      if (ALGO == PGPE) sB[e] = cB[b0 + e];
    }
    __syncthreads();
    if (active) {
#pragma unroll 2
      for (int e = 0; e < nb; ++e) {
        const float4 z = normal4(ph, (uint32_t)(q + s.q0), sdir[e], t);
        accumulate<ALGO>(acc, z, sA[e], ALGO == PGPE ? sB[e] : 0.0);
      }
    }
  }
  if (ALGO == PGPE || ALGO == SNES) {
#pragma unroll
    for (int k = 0; k < 4; ++k) acc.b[k] = __dsub_rn(acc.b[k], acc.wsum);
  }
  const int64_t D2 = 2 * s.D;
  if (nchunk > 1) {
    // publish partials, elect the last CTA of this (run, quad tile)
    if (active) {
      double* P = s.Gchunk + ((int64_t)chunk * s.R + r) * D2;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (4 * q + k < s.D) {
          P[4 * q + k] = acc.a[k];
          if (ALGO != OPENAI_ES && ALGO != ARS) P[s.D + 4 * q + k] = acc.b[k];
        }
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t prev = atomicAdd(&s.arrive[(int64_t)r * bpr + qb], 1u);
      sh_last = (prev == (uint32_t)(nchunk - 1));
      if (sh_last) s.arrive[(int64_t)r * bpr + qb] = 0u;
    }
    __syncthreads();
    if (!sh_last) return;
    __threadfence();
    if (active) {
#pragma unroll
      for (int k = 0; k < 4; ++k) acc.a[k] = acc.b[k] = 0.0;
      for (int c = 0; c < nchunk; ++c) {
        const double* P = s.Gchunk + ((int64_t)c * s.R + r) * D2;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (4 * q + k < s.D) {
            acc.a[k] = __dadd_rn(acc.a[k], __ldcg(P + 4 * q + k));
            if (ALGO != OPENAI_ES && ALGO != ARS)
              acc.b[k] = __dadd_rn(acc.b[k], __ldcg(P + s.D + 4 * q + k));
          }
        }
      }
    }
  }
  if (fused) {
    apply_update<ALGO>(s, r, q, active, acc.a, acc.b, qb, bpr, red);
  } else if (active) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (4 * q + k < s.D) {
        s.G[gidx(s, 0, r, 4 * q + k)] = acc.a[k];
        if (ALGO != OPENAI_ES && ALGO != ARS) s.G[gidx(s, 1, r, 4 * q + k)] = acc.b[k];
      }
    }
  }
}

// W > 1: after the all-reduce of s.G, apply the update.
template <int ALGO>
__global__ void __launch_bounds__(TT) update_kernel(DevState s, int bpr) {
  __shared__ double red[TT / 32];
  const int r = blockIdx.x / bpr;
  const int qb = blockIdx.x % bpr;
  const int64_t q = (int64_t)qb * TT + threadIdx.x;
  const bool active = q < s.Q;
  double G0[4] = {0, 0, 0, 0}, G1[4] = {0, 0, 0, 0};
  if (active) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (4 * q + k < s.D) {
        G0[k] = s.G[gidx(s, 0, r, 4 * q + k)];
        if (ALGO != OPENAI_ES && ALGO != ARS) G1[k] = s.G[gidx(s, 1, r, 4 * q + k)];
      }
    }
  }
  apply_update<ALGO>(s, r, q, active, G0, G1, qb, bpr, red);
}

// Fixed-order sum of run r's per-block norm partials (valid in thread 0).
__device__ __forceinline__ double normpart_total(const DevState& s, int r, int bpr, double* red) {
  double v = 0.0;
  for (int b = threadIdx.x; b < bpr; b += blockDim.x) v = __dadd_rn(v, __ldcg(&s.normpart[(int64_t)r * bpr + b]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double n2 = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) n2 = __dadd_rn(n2, red[k]);
  return n2;
}

// Sep-CMA-ES phase 2: global ‖p_σ'‖ (fixed-order sum of the block partials), σ', h_σ.
// D-sharded contexts split it: sepcma_n2_kernel writes this rank's ‖p_σ'‖² share to s.n2, the
// shares are summed over ranks (NCCL or the caller), then sepcma_norm_kernel reads s.n2.
// (Also ClipUp's shares under the peer-memory tell: ‖g‖² at off 0, ‖v'‖² at off R.)
__global__ void sepcma_n2_kernel(DevState s, int bpr, int off) {
  __shared__ double red[32];
  const double n2 = normpart_total(s, blockIdx.x, bpr, red);
  if (threadIdx.x == 0) s.n2[off + blockIdx.x] = n2;
}

// σ' and h_σ of run r from the global ‖p_σ'‖² (one thread).
__device__ __forceinline__ void sepcma_sigma(const DevState& s, int r, double n2) {
  RunScal& rs = s.rs[r];
  GenScal& gs = s.gs[r];
  const double norm = sqrt(n2);
  const double Dd = (double)s.Dg;
  const float sig_new = __fmul_rn(
      gs.sigma, (float)exp(__dmul_rn(__ddiv_rn(rs.c_sigma, rs.d_sigma),
                                     __dsub_rn(__ddiv_rn(norm, rs.chi_d), 1.0))));
  const double lhs = norm / sqrt(1.0 - pow(1.0 - rs.c_sigma, 2.0 * (double)(gs.t + 1)));
  gs.hsig = lhs < (1.4 + 2.0 / (Dd + 1.0)) * rs.chi_d;
  gs.sigma_new = sig_new;
  rs.sigma = sig_new;
}

__global__ void sepcma_norm_kernel(DevState s, int bpr) {
  __shared__ double red[32];
  pdl_enter();
  const int r = blockIdx.x;
  const double n2 = s.dshard ? s.n2[r] : normpart_total(s, r, bpr, red);
  if (threadIdx.x == 0) sepcma_sigma(s, r, n2);
}

// The run's p_c / C coefficients (binary64 → binary32, as the oracle rounds them), once per run.
struct PcCoef {
  float omcc, kc, aC, c1f, cmuf;
};
__device__ __forceinline__ PcCoef sepcma_pc_coef(const DevState& s, int r) {
  const RunScal& rs = s.rs[r];
  const GenScal& gs = s.gs[r];
  const double hs = gs.hsig ? 1.0 : 0.0;
  PcCoef k;
  k.omcc = (float)(1.0 - rs.c_c);
  k.kc = gs.hsig ? (float)sqrt(rs.c_c * (2.0 - rs.c_c) * rs.mueff) : 0.0f;
  k.aC = (float)(1.0 - rs.c_1 - rs.c_mu + (1.0 - hs) * rs.c_1 * rs.c_c * (2.0 - rs.c_c));
  k.c1f = (float)rs.c_1;
  k.cmuf = (float)rs.c_mu;
  return k;
}

// p_c and C of element idx (run r, dim d) from Z, Q (s.G) and h_σ.
__device__ __forceinline__ void sepcma_pc_elem(const DevState& s, int r, int64_t d,
                                               const PcCoef& k) {
  const float omcc = k.omcc, kc = k.kc, aC = k.aC, c1f = k.c1f, cmuf = k.cmuf;
  const float Z = (float)__ldcg(&s.G[gidx(s, 0, r, d)]);
  const float Qv = (float)__ldcg(&s.G[gidx(s, 1, r, d)]);
  const int64_t idx = (int64_t)r * s.D + d;
  const float C0 = s.vec[F_C][idx];
  const float y = __fmul_rn(__fsqrt_rn(C0), Z);
  const float pcn = __fadd_rn(__fmul_rn(omcc, s.vec[F_PC][idx]), __fmul_rn(kc, y));
  s.vec[F_PC][idx] = pcn;
  s.vec[F_C][idx] = __fadd_rn(__fadd_rn(__fmul_rn(aC, C0), __fmul_rn(c1f, __fmul_rn(pcn, pcn))),
                              __fmul_rn(cmuf, __fmul_rn(C0, Qv)));
}

// f2: the all-reduce of the direction sums and the update, fused over peer memory.
// Rank w owns quads [Q·w/W, Q·(w+1)/W) of every run: it reads the W partial sums of its slice from
// the peers' buffers (NVLink loads; summed in rank order, so every rank and the emulation agree
// bit for bit), applies the update to the slice (its optimizer state is the only copy — the
// "memory split across devices" of P:226), and writes the updated mean / σ_d / best_x of the
// slice into every peer's state (NVLink stores). Compute and communication are one kernel; the
// stream-ordered barriers around it are the caller's (es_tell uses two 4-byte NCCL all-reduces).
template <int ALGO>
__global__ void __launch_bounds__(TT) p2p_apply_kernel(DevState s, PeerTable pt, int64_t qa,
                                                       int64_t qe, int bps) {
  __shared__ double red[TT / 32];
  const int r = blockIdx.x / bps;
  const int64_t q = qa + (int64_t)(blockIdx.x % bps) * TT + threadIdx.x;
  const bool active = q < qe;
  constexpr bool kTwo = !(ALGO == OPENAI_ES || ALGO == ARS);
  double G0[4] = {0.0, 0.0, 0.0, 0.0}, G1[4] = {0.0, 0.0, 0.0, 0.0};
  if (active) {
    for (int v = 0; v < pt.W; ++v) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t d = 4 * q + k;
        if (d < s.D) {
          G0[k] = __dadd_rn(G0[k], __ldcg(pt.G[v] + gidx(s, 0, r, d)));
          if (kTwo) G1[k] = __dadd_rn(G1[k], __ldcg(pt.G[v] + gidx(s, 1, r, d)));
        }
      }
    }
  }
  apply_update<ALGO>(s, r, q, active, G0, G1, blockIdx.x % bps, bps, red);
  if (!active) return;
  constexpr int kF[3] = {F_MEAN, F_BEST_X, F_SIGMA_D};
  constexpr int nf = (ALGO == PGPE || ALGO == SNES) ? 3 : 2;
  for (int v = 0; v < pt.W; ++v) {
    if (v == s.rank) continue;
#pragma unroll
    for (int fi = 0; fi < nf; ++fi) {
      const float* src = s.vec[kF[fi]];
      float* dst = pt.vec[v][kF[fi]];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t d = 4 * q + k;
        if (d < s.D) __stcg(dst + (int64_t)r * s.D + d, src[(int64_t)r * s.D + d]);
      }
    }
  }
}

cudaError_t launch_p2p_apply(const DevState& s, const PeerTable& pt, bool clipup, cudaStream_t st,
                             int* nk) {
  const int64_t qa = s.Q * s.rank / s.W, qe = s.Q * (s.rank + 1) / s.W;
  const int bps = (int)std::max<int64_t>(1, (qe - qa + TT - 1) / TT);
  const unsigned g = (unsigned)(s.R * bps);
  if (nk) *nk = (s.algo == SEP_CMA_ES || clipup) ? 2 : 1;
  switch (s.algo) {
    case OPENAI_ES: p2p_apply_kernel<OPENAI_ES><<<g, TT, 0, st>>>(s, pt, qa, qe, bps); break;
    case PGPE: p2p_apply_kernel<PGPE><<<g, TT, 0, st>>>(s, pt, qa, qe, bps); break;
    case SNES: p2p_apply_kernel<SNES><<<g, TT, 0, st>>>(s, pt, qa, qe, bps); break;
    case ARS: p2p_apply_kernel<ARS><<<g, TT, 0, st>>>(s, pt, qa, qe, bps); break;
    case SEP_CMA_ES:
      p2p_apply_kernel<SEP_CMA_ES><<<g, TT, 0, st>>>(s, pt, qa, qe, bps);
      sepcma_n2_kernel<<<s.R, 256, 0, st>>>(s, bps, 0);  // this slice's ‖p_σ'‖² share → s.n2
      break;
    default: return cudaErrorInvalidValue;
  }
  // ClipUp parked g in the slice and left ‖g‖² block partials: this slice's share → s.n2[0, R)
  if (clipup) sepcma_n2_kernel<<<s.R, 256, 0, st>>>(s, bps, 0);
  return cudaGetLastError();
}

// Sep-CMA-ES under the peer-memory tell, after a barrier: the global ‖p_σ'‖² (peer n2 shares in
// rank order → identical σ', h_σ on every rank), then p_c and C of this rank's slice, and C's slice
// stored into every peer (the ask needs the full C).
__global__ void p2p_sepcma_sigma_kernel(DevState s, PeerTable pt) {
  if (threadIdx.x != 0) return;
  const int r = blockIdx.x;
  double n2 = 0.0;
  for (int v = 0; v < pt.W; ++v) n2 = __dadd_rn(n2, __ldcg(pt.n2[v] + r));
  sepcma_sigma(s, r, n2);
}

__global__ void __launch_bounds__(256) p2p_sepcma_pc_kernel(DevState s, PeerTable pt, int64_t d0,
                                                            int64_t d1) {
  const int r = blockIdx.y;
  const int64_t d = d0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= d1) return;
  sepcma_pc_elem(s, r, d, sepcma_pc_coef(s, r));
  const int64_t idx = (int64_t)r * s.D + d;
  const float c = s.vec[F_C][idx];
  for (int v = 0; v < pt.W; ++v)
    if (v != s.rank) __stcg(pt.vec[v][F_C] + idx, c);
}


// f2 NVLS variant of p2p_apply_kernel: the W partial sums of the slice are added inside the switch
// (multimem.ld_reduce on the multicast alias of every rank's G), and the updated slice is
// broadcast with one multimem.st per value. Summation order is the switch's, so results can differ
// from the rank-ordered P2P / NCCL paths in the last binary64 bits.
__device__ __forceinline__ double mm_ld_add_f64(const double* mc) {
  double v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f64 %0, [%1];" : "=d"(v) : "l"(mc) : "memory");
  return v;
}
__device__ __forceinline__ void mm_st_f32(float* mc, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "f"(v) : "memory");
}

template <int ALGO>
__global__ void __launch_bounds__(TT) nvls_apply_kernel(DevState s, NvlsView v, int64_t qa,
                                                        int64_t qe, int bps) {
  __shared__ double red[TT / 32];
  asm volatile("fence.proxy.alias;" ::: "memory");
  const int r = blockIdx.x / bps;
  const int64_t q = qa + (int64_t)(blockIdx.x % bps) * TT + threadIdx.x;
  const bool active = q < qe;
  constexpr bool kTwo = !(ALGO == OPENAI_ES || ALGO == ARS);
  double G0[4] = {0.0, 0.0, 0.0, 0.0}, G1[4] = {0.0, 0.0, 0.0, 0.0};
  if (active) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t d = 4 * q + k;
      if (d < s.D) {
        G0[k] = mm_ld_add_f64(v.G + gidx(s, 0, r, d));
        if (kTwo) G1[k] = mm_ld_add_f64(v.G + gidx(s, 1, r, d));
      }
    }
  }
  apply_update<ALGO>(s, r, q, active, G0, G1, 0, 1, red);
  if (active) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t d = 4 * q + k;
      if (d >= s.D) break;
      const int64_t idx = (int64_t)r * s.D + d;
      mm_st_f32(v.mean + idx, s.vec[F_MEAN][idx]);
      mm_st_f32(v.best + idx, s.vec[F_BEST_X][idx]);
      if (v.sig) mm_st_f32(v.sig + idx, s.vec[F_SIGMA_D][idx]);
    }
  }
  asm volatile("fence.proxy.alias;" ::: "memory");
}

cudaError_t launch_nvls_apply(const DevState& s, const NvlsView& v, cudaStream_t st) {
  const int64_t qa = s.Q * s.rank / s.W, qe = s.Q * (s.rank + 1) / s.W;
  const int bps = (int)std::max<int64_t>(1, (qe - qa + TT - 1) / TT);
  const unsigned g = (unsigned)(s.R * bps);
  switch (s.algo) {
    case OPENAI_ES: nvls_apply_kernel<OPENAI_ES><<<g, TT, 0, st>>>(s, v, qa, qe, bps); break;
    case PGPE: nvls_apply_kernel<PGPE><<<g, TT, 0, st>>>(s, v, qa, qe, bps); break;
    case SNES: nvls_apply_kernel<SNES><<<g, TT, 0, st>>>(s, v, qa, qe, bps); break;
    case ARS: nvls_apply_kernel<ARS><<<g, TT, 0, st>>>(s, v, qa, qe, bps); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Sep-CMA-ES phase 3: p_c and C from Z, Q (s.G) and h_σ.
__global__ void __launch_bounds__(256) sepcma_pc_kernel(DevState s) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)s.R * s.D) return;
  sepcma_pc_elem(s, (int)(gid / s.D), gid % s.D, sepcma_pc_coef(s, (int)(gid / s.D)));
}

// ClipUp (Toklu et al. 2020), phases after the gradient g is parked in s.G:
//   norm(0): inv = 1/‖g‖ (0 if ‖g‖ = 0)      vel: v' = μ v + lr (g · inv), ‖v'‖² partials
//   norm(1): clip = max_speed/‖v'‖ if ‖v'‖ > max_speed else 1      apply: v = v' clip, m −= v.
// Runs using another optimizer skip every phase.
__device__ __forceinline__ void clipup_scalar(const DevState& s, int r, double n2, int phase) {
  const double n = sqrt(n2);
  GenScal& gs = s.gs[r];
  if (phase == 0) {
    gs.clip_inv = n > 0.0 ? (float)(1.0 / n) : 0.0f;
  } else {
    const double ms = (double)s.rs[r].max_speed;
    gs.clip_inv = n > ms ? (float)(ms / n) : 1.0f;
  }
}

__global__ void clipup_norm_kernel(DevState s, int bpr, int phase) {
  __shared__ double red[32];
  const int r = blockIdx.x;
  if (s.rs[r].optimizer != OPT_CLIPUP) return;
  const double n2 = normpart_total(s, r, bpr, red);
  if (threadIdx.x == 0) clipup_scalar(s, r, n2, phase);
}

// Quads [qa, qe) of every run (the whole run, or a peer-memory rank's slice), bpr blocks each.
__global__ void __launch_bounds__(TT) clipup_vel_kernel(DevState s, int bpr, int64_t qa,
                                                        int64_t qe) {
  __shared__ double red[TT / 32];
  const int r = blockIdx.x / bpr, qb = blockIdx.x % bpr;
  const RunScal& rs = s.rs[r];
  if (rs.optimizer != OPT_CLIPUP) return;              // block-uniform
  const GenScal& gs = s.gs[r];
  const int64_t q = qa + (int64_t)qb * TT + threadIdx.x;
  double v2 = 0.0;
  if (q < qe) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t d = 4 * q + k;
      if (d >= s.D) break;
      const int64_t idx = (int64_t)r * s.D + d;
      const float g = (float)s.G[gidx(s, 0, r, d)];
      const float vn = __fmaf_rn(rs.momentum, s.vec[F_ADAM_M][idx],
                                 __fmul_rn(gs.lr, __fmul_rn(g, gs.clip_inv)));
      s.vec[F_ADAM_M][idx] = vn;
      if (d < s.Dx) v2 = __dadd_rn(v2, __dmul_rn((double)vn, (double)vn));
    }
  }
  const double tot = block_sum_tt(v2, red);
  if (threadIdx.x == 0) s.normpart[(int64_t)r * bpr + qb] = tot;
}

__global__ void __launch_bounds__(256) clipup_apply_kernel(DevState s) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)s.R * s.D) return;
  const int r = (int)(gid / s.D);
  if (s.rs[r].optimizer != OPT_CLIPUP) return;
  const float v = __fmul_rn(s.vec[F_ADAM_M][gid], s.gs[r].clip_inv);
  s.vec[F_ADAM_M][gid] = v;
  s.vec[F_MEAN][gid] = __fsub_rn(s.vec[F_MEAN][gid], v);
}

int tell_blocks_per_run(const DevState& s) { return (int)((s.Q + TT - 1) / TT); }

// Entry-chunk size: choose echunk minimising the estimated makespan of the tell grid. Each CTA costs
// (its entries + c0) entry-times, c0 ≈ the per-CTA fixed cost (coefficient staging, partial
// write-back, last-CTA reduction); `ent[r]` is run r's expected entry count on this rank (P, N, or
// Sep-CMA-ES's μ_r). For grids up to 2^16 CTAs the makespan is simulated the way the block
// scheduler dispatches (blockIdx.x fastest, each CTA onto the earliest-free of `slots` resident
// slots); beyond that, waves(n) · (max entries/n + c0).
template <int ALGO>
static TellSplit pick_split_t(const DevState& s, const std::vector<int>& ent) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tell_kernel<ALGO>, TT, 0);
  occ = std::max(occ, 1);
  const int64_t slots = (int64_t)sm_count() * occ;
  const int bpr = tell_blocks_per_run(s);
  const int64_t blocks = (int64_t)s.R * bpr;
  int emax = 1;
  for (int e : ent) emax = std::max(emax, e);
  const double c0 = 8.0;
  TellSplit best{1, emax};
  double best_t = 1e300;
  std::vector<double> heap;
  for (int n = 1; n <= std::min(64, emax); ++n) {
    const int ec = (emax + n - 1) / n;
    if (n > 1 && (emax + ec - 1) / ec != n) continue;         // same echunk as a smaller n
    int64_t nit = 0;                                           // grid.y ≤ 65535 work items
    for (int e : ent) nit += std::max(1, (e + ec - 1) / ec);
    if (n > 1 && nit > 65535) break;
    double tn;
    if (blocks * n <= 65536) {
      heap.assign((size_t)slots, 0.0);                         // min-heap of slot free times
      std::make_heap(heap.begin(), heap.end(), std::greater<double>());
      for (int y = 0; y < n; ++y) {
        for (int r = 0; r < s.R; ++r) {
          const int nch = std::max(1, (ent[r] + ec - 1) / ec);
          if (y >= nch) continue;                    // no CTA: the item table skips it
          const double len = std::min(ec, ent[r] - y * ec) + c0;
          for (int b = 0; b < bpr; ++b) {
            std::pop_heap(heap.begin(), heap.end(), std::greater<double>());
            heap.back() += len;
            std::push_heap(heap.begin(), heap.end(), std::greater<double>());
          }
        }
      }
      tn = *std::max_element(heap.begin(), heap.end());
    } else {
      tn = (double)((blocks * n + slots - 1) / slots) * ((double)ec + c0);
    }
    if (tn < best_t * 0.999) { best_t = tn; best = TellSplit{n, ec}; }
  }
  return best;
}

TellSplit tell_pick_split(const DevState& s, const std::vector<int>& ent) {
  if (const char* e = std::getenv("ES_TELL_ECHUNK")) {     // A/B switch for profiling
    int emax = 1;
    for (int v : ent) emax = std::max(emax, v);
    const int ec = std::max(1, std::min(emax, std::atoi(e)));
    return TellSplit{(emax + ec - 1) / ec, ec};
  }
  switch (s.algo) {
    case OPENAI_ES: return pick_split_t<OPENAI_ES>(s, ent);
    case PGPE: return pick_split_t<PGPE>(s, ent);
    case SNES: return pick_split_t<SNES>(s, ent);
    case ARS: return pick_split_t<ARS>(s, ent);
    default: return pick_split_t<SEP_CMA_ES>(s, ent);
  }
}

std::vector<int4> tell_items(int R, const std::vector<int>& ent, const TellSplit& sp) {
  std::vector<int4> it;
  for (int y = 0; y < sp.nchunk; ++y)            // chunk-major: the block scheduler starts every
    for (int r = 0; r < R; ++r) {                // run's first chunk before anyone's second
      const int nch = std::max(1, (ent[r] + sp.echunk - 1) / sp.echunk);
      if (y < nch) it.push_back(make_int4(r, y, nch, 0));
    }
  return it;
}

template <int ALGO>
static void launch_tell_t(const DevState& s, bool fused, TellSplit sp, cudaStream_t st) {
  dim3 grid((unsigned)tell_blocks_per_run(s), (unsigned)sp.nitems);
  // a launch error stays the thread's last error (launch_tell_reduce returns it)
  (void)launch_pdl(tell_kernel<ALGO>, grid, dim3(TT), 0, st, s, (const int4*)sp.items, sp.echunk,
                   fused ? 1 : 0);
}

cudaError_t launch_tell_reduce(const DevState& s, bool fused, TellSplit sp, cudaStream_t st) {
  switch (s.algo) {
    case OPENAI_ES: launch_tell_t<OPENAI_ES>(s, fused, sp, st); break;
    case PGPE: launch_tell_t<PGPE>(s, fused, sp, st); break;
    case SNES: launch_tell_t<SNES>(s, fused, sp, st); break;
    case ARS: launch_tell_t<ARS>(s, fused, sp, st); break;
    default: launch_tell_t<SEP_CMA_ES>(s, fused, sp, st); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_tell_update(const DevState& s, cudaStream_t st) {
  const int bpr = tell_blocks_per_run(s);
  const unsigned g = (unsigned)(s.R * bpr);
  switch (s.algo) {
    case OPENAI_ES: update_kernel<OPENAI_ES><<<g, TT, 0, st>>>(s, bpr); break;
    case PGPE: update_kernel<PGPE><<<g, TT, 0, st>>>(s, bpr); break;
    case SNES: update_kernel<SNES><<<g, TT, 0, st>>>(s, bpr); break;
    case ARS: update_kernel<ARS><<<g, TT, 0, st>>>(s, bpr); break;
    default: update_kernel<SEP_CMA_ES><<<g, TT, 0, st>>>(s, bpr); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_sepcma_norm(const DevState& s, cudaStream_t st) {
  sepcma_norm_kernel<<<s.R, 256, 0, st>>>(s, tell_blocks_per_run(s));
  return cudaGetLastError();
}

cudaError_t launch_sepcma_n2(const DevState& s, cudaStream_t st) {
  sepcma_n2_kernel<<<s.R, 256, 0, st>>>(s, tell_blocks_per_run(s), 0);
  return cudaGetLastError();
}

// Small D (≤ 16384 dims per run): phase 2 in ONE launch, a CTA per run — ‖p_σ'‖, σ', h_σ, then
// p_c and C of the run's dims by the same CTA (saves the second launch and its ramp; C2: 2 → 1).
__global__ void __launch_bounds__(256) sepcma_finish_kernel(DevState s, int bpr) {
  __shared__ double red[32];
  pdl_enter();
  const int r = blockIdx.x;
  const double n2 = s.dshard ? s.n2[r] : normpart_total(s, r, bpr, red);
  if (threadIdx.x == 0) sepcma_sigma(s, r, n2);
  __syncthreads();                               // h_σ (global, this CTA's own write) visible
  const PcCoef k = sepcma_pc_coef(s, r);          // once per thread, not per element
  for (int64_t d = threadIdx.x; d < s.D; d += blockDim.x) sepcma_pc_elem(s, r, d, k);
}

cudaError_t launch_sepcma_finish(const DevState& s, cudaStream_t st, int* nk) {
  const int bpr = tell_blocks_per_run(s);
  if (s.D <= 16384) {
    if (nk) *nk = 1;
    return launch_pdl(sepcma_finish_kernel, dim3(s.R), dim3(256), 0, st, s, bpr);
  }
  sepcma_norm_kernel<<<s.R, 256, 0, st>>>(s, bpr);
  const int64_t n = (int64_t)s.R * s.D;
  sepcma_pc_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s);
  if (nk) *nk = 2;
  return cudaGetLastError();
}

cudaError_t launch_clipup_finish(const DevState& s, cudaStream_t st, int* nk) {
  const int bpr = tell_blocks_per_run(s);
  const int64_t n = (int64_t)s.R * s.D;
  clipup_norm_kernel<<<s.R, 256, 0, st>>>(s, bpr, 0);
  clipup_vel_kernel<<<(unsigned)(s.R * bpr), TT, 0, st>>>(s, bpr, 0, s.Q);
  clipup_norm_kernel<<<s.R, 256, 0, st>>>(s, bpr, 1);
  clipup_apply_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s);
  if (nk) *nk = 4;
  return cudaGetLastError();
}

// ClipUp under the peer-memory tell, two phases after the apply kernel, each after a barrier:
//   phase 0: 1/‖g‖ from the ranks' ‖g‖² shares (rank order), v' = μ v + lr g/‖g‖ on the slice,
//            the slice's ‖v'‖² share → s.n2[R, 2R) (a second slot: peers may still read [0, R));
//   phase 1: the clip factor from the ‖v'‖² shares, v = v'·clip, m −= v on the slice, and the
//            slice's mean stored into every peer (the velocity stays with its owner).
__global__ void p2p_clipup_norm_kernel(DevState s, PeerTable pt, int phase) {
  const int r = blockIdx.x;
  if (threadIdx.x != 0 || s.rs[r].optimizer != OPT_CLIPUP) return;
  double n2 = 0.0;
  for (int v = 0; v < pt.W; ++v) n2 = __dadd_rn(n2, __ldcg(pt.n2[v] + phase * s.R + r));
  clipup_scalar(s, r, n2, phase);
}

__global__ void __launch_bounds__(256) p2p_clipup_apply_kernel(DevState s, PeerTable pt,
                                                               int64_t d0, int64_t d1) {
  const int r = blockIdx.y;
  const int64_t d = d0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= d1 || s.rs[r].optimizer != OPT_CLIPUP) return;
  const int64_t idx = (int64_t)r * s.D + d;
  const float v = __fmul_rn(s.vec[F_ADAM_M][idx], s.gs[r].clip_inv);
  s.vec[F_ADAM_M][idx] = v;
  const float m = __fsub_rn(s.vec[F_MEAN][idx], v);
  s.vec[F_MEAN][idx] = m;
  for (int w = 0; w < pt.W; ++w)
    if (w != s.rank) __stcg(pt.vec[w][F_MEAN] + idx, m);
}

cudaError_t launch_p2p_finish(const DevState& s, const PeerTable& pt, int phase, cudaStream_t st,
                              int* nk) {
  if (nk) *nk = 0;
  const int64_t qa = s.Q * s.rank / s.W, qe = s.Q * (s.rank + 1) / s.W;
  const int64_t d0 = 4 * qa, d1 = std::min<int64_t>(4 * qe, s.D);
  const int64_t n = std::max<int64_t>(1, d1 - d0);
  const dim3 eg((unsigned)((n + 255) / 256), (unsigned)s.R);
  if (s.algo == SEP_CMA_ES) {
    p2p_sepcma_sigma_kernel<<<s.R, 32, 0, st>>>(s, pt);
    p2p_sepcma_pc_kernel<<<eg, 256, 0, st>>>(s, pt, d0, d1);
    if (nk) *nk = 2;
  } else if (phase == 0) {
    const int bps = (int)std::max<int64_t>(1, (qe - qa + TT - 1) / TT);
    p2p_clipup_norm_kernel<<<s.R, 32, 0, st>>>(s, pt, 0);
    clipup_vel_kernel<<<(unsigned)(s.R * bps), TT, 0, st>>>(s, bps, qa, qe);
    sepcma_n2_kernel<<<s.R, 256, 0, st>>>(s, bps, s.R);
    if (nk) *nk = 3;
  } else {
    p2p_clipup_norm_kernel<<<s.R, 32, 0, st>>>(s, pt, 1);
    p2p_clipup_apply_kernel<<<eg, 256, 0, st>>>(s, pt, d0, d1);
    if (nk) *nk = 2;
  }
  return cudaGetLastError();
}

// ClipUp on a D-sharded context (f1 × f3): the norms are sums of the ranks' shares, formed by
// NCCL (es_tell) or by the caller (es_tell_local / es_tell_apply), and read from s.n2:
//   after the fused tell  this rank's ‖g‖² share → s.n2 (launch_sepcma_n2)
//   phase 0               1/‖g‖ from the summed s.n2; v' = μv + lr·g/‖g‖ on the local dims; this
//                         rank's ‖v'‖² share → s.n2 (halo dims are not counted: d < Dx)
//   phase 1               the max_speed clip from the summed s.n2; v = v'·clip, m −= v.
__global__ void clipup_scalar_kernel(DevState s, int phase) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= s.R || s.rs[r].optimizer != OPT_CLIPUP) return;
  clipup_scalar(s, r, s.n2[r], phase);
}

cudaError_t launch_clipup_dshard_phase(const DevState& s, int phase, cudaStream_t st, int* nk) {
  const unsigned rb = (unsigned)((s.R + 127) / 128);
  clipup_scalar_kernel<<<rb, 128, 0, st>>>(s, phase);
  if (phase == 0) {
    const int bpr = tell_blocks_per_run(s);
    clipup_vel_kernel<<<(unsigned)(s.R * bpr), TT, 0, st>>>(s, bpr, 0, s.Q);
    sepcma_n2_kernel<<<s.R, 256, 0, st>>>(s, bpr, 0);
    if (nk) *nk = 3;
  } else {
    const int64_t n = (int64_t)s.R * s.D;
    clipup_apply_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s);
    if (nk) *nk = 2;
  }
  return cudaGetLastError();
}

}  // namespace esb
