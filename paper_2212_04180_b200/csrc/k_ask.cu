// k_ask.cu — K1 init, K2 ask (Philox noise fused with antithetic mirroring and x = m + σz), and
// the synthetic-fitness generator of the tell sweep.
//
// K2 mapping: one thread owns (run r, quad q = 4 consecutive dims) and a chunk of directions; it
// loads m and the per-dim scale once, then per direction makes ONE Philox call (4 normals) and
// writes one float4 per member row (two rows per direction for antithetic pairs). Consecutive
// threads own consecutive quads, so each warp store is a 512-B contiguous segment of one row.
// Bound: the HBM write of x (4·N·D bytes) for antithetic strategies; the Philox/Box–Muller issue
// rate for SNES / Sep-CMA (one direction per member). See DESIGN.md §Kernels.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "es_internal.h"
#include "noise.cuh"

namespace esb {

static constexpr int kAskThreads = 128;

__global__ void __launch_bounds__(256) init_kernel(DevState s) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)s.R * s.Q) return;
  const int r = (int)(gid / s.Q);
  const uint32_t q = (uint32_t)(gid % s.Q);
  const RunScal& rs = s.rs[r];
  const Philox ph(rs.seed);
  const uint4 o = ph((uint32_t)(q + s.q0), 0u, 0u, TAG_INIT);
  const float span = __fsub_rn(rs.init_max, rs.init_min);
  const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t d = 4 * (int64_t)q + k;
    if (d >= s.D) break;
    const int64_t idx = (int64_t)r * s.D + d;
    const float m = __fmaf_rn(span, uni_b(ow[k]), rs.init_min);   // N6
    s.vec[F_MEAN][idx] = m;
    s.vec[F_BEST_X][idx] = m;
    if (s.vec[F_SIGMA_D]) s.vec[F_SIGMA_D][idx] = rs.sigma_init;
    if (s.vec[F_ADAM_M]) { s.vec[F_ADAM_M][idx] = 0.0f; s.vec[F_ADAM_V][idx] = 0.0f; }
    if (s.vec[F_PSIGMA]) {
      s.vec[F_PSIGMA][idx] = 0.0f;
      s.vec[F_PC][idx] = 0.0f;
      if (s.vec[F_C]) s.vec[F_C][idx] = 1.0f;
    }
  }
}

cudaError_t launch_init(const DevState& s, cudaStream_t st) {
  const int64_t n = (int64_t)s.R * s.Q;
  init_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s);
  return cudaGetLastError();
}

// Per-dimension scale of the sample for this algorithm (N6): x = fma(±scale, z, m).
template <int ALGO>
__device__ __forceinline__ float ask_scale(const DevState& s, const RunScal& rs, int64_t idx) {
  if (ALGO == OPENAI_ES || ALGO == ARS) return rs.sigma;
  if (ALGO == PGPE || ALGO == SNES) return s.vec[F_SIGMA_D][idx];
  return __fmul_rn(rs.sigma, __fsqrt_rn(s.vec[F_C][idx]));
}

// IMG 1: also write fp16(x) into x16 (N14′, the MLP fitness's parameter image); IMG 2: write the
// split image of N14 — plane 0 fp16(x·2^8), plane 1 fp16(x·2^8 − hi), planes R·Nloc·D apart (the
// fp32-accurate MLP's operands). x may be NULL with an image.
// CLIP: clamp the members into the run's box [clip_lo, clip_hi] (the z the tell regenerates
// is unclipped). Instantiated only when some run has bounds.
__device__ __forceinline__ void store_img(__half* h, const float* v, int mode, int64_t plane) {
  if (mode == 1) {
    __half2 a0 = __floats2half2_rn(v[0], v[1]), a1 = __floats2half2_rn(v[2], v[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a0);
    u.y = *reinterpret_cast<uint32_t*>(&a1);
    __stcs(reinterpret_cast<uint2*>(h), u);
  } else {                                  // mode 2: v is already x·2⁸ (see ask_kernel)
    float r[4];
    const float* sc = v;
    __half2 a0 = __floats2half2_rn(sc[0], sc[1]), a1 = __floats2half2_rn(sc[2], sc[3]);
    const float2 b0 = __half22float2(a0), b1 = __half22float2(a1);
    r[0] = __fsub_rn(sc[0], b0.x); r[1] = __fsub_rn(sc[1], b0.y);
    r[2] = __fsub_rn(sc[2], b1.x); r[3] = __fsub_rn(sc[3], b1.y);
    __half2 c0 = __floats2half2_rn(r[0], r[1]), c1 = __floats2half2_rn(r[2], r[3]);
    uint2 u, w;
    u.x = *reinterpret_cast<uint32_t*>(&a0);
    u.y = *reinterpret_cast<uint32_t*>(&a1);
    w.x = *reinterpret_cast<uint32_t*>(&c0);
    w.y = *reinterpret_cast<uint32_t*>(&c1);
    __stcs(reinterpret_cast<uint2*>(h), u);
    __stcs(reinterpret_cast<uint2*>(h + plane), w);
  }
}

template <int ALGO, bool V4, int IMG, bool CLIP>
__global__ void __launch_bounds__(kAskThreads) ask_kernel(DevState s, float* __restrict__ x,
                                                           __half* __restrict__ x16, int bpr,
                                                           int dpt) {
  pdl_enter();
  constexpr bool kAnti = is_anti(ALGO);
  const int r = blockIdx.x / bpr;
  const int64_t q = (int64_t)(blockIdx.x % bpr) * kAskThreads + threadIdx.x;
  if (q >= s.Qx) return;
  const int Ploc = kAnti ? s.Nloc / 2 : s.Nloc;
  const int i0 = blockIdx.y * dpt;
  const int i1 = min(Ploc, i0 + dpt);
  if (i0 >= i1) return;
  const RunScal& rs = s.rs[r];
  const Philox ph(rs.seed);
  const uint32_t t = rs.t;
  const int64_t base = (int64_t)r * s.D + 4 * q;
  // IMG 2 (the split image of x·2⁸): m, the scale and the box are pre-multiplied by 2⁸, so the
  // FFMA yields x·2⁸ directly — fma(2⁸σ, z, 2⁸m) = 2⁸·fma(σ, z, m) exactly (a power of two), and
  // so is the clamp; x itself, when written, is that times 2⁻⁸ (exact)
  constexpr float kPre = IMG == 2 ? 256.0f : 1.0f;
  float m[4], sc[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool ok = 4 * q + k < s.D;
    m[k] = ok ? __fmul_rn(s.vec[F_MEAN][base + k], kPre) : 0.0f;
    sc[k] = ok ? __fmul_rn(ask_scale<ALGO>(s, rs, base + k), kPre) : 0.0f;
  }
  const int dir0 = s.rank * Ploc;
  const float lo = CLIP ? __fmul_rn(rs.clip_lo, kPre) : 0.0f, hi = CLIP ? __fmul_rn(rs.clip_hi, kPre) : 0.0f;
  // row pointers advance by one direction's rows per iteration (no per-iteration 64-bit multiply)
  const int64_t step = (kAnti ? 2 : 1) * s.Dx;
  const int64_t first = (int64_t)r * s.Nloc * s.Dx + 4 * q + (int64_t)i0 * step;
  float* p0 = x ? x + first : nullptr;
  __half* h0 = IMG ? x16 + first : nullptr;
  const int64_t plane = (int64_t)s.R * s.Nloc * s.Dx;     // IMG 2: hi → lo plane distance
#pragma unroll 4
  for (int il = i0; il < i1; ++il, p0 += (x ? step : 0), h0 += (IMG ? step : 0)) {
    const float4 z = normal4(ph, (uint32_t)(q + s.q0), (uint32_t)(dir0 + il), t);
    const float zz[4] = {z.x, z.y, z.z, z.w};
    float xp[4], xm[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      xp[k] = __fmaf_rn(sc[k], zz[k], m[k]);
      if (kAnti) xm[k] = __fmaf_rn(-sc[k], zz[k], m[k]);
      if (CLIP) {
        xp[k] = fminf(fmaxf(xp[k], lo), hi);
        if (kAnti) xm[k] = fminf(fmaxf(xm[k], lo), hi);
      }
    }
    if (IMG) {            // D % 4 == 0 is required for this path (8-byte stores)
      store_img(h0, xp, IMG, plane);
      if (kAnti) store_img(h0 + s.Dx, xm, IMG, plane);
      if (!p0) continue;
      if (IMG == 2) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          xp[k] = __fmul_rn(xp[k], 1.0f / 256.0f);
          if (kAnti) xm[k] = __fmul_rn(xm[k], 1.0f / 256.0f);
        }
      }
    }
    if (V4) {
      __stcs(reinterpret_cast<float4*>(p0), make_float4(xp[0], xp[1], xp[2], xp[3]));
      if (kAnti)
        __stcs(reinterpret_cast<float4*>(p0 + s.Dx), make_float4(xm[0], xm[1], xm[2], xm[3]));
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (4 * q + k < s.Dx) {
          p0[k] = xp[k];
          if (kAnti) p0[s.Dx + k] = xm[k];
        }
      }
    }
  }
}

template <int ALGO, bool CLIP>
static cudaError_t launch_ask_t(const DevState& s, float* x, __half* x16, int img, cudaStream_t st) {
  constexpr bool kAnti = is_anti(ALGO);
  const int Ploc = kAnti ? s.Nloc / 2 : s.Nloc;
  const int bpr = (int)((s.Qx + kAskThreads - 1) / kAskThreads);
  // Enough (thread, direction-chunk) items for ~4 waves of 16 warps/SM, ≥ 16 directions each.
  const int64_t quads = (int64_t)s.R * bpr * kAskThreads;
  const int64_t want = (int64_t)sm_count() * 2048 * 4;
  int nchunk = (int)std::min<int64_t>(std::max<int64_t>(1, want / std::max<int64_t>(quads, 1)),
                                      std::max(1, Ploc / 16));   // ≥ 16 directions per thread (C3: 16 vs 4 = 27.1 vs 29.3 µs)
  nchunk = std::min(nchunk, 65535);
  if (const char* e = std::getenv("ES_ASK_DPT")) {     // A/B switch for profiling
    const int d = std::max(1, std::atoi(e));
    nchunk = std::max(1, std::min(65535, (Ploc + d - 1) / d));
  }
  const int dpt = (Ploc + nchunk - 1) / nchunk;
  nchunk = (Ploc + dpt - 1) / dpt;
  dim3 grid((unsigned)(s.R * bpr), (unsigned)nchunk);
  const dim3 blk(kAskThreads);
  if (x16 && img == 2) return launch_pdl(ask_kernel<ALGO, true, 2, CLIP>, grid, blk, 0, st, s, x, x16, bpr, dpt);
  if (x16) return launch_pdl(ask_kernel<ALGO, true, 1, CLIP>, grid, blk, 0, st, s, x, x16, bpr, dpt);
  const bool v4 = (s.Dx % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  __half* none = nullptr;
  if (v4) return launch_pdl(ask_kernel<ALGO, true, 0, CLIP>, grid, blk, 0, st, s, x, none, bpr, dpt);
  return launch_pdl(ask_kernel<ALGO, false, 0, CLIP>, grid, blk, 0, st, s, x, none, bpr, dpt);
}

template <bool CLIP>
static cudaError_t launch_ask_c(const DevState& s, float* x, __half* x16, int img, cudaStream_t st) {
  switch (s.algo) {
    case OPENAI_ES: return launch_ask_t<OPENAI_ES, CLIP>(s, x, x16, img, st);
    case PGPE: return launch_ask_t<PGPE, CLIP>(s, x, x16, img, st);
    case SNES: return launch_ask_t<SNES, CLIP>(s, x, x16, img, st);
    case ARS: return launch_ask_t<ARS, CLIP>(s, x, x16, img, st);
    default: return launch_ask_t<SEP_CMA_ES, CLIP>(s, x, x16, img, st);
  }
}

cudaError_t launch_ask16(const DevState& s, float* x, __half* x16, cudaStream_t st) {
  return s.any_clip ? launch_ask_c<true>(s, x, x16, 1, st) : launch_ask_c<false>(s, x, x16, 1, st);
}

// N14 split image (plane distance R·Nloc·D), x optional
cudaError_t launch_ask_split(const DevState& s, float* x, __half* img, cudaStream_t st) {
  return s.any_clip ? launch_ask_c<true>(s, x, img, 2, st) : launch_ask_c<false>(s, x, img, 2, st);
}

cudaError_t launch_ask(const DevState& s, float* x, cudaStream_t st) {
  return launch_ask16(s, x, nullptr, st);
}

// N15: f_j = u_b(o_{j mod 4}) of counter (⌊j/4⌋, 0, t, 4), for this rank's members.
__global__ void synth_kernel(DevState s, float* __restrict__ f) {
  pdl_enter();
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)s.R * s.Nloc) return;
  const int r = (int)(gid / s.Nloc);
  const int jl = (int)(gid % s.Nloc);
  const int j = s.rank * s.Nloc + jl;
  const RunScal& rs = s.rs[r];
  const Philox ph(rs.seed);
  const uint4 o = ph((uint32_t)(j / 4), 0u, rs.t, TAG_SYNTH);
  const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
  f[gid] = uni_b(ow[j % 4]);
}

cudaError_t launch_synth(const DevState& s, float* f, cudaStream_t st) {
  const int64_t n = (int64_t)s.R * s.Nloc;
  return launch_pdl(synth_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, st, s, f);
}

}  // namespace esb
