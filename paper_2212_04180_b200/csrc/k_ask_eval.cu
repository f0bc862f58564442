// k_ask_eval.cu — K8: fused ask + BBOB evaluate.
//
// The ask kernel's thread mapping (run, 4-dim quad, chunk of directions) is kept; after forming
// the member rows x = m ± σ⊙z (N6) the thread adds their Sphere / Rosenbrock / Rastrigin terms
// (N7, binary64) and the warp reduces them per member, so x never has to be re-read from HBM and
// — when the caller passes x = NULL — is never materialised at all (memory O(R·D)). Per
// (member, 512-dim block) the partial goes to a small binary64 buffer; a finalize kernel sums the
// blocks of each member in fixed order (deterministic, run to run and across launch shapes).
// Rosenbrock's cross-quad pair (x_{4q+3}, x_{4q+4}) comes from the next lane by shuffle; lane 31
// regenerates the first normal of quad q+1 itself (one extra Philox call per 32 quads).
#include <algorithm>

#include "es_internal.h"
#include "fitness.cuh"

namespace esb {

static constexpr int kAE = 128;      // threads per block (4 warps, 512 dims)
static constexpr int kMaxDpt = 32;   // directions per thread-chunk (red buffer bound)
static constexpr int kAEB = 8;       // directions per batch of the warp's column sums

template <int ALGO>
__device__ __forceinline__ float ae_scale(const DevState& s, const RunScal& rs, int64_t idx) {
  if (ALGO == OPENAI_ES || ALGO == ARS) return rs.sigma;
  if (ALGO == PGPE || ALGO == SNES) return s.vec[F_SIGMA_D][idx];
  return __fmul_rn(rs.sigma, __fsqrt_rn(s.vec[F_C][idx]));
}

template <int ALGO, int FN, bool WX, bool V4>
__global__ void __launch_bounds__(kAE) ask_eval_kernel(DevState s, float* __restrict__ x,
                                                       double* __restrict__ part, int bpr,
                                                       int dpt) {
  constexpr bool kAnti = is_anti(ALGO);
  constexpr int M = kAnti ? 2 : 1;
  __shared__ double red[4][kMaxDpt * 2];
  // per warp: each lane's binary64 partial of the batch's members, [member][lane] with a 33-word
  // row pitch (the column sums below read down a row: no bank conflicts)
  __shared__ double col[4][kAEB * M][33];
  const int r = blockIdx.x / bpr, qb = blockIdx.x % bpr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t q = (int64_t)qb * kAE + threadIdx.x;
  const bool active = q < s.Q;    // state quads: a D-shard's halo quad feeds the shuffled xn
  const int Ploc = kAnti ? s.Nloc / 2 : s.Nloc;
  const int i0 = blockIdx.y * dpt, i1 = min(Ploc, i0 + dpt);
  if (i0 >= i1) return;                               // block-uniform
  const RunScal& rs = s.rs[r];
  const Philox ph(rs.seed);
  const uint32_t t = rs.t;
  const int64_t base = (int64_t)r * s.D + 4 * q;
  float m[4], sc[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool ok = active && 4 * q + k < s.D;
    m[k] = ok ? s.vec[F_MEAN][base + k] : 0.0f;
    sc[k] = ok ? ae_scale<ALGO>(s, rs, base + k) : 0.0f;
  }
  // Rosenbrock successor of this quad's last element (dim 4q+4), needed by lane 31 only
  const bool has_next = active && 4 * q + 4 < s.D;
  float mN = 0.0f, scN = 0.0f;
  if (FN == FN_ROSENBROCK && lane == 31 && has_next) {
    mN = s.vec[F_MEAN][base + 4];
    scN = ae_scale<ALGO>(s, rs, base + 4);
  }
  const int dir0 = s.rank * Ploc;
  const bool clip = rs.clip != 0;                     // box bounds, block-uniform
  const float lo = rs.clip_lo, hi = rs.clip_hi;
  float* xr = x ? x + (int64_t)r * s.Nloc * s.Dx + 4 * q : nullptr;
  for (int ib = i0; ib < i1; ib += kAEB) {
    const int ie = min(i1, ib + kAEB);
#pragma unroll 2
    for (int il = ib; il < ie; ++il) {
      const uint32_t dir = (uint32_t)(dir0 + il);
      const float4 z = normal4(ph, (uint32_t)(q + s.q0), dir, t);
      const float zz[4] = {z.x, z.y, z.z, z.w};
      float xv[M][4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        xv[0][k] = __fmaf_rn(sc[k], zz[k], m[k]);
        if (kAnti) xv[M - 1][k] = __fmaf_rn(-sc[k], zz[k], m[k]);
        if (clip) {
#pragma unroll
          for (int h = 0; h < M; ++h) xv[h][k] = fminf(fmaxf(xv[h][k], lo), hi);
        }
      }
      if (WX && q < s.Qx) {                             // owned quads only
        const int64_t row = kAnti ? 2 * (int64_t)il : il;
#pragma unroll
        for (int h = 0; h < M; ++h) {
          float* p0 = xr + (row + h) * s.Dx;
          if (V4) {
            __stcs(reinterpret_cast<float4*>(p0), make_float4(xv[h][0], xv[h][1], xv[h][2], xv[h][3]));
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (4 * q + k < s.Dx) p0[k] = xv[h][k];
          }
        }
      }
      float nx[M];
#pragma unroll
      for (int h = 0; h < M; ++h) nx[h] = 0.0f;
      if (FN == FN_ROSENBROCK) {
#pragma unroll
        for (int h = 0; h < M; ++h) nx[h] = __shfl_down_sync(0xffffffffu, xv[h][0], 1);
        if (lane == 31 && has_next) {
          const float zN = normal4(ph, (uint32_t)(q + 1 + s.q0), dir, t).x;
          nx[0] = __fmaf_rn(scN, zN, mN);
          if (kAnti) nx[M - 1] = __fmaf_rn(-scN, zN, mN);
          if (clip) {
#pragma unroll
            for (int h = 0; h < M; ++h) nx[h] = fminf(fmaxf(nx[h], lo), hi);
          }
        }
      }
#pragma unroll
      for (int h = 0; h < M; ++h) {
        FitAcc acc;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t d = 4 * q + k;
          if (active && d < s.Dx) {                    // a D-shard's halo dim only feeds xn
            const float xn = k < 3 ? xv[h][k + 1] : nx[h];
            fit_add<FN>(acc, xv[h][k], xn, d + 1 < s.D);
          }
        }
        col[warp][M * (il - ib) + h][lane] = fit_total<FN>(acc);
      }
    }
    // the members' sums over the warp's 32 lanes, one member per lane, in lane order (instead of a
    // 5-round shuffle reduction per member: the reduction cost per member falls from 15 warp
    // instructions to 2 × 32 / (8·M) plus one store)
    __syncwarp();
    if (lane < M * (ie - ib)) {
      double v = 0.0;
#pragma unroll 8
      for (int k = 0; k < 32; ++k) v = __dadd_rn(v, col[warp][lane][k]);
      red[warp][M * (ib - i0) + lane] = v;
    }
    __syncwarp();
  }
  __syncthreads();
  const int cnt = M * (i1 - i0);
  for (int idx = threadIdx.x; idx < cnt; idx += kAE) {
    const double v = __dadd_rn(__dadd_rn(__dadd_rn(red[0][idx], red[1][idx]), red[2][idx]),
                               red[3][idx]);
    const int jl = M * i0 + idx;                     // local member index
    part[((int64_t)r * s.Nloc + jl) * bpr + qb] = v;
  }
}

// f (fp32) or, for a D-shard, the member's binary64 partial over the owned dims (fpart).
__global__ void ae_finalize_kernel(const double* __restrict__ part, int64_t rows, int bpr,
                                   float* __restrict__ f, double* __restrict__ fpart) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= rows) return;
  double v = 0.0;
  for (int b = 0; b < bpr; ++b) v = __dadd_rn(v, part[j * bpr + b]);
  if (fpart) fpart[j] = v;
  else f[j] = (float)v;
}

__global__ void partial_to_fitness_kernel(const double* __restrict__ fsum, int64_t n,
                                          float* __restrict__ f) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) f[j] = (float)fsum[j];
}

cudaError_t launch_partial_to_fitness(const double* fsum, int64_t n, float* f, cudaStream_t st) {
  partial_to_fitness_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(fsum, n, f);
  return cudaGetLastError();
}

// Weight decay: out_j = f_j + λ_r Σ_b part[j][b] (the member's ‖x_j‖², binary64).
__global__ void wd_finalize_kernel(DevState s, const double* __restrict__ part, int bpr,
                                   const float* f, float* out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= (int64_t)s.R * s.Nloc) return;
  const float wd = s.rs[j / s.Nloc].weight_decay;
  const float fj = f[j];
  if (wd == 0.0f) { out[j] = fj; return; }
  double v = 0.0;
  for (int b = 0; b < bpr; ++b) v = __dadd_rn(v, part[j * bpr + b]);
  out[j] = (float)__dadd_rn((double)fj, __dmul_rn((double)wd, v));
}

int ask_eval_blocks_per_run(const DevState& s) { return (int)((s.Q + kAE - 1) / kAE); }

template <int ALGO, int FN>
static void launch_ae_t(const DevState& s, float* x, double* part, dim3 grid, int bpr, int dpt,
                        cudaStream_t st) {
  const bool v4 = x && (s.Dx % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  if (!x) ask_eval_kernel<ALGO, FN, false, false><<<grid, kAE, 0, st>>>(s, x, part, bpr, dpt);
  else if (v4) ask_eval_kernel<ALGO, FN, true, true><<<grid, kAE, 0, st>>>(s, x, part, bpr, dpt);
  else ask_eval_kernel<ALGO, FN, true, false><<<grid, kAE, 0, st>>>(s, x, part, bpr, dpt);
}

template <int ALGO>
static void launch_ae_a(int fn, const DevState& s, float* x, double* part, dim3 grid, int bpr,
                        int dpt, cudaStream_t st) {
  if (fn == FN_SPHERE) launch_ae_t<ALGO, FN_SPHERE>(s, x, part, grid, bpr, dpt, st);
  else if (fn == FN_ROSENBROCK) launch_ae_t<ALGO, FN_ROSENBROCK>(s, x, part, grid, bpr, dpt, st);
  else launch_ae_t<ALGO, FN_RASTRIGIN>(s, x, part, grid, bpr, dpt, st);
}

static dim3 ae_grid(const DevState& s, int& bpr, int& dpt) {
  const bool anti = is_anti(s.algo);
  const int Ploc = anti ? s.Nloc / 2 : s.Nloc;
  bpr = ask_eval_blocks_per_run(s);
  const int64_t quads = (int64_t)s.R * bpr * kAE;
  const int64_t want = (int64_t)sm_count() * 2048 * 4;
  int nchunk = (int)std::max<int64_t>(1, want / std::max<int64_t>(quads, 1));
  nchunk = std::max(nchunk, (Ploc + kMaxDpt - 1) / kMaxDpt);
  nchunk = std::min(nchunk, std::max(1, Ploc));
  dpt = (Ploc + nchunk - 1) / nchunk;
  nchunk = (Ploc + dpt - 1) / dpt;
  return dim3((unsigned)(s.R * bpr), (unsigned)nchunk);
}

// ‖x_j‖² of the regenerated (clipped) members = the Sphere pass of the fused kernel without the
// x write, then the weight-decay finalize.
cudaError_t launch_weight_decay(const DevState& s, double* part, const float* f, float* out,
                                cudaStream_t st) {
  int bpr, dpt;
  const dim3 grid = ae_grid(s, bpr, dpt);
  switch (s.algo) {
    case OPENAI_ES: launch_ae_t<OPENAI_ES, FN_SPHERE>(s, nullptr, part, grid, bpr, dpt, st); break;
    case PGPE: launch_ae_t<PGPE, FN_SPHERE>(s, nullptr, part, grid, bpr, dpt, st); break;
    case SNES: launch_ae_t<SNES, FN_SPHERE>(s, nullptr, part, grid, bpr, dpt, st); break;
    case ARS: launch_ae_t<ARS, FN_SPHERE>(s, nullptr, part, grid, bpr, dpt, st); break;
    default: launch_ae_t<SEP_CMA_ES, FN_SPHERE>(s, nullptr, part, grid, bpr, dpt, st); break;
  }
  const int64_t rows = (int64_t)s.R * s.Nloc;
  wd_finalize_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(s, part, bpr, f, out);
  return cudaGetLastError();
}

// out = f + weight_decay·‖x‖² from per-member squared norms already summed (over the D-shard
// ranks): the finalize with one partial per member.
cudaError_t launch_wd_apply(const DevState& s, const double* sqnorm, const float* f, float* out,
                            cudaStream_t st) {
  const int64_t rows = (int64_t)s.R * s.Nloc;
  wd_finalize_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(s, sqnorm, 1, f, out);
  return cudaGetLastError();
}

static cudaError_t ask_eval_impl(const DevState& s, int fn, float* x, double* part, float* f,
                                 double* fpart, cudaStream_t st);

cudaError_t launch_ask_eval(const DevState& s, int fn, float* x, double* part, float* f,
                            cudaStream_t st) {
  return ask_eval_impl(s, fn, x, part, f, nullptr, st);
}

cudaError_t launch_ask_eval_partial(const DevState& s, int fn, float* x, double* part,
                                    double* fpart, cudaStream_t st) {
  return ask_eval_impl(s, fn, x, part, nullptr, fpart, st);
}

// Two kernels: the fused ask+evaluate and the per-member block sum.
static cudaError_t ask_eval_impl(const DevState& s, int fn, float* x, double* part, float* f,
                                 double* fpart, cudaStream_t st) {
  int bpr, dpt;
  const dim3 grid = ae_grid(s, bpr, dpt);
  switch (s.algo) {
    case OPENAI_ES: launch_ae_a<OPENAI_ES>(fn, s, x, part, grid, bpr, dpt, st); break;
    case PGPE: launch_ae_a<PGPE>(fn, s, x, part, grid, bpr, dpt, st); break;
    case SNES: launch_ae_a<SNES>(fn, s, x, part, grid, bpr, dpt, st); break;
    case ARS: launch_ae_a<ARS>(fn, s, x, part, grid, bpr, dpt, st); break;
    default: launch_ae_a<SEP_CMA_ES>(fn, s, x, part, grid, bpr, dpt, st); break;
  }
  const int64_t rows = (int64_t)s.R * s.Nloc;
  ae_finalize_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(part, rows, bpr, f, fpart);
  return cudaGetLastError();
}

}  // namespace esb
