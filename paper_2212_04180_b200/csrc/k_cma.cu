// k_cma.cu — SURVEY §8(f) row f4: full-covariance CMA-ES ("weighted recombination-based mean
// updates and iterative covariance matrix estimation ... evolution paths"; Table 1) with the
// sampling reparametrisation the paper names, "the Cholesky decomposition of a covariance matrix"
// (P:106). Readings in DESIGN.md §2 (R-CMA).
//
// One generation, R runs batched in the grid:
//   ask   K-z      z_j = N2 normals (counter (⌊d/4⌋, j, t, ASK)), stored [R][N][D]
//         K-samp   Y = Z·Aᵀ (A lower-triangular: an output tile's K range stops at its last dim),
//                  x = clip(m + σ·y); Y stored for the tell
//   tell  (rank kernel as Sep-CMA-ES: weights by sorted position)
//         K-vec    ȳ = Σ w_j y_j, z̄ = Σ w_j z_j (binary64) → m, p_σ, ‖p_σ‖² partials, best_x
//         (sepcma_norm_kernel: σ', h_σ)    K-pc  p_c
//         K-cov    C ← a·C + c₁ p_c p_cᵀ + c_μ Σ w_j y_j y_jᵀ on lower tiles, mirrored (exactly symmetric)
//         K-chol   every k-th tell: blocked right-looking Cholesky of C (64-wide panels: diagonal
//                  block in binary64 in shared memory, row-parallel triangular solve, tiled trailing
//                  update); a run whose C is not positive definite keeps its previous factor.
// The contractions here are FP32 FFMA tiles on the CUDA cores.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "es_internal.h"
#include "noise.cuh"

namespace esb {

static constexpr int kTB = 64;    // output tile (rows × cols)
static constexpr int kTK = 16;    // K step
static constexpr int kNB = 64;    // Cholesky panel width

__global__ void cma_init_kernel(DevState s) {
  const int64_t DD = s.D * s.D, n = (int64_t)s.R * DD;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rem = g % DD;
    const float v = (rem / s.D == rem % s.D) ? 1.0f : 0.0f;
    s.cov[g] = v;
    s.chol[g] = v;
  }
  if (blockIdx.x == 0)
    for (int r = threadIdx.x; r < s.R; r += blockDim.x) s.chol_fail[r] = 0;
}

cudaError_t launch_cma_init(const DevState& s, cudaStream_t st) {
  const int64_t n = (int64_t)s.R * s.D * s.D;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
  cma_init_kernel<<<std::max(blocks, 1), 256, 0, st>>>(s);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------- ask
__global__ void __launch_bounds__(128) cma_z_kernel(DevState s, int bpr, int jpb) {
  const int r = blockIdx.x / bpr;
  const int64_t q = (int64_t)(blockIdx.x % bpr) * 128 + threadIdx.x;
  if (q >= s.Q) return;
  const int j0 = blockIdx.y * jpb, j1 = min(s.N, j0 + jpb);
  const RunScal& rs = s.rs[r];
  const Philox ph(rs.seed);
  const uint32_t t = rs.t;
  const bool v4 = (s.D & 3) == 0;
  for (int j = j0; j < j1; ++j) {
    const float4 z = normal4(ph, (uint32_t)(q + s.q0), (uint32_t)j, t);
    float* p = s.zbuf + ((int64_t)r * s.N + j) * s.D + 4 * q;
    if (v4) {
      *reinterpret_cast<float4*>(p) = z;
    } else {
      const float zz[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (4 * q + k < s.D) p[k] = zz[k];
    }
  }
}

// Y = Z·Aᵀ for one 64-member × 64-dim tile of run blockIdx.z; 256 threads × (4 members × 4 dims),
// FP32 FFMA in k order. Epilogue x = clip(fma(σ, y, m)) — the same expression best_x uses. Every
// rank samples all N members (Y feeds the replicated tell); x holds only this rank's members
// [rank·Nloc, (rank+1)·Nloc), locally indexed (population sharding).
__global__ void __launch_bounds__(256) cma_sample_kernel(DevState s, float* __restrict__ x) {
  __shared__ __align__(16) float Zs[kTK][kTB + 4];
  __shared__ __align__(16) float As[kTK][kTB + 4];
  const int r = blockIdx.z;
  const int64_t D = s.D;
  const int d0 = blockIdx.x * kTB, j0 = blockIdx.y * kTB;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const float* Z = s.zbuf + (int64_t)r * s.N * D;
  const float* A = s.chol + (int64_t)r * D * D;
  const int lr = threadIdx.x >> 2, lk = (threadIdx.x & 3) * 4;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) acc[i][jj] = 0.0f;
  const int kend = (int)std::min<int64_t>(D, d0 + kTB);      // A[d][k] = 0 for k > d
  for (int k0 = 0; k0 < kend; k0 += kTK) {
    const int jr = j0 + lr, dr = d0 + lr;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + lk + u;
      Zs[lk + u][lr] = (jr < s.N && k < D) ? Z[(int64_t)jr * D + k] : 0.0f;
      As[lk + u][lr] = (dr < D && k < D) ? A[(int64_t)dr * D + k] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&Zs[kk][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&As[kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) acc[i][jj] = __fmaf_rn(av[i], bv[jj], acc[i][jj]);
    }
    __syncthreads();
  }
  const RunScal& rs = s.rs[r];
  const float sig = rs.sigma;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int j = j0 + ty * 4 + i;
    if (j >= s.N) continue;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int d = d0 + tx * 4 + jj;
      if (d >= D) continue;
      const int64_t o = ((int64_t)r * s.N + j) * D + d;
      s.ybuf[o] = acc[i][jj];
      const int jl = j - s.rank * s.Nloc;
      if (x && jl >= 0 && jl < s.Nloc) {
        float xv = __fmaf_rn(sig, acc[i][jj], s.vec[F_MEAN][(int64_t)r * D + d]);
        if (rs.clip) xv = fminf(fmaxf(xv, rs.clip_lo), rs.clip_hi);
        x[((int64_t)r * s.Nloc + jl) * D + d] = xv;
      }
    }
  }
}

cudaError_t launch_cma_ask(const DevState& s, float* x, cudaStream_t st, int* nk) {
  const int bpr = (int)((s.Q + 127) / 128);
  const int64_t quads = (int64_t)s.R * bpr * 128;
  const int64_t want = (int64_t)sm_count() * 2048 * 4;
  int nchunk = (int)std::min<int64_t>(std::max<int64_t>(1, want / std::max<int64_t>(quads, 1)),
                                      std::max(1, s.N / 4));
  nchunk = std::min(nchunk, 65535);
  const int jpb = (s.N + nchunk - 1) / nchunk;
  nchunk = (s.N + jpb - 1) / jpb;
  cma_z_kernel<<<dim3((unsigned)(s.R * bpr), (unsigned)nchunk), 128, 0, st>>>(s, bpr, jpb);
  static const bool simt = std::getenv("ES_CMA_SIMT") != nullptr;   // A/B switch for profiling
  if (!simt && cma_tc_supported(s)) {
    const cudaError_t e = launch_cma_sample_tc(s, x, st);
    if (nk) *nk = 2;
    return e;
  }
  const dim3 g((unsigned)((s.D + kTB - 1) / kTB), (unsigned)((s.N + kTB - 1) / kTB), (unsigned)s.R);
  cma_sample_kernel<<<g, 256, 0, st>>>(s, x);
  if (nk) *nk = 2;
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------ tell
__device__ __forceinline__ double block_sum128(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) t = __dadd_rn(t, red[k]);
  return t;
}

// ȳ, z̄ over the weighted sorted positions; m, p_σ, best_x; ȳ to s.G[0] for p_c and C.
// Block = 32 dims × 8 entry groups (each group sums every 8th entry, the groups are then added in
// group order: a fixed summation order); grid = R × ⌈D/32⌉.
static constexpr int kVecDims = 32, kVecGroups = 8;
__global__ void __launch_bounds__(256) cma_tellvec_kernel(DevState s, int bpr) {
  __shared__ double sy[kVecGroups][kVecDims], sz[kVecGroups][kVecDims];
  const int r = blockIdx.y;
  const int lane = threadIdx.x & (kVecDims - 1), grp = threadIdx.x / kVecDims;
  const int64_t D = s.D;
  const int64_t d = (int64_t)blockIdx.x * kVecDims + lane;
  const GenScal& gs = s.gs[r];
  const RunScal& rs = s.rs[r];
  const int ne = gs.nentries;
  const uint32_t* dir = s.dir + (int64_t)r * s.N;
  const double* cA = s.coefA + (int64_t)r * s.N;
  const float* Y = s.ybuf + (int64_t)r * s.N * D;
  const float* Z = s.zbuf + (int64_t)r * s.N * D;
  double yb = 0.0, zb = 0.0;
  if (d < D) {
    for (int e = grp; e < ne; e += kVecGroups) {
      const int64_t row = (int64_t)dir[e] * D;
      const double w = cA[e];
      yb = __fma_rn(w, (double)Y[row + d], yb);
      zb = __fma_rn(w, (double)Z[row + d], zb);
    }
  }
  sy[grp][lane] = yb;
  sz[grp][lane] = zb;
  __syncthreads();
  if (grp != 0) return;
  yb = zb = 0.0;
#pragma unroll
  for (int k = 0; k < kVecGroups; ++k) {
    yb = __dadd_rn(yb, sy[k][lane]);
    zb = __dadd_rn(zb, sz[k][lane]);
  }
  double norm2 = 0.0;
  if (d < D) {
    const float omcs = (float)__dsub_rn(1.0, rs.c_sigma);
    const float ks = (float)sqrt(__dmul_rn(__dmul_rn(rs.c_sigma, __dsub_rn(2.0, rs.c_sigma)), rs.mueff));
    const int64_t idx = (int64_t)r * D + d;
    const float mean = s.vec[F_MEAN][idx];
    if (gs.improved) {                             // the member as asked (pre-update m, σ)
      float xb = __fmaf_rn(gs.sigma, Y[(int64_t)gs.jbest * D + d], mean);
      if (rs.clip) xb = fminf(fmaxf(xb, rs.clip_lo), rs.clip_hi);
      s.vec[F_BEST_X][idx] = xb;
    }
    s.vec[F_MEAN][idx] = __fadd_rn(mean, __fmul_rn(gs.sigma, (float)yb));
    const float ps = __fadd_rn(__fmul_rn(omcs, s.vec[F_PSIGMA][idx]), __fmul_rn(ks, (float)zb));
    s.vec[F_PSIGMA][idx] = ps;
    norm2 = __dmul_rn((double)ps, (double)ps);
    s.G[idx] = yb;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) norm2 = __dadd_rn(norm2, __shfl_xor_sync(0xffffffffu, norm2, o));
  if (lane == 0) s.normpart[(int64_t)r * bpr + blockIdx.x] = norm2;
}

// σ', h_σ from the per-block ‖p_σ'‖² partials (bpr = ⌈D/32⌉ of them per run)
__global__ void cma_norm_kernel(DevState s, int bpr) {
  __shared__ double red[32];
  const int r = blockIdx.x;
  double v = 0.0;
  for (int b = threadIdx.x; b < bpr; b += blockDim.x) v = __dadd_rn(v, s.normpart[(int64_t)r * bpr + b]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double n2 = 0.0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) n2 = __dadd_rn(n2, red[k]);
  RunScal& rs = s.rs[r];
  GenScal& gs = s.gs[r];
  const double norm = sqrt(n2);
  const float sig_new = __fmul_rn(
      gs.sigma, (float)exp(__dmul_rn(__ddiv_rn(rs.c_sigma, rs.d_sigma),
                                     __dsub_rn(__ddiv_rn(norm, rs.chi_d), 1.0))));
  const double lhs = norm / sqrt(1.0 - pow(1.0 - rs.c_sigma, 2.0 * (double)(gs.t + 1)));
  gs.hsig = lhs < (1.4 + 2.0 / ((double)s.Dg + 1.0)) * rs.chi_d;
  gs.sigma_new = sig_new;
  rs.sigma = sig_new;
}

__global__ void __launch_bounds__(256) cma_pc_kernel(DevState s) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)s.R * s.D) return;
  const int r = (int)(gid / s.D);
  const RunScal& rs = s.rs[r];
  const GenScal& gs = s.gs[r];
  const float omcc = (float)(1.0 - rs.c_c);
  const float kc = gs.hsig ? (float)sqrt(rs.c_c * (2.0 - rs.c_c) * rs.mueff) : 0.0f;
  s.vec[F_PC][gid] = __fadd_rn(__fmul_rn(omcc, s.vec[F_PC][gid]), __fmul_rn(kc, (float)s.G[gid]));
}

// C ← a·C + c₁ p_c p_cᵀ + c_μ Σ_e w_e y_e y_eᵀ (lower tiles; mirrored).
__global__ void __launch_bounds__(256) cma_cov_kernel(DevState s) {
  __shared__ __align__(16) float Ui[kTK][kTB + 4];
  __shared__ __align__(16) float Uj[kTK][kTB + 4];
  const int r = blockIdx.y;
  int I, J;
  lower_tile(blockIdx.x, I, J);
  const int64_t D = s.D;
  const int i0 = I * kTB, j0 = J * kTB;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const GenScal& gs = s.gs[r];
  const RunScal& rs = s.rs[r];
  const int ne = gs.nentries;
  const uint32_t* dir = s.dir + (int64_t)r * s.N;
  const double* cA = s.coefA + (int64_t)r * s.N;
  const float* Y = s.ybuf + (int64_t)r * s.N * D;
  float acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0f;
  const int le = threadIdx.x >> 4, lc = (threadIdx.x & 15) * 4;   // 16 entries × 64 cols
  for (int e0 = 0; e0 < ne; e0 += kTK) {
    const int e = e0 + le;
    const bool ok = e < ne;
    const int64_t row = ok ? (int64_t)dir[e] * D : 0;
    const float w = ok ? (float)cA[e] : 0.0f;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int ci = i0 + lc + u, cj = j0 + lc + u;
      Ui[le][lc + u] = (ok && ci < D) ? __fmul_rn(w, Y[row + ci]) : 0.0f;
      Uj[le][lc + u] = (ok && cj < D) ? Y[row + cj] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&Ui[kk][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Uj[kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = __fmaf_rn(av[p], bv[q], acc[p][q]);
    }
    __syncthreads();
  }
  const double hs = gs.hsig ? 1.0 : 0.0;
  const float af = (float)(1.0 - rs.c_1 - rs.c_mu + (1.0 - hs) * rs.c_1 * rs.c_c * (2.0 - rs.c_c));
  const float c1f = (float)rs.c_1, cmuf = (float)rs.c_mu;
  float* C = s.cov + (int64_t)r * D * D;
  const float* pc = s.vec[F_PC] + (int64_t)r * D;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int i = i0 + ty * 4 + p;
    if (i >= D) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + tx * 4 + q;
      if (j > i) continue;                         // lower triangle; mirrored below
      const float c = __fadd_rn(__fadd_rn(__fmul_rn(af, C[(int64_t)i * D + j]),
                                          __fmul_rn(__fmul_rn(c1f, pc[i]), pc[j])),
                                __fmul_rn(cmuf, acc[p][q]));
      C[(int64_t)i * D + j] = c;
      C[(int64_t)j * D + i] = c;
    }
  }
}

// ---------------------------------------------------------------------------------- Cholesky
__device__ __forceinline__ bool chol_due(const DevState& s, int r) { return chol_due_rs(s.rs[r]); }

// W ← lower(C): the factorisation reads and writes nothing above the diagonal. One row per
// block iteration, float4 when rows are 16-B aligned (the ≤ 3 entries past the diagonal that a
// last float4 carries are never read).
__global__ void __launch_bounds__(256) chol_copy_kernel(DevState s) {
  const int r = blockIdx.y;
  if (!chol_due(s, r)) return;
  const int64_t D = s.D, DD = D * D;
  const float* C = s.cov + (int64_t)r * DD;
  float* Wk = s.cw + (int64_t)r * DD;
  const bool v4 = (D & 3) == 0;
  for (int64_t i = blockIdx.x; i < D; i += gridDim.x) {
    if (v4) {
      const float4* src = reinterpret_cast<const float4*>(C + i * D);
      float4* dst = reinterpret_cast<float4*>(Wk + i * D);
      for (int64_t c = threadIdx.x; c < (i + 4) / 4; c += blockDim.x) dst[c] = src[c];
    } else {
      for (int64_t c = threadIdx.x; c <= i; c += blockDim.x) Wk[i * D + c] = C[i * D + c];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) s.chol_fail[r] = 0;
}

// ---- 64 × 64 diagonal block: left-looking, one warp per 32 × 32 step, rows in shared memory.
// Row stride 36 floats: 16-B aligned rows for LDS.128, and a lane's own-row LDS.128 spreads over
// the banks in the minimum 4 wavefronts.
static constexpr int kLs = 36;

// Dot product of two 32-float shared-memory rows (x: this lane's, r: broadcast), 4 partial sums.
__device__ __forceinline__ float dot32_smem(const float* x, const float* r) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 a = reinterpret_cast<const float4*>(x)[q];
    const float4 b = reinterpret_cast<const float4*>(r)[q];
    s0 = __fmaf_rn(a.x, b.x, s0);
    s1 = __fmaf_rn(a.y, b.y, s1);
    s2 = __fmaf_rn(a.z, b.z, s2);
    s3 = __fmaf_rn(a.w, b.w, s3);
  }
  return __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
}

// 1/√d and √d to ~1 ulp: the MUFU estimate plus one Newton step (no IEEE slow-path branches on
// the serial chain).
__device__ __forceinline__ void rsqrt_sqrt(float d, float& inv, float& piv) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(d));
  const float h = __fmul_rn(0.5f, d);
  y = __fmul_rn(y, __fmaf_rn(-h, __fmul_rn(y, y), 1.5f));
  inv = y;
  piv = __fmul_rn(d, y);
}

// 32 × 32 Cholesky by one warp, left-looking (column j from the finished columns k < j):
//   c_i = A[i][j] − Σ_{k<j} L[i][k]·L[j][k],  L[j][j] = √c_j,  L[i][j] = c_i / L[j][j] (i > j).
// Lane i owns row i. A: [32][33] input; L: [32][kLs] output rows, ZERO on entry (so the dot
// product may run over all 32 k: the not-yet-computed entries are 0). dinv[j] = 1/L[j][j].
// One shuffle (the pivot) and one __syncwarp per column. Returns false if a pivot is not positive.
__device__ bool warp_chol32(const float (*A)[33], float (*L)[kLs], float* dinv, int lane) {
  bool ok = true;
#pragma unroll 1
  for (int j = 0; j < 32; ++j) {
    const float c = __fsub_rn(A[lane][j], dot32_smem(L[lane], L[j]));
    const float d = __shfl_sync(0xffffffffu, c, j);
    ok = ok && d > 0.0f;
    float inv = 1.0f, piv = 1.0f;
    if (d > 0.0f) rsqrt_sqrt(d, inv, piv);
    const float v = lane == j ? piv : (lane > j ? __fmul_rn(c, inv) : 0.0f);
    L[lane][j] = v;
    if (lane == j) dinv[j] = inv;
    __syncwarp();
  }
  return ok;
}

// Diagonal block [kb, kb+64)² (the last may be narrower) as a 2 × 2 blocked Cholesky of 32 × 32
// tiles: warp 0 factors L00; warp 1 solves L10 = A10·L00⁻ᵀ (left-looking forward substitution,
// x_j = (a_j − Σ_{k<j} x_k L00[j][k]) / L00[j][j]) and forms A11 − L10·L10ᵀ; warp 0 factors L11.
// Every step is a rolled loop over shared-memory rows (instruction-cache resident; the earlier
// fully unrolled register form was instruction-fetch-bound). fp32 throughout. Latency-bound:
// one serial 64-column chain per run.
__global__ void __launch_bounds__(64) chol_diag_kernel(DevState s, int kb) {
  __shared__ __align__(16) float L0[32][kLs];   // L00 rows
  __shared__ __align__(16) float L1[32][kLs];   // L11 rows
  __shared__ __align__(16) float X[32][kLs];    // L10 rows
  __shared__ float A0[32][33];                  // A00 (identity-padded)
  __shared__ float A1[32][33];                  // A11, then A11 − L10·L10ᵀ
  __shared__ float B[32][33];                   // A10
  __shared__ float dinv0[32], dinv1[32];
  __shared__ int bad;
  const int r = blockIdx.x;
  if (!chol_due(s, r) || s.chol_fail[r]) return;
  const int64_t D = s.D;
  const int b = (int)std::min<int64_t>(kNB, D - kb);
  const int b1 = b - 32;
  float* Wk = s.cw + (int64_t)r * D * D;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto at = [&](int i, int j) -> float& { return Wk[(int64_t)(kb + i) * D + kb + j]; };
  if (threadIdx.x == 0) bad = 0;
#pragma unroll 4
  for (int k = 0; k < 32; ++k) {               // zero the L rows; stage the inputs (row = lane)
    if (warp == 0) {
      L0[lane][k] = 0.0f;
      L1[lane][k] = 0.0f;
      A0[lane][k] = (lane < b && k <= lane && k < b) ? at(lane, k) : (k == lane ? 1.0f : 0.0f);
    } else {
      X[lane][k] = 0.0f;
      B[lane][k] = b1 > 0 && lane < b1 ? at(32 + lane, k) : 0.0f;
      A1[lane][k] = (lane < b1 && k <= lane && k < b1) ? at(32 + lane, 32 + k) : (k == lane ? 1.0f : 0.0f);
    }
  }
  __syncthreads();
  if (warp == 0) {
    if (!warp_chol32(A0, L0, dinv0, lane)) bad = 1;
#pragma unroll 4
    for (int k = 0; k < 32; ++k)
      if (lane < b && k <= lane && k < b) at(lane, k) = L0[lane][k];
  }
  __syncthreads();
  if (b1 <= 0) {
    if (threadIdx.x == 0 && bad) s.chol_fail[r] = 1;
    return;
  }
  if (warp == 1) {
#pragma unroll 1
    for (int j = 0; j < 32; ++j) {               // L10: left-looking forward substitution
      const float c = __fsub_rn(B[lane][j], dot32_smem(X[lane], L0[j]));
      X[lane][j] = __fmul_rn(c, dinv0[j]);
      __syncwarp();
    }
#pragma unroll 4
    for (int k = 0; k < 32; ++k)
      if (lane < b1) at(32 + lane, k) = X[lane][k];
#pragma unroll 2
    for (int k = 0; k < 32; ++k) {               // A11 − L10·L10ᵀ, row `lane`, k ≤ lane
      if (lane < b1 && k <= lane && k < b1)
        A1[lane][k] = __fsub_rn(A1[lane][k], dot32_smem(X[lane], X[k]));
    }
  }
  __syncthreads();
  if (warp == 0) {
    if (!warp_chol32(A1, L1, dinv1, lane)) bad = 1;
#pragma unroll 4
    for (int k = 0; k < 32; ++k)
      if (lane < b1 && k <= lane && k < b1) at(32 + lane, 32 + k) = L1[lane][k];
  }
  __syncthreads();
  if (threadIdx.x == 0 && bad) s.chol_fail[r] = 1;
}

// Panel rows i ≥ kb+64: solve x·L11ᵀ = W[i][kb:kb+64] by forward substitution, one row per thread,
// the row held in registers (fully unrolled; many warps share the code, so it stays cached).
static constexpr int kPanelRows = 128;
__global__ void __launch_bounds__(kPanelRows) chol_panel_kernel(DevState s, int kb) {
  __shared__ float L11[kNB][kNB + 1];
  __shared__ float dinv[kNB];
  const int r = blockIdx.y;
  if (!chol_due(s, r) || s.chol_fail[r]) return;
  const int64_t D = s.D;
  float* Wk = s.cw + (int64_t)r * D * D;
  for (int e = threadIdx.x; e < kNB * kNB; e += blockDim.x) {
    const int i = e >> 6, j = e & (kNB - 1);
    L11[i][j] = j <= i ? Wk[(int64_t)(kb + i) * D + kb + j] : 0.0f;
  }
  __syncthreads();
  if (threadIdx.x < kNB) dinv[threadIdx.x] = 1.0f / L11[threadIdx.x][threadIdx.x];
  __syncthreads();
  const int64_t i = kb + kNB + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= D) return;
  float* row = Wk + i * D + kb;
  float x[kNB];
  const bool v4 = (D & 3) == 0;                   // rows 16-B aligned (kb is a multiple of 64)
#pragma unroll
  for (int j = 0; j < kNB; j += 4) {
    if (v4) {
      const float4 v = *reinterpret_cast<const float4*>(row + j);
      x[j] = v.x; x[j + 1] = v.y; x[j + 2] = v.z; x[j + 3] = v.w;
    } else {
      x[j] = row[j]; x[j + 1] = row[j + 1]; x[j + 2] = row[j + 2]; x[j + 3] = row[j + 3];
    }
  }
#pragma unroll
  for (int j = 0; j < kNB; ++j) {
    float a0 = x[j], a1 = 0.0f;
#pragma unroll
    for (int k = 0; k + 1 < j; k += 2) {
      a0 = __fmaf_rn(-x[k], L11[j][k], a0);
      a1 = __fmaf_rn(-x[k + 1], L11[j][k + 1], a1);
    }
    if (j & 1) a0 = __fmaf_rn(-x[j - 1], L11[j][j - 1], a0);
    x[j] = __fmul_rn(__fadd_rn(a0, a1), dinv[j]);
  }
#pragma unroll
  for (int j = 0; j < kNB; j += 4) {
    if (v4) {
      *reinterpret_cast<float4*>(row + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
    } else {
      row[j] = x[j]; row[j + 1] = x[j + 1]; row[j + 2] = x[j + 2]; row[j + 3] = x[j + 3];
    }
  }
}

// Trailing update W[i][j] −= Σ_k L21[i][k] L21[j][k] on the lower tiles of [kb+b, D)².
__global__ void __launch_bounds__(256) chol_update_kernel(DevState s, int kb) {
  __shared__ __align__(16) float Pi[kTK][kTB + 4];
  __shared__ __align__(16) float Pj[kTK][kTB + 4];
  const int r = blockIdx.y;
  if (!chol_due(s, r) || s.chol_fail[r]) return;
  const int64_t D = s.D;
  const int b = (int)std::min<int64_t>(kNB, D - kb);
  const int64_t t0 = kb + b;
  int I, J;
  lower_tile(blockIdx.x, I, J);
  const int64_t i0 = t0 + (int64_t)I * kTB, j0 = t0 + (int64_t)J * kTB;
  if (i0 >= D) return;
  float* Wk = s.cw + (int64_t)r * D * D;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int lr = threadIdx.x >> 2, lk = (threadIdx.x & 3) * 4;
  float acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = 0.0f;
  for (int k0 = 0; k0 < b; k0 += kTK) {
    const int64_t ri = i0 + lr, rj = j0 + lr;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = k0 + lk + u;
      Pi[lk + u][lr] = (ri < D && k < b) ? Wk[ri * D + kb + k] : 0.0f;
      Pj[lk + u][lr] = (rj < D && k < b) ? Wk[rj * D + kb + k] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kTK; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&Pi[kk][ty * 4]);
      const float4 c = *reinterpret_cast<const float4*>(&Pj[kk][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = __fmaf_rn(av[p], cv[q], acc[p][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int64_t i = i0 + ty * 4 + p;
    if (i >= D) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t j = j0 + tx * 4 + q;
      if (j > i) continue;
      Wk[i * D + j] = __fsub_rn(Wk[i * D + j], acc[p][q]);
    }
  }
}

// A ← lower(W) for runs whose refresh succeeded.
__global__ void __launch_bounds__(256) chol_commit_kernel(DevState s) {
  const int r = blockIdx.y;
  if (!chol_due(s, r) || s.chol_fail[r]) return;
  const int64_t D = s.D, DD = D * D;
  const float* Wk = s.cw + (int64_t)r * DD;
  float* A = s.chol + (int64_t)r * DD;                 // its upper triangle is 0 from cma_init on
  const bool v4 = (D & 3) == 0;
  for (int64_t i = blockIdx.x; i < D; i += gridDim.x) {
    if (v4) {
      const float4* src = reinterpret_cast<const float4*>(Wk + i * D);
      float4* dst = reinterpret_cast<float4*>(A + i * D);
      for (int64_t c = threadIdx.x; c < (i + 4) / 4; c += blockDim.x) {
        float4 v = src[c];
        const int64_t j = 4 * c;
        if (j + 1 > i) v.y = 0.0f;
        if (j + 2 > i) v.z = 0.0f;
        if (j + 3 > i) v.w = 0.0f;
        dst[c] = v;
      }
    } else {
      for (int64_t c = threadIdx.x; c <= i; c += blockDim.x) A[i * D + c] = Wk[i * D + c];
    }
  }
}

cudaError_t launch_cma_tell(const DevState& s, bool refresh, cudaStream_t st, int* nk) {
  int n = 0;
  const int bpr = (int)((s.D + kVecDims - 1) / kVecDims);    // ≤ normpart's R·⌈Q/128⌉·… capacity
  cma_tellvec_kernel<<<dim3((unsigned)bpr, (unsigned)s.R), 256, 0, st>>>(s, bpr);
  cma_norm_kernel<<<s.R, 256, 0, st>>>(s, bpr);
  const int64_t RD = (int64_t)s.R * s.D;
  cma_pc_kernel<<<(unsigned)((RD + 255) / 256), 256, 0, st>>>(s);
  static const bool simt = std::getenv("ES_CMA_SIMT") != nullptr;   // A/B switch for profiling
  const bool tc = !simt && syrk_tc_supported(s);
  if (tc) {
    if (cudaError_t e = launch_cma_cov_tc(s, st)) return e;
    n += 5;
  } else {
    const int T = (int)((s.D + kTB - 1) / kTB);
    cma_cov_kernel<<<dim3((unsigned)(T * (T + 1) / 2), (unsigned)s.R), 256, 0, st>>>(s);
    n += 4;
  }
  if (refresh) {
    const unsigned cb = (unsigned)std::min<int64_t>(s.D, 1024);   // one row per block iteration
    chol_copy_kernel<<<dim3(cb, (unsigned)s.R), 256, 0, st>>>(s);
    n += 1;
    for (int64_t kb = 0; kb < s.D; kb += kNB) {
      chol_diag_kernel<<<s.R, 64, 0, st>>>(s, (int)kb);
      const int64_t rest = s.D - kb - std::min<int64_t>(kNB, s.D - kb);
      n += 1;
      if (rest > 0) {
        chol_panel_kernel<<<dim3((unsigned)((rest + kPanelRows - 1) / kPanelRows), (unsigned)s.R),
                            kPanelRows, 0, st>>>(s, (int)kb);
        if (tc) {
          if (cudaError_t e = launch_chol_update_tc(s, (int)kb, st)) return e;
        } else {
          const int Tt = (int)((rest + kTB - 1) / kTB);
          chol_update_kernel<<<dim3((unsigned)(Tt * (Tt + 1) / 2), (unsigned)s.R), 256, 0, st>>>(
              s, (int)kb);
        }
        n += 2;
      }
    }
    chol_commit_kernel<<<dim3(cb, (unsigned)s.R), 256, 0, st>>>(s);
    n += 1;
  }
  if (nk) *nk = n + 1;
  return cudaGetLastError();
}

}  // namespace esb
