// k_eval.cu — K3 batched analytic fitness (Sphere / Rosenbrock / Rastrigin, NUMERICS N7).
//
// f_j = Σ_d term(x_jd): per-term arithmetic in double (exactly the oracle's operations), binary64
// accumulation in a fixed per-thread stride order followed by a fixed butterfly / tree, one final
// rounding to binary32. HBM-read bound (4·D bytes per member); x is streamed with float4 loads
// when D % 4 == 0. Short rows (D ≤ 4096): one warp per member. Long rows: one CTA per member.
#include <algorithm>
#include <atomic>

#include "es_internal.h"
#include "fitness.cuh"

namespace esb {

// Accumulate this thread's strided share of one row's range [qa, qb) — quads (V4) or elements:
// qa + lane0, qa + lane0 + stride, ... (a Rosenbrock pair term belongs to its first element's range)
template <int FN, bool V4>
__device__ __forceinline__ double row_partial(const float* __restrict__ row, int64_t D, int64_t qa,
                                              int64_t qb, int64_t lane0, int64_t stride) {
  FitAcc acc;
  if (V4 && FN != FN_ROSENBROCK) {
    // quad indices within a row fit 32 bits: 32-bit compares and increments; a quad past the
    // range is neither loaded nor zero-filled (the consuming loop stops before it). Same
    // per-thread order as the general loop below.
    constexpr int kU = 4;
    const int Q = (int)qb, st = (int)stride;
    const float4* row4 = reinterpret_cast<const float4*>(row);
    for (int q0 = (int)(qa + lane0); q0 < Q; q0 += kU * st) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (q0 + u * st < Q) v[u] = __ldcs(row4 + q0 + u * st);
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (q0 + u * st >= Q) break;
        fit_add<FN>(acc, v[u].x, v[u].y, true);
        fit_add<FN>(acc, v[u].y, v[u].z, true);
        fit_add<FN>(acc, v[u].z, v[u].w, true);
        fit_add<FN>(acc, v[u].w, 0.0f, false);
      }
    }
  } else if (V4) {
    // kU float4 loads issued before any is consumed (the loop was load-latency bound: one
    // 16-byte load in flight per thread); the accumulation order per thread is unchanged
    constexpr int kU = 4;
    const int64_t Q = qb;
    for (int64_t q0 = qa + lane0; q0 < Q; q0 += kU * stride) {
      float4 v[kU];
      float nx[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t q = q0 + u * stride;
        v[u] = q < Q ? __ldcs(reinterpret_cast<const float4*>(row) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        nx[u] = (FN == FN_ROSENBROCK && 4 * q + 4 < D) ? __ldg(row + 4 * q + 4) : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t q = q0 + u * stride;
        if (q >= Q) break;
        const bool nn = (FN == FN_ROSENBROCK) && (4 * q + 4 < D);
        if (FN == FN_ROSENBROCK) {
          // each element converted to binary64 once (it is the b of one pair and the a of the
          // next): 5 converts per quad instead of 8, the same binary64 terms
          const double d0 = v[u].x, d1 = v[u].y, d2 = v[u].z, d3 = v[u].w;
          acc.a = rosen_acc_d(acc.a, d0, d1);
          acc.a = rosen_acc_d(acc.a, d1, d2);
          acc.a = rosen_acc_d(acc.a, d2, d3);
          if (nn) acc.a = rosen_acc_d(acc.a, d3, (double)nx[u]);
        } else {
          fit_add<FN>(acc, v[u].x, v[u].y, true);
          fit_add<FN>(acc, v[u].y, v[u].z, true);
          fit_add<FN>(acc, v[u].z, v[u].w, true);
          fit_add<FN>(acc, v[u].w, nx[u], nn);
        }
      }
    }
  } else {
    for (int64_t d = qa + lane0; d < qb; d += stride) {
      const bool nn = d + 1 < D;
      const float b = (FN == FN_ROSENBROCK && nn) ? __ldg(row + d + 1) : 0.0f;
      fit_add<FN>(acc, __ldg(row + d), b, nn);
    }
  }
  return fit_total<FN>(acc);
}

__device__ __forceinline__ double warp_sum(double v) { return warp_sum_d(v); }

// Short rows: one warp per row. (A grid-stride loop over rows with 8 resident CTAs per SM was
// measured slower at C2: 121.5 vs 115 µs — the per-row load → reduce → next-row chain of a
// persistent warp hides less latency than fresh warps do.)
template <int FN, bool V4>
__global__ void __launch_bounds__(256, FN == FN_ROSENBROCK ? 6 : 8) eval_warp_kernel(const float* __restrict__ x, int64_t n,
                                                        int64_t D, float* __restrict__ f) {
  pdl_enter();
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  const int lane = threadIdx.x & 31;
  const double acc = warp_sum(row_partial<FN, V4>(x + row * D, D, 0, V4 ? D / 4 : D, lane, 32));
  if (lane == 0) f[row] = (float)acc;
}

template <int FN, bool V4, int T>
__global__ void __launch_bounds__(T) eval_block_kernel(const float* __restrict__ x, int64_t D,
                                                       float* __restrict__ f) {
  __shared__ double part[T / 32];
  pdl_enter();
  const int64_t row = blockIdx.x;
  double acc = warp_sum(row_partial<FN, V4>(x + row * D, D, 0, V4 ? D / 4 : D, threadIdx.x, T));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < T / 32 ? part[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) f[row] = (float)v;
  }
}

// Long rows, few members: a cluster of C CTAs per row (grid (C, n), cluster (C, 1, 1)), CTA c
// summing the row's c-th range; CTA 0 adds the C block sums in rank order over distributed shared
// memory. (One 1024-thread CTA per row left C3's 256 rows in two waves at one CTA per SM.)
template <int FN, bool V4>
__global__ void __launch_bounds__(256, 6) eval_cluster_kernel(const float* __restrict__ x, int64_t D,
                                                           float* __restrict__ f) {
  __shared__ double part[8];
  __shared__ double csum;
  pdl_enter();
  const int C = gridDim.x, c = blockIdx.x;
  const int64_t row = blockIdx.y;
  const int64_t Q = V4 ? D / 4 : D, per = (Q + C - 1) / C;
  const int64_t qa = min(Q, c * per), qb = min(Q, qa + per);
  const double acc = warp_sum(row_partial<FN, V4>(x + row * D, D, qa, qb, threadIdx.x, 256));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t = __dadd_rn(t, part[k]);
    csum = t;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (c == 0 && threadIdx.x == 0) {
    double t = 0.0;
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(&csum);
    for (int k = 0; k < C; ++k) {
      double v;
      asm volatile("{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %1, %2;\n\t"
                   "ld.shared::cluster.f64 %0, [ra];\n\t}"
                   : "=d"(v) : "r"(a), "r"(k) : "memory");
      t = __dadd_rn(t, v);
    }
    f[row] = (float)t;
  }
  // no CTA leaves while CTA 0 may still read its block sum
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int FN, bool V4>
static cudaError_t launch_cluster(const float* x, int64_t n, int64_t D, float* f, int C,
                                  cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)C, (unsigned)n);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, eval_cluster_kernel<FN, V4>, x, D, f);
}

template <int FN, bool V4>
static void launch_fn(const float* x, int64_t n, int64_t D, float* f, cudaStream_t st) {
  cudaError_t e;
  if (D <= 4096) {
    e = launch_pdl(eval_warp_kernel<FN, V4>, dim3((unsigned)((n + 7) / 8)), dim3(256), 0, st, x, n, D, f);
  } else if (n < 4 * sm_count() && n <= 65535 &&
             std::min<int64_t>(8, (6 * sm_count() + n - 1) / n) > 1) {
    // as many CTAs per row as keep the grid in one wave of resident CTAs; ≥ 2048 elements each
    static std::atomic<int> occ{0};
    if (occ.load() == 0) {
      int o = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, eval_cluster_kernel<FN, V4>, 256, 0);
      occ.store(std::max(1, o));
    }
    const int64_t Q = V4 ? D / 4 : D;
    const int C = (int)std::min<int64_t>({8, (int64_t)occ.load() * sm_count() / n,
                                          std::max<int64_t>(1, Q / (V4 ? 512 : 2048))});
    e = C > 1 ? launch_cluster<FN, V4>(x, n, D, f, C, st)
              : launch_pdl(eval_block_kernel<FN, V4, 256>, dim3((unsigned)n), dim3(256), 0, st, x, D, f);
  } else if (D <= 65536 || n >= 4 * sm_count()) {
    e = launch_pdl(eval_block_kernel<FN, V4, 256>, dim3((unsigned)n), dim3(256), 0, st, x, D, f);
  } else {
    e = launch_pdl(eval_block_kernel<FN, V4, 1024>, dim3((unsigned)n), dim3(1024), 0, st, x, D, f);
  }
  (void)e;   // a launch error stays the thread's last error (launch_eval_bbob returns it)
}

cudaError_t launch_eval_bbob(int fn, const float* x, int64_t n, int64_t D, float* f,
                             cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const bool v4 = (D % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  switch (fn * 2 + (v4 ? 1 : 0)) {
    case 0: launch_fn<FN_SPHERE, false>(x, n, D, f, st); break;
    case 1: launch_fn<FN_SPHERE, true>(x, n, D, f, st); break;
    case 2: launch_fn<FN_ROSENBROCK, false>(x, n, D, f, st); break;
    case 3: launch_fn<FN_ROSENBROCK, true>(x, n, D, f, st); break;
    case 4: launch_fn<FN_RASTRIGIN, false>(x, n, D, f, st); break;
    default: launch_fn<FN_RASTRIGIN, true>(x, n, D, f, st); break;
  }
  return cudaGetLastError();
}

}  // namespace esb
