// k_eval.cu — K3 batched analytic fitness (Sphere / Rosenbrock / Rastrigin, NUMERICS N7).
//
// f_j = Σ_d term(x_jd): per-term arithmetic in double (exactly the oracle's operations), binary64
// accumulation in a fixed per-thread stride order followed by a fixed butterfly / tree, one final
// rounding to binary32. HBM-read bound (4·D bytes per member); x is streamed with float4 loads
// when D % 4 == 0. Short rows (D ≤ 4096): one warp per member. Long rows: one CTA per member.
#include <algorithm>

#include "es_internal.h"
#include "fitness.cuh"

namespace esb {

// Accumulate this thread's strided share of one row: quads q = lane0, lane0+stride, ...
template <int FN, bool V4>
__device__ __forceinline__ double row_partial(const float* __restrict__ row, int64_t D,
                                              int64_t lane0, int64_t stride) {
  FitAcc acc;
  if (V4) {
    // kU float4 loads issued before any is consumed (the loop was load-latency bound: one
    // 16-byte load in flight per thread); the accumulation order per thread is unchanged
    constexpr int kU = 4;
    const int64_t Q = D / 4;
    for (int64_t q0 = lane0; q0 < Q; q0 += kU * stride) {
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
          acc.a = __dadd_rn(acc.a, rosen_term_d(d0, d1));
          acc.a = __dadd_rn(acc.a, rosen_term_d(d1, d2));
          acc.a = __dadd_rn(acc.a, rosen_term_d(d2, d3));
          if (nn) acc.a = __dadd_rn(acc.a, rosen_term_d(d3, (double)nx[u]));
        } else {
          fit_add<FN>(acc, v[u].x, v[u].y, true);
          fit_add<FN>(acc, v[u].y, v[u].z, true);
          fit_add<FN>(acc, v[u].z, v[u].w, true);
          fit_add<FN>(acc, v[u].w, nx[u], nn);
        }
      }
    }
  } else {
    for (int64_t d = lane0; d < D; d += stride) {
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
__global__ void __launch_bounds__(256) eval_warp_kernel(const float* __restrict__ x, int64_t n,
                                                        int64_t D, float* __restrict__ f) {
  pdl_enter();
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= n) return;
  const int lane = threadIdx.x & 31;
  const double acc = warp_sum(row_partial<FN, V4>(x + row * D, D, lane, 32));
  if (lane == 0) f[row] = (float)acc;
}

template <int FN, bool V4, int T>
__global__ void __launch_bounds__(T) eval_block_kernel(const float* __restrict__ x, int64_t D,
                                                       float* __restrict__ f) {
  __shared__ double part[T / 32];
  pdl_enter();
  const int64_t row = blockIdx.x;
  double acc = warp_sum(row_partial<FN, V4>(x + row * D, D, threadIdx.x, T));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < T / 32 ? part[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) f[row] = (float)v;
  }
}

template <int FN, bool V4>
static void launch_fn(const float* x, int64_t n, int64_t D, float* f, cudaStream_t st) {
  cudaError_t e;
  if (D <= 4096) {
    e = launch_pdl(eval_warp_kernel<FN, V4>, dim3((unsigned)((n + 7) / 8)), dim3(256), 0, st, x, n, D, f);
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
