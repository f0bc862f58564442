// k_eval.cu — K3 batched analytic fitness (Sphere / Rosenbrock / Rastrigin, NUMERICS N7).
//
// f_j = Σ_d term(x_jd): per-term arithmetic in double (exactly the oracle's operations), binary64
// accumulation in a fixed per-thread stride order followed by a fixed butterfly / tree, one final
// rounding to binary32. HBM-read bound (4·D bytes per member); x is streamed with float4 loads
// when D % 4 == 0. Short rows (D ≤ 4096): one warp per member. Long rows: one CTA per member.
#include <algorithm>

#include "es_internal.h"
#include "noise.cuh"

namespace esb {

enum { FN_SPHERE = 0, FN_ROSENBROCK = 1, FN_RASTRIGIN = 2 };

template <int FN>
__device__ __forceinline__ double term(float a, float b, bool has_next) {
  if (FN == FN_SPHERE) return __dmul_rn((double)a, (double)a);
  if (FN == FN_ROSENBROCK) {
    if (!has_next) return 0.0;
    const double da = a, db = b;
    const double t1 = __dsub_rn(db, __dmul_rn(da, da));
    const double t2 = __dsub_rn(1.0, da);
    return __dadd_rn(__dmul_rn(100.0, __dmul_rn(t1, t1)), __dmul_rn(t2, t2));
  }
  return 0.0;   // Rastrigin accumulates two sums instead (rast_acc)
}

// Rastrigin (N7): Σx² and ΣS² accumulated separately with exact-product DFMAs, combined once;
// S = sin(π·min(fr, 1 − fr)) by the degree-5 polynomial of N7.
__device__ __forceinline__ void rast_acc(float a, double& ax, double& as) {
  const float ab = fabsf(a);
  const float fr = __fsub_rn(ab, floorf(ab));
  const double S = (double)sinpi_half(fminf(fr, __fsub_rn(1.0f, fr)));
  const double da = (double)a;
  ax = __fma_rn(da, da, ax);
  as = __fma_rn(S, S, as);
}

// Accumulate this thread's strided share of one row: quads q = lane0, lane0+stride, ...
template <int FN, bool V4>
__device__ __forceinline__ double row_partial(const float* __restrict__ row, int64_t D,
                                              int64_t lane0, int64_t stride) {
  double acc = 0.0;
  if (FN == FN_RASTRIGIN) {
    double ax = 0.0, as = 0.0;
    if (V4) {
      for (int64_t q = lane0; q < D / 4; q += stride) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(row) + q);
        rast_acc(v.x, ax, as);
        rast_acc(v.y, ax, as);
        rast_acc(v.z, ax, as);
        rast_acc(v.w, ax, as);
      }
    } else {
      for (int64_t d = lane0; d < D; d += stride) rast_acc(__ldg(row + d), ax, as);
    }
    return __fma_rn(20.0, as, ax);
  }
  if (FN == FN_SPHERE) {
    if (V4) {
      for (int64_t q = lane0; q < D / 4; q += stride) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(row) + q);
        acc = __fma_rn((double)v.x, (double)v.x, acc);   // exact product: = mul-then-add
        acc = __fma_rn((double)v.y, (double)v.y, acc);
        acc = __fma_rn((double)v.z, (double)v.z, acc);
        acc = __fma_rn((double)v.w, (double)v.w, acc);
      }
    } else {
      for (int64_t d = lane0; d < D; d += stride) {
        const double v = __ldg(row + d);
        acc = __fma_rn(v, v, acc);
      }
    }
    return acc;
  }
  if (V4) {
    const int64_t Q = D / 4;
    for (int64_t q = lane0; q < Q; q += stride) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(row) + q);
      float nx = 0.0f;
      const bool nn = (FN == FN_ROSENBROCK) && (4 * q + 4 < D);
      if (FN == FN_ROSENBROCK && nn) nx = __ldg(row + 4 * q + 4);
      acc = __dadd_rn(acc, term<FN>(v.x, v.y, true));
      acc = __dadd_rn(acc, term<FN>(v.y, v.z, true));
      acc = __dadd_rn(acc, term<FN>(v.z, v.w, true));
      acc = __dadd_rn(acc, term<FN>(v.w, nx, nn));
    }
  } else {
    for (int64_t d = lane0; d < D; d += stride) {
      const bool nn = d + 1 < D;
      const float b = (FN == FN_ROSENBROCK && nn) ? __ldg(row + d + 1) : 0.0f;
      acc = __dadd_rn(acc, term<FN>(__ldg(row + d), b, nn));
    }
  }
  return acc;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int FN, bool V4>
__global__ void __launch_bounds__(256) eval_warp_kernel(const float* __restrict__ x, int64_t n,
                                                        int64_t D, float* __restrict__ f) {
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
  if (D <= 4096) {
    eval_warp_kernel<FN, V4><<<(unsigned)((n + 7) / 8), 256, 0, st>>>(x, n, D, f);
  } else if (D <= 65536 || n >= 4 * sm_count()) {
    eval_block_kernel<FN, V4, 256><<<(unsigned)n, 256, 0, st>>>(x, D, f);
  } else {
    eval_block_kernel<FN, V4, 1024><<<(unsigned)n, 1024, 0, st>>>(x, D, f);
  }
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
