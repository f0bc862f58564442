// fitness.cuh — per-element BBOB fitness accumulation (NUMERICS N7), shared by the standalone
// evaluation kernel (k_eval.cu) and the fused ask+evaluate kernel (k_ask_eval.cu).
// Binary64 accumulation; Sphere uses exact-product DFMAs (= the oracle's mul-then-add), Rastrigin
// accumulates Σx² and ΣS² separately and combines them once as Σx² + 20·ΣS² (N7). The binary32 →
// binary64 converts of S and |x| are bit assemblies on the FMA pipe; rint stays on the XU.
#pragma once
#include "noise.cuh"

namespace esb {

enum { FN_SPHERE = 0, FN_ROSENBROCK = 1, FN_RASTRIGIN = 2 };

struct FitAcc {
  double a = 0.0, b = 0.0;
};

// acc + Rosenbrock term of the pair (x_d, x_{d+1}) in binary64 with contracted operations
// (NUMERICS N7, GPU detail): t1 = fma(−a, a, b), acc = fma(1 − a, 1 − a, acc), then
// acc = fma(100·t1, t1, acc) — 5 FP64 instructions instead of the oracle's 7 + the sum's add; each
// result is binary64-accurate (a few 2⁻⁵³ relative), the same ≤ 1 ulp binary32 bar.
__device__ __forceinline__ double rosen_acc_d(double acc, double da, double db) {
  const double t1 = __fma_rn(-da, da, db);
  const double t2 = __dsub_rn(1.0, da);
  acc = __fma_rn(t2, t2, acc);
  return __fma_rn(__dmul_rn(100.0, t1), t1, acc);
}

// (double)v for v ≥ 0 without the XU-pipe F2F convert: the binary64 bits of a positive normal
// binary32 with bits u are u·2²⁹ + (896 << 52) — one IMAD.WIDE on the FMA pipe. Exact for normal
// v; v = 0 or subnormal becomes a ~2⁻¹²⁷-scale value whose square (≤ 2⁻²⁵⁰) cannot move a
// binary64 sum of the BBOB terms, nor its binary32 rounding (a sum that small rounds to 0).
__device__ __forceinline__ double pos_f2d(float v) {
  const uint64_t b = (uint64_t)__float_as_uint(v) * (1ull << 29) + 0x3800000000000000ull;
  return __longlong_as_double((long long)b);
}

// Add element x (and, for Rosenbrock, the pair term with its successor xn when has_next).
template <int FN>
__device__ __forceinline__ void fit_add(FitAcc& acc, float x, float xn, bool has_next) {
  if (FN == FN_SPHERE) {
    const double d = (double)x;
    acc.a = __fma_rn(d, d, acc.a);
  } else if (FN == FN_ROSENBROCK) {
    if (has_next) acc.a = rosen_acc_d(acc.a, (double)x, (double)xn);
  } else {
    // b = min(fr, 1 − fr) of N7 is the distance from x to the nearest integer: bq = x − rint(x)
    // is exact (Sterbenz; rint(x) = 0 for |x| < 1/2) and |bq| = b bit for bit, ties and |x| ≥ 2^23
    // included. S is odd in b and its polynomial even, so S = |bq|·P(bq²) (the |·| is an operand
    // modifier). Per element: FRND (the one XU instruction), FADD, the 7-op polynomial, two
    // IMAD.WIDE bit-assembled converts (FMA pipe), the |x| materialisation and two DFMAs.
    const float bq = __fsub_rn(x, rintf(x));
    const double S = pos_f2d(__fmul_rn(fabsf(bq), sinpi_P(__fmul_rn(bq, bq))));   // S ∈ [0, 1]
    const double d = pos_f2d(fabsf(x));
    acc.a = __fma_rn(d, d, acc.a);
    acc.b = __fma_rn(S, S, acc.b);
  }
}

template <int FN>
__device__ __forceinline__ double fit_total(const FitAcc& acc) {
  return FN == FN_RASTRIGIN ? __fma_rn(20.0, acc.b, acc.a) : acc.a;
}

// tanh to ≤ 5·10⁻⁷ relative (NUMERICS N14): the odd [9/8] rational x·p(x²)/q(x²) (p₀ = q₀ = 1) on
// x clamped to ±7.9053 (where it reaches ±1 in binary32); ONE MUFU (rcp) — a 1 − 2/(1 + e^{2x})
// form loads the XU pipe twice. 3.0·10⁻⁷ modelled in binary32 (+ the reciprocal's ulp: ≤ 4.2·10⁻⁷);
// tested on a dense sweep. 14 instructions per value (the earlier [13/6] form took 15).
__device__ __forceinline__ float tanh32(float x) {
  const float xc = fminf(fmaxf(x, -7.90531110763549805f), 7.90531110763549805f);
  const float s = __fmul_rn(xc, xc);
  float p = 0x1.08dd48p-26f;
  p = __fmaf_rn(p, s, 0x1.715eecp-16f);
  p = __fmaf_rn(p, s, 0x1.d50d80p-9f);
  p = __fmaf_rn(p, s, 0x1.13763cp-3f);
  p = __fmaf_rn(p, s, 1.0f);
  p = __fmul_rn(xc, p);
  float q = 0x1.cd6b4ap-21f;
  q = __fmaf_rn(q, s, 0x1.66ecccp-12f);
  q = __fmaf_rn(q, s, 0x1.ad1bd8p-6f);
  q = __fmaf_rn(q, s, 0x1.df1070p-2f);
  q = __fmaf_rn(q, s, 1.0f);
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
  return __fmul_rn(p, r);     // tiny |x|: p/q = x (p0 = q0 = 1), no select needed
}

// 2⁸·tanh(x) — tanh32 with p's coefficients scaled by 2⁸ (exact: a power of two), so the value is
// bit for bit fmul(tanh32(x), 256): the fp32 MLP's hidden activations enter the binary16 split
// pre-scaled without a multiply per value.
__device__ __forceinline__ float tanh32_x256(float x) {
  const float xc = fminf(fmaxf(x, -7.90531110763549805f), 7.90531110763549805f);
  const float s = __fmul_rn(xc, xc);
  float p = 0x1.08dd48p-18f;
  p = __fmaf_rn(p, s, 0x1.715eecp-8f);
  p = __fmaf_rn(p, s, 0x1.d50d80p-1f);
  p = __fmaf_rn(p, s, 0x1.13763cp+5f);
  p = __fmaf_rn(p, s, 256.0f);
  p = __fmul_rn(xc, p);
  float q = 0x1.cd6b4ap-21f;
  q = __fmaf_rn(q, s, 0x1.66ecccp-12f);
  q = __fmaf_rn(q, s, 0x1.ad1bd8p-6f);
  q = __fmaf_rn(q, s, 0x1.df1070p-2f);
  q = __fmaf_rn(q, s, 1.0f);
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
  return __fmul_rn(p, r);
}

// tanh of an activation that is rounded to binary16 next (N14′ hidden layers): the odd [7/6]
// rational x·p(x²)/q(x²) on x clamped to ±4.6 — past it tanh rounds to ±1 in binary16, and the
// rational's value there, 0.99979794, is above 1 − 2⁻¹² — ≤ 2.8·10⁻⁷ relative inside (modelled in
// binary32); 12 instructions per value instead of tanh32's 14.
__device__ __forceinline__ float tanh16h(float x) {
  const float xc = fminf(fmaxf(x, -4.6f), 4.6f);
  const float s = __fmul_rn(xc, xc);
  float p = 0x1.6cb52ep-18f;
  p = __fmaf_rn(p, s, 0x1.4e0136p-9f);
  p = __fmaf_rn(p, s, 0x1.01c874p-3f);
  p = __fmaf_rn(p, s, 1.0f);
  p = __fmul_rn(xc, p);
  float q = 0x1.6cb002p-13f;
  q = __fmaf_rn(q, s, 0x1.6d1718p-6f);
  q = __fmaf_rn(q, s, 0x1.d6397cp-2f);
  q = __fmaf_rn(q, s, 1.0f);
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
  return __fmul_rn(p, r);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace esb
