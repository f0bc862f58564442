// k_cma_tc.cu — SURVEY §8(f) f4: CMA-ES sampling y = A·z as a dense contraction on the 5th-generation
// tensor cores ("reparametrization ... Cholesky decomposition", sped up on accelerators).
//
// Per run r: Y[r] (N × D) = Z[r] (N × D) · A[r]ᵀ (D × D, lower-triangular). One CTA computes a
// 128-member × 128-dim tile with tcgen05.mma.kind::tf32 (M = 128, N = 128, K = 8), fp32 accumulator
// in 128 TMEM columns. fp32 accuracy from the 3-pass split: every operand x = big + small with
// big = x with its low 13 mantissa bits cleared — exactly what the tensor core reads from the raw
// fp32 tile, so the raw tile IS big — and small = x − big (exact in fp32; the MMA keeps its top 11
// bits, 2⁻²¹|x|), and
//   a·b ≈ big_a·big_b + big_a·small_b + small_a·big_b      (the dropped small·small is ~2⁻²⁰ |ab|).
// An output tile's K range stops at its last dim (A[d][k] = 0 for k > d).
//
// Warp roles (256 threads): warp 0 lane 0 — TMA producer (Z and A tiles, [128 rows × 32 k] fp32,
// K-major SWIZZLE_128B, 3-stage ring); warp 1 — TMEM allocation + the single MMA-issuing thread;
// warps 4–7 — write each landed stage's small parts into the tile's twin (one FADD per element), then
// the epilogue: tcgen05.ld (TMEM lane = member row), x = fma(σ, y, m) (+ box clip), Y and x out.
#include <cuda.h>

#include <algorithm>

#include "es_internal.h"
#include "tcgen05.cuh"

namespace esb {

static constexpr int kTcStages = 3;
static constexpr int kTcTile = 128 * 32 * 4;               // [128 rows × 32 k] fp32 = 16 KB
static constexpr int kTcStageBytes = 4 * kTcTile;          // Z big/small, A big/small
static constexpr int kTcSmem = kTcStages * kTcStageBytes + 1024 + 256;

struct CmaTcParams {
  CUtensorMap tz, ta;          // Z [R][N][D], A [R][D][D] as 3-D (k, row, run) fp32 maps
  float* y;                    // [R][N][D]
  float* x;                    // [R][Nloc][D] (this rank's members) or nullptr
  const float* mean;           // [R][D]
  const RunScal* rs;
  int N;
  int jl0, Nloc;               // this rank's members [jl0, jl0 + Nloc) (population sharding)
  int64_t D;
};

// Instruction descriptor, kind::tf32: D f32 (bit 4), A/B tf32 (format 2 at bits 7 and 10), both
// K-major, N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// The tf32 value the tensor core reads from an fp32 operand: the low 13 mantissa bits ignored.
__device__ __forceinline__ float tf32_trunc(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__global__ void __launch_bounds__(256, 1) cma_sample_tc_kernel(const __grid_constant__ CmaTcParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTcStages * kTcStageBytes);
  uint64_t* full = bars;                       // [kTcStages] TMA landed
  uint64_t* split = bars + kTcStages;          // [kTcStages] big/small written
  uint64_t* empty = bars + 2 * kTcStages;      // [kTcStages] MMAs done with the stage
  uint64_t* accum = bars + 3 * kTcStages;      // accumulator complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * kTcStages + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.z;
  const int d0 = blockIdx.x * 128, j0 = blockIdx.y * 128;
  const int64_t D = P.D;
  const int kend = (int)std::min<int64_t>(D, d0 + 128);
  const int nchunk = (kend + 31) / 32;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&split[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {                                   // TMA producer
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tz)));
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.ta)));
      for (int c = 0; c < nchunk; ++c) {
        const int s = c % kTcStages;
        const uint32_t ph = (uint32_t)(c / kTcStages) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        uint8_t* st = smem + s * kTcStageBytes;
        mbar_expect_tx(&full[s], 2 * kTcTile);
        tma_load_3d(st, &P.tz, c * 32, j0, r, &full[s]);                // Z big (raw)
        tma_load_3d(st + 2 * kTcTile, &P.ta, c * 32, d0, r, &full[s]);  // A big (raw)
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {                                   // MMA issuer
      const uint32_t idesc = idesc_tf32(128, 128);
      const uint32_t base = smem_u32(smem);
      for (int c = 0; c < nchunk; ++c) {
        const int s = c % kTcStages;
        mbar_wait(&split[s], (uint32_t)(c / kTcStages) & 1u);
        tc_fence_after();
        const uint32_t zb = base + s * kTcStageBytes, zs = zb + kTcTile;
        const uint32_t ab = zb + 2 * kTcTile, as = zb + 3 * kTcTile;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {                // K = 8 tf32 = 32 B per instruction
          const uint32_t o = ks * 32;
          mma_tf32(tmem, smem_desc(zb + o), smem_desc(ab + o), idesc, (c | ks) != 0);
          mma_tf32(tmem, smem_desc(zb + o), smem_desc(as + o), idesc, 1);
          mma_tf32(tmem, smem_desc(zs + o), smem_desc(ab + o), idesc, 1);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(accum);
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int t = threadIdx.x - 128;                   // 0..127
    for (int c = 0; c < nchunk; ++c) {                 // split each landed stage
      const int s = c % kTcStages;
      mbar_wait(&full[s], (uint32_t)(c / kTcStages) & 1u);
      uint8_t* st = smem + s * kTcStageBytes;
#pragma unroll
      for (int op = 0; op < 2; ++op) {                 // Z tile, then A tile
        const float4* raw = reinterpret_cast<const float4*>(st + op * 2 * kTcTile);
        float4* small = reinterpret_cast<float4*>(st + op * 2 * kTcTile + kTcTile);
#pragma unroll
        for (int i = 0; i < kTcTile / 16 / 128; ++i) {
          const int o = t + 128 * i;
          const float4 v = raw[o];
          small[o] = make_float4(__fsub_rn(v.x, tf32_trunc(v.x)), __fsub_rn(v.y, tf32_trunc(v.y)),
                                 __fsub_rn(v.z, tf32_trunc(v.z)), __fsub_rn(v.w, tf32_trunc(v.w)));
        }
      }
      fence_async_smem();
      named_bar(1, 128);
      if (t == 0) mbar_arrive(&split[s]);
    }
    // epilogue: lane quarter q = warp & 3 → member rows j0 + 32q + lane. Each 32 × 32 sub-tile is
    // transposed through shared memory (the ring is idle once the accumulator is complete) so that
    // every store is one member's 32 consecutive dims — a full 128-B line, not 32 scattered words.
    mbar_wait(accum, 0);
    tc_fence_after();
    const int q = warp & 3;
    const RunScal& rs = P.rs[r];
    const float sig = rs.sigma;
    const float* m = P.mean + (int64_t)r * D;
    float (*T)[33] = reinterpret_cast<float (*)[33]>(smem + q * (32 * 33 * 4));
    for (int c0 = 0; c0 < 128; c0 += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) T[lane][i] = v[i];
      __syncwarp();
      const int64_t d = d0 + c0 + lane;
      const bool dok = d < D;
      const float md = dok ? m[d] : 0.0f;
#pragma unroll 4
      for (int rr = 0; rr < 32; ++rr) {
        const int j = j0 + q * 32 + rr;
        if (j >= P.N || !dok) continue;
        const float yv = T[rr][lane];
        const int64_t o = ((int64_t)r * P.N + j) * D + d;
        P.y[o] = yv;
        const int jl = j - P.jl0;
        if (P.x && jl >= 0 && jl < P.Nloc) {
          float xv = __fmaf_rn(sig, yv, md);
          if (rs.clip) xv = fminf(fmaxf(xv, rs.clip_lo), rs.clip_hi);
          P.x[((int64_t)r * P.Nloc + jl) * D + d] = xv;
        }
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
  }
}


// (k, row, run) fp32 view of a [runs][rows][D] array: box 32 k × 128 rows × 1 run lands in smem in
// the UMMA K-major SWIZZLE_128B layout; out-of-range rows / k are zero-filled.
static bool encode_rows(CUtensorMap* m, const float* base, int64_t D, int64_t rows, int runs) {
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)rows, (cuuint64_t)runs};
  const cuuint64_t strides[2] = {(cuuint64_t)D * 4, (cuuint64_t)(D * rows * 4)};
  const cuuint32_t box[3] = {32, 128, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool cma_tc_supported(const DevState& s) { return (s.D % 4) == 0 && encode_tiled_fn() != nullptr; }

cudaError_t launch_cma_sample_tc(const DevState& s, float* x, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_attr_once((const void*)cma_sample_tc_kernel, kTcSmem, attr)) return e;
  CmaTcParams P;
  if (!encode_rows(&P.tz, s.zbuf, s.D, s.N, s.R) || !encode_rows(&P.ta, s.chol, s.D, s.D, s.R))
    return cudaErrorInvalidValue;
  P.y = s.ybuf;
  P.x = x;
  P.mean = s.vec[F_MEAN];
  P.rs = s.rs;
  P.N = s.N;
  P.jl0 = s.rank * s.Nloc;
  P.Nloc = s.Nloc;
  P.D = s.D;
  const dim3 g((unsigned)((s.D + 127) / 128), (unsigned)((s.N + 127) / 128), (unsigned)s.R);
  cma_sample_tc_kernel<<<g, 256, kTcSmem, st>>>(P);
  return cudaGetLastError();
}

}  // namespace esb
