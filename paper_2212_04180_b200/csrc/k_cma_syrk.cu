// k_cma_syrk.cu — SURVEY §8(f) f4: the two symmetric rank-k updates of full-covariance CMA-ES on the
// 5th-generation tensor cores (the dense contractions of P:62 / P:177's covariance adaptation and of
// the Cholesky refresh behind P:106's sampling):
//   CHOL  the blocked factorisation's trailing update  W[i][j] −= Σ_{k∈panel} W[i][k]·W[j][k]
//         over the lower tiles of [t0, D)² (K = the 64 panel columns, read in place from W);
//   COV   the rank-μ covariance update  C[i][j] ← a·C[i][j] + c₁·p_c[i]·p_c[j] + c_μ·Σ_e U[i][e]·V[j][e]
//         with U[i][e] = w_e·y_e[i], V[j][e] = y_e[j] (transposed by cma_gather_t_kernel so that the
//         contraction index e is contiguous, i.e. both operands K-major), mirrored into the upper
//         triangle.
// One CTA per 128 × 128 lower tile (I ≥ J) and run: tcgen05.mma.kind::tf32 (M = N = 128, K = 8),
// fp32 accumulator in 128 TMEM columns, fp32 accuracy from the same 3-pass split as the sampling
// kernel (k_cma_tc.cu): the raw fp32 tile is the truncated big part, the converter warps write
// small = x − big into its twin, and big·big + big·small + small·big is accumulated.
// Warp roles (256 threads): warp 0 lane 0 TMA producer (2-stage ring of [128 rows × 32 k] fp32
// tiles, K-major SWIZZLE_128B); warp 1 TMEM allocation + the MMA-issuing thread; warps 4–7 the
// converters, then the epilogue (tcgen05.ld → 32 × 32 transposes through shared memory, so every
// global access is one row's 32 consecutive floats).
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "es_internal.h"
#include "tcgen05.cuh"

namespace esb {

static constexpr int kSyStages = 2;
static constexpr int kSyTile = 128 * 32 * 4;               // [128 rows × 32 k] fp32 = 16 KB
static constexpr int kSyStageBytes = 4 * kSyTile;          // A raw/small, B raw/small
static constexpr int kSySmem = kSyStages * kSyStageBytes + 1024 + 256;

enum SyrkMode : int { SYRK_CHOL = 0, SYRK_COV = 1 };

struct SyrkParams {
  CUtensorMap ta, tb;          // (k, row, run) fp32 maps of the two operands
  float* out;                  // [R][D][D]: W (CHOL) or C (COV)
  const float* pc;             // COV: p_c [R][D]
  const RunScal* rs;
  const GenScal* gs;
  const int32_t* fail;         // CHOL: chol_fail
  int64_t D;
  int t0;                      // first row / column of the updated region
  int k0;                      // first k of the operands
  int kchunks;                 // CHOL: 32-wide k chunks (COV: from the run's entry count)
  int mode;
};

__device__ __forceinline__ uint32_t idesc_tf32_128() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(128 >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ float trunc_tf32(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__global__ void __launch_bounds__(256, 1) syrk_tc_kernel(const __grid_constant__ SyrkParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int r = blockIdx.y;
  const RunScal& rs = P.rs[r];
  if (P.mode == SYRK_CHOL && (!chol_due_rs(rs) || P.fail[r])) return;
  int I, J;
  lower_tile(blockIdx.x, I, J);
  const int64_t D = P.D;
  const int i0 = P.t0 + I * 128, j0 = P.t0 + J * 128;
  if (i0 >= D) return;
  const int nchunk = P.mode == SYRK_CHOL ? P.kchunks : (P.gs[r].nentries + 31) / 32;
  if (nchunk <= 0) return;   // (COV always has entries)

  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSyStages * kSyStageBytes);
  uint64_t* full = bars;
  uint64_t* split = bars + kSyStages;
  uint64_t* empty = bars + 2 * kSyStages;
  uint64_t* accum = bars + 3 * kSyStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * kSyStages + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSyStages; ++s) {
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
      for (int c = 0; c < nchunk; ++c) {
        const int s = c % kSyStages;
        mbar_wait(&empty[s], ((uint32_t)(c / kSyStages) & 1u) ^ 1u);
        uint8_t* st = smem + s * kSyStageBytes;
        mbar_expect_tx(&full[s], 2 * kSyTile);
        tma_load_3d(st, &P.ta, P.k0 + c * 32, i0, r, &full[s]);
        tma_load_3d(st + 2 * kSyTile, &P.tb, P.k0 + c * 32, j0, r, &full[s]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {                                   // MMA issuer: D[i][j] += A[i][k]·B[j][k]
      const uint32_t idesc = idesc_tf32_128();
      const uint32_t base = smem_u32(smem);
      for (int c = 0; c < nchunk; ++c) {
        const int s = c % kSyStages;
        mbar_wait(&split[s], (uint32_t)(c / kSyStages) & 1u);
        tc_fence_after();
        const uint32_t ab = base + s * kSyStageBytes, as = ab + kSyTile;
        const uint32_t bb = ab + 2 * kSyTile, bs = ab + 3 * kSyTile;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t o = ks * 32;
          mma_tf32_ss(tmem, smem_desc(ab + o), smem_desc(bb + o), idesc, (c | ks) != 0);
          mma_tf32_ss(tmem, smem_desc(ab + o), smem_desc(bs + o), idesc, 1);
          mma_tf32_ss(tmem, smem_desc(as + o), smem_desc(bb + o), idesc, 1);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(accum);
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int t = threadIdx.x - 128;
    for (int c = 0; c < nchunk; ++c) {                 // small parts of each landed stage
      const int s = c % kSyStages;
      mbar_wait(&full[s], (uint32_t)(c / kSyStages) & 1u);
      uint8_t* st = smem + s * kSyStageBytes;
#pragma unroll
      for (int op = 0; op < 2; ++op) {
        const float4* raw = reinterpret_cast<const float4*>(st + op * 2 * kSyTile);
        float4* small = reinterpret_cast<float4*>(st + op * 2 * kSyTile + kSyTile);
#pragma unroll
        for (int i = 0; i < kSyTile / 16 / 128; ++i) {
          const int o = t + 128 * i;
          const float4 v = raw[o];
          small[o] = make_float4(__fsub_rn(v.x, trunc_tf32(v.x)), __fsub_rn(v.y, trunc_tf32(v.y)),
                                 __fsub_rn(v.z, trunc_tf32(v.z)), __fsub_rn(v.w, trunc_tf32(v.w)));
        }
      }
      fence_async_smem();
      named_bar(1, 128);
      if (t == 0) mbar_arrive(&split[s]);
    }
  }
  // epilogue, all 8 warps: quarter q = warp & 3 holds rows i0 + 32q + lane (its TMEM lanes); warps
  // 0–3 take columns j0 + [0, 64), warps 4–7 j0 + [64, 128). Every global access below is issued
  // as a batch of 32 independent row-segment loads before any store (one memory latency per
  // 32 × 32 sub-tile, not one per row).
  __syncwarp();
  mbar_wait(accum, 0);
  tc_fence_after();
  {
    const int q = warp & 3, h = warp >> 2;
    const int i = i0 + q * 32 + lane;
    float* M = P.out + (int64_t)r * D * D;
    float (*T)[33] = reinterpret_cast<float (*)[33]>(smem + warp * (32 * 33 * 4));
    float af = 0.f, c1f = 0.f, cmuf = 0.f, pci = 0.f;
    const float* pc = nullptr;
    if (P.mode == SYRK_COV) {
      const GenScal& gs = P.gs[r];
      const double hs = gs.hsig ? 1.0 : 0.0;
      af = (float)(1.0 - rs.c_1 - rs.c_mu + (1.0 - hs) * rs.c_1 * rs.c_c * (2.0 - rs.c_c));
      c1f = (float)rs.c_1;
      cmuf = (float)rs.c_mu;
      pc = P.pc + (int64_t)r * D;
      pci = i < D ? pc[i] : 0.0f;
    }
    for (int c0 = 64 * h; c0 < 64 * h + 64; c0 += 32) {
      if (j0 + c0 > i0 + q * 32 + 31) break;           // the warp's 32 rows are all above these columns
      float v[32], w[32];
      tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, v);
      if (P.mode == SYRK_COV) {
        // new (i, j) from C[j][i] (= C[i][j]: C is symmetric), written to C[j][i] for j < i (the
        // mirror; lanes run along i, so coalesced) and staged for the lower store
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int j = j0 + c0 + k;
          w[k] = (i < D && j <= i) ? M[(int64_t)j * D + i] : 0.0f;
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int j = j0 + c0 + k;
          if (i < D && j <= i) {
            const float cv = __fadd_rn(__fadd_rn(__fmul_rn(af, w[k]),
                                                 __fmul_rn(__fmul_rn(c1f, pci), pc[j])),
                                       __fmul_rn(cmuf, v[k]));
            if (j < i) M[(int64_t)j * D + i] = cv;
            v[k] = cv;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 32; ++k) T[lane][k] = v[k];
      __syncwarp();
      const int jj = j0 + c0 + lane;
      if (P.mode == SYRK_CHOL) {
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) {
          const int ii = i0 + q * 32 + rr;
          w[rr] = (ii < D && jj <= ii) ? M[(int64_t)ii * D + jj] : 0.0f;
        }
      }
#pragma unroll
      for (int rr = 0; rr < 32; ++rr) {
        const int ii = i0 + q * 32 + rr;
        if (ii < D && jj <= ii)
          M[(int64_t)ii * D + jj] = P.mode == SYRK_CHOL ? __fsub_rn(w[rr], T[rr][lane]) : T[rr][lane];
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

// COV operands: Ut[r][d][e] = w_e·y_e[d] and Vt[r][d][e] = y_e[d] for the run's selected entries
// e < nentries (y_e = Y[dir_e], w_e = its recombination weight, as cma_cov_kernel forms them), zero
// for nentries ≤ e < Kp. 32 × 32 tiles transposed through shared memory: both the row reads of Y
// and the writes (32 consecutive e of one d) are coalesced.
__global__ void __launch_bounds__(256) cma_gather_t_kernel(DevState s) {
  __shared__ float tu[32][33], tv[32][33];
  const int r = blockIdx.z;
  const int e0 = blockIdx.y * 32;
  const int64_t d0 = (int64_t)blockIdx.x * 32;
  const int ne = s.gs[r].nentries;
  const int64_t D = s.D;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 8 rows of 32
  const float* Y = s.ybuf + (int64_t)r * s.N * D;
  for (int k = ty; k < 32; k += 8) {
    const int e = e0 + k;
    const int64_t d = d0 + tx;
    float y = 0.0f, w = 0.0f;
    if (e < ne && d < D) {
      y = Y[(int64_t)s.dir[(int64_t)r * s.N + e] * D + d];
      w = (float)s.coefA[(int64_t)r * s.N + e];
    }
    tu[k][tx] = __fmul_rn(w, y);
    tv[k][tx] = y;
  }
  __syncthreads();
  const int64_t base = (int64_t)r * D * s.kp;
  for (int k = ty; k < 32; k += 8) {
    const int64_t d = d0 + k;
    if (d >= D) continue;
    s.ut[base + d * s.kp + e0 + tx] = tu[tx][k];
    s.vt[base + d * s.kp + e0 + tx] = tv[tx][k];
  }
}

// (k, row, run) fp32 view of [runs][rows][ld] (k < kdim valid): box 32 k × 128 rows × 1 run in the
// UMMA K-major SWIZZLE_128B layout; out-of-range rows / k read as zero.
static bool encode_kmajor(CUtensorMap* m, const float* base, int64_t kdim, int64_t ld, int64_t rows,
                          int runs) {
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)kdim, (cuuint64_t)rows, (cuuint64_t)runs};
  const cuuint64_t strides[2] = {(cuuint64_t)ld * 4, (cuuint64_t)(ld * rows * 4)};
  const cuuint32_t box[3] = {32, 128, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static cudaError_t syrk_attr() {
  static std::atomic<uint64_t> done{0};
  return smem_attr_once((const void*)syrk_tc_kernel, kSySmem, done);
}

bool syrk_tc_supported(const DevState& s) { return (s.D % 4) == 0 && encode_tiled_fn() != nullptr; }

// Trailing update after the panel at kb (b = 64 columns; rows and columns from t0 = kb + 64).
cudaError_t launch_chol_update_tc(const DevState& s, int kb, cudaStream_t st) {
  if (cudaError_t e = syrk_attr()) return e;
  SyrkParams P;
  std::memset(&P, 0, sizeof P);
  // W as (k, row, run); the panel is columns [kb, kb+64) of rows ≥ t0
  if (!encode_kmajor(&P.ta, s.cw, s.D, s.D, s.D, s.R)) return cudaErrorInvalidValue;
  P.tb = P.ta;
  P.out = s.cw;
  P.rs = s.rs;
  P.gs = s.gs;
  P.fail = s.chol_fail;
  P.D = s.D;
  P.t0 = kb + 64;
  P.k0 = kb;
  P.kchunks = 2;
  P.mode = SYRK_CHOL;
  const int T = (int)((s.D - P.t0 + 127) / 128);
  syrk_tc_kernel<<<dim3((unsigned)(T * (T + 1) / 2), (unsigned)s.R), 256, kSySmem, st>>>(P);
  return cudaGetLastError();
}

// C ← a·C + c₁ p_c p_cᵀ + c_μ Σ_e w_e y_e y_eᵀ: the transposed gather, then the tensor-core SYRK
// over the lower tiles of [0, D)² (k chunks from each run's entry count), mirrored.
cudaError_t launch_cma_cov_tc(const DevState& s, cudaStream_t st) {
  if (cudaError_t e = syrk_attr()) return e;
  const int nek = (int)((s.N + 31) / 32);            // entry chunks covering any run's μ
  cma_gather_t_kernel<<<dim3((unsigned)((s.D + 31) / 32), (unsigned)nek, (unsigned)s.R), 256, 0,
                        st>>>(s);
  SyrkParams P;
  std::memset(&P, 0, sizeof P);
  if (!encode_kmajor(&P.ta, s.ut, s.kp, s.kp, s.D, s.R) ||
      !encode_kmajor(&P.tb, s.vt, s.kp, s.kp, s.D, s.R))
    return cudaErrorInvalidValue;
  P.out = s.cov;
  P.pc = s.vec[F_PC];
  P.rs = s.rs;
  P.gs = s.gs;
  P.D = s.D;
  P.mode = SYRK_COV;
  const int T = (int)((s.D + 127) / 128);
  syrk_tc_kernel<<<dim3((unsigned)(T * (T + 1) / 2), (unsigned)s.R), 256, kSySmem, st>>>(P);
  return cudaGetLastError();
}

}  // namespace esb
