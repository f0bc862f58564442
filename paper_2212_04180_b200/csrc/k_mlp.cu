// k_mlp.cu — K4: synthetic-MLP fitness on the 5th-generation tensor cores (NUMERICS N14, N14′;
// P:212 "MLP", topology P:268–270). Per population member: L chained [128 × w_{l-1}]·[w_{l-1} × w_l]
// GEMMs (batch 128), tanh, and the MSE against the teacher's outputs. Two kernels:
//
// mlp_kernel (N14′, the fp16-image approximation): one persistent CTA per SM walks the members.
//   warp 0 (TMA mode)  producer: the ask's fp16 image streamed with TMA in [128 n × 64 k]
//                      SWIZZLE_128B tiles (6-stage ring), one bulk L2 prefetch per (layer,
//                      n-tile) block ahead; (non-TMA mode: 8 warps converting fp32 x to fp16)
//   warps 1–16         epilogue: tcgen05.ld the fp32 accumulator (TMEM lane = batch row), + bias,
//                      tanh, round to fp16, park in TMEM, then write the next layer's A operand
//                      (smem) per 128-k group; last layer: squared error vs. the teacher
//   warp 17            TMEM allocator + the MMA loop (whole warp, one elected lane issuing
//                      tcgen05.mma.kind::f16 M=128 N=128 K=16; fp32 accumulation in 512 TMEM columns)
// mlp32_kernel (N14, the definition, fp32-accurate): CTA pairs (2-CTA clusters), see below.
// The activations never leave the SM (A: 128 KB smem); weights are read from HBM exactly once.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "es_internal.h"
#include "fitness.cuh"   // tanh32 (N14)
#include "noise.cuh"
#include "tcgen05.cuh"   // PTX helpers: mbarriers, TMA, UMMA descriptors, tcgen05 mma/ld/st

namespace esb {

static constexpr int kBatch = 128;
static constexpr int kMaxLayers = 15;
static constexpr int kStages = 6;
static constexpr int kProdWarps = 8, kEpiWarps = 16;
static constexpr int kThreads = (kProdWarps + kEpiWarps + 1) * 32;
// TMA mode: one producer warp (a single thread issues the tile copies) instead of eight.
// (32 epilogue warps of 16 columns would double the warps per scheduler for the latency-bound
// epilogue, but 34 warps exceed the 1024-thread CTA limit; the code is generic in the count)
static constexpr int kEpiWarpsTma = 16;
static constexpr int kThreadsTma = (1 + kEpiWarpsTma + 1) * 32;
static constexpr int kTileBytes = 128 * 128;              // [128 rows × 64 k] fp16 = 16 KB
static constexpr int kABytes = 8 * kTileBytes;            // A: up to K = 512 (8 k-blocks)
static constexpr int kSmemBytes = kABytes + kStages * kTileBytes + 3072;   // + barriers, fp32 bias
static_assert(kSmemBytes <= 232448, "fp16-image MLP kernel exceeds 227 KB of shared memory");
#ifndef ES_MLP16_AHEAD
#define ES_MLP16_AHEAD 1   // L2 look-ahead of the fp16-image MLP producer, in (layer, n-tile) blocks
                           // (measured at C4: 1 → 1.72 ms, 2 → 1.79)
#endif

// ES_MLP_TRACE (profiling builds only): per-role wait / busy cycle totals of CTA 0, printed at exit.
#ifdef ES_MLP_TRACE
#define TR_DECL(v) long long v = 0
#define TR_T0(t) const long long t = clock64()
#define TR_ACC(v, t) v += clock64() - t
#else
#define TR_DECL(v)
#define TR_T0(t)
#define TR_ACC(v, t)
#endif

struct MlpParams {
  int nl;                       // layers L
  int w[kMaxLayers + 1];        // widths
  int kpad[kMaxLayers + 1];     // w rounded up to 64 (as K of the next layer)
  int npad[kMaxLayers + 1];     // w rounded up to 128 (as N)
  int64_t off[kMaxLayers + 1];  // offset of W_l in a parameter vector (l = 1..L)
  int64_t D;
  const float* x;               // [n][D]
  int64_t n;
  float* f;                     // [n] fitness (mode 0)
  const __half* uimg;           // layer-1 A image (pre-swizzled)
  float* Y;                     // [128][w_L] teacher outputs (read in mode 0, written in mode 1)
  int mode;
  const __half* x16;            // TMA mode: the fp16 parameter image [n][D] (N14′)
  CUtensorMap tmap[kMaxLayers + 1];   // TMA mode: per layer, 3-D (in, out, member) fp16 tiles
  // fp32-accurate kernel (N14): per batch half, the layer-1 A image of the scaled hi/lo split of U
  const __half* uimg32[2];
  float* Y32;                   // [128][w_L] teacher outputs of the fp32-accurate kernel
  const __half* img;            // split image [2][n][D] (hi plane, lo plane); biases read here
  CUtensorMap tmap32[2][kMaxLayers + 1];   // per plane (hi, lo) and layer: [64 n × 64 k] boxes
  double* part;                 // [n][2] per-half squared-error sums
  uint32_t* cnt;                // [n] arrival counters (zero between launches)
};

struct MlpProblem {
  MlpParams p;                  // x/n/f/mode filled per launch
  __half* uimg = nullptr;
  float* Y = nullptr;
  float* theta = nullptr;
  __half* uimg32 = nullptr;     // [2 halves][kpad0/64 k-blocks][128 rows][64] fp16
  float* Y32 = nullptr;
  double* part = nullptr;
  uint32_t* cnt = nullptr;
  __half* img = nullptr;        // split image [2][cap][D] (hi, lo planes of x·2^8)
  int64_t cap = 0;              // members part/cnt/img can hold
};


// Byte offset of the 16-byte chunk c (k = 8c..8c+7) of row r in a [rows × 64] fp16 K-major
// SWIZZLE_128B tile: 8-row groups of 1024 B, chunk index XOR (row mod 8).
__host__ __device__ __forceinline__ uint32_t swz(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

__device__ __forceinline__ uint4 pack8(const float* v) {
  uint4 o;
  __half2 h0 = __floats2half2_rn(v[0], v[1]), h1 = __floats2half2_rn(v[2], v[3]);
  __half2 h2 = __floats2half2_rn(v[4], v[5]), h3 = __floats2half2_rn(v[6], v[7]);
  o.x = *reinterpret_cast<uint32_t*>(&h0);
  o.y = *reinterpret_cast<uint32_t*>(&h1);
  o.z = *reinterpret_cast<uint32_t*>(&h2);
  o.w = *reinterpret_cast<uint32_t*>(&h3);
  return o;
}

// ---------------------------------------------------------------- the fitness kernel
template <bool TMA>
__global__ void __launch_bounds__(TMA ? kThreadsTma : kThreads, 1)
    mlp_kernel(const __grid_constant__ MlpParams P) {
  constexpr int kProd = TMA ? 1 : kProdWarps;          // producer warps
  constexpr int EW = TMA ? kEpiWarpsTma : kEpiWarps;    // epilogue warps
  constexpr int CW = 128 / (EW / 4);                    // columns per epilogue warp per n-tile
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* A = smem;                                 // [8][128 rows][64] fp16
  uint8_t* Bst = smem + kABytes;                     // [kStages][128 rows][64] fp16
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kABytes + kStages * kTileBytes);
  uint64_t* full = bars;                             // [kStages]
  uint64_t* empty = bars + kStages;                  // [kStages]
  uint64_t* dready = bars + 2 * kStages;             // [4] per 128-column n-tile of a layer
  uint64_t* aready = bars + 2 * kStages + 4;         // [4] per 128-k group of A
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 8);
  float* red = reinterpret_cast<float*>(bars + 2 * kStages + 9);   // [EW] (≤ 128 B)
  // TMA mode: the layer's fp16 bias, staged once per layer (≤ 512 values)
  float* bias_s = reinterpret_cast<float*>(smem + kABytes + kStages * kTileBytes + 512);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (smem_u32(smem) & 1023) __trap();               // SWIZZLE_128B needs 1024-B alignment

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], TMA ? 1 : kProdWarps);
      mbar_init(&empty[s], 1);
    }
    for (int k = 0; k < 4; ++k) mbar_init(&dready[k], 1);
    for (int k = 0; k < 4; ++k) mbar_init(&aready[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kProd + EW) {                          // TMEM: 512 fp32 columns × 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int L = P.nl;

  if (TMA && warp == 0) {
    // ------------------------------------------------------------ TMA producer (fp16 image):
    // whole warp, warp-uniform counters, one elected lane issues
    {
      if (lane == 0)
        for (int l = 1; l <= L; ++l)
          asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tmap[l])));
      __syncwarp();
      int stage = 0;
      uint32_t phase = 0;
      TR_DECL(tr_empty);
      TR_T0(tr_start);
      // L2 look-ahead by (layer, n-tile) block: contiguous rows, plain bulk L2 prefetches of 16 KB
      // per lane, two blocks ahead (the TMA engine only serves the tile loads)
      int64_t pm = blockIdx.x;
      int pl = 1, pnt = 0;
      const uintptr_t img_end = reinterpret_cast<uintptr_t>(P.x16) + (uintptr_t)P.n * P.D * 2;
      auto prefetch_block = [&]() {
        if (pm >= P.n) return;
        const int in = P.w[pl - 1], rows = min(128, P.w[pl] - pnt * 128);
        if (rows > 0) {
          const uintptr_t b0 = reinterpret_cast<uintptr_t>(P.x16) +
                               (uintptr_t)(pm * P.D + P.off[pl] + (int64_t)pnt * 128 * in) * 2;
          const uintptr_t lo = b0 & ~(uintptr_t)15;
          const uintptr_t hi = min(img_end, b0 + (uintptr_t)rows * in * 2 + 15) & ~(uintptr_t)15;
          for (uintptr_t o = lo + (uintptr_t)lane * 16384u; o < hi; o += 32u * 16384u)
            prefetch_l2(reinterpret_cast<const void*>(o), (uint32_t)min((uintptr_t)16384u, hi - o));
        }
        if (pnt == 0 && lane == 31) {                // the layer's bias (staged at layer start)
          const int out = P.w[pl];
          const uintptr_t b0 = reinterpret_cast<uintptr_t>(P.x16) +
                               (uintptr_t)(pm * P.D + P.off[pl] + (int64_t)out * in) * 2;
          const uintptr_t lo = b0 & ~(uintptr_t)15;
          const uintptr_t hi = min(img_end, b0 + (uintptr_t)out * 2 + 15) & ~(uintptr_t)15;
          if (hi > lo) prefetch_l2(reinterpret_cast<const void*>(lo), (uint32_t)(hi - lo));
        }
        if (++pnt == (P.npad[pl] >> 7)) {
          pnt = 0;
          if (++pl > L) { pl = 1; pm += gridDim.x; }
        }
      };
      for (int k = 0; k < ES_MLP16_AHEAD; ++k) prefetch_block();
      for (int64_t m = blockIdx.x; m < P.n; m += gridDim.x) {
        for (int l = 1; l <= L; ++l) {
          const int nt_n = P.npad[l] >> 7, kc_n = P.kpad[l - 1] >> 6;
          for (int nt = 0; nt < nt_n; ++nt) {
            prefetch_block();
            for (int kc = 0; kc < kc_n; ++kc) {
              TR_T0(tw);
              mbar_wait(&empty[stage], phase ^ 1);
              TR_ACC(tr_empty, tw);
              mbar_expect_tx_w(&full[stage], kTileBytes);
              tma_load_3d_w(Bst + stage * kTileBytes, &P.tmap[l], kc * 64, nt * 128, (int)m,
                            &full[stage]);
              if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
#ifdef ES_MLP_TRACE
      if (blockIdx.x == 0 && lane == 0)
        printf("mlp16 trace producer: total %lld wait_empty %lld\n", clock64() - tr_start, tr_empty);
#endif
    }
    __syncwarp();
  } else if (!TMA && warp < kProdWarps) {
    // ------------------------------------------------------------ producers
    const int t = threadIdx.x;                       // 0..255
    int stage = 0;
    uint32_t phase = 0;
    // Task stream: (member, layer, n-tile, k-chunk). The 128 weight rows of one (layer, n-tile)
    // are one contiguous block; when a block starts, warp 0 asks the TMA engine to prefetch the
    // NEXT block into L2 (cp.async.bulk.prefetch), so the LDG.128s below hit L2 and the HBM stream
    // does not depend on the producers' own load parallelism.
    auto block_of = [&](int64_t m, int l, int nt, const float** ptr, uint32_t* bytes) {
      const int in = P.w[l - 1], out = P.w[l];
      const int rows = min(128, out - nt * 128);
      *ptr = P.x + m * P.D + P.off[l] + (int64_t)nt * 128 * in;
      *bytes = rows > 0 ? (uint32_t)rows * in * 4u : 0u;
    };
    auto prefetch_block = [&](int64_t m, int l, int nt) {
      // next (layer, n-tile) after (m, l, nt) in stream order
      if (++nt >= (P.npad[l] >> 7)) { nt = 0; if (++l > L) { l = 1; m += gridDim.x; } }
      if (m >= P.n) return;
      const float* ptr;
      uint32_t bytes;
      block_of(m, l, nt, &ptr, &bytes);
      const uint32_t chunk = 8192;
      for (uint32_t o = lane * chunk; o < bytes; o += 32 * chunk)
        prefetch_l2(reinterpret_cast<const char*>(ptr) + o, min(chunk, bytes - o));
    };
    if (warp == 0 && blockIdx.x < P.n) {
      const float* ptr;
      uint32_t bytes;
      block_of(blockIdx.x, 1, 0, &ptr, &bytes);
      for (uint32_t o = lane * 8192u; o < bytes; o += 32 * 8192u)
        prefetch_l2(reinterpret_cast<const char*>(ptr) + o, min(8192u, bytes - o));
    }
    for (int64_t m = blockIdx.x; m < P.n; m += gridDim.x) {
      const float* xm = P.x + m * P.D;
      for (int l = 1; l <= L; ++l) {
        const int in = P.w[l - 1], out = P.w[l];
        const float* W = xm + P.off[l];
        const int nt_n = P.npad[l] >> 7, kc_n = P.kpad[l - 1] >> 6;
        for (int tile = 0; tile < nt_n * kc_n; ++tile) {
          const int nt = tile / kc_n, kc = tile % kc_n;
          if (kc == 0 && warp == 0) prefetch_block(m, l, nt);
          mbar_wait(&empty[stage], phase ^ 1);
          float4 v[8];
#pragma unroll
          for (int j = 0; j < 4; ++j) {              // 1024 chunks of 8 k per tile, 4 per thread
            const int ch = t + 256 * j, r = ch >> 3, c = ch & 7;
            const int n = nt * 128 + r, k = kc * 64 + c * 8;
            if (n < out && k < in) {
              const float4* src = reinterpret_cast<const float4*>(W + (int64_t)n * in + k);
              v[2 * j] = __ldcs(src);
              v[2 * j + 1] = __ldcs(src + 1);
            } else {
              v[2 * j] = v[2 * j + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
          uint8_t* dst = Bst + stage * kTileBytes;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int ch = t + 256 * j, r = ch >> 3, c = ch & 7;
            const float e[8] = {v[2 * j].x, v[2 * j].y, v[2 * j].z, v[2 * j].w,
                                v[2 * j + 1].x, v[2 * j + 1].y, v[2 * j + 1].z, v[2 * j + 1].w};
            *reinterpret_cast<uint4*>(dst + swz(r, c)) = pack8(e);
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[stage]);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp < kProd + EW) {
    // ------------------------------------------------------------ epilogue
    const int e = warp - kProd;                      // 0..EW-1
    // a warp may only tcgen05.ld the TMEM lane quarter (warp id mod 4); part = CW-column group
    const int q = warp & 3, part = e >> 2;
    const int row = q * 32 + lane;                   // batch row = TMEM lane
    const int et = threadIdx.x - kProd * 32;         // 0..511
    uint32_t dphase = 0;                             // bit k: parity of dready[k]
    TR_DECL(tr_dready);
    TR_T0(tr_start);
    for (int64_t m = blockIdx.x; m < P.n; m += gridDim.x) {
      const float* xm = P.x + m * P.D;
      // A <- layer-1 inputs (fp16 image, L2-resident)
      {
        const int bytes = (P.kpad[0] >> 6) * kTileBytes;
        const uint4* src = reinterpret_cast<const uint4*>(P.uimg);
        for (int o = et; o < bytes / 16; o += EW * 32)
          reinterpret_cast<uint4*>(A)[o] = __ldg(src + o);
        fence_async_smem();
        named_bar(1, EW * 32);
        if (et == 0)
          for (int g = 0; g < (P.kpad[0] + 127) >> 7; ++g) mbar_arrive(&aready[g]);
      }
      float sq = 0.0f;
      for (int l = 1; l <= L; ++l) {
        const int in = P.w[l - 1], out = P.w[l];
        const float* bias = TMA ? nullptr : xm + P.off[l] + (int64_t)out * in;
        const __half* bias16 = TMA ? P.x16 + m * P.D + P.off[l] + (int64_t)out * in : nullptr;
        const int ntl = P.npad[l] >> 7;              // n-tiles (dready barriers) of this layer
        if (TMA) {
          // stage the bias while the layer's MMAs run (its HBM latency was exposed per chunk)
          // staged as fp32 (the fp16 values exactly): one conversion per column, not per element
          for (int o = et; o < (out >> 3); o += EW * 32) {
            const uint4 hb = __ldg(reinterpret_cast<const uint4*>(bias16) + o);
            const __half* hh = reinterpret_cast<const __half*>(&hb);
            float4* d4 = reinterpret_cast<float4*>(bias_s + 8 * o);
            d4[0] = make_float4(__half2float(hh[0]), __half2float(hh[1]), __half2float(hh[2]), __half2float(hh[3]));
            d4[1] = make_float4(__half2float(hh[4]), __half2float(hh[5]), __half2float(hh[6]), __half2float(hh[7]));
          }
          for (int n = (out & ~7) + et; n < P.npad[l]; n += EW * 32)
            bias_s[n] = n < out ? __half2float(bias16[n]) : 0.0f;   // padded columns finite
          named_bar(1, EW * 32);
        }

        // hidden layers also zero-fill the padded K columns [out, kpad) of the next A. The next
        // A overwrites this layer's A, which the remaining n-tiles' MMAs are still reading, so the
        // packed fp16 results wait in TMEM — in the first 16 of the chunk's own (already read)
        // accumulator columns — until the layer's last n-tile has completed. Each n-tile's 128
        // columns are split over the four parts (32 each), so all 16 warps work on every tile as
        // soon as it completes and the last tile's epilogue is short.
        const int cend = l < L ? P.kpad[l] : out;
        const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
        // next layer's A, k group t, from the packed fp16 results parked in TMEM (zeros past out)
        auto write_a = [&](int t) {
          const int c0 = t * 128 + part * CW;
          if (c0 >= cend) return;
          uint4 h[4] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0),
                        make_uint4(0, 0, 0, 0)};
          if (c0 < out) {
            if (CW == 32) tmem_ld16(trow + (uint32_t)c0, h);
            else tmem_ld8(trow + (uint32_t)c0, h);
          }
#pragma unroll
          for (int c = 0; c < CW / 8; ++c) {         // CW/8 chunks of 8 k in k-block c0/64
            const int kb = c0 >> 6, ck = ((c0 & 63) >> 3) + c;
            *reinterpret_cast<uint4*>(A + kb * kTileBytes + swz(row, ck)) = h[c];
          }
        };
        for (int t = 0; t < ntl; ++t) {
          TR_T0(td);
          mbar_wait(&dready[t], (dphase >> t) & 1u);
          TR_ACC(tr_dready, td);
          tc_fence_after();
          if (l < L && t == ntl - 1 && t > 0) {
            // every MMA of this layer is done: A is free. k groups 0 … ntl−2 go first, so the
            // next layer's MMAs start on them while this last tile's epilogue runs
            for (int g = 0; g < ntl - 1; ++g) write_a(g);
            fence_async_smem();
            tc_fence_before();
            named_bar(1, EW * 32);
            if (et == 0)
              for (int g = 0; g < ntl - 1; ++g) mbar_arrive(&aready[g]);
          }
          const int c0 = t * 128 + part * CW;
          if (c0 >= cend || c0 >= out) continue;     // padded K columns: zeros, written below
          float v[CW];
          if (CW == 32) tmem_ld32(trow + (uint32_t)c0, v);
          else tmem_ld16f(trow + (uint32_t)c0, v);
          // bias (N14: fp16(b), uniform across the warp → broadcast loads)
          if (TMA) {
            // branch-free (the tanh chains interleave): past `out` the accumulator (zero-filled
            // weight rows) and the staged bias (padded with 0) are 0, and tanh(0) = 0
            // hidden layers: tanh16h (the value is rounded to binary16 next); the output layer
            // keeps tanh32 (its activation enters the squared error in fp32)
            if (l < L) {
#pragma unroll
              for (int i = 0; i < CW; i += 4) {
                const float4 b4 = *reinterpret_cast<const float4*>(bias_s + c0 + i);
                v[i] = tanh16h(__fadd_rn(v[i], b4.x));
                v[i + 1] = tanh16h(__fadd_rn(v[i + 1], b4.y));
                v[i + 2] = tanh16h(__fadd_rn(v[i + 2], b4.z));
                v[i + 3] = tanh16h(__fadd_rn(v[i + 3], b4.w));
              }
            } else {
#pragma unroll
              for (int i = 0; i < CW; i += 4) {
                const float4 b4 = *reinterpret_cast<const float4*>(bias_s + c0 + i);
                v[i] = tanh32(__fadd_rn(v[i], b4.x));
                v[i + 1] = tanh32(__fadd_rn(v[i + 1], b4.y));
                v[i + 2] = tanh32(__fadd_rn(v[i + 2], b4.z));
                v[i + 3] = tanh32(__fadd_rn(v[i + 3], b4.w));
              }
            }
          } else if (c0 + CW <= out) {
            // the same activations as the TMA path: tanh16h for hidden layers, tanh32 last
            auto act = [&](float a) { return l < L ? tanh16h(a) : tanh32(a); };
#pragma unroll
            for (int i = 0; i < CW; i += 4) {
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + c0 + i));
              v[i] = act(__fadd_rn(v[i], __half2float(__float2half_rn(b4.x))));
              v[i + 1] = act(__fadd_rn(v[i + 1], __half2float(__float2half_rn(b4.y))));
              v[i + 2] = act(__fadd_rn(v[i + 2], __half2float(__float2half_rn(b4.z))));
              v[i + 3] = act(__fadd_rn(v[i + 3], __half2float(__float2half_rn(b4.w))));
            }
          } else {
            auto act = [&](float a) { return l < L ? tanh16h(a) : tanh32(a); };
#pragma unroll
            for (int i = 0; i < CW; ++i) {
              const int n = c0 + i;
              v[i] = n < out ? act(__fadd_rn(v[i], __half2float(__float2half_rn(__ldg(bias + n)))))
                             : 0.0f;
            }
          }
          if (l < L) {
            uint4 h[CW / 8];
#pragma unroll
            for (int c = 0; c < CW / 8; ++c) h[c] = pack8(v + 8 * c);
            if (CW == 32) tmem_st16(trow + (uint32_t)c0, h);
            else tmem_st8(trow + (uint32_t)c0, h);
          } else if (P.mode == 0) {
            const float* yr = P.Y + (int64_t)row * out;
#pragma unroll
            for (int i = 0; i < CW; ++i) {
              const int n = c0 + i;
              if (n < out) {
                const float d = __fsub_rn(v[i], __ldg(yr + n));
                sq = __fmaf_rn(d, d, sq);
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < CW; ++i)
              if (c0 + i < out) P.Y[(int64_t)row * out + c0 + i] = v[i];
          }
        }
        if (l < L) write_a(ntl - 1);
        dphase ^= (1u << ntl) - 1u;                  // every n-tile barrier completed once
        tc_fence_before();
        if (l < L) {
          fence_async_smem();
          named_bar(1, EW * 32);
          if (et == 0) mbar_arrive(&aready[ntl - 1]);
        }
      }
      // fitness = Σ squares / (B · w_L)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
      if (lane == 0) red[e] = sq;
      named_bar(1, EW * 32);
      if (et == 0 && P.mode == 0) {
        double tot = 0.0;
        for (int k = 0; k < EW; ++k) tot += (double)red[k];
        P.f[m] = (float)(tot / ((double)kBatch * P.w[L]));
      }
      named_bar(1, EW * 32);
    }
#ifdef ES_MLP_TRACE
    if (TMA && blockIdx.x == 0 && et == 0)
      printf("mlp16 trace epi: total %lld dready %lld\n", clock64() - tr_start, tr_dready);
#endif
  } else {
    // ------------------------------------------------------------ MMA issuer (whole warp: the
    // loop's values stay warp-uniform; one elected lane issues each tcgen05 instruction)
    {
      const uint32_t idesc = idesc_f16(128, 128);
      int stage = 0;
      uint32_t phase = 0, aphase = 0;
      const uint32_t a_base = smem_u32(A), b_base = smem_u32(Bst);
      const uint64_t da0 = smem_desc(a_base), db0 = smem_desc(b_base);
      TR_DECL(tr_aready); TR_DECL(tr_full);
      TR_T0(tr_start);
      for (int64_t m = blockIdx.x; m < P.n; m += gridDim.x) {
        for (int l = 1; l <= L; ++l) {
          const int nt_n = P.npad[l] >> 7, kc_n = P.kpad[l - 1] >> 6;
          for (int nt = 0; nt < nt_n; ++nt) {
            const uint32_t dt = tmem + (uint32_t)(nt * 128);
            for (int kc = 0; kc < kc_n; ++kc) {
              if (nt == 0 && (kc & 1) == 0) {        // A's k group kc/2 (128 k) is written
                const int g = kc >> 1;
                TR_T0(ta);
                mbar_wait_cluster(&aready[g], (aphase >> g) & 1u);
                TR_ACC(tr_aready, ta);
                aphase ^= 1u << g;
                tc_fence_after();
              }
              TR_T0(tf);
              mbar_wait(&full[stage], phase);
              TR_ACC(tr_full, tf);
              tc_fence_after();
              // K = 16 per instruction, 64 per tile; descriptor = base + (byte offset >> 4)
              mma4k_commit_w(dt, da0 + (uint32_t)((kc * kTileBytes) >> 4),
                             db0 + (uint32_t)((stage * kTileBytes) >> 4), idesc, kc != 0,
                             &empty[stage]);          // ... and frees the stage when they finish
              // n-tile nt's accumulator is complete: its epilogue quarter starts while the
              // remaining n-tiles of the layer are still being multiplied
              if (kc == kc_n - 1) mma_commit_w(&dready[nt]);
              if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
#ifdef ES_MLP_TRACE
      if (TMA && blockIdx.x == 0 && lane == 0)
        printf("mlp16 trace mma: total %lld wait_aready %lld wait_full %lld\n", clock64() - tr_start,
               tr_aready, tr_full);
#endif
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kProd + EW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------- fp32-accurate kernel (N14)
// The definition (N14) is the MLP of the fp32 parameters. Each operand a is split into two binary16
// parts of the scaled value a·2^8: hi = fp16(a·2^8), lo = fp16(a·2^8 − hi) (≈ 22 significant bits
// together; the 2^8 scale keeps lo out of the binary16 subnormal range for |a| ≥ 2^-10, below which
// its absolute error is ≤ 2^-33). One 2-CTA cluster per member, CTA h holding batch rows
// 64h … 64h+63 as A = [A_hi; A_lo] (128 rows). CTA 0 issues `tcgen05.mma.cta_group::2` with M = 256
// (both CTAs' rows) and N = 128 output columns, W_hi and W_lo products accumulated into the same
// TMEM columns, so in each CTA row b + row 64+b of D = (A_hi + A_lo)(W_hi + W_lo)[b] = 2^16·(h·W)[b]
// to fp32 accuracy (the lo·lo product is negligible and free). The weights are the population's
// split image — two binary16 planes [2][n][D] written by the ask (or mlp_split_kernel) — and each
// CTA TMA-loads ITS 64 of the tile's 128 weight rows of both planes (the pair MMA takes B rows
// 0–63 from CTA 0's shared memory and 64–127 from CTA 1's), the bytes counted on CTA 0's barrier;
// the MMA's multicast commits free both CTAs' stages and signal both epilogues; the epilogues
// arrive on CTA 0's per-128-k-group `aready` barriers remotely. The pair's squared-error halves are
// combined in a fixed order by whichever CTA finishes second. Epilogue: the hi warp (lanes 0–63)
// and lo warp (64–127) of a column part swap 16 columns through shared memory so both finish 16
// columns (bias, tanh, split into the next A, parked in TMEM until A is free). Stages hold 64 k
// (128-byte SWIZZLE_128B rows): the TMA unit's cost goes with the number of rows it moves, and
// 128-byte rows halve it against [128 n × 32 k] 64-byte-row tiles (C4: 4.31 vs 4.62 ms).
#ifndef ES_MLP_AHEAD
#define ES_MLP_AHEAD 1   // L2 look-ahead of the fp32 MLP producer, in (layer, n-tile) blocks
                         // (measured at C4: 1 → 4.54 ms, 2 → 4.66, 3 → 4.94)
#endif
static constexpr int kStages32 = 5;
static constexpr int kH32Bytes = 64 * 128;                       // [64 n × 64 k] fp16 = 8 KB
static constexpr int kStage32Bytes = 2 * kH32Bytes;              // this CTA's hi half + lo half
static constexpr int kXbufBytes = 8 * 2 * 8 * 32 * 4;            // 8 pairs × 2 dirs × 8 cols × 32
static constexpr int kBias32Bytes = 512 * 4;                     // the layer's fp32 bias
static constexpr int kSmem32Bytes =
    kABytes + kStages32 * kStage32Bytes + kXbufBytes + kBias32Bytes + 1024;
static_assert(kSmem32Bytes <= 232448, "fp32 MLP kernel exceeds 227 KB of shared memory");
static constexpr int kThreads32 = (1 + kEpiWarps + 1) * 32;
static constexpr float kSplitScale = 256.0f, kUnscale = 1.0f / 65536.0f;

// hi / lo binary16 parts of 8 values already scaled by 2⁸
__device__ __forceinline__ void split8s(const float* s, uint4& hi, uint4& lo) {
  float r[8];
  hi = pack8(s);
  const __half* h = reinterpret_cast<const __half*>(&hi);
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = __fsub_rn(s[i], __half2float(h[i]));
  lo = pack8(r);
}

// hi / lo binary16 parts of 8 scaled values
__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  float s[8], r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) s[i] = __fmul_rn(v[i], kSplitScale);
  hi = pack8(s);
  const __half* h = reinterpret_cast<const __half*>(&hi);
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = __fsub_rn(s[i], __half2float(h[i]));
  lo = pack8(r);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads32, 1)
    mlp32_kernel(const __grid_constant__ MlpParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* A = smem;                                              // [8][128 rows][64] fp16
  uint8_t* Bst = smem + kABytes;                                  // [5][hi, lo][64][64] fp16
  float* xbuf = reinterpret_cast<float*>(smem + kABytes + kStages32 * kStage32Bytes);
  float* bias_s = reinterpret_cast<float*>(smem + kABytes + kStages32 * kStage32Bytes + kXbufBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kABytes + kStages32 * kStage32Bytes +
                                               kXbufBytes + kBias32Bytes);
  uint64_t* full = bars;                                          // [kStages32]
  uint64_t* empty = bars + kStages32;
  uint64_t* dready = bars + 2 * kStages32;                        // [4]
  uint64_t* aready = bars + 2 * kStages32 + 4;                    // [4] per 128-k group of A
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages32 + 8);
  double* red = reinterpret_cast<double*>(bars + 2 * kStages32 + 9);   // [kEpiWarps]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = blockIdx.x & 1;
  const int64_t pair = blockIdx.x >> 1, npair = gridDim.x >> 1;
  if (smem_u32(smem) & 1023) __trap();

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages32; ++s) {
      mbar_init(&full[s], 1);                    // CTA 0's: its producer's expect_tx
      mbar_init(&empty[s], 1);                   // the pair MMA's multicast commit
    }
    for (int k = 0; k < 4; ++k) mbar_init(&dready[k], 1);
    for (int k = 0; k < 4; ++k) mbar_init(&aready[k], 2);   // CTA 0's: both CTAs' epilogues
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1 + kEpiWarps) {                   // the same warp in both CTAs of the pair
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();                            // the peer's barriers exist before any signal
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int L = P.nl;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (split image):
    // the whole warp runs the loop (warp-uniform counters, no divisions); one elected lane issues
    {
      if (lane == 0)
        for (int l = 1; l <= L; ++l) {
          asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tmap32[0][l])));
          asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tmap32[1][l])));
        }
      __syncwarp();
      int stage = 0;
      uint32_t phase = 0;
      TR_DECL(tr_empty);
      TR_T0(tr_start);
      // L2 look-ahead by (layer, n-tile) block: the block's rows of this CTA's plane are one
      // contiguous range (≤ 128 rows × in × 2 B), prefetched with plain bulk L2 prefetches, 16 KB
      // per lane, two blocks ahead of the loads — the TMA engine only serves the tile loads
      // (tensor prefetches, one per tile and plane, had doubled its 64-B row requests)
      int64_t pm = pair;
      int pl = 1, pnt = 0;
      const char* plane0 = reinterpret_cast<const char*>(P.img + (int64_t)half * P.n * P.D);
      const uintptr_t plane_end = reinterpret_cast<uintptr_t>(plane0) + (uintptr_t)P.n * P.D * 2;
      auto prefetch_block = [&]() {
        if (pm >= P.n) return;
        const int in = P.w[pl - 1], rows = min(128, P.w[pl] - pnt * 128);
        if (rows > 0) {
          const uintptr_t b0 = reinterpret_cast<uintptr_t>(plane0) +
                               (uintptr_t)(pm * P.D + P.off[pl] + (int64_t)pnt * 128 * in) * 2;
          const uintptr_t lo = b0 & ~(uintptr_t)15;
          const uintptr_t hi = min(plane_end, b0 + (uintptr_t)rows * in * 2 + 15) & ~(uintptr_t)15;
          for (uintptr_t o = lo + (uintptr_t)lane * 16384u; o < hi; o += 32u * 16384u)
            prefetch_l2(reinterpret_cast<const void*>(o), (uint32_t)min((uintptr_t)16384u, hi - o));
        }
        if (pnt == 0 && lane == 31) {                // the layer's bias (this plane's part)
          const int out = P.w[pl];
          const uintptr_t b0 = reinterpret_cast<uintptr_t>(plane0) +
                               (uintptr_t)(pm * P.D + P.off[pl] + (int64_t)out * in) * 2;
          const uintptr_t lo = b0 & ~(uintptr_t)15;
          const uintptr_t hi = min(plane_end, b0 + (uintptr_t)out * 2 + 15) & ~(uintptr_t)15;
          if (hi > lo) prefetch_l2(reinterpret_cast<const void*>(lo), (uint32_t)(hi - lo));
        }
        if (++pnt == (P.npad[pl] >> 7)) {
          pnt = 0;
          if (++pl > L) { pl = 1; pm += npair; }
        }
      };
      for (int k = 0; k < ES_MLP_AHEAD; ++k) prefetch_block();
      for (int64_t m = pair; m < P.n; m += npair) {
        for (int l = 1; l <= L; ++l) {
          const int nt_n = P.npad[l] >> 7, kc_n = P.kpad[l - 1] >> 6;
          for (int nt = 0; nt < nt_n; ++nt) {
            prefetch_block();
            for (int kc = 0; kc < kc_n; ++kc) {
              // the pair MMA (M = 256, N = 128) takes B rows 0–63 from CTA 0 and 64–127 from CTA 1:
              // each CTA loads its 64 rows of both planes; the bytes count on CTA 0's barrier
              TR_T0(tw);
              mbar_wait(&empty[stage], phase ^ 1);
              TR_ACC(tr_empty, tw);
              if (half == 0) mbar_expect_tx_w(&full[stage], 2 * kStage32Bytes);
              uint8_t* dst = Bst + stage * kStage32Bytes;
              const int n0 = nt * 128 + half * 64;
              tma_load_3d_2sm_w(dst, &P.tmap32[0][l], kc * 64, n0, (int)m, &full[stage]);
              tma_load_3d_2sm_w(dst + kH32Bytes, &P.tmap32[1][l], kc * 64, n0, (int)m, &full[stage]);
              if (++stage == kStages32) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
#ifdef ES_MLP_TRACE
      if (blockIdx.x == 0 && lane == 0)
        printf("mlp32 trace producer: total %lld wait_empty %lld\n", clock64() - tr_start, tr_empty);
#endif
    }
    __syncwarp();
  } else if (warp < 1 + kEpiWarps) {
    // ------------------------------------------------------------ epilogue
    // Warp pair (hi, lo) = (q, q ^ 2) of one 32-column part: the hi warp's lanes hold the A_hi
    // rows' accumulators D[b], the lo warp's D[64 + b], both for batch row b. They swap 16 columns
    // through shared memory, so BOTH finish 16 columns of b = D[b] + D[64+b]: the hi warp columns
    // 0–15 of the part, the lo warp 16–31 (+ bias, tanh, split, or the squared error).
    const int e = warp - 1;                          // 0..15
    const int q = warp & 3, part = e >> 2;           // TMEM lane quarter, 32-column quarter
    const bool hiw = q < 2;                          // lanes 0–63: the A_hi rows
    const int prid = part * 2 + (q & 1);             // named barrier of the pair
    const int side = hiw ? 0 : 16;                   // this warp's 16 result columns in the part
    // [2 col quads][32 lanes] float4 I write / the peer wrote (16-byte accesses: 4 per round)
    float4* xmine = reinterpret_cast<float4*>(xbuf + (prid * 2 + (hiw ? 0 : 1)) * (8 * 32));
    const float4* xpeer = reinterpret_cast<const float4*>(xbuf + (prid * 2 + (hiw ? 1 : 0)) * (8 * 32));
    const int rh = (q & 1) * 32 + lane;              // batch row within the half (A rows rh, 64+rh)
    const int brow = half * 64 + rh;                 // batch row of this lane
    const int et = threadIdx.x - 32;                 // 0..511
    uint32_t dphase = 0;
    TR_DECL(tr_dready); TR_DECL(tr_tile); TR_DECL(tr_awrite); TR_DECL(tr_bias);
    TR_T0(tr_start);
    for (int64_t m = pair; m < P.n; m += npair) {
      const __half* bhi = P.img + m * P.D;             // this member's hi / lo planes
      const __half* blo = P.img + (P.n + m) * P.D;
      {
        const int bytes = (P.kpad[0] >> 6) * kTileBytes;
        const uint4* src = reinterpret_cast<const uint4*>(P.uimg32[half]);
        for (int o = et; o < bytes / 16; o += kEpiWarps * 32)
          reinterpret_cast<uint4*>(A)[o] = __ldg(src + o);
        fence_async_smem();
        named_bar(1, kEpiWarps * 32);
        if (et == 0)
          for (int g = 0; g < (P.kpad[0] + 127) >> 7; ++g) mbar_arrive_remote(&aready[g], 0);
      }
      double sq = 0.0;
      for (int l = 1; l <= L; ++l) {
        const int in = P.w[l - 1], out = P.w[l];
        const int64_t boff = P.off[l] + (int64_t)out * in;   // b_l inside the layer block
        const int ntl = P.npad[l] >> 7;
        const int cend = l < L ? P.kpad[l] : out;
        // b = (hi + lo)·2^-8 (exact in fp32: ≤ 22 significant bits), staged while the MMAs run
        TR_T0(tb);
        for (int n = et; n < P.npad[l]; n += kEpiWarps * 32)
          bias_s[n] = n < out ? __fmul_rn(__fadd_rn(__half2float(bhi[boff + n]),
                                                    __half2float(blo[boff + n])), 1.0f / kSplitScale)
                              : 0.0f;
        named_bar(1, kEpiWarps * 32);
        TR_ACC(tr_bias, tb);
        const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
        // next layer's A, k group t (rows rh: hi split, 64 + rh: lo split) from the split values
        // parked in TMEM; padded K columns [out, kpad) written as zeros
        auto write_a = [&](int t) {
          const int cb = t * 128 + part * 32 + side;
          if (cb >= cend) return;
          uint4 h[4] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0),
                        make_uint4(0, 0, 0, 0)};
          if (cb - side < out) tmem_ld16(trow + (uint32_t)cb, h);
          const int kb = cb >> 6, ck = (cb & 63) >> 3;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            *reinterpret_cast<uint4*>(A + kb * kTileBytes + swz(rh, ck + c)) = h[c];
            *reinterpret_cast<uint4*>(A + kb * kTileBytes + swz(64 + rh, ck + c)) = h[2 + c];
          }
        };
        for (int t = 0; t < ntl; ++t) {
          TR_T0(td);
          mbar_wait(&dready[t], (dphase >> t) & 1u);
          TR_ACC(tr_dready, td);
          TR_T0(tt);
          tc_fence_after();
          if (l < L && t == ntl - 1 && t > 0) {
            // every MMA of this layer is done: A is free. Groups 0 … ntl−2 go first, so the next
            // layer's MMAs start on them while this last tile's epilogue runs
            for (int g = 0; g < ntl - 1; ++g) write_a(g);
            fence_async_smem();
            tc_fence_before();
            named_bar(1, kEpiWarps * 32);
            if (et == 0)
              for (int g = 0; g < ntl - 1; ++g) mbar_arrive_remote(&aready[g], 0);
          }
          const int c0 = t * 128 + part * 32;
          if (c0 >= cend || c0 >= out) continue;     // both warps of the pair skip together
          float v[32];
          tmem_ld32(trow + (uint32_t)c0, v);
          // swap the peer's half of the 32 columns in two rounds of 8 through one 8-column buffer
          // per direction (4 barriers of the pair: the buffer is rewritten only after the peer
          // has read it)
          float x[16];
#pragma unroll
          for (int rr = 0; rr < 2; ++rr) {
            named_bar(2 + prid, 64);
            // warp-uniform roles (no per-value selects): the hi warp hands over columns 16–31
            // of the part and finishes 0–15, the lo warp the reverse
            if (hiw) {
              xmine[lane] = make_float4(v[16 + 8 * rr], v[17 + 8 * rr], v[18 + 8 * rr], v[19 + 8 * rr]);
              xmine[32 + lane] = make_float4(v[20 + 8 * rr], v[21 + 8 * rr], v[22 + 8 * rr], v[23 + 8 * rr]);
            } else {
              xmine[lane] = make_float4(v[8 * rr], v[1 + 8 * rr], v[2 + 8 * rr], v[3 + 8 * rr]);
              xmine[32 + lane] = make_float4(v[4 + 8 * rr], v[5 + 8 * rr], v[6 + 8 * rr], v[7 + 8 * rr]);
            }
            named_bar(2 + prid, 64);
            const float4 p0 = xpeer[lane], p1 = xpeer[32 + lane];
            const float pv[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
            if (hiw) {
#pragma unroll
              for (int i = 0; i < 8; ++i) x[8 * rr + i] = __fadd_rn(v[8 * rr + i], pv[i]);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) x[8 * rr + i] = __fadd_rn(v[16 + 8 * rr + i], pv[i]);
            }
          }
          const int cb = c0 + side;                  // first of this warp's 16 columns
          // a = D·2^-16 + b (the product by 2^-16 is exact), h = tanh(a)
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            const float4 b4 = *reinterpret_cast<const float4*>(bias_s + cb + i);
            const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
            // branch-free over the 16 columns (so the 16 tanh chains interleave): past `out` the
            // accumulator (zero-filled weight rows) and the staged bias are 0, and tanh(0) = 0
            // hidden layers: 2⁸·tanh (the split's scale folded into the rational's numerator)
            if (l < L) {
#pragma unroll
              for (int u = 0; u < 4; ++u) x[i + u] = tanh32_x256(__fmaf_rn(x[i + u], kUnscale, bb[u]));
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u) x[i + u] = tanh32(__fmaf_rn(x[i + u], kUnscale, bb[u]));
            }
          }
          if (l < L) {
            uint4 h[4];                              // hi split of 16 columns, then the lo split
            split8s(x, h[0], h[2]);
            split8s(x + 8, h[1], h[3]);
            tmem_st16(trow + (uint32_t)cb, h);       // parked in this lane's consumed columns
          } else if (P.mode == 0) {
            const float* yr = P.Y32 + (int64_t)brow * out;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int n = cb + i;
              if (n < out) {
                const double d = (double)x[i] - (double)__ldg(yr + n);
                sq = __fma_rn(d, d, sq);
              }
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (cb + i < out) P.Y32[(int64_t)brow * out + cb + i] = x[i];
          }
          TR_ACC(tr_tile, tt);
        }
        TR_T0(ta);
        if (l < L) write_a(ntl - 1);
        dphase ^= (1u << ntl) - 1u;
        tc_fence_before();
        if (l < L) {
          fence_async_smem();
          named_bar(1, kEpiWarps * 32);
          if (et == 0) mbar_arrive_remote(&aready[ntl - 1], 0);
        }
        TR_ACC(tr_awrite, ta);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
      if (lane == 0) red[e] = sq;
      named_bar(1, kEpiWarps * 32);
      if (et == 0 && P.mode == 0) {
        double tot = 0.0;
        for (int k = 0; k < kEpiWarps; ++k) tot = __dadd_rn(tot, red[k]);
        // combine the two halves in a fixed order, whichever CTA arrives second
        P.part[2 * m + half] = tot;
        __threadfence();
        const uint32_t prev = atomicAdd(&P.cnt[m], 1u);
        if (prev == 1u) {
          __threadfence();
          const double s2 = __dadd_rn(__ldcg(&P.part[2 * m]), __ldcg(&P.part[2 * m + 1]));
          P.f[m] = (float)(s2 / ((double)kBatch * P.w[L]));
          P.cnt[m] = 0u;
        }
      }
      named_bar(1, kEpiWarps * 32);
    }
#ifdef ES_MLP_TRACE
    if (blockIdx.x == 0 && (et == 0 || et == 32 * 8))
      printf("mlp32 trace epi warp %d: total %lld dready %lld tiles %lld awrite %lld bias %lld\n", e,
             clock64() - tr_start, tr_dready, tr_tile, tr_awrite, tr_bias);
#endif
  } else {
    // ------------------------------------------------------------ MMA issuer: CTA 0 of the pair
    // (whole warp, one elected lane issues); M = 256 = both CTAs' [A_hi; A_lo] rows, N = 128
    if (half == 0) {
      const uint32_t idesc = idesc_f16(256, 128);
      int stage = 0;
      uint32_t phase = 0, aphase = 0;                // aphase bit g: parity of aready[g]
      const uint32_t a_base = smem_u32(A), b_base = smem_u32(Bst);
      const uint64_t da0 = smem_desc(a_base), db0 = smem_desc(b_base);   // SWIZZLE_128B, 64-k rows
      TR_DECL(tr_aready); TR_DECL(tr_full);
      TR_T0(tr_start);
      for (int64_t m = pair; m < P.n; m += npair) {
        for (int l = 1; l <= L; ++l) {
          const int nt_n = P.npad[l] >> 7, kc_n = P.kpad[l - 1] >> 6;
          for (int nt = 0; nt < nt_n; ++nt) {
            const uint32_t dt = tmem + (uint32_t)(nt * 128);
            for (int kc = 0; kc < kc_n; ++kc) {
              if (nt == 0 && (kc & 1) == 0) {        // A's k group kc/2 (128 k) is written
                const int g = kc >> 1;
                TR_T0(ta);
                mbar_wait(&aready[g], (aphase >> g) & 1u);
                TR_ACC(tr_aready, ta);
                aphase ^= 1u << g;
                tc_fence_after();
              }
              TR_T0(tf);
              mbar_wait(&full[stage], phase);
              TR_ACC(tr_full, tf);
              tc_fence_after();
              // K = 16 per instruction, 64 per stage: descriptors = base + (byte offset >> 4)
              // (the 14-bit address field cannot carry: shared memory < 256 KB)
              const uint32_t ao = (uint32_t)(kc * kTileBytes) >> 4;
              const uint32_t bo = (uint32_t)(stage * kStage32Bytes) >> 4;
              mma8_commit_2sm_w(dt, da0 + ao, db0 + bo, db0 + bo + (kH32Bytes >> 4), idesc, kc != 0,
                                &empty[stage], 3);      // ... and frees the stage in both CTAs
              if (kc == kc_n - 1) mma_commit_2sm_mc_w(&dready[nt], 3);
              if (++stage == kStages32) { stage = 0; phase ^= 1; }
            }
          }
        }
      }
#ifdef ES_MLP_TRACE
      if (blockIdx.x == 0 && lane == 0)
        printf("mlp32 trace mma: total %lld wait_aready %lld wait_full %lld\n", clock64() - tr_start,
               tr_aready, tr_full);
#endif
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();                            // no CTA leaves while its peer may still signal it
  if (warp == 1 + kEpiWarps) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// fp32 parameters → the split image [2][n][D] (plane 0 = hi, plane 1 = lo), 8 values per thread.
__global__ void mlp_split_kernel(const float* __restrict__ x, int64_t total, __half* __restrict__ img) {
  const int64_t i8 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (i8 >= total) return;
  float v[8];
  if (i8 + 8 <= total && ((reinterpret_cast<uintptr_t>(x + i8) & 15) == 0)) {
    const float4 a = __ldcs(reinterpret_cast<const float4*>(x + i8));
    const float4 b = __ldcs(reinterpret_cast<const float4*>(x + i8) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = i8 + i < total ? x[i8 + i] : 0.0f;
  }
  uint4 hi, lo;
  split8(v, hi, lo);
  if (i8 + 8 <= total) {
    __stcs(reinterpret_cast<uint4*>(img + i8), hi);
    __stcs(reinterpret_cast<uint4*>(img + total + i8), lo);
  } else {
    const __half* h = reinterpret_cast<const __half*>(&hi);
    const __half* g = reinterpret_cast<const __half*>(&lo);
    for (int i = 0; i < 8 && i8 + i < total; ++i) {
      img[i8 + i] = h[i];
      img[total + i8 + i] = g[i];
    }
  }
}

// U (DATA stream) → the layer-1 A images of the fp32-accurate kernel: for batch half h, rows
// 0–63 = hi(U[64h + r]·2^8), rows 64–127 = lo (same pre-swizzled layout as mlp_uimg_kernel).
__global__ void mlp_uimg32_kernel(uint64_t seed, int w0, int kpad0, __half* img) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;   // one thread per (half, row, 8-k chunk)
  const int chunks = kpad0 / 8;
  if (idx >= 2 * 64 * chunks) return;
  const int hf = idx / (64 * chunks), r = (idx / chunks) % 64, cc = idx % chunks;
  const Philox ph(seed);
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; i += 4) {
    const int k = cc * 8 + i;
    if (k < w0) {
      const float4 z = normal4(ph, (uint32_t)(k / 4), (uint32_t)(64 * hf + r), 0u, TAG_DATA);
      v[i] = z.x; v[i + 1] = z.y; v[i + 2] = z.z; v[i + 3] = z.w;
    } else {
      v[i] = v[i + 1] = v[i + 2] = v[i + 3] = 0.f;
    }
  }
  uint4 hi, lo;
  split8(v, hi, lo);
  const int kb = cc / 8, c = cc % 8;
  uint8_t* base = reinterpret_cast<uint8_t*>(img) + (size_t)hf * (kpad0 / 64) * kTileBytes +
                  kb * kTileBytes;
  *reinterpret_cast<uint4*>(base + swz(r, c)) = hi;
  *reinterpret_cast<uint4*>(base + swz(64 + r, c)) = lo;
}

// ---------------------------------------------------------------- problem setup kernels
// U (DATA stream) → fp16 → the pre-swizzled layer-1 A image.
__global__ void mlp_uimg_kernel(uint64_t seed, int w0, int kpad0, __half* img) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;   // one thread per (row, 8-k chunk)
  const int chunks = kpad0 / 8;
  if (idx >= kBatch * chunks) return;
  const int r = idx / chunks, cc = idx % chunks;
  const Philox ph(seed);
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; i += 4) {
    const int k = cc * 8 + i;
    if (k < w0) {
      const float4 z = normal4(ph, (uint32_t)(k / 4), (uint32_t)r, 0u, TAG_DATA);
      v[i] = z.x; v[i + 1] = z.y; v[i + 2] = z.z; v[i + 3] = z.w;
    } else {
      v[i] = v[i + 1] = v[i + 2] = v[i + 3] = 0.f;
    }
  }
  const int kb = cc / 8, c = cc % 8;
  uint8_t* base = reinterpret_cast<uint8_t*>(img) + kb * kTileBytes + swz(r, c);
  *reinterpret_cast<uint4*>(base) = pack8(v);
}

// θ* (TEACHER stream): W*_l[n][k] = z ⊗ (float)(1/√in), b* = 0.
__global__ void mlp_teacher_kernel(uint64_t seed, int l, int in, int out, float scale,
                                   float* W) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)out * in + out) return;
  if (idx >= (int64_t)out * in) {
    W[idx] = 0.0f;
    return;
  }
  const int n = (int)(idx / in), k = (int)(idx % in);
  const Philox ph(seed);
  const float4 z = normal4(ph, (uint32_t)(k / 4), (uint32_t)(4096 * l + n), 0u, TAG_TEACHER);
  W[idx] = __fmul_rn(f4get(z, k % 4), scale);
}

void mlp_problem_destroy(void* prob);
static cudaError_t mlp_reserve(MlpProblem* pr, int64_t n, cudaStream_t st);

static void fill_params(MlpParams& p, const int32_t* widths, int nw) {
  p.nl = nw - 1;
  int64_t off = 0;
  for (int l = 0; l < nw; ++l) {
    p.w[l] = widths[l];
    p.kpad[l] = (widths[l] + 63) / 64 * 64;
    p.npad[l] = (widths[l] + 127) / 128 * 128;
  }
  for (int l = 1; l < nw; ++l) {
    p.off[l] = off;
    off += (int64_t)widths[l - 1] * widths[l] + widths[l];
  }
  p.off[0] = 0;
  p.D = off;
}

// Per plane and layer: the split image viewed as a 3-D tensor (k = in, n = out, member) with
// strides (2 B, in·2 B, D·2 B); a box of 64 k × 64 n × 1 member lands in smem in the UMMA K-major
// SWIZZLE_128B layout of one plane of a stage (rows past `out` / columns past `in` are zero-filled).
static cudaError_t encode_maps32(MlpParams& q, const __half* img, int64_t n) {
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc) return cudaErrorNotSupported;
  for (int pl = 0; pl < 2; ++pl) {
    const __half* base = img + (size_t)pl * n * q.D;
    for (int l = 1; l <= q.nl; ++l) {
      const cuuint64_t dims[3] = {(cuuint64_t)q.w[l - 1], (cuuint64_t)q.w[l], (cuuint64_t)n};
      const cuuint64_t strides[2] = {(cuuint64_t)q.w[l - 1] * 2, (cuuint64_t)q.D * 2};
      const cuuint32_t box[3] = {64, 64, 1};        // one CTA's half of a [128 n × 64 k] tile
      const cuuint32_t es[3] = {1, 1, 1};
      CUresult r = enc(&q.tmap32[pl][l], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
                       const_cast<__half*>(base + q.off[l]), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
  }
  return cudaSuccess;
}

// fp32-accurate kernel on the split image img [2][n][D]
static cudaError_t launch_mlp32(MlpParams q, const __half* img, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  if (cudaError_t e = smem_attr_once((const void*)mlp32_kernel, kSmem32Bytes, attr)) return e;
  if (cudaError_t e = encode_maps32(q, img, q.n)) return e;
  q.img = img;
  // persistent: as many CTA pairs as can be co-resident (not every SM has a cluster partner),
  // so that no pair waits for a second wave
  static std::atomic<int> max_pairs{0};
  int mp = max_pairs.load();
  if (mp == 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * (unsigned)std::max(1, sm_count() / 2));
    cfg.blockDim = dim3(kThreads32);
    cfg.dynamicSmemBytes = kSmem32Bytes;
    cudaLaunchAttribute at{};
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = 2; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&mp, (const void*)mlp32_kernel, &cfg) != cudaSuccess || mp < 1)
      mp = std::max(1, sm_count() / 2);
    max_pairs.store(mp);
  }
  const int pairs = (int)std::min<int64_t>(q.n, mp);
  mlp32_kernel<<<2 * pairs, kThreads32, kSmem32Bytes, st>>>(q);
  return cudaGetLastError();
}

static cudaError_t launch_split(const float* x, int64_t total, __half* img, cudaStream_t st) {
  const int64_t thr = (total + 7) / 8;
  mlp_split_kernel<<<(unsigned)((thr + 255) / 256), 256, 0, st>>>(x, total, img);
  return cudaGetLastError();
}

static cudaError_t launch_mlp(const MlpParams& p, cudaStream_t st) {
  static std::atomic<uint64_t> attr0{0}, attr1{0};
  if (cudaError_t e = smem_attr_once((const void*)mlp_kernel<false>, kSmemBytes, attr0)) return e;
  if (cudaError_t e = smem_attr_once((const void*)mlp_kernel<true>, kSmemBytes, attr1)) return e;
  const int grid = (int)std::min<int64_t>(p.n, sm_count());
  if (p.x16) mlp_kernel<true><<<grid, kThreadsTma, kSmemBytes, st>>>(p);
  else mlp_kernel<false><<<grid, kThreads, kSmemBytes, st>>>(p);
  return cudaGetLastError();
}


// Per layer: the fp16 image viewed as a 3-D tensor (k = in, n = out, member) with strides
// (2 B, in·2 B, D·2 B); a box of 64 k × 128 n × 1 member lands in smem in exactly the UMMA
// K-major SWIZZLE_128B layout of a B stage (rows past `out` / columns past `in` are zero-filled).
static cudaError_t encode_maps(MlpParams& q, const __half* x16, int64_t n) {
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc) return cudaErrorNotSupported;
  for (int l = 1; l <= q.nl; ++l) {
    const cuuint64_t dims[3] = {(cuuint64_t)q.w[l - 1], (cuuint64_t)q.w[l], (cuuint64_t)n};
    const cuuint64_t strides[2] = {(cuuint64_t)q.w[l - 1] * 2, (cuuint64_t)q.D * 2};
    const cuuint32_t box[3] = {64, 128, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&q.tmap[l], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
                     const_cast<__half*>(x16 + q.off[l]), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

void* mlp_problem_create(const int32_t* widths, int32_t nw, int32_t batch, uint64_t seed,
                         cudaStream_t st, std::string* err) {
  if (batch != kBatch) { *err = "unsupported: batch must be 128"; return nullptr; }
  if (nw < 2 || nw > kMaxLayers + 1) { *err = "need 2..16 widths"; return nullptr; }
  for (int l = 0; l < nw; ++l) {
    if (widths[l] < 16 || widths[l] % 16 || widths[l] > 512) {
      *err = "unsupported: widths must be multiples of 16 in [16, 512]";
      return nullptr;
    }
  }
  MlpProblem* pr = new MlpProblem();
  fill_params(pr->p, widths, nw);
  const MlpParams& p = pr->p;
  cudaError_t e = cudaSuccess;
  const size_t img = (size_t)(p.kpad[0] / 64) * kTileBytes;
  if ((e = cudaMalloc(&pr->uimg, img)) != cudaSuccess ||
      (e = cudaMalloc(&pr->Y, (size_t)kBatch * widths[nw - 1] * sizeof(float))) != cudaSuccess ||
      (e = cudaMalloc(&pr->theta, (size_t)p.D * sizeof(float))) != cudaSuccess) {
    *err = std::string("allocation: ") + cudaGetErrorString(e);
    mlp_problem_destroy(pr);
    return nullptr;
  }
  const int nthr = kBatch * (p.kpad[0] / 8);
  mlp_uimg_kernel<<<(nthr + 255) / 256, 256, 0, st>>>(seed, widths[0], p.kpad[0], pr->uimg);
  for (int l = 1; l < nw; ++l) {
    const int64_t cnt = (int64_t)widths[l] * widths[l - 1] + widths[l];
    const float sc = (float)(1.0 / std::sqrt((double)widths[l - 1]));
    mlp_teacher_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(
        seed, l, widths[l - 1], widths[l], sc, pr->theta + p.off[l]);
  }
  if ((e = cudaMalloc(&pr->uimg32, 2 * img)) != cudaSuccess ||
      (e = cudaMalloc(&pr->Y32, (size_t)kBatch * widths[nw - 1] * sizeof(float))) != cudaSuccess) {
    *err = std::string("allocation: ") + cudaGetErrorString(e);
    mlp_problem_destroy(pr);
    return nullptr;
  }
  {
    const int n32 = 2 * 64 * (p.kpad[0] / 8);
    mlp_uimg32_kernel<<<(n32 + 255) / 256, 256, 0, st>>>(seed, widths[0], p.kpad[0], pr->uimg32);
  }
  pr->p.uimg = pr->uimg;
  pr->p.Y = pr->Y;
  pr->p.x16 = nullptr;
  pr->p.uimg32[0] = pr->uimg32;
  pr->p.uimg32[1] = pr->uimg32 + img / sizeof(__half);
  pr->p.Y32 = pr->Y32;
  pr->p.part = nullptr;
  pr->p.cnt = nullptr;
  MlpParams q = pr->p;
  q.x = pr->theta;
  q.n = 1;
  q.f = nullptr;
  q.mode = 1;                                   // write Y* = g_L(θ*) (both kernels)
  if ((e = mlp_reserve(pr, 1, st)) != cudaSuccess || (e = launch_mlp(q, st)) != cudaSuccess ||
      (e = launch_split(pr->theta, p.D, pr->img, st)) != cudaSuccess ||
      (e = launch_mlp32(q, pr->img, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess) {
    *err = std::string("teacher forward: ") + cudaGetErrorString(e);
    mlp_problem_destroy(pr);
    return nullptr;
  }
  return pr;
}

// per-member buffers of the fp32-accurate kernel — the split image [2][n][D] and the two half
// sums + a counter — grown on demand (outside any stream capture: es_set_mlp_problem reserves a
// whole population)
static cudaError_t mlp_reserve(MlpProblem* pr, int64_t n, cudaStream_t st) {
  if (n <= pr->cap) return cudaSuccess;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  cudaFree(pr->part);
  cudaFree(pr->cnt);
  cudaFree(pr->img);
  pr->part = nullptr;
  pr->cnt = nullptr;
  pr->img = nullptr;
  pr->cap = 0;
  if ((e = cudaMalloc(&pr->part, (size_t)n * 2 * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&pr->cnt, (size_t)n * sizeof(uint32_t))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&pr->img, (size_t)n * 2 * pr->p.D * sizeof(__half))) != cudaSuccess) return e;
  if ((e = cudaMemset(pr->cnt, 0, (size_t)n * sizeof(uint32_t))) != cudaSuccess) return e;
  pr->cap = n;
  return cudaSuccess;
}

cudaError_t mlp_problem_reserve(void* prob, int64_t n, cudaStream_t st) {
  return mlp_reserve(static_cast<MlpProblem*>(prob), n, st);
}

// the split image buffer for n members (the fused ask writes it), or nullptr on failure
__half* mlp_problem_image(void* prob, int64_t n, cudaStream_t st) {
  MlpProblem* pr = static_cast<MlpProblem*>(prob);
  return mlp_reserve(pr, n, st) == cudaSuccess ? pr->img : nullptr;
}

void mlp_problem_destroy(void* prob) {
  MlpProblem* pr = static_cast<MlpProblem*>(prob);
  if (!pr) return;
  cudaFree(pr->uimg);
  cudaFree(pr->Y);
  cudaFree(pr->theta);
  cudaFree(pr->uimg32);
  cudaFree(pr->Y32);
  cudaFree(pr->part);
  cudaFree(pr->cnt);
  cudaFree(pr->img);
  delete pr;
}

int64_t mlp_problem_dims(const void* prob) {
  return prob ? static_cast<const MlpProblem*>(prob)->p.D : -1;
}

// N14 (the definition) on the split image the ask already wrote into mlp_problem_image(n).
cudaError_t launch_mlp_eval_img(void* prob, int64_t n, float* f, cudaStream_t st) {
  MlpProblem* pr = static_cast<MlpProblem*>(prob);
  if (n == 0) return cudaSuccess;
  if (n > pr->cap) return cudaErrorInvalidValue;
  MlpParams q = pr->p;
  q.x = nullptr;
  q.x16 = nullptr;
  q.n = n;
  q.f = f;
  q.mode = 0;
  q.part = pr->part;
  q.cnt = pr->cnt;
  return launch_mlp32(q, pr->img, st);
}

// N14 (the definition) on fp32 parameters: split pass, then the fp32-accurate kernel.
cudaError_t launch_mlp_eval(void* prob, const float* x, int64_t n, float* f, cudaStream_t st) {
  MlpProblem* pr = static_cast<MlpProblem*>(prob);
  if (n == 0) return cudaSuccess;
  if (cudaError_t e = mlp_reserve(pr, n, st)) return e;
  if (cudaError_t e = launch_split(x, n * pr->p.D, pr->img, st)) return e;
  return launch_mlp_eval_img(prob, n, f, st);
}

// N14′ (the fp16-image approximation) on fp32 parameters: the producers round to binary16.
cudaError_t launch_mlp_eval_f16(void* prob, const float* x, int64_t n, float* f, cudaStream_t st) {
  MlpProblem* pr = static_cast<MlpProblem*>(prob);
  if (reinterpret_cast<uintptr_t>(x) & 15) return cudaErrorMisalignedAddress;
  MlpParams q = pr->p;
  q.x = x;
  q.x16 = nullptr;
  q.n = n;
  q.f = f;
  q.mode = 0;
  return launch_mlp(q, st);
}

// N14′: fitness of the fp16 parameter image written by the ask kernel (TMA producer).
cudaError_t launch_mlp_eval16(void* prob, const __half* x16, int64_t n, float* f,
                              cudaStream_t st) {
  MlpProblem* pr = static_cast<MlpProblem*>(prob);
  if (reinterpret_cast<uintptr_t>(x16) & 15) return cudaErrorMisalignedAddress;
  MlpParams q = pr->p;
  q.x = nullptr;
  q.x16 = x16;
  q.n = n;
  q.f = f;
  q.mode = 0;
  cudaError_t e = encode_maps(q, x16, n);
  if (e != cudaSuccess) return e;
  return launch_mlp(q, st);
}

// es_get helpers for tests: teacher parameters and targets (device pointers).
const float* mlp_problem_theta(const void* prob) { return static_cast<const MlpProblem*>(prob)->theta; }
const float* mlp_problem_targets(const void* prob) { return static_cast<const MlpProblem*>(prob)->Y32; }
const float* mlp_problem_targets_f16(const void* prob) { return static_cast<const MlpProblem*>(prob)->Y; }

}  // namespace esb
