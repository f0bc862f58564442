// k_rank.cu — K5: per-run ranking and fitness shaping (NUMERICS N9–N11), best tracking and the
// per-generation scalars, one CTA per run.
//
// Keys: fp32 fitness → order-preserving u32 (NaN worst, ±0 equal) packed with the member index
// into a u64, bitonic-sorted in shared memory (N ≤ 16384 → ≤ 128 KB). Tie groups [s, e] come from
// two binary searches on the sorted high words. Shaping (P:213 centered rank; P:369 SNES
// utilities; P:286 Sep-CMA elite weights) and the tell's per-direction coefficients are written
// here so that the tell kernel only streams (direction, coefficient) pairs.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include <cooperative_groups.h>

#include "es_internal.h"

namespace esb {

__device__ __forceinline__ uint32_t rank_key(float f) {
  if (f != f) return 0xFFFFFFFFu;
  if (f == 0.0f) return 0x80000000u;
  const uint32_t b = __float_as_uint(f);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int k = 0; k < nw; ++k) t = __dadd_rn(t, red[k]);   // fixed order, every thread
  return t;
}

// The generation's scalars (one thread): best tracking, schedules, Adam bias
// corrections, the tell's entry count. jbest = member at sorted position 0, fb its fitness,
// nw = Sep-CMA-ES / CMA-ES weighted positions (end of μ−1's tie group + 1).
__device__ void write_genscal(const DevState& s, int r, int jbest, float fb, int nw, double bbar,
                              float ars_scale) {
  const int N = s.N;
  const bool anti = is_anti(s.algo);
  RunScal& w = s.rs[r];
  // every field is read before the first store: the stores may alias them, so a field read after
  // one would be another dependent global round trip on this single thread
  const uint32_t t = w.t;
  const float best_f = w.best_f, lr = w.lr, sigma = w.sigma;
  const int ars_k = w.ars_k;
  const double b1pow = w.b1pow, b2pow = w.b2pow;
  const float beta1 = w.beta1, beta2 = w.beta2, lrate_decay = w.lrate_decay,
              lrate_limit = w.lrate_limit, sigma_decay = w.sigma_decay, sigma_limit = w.sigma_limit;
  GenScal g;
  g.t = t;
  g.jbest = jbest;
  g.improved = fb < best_f;                   // strict; false for NaN
  g.lr = lr;
  g.sigma = sigma;
  g.nentries = (s.algo == ARS || s.algo == PGPE) ? ars_k
                                                 : (anti ? N / 2 : (s.algo == SNES ? N : nw));
  g.ars_scale = ars_scale;
  g.clip_inv = 0.0f;
  g.bbar = bbar;
  g.bc1 = g.bc2 = 1.0f;
  g.sigma_new = sigma;
  g.hsig = 0;
  if (g.improved) w.best_f = fb;
  if (anti) {
    const double b1 = __dmul_rn(b1pow, (double)beta1);
    const double b2 = __dmul_rn(b2pow, (double)beta2);
    g.bc1 = (float)__dsub_rn(1.0, b1);
    g.bc2 = (float)__dsub_rn(1.0, b2);
    w.b1pow = b1;
    w.b2pow = b2;
    w.lr = fmaxf(__fmul_rn(lr, lrate_decay), lrate_limit);
    if (s.algo == OPENAI_ES || s.algo == ARS)
      w.sigma = fmaxf(__fmul_rn(sigma, sigma_decay), sigma_limit);
  }
  w.t = t + 1;
  s.gs[r] = g;
}

// Sorted (key, index) pairs → tie groups, shaping, tell coefficients and the generation's
// scalars (N9–N12 bookkeeping). `keys` is the run's sorted array (shared or global memory).
// fit: the run's fitness in sorted-input order (shared memory when the caller staged it there —
// load_key also writes the global copy es_get reads).
// aux (optional, N ≤ kAuxMaxN): on-chip copies — [N] shaped, [N] tie ends, [N] perm, and the
// run's position weights prefetched by the caller — so the second half reads no global value
// this CTA has just written (each such read was a dependent L2 round trip).
static constexpr int kAuxMaxN = 4096;
struct RankAux {
  float* shaped;
  int32_t* E;
  int32_t* perm;
  const float* wpos;
};

__device__ void rank_finish(const DevState& s, int r, const uint64_t* keys, double* red,
                            int32_t* sh_nw_p, const float* fit, RankAux aux = RankAux{}) {
  const int N = s.N, T = blockDim.x;
  int32_t& sh_nw = *sh_nw_p;
  // tie groups and shaping
  const RunScal& rs = s.rs[r];
  int32_t* perm = s.perm + (int64_t)r * N;
  int32_t* S = s.rs_s + (int64_t)r * N;
  int32_t* E = s.rs_e + (int64_t)r * N;
  float* shaped = s.shaped + (int64_t)r * N;
  const float* wpos = aux.wpos ? aux.wpos : s.wpos + (int64_t)r * N;
  const bool on_chip = aux.shaped != nullptr;
  const float* shaped_r = on_chip ? aux.shaped : shaped;   // read side after the barrier
  const int32_t* E_r = on_chip ? aux.E : E;
  const int32_t* perm_r = on_chip ? aux.perm : perm;
  const bool anti = is_anti(s.algo);
  // z-score shaping: population mean and std of the fitness, binary64
  double zmu = 0.0, zsd = 1.0;
  const bool zscore = anti && s.algo != ARS && rs.shaping == 2;
  if (zscore) {
    double part = 0.0;
    for (int j = threadIdx.x; j < N; j += T) part = __dadd_rn(part, (double)fit[j]);
    zmu = block_sum(part, red) / (double)N;
    part = 0.0;
    for (int j = threadIdx.x; j < N; j += T) {
      const double d = __dsub_rn((double)fit[j], zmu);
      part = __dadd_rn(part, __dmul_rn(d, d));
    }
    zsd = __dadd_rn(sqrt(block_sum(part, red) / (double)N), 1e-8);
  }
  for (int p = threadIdx.x; p < N; p += T) {
    const uint64_t v = keys[p];
    const uint32_t key = (uint32_t)(v >> 32);
    const int j = (int)(uint32_t)v;
    int lo = 0, hi = p;                   // first position with key ≥ key
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((uint32_t)(keys[mid] >> 32) < key) lo = mid + 1; else hi = mid;
    }
    const int sj = lo;
    lo = p; hi = N;                       // first position with key > key
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((uint32_t)(keys[mid] >> 32) <= key) lo = mid + 1; else hi = mid;
    }
    const int ej = lo - 1;
    perm[p] = j;
    S[j] = sj;
    E[j] = ej;
    s.pos[(int64_t)r * N + j] = p;
    if (on_chip) {
      aux.perm[p] = j;
      aux.E[j] = ej;
    }
    float val;
    if (s.algo == ARS || (anti && rs.shaping == 1)) {
      val = fit[j];                                                      // raw fitness
    } else if (zscore) {
      val = (float)__ddiv_rn(__dsub_rn((double)fit[j], zmu), zsd);
    } else if (anti) {
      val = __fdiv_rn((float)(sj + ej - (N - 1)), (float)(2 * (N - 1)));  // N10
    } else {
      float acc = 0.0f;                                                                       // N11
      for (int q = sj; q <= ej; ++q) acc = __fadd_rn(acc, wpos[q]);
      val = __fdiv_rn(acc, (float)(ej - sj + 1));
    }
    shaped[j] = val;
    if (on_chip) aux.shaped[j] = val;
  }
  __syncthreads();
  // per-entry tell coefficients
  uint32_t* dir = s.dir + (int64_t)r * N;
  double* cA = s.coefA + (int64_t)r * N;
  double* cB = s.coefB + (int64_t)r * N;
  double bbar = 0.0;
  if (s.algo == PGPE) {
    double part = 0.0;
    for (int j = threadIdx.x; j < N; j += T) part = __dadd_rn(part, (double)shaped_r[j]);
    bbar = block_sum(part, red) / (double)N;
  }
  float ars_scale = 0.0f;
  // PGPE with elite pairs (k < N/2, reading Q13b) selects its entries with ARS's rule
  const bool elite_sel = s.algo == ARS || (s.algo == PGPE && rs.ars_k < N / 2);
  if (elite_sel) {
    // ARS: pairs ordered by (key(min(f+, f−)), pair index) = by the position of
    // their better member; pair i is "first seen" at p = min(pos(2i), pos(2i+1)). A block scan over
    // positions gives each first-seen pair its order; the first k are the elite directions.
    const int32_t* pos = s.pos + (int64_t)r * N;
    const int k = rs.ars_k;
    const int per = (N + T - 1) / T, p0 = threadIdx.x * per, p1 = min(N, p0 + per);
    int cnt = 0;
    for (int p = p0; p < p1; ++p) cnt += pos[perm_r[p] ^ 1] > p;
    // exclusive scan of cnt over the block (fixed order)
    int* scan = reinterpret_cast<int*>(red);          // ≤ 32 warps: warp totals
    int v = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) >= o) v += u;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 31) scan[threadIdx.x >> 5] = v;
    __syncthreads();
    int wbase = 0;
    for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) wbase += scan[w];
    int idx = wbase + v - cnt;
    double psum = 0.0;
    for (int p = p0; p < p1; ++p) {
      if (pos[perm_r[p] ^ 1] > p) {
        if (idx < k) {
          const int i = perm_r[p] >> 1;
          dir[idx] = (uint32_t)i;
          if (s.algo == ARS) {         // raw differences; σ_R below
            cA[idx] = __dsub_rn((double)fit[2 * i], (double)fit[2 * i + 1]);
            psum = __dadd_rn(psum, __dadd_rn((double)fit[2 * i], (double)fit[2 * i + 1]));
          } else {                     // PGPE: shaped coefficients, whole-population baseline
            const double cp = shaped_r[2 * i], cm = shaped_r[2 * i + 1];
            cA[idx] = __dsub_rn(cp, cm);
            cB[idx] = __dsub_rn(__dmul_rn(__dadd_rn(cp, cm), 0.5), bbar);
          }
        }
        ++idx;
      }
    }
    __syncthreads();
    if (s.algo == ARS) {               // block-uniform
      const double mu = block_sum(psum, red) / (2.0 * k);
      double pv = 0.0;
      for (int e = threadIdx.x; e < k; e += T) {
        const int i = (int)dir[e];
        const double a = __dsub_rn((double)fit[2 * i], mu), b = __dsub_rn((double)fit[2 * i + 1], mu);
        pv = __dadd_rn(pv, __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)));
      }
      const double sr = sqrt(block_sum(pv, red) / (2.0 * k));
      if (sr > 0.0) ars_scale = (float)((double)rs.lr / ((double)k * sr));
    }
  } else if (anti) {
    for (int i = threadIdx.x; i < N / 2; i += T) {
      const double cp = shaped_r[2 * i], cm = shaped_r[2 * i + 1];
      dir[i] = (uint32_t)i;
      cA[i] = __dsub_rn(cp, cm);
      if (s.algo == PGPE) cB[i] = __dsub_rn(__dmul_rn(__dadd_rn(cp, cm), 0.5), bbar);
    }
  } else if (s.algo == SNES) {
    for (int j = threadIdx.x; j < N; j += T) {
      dir[j] = (uint32_t)j;
      cA[j] = (double)shaped_r[j];
    }
  } else {
    if (threadIdx.x == 0) sh_nw = E_r[(uint32_t)keys[rs.mu - 1]] + 1;   // end of μ−1's tie group
    __syncthreads();
    for (int p = threadIdx.x; p < sh_nw; p += T) {
      const int j = perm_r[p];
      dir[p] = (uint32_t)j;
      cA[p] = (double)shaped_r[j];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int jbest = (int)(uint32_t)keys[0];            // = perm[0], without the global round trip
    write_genscal(s, r, jbest, fit[jbest], sh_nw, bbar, ars_scale);
  }
}

// fsrc layout [W][R][Nloc] (for W == 1 simply [R][N]).
__device__ __forceinline__ uint64_t load_key(const DevState& s, const float* __restrict__ fsrc,
                                             int r, int p, float* fs = nullptr) {
  if (p >= s.N) return ~0ull;
  const int w = p / s.Nloc, jl = p % s.Nloc;
  const float f = fsrc[((int64_t)w * s.R + r) * s.Nloc + jl];
  s.fit[(int64_t)r * s.N + p] = f;
  if (fs) fs[p] = f;
  return ((uint64_t)rank_key(f) << 32) | (uint32_t)p;
}

// The on-chip finish arrays after the keys and fitness (N ≤ kAuxMaxN; the launch sizes the shared
// memory accordingly), with the run's position weights prefetched while the keys load and sort.
__device__ __forceinline__ RankAux rank_aux(const DevState& s, int r, float* base, int npad) {
  if (npad > kAuxMaxN) return RankAux{};
  RankAux a;
  a.shaped = base;
  a.E = reinterpret_cast<int32_t*>(base + npad);
  a.perm = reinterpret_cast<int32_t*>(base + 2 * npad);
  float* w = base + 3 * npad;
  const float* wg = s.wpos + (int64_t)r * s.N;
  for (int p = threadIdx.x; p < s.N; p += blockDim.x) w[p] = wg[p];
  a.wpos = w;                                      // visible after the caller's barrier
  return a;
}

// In-shared-memory bitonic steps k ∈ [k0, k1], all j < k (indices global: direction (g & k)).
__device__ __forceinline__ void bitonic_smem(uint64_t* keys, int n, int64_t gbase, int k0,
                                             int k1, int jmax) {
  const int T = blockDim.x;
  for (int k = k0; k <= k1; k <<= 1) {
    for (int j = min(k >> 1, jmax); j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < (n >> 1); i += T) {
        const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
        const int hi = lo + j;
        const uint64_t a = keys[lo], b = keys[hi];
        const bool up = ((gbase + lo) & k) == 0;
        if ((a > b) == up) {
          keys[lo] = b;
          keys[hi] = a;
        }
      }
      __syncthreads();
    }
  }
}

// Whole-block bitonic sort of npad = E·T keys held in registers, blocked layout (thread t owns
// elements t·E .. t·E+E−1). Stride j < E: in-register compare-exchange; E ≤ j < 32E: partner in the
// same warp, exchanged with shuffles; j ≥ 32E: through shared memory (two barriers). Same network
// (and so the same result) as bitonic_smem, with a barrier only on the shared-memory strides.
template <int E, int J>
__device__ __forceinline__ void reg_stage(uint64_t (&a)[E], int t, int k) {
  if constexpr (J < E) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e & J) continue;                           // static: e, J are compile-time here
      const int e2 = e | J;
      const bool asc = (((t * E + e) & k) == 0);
      const uint64_t x = a[e], y = a[e2];
      if ((x > y) == asc) { a[e] = y; a[e2] = x; }
    }
  }
}

template <int E>
__device__ __forceinline__ void bitonic_regs(uint64_t* keys, int npad) {
  const int t = threadIdx.x;
  uint64_t a[E];
#pragma unroll
  for (int e = 0; e < E; ++e) a[e] = keys[t * E + e];
  for (int k = 2; k <= npad; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j < E) {
        if (j == 1) reg_stage<E, 1>(a, t, k);
        else if (j == 2) reg_stage<E, 2>(a, t, k);
        else if (j == 4) reg_stage<E, 4>(a, t, k);
        else reg_stage<E, 8>(a, t, k);
      } else if (j < 32 * E) {
        // j, k ≥ E: direction and half depend on the thread only (g = t·E + e, e < E ≤ j)
        const int lm = j / E;                          // partner lane mask
        const bool keep_min = (((t * E) & j) == 0) == (((t * E) & k) == 0);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t o = __shfl_xor_sync(0xffffffffu, a[e], lm);
          a[e] = keep_min ? (a[e] < o ? a[e] : o) : (a[e] > o ? a[e] : o);
        }
      } else {
        const bool keep_min = (((t * E) & j) == 0) == (((t * E) & k) == 0);
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) keys[t * E + e] = a[e];
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint64_t o = keys[(t * E + e) ^ j];
          a[e] = keep_min ? (a[e] < o ? a[e] : o) : (a[e] > o ? a[e] : o);
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) keys[t * E + e] = a[e];
  __syncthreads();
}

// 8192 < N ≤ 16384: one CTA per run, the classic shared-memory network (16 keys per thread would
// not fit the register file at 1024 threads).
__global__ void rank_kernel_smem(DevState s, const float* __restrict__ fsrc, int npad) {
  extern __shared__ uint64_t keys[];              // [npad] keys, then [npad] fitness values
  __shared__ double red[32];
  __shared__ int32_t sh_nw;
  pdl_enter();
  const int r = blockIdx.x;
  float* fs = reinterpret_cast<float*>(keys + npad);
  const RankAux aux = rank_aux(s, r, fs + npad, npad);
  for (int p = threadIdx.x; p < npad; p += blockDim.x) keys[p] = load_key(s, fsrc, r, p, fs);
  __syncthreads();
  bitonic_smem(keys, npad, 0, 2, npad, npad);
  rank_finish(s, r, keys, red, &sh_nw, fs, aux);
}

// N ≤ 8192: one CTA per run, the sort in registers (+ shared memory for the long strides).
template <int E>
__global__ void rank_kernel(DevState s, const float* __restrict__ fsrc, int npad) {
  extern __shared__ uint64_t keys[];
  __shared__ double red[32];
  __shared__ int32_t sh_nw;
  pdl_enter();
  const int r = blockIdx.x;
  float* fs = reinterpret_cast<float*>(keys + npad);   // the fitness, kept on chip for the finish
  const RankAux aux = rank_aux(s, r, fs + npad, npad);
  for (int p = threadIdx.x; p < npad; p += blockDim.x) keys[p] = load_key(s, fsrc, r, p, fs);
  __syncthreads();
  bitonic_regs<E>(keys, npad);
  rank_finish(s, r, keys, red, &sh_nw, fs, aux);
}

// N > 16384: hybrid bitonic sort over global memory. Chunks of kChunk keys are sorted and merged
// in shared memory; only the strides j ≥ kChunk go through global memory, one launch each.
static constexpr int kChunk = 16384;

__global__ void rank_chunk_sort_kernel(DevState s, const float* __restrict__ fsrc,
                                       uint64_t* __restrict__ gkeys, int npad) {
  extern __shared__ uint64_t keys[];
  const int nch = npad / kChunk;
  const int r = blockIdx.x / nch, c = blockIdx.x % nch;
  const int64_t g0 = (int64_t)c * kChunk;
  for (int p = threadIdx.x; p < kChunk; p += blockDim.x)
    keys[p] = load_key(s, fsrc, r, (int)(g0 + p));
  __syncthreads();
  bitonic_smem(keys, kChunk, g0, 2, kChunk, kChunk);
  uint64_t* out = gkeys + (int64_t)r * npad + g0;
  for (int p = threadIdx.x; p < kChunk; p += blockDim.x) out[p] = keys[p];
}

__global__ void rank_global_step_kernel(uint64_t* __restrict__ gkeys, int npad, int k, int j,
                                        int R) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t half = npad >> 1;
  if (i >= (int64_t)R * half) return;
  const int r = (int)(i / half);
  const int ii = (int)(i % half);
  const int lo = ((ii & ~(j - 1)) << 1) | (ii & (j - 1));
  uint64_t* kr = gkeys + (int64_t)r * npad;
  const uint64_t a = kr[lo], b = kr[lo + j];
  const bool up = (lo & k) == 0;
  if ((a > b) == up) {
    kr[lo] = b;
    kr[lo + j] = a;
  }
}

__global__ void rank_chunk_merge_kernel(uint64_t* __restrict__ gkeys, int npad, int k) {
  extern __shared__ uint64_t keys[];
  const int nch = npad / kChunk;
  const int r = blockIdx.x / nch, c = blockIdx.x % nch;
  const int64_t g0 = (int64_t)c * kChunk;
  uint64_t* io = gkeys + (int64_t)r * npad + g0;
  for (int p = threadIdx.x; p < kChunk; p += blockDim.x) keys[p] = io[p];
  __syncthreads();
  bitonic_smem(keys, kChunk, g0, k, k, kChunk >> 1);
  for (int p = threadIdx.x; p < kChunk; p += blockDim.x) io[p] = keys[p];
}

__global__ void rank_finish_kernel(DevState s, const uint64_t* __restrict__ gkeys, int npad) {
  __shared__ double red[32];
  __shared__ int32_t sh_nw;
  rank_finish(s, blockIdx.x, gkeys + (int64_t)blockIdx.x * npad, red, &sh_nw,
              s.fit + (int64_t)blockIdx.x * s.N);
}

// Few runs (R ≤ kCountMaxR), N ≤ kCountMaxN, and a shaping that is a per-member function of the
// ranks (centered rank, raw, SNES / Sep-CMA weights — s.rank_par): rank by COUNTING, in ONE launch
// spread over the whole GPU (the single-CTA sort is latency-bound at R = 1). For member j with key
// k_j (N9):  lt_j = #{i : k_i < k_j},  le_j = #{i : k_i ≤ k_j},  pos_j = #{i : (k_i, i) < (k_j, j)}
// — the tie group is [s_j, e_j] = [lt_j, le_j − 1] and pos_j the (key, index) sort position, so
// no sorted array is needed. Grid: j-tiles × i-ranges × runs; each CTA adds its i-range's counts
// with integer atomics (order-free, deterministic). The last CTA of a j-tile (arrival counter)
// finishes its 256 members: tie group, shaped value (N10 / N11 / raw), perm, the tell's
// (direction, coefficient) entries; the last j-tile of a run writes the generation's scalars
// (and subtracts PGPE's baseline, N12). Counters are cleared for the next generation on the way.
// N ≤ 256 at any run count: one CTA per run holds the whole run (no atomics, no arrivals).
static constexpr int kCountMaxR = 16, kCountMaxN = 16384, kCountT = 256;
static constexpr int kCountMaxTiles = kCountMaxN / kCountT;

// rcnt layout: [3][R][N] counters (pos, lt, le), then [R][kCountMaxTiles] j-tile arrivals, [R]
// run arrivals, [R][2] slots (jbest, nw).
__device__ __forceinline__ uint32_t* rc_tile(const DevState& s) { return s.rcnt + 3 * (int64_t)s.R * s.N; }
__device__ __forceinline__ uint32_t* rc_run(const DevState& s) { return rc_tile(s) + (int64_t)s.R * kCountMaxTiles; }
__device__ __forceinline__ uint32_t* rc_slot(const DevState& s) { return rc_run(s) + s.R; }

__device__ __forceinline__ float fit_at(const DevState& s, const float* __restrict__ fsrc, int r,
                                        int p) {
  const int w = p / s.Nloc, jl = p % s.Nloc;
  return fsrc[((int64_t)w * s.R + r) * s.Nloc + jl];
}

__global__ void __launch_bounds__(kCountT) rank_count_kernel(DevState s,
                                                             const float* __restrict__ fsrc,
                                                             int ilen) {
  __shared__ uint32_t tile[kCountT];
  __shared__ float sval[kCountT];
  __shared__ double red[32];
  __shared__ int sh_last;
#ifdef ES_RANK_TRACE
  long long rtr[12];
  int nrt = 0;
#define RKT() do { if (nrt < 12) rtr[nrt++] = clock64(); } while (0)
#else
#define RKT() do { } while (0)
#endif
  RKT();
  pdl_enter();
  RKT();
  const int N = s.N, r = blockIdx.z, jt = gridDim.x, ni = gridDim.y;
  // the run's hyperparameters, loaded before any store (a load after a store to another array
  // cannot be hoisted above it: one more dependent round trip each)
  const int rs_shaping = s.rs[r].shaping, rs_mu = s.rs[r].mu;
  const int j = blockIdx.x * kCountT + threadIdx.x;
  const float fj = j < N ? fit_at(s, fsrc, r, j) : 0.0f;
  const uint32_t kj = j < N ? rank_key(fj) : 0xFFFFFFFFu;
  RKT();
  const int i0 = blockIdx.y * ilen, i1 = min(N, i0 + ilen);
  const int jt0 = blockIdx.x * kCountT;
  uint32_t cpos = 0, clt = 0, cle = 0;
  const bool solo = jt == 1 && ni == 1;
  for (int b = i0; b < i1; b += kCountT) {
    const int n = min(kCountT, i1 - b);
    __syncthreads();
    // one CTA for the run: the tile is its own keys (no second load of the fitness)
    if (threadIdx.x < n) tile[threadIdx.x] = solo ? kj : rank_key(fit_at(s, fsrc, r, b + threadIdx.x));
    __syncthreads();
    uint32_t lt = 0, le = 0;
    if (n == kCountT) {
      // 16-byte broadcast reads, 8 in flight (a scalar read per key was ≈ 22 cycles per key)
      const uint4* t4 = reinterpret_cast<const uint4*>(tile);
#pragma unroll 8
      for (int e = 0; e < kCountT / 4; ++e) {
        const uint4 k4 = t4[e];
        lt += (k4.x < kj) + (k4.y < kj) + (k4.z < kj) + (k4.w < kj);
        le += (k4.x <= kj) + (k4.y <= kj) + (k4.z <= kj) + (k4.w <= kj);
      }
    } else {
      for (int e = 0; e < n; ++e) {
        const uint32_t k = tile[e];
        lt += k < kj;
        le += k <= kj;
      }
    }
    clt += lt;
    cle += le;
    if (b + n <= jt0) {
      cpos += le;                           // every i of the tile precedes every j of this j-tile
    } else if (b >= jt0 + kCountT) {
      cpos += lt;                           // every i follows
    } else {                                // the j-tile itself: (key, index) order, i.e. lt
      cpos += lt;                           // + the equal keys of smaller index (ties only)
      if (le - lt > 1u) {
        const int ne = min(j - b, n);
        for (int e = 0; e < ne; ++e) cpos += tile[e] == kj;
      }
    }
  }
  RKT();
  const int64_t RN = (int64_t)s.R * N, rj = (int64_t)r * N + j;
  // one CTA covers the whole run (N ≤ 256): the counts are final in registers — no atomics,
  // arrival counters or fences (the multi-CTA path's four global round trips are its latency)
  if (!solo) {
    if (j < N) {
      if (cpos) atomicAdd(&s.rcnt[rj], cpos);
      if (clt) atomicAdd(&s.rcnt[RN + rj], clt);
      if (cle) atomicAdd(&s.rcnt[2 * RN + rj], cle);
    }
    // ---- the last i-range CTA of this j-tile finishes its members
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t* tc = rc_tile(s) + (int64_t)r * kCountMaxTiles + blockIdx.x;
      sh_last = atomicAdd(tc, 1u) == (uint32_t)(ni - 1);
      if (sh_last) *tc = 0u;
    }
    __syncthreads();
    if (!sh_last) return;
    __threadfence();
  }
  const bool anti = is_anti(s.algo), cmaish = s.algo == SEP_CMA_ES || s.algo == CMA_ES;
  float val = 0.0f;
  int pos = 0;
  __shared__ int sh_jbest, sh_nw;
  __shared__ float sh_fbest;
  if (j < N) {
    int sj, ej;
    if (solo) {
      pos = (int)cpos;
      sj = (int)clt;
      ej = (int)cle - 1;
    } else {
      pos = (int)__ldcg(&s.rcnt[rj]);
      sj = (int)__ldcg(&s.rcnt[RN + rj]);
      ej = (int)__ldcg(&s.rcnt[2 * RN + rj]) - 1;
      s.rcnt[rj] = 0u;
      s.rcnt[RN + rj] = 0u;
      s.rcnt[2 * RN + rj] = 0u;
    }
    // the shaped value first: its weight loads then precede this thread's stores
    if (anti && rs_shaping == 1) {
      val = fj;                                                          // raw fitness
    } else if (anti) {
      val = __fdiv_rn((float)(sj + ej - (N - 1)), (float)(2 * (N - 1)));  // N10
    } else {
      const float* wpos = s.wpos + (int64_t)r * N;                        // N11
      float acc = 0.0f;
      for (int q = sj; q <= ej; ++q) acc = __fadd_rn(acc, wpos[q]);
      val = __fdiv_rn(acc, (float)(ej - sj + 1));
    }
    s.perm[(int64_t)r * N + pos] = j;
    s.rs_s[rj] = sj;
    s.rs_e[rj] = ej;
    s.pos[rj] = pos;
    s.fit[rj] = fj;
    s.shaped[rj] = val;
    if (solo) {
      if (pos == 0) {
        sh_jbest = j;
        sh_fbest = fj;
      }
      if (cmaish && pos == rs_mu - 1) sh_nw = ej + 1;
    } else {
      if (pos == 0) rc_slot(s)[2 * r] = (uint32_t)j;
      if (cmaish && pos == rs_mu - 1) rc_slot(s)[2 * r + 1] = (uint32_t)(ej + 1);
    }
  }
  RKT();
  sval[threadIdx.x] = val;
  __syncthreads();
  RKT();
  uint32_t* dir = s.dir + (int64_t)r * N;
  double* cA = s.coefA + (int64_t)r * N;
  double* cB = s.coefB + (int64_t)r * N;
  double part = 0.0;
  double cb_pre = 0.0;                      // PGPE (cp + cm)/2 of this thread's pair
  if (anti) {
    if (j < N && !(j & 1)) {               // pair i = j/2 (N even; the partner is in this tile)
      const int i = j >> 1;
      const double cp = sval[threadIdx.x], cm = sval[threadIdx.x + 1];
      dir[i] = (uint32_t)i;
      cA[i] = __dsub_rn(cp, cm);
      if (s.algo == PGPE) {
        cb_pre = __dmul_rn(__dadd_rn(cp, cm), 0.5);
        if (!solo) cB[i] = cb_pre;         // − b̄ by the last tile
      }
    }
    if (s.algo == PGPE) part = j < N ? (double)val : 0.0;
  } else if (j < N) {
    const int e = cmaish ? pos : j;         // Sep-CMA: entries in sorted order (the first nw count)
    dir[e] = (uint32_t)j;
    cA[e] = (double)val;
  }
  if (s.algo == PGPE) {
    const double t = block_sum(part, red);
    if (solo) {                               // the baseline and the generation's scalars here
      const double bbar = t / (double)N;
      // the pair's thread still holds (cp + cm)/2: one store, no read back of cB
      if (j < N && !(j & 1)) cB[j >> 1] = __dsub_rn(cb_pre, bbar);
      RKT();
      if (threadIdx.x == 0) write_genscal(s, r, sh_jbest, sh_fbest, 0, bbar, 0.0f);
#ifdef ES_RANK_TRACE
      RKT();
      if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
        printf("rank trace pgpe:");
        for (int i = 1; i < nrt; ++i) printf(" %lld", rtr[i] - rtr[i - 1]);
        printf("\n");
      }
#endif
      return;
    }
    if (threadIdx.x == 0) s.rbpart[(int64_t)r * kCountMaxTiles + blockIdx.x] = t;
  }
  if (solo) {
    __syncthreads();
    RKT();
    if (threadIdx.x == 0)
      write_genscal(s, r, sh_jbest, sh_fbest, cmaish ? sh_nw : 0, 0.0, 0.0f);
#ifdef ES_RANK_TRACE
    RKT();
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
      printf("rank trace:");
      for (int i = 1; i < nrt; ++i) printf(" %lld", rtr[i] - rtr[i - 1]);
      printf("\n");
    }
#endif
    return;
  }
  // ---- the last j-tile of the run: the generation's scalars
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t* rc = rc_run(s) + r;
    sh_last = atomicAdd(rc, 1u) == (uint32_t)(jt - 1);
    if (sh_last) *rc = 0u;
  }
  __syncthreads();
  if (!sh_last) return;
  __threadfence();
  double bbar = 0.0;
  if (s.algo == PGPE) {
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int b = 0; b < jt; ++b) t = __dadd_rn(t, __ldcg(&s.rbpart[(int64_t)r * kCountMaxTiles + b]));
      red[0] = t / (double)N;
    }
    __syncthreads();
    bbar = red[0];
    for (int i = threadIdx.x; i < N / 2; i += blockDim.x) cB[i] = __dsub_rn(__ldcg(&cB[i]), bbar);
  }
  if (threadIdx.x == 0) {
    const int jbest = (int)__ldcg(&rc_slot(s)[2 * r]);
    const int nw = cmaish ? (int)__ldcg(&rc_slot(s)[2 * r + 1]) : 0;
    write_genscal(s, r, jbest, __ldcg(&s.fit[(int64_t)r * N + jbest]), nw, bbar, 0.0f);
  }
}

// (For many runs the per-run register bitonic sort stays faster: counting at R = 512, N = 256
// measured 22.8 vs 15 µs per launch.)

// Few runs (R ≤ kCountMaxR) with 4096 < N ≤ 65536 and per-member shaping: an LSD radix RANK in
// ONE cooperative launch. A tile of 2048 keys per CTA (256 threads × 8, striped so that position
// = tile·2048 + slot·256 + thread); four 8-bit passes of a stable counting sort of the (key,
// index) pairs — warp-level __match_any_sync ranks, a (slot, warp) prefix per digit in shared
// memory, per-tile digit totals in global memory, every CTA deriving its own digit offsets after a
// grid sync (no separate scan phase) — then the finish over the sorted keys spread over all CTAs
// (tie groups by neighbour checks, binary search only inside a tie run). Sorting by (key, index)
// through a stable LSD sort gives exactly N9's order. Nine grid syncs replace the counting path's
// N² compares (88 µs at N = 16384) and the hybrid sort's single-CTA finish (0.52 ms at 65536).
static constexpr int kRadT = 256, kRadE = 8, kRadTile = kRadT * kRadE, kRadMaxBlk = 32;
static constexpr int kRadMinN = 4097, kRadMaxN = kRadTile * kRadMaxBlk;

__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += u;
  }
  __syncthreads();
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  uint32_t base = 0;
  for (int k = 0; k < w; ++k) base += wsum[k];
  return base + x - v;
}

// Grid barrier for the cooperative launch (all CTAs co-resident): a monotone arrival counter,
// spun on without back-off (the cooperative-groups grid sync measured ~4 µs per barrier here).
// `ctr[0]` counts arrivals, `ctr[1]` departures; the last CTA to leave the kernel resets both.
__device__ __forceinline__ unsigned __smid_dummy() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
struct GridBar {
  unsigned* ctr;
  unsigned n, k = 0;
  __device__ void sync() {
    __syncthreads();
    if (threadIdx.x == 0) {
      ++k;
      __threadfence();                           // cumulative: the CTA's writes, ordered by the barrier
      atomicAdd(&ctr[0], 1u);
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      } while (v < k * n);
    }
    __syncthreads();
  }
  __device__ void leave() {
    if (threadIdx.x == 0 && atomicAdd(&ctr[1], 1u) == n - 1) {
      ctr[0] = 0u;                               // every CTA has passed every barrier
      ctr[1] = 0u;
    }
  }
};

__global__ void __launch_bounds__(kRadT, 4) rank_radix_kernel(DevState s, const float* __restrict__ fsrc,
                                                           int nblk) {
  GridBar grid{s.rrad_bar, gridDim.x * gridDim.y};
#ifdef ES_RADIX_TRACE
  long long tr[16];
  int ntr = 0;
  tr[ntr++] = clock64();
#define RTR() do { if (ntr < 16) tr[ntr++] = clock64(); } while (0)
#else
#define RTR() do { } while (0)
#endif
  __shared__ uint16_t cnt[kRadE][kRadT / 32][256];
  __shared__ uint32_t off[256];
  __shared__ uint32_t wsum[kRadT / 32];
  __shared__ double red[32];
  const int N = s.N, R = s.R, r = blockIdx.y, b = blockIdx.x, t = threadIdx.x;
  const int w = t >> 5, lane = t & 31;
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t* const base = s.rrad;
  uint32_t* const K0 = base + (size_t)r * N;
  uint32_t* const K1 = base + (size_t)(2 * R + r) * N;
  uint32_t* const I0 = base + (size_t)(R + r) * N;
  uint32_t* const I1 = base + (size_t)(3 * R + r) * N;
  uint32_t* hist = base + (size_t)4 * R * N + (size_t)r * 256 * kRadMaxBlk;   // [digit][tile]
  uint32_t k[kRadE], id[kRadE];
  bool v[kRadE];
#pragma unroll
  for (int e = 0; e < kRadE; ++e) {
    const int i = b * kRadTile + e * kRadT + t;
    v[e] = i < N;
    k[e] = v[e] ? rank_key(fit_at(s, fsrc, r, i)) : 0u;
    id[e] = (uint32_t)i;
  }
  for (int pass = 0; pass < 4; ++pass) {
    const int sh = 8 * pass;
    uint32_t* cz = reinterpret_cast<uint32_t*>(&cnt[0][0][0]);
    for (int i = t; i < kRadE * (kRadT / 32) * 256 / 2; i += kRadT) cz[i] = 0u;
    __syncthreads();
    uint32_t rk[kRadE];
#pragma unroll
    for (int e = 0; e < kRadE; ++e) {
      const uint32_t act = __ballot_sync(0xffffffffu, v[e]);
      rk[e] = 0u;
      if (v[e]) {
        const uint32_t d = (k[e] >> sh) & 255u;
        const uint32_t peers = __match_any_sync(act, d);
        rk[e] = __popc(peers & lt_mask);
        if (rk[e] == 0u) cnt[e][w][d] = (uint16_t)__popc(peers);
      }
    }
    __syncthreads();
    uint32_t run = 0;                             // thread t = digit: prefix over (slot, warp)
    {
      uint16_t c[kRadE * (kRadT / 32)];           // all 64 loads in flight, then the prefix
#pragma unroll
      for (int k2 = 0; k2 < kRadE * (kRadT / 32); ++k2) c[k2] = cnt[k2 / (kRadT / 32)][k2 % (kRadT / 32)][t];
#pragma unroll
      for (int k2 = 0; k2 < kRadE * (kRadT / 32); ++k2) {
        cnt[k2 / (kRadT / 32)][k2 % (kRadT / 32)][t] = (uint16_t)run;
        run += c[k2];
      }
    }
    hist[t * kRadMaxBlk + b] = run;
    RTR();
    grid.sync();
    RTR();
    uint32_t T = 0, Pb = 0;
    {
      uint32_t h[kRadMaxBlk];                     // all tile totals in flight at once
#pragma unroll
      for (int bb = 0; bb < kRadMaxBlk; ++bb) h[bb] = bb < nblk ? __ldcg(&hist[t * kRadMaxBlk + bb]) : 0u;
#pragma unroll
      for (int bb = 0; bb < kRadMaxBlk; ++bb) {
        T += h[bb];
        if (bb < b) Pb += h[bb];
      }
    }
    off[t] = block_excl_scan256(T, wsum) + Pb;
    __syncthreads();
    uint32_t* Ko = (pass & 1) ? K1 : K0;
    uint32_t* Io = (pass & 1) ? I1 : I0;
#pragma unroll
    for (int e = 0; e < kRadE; ++e) {
      if (!v[e]) continue;
      const uint32_t d = (k[e] >> sh) & 255u;
      const uint32_t dst = off[d] + cnt[e][w][d] + rk[e];
      Ko[dst] = k[e];
      Io[dst] = id[e];
    }
    grid.sync();
#pragma unroll
    for (int e = 0; e < kRadE; ++e) {
      const int i = b * kRadTile + e * kRadT + t;
      if (v[e]) {
        k[e] = __ldcg(&Ko[i]);
        id[e] = __ldcg(&Io[i]);
      }
    }
  }
  RTR();
  // ---- finish: positions of this tile in the sorted order (pass 3 wrote buffer 1)
  const uint32_t* SK = K1;
  const RunScal& rs = s.rs[r];
  const bool anti = is_anti(s.algo), cmaish = s.algo == SEP_CMA_ES || s.algo == CMA_ES;
  uint32_t* dir = s.dir + (int64_t)r * N;
  double* cA = s.coefA + (int64_t)r * N;
  double* cB = s.coefB + (int64_t)r * N;
  double part = 0.0;
  // the tile's sorted keys in shared memory (the digit counters are free now): neighbour checks and
  // tie-run searches stay on chip unless a tie run crosses the tile edge; the fitness values of
  // the tile's members are fetched up front (independent loads)
  uint32_t* skt = reinterpret_cast<uint32_t*>(&cnt[0][0][0]);
  const int tlen = min(kRadTile, N - b * kRadTile);
  __syncthreads();
#pragma unroll
  for (int e = 0; e < kRadE; ++e) skt[e * kRadT + t] = k[e];
  float fv[kRadE];
#pragma unroll
  for (int e = 0; e < kRadE; ++e) fv[e] = v[e] ? fit_at(s, fsrc, r, (int)id[e]) : 0.0f;
  __syncthreads();
#pragma unroll
  for (int e = 0; e < kRadE; ++e) {
    if (!v[e]) continue;
    const int pl = e * kRadT + t, p = b * kRadTile + pl;
    const uint32_t key = k[e];
    const int j = (int)id[e];
    int sj = p, ej = p;
    const uint32_t kprev = pl > 0 ? skt[pl - 1] : (p > 0 ? __ldcg(&SK[p - 1]) : ~key);
    if (kprev == key) {                           // inside a tie run: its first position
      int lo, hi;
      if (skt[0] != key) { lo = 0; hi = pl; } else { lo = -b * kRadTile; hi = 0; }
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const uint32_t km = mid >= 0 ? skt[mid] : __ldcg(&SK[b * kRadTile + mid]);
        if (km < key) lo = mid + 1; else hi = mid;
      }
      sj = b * kRadTile + lo;
    }
    const uint32_t knext = pl + 1 < tlen ? skt[pl + 1] : (p + 1 < N ? __ldcg(&SK[p + 1]) : ~key);
    if (knext == key) {                           // its last position
      int lo, hi;
      if (skt[tlen - 1] != key) { lo = pl; hi = tlen; } else { lo = tlen - 1; hi = N - b * kRadTile; }
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const uint32_t km = mid < tlen ? skt[mid] : __ldcg(&SK[b * kRadTile + mid]);
        if (km <= key) lo = mid + 1; else hi = mid;
      }
      ej = b * kRadTile + lo - 1;
    }
    const int64_t rj = (int64_t)r * N + j;
    const float fj = fv[e];
    s.perm[(int64_t)r * N + p] = j;
    s.rs_s[rj] = sj;
    s.rs_e[rj] = ej;
    s.pos[rj] = p;
    s.fit[rj] = fj;
    float val;
    if (anti && rs.shaping == 1) {
      val = fj;
    } else if (anti) {
      val = __fdiv_rn((float)(sj + ej - (N - 1)), (float)(2 * (N - 1)));   // N10
    } else {
      const float* wpos = s.wpos + (int64_t)r * N;                         // N11
      float acc = 0.0f;
      for (int q = sj; q <= ej; ++q) acc = __fadd_rn(acc, wpos[q]);
      val = __fdiv_rn(acc, (float)(ej - sj + 1));
    }
    s.shaped[rj] = val;
    if (cmaish) { dir[p] = (uint32_t)j; cA[p] = (double)val; }
    else if (!anti) { dir[j] = (uint32_t)j; cA[j] = (double)val; }
    if (p == 0) rc_slot(s)[2 * r] = (uint32_t)j;
    if (cmaish && p == rs.mu - 1) rc_slot(s)[2 * r + 1] = (uint32_t)(ej + 1);
    part += (double)val;
  }
  RTR();
  if (s.algo == PGPE) {
    const double tsum = block_sum(part, red);
    if (t == 0) s.rbpart[(int64_t)r * kCountMaxTiles + b] = tsum;
  }
  grid.sync();
  RTR();
  double bbar = 0.0;
  if (s.algo == PGPE) {                           // every CTA sums the tile partials in order
    double pb[kRadMaxBlk];
#pragma unroll
    for (int bb = 0; bb < kRadMaxBlk; ++bb)
      pb[bb] = bb < nblk ? __ldcg(&s.rbpart[(int64_t)r * kCountMaxTiles + bb]) : 0.0;
    double tsum = 0.0;
#pragma unroll
    for (int bb = 0; bb < kRadMaxBlk; ++bb) tsum = __dadd_rn(tsum, pb[bb]);
    bbar = tsum / (double)N;
  }
  if (anti) {                                     // pair coefficients, 1024 pairs per tile
    const float* sh = s.shaped + (int64_t)r * N;
    for (int i = b * (kRadTile / 2) + t; i < min(N / 2, (b + 1) * (kRadTile / 2)); i += kRadT) {
      const double cp = __ldcg(&sh[2 * i]), cm = __ldcg(&sh[2 * i + 1]);
      dir[i] = (uint32_t)i;
      cA[i] = __dsub_rn(cp, cm);
      if (s.algo == PGPE) cB[i] = __dsub_rn(__dmul_rn(__dadd_rn(cp, cm), 0.5), bbar);
    }
  }
  if (b == 0 && t == 0) {
    const int jbest = (int)__ldcg(&rc_slot(s)[2 * r]);
    const int nw = cmaish ? (int)__ldcg(&rc_slot(s)[2 * r + 1]) : 0;
    write_genscal(s, r, jbest, __ldcg(&s.fit[(int64_t)r * N + jbest]), nw, bbar, 0.0f);
  }
  grid.leave();
#ifdef ES_RADIX_TRACE
  RTR();
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    printf("radix trace:");
    for (int i = 1; i < ntr; ++i) printf(" %lld", tr[i] - tr[i - 1]);
    printf("\n");
  }
  if (threadIdx.x == 0 && ntr >= 12)
    printf("radix cta %d finish %lld smid %u\n", blockIdx.x, tr[10] - tr[9], __smid_dummy());
#endif
}

static int radix_min_n() {                      // A/B switch for profiling (ES_RADIX_MIN_N)
  static const int v = [] {
    const char* e = std::getenv("ES_RADIX_MIN_N");
    return e ? std::max(2, std::atoi(e)) : kRadMinN;
  }();
  return v;
}
// the cooperative grid (tiles × runs) must be co-resident
static int radix_max_ctas() {
  static std::atomic<int> v{0};
  int m = v.load();
  if (m == 0) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rank_radix_kernel, kRadT, 0);
    m = std::max(1, occ) * sm_count();
    v.store(m);
  }
  return m;
}
static bool use_radix(const DevState& s) {
  return s.rank_par && s.rrad && s.R <= kCountMaxR && s.N >= radix_min_n() && s.N <= kRadMaxN &&
         s.R * ((s.N + kRadTile - 1) / kRadTile) <= radix_max_ctas();
}

static bool use_count(const DevState& s) {
  // N ≤ 256: one counting CTA per run (no cross-CTA traffic) for any number of runs (A/B switch
  // ES_COUNT_MANY=0 keeps the per-run bitonic sort for R > 16)
  static const bool many = [] {
    const char* e = std::getenv("ES_COUNT_MANY");
    return !(e && e[0] == '0');
  }();
  if (s.rank_par && many && s.N <= kCountT && s.R <= 65535) return true;
  return s.rank_par && s.R <= kCountMaxR && s.N <= kCountMaxN && !use_radix(s);
}

cudaError_t launch_rank(const DevState& s, const float* fsrc, cudaStream_t st) {
  if (use_radix(s)) {
    int nblk = (s.N + kRadTile - 1) / kRadTile;
    dim3 grid((unsigned)nblk, (unsigned)s.R);
    DevState sc = s;
    const float* fs = fsrc;
    void* args[] = {(void*)&sc, (void*)&fs, (void*)&nblk};
    return cudaLaunchCooperativeKernel((const void*)rank_radix_kernel, grid, dim3(kRadT), args, 0, st);
  }
  if (use_count(s)) {
    const int jt = (s.N + kCountT - 1) / kCountT;
    const int want = 2 * sm_count();
    int ni = std::max(1, std::min(jt, want / std::max(1, s.R * jt)));
    const int ilen = ((s.N + ni - 1) / ni + kCountT - 1) / kCountT * kCountT;
    ni = (s.N + ilen - 1) / ilen;
    return launch_pdl(rank_count_kernel, dim3((unsigned)jt, (unsigned)ni, (unsigned)s.R),
                      dim3(kCountT), 0, st, s, fsrc, ilen);
  }
  int npad = 1;
  while (npad < s.N) npad <<= 1;
  static std::atomic<uint64_t> attr[6];
  {
    const void* fs[6] = {(const void*)rank_kernel<2>, (const void*)rank_kernel<4>,
                         (const void*)rank_kernel<8>, (const void*)rank_kernel_smem,
                         (const void*)rank_chunk_sort_kernel, (const void*)rank_chunk_merge_kernel};
    for (int i = 0; i < 6; ++i)
      if (cudaError_t e = smem_attr_once(fs[i], 200 * 1024, attr[i])) return e;
  }
  if (npad <= kChunk) {
    // E keys per thread: 2 while the block grows to 1024 threads, then 4, 8, 16 (npad ≥ 64)
    const int pad = std::max(npad, 64);
    const int T = std::min(1024, pad / 2);
    const int E = pad / T;
    // keys + fitness (+ the finish's on-chip arrays and weights for pad ≤ kAuxMaxN)
    const size_t sm = (size_t)pad * (sizeof(uint64_t) + sizeof(float)) +
                      (pad <= kAuxMaxN ? (size_t)pad * 16 : 0);
    switch (E) {
      case 2: return launch_pdl(rank_kernel<2>, dim3(s.R), dim3(T), sm, st, s, fsrc, pad);
      case 4: return launch_pdl(rank_kernel<4>, dim3(s.R), dim3(T), sm, st, s, fsrc, pad);
      case 8: return launch_pdl(rank_kernel<8>, dim3(s.R), dim3(T), sm, st, s, fsrc, pad);
      default: return launch_pdl(rank_kernel_smem, dim3(s.R), dim3(T), sm, st, s, fsrc, pad);
    }
  }
  const int nch = npad / kChunk;
  const size_t smem = (size_t)kChunk * sizeof(uint64_t);
  rank_chunk_sort_kernel<<<s.R * nch, 1024, smem, st>>>(s, fsrc, s.gkeys, npad);
  const int64_t pairs = (int64_t)s.R * (npad >> 1);
  for (int k = 2 * kChunk; k <= npad; k <<= 1) {
    for (int j = k >> 1; j >= kChunk; j >>= 1)
      rank_global_step_kernel<<<(unsigned)((pairs + 255) / 256), 256, 0, st>>>(s.gkeys, npad, k,
                                                                            j, s.R);
    rank_chunk_merge_kernel<<<s.R * nch, 1024, smem, st>>>(s.gkeys, npad, k);
  }
  rank_finish_kernel<<<s.R, 1024, 0, st>>>(s, s.gkeys, npad);
  return cudaGetLastError();
}

int rank_launches(const DevState& s) {
  if (use_radix(s) || use_count(s)) return 1;
  int npad = 1, n = 1;
  while (npad < s.N) npad <<= 1;
  if (npad <= kChunk) return 1;
  n = 2;
  for (int k = 2 * kChunk; k <= npad; k <<= 1) {
    for (int j = k >> 1; j >= kChunk; j >>= 1) ++n;
    ++n;
  }
  return n;
}

}  // namespace esb
