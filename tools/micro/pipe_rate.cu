// Issue-rate micro-benchmark: warp-instructions per clock per SM for single SASS forms and mixes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rate pipe_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kIters = 4096, kChains = 8;

#define BODY(...)                                                              \
  _Pragma("unroll 4") for (int it = 0; it < kIters; ++it) {                    \
    _Pragma("unroll") for (int c = 0; c < kChains; ++c) { __VA_ARGS__ }                \
  }

template <int K>
__global__ void __launch_bounds__(256) kern(float* out, float s) {
  float f[kChains], g[kChains];
  unsigned u[kChains], v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    f[c] = s * (threadIdx.x + c); g[c] = s + c;
    u[c] = threadIdx.x * 7 + c; v[c] = threadIdx.x ^ c;
  }
  if (K == 0) {  // FFMA R,R,R,R (0x223)
    BODY(asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[c]) : "f"(g[c]), "f"(g[(c + 1) % kChains]));)
  } else if (K == 1) {  // FFMA R,R,R,imm (0x423)
    BODY(asm volatile("fma.rn.f32 %0, %0, %1, 0f3E18C294;" : "+f"(f[c]) : "f"(g[c]));)
  } else if (K == 2) {  // FFMA R,R,imm,R (0x823)
    BODY(asm volatile("fma.rn.f32 %0, %0, 0f3E18C294, %1;" : "+f"(f[c]) : "f"(g[c]));)
  } else if (K == 3) {  // FMUL R,R,R
    BODY(asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(f[c]) : "f"(g[c]));)
  } else if (K == 4) {  // FADD R,R,imm
    BODY(asm volatile("add.rn.f32 %0, %0, 0f4B400000;" : "+f"(f[c]));)
  } else if (K == 5) {  // IMAD.WIDE.U32 imm
    BODY(asm volatile("mul.lo.u32 %0, %0, 3528531795;" : "+r"(u[c]));)
  } else if (K == 6) {  // LOP3
    BODY(asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[c]) : "r"(v[c]), "r"(v[(c + 1) % kChains]));)
  } else if (K == 7) {  // IADD3
    BODY(asm volatile("add.u32 %0, %0, %1;" : "+r"(u[c]) : "r"(v[c]));)
  } else if (K == 8) {  // mix: FFMA 0x423 + LOP3 1:1
    BODY(asm volatile("fma.rn.f32 %0, %0, %1, 0f3E18C294;" : "+f"(f[c]) : "f"(g[c]));
         asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[c]) : "r"(v[c]), "r"(v[(c + 1) % kChains]));)
  } else if (K == 9) {  // mix: FFMA 0x223 + LOP3 1:1
    BODY(asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[c]) : "f"(g[c]), "f"(g[(c + 1) % kChains]));
         asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(u[c]) : "r"(v[c]), "r"(v[(c + 1) % kChains]));)
  } else if (K == 10) {  // mul.hi.u32 (IMAD.HI)
    BODY(asm volatile("mul.hi.u32 %0, %0, 3528531795;" : "+r"(u[c]));)
  } else if (K == 11) {  // mix: IMAD.WIDE + LOP3 1:1
    BODY({ unsigned long long w; asm volatile("mul.wide.u32 %0, %1, 3528531795;" : "=l"(w) : "r"(u[c])); u[c] ^= (unsigned)(w >> 32) ^ (unsigned)w; })
  } else if (K == 12) {  // MUFU.LG2
    BODY(asm volatile("lg2.approx.f32 %0, %0;" : "+f"(f[c]));)
  } else if (K == 13) {  // mix: FFMA 0x823 + FFMA 0x423
    BODY(asm volatile("fma.rn.f32 %0, %0, 0f3E18C294, %1;" : "+f"(f[c]) : "f"(g[c]));
         asm volatile("fma.rn.f32 %0, %0, %1, 0f3E18C294;" : "+f"(g[c]) : "f"(f[(c + 3) % kChains]));)
  } else if (K == 14) {  // HFMA2
    BODY({ unsigned h = u[c]; asm volatile("fma.rn.f16x2 %0, %0, %1, %2;" : "+r"(h) : "r"(v[c]), "r"(v[(c+1)%kChains])); u[c] = h; })
  } else if (K == 15) {  // F2F / I2F style: cvt.rn.f32.u32
    BODY(asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(f[c]) : "r"(u[c])); u[c] += 1;)
  }
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc += f[c] + g[c] + (float)u[c];
  if (acc == 1.2345f) out[threadIdx.x] = acc;
}

template <int K>
void run(const char* name, int ops_per_chain_iter) {
  float* out; cudaMalloc(&out, 1024 * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  dim3 grid(sms * 8), block(256);
  kern<K><<<grid, block>>>(out, 1.0f);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<K><<<grid, block>>>(out, 1.0f);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double warp_instr = (double)grid.x * 8 * kIters * kChains * ops_per_chain_iter;
  double per_sm_per_s = warp_instr / sms / (ms * 1e-3);
  printf("%-28s %8.3f ms  %.3f warp-instr/clk/SM at 1965 MHz  (%.3f at attr clk %d MHz)\n", name, ms,
         per_sm_per_s / 1.965e9, per_sm_per_s / (clk * 1e3), clk / 1000);
  cudaFree(out);
}

int main() {
  run<0>("FFMA rrr (223)", 1);
  run<1>("FFMA rr,imm-add (423)", 1);
  run<2>("FFMA r,imm-mul,r (823)", 1);
  run<3>("FMUL rr", 1);
  run<4>("FADD r,imm", 1);
  run<5>("IMAD.LO imm", 1);
  run<6>("LOP3", 1);
  run<7>("IADD", 1);
  run<8>("FFMA423+LOP3", 2);
  run<9>("FFMA223+LOP3", 2);
  run<10>("IMAD.HI imm", 1);
  run<11>("IMAD.WIDE+2LOP", 1);
  run<12>("MUFU.LG2", 1);
  run<13>("FFMA823+FFMA423", 2);
  run<14>("HFMA2", 1);
  run<15>("I2F", 1);
  return 0;
}
