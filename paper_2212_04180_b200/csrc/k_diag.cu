// k_diag.cu — device evaluation of single NUMERICS primitives for the exhaustive parity tests
// (es_debug_primitive). Uses exactly the device functions the hot kernels use.
#include "es_internal.h"
#include "fitness.cuh"
#include "noise.cuh"

namespace esb {

__global__ void prim_kernel(int which, const void* __restrict__ in, void* __restrict__ out,
                            int64_t n) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  if (which == 0 || which == 3) {
    const uint32_t* a = static_cast<const uint32_t*>(in) + 6 * k;
    const uint64_t seed = (uint64_t)a[4] | ((uint64_t)a[5] << 32);
    const Philox ph(seed);
    const uint4 o = ph(a[0], a[1], a[2], a[3]);
    if (which == 0) {
      reinterpret_cast<uint4*>(out)[k] = o;
    } else {
      reinterpret_cast<float4*>(out)[k] = box_muller4(o);
    }
  } else if (which == 5) {
    static_cast<float*>(out)[k] = sinpi_half(static_cast<const float*>(in)[k]);
  } else if (which == 4) {
    static_cast<float*>(out)[k] = rho_sqrt(static_cast<const float*>(in)[k]);
  } else if (which == 6) {
    static_cast<float*>(out)[k] = tanh32(static_cast<const float*>(in)[k]);
  } else if (which == 7) {
    static_cast<float*>(out)[k] = tanh16h(static_cast<const float*>(in)[k]);
  } else if (which == 1) {
    static_cast<float*>(out)[k] = ln_poly(static_cast<const float*>(in)[k]);
  } else {
    float c, s;
    sincos2pi_poly(static_cast<const float*>(in)[k], c, s);
    reinterpret_cast<float2*>(out)[k] = make_float2(c, s);
  }
}

cudaError_t launch_primitive(int which, const void* in, void* out, int64_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  prim_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(which, in, out, n);
  return cudaGetLastError();
}

}  // namespace esb
