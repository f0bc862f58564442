// k_nvls.cu — SURVEY §8(f) f2, NVLS variant, host side (the kernel is k_tell.cu:nvls_apply_kernel):
// the population-sharded tell's all-reduce done INSIDE the NVSwitch ("aggregated via map-reduce"; B200 NVLink SHARP). Every rank binds one
// symmetric buffer — [direction sums G (2·R·D binary64) | mean | best_x | σ_d] — to a multicast
// object; ONE kernel per rank then, for its quad slice, reads Σ_ranks G with
// `multimem.ld_reduce.add.f64` (the switch adds the W copies), applies the update to the slice
// (optimizer state local to the rank), and broadcasts the slice's mean / best_x / σ_d to every
// rank with `multimem.st` (one store, replicated by the switch). Host side: the multicast object
// lifecycle through the CUDA driver's VMM API (fabric handles, so that the 64-byte handle can be
// exchanged over any transport), reached through the runtime's driver entry points.
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "es_internal.h"

namespace esb {

// ------------------------------------------------------------------------------- driver calls
#define ES_DRV(name) static decltype(&::name) p_##name = nullptr;
ES_DRV(cuMemCreate)
ES_DRV(cuMemRelease)
ES_DRV(cuMemAddressReserve)
ES_DRV(cuMemAddressFree)
ES_DRV(cuMemMap)
ES_DRV(cuMemUnmap)
ES_DRV(cuMemSetAccess)
ES_DRV(cuMemGetAllocationGranularity)
ES_DRV(cuMulticastCreate)
ES_DRV(cuMulticastAddDevice)
ES_DRV(cuMulticastBindMem)
ES_DRV(cuMulticastUnbind)
ES_DRV(cuMulticastGetGranularity)
ES_DRV(cuMemExportToShareableHandle)
ES_DRV(cuMemImportFromShareableHandle)
#undef ES_DRV

static bool drv_load() {
  static int ok = -1;
  if (ok >= 0) return ok == 1;
  auto get = [](const char* n, void** f) {
    cudaDriverEntryPointQueryResult q;
    return cudaGetDriverEntryPoint(n, f, cudaEnableDefault, &q) == cudaSuccess &&
           q == cudaDriverEntryPointSuccess;
  };
  ok = get("cuMemCreate", (void**)&p_cuMemCreate) && get("cuMemRelease", (void**)&p_cuMemRelease) &&
       get("cuMemAddressReserve", (void**)&p_cuMemAddressReserve) &&
       get("cuMemAddressFree", (void**)&p_cuMemAddressFree) && get("cuMemMap", (void**)&p_cuMemMap) &&
       get("cuMemUnmap", (void**)&p_cuMemUnmap) && get("cuMemSetAccess", (void**)&p_cuMemSetAccess) &&
       get("cuMemGetAllocationGranularity", (void**)&p_cuMemGetAllocationGranularity) &&
       get("cuMulticastCreate", (void**)&p_cuMulticastCreate) &&
       get("cuMulticastAddDevice", (void**)&p_cuMulticastAddDevice) &&
       get("cuMulticastBindMem", (void**)&p_cuMulticastBindMem) &&
       get("cuMulticastUnbind", (void**)&p_cuMulticastUnbind) &&
       get("cuMulticastGetGranularity", (void**)&p_cuMulticastGetGranularity) &&
       get("cuMemExportToShareableHandle", (void**)&p_cuMemExportToShareableHandle) &&
       get("cuMemImportFromShareableHandle", (void**)&p_cuMemImportFromShareableHandle)
           ? 1 : 0;
  return ok == 1;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Symmetric layout, identical on every rank.
static void nvls_layout(const DevState& s, NvlsHost& h) {
  const size_t RD = (size_t)s.R * s.D;
  size_t o = 0;
  h.off_g = o;   o = align_up(o + 2 * RD * sizeof(double), 256);
  h.off_mean = o; o = align_up(o + RD * sizeof(float), 256);
  h.off_best = o; o = align_up(o + RD * sizeof(float), 256);
  h.off_sig = s.vec[F_SIGMA_D] ? o : (size_t)-1;
  if (s.vec[F_SIGMA_D]) o = align_up(o + RD * sizeof(float), 256);
  h.used = o;
}

const char* nvls_open(const DevState& s, NvlsHost& h, void* handle, bool creator) {
  if (!drv_load()) return "CUDA driver VMM / multicast entry points unavailable";
  int ord = 0;
  cudaGetDevice(&ord);
  h.dev = (CUdevice)ord;
  nvls_layout(s, h);
  CUmulticastObjectProp mp;
  std::memset(&mp, 0, sizeof mp);
  mp.numDevices = (unsigned)s.W;
  // a single-rank team needs no export (and so no fabric / IMEX channel)
  mp.handleTypes = s.W > 1 ? CU_MEM_HANDLE_TYPE_FABRIC : CU_MEM_HANDLE_TYPE_NONE;
  size_t mgran = 0, pgran = 0;
  mp.size = h.used;
  if (p_cuMulticastGetGranularity(&mgran, &mp, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS)
    return "cuMulticastGetGranularity failed (no multicast support?)";
  CUmemAllocationProp pp;
  std::memset(&pp, 0, sizeof pp);
  pp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  pp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  pp.location.id = ord;
  if (p_cuMemGetAllocationGranularity(&pgran, &pp, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS)
    return "cuMemGetAllocationGranularity failed";
  h.gran = std::max(mgran, pgran);
  h.bytes = align_up(h.used, h.gran);
  mp.size = h.bytes;
  if (creator) {
    if (p_cuMulticastCreate(&h.mc, &mp) != CUDA_SUCCESS) return "cuMulticastCreate failed";
    if (s.W > 1 &&
        p_cuMemExportToShareableHandle(handle, h.mc, CU_MEM_HANDLE_TYPE_FABRIC, 0) != CUDA_SUCCESS)
      return "cuMemExportToShareableHandle(FABRIC) failed";
  } else if (p_cuMemImportFromShareableHandle(&h.mc, handle, CU_MEM_HANDLE_TYPE_FABRIC) != CUDA_SUCCESS) {
    return "cuMemImportFromShareableHandle(FABRIC) failed";
  }
  h.have_mc = true;
  if (p_cuMulticastAddDevice(h.mc, h.dev) != CUDA_SUCCESS) return "cuMulticastAddDevice failed";
  if (p_cuMemCreate(&h.phys, h.bytes, &pp, 0) != CUDA_SUCCESS) return "cuMemCreate failed";
  h.have_phys = true;
  CUmemAccessDesc ad;
  ad.location = pp.location;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (p_cuMemAddressReserve(&h.uva, h.bytes, h.gran, 0, 0) != CUDA_SUCCESS ||
      p_cuMemMap(h.uva, h.bytes, 0, h.phys, 0) != CUDA_SUCCESS ||
      p_cuMemSetAccess(h.uva, h.bytes, &ad, 1) != CUDA_SUCCESS)
    return "mapping the symmetric buffer failed";
  h.stage = 1;
  return nullptr;
}

// After EVERY rank has added its device (caller's barrier): bind this rank's memory and map the
// multicast address range.
const char* nvls_bind(NvlsHost& h) {
  if (h.stage != 1) return "nvls_bind before nvls_open";
  if (p_cuMulticastBindMem(h.mc, 0, h.phys, 0, h.bytes, 0) != CUDA_SUCCESS)
    return "cuMulticastBindMem failed";
  CUmemAccessDesc ad;
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = (int)h.dev;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (p_cuMemAddressReserve(&h.mcva, h.bytes, h.gran, 0, 0) != CUDA_SUCCESS ||
      p_cuMemMap(h.mcva, h.bytes, 0, h.mc, 0) != CUDA_SUCCESS ||
      p_cuMemSetAccess(h.mcva, h.bytes, &ad, 1) != CUDA_SUCCESS)
    return "mapping the multicast range failed";
  h.stage = 2;
  return nullptr;
}

void nvls_close(NvlsHost& h) {
  if (!drv_load()) return;
  if (h.mcva) { p_cuMemUnmap(h.mcva, h.bytes); p_cuMemAddressFree(h.mcva, h.bytes); }
  if (h.stage == 2) p_cuMulticastUnbind(h.mc, h.dev, 0, h.bytes);
  if (h.uva) { p_cuMemUnmap(h.uva, h.bytes); p_cuMemAddressFree(h.uva, h.bytes); }
  if (h.have_phys) p_cuMemRelease(h.phys);
  if (h.have_mc) p_cuMemRelease(h.mc);
  h = NvlsHost{};
}

}  // namespace esb
