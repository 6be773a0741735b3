// Translation unit of the r02 sine-domain operator (sop_kernels.cuh) and its
// host launcher (sop.h); compiled separately from fde.cu.
#include <cuda_runtime.h>

#include "sop.h"
#include "sop_kernels.cuh"

namespace fde {
namespace sop {

template <int U, bool ONEWAVE>
static cudaError_t launch_k(const SopArgs& a, cudaStream_t st) {
  constexpr int UPC = sop_upc<U>();
  const size_t smem = (size_t)UPC * Geo<U>::SLOTS * sizeof(double2);
  auto kern = k_sop<U, ONEWAVE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<a.total_warps / UPC, U * UPC, smem, st>>>(a);   // total_warps: units over the batch
  return cudaGetLastError();
}

// m = 1024: the 128-register instantiation when every unit of the launch is
// resident at once (8 per SM), else 144 (sop_maxreg)
template <int U>
static cudaError_t launch_u(const SopArgs& a, cudaStream_t st) {
  if (U != 64) return launch_k<U, false>(a, st);
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
#ifndef FDE_SOP_ONEWAVE
#define FDE_SOP_ONEWAVE 1
#endif
  return (FDE_SOP_ONEWAVE && a.total_warps <= 8 * sms) ? launch_k<U, true>(a, st) : launch_k<U, false>(a, st);
}

bool supported(int m) { return m == 512 || m == 1024 || m == 2048 || m == 4096; }

cudaError_t launch(const SopArgs& a, cudaStream_t st) {
  switch (a.m) {
    case 512: return launch_u<32>(a, st);
    case 1024: return launch_u<64>(a, st);
    case 2048: return launch_u<128>(a, st);
    case 4096: return launch_u<256>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

int warps_for(int m, int batch) { return batch * m; }   // units (CTAs): 2·npairs = m per RHS

}  // namespace sop
}  // namespace fde

#if FDE_SOP_TRACE
// measurement builds only (-DFDE_SOP_TRACE=1): the last k_sop launch's trace
extern "C" int fde_debug_sop_trace(unsigned long long* host, int n) {
  if (n > 8192 * 8) n = 8192 * 8;
  return (int)cudaMemcpyFromSymbol(host, fde::sop::g_sop_trace, sizeof(unsigned long long) * n);
}
#endif
