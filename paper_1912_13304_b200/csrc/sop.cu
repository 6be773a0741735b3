// Translation unit of the r02 sine-domain operator (sop_kernels.cuh) and its
// host launcher (sop.h); compiled separately from fde.cu.
#include <cuda_runtime.h>

#include "sop.h"
#include "sop_kernels.cuh"
#include "stau_kernels.cuh"

namespace fde {
namespace sop {

template <int U, bool ONEWAVE>
static cudaError_t launch_k(const SopArgs& a, const SopMaps& maps, cudaStream_t st) {
  constexpr int UPC = sop_upc<U>();
#ifndef FDE_SOP_SMEM_PAD
#define FDE_SOP_SMEM_PAD 0   // measurement builds only: extra dynamic smem per CTA (limits units per SM)
#endif
  const size_t smem = (size_t)UPC * Geo<U>::SLOTS * sizeof(double2) + FDE_SOP_SMEM_PAD;
  auto kern = k_sop<U, ONEWAVE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<a.total_warps / UPC, U * UPC, smem, st>>>(a, maps);   // total_warps: units over the batch
  return cudaGetLastError();
}

// m = 1024: the 128-register instantiation when every unit of the launch is
// resident at once (8 per SM), else 144 (sop_maxreg)
template <int U>
static cudaError_t launch_u(const SopArgs& a, const SopMaps& maps, cudaStream_t st) {
  if (U != 64) return launch_k<U, false>(a, maps, st);
  int dev = 0, sms = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
#ifndef FDE_SOP_ONEWAVE
#define FDE_SOP_ONEWAVE 1
#endif
  return (FDE_SOP_ONEWAVE && a.total_warps <= 8 * sms) ? launch_k<U, true>(a, maps, st)
                                                       : launch_k<U, false>(a, maps, st);
}

bool supported(int m) { return m == 512 || m == 1024 || m == 2048 || m == 4096; }

cudaError_t launch(const SopArgs& a, const SopMaps& maps, cudaStream_t st) {
  switch (a.m) {
    case 512: return launch_u<32>(a, maps, st);
    case 1024: return launch_u<64>(a, maps, st);
    case 2048: return launch_u<128>(a, maps, st);
    case 4096: return launch_u<256>(a, maps, st);
    default: return cudaErrorInvalidValue;
  }
}

// TMA descriptors of the 2D arrays [batch][n][pitch] (fp64) with a box of
// 2 columns × 256 rows (the column units' staging, sop_kernels.cuh)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
cudaError_t make_maps(SopMaps* maps, const double* z, const double* p, const double* p2, const double* wc, int n,
                      int pitch, int batch) {
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess) return e;
    if (q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  const cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)n, (cuuint64_t)batch};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch * sizeof(double), (cuuint64_t)n * pitch * sizeof(double)};
  const cuuint32_t box[3] = {2, 256, 1}, estr[3] = {1, 1, 1};
  const double* src[4] = {z, p, p2, wc};
  CUtensorMap* dst[4] = {&maps->z, &maps->p, &maps->p2, &maps->wc};
  for (int i = 0; i < 4; ++i) {
    const CUresult r = encode(dst[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(src[i]), dims, strides,
                              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

int warps_for(int m, int batch) { return batch * m; }   // units (CTAs): 2·npairs = m per RHS

// ---- 2D τ-solve on the r02 transform engine (stau_kernels.cuh)
template <int U>
static cudaError_t stau_k(bool cols, const StauArgs& a, const StauMaps* maps, int batch, cudaStream_t st) {
  const size_t smem = (size_t)Geo<U>::SLOTS * sizeof(double2);
  const dim3 grid((a.n + 1) / 2, batch);
  if (cols) {
    cudaError_t e = cudaFuncSetAttribute(k_stau_cols<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_stau_cols<U><<<grid, U, smem, st>>>(a, *maps);
  } else {
    cudaError_t e = cudaFuncSetAttribute(k_stau_rows<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_stau_rows<U><<<grid, U, smem, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t stau_launch(bool cols, const StauArgs& a, const StauMaps* maps, int batch, cudaStream_t st) {
  switch (a.m) {
    case 512: return stau_k<32>(cols, a, maps, batch, st);
    case 1024: return stau_k<64>(cols, a, maps, batch, st);
    case 2048: return stau_k<128>(cols, a, maps, batch, st);
    case 4096: return stau_k<256>(cols, a, maps, batch, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t make_stau_maps(StauMaps* maps, const double* t1, const double* t2, int n, int batch) {
  SopMaps tmp;
  // the same descriptor shape as the sop column staging: [batch][n][m], box 2 × 256
  cudaError_t e = make_maps(&tmp, t1, t2, t1, t2, n, n + 1, batch);
  if (e != cudaSuccess) return e;
  maps->t1 = tmp.z;
  maps->t2 = tmp.p;
  return cudaSuccess;
}

}  // namespace sop
}  // namespace fde

#if FDE_SOP_TRACE
// measurement builds only (-DFDE_SOP_TRACE=1): the last k_sop launch's trace
extern "C" int fde_debug_sop_trace(unsigned long long* host, int n) {
  if (n > 8192 * 8) n = 8192 * 8;
  return (int)cudaMemcpyFromSymbol(host, fde::sop::g_sop_trace, sizeof(unsigned long long) * n);
}
#endif
