// Host interface of the r02 sine-domain operator kernel (sop.cu).
#pragma once
#include <cuda_runtime.h>

#include "sop_kernels.cuh"

namespace fde {
namespace sop {

bool supported(int m);                                // m = n+1 the kernel is instantiated for
int warps_for(int m, int batch);                      // SopArgs::total_warps: the units (CTAs) over the batch
cudaError_t launch(const SopArgs& a, const SopMaps& maps, cudaStream_t st);
// TMA descriptors of ẑ, the two p̂ buffers and w_c (layout [batch][n][pitch])
cudaError_t make_maps(SopMaps* maps, const double* z, const double* p, const double* p2, const double* wc, int n,
                      int pitch, int batch);

}  // namespace sop
}  // namespace fde
