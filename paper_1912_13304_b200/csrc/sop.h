// Host interface of the r02 sine-domain operator kernel (sop.cu).
#pragma once
#include <cuda_runtime.h>

#include "sop_kernels.cuh"

namespace fde {
namespace sop {

bool supported(int m);                                // m = n+1 the kernel is instantiated for
int warps_for(int m, int batch);                      // SopArgs::total_warps: the units (CTAs) over the batch
cudaError_t launch(const SopArgs& a, cudaStream_t st);

}  // namespace sop
}  // namespace fde
