// Host interface of the r02 sine-domain operator kernel (sop.cu).
#pragma once
#include <cuda_runtime.h>

#include "sop_kernels.cuh"
#include "stau_kernels.cuh"

namespace fde {
namespace sop {

bool supported(int m);                                // m = n+1 the kernel is instantiated for
int warps_for(int m, int batch);                      // SopArgs::total_warps: the units (CTAs) over the batch
cudaError_t launch(const SopArgs& a, const SopMaps& maps, cudaStream_t st);
// TMA descriptors of ẑ, the two p̂ buffers and w_c (layout [batch][n][pitch])
cudaError_t make_maps(SopMaps* maps, const double* z, const double* p, const double* p2, const double* wc, int n,
                      int pitch, int batch);
// 2D τ-solve passes on the same transform engine (stau_kernels.cuh): rows DST
// (cols = false) or the columns τ core t1 → t2 (cols = true, pitch m, TMA)
cudaError_t stau_launch(bool cols, const StauArgs& a, const StauMaps* maps, int batch, cudaStream_t st);
cudaError_t make_stau_maps(StauMaps* maps, const double* t1, const double* t2, int n, int batch);

}  // namespace sop
}  // namespace fde
