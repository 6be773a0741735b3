// P_tri: the tridiagonal part of M (Table 2; reading R19),
// 1D only. z = P_tri⁻¹ r by parallel cyclic reduction in one CTA per RHS: in
// log2(n) steps every equation eliminates its neighbours at distance s, all
// equations at once (the B200 form of the paper's O(n) Thomas solve, which is
// inherently sequential). Coefficients (sub, diag, sup) are read from the
// handle's tables; the system lives in shared memory (4 n doubles).
#pragma once
#include "line_kernels.cuh"

namespace fde {

constexpr int TRI_THREADS = 1024;
constexpr int TRI_PER_THREAD = 4;   // n <= 4096

__global__ void __launch_bounds__(TRI_THREADS) k_tri_pcr(const double* __restrict__ sub, const double* __restrict__ diag,
                                                          const double* __restrict__ sup, const double* __restrict__ r,
                                                          double* __restrict__ z, int n, const int* gate) {
  FDE_PDL_ENTRY();
  if (gate && *gate == 0) return;
  extern __shared__ double tsm[];
  double* A = tsm;
  double* B = tsm + n;
  double* C = tsm + 2 * n;
  double* D = tsm + 3 * n;
  const size_t o = (size_t)blockIdx.y * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    A[i] = i > 0 ? sub[i] : 0.0;
    B[i] = diag[i];
    C[i] = i < n - 1 ? sup[i] : 0.0;
    D[i] = r[o + i];
  }
  __syncthreads();
  for (int s = 1; s < n; s <<= 1) {
    double na[TRI_PER_THREAD], nb[TRI_PER_THREAD], nc[TRI_PER_THREAD], nd[TRI_PER_THREAD];
#pragma unroll
    for (int u = 0; u < TRI_PER_THREAD; ++u) {
      const int i = threadIdx.x + u * blockDim.x;
      if (i >= n) continue;
      // out-of-range neighbours act as identity rows (a = c = d = 0, b = 1)
      const bool lo = i - s >= 0, hi = i + s < n;
      const double am = lo ? A[i - s] : 0.0, bm = lo ? B[i - s] : 1.0, cm = lo ? C[i - s] : 0.0, dm = lo ? D[i - s] : 0.0;
      const double ap = hi ? A[i + s] : 0.0, bp = hi ? B[i + s] : 1.0, cp = hi ? C[i + s] : 0.0, dp = hi ? D[i + s] : 0.0;
      const double k1 = A[i] / bm, k2 = C[i] / bp;
      na[u] = -am * k1;
      nc[u] = -cp * k2;
      nb[u] = B[i] - cm * k1 - ap * k2;
      nd[u] = D[i] - dm * k1 - dp * k2;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < TRI_PER_THREAD; ++u) {
      const int i = threadIdx.x + u * blockDim.x;
      if (i >= n) continue;
      A[i] = na[u];
      B[i] = nb[u];
      C[i] = nc[u];
      D[i] = nd[u];
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) z[o + i] = D[i] / B[i];
}

}  // namespace fde
