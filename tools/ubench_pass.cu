// Floor of one line pass at n = 1023 (1023 x 1023 fp64, 8.4 MB in + 8.4 MB out,
// warm L2): grid-stride copy vs the line-kernel launch geometries with their
// load/store patterns but no transform. CUDA events, median of 50.
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void k_copy(const double* __restrict__ x, double* __restrict__ y, long long n) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) y[e] = x[e];
}
// rows: one pair of rows per group of P threads, R points per thread at stride P
template <int P, int R, int FPC, bool SYNC>
__global__ void k_rows(const double* __restrict__ x, double* __restrict__ y, int n, int nlines) {
  const int f = threadIdx.x / P, t = threadIdx.x % P;
  const int g = blockIdx.x * FPC + f;
  const int l0 = 2 * g, l1 = 2 * g + 1;
  double2 v[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int p = q * P + t;
    v[q].x = (p < n && l0 < nlines) ? x[(long long)l0 * n + p] : 0.0;
    v[q].y = (p < n && l1 < nlines) ? x[(long long)l1 * n + p] : 0.0;
  }
  if (SYNC) __syncthreads();
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int p = q * P + t;
    if (p < n && l0 < nlines) y[(long long)l0 * n + p] = v[q].x * 2.0;
    if (p < n && l1 < nlines) y[(long long)l1 * n + p] = v[q].y * 2.0;
  }
}
template <int P, int R, int FPC>
__global__ void k_cols(const double* __restrict__ x, double* __restrict__ y, int n, int nlines) {
  const int f = threadIdx.x % FPC, t = threadIdx.x / FPC;
  const int g = blockIdx.x * FPC + f;
  const int l0 = 2 * g, l1 = 2 * g + 1;
  double2 v[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int p = q * P + t;
    v[q].x = (p < n && l0 < nlines) ? x[(long long)p * n + l0] : 0.0;
    v[q].y = (p < n && l1 < nlines) ? x[(long long)p * n + l1] : 0.0;
  }
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int p = q * P + t;
    if (p < n && l0 < nlines) y[(long long)p * n + l0] = v[q].x * 2.0;
    if (p < n && l1 < nlines) y[(long long)p * n + l1] = v[q].y * 2.0;
  }
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<float> ts;
  for (int i = 0; i < 60; ++i) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (i >= 10) ts.push_back(ms * 1e3f);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

int main() {
  const int n = 1023; const long long N = (long long)n * n;
  double *x, *y;
  cudaMalloc(&x, N * 8); cudaMalloc(&y, N * 8);
  cudaMemset(x, 0, N * 8);
  printf("copy grid-stride 592x256: %.2f us\n", timeit([&] { k_copy<<<592, 256>>>(x, y, N); }));
  printf("copy grid-stride 4096x256: %.2f us\n", timeit([&] { k_copy<<<4096, 256>>>(x, y, N); }));
  printf("empty kernel: %.2f us\n", timeit([&] { k_copy<<<1, 32>>>(x, y, 0); }));
  printf("rows P=128 R=16 FPC=1 (toeplitz geometry): %.2f us\n", timeit([&] { k_rows<128, 8, 1, true><<<512, 128>>>(x, y, n, n); }));
  printf("rows P=64 R=16 FPC=1: %.2f us\n", timeit([&] { k_rows<64, 16, 1, true><<<512, 64>>>(x, y, n, n); }));
  printf("rows P=128 R=8 FPC=1: %.2f us\n", timeit([&] { k_rows<128, 8, 1, true><<<512, 128>>>(x, y, n, n); }));
  printf("rows P=256 R=4 FPC=1: %.2f us\n", timeit([&] { k_rows<256, 4, 1, true><<<512, 256>>>(x, y, n, n); }));
  printf("cols P=64 R=16 FPC=2: %.2f us\n", timeit([&] { k_cols<64, 16, 2><<<256, 128>>>(x, y, n, n); }));
  printf("cols P=128 R=8 FPC=2: %.2f us\n", timeit([&] { k_cols<128, 8, 2><<<256, 256>>>(x, y, n, n); }));
  printf("cols P=64 R=16 FPC=8: %.2f us\n", timeit([&] { k_cols<64, 16, 8><<<64, 512>>>(x, y, n, n); }));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
