// Latency / throughput probes for the FP64 and shared-memory paths the FFT
// engine uses (one warp per SMSP vs many): dependent DADD/DFMA chains,
// independent chains (ILP), LDS.128 round trips.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void k_dadd(double* out, int iters, double s) {
  double a[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = a[i] * s + 1e-9;  // DFMA chain
  }
  long long t1 = clock64();
  double r = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
  if (threadIdx.x == 0 && blockIdx.x == 0) printf("  dfma ILP=%d threads=%d: %.2f cycles per dependent step (per warp)\n", ILP, blockDim.x, (double)(t1 - t0) / iters);
}

__global__ void k_lds(double* out, int iters) {
  __shared__ double2 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(i, 0);
  __syncthreads();
  int idx = threadIdx.x;
  long long t0 = clock64();
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    double2 v = sm[idx & 1023];
    idx = (int)v.x + 1;   // dependent
    acc += v.y;
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc + idx;
  if (threadIdx.x == 0) printf("  lds.128 dependent latency: %.2f cycles (threads=%d)\n", (double)(t1 - t0) / iters, blockDim.x);
}

int main() {
  double* d;
  cudaMalloc(&d, 1 << 24);
  int it = 4096;
  k_dadd<1><<<1, 32>>>(d, it, 1.0000001); cudaDeviceSynchronize();
  k_dadd<1><<<1, 32>>>(d, it, 1.0000001); cudaDeviceSynchronize();
  k_dadd<2><<<1, 32>>>(d, it, 1.0000001); cudaDeviceSynchronize();
  k_dadd<4><<<1, 32>>>(d, it, 1.0000001); cudaDeviceSynchronize();
  k_dadd<8><<<1, 32>>>(d, it, 1.0000001); cudaDeviceSynchronize();
  k_dadd<16><<<1, 32>>>(d, it, 1.0000001); cudaDeviceSynchronize();
  k_dadd<8><<<1, 128>>>(d, it, 1.0000001); cudaDeviceSynchronize();
  k_dadd<8><<<1, 512>>>(d, it, 1.0000001); cudaDeviceSynchronize();
  k_dadd<8><<<1, 1024>>>(d, it, 1.0000001); cudaDeviceSynchronize();
  k_lds<<<1, 32>>>(d, it); cudaDeviceSynchronize();
  k_lds<<<1, 32>>>(d, it); cudaDeviceSynchronize();
  k_lds<<<1, 512>>>(d, it); cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
