// Microbenchmarks that fix the roofline denominators the bench does not get
// from MEASURED_PEAKS.json: FP64 FMA throughput, FP64 DMMA (mma.sync) rate,
// shared-memory bandwidth for 16-byte elements, fp64 copy bandwidth, and the
// per-node cost of a chain of tiny kernels replayed as a CUDA graph.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

__global__ void dadd_kernel(double* out, int iters, double a) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 += a; x1 += a; x2 += a; x3 += a; x4 += a; x5 += a; x6 += a; x7 += a;
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

// DMMA m8n8k4 fp64: 2*8*8*4 = 512 flop per warp-instruction
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = c[0][0] + c[1][1] + c[2][0] + c[3][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void smem_kernel(double* out, int iters) {
  __shared__ double2 buf[2048];
  int t = threadIdx.x;
  for (int i = t; i < 2048; i += blockDim.x) buf[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double2 v = buf[(t + k * 256 + i) & 2047];
      acc.x += v.x; acc.y += v.y;
    }
  }
  if (acc.x == 12345.678) out[0] = acc.y;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

__global__ void empty_kernel(int* p) { if (threadIdx.x == 1000000) p[0] = 1; }

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu, \"clock_khz\": %d",
         prop.name, sms, prop.l2CacheSize, prop.sharedMemPerBlockOptin, prop.clockRate);
  double* d_out; CK(cudaMalloc(&d_out, 64));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;
  // FP64 FMA
  {
    int iters = 4096, blocks = sms * 8, threads = 256;
    dfma_kernel<<<blocks, threads>>>(d_out, 16, 0.999, 1e-3);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    dfma_kernel<<<blocks, threads>>>(d_out, iters, 0.999, 1e-3);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf(", \"fp64_fma_tflops\": %.3f", flops / (ms * 1e-3) / 1e12);
    CK(cudaEventRecord(e0));
    dadd_kernel<<<blocks, threads>>>(d_out, iters, 1e-3);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double ops = 8.0 * 16 * (double)iters * blocks * threads;
    printf(", \"fp64_add_gops\": %.1f", ops / (ms * 1e-3) / 1e9);
  }
  // DMMA
  {
    int iters = 4096, blocks = sms * 8, threads = 256;
    dmma_kernel<<<blocks, threads>>>(d_out, 16);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    dmma_kernel<<<blocks, threads>>>(d_out, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double flops = 512.0 * 4 * (double)iters * blocks * (threads / 32);
    printf(", \"fp64_dmma_tflops\": %.3f", flops / (ms * 1e-3) / 1e12);
  }
  // smem
  {
    int iters = 4096, blocks = sms * 4, threads = 256;
    smem_kernel<<<blocks, threads>>>(d_out, 16);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    smem_kernel<<<blocks, threads>>>(d_out, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double bytes = 16.0 * 8 * (double)iters * blocks * threads;
    printf(", \"smem_tbs_chip\": %.2f", bytes / (ms * 1e-3) / 1e12);
  }
  // copy bandwidth fp64
  {
    size_t n = (size_t)1 << 27;  // 2 GiB of double2 per buffer
    double2 *a, *b;
    CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
    CK(cudaMemset(a, 0, n * 16));
    copy_kernel<<<sms * 8, 512>>>(a, b, n);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      copy_kernel<<<sms * 8, 512>>>(a, b, n);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    printf(", \"copy_gbs\": %.1f", 2.0 * n * 16 / (best * 1e-3) / 1e9);
    // L2-resident copy: 32 MB working set
    size_t n2 = (size_t)1 << 21;
    best = 1e30f;
    for (int r = 0; r < 20; ++r) {
      CK(cudaEventRecord(e0));
      for (int k = 0; k < 10; ++k) copy_kernel<<<sms * 8, 512>>>(a, b, n2);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    printf(", \"l2_copy_gbs_32MB\": %.1f", 10 * 2.0 * n2 * 16 / (best * 1e-3) / 1e9);
    CK(cudaFree(a)); CK(cudaFree(b));
  }
  // graph of 100 tiny kernels
  {
    cudaStream_t s; CK(cudaStreamCreate(&s));
    int* p; CK(cudaMalloc(&p, 4));
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int k = 0; k < 100; ++k) empty_kernel<<<sms, 128, 0, s>>>(p);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      CK(cudaEventRecord(e0, s));
      CK(cudaGraphLaunch(ge, s));
      CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    printf(", \"graph_us_per_node\": %.3f", best * 1e3 / 100);
    best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      CK(cudaEventRecord(e0, s));
      for (int k = 0; k < 100; ++k) empty_kernel<<<sms, 128, 0, s>>>(p);
      CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    printf(", \"stream_us_per_launch\": %.3f", best * 1e3 / 100);
  }
  printf("}\n");
  return 0;
}
