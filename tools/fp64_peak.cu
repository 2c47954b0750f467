// DFMA throughput microbenchmark: measures the fp64 FMA peak of this GPU.
// Each thread runs 8 independent FMA chains; flops = 2 * chains * iters * threads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += r[i];
  if (s == 12345.678) out[0] = s;
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  double* d; cudaMalloc(&d, 8);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 20000;
  dfma_kernel<<<blocks, threads>>>(d, 100, 0.999999, 1e-7);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * (double)iters * blocks * threads;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"fp64_tflops\": %.3f, \"ms\": %.3f, \"sms\": %d, \"clock_khz\": %d, \"l2_bytes\": %d, \"err\": \"%s\"}\n",
         flops / (best * 1e-3) / 1e12, best, p.multiProcessorCount, clk, p.l2CacheSize,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
