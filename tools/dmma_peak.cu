// fp64 tensor-core (DMMA m8n8k4) throughput microbenchmark vs DFMA.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(c[2 * i], c[2 * i + 1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 1.2345) out[0] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 4; warps <= 16; warps *= 2) {
    int blocks = p.multiProcessorCount * 2, threads = 32 * warps / 2, iters = 4000;
    k_dmma<<<blocks, threads>>>(d, 10);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      k_dmma<<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 256 * 8 * (double)iters * blocks * (threads / 32);
    printf("{\"dmma_tflops\": %.3f, \"warps_per_sm\": %d, \"ms\": %.3f, \"err\": \"%s\"}\n",
           flops / (best * 1e-3) / 1e12, warps, best, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
