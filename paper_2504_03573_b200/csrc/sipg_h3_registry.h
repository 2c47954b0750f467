// Kernel registry of the config-4 hybrid kernels (sipg_h3.cu).
#pragma once
#include <stddef.h>
#include <vector>
#include "sipg_h3.cuh"

using H3Fn = void (*)(const H3Plan, const int, const double*, double*);
// __constant__ tables of a (shape, n) instantiation: D, A, psi, E, ED, pts, W (plan3d.ClassTables3 parts)
using H3UploadFn = cudaError_t (*)(const double* D, const double* A, const double* psi, const double* E,
                                   const double* ED, const double* pts, const double* W);
struct H3Entry {
  int shape, n;
  H3Fn pub, apply;
  int threads;         // CTA threads: epc teams of q^2 threads
  int epc;             // elements per CTA
  size_t smem_pub, smem_apply;
  H3UploadFn upload;
};
void sipg_register_h3(std::vector<H3Entry>& v);
// the slot kernels over the work-list records [first, first + count): the flux kernel (identity-map
// or mapped list) between publish and apply, the trace-map kernel (mapped list) right after publish
void sipg_h3c_flux_launch(const H3Plan& P, int64_t first, int64_t count, bool mapped, int sms, cudaStream_t stream);
void sipg_h3c_map_launch(const H3Plan& P, int64_t first, int64_t count, int sms, cudaStream_t stream);
