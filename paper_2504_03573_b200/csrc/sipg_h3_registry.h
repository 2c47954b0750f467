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
  int gen;             // 1: register-column kernels (sipg_h3c.cuh); 0: first generation (sipg_h3.cuh)
  H3Fn pub, apply;
  int threads;
  int epc;             // elements per CTA (generation 1 packs several q^2-thread teams into a CTA)
  size_t smem_pub, smem_apply;
  H3UploadFn upload;
};
void sipg_register_h3(std::vector<H3Entry>& v);
// generation 1: the flux kernel (one warp per slot) over cslots[first, first + count), between publish and apply
void sipg_h3c_flux_launch(const H3Plan& P, int64_t first, int64_t count, bool mapped, int sms, cudaStream_t stream);
// generation 1: the trace-map kernel over the same work list, right after the publish kernels of those slots
void sipg_h3c_map_launch(const H3Plan& P, int64_t first, int64_t count, int sms, cudaStream_t stream);
