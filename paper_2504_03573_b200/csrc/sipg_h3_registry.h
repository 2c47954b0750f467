// Kernel registry of the config-4 hybrid kernels (sipg_h3.cu).
#pragma once
#include <stddef.h>
#include <vector>
#include "sipg_h3.cuh"

using H3Fn = void (*)(const H3Plan, const int, const double*, double*);
using H3UploadFn = cudaError_t (*)(const double* D, const double* A, const double* psi);
struct H3Entry {
  int shape, n;
  H3Fn pub, apply;
  int threads;
  size_t smem_pub, smem_apply;
  H3UploadFn upload;   // __constant__ tables of this (shape, n) instantiation
};
void sipg_register_h3(std::vector<H3Entry>& v);
