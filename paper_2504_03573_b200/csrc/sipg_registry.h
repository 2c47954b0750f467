// Kernel registry: each shape's translation unit instantiates its templates.
#pragma once
#include <stddef.h>
#include <vector>
#include "sipg_plan.h"

using KernelFn = void (*)(const DevPlan, const int, const double*, double*);
using UploadFn = cudaError_t (*)(const double* V, const double* D, const double* W, const double* dVend);

// kind: 6/7 = planes-consuming hex kernel (k_hexp) without / with fast shared traces,
//       0 = generic smem kernel, one CTA per element (any basis / rule / geometry),
//       5 = the same element routine, one warp per element (2-D shapes, persistent),
//       4 = register-column hex kernel (k_hex), conforming + boundary faces only,
//       2 = register-column hex kernel with the generic face path
struct KernelEntry {
  int shape, n, q, geom, kind;
  KernelFn fn;
  int threads;
  size_t smem;          // dynamic shared memory bytes
  UploadFn upload;      // constant-table upload (kinds 1, 2)
};

using PlanesFn = void (*)(const DevPlan, const int, const double*);
struct PlanesEntry {
  int shape, n, q;
  PlanesFn fn;
};
void sipg_register_planes(std::vector<PlanesEntry>& v);
void sipg_register_planes_quad(std::vector<PlanesEntry>& v);
void sipg_register_planes_tri(std::vector<PlanesEntry>& v);

void sipg_register_quad(std::vector<KernelEntry>& v);
void sipg_register_tri(std::vector<KernelEntry>& v);
void sipg_register_hex(std::vector<KernelEntry>& v);

#include <cuda_runtime.h>
#ifdef __CUDACC__
// warps (elements in flight) per CTA of the 2-D warp-per-element kernels
#ifndef SIPG_WPC
#define SIPG_WPC 8
#endif
template <int SHAPE, int N, int Q, int GEOM>
KernelEntry sipg_entry();
#define SIPG_DEFINE_ENTRY                                                                    \
  template <int SHAPE, int N, int Q, int GEOM>                                               \
  KernelEntry sipg_entry() {                                                                 \
    using C = sipg::Cfg<SHAPE, N, Q>;                                                        \
    if (SHAPE == SHAPE_HEX)                                                                  \
      return KernelEntry{SHAPE, N, Q, GEOM, 0, &sipg::k_apply<SHAPE, N, Q, GEOM>, C::NT,     \
                         sizeof(double) * (size_t)C::TOTAL, nullptr};                        \
    return KernelEntry{SHAPE, N, Q, GEOM, 5, &sipg::k_apply_w<SHAPE, N, Q, GEOM, SIPG_WPC>,      \
                       32 * SIPG_WPC, sizeof(double) * (size_t)(C::TABP + SIPG_WPC * C::ESZ), nullptr};            \
  }                                                                                          \
  /* 2-D shapes also get the CTA-per-element kernel (kind 0): small classes (configs 0 / 1) */  \
  /* are latency-bound and run every element at once, 64 threads each instead of one warp */   \
  template <int SHAPE, int N, int Q, int GEOM>                                               \
  KernelEntry sipg_entry_cta() {                                                             \
    using C = sipg::Cfg<SHAPE, N, Q>;                                                        \
    return KernelEntry{SHAPE, N, Q, GEOM, 0, &sipg::k_apply<SHAPE, N, Q, GEOM>, C::NT,       \
                       sizeof(double) * (size_t)C::TOTAL, nullptr};                          \
  }
#define SIPG_ENTRIES_NQ(S, N)                                                                \
  v.push_back(sipg_entry<S, N, N + 1, GEOM_REGULAR>());                                      \
  v.push_back(sipg_entry<S, N, N + 1, GEOM_POINTWISE>());                                    \
  if (S != SHAPE_HEX) {                                                                      \
    v.push_back(sipg_entry_cta<S, N, N + 1, GEOM_REGULAR>());                                \
    v.push_back(sipg_entry_cta<S, N, N + 1, GEOM_POINTWISE>());                              \
  }
#define SIPG_HEX_PLANES(N)                                                                   \
  v.push_back(KernelEntry{SHAPE_HEX, N, N + 1, GEOM_REGULAR, 6, &sipg::k_hexp<N, N + 1, false>,    \
                          (N + 1) * (N + 1), sipg::HexPlanes<N, N + 1, false>::smem_bytes(),      \
                          &sipg::hex_fast_upload<N, N + 1>});                                    \
  v.push_back(KernelEntry{SHAPE_HEX, N, N + 1, GEOM_REGULAR, 7, &sipg::k_hexp<N, N + 1, true>,     \
                          (N + 1) * (N + 1), sipg::HexPlanes<N, N + 1, true>::smem_bytes(),       \
                          &sipg::hex_fast_upload<N, N + 1>})
#define SIPG_HEX_FAST(N)                                                                     \
  v.push_back(KernelEntry{SHAPE_HEX, N, N + 1, GEOM_REGULAR, 4, &sipg::k_hex<N, N + 1, false>,  \
                          (N + 1) * (N + 1), sipg::HexFast<N, N + 1>::smem_bytes(false),         \
                          &sipg::hex_fast_upload<N, N + 1>});                                   \
  v.push_back(KernelEntry{SHAPE_HEX, N, N + 1, GEOM_REGULAR, 2, &sipg::k_hex<N, N + 1, true>,   \
                          (N + 1) * (N + 1), sipg::HexFast<N, N + 1>::smem_bytes(true),          \
                          &sipg::hex_fast_upload<N, N + 1>})
#endif
