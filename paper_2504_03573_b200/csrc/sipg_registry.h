// Kernel registry: each shape's translation unit instantiates its templates.
#pragma once
#include <stddef.h>
#include <vector>
#include "sipg_plan.h"

using KernelFn = void (*)(const DevPlan, const int, const double*, double*);

struct KernelEntry {
  int shape, n, q, geom;
  KernelFn fn;
  int threads;
  size_t smem;
};

void sipg_register_quad(std::vector<KernelEntry>& v);
void sipg_register_tri(std::vector<KernelEntry>& v);
void sipg_register_hex(std::vector<KernelEntry>& v);

#ifdef __CUDACC__
template <int SHAPE, int N, int Q, int GEOM>
KernelEntry sipg_entry();
#define SIPG_DEFINE_ENTRY                                                                    \
  template <int SHAPE, int N, int Q, int GEOM>                                               \
  KernelEntry sipg_entry() {                                                                 \
    using C = sipg::Cfg<SHAPE, N, Q>;                                                        \
    return KernelEntry{SHAPE, N, Q, GEOM, &sipg::k_apply<SHAPE, N, Q, GEOM>, C::NT,          \
                       sizeof(double) * (size_t)C::TOTAL};                                   \
  }
#define SIPG_ENTRIES_NQ(S, N)                                                                \
  v.push_back(sipg_entry<S, N, N + 1, GEOM_REGULAR>());                                      \
  v.push_back(sipg_entry<S, N, N + 1, GEOM_POINTWISE>())
#endif
