// sm_100a kernels for quad elements (templates in sipg_kernels.cuh).
#include "sipg_kernels.cuh"
#include "sipg_registry.h"
SIPG_DEFINE_ENTRY
void sipg_register_quad(std::vector<KernelEntry>& v) {
  SIPG_ENTRIES_NQ(SHAPE_QUAD, 2);
  SIPG_ENTRIES_NQ(SHAPE_QUAD, 3);
  SIPG_ENTRIES_NQ(SHAPE_QUAD, 4);
  SIPG_ENTRIES_NQ(SHAPE_QUAD, 5);
  SIPG_ENTRIES_NQ(SHAPE_QUAD, 6);
  SIPG_ENTRIES_NQ(SHAPE_QUAD, 7);
  SIPG_ENTRIES_NQ(SHAPE_QUAD, 8);
  SIPG_ENTRIES_NQ(SHAPE_QUAD, 9);
  SIPG_ENTRIES_NQ(SHAPE_QUAD, 10);
}

void sipg_register_planes_quad(std::vector<PlanesEntry>& v) {
  v.push_back(PlanesEntry{SHAPE_QUAD, 2, 3, &sipg::k_traces2d<SHAPE_QUAD, 2, 3>});
  v.push_back(PlanesEntry{SHAPE_QUAD, 3, 4, &sipg::k_traces2d<SHAPE_QUAD, 3, 4>});
  v.push_back(PlanesEntry{SHAPE_QUAD, 4, 5, &sipg::k_traces2d<SHAPE_QUAD, 4, 5>});
  v.push_back(PlanesEntry{SHAPE_QUAD, 5, 6, &sipg::k_traces2d<SHAPE_QUAD, 5, 6>});
  v.push_back(PlanesEntry{SHAPE_QUAD, 6, 7, &sipg::k_traces2d<SHAPE_QUAD, 6, 7>});
  v.push_back(PlanesEntry{SHAPE_QUAD, 7, 8, &sipg::k_traces2d<SHAPE_QUAD, 7, 8>});
  v.push_back(PlanesEntry{SHAPE_QUAD, 8, 9, &sipg::k_traces2d<SHAPE_QUAD, 8, 9>});
  v.push_back(PlanesEntry{SHAPE_QUAD, 9, 10, &sipg::k_traces2d<SHAPE_QUAD, 9, 10>});
  v.push_back(PlanesEntry{SHAPE_QUAD, 10, 11, &sipg::k_traces2d<SHAPE_QUAD, 10, 11>});
}
