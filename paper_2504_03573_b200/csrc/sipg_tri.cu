// sm_100a kernels for tri elements (templates in sipg_kernels.cuh).
#include "sipg_kernels.cuh"
#include "sipg_registry.h"
SIPG_DEFINE_ENTRY
void sipg_register_tri(std::vector<KernelEntry>& v) {
  SIPG_ENTRIES_NQ(SHAPE_TRI, 2);
  SIPG_ENTRIES_NQ(SHAPE_TRI, 3);
  SIPG_ENTRIES_NQ(SHAPE_TRI, 4);
  SIPG_ENTRIES_NQ(SHAPE_TRI, 5);
  SIPG_ENTRIES_NQ(SHAPE_TRI, 6);
  SIPG_ENTRIES_NQ(SHAPE_TRI, 7);
  SIPG_ENTRIES_NQ(SHAPE_TRI, 8);
  SIPG_ENTRIES_NQ(SHAPE_TRI, 9);
  SIPG_ENTRIES_NQ(SHAPE_TRI, 10);
}

void sipg_register_planes_tri(std::vector<PlanesEntry>& v) {
  v.push_back(PlanesEntry{SHAPE_TRI, 2, 3, &sipg::k_traces2d<SHAPE_TRI, 2, 3>});
  v.push_back(PlanesEntry{SHAPE_TRI, 3, 4, &sipg::k_traces2d<SHAPE_TRI, 3, 4>});
  v.push_back(PlanesEntry{SHAPE_TRI, 4, 5, &sipg::k_traces2d<SHAPE_TRI, 4, 5>});
  v.push_back(PlanesEntry{SHAPE_TRI, 5, 6, &sipg::k_traces2d<SHAPE_TRI, 5, 6>});
  v.push_back(PlanesEntry{SHAPE_TRI, 6, 7, &sipg::k_traces2d<SHAPE_TRI, 6, 7>});
  v.push_back(PlanesEntry{SHAPE_TRI, 7, 8, &sipg::k_traces2d<SHAPE_TRI, 7, 8>});
  v.push_back(PlanesEntry{SHAPE_TRI, 8, 9, &sipg::k_traces2d<SHAPE_TRI, 8, 9>});
  v.push_back(PlanesEntry{SHAPE_TRI, 9, 10, &sipg::k_traces2d<SHAPE_TRI, 9, 10>});
  v.push_back(PlanesEntry{SHAPE_TRI, 10, 11, &sipg::k_traces2d<SHAPE_TRI, 10, 11>});
}
