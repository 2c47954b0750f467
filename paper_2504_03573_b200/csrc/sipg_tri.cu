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
