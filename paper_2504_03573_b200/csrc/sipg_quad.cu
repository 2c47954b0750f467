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
