// sm_100a kernels for hex elements (templates in sipg_kernels.cuh).
#include "sipg_kernels.cuh"
#include "sipg_hex_fast.cuh"
#include "sipg_hex_mma.cuh"
#include "sipg_hex_warp.cuh"
#include "sipg_registry.h"
SIPG_DEFINE_ENTRY
void sipg_register_hex(std::vector<KernelEntry>& v) {
  SIPG_ENTRIES_NQ(SHAPE_HEX, 2);
  SIPG_ENTRIES_NQ(SHAPE_HEX, 3);
  SIPG_ENTRIES_NQ(SHAPE_HEX, 4);
  SIPG_ENTRIES_NQ(SHAPE_HEX, 5);
  SIPG_ENTRIES_NQ(SHAPE_HEX, 6);
  SIPG_ENTRIES_NQ(SHAPE_HEX, 7);
  SIPG_ENTRIES_NQ(SHAPE_HEX, 8);
  SIPG_ENTRIES_NQ(SHAPE_HEX, 9);
  SIPG_HEX_MMA(2);
  SIPG_HEX_MMA(3);
  SIPG_HEX_MMA(4);
  SIPG_HEX_MMA(5);
  SIPG_HEX_MMA(6);
  SIPG_HEX_MMA(7);
  SIPG_HEX_FAST(8);
  SIPG_HEX_FAST(9);
}
