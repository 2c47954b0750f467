// sm_100a kernels for hex elements (templates in sipg_kernels.cuh).
#include "sipg_kernels.cuh"
#include "sipg_hex_fast.cuh"
#include "sipg_hex_planes.cuh"
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
  SIPG_HEX_FAST(2);
  SIPG_HEX_FAST(3);
  SIPG_HEX_FAST(4);
  SIPG_HEX_FAST(5);
  SIPG_HEX_FAST(6);
  SIPG_HEX_FAST(7);
  SIPG_HEX_FAST(8);
  SIPG_HEX_FAST(9);
  SIPG_HEX_PLANES(2);
  SIPG_HEX_PLANES(3);
  SIPG_HEX_PLANES(4);
  SIPG_HEX_PLANES(5);
  SIPG_HEX_PLANES(6);
  SIPG_HEX_PLANES(7);
  SIPG_HEX_PLANES(8);
  SIPG_HEX_PLANES(9);
}

void sipg_register_planes(std::vector<PlanesEntry>& v) {
  v.push_back(PlanesEntry{SHAPE_HEX, 2, 3, &sipg::k_planes<2, 3>});
  v.push_back(PlanesEntry{SHAPE_HEX, 3, 4, &sipg::k_planes<3, 4>});
  v.push_back(PlanesEntry{SHAPE_HEX, 4, 5, &sipg::k_planes<4, 5>});
  v.push_back(PlanesEntry{SHAPE_HEX, 5, 6, &sipg::k_planes<5, 6>});
  v.push_back(PlanesEntry{SHAPE_HEX, 6, 7, &sipg::k_planes<6, 7>});
  v.push_back(PlanesEntry{SHAPE_HEX, 7, 8, &sipg::k_planes<7, 8>});
  v.push_back(PlanesEntry{SHAPE_HEX, 8, 9, &sipg::k_planes<8, 9>});
  v.push_back(PlanesEntry{SHAPE_HEX, 9, 10, &sipg::k_planes<9, 10>});
}
