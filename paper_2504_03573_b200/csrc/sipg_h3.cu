// Instantiations of the config-4 hybrid hex / prism / tet kernels (sipg_h3c.cuh), n_modes 2..7, and
// the launchers of the slot kernels (trace maps, flux).
#include <vector>
#include "sipg_h3c.cuh"
#include "sipg_h3_registry.h"

namespace {
template <int S, int N>
H3Entry entry() {
  using C = h3c::CfgC<S, N>;
  return H3Entry{S, N, &h3c::k_h3c<S, N, 1>, &h3c::k_h3c<S, N, 0>, C::NTC, C::E, C::smem_bytes(1),
                 C::smem_bytes(0), &h3c::h3c_upload<S, N>};
}
template <int S>
void add(std::vector<H3Entry>& v) {
  v.push_back(entry<S, 2>());
  v.push_back(entry<S, 3>());
  v.push_back(entry<S, 4>());
  v.push_back(entry<S, 5>());
  v.push_back(entry<S, 6>());
  v.push_back(entry<S, 7>());
}

// persistent grid of the mapped-slot kernels: resident CTAs per SM x SMs (capped by the work)
template <bool FLUX>
unsigned slot_grid(int64_t count, int sms) {
  static int occ = 0;
  if (!occ) {
    cudaFuncSetAttribute(h3c::k_h3c_slot<FLUX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)h3c::h3c_slot_smem<FLUX>());
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, h3c::k_h3c_slot<FLUX>, 32 * H3C_SLOT_WPB,
                                                      h3c::h3c_slot_smem<FLUX>()) != cudaSuccess || occ <= 0)
      occ = 4;
  }
  const int64_t need = (count + H3C_SLOT_WPB - 1) / H3C_SLOT_WPB, cap = (int64_t)occ * sms;
  return (unsigned)(need < cap ? need : cap);
}
}  // namespace

void sipg_register_h3(std::vector<H3Entry>& v) {
  add<H3_HEX>(v);
  add<H3_PRISM>(v);
  add<H3_TET>(v);
}

void sipg_h3c_flux_launch(const H3Plan& P, int64_t first, int64_t count, bool mapped, int sms, cudaStream_t stream) {
  if (count <= 0) return;
  if (mapped)
    h3c::k_h3c_slot<true><<<slot_grid<true>(count, sms), 32 * H3C_SLOT_WPB, h3c::h3c_slot_smem<true>(), stream>>>(P, first, count);
  else
    h3c::k_h3c_flux_id<<<(unsigned)((count + 7) / 8), 256, 0, stream>>>(P, first, count);
}

void sipg_h3c_map_launch(const H3Plan& P, int64_t first, int64_t count, int sms, cudaStream_t stream) {
  if (count <= 0) return;
  h3c::k_h3c_slot<false><<<slot_grid<false>(count, sms), 32 * H3C_SLOT_WPB, h3c::h3c_slot_smem<false>(), stream>>>(P, first, count);
}
