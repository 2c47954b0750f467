// Instantiations of the config-4 hybrid hex / prism / tet kernels (sipg_h3.cuh), n_modes 2..7.
#include <vector>
#include "sipg_h3.cuh"
#include "sipg_h3_registry.h"

namespace {
template <int S, int N>
H3Entry entry() {
  using C = h3::Cfg<S, N>;
  return H3Entry{S, N, &h3::k_h3<S, N, true>, &h3::k_h3<S, N, false>, h3::nthreads<N + 1>(), C::smem_bytes(true),
                 C::smem_bytes(false), &h3::h3_upload<S, N>};
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
}  // namespace

void sipg_register_h3(std::vector<H3Entry>& v) {
  add<H3_HEX>(v);
  add<H3_PRISM>(v);
  add<H3_TET>(v);
}
