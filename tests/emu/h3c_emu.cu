// TEST INFRASTRUCTURE ONLY (never linked into libsipg.so): runs the element body of the config-4
// register-column kernels (paper_2504_03573_b200/csrc/sipg_h3c.cuh) on the host, thread after thread
// between the barriers, on a flattened plan3d plan.  tests/test_h3c_emu.py compares it with the numpy
// emulation of the plan (oracle/h3_emulate.py) — indexing and phase-order bugs show up on CPU.
#define H3C_HOST_EMU 1
#include <cmath>
#include <cstring>
#include <vector>
#include "../../paper_2504_03573_b200/csrc/sipg_h3c.cuh"
#include "sipg.h"

namespace {
template <int Q>
void eo_build(const double* D, double* eo) {
  constexpr int H = Q / 2, EO = h3::eo_size<Q>();
  for (int t = 0; t < 2; ++t)
    for (int a = 0; a < 3; ++a) {
      const double* Da = D + a * Q * Q;
      auto M = [&](int k, int j) { return t == 0 ? Da[k * Q + j] : Da[j * Q + k]; };
      double* o = eo + (t * 3 + a) * EO;
      for (int k = 0; k < H; ++k)
        for (int j = 0; j < H; ++j) {
          o[k * H + j] = 0.5 * (M(k, j) + M(k, Q - 1 - j));
          o[H * H + k * H + j] = 0.5 * (M(k, j) - M(k, Q - 1 - j));
        }
      for (int k = 0; k < H; ++k) {
        o[2 * H * H + k] = (Q & 1) ? M(k, H) : 0.0;
        o[2 * H * H + H + k] = (Q & 1) ? M(H, k) : 0.0;
      }
    }
}

template <int S, int N>
void run_class(const H3Plan& P, const sipg_h3_desc* d, int cls, const double* x, double* y, int phases) {
  using C = h3c::CfgC<S, N>;
  using T = h3c::HostTabs<S, N>;
  constexpr int Q = N + 1;
  const int32_t* cd = d->class_desc + cls * CD3_WORDS;
  const double* tab = d->tables;
  constexpr int NA = S == H3_HEX ? N : N + 1;
  std::memcpy(T::A, tab + cd[CD3_T_A], sizeof(double) * Q * NA);
  if (S == H3_PRISM) std::memcpy(T::P, tab + cd[CD3_T_C], sizeof(double) * Q * N);
  eo_build<Q>(tab + cd[CD3_T_D], T::E);
  for (int i = 0; i < 6 * Q; ++i) {
    T::X[i] = tab[cd[CD3_T_E] + i];
    T::X[6 * Q + i] = tab[cd[CD3_T_ED] + i];
  }
  for (int k = 0; k < Q; ++k) {
    T::X[12 * Q + k] = 1.0 + tab[cd[CD3_T_PTS] + k];
    T::X[13 * Q + k] = tab[cd[CD3_T_W] + k];
  }
  const int G = 3;   // a few "CTAs": exercises the double-buffered element pipeline
  for (int b = 0; b < G; ++b) {
    // shared memory exactly as large as the kernel's (NaN-filled: reads of unwritten words show up)
    if (phases == 0) {
      std::vector<double> sm(C::smem_bytes(1) / 8 + 1, NAN);
      h3c::body<S, N, 1>(P, cls, x, y, b, G, sm.data());
    } else {
      std::vector<double> sm(C::smem_bytes(0) / 8 + 1, NAN);
      h3c::body<S, N, 0>(P, cls, x, y, b, G, sm.data());
    }
  }
}

template <int S>
bool dispatch_n(const H3Plan& P, const sipg_h3_desc* d, int cls, int n, const double* x, double* y, int phase) {
  switch (n) {
    case 2: run_class<S, 2>(P, d, cls, x, y, phase); return true;
    case 3: run_class<S, 3>(P, d, cls, x, y, phase); return true;
    case 4: run_class<S, 4>(P, d, cls, x, y, phase); return true;
    case 5: run_class<S, 5>(P, d, cls, x, y, phase); return true;
    case 6: run_class<S, 6>(P, d, cls, x, y, phase); return true;
    case 7: run_class<S, 7>(P, d, cls, x, y, phase); return true;
  }
  return false;
}
}  // namespace

// own-grid flux buffer layout (as sipg_h3_plan_create): fb_off[n_elements + 1], returns the total
extern "C" int64_t h3c_emu_fb_layout(const sipg_h3_desc* d, int64_t* fb_off) {
  std::vector<int32_t> q2(d->n_elements, 0);
  for (int c = 0; c < d->n_classes; ++c) {
    const int32_t* cd = d->class_desc + c * CD3_WORDS;
    for (int i = 0; i < cd[CD3_COUNT]; ++i) q2[d->class_elems[cd[CD3_ELEM_OFF] + i]] = cd[CD3_Q] * cd[CD3_Q];
  }
  fb_off[0] = 0;
  for (int64_t e = 0; e < d->n_elements; ++e)
    fb_off[e + 1] = fb_off[e] + 2ll * q2[e] * (d->slot_off[e + 1] - d->slot_off[e]);
  return fb_off[d->n_elements];
}

// phase 0: publish every class into pub; phase 3: the trace maps of the staged slots; phase 2: the fluxes of every class (reads pub) into fb;
// phase 1: apply every class (reads fb) into y
// u hand-over buffer layout (as sipg_h3_plan_create): ug_off[n_elements + 1], returns the total
extern "C" int64_t h3c_emu_ug_layout(const sipg_h3_desc* d, int64_t* ug_off) {
  std::vector<int64_t> q(d->n_elements, 0);
  for (int c = 0; c < d->n_classes; ++c) {
    const int32_t* cd = d->class_desc + c * CD3_WORDS;
    for (int i = 0; i < cd[CD3_COUNT]; ++i) q[d->class_elems[cd[CD3_ELEM_OFF] + i]] = cd[CD3_Q];
  }
  ug_off[0] = 0;
  for (int64_t e = 0; e < d->n_elements; ++e) ug_off[e + 1] = ug_off[e] + ((q[e] * q[e] * q[e] + 1) & ~1ll);
  return ug_off[d->n_elements];
}

extern "C" int h3c_emu_run(const sipg_h3_desc* d, const double* x, double* y, double* pub, double* fb,
                           const int64_t* fb_off, double* ug, const int64_t* ug_off, int phase) {
  // the flux kernel's work list, as sipg_h3_plan_create builds it
  std::vector<int32_t> qe(d->n_elements, 0);
  std::vector<H3FluxRec> fr;
  for (int c = 0; c < d->n_classes; ++c) {
    const int32_t* cd = d->class_desc + c * CD3_WORDS;
    for (int i = 0; i < cd[CD3_COUNT]; ++i) qe[d->class_elems[cd[CD3_ELEM_OFF] + i]] = cd[CD3_Q];
  }
  const H3Slot* sl = (const H3Slot*)d->slots;
  for (int64_t i = 0; i < d->n_elements; ++i) {
    const int32_t e = d->class_elems[i];
    for (int64_t q = d->slot_off[e]; q < d->slot_off[e + 1]; ++q) {
      const H3Slot& s0 = sl[q];
      fr.push_back(H3FluxRec{s0.pub_self, s0.pub_other, (fb_off[e] + 2ll * qe[e] * qe[e] * (q - d->slot_off[e])) * 16 + qe[e],
                             s0.tau, s0.sJ, s0.nt, s0.mkind | (s0.kind << 8), s0.nab, s0.moff, s0.moff2, s0.wtoff});
    }
  }
  std::vector<long long> es((size_t)d->n_elements * 6);
  for (int64_t i = 0; i < d->n_elements; ++i) {
    const int32_t e = d->class_elems[i];
    long long* r = es.data() + 6 * i;
    r[0] = e; r[1] = d->slot_off[e + 1] - d->slot_off[e]; r[2] = d->dof_off[e]; r[3] = d->slot_off[e];
    r[4] = fb_off[e]; r[5] = ug_off[e];
  }
  H3Plan P{d->class_desc, d->class_elems, d->dof_off, d->elem_geom, d->slot_off, (const H3Slot*)d->slots,
           d->tables, pub, d->lambda, fb, fb_off, fr.data(), ug, ug_off, es.data()};
  auto lanes = [&](auto&& f) { for (int lane = 0; lane < 32; ++lane) f(lane); };
  if (phase == 3) {   // the trace-map kernel, after the publish kernels (mapped slots)
    for (size_t i = 0; i < fr.size(); ++i) {
      if ((fr[i].mk_kind & 255) == MAP_ID) continue;
      std::vector<double> st(H3C_ST_MAP, NAN), tmp(2 * h3::TMAX, NAN);
      h3c::slot_stage<false>(P, fr[i], st.data(), lanes);
      h3c::map_compute(P, fr[i], st.data(), tmp.data(), lanes, [] {});
    }
    return 0;
  }
  if (phase == 2) {   // the flux kernels: identity-map slots streaming, mapped slots staged
    for (size_t i = 0; i < fr.size(); ++i) {
      if ((fr[i].mk_kind & 255) == MAP_ID) {
        h3c::flux_ident(P, (int64_t)i, lanes);
      } else {
        std::vector<double> st(H3C_ST_FLUX, NAN), tv(2 * h3::TMAX, NAN);
        h3c::slot_stage<true>(P, fr[i], st.data(), lanes);
        h3c::flux_compute(P, fr[i], st.data(), tv.data(), lanes, [] {});
      }
    }
    return 0;
  }
  for (int c = 0; c < d->n_classes; ++c) {
    const int32_t* cd = d->class_desc + c * CD3_WORDS;
    if (cd[CD3_COUNT] <= 0) continue;
    bool ok = false;
    if (cd[CD3_SHAPE] == H3_HEX) ok = dispatch_n<H3_HEX>(P, d, c, cd[CD3_N], x, y, phase);
    if (cd[CD3_SHAPE] == H3_PRISM) ok = dispatch_n<H3_PRISM>(P, d, c, cd[CD3_N], x, y, phase);
    if (cd[CD3_SHAPE] == H3_TET) ok = dispatch_n<H3_TET>(P, d, c, cd[CD3_N], x, y, phase);
    if (!ok) return 1;
  }
  return 0;
}
