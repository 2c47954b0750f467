// Config 4: the SIP-Helmholtz apply on 3-D hybrid hex / prism / tet meshes (sm_100a, fp64) -- the
// reference's two-phase apply (pkg/src/dgsipg/sipg.py:558-602) on the shared-trace route
// (sipg.py:513-554, 653-677), extended to prisms and tets as restated in oracle/hybrid3d.py; plan
// layout: paper_2504_03573_b200/plan3d.py, shared definitions: sipg_h3.cuh.  The first generation of
// these kernels (round 1) kept four q^3 arrays per element in shared memory and ran at 85 % of the
// shared-memory data pipe's wavefront peak (ncu); this generation is organised around registers:
//   * one CTA of q^2 threads per element; thread (k1, k2) owns the q points (., k1, k2) along eta0 in
//     REGISTERS: the last BwdTrans stage, PhysDeriv along eta0, the volume terms, every face lift,
//     D0^T and the first IProduct stage never touch shared memory;
//   * eta1 / eta2 derivatives are one line per thread through two (bank-padded) q^3 buffers,
//     even-odd factorised with __constant__ operands;
//   * three kernels per class.  publish: own traces (u, n.grad u) of every coupling at its trace
//     points.  flux: the SIP flux of every coupling from the published own and partner traces and
//     the transposed trace maps back onto the own face grid (the reference's per-interface phase 2,
//     sipg.py:607-661) -- all the irregular, DRAM-latency-bound work, in a kernel that needs few
//     registers and runs at full occupancy.  apply: the element-local work; the own-grid fluxes
//     arrive by cp.async behind BwdTrans / PhysDeriv and are lifted straight into the register
//     columns, faces compile-time unrolled (one-hot GLL endpoint rows touch the boundary columns only);
//   * the publish kernel takes u and d/d eta_fixed on the faces from the register columns (eta0
//     faces) or from one line read per thread (eta1 / eta2 faces) and the tangential derivatives as
//     even-odd lines on the face grids.
// The element body is written against a tiny execution abstraction (par / sync) so that the very
// same code runs on the host, thread after thread, in the CPU test of the kernel logic
// (tests/emu, -DH3C_HOST_EMU; test infrastructure, not part of libsipg.so).
#pragma once
#include <type_traits>
#include "sipg_h3.cuh"

#ifdef H3C_HOST_EMU
#define H3C_HD __host__ __device__ __forceinline__
#else
#define H3C_HD __device__ __forceinline__
#endif
#if defined(__CUDA_ARCH__)
#define H3C_LDG(p) __ldg(p)
#else
#define H3C_LDG(p) (*(p))
#endif

// build knobs (measured variants, tools/h3c_variants.sh)
#ifndef H3C_MAP_U8
#define H3C_MAP_U8 1        // transposed-map contractions: eight predicated, unrolled steps
#endif
#ifndef H3C_ITEM_U
#define H3C_ITEM_U 0        // ragged tet stages: item loops unrolled (measured slower: spills)
#endif
#ifndef H3C_PACK
#define H3C_PACK 1          // several elements per CTA (teams of q^2 threads) so that the warps are full
#endif
#ifndef H3C_E5
#define H3C_E5 5
#endif
#ifndef H3C_E6
#define H3C_E6 7
#endif
#ifndef H3C_E7
#define H3C_E7 5
#endif
#ifndef H3C_E8
#define H3C_E8 1
#endif
#ifndef H3C_TET_FUSE1
#define H3C_TET_FUSE1 1     // tets: the ragged eta2 stage recomputed per thread inside the fused register stage
#endif
#if H3C_MAP_U8
#define H3C_MAPLOOP(i, n) _Pragma("unroll") for (int i = 0; i < 8; ++i) if (i < (n))
#else
#define H3C_MAPLOOP(i, n) for (int i = 0; i < (n); ++i)
#endif
#if H3C_ITEM_U
#define H3C_ITEM_UNROLL _Pragma("unroll")
#else
#define H3C_ITEM_UNROLL _Pragma("unroll 1")
#endif
#ifndef SIPG_H3C_MINB8
#define SIPG_H3C_MINB8 7            // resident CTAs per SM the registers must allow, q = 8 (64 threads)
#endif

namespace h3c {
using h3::Chain;
using h3::TMAX;

// E | ED endpoint rows (6 q each, row (axis * 2 + (side > 0))), 1 + eta0 points, eta0 weights
template <int S, int N> __constant__ double c3X[14 * (N + 1)];

#ifdef H3C_HOST_EMU
template <int S, int N>
struct HostTabs {
  static double A[(N + 1) * (N + 1)], P[(N + 1) * N], E[6 * h3::eo_size<N + 1>()], X[14 * (N + 1)];
};
template <int S, int N> double HostTabs<S, N>::A[(N + 1) * (N + 1)];
template <int S, int N> double HostTabs<S, N>::P[(N + 1) * N];
template <int S, int N> double HostTabs<S, N>::E[6 * h3::eo_size<N + 1>()];
template <int S, int N> double HostTabs<S, N>::X[14 * (N + 1)];
#endif
#if defined(__CUDA_ARCH__) || !defined(H3C_HOST_EMU)
#define H3C_TA (h3::c3A<S, N>)
#define H3C_TP (h3::c3P<S, N>)
#define H3C_TE (h3::c3E<S, N>)
#define H3C_TX (c3X<S, N>)
#else
#define H3C_TA (HostTabs<S, N>::A)
#define H3C_TP (HostTabs<S, N>::P)
#define H3C_TE (HostTabs<S, N>::E)
#define H3C_TX (HostTabs<S, N>::X)
#endif

// (fixed axis, side, run axis 0, run axis 1) per shape and local face (plan3d.FACES)
H3C_HD constexpr int fc(int S, int f, int w) {
  constexpr int T[3][6][4] = {
      {{0, -1, 1, 2}, {0, 1, 1, 2}, {1, -1, 0, 2}, {1, 1, 0, 2}, {2, -1, 0, 1}, {2, 1, 0, 1}},
      {{2, -1, 0, 1}, {1, -1, 0, 2}, {0, 1, 1, 2}, {1, 1, 0, 2}, {0, -1, 1, 2}, {0, 0, 0, 0}},
      {{2, -1, 0, 1}, {1, -1, 0, 2}, {0, 1, 1, 2}, {0, -1, 1, 2}, {0, 0, 0, 0}, {0, 0, 0, 0}},
  };
  return T[S][f][w];
}
// the same for a run-time face: the __constant__ copy on the device (no per-thread table)
H3C_HD int fcr(int S, int f, int w) {
#if defined(__CUDA_ARCH__)
  return h3::c_faces[S][f][w];
#else
  return fc(S, f, w);
#endif
}
// GLL axes (endpoint rows one-hot): hex all, prism eta1 (plan3d.AXIS_KINDS)
H3C_HD constexpr bool gll_axis(int S, int a) { return S == H3_HEX || (S == H3_PRISM && a == 1); }

template <int S>
H3C_HD Chain chain_t(double p0, double p1, double r1, double r2) {
  Chain c{1.0, 0.0, 0.0, 1.0, 0.0};
  if (S == H3_PRISM) {
    c.c00 = 2.0 * r2;
    c.c02 = p0 * r2;
  } else if (S == H3_TET) {
    const double r12 = r1 * r2;
    c.c00 = 4.0 * r12;
    c.c01 = c.c02 = 2.0 * p0 * r12;
    c.c11 = 2.0 * r2;
    c.c12 = p1 * r2;
  }
  return c;
}
// chain at own-face-grid point (ia, ib) of a face (h3::face_chain)
template <int S>
H3C_HD Chain face_chain(const double* pts, const double* R, int Q, int fx, int sd, int ra, int rb, int ia, int ib) {
  if (S == H3_HEX) return Chain{1.0, 0.0, 0.0, 1.0, 0.0};
  const double ea = *(pts + ra * Q + ia), eb = *(pts + rb * Q + ib);
  const double rra = *(R + ra * Q + ia), rrb = *(R + rb * Q + ib);
  const double es = (double)sd, rs = sd < 0 ? 0.5 : 0.0;
  const double e0 = fx == 0 ? es : (ra == 0 ? ea : eb);
  const double e1 = fx == 1 ? es : (ra == 1 ? ea : eb);
  const double r1 = fx == 1 ? rs : (ra == 1 ? rra : rrb);
  const double r2 = fx == 2 ? rs : (ra == 2 ? rra : rrb);
  return chain_t<S>(1.0 + e0, 1.0 + e1, r1, r2);
}

H3C_HD const H3Slot& slot_hdr(const double* hdr, int s) { return *reinterpret_cast<const H3Slot*>(hdr + 12 * s); }

// items of a batch of <= 4 slots (h3::Batch)
struct Batch {
  int b0, o1, o2, o3, tot;
  template <typename CountFn>
  H3C_HD Batch(int b0_, int nb, CountFn cnt) : b0(b0_) {
    const int c0 = nb > 0 ? cnt(b0) : 0;
    const int c1 = nb > 1 ? cnt(b0 + 1) : 0;
    const int c2 = nb > 2 ? cnt(b0 + 2) : 0;
    const int c3 = nb > 3 ? cnt(b0 + 3) : 0;
    o1 = c0;
    o2 = o1 + c1;
    o3 = o2 + c2;
    tot = o3 + c3;
  }
  H3C_HD int slot(int& it) const {
    const int j = (it >= o1) + (it >= o2) + (it >= o3);
    it -= j == 0 ? 0 : (j == 1 ? o1 : (j == 2 ? o2 : o3));
    return b0 + j;
  }
};

// full even-odd line: out = M in for the operator block at T[off] (Pe | Po | mc | mr, sipg_h3.cuh)
template <int Q, typename Tab>
H3C_HD void eo_full(const Tab& T, const int off, const double (&in)[Q], double (&out)[Q]) {
  constexpr int H = Q / 2;
  double sm[H > 0 ? H : 1], df[H > 0 ? H : 1];
#pragma unroll
  for (int j = 0; j < H; ++j) {
    sm[j] = in[j] + in[Q - 1 - j];
    df[j] = in[j] - in[Q - 1 - j];
  }
#pragma unroll
  for (int k = 0; k < H; ++k) {
    double e = 0.0, o = 0.0;
#pragma unroll
    for (int j = 0; j < H; ++j) {
      e = fma(T[off + k * H + j], sm[j], e);
      o = fma(T[off + H * H + k * H + j], df[j], o);
    }
    if (Q & 1) e = fma(T[off + 2 * H * H + k], in[H], e);
    out[k] = e + o;
    out[Q - 1 - k] = o - e;
  }
  if (Q & 1) {
    double m = 0.0;
#pragma unroll
    for (int j = 0; j < H; ++j) m = fma(T[off + 2 * H * H + H + j], df[j], m);
    out[H] = m;
  }
}

template <int K, int J, typename Tab>
H3C_HD void cmat(const Tab& M, const int off, const double (&in)[J], double (&out)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double a = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) a = fma(M[off + k * J + j], in[j], a);
    out[k] = a;
  }
}
template <int K, int J, typename Tab>
H3C_HD void cmatT(const Tab& M, const int off, const double (&in)[K], double (&out)[J]) {
#pragma unroll
  for (int j = 0; j < J; ++j) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) a = fma(M[off + k * J + j], in[k], a);
    out[j] = a;
  }
}

template <int S, int N>
struct CfgC {
  static constexpr int Q = N + 1, Q2 = Q * Q, NT = Q2;   // NT: threads of one element (its team)
  // elements (teams) per CTA: q^2 threads each, packed without padding so the warps are full
  // (q = 6: 36 threads would leave a 4-lane second warp; seven elements fill 252 of 256 lanes)
  static constexpr int E = H3C_PACK ? (Q <= 3 ? 3 : (Q == 4 ? 2 : (Q == 5 ? H3C_E5 : (Q == 6 ? H3C_E6 : (Q == 7 ? H3C_E7 : H3C_E8))))) : 1;
  static constexpr int NTC = E * NT;                     // CTA threads
  static constexpr int SJ = (Q & 1) ? Q : Q + 1, SI = Q * SJ, BUF = Q * SI;   // odd row stride
  static constexpr int NF = S == H3_HEX ? 6 : (S == H3_PRISM ? 5 : 4);
  static constexpr int NTRI = N * (N + 1) / 2, NG = N + 1;
  static constexpr int NPM = NTRI + (S == H3_TET ? 1 : 0);
  static constexpr int NA = S == H3_HEX ? N : N + 1;
  static constexpr int NC = S == H3_HEX ? N * N * N : (S == H3_PRISM ? N * NTRI : N * (N + 1) * (N + 2) / 6);
  static constexpr int NCP = (NC + 1) & ~1;
  static constexpr int S1 = S == H3_HEX ? N * N * Q : NPM * Q;
  static constexpr int NSMAX = S == H3_HEX ? 12 : (S == H3_PRISM ? 8 : 4);
  static constexpr int SLOTD = 12;
  static constexpr int SB = 4;                                  // slots per map batch
  static constexpr int TB = S == H3_HEX ? 0 : NPM * Q;
  static constexpr int NCD = S == H3_TET ? N * (N - 1) / 2 + 1 : 0;            // distinct eta2 rows of a tet class
  static constexpr int TABD = (3 * Q + 3 * Q + Q2 + 6 * Q + TB + NCD * Q + 1) & ~1;   // pts R W12 E B Cd
  static constexpr int imax(int a, int b) { return a > b ? a : b; }
  static constexpr int SCR_P = (BUF + S1 + 1) & ~1;                            // publish: u, s1
  static constexpr int FBN = NSMAX * 2 * Q2;                                   // own-grid fluxes of an element
  static constexpr int NI = 2 * NPM + 2 + NC + NCD + 8;   // gof, minfo, rinfo, cdrep
  // kernel modes: 0 apply, 1 publish.  Shared memory: ring | class tables | one block per team | int tables
  static constexpr int RING = (3 * E * 6 + 1) & ~1;
  static constexpr int UBP = (Q2 * Q + 1) & ~1;                                // apply: the element's u, q^3 (unpadded)
  static constexpr int teamd(int mode) {
    return mode == 1 ? 2 * NCP + 2 * NSMAX * SLOTD + NF * 4 * Q2 + SCR_P
                     : (H3C_UHAND ? UBP : 2 * NCP) + 2 * NSMAX * SLOTD + 2 * H3_EGEO + FBN + 2 * BUF;   // every term even
  }
  static constexpr int doubles(int mode) { return RING + TABD + E * teamd(mode); }
  static constexpr size_t smem_bytes(int mode) { return sizeof(double) * doubles(mode) + sizeof(int) * NI; }
};

// triangle pseudo-mode -> group (row 0 -> 0 except (0,1) -> 1, row 1 -> 2, row i >= 2 -> i + 1; the tet apex
// pseudo-mode -> 1), and for tets the packed tables of the ragged eta2 stage.  The eta2 functions of a
// tet mode (i, j, k) depend on the triangle mode's degree d = max(i + j, 1) and on k only
// (plan3d.collapse_rows), so the class's C table (n_c x q) is kept as its n (n - 1) / 2 + 1 distinct
// rows: cdrep[row] = a row of the plan's table holding it, minfo[m] = first mode | count << 8 | first
// distinct row << 16, rinfo[r] = triangle pseudo-mode | distinct row << 8.  By one thread.
template <int S, int N>
H3C_HD void build_int_tables(int* gof, int* minfo, int* rinfo, int* cdrep) {
  using C = CfgC<S, N>;
  int m = 0;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N - i; ++j, ++m) gof[m] = i == 0 ? (j == 1 ? 1 : 0) : (i == 1 ? 2 : i + 1);
  if (S == H3_TET) {
    gof[C::NTRI] = 1;
    int doff[N + 1];
    doff[1] = 0;
    for (int d = 1; d < N; ++d) doff[d + 1] = doff[d] + (N - d);
    int r = 0, mm = 0;
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N - i; ++j, ++mm) {
        const int d = (i + j) > 1 ? i + j : 1;
        minfo[mm] = r | ((N - d) << 8) | (doff[d] << 16);
        for (int k = 0; k < N - d; ++k) {
          cdrep[doff[d] + k] = r;
          rinfo[r++] = mm | ((doff[d] + k) << 8);
        }
      }
    minfo[C::NTRI] = r | (1 << 8) | (doff[N] << 16);   // apex: one mode, the last distinct row
    cdrep[doff[N]] = r;
    rinfo[r] = C::NTRI | (doff[N] << 8);
  }
}

// compile-time loop over the local faces
template <int F0, int F1, typename Fn>
H3C_HD void for_faces(Fn&& fn) {
  if constexpr (F0 < F1) {
    fn(std::integral_constant<int, F0>{});
    for_faces<F0 + 1, F1>(fn);
  }
}

template <int S, int N, int MODE>
H3C_HD void body(const H3Plan& P, const int cls, const double* __restrict__ x, double* __restrict__ y, const int bid,
                 const int G, double* sm) {
  using C = CfgC<S, N>;
  constexpr bool PUB = MODE == 1, APP = MODE == 0;
  constexpr int Q = C::Q, Q2 = C::Q2, NT = C::NT, SJ = C::SJ, SI = C::SI, BUF = C::BUF, NF = C::NF, SB = C::SB;
  constexpr int EOS = h3::eo_size<Q>(), NA = C::NA;
  constexpr int XE = 0, XED = 6 * Q, XP0 = 12 * Q, XW0 = 13 * Q;   // c3X sections
  struct TS {
    double u[Q], d0[Q], d1[Q], d2[Q];
  };
#if defined(__CUDA_ARCH__) || !defined(H3C_HOST_EMU)
  TS ts_;
  auto par = [&](auto&& f) { f((int)threadIdx.x, ts_); };
  auto sync = [&]() { __syncthreads(); };
#else
  static thread_local TS tsa[C::NTC];
  auto par = [&](auto&& f) {
    for (int lt = 0; lt < C::NTC; ++lt) f(lt, tsa[lt]);
  };
  auto sync = [&]() {};
#endif
  // ---- shared memory (CfgC::doubles): ring | class tables | team blocks | int tables
  constexpr int E = C::E, NTC = C::NTC, TEAMD = C::teamd(MODE);
  long long* ring = reinterpret_cast<long long*>(sm);                  // [3][E][6] element scalars (e, ns, dof, sb, fbo, ugo)
  double* pts = sm + C::RING;
  double* Rt = pts + 3 * Q;
  double* W12 = Rt + 3 * Q;
  double* Et = W12 + Q2;
  double* Bt = Et + 6 * Q;
  double* Cd = Bt + C::TB;                                          // tets: distinct eta2 rows [NCD][Q]
  double* teams = sm + C::RING + C::TABD;
  // per team (element): coefficients [2][NCP] | slot headers [2][NSMAX][12] | apply: geometry [2][8], own-grid
  // fluxes [ns][2][Q2], B0, B1 (padded q^3 buffers; BwdTrans s2, s1) | publish: face arrays [NF][4][Q2], u, s1
  constexpr bool UH = APP && H3C_UHAND;   // apply: u arrives from the publish kernel (one q^3 buffer, no coefficients)
  constexpr int O_H = UH ? C::UBP : 2 * C::NCP, O_E = O_H + 2 * C::NSMAX * C::SLOTD, O_F = O_E + 2 * H3_EGEO;
  constexpr int O_B0 = APP ? O_F + C::FBN : O_E + NF * 4 * Q2;
  int* gof = reinterpret_cast<int*>(teams + E * TEAMD);
  int* minfo = gof + C::NPM + 1;
  int* rinfo = minfo + C::NPM + 1;
  int* cdrep = rinfo + C::NC + 1;
  // a thread's team (element) and its buffers: the first statement of every element-work phase
#define H3C_TEAM(ltc)                                                                  \
  const int tm = (ltc) / NT, lt = (ltc) - tm * NT;                                     \
  const long long* rg_ = ring + 6 * (slot * E + tm);                                   \
  const int ns = (int)rg_[1];                                                          \
  if (ns < 0) return;                                                                  \
  const int64_t dof = rg_[2], fbo = rg_[4], ugo = rg_[5];                              \
  double* tmb_ = teams + tm * TEAMD;                                                    \
  const double* c = tmb_ + bsel * C::NCP;                                               \
  const double* hdr = tmb_ + O_H + bsel * C::NSMAX * C::SLOTD;                          \
  const double* eg = tmb_ + O_E + bsel * H3_EGEO;                                       \
  double* fbuf = tmb_ + O_F;                                                            \
  double* FL = tmb_ + O_E;                                                              \
  double* B0 = tmb_ + O_B0;                                                             \
  double* B1 = B0 + BUF;                                                               \
  double* s2 = B0;                                                                     \
  double* s1 = B0 + BUF;                                                               \
  (void)dof; (void)fbo; (void)ugo; (void)c; (void)hdr; (void)eg; (void)fbuf; (void)FL; (void)B1; (void)s2; (void)s1; (void)lt

  const int32_t* cd = P.cd + cls * CD3_WORDS;
  const int count = cd[CD3_COUNT];
  const double* tab = P.tab;
  const double* Ct = S == H3_TET ? tab + cd[CD3_T_C] : tab;
  {
    par([&](int lt, TS&) {
      auto cp = [&](double* dst, const double* src, int n) {
        for (int r = lt; r < n; r += NTC) dst[r] = H3C_LDG(src + r);
      };
      cp(pts, tab + cd[CD3_T_PTS], 3 * Q);
      cp(Rt, tab + cd[CD3_T_R], 3 * Q);
      cp(W12, tab + cd[CD3_T_W] + Q, Q2);
      cp(Et, tab + cd[CD3_T_E], 6 * Q);
      if (S != H3_HEX) cp(Bt, tab + cd[CD3_T_B], C::TB);
      if (S != H3_HEX && lt == 0) build_int_tables<S, N>(gof, minfo, rinfo, cdrep);
    });
    if (S == H3_TET) {
      sync();
      par([&](int lt, TS&) {
        for (int r = lt; r < C::NCD * Q; r += NTC) Cd[r] = H3C_LDG(Ct + cdrep[r / Q] * Q + r % Q);
      });
    }
  }

  // ---- element pipeline: scalars two elements ahead; coefficients + slot headers + geometry one
  // element ahead (cp.async into the other buffer); apply: the element's own-grid fluxes (written by
  // the flux kernel) at the top of the element, consumed after BwdTrans / PhysDeriv
  const int32_t* ce = P.class_elems + cd[CD3_ELEM_OFF];
  // element scalars through a 3-deep ring in shared memory (one thread loads them two elements ahead;
  // nothing of the pipeline is carried in registers)
  // group gi of the class list = elements gi E .. gi E + E - 1, one per team (ns = -1: none)
  auto scalars = [&](int gi, int slot) {
    par([&](int lt, TS&) {
      if (lt < E) {
        const int i = gi * E + lt;
        long long* r = ring + 6 * (slot * E + lt);
        if (i < count) {
          const long long* src = P.escal + 6 * (long long)(cd[CD3_ELEM_OFF] + i);
#if defined(__CUDA_ARCH__)
          __pipeline_memcpy_async(r, src, 16);
          __pipeline_memcpy_async(r + 2, src + 2, 16);
          __pipeline_memcpy_async(r + 4, src + 4, 16);
#else
          for (int q = 0; q < 6; ++q) r[q] = src[q];
#endif
        } else {
          r[1] = -1;
        }
      }
#if defined(__CUDA_ARCH__)
      __pipeline_commit();
#endif
    });
  };
  auto issue = [&](int buf, int slot, bool on) {   // coefficients (not with the u hand-over), slot headers, geometry
    par([&](int ltc, TS&) {
      const int tm = ltc / NT, lt = ltc - tm * NT;
      const long long* r = ring + 6 * (slot * E + tm);
      const int e = (int)r[0], ns = on ? (int)r[1] : -1;
      const int64_t dof = r[2], sb = r[3];
      double* tb_ = teams + tm * TEAMD;
      double* cd_ = tb_ + buf * C::NCP;
      double* hd_ = tb_ + O_H + buf * C::NSMAX * C::SLOTD;
      double* eb_ = tb_ + O_E + buf * H3_EGEO;
      const double* src = reinterpret_cast<const double*>(P.slots + sb);
#if defined(__CUDA_ARCH__)
      if (ns >= 0) {
        if (!UH)
          for (int r = lt; r < C::NC; r += NT) __pipeline_memcpy_async(cd_ + r, x + dof + r, sizeof(double));
        for (int r = lt; r < ns * C::SLOTD; r += NT) __pipeline_memcpy_async(hd_ + r, src + r, sizeof(double));
        if (APP && lt < H3_EGEO / 2)
          __pipeline_memcpy_async(eb_ + 2 * lt, P.egeo + (int64_t)e * H3_EGEO + 2 * lt, 2 * sizeof(double));
      }
      __pipeline_commit();
#else
      if (ns >= 0) {
        if (!UH)
          for (int r = lt; r < C::NC; r += NT) cd_[r] = x[dof + r];
        for (int r = lt; r < ns * C::SLOTD; r += NT) hd_[r] = src[r];
        if (APP && lt < H3_EGEO / 2) {
          eb_[2 * lt] = P.egeo[(int64_t)e * H3_EGEO + 2 * lt];
          eb_[2 * lt + 1] = P.egeo[(int64_t)e * H3_EGEO + 2 * lt + 1];
        }
      }
#endif
    });
  };
  auto issue_u = [&](int slot, bool on) {   // the element's u (q^3 doubles, ug_off even: 16-byte pieces; odd tail 8)
    par([&](int ltc, TS&) {
      const int tm = ltc / NT, lt = ltc - tm * NT;
      const long long* r = ring + 6 * (slot * E + tm);
      const int ns = on ? (int)r[1] : -1;
      const double* src = P.ug + r[5];
      double* ub = teams + tm * TEAMD;
      constexpr int Q3 = Q2 * Q;
#if defined(__CUDA_ARCH__)
      if (ns >= 0) {
        for (int q = lt; q < Q3 / 2; q += NT) __pipeline_memcpy_async(ub + 2 * q, src + 2 * q, 2 * sizeof(double));
        if ((Q3 & 1) && lt == 0) __pipeline_memcpy_async(ub + Q3 - 1, src + Q3 - 1, sizeof(double));
      }
      __pipeline_commit();
#else
      if (ns >= 0)
        for (int q = lt; q < Q3; q += NT) ub[q] = src[q];
#endif
    });
  };
  auto issue_fb = [&](int slot) {   // ns * 2 * Q2 doubles per team, 16-byte pieces (fb_off is even)
    par([&](int ltc, TS&) {
      const int tm = ltc / NT, lt = ltc - tm * NT;
      const long long* r = ring + 6 * (slot * E + tm);
      const int ns = (int)r[1];
      const double* src = P.fb + r[4];
      double* fbuf = teams + tm * TEAMD + O_F;
#if defined(__CUDA_ARCH__)
      for (int q = lt; q < ns * Q2; q += NT) __pipeline_memcpy_async(fbuf + 2 * q, src + 2 * q, 2 * sizeof(double));
      __pipeline_commit();
#else
      for (int q = lt; q < ns * 2 * Q2; q += NT) fbuf[q] = src[q];
#endif
    });
  };
  const int ngroups = (count + E - 1) / E;
  scalars(bid, 0);
  scalars(bid + G, 1);
#if defined(__CUDA_ARCH__)
  __pipeline_wait_prior(0);
#endif
  sync();
  issue(0, 0, bid < ngroups);
  if (UH) issue_u(0, bid < ngroups);
  int it_el = 0;
  for (int gi = bid; gi < ngroups; gi += G, ++it_el) {
    const int bsel = it_el & 1;
    const int slot = it_el % 3, slot_n = (it_el + 1) % 3, slot_nn = (it_el + 2) % 3;
#if defined(__CUDA_ARCH__)
    __pipeline_wait_prior(0);
#endif
    sync();
    issue(bsel ^ 1, slot_n, gi + G < ngroups);
    scalars(gi + 2 * G, slot_nn);
    if (APP) issue_fb(slot);

    if (UH) {
      // ================= apply with the u hand-over: the column from the publish kernel's u ==========
      par([&](int ltc, TS& ts) {
        H3C_TEAM(ltc);
        const int ta = lt / Q, tb_ = lt % Q;
        const double* ub = tmb_;
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          ts.u[k] = ub[k * Q2 + lt];
          B0[k * SI + ta * SJ + tb_] = ts.u[k];
        }
        eo_full<Q>(H3C_TE, 0 * EOS, ts.u, ts.d0);
      });
      sync();
      issue_u(slot_n, gi + G < ngroups);   // the u buffer is free again: the next element's u, a whole element ahead
    } else {
    // ================= BwdTrans (stdregions.py:575-597): u column in registers ====================
    if (S == H3_HEX) {
      par([&](int ltc, TS&) {
        H3C_TEAM(ltc);
        if (lt < N * N) {                      // (i0, i1): i2 -> k2
          double col[N], out[Q];
#pragma unroll
          for (int i = 0; i < N; ++i) col[i] = c[lt * N + i];
          cmat<Q, N>(H3C_TA, 0, col, out);
#pragma unroll
          for (int k = 0; k < Q; ++k) s1[lt * Q + k] = out[k];
        }
      });
      sync();
      par([&](int ltc, TS&) {
        H3C_TEAM(ltc);
        if (lt < N * Q) {                      // (i0, k2): i1 -> k1
          const int i0 = lt / Q, k2 = lt % Q;
          double col[N], out[Q];
#pragma unroll
          for (int i = 0; i < N; ++i) col[i] = s1[(i0 * N + i) * Q + k2];
          cmat<Q, N>(H3C_TA, 0, col, out);
#pragma unroll
          for (int k = 0; k < Q; ++k) s2[i0 * SI + k * SJ + k2] = out[k];
        }
      });
      sync();
    } else if (S == H3_PRISM || !H3C_TET_FUSE1) {
      // stage 1: the innermost family (prism: psi on eta1 per triangle mode; tet: C rows on eta2)
      par([&](int ltc, TS&) {
        H3C_TEAM(ltc);
        if (S == H3_PRISM) {
          for (int m = lt; m < C::NPM; m += NT) {
            double col[N], out[Q];
#pragma unroll
            for (int l = 0; l < N; ++l) col[l] = c[m * N + l];
            cmat<Q, N>(H3C_TP, 0, col, out);
#pragma unroll
            for (int k = 0; k < Q; ++k) s1[m * Q + k] = out[k];
          }
        } else {
          H3C_ITEM_UNROLL
          for (int rr = 0; rr < (C::NPM * Q + NT - 1) / NT; ++rr) {
            const int o = lt + rr * NT;
            if (o < C::NPM * Q) {
              const int k = o % Q, m = o / Q;
              double a = 0.0;
              const int inf = minfo[m], r0 = inf & 255, cn = (inf >> 8) & 255;
              const double* Cr = Cd + (inf >> 16) * Q + k;
#pragma unroll
              for (int kk = 0; kk < (N - 1 > 1 ? N - 1 : 1); ++kk)
                if (kk < cn) a = fma(Cr[kk * Q], c[r0 + kk], a);
              s1[o] = a;
            }
          }
        }
      });
      sync();
    }
    // last stages, in registers: thread (k1, k2) sums every triangle mode's B x s1 product into its
    // group's accumulator (compile-time mode -> group map, no shared-memory s2) and applies A along eta0
    par([&](int ltc, TS& ts) {
      H3C_TEAM(ltc);
      const int ta = lt / Q, tb_ = lt % Q;
      double col[NA];
      if (S == H3_HEX) {
#pragma unroll
        for (int g = 0; g < NA; ++g) col[g] = s2[g * SI + ta * SJ + tb_];
      } else {
        // prism: B on eta2, s1 over eta1; tet: B on eta1, s1 over eta2
        const double* Bk = Bt + (S == H3_PRISM ? tb_ : ta);
        const double* sk = s1 + (S == H3_PRISM ? ta : tb_);
#pragma unroll
        for (int g = 0; g < NA; ++g) col[g] = 0.0;
        int m = 0, r = 0;
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int j = 0; j < N - i; ++j, ++m) {
            const int g = i == 0 ? (j == 1 ? 1 : 0) : (i == 1 ? 2 : i + 1);
            if (S == H3_TET && H3C_TET_FUSE1) {
              // s1[m][k2] = sum_k Cd[d][k][k2] c[r + k] on the fly (every index a compile-time constant;
              // c is a broadcast read): no ragged item loop, no barrier, q-fold redundant but short
              const int d = (i + j) > 1 ? i + j : 1, cn = N - d, row = (d - 1) * (2 * N - d) / 2;
              double sv = 0.0;
#pragma unroll
              for (int k = 0; k < cn; ++k) sv = fma(Cd[(row + k) * Q + tb_], c[r + k], sv);
              r += cn;
              col[g] = fma(Bk[m * Q], sv, col[g]);
            } else {
              col[g] = fma(Bk[m * Q], sk[m * Q], col[g]);
            }
          }
        if (S == H3_TET) {   // apex pseudo-mode
          const double sv = H3C_TET_FUSE1 ? Cd[(C::NCD - 1) * Q + tb_] * c[r] : sk[C::NTRI * Q];
          col[1] = fma(Bk[C::NTRI * Q], sv, col[1]);
        }
      }
      cmat<Q, NA>(H3C_TA, 0, col, ts.u);
    });

    }   // BwdTrans (not with the u hand-over)

    if (PUB) {
      // ================= publish: own traces (u, n.grad u) of every coupling =====================
      // FL[f] = (u, d u / d eta_fixed, d u / d eta_ra, d u / d eta_rb) on the own face grid
      par([&](int ltc, TS& ts) {
        H3C_TEAM(ltc);
        const int ta = lt / Q, tb_ = lt % Q;
        for_faces<0, NF>([&](auto Fc) {
          constexpr int f = decltype(Fc)::value;
          if constexpr (fc(S, f, 0) == 0) {
            constexpr int row = fc(S, f, 1) > 0 ? 1 : 0;
            double uf = 0.0, un = 0.0;
#pragma unroll
            for (int k = 0; k < Q; ++k) {
              uf = fma(H3C_TX[XE + row * Q + k], ts.u[k], uf);
              un = fma(H3C_TX[XED + row * Q + k], ts.u[k], un);
            }
            FL[f * 4 * Q2 + lt] = uf;
            FL[f * 4 * Q2 + Q2 + lt] = un;
          }
        });
#pragma unroll
        for (int k = 0; k < Q; ++k) B0[k * SI + ta * SJ + tb_] = ts.u[k];
        if (H3C_UHAND) {   // u for the apply kernel (coalesced: consecutive threads, consecutive points)
          double* ue = P.ug + ugo;
#pragma unroll
          for (int k = 0; k < Q; ++k) ue[k * Q2 + lt] = ts.u[k];
        }
      });
      sync();
      par([&](int ltc, TS&) {
        H3C_TEAM(ltc);
        const int ta = lt / Q, tb_ = lt % Q;
        double v[Q], w[Q];
#pragma unroll
        for (int m = 0; m < Q; ++m) {
          v[m] = B0[ta * SI + m * SJ + tb_];   // line along eta1: (k0 = ta, k2 = tb)
          w[m] = B0[ta * SI + tb_ * SJ + m];   // line along eta2: (k0 = ta, k1 = tb)
        }
        for_faces<0, NF>([&](auto Fc) {
          constexpr int f = decltype(Fc)::value;
          constexpr int fx = fc(S, f, 0);
          if constexpr (fx != 0) {
            constexpr int row = fx * 2 + (fc(S, f, 1) > 0 ? 1 : 0);
            double uf = 0.0, un = 0.0;
#pragma unroll
            for (int k = 0; k < Q; ++k) {
              const double val = fx == 1 ? v[k] : w[k];
              uf = fma(H3C_TX[XE + row * Q + k], val, uf);
              un = fma(H3C_TX[XED + row * Q + k], val, un);
            }
            FL[f * 4 * Q2 + lt] = uf;
            FL[f * 4 * Q2 + Q2 + lt] = un;
          }
        });
      });
      sync();
      // tangential derivatives: one face-grid line per task (face, direction, line)
      par([&](int ltc, TS&) {
        H3C_TEAM(ltc);
        for (int task = lt; task < NF * 2 * Q; task += NT) {
          const int f = task / (2 * Q), dir = (task / Q) & 1, line = task % Q;
          const int base = dir ? line * Q : line, st = dir ? 1 : Q;
          const double* fu = FL + f * 4 * Q2;
          double in[Q], out[Q];
#pragma unroll
          for (int j = 0; j < Q; ++j) in[j] = fu[base + j * st];
          const int axis = fcr(S, f, dir ? 3 : 2);
          if (S == H3_PRISM && axis == 1) eo_full<Q>(H3C_TE, 1 * EOS, in, out);
          else eo_full<Q>(H3C_TE, 0, in, out);
          double* fo = FL + f * 4 * Q2 + (2 + dir) * Q2;
#pragma unroll
          for (int j = 0; j < Q; ++j) fo[base + j * st] = out[j];
        }
      });
      sync();
      // n.grad u at own face point a = lt of every face; identity-map couplings publish directly
      par([&](int ltc, TS&) {
        H3C_TEAM(ltc);
        double* fbe = P.fb + fbo;
        int s = 0;
        // one coupling per face and every face coupled (always so for tets): slot f is face f, and the
        // header reads below are at compile-time offsets instead of a dependent search through the slots
        const bool onefc = C::NSMAX == NF && ns == NF;
        for_faces<0, NF>([&](auto Fc) {
          constexpr int f = decltype(Fc)::value;
          constexpr int fx = fc(S, f, 0), sd = fc(S, f, 1), ra = fc(S, f, 2), rb = fc(S, f, 3);
          if (onefc) s = f;
          if (onefc || (s < ns && slot_hdr(hdr, s).face == f)) {
            const H3Slot& h = slot_hdr(hdr, s);
            double* Ff = FL + f * 4 * Q2;
            const Chain ch = face_chain<S>(pts, Rt, Q, fx, sd, ra, rb, lt / Q, lt % Q);
            const double g0 = ch.c00 * h.v[0] + ch.c01 * h.v[1] + ch.c02 * h.v[2];
            const double g1 = ch.c11 * h.v[1] + ch.c12 * h.v[2];
            const double g2 = h.v[2];
            const double gf = fx == 0 ? g0 : (fx == 1 ? g1 : g2);
            const double ga = ra == 0 ? g0 : (ra == 1 ? g1 : g2);
            const double gb = rb == 0 ? g0 : (rb == 1 ? g1 : g2);
            const double uf = Ff[lt];
            const double gv = gf * Ff[Q2 + lt] + ga * Ff[2 * Q2 + lt] + gb * Ff[3 * Q2 + lt];
            Ff[Q2 + lt] = gv;
            for (const int s1_ = onefc ? s + 1 : ns; s < s1_ && (onefc || slot_hdr(hdr, s).face == f); ++s) {
              const H3Slot& hs = slot_hdr(hdr, s);
              if (hs.mkind == MAP_ID) {
                reinterpret_cast<double2*>(P.pub + hs.pub_self)[lt] = make_double2(uf, gv);
              } else {   // staged on the own face grid for the trace-map kernel (fb is free until the flux kernel)
                fbe[s * 2 * Q2 + lt] = uf;
                fbe[s * 2 * Q2 + Q2 + lt] = gv;
              }
            }
          }
        });
      });
      continue;
    }

    // ================= apply: PhysDeriv (stdregions.py:658-674) ==================================
    // eta0 in registers; eta1 / eta2 one line per thread through B0 / B1
    if (!UH) {
      par([&](int ltc, TS& ts) {
        H3C_TEAM(ltc);
        const int ta = lt / Q, tb_ = lt % Q;
#pragma unroll
        for (int k = 0; k < Q; ++k) B0[k * SI + ta * SJ + tb_] = ts.u[k];
        eo_full<Q>(H3C_TE, 0 * EOS, ts.u, ts.d0);
      });
      sync();
    }
    par([&](int ltc, TS& ts) {
      H3C_TEAM(ltc);
      const int ta = lt / Q, tb_ = lt % Q;
      double v[Q], w[Q];
#pragma unroll
      for (int m = 0; m < Q; ++m) {
        v[m] = B0[ta * SI + m * SJ + tb_];
        w[m] = B0[ta * SI + tb_ * SJ + m];
      }
      eo_full<Q>(H3C_TE, 1 * EOS, v, ts.d1);
      eo_full<Q>(H3C_TE, 2 * EOS, w, ts.d2);
#pragma unroll
      for (int r = 0; r < Q; ++r) B1[ta * SI + r * SJ + tb_] = ts.d1[r];
    });
    sync();   // every line of B0 read
    par([&](int ltc, TS& ts) {
      H3C_TEAM(ltc);
      const int ta = lt / Q, tb_ = lt % Q;
#pragma unroll
      for (int r = 0; r < Q; ++r) B0[ta * SI + tb_ * SJ + r] = ts.d2[r];
    });
    // ================= volume terms (sipg.py:575-582) + face lifts, in registers ==================
#if defined(__CUDA_ARCH__)
    __pipeline_wait_prior(UH ? 1 : 0);   // this element's own-grid fluxes (the next element's u may still be in flight)
#endif
    sync();
    par([&](int ltc, TS& ts) {
      H3C_TEAM(ltc);
      const int ta = lt / Q, tb_ = lt % Q;
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        ts.d1[k] = B1[k * SI + ta * SJ + tb_];
        ts.d2[k] = B0[k * SI + ta * SJ + tb_];
      }
      const double lam = P.lam;
      const double tp1 = 1.0 + pts[Q + ta], tr1 = Rt[Q + ta], tr2 = Rt[2 * Q + tb_];   // this thread's (eta1, eta2)
      const double dJ = eg[0], S00 = eg[1], S01 = eg[2], S02 = eg[3], S11 = eg[4], S12 = eg[5], S22 = eg[6];
      const double jw12 = dJ * W12[lt];
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        const Chain ch = chain_t<S>(H3C_TX[XP0 + k], tp1, tr1, tr2);
        const double jw = jw12 * H3C_TX[XW0 + k];
        const double e0 = ts.d0[k], e1 = ts.d1[k], e2 = ts.d2[k];
        const double x0 = ch.c00 * e0, x1 = ch.c01 * e0 + ch.c11 * e1, x2 = ch.c02 * e0 + ch.c12 * e1 + e2;
        const double f0 = S00 * x0 + S01 * x1 + S02 * x2;
        const double f1 = S01 * x0 + S11 * x1 + S12 * x2;
        const double f2 = S02 * x0 + S12 * x1 + S22 * x2;
        ts.u[k] = lam * jw * ts.u[k];
        ts.d0[k] = jw * (ch.c00 * f0 + ch.c01 * f1 + ch.c02 * f2);
        ts.d1[k] = jw * (ch.c11 * f1 + ch.c12 * f2);
        ts.d2[k] = jw * f2;
      }
      // lift (the reference's scatter + final sweep, sipg.py:663-693), per local face f with own-grid
      // fluxes (fv, fd) summed over its one or two couplings:
      //   W0(k) += E[k_fixed] fv(a),  W_c(k) += E[k_fixed] ((G n)_c fd)(a),  (G n) from the collapse chain
      int s = 0;
      const bool onefc = C::NSMAX == NF && ns == NF;   // tets: slot f is face f (compile-time header offsets)
      for_faces<0, NF>([&](auto Fc) {
        constexpr int f = decltype(Fc)::value;
        constexpr int fx = fc(S, f, 0), sd = fc(S, f, 1), hi = sd > 0 ? 1 : 0;
        constexpr bool onehot = gll_axis(S, fx);
        constexpr int kend = hi ? Q - 1 : 0;
        constexpr double rs = sd < 0 ? 0.5 : 0.0, ps = 1.0 + sd;
        if (onefc) s = f;
        else if (!(s < ns && slot_hdr(hdr, s).face == f)) return;
        const H3Slot& h = slot_hdr(hdr, s);
        const double v0 = h.v[0], v1 = h.v[1], v2 = h.v[2];
        const double* F0 = fbuf + s * 2 * Q2;
        const bool two = C::NSMAX > NF && s + 1 < ns && slot_hdr(hdr, s + 1).face == f;   // tets: one coupling per face
        const double* F1 = two ? F0 + 2 * Q2 : F0;
        const double w2nd = two ? 1.0 : 0.0;
        s += two ? 2 : 1;
        if constexpr (fx == 0) {
          const double fv = F0[lt] + w2nd * F1[lt], fd = F0[Q2 + lt] + w2nd * F1[Q2 + lt];
          const Chain ch = chain_t<S>(ps, tp1, tr1, tr2);
          const double l1 = (ch.c00 * v0 + ch.c01 * v1 + ch.c02 * v2) * fd;
          const double l2 = (ch.c11 * v1 + ch.c12 * v2) * fd, l3 = v2 * fd;
#pragma unroll
          for (int k = 0; k < Q; ++k) {
            if (onehot && k != kend) continue;
            const double ek = H3C_TX[XE + hi * Q + k];
            ts.u[k] = fma(ek, fv, ts.u[k]);
            ts.d0[k] = fma(ek, l1, ts.d0[k]);
            ts.d1[k] = fma(ek, l2, ts.d1[k]);
            ts.d2[k] = fma(ek, l3, ts.d2[k]);
          }
        } else {
          const int kf = fx == 1 ? ta : tb_, ko = fx == 1 ? tb_ : ta;   // own index on the fixed / other axis
          if (onehot && kf != kend) return;
          const double ek = Et[(fx * 2 + hi) * Q + kf];
#pragma unroll
          for (int k = 0; k < Q; ++k) {
            const int a = k * Q + ko;
            const double fv = F0[a] + w2nd * F1[a], fd = ek * (F0[Q2 + a] + w2nd * F1[Q2 + a]);
            // the chain at face point (eta0 = point k, the other run axis at this thread's index)
            const Chain ch = fx == 1 ? chain_t<S>(H3C_TX[XP0 + k], ps, rs, tr2)
                                     : chain_t<S>(H3C_TX[XP0 + k], tp1, tr1, rs);
            ts.u[k] = fma(ek, fv, ts.u[k]);
            ts.d0[k] = fma(ch.c00 * v0 + ch.c01 * v1 + ch.c02 * v2, fd, ts.d0[k]);
            ts.d1[k] = fma(ch.c11 * v1 + ch.c12 * v2, fd, ts.d1[k]);
            ts.d2[k] = fma(v2, fd, ts.d2[k]);
          }
        }
      });
      // ================= T = W0 + sum_a D_a^T W_a (IProductDeriv, stdregions.py:620-656) ==========
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        B0[k * SI + ta * SJ + tb_] = ts.d1[k];
        B1[k * SI + ta * SJ + tb_] = ts.d2[k];
      }
      double r[Q];
      eo_full<Q>(H3C_TE, 3 * EOS, ts.d0, r);
#pragma unroll
      for (int k = 0; k < Q; ++k) ts.u[k] += r[k];
    });
    sync();
    par([&](int ltc, TS&) {
      H3C_TEAM(ltc);
      const int ta = lt / Q, tb_ = lt % Q;
      double v[Q], w[Q], r1[Q], r2[Q];
#pragma unroll
      for (int m = 0; m < Q; ++m) {
        v[m] = B0[ta * SI + m * SJ + tb_];
        w[m] = B1[ta * SI + tb_ * SJ + m];
      }
      eo_full<Q>(H3C_TE, 4 * EOS, v, r1);
      eo_full<Q>(H3C_TE, 5 * EOS, w, r2);
#pragma unroll
      for (int m = 0; m < Q; ++m) {
        B0[ta * SI + m * SJ + tb_] = r1[m];
        B1[ta * SI + tb_ * SJ + m] = r2[m];
      }
    });
    sync();
    // ================= IProduct (stdregions.py:599-618): y = Phi^T T ==============================
    par([&](int ltc, TS& ts) {
      H3C_TEAM(ltc);
      const int ta = lt / Q, tb_ = lt % Q;
#pragma unroll
      for (int k = 0; k < Q; ++k) ts.u[k] += B0[k * SI + ta * SJ + tb_] + B1[k * SI + ta * SJ + tb_];
      double o[NA];
      cmatT<Q, NA>(H3C_TA, 0, ts.u, o);
#pragma unroll
      for (int g = 0; g < NA; ++g) s2[g * SI + ta * SJ + tb_] = o[g];
    });
    sync();
    if (S == H3_HEX) {
      par([&](int ltc, TS&) {
        H3C_TEAM(ltc);
        if (lt < N * Q) {                      // (i0, k2): k1 -> i1
          const int i0 = lt / Q, k2 = lt % Q;
          double col[Q], out[N];
#pragma unroll
          for (int k = 0; k < Q; ++k) col[k] = s2[i0 * SI + k * SJ + k2];
          cmatT<Q, N>(H3C_TA, 0, col, out);
#pragma unroll
          for (int i = 0; i < N; ++i) s1[(i0 * N + i) * Q + k2] = out[i];
        }
      });
      sync();
      par([&](int ltc, TS&) {
        H3C_TEAM(ltc);
        if (lt < N * N) {                      // (i0, i1): k2 -> i2
          double col[Q], out[N];
#pragma unroll
          for (int k = 0; k < Q; ++k) col[k] = s1[lt * Q + k];
          cmatT<Q, N>(H3C_TA, 0, col, out);
#pragma unroll
          for (int i = 0; i < N; ++i) y[dof + lt * N + i] = out[i];
        }
      });
    } else {
      par([&](int ltc, TS&) {
        H3C_TEAM(ltc);
        H3C_ITEM_UNROLL
        for (int rr = 0; rr < (C::NPM * Q + NT - 1) / NT; ++rr) {
          const int o = lt + rr * NT;
          if (o >= C::NPM * Q) break;
          const int k = o % Q, m = o / Q, g = gof[m];
          const double* Br = Bt + m * Q;
          double a = 0.0;
          if (S == H3_PRISM) {   // s1[m][k1] = sum_k2 B[m][k2] s2[g][k1][k2]
#pragma unroll
            for (int k2 = 0; k2 < Q; ++k2) a = fma(Br[k2], s2[g * SI + k * SJ + k2], a);
          } else {               // s1[m][k2] = sum_k1 B[m][k1] s2[g][k1][k2]
#pragma unroll
            for (int k1 = 0; k1 < Q; ++k1) a = fma(Br[k1], s2[g * SI + k1 * SJ + k], a);
          }
          s1[o] = a;
        }
      });
      sync();
      par([&](int ltc, TS&) {
        H3C_TEAM(ltc);
        if (S == H3_PRISM) {
          for (int m = lt; m < C::NPM; m += NT) {
            double col[Q], out[N];
#pragma unroll
            for (int k = 0; k < Q; ++k) col[k] = s1[m * Q + k];
            cmatT<Q, N>(H3C_TP, 0, col, out);
#pragma unroll
            for (int l = 0; l < N; ++l) y[dof + m * N + l] = out[l];
          }
        } else {
          H3C_ITEM_UNROLL
          for (int rr = 0; rr < (C::NC + NT - 1) / NT; ++rr) {
            const int r = lt + rr * NT;
            if (r >= C::NC) break;
            const int inf = rinfo[r], m = inf & 255;
            const double* Cr = Cd + (inf >> 8) * Q;
            double a = 0.0;
#pragma unroll
            for (int k2 = 0; k2 < Q; ++k2) a = fma(Cr[k2], s1[m * Q + k2], a);
            y[dof + r] = a;
          }
        }
      });
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Slot kernels, one warp per coupling side (slot), any shape / order, over work lists of 64-byte
// records (identity-map and mapped slots separately, so the warps of a launch do uniform work).
//   trace maps (mapped slots): the own traces (u, n.grad u) the publish kernel staged on the own face
//     grid (in fb), interpolated to the coupling's trace points (trace.py:172-199 transfers; tensor
//     X (x) Y, row-structured for subface quads, or dense) -> published;
//   flux: the SIP flux at the trace points (sipg.py:622-650, 663-677) from the published own and
//     partner traces (boundary: jump 2u, average g), then the transposed trace map onto the owning
//     element's face grid: fb[slot] = (fv, fd) -- the reference's per-interface phase 2
//     (sipg.py:607-661).
// Identity-map flux is a pure streaming kernel (one slot per warp).  The mapped kernels are
// persistent: a warp walks its slots with the next slot's inputs (and the record after that) in
// flight by cp.async while it computes -- the dependent record -> data -> store chain of a slot is
// several DRAM latencies long, and without the prefetch these kernels ran at a fifth of the HBM rate.
#define H3C_SLOT_WPB 4                       // warps per CTA
H3C_HD int div_small(int it, unsigned rcp) { return (int)(((unsigned)it * rcp) >> 16); }   // it < 600, divisor <= 8

#if defined(__CUDA_ARCH__)
// fp64 tensor-core tile D(8x8) += A(8x4) B(4x8): lane l = 4 g + t holds A[g][t], B[t][g], D[g][2t], D[g][2t+1]
__device__ __forceinline__ void dmma884(double& d0, double& d1, const double a, const double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
#endif

// staged inputs of a mapped slot (doubles): map: own-grid (u | g), 2 q^2;  flux: own traces (u, g)
// interleaved [0, 2 TMAX), partner traces [2 TMAX, 4 TMAX), trace weights [4 TMAX, 5 TMAX)
#define H3C_ST_MAP (2 * h3::TMAX)
#define H3C_ST_FLUX (5 * h3::TMAX)
template <bool FLUX, typename Par>
H3C_HD void slot_stage(const H3Plan& P, const H3FluxRec& hr, double* st, Par par) {
  const H3FluxRec h = hr;   // the record (shared-memory ring) in registers
  const int Q = (int)(h.fb_q & 15), Q2 = Q * Q;
  par([&](int lane) {
#if defined(__CUDA_ARCH__)
    if (FLUX) {
      const double* own = P.pub + h.pub_self;
      const double* nbr = P.pub + h.pub_other;
      for (int r = lane; r < h.nt; r += 32) {
        __pipeline_memcpy_async(st + 2 * r, own + 2 * r, 16);
        if (h.mk_kind >> 8) __pipeline_memcpy_async(st + 2 * TMAX + 2 * r, nbr + 2 * r, 16);
        __pipeline_memcpy_async(st + 4 * TMAX + r, P.tab + h.wtoff + r, 8);
      }
    } else {
      const double* og = P.fb + (h.fb_q >> 4);
      for (int r = lane; r < Q2; r += 32) __pipeline_memcpy_async(st + 2 * r, og + 2 * r, 16);
    }
#else
    if (FLUX) {
      for (int r = lane; r < h.nt; r += 32) {
        st[2 * r] = P.pub[h.pub_self + 2 * r];
        st[2 * r + 1] = P.pub[h.pub_self + 2 * r + 1];
        if (h.mk_kind >> 8) {
          st[2 * TMAX + 2 * r] = P.pub[h.pub_other + 2 * r];
          st[2 * TMAX + 2 * r + 1] = P.pub[h.pub_other + 2 * r + 1];
        }
        st[4 * TMAX + r] = P.tab[h.wtoff + r];
      }
    } else {
      for (int r = lane; r < 2 * Q2; r += 32) st[r] = P.fb[(h.fb_q >> 4) + r];
    }
#endif
  });
}

// trace map of a staged slot: st = own-grid (u | g); tmp: 2 TMAX doubles
template <typename Par, typename Sync>
H3C_HD void map_compute(const H3Plan& P, const H3FluxRec& hr, const double* st, double* tmp, Par par, Sync sync) {
  const H3FluxRec h = hr;
  const int mkind = h.mk_kind & 255;
  const int Q = (int)(h.fb_q & 15), Q2 = Q * Q;
  const unsigned rq = 65536u / Q + 1;
  const double* tab = P.tab;
  double2* dst = reinterpret_cast<double2*>(P.pub + h.pub_self);
  const double* fu = st;
  const double* fg = st + Q2;
  const int n1 = h.nab & 255, n2 = (h.nab >> 8) & 255, sw = (h.nab >> 16) & 1;
#if defined(__CUDA_ARCH__)
  if (mkind == MAP_TENSOR) {
    // t_f = X F_f Y^T (f = u, g) as two 8 x 8 x 8 tensor-core products per field, zero-padded:
    // T_f = X F_f, then t_f = T_f Y^T with T_f passed from the accumulator to the A layout by shuffles
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const double* X = tab + h.moff;
    const double* Y = tab + h.moff2;
    double cu0 = 0.0, cu1 = 0.0, cg0 = 0.0, cg1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int ia = 4 * ks + t;
      const bool ok = ia < Q && g < Q;
      const double a = (g < n1 && ia < Q) ? __ldg(X + g * Q + ia) : 0.0;
      const double bu = ok ? fu[ia * Q + g] : 0.0, bg = ok ? fg[ia * Q + g] : 0.0;
      dmma884(cu0, cu1, a, bu);
      dmma884(cg0, cg1, a, bg);
    }
    double tu0 = 0.0, tu1 = 0.0, tg0 = 0.0, tg1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int src = (lane & ~3) + 2 * ks + (t >> 1), ib = 4 * ks + t;
      const double xu0 = __shfl_sync(0xffffffffu, cu0, src), xu1 = __shfl_sync(0xffffffffu, cu1, src);
      const double xg0 = __shfl_sync(0xffffffffu, cg0, src), xg1 = __shfl_sync(0xffffffffu, cg1, src);
      const double au = (t & 1) ? xu1 : xu0, ag = (t & 1) ? xg1 : xg0;
      const double b = (g < n2 && ib < Q) ? __ldg(Y + g * Q + ib) : 0.0;
      dmma884(tu0, tu1, au, b);
      dmma884(tg0, tg1, ag, b);
    }
    if (g < n1) {
      const int r2 = 2 * t;
      if (r2 < n2) dst[sw ? r2 * n1 + g : g * n2 + r2] = make_double2(tu0, tg0);
      if (r2 + 1 < n2) dst[sw ? (r2 + 1) * n1 + g : g * n2 + r2 + 1] = make_double2(tu1, tg1);
    }
    return;
  }
#endif
#if defined(__CUDA_ARCH__)
  if (mkind == MAP_ROW) {
    // tmp[pb][i_par] = sum_i_perp Y[pb][i_perp] f(i_par, i_perp) as one 8 x 8 x 8 tensor-core product per field
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const double* Y = tab + h.moff2;
    double cu0 = 0.0, cu1 = 0.0, cg0 = 0.0, cg1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int ip = 4 * ks + t;
      const bool ok = ip < Q && g < Q;
      const int o = sw ? g * Q + ip : ip * Q + g;
      const double a = (g < n2 && ip < Q) ? __ldg(Y + g * Q + ip) : 0.0;
      const double bu = ok ? fu[o] : 0.0, bg = ok ? fg[o] : 0.0;
      dmma884(cu0, cu1, a, bu);
      dmma884(cg0, cg1, a, bg);
    }
    if (g < n2) {
      const int ib = 2 * t;
      if (ib < Q) {
        tmp[g * Q + ib] = cu0;
        tmp[TMAX + g * Q + ib] = cg0;
      }
      if (ib + 1 < Q) {
        tmp[g * Q + ib + 1] = cu1;
        tmp[TMAX + g * Q + ib + 1] = cg1;
      }
    }
  } else
#endif
  par([&](int lane) {
    const int tot = mkind == MAP_TENSOR ? n1 * Q : (mkind == MAP_ROW ? n2 * Q : h.nt);
    for (int it = lane; it < tot; it += 32) {
      double a0 = 0.0, a1 = 0.0;
      const int r1 = div_small(it, rq), ib = it - r1 * Q;
      if (mkind == MAP_ROW) {          // tmp[pb][i_par] = sum_i_perp Y[pb][i_perp] f(i_par, i_perp)
        const double* Yr = tab + h.moff2 + r1 * Q;
        H3C_MAPLOOP(ip, Q) {
          const double m = H3C_LDG(Yr + ip);
          const int o = sw ? ib * Q + ip : ip * Q + ib;
          a0 = fma(m, fu[o], a0);
          a1 = fma(m, fg[o], a1);
        }
        tmp[it] = a0;
        tmp[TMAX + it] = a1;
      } else if (mkind == MAP_TENSOR) {
        const double* X = tab + h.moff + r1 * Q;
        H3C_MAPLOOP(ia, Q) {
          const double m = H3C_LDG(X + ia);
          a0 = fma(m, fu[ia * Q + ib], a0);
          a1 = fma(m, fg[ia * Q + ib], a1);
        }
        tmp[it] = a0;
        tmp[TMAX + it] = a1;
      } else {                         // dense
        const double* M = tab + h.moff + (int64_t)it * Q2;
        for (int a = 0; a < Q2; ++a) {
          const double m = H3C_LDG(M + a);
          a0 = fma(m, fu[a], a0);
          a1 = fma(m, fg[a], a1);
        }
        dst[it] = make_double2(a0, a1);
      }
    }
  });
  if (mkind == MAP_DENSE) return;
  sync();
#if defined(__CUDA_ARCH__)
  if (mkind == MAP_ROW) {
    // t_f[pa, pb] = sum_i_par X[pb][pa][i_par] tmp_f[pb][i_par]: per trace row pb one 8 x 8 x 8 tensor-core
    // product whose B operand holds the two fields (u, n.grad u) in its first two columns
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const double* X = tab + h.moff;
    for (int pb = 0; pb < n2; ++pb) {
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int ip = 4 * ks + t;
        const double a = (g < n1 && ip < Q) ? __ldg(X + (pb * n1 + g) * Q + ip) : 0.0;
        const double b = (g < 2 && ip < Q) ? tmp[g * TMAX + pb * Q + ip] : 0.0;
        dmma884(c0, c1, a, b);
      }
      if (t == 0 && g < n1) dst[g * n2 + pb] = make_double2(c0, c1);   // C[pa = g][field 0, 1]
    }
    return;
  }
#endif
  const unsigned rn2 = 65536u / n2 + 1;
  par([&](int lane) {
    for (int it = lane; it < h.nt; it += 32) {
      const int r1 = div_small(it, rn2), r2 = it - r1 * n2;
      int p;
      const double *Y, *m0, *m1;
      if (mkind == MAP_ROW) {   // t[pa, pb] = sum_i_par X[pb][pa][i_par] tmp[pb][i_par]  (r1 = pa, r2 = pb)
        p = it;
        Y = tab + h.moff + (r2 * n1 + r1) * Q;
        m0 = tmp + r2 * Q;
        m1 = tmp + TMAX + r2 * Q;
      } else {
        p = sw ? r2 * n1 + r1 : r1 * n2 + r2;
        Y = tab + h.moff2 + r2 * Q;
        m0 = tmp + r1 * Q;
        m1 = tmp + TMAX + r1 * Q;
      }
      double a0 = 0.0, a1 = 0.0;
      H3C_MAPLOOP(ib, Q) {
        const double m = H3C_LDG(Y + ib);
        a0 = fma(m, m0[ib], a0);
        a1 = fma(m, m1[ib], a1);
      }
      dst[p] = make_double2(a0, a1);
    }
  });
}

// flux + transposed map of a staged mapped slot (st as slot_stage<true>; its own-trace part is reused
// for the first contraction); tv: 2 TMAX doubles
template <typename Par, typename Sync>
H3C_HD void flux_compute(const H3Plan& P, const H3FluxRec& hr, double* st, double* tv, Par par, Sync sync) {
  const H3FluxRec h = hr;
  const int Q = (int)(h.fb_q & 15), Q2 = Q * Q, mkind = h.mk_kind & 255, kind = h.mk_kind >> 8;
  const unsigned rq = 65536u / Q + 1;
  double* fb = P.fb + (h.fb_q >> 4);
  const double* tab = P.tab;
  double* tmp = st;                // first contraction (over the consumed own traces)
  par([&](int lane) {              // flux at the trace points: tv[p], tv[TMAX + p]
    for (int p = lane; p < h.nt; p += 32) {
      const double ut = st[2 * p], gt = st[2 * p + 1];
      const double un = kind ? st[2 * TMAX + 2 * p] : -ut, gn = kind ? st[2 * TMAX + 2 * p + 1] : -gt;
      const double j = ut - un, cc = 0.5 * (gt - gn);
      const double w = h.sJ * st[4 * TMAX + p];
      tv[p] = (h.tau * j - cc) * w;
      tv[TMAX + p] = -0.5 * j * w;
    }
  });
  sync();
  const int n1 = h.nab & 255, n2 = (h.nab >> 8) & 255, sw = (h.nab >> 16) & 1;
#if defined(__CUDA_ARCH__)
  if (mkind == MAP_TENSOR) {
    // F_f = X^T G_f Y (f = fv, fd; G_f the flux on the n1 x n2 trace grid): U_f = G_f Y, F_f = X^T U_f
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const double* X = tab + h.moff;
    const double* Y = tab + h.moff2;
    double uv0 = 0.0, uv1 = 0.0, ud0 = 0.0, ud1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int r2 = 4 * ks + t;
      const bool ok = g < n1 && r2 < n2;
      const int p = sw ? r2 * n1 + g : g * n2 + r2;
      const double av = ok ? tv[p] : 0.0, ad = ok ? tv[TMAX + p] : 0.0;
      const double b = (r2 < n2 && g < Q) ? __ldg(Y + r2 * Q + g) : 0.0;
      dmma884(uv0, uv1, av, b);
      dmma884(ud0, ud1, ad, b);
    }
    double fv0 = 0.0, fv1 = 0.0, fd0 = 0.0, fd1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int r1 = 4 * ks + t, src = r1 * 4 + (g >> 1);
      const double xv0 = __shfl_sync(0xffffffffu, uv0, src), xv1 = __shfl_sync(0xffffffffu, uv1, src);
      const double xd0 = __shfl_sync(0xffffffffu, ud0, src), xd1 = __shfl_sync(0xffffffffu, ud1, src);
      const double bv = (g & 1) ? xv1 : xv0, bd = (g & 1) ? xd1 : xd0;
      const double a = (r1 < n1 && g < Q) ? __ldg(X + r1 * Q + g) : 0.0;
      dmma884(fv0, fv1, a, bv);
      dmma884(fd0, fd1, a, bd);
    }
    if (g < Q) {
      const int ib = 2 * t;
      if (ib < Q) {
        fb[g * Q + ib] = fv0;
        fb[Q2 + g * Q + ib] = fd0;
      }
      if (ib + 1 < Q) {
        fb[g * Q + ib + 1] = fv1;
        fb[Q2 + g * Q + ib + 1] = fd1;
      }
    }
    return;
  }
#endif
#if defined(__CUDA_ARCH__)
  if (mkind == MAP_ROW) {
    // tmp_f[pb][i_par] = sum_pa X[pb][pa][i_par] g_f[pa, pb]: per trace row pb one tensor-core product,
    // the two fields (fv, fd) in the first two columns of B
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const double* X = tab + h.moff;
    for (int pb = 0; pb < n2; ++pb) {
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int pa = 4 * ks + t;
        const double a = (g < Q && pa < n1) ? __ldg(X + (pb * n1 + pa) * Q + g) : 0.0;   // A[i_par = g][pa]
        const double b = (g < 2 && pa < n1) ? tv[g * TMAX + pa * n2 + pb] : 0.0;          // B[pa][field g]
        dmma884(c0, c1, a, b);
      }
      if (t == 0 && g < Q) {
        tmp[pb * Q + g] = c0;
        tmp[TMAX + pb * Q + g] = c1;
      }
    }
  } else
#endif
  // transposed map, stage 1: tensor / row first contraction, dense complete -> tmp
  par([&](int lane) {
    const int tot = mkind == MAP_ROW ? n2 * Q : (mkind == MAP_TENSOR ? n1 * Q : Q2);
    for (int it = lane; it < tot; it += 32) {
      double a0 = 0.0, a1 = 0.0;
      const int r1 = div_small(it, rq), ib = it - r1 * Q;
      if (mkind == MAP_ROW) {   // tmp[pb][i_par] = sum_pa X[pb][pa][i_par] g[pa, pb]
        H3C_MAPLOOP(pa, n1) {
          const double m = H3C_LDG(tab + h.moff + (r1 * n1 + pa) * Q + ib);
          a0 = fma(m, tv[pa * n2 + r1], a0);
          a1 = fma(m, tv[TMAX + pa * n2 + r1], a1);
        }
      } else if (mkind == MAP_TENSOR) {
        const double* Yc = tab + h.moff2 + ib;
        const int pst = sw ? n1 : 1;
        const int p0 = sw ? r1 : r1 * n2;
        H3C_MAPLOOP(r2, n2) {
          const double m = H3C_LDG(Yc + r2 * Q);
          a0 = fma(m, tv[p0 + r2 * pst], a0);
          a1 = fma(m, tv[TMAX + p0 + r2 * pst], a1);
        }
      } else {                    // dense: F(a) = sum_p M[p][a] g[p]
        for (int p = 0; p < h.nt; ++p) {
          const double m = H3C_LDG(tab + h.moff + (int64_t)p * Q2 + it);
          a0 = fma(m, tv[p], a0);
          a1 = fma(m, tv[TMAX + p], a1);
        }
      }
      tmp[it] = a0;
      tmp[TMAX + it] = a1;
    }
  });
  sync();
#if defined(__CUDA_ARCH__)
  if (mkind == MAP_ROW) {
    // F(i_par, i_perp) = sum_pb tmp[pb][i_par] Y[pb][i_perp]: one 8 x 8 x 8 tensor-core product per field
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const double* Y = tab + h.moff2;
    double fv0 = 0.0, fv1 = 0.0, fd0 = 0.0, fd1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int pb = 4 * ks + t;
      const bool ok = pb < n2 && g < Q;
      const double av = ok ? tmp[pb * Q + g] : 0.0, ad = ok ? tmp[TMAX + pb * Q + g] : 0.0;   // A[i_par = g][pb]
      const double b = ok ? __ldg(Y + pb * Q + g) : 0.0;                                      // B[pb][i_perp = g]
      dmma884(fv0, fv1, av, b);
      dmma884(fd0, fd1, ad, b);
    }
    if (g < Q) {   // C[i_par = g][i_perp = 2 t, 2 t + 1]
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int iperp = 2 * t + e;
        if (iperp < Q) {
          const int a = sw ? g * Q + iperp : iperp * Q + g;
          fb[a] = e ? fv1 : fv0;
          fb[Q2 + a] = e ? fd1 : fd0;
        }
      }
    }
    return;
  }
#endif
  // stage 2: second contraction onto the own face grid -> fb
  par([&](int lane) {
    for (int a = lane; a < Q2; a += 32) {
      double a0 = 0.0, a1 = 0.0;
      const int ia = div_small(a, rq), ib = a - ia * Q;
      if (mkind == MAP_ROW) {   // F(i_par, i_perp) = sum_pb Y[pb][i_perp] tmp[pb][i_par]
        const int ipar = sw ? ia : ib, iperp = sw ? ib : ia;   // sw: the perp flag of a row map
        H3C_MAPLOOP(pb, n2) {
          const double m = H3C_LDG(tab + h.moff2 + pb * Q + iperp);
          a0 = fma(m, tmp[pb * Q + ipar], a0);
          a1 = fma(m, tmp[TMAX + pb * Q + ipar], a1);
        }
      } else if (mkind == MAP_TENSOR) {
        const double* Xc = tab + h.moff + ia;
        const double* t0 = tmp + ib;
        H3C_MAPLOOP(r1, n1) {
          const double m = H3C_LDG(Xc + r1 * Q);
          a0 = fma(m, t0[r1 * Q], a0);
          a1 = fma(m, t0[TMAX + r1 * Q], a1);
        }
      } else {
        a0 = tmp[a];
        a1 = tmp[TMAX + a];
      }
      fb[a] = a0;
      fb[Q2 + a] = a1;
    }
  });
}

// identity-map flux: trace grid = own face grid, straight from global to global
template <typename Par>
H3C_HD void flux_ident(const H3Plan& P, const int64_t i, Par par) {
  const H3FluxRec h = P.frec[i];
  const int Q = (int)(h.fb_q & 15), Q2 = Q * Q, kind = h.mk_kind >> 8;
  double* fb = P.fb + (h.fb_q >> 4);
  par([&](int lane) {
    double2 own[2], nbv[2];
    double wv[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int p = lane + 32 * r;
      own[r] = nbv[r] = make_double2(0.0, 0.0);
      wv[r] = 0.0;
      if (p < h.nt) {
        own[r] = H3C_LDG(reinterpret_cast<const double2*>(P.pub + h.pub_self) + p);
        if (kind) nbv[r] = H3C_LDG(reinterpret_cast<const double2*>(P.pub + h.pub_other) + p);
        wv[r] = H3C_LDG(P.tab + h.wtoff + p);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int p = lane + 32 * r;
      if (p < h.nt) {
        const double ut = own[r].x, gt = own[r].y;
        const double un = kind ? nbv[r].x : -ut, gn = kind ? nbv[r].y : -gt;
        const double j = ut - un, cc = 0.5 * (gt - gn);
        const double w = h.sJ * wv[r];
        fb[p] = (h.tau * j - cc) * w;
        fb[Q2 + p] = -0.5 * j * w;
      }
    }
  });
}

// identity-map records [first, first + count), one per warp
__global__ void __launch_bounds__(256, 6) k_h3c_flux_id(const H3Plan P, const int64_t first, const int64_t count) {
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= count) return;
  flux_ident(P, first + i, [&](auto&& f) { f((int)(threadIdx.x & 31)); });
}

// mapped records [first, first + count): persistent warps; the inputs of the next H3C_SLOT_DEPTH slots
// (and the records after them) are in flight by cp.async while a slot computes
#ifndef H3C_SLOT_DEPTH
#define H3C_SLOT_DEPTH 1
#endif
template <bool FLUX>
__global__ void __launch_bounds__(32 * H3C_SLOT_WPB) k_h3c_slot(const H3Plan P, const int64_t first, const int64_t count) {
  constexpr int ST = FLUX ? H3C_ST_FLUX : H3C_ST_MAP;
  constexpr int D = H3C_SLOT_DEPTH, NB = D + 1, NR = 2 * D + 1;   // staging buffers, record ring
  constexpr int PW = NR * 8 + NB * ST + 2 * TMAX;   // per warp: record ring | staged inputs | flux values / map tmp
  extern __shared__ __align__(16) double sm_[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* my = sm_ + w * PW;
  H3FluxRec* ring = reinterpret_cast<H3FluxRec*>(my);
  double* st = my + NR * 8;
  double* tmp = st + NB * ST;
  const int64_t W = (int64_t)gridDim.x * H3C_SLOT_WPB;
  const int64_t i0 = (int64_t)blockIdx.x * H3C_SLOT_WPB + w;
  auto par = [&](auto&& f) { f(lane); };
  auto sync = [&]() { __syncwarp(); };
  if (i0 >= count) return;
  const int n = (int)((count - i0 + W - 1) / W);   // this warp's slots: i0, i0 + W, ...
  auto fetch_rec = [&](int j) {                    // 64 bytes: lanes 0..3, 16 bytes each
    if (j < n && lane < 4)
      __pipeline_memcpy_async(reinterpret_cast<char*>(ring + j % NR) + 16 * lane,
                              reinterpret_cast<const char*>(P.frec + first + i0 + j * W) + 16 * lane, 16);
  };
  // record j is issued 2 D groups before its slot computes and D groups before its inputs are staged
  for (int j = 0; j < 2 * D; ++j) fetch_rec(j);
  __pipeline_commit();
  __pipeline_wait_prior(0);
  __syncwarp();
  for (int j = 0; j < D; ++j) {
    if (j < n) slot_stage<FLUX>(P, ring[j % NR], st + (j % NB) * ST, par);
    __pipeline_commit();
  }
  for (int j = 0; j < n; ++j) {
    __pipeline_wait_prior(D - 1);   // the inputs of slot j (and every older group) have landed
    __syncwarp();
    if (j + D < n) slot_stage<FLUX>(P, ring[(j + D) % NR], st + ((j + D) % NB) * ST, par);
    fetch_rec(j + 2 * D);
    __pipeline_commit();
    if (FLUX) flux_compute(P, ring[j % NR], st + (j % NB) * ST, tmp, par, sync);
    else map_compute(P, ring[j % NR], st + (j % NB) * ST, tmp, par, sync);
    __syncwarp();
  }
}
template <bool FLUX>
constexpr size_t h3c_slot_smem() {
  return sizeof(double) * H3C_SLOT_WPB * ((2 * H3C_SLOT_DEPTH + 1) * 8 + (H3C_SLOT_DEPTH + 1) * (FLUX ? H3C_ST_FLUX : H3C_ST_MAP) + 2 * TMAX);
}

// resident CTAs per SM the register allocation must allow, per q (apply | publish)
#if H3C_PACK   // CTAs of 64 (q = 8), 245, 252, 125 (q = 7, 6, 5) threads
#ifndef H3C_MINB_A
#define H3C_MINB_A(Q) ((Q) >= 8 ? 8 : ((Q) == 7 ? 2 : ((Q) == 6 ? 2 : ((Q) == 5 ? 5 : 8))))
#endif
#ifndef H3C_MINB_P
#define H3C_MINB_P(Q) ((Q) >= 8 ? 10 : ((Q) == 7 ? 2 : ((Q) == 6 ? 3 : ((Q) == 5 ? 6 : 8))))
#endif
#else
#ifndef H3C_MINB_A
#define H3C_MINB_A(Q) ((Q) >= 8 ? 8 : ((Q) == 7 ? 8 : ((Q) == 6 ? 10 : 20)))
#endif
#ifndef H3C_MINB_P
#define H3C_MINB_P(Q) ((Q) >= 8 ? 10 : ((Q) == 7 ? 10 : ((Q) == 6 ? 12 : 24)))
#endif
#endif
template <int Q, int MODE, int S = 0>
constexpr int h3c_minb() {   // the prism n = 7 publish kernel spills at 96 registers (measured 0.172 -> 0.148 ms with 8 CTAs)
  return MODE == 1 ? ((S == H3_PRISM && Q >= 8 && H3C_MINB_P(Q) > 8) ? 8 : H3C_MINB_P(Q)) : H3C_MINB_A(Q);
}

// registers per thread for that many resident CTAs (__maxnreg__: ptxas otherwise stops at 128 for the
// 64-thread classes even where the bound allows 144)
template <int Q, int MODE>
constexpr int h3c_regs() {
  const int warps = (Q * Q + 31) / 32, r = 65536 / (h3c_minb<Q, MODE>() * warps * 32) / 8 * 8;
  return r > 255 ? 255 : r;
}
#ifndef H3C_USE_MAXNREG
#define H3C_USE_MAXNREG 0
#endif
template <int S, int N, int MODE>
#if H3C_USE_MAXNREG
__global__ void __launch_bounds__(CfgC<S, N>::NTC) __maxnreg__((h3c_regs<N + 1, MODE>()))
#else
__global__ void __launch_bounds__(CfgC<S, N>::NTC, h3c_minb<N + 1, MODE, S>())
#endif
k_h3c(const H3Plan P, const int cls, const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ __align__(16) double h3c_sm[];
  body<S, N, MODE>(P, cls, x, y, (int)blockIdx.x, (int)gridDim.x, h3c_sm);
}

// __constant__ tables of one (shape, n) instantiation: the h3 tables (D, A, psi, even-odd blocks)
// plus the endpoint rows, 1 + eta0 and the eta0 weights
template <int S, int N>
cudaError_t h3c_upload(const double* D, const double* A, const double* psi, const double* E, const double* ED,
                       const double* pts, const double* W) {
  constexpr int Q = N + 1;
  cudaError_t e = h3::h3_upload<S, N>(D, A, psi);
  if (e != cudaSuccess) return e;
  double xt[14 * Q];
  for (int i = 0; i < 6 * Q; ++i) {
    xt[i] = E[i];
    xt[6 * Q + i] = ED[i];
  }
  for (int k = 0; k < Q; ++k) {
    xt[12 * Q + k] = 1.0 + pts[k];
    xt[13 * Q + k] = W[k];
  }
  return cudaMemcpyToSymbol(c3X<S, N>, xt, sizeof(double) * 14 * Q);
}

}  // namespace h3c
