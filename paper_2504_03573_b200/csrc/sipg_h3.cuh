// Config 4: the SIP-Helmholtz apply on 3-D hybrid hex / prism / tet meshes (sm_100a, fp64).
//
// The reference's two-phase apply (pkg/src/dgsipg/sipg.py:558-602) on the shared-trace route
// (sipg.py:513-554 trace rule / geometry, 653-661 TracePhysEval, 663-677 absorb), extended to
// prisms and tets (collapsed-coordinate modified-modal bases built like the reference triangle,
// stdregions.py:266-383; restated and property-tested in oracle/hybrid3d.py).  Plan layout:
// paper_2504_03573_b200/plan3d.py.
//
// Two kernels per element class (shape, n), persistent CTAs, one element at a time per CTA:
//   k_h3<S, N, true>  (publish): BwdTrans -> per interior coupling, u and n.grad u on the element's
//                     own face grid (endpoint rows E and E D along the fixed axis, collocation along
//                     the face for the tangential derivatives), mapped to the coupling's trace
//                     points (identity, tensor X (x) Y, or dense for subface quads) -> published.
//   k_h3<S, N, false> (apply):   BwdTrans, PhysDeriv, own traces of every coupling at once, the
//                     volume terms lambda jw u and jw G G^T grad u in place, then per batch of
//                     couplings the partner's published traces, the SIP flux (jump, average,
//                     penalty), the transposed maps and the transposed endpoint rows into the
//                     volume-point accumulators; one transposed pass
//                     y = Phi^T (W0 + sum_k D_k^T W_k)   (IProduct + IProductDeriv, sipg.py:575-582).
// Every element's y is written by exactly one CTA (no atomics, deterministic).
#pragma once
#include <cuda_pipeline.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define SIPG_H3_ABI_VERSION 1
// build knobs (measured variants; the defaults are the fastest measured)
#ifndef SIPG_H3_NT64_QMAX
#define SIPG_H3_NT64_QMAX 6         // classes with q <= this run 64-thread CTAs, the others 128
#endif
#ifndef SIPG_H3_TET_SPLIT
#define SIPG_H3_TET_SPLIT 0         // tets: split pencils over two halves of the output line too
#endif
#ifndef SIPG_H3_APP_MINB_HI
#define SIPG_H3_APP_MINB_HI 6       // resident apply CTAs per SM the registers must allow (128-thread classes)
#endif
#ifndef SIPG_H3_EGEO_ASYNC
#define SIPG_H3_EGEO_ASYNC 1        // element geometry by cp.async with the coefficients (else __ldg in the loop)
#endif
#ifndef SIPG_H3_PUB_DIRECT
#define SIPG_H3_PUB_DIRECT 1        // identity-map slots publish straight from the face-grid pass
#endif
#ifndef SIPG_H3_EO
#define SIPG_H3_EO 1                // even-odd factorised PhysDeriv / PhysDeriv^T pencils
#endif
#ifndef SIPG_H3_FUSE_LIFT
#define SIPG_H3_FUSE_LIFT 0         // first slot batch: flux before PhysDeriv, its lift in the volume-term pass
#endif

enum { H3_HEX = 0, H3_PRISM = 1, H3_TET = 2 };
#define CD3_WORDS 16
enum {
  CD3_SHAPE = 0, CD3_N, CD3_Q, CD3_NC, CD3_COUNT, CD3_ELEM_OFF, CD3_T_PTS, CD3_T_D, CD3_T_W, CD3_T_E,
  CD3_T_A, CD3_T_B, CD3_T_C, CD3_ROLE, CD3_T_R, CD3_T_ED
};
enum { MAP_ID = 0, MAP_TENSOR = 1, MAP_DENSE = 2, MAP_ROW = 3 };
#define H3_EGEO 8

struct H3Slot {   // numpy dtype plan3d.SLOT
  int32_t face, kind, nt, mkind, moff, moff2, nab, wtoff, elem, partner;
  int64_t pub_self, pub_other;
  double tau, sJ, v[3];
};
static_assert(sizeof(H3Slot) == 96, "H3Slot layout");

struct H3Plan {
  const int32_t* cd;
  const int32_t* class_elems;
  const int64_t* dof_off;
  const double* egeo;
  const int64_t* slot_off;
  const H3Slot* slots;
  const double* tab;
  double* pub;
  double lam;
  // register-column kernels (sipg_h3c.cuh): own-grid fluxes (fv, fd) per slot, written by the flux
  // kernels; element e's slots are contiguous from fb_off[e], 2 q^2 doubles each
  double* fb;
  const int64_t* fb_off;
  const struct H3FluxRec* frec;   // the flux kernel's work list: one record per slot, class-list order
};
// what the flux kernel needs of a slot, 64 bytes, in work-list order (built by sipg_h3_plan_create)
struct H3FluxRec {
  int64_t pub_self, pub_other, fb_q;   // fb_q = (offset into fb) * 16 + q of the owning element
  double tau, sJ;
  int32_t nt, mk_kind, nab, moff, moff2, wtoff;   // mk_kind = mkind | kind << 8
};
static_assert(sizeof(H3FluxRec) == 64, "H3FluxRec layout");

namespace h3 {

// padded volume layout per kernel kind (measured: the publish kernels gain, the apply kernels lose
// the occupancy the larger arrays cost)
#ifndef SIPG_H3_PAD_PUB
#define SIPG_H3_PAD_PUB 1
#endif
#ifndef SIPG_H3_PAD_APPLY
#define SIPG_H3_PAD_APPLY 0
#endif
template <bool PUB>
constexpr bool h3_pad() { return PUB ? SIPG_H3_PAD_PUB : SIPG_H3_PAD_APPLY; }
template <int Q, bool PD>
constexpr int H3_SJ() { return (PD && !(Q & 1)) ? Q + 1 : Q; }

// threads per CTA: 256 for q >= 8 (512 volume points), else 128
template <int Q>
constexpr int nthreads() { return Q <= SIPG_H3_NT64_QMAX ? 64 : 128; }
constexpr int TMAX = 64;   // trace points per coupling: q_t = max(q_L, q_R) <= 8

template <int S, int N>
struct Cfg {
  static constexpr int Q = N + 1, Q2 = Q * Q, Q3 = Q2 * Q;
  // padded volume layout (k0, k1, k2) -> k0 SI + k1 SJ + k2: odd row stride, so the pencils along
  // every axis hit distinct shared-memory banks (ncu: the h3 kernels are bound by the LSU data pipe,
  // a quarter to a third of whose wavefronts were bank-conflict replays with the dense layout)
  template <bool PD>
  static constexpr int sj() { return H3_SJ<Q, PD>(); }
  template <bool PD>
  static constexpr int v3() { return Q * Q * H3_SJ<Q, PD>(); }
  static constexpr int NTRI = N * (N + 1) / 2;
  static constexpr int NG = N + 1;                                   // triangle direction-1 groups
  static constexpr int NPM = NTRI + (S == H3_TET ? 1 : 0);           // + tet apex pseudo-mode
  static constexpr int NC = S == H3_HEX ? N * N * N : (S == H3_PRISM ? N * NTRI : N * (N + 1) * (N + 2) / 6);
  static constexpr int S1 = S == H3_HEX ? N * N * Q : NPM * Q;
  static constexpr int S2 = (S == H3_HEX ? N : NG) * Q * H3_SJ<Q, true>();   // sized for the padded layout
  static constexpr int NCP = (NC + 1) & ~1;
  static constexpr int NI = 4 * NPM + 4 + NC + 16;                   // int tables + batch offsets
  static constexpr int NSMAX = S == H3_HEX ? 12 : (S == H3_PRISM ? 8 : 4);   // slots per element
  static constexpr int SB = 4;                                       // slots per map batch
  static constexpr int SLOTD = 12;                                   // doubles per slot header
  // class tables staged in shared memory once per CTA (persistent kernels)
  static constexpr int TA = S == H3_HEX ? Q * N : Q * NG;
  static constexpr int TB = S == H3_HEX ? 0 : NPM * Q;
  static constexpr int TC = S == H3_HEX ? 0 : (S == H3_PRISM ? Q * N : NC * Q);
  // small 1-D tables + the ragged triangle-group rows B (and the tet C rows) in shared memory;
  // A / D / prism psi are __constant__ (register pencils)
  static constexpr int TABD = (6 * Q + 3 * Q2 + (Q + Q2) + 12 * Q + TB + 1) & ~1;   // even: 16-B cp.async after it; tet C rows: global (L1)
  static constexpr int SCR = (S1 + S2) > SB * 4 * TMAX ? (S1 + S2) : SB * 4 * TMAX;   // BwdTrans | traces
  // coefficients and slot headers are double-buffered: the next element's arrive (cp.async) while
  // the current one computes
  // the publish kernel has no derivative arrays (3 Q^3 doubles less: more CTAs per SM)
  static constexpr int doubles(bool pub) {
    return TABD + 2 * NCP + (pub ? v3<h3_pad<true>()>() : 4 * v3<h3_pad<false>()>()) + NSMAX * (2 * Q2 + 2 * SLOTD) +
           2 * H3_EGEO + SCR;
  }
  static constexpr size_t smem_bytes(bool pub) { return sizeof(double) * doubles(pub) + sizeof(int) * NI; }
};

// (fixed axis, side, run axis 0, run axis 1) per shape and local face (plan3d.FACES)
__constant__ int8_t c_faces[3][6][4] = {
    {{0, -1, 1, 2}, {0, 1, 1, 2}, {1, -1, 0, 2}, {1, 1, 0, 2}, {2, -1, 0, 1}, {2, 1, 0, 1}},
    {{2, -1, 0, 1}, {1, -1, 0, 2}, {0, 1, 1, 2}, {1, 1, 0, 2}, {0, -1, 1, 2}, {0, 0, 0, 0}},
    {{2, -1, 0, 1}, {1, -1, 0, 2}, {0, 1, 1, 2}, {0, -1, 1, 2}, {0, 0, 0, 0}, {0, 0, 0, 0}},
};

// collapse chain d eta_k / d xi_j (upper triangular, c22 = 1, c10 = c20 = c21 = 0) from
// p0 = 1 + eta0, p1 = 1 + eta1, r1 = 1 / (1 - eta1), r2 = 1 / (1 - eta2)
struct Chain {
  double c00, c01, c02, c11, c12;
};
template <int S>
__device__ __forceinline__ Chain chain_t(double p0, double p1, double r1, double r2) {
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

// chain at own-face-grid point (ia, ib) of a face (fixed axis fx at side sd, run axes ra, rb)
template <int S>
__device__ __forceinline__ Chain face_chain(const double* __restrict__ pts, const double* __restrict__ R, int Q,
                                            int fx, int sd, int ra, int rb, int ia, int ib) {
  if (S == H3_HEX) return Chain{1.0, 0.0, 0.0, 1.0, 0.0};
  // eta = +1 occurs only on axis 0 (tet / prism slanted face), where r is unused
  const double ea = *(pts + ra * Q + ia), eb = *(pts + rb * Q + ib);
  const double rra = *(R + ra * Q + ia), rrb = *(R + rb * Q + ib);
  const double es = (double)sd, rs = sd < 0 ? 0.5 : 0.0;
  const double e0 = fx == 0 ? es : (ra == 0 ? ea : eb);
  const double e1 = fx == 1 ? es : (ra == 1 ? ea : eb);
  const double r1 = fx == 1 ? rs : (ra == 1 ? rra : rrb);
  const double r2 = fx == 2 ? rs : (ra == 2 ? rra : rrb);
  return chain_t<S>(1.0 + e0, 1.0 + e1, r1, r2);
}

// group of triangle pseudo-mode (i, j) (plan tri_tables gid): row 0 -> 0 except (0,1) -> 1,
// row 1 -> 2, row i >= 2 -> i + 1; the tet apex pseudo-mode -> 1 (A = 1)
template <int S, int N>
__device__ void build_int_tables(int* gstart, int* gmem, int* gof, int* coff, int* mofr) {
  using C = Cfg<S, N>;
  if (threadIdx.x != 0) return;
  int cnt[C::NG + 1];
  for (int g = 0; g <= C::NG; ++g) cnt[g] = 0;
  int m = 0;
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N - i; ++j, ++m) {
      const int g = i == 0 ? (j == 1 ? 1 : 0) : (i == 1 ? 2 : i + 1);
      gof[m] = g;
      ++cnt[g];
    }
  if (S == H3_TET) {
    gof[C::NTRI] = 1;
    ++cnt[1];
  }
  gstart[0] = 0;
  for (int g = 0; g < C::NG; ++g) gstart[g + 1] = gstart[g] + cnt[g];
  int fill[C::NG];
  for (int g = 0; g < C::NG; ++g) fill[g] = gstart[g];
  for (int mm = 0; mm < C::NPM; ++mm) gmem[fill[gof[mm]]++] = mm;
  if (S == H3_TET) {   // tet modes: per triangle mode (degree d = max(i+j, 1)) n - d of them, apex last
    int r = 0, mm = 0;
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N - i; ++j, ++mm) {
        const int d = (i + j) > 1 ? i + j : 1;
        coff[mm] = r;
        for (int k = 0; k < N - d; ++k) mofr[r++] = mm;
      }
    coff[C::NTRI] = r;
    mofr[r++] = C::NTRI;
    coff[C::NTRI + 1] = r;
  }
}


// ---------------------------------------------------------------------------------------------
// Register pencils with __constant__ 1-D tables (the k_hex recipe): a thread loads one line of
// values along an axis into registers and produces the whole output line; with the loops fully
// unrolled every table entry is a compile-time constant-bank operand of its DFMA (uniform
// across the warp), so a contraction costs one shared-memory load per input value.
template <int S, int N> __constant__ double c3D[3 * (N + 1) * (N + 1)];                 // D_a[k][j]
template <int S, int N> __constant__ double c3A[(N + 1) * (S == H3_HEX ? N : N + 1)];   // A[k][g] / V[k][i]
template <int S, int N> __constant__ double c3P[(N + 1) * N];                           // prism psi[k][l]

// Even-odd (parity) factorisation of the collocation derivatives.  GL and GLL points are symmetric,
// so D[Q-1-k][Q-1-j] = -D[k][j] (and the same for D^T): with s_j = in_j + in_{Q-1-j},
// d_j = in_j - in_{Q-1-j} (j < H = Q/2) and, for odd Q, the middle value in_H,
//   E_k = sum_j Pe[k][j] s_j + mc[k] in_H,   O_k = sum_j Po[k][j] d_j,
//   out_k = E_k + O_k,   out_{Q-1-k} = O_k - E_k,   out_H = sum_j mr[j] d_j,
// with Pe = (D[k][j] + D[k][Q-1-j]) / 2, Po = (D[k][j] - D[k][Q-1-j]) / 2, mc[k] = D[k][H],
// mr[j] = D[H][j]: 2 H^2 (+2H) FMAs per line instead of Q^2.  Per (operator t: 0 = D, 1 = D^T,
// axis a) a block of EO doubles: Pe | Po | mc | mr.
template <int Q>
constexpr int eo_size() { return 2 * (Q / 2) * (Q / 2) + 2 * (Q / 2); }
template <int S, int N> __constant__ double c3E[6 * eo_size<N + 1>()];

// out_k for k in [K0, K0 + KN) (and their mirrors), plus the middle row when MID
template <int Q, int K0, int KN, bool MID, typename Tab>
__device__ __forceinline__ void eo_lines(const Tab& T, int off, const double (&in)[Q], double* out) {
  constexpr int H = Q / 2;
  double sm[H], df[H];
#pragma unroll
  for (int j = 0; j < H; ++j) {
    sm[j] = in[j] + in[Q - 1 - j];
    df[j] = in[j] - in[Q - 1 - j];
  }
#pragma unroll
  for (int kk = 0; kk < KN; ++kk) {
    const int k = K0 + kk;
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
  if ((Q & 1) && MID) {
    double m = 0.0;
#pragma unroll
    for (int j = 0; j < H; ++j) m = fma(T[off + 2 * H * H + H + j], df[j], m);
    out[H] = m;
  }
}

// the lines eo_lines produced, stored (ACC: accumulated) at stride st
template <int Q, int K0, int KN, bool MID, bool ACC>
__device__ __forceinline__ void eo_store(const double* out, double* d, int st) {
#pragma unroll
  for (int kk = 0; kk < KN; ++kk) {
    const int k = K0 + kk;
    if (ACC) {
      d[k * st] += out[k];
      d[(Q - 1 - k) * st] += out[Q - 1 - k];
    } else {
      d[k * st] = out[k];
      d[(Q - 1 - k) * st] = out[Q - 1 - k];
    }
  }
  if ((Q & 1) && MID) {
    if (ACC) d[(Q / 2) * st] += out[Q / 2];
    else d[(Q / 2) * st] = out[Q / 2];
  }
}

// one pencil line through the even-odd operator block `blk`, part `part` of KS
template <int S, int N, int KS, bool ACC>
__device__ __forceinline__ void eo_pencil(int blk, int part, const double (&col)[N + 1], double* dst, int st) {
  constexpr int Q = N + 1, H = Q / 2, KA = KS == 1 ? H : (H + 1) / 2;
  double out[Q];
  if (KS == 1) {
    eo_lines<Q, 0, H, true>(c3E<S, N>, blk * eo_size<Q>(), col, out);
    eo_store<Q, 0, H, true, ACC>(out, dst, st);
  } else if (part == 0) {
    eo_lines<Q, 0, KA, false>(c3E<S, N>, blk * eo_size<Q>(), col, out);
    eo_store<Q, 0, KA, false, ACC>(out, dst, st);
  } else {
    eo_lines<Q, KA, H - KA, true>(c3E<S, N>, blk * eo_size<Q>(), col, out);
    eo_store<Q, KA, H - KA, true, ACC>(out, dst, st);
  }
}

template <int S, int N>
cudaError_t h3_upload(const double* D, const double* A, const double* psi) {
  constexpr int Q = N + 1, NA = S == H3_HEX ? N : N + 1, H = Q / 2, EO = eo_size<Q>();
  cudaError_t e = cudaMemcpyToSymbol(c3D<S, N>, D, sizeof(double) * 3 * Q * Q);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c3A<S, N>, A, sizeof(double) * Q * NA);
  if (e == cudaSuccess && S == H3_PRISM) e = cudaMemcpyToSymbol(c3P<S, N>, psi, sizeof(double) * Q * N);
  if (e != cudaSuccess) return e;
  double eo[6 * EO];
  for (int t = 0; t < 2; ++t)
    for (int a = 0; a < 3; ++a) {
      const double* Da = D + a * Q * Q;
      auto M = [&](int k, int j) { return t == 0 ? Da[k * Q + j] : Da[j * Q + k]; };   // D or D^T
      double* o = eo + (t * 3 + a) * EO;
      double scale = 0.0, asym = 0.0;
      for (int k = 0; k < Q; ++k)
        for (int j = 0; j < Q; ++j) {
          scale = fmax(scale, fabs(M(k, j)));
          asym = fmax(asym, fabs(M(Q - 1 - k, Q - 1 - j) + M(k, j)));
        }
      if (asym > 1e-12 * scale) return cudaErrorInvalidValue;   // points not symmetric: no parity split
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
  return cudaMemcpyToSymbol(c3E<S, N>, eo, sizeof(double) * 6 * EO);
}

// out[k] = sum_j M[k][j] in[j]  (M row-major K x J in constant memory at compile-time offset)
template <int K, int J, typename Tab>
__device__ __forceinline__ void cmat(const Tab& M, int off, const double (&in)[J], double (&out)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double a = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) a = fma(M[off + k * J + j], in[j], a);
    out[k] = a;
  }
}
// out[j] = sum_k M[k][j] in[k]  (transposed)
template <int K, int J, typename Tab>
__device__ __forceinline__ void cmatT(const Tab& M, int off, const double (&in)[K], double (&out)[J]) {
#pragma unroll
  for (int j = 0; j < J; ++j) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) a = fma(M[off + k * J + j], in[k], a);
    out[j] = a;
  }
}

// rows [R0, R0 + KR) of out = M in  /  columns [C0, C0 + KC) of out = M^T in
template <int R0, int KR, int J, typename Tab>
__device__ __forceinline__ void cmat_rows(const Tab& M, int off, const double (&in)[J], double* out) {
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    double a = 0.0;
#pragma unroll
    for (int j = 0; j < J; ++j) a = fma(M[off + (R0 + k) * J + j], in[j], a);
    out[k] = a;
  }
}
template <int C0, int KC, int K, int J, typename Tab>
__device__ __forceinline__ void cmatT_cols(const Tab& M, int off, const double (&in)[K], double* out) {
#pragma unroll
  for (int j = 0; j < KC; ++j) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) a = fma(M[off + k * J + C0 + j], in[k], a);
    out[j] = a;
  }
}

// Pencil work is split in two halves of the output line when Q^2 pencils would leave half of the
// threads idle (2 Q^2 <= NT): part = item / Q^2 (warp-uniform for q = 8)
template <int S, int Q>
constexpr int pencil_split() { return ((S != H3_TET || SIPG_H3_TET_SPLIT) && 2 * Q * Q <= nthreads<Q>()) ? 2 : 1; }

// du_a = D_a u along each eta axis: Q^2 pencils per axis (one compile-time axis per loop: a runtime
// axis switch over three unrolled constant-operand contractions makes ptxas spill)
template <int S, int N, int A, bool PD>
__device__ __forceinline__ void pencil_deriv_axis(const double* __restrict__ u, double* __restrict__ du) {
  constexpr int Q = N + 1, Q2 = Q * Q, NT = nthreads<Q>(), KS = pencil_split<S, Q>();
  constexpr int SJ = H3_SJ<Q, PD>(), SI = Q * SJ, V3 = Q * SI;
  constexpr int KP = (Q + 1) / 2;
  constexpr int st = A == 0 ? SI : (A == 1 ? SJ : 1);
  for (int it = threadIdx.x; it < KS * Q2; it += NT) {
    const int r = it % Q2, part = it / Q2;
    const int ra = r / Q, rb = r % Q;
    const int base = A == 0 ? ra * SJ + rb : (A == 1 ? ra * SI + rb : ra * SI + rb * SJ);
    double col[Q], out[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) col[j] = u[base + j * st];
    double* d = du + A * V3 + base;
    if (SIPG_H3_EO) {      // even-odd: parts split the mirrored output pairs
      eo_pencil<S, N, KS, false>(A, part, col, d, st);
    } else if (KS == 1) {
      cmat_rows<0, Q, Q>(c3D<S, N>, A * Q2, col, out);
#pragma unroll
      for (int k = 0; k < Q; ++k) d[k * st] = out[k];
    } else if (part == 0) {
      cmat_rows<0, KP, Q>(c3D<S, N>, A * Q2, col, out);
#pragma unroll
      for (int k = 0; k < KP; ++k) d[k * st] = out[k];
    } else {
      cmat_rows<KP, Q - KP, Q>(c3D<S, N>, A * Q2, col, out);
#pragma unroll
      for (int k = 0; k < Q - KP; ++k) d[(KP + k) * st] = out[k];
    }
  }
}
template <int S, int N, bool PD>
__device__ void pencil_deriv(const double* __restrict__ u, double* __restrict__ du) {
  pencil_deriv_axis<S, N, 0, PD>(u, du);
  pencil_deriv_axis<S, N, 1, PD>(u, du);
  pencil_deriv_axis<S, N, 2, PD>(u, du);
}

// T = W0 + sum_a D_a^T W_a, in place into W0 (three passes, one per axis)
template <int S, int N, int A, bool PD>
__device__ __forceinline__ void pencil_dt_axis(double* __restrict__ W0, const double* __restrict__ W) {
  constexpr int Q = N + 1, Q2 = Q * Q, NT = nthreads<Q>(), KS = pencil_split<S, Q>();
  constexpr int SJ = H3_SJ<Q, PD>(), SI = Q * SJ, V3 = Q * SI;
  constexpr int KP = (Q + 1) / 2;
  constexpr int st = A == 0 ? SI : (A == 1 ? SJ : 1);
  for (int it = threadIdx.x; it < KS * Q2; it += NT) {
    const int r = it % Q2, part = it / Q2;
    const int ra = r / Q, rb = r % Q;
    const int base = A == 0 ? ra * SJ + rb : (A == 1 ? ra * SI + rb : ra * SI + rb * SJ);
    double col[Q], out[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) col[j] = W[A * V3 + base + j * st];
    double* w0 = W0 + base;
    if (SIPG_H3_EO) {      // even-odd with the D^T blocks
      eo_pencil<S, N, KS, true>(3 + A, part, col, w0, st);
    } else if (KS == 1) {
      cmatT_cols<0, Q, Q, Q>(c3D<S, N>, A * Q2, col, out);
#pragma unroll
      for (int k = 0; k < Q; ++k) w0[k * st] += out[k];
    } else if (part == 0) {
      cmatT_cols<0, KP, Q, Q>(c3D<S, N>, A * Q2, col, out);
#pragma unroll
      for (int k = 0; k < KP; ++k) w0[k * st] += out[k];
    } else {
      cmatT_cols<KP, Q - KP, Q, Q>(c3D<S, N>, A * Q2, col, out);
#pragma unroll
      for (int k = 0; k < Q - KP; ++k) w0[(KP + k) * st] += out[k];
    }
  }
}
template <int S, int N, bool PD>
__device__ void pencil_dt(double* __restrict__ W0, const double* __restrict__ W) {
  pencil_dt_axis<S, N, 0, PD>(W0, W);
  __syncthreads();
  pencil_dt_axis<S, N, 1, PD>(W0, W);
  __syncthreads();
  pencil_dt_axis<S, N, 2, PD>(W0, W);
  __syncthreads();
}

// u[k0][k12] = sum_g A[k0][g] s2[g][k12]   (outermost BwdTrans stage, all shapes)
template <int S, int N, bool PD>
__device__ void pencil_stage_a(const double* __restrict__ s2, double* __restrict__ u) {
  constexpr int Q = N + 1, Q2 = Q * Q, NA = S == H3_HEX ? N : N + 1, NT = nthreads<Q>(), KS = pencil_split<S, Q>();
  constexpr int SJ = H3_SJ<Q, PD>(), SI = Q * SJ;
  constexpr int KP = (Q + 1) / 2;
  for (int it = threadIdx.x; it < KS * Q2; it += NT) {
    const int r0 = it % Q2, part = it / Q2;
    const int r = (r0 / Q) * SJ + r0 % Q;
    double col[NA], out[Q];
#pragma unroll
    for (int g = 0; g < NA; ++g) col[g] = s2[g * SI + r];
    if (KS == 1) {
      cmat_rows<0, Q, NA>(c3A<S, N>, 0, col, out);
#pragma unroll
      for (int k = 0; k < Q; ++k) u[k * SI + r] = out[k];
    } else if (part == 0) {
      cmat_rows<0, KP, NA>(c3A<S, N>, 0, col, out);
#pragma unroll
      for (int k = 0; k < KP; ++k) u[k * SI + r] = out[k];
    } else {
      cmat_rows<KP, Q - KP, NA>(c3A<S, N>, 0, col, out);
#pragma unroll
      for (int k = 0; k < Q - KP; ++k) u[(KP + k) * SI + r] = out[k];
    }
  }
}

// s2[g][k12] = sum_k0 A[k0][g] T[k0][k12]   (its transpose)
template <int S, int N, bool PD>
__device__ void pencil_stage_a_t(const double* __restrict__ T, double* __restrict__ s2) {
  constexpr int Q = N + 1, Q2 = Q * Q, NA = S == H3_HEX ? N : N + 1, NT = nthreads<Q>(), KS = pencil_split<S, Q>();
  constexpr int SJ = H3_SJ<Q, PD>(), SI = Q * SJ;
  constexpr int GP = (NA + 1) / 2;
  for (int it = threadIdx.x; it < KS * Q2; it += NT) {
    const int r0 = it % Q2, part = it / Q2;
    const int r = (r0 / Q) * SJ + r0 % Q;
    double col[Q], out[NA];
#pragma unroll
    for (int k = 0; k < Q; ++k) col[k] = T[k * SI + r];
    if (KS == 1) {
      cmatT_cols<0, NA, Q, NA>(c3A<S, N>, 0, col, out);
#pragma unroll
      for (int g = 0; g < NA; ++g) s2[g * SI + r] = out[g];
    } else if (part == 0) {
      cmatT_cols<0, GP, Q, NA>(c3A<S, N>, 0, col, out);
#pragma unroll
      for (int g = 0; g < GP; ++g) s2[g * SI + r] = out[g];
    } else {
      cmatT_cols<GP, NA - GP, Q, NA>(c3A<S, N>, 0, col, out);
#pragma unroll
      for (int g = 0; g < NA - GP; ++g) s2[(GP + g) * SI + r] = out[g];
    }
  }
}

// u = Phi c on the q^3 grid (generalised tensor product; stages as plan3d.ClassTables3 tables)
template <int S, int N, bool PD>
__device__ void bwd(const double* __restrict__ c, double* __restrict__ u, double* s1, double* s2,
                    const double* __restrict__ A, const double* __restrict__ B, const double* __restrict__ Ct,
                    const int* gstart, const int* gmem, const int* coff) {
  using C = Cfg<S, N>;
  constexpr int Q = C::Q, NG = C::NG, NT = nthreads<Q>();
  const int t = threadIdx.x;
  if (S == H3_HEX) {
    for (int r = t; r < N * N; r += NT) {        // (i0, i1) pencils: i2 -> k2
      double col[N], out[Q];
#pragma unroll
      for (int i = 0; i < N; ++i) col[i] = c[r * N + i];
      cmat<Q, N>(c3A<S, N>, 0, col, out);
#pragma unroll
      for (int k = 0; k < Q; ++k) s1[r * Q + k] = out[k];
    }
    __syncthreads();
    for (int r = t; r < N * Q; r += NT) {        // (i0, k2) pencils: i1 -> k1
      const int i0 = r / Q, k2 = r % Q;
      double col[N], out[Q];
#pragma unroll
      for (int i = 0; i < N; ++i) col[i] = s1[(i0 * N + i) * Q + k2];
      cmat<Q, N>(c3A<S, N>, 0, col, out);
#pragma unroll
      for (int k = 0; k < Q; ++k) s2[i0 * C::template sj<PD>() * Q + k * C::template sj<PD>() + k2] = out[k];
    }
    __syncthreads();
    pencil_stage_a<S, N, PD>(s2, u);
    __syncthreads();
    return;
  }
  // stage 1: the innermost family (prism: psi on eta1 per triangle mode; tet: C rows on eta2)
  if (S == H3_PRISM) {
    for (int m = t; m < C::NPM; m += NT) {     // triangle-mode pencils: l -> k1
      double col[N], out[Q];
#pragma unroll
      for (int l = 0; l < N; ++l) col[l] = c[m * N + l];
      cmat<Q, N>(c3P<S, N>, 0, col, out);
#pragma unroll
      for (int k = 0; k < Q; ++k) s1[m * Q + k] = out[k];
    }
  } else {
    for (int o = t; o < C::NPM * Q; o += NT) {
      const int k = o % Q, m = o / Q;
      double a = 0.0;
      const int r0 = coff[m], cnt = coff[m + 1] - r0;   // <= N - 1 modes per triangle mode
#pragma unroll
      for (int kk = 0; kk < N - 1; ++kk)
        if (kk < cnt) a = fma(Ct[(r0 + kk) * Q + k], c[r0 + kk], a);
      s1[o] = a;
    }
  }
  __syncthreads();
  // stage 2: group sums with the B rows (prism: B on eta2, s1 over eta1; tet: B on eta1, s1 over eta2)
  // (g, ko, part) pencils over a part of kb: prism kb = k2, ko = k1; tet kb = k1, ko = k2 (the kb
  // range is split so that every thread has work)
  {
    constexpr int KS = (NT / (NG * Q)) < 1 ? 1 : ((NT / (NG * Q)) > Q ? Q : NT / (NG * Q));
    constexpr int KP = (Q + KS - 1) / KS;
    for (int it = t; it < NG * Q * KS; it += NT) {
      const int part = it % KS, go = it / KS;
      const int g = go / Q, ko = go % Q;
      const int kb0 = part * KP;
      double out[KP];
#pragma unroll
      for (int k = 0; k < KP; ++k) out[k] = 0.0;
      constexpr int GMAX = N - 1 > 2 ? N - 1 : 2;   // members per group (tet n = 2: vertex + apex)
      const int q0 = gstart[g], cntg = gstart[g + 1] - q0;
#pragma unroll
      for (int qq = 0; qq < GMAX; ++qq) {
        if (qq >= cntg) break;
        const int m = gmem[q0 + qq];
        const double sv = s1[m * Q + ko];
        const double* Br = B + m * Q + kb0;
#pragma unroll
        for (int k = 0; k < KP; ++k)
          if (kb0 + k < Q) out[k] = fma(Br[k], sv, out[k]);
      }
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        if (kb0 + k >= Q) break;
        if (S == H3_PRISM) s2[g * C::template sj<PD>() * Q + ko * C::template sj<PD>() + kb0 + k] = out[k];
        else s2[g * C::template sj<PD>() * Q + (kb0 + k) * C::template sj<PD>() + ko] = out[k];
      }
    }
  }
  __syncthreads();
  pencil_stage_a<S, N, PD>(s2, u);
  __syncthreads();
}

// y = Phi^T T (transposed stages), written to global
template <int S, int N, bool PD>
__device__ void bwd_t(const double* __restrict__ T, double* __restrict__ y, double* s1, double* s2,
                      const double* __restrict__ A, const double* __restrict__ B, const double* __restrict__ Ct,
                      const int* gof, const int* mofr) {
  using C = Cfg<S, N>;
  constexpr int Q = C::Q, NT = nthreads<Q>();
  const int t = threadIdx.x;
  if (S == H3_HEX) {
    pencil_stage_a_t<S, N, PD>(T, s2);             // k0 -> i0
    __syncthreads();
    for (int r = t; r < N * Q; r += NT) {        // (i0, k2) pencils: k1 -> i1
      const int i0 = r / Q, k2 = r % Q;
      double col[Q], out[N];
#pragma unroll
      for (int k = 0; k < Q; ++k) col[k] = s2[i0 * C::template sj<PD>() * Q + k * C::template sj<PD>() + k2];
      cmatT<Q, N>(c3A<S, N>, 0, col, out);
#pragma unroll
      for (int i = 0; i < N; ++i) s1[(i0 * N + i) * Q + k2] = out[i];
    }
    __syncthreads();
    for (int r = t; r < N * N; r += NT) {        // (i0, i1) pencils: k2 -> i2
      double col[Q], out[N];
#pragma unroll
      for (int k = 0; k < Q; ++k) col[k] = s1[r * Q + k];
      cmatT<Q, N>(c3A<S, N>, 0, col, out);
#pragma unroll
      for (int i = 0; i < N; ++i) y[r * N + i] = out[i];
    }
    return;
  }
  pencil_stage_a_t<S, N, PD>(T, s2);
  __syncthreads();
  for (int o = t; o < C::NPM * Q; o += NT) {
    const int k = o % Q, m = o / Q, g = gof[m];
    double a = 0.0;
    if (S == H3_PRISM) {   // s1[m][k1] = sum_k2 B[m][k2] s2[g][k1][k2]
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) a = fma(B[m * Q + k2], s2[g * C::template sj<PD>() * Q + k * C::template sj<PD>() + k2], a);
    } else {               // s1[m][k2] = sum_k1 B[m][k1] s2[g][k1][k2]
#pragma unroll
      for (int k1 = 0; k1 < Q; ++k1) a = fma(B[m * Q + k1], s2[g * C::template sj<PD>() * Q + k1 * C::template sj<PD>() + k], a);
    }
    s1[o] = a;
  }
  __syncthreads();
  if (S == H3_PRISM) {
    for (int m = t; m < C::NPM; m += NT) {     // triangle-mode pencils: k1 -> l
      double col[Q], out[N];
#pragma unroll
      for (int k = 0; k < Q; ++k) col[k] = s1[m * Q + k];
      cmatT<Q, N>(c3P<S, N>, 0, col, out);
#pragma unroll
      for (int l = 0; l < N; ++l) y[m * N + l] = out[l];
    }
    return;
  }
  for (int r = t; r < C::NC; r += NT) {
    double a = 0.0;
    {
      const int m = mofr[r];
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) a = fma(Ct[r * Q + k2], s1[m * Q + k2], a);
    }
    y[r] = a;
  }
}

// ---------------------------------------------------------------------------------------------
// per-element shared-memory layout
template <int S, int N>
struct Lay {
  using C = Cfg<S, N>;
  double *c, *u, *du, *s1, *s2, *F, *hdr, *tb, *cbuf, *hbuf, *ebuf;
  double *pts, *R, *D, *W, *E, *ED, *B, *Ct;
  int *gstart, *gmem, *gof, *coff, *mofr;
  __device__ Lay(double* sm, bool pub) {
    constexpr int Q = C::Q, Q2 = C::Q2;
    pts = sm;
    R = pts + 3 * Q;
    D = R + 3 * Q;
    W = D + 3 * Q2;          // w0 (Q) then w1 w2 Duffy (Q2)
    E = W + Q + Q2;
    ED = E + 6 * Q;
    B = ED + 6 * Q;
    Ct = B + C::TB;
    cbuf = sm + C::TABD;                 // [2][NCP]
    c = cbuf;
    u = cbuf + 2 * C::NCP;
    du = u + (pub ? C::template v3<h3_pad<true>()>() : C::template v3<h3_pad<false>()>());
    F = du + (pub ? 0 : 3 * C::template v3<h3_pad<false>()>());   // [NSMAX][2][Q2]: own-face-grid arrays per slot
    hbuf = F + C::NSMAX * 2 * C::Q2;     // [2][NSMAX][12]: slot headers
    hdr = hbuf;
    ebuf = hbuf + 2 * C::NSMAX * C::SLOTD;   // [2][H3_EGEO]: element geometry, double-buffered
    tb = ebuf + 2 * H3_EGEO;             // [SB][4][TMAX]: trace values / flux / map temporaries,
    s1 = tb;                             // shared with the BwdTrans stages (never live together)
    s2 = s1 + C::S1;
    gstart = (int*)(tb + C::SCR);
    gmem = gstart + C::NPM + 2;
    gof = gmem + C::NPM;
    coff = gof + C::NPM;
    mofr = coff + C::NPM + 2;
  }
};

__device__ __forceinline__ const H3Slot& slot_hdr(const double* hdr, int s) {
  return *reinterpret_cast<const H3Slot*>(hdr + 12 * s);
}

// items of a batch of <= 4 slots [b0, b0 + nb): prefix offsets computed once per phase, the slot of
// an item found with three compares (no loops over slot headers per item)
struct Batch {
  int b0, o1, o2, o3, tot;
  template <typename CountFn>
  __device__ __forceinline__ Batch(int b0_, int nb, CountFn cnt) : b0(b0_) {
    const int c0 = cnt(b0);
    const int c1 = nb > 1 ? cnt(b0 + 1) : 0;
    const int c2 = nb > 2 ? cnt(b0 + 2) : 0;
    const int c3 = nb > 3 ? cnt(b0 + 3) : 0;
    o1 = c0;
    o2 = o1 + c1;
    o3 = o2 + c2;
    tot = o3 + c3;
  }
  // global item -> slot; `it` becomes the index within the slot
  __device__ __forceinline__ int slot(int& it) const {
    const int j = (it >= o1) + (it >= o2) + (it >= o3);
    it -= j == 0 ? 0 : (j == 1 ? o1 : (j == 2 ? o2 : o3));
    return b0 + j;
  }
};

__device__ __forceinline__ void unpack_nab(int nab, int& n1, int& n2, int& swap) {
  n1 = nab & 255;
  n2 = (nab >> 8) & 255;
  swap = (nab >> 16) & 1;
}

// own-face-grid arrays (F[s][0], F[s][1]) -> trace arrays (tb[j][0], tb[j][1]) for the slots of a
// batch; with `pub`, the trace values go straight to the published buffer instead
template <int Q>
__device__ void map_forward(const double* hdr, const double* F, double* tb, int b0, int nb, const double* tab,
                            double* pub, bool only_interior, bool skip_identity = false) {
  constexpr int Q2 = Q * Q, NT = nthreads<Q>();
  const int t = threadIdx.x;
  auto active = [&](int s) {
    const H3Slot& h = slot_hdr(hdr, s);
    return (!only_interior || h.kind == 1) && !(skip_identity && h.mkind == MAP_ID);
  };
  // stage 1: tensor X contraction over own axis 0; dense and identity complete here
  auto c1 = [&](int s) -> int {
    if (!active(s)) return 0;
    const H3Slot& h = slot_hdr(hdr, s);
    if (h.mkind == MAP_TENSOR) return (h.nab & 255) * Q;
    if (h.mkind == MAP_ROW) return ((h.nab >> 8) & 255) * Q;
    return h.mkind == MAP_DENSE ? h.nt : Q2;
  };
  const Batch B1(b0, nb, c1);
  for (int it0 = t; it0 < B1.tot; it0 += NT) {
    int it = it0;
    const int s = B1.slot(it);
    const H3Slot& h = slot_hdr(hdr, s);
    const double* fu = F + s * 2 * Q2;
    const double* fg = fu + Q2;
    double* tu = tb + (s - b0) * 4 * TMAX;
    double* tg = tu + TMAX;
    if (h.mkind == MAP_ROW) {
      // subface quad side: tmp[pb][i_par] = sum_i_perp Y[pb][i_perp] f(i_par, i_perp)
      const int pb = it / Q, ipar = it % Q, perp = (h.nab >> 16) & 1;
      const double* Yr = tab + h.moff2 + pb * Q;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int ip = 0; ip < Q; ++ip) {
        const double m = __ldg(Yr + ip);
        const int o = perp ? ipar * Q + ip : ip * Q + ipar;
        a0 = fma(m, fu[o], a0);
        a1 = fma(m, fg[o], a1);
      }
      tu[2 * TMAX + it] = a0;
      tu[3 * TMAX + it] = a1;
    } else if (h.mkind == MAP_TENSOR) {
      const int r1 = it / Q, ib = it % Q;
      const double* X = tab + h.moff + r1 * Q;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int ia = 0; ia < Q; ++ia) {
        const double m = __ldg(X + ia);
        a0 = fma(m, fu[ia * Q + ib], a0);
        a1 = fma(m, fg[ia * Q + ib], a1);
      }
      tu[2 * TMAX + it] = a0;
      tu[3 * TMAX + it] = a1;
    } else {
      double a0, a1;
      if (h.mkind == MAP_DENSE) {
        const double* M = tab + h.moff + (int64_t)it * Q2;
        a0 = 0.0;
        a1 = 0.0;
        for (int a = 0; a < Q2; ++a) {
          const double m = __ldg(M + a);
          a0 = fma(m, fu[a], a0);
          a1 = fma(m, fg[a], a1);
        }
      } else {
        a0 = fu[it];
        a1 = fg[it];
      }
      if (pub) {
        double* dst = pub + h.pub_self;
        dst[2 * it] = a0;
        dst[2 * it + 1] = a1;
      } else {
        tu[it] = a0;
        tg[it] = a1;
      }
    }
  }
  __syncthreads();
  // stage 2: tensor Y contraction over own axis 1
  auto c2 = [&](int s) -> int {
    if (!active(s)) return 0;
    const H3Slot& h = slot_hdr(hdr, s);
    return (h.mkind == MAP_TENSOR || h.mkind == MAP_ROW) ? h.nt : 0;
  };
  const Batch B2(b0, nb, c2);
  if (B2.tot == 0) return;
  for (int it0 = t; it0 < B2.tot; it0 += NT) {
    int it = it0;
    const int s = B2.slot(it);
    const H3Slot& h = slot_hdr(hdr, s);
    int n1, n2, sw;
    unpack_nab(h.nab, n1, n2, sw);
    double* tu = tb + (s - b0) * 4 * TMAX;
    int p;
    const double *Y, *m0, *m1;
    if (h.mkind == MAP_ROW) {   // t[pa, pb] = sum_i_par X[pb][pa][i_par] tmp[pb][i_par]
      const int pa = it / n2, pb = it % n2;
      p = it;
      Y = tab + h.moff + (pb * n1 + pa) * Q;
      m0 = tu + 2 * TMAX + pb * Q;
      m1 = tu + 3 * TMAX + pb * Q;
    } else {
      const int r1 = it / n2, r2 = it % n2;
      p = sw ? r2 * n1 + r1 : r1 * n2 + r2;
      Y = tab + h.moff2 + r2 * Q;
      m0 = tu + 2 * TMAX + r1 * Q;
      m1 = tu + 3 * TMAX + r1 * Q;
    }
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int ib = 0; ib < Q; ++ib) {
      const double m = __ldg(Y + ib);
      a0 = fma(m, m0[ib], a0);
      a1 = fma(m, m1[ib], a1);
    }
    if (pub) {
      double* dst = pub + h.pub_self;
      dst[2 * p] = a0;
      dst[2 * p + 1] = a1;
    } else {
      tu[p] = a0;
      tu[TMAX + p] = a1;
    }
  }
  __syncthreads();
}

// trace arrays (tb[j][0], tb[j][1]) -> own-face-grid arrays F[s][0], F[s][1] (transposed maps)
template <int S, int Q>
__device__ void map_transpose(const double* hdr, double* F, double* tb, int b0, int nb, const double* tab,
                              const double* pts, const double* R) {
  constexpr int Q2 = Q * Q, NT = nthreads<Q>();
  const int t = threadIdx.x;
  auto c1 = [&](int s) -> int {
    const H3Slot& h = slot_hdr(hdr, s);
    if (h.mkind == MAP_ROW) return ((h.nab >> 8) & 255) * Q;
    return h.mkind == MAP_TENSOR ? (h.nab & 255) * Q : 0;
  };
  const Batch B1(b0, nb, c1);
  if (B1.tot > 0) {
    for (int it0 = t; it0 < B1.tot; it0 += NT) {
      int it = it0;
      const int s = B1.slot(it);
      const H3Slot& h = slot_hdr(hdr, s);
      int n1, n2, sw;
      unpack_nab(h.nab, n1, n2, sw);
      const int r1 = it / Q, ib = it % Q;
      double* tv = tb + (s - b0) * 4 * TMAX;
      double a0 = 0.0, a1 = 0.0;
      if (h.mkind == MAP_ROW) {   // tmp[pb][i_par] = sum_pa X[pb][pa][i_par] g[pa, pb]
        for (int pa = 0; pa < n1; ++pa) {
          const double m = __ldg(tab + h.moff + (r1 * n1 + pa) * Q + ib);
          a0 = fma(m, tv[pa * n2 + r1], a0);
          a1 = fma(m, tv[TMAX + pa * n2 + r1], a1);
        }
        tv[2 * TMAX + it] = a0;
        tv[3 * TMAX + it] = a1;
        continue;
      }
      const double* Yc = tab + h.moff2 + ib;
      const int pst = sw ? n1 : 1;
      int p = sw ? r1 : r1 * n2;
      for (int r2 = 0; r2 < n2; ++r2, p += pst) {
        const double m = __ldg(Yc + r2 * Q);
        a0 = fma(m, tv[p], a0);
        a1 = fma(m, tv[TMAX + p], a1);
      }
      tv[2 * TMAX + it] = a0;
      tv[3 * TMAX + it] = a1;
    }
    __syncthreads();
  }
  const int n2tot = nb * Q2;
  for (int it0 = t; it0 < n2tot; it0 += NT) {
    const int s = b0 + it0 / Q2, a = it0 % Q2;
    const H3Slot& h = slot_hdr(hdr, s);
    double* tv = tb + (s - b0) * 4 * TMAX;
    double a0, a1;
    if (h.mkind == MAP_ROW) {   // F(i_par, i_perp) = sum_pb Y[pb][i_perp] tmp[pb][i_par]
      const int n2 = (h.nab >> 8) & 255, perp = (h.nab >> 16) & 1;
      const int ipar = perp ? a / Q : a % Q, iperp = perp ? a % Q : a / Q;
      a0 = 0.0;
      a1 = 0.0;
      for (int pb = 0; pb < n2; ++pb) {
        const double m = __ldg(tab + h.moff2 + pb * Q + iperp);
        a0 = fma(m, tv[2 * TMAX + pb * Q + ipar], a0);
        a1 = fma(m, tv[3 * TMAX + pb * Q + ipar], a1);
      }
    } else if (h.mkind == MAP_TENSOR) {
      const int n1 = h.nab & 255, ia = a / Q, ib = a % Q;
      a0 = 0.0;
      a1 = 0.0;
      const double* Xc = tab + h.moff + ia;
      const double* t0 = tv + 2 * TMAX + ib;
#pragma unroll 4
      for (int r1 = 0; r1 < n1; ++r1) {
        const double m = __ldg(Xc + r1 * Q);
        a0 = fma(m, t0[r1 * Q], a0);
        a1 = fma(m, t0[TMAX + r1 * Q], a1);
      }
    } else if (h.mkind == MAP_DENSE) {
      a0 = 0.0;
      a1 = 0.0;
      for (int p = 0; p < h.nt; ++p) {
        const double m = __ldg(tab + h.moff + (int64_t)p * Q2 + a);
        a0 = fma(m, tv[p], a0);
        a1 = fma(m, tv[TMAX + p], a1);
      }
    } else {
      a0 = tv[a];
      a1 = tv[TMAX + a];
    }
    F[s * 2 * Q2 + a] = a0;
    F[s * 2 * Q2 + Q2 + a] = a1;
  }
  __syncthreads();
  // (G n)_k fd on the own face grid for the scatter (the chain evaluated once per face point), into
  // the now consumed trace buffers
  for (int it0 = t; it0 < n2tot; it0 += NT) {
    const int s = b0 + it0 / Q2, a = it0 % Q2;
    const H3Slot& h = slot_hdr(hdr, s);
    const int fx = c_faces[S][h.face][0], sd = c_faces[S][h.face][1];
    const int ra = c_faces[S][h.face][2], rb = c_faces[S][h.face][3];
    const Chain ch = face_chain<S>(pts, R, Q, fx, sd, ra, rb, a / Q, a % Q);
    const double fd = F[s * 2 * Q2 + Q2 + a];
    double* gd = tb + (s - b0) * 4 * TMAX;
    gd[a] = (ch.c00 * h.v[0] + ch.c01 * h.v[1] + ch.c02 * h.v[2]) * fd;
    gd[Q2 + a] = (ch.c11 * h.v[1] + ch.c12 * h.v[2]) * fd;
    gd[2 * Q2 + a] = h.v[2] * fd;
  }
  __syncthreads();
}

// resident CTAs per SM the register allocation must allow (q >= 7: 128 threads, else 64)
#ifndef SIPG_H3_PUB_MINB_HI
#define SIPG_H3_PUB_MINB_HI 6
#endif
#ifndef SIPG_H3_PUB_MINB_LO
#define SIPG_H3_PUB_MINB_LO 12
#endif
template <bool PUB, int Q>
constexpr int h3_minb() {
  return PUB ? (Q > SIPG_H3_NT64_QMAX ? SIPG_H3_PUB_MINB_HI : SIPG_H3_PUB_MINB_LO)
             : (Q > SIPG_H3_NT64_QMAX ? SIPG_H3_APP_MINB_HI : 12);
}

template <int S, int N, bool PUB>
__global__ void __launch_bounds__(nthreads<N + 1>(), h3_minb<PUB, N + 1>()) k_h3(const H3Plan P, const int cls, const double* __restrict__ x,
                                                          double* __restrict__ y) {
  using C = Cfg<S, N>;
  constexpr int Q = C::Q, Q2 = C::Q2, Q3 = C::Q3, NT = nthreads<Q>();
  constexpr bool PD = h3_pad<PUB>();   // volume layout of this kernel kind
  extern __shared__ double sm[];
  Lay<S, N> L(sm, PUB);
  const int t = threadIdx.x;
  const int32_t* cd = P.cd + cls * CD3_WORDS;
  const int count = cd[CD3_COUNT];
  {   // stage the class tables (a few KB) in shared memory
    auto cp = [&](double* dst, int word, int n) {
      const double* src = P.tab + cd[word];
      for (int r = t; r < n; r += NT) dst[r] = __ldg(src + r);
    };
    cp(L.pts, CD3_T_PTS, 3 * Q);
    cp(L.R, CD3_T_R, 3 * Q);
    cp(L.D, CD3_T_D, 3 * Q2);
    cp(L.W, CD3_T_W, Q + Q2);
    cp(L.E, CD3_T_E, 6 * Q);
    cp(L.ED, CD3_T_ED, 6 * Q);
    if (S != H3_HEX) cp(L.B, CD3_T_B, C::TB);
  }
  const double* pts = L.pts;
  const double* Rt = L.R;
  const double* Dt = L.D;
  const double* Wr = L.W;
  const double* Et = L.E;
  const double* EDt = L.ED;
  const double* At = P.tab + cd[CD3_T_A];
  const double* Bt = S == H3_HEX ? At : L.B;
  const double* Ct = S == H3_TET ? P.tab + cd[CD3_T_C] : At;
  if (S != H3_HEX) build_int_tables<S, N>(L.gstart, L.gmem, L.gof, L.coff, L.mofr);
  // element pipeline: scalars (element id, DoF and slot offsets) two elements ahead in registers,
  // coefficients + slot headers one element ahead by cp.async into the other buffer
  const int G = gridDim.x;
  const int32_t* ce = P.class_elems + cd[CD3_ELEM_OFF];
  auto scalars = [&](int i, int& e, int64_t& dof, int64_t& sb, int& ns) {
    if (i < count) {
      e = __ldg(ce + i);
      dof = __ldg(P.dof_off + e);
      sb = __ldg(P.slot_off + e);
      ns = (int)(__ldg(P.slot_off + e + 1) - sb);
    }
  };
  // coefficients, slot headers and (apply) the element geometry of the next element, by cp.async
  auto issue = [&](int buf, int e, int64_t dof, int64_t sb, int ns) {
    double* cd_ = L.cbuf + buf * C::NCP;
    double* hd_ = L.hbuf + buf * C::NSMAX * C::SLOTD;
    for (int r = t; r < C::NC; r += NT) __pipeline_memcpy_async(cd_ + r, x + dof + r, sizeof(double));
    const double* src = reinterpret_cast<const double*>(P.slots + sb);
    for (int r = t; r < ns * C::SLOTD; r += NT) __pipeline_memcpy_async(hd_ + r, src + r, sizeof(double));
    if (!PUB && SIPG_H3_EGEO_ASYNC && t < H3_EGEO / 2)
      __pipeline_memcpy_async(L.ebuf + buf * H3_EGEO + 2 * t, P.egeo + (int64_t)e * H3_EGEO + 2 * t, 2 * sizeof(double));
    __pipeline_commit();
  };
  int64_t dof_n = 0, sb_n = 0, dof_nn = 0, sb_nn = 0;   // next and next-but-one element
  int ns_n = 0, ns_nn = 0, e_n = 0, e_nn = 0;
  scalars(blockIdx.x, e_n, dof_n, sb_n, ns_n);
  if ((int)blockIdx.x < count) issue(0, e_n, dof_n, sb_n, ns_n);
  scalars(blockIdx.x + G, e_nn, dof_nn, sb_nn, ns_nn);
  int it_el = 0;
  for (int i = blockIdx.x; i < count; i += G, ++it_el) {
    const int bsel = it_el & 1;
    __pipeline_wait_prior(0);
    __syncthreads();
    L.c = L.cbuf + bsel * C::NCP;
    L.hdr = L.hbuf + bsel * C::NSMAX * C::SLOTD;
    const double* eg = SIPG_H3_EGEO_ASYNC ? L.ebuf + bsel * H3_EGEO : P.egeo + (int64_t)__ldg(ce + i) * H3_EGEO;
    const int64_t dof = dof_n;
    const int ns = ns_n;
    if (i + G < count) issue(bsel ^ 1, e_nn, dof_nn, sb_nn, ns_nn);
    dof_n = dof_nn;
    sb_n = sb_nn;
    ns_n = ns_nn;
    e_n = e_nn;
    scalars(i + 2 * G, e_nn, dof_nn, sb_nn, ns_nn);
    bwd<S, N, PD>(L.c, L.u, L.s1, L.s2, At, Bt, Ct, L.gstart, L.gmem, L.coff);
    if (PUB) {
      // own-face-grid u and n.grad u of the interior slots from u alone: endpoint rows for u and
      // d/d eta_fixed (E D), collocation on the face grid for the two tangential derivatives
      for (int it = t; it < ns * Q2; it += NT) {
        const int s = it / Q2, a = it % Q2;
        const H3Slot& h = slot_hdr(L.hdr, s);
        const int fx = c_faces[S][h.face][0], sd = c_faces[S][h.face][1];
        const int ra = c_faces[S][h.face][2], rb = c_faces[S][h.face][3];
        const int st_f = fx == 0 ? C::template sj<PD>() * Q : (fx == 1 ? C::template sj<PD>() : 1);
        const int st_a = ra == 0 ? C::template sj<PD>() * Q : (ra == 1 ? C::template sj<PD>() : 1);
        const int st_b = rb == 0 ? C::template sj<PD>() * Q : (rb == 1 ? C::template sj<PD>() : 1);
        const double* E = Et + (fx * 2 + (sd > 0)) * Q;
        const double* ED = EDt + (fx * 2 + (sd > 0)) * Q;
        const int base = (a / Q) * st_a + (a % Q) * st_b;
        double uf = 0.0, un = 0.0;
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          const double uv = L.u[base + k * st_f];
          uf = fma(*(E + k), uv, uf);
          un = fma(*(ED + k), uv, un);
        }
        L.F[s * 2 * Q2 + a] = uf;
        L.F[s * 2 * Q2 + Q2 + a] = un;
      }
      __syncthreads();
      for (int it = t; it < ns * Q2; it += NT) {
        const int s = it / Q2, a = it % Q2;
        const H3Slot& h = slot_hdr(L.hdr, s);
        const int fx = c_faces[S][h.face][0], sd = c_faces[S][h.face][1];
        const int ra = c_faces[S][h.face][2], rb = c_faces[S][h.face][3];
        const int ia = a / Q, ib = a % Q;
        const double* fu = L.F + s * 2 * Q2;
        double da = 0.0, db = 0.0;
#pragma unroll
        for (int j = 0; j < Q; ++j) {
          da = fma(*(Dt + ra * Q2 + ia * Q + j), fu[j * Q + ib], da);
          db = fma(*(Dt + rb * Q2 + ib * Q + j), fu[ia * Q + j], db);
        }
        const Chain ch = face_chain<S>(pts, Rt, Q, fx, sd, ra, rb, ia, ib);
        const double g0 = ch.c00 * h.v[0] + ch.c01 * h.v[1] + ch.c02 * h.v[2];
        const double g1 = ch.c11 * h.v[1] + ch.c12 * h.v[2];
        const double g2 = h.v[2];
        const double gf = fx == 0 ? g0 : (fx == 1 ? g1 : g2);
        const double ga = ra == 0 ? g0 : (ra == 1 ? g1 : g2);
        const double gb = rb == 0 ? g0 : (rb == 1 ? g1 : g2);
        const double gv = gf * fu[Q2 + a] + ga * da + gb * db;
        if (SIPG_H3_PUB_DIRECT && h.mkind == MAP_ID)   // own face grid = trace grid: straight to the published buffer
          reinterpret_cast<double2*>(P.pub + h.pub_self)[a] = make_double2(fu[a], gv);
        else
          L.F[s * 2 * Q2 + Q2 + a] = gv;
      }
      bool mapped = false;
      for (int j = 0; j < ns; ++j) mapped |= !SIPG_H3_PUB_DIRECT || slot_hdr(L.hdr, j).mkind != MAP_ID;
      if (mapped) {
        __syncthreads();
        for (int b0 = 0; b0 < ns; b0 += C::SB)
          map_forward<Q>(L.hdr, L.F, L.tb, b0, min(C::SB, ns - b0), P.tab, P.pub, false, SIPG_H3_PUB_DIRECT);
      }
      continue;
    }
    // SIP flux at the trace points of the slots [b0, b0 + nb) (sipg.py:622-650, 663-677) from the
    // published own and partner traces (the publish kernel evaluated both; boundary: jump 2u,
    // average g), then the transposed maps onto the own face grids: fv / fd in F, (G n)_k fd in the
    // trace scratch.  Needs only the trace scratch, so the first batch runs right after BwdTrans
    // and its lift rides on the volume-term pass below (SIPG_H3_FUSE_LIFT).
    auto face_batch = [&](const int b0, const int nb) {
        // SIP flux at the trace points (sipg.py:622-650, 663-677) from the published own and partner
        // traces (the publish kernel evaluated both); boundary: jump 2u, average g
        {
          auto cnt = [&](int s) -> int { return slot_hdr(L.hdr, s).nt; };
          const Batch BF(b0, nb, cnt);
          for (int it0 = t; it0 < BF.tot; it0 += NT) {
            int p = it0;
            const int s = BF.slot(p);
            const H3Slot& h = slot_hdr(L.hdr, s);
            double* tv = L.tb + (s - b0) * 4 * TMAX;
            const double2 own = __ldg(reinterpret_cast<const double2*>(P.pub + h.pub_self) + p);
            const double ut = own.x, gt = own.y;
            double un, gn;
            if (h.kind) {
              const double2 nbv = __ldg(reinterpret_cast<const double2*>(P.pub + h.pub_other) + p);
              un = nbv.x;
              gn = nbv.y;
            } else {
              un = -ut;
              gn = -gt;
            }
            const double j = ut - un, cc = 0.5 * (gt - gn);
            const double w = h.sJ * __ldg(P.tab + h.wtoff + p);
            tv[p] = (h.tau * j - cc) * w;
            tv[TMAX + p] = -0.5 * j * w;
          }
        }
        __syncthreads();
        map_transpose<S, Q>(L.hdr, L.F, L.tb, b0, nb, P.tab, pts, Rt);
    };
    // the lift of a batch's faces at one volume point: the transposed endpoint rows of fv and of the
    // (G n)_k fd arrays (the reference's scatter + final sweep)
    // a batch's face geometry packed into registers: per slot 3 bits (fixed axis * 2 + side)
    struct Lift {
      int pack, nb, b0;
    };
    auto lift_setup = [&](Lift& lf, const int b0, const int nb) {
      lf.nb = nb;
      lf.b0 = b0;
      lf.pack = 0;
#pragma unroll
      for (int j = 0; j < C::SB; ++j) {
        const int face = slot_hdr(L.hdr, j < nb ? b0 + j : b0).face;
        lf.pack |= (c_faces[S][face][0] * 2 + (c_faces[S][face][1] > 0)) << (3 * j);
      }
    };
    auto lift_at = [&](const Lift& lf, int k0, int k1, int k2, double& w0, double& w1, double& w2, double& w3) {
#pragma unroll
      for (int j = 0; j < C::SB; ++j) {
        if (j >= lf.nb) break;
        const int code = (lf.pack >> (3 * j)) & 7, fx = code >> 1;
        const int kf = fx == 0 ? k0 : (fx == 1 ? k1 : k2);
        const int a = fx == 0 ? k1 * Q + k2 : (fx == 1 ? k0 * Q + k2 : k0 * Q + k1);
        const double ek = Et[code * Q + kf];
        if (S != H3_TET && ek == 0.0) continue;   // GLL endpoint rows are one-hot
        const double* Fs = L.F + (lf.b0 + j) * 2 * Q2;
        const double* Gs = L.tb + j * 4 * TMAX;
        w0 = fma(ek, Fs[a], w0);
        w1 = fma(ek, Gs[a], w1);
        w2 = fma(ek, Gs[Q2 + a], w2);
        w3 = fma(ek, Gs[2 * Q2 + a], w3);
      }
    };
    constexpr bool FUSE = SIPG_H3_FUSE_LIFT;
    const int nb0 = ns < C::SB ? ns : C::SB;
    if (FUSE && nb0 > 0) face_batch(0, nb0);
    // PhysDeriv: collocation along each eta axis (stdregions.py:658-674)
    pencil_deriv<S, N, PD>(L.u, L.du);
    __syncthreads();
    // volume terms (sipg.py:575-582), in place: W0 = lambda jw u (u), W_k = jw (G G^T grad u)_k (du),
    // plus the first face batch's lift
    {
      Lift lf0;
      lift_setup(lf0, 0, FUSE ? nb0 : 0);
      const double lam = P.lam;
      double mt[7];
#pragma unroll
      for (int q = 0; q < 7; ++q) mt[q] = FUSE ? 0.0 : eg[q];   // hoisted (the fused lift re-reads: spills)
      for (int o0 = t; o0 < Q3; o0 += NT) {
        const double dJ = FUSE ? eg[0] : mt[0], S00 = FUSE ? eg[1] : mt[1], S01 = FUSE ? eg[2] : mt[2],
                     S02 = FUSE ? eg[3] : mt[3], S11 = FUSE ? eg[4] : mt[4], S12 = FUSE ? eg[5] : mt[5],
                     S22 = FUSE ? eg[6] : mt[6];
        const int k0 = o0 / Q2, k1 = (o0 / Q) % Q, k2 = o0 % Q;
        const int o = k0 * C::template sj<PD>() * Q + k1 * C::template sj<PD>() + k2;
        const Chain ch = chain_t<S>(1.0 + *(pts + k0), 1.0 + *(pts + Q + k1), *(Rt + Q + k1),
                                    *(Rt + 2 * Q + k2));
        const double jw = dJ * Wr[k0] * Wr[Q + k1 * Q + k2];
        const double d0 = L.du[o], d1 = L.du[C::template v3<PD>() + o], d2 = L.du[2 * C::template v3<PD>() + o];
        const double x0 = ch.c00 * d0, x1 = ch.c01 * d0 + ch.c11 * d1, x2 = ch.c02 * d0 + ch.c12 * d1 + d2;
        const double f0 = S00 * x0 + S01 * x1 + S02 * x2;
        const double f1 = S01 * x0 + S11 * x1 + S12 * x2;
        const double f2 = S02 * x0 + S12 * x1 + S22 * x2;
        double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
        if (FUSE) lift_at(lf0, k0, k1, k2, w0, w1, w2, w3);
        L.u[o] = fma(lam * jw, L.u[o], w0);
        L.du[o] = fma(jw, ch.c00 * f0 + ch.c01 * f1 + ch.c02 * f2, w1);
        L.du[C::template v3<PD>() + o] = fma(jw, ch.c11 * f1 + ch.c12 * f2, w2);
        L.du[2 * C::template v3<PD>() + o] = fma(jw, f2, w3);
      }
    }
    __syncthreads();
    for (int b0 = FUSE ? C::SB : 0; b0 < ns; b0 += C::SB) {
      const int nb = min(C::SB, ns - b0);
      face_batch(b0, nb);
      {
        Lift lf;
        lift_setup(lf, b0, nb);
        for (int o0 = t; o0 < Q3; o0 += NT) {
          const int k0 = o0 / Q2, k1 = (o0 / Q) % Q, k2 = o0 % Q;
          const int o = k0 * C::template sj<PD>() * Q + k1 * C::template sj<PD>() + k2;
          double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
          lift_at(lf, k0, k1, k2, w0, w1, w2, w3);
          L.u[o] += w0;
          L.du[o] += w1;
          L.du[C::template v3<PD>() + o] += w2;
          L.du[2 * C::template v3<PD>() + o] += w3;
        }
      }
      __syncthreads();
    }
    // T = W0 + sum_k D_k^T W_k  (in place)
    pencil_dt<S, N, PD>(L.u, L.du);
    bwd_t<S, N, PD>(L.u, y + dof, L.s1, L.s2, At, Bt, Ct, L.gof, L.mofr);
    __syncthreads();
  }
}

}  // namespace h3
