// Config 4: shared definitions of the hybrid hex / prism / tet kernels (sm_100a, fp64) -- the plan
// structures of paper_2504_03573_b200/plan3d.py as the kernels see them, the per-(shape, n)
// __constant__ 1-D tables and their upload.  The kernels themselves: sipg_h3c.cuh.
//
// The reference's two-phase apply (pkg/src/dgsipg/sipg.py:558-602) on the shared-trace route
// (sipg.py:513-554 trace rule / geometry, 653-661 TracePhysEval, 663-677 absorb), extended to
// prisms and tets (collapsed-coordinate modified-modal bases built like the reference triangle,
// stdregions.py:266-383; restated and property-tested in oracle/hybrid3d.py).
#pragma once
#include <cuda_pipeline.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#define SIPG_H3_ABI_VERSION 1
// build knob: the publish kernels hand u (q^3 grid, 0.74 GB at 48^3) to the apply kernels, which then skip
// their BwdTrans.  Measured on cfg4: 3.87 -> 3.78 ms (tet n = 7 apply 0.395 -> 0.346 ms, the publish kernels
// 4 % slower), for 1.5 GB more DRAM traffic per apply and an apply kernel that moves 6 x its algorithmic
// bytes; left off.
#ifndef H3C_UHAND
#define H3C_UHAND 0
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
  // u on the q^3 grid, handed from the publish kernels to the apply kernels (element e from ug_off[e])
  double* ug;
  const int64_t* ug_off;
  // per class-list position: (element, n_slots, dof offset, first slot, fb offset, ug offset), 48 bytes -- what a
  // CTA needs to start an element, fetched by cp.async (no dependent global loads in the element loop)
  const long long* escal;
};
// what the flux kernel needs of a slot, 64 bytes, in work-list order (built by sipg_h3_plan_create)
struct H3FluxRec {
  int64_t pub_self, pub_other, fb_q;   // fb_q = (offset into fb) * 16 + q of the owning element
  double tau, sJ;
  int32_t nt, mk_kind, nab, moff, moff2, wtoff;   // mk_kind = mkind | kind << 8
};
static_assert(sizeof(H3FluxRec) == 64, "H3FluxRec layout");

namespace h3 {

constexpr int TMAX = 64;   // trace points per coupling: q_t = max(q_L, q_R) <= 8

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

// Register pencils with __constant__ 1-D tables: a thread loads one line of values along an axis into
// registers and produces the whole output line; with the loops fully unrolled every table entry is a
// compile-time constant-bank operand of its DFMA (uniform across the warp).
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

template <int S, int N>
cudaError_t h3_upload(const double* D, const double* A, const double* psi) {
  constexpr int Q = N + 1, NA = S == H3_HEX ? N : N + 1, H = Q / 2, EO = eo_size<Q>();
  cudaError_t e = cudaMemcpyToSymbol(c3A<S, N>, A, sizeof(double) * Q * NA);
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

}  // namespace h3
