#pragma once
// SIP-Helmholtz matrix-free apply, fp64, sm_100a.
//
// One fused kernel per element class (shape, n_modes, n_quad, geometry mode).
// Each CTA owns one element and writes its output coefficients exactly once
// (no atomics, deterministic):
//   1. BwdTrans        u  = (V x V x V) c                      (reference stdregions.py:575-597)
//   2. PhysDeriv       du_k = D_k u                              (stdregions.py:658-674)
//   3. trace values    own u, du on each face; the neighbour's u, du evaluated on
//                      ITS face grid straight from its coefficients (sum-factorised
//                      TracePhysEval, stdregions.py:704-758) — no trace buffers
//   4. SIP flux        jump / average / penalty per face point   (sipg.py:607-677)
//                      gather / certified p2p on the own face grid, shared trace on
//                      the trace grid with exact 1-D transfers  (trace.py:172-206)
//   5. lift            face fluxes folded into the volume point arrays (the
//                      reference's scatter + final sweep, sipg.py:663-693)
//   6. one transposed pass  y = IProduct(lam jw u + sum_k D_k^T (K du)_k + faces)
//                      using dV_k = D_k V (exact for q >= n), stdregions.py:600-655
#include <cuda_runtime.h>
#include <stdint.h>
#include "sipg_plan.h"

namespace sipg {

constexpr int QMAX = 11;   // largest supported points per direction
constexpr int NMAX = 10;   // largest supported modes per direction

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

__device__ __forceinline__ void cp_async8_(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit_() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all_() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// coefficient read that works for global (read-only path) and staged shared data
__device__ __forceinline__ double c_at(const double* p) { return __isShared(p) ? *p : __ldg(p); }

// A "team" works on one element: a whole CTA or a single warp.
struct CtaTeam { static __device__ __forceinline__ void sync() { __syncthreads(); } };
struct WarpTeam { static __device__ __forceinline__ void sync() { __syncwarp(); } };

// ---------------------------------------------------------------------------
// compile-time tensor contraction on shared memory.
// in: dims (S0,S1,S2) row-major, contract axis AX (size K) with M:
//   !TR: out[..r..] = sum_k M[r*K+k] in[..k..]   (M is R x K)
//    TR: out[..r..] = sum_k M[k*R+r] in[..k..]   (M is K x R, transposed use)
template <int S0, int S1, int S2, int AX, int R, bool TR, bool ACC>
__device__ __forceinline__ void contract(const double* __restrict__ in, double* __restrict__ out,
                                         const double* __restrict__ M, int tid, int nt) {
  constexpr int K = AX == 0 ? S0 : (AX == 1 ? S1 : S2);
  constexpr int O1 = AX == 1 ? R : S1, O2 = AX == 2 ? R : S2;
  constexpr int is0 = S1 * S2, is1 = S2;
  constexpr int os0 = O1 * O2, os1 = O2;
  constexpr int isk = AX == 0 ? is0 : (AX == 1 ? is1 : 1);
  constexpr int osk = AX == 0 ? os0 : (AX == 1 ? os1 : 1);
  constexpr int A = AX == 0 ? S1 : S0;
  constexpr int B = AX == 2 ? S1 : S2;
  constexpr int ia = AX == 0 ? is1 : is0, ib = AX == 2 ? is1 : 1;
  constexpr int oa = AX == 0 ? os1 : os0, ob = AX == 2 ? os1 : 1;
  for (int line = tid; line < A * B; line += nt) {
    const int a = line / B, b = line - (line / B) * B;
    const double* src = in + a * ia + b * ib;
    double* dst = out + a * oa + b * ob;
    double v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = src[k * isk];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) acc = fma(TR ? M[k * R + r] : M[r * K + k], v[k], acc);
      if (ACC) dst[r * osk] += acc; else dst[r * osk] = acc;
    }
  }
}

// ---------------------------------------------------------------------------
// face topology
struct FaceTopo { int fixed, side, run0, run1; };

__device__ __forceinline__ FaceTopo face_topo(int shape, int f) {
  FaceTopo t;
  if (shape == SHAPE_TRI) {
    if (f == 0) { t.fixed = 1; t.side = -1; t.run0 = 0; }
    else { t.fixed = 0; t.side = (f == 1) ? 1 : -1; t.run0 = 1; }
    t.run1 = -1;
    return t;
  }
  t.fixed = f >> 1;
  t.side = (f & 1) ? 1 : -1;
  if (shape == SHAPE_QUAD) { t.run0 = 1 - t.fixed; t.run1 = -1; }
  else { t.run0 = t.fixed == 0 ? 1 : 0; t.run1 = t.fixed == 2 ? 1 : 2; }
  return t;
}

// triangle collapse chain d eta/d xi at a face parameter: returns (c00, c01); c10=0, c11=1
__device__ __forceinline__ void tri_chain(int f, double p, double& c00, double& c01) {
  if (f == 0) { c00 = 1.0; c01 = 0.5 * (1.0 + p); }                 // eta2 = -1, eta1 = p
  else { const double s = (f == 1) ? 1.0 : -1.0; c00 = 2.0 / (1.0 - p); c01 = (1.0 + s) / (1.0 - p); }
}

// ---------------------------------------------------------------------------
// neighbour trace evaluation from coefficients, on the neighbour's own face grid.
// out[0*FP + p] = u, out[(1+k)*FP + p] = du/deta_k (neighbour axes).  Returns the
// number of face points.  Runtime sizes: only used for the face part.
template <class TM = CtaTeam>
static __device__ int eval_face_from_coeffs(const DevPlan& P, int e, int f, const double* __restrict__ x,
                                     double* __restrict__ out, int FP, double* __restrict__ scr,
                                     int tid, int nt, const double* staged = nullptr) {
  const int* cd = P.cd + P.elem_class[e] * CD_WORDS;
  const int shape = cd[CD_SHAPE], n = cd[CD_N];
  const double* c = staged ? staged : x + P.dof_off[e];
  const double* T = P.tab;
  const FaceTopo ft = face_topo(shape, f);
  if (shape == SHAPE_TRI) {
    const int ng = n + 1, nc = cd[CD_NC];
    const double* gst = T + cd[TR_GSTART];
    const double* gmo = T + cd[TR_GID];
    if (f == 0) {
      // eta2 = -1: contract direction 2 first, then direction-1 tables at the GL points
      const int q = cd[CD_Q0];
      double* tg = scr;          // ng
      double* dtg = scr + ng;    // ng
      for (int g = tid; g < ng; g += nt) {
        double a = 0.0, b = 0.0;
        const int j0 = (int)ldg(gst + g), j1 = (int)ldg(gst + g + 1);
        for (int j = j0; j < j1; ++j) {
          const int m = (int)ldg(gmo + j);
          const double cm = c_at(c + m);
          a = fma(ldg(T + cd[TR_BM1] + m), cm, a);
          b = fma(ldg(T + cd[TR_DBM1] + m), cm, b);
        }
        tg[g] = a; dtg[g] = b;
      }
      TM::sync();
      const double* A = T + cd[TR_A];
      const double* dA = T + cd[TR_DA];
      for (int p = tid; p < q; p += nt) {
        double u = 0.0, d0 = 0.0, d1 = 0.0;
        for (int g = 0; g < ng; ++g) {
          const double a = ldg(A + p * ng + g);
          u = fma(a, tg[g], u);
          d0 = fma(ldg(dA + p * ng + g), tg[g], d0);
          d1 = fma(a, dtg[g], d1);
        }
        out[p] = u; out[FP + p] = d0; out[2 * FP + p] = d1;
      }
      TM::sync();
      return q;
    }
    // eta1 = side: direction-1 row at the endpoint, direction-2 tables at the GL points
    const int q = cd[CD_Q1];
    const double* arow = T + cd[TR_AEND] + (ft.side > 0 ? ng : 0);
    const double* darow = T + cd[TR_DAEND] + (ft.side > 0 ? ng : 0);
    const double* B = T + cd[TR_B];
    const double* dB = T + cd[TR_DB];
    for (int p = tid; p < q; p += nt) {
      double u = 0.0, d0 = 0.0, d1 = 0.0;
      for (int g = 0; g < ng; ++g) {
        const double a = ldg(arow + g), da = ldg(darow + g);
        const int j0 = (int)ldg(gst + g), j1 = (int)ldg(gst + g + 1);
        double s = 0.0, ds = 0.0;
        for (int j = j0; j < j1; ++j) {
          const int m = (int)ldg(gmo + j);
          const double cm = c_at(c + m);
          s = fma(ldg(B + p * nc + m), cm, s);
          ds = fma(ldg(dB + p * nc + m), cm, ds);
        }
        u = fma(a, s, u);
        d0 = fma(da, s, d0);
        d1 = fma(a, ds, d1);
      }
      out[p] = u; out[FP + p] = d0; out[2 * FP + p] = d1;
    }
    TM::sync();
    return q;
  }
  const int d = shape == SHAPE_HEX ? 3 : 2;
  const int a = ft.fixed;
  const int* ax = cd + CD_TAX;
  const double* vend = T + ax[8 * a + TX_VEND] + (ft.side > 0 ? n : 0);
  const double* dvend = T + ax[8 * a + TX_DVEND] + (ft.side > 0 ? n : 0);
  const int b0 = ft.run0;
  const int q0 = cd[CD_Q0 + b0];
  const double* V0 = T + ax[8 * b0 + TX_V];
  const double* dV0 = T + ax[8 * b0 + TX_DV];
  const int sa = (d == 3) ? (a == 0 ? n * n : (a == 1 ? n : 1)) : (a == 0 ? n : 1);
  if (d == 2) {
    const int sb = b0 == 0 ? n : 1;
    double* pv = scr;
    double* pd = scr + n;
    for (int i = tid; i < n; i += nt) {
      double s = 0.0, t = 0.0;
      for (int k = 0; k < n; ++k) {
        const double cv = c_at(c + k * sa + i * sb);
        s = fma(ldg(vend + k), cv, s);
        t = fma(ldg(dvend + k), cv, t);
      }
      pv[i] = s; pd[i] = t;
    }
    TM::sync();
    for (int p = tid; p < q0; p += nt) {
      double u = 0.0, du = 0.0, dn = 0.0;
      for (int i = 0; i < n; ++i) {
        const double v = ldg(V0 + p * n + i);
        u = fma(v, pv[i], u);
        du = fma(ldg(dV0 + p * n + i), pv[i], du);
        dn = fma(v, pd[i], dn);
      }
      out[p] = u;
      out[(1 + b0) * FP + p] = du;
      out[(1 + a) * FP + p] = dn;
    }
    TM::sync();
    return q0;
  }
  const int b1 = ft.run1;
  const int q1 = cd[CD_Q0 + b1];
  const double* V1 = T + ax[8 * b1 + TX_V];
  const double* dV1 = T + ax[8 * b1 + TX_DV];
  const int s0 = b0 == 0 ? n * n : (b0 == 1 ? n : 1);
  const int s1 = b1 == 0 ? n * n : (b1 == 1 ? n : 1);
  double* pv = scr;                  // n*n plane of V-contracted coefficients
  double* pd = pv + n * n;           // n*n plane, dV-contracted (normal derivative)
  double* tv = pd + n * n;           // q0*n
  double* td = tv + q0 * n;          // q0*n (dV along run0)
  double* tp = td + q0 * n;          // q0*n (from pd)
  for (int i = tid; i < n * n; i += nt) {
    const int i0 = i / n, i1 = i - i0 * n;
    double s = 0.0, t = 0.0;
    for (int k = 0; k < n; ++k) {
      const double cv = c_at(c + k * sa + i0 * s0 + i1 * s1);
      s = fma(ldg(vend + k), cv, s);
      t = fma(ldg(dvend + k), cv, t);
    }
    pv[i] = s; pd[i] = t;
  }
  TM::sync();
  for (int i = tid; i < q0 * n; i += nt) {
    const int p0 = i / n, i1 = i - p0 * n;
    double s = 0.0, t = 0.0, r = 0.0;
    for (int k = 0; k < n; ++k) {
      const double v = ldg(V0 + p0 * n + k);
      s = fma(v, pv[k * n + i1], s);
      t = fma(ldg(dV0 + p0 * n + k), pv[k * n + i1], t);
      r = fma(v, pd[k * n + i1], r);
    }
    tv[i] = s; td[i] = t; tp[i] = r;
  }
  TM::sync();
  for (int i = tid; i < q0 * q1; i += nt) {
    const int p0 = i / q1, p1 = i - p0 * q1;
    double u = 0.0, d1 = 0.0, d0 = 0.0, dn = 0.0;
    for (int k = 0; k < n; ++k) {
      const double v = ldg(V1 + p1 * n + k);
      u = fma(v, tv[p0 * n + k], u);
      d1 = fma(ldg(dV1 + p1 * n + k), tv[p0 * n + k], d1);
      d0 = fma(v, td[p0 * n + k], d0);
      dn = fma(v, tp[p0 * n + k], dn);
    }
    out[i] = u;
    out[(1 + b0) * FP + i] = d0;
    out[(1 + b1) * FP + i] = d1;
    out[(1 + a) * FP + i] = dn;
  }
  TM::sync();
  return q0 * q1;
}

// ---------------------------------------------------------------------------
// transfers between face grids: per flux axis 1-D matrices (pool), optional swap.
// forward: in (n0 x n1) -> out (m0 x m1); T0: m0 x n_sig0, T1: m1 x n_sig1.
template <class TM = CtaTeam>
static __device__ void xfer_fwd(const double* __restrict__ in, int FPin, int n0, int n1,
                         double* __restrict__ out, int FPout, int m0, int m1,
                         const double* __restrict__ T0, const double* __restrict__ T1, bool swap,
                         int nf, double* __restrict__ tmp, int fd, int tid, int nt) {
  if (fd == 1) {
    for (int i = tid; i < nf * m0; i += nt) {
      const int fl = i / m0, t = i - fl * m0;
      double s = 0.0;
      for (int k = 0; k < n0; ++k) s = fma(ldg(T0 + t * n0 + k), in[fl * FPin + k], s);
      out[fl * FPout + t] = s;
    }
    TM::sync();
    return;
  }
  if (!swap) {
    // tmp[s0][t1] = sum_s1 T1[t1][s1] in[s0][s1]
    for (int i = tid; i < nf * n0 * m1; i += nt) {
      const int fl = i / (n0 * m1), r = i - fl * n0 * m1, s0 = r / m1, t1 = r - s0 * m1;
      double s = 0.0;
      for (int k = 0; k < n1; ++k) s = fma(ldg(T1 + t1 * n1 + k), in[fl * FPin + s0 * n1 + k], s);
      tmp[fl * QMAX * QMAX + s0 * m1 + t1] = s;
    }
    TM::sync();
    for (int i = tid; i < nf * m0 * m1; i += nt) {
      const int fl = i / (m0 * m1), r = i - fl * m0 * m1, t0 = r / m1, t1 = r - t0 * m1;
      double s = 0.0;
      for (int k = 0; k < n0; ++k) s = fma(ldg(T0 + t0 * n0 + k), tmp[fl * QMAX * QMAX + k * m1 + t1], s);
      out[fl * FPout + r] = s;
    }
  } else {
    // T0: m0 x n1, T1: m1 x n0.  tmp[t1][s1] = sum_s0 T1[t1][s0] in[s0][s1]
    for (int i = tid; i < nf * m1 * n1; i += nt) {
      const int fl = i / (m1 * n1), r = i - fl * m1 * n1, t1 = r / n1, s1 = r - t1 * n1;
      double s = 0.0;
      for (int k = 0; k < n0; ++k) s = fma(ldg(T1 + t1 * n0 + k), in[fl * FPin + k * n1 + s1], s);
      tmp[fl * QMAX * QMAX + t1 * n1 + s1] = s;
    }
    TM::sync();
    for (int i = tid; i < nf * m0 * m1; i += nt) {
      const int fl = i / (m0 * m1), r = i - fl * m0 * m1, t0 = r / m1, t1 = r - t0 * m1;
      double s = 0.0;
      for (int k = 0; k < n1; ++k) s = fma(ldg(T0 + t0 * n1 + k), tmp[fl * QMAX * QMAX + t1 * n1 + k], s);
      out[fl * FPout + r] = s;
    }
  }
  TM::sync();
}

// transpose: in (m0 x m1) on the flux grid -> out (n0 x n1) on the source grid
template <class TM = CtaTeam>
static __device__ void xfer_bwd(const double* __restrict__ in, int FPin, int m0, int m1,
                         double* __restrict__ out, int FPout, int n0, int n1,
                         const double* __restrict__ T0, const double* __restrict__ T1, bool swap,
                         int nf, double* __restrict__ tmp, int fd, int tid, int nt) {
  if (fd == 1) {
    for (int i = tid; i < nf * n0; i += nt) {
      const int fl = i / n0, s0 = i - fl * n0;
      double s = 0.0;
      for (int t = 0; t < m0; ++t) s = fma(ldg(T0 + t * n0 + s0), in[fl * FPin + t], s);
      out[fl * FPout + s0] = s;
    }
    TM::sync();
    return;
  }
  if (!swap) {
    // tmp[t0][s1] = sum_t1 T1[t1][s1] in[t0][t1];  out[s0][s1] = sum_t0 T0[t0][s0] tmp[t0][s1]
    for (int i = tid; i < nf * m0 * n1; i += nt) {
      const int fl = i / (m0 * n1), r = i - fl * m0 * n1, t0 = r / n1, s1 = r - t0 * n1;
      double s = 0.0;
      for (int t1 = 0; t1 < m1; ++t1) s = fma(ldg(T1 + t1 * n1 + s1), in[fl * FPin + t0 * m1 + t1], s);
      tmp[fl * QMAX * QMAX + t0 * n1 + s1] = s;
    }
    TM::sync();
    for (int i = tid; i < nf * n0 * n1; i += nt) {
      const int fl = i / (n0 * n1), r = i - fl * n0 * n1, s0 = r / n1, s1 = r - s0 * n1;
      double s = 0.0;
      for (int t0 = 0; t0 < m0; ++t0) s = fma(ldg(T0 + t0 * n0 + s0), tmp[fl * QMAX * QMAX + t0 * n1 + s1], s);
      out[fl * FPout + r] = s;
    }
  } else {
    // out[s0][s1] = sum T0[t0][s1] T1[t1][s0] in[t0][t1]
    for (int i = tid; i < nf * m1 * n1; i += nt) {
      const int fl = i / (m1 * n1), r = i - fl * m1 * n1, t1 = r / n1, s1 = r - t1 * n1;
      double s = 0.0;
      for (int t0 = 0; t0 < m0; ++t0) s = fma(ldg(T0 + t0 * n1 + s1), in[fl * FPin + t0 * m1 + t1], s);
      tmp[fl * QMAX * QMAX + t1 * n1 + s1] = s;
    }
    TM::sync();
    for (int i = tid; i < nf * n0 * n1; i += nt) {
      const int fl = i / (n0 * n1), r = i - fl * n0 * n1, s0 = r / n1, s1 = r - s0 * n1;
      double s = 0.0;
      for (int t1 = 0; t1 < m1; ++t1) s = fma(ldg(T1 + t1 * n0 + s0), tmp[fl * QMAX * QMAX + t1 * n1 + s1], s);
      out[fl * FPout + r] = s;
    }
  }
  TM::sync();
}

// ---------------------------------------------------------------------------
// geometry on a flux grid

// self: swj(t) and Gn_k(t), k < d.  nf = flux grid size.
__device__ __forceinline__ double self_geom(const DevPlan& P, const FaceRec& r, int shape, int f, int d,
                                            int t, int nflux, double* gn) {
  const double* T = P.tab;
  if (r.flags & F_SELF_PW) {
    const double* g = P.fgeo + r.geo;
    for (int k = 0; k < d; ++k) gn[k] = g[nflux + k * nflux + t];
    return g[t];
  }
  const int t0 = (r.nt1 > 1) ? t / r.nt1 : t;
  const int t1 = (r.nt1 > 1) ? t - t0 * r.nt1 : 0;
  double w = ldg(T + r.wt0 + t0);
  if (r.nt1 > 1) w *= ldg(T + r.wt1 + t1);
  if (shape == SHAPE_TRI) {
    double p = ldg(T + r.wt0 + r.nt0 + t0);
    if (r.flags & F_SELF_NEG) p = -p;
    double c00, c01;
    tri_chain(f, p, c00, c01);
    gn[0] = c00 * r.gs[0] + c01 * r.gs[1];
    gn[1] = r.gs[1];
  } else {
    for (int k = 0; k < d; ++k) gn[k] = r.gs[k];
  }
  return r.sJ * w;
}

// other side's Gn at point t of the grid it is evaluated on
__device__ __forceinline__ void other_gn(const DevPlan& P, const FaceRec& r, int d, int t, int nflux,
                                         double* gn) {
  const double* T = P.tab;
  const int shape_o = P.cd[P.elem_class[r.nbr] * CD_WORDS + CD_SHAPE];
  if (r.type == FT_DIRECT) {
    // on the neighbour's own face grid, its own normal (its own record)
    const FaceRec& o = P.recs[r.nbr_rec];
    const int no = o.nt0 * o.nt1;
    if (r.flags & F_OTHER_PW) {
      const double* g = P.fgeo + o.geo;
      for (int k = 0; k < d; ++k) gn[k] = g[no + k * no + t];
      return;
    }
    if (shape_o == SHAPE_TRI) {
      const double p = ldg(T + o.wt0 + o.nt0 + t);
      double c00, c01;
      tri_chain(r.nbr_face, p, c00, c01);
      gn[0] = c00 * r.go[0] + c01 * r.go[1];
      gn[1] = r.go[1];
    } else {
      for (int k = 0; k < d; ++k) gn[k] = r.go[k];
    }
    return;
  }
  // shared: on the trace grid
  if (r.flags & F_OTHER_PW) {
    const double* g = P.fgeo + r.geo;
    for (int k = 0; k < d; ++k) gn[k] = g[nflux + d * nflux + k * nflux + t];
    return;
  }
  if (shape_o == SHAPE_TRI) {
    const int t0 = (r.nt1 > 1) ? t / r.nt1 : t;
    double p = ldg(T + r.wt0 + r.nt0 + t0);
    if (r.flags & F_OTHER_NEG) p = -p;
    double c00, c01;
    tri_chain(r.nbr_face, p, c00, c01);
    gn[0] = c00 * r.go[0] + c01 * r.go[1];
    gn[1] = r.go[1];
  } else {
    for (int k = 0; k < d; ++k) gn[k] = r.go[k];
  }
}

// ---------------------------------------------------------------------------
template <int SHAPE> struct ShapeDim { static constexpr int D = SHAPE == SHAPE_HEX ? 3 : 2; };

template <int SHAPE, int N, int Q>
struct Cfg {
  static constexpr int D = ShapeDim<SHAPE>::D;
  static constexpr int NF = SHAPE == SHAPE_HEX ? 6 : (SHAPE == SHAPE_QUAD ? 4 : 3);
  static constexpr int NC = SHAPE == SHAPE_TRI ? N * (N + 1) / 2 : (D == 3 ? N * N * N : N * N);
  static constexpr int NP = D == 3 ? Q * Q * Q : Q * Q;
  static constexpr int NS = D == 3 ? Q * Q : Q;              // own face points
  static constexpr int FP = D == 3 ? QMAX * QMAX : QMAX;     // face-field stride
  static constexpr int NT = D == 3 ? 128 : 64;
  static constexpr int TABSZ = SHAPE == SHAPE_TRI
      ? (2 * Q * (N + 1) + 3 * Q * Q + 2 * Q + Q * NC + NC + 4 * Q + 2 * Q + (N + 2) + NC)
      : D * (Q * N + Q * Q + Q + 2 * Q);
  static constexpr int TABP = (TABSZ + 1) & ~1;
  // element scratch layout (doubles)
  static constexpr int e_c = 0;
  static constexpr int e_u = e_c + ((NC + 1) & ~1);
  static constexpr int e_du = e_u + NP;
  static constexpr int e_t1 = e_du + D * NP;
  static constexpr int e_t2 = e_t1 + NP;
  static constexpr int e_fb = e_t2 + NP;
  static constexpr int e_fs = e_fb + NF * (1 + D) * NS;
  // face scratch: us(4FP) uo(4FP) xo(4FP) xs(4FP) ff(4FP) tmp(4 QMAX^2, 3-D) nbr
  static constexpr int FSZ = D == 3 ? 5 * 4 * FP + 4 * QMAX * QMAX + 2 * NMAX * NMAX + 3 * QMAX * NMAX
                                    : 5 * 4 * FP + 2 * (NMAX + 2);
  static constexpr int NBK = NMAX * NMAX + 2;                 // staged neighbour block (2-D)
  static constexpr int e_rec = (e_fs + FSZ + 1) & ~1;          // NF face records (16 doubles each)
  static constexpr int e_nb = e_rec + NF * 16;
  // 2-D warp kernel: next element's coefficients and records, double-buffered (prefetched)
  static constexpr int NCP = (NC + 1) & ~1;
  static constexpr int e_pre = e_nb + (D == 2 ? NF * NBK : 0);
  static constexpr int RPW = NF * 16 + 2 * NF;    // prefetched records + their rec_ext words
  static constexpr int ESZ = e_pre + (D == 2 ? 2 * (NCP + RPW) : 0);
  static constexpr int TOTAL = TABP + ESZ;
};

// own face values (u and du_k) on the own face grid from the volume arrays
template <int SHAPE, int N, int Q>
__device__ __forceinline__ void restrict_face(const double* u, const double* du, const double* Ltab,
                                              int gllmask, int f, double* us, int tid, int nt) {
  using C = Cfg<SHAPE, N, Q>;
  constexpr int D = C::D;
  const FaceTopo ft = face_topo(SHAPE, f);
  const int a = ft.fixed;
  const bool gll = (gllmask >> a) & 1;
  const double* Lrow = Ltab + a * 2 * Q + (ft.side > 0 ? Q : 0);
  for (int i = tid; i < C::NS * (1 + D); i += nt) {
    const int fl = i / C::NS, p = i - fl * C::NS;
    const double* src = fl == 0 ? u : du + (fl - 1) * C::NP;
    int base, sa;
    if (D == 2) {
      sa = a == 0 ? Q : 1;
      base = p * (a == 0 ? 1 : Q);
    } else {
      const int p0 = p / Q, p1 = p - p0 * Q;
      const int s0 = ft.run0 == 0 ? Q * Q : (ft.run0 == 1 ? Q : 1);
      const int s1 = ft.run1 == 0 ? Q * Q : (ft.run1 == 1 ? Q : 1);
      sa = a == 0 ? Q * Q : (a == 1 ? Q : 1);
      base = p0 * s0 + p1 * s1;
    }
    double v;
    if (gll) {
      v = src[base + (ft.side > 0 ? (Q - 1) * sa : 0)];
    } else {
      v = 0.0;
      for (int k = 0; k < Q; ++k) v = fma(Lrow[k], src[base + k * sa], v);
    }
    us[fl * C::FP + p] = v;
  }
}

template <int SHAPE, int N, int Q>
__device__ __forceinline__ void fold_face(double* P0, double* Pk, const double* Ltab, int gllmask, int f,
                                          const double* fb, int tid, int nt) {
  using C = Cfg<SHAPE, N, Q>;
  constexpr int D = C::D;
  const FaceTopo ft = face_topo(SHAPE, f);
  const int a = ft.fixed;
  const bool gll = (gllmask >> a) & 1;
  const double* Lrow = Ltab + a * 2 * Q + (ft.side > 0 ? Q : 0);
  for (int i = tid; i < C::NS * (1 + D); i += nt) {
    const int fl = i / C::NS, p = i - fl * C::NS;
    double* dst = fl == 0 ? P0 : Pk + (fl - 1) * C::NP;
    int base, sa;
    if (D == 2) {
      sa = a == 0 ? Q : 1;
      base = p * (a == 0 ? 1 : Q);
    } else {
      const int p0 = p / Q, p1 = p - p0 * Q;
      const int s0 = ft.run0 == 0 ? Q * Q : (ft.run0 == 1 ? Q : 1);
      const int s1 = ft.run1 == 0 ? Q * Q : (ft.run1 == 1 ? Q : 1);
      sa = a == 0 ? Q * Q : (a == 1 ? Q : 1);
      base = p0 * s0 + p1 * s1;
    }
    const double v = fb[fl * C::NS + p];
    if (gll) {
      dst[base + (ft.side > 0 ? (Q - 1) * sa : 0)] += v;
    } else {
      for (int k = 0; k < Q; ++k) dst[base + k * sa] += Lrow[k] * v;
    }
  }
}

// Flux of one face on the own face grid (any coupling type).  `us` holds the
// own u, du_k at the own face points (stride FP, filled and synced by the
// caller); the result fbf holds (fv, fd Gn_k) on the own face grid (stride NS).
// Scratch layout of fscr: uo, xo, xs, ff (4*FP each), tmp (4*QMAX^2), nscr.
template <int SHAPE, int N, int Q, class TM = CtaTeam>
__device__ __noinline__ void generic_face(const DevPlan& P, const FaceRec& r, const int f,
                                          const double* __restrict__ x, double* __restrict__ us,
                                          double* __restrict__ fbf, double* __restrict__ fscr,
                                          const int tid, const int nt, const double* staged = nullptr,
                                          const bool staged_traces = false, const int staged_q = 0) {
  using C = Cfg<SHAPE, N, Q>;
  constexpr int D = C::D, NS = C::NS, FP = C::FP;
  const double* T = P.tab;
  const int fd = D - 1;
  double* uo = fscr;
  double* xo = uo + 4 * FP;
  double* xs = xo + 4 * FP;
  double* ff = xs + 4 * FP;
  double* tmp = ff + 4 * FP;
  double* nscr = tmp + (D == 3 ? 4 * QMAX * QMAX : 0);
  int no = 0;
  int qo0 = 0, qo1 = 1;
  if (r.type != FT_BOUNDARY) {
    TM::sync();
    if (staged_traces) {      // published traces of the neighbour face: u, du_0, du_1 on its grid
      no = staged_q;
      for (int i = tid; i < 3 * no; i += nt) {
        const int fl = i / no, pp = i - fl * no;
        uo[fl * FP + pp] = staged[i];
      }
      TM::sync();
    } else {
      no = eval_face_from_coeffs<TM>(P, r.nbr, r.nbr_face, x, uo, FP, nscr, tid, nt, staged);
    }
    if (staged_traces && D == 2) {
      qo0 = staged_q;
      qo1 = 1;
    } else {
      const int* cdo = P.cd + P.elem_class[r.nbr] * CD_WORDS;
      const FaceTopo fto = face_topo(cdo[CD_SHAPE], r.nbr_face);
      qo0 = cdo[CD_Q0 + fto.run0];
      qo1 = fto.run1 >= 0 ? cdo[CD_Q0 + fto.run1] : 1;
    }
  }
  TM::sync();
  const double tau = r.tau;
  if (r.type != FT_SHARED) {
    // flux on the own face grid
    if (r.type == FT_DIRECT) {
      // g_o on the other grid, then (u_o, g_o) -> own grid
      for (int p = tid; p < no; p += nt) {
        double gn[3];
        other_gn(P, r, D, p, no, gn);
        double g = 0.0;
        for (int k = 0; k < D; ++k) g = fma(gn[k], uo[(1 + k) * FP + p], g);
        uo[FP + p] = g;      // field 1 now holds g_o (du_0 no longer needed)
      }
      TM::sync();
      if (!(r.flags & F_OTHER_ID)) {
        const int q0s = (SHAPE == SHAPE_TRI || D == 2) ? NS : Q;
        const int q1s = D == 3 ? Q : 1;
        xfer_fwd<TM>(uo, FP, qo0, qo1, xo, FP, q0s, q1s, T + r.to0, D == 3 ? T + r.to1 : nullptr,
                 (r.flags & F_OTHER_SWAP) != 0, 2, tmp, fd, tid, nt);
      } else {
        for (int p = tid; p < NS; p += nt) { xo[p] = uo[p]; xo[FP + p] = uo[FP + p]; }
        TM::sync();
      }
    }
    for (int p = tid; p < NS; p += nt) {
      double gn[3];
      const double swj = self_geom(P, r, SHAPE, f, D, p, NS, gn);
      double gs = 0.0;
      for (int k = 0; k < D; ++k) gs = fma(gn[k], us[(1 + k) * FP + p], gs);
      double jump, avg;
      if (r.type == FT_BOUNDARY) {
        jump = 2.0 * us[p];
        avg = gs;
      } else {
        jump = us[p] - xo[p];
        avg = 0.5 * (gs - xo[FP + p]);
      }
      const double fv = (tau * jump - avg) * swj;
      const double fdd = -0.5 * jump * swj;
      fbf[p] = fv;
      for (int k = 0; k < D; ++k) fbf[(1 + k) * NS + p] = fdd * gn[k];
    }
    TM::sync();
    return;
  }
  // ---- shared trace: flux on the trace grid
  const int m0 = r.nt0, m1 = r.nt1, nflux = m0 * m1;
  const bool same_self = (r.flags & F_SELF_ID) != 0;
  if (!same_self) {
    const int q0s = D == 3 ? Q : NS;
    const int q1s = D == 3 ? Q : 1;
    xfer_fwd<TM>(us, FP, q0s, q1s, xs, FP, m0, m1, T + r.ts0, D == 3 ? T + r.ts1 : nullptr,
             (r.flags & F_SELF_SWAP) != 0, 1 + D, tmp, fd, tid, nt);
  }
  const double* vs = same_self ? us : xs;
  if (!(r.flags & F_OTHER_ID)) {
    xfer_fwd<TM>(uo, FP, qo0, qo1, xo, FP, m0, m1, T + r.to0, D == 3 ? T + r.to1 : nullptr,
             (r.flags & F_OTHER_SWAP) != 0, 1 + D, tmp, fd, tid, nt);
  }
  const double* vo = (r.flags & F_OTHER_ID) ? uo : xo;
  for (int t = tid; t < nflux; t += nt) {
    double gns[3], gno[3];
    const double swj = self_geom(P, r, SHAPE, f, D, t, nflux, gns);
    other_gn(P, r, D, t, nflux, gno);
    double gs = 0.0, go = 0.0;
    for (int k = 0; k < D; ++k) {
      gs = fma(gns[k], vs[(1 + k) * FP + t], gs);
      go = fma(gno[k], vo[(1 + k) * FP + t], go);
    }
    const double jump = vs[t] - vo[t];
    const double avg = 0.5 * (gs - go);
    const double fv = (tau * jump - avg) * swj;
    const double fdd = -0.5 * jump * swj;
    ff[t] = fv;
    for (int k = 0; k < D; ++k) ff[(1 + k) * FP + t] = fdd * gns[k];
  }
  TM::sync();
  if (same_self) {
    for (int i = tid; i < (1 + D) * NS; i += nt) {
      const int fl = i / NS, p = i - fl * NS;
      fbf[i] = ff[fl * FP + p];
    }
    TM::sync();
  } else {
    const int q0s = D == 3 ? Q : NS;
    const int q1s = D == 3 ? Q : 1;
    xfer_bwd<TM>(ff, FP, m0, m1, fbf, NS, q0s, q1s, T + r.ts0, D == 3 ? T + r.ts1 : nullptr,
             (r.flags & F_SELF_SWAP) != 0, 1 + D, tmp, fd, tid, nt);
  }
}

// Stage the class's 1-D tables into shared memory (layout: see apply_elem).
template <int SHAPE, int N, int Q>
__device__ __forceinline__ void stage_tables(const DevPlan& P, const int* cd, double* tb, int tid, int nt) {
  using C = Cfg<SHAPE, N, Q>;
  constexpr int D = C::D, NC = C::NC;
  const double* T = P.tab;
  double *V = tb, *Dm, *W, *Lt;
  double *A = nullptr, *dA = nullptr, *Bt = nullptr, *gidd = nullptr, *refw = nullptr, *eta0 = nullptr,
         *eta1 = nullptr, *gst = nullptr, *gmo = nullptr;
  if (SHAPE != SHAPE_TRI) {
    Dm = V + D * Q * N;
    W = Dm + D * Q * Q;
    Lt = W + D * Q;
    for (int ax = 0; ax < D; ++ax) {
      const int* t = cd + CD_TAX + 8 * ax;
      for (int i = tid; i < Q * N; i += nt) V[ax * Q * N + i] = ldg(T + t[TX_V] + i);
      for (int i = tid; i < Q * Q; i += nt) Dm[ax * Q * Q + i] = ldg(T + t[TX_D] + i);
      for (int i = tid; i < Q; i += nt) W[ax * Q + i] = ldg(T + t[TX_W] + i);
      for (int i = tid; i < 2 * Q; i += nt) Lt[ax * 2 * Q + i] = ldg(T + t[TX_LEND] + i);
    }
  } else {
    constexpr int NG = N + 1;
    A = tb;
    dA = A + Q * NG;
    Dm = dA + Q * NG;             // D0 then D1
    W = Dm + 2 * Q * Q;           // w0, w1
    Bt = W + 2 * Q;               // B (Q x NC)
    gidd = Bt + Q * NC;           // group of each mode
    Lt = gidd + NC;               // L0 (2Q), L1 (2Q)
    refw = Lt + 4 * Q;            // Q*Q
    eta0 = refw + Q * Q;          // Q
    eta1 = eta0 + Q;              // Q
    gst = eta1 + Q;               // group starts (NG + 1)
    gmo = gst + NG + 1;           // modes ordered by group (NC)
    for (int i = tid; i < Q * NG; i += nt) { A[i] = ldg(T + cd[TR_A] + i); dA[i] = ldg(T + cd[TR_DA] + i); }
    for (int i = tid; i < Q * Q; i += nt) {
      Dm[i] = ldg(T + cd[TR_D0] + i);
      Dm[Q * Q + i] = ldg(T + cd[TR_D1] + i);
      refw[i] = ldg(T + cd[TR_REFW] + i);
    }
    for (int i = tid; i < Q; i += nt) {
      W[i] = ldg(T + cd[TR_W0] + i); W[Q + i] = ldg(T + cd[TR_W1] + i);
      eta0[i] = ldg(T + cd[TR_PTS0] + i); eta1[i] = ldg(T + cd[TR_PTS1] + i);
    }
    for (int i = tid; i < Q * NC; i += nt) Bt[i] = ldg(T + cd[TR_B] + i);
    for (int i = tid; i < 2 * Q; i += nt) { Lt[i] = ldg(T + cd[TR_L0] + i); Lt[2 * Q + i] = ldg(T + cd[TR_L1] + i); }
    for (int i = tid; i < NG + 1; i += nt) gst[i] = ldg(T + cd[TR_GSTART] + i);
    for (int i = tid; i < NC; i += nt) gmo[i] = ldg(T + cd[TR_GID] + i);
    for (int g = tid; g < NG; g += nt) {
      const int j0 = (int)ldg(T + cd[TR_GSTART] + g), j1 = (int)ldg(T + cd[TR_GSTART] + g + 1);
      for (int j = j0; j < j1; ++j) gidd[(int)ldg(T + cd[TR_GID] + j)] = (double)g;
    }
  }
}

// One element: volume terms, faces, lift, transposed pass; written to y once.
// `es` is the element's scratch (Cfg layout without the table region), `tb`
// the staged tables; the team (CTA or warp) is tid / nt with TM::sync().
// PREF (2-D warp kernel): the element's coefficients (cpre) and face records (rpre) were
// prefetched by the caller during the previous element, and dof_pre is its DoF offset.
template <int SHAPE, int N, int Q, int GEOM, class TM, bool PREF = false>
__device__ __forceinline__ void apply_elem(const DevPlan& P, const int* cd, const int i_el,
                                           const double* __restrict__ x, double* __restrict__ y,
                                           double* es, const double* tb, const int tid, const int nt,
                                           double* cpre = nullptr, FaceRec* rpre = nullptr, int64_t dof_pre = 0) {
  using C = Cfg<SHAPE, N, Q>;
  constexpr int D = C::D, NP = C::NP, NS = C::NS, FP = C::FP, NC = C::NC;
  const int64_t dof0 = PREF ? dof_pre : P.dof_off[P.class_elems[cd[CD_ELEM_OFF] + i_el]];
  const int gllmask = cd[CD_GLLMASK];
  double* c = PREF ? cpre : es + C::e_c;
  double* u = es + C::e_u;
  double* du = es + C::e_du;
  double* t1 = es + C::e_t1;
  double* t2 = es + C::e_t2;
  double* fb = es + C::e_fb;
  double* fs = es + C::e_fs;
  // table pointers (layout of stage_tables)
  const double *V = tb, *Dm, *W, *Lt;
  const double *A = nullptr, *dA = nullptr, *Bt = nullptr, *gidd = nullptr, *refw = nullptr, *eta0 = nullptr,
               *eta1 = nullptr, *gst = nullptr, *gmo = nullptr;
  if (SHAPE != SHAPE_TRI) {
    Dm = V + D * Q * N;
    W = Dm + D * Q * Q;
    Lt = W + D * Q;
  } else {
    constexpr int NG = N + 1;
    A = tb;
    dA = A + Q * NG;
    Dm = dA + Q * NG;
    W = Dm + 2 * Q * Q;
    Bt = W + 2 * Q;
    gidd = Bt + Q * NC;
    Lt = gidd + NC;
    refw = Lt + 4 * Q;
    eta0 = refw + Q * Q;
    eta1 = eta0 + Q;
    gst = eta1 + Q;
    gmo = gst + NG + 1;
  }
  // 2-D: records and neighbour coefficient blocks fetched asynchronously up front
  FaceRec* srec = PREF ? rpre : reinterpret_cast<FaceRec*>(es + C::e_rec);
  double* snb = es + C::e_nb;
  const int rbase = cd[CD_REC_OFF] + i_el * C::NF;
  if (D == 2 && !PREF) {
    for (int i = tid; i < C::NF * 16; i += nt)
      cp_async8_(reinterpret_cast<double*>(srec) + i, reinterpret_cast<const double*>(P.recs + rbase) + i);
    cp_async_commit_();
  }
  if (!PREF)
    for (int i = tid; i < NC; i += nt) c[i] = ldg(x + dof0 + i);
  if (D == 2) {
    if (!PREF) cp_async_wait_all_();
    TM::sync();
    for (int f = 0; f < C::NF; ++f) {
      if (srec[f].type == FT_BOUNDARY) continue;
      const int64_t ext = PREF ? reinterpret_cast<const int64_t*>(srec + C::NF)[2 * f]
                               : (P.rec_ext ? P.rec_ext[2 * (rbase + f)] : -1);
      if (ext >= 0 && P.planes) {          // published neighbour traces (3 fields x q_o)
        const int qo = (int)(ext >> 48);
        const double* src = P.planes + (ext & ((int64_t(1) << 48) - 1));
        for (int i = tid; i < 3 * qo; i += nt) cp_async8_(snb + f * C::NBK + i, src + i);
      } else {
        const int no = P.cd[P.elem_class[srec[f].nbr] * CD_WORDS + CD_NC];
        const double* src = x + srec[f].nbr_dof;
        for (int i = tid; i < no; i += nt) cp_async8_(snb + f * C::NBK + i, src + i);
      }
    }
    cp_async_commit_();
  }
  TM::sync();

  // ---- 1-2. BwdTrans and PhysDeriv
  if (SHAPE == SHAPE_HEX) {
    contract<N, N, N, 0, Q, false, false>(c, t1, V, tid, nt);
    TM::sync();
    contract<Q, N, N, 1, Q, false, false>(t1, t2, V + Q * N, tid, nt);
    TM::sync();
    contract<Q, Q, N, 2, Q, false, false>(t2, u, V + 2 * Q * N, tid, nt);
    TM::sync();
    contract<Q, Q, Q, 0, Q, false, false>(u, du, Dm, tid, nt);
    contract<Q, Q, Q, 1, Q, false, false>(u, du + NP, Dm + Q * Q, tid, nt);
    contract<Q, Q, Q, 2, Q, false, false>(u, du + 2 * NP, Dm + 2 * Q * Q, tid, nt);
  } else if (SHAPE == SHAPE_QUAD) {
    contract<N, N, 1, 0, Q, false, false>(c, t1, V, tid, nt);
    TM::sync();
    contract<Q, N, 1, 1, Q, false, false>(t1, u, V + Q * N, tid, nt);
    TM::sync();
    contract<Q, Q, 1, 0, Q, false, false>(u, du, Dm, tid, nt);
    contract<Q, Q, 1, 1, Q, false, false>(u, du + NP, Dm + Q * Q, tid, nt);
  } else {
    constexpr int NG = N + 1;
    // t1[g][b] = sum_{m in g} B[b][m] c[m]
    for (int i = tid; i < NG * Q; i += nt) {
      const int g = i / Q, b = i - g * Q;
      double s = 0.0;
      const int j0 = (int)gst[g], j1 = (int)gst[g + 1];
      for (int j = j0; j < j1; ++j) {
        const int m = (int)gmo[j];
        s = fma(Bt[b * NC + m], c[m], s);
      }
      t1[i] = s;
    }
    TM::sync();
    contract<NG, Q, 1, 0, Q, false, false>(t1, u, A, tid, nt);    // u[a][b] = sum_g A[a][g] t1[g][b]
    TM::sync();
    contract<Q, Q, 1, 0, Q, false, false>(u, du, Dm, tid, nt);
    contract<Q, Q, 1, 1, Q, false, false>(u, du + NP, Dm + Q * Q, tid, nt);
  }
  TM::sync();

  // ---- 3-4. faces: flux on each face, stored on the own face grid in fb
  double* us = fs;              // 4 fields x FP, own face grid
  if (D == 2) cp_async_wait_all_();
  TM::sync();
  for (int f = 0; f < C::NF; ++f) {
    const FaceRec r = D == 2 ? srec[f] : P.recs[rbase + f];
    restrict_face<SHAPE, N, Q>(u, du, Lt, gllmask, f, us, tid, nt);
    TM::sync();
    const int64_t ext = (D == 2 && P.rec_ext && r.type != FT_BOUNDARY)
                            ? (PREF ? reinterpret_cast<const int64_t*>(srec + C::NF)[2 * f] : P.rec_ext[2 * (rbase + f)])
                            : -1;
    const bool pub = D == 2 && ext >= 0 && P.planes != nullptr;
    generic_face<SHAPE, N, Q, TM>(P, r, f, x, us, fb + f * (1 + D) * NS, fs + 4 * FP, tid, nt,
                                  D == 2 ? snb + f * C::NBK : nullptr, pub, pub ? (int)(ext >> 48) : 0);
    TM::sync();
  }

  // ---- volume point arrays: u -> P0 = lam jw u, du -> P_k = (jw G G^T du)_k
  {
    const double lam = P.lam;
    const double* eg = P.egeo + cd[CD_EGEO_OFF] + (int64_t)i_el * cd[CD_EGEO_STRIDE];
    for (int p = tid; p < NP; p += nt) {
      double jw, K[6];
      if (GEOM == GEOM_POINTWISE) {
        constexpr int NSYM = D == 3 ? 6 : 3;
        jw = eg[p];
#pragma unroll
        for (int s = 0; s < NSYM; ++s) K[s] = eg[(1 + s) * NP + p];
      } else if (SHAPE == SHAPE_TRI) {
        const int a = p / Q, b = p - a * Q;
        jw = eg[0] * refw[p];
        const double e1 = eta0[a], e2 = eta1[b];
        const double c00 = 2.0 / (1.0 - e2), c01 = (1.0 + e1) / (1.0 - e2);
        const double S00 = eg[1], S01 = eg[2], S11 = eg[3];
        const double m00 = c00 * S00 + c01 * S01, m01 = c00 * S01 + c01 * S11;
        K[0] = jw * (m00 * c00 + m01 * c01);
        K[1] = jw * m01;
        K[2] = jw * S11;
      } else {
        double w;
        if (D == 3) {
          const int a0 = p / (Q * Q), r0 = p - a0 * Q * Q, a1 = r0 / Q, a2 = r0 - a1 * Q;
          w = W[a0] * W[Q + a1] * W[2 * Q + a2];
        } else {
          const int a0 = p / Q, a1 = p - a0 * Q;
          w = W[a0] * W[Q + a1];
        }
        jw = eg[0] * w;
        constexpr int NSYM = D == 3 ? 6 : 3;
#pragma unroll
        for (int s = 0; s < NSYM; ++s) K[s] = jw * eg[1 + s];
      }
      const double uv = u[p];
      if (D == 3) {
        const double d0 = du[p], d1 = du[NP + p], d2 = du[2 * NP + p];
        du[p] = K[0] * d0 + K[1] * d1 + K[2] * d2;
        du[NP + p] = K[1] * d0 + K[3] * d1 + K[4] * d2;
        du[2 * NP + p] = K[2] * d0 + K[4] * d1 + K[5] * d2;
      } else {
        const double d0 = du[p], d1 = du[NP + p];
        du[p] = K[0] * d0 + K[1] * d1;
        du[NP + p] = K[1] * d0 + K[2] * d1;
      }
      u[p] = lam * jw * uv;
    }
  }
  TM::sync();
  // ---- 5. fold face fluxes (faces sequentially: they share edge points)
  for (int f = 0; f < C::NF; ++f) {
    fold_face<SHAPE, N, Q>(u, du, Lt, gllmask, f, fb + f * (1 + D) * NS, tid, nt);
    TM::sync();
  }
  // ---- 6. R = P0 + sum_k D_k^T P_k, then IProduct
  if (SHAPE == SHAPE_HEX) {
    contract<Q, Q, Q, 0, Q, true, true>(du, u, Dm, tid, nt);
    TM::sync();
    contract<Q, Q, Q, 1, Q, true, true>(du + NP, u, Dm + Q * Q, tid, nt);
    TM::sync();
    contract<Q, Q, Q, 2, Q, true, true>(du + 2 * NP, u, Dm + 2 * Q * Q, tid, nt);
    TM::sync();
    contract<Q, Q, Q, 0, N, true, false>(u, t1, V, tid, nt);
    TM::sync();
    contract<N, Q, Q, 1, N, true, false>(t1, t2, V + Q * N, tid, nt);
    TM::sync();
    contract<N, N, Q, 2, N, true, false>(t2, c, V + 2 * Q * N, tid, nt);
  } else if (SHAPE == SHAPE_QUAD) {
    contract<Q, Q, 1, 0, Q, true, true>(du, u, Dm, tid, nt);
    TM::sync();
    contract<Q, Q, 1, 1, Q, true, true>(du + NP, u, Dm + Q * Q, tid, nt);
    TM::sync();
    contract<Q, Q, 1, 0, N, true, false>(u, t1, V, tid, nt);
    TM::sync();
    contract<N, Q, 1, 1, N, true, false>(t1, c, V + Q * N, tid, nt);
  } else {
    constexpr int NG = N + 1;
    contract<Q, Q, 1, 0, Q, true, true>(du, u, Dm, tid, nt);
    TM::sync();
    contract<Q, Q, 1, 1, Q, true, true>(du + NP, u, Dm + Q * Q, tid, nt);
    TM::sync();
    contract<Q, Q, 1, 0, NG, true, false>(u, t1, A, tid, nt);    // s[g][b] = sum_a A[a][g] R[a][b]
    TM::sync();
    for (int m = tid; m < NC; m += nt) {
      const int g = (int)gidd[m];
      double s = 0.0;
      for (int b = 0; b < Q; ++b) s = fma(Bt[b * NC + m], t1[g * Q + b], s);
      c[m] = s;
    }
  }
  TM::sync();
  for (int i = tid; i < NC; i += nt) y[dof0 + i] = c[i];
  TM::sync();
}

// Phase 1 (2-D): every element publishes u, du/deta_0, du/deta_1 on each of its
// faces' own grids (the reference's trace publish, sipg.py:585-592, with the
// eta-gradient instead of the normal derivative so a shared trace can apply
// its own metric).  One warp per element, persistent.
template <int SHAPE, int N, int Q>
__global__ void __launch_bounds__(256)
k_traces2d(const DevPlan P, const int cls, const double* __restrict__ x) {
  using C = Cfg<SHAPE, N, Q>;
  constexpr int NF = C::NF, FP = QMAX;
  __shared__ double sc[8][C::NC + 2];
  __shared__ double so[8][3 * FP + 2 * (NMAX + 2)];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int* cd = P.cd + cls * CD_WORDS;
  const int count = cd[CD_COUNT];
  const int* elist = P.class_elems + cd[CD_ELEM_OFF];
  for (int iel = blockIdx.x * 8 + warp; iel < count; iel += gridDim.x * 8) {
    const int e = elist[iel];
    const double* xe = x + P.dof_off[e];
    for (int i = lane; i < C::NC; i += 32) sc[warp][i] = __ldg(xe + i);
    __syncwarp();
    double* out = P.planes + P.plane_off[e];
    for (int f = 0; f < NF; ++f) {
      const int q = eval_face_from_coeffs<WarpTeam>(P, e, f, x, so[warp], FP, so[warp] + 3 * FP, lane, 32,
                                                    sc[warp]);
      for (int i = lane; i < 3 * q; i += 32) out[f * 3 * Q + i] = so[warp][(i / q) * FP + (i - (i / q) * q)];
      __syncwarp();
    }
  }
}

template <int SHAPE, int N, int Q, int GEOM>
__global__ void __launch_bounds__(Cfg<SHAPE, N, Q>::NT)
k_apply(const DevPlan P, const int cls, const double* __restrict__ x, double* __restrict__ y) {
  using C = Cfg<SHAPE, N, Q>;
  extern __shared__ double sm[];
  const int* cd = P.cd + cls * CD_WORDS;
  stage_tables<SHAPE, N, Q>(P, cd, sm, threadIdx.x, blockDim.x);
  apply_elem<SHAPE, N, Q, GEOM, CtaTeam>(P, cd, blockIdx.x, x, y, sm + C::TABP, sm, threadIdx.x, blockDim.x);
}

// Warp-per-element variant (2-D shapes): WPC independent warps per CTA share the
// staged tables; each warp walks the class's elements with stride gridDim.x*WPC.
template <int SHAPE, int N, int Q, int GEOM, int WPC>
__global__ void __launch_bounds__(32 * WPC)
k_apply_w(const DevPlan P, const int cls, const double* __restrict__ x, double* __restrict__ y) {
  using C = Cfg<SHAPE, N, Q>;
  extern __shared__ double sm[];
  const int* cd = P.cd + cls * CD_WORDS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  stage_tables<SHAPE, N, Q>(P, cd, sm, threadIdx.x, blockDim.x);
  __syncthreads();
  double* es = sm + C::TABP + warp * C::ESZ;
  const int count = cd[CD_COUNT];
  const int* elist = P.class_elems + cd[CD_ELEM_OFF];
  const int stride = gridDim.x * WPC;
  // software pipeline across the warp's elements: element k+1's records and coefficients are
  // copied (cp.async) while element k computes; DoF offsets are loaded one more element ahead
  double* cb = es + C::e_pre;
  double* rbd = es + C::e_pre + 2 * C::NCP;     // [2][NF records | 2 NF rec_ext words]
  auto issue = [&](int iel, int b, int64_t dof) {
    const int64_t r0 = cd[CD_REC_OFF] + (int64_t)iel * C::NF;
    const double* rs = reinterpret_cast<const double*>(P.recs + r0);
    double* rd = rbd + b * C::RPW;
    for (int i = lane; i < C::NF * 16; i += 32) cp_async8_(rd + i, rs + i);
    if (P.rec_ext)
      for (int i = lane; i < 2 * C::NF; i += 32)
        cp_async8_(rd + C::NF * 16 + i, reinterpret_cast<const double*>(P.rec_ext + 2 * r0) + i);
      else if (lane < 2 * C::NF) rd[C::NF * 16 + lane] = __longlong_as_double(-1ll);
    for (int i = lane; i < C::NC; i += 32) cp_async8_(cb + b * C::NCP + i, x + dof + i);
    cp_async_commit_();
  };
  int i_el = blockIdx.x * WPC + warp;
  int64_t dcur = 0, dnext = 0;
  if (i_el < count) {
    dcur = P.dof_off[elist[i_el]];
    issue(i_el, 0, dcur);
    if (i_el + stride < count) dnext = P.dof_off[elist[i_el + stride]];
  }
  for (int k = 0; i_el < count; i_el += stride, ++k) {
    const int b = k & 1;
    cp_async_wait_all_();   // this element's prefetch (and the previous element's groups)
    __syncwarp();
    const int64_t dthis = dcur;
    if (i_el + stride < count) {
      issue(i_el + stride, b ^ 1, dnext);
      dcur = dnext;
      if (i_el + 2 * stride < count) dnext = P.dof_off[elist[i_el + 2 * stride]];
    }
    apply_elem<SHAPE, N, Q, GEOM, WarpTeam, true>(P, cd, i_el, x, y, es, sm, lane, 32, cb + b * C::NCP,
                                                  reinterpret_cast<FaceRec*>(rbd + b * C::RPW), dthis);
  }
}

}  // namespace sipg
