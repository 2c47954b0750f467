// Config 4: the SIP-Helmholtz apply on 3-D hybrid hex / prism / tet meshes (sm_100a, fp64).
//
// The reference's two-phase apply (pkg/src/dgsipg/sipg.py:558-602) on the shared-trace route
// (sipg.py:513-554 trace rule / geometry, 653-661 TracePhysEval, 663-677 absorb), extended to
// prisms and tets (collapsed-coordinate modified-modal bases built like the reference triangle,
// stdregions.py:266-383; restated and property-tested in oracle/hybrid3d.py).  Plan layout:
// paper_2504_03573_b200/plan3d.py.
//
// Two kernels per element class (shape, n), one CTA per element:
//   k_h3<S, N, true>  (publish): BwdTrans -> PhysDeriv -> per interior coupling, u and n.grad u on
//                     the element's own face grid (endpoint rows along the fixed axis), mapped to
//                     the coupling's trace points (identity or a dense nt x q^2 map) -> published.
//   k_h3<S, N, false> (apply):   the same own traces, the partner's published traces, the SIP flux
//                     (jump, average, penalty), lifted by the transposed map and the transposed
//                     endpoint rows into the volume-point accumulators, plus the volume terms
//                     lambda jw u and jw G G^T grad u; then one transposed pass
//                     y = Phi^T (W0 + sum_k D_k^T W_k)   (IProduct + IProductDeriv, sipg.py:575-582).
// Every element's y is written by exactly one CTA (no atomics, deterministic).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define SIPG_H3_ABI_VERSION 1

enum { H3_HEX = 0, H3_PRISM = 1, H3_TET = 2 };
#define CD3_WORDS 16
enum {
  CD3_SHAPE = 0, CD3_N, CD3_Q, CD3_NC, CD3_COUNT, CD3_ELEM_OFF, CD3_T_PTS, CD3_T_D, CD3_T_W, CD3_T_E,
  CD3_T_A, CD3_T_B, CD3_T_C, CD3_ROLE
};
#define H3_EGEO 8

struct H3Slot {   // numpy dtype plan3d.SLOT
  int32_t face, kind, nt, mkind, moff, wtoff, elem, partner;
  int64_t pub_self, pub_other;
  double tau, sJ, v[3], pad;
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
};

namespace h3 {

constexpr int NT = 128;
constexpr int TMAX = 64;   // trace points per coupling: q_t = max(q_L, q_R) <= 8

template <int S, int N>
struct Cfg {
  static constexpr int Q = N + 1, Q2 = Q * Q, Q3 = Q2 * Q;
  static constexpr int NTRI = N * (N + 1) / 2;
  static constexpr int NG = N + 1;                                   // triangle direction-1 groups
  static constexpr int NPM = NTRI + (S == H3_TET ? 1 : 0);           // + tet apex pseudo-mode
  static constexpr int NC = S == H3_HEX ? N * N * N : (S == H3_PRISM ? N * NTRI : N * (N + 1) * (N + 2) / 6);
  static constexpr int S1 = S == H3_HEX ? N * N * Q : NPM * Q;
  static constexpr int S2 = S == H3_HEX ? N * Q2 : NG * Q2;
  static constexpr int NCP = (NC + 1) & ~1;
  static constexpr int NI = 4 * NPM + 4 + NC;                        // int tables
  static constexpr int doubles(bool pub) {
    return NCP + 4 * Q3 + (pub ? 0 : 4 * Q3) + S1 + S2 + 5 * Q2 + 4 * TMAX;
  }
  static constexpr size_t smem_bytes(bool pub) { return sizeof(double) * doubles(pub) + sizeof(int) * NI; }
};

// (fixed axis, side, run axis 0, run axis 1) per shape and local face (plan3d.FACES)
__constant__ int8_t c_faces[3][6][4] = {
    {{0, -1, 1, 2}, {0, 1, 1, 2}, {1, -1, 0, 2}, {1, 1, 0, 2}, {2, -1, 0, 1}, {2, 1, 0, 1}},
    {{2, -1, 0, 1}, {1, -1, 0, 2}, {0, 1, 1, 2}, {1, 1, 0, 2}, {0, -1, 1, 2}, {0, 0, 0, 0}},
    {{2, -1, 0, 1}, {1, -1, 0, 2}, {0, 1, 1, 2}, {0, -1, 1, 2}, {0, 0, 0, 0}, {0, 0, 0, 0}},
};

// collapse chain d eta_k / d xi_j (upper triangular, c22 = 1, c10 = c20 = c21 = 0)
struct Chain {
  double c00, c01, c02, c11, c12;
};
template <int S>
__device__ __forceinline__ Chain chain(double e0, double e1, double e2) {
  Chain c{1.0, 0.0, 0.0, 1.0, 0.0};
  if (S == H3_PRISM) {
    const double r = 1.0 / (1.0 - e2);
    c.c00 = 2.0 * r;
    c.c02 = (1.0 + e0) * r;
  } else if (S == H3_TET) {
    const double r2 = 1.0 / (1.0 - e2), r12 = r2 / (1.0 - e1);
    c.c00 = 4.0 * r12;
    c.c01 = c.c02 = 2.0 * (1.0 + e0) * r12;
    c.c11 = 2.0 * r2;
    c.c12 = (1.0 + e1) * r2;
  }
  return c;
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

// u = Phi c on the q^3 grid (generalised tensor product; stages as plan3d.ClassTables3 tables)
template <int S, int N>
__device__ void bwd(const double* __restrict__ c, double* __restrict__ u, double* s1, double* s2,
                    const double* __restrict__ A, const double* __restrict__ B, const double* __restrict__ Ct,
                    const int* gstart, const int* gmem, const int* coff) {
  using C = Cfg<S, N>;
  constexpr int Q = C::Q, Q2 = C::Q2, Q3 = C::Q3, NG = C::NG;
  const int t = threadIdx.x;
  if (S == H3_HEX) {
    for (int o = t; o < N * N * Q; o += NT) {
      const int k2 = o % Q, i01 = o / Q;
      double a = 0.0;
#pragma unroll
      for (int i2 = 0; i2 < N; ++i2) a = fma(__ldg(A + k2 * N + i2), c[i01 * N + i2], a);
      s1[o] = a;
    }
    __syncthreads();
    for (int o = t; o < N * Q2; o += NT) {
      const int k2 = o % Q, k1 = (o / Q) % Q, i0 = o / Q2;
      double a = 0.0;
#pragma unroll
      for (int i1 = 0; i1 < N; ++i1) a = fma(__ldg(A + k1 * N + i1), s1[(i0 * N + i1) * Q + k2], a);
      s2[o] = a;
    }
    __syncthreads();
    for (int o = t; o < Q3; o += NT) {
      const int k12 = o % Q2, k0 = o / Q2;
      double a = 0.0;
#pragma unroll
      for (int i0 = 0; i0 < N; ++i0) a = fma(__ldg(A + k0 * N + i0), s2[i0 * Q2 + k12], a);
      u[o] = a;
    }
    __syncthreads();
    return;
  }
  // stage 1: the innermost family (prism: psi on eta1 per triangle mode; tet: C rows on eta2)
  for (int o = t; o < C::NPM * Q; o += NT) {
    const int k = o % Q, m = o / Q;
    double a = 0.0;
    if (S == H3_PRISM) {
#pragma unroll
      for (int l = 0; l < N; ++l) a = fma(__ldg(Ct + k * N + l), c[m * N + l], a);
    } else {
      for (int r = coff[m]; r < coff[m + 1]; ++r) a = fma(__ldg(Ct + r * Q + k), c[r], a);
    }
    s1[o] = a;
  }
  __syncthreads();
  // stage 2: group sums with the B rows (prism: B on eta2, s1 over eta1; tet: B on eta1, s1 over eta2)
  for (int o = t; o < NG * Q2; o += NT) {
    const int k2 = o % Q, k1 = (o / Q) % Q, g = o / Q2;
    const int kb = S == H3_PRISM ? k2 : k1, ko = S == H3_PRISM ? k1 : k2;
    double a = 0.0;
    for (int q = gstart[g]; q < gstart[g + 1]; ++q) {
      const int m = gmem[q];
      a = fma(__ldg(B + m * Q + kb), s1[m * Q + ko], a);
    }
    s2[o] = a;
  }
  __syncthreads();
  for (int o = t; o < Q3; o += NT) {
    const int k12 = o % Q2, k0 = o / Q2;
    double a = 0.0;
#pragma unroll
    for (int g = 0; g < NG; ++g) a = fma(__ldg(A + k0 * NG + g), s2[g * Q2 + k12], a);
    u[o] = a;
  }
  __syncthreads();
}

// y = Phi^T T (transposed stages), written to global
template <int S, int N>
__device__ void bwd_t(const double* __restrict__ T, double* __restrict__ y, double* s1, double* s2,
                      const double* __restrict__ A, const double* __restrict__ B, const double* __restrict__ Ct,
                      const int* gof, const int* mofr) {
  using C = Cfg<S, N>;
  constexpr int Q = C::Q, Q2 = C::Q2, NG = C::NG;
  const int t = threadIdx.x;
  if (S == H3_HEX) {
    for (int o = t; o < N * Q2; o += NT) {
      const int k12 = o % Q2, i0 = o / Q2;
      double a = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < Q; ++k0) a = fma(__ldg(A + k0 * N + i0), T[k0 * Q2 + k12], a);
      s2[o] = a;
    }
    __syncthreads();
    for (int o = t; o < N * N * Q; o += NT) {
      const int k2 = o % Q, i1 = (o / Q) % N, i0 = o / (N * Q);
      double a = 0.0;
#pragma unroll
      for (int k1 = 0; k1 < Q; ++k1) a = fma(__ldg(A + k1 * N + i1), s2[(i0 * Q + k1) * Q + k2], a);
      s1[o] = a;
    }
    __syncthreads();
    for (int o = t; o < N * N * N; o += NT) {
      const int i2 = o % N, i01 = o / N;
      double a = 0.0;
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) a = fma(__ldg(A + k2 * N + i2), s1[i01 * Q + k2], a);
      y[o] = a;
    }
    return;
  }
  for (int o = t; o < NG * Q2; o += NT) {
    const int k12 = o % Q2, g = o / Q2;
    double a = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < Q; ++k0) a = fma(__ldg(A + k0 * NG + g), T[k0 * Q2 + k12], a);
    s2[o] = a;
  }
  __syncthreads();
  for (int o = t; o < C::NPM * Q; o += NT) {
    const int k = o % Q, m = o / Q, g = gof[m];
    double a = 0.0;
    if (S == H3_PRISM) {   // s1[m][k1] = sum_k2 B[m][k2] s2[g][k1][k2]
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) a = fma(__ldg(B + m * Q + k2), s2[(g * Q + k) * Q + k2], a);
    } else {               // s1[m][k2] = sum_k1 B[m][k1] s2[g][k1][k2]
#pragma unroll
      for (int k1 = 0; k1 < Q; ++k1) a = fma(__ldg(B + m * Q + k1), s2[(g * Q + k1) * Q + k], a);
    }
    s1[o] = a;
  }
  __syncthreads();
  for (int r = t; r < C::NC; r += NT) {
    double a = 0.0;
    if (S == H3_PRISM) {
      const int m = r / N, l = r % N;
#pragma unroll
      for (int k1 = 0; k1 < Q; ++k1) a = fma(__ldg(Ct + k1 * N + l), s1[m * Q + k1], a);
    } else {
      const int m = mofr[r];
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) a = fma(__ldg(Ct + r * Q + k2), s1[m * Q + k2], a);
    }
    y[r] = a;
  }
}

template <int S, int N, bool PUB>
__global__ void __launch_bounds__(NT) k_h3(const H3Plan P, const int cls, const double* __restrict__ x,
                                           double* __restrict__ y) {
  using C = Cfg<S, N>;
  constexpr int Q = C::Q, Q2 = C::Q2, Q3 = C::Q3;
  extern __shared__ double sm[];
  double* c = sm;
  double* u = c + C::NCP;
  double* du = u + Q3;
  double* W = du + 3 * Q3;
  double* s1 = W + (PUB ? 0 : 4 * Q3);
  double* s2 = s1 + C::S1;
  double* gnc = s2 + C::S2;      // 3 Q2: G.n per own-face-grid point
  double* fa = gnc + 3 * Q2;     // own-grid u, then lifted fv
  double* fb = fa + Q2;          // own-grid n.grad u, then lifted fd
  double* tr = fb + Q2;          // 4 TMAX: trace u, g, fv, fd
  int* gstart = (int*)(tr + 4 * TMAX);
  int* gmem = gstart + C::NPM + 2;
  int* gof = gmem + C::NPM;
  int* coff = gof + C::NPM;
  int* mofr = coff + C::NPM + 2;
  const int t = threadIdx.x;
  const int32_t* cd = P.cd + cls * CD3_WORDS;
  const int count = cd[CD3_COUNT];
  const double* pts = P.tab + cd[CD3_T_PTS];
  const double* Dt = P.tab + cd[CD3_T_D];
  const double* Wr = P.tab + cd[CD3_T_W];
  const double* Et = P.tab + cd[CD3_T_E];
  const double* At = P.tab + cd[CD3_T_A];
  const double* Bt = S == H3_HEX ? At : P.tab + cd[CD3_T_B];
  const double* Ct = S == H3_HEX ? At : P.tab + cd[CD3_T_C];
  if (S != H3_HEX) build_int_tables<S, N>(gstart, gmem, gof, coff, mofr);
  __syncthreads();
  for (int i = blockIdx.x; i < count; i += gridDim.x) {
    const int e = P.class_elems[cd[CD3_ELEM_OFF] + i];
    const int64_t dof = P.dof_off[e];
    for (int r = t; r < C::NC; r += NT) c[r] = __ldg(x + dof + r);
    __syncthreads();
    bwd<S, N>(c, u, s1, s2, At, Bt, Ct, gstart, gmem, coff);
    // PhysDeriv: collocation along each eta axis (stdregions.py:658-674)
    for (int o = t; o < Q3; o += NT) {
      const int k0 = o / Q2, k1 = (o / Q) % Q, k2 = o % Q;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        a0 = fma(__ldg(Dt + k0 * Q + j), u[j * Q2 + k1 * Q + k2], a0);
        a1 = fma(__ldg(Dt + Q2 + k1 * Q + j), u[k0 * Q2 + j * Q + k2], a1);
        a2 = fma(__ldg(Dt + 2 * Q2 + k2 * Q + j), u[k0 * Q2 + k1 * Q + j], a2);
      }
      du[o] = a0;
      du[Q3 + o] = a1;
      du[2 * Q3 + o] = a2;
      if (!PUB) W[o] = W[Q3 + o] = W[2 * Q3 + o] = W[3 * Q3 + o] = 0.0;
    }
    __syncthreads();
    const int64_t sb = P.slot_off[e], se = P.slot_off[e + 1];
    for (int64_t si = sb; si < se; ++si) {
      const H3Slot* sl = P.slots + si;
      const int kind = sl->kind;
      if (PUB && kind == 0) continue;
      const int face = sl->face, nt = sl->nt, mk = sl->mkind;
      const int fx = c_faces[S][face][0], sd = c_faces[S][face][1], ra = c_faces[S][face][2],
                rb = c_faces[S][face][3];
      const int st_f = fx == 0 ? Q2 : (fx == 1 ? Q : 1);
      const int st_a = ra == 0 ? Q2 : (ra == 1 ? Q : 1);
      const int st_b = rb == 0 ? Q2 : (rb == 1 ? Q : 1);
      const double* E = Et + (fx * 2 + (sd > 0)) * Q;
      const double v0 = sl->v[0], v1 = sl->v[1], v2 = sl->v[2];
      // 1. own face grid: u and n.grad u through the endpoint rows of the fixed axis (face_values_from_phys)
      for (int a = t; a < Q2; a += NT) {
        const int ia = a / Q, ib = a % Q;
        const int base = ia * st_a + ib * st_b;
        double uf = 0.0, d0 = 0.0, d1 = 0.0, d2 = 0.0;
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          const double ek = __ldg(E + k);
          const int vi = base + k * st_f;
          uf = fma(ek, u[vi], uf);
          d0 = fma(ek, du[vi], d0);
          d1 = fma(ek, du[Q3 + vi], d1);
          d2 = fma(ek, du[2 * Q3 + vi], d2);
        }
        double eta[3];
        eta[fx] = (double)sd;
        eta[ra] = __ldg(pts + ra * Q + ia);
        eta[rb] = __ldg(pts + rb * Q + ib);
        const Chain ch = chain<S>(eta[0], eta[1], eta[2]);
        const double g0 = ch.c00 * v0 + ch.c01 * v1 + ch.c02 * v2;
        const double g1 = ch.c11 * v1 + ch.c12 * v2;
        const double g2 = v2;
        gnc[a] = g0;
        gnc[Q2 + a] = g1;
        gnc[2 * Q2 + a] = g2;
        fa[a] = uf;
        fb[a] = g0 * d0 + g1 * d1 + g2 * d2;
      }
      __syncthreads();
      // 2. to the trace points
      const double* M = mk ? P.tab + sl->moff : nullptr;
      double* ut = tr;
      double* gt = tr + TMAX;
      if (mk) {
        for (int p = t; p < nt; p += NT) {
          double a0 = 0.0, a1 = 0.0;
          const double* row = M + (int64_t)p * Q2;
          for (int a = 0; a < Q2; ++a) {
            const double m = __ldg(row + a);
            a0 = fma(m, fa[a], a0);
            a1 = fma(m, fb[a], a1);
          }
          ut[p] = a0;
          gt[p] = a1;
        }
      } else {
        ut = fa;
        gt = fb;
      }
      __syncthreads();
      if (PUB) {
        double* dst = P.pub + sl->pub_self;
        for (int p = t; p < nt; p += NT) {
          dst[2 * p] = ut[p];
          dst[2 * p + 1] = gt[p];
        }
        __syncthreads();
        continue;
      }
      // 3. SIP flux at the trace points (sipg.py:622-650, 663-677): boundary jump 2u, average g
      double* fv = tr + 2 * TMAX;
      double* fd = tr + 3 * TMAX;
      {
        const double tau = sl->tau, sJ = sl->sJ;
        const double* wt = P.tab + sl->wtoff;
        const double* nb = kind ? P.pub + sl->pub_other : nullptr;
        for (int p = t; p < nt; p += NT) {
          const double un = kind ? nb[2 * p] : -ut[p];
          const double gn = kind ? nb[2 * p + 1] : -gt[p];
          const double j = ut[p] - un, cc = 0.5 * (gt[p] - gn);
          const double w = sJ * __ldg(wt + p);
          fv[p] = (tau * j - cc) * w;
          fd[p] = -0.5 * j * w;
        }
      }
      __syncthreads();
      // 4. back to the own face grid (transposed map)
      const double* fvA = fv;
      const double* fdA = fd;
      if (mk) {
        for (int a = t; a < Q2; a += NT) {
          double a0 = 0.0, a1 = 0.0;
          for (int p = 0; p < nt; ++p) {
            const double m = __ldg(M + (int64_t)p * Q2 + a);
            a0 = fma(m, fv[p], a0);
            a1 = fma(m, fd[p], a1);
          }
          fa[a] = a0;
          fb[a] = a1;
        }
        fvA = fa;
        fdA = fb;
        __syncthreads();
      }
      // 5. transposed endpoint rows into the volume accumulators (the reference's scatter + final sweep)
      for (int o = t; o < Q * Q2; o += NT) {
        const int k = o / Q2, a = o % Q2;
        const int vi = (a / Q) * st_a + (a % Q) * st_b + k * st_f;
        const double ek = __ldg(E + k);
        const double fvk = ek * fvA[a], fdk = ek * fdA[a];
        W[vi] += fvk;
        W[Q3 + vi] = fma(gnc[a], fdk, W[Q3 + vi]);
        W[2 * Q3 + vi] = fma(gnc[Q2 + a], fdk, W[2 * Q3 + vi]);
        W[3 * Q3 + vi] = fma(gnc[2 * Q2 + a], fdk, W[3 * Q3 + vi]);
      }
      __syncthreads();
    }
    if (PUB) continue;
    // volume terms (sipg.py:575-582): lambda jw u, jw G G^T grad u with G = chain * dxi/dx
    {
      const double* eg = P.egeo + (int64_t)e * H3_EGEO;
      const double dJ = __ldg(eg), S00 = __ldg(eg + 1), S01 = __ldg(eg + 2), S02 = __ldg(eg + 3),
                   S11 = __ldg(eg + 4), S12 = __ldg(eg + 5), S22 = __ldg(eg + 6);
      const double lam = P.lam;
      for (int o = t; o < Q3; o += NT) {
        const int k0 = o / Q2, k1 = (o / Q) % Q, k2 = o % Q;
        const Chain ch = chain<S>(__ldg(pts + k0), __ldg(pts + Q + k1), __ldg(pts + 2 * Q + k2));
        const double jw = dJ * __ldg(Wr + o);
        const double d0 = du[o], d1 = du[Q3 + o], d2 = du[2 * Q3 + o];
        const double x0 = ch.c00 * d0, x1 = ch.c01 * d0 + ch.c11 * d1, x2 = ch.c02 * d0 + ch.c12 * d1 + d2;
        const double f0 = S00 * x0 + S01 * x1 + S02 * x2;
        const double f1 = S01 * x0 + S11 * x1 + S12 * x2;
        const double f2 = S02 * x0 + S12 * x1 + S22 * x2;
        W[o] = fma(lam * jw, u[o], W[o]);
        W[Q3 + o] += jw * (ch.c00 * f0 + ch.c01 * f1 + ch.c02 * f2);
        W[2 * Q3 + o] += jw * (ch.c11 * f1 + ch.c12 * f2);
        W[3 * Q3 + o] += jw * f2;
      }
    }
    __syncthreads();
    // T = W0 + sum_k D_k^T W_k  (into u)
    for (int o = t; o < Q3; o += NT) {
      const int k0 = o / Q2, k1 = (o / Q) % Q, k2 = o % Q;
      double a = W[o];
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        a = fma(__ldg(Dt + j * Q + k0), W[Q3 + j * Q2 + k1 * Q + k2], a);
        a = fma(__ldg(Dt + Q2 + j * Q + k1), W[2 * Q3 + k0 * Q2 + j * Q + k2], a);
        a = fma(__ldg(Dt + 2 * Q2 + j * Q + k2), W[3 * Q3 + k0 * Q2 + k1 * Q + j], a);
      }
      u[o] = a;
    }
    __syncthreads();
    bwd_t<S, N>(u, y + dof, s1, s2, At, Bt, Ct, gof, mofr);
    __syncthreads();
  }
}

}  // namespace h3
