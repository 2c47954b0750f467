// Published face planes + planes-consuming hexahedron kernel (sm_100a, fp64).
//
// k_planes (phase 1, one pass over x): every hex element publishes, for each of
// its six faces, the boundary-mode plane (the modes that do not vanish on the
// face) and the normal-derivative plane sum_i psi_i'(+-1) c[.., i, ..] — the
// face trace of u and d_n u in modal form, N^2 doubles each.  This is the
// reference's phase-1 trace publish (sipg.py:585-592) in the form a
// sum-factorised neighbour evaluation needs, and the multi-GPU halo unit.
//
// k_hexp (phase 2): the register-column volume kernel of k_hex, with every
// neighbour face (conforming, or p-nonconforming shared trace) read as its two
// planes (one TMA bulk copy per face): conforming faces evaluate them on the own
// face grid with the element's V; shared traces evaluate them at the trace
// points with the other side's 1-D tables E_k = psi(other's parameter of t_k),
// interpolate the own trace to the trace grid (1-D matrices), form the SIP flux
// there with the trace quadrature, and fold it back with the transposed
// interpolation (reference sipg.py:513-554, 640-650) — all exact for q >= n.
#pragma once
#include "sipg_kernels.cuh"
#include "sipg_hex_fast.cuh"

namespace sipg {

template <int N, int Q>
__global__ void __launch_bounds__(128)
k_planes(const DevPlan P, const int cls, const double* __restrict__ x) {
  constexpr int N3 = N * N * N, NN = (N * N + 1) & ~1;
  __shared__ double c[N3];
  const int t = threadIdx.x;
  const int* cd = P.cd + cls * CD_WORDS;
  const int count = cd[CD_COUNT];
  const int* elist = P.class_elems + cd[CD_ELEM_OFF];
  for (int iel = blockIdx.x; iel < count; iel += gridDim.x) {
    const int e = elist[iel];
    const double* xe = x + P.dof_off[e];
    for (int i = t; i < N3; i += 128) c[i] = __ldg(xe + i);
    __syncthreads();
    double* out = P.planes + P.plane_off[e];
    for (int it = t; it < 6 * N * N; it += 128) {
      const int f = it / (N * N), r = it - f * (N * N);
      const int i0 = r / N, i1 = r - (r / N) * N;
      const int a = f >> 1, hi = f & 1;
      const int b0 = a == 0 ? 1 : 0, b1 = a == 2 ? 1 : 2;
      const int base = i0 * hex_stride(b0, N) + i1 * hex_stride(b1, N), sa = hex_stride(a, N);
      double pd = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) pd = fma(hxDVE<N, Q>[hi * N + i], c[base + i * sa], pd);
      out[f * 2 * NN + r] = c[base + (hi ? (N - 1) * sa : 0)];
      out[f * 2 * NN + NN + r] = pd;
    }
    __syncthreads();
  }
}

// Shared-trace scratch layout (doubles, from SHX): tables E0, E1 (QM x NM), I0, I1 (QM x QM),
// weights (2 QM), T (2 QM NM), UO (2 QM^2), SI (2 QM^2), SS (2 QM^2), FL (2 QM^2), G (2 QM^2)
// QM / NM: the instantiation's largest trace size / neighbour order (sizes the scratch: a class of
// order N only takes fast shared faces with neighbours of order <= N + SIPG_SF_RANGE, plan.py)
template <int QM, int NM>
struct ShScr {
  static constexpr int QMX = QM, NMX = NM;
  double* base;
  __device__ double* tE0() const { return base; }
  __device__ double* tE1() const { return base + QM * NM; }
  __device__ double* tI0() const { return base + 2 * QM * NM; }
  __device__ double* tI1() const { return base + 2 * QM * NM + QM * QM; }
  __device__ double* tw0() const { return base + 2 * QM * NM + 2 * QM * QM; }
  __device__ double* tw1() const { return tw0() + 2 * QM; }
  __device__ double* sT() const { return tw1() + 2 * QM; }
  __device__ double* sUO() const { return sT() + 2 * QM * NM; }
  __device__ double* sSI() const { return sUO() + 2 * QM * QM; }
  __device__ double* sSS() const { return sSI() + 2 * QM * QM; }
  __device__ double* sFL() const { return sSS() + 2 * QM * QM; }
  __device__ double* sG() const { return sFL() + 2 * QM * QM; }
  static constexpr int doubles() { return 4 * QM * NM + 12 * QM * QM + 4 * QM + 16; }
};

// One fast shared-trace face (F_FAST_SHARED): the neighbour's published planes evaluated at the
// trace points with its 1-D tables, the own trace interpolated there, the SIP flux on the trace
// grid (self normal n, other -n, one metric: reference sipg.py:640-650) and the transposed
// interpolation back to the own face grid.  NO / QT > 0: compile-time neighbour order and trace
// size (the common cases, fully unrolled); 0: runtime sizes.  Called by every thread of the CTA.
template <int N, int Q, int NO, int QT, class SC>
__device__ __noinline__ void shared_face(const int no_rt, const int qt_rt, const int t, const int f,
                                         const FaceRec& r, const int64_t e01, const double* pl,
                                         const double* __restrict__ T, const double* OWN, double* FVD,
                                         const SC sc) {
  constexpr int NT = Q * Q, QQ = Q * Q;
  const int no = NO ? NO : no_rt, qt = QT ? QT : qt_rt;
  double *tE0 = sc.tE0(), *tE1 = sc.tE1(), *tI0 = sc.tI0(), *tI1 = sc.tI1(), *tw0 = sc.tw0(), *tw1 = sc.tw1();
  double *sT = sc.sT(), *sUO = sc.sUO(), *sSI = sc.sSI(), *sSS = sc.sSS(), *sFL = sc.sFL(), *sG = sc.sG();
  const double* gE0 = T + (int)(e01 & 0xffffffff);
  const double* gE1 = T + (int)(e01 >> 32);
  const bool sid = (r.flags & F_SELF_ID) != 0;
  for (int i = t; i < qt * no; i += NT) { tE0[i] = __ldg(gE0 + i); tE1[i] = __ldg(gE1 + i); }
  if (!sid)
    for (int i = t; i < qt * Q; i += NT) { tI0[i] = __ldg(T + r.ts0 + i); tI1[i] = __ldg(T + r.ts1 + i); }
  for (int i = t; i < qt; i += NT) { tw0[i] = __ldg(T + r.wt0 + i); tw1[i] = __ldg(T + r.wt1 + i); }
  __syncthreads();
  const int nno = (no * no + 1) & ~1;
  // other: planes -> trace points, axis 0
#pragma unroll 2
  for (int it = t; it < 2 * qt * no; it += NT) {
    const int plx = it / (qt * no), r0 = it - plx * qt * no, p0 = r0 / no, i1 = r0 - p0 * no;
    double s = 0.0;
#pragma unroll
    for (int i0 = 0; i0 < (NO ? NO : SC::NMX); ++i0)
      if (NO || i0 < no) s = fma(tE0[p0 * no + i0], pl[plx * nno + i0 * no + i1], s);
    sT[it] = s;
  }
  // own: face grid -> trace points, axis 0
  if (!sid)
#pragma unroll 2
    for (int it = t; it < 2 * qt * Q; it += NT) {
      const int plx = it / (qt * Q), r0 = it - plx * qt * Q, p0 = r0 / Q, q1 = r0 - p0 * Q;
      const double* o = OWN + f * 2 * QQ + plx * QQ;
      double s = 0.0;
#pragma unroll
      for (int q0 = 0; q0 < Q; ++q0) s = fma(tI0[p0 * Q + q0], o[q0 * Q + q1], s);
      sSI[it] = s;
    }
  __syncthreads();
  // axis 1 for both
#pragma unroll 2
  for (int it = t; it < 2 * qt * qt; it += NT) {
    const int plx = it / (qt * qt), r0 = it - plx * qt * qt, p0 = r0 / qt, p1 = r0 - p0 * qt;
    double s = 0.0;
#pragma unroll
    for (int i1 = 0; i1 < (NO ? NO : SC::NMX); ++i1)
      if (NO || i1 < no) s = fma(tE1[p1 * no + i1], sT[plx * qt * no + p0 * no + i1], s);
    sUO[it] = s;
    if (!sid) {
      double w = 0.0;
#pragma unroll
      for (int q1 = 0; q1 < Q; ++q1) w = fma(tI1[p1 * Q + q1], sSI[plx * qt * Q + p0 * Q + q1], w);
      sSS[it] = w;
    }
  }
  __syncthreads();
  const int ao = r.nbr_face >> 1;
  const double goa = r.go[ao], sJ = r.sJ, tau = r.tau;
  for (int p = t; p < qt * qt; p += NT) {
    const int p0 = p / qt, p1 = p - p0 * qt;
    const double us = sid ? OWN[f * 2 * QQ + p] : sSS[p];
    const double gs = sid ? OWN[f * 2 * QQ + QQ + p] : sSS[qt * qt + p];
    const double jump = us - sUO[p];
    const double avg = 0.5 * (gs - goa * sUO[qt * qt + p]);
    const double swj = sJ * tw0[p0] * tw1[p1];
    const double fv = (tau * jump - avg) * swj, fd = -0.5 * jump * swj;
    if (sid) {
      FVD[f * 2 * QQ + p] = fv;
      FVD[f * 2 * QQ + QQ + p] = fd;
    } else {
      sFL[p] = fv;
      sFL[qt * qt + p] = fd;
    }
  }
  if (!sid) {
    __syncthreads();
    // back to the own face grid: transposed interpolation along both axes
#pragma unroll 2
    for (int it = t; it < 2 * Q * qt; it += NT) {
      const int plx = it / (Q * qt), r0 = it - plx * Q * qt, q0 = r0 / qt, p1 = r0 - q0 * qt;
      double s = 0.0;
#pragma unroll
      for (int p0 = 0; p0 < (QT ? QT : SC::QMX); ++p0)
        if (QT || p0 < qt) s = fma(tI0[p0 * Q + q0], sFL[plx * qt * qt + p0 * qt + p1], s);
      sG[it] = s;
    }
    __syncthreads();
    for (int it = t; it < 2 * QQ; it += NT) {
      const int plx = it / QQ, r0 = it - plx * QQ, q0 = r0 / Q, q1 = r0 - q0 * Q;
      double s = 0.0;
#pragma unroll
      for (int p1 = 0; p1 < (QT ? QT : SC::QMX); ++p1)
        if (QT || p1 < qt) s = fma(tI1[p1 * Q + q1], sG[plx * Q * qt + q0 * qt + p1], s);
      FVD[f * 2 * QQ + it] = s;
    }
  }
}

// compiled neighbour-order variants: |NO - N| <= SIPG_SF_RANGE (code size vs instruction cache)
#ifndef SIPG_SF_RANGE
#define SIPG_SF_RANGE 3
#endif
// neighbour orders |NO - N| <= SIPG_SF_CRANGE get a compiled (fully unrolled) variant, the rest the
// runtime-size one (code size vs instruction cache: ncu shows 35 % no-instruction stalls at 3)
#ifndef SIPG_SF_CRANGE
#define SIPG_SF_CRANGE SIPG_SF_RANGE
#endif
// 0: every shared face takes the runtime-size variant (one copy of the code: instruction cache)
#ifndef SIPG_SF_COMPILED
#define SIPG_SF_COMPILED 1
#endif
// compile-time dispatch over the neighbour order NO in [LO, HI] (trace size max(Q, NO + 1),
// the GLL / GLL case F_FAST_SHARED covers); anything else takes the runtime-size variant
template <int N, int Q, int LO, int HI, class SC>
__device__ __forceinline__ void sf_dispatch(const int no, const int qt, const int t, const int f, const FaceRec& r,
                                            const int64_t e01, const double* pl, const double* T,
                                            const double* OWN, double* FVD, const SC sc) {
  if constexpr (LO > HI || !SIPG_SF_COMPILED) {
    shared_face<N, Q, 0, 0>(no, qt, t, f, r, e01, pl, T, OWN, FVD, sc);
  } else {
    constexpr int QTV = Q > LO + 1 ? Q : LO + 1;
    if (LO != N && no == LO && qt == QTV)
      shared_face<N, Q, LO, QTV>(no, qt, t, f, r, e01, pl, T, OWN, FVD, sc);
    else
      sf_dispatch<N, Q, LO + 1, HI>(no, qt, t, f, r, e01, pl, T, OWN, FVD, sc);
  }
}

template <int N, int Q, bool SH>
struct HexPlanes {
  static constexpr int NT = Q * Q;
  static constexpr int SJ = (Q & 1) ? Q : Q + 1;
  static constexpr int SI = Q * SJ;
  static constexpr int BUF = Q * SI;
  static constexpr int N3 = N * N * N;
  static constexpr int QQ = Q * Q;
  static constexpr int BLK = (N3 + 2 + 1) & ~1;
  // neighbour orders of the fast faces: <= N + SIPG_SF_RANGE (F_FAST_SHARED is set only then, plan.py)
  static constexpr int NM = N + SIPG_SF_RANGE < NMAX ? N + SIPG_SF_RANGE : NMAX;
  static constexpr int QM0 = Q > NM + 1 ? Q : NM + 1;
  static constexpr int QM = QM0 < QMAX ? QM0 : QMAX;
  static constexpr int NNX = NM * NM + 2;              // one plane slot
  static constexpr int RECW = 96 + 12;                 // 6 records + 6 x 2 ext words (doubles)
  // face-phase scratch: U2 (6 x 2 x QQ), OWN (6 x 2 x QQ), FVD (6 x 2 x QQ), T1 (12 Q N)
  static constexpr int FACE = 36 * QQ + 12 * Q * N;
  // shared-trace scratch (SH): tables, T, UO, SI, SS, FL, G
  static constexpr int SHS = SH ? ShScr<QM, NM>::doubles() : 0;
  static constexpr int S0 = 3 * BUF > FACE + SHS ? 3 * BUF : FACE + SHS;
  static constexpr int SCR = (S0 + 1) & ~1;
  // dynamic shared memory (doubles): REC[2] | CO[2] | NBP[6] | S
  static constexpr int O_REC = 0;
  static constexpr int O_CO = 2 * RECW;
  static constexpr int O_NB = O_CO + 2 * BLK;
  static constexpr int O_S = O_NB + 6 * 2 * NNX;
  static size_t smem_bytes() { return sizeof(double) * (size_t)(O_S + SCR); }
};

template <int N, int Q, bool SH>
__global__ void __launch_bounds__(Q * Q, (Q <= 8 ? SIPG_HEX_MINB : 1))
k_hexp(const DevPlan P, const int cls, const double* __restrict__ x, double* __restrict__ y) {
  using H = HexPlanes<N, Q, SH>;
  constexpr int NT = H::NT, SJ = H::SJ, SI = H::SI, BUF = H::BUF, N3 = H::N3, QQ = H::QQ, NNX = H::NNX;
  extern __shared__ __align__(16) double dsm[];
  double* NBP = dsm + H::O_NB;
  double* S = dsm + H::O_S;
  __shared__ double sW[Q];
  __shared__ int sk[6];               // 1 fast conforming, 2 boundary, 3 fast shared
  __shared__ int soff[8];
  __shared__ int sno[6];              // neighbour n_modes
  __shared__ __align__(8) uint64_t mbar[3];
  double* B0 = S;
  double* B1 = S + BUF;
  double* B2 = S + 2 * BUF;
  const int t = threadIdx.x;
  const int ta = t / Q, tb = t - (t / Q) * Q;
  const int* cd = P.cd + cls * CD_WORDS;
  const int count = cd[CD_COUNT];
  const int* elist = P.class_elems + cd[CD_ELEM_OFF];
  const double lam = P.lam;
  const double* T = P.tab;
  if (t == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&mbar[2], 6);
    fence_proxy_async();
  }
  if (t < Q) sW[t] = hxW<N, Q>[t];
  __syncthreads();
  auto issue_own = [&](int iel, int st) {
    const int64_t r0 = cd[CD_REC_OFF] + (int64_t)iel * 6;
    double* rec = dsm + H::O_REC + st * H::RECW;
    bulk_g2s(rec, P.recs + r0, 6 * sizeof(FaceRec), &mbar[st]);
    bulk_g2s(rec + 96, P.rec_ext + 2 * r0, 6 * 16, &mbar[st]);
    unsigned nb;
    soff[st] = bulk_block(dsm + H::O_CO + st * H::BLK, x + P.dof_off[elist[iel]], N3, &mbar[st], &nb);
    mbar_expect_tx(&mbar[st], 6 * sizeof(FaceRec) + 96 + nb);
    cp_async_commit();
  };
  if (t == 0 && blockIdx.x < count) issue_own(blockIdx.x, 0);

  int kk = 0;
  for (int iel = blockIdx.x; iel < count; iel += gridDim.x, ++kk) {
    const int st = kk & 1;
    const bool more = iel + (int)gridDim.x < count;
    if (t == 0 && more) issue_own(iel + gridDim.x, st ^ 1);
    if (t == 0) {
      if (more) cp_async_wait<1>(); else cp_async_wait<0>();
    }
    mbar_wait(&mbar[st], (kk >> 1) & 1);
    __syncthreads();
    const double* rec = dsm + H::O_REC + st * H::RECW;
    const FaceRec* srec = reinterpret_cast<const FaceRec*>(rec);
    const int64_t* sext = reinterpret_cast<const int64_t*>(rec + 96);
    const double* C = dsm + H::O_CO + st * H::BLK + soff[st];
    const int64_t dof0 = P.dof_off[elist[iel]];
    if (t < 6) {
      const int fl = srec[t].flags, ty = srec[t].type;
      sk[t] = (ty == FT_DIRECT && (fl & F_FAST_HEX)) ? 1
            : (ty == FT_BOUNDARY && !(fl & F_SELF_PW)) ? 2
            : (ty == FT_SHARED && (fl & F_FAST_SHARED)) ? 3 : 0;
    }
    if (t >= NT - 6) {      // neighbour face planes, one bulk copy per face: the last 6 threads
                            // (NT >= 9); thread 0 issues the next-element prefetch
      const int f = t - (NT - 6);
      const int64_t ext = sext[2 * f];
      unsigned nb = 0;
      const int ty = srec[f].type, fl = srec[f].flags;
      const bool use = (ty == FT_DIRECT && (fl & F_FAST_HEX)) || (ty == FT_SHARED && (fl & F_FAST_SHARED));
      if (use && ext >= 0) {
        const int no = (int)(ext >> 48);
        const int nn = (no * no + 1) & ~1;
        const int64_t off = ext & ((int64_t(1) << 48) - 1);
        bulk_g2s(NBP + f * 2 * NNX, P.planes + off, 2 * nn * 8, &mbar[2]);
        nb = 2 * nn * 8;
        sno[f] = no;
      }
      mbar_expect_tx(&mbar[2], nb);
    }

    // ---- BwdTrans (k_hex register-column scheme)
    if (ta < N && tb < N) {
      double v[N], o[Q];
#pragma unroll
      for (int c = 0; c < N; ++c) v[c] = C[(ta * N + tb) * N + c];
      eo_fwdV<N, Q>(v, o);
#pragma unroll
      for (int k = 0; k < Q; ++k) B1[ta * SI + tb * SJ + k] = o[k];
    }
    __syncthreads();
    if (ta < N) {
      double v[N], o[Q];
#pragma unroll
      for (int b = 0; b < N; ++b) v[b] = B1[ta * SI + b * SJ + tb];
      eo_fwdV<N, Q>(v, o);
#pragma unroll
      for (int j = 0; j < Q; ++j) B2[ta * SI + j * SJ + tb] = o[j];
    }
    __syncthreads();
    double u[Q], d0[Q], d1[Q], d2[Q];
    {
      double v[N];
#pragma unroll
      for (int a = 0; a < N; ++a) v[a] = B2[a * SI + ta * SJ + tb];
      eo_fwdV<N, Q>(v, u);
    }
#pragma unroll
    for (int i = 0; i < Q; ++i) B0[i * SI + ta * SJ + tb] = u[i];
    eo_fwdD<N, Q>(u, d0);
    __syncthreads();
    {
      double v[Q], w[Q];
#pragma unroll
      for (int m = 0; m < Q; ++m) {
        v[m] = B0[ta * SI + m * SJ + tb];
        w[m] = B0[ta * SI + tb * SJ + m];
      }
      eo_fwdD<N, Q>(v, d1);
      eo_fwdD<N, Q>(w, d2);
#pragma unroll
      for (int r = 0; r < Q; ++r) {
        B1[ta * SI + r * SJ + tb] = d1[r];
        B2[ta * SI + tb * SJ + r] = d2[r];
      }
    }
    mbar_wait(&mbar[2], kk & 1);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      d1[i] = B1[i * SI + ta * SJ + tb];
      d2[i] = B2[i * SI + ta * SJ + tb];
    }
    __syncthreads();   // S is face scratch from here on

    double* U2 = S;                    // [f][pl][p0][p1]   neighbour trace on the own grid (fast)
    double* OWN = U2 + 12 * QQ;        // [f][pl][p0][p1]   own (u, g_s) on the own grid
    double* FVD = OWN + 12 * QQ;       // [f][pl][p0][p1]   (fv, fd) on the own grid
    double* T1 = FVD + 12 * QQ;        // [f][pl][p0][i1]   stage-1 tiles (fast)
    double* SHX = T1 + 12 * Q * N;     // shared-trace scratch
    // ---- fast faces: stage 1 / 2 of V P V^T from the published planes
    for (int it = t; it < 12 * N; it += NT) {
      const int fp = it / N, i1 = it - (it / N) * N;
      if (sk[fp >> 1] != 1) continue;
      const double* pl = NBP + (fp >> 1) * 2 * NNX + (fp & 1) * ((N * N + 1) & ~1);
      double v[N], o[Q];
#pragma unroll
      for (int i0 = 0; i0 < N; ++i0) v[i0] = pl[i0 * N + i1];
      eo_fwdV<N, Q>(v, o);
#pragma unroll
      for (int p0 = 0; p0 < Q; ++p0) T1[fp * Q * N + p0 * N + i1] = o[p0];
    }
    // ---- own (u, g_s) on every face grid (owners publish)
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      if (sk[f] == 0) continue;
      const double g0 = srec[f].gs[0], g1 = srec[f].gs[1], g2 = srec[f].gs[2];
      double* o = OWN + f * 2 * QQ;
      const int a = f >> 1, hi = f & 1;
      if (a == 0) {
        const int i = hi ? Q - 1 : 0;
        o[ta * Q + tb] = u[i];
        o[QQ + ta * Q + tb] = g0 * d0[i] + g1 * d1[i] + g2 * d2[i];
      } else if (a == 1 ? (ta == (hi ? Q - 1 : 0)) : (tb == (hi ? Q - 1 : 0))) {
        const int q1 = a == 1 ? tb : ta;
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          o[i * Q + q1] = u[i];
          o[QQ + i * Q + q1] = g0 * d0[i] + g1 * d1[i] + g2 * d2[i];
        }
      }
    }
    __syncthreads();
    for (int it = t; it < 12 * Q; it += NT) {
      const int fp = it / Q, p0 = it - (it / Q) * Q;
      if (sk[fp >> 1] != 1) continue;
      double v[N], o[Q];
#pragma unroll
      for (int i1 = 0; i1 < N; ++i1) v[i1] = T1[fp * Q * N + p0 * N + i1];
      eo_fwdV<N, Q>(v, o);
#pragma unroll
      for (int p1 = 0; p1 < Q; ++p1) U2[fp * QQ + p0 * Q + p1] = o[p1];
    }
    // ---- fast shared traces, one face at a time (runtime trace / neighbour sizes)
    if (SH) {
      for (int f = 0; f < 6; ++f) {
        if (sk[f] != 3) continue;
        __syncthreads();
        const FaceRec& r = srec[f];
        ShScr<H::QM, H::NM> sc{SHX};
        sf_dispatch<N, Q, (N - SIPG_SF_CRANGE > 2 ? N - SIPG_SF_CRANGE : 2),
                    (N + SIPG_SF_CRANGE < NMAX ? N + SIPG_SF_CRANGE : NMAX)>(
            sno[f], r.nt0, t, f, r, sext[2 * f + 1], NBP + f * 2 * NNX, T, OWN, FVD, sc);
      }
    }
    __syncthreads();
    // ---- flux at every point of the fast / boundary faces
    for (int it = t; it < 6 * QQ; it += NT) {
      const int f = it / QQ, p = it - (it / QQ) * QQ;
      const int kind = sk[f];
      if (kind != 1 && kind != 2) continue;
      const FaceRec& r = srec[f];
      const int p0 = p / Q, p1 = p - (p / Q) * Q;
      const double* o = OWN + f * 2 * QQ;
      const double swj = r.sJ * sW[p0] * sW[p1];
      const double us = o[p], gs = o[QQ + p];
      double jump, avg;
      if (kind == 2) {
        jump = 2.0 * us;
        avg = gs;
      } else {
        jump = us - U2[(2 * f) * QQ + p];
        avg = 0.5 * (gs - r.go[r.nbr_face >> 1] * U2[(2 * f + 1) * QQ + p]);
      }
      FVD[f * 2 * QQ + p] = (r.tau * jump - avg) * swj;
      FVD[f * 2 * QQ + QQ + p] = -0.5 * jump * swj;
    }
    __syncthreads();

    // ---- volume metric, then lift (fv, fd G n) of every face into the owned points
    {
      const double* eg = P.egeo + cd[CD_EGEO_OFF] + (int64_t)iel * cd[CD_EGEO_STRIDE];
      const double J = eg[0];
      const double K0 = eg[1], K1 = eg[2], K2 = eg[3], K3 = eg[4], K4 = eg[5], K5 = eg[6];
      const double wjk = sW[ta] * sW[tb];
#pragma unroll
      for (int i = 0; i < Q; ++i) {
        const double jw = J * hxW<N, Q>[i] * wjk;
        const double ui = u[i], g0 = d0[i], g1 = d1[i], g2 = d2[i];
        u[i] = lam * jw * ui;
        d0[i] = jw * (K0 * g0 + K1 * g1 + K2 * g2);
        d1[i] = jw * (K1 * g0 + K3 * g1 + K4 * g2);
        d2[i] = jw * (K2 * g0 + K4 * g1 + K5 * g2);
      }
    }
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      if (sk[f] == 0) continue;
      const double gsa = srec[f].gs[0], gsb = srec[f].gs[1], gsc = srec[f].gs[2];
      const double* fvd = FVD + f * 2 * QQ;
      const int a = f >> 1, hi = f & 1;
      if (a == 0) {
        const int i = hi ? Q - 1 : 0;
        const double fv = fvd[ta * Q + tb], fd = fvd[QQ + ta * Q + tb];
        u[i] += fv;
        d0[i] = fma(fd, gsa, d0[i]);
        d1[i] = fma(fd, gsb, d1[i]);
        d2[i] = fma(fd, gsc, d2[i]);
      } else if (a == 1 ? (ta == (hi ? Q - 1 : 0)) : (tb == (hi ? Q - 1 : 0))) {
        const int q1 = a == 1 ? tb : ta;
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          const double fv = fvd[i * Q + q1], fd = fvd[QQ + i * Q + q1];
          u[i] += fv;
          d0[i] = fma(fd, gsa, d0[i]);
          d1[i] = fma(fd, gsb, d1[i]);
          d2[i] = fma(fd, gsc, d2[i]);
        }
      }
    }
    __syncthreads();   // FVD / S reused below

    // ---- R = P0 + D0^T P1 (registers) + D1^T P2 + D2^T P3, then IProduct
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      B1[i * SI + ta * SJ + tb] = d1[i];
      B2[i * SI + ta * SJ + tb] = d2[i];
    }
    {
      double rr[Q];
      eo_trD<N, Q>(d0, rr);
#pragma unroll
      for (int i = 0; i < Q; ++i) u[i] += rr[i];
    }
    __syncthreads();
    {
      double v[Q], w[Q];
#pragma unroll
      for (int m = 0; m < Q; ++m) {
        v[m] = B1[ta * SI + m * SJ + tb];
        w[m] = B2[ta * SI + tb * SJ + m];
      }
      eo_trD<N, Q>(v, d1);
      eo_trD<N, Q>(w, d2);
#pragma unroll
      for (int r = 0; r < Q; ++r) {
        B1[ta * SI + r * SJ + tb] = d1[r];
        B2[ta * SI + tb * SJ + r] = d2[r];
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < Q; ++i) u[i] += B1[i * SI + ta * SJ + tb] + B2[i * SI + ta * SJ + tb];
    {
      double o[N];
      eo_bwdV<N, Q>(u, o);
#pragma unroll
      for (int a = 0; a < N; ++a) B0[a * SI + ta * SJ + tb] = o[a];
    }
    __syncthreads();
    if (ta < N) {
      double v[Q], o[N];
#pragma unroll
      for (int j = 0; j < Q; ++j) v[j] = B0[ta * SI + j * SJ + tb];
      eo_bwdV<N, Q>(v, o);
#pragma unroll
      for (int b = 0; b < N; ++b) B1[ta * SI + b * SJ + tb] = o[b];
    }
    __syncthreads();
    if (ta < N && tb < N) {
      double v[Q], o[N];
#pragma unroll
      for (int k = 0; k < Q; ++k) v[k] = B1[ta * SI + tb * SJ + k];
      eo_bwdV<N, Q>(v, o);
      double* ye = y + dof0 + (ta * N + tb) * N;
#pragma unroll
      for (int c = 0; c < N; ++c) ye[c] = o[c];
    }
    fence_proxy_async();
    __syncthreads();
  }
}

}  // namespace sipg
