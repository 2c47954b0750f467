// Register-column hexahedron kernel (sm_100a, fp64): modified-modal basis on
// GLL points, affine elements.  One CTA of Q*Q threads per element; thread
// (j,k) owns the Q points (i, j, k) along axis 0 in registers, so the axis-0
// contractions of BwdTrans / PhysDeriv / PhysDeriv^T / IProduct are in-register
// and only the axis-1/2 contractions go through (bank-padded) shared memory.
// 1-D tables live in __constant__ memory per (N, Q) instantiation and are read
// as uniform operands of DFMA.
//
// Data movement: the element's and its six neighbours' coefficients are
// fetched with cp.async at kernel entry (the neighbour copies complete behind
// BwdTrans/PhysDeriv).  Faces flagged F_FAST_HEX (conforming same-class
// neighbour, identity grid, constant metric) and constant-metric boundary faces
// are evaluated together: the neighbour trace (u, du_normal) on the shared face
// grid from its coefficients (boundary-mode plane + normal-derivative plane, two
// sum-factorised 2-D passes), the flux at every face point, and the lift folded
// into the owning thread's register point arrays (no scatter, no atomics).  Any
// other coupling (shared trace, p2p, orientation transfers, pointwise metric)
// goes through generic_face() in dynamic shared memory (GEN instantiations).
#pragma once
#include "sipg_kernels.cuh"

namespace sipg {

template <int N, int Q> __constant__ double hxV[Q * N];     // psi_i(x_p), [p][i]
template <int N, int Q> __constant__ double hxD[Q * Q];     // collocation derivative
template <int N, int Q> __constant__ double hxW[Q];         // GLL weights
template <int N, int Q> __constant__ double hxDVE[2 * N];   // psi_i'(-1), psi_i'(+1)

// Even-odd (parity) factorisation of the 1-D operators.  On symmetric GLL points
// x_{Q-1-p} = -x_p the modified-modal modes satisfy psi_0(-x) = psi_{N-1}(x) and
// psi_c(-x) = (-1)^(c-1) psi_c(x) (bubbles), and the collocation derivative
// D[Q-1-p][Q-1-m] = -D[p][m]; every contraction splits into an even and an odd
// half of about a quarter of the size each (half the FMAs).  Tables (built and
// checked on the host by hex_fast_upload):
//   VE[p][a], p < H:  a = 0: (psi_0 + psi_{N-1})/2 (= 1/2), a >= 1: psi_{2a-1}
//   VO[p][b], p < QH: b = 0: (psi_0 - psi_{N-1})/2,        b >= 1: psi_{2b}
//   DP[p][m] = (D[p][m] + D[p][Q-1-m]) / 2, p < QH, m < H
//   DM[p][m] = (D[p][m] - D[p][Q-1-m]) / 2, p < H,  m < QH
template <int N, int Q> struct EO {
  static constexpr int H = (Q + 1) / 2, QH = Q / 2, NE = 1 + (N - 1) / 2, NO = 1 + (N - 2) / 2;
};
template <int N, int Q> __constant__ double eoVE[EO<N, Q>::H * EO<N, Q>::NE];
template <int N, int Q> __constant__ double eoVO[EO<N, Q>::QH * EO<N, Q>::NO];
template <int N, int Q> __constant__ double eoDP[EO<N, Q>::QH * EO<N, Q>::H];
template <int N, int Q> __constant__ double eoDM[EO<N, Q>::H * EO<N, Q>::QH];

// u[p] = sum_c V[p][c] v[c]
template <int N, int Q>
__device__ __forceinline__ void eo_fwdV(const double (&v)[N], double (&u)[Q]) {
  using E = EO<N, Q>;
  double ve[E::NE], vo[E::NO];
  ve[0] = v[0] + v[N - 1];
  vo[0] = v[0] - v[N - 1];
#pragma unroll
  for (int a = 1; a < E::NE; ++a) ve[a] = v[2 * a - 1];
#pragma unroll
  for (int b = 1; b < E::NO; ++b) vo[b] = v[2 * b];
#pragma unroll
  for (int p = 0; p < E::H; ++p) {
    double e = 0.0, o = 0.0;
#pragma unroll
    for (int a = 0; a < E::NE; ++a) e = fma(eoVE<N, Q>[p * E::NE + a], ve[a], e);
    if (p < E::QH) {
#pragma unroll
      for (int b = 0; b < E::NO; ++b) o = fma(eoVO<N, Q>[p * E::NO + b], vo[b], o);
      u[p] = e + o;
      u[Q - 1 - p] = e - o;
    } else {
      u[p] = e;   // middle point (odd Q)
    }
  }
}

// o[c] = sum_p V[p][c] u[p]
template <int N, int Q>
__device__ __forceinline__ void eo_bwdV(const double (&u)[Q], double (&o)[N]) {
  using E = EO<N, Q>;
  double sp[E::H], sm[E::QH];
#pragma unroll
  for (int p = 0; p < E::QH; ++p) {
    sp[p] = u[p] + u[Q - 1 - p];
    sm[p] = u[p] - u[Q - 1 - p];
  }
  if (Q & 1) sp[E::H - 1] = u[E::QH];
  double oe[E::NE], oo[E::NO];
#pragma unroll
  for (int a = 0; a < E::NE; ++a) {
    double acc = 0.0;
#pragma unroll
    for (int p = 0; p < E::H; ++p) acc = fma(eoVE<N, Q>[p * E::NE + a], sp[p], acc);
    oe[a] = acc;
  }
#pragma unroll
  for (int b = 0; b < E::NO; ++b) {
    double acc = 0.0;
#pragma unroll
    for (int p = 0; p < E::QH; ++p) acc = fma(eoVO<N, Q>[p * E::NO + b], sm[p], acc);
    oo[b] = acc;
  }
  o[0] = oe[0] + oo[0];
  o[N - 1] = oe[0] - oo[0];
#pragma unroll
  for (int a = 1; a < E::NE; ++a) o[2 * a - 1] = oe[a];
#pragma unroll
  for (int b = 1; b < E::NO; ++b) o[2 * b] = oo[b];
}

// d[p] = sum_m D[p][m] u[m]
template <int N, int Q>
__device__ __forceinline__ void eo_fwdD(const double (&u)[Q], double (&d)[Q]) {
  using E = EO<N, Q>;
  double sp[E::H], sm[E::QH];
#pragma unroll
  for (int m = 0; m < E::QH; ++m) {
    sp[m] = u[m] + u[Q - 1 - m];
    sm[m] = u[m] - u[Q - 1 - m];
  }
  if (Q & 1) sp[E::H - 1] = u[E::QH];
#pragma unroll
  for (int p = 0; p < E::H; ++p) {
    double o = 0.0;
#pragma unroll
    for (int m = 0; m < E::QH; ++m) o = fma(eoDM<N, Q>[p * E::QH + m], sm[m], o);
    if (p < E::QH) {
      double e = 0.0;
#pragma unroll
      for (int m = 0; m < E::H; ++m) e = fma(eoDP<N, Q>[p * E::H + m], sp[m], e);
      d[p] = e + o;
      d[Q - 1 - p] = o - e;
    } else {
      d[p] = o;
    }
  }
}

// r[m] = sum_p D[p][m] g[p]
template <int N, int Q>
__device__ __forceinline__ void eo_trD(const double (&g)[Q], double (&r)[Q]) {
  using E = EO<N, Q>;
  double gp[E::H], gm[E::QH];
#pragma unroll
  for (int p = 0; p < E::QH; ++p) {
    gp[p] = g[p] + g[Q - 1 - p];
    gm[p] = g[p] - g[Q - 1 - p];
  }
  if (Q & 1) gp[E::H - 1] = g[E::QH];
#pragma unroll
  for (int m = 0; m < E::H; ++m) {
    double yv = 0.0;
#pragma unroll
    for (int p = 0; p < E::QH; ++p) yv = fma(eoDP<N, Q>[p * E::H + m], gm[p], yv);
    if (m < E::QH) {
      double xv = 0.0;
#pragma unroll
      for (int p = 0; p < E::H; ++p) xv = fma(eoDM<N, Q>[p * E::QH + m], gp[p], xv);
      r[m] = xv + yv;
      r[Q - 1 - m] = yv - xv;
    } else {
      r[m] = yv;
    }
  }
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int PENDING>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(PENDING) : "memory"); }

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  unsigned long long state;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
               : "=l"(state) : "r"(smem_u32(bar)), "r"(bytes) : "memory");
  (void)state;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// TMA 1-D bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Copy n doubles at 8-byte-aligned global src into a shared region laid out so
// that the 16-byte-aligned body can go through one TMA bulk copy; the (at most
// one) unaligned head and tail doubles are plain loads.  Returns the offset of
// element 0 inside `region` (region must be 16-byte aligned, n + 2 doubles).
// Returns the bulk byte count through *bytes (to be expected on `bar`).
__device__ __forceinline__ int bulk_block(double* region, const double* src, int n, uint64_t* bar,
                                          unsigned* bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src);
  const int o = (a & 15) ? 1 : 0;
  const uintptr_t b0 = (a + 15) & ~uintptr_t(15);
  const uintptr_t e = a + 8 * (uintptr_t)n;
  const uintptr_t b1 = e & ~uintptr_t(15);
  // unaligned head / tail doubles: 8-byte cp.async (asynchronous; the issuing
  // thread completes them with cp_async_wait<0>() before the consumers' barrier)
  if (o) cp_async8(region + o, src);
  if (e != b1) cp_async8(region + o + n - 1, src + n - 1);
  const unsigned nb = b1 > b0 ? (unsigned)(b1 - b0) : 0u;
  if (nb) bulk_g2s(region + o + (int)((b0 - a) >> 3), reinterpret_cast<const void*>(b0), nb, bar);
  *bytes = nb;
  return o;
}

template <int N, int Q>
struct HexFast {
  static constexpr int NT = Q * Q;
  static constexpr int SJ = (Q & 1) ? Q : Q + 1;   // odd row stride: conflict-free strided lines
  static constexpr int SI = Q * SJ;
  static constexpr int BUF = Q * SI;
  static constexpr int N3 = N * N * N;
  static constexpr int BLK = (N3 + 2 + 1) & ~1;    // one coefficient block (+ alignment slack), even
  // neighbour region: 6 coefficient blocks; later stage-1 output + face flux buffers
  static constexpr int NBR = 6 * BLK > 12 * Q * N + 16 * Q * Q ? 6 * BLK : 12 * Q * N + 16 * Q * Q;
  // scratch: 2 padded Q^3 buffers; later the neighbour planes (12 N^2), then (overlaid) the
  // stage-2 traces (12 Q^2).  Kept small so that 7 CTAs fit per SM (Q = 8: 30 KB per CTA).
  static constexpr int SF = 12 * N * N > 12 * Q * Q ? 12 * N * N : 12 * Q * Q;
  static constexpr int SCR0 = 2 * BUF > SF ? 2 * BUF : SF;
  static constexpr int SCR = (SCR0 + 1) & ~1;
  // generic-face scratch (dynamic smem): us (4 FP), fscr, fb (6*4*Q*Q)
  static constexpr int FP = QMAX * QMAX;
  static constexpr int GFB = 4 * FP + 16 * FP + 4 * QMAX * QMAX + 2 * NMAX * NMAX + 3 * QMAX * NMAX;
  static constexpr int GSZ = GFB + 6 * 4 * Q * Q;
  // dynamic shared memory (doubles, 16-byte aligned regions):
  //   REC[2] (6 records = 96 doubles each) | CO own coefficients | NB | S | generic scratch
  // (the next element's coefficients land in CO as soon as BwdTrans has consumed the current ones)
  static constexpr int O_REC = 0;
  static constexpr int O_CO = 2 * 96;
  static constexpr int O_NB = O_CO + BLK;
  static constexpr int O_S = O_NB + NBR;
  static constexpr int O_G = O_S + SCR;
  static size_t smem_bytes(bool gen) { return sizeof(double) * (size_t)(O_G + (gen ? GSZ : 0)); }
};

__device__ __forceinline__ int hex_stride(int axis, int n) { return axis == 0 ? n * n : (axis == 1 ? n : 1); }

// Persistent: CTA b processes elements b, b + gridDim.x, ... of the class.  The
// next element's face records and coefficients stream in (TMA bulk copies on an
// mbarrier) while the current one computes; the neighbours' coefficients
// stream in behind BwdTrans / PhysDeriv.
// 6 resident CTAs per SM for Q <= 8 (caps registers at 168: measured 498 us vs
// 545 us unconstrained and 525 us with 8 CTAs / 128 registers, cfg3a)
#ifndef SIPG_HEX_MINB
#define SIPG_HEX_MINB 7
#endif
template <int N, int Q, bool GEN>
__global__ void __launch_bounds__(Q * Q, (Q <= 8 ? SIPG_HEX_MINB : 1))
k_hex(const DevPlan P, const int cls, const double* __restrict__ x, double* __restrict__ y) {
  using H = HexFast<N, Q>;
  constexpr int NT = H::NT, SJ = H::SJ, SI = H::SI, BUF = H::BUF, N3 = H::N3, QQ = Q * Q;
  extern __shared__ __align__(16) double dsm[];
  double* NB = dsm + H::O_NB;
  double* S = dsm + H::O_S;
  double* gsm = dsm + H::O_G;
  __shared__ double sW[Q];
  __shared__ int sk[6];               // 1 fast conforming, 2 boundary, 0 generic
  __shared__ int soff[8];
  __shared__ int64_t sdof[2];
  __shared__ int fpar[6][4];          // neighbour plane strides (b0, b1, fixed axis), side             // block offsets (own coefficients per stage, neighbours)
  __shared__ __align__(8) uint64_t mbar[3];   // records+own [stage 0, 1], neighbours
  double* B0 = S;
  double* B1 = S + BUF;
  const int t = threadIdx.x;
  const int ta = t / Q, tb = t - (t / Q) * Q;
  const int* cd = P.cd + cls * CD_WORDS;
  const int count = cd[CD_COUNT];
  const int* elist = P.class_elems + cd[CD_ELEM_OFF];
  const double lam = P.lam;
  if (t == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&mbar[2], 6);
    fence_proxy_async();
  }
  if (t < Q) sW[t] = hxW<N, Q>[t];
  __syncthreads();
  // issue records + own coefficients of element `iel` into stage `st`
  // (thread 0) dof offsets are loaded one issue ahead so the TMA issue never waits on the
  // elist -> dof_off load chain
  auto issue_own = [&](int iel, int st, int64_t dof) {
    const FaceRec* rsrc = P.recs + cd[CD_REC_OFF] + (int64_t)iel * 6;
    bulk_g2s(dsm + H::O_REC + st * 96, rsrc, 6 * sizeof(FaceRec), &mbar[st]);
    unsigned nb;
    sdof[st] = dof;
    soff[st] = bulk_block(dsm + H::O_CO, x + dof, N3, &mbar[st], &nb);
    mbar_expect_tx(&mbar[st], 6 * sizeof(FaceRec) + nb);
    cp_async_commit();
  };
  int64_t dnext = 0;
  if (t == 0 && blockIdx.x < count) {
    issue_own(blockIdx.x, 0, P.dof_off[elist[blockIdx.x]]);
    if (blockIdx.x + gridDim.x < count) dnext = P.dof_off[elist[blockIdx.x + gridDim.x]];
  }

  int k = 0;
  for (int iel = blockIdx.x; iel < count; iel += gridDim.x, ++k) {
  const int st = k & 1;
  const bool more = iel + (int)gridDim.x < count;
  if (t == 0) cp_async_wait<0>();
  mbar_wait(&mbar[st], (k >> 1) & 1);
  __syncthreads();
  const FaceRec* srec = reinterpret_cast<const FaceRec*>(dsm + H::O_REC + st * 96);
  const double* C = dsm + H::O_CO + soff[st];
  const int64_t dof0 = sdof[st];
  if (t < 6) {
    const int fl = srec[t].flags, ty = srec[t].type;
    sk[t] = (ty == FT_DIRECT && (fl & F_FAST_HEX)) ? 1 : ((ty == FT_BOUNDARY && !(fl & F_SELF_PW)) ? 2 : 0);
#ifdef SIPG_INSTRUMENT
    if (!GEN && (P.debug & 2)) sk[t] = 0;   // instrumentation build only (SIPG_DEBUG=2): no face work
#endif
  }
  if (t >= NT - 6) {      // neighbour blocks, one per thread: the last 6 threads (NT >= 9),
                          // never thread 0 (which issues the next-element prefetch)
    const int f = t - (NT - 6);
    unsigned nb = 0;
    const FaceRec& rf = srec[f];
    if (rf.type == FT_DIRECT && (rf.flags & F_FAST_HEX)) {
      soff[2 + f] = bulk_block(NB + f * H::BLK, x + rf.nbr_dof, N3, &mbar[2], &nb);
      const int ao = rf.nbr_face >> 1;
      fpar[f][0] = hex_stride(ao == 0 ? 1 : 0, N);
      fpar[f][1] = hex_stride(ao == 2 ? 1 : 2, N);
      fpar[f][2] = hex_stride(ao, N);
      fpar[f][3] = rf.nbr_face & 1;
    }
    mbar_expect_tx(&mbar[2], nb);
    cp_async_commit();
  }

  // ---- BwdTrans: axis 2 (thread (a,b)), axis 1 (thread (a,k)), axis 0 (thread (j,k))
  if (ta < N && tb < N) {
    double v[N], o[Q];
#pragma unroll
    for (int c = 0; c < N; ++c) v[c] = C[(ta * N + tb) * N + c];
    eo_fwdV<N, Q>(v, o);
#pragma unroll
    for (int k = 0; k < Q; ++k) B1[ta * SI + tb * SJ + k] = o[k];
  }
  fence_proxy_async();   // the reads of CO above before the next element's TMA writes into it
  __syncthreads();
  if (t == 0 && more) {
    issue_own(iel + gridDim.x, st ^ 1, dnext);
    if (iel + 2 * (int)gridDim.x < count) dnext = P.dof_off[elist[iel + 2 * gridDim.x]];
  }
  if (ta < N) {
    double v[N], o[Q];
#pragma unroll
    for (int b = 0; b < N; ++b) v[b] = B1[ta * SI + b * SJ + tb];
    eo_fwdV<N, Q>(v, o);
#pragma unroll
    for (int j = 0; j < Q; ++j) B0[ta * SI + j * SJ + tb] = o[j];
  }
  __syncthreads();
  double u[Q], d0[Q], d1[Q], d2[Q];
  {
    double v[N];
#pragma unroll
    for (int a = 0; a < N; ++a) v[a] = B0[a * SI + ta * SJ + tb];
    eo_fwdV<N, Q>(v, u);
  }
  // ---- PhysDeriv: axis 0 in registers; axes 1, 2 through shared memory
#pragma unroll
  for (int i = 0; i < Q; ++i) B0[i * SI + ta * SJ + tb] = u[i];
  eo_fwdD<N, Q>(u, d0);
  __syncthreads();
  {
    double v[Q], w[Q];
#pragma unroll
    for (int m = 0; m < Q; ++m) {
      v[m] = B0[ta * SI + m * SJ + tb];     // line along axis 1: thread (i=ta, k=tb)
      w[m] = B0[ta * SI + tb * SJ + m];     // line along axis 2: thread (i=ta, j=tb)
    }
    eo_fwdD<N, Q>(v, d1);
    eo_fwdD<N, Q>(w, d2);
#pragma unroll
    for (int r = 0; r < Q; ++r) B1[ta * SI + r * SJ + tb] = d1[r];
    __syncthreads();   // every line of B0 read
#pragma unroll
    for (int r = 0; r < Q; ++r) B0[ta * SI + tb * SJ + r] = d2[r];
  }
  if (t >= NT - 6) cp_async_wait<0>();
  mbar_wait(&mbar[2], k & 1);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    d1[i] = B1[i * SI + ta * SJ + tb];
    d2[i] = B0[i * SI + ta * SJ + tb];
  }
  __syncthreads();   // S reused from here on

  // ---- fast faces: neighbour (u, du_normal) on the face grid from its coefficients
  double* NP = S;                      // [f][pl][i0][i1], 12 N^2
  double* U2 = S;                      // [f][pl][p0][p1], 12 Q^2 (overlays NP once stage 1 is done)
  double* T1 = NB;                     // [f][pl][p0][i1], 12 Q N (neighbour blocks dead by then)
  double* OWN = NB + 12 * Q * N;       // faces 2..5: own (u, g_s) [f-2][2][QQ]
  double* FVD = OWN + 8 * QQ;          // faces 2..5: (fv, fd) [f-2][2][QQ]
  if (t < N * N) {
    const int i0 = t / N, i1 = t - (t / N) * N;
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      if (sk[f] != 1) continue;
      const double* c = NB + f * H::BLK + soff[2 + f] + i0 * fpar[f][0] + i1 * fpar[f][1];
      const int sa = fpar[f][2], hi = fpar[f][3];
      double pd = 0.0;
      if (hi) {   // face-uniform branch: both endpoint rows stay compile-time constant operands
#pragma unroll
        for (int i = 0; i < N; ++i) pd = fma(hxDVE<N, Q>[N + i], c[i * sa], pd);
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i) pd = fma(hxDVE<N, Q>[i], c[i * sa], pd);
      }
      NP[(2 * f) * N * N + t] = c[hi ? (N - 1) * sa : 0];   // modified-modal boundary mode
      NP[(2 * f + 1) * N * N + t] = pd;
    }
  }
  __syncthreads();
  for (int it = t; it < 12 * N; it += NT) {      // stage 1: contract i0 -> p0 (line over i0 at fixed i1)
    const int fp = it / N, i1 = it - (it / N) * N;
    if (sk[fp >> 1] != 1) continue;
    double v[N], o[Q];
#pragma unroll
    for (int i0 = 0; i0 < N; ++i0) v[i0] = NP[fp * N * N + i0 * N + i1];
    eo_fwdV<N, Q>(v, o);
#pragma unroll
    for (int p0 = 0; p0 < Q; ++p0) T1[fp * Q * N + p0 * N + i1] = o[p0];
  }
  __syncthreads();
  for (int it = t; it < 12 * Q; it += NT) {      // stage 2: contract i1 -> p1
    const int fp = it / Q, p0 = it - (it / Q) * Q;
    if (sk[fp >> 1] != 1) continue;
    double v[N], o[Q];
#pragma unroll
    for (int i1 = 0; i1 < N; ++i1) v[i1] = T1[fp * Q * N + p0 * N + i1];
    eo_fwdV<N, Q>(v, o);
#pragma unroll
    for (int p1 = 0; p1 < Q; ++p1) U2[fp * QQ + p0 * Q + p1] = o[p1];
  }
  // ---- generic faces (dynamic shared memory; GEN instantiations only)
  double* gfb = gsm + H::GFB;
  if (GEN) {
    __syncthreads();
    for (int f = 0; f < 6; ++f) {
      if (sk[f] != 0) continue;
      const int a = f >> 1, hi = f & 1;
      double* us = gsm;
      if (a == 0) {
        const int i = hi ? Q - 1 : 0;
        const int p = ta * Q + tb;
        us[p] = u[i]; us[H::FP + p] = d0[i]; us[2 * H::FP + p] = d1[i]; us[3 * H::FP + p] = d2[i];
      } else if ((a == 1 && ta == (hi ? Q - 1 : 0)) || (a == 2 && tb == (hi ? Q - 1 : 0))) {
        const int q1 = a == 1 ? tb : ta;
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          const int p = i * Q + q1;
          us[p] = u[i]; us[H::FP + p] = d0[i]; us[2 * H::FP + p] = d1[i]; us[3 * H::FP + p] = d2[i];
        }
      }
      __syncthreads();
      generic_face<SHAPE_HEX, N, Q>(P, srec[f], f, x, us, gfb + f * 4 * QQ, gsm + 4 * H::FP, t, NT);
      __syncthreads();
    }
  }
  // ---- faces 2..5: owners publish own (u, g_s); the flux is computed cooperatively
#pragma unroll
  for (int f = 2; f < 6; ++f) {
    const int a = f >> 1, hi = f & 1;
    const bool own = a == 1 ? (ta == (hi ? Q - 1 : 0)) : (tb == (hi ? Q - 1 : 0));
    if (sk[f] == 0 || !own) continue;
    const double g0 = srec[f].gs[0], g1 = srec[f].gs[1], g2 = srec[f].gs[2];
    const int q1 = a == 1 ? tb : ta;
    double* o = OWN + (f - 2) * 2 * QQ;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      o[i * Q + q1] = u[i];
      o[QQ + i * Q + q1] = g0 * d0[i] + g1 * d1[i] + g2 * d2[i];
    }
  }
  __syncthreads();
  for (int it = t; it < 4 * QQ; it += NT) {
    const int f = 2 + it / QQ, p = it - (it / QQ) * QQ;
    const int kind = sk[f];
    if (kind == 0) continue;
    const FaceRec& r = srec[f];
    const int p0 = p / Q, p1 = p - (p / Q) * Q;
    const double* o = OWN + (f - 2) * 2 * QQ;
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
    FVD[(f - 2) * 2 * QQ + p] = (r.tau * jump - avg) * swj;
    FVD[(f - 2) * 2 * QQ + QQ + p] = -0.5 * jump * swj;
  }
  // ---- faces 0/1 (points i = 0 and i = Q-1 of every thread): flux in registers
  double fv01[2], fd01[2];
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    const int i = f ? Q - 1 : 0;
    const int kind = sk[f];
    fv01[f] = 0.0;
    fd01[f] = 0.0;
    if (kind == 0) continue;
    const FaceRec& r = srec[f];
    const int p = ta * Q + tb;
    const double swj = r.sJ * sW[ta] * sW[tb];
    const double gs = r.gs[0] * d0[i] + r.gs[1] * d1[i] + r.gs[2] * d2[i];
    double jump, avg;
    if (kind == 2) {
      jump = 2.0 * u[i];
      avg = gs;
    } else {
      jump = u[i] - U2[(2 * f) * QQ + p];
      avg = 0.5 * (gs - r.go[r.nbr_face >> 1] * U2[(2 * f + 1) * QQ + p]);
    }
    fv01[f] = (r.tau * jump - avg) * swj;
    fd01[f] = -0.5 * jump * swj;
  }
  __syncthreads();

  // ---- volume metric + lift of the face fluxes, per owned point
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
  // lift: faces 0/1 at i = 0 / Q-1 of every column (registers), faces 2..5 on the edge columns
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    const int i = f ? Q - 1 : 0;
    if (sk[f] == 0) {
      if (GEN) {
        const double* fbf = gfb + f * 4 * QQ;
        const int p = ta * Q + tb;
        u[i] += fbf[p]; d0[i] += fbf[QQ + p]; d1[i] += fbf[2 * QQ + p]; d2[i] += fbf[3 * QQ + p];
      }
      continue;
    }
    const double fv = fv01[f], fd = fd01[f];
    u[i] += fv;
    d0[i] = fma(fd, srec[f].gs[0], d0[i]);
    d1[i] = fma(fd, srec[f].gs[1], d1[i]);
    d2[i] = fma(fd, srec[f].gs[2], d2[i]);
  }
#pragma unroll
  for (int f = 2; f < 6; ++f) {
    const int a = f >> 1, hi = f & 1;
    const bool own = a == 1 ? (ta == (hi ? Q - 1 : 0)) : (tb == (hi ? Q - 1 : 0));
    if (!own) continue;
    const int q1 = a == 1 ? tb : ta;
    if (sk[f] == 0) {
      if (GEN) {
        const double* fbf = gfb + f * 4 * QQ;
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          const int p = i * Q + q1;
          u[i] += fbf[p]; d0[i] += fbf[QQ + p]; d1[i] += fbf[2 * QQ + p]; d2[i] += fbf[3 * QQ + p];
        }
      }
      continue;
    }
    const double gsa = srec[f].gs[0], gsb = srec[f].gs[1], gsc = srec[f].gs[2];
    const double* fvd = FVD + (f - 2) * 2 * QQ;
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      const double fv = fvd[i * Q + q1], fd = fvd[QQ + i * Q + q1];
      u[i] += fv;
      d0[i] = fma(fd, gsa, d0[i]);
      d1[i] = fma(fd, gsb, d1[i]);
      d2[i] = fma(fd, gsc, d2[i]);
    }
  }

  // ---- R = P0 + D0^T P1 (registers) + D1^T P2 + D2^T P3 (shared memory)
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    B0[i * SI + ta * SJ + tb] = d1[i];
    B1[i * SI + ta * SJ + tb] = d2[i];
  }
  {
    double r[Q];
    eo_trD<N, Q>(d0, r);
#pragma unroll
    for (int i = 0; i < Q; ++i) u[i] += r[i];
  }
  __syncthreads();
  {
    double v[Q], w[Q];
#pragma unroll
    for (int m = 0; m < Q; ++m) {
      v[m] = B0[ta * SI + m * SJ + tb];   // (i=ta, ., k=tb)
      w[m] = B1[ta * SI + tb * SJ + m];   // (i=ta, j=tb, .)
    }
    eo_trD<N, Q>(v, d1);
    eo_trD<N, Q>(w, d2);
#pragma unroll
    for (int r = 0; r < Q; ++r) {
      B0[ta * SI + r * SJ + tb] = d1[r];
      B1[ta * SI + tb * SJ + r] = d2[r];
    }
  }
  __syncthreads();
  // ---- IProduct: axis 0 in registers (thread (j,k)), then axes 1 and 2
#pragma unroll
  for (int i = 0; i < Q; ++i) u[i] += B0[i * SI + ta * SJ + tb] + B1[i * SI + ta * SJ + tb];
  {
    double o[N];
    eo_bwdV<N, Q>(u, o);
#pragma unroll
    for (int a = 0; a < N; ++a) B0[a * SI + ta * SJ + tb] = o[a];
  }
  __syncthreads();
  if (ta < N) {                                     // thread (a, k): contract j -> b
    double v[Q], o[N];
#pragma unroll
    for (int j = 0; j < Q; ++j) v[j] = B0[ta * SI + j * SJ + tb];
    eo_bwdV<N, Q>(v, o);
#pragma unroll
    for (int b = 0; b < N; ++b) B1[ta * SI + b * SJ + tb] = o[b];
  }
  __syncthreads();
  if (ta < N && tb < N) {                           // thread (a, b): contract k -> c, write y
    double v[Q], o[N];
#pragma unroll
    for (int k = 0; k < Q; ++k) v[k] = B1[ta * SI + tb * SJ + k];
    eo_bwdV<N, Q>(v, o);
    double* ye = y + dof0 + (ta * N + tb) * N;
#pragma unroll
    for (int c = 0; c < N; ++c) ye[c] = o[c];
  }
  fence_proxy_async();   // generic accesses of this element before the next TMA writes
  __syncthreads();
  }  // element loop
}

// Upload the constant tables of one (N, Q) instantiation (from the plan's pool).
// The even-odd tables are derived here and checked by reassembling V and D from
// them (the parity symmetry holds for modified-modal modes on GLL points).
template <int N, int Q>
cudaError_t hex_fast_upload(const double* V, const double* D, const double* W, const double* dVend) {
  using E = EO<N, Q>;
  double ve[E::H * E::NE], vo[E::QH * E::NO], dp[E::QH * E::H], dm[E::H * E::QH];
  for (int p = 0; p < E::H; ++p) {
    ve[p * E::NE] = 0.5 * (V[p * N] + V[p * N + N - 1]);
    for (int a = 1; a < E::NE; ++a) ve[p * E::NE + a] = V[p * N + 2 * a - 1];
  }
  for (int p = 0; p < E::QH; ++p) {
    vo[p * E::NO] = 0.5 * (V[p * N] - V[p * N + N - 1]);
    for (int b = 1; b < E::NO; ++b) vo[p * E::NO + b] = V[p * N + 2 * b];
  }
  for (int p = 0; p < E::QH; ++p)
    for (int m = 0; m < E::H; ++m) dp[p * E::H + m] = 0.5 * (D[p * Q + m] + D[p * Q + Q - 1 - m]);
  for (int p = 0; p < E::H; ++p)
    for (int m = 0; m < E::QH; ++m) dm[p * E::QH + m] = 0.5 * (D[p * Q + m] - D[p * Q + Q - 1 - m]);
  // check: apply the even-odd forms (same formulas as eo_fwdV / eo_fwdD / eo_bwdV / eo_trD)
  // to unit vectors and compare with V, D, V^T, D^T
  double vmax = 0.0, dmax = 0.0, verr = 0.0, derr = 0.0;
  for (int c = 0; c < N; ++c) {             // column c of V; row c of V^T
    double v[N] = {}, u[Q];
    v[c] = 1.0;
    double vev[E::NE], vov[E::NO];
    vev[0] = v[0] + v[N - 1];
    vov[0] = v[0] - v[N - 1];
    for (int a = 1; a < E::NE; ++a) vev[a] = v[2 * a - 1];
    for (int b = 1; b < E::NO; ++b) vov[b] = v[2 * b];
    for (int p = 0; p < E::H; ++p) {
      double ev = 0.0, ov = 0.0;
      for (int a = 0; a < E::NE; ++a) ev += ve[p * E::NE + a] * vev[a];
      if (p < E::QH) {
        for (int b = 0; b < E::NO; ++b) ov += vo[p * E::NO + b] * vov[b];
        u[p] = ev + ov;
        u[Q - 1 - p] = ev - ov;
      } else {
        u[p] = ev;
      }
    }
    for (int p = 0; p < Q; ++p) {
      vmax = fmax(vmax, fabs(V[p * N + c]));
      verr = fmax(verr, fabs(u[p] - V[p * N + c]));
    }
  }
  for (int m = 0; m < Q; ++m) {             // column m of D
    double u[Q] = {}, d[Q], sp[E::H], sm[E::QH > 0 ? E::QH : 1];
    u[m] = 1.0;
    for (int k = 0; k < E::QH; ++k) {
      sp[k] = u[k] + u[Q - 1 - k];
      sm[k] = u[k] - u[Q - 1 - k];
    }
    if (Q & 1) sp[E::H - 1] = u[E::QH];
    for (int p = 0; p < E::H; ++p) {
      double ov = 0.0;
      for (int k = 0; k < E::QH; ++k) ov += dm[p * E::QH + k] * sm[k];
      if (p < E::QH) {
        double ev = 0.0;
        for (int k = 0; k < E::H; ++k) ev += dp[p * E::H + k] * sp[k];
        d[p] = ev + ov;
        d[Q - 1 - p] = ov - ev;
      } else {
        d[p] = ov;
      }
    }
    for (int p = 0; p < Q; ++p) {
      dmax = fmax(dmax, fabs(D[p * Q + m]));
      derr = fmax(derr, fabs(d[p] - D[p * Q + m]));
    }
  }
  if (verr > 1e-13 * (vmax > 1.0 ? vmax : 1.0) || derr > 1e-12 * (dmax > 1.0 ? dmax : 1.0))
    return cudaErrorInvalidValue;   // tables lack the parity symmetry: not a GLL / modified-modal class
  cudaError_t e;
  if ((e = cudaMemcpyToSymbol(eoVE<N, Q>, ve, sizeof(ve))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(eoVO<N, Q>, vo, sizeof(vo))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(eoDP<N, Q>, dp, sizeof(dp))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(eoDM<N, Q>, dm, sizeof(dm))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(hxV<N, Q>, V, sizeof(double) * Q * N)) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(hxD<N, Q>, D, sizeof(double) * Q * Q)) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(hxW<N, Q>, W, sizeof(double) * Q)) != cudaSuccess) return e;
  return cudaMemcpyToSymbol(hxDVE<N, Q>, dVend, sizeof(double) * 2 * N);
}

}  // namespace sipg
