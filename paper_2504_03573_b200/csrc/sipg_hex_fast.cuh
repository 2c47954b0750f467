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
  // scratch: 3 padded Q^3 buffers; later planes (12 N^2) + stage-2 output (12 Q^2)
  static constexpr int SCR0 = 3 * BUF > 12 * N * N + 12 * Q * Q ? 3 * BUF : 12 * N * N + 12 * Q * Q;
  static constexpr int SCR = (SCR0 + 1) & ~1;
  // generic-face scratch (dynamic smem): us (4 FP), fscr, fb (6*4*Q*Q)
  static constexpr int FP = QMAX * QMAX;
  static constexpr int GFB = 4 * FP + 16 * FP + 4 * QMAX * QMAX + 2 * NMAX * NMAX + 3 * QMAX * NMAX;
  static constexpr int GSZ = GFB + 6 * 4 * Q * Q;
  // dynamic shared memory (doubles, 16-byte aligned regions):
  //   REC[2] (6 records = 96 doubles each) | CO[2] own coefficients | NB | S | generic scratch
  static constexpr int O_REC = 0;
  static constexpr int O_CO = 2 * 96;
  static constexpr int O_NB = O_CO + 2 * BLK;
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
#define SIPG_HEX_MINB 6
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
  __shared__ int fpar[6][4];          // neighbour plane strides (b0, b1, fixed axis), side             // block offsets (own coefficients per stage, neighbours)
  __shared__ __align__(8) uint64_t mbar[3];   // records+own [stage 0, 1], neighbours
  double* B0 = S;
  double* B1 = S + BUF;
  double* B2 = S + 2 * BUF;
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
  auto issue_own = [&](int iel, int st) {
    const FaceRec* rsrc = P.recs + cd[CD_REC_OFF] + (int64_t)iel * 6;
    bulk_g2s(dsm + H::O_REC + st * 96, rsrc, 6 * sizeof(FaceRec), &mbar[st]);
    unsigned nb;
    soff[st] = bulk_block(dsm + H::O_CO + st * H::BLK, x + P.dof_off[elist[iel]], N3, &mbar[st], &nb);
    mbar_expect_tx(&mbar[st], 6 * sizeof(FaceRec) + nb);
    cp_async_commit();
  };
  if (t == 0 && blockIdx.x < count) issue_own(blockIdx.x, 0);

  int k = 0;
  for (int iel = blockIdx.x; iel < count; iel += gridDim.x, ++k) {
  const int st = k & 1;
  const bool more = iel + (int)gridDim.x < count;
  if (t == 0 && more) issue_own(iel + gridDim.x, st ^ 1);
  if (t == 0) {
    if (more) cp_async_wait<1>(); else cp_async_wait<0>();
  }
  mbar_wait(&mbar[st], (k >> 1) & 1);
  __syncthreads();
  const FaceRec* srec = reinterpret_cast<const FaceRec*>(dsm + H::O_REC + st * 96);
  const double* C = dsm + H::O_CO + st * H::BLK + soff[st];
  const int e = elist[iel];
  const int64_t dof0 = P.dof_off[e];
  if (t < 6) {
    const int fl = srec[t].flags, ty = srec[t].type;
    sk[t] = (ty == FT_DIRECT && (fl & F_FAST_HEX)) ? 1 : ((ty == FT_BOUNDARY && !(fl & F_SELF_PW)) ? 2 : 0);
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
#pragma unroll
    for (int k = 0; k < Q; ++k) o[k] = 0.0;
#pragma unroll
    for (int c = 0; c < N; ++c)
#pragma unroll
      for (int k = 0; k < Q; ++k) o[k] = fma(hxV<N, Q>[k * N + c], v[c], o[k]);
#pragma unroll
    for (int k = 0; k < Q; ++k) B1[ta * SI + tb * SJ + k] = o[k];
  }
  __syncthreads();
  if (ta < N) {
    double v[N], o[Q];
#pragma unroll
    for (int b = 0; b < N; ++b) v[b] = B1[ta * SI + b * SJ + tb];
#pragma unroll
    for (int j = 0; j < Q; ++j) o[j] = 0.0;
#pragma unroll
    for (int b = 0; b < N; ++b)
#pragma unroll
      for (int j = 0; j < Q; ++j) o[j] = fma(hxV<N, Q>[j * N + b], v[b], o[j]);
#pragma unroll
    for (int j = 0; j < Q; ++j) B2[ta * SI + j * SJ + tb] = o[j];
  }
  __syncthreads();
  double u[Q], d0[Q], d1[Q], d2[Q];
  {
    double v[N];
#pragma unroll
    for (int a = 0; a < N; ++a) v[a] = B2[a * SI + ta * SJ + tb];
#pragma unroll
    for (int i = 0; i < Q; ++i) u[i] = 0.0;
#pragma unroll
    for (int a = 0; a < N; ++a)
#pragma unroll
      for (int i = 0; i < Q; ++i) u[i] = fma(hxV<N, Q>[i * N + a], v[a], u[i]);
  }
  // ---- PhysDeriv: axis 0 in registers; axes 1, 2 through shared memory
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    d0[i] = 0.0;
    B0[i * SI + ta * SJ + tb] = u[i];
  }
#pragma unroll
  for (int m = 0; m < Q; ++m)
#pragma unroll
    for (int i = 0; i < Q; ++i) d0[i] = fma(hxD<N, Q>[i * Q + m], u[m], d0[i]);
  __syncthreads();
  {
    double v[Q], w[Q];
#pragma unroll
    for (int m = 0; m < Q; ++m) {
      v[m] = B0[ta * SI + m * SJ + tb];     // line along axis 1: thread (i=ta, k=tb)
      w[m] = B0[ta * SI + tb * SJ + m];     // line along axis 2: thread (i=ta, j=tb)
    }
#pragma unroll
    for (int r = 0; r < Q; ++r) {
      d1[r] = 0.0;
      d2[r] = 0.0;
    }
#pragma unroll
    for (int m = 0; m < Q; ++m)
#pragma unroll
      for (int r = 0; r < Q; ++r) {
        d1[r] = fma(hxD<N, Q>[r * Q + m], v[m], d1[r]);
        d2[r] = fma(hxD<N, Q>[r * Q + m], w[m], d2[r]);
      }
#pragma unroll
    for (int r = 0; r < Q; ++r) {
      B1[ta * SI + r * SJ + tb] = d1[r];
      B2[ta * SI + tb * SJ + r] = d2[r];
    }
  }
  if (t >= NT - 6) cp_async_wait<0>();
  mbar_wait(&mbar[2], k & 1);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    d1[i] = B1[i * SI + ta * SJ + tb];
    d2[i] = B2[i * SI + ta * SJ + tb];
  }
  __syncthreads();   // S reused from here on

  // ---- fast faces: neighbour (u, du_normal) on the face grid from its coefficients
  double* NP = S;                      // [f][pl][i0][i1], 12 N^2
  double* U2 = S + 12 * N * N;         // [f][pl][p0][p1], 12 Q^2
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
      const double* dve = &hxDVE<N, Q>[hi * N];
      double pd = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) pd = fma(dve[i], c[i * sa], pd);
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
#pragma unroll
    for (int p0 = 0; p0 < Q; ++p0) o[p0] = 0.0;
#pragma unroll
    for (int i0 = 0; i0 < N; ++i0)
#pragma unroll
      for (int p0 = 0; p0 < Q; ++p0) o[p0] = fma(hxV<N, Q>[p0 * N + i0], v[i0], o[p0]);
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
#pragma unroll
    for (int p1 = 0; p1 < Q; ++p1) o[p1] = 0.0;
#pragma unroll
    for (int i1 = 0; i1 < N; ++i1)
#pragma unroll
      for (int p1 = 0; p1 < Q; ++p1) o[p1] = fma(hxV<N, Q>[p1 * N + i1], v[i1], o[p1]);
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
    B1[i * SI + ta * SJ + tb] = d1[i];
    B2[i * SI + ta * SJ + tb] = d2[i];
  }
#pragma unroll
  for (int m = 0; m < Q; ++m)
#pragma unroll
    for (int i = 0; i < Q; ++i) u[i] = fma(hxD<N, Q>[m * Q + i], d0[m], u[i]);
  __syncthreads();
  {
    double v[Q], w[Q];
#pragma unroll
    for (int m = 0; m < Q; ++m) {
      v[m] = B1[ta * SI + m * SJ + tb];   // (i=ta, ., k=tb)
      w[m] = B2[ta * SI + tb * SJ + m];   // (i=ta, j=tb, .)
    }
#pragma unroll
    for (int r = 0; r < Q; ++r) {
      d1[r] = 0.0;
      d2[r] = 0.0;
    }
#pragma unroll
    for (int m = 0; m < Q; ++m)
#pragma unroll
      for (int r = 0; r < Q; ++r) {
        d1[r] = fma(hxD<N, Q>[m * Q + r], v[m], d1[r]);
        d2[r] = fma(hxD<N, Q>[m * Q + r], w[m], d2[r]);
      }
#pragma unroll
    for (int r = 0; r < Q; ++r) {
      B1[ta * SI + r * SJ + tb] = d1[r];
      B2[ta * SI + tb * SJ + r] = d2[r];
    }
  }
  __syncthreads();
  // ---- IProduct: axis 0 in registers (thread (j,k)), then axes 1 and 2
#pragma unroll
  for (int i = 0; i < Q; ++i) u[i] += B1[i * SI + ta * SJ + tb] + B2[i * SI + ta * SJ + tb];
  {
    double o[N];
#pragma unroll
    for (int a = 0; a < N; ++a) o[a] = 0.0;
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
      for (int a = 0; a < N; ++a) o[a] = fma(hxV<N, Q>[i * N + a], u[i], o[a]);
#pragma unroll
    for (int a = 0; a < N; ++a) B0[a * SI + ta * SJ + tb] = o[a];
  }
  __syncthreads();
  if (ta < N) {                                     // thread (a, k): contract j -> b
    double v[Q], o[N];
#pragma unroll
    for (int j = 0; j < Q; ++j) v[j] = B0[ta * SI + j * SJ + tb];
#pragma unroll
    for (int b = 0; b < N; ++b) o[b] = 0.0;
#pragma unroll
    for (int j = 0; j < Q; ++j)
#pragma unroll
      for (int b = 0; b < N; ++b) o[b] = fma(hxV<N, Q>[j * N + b], v[j], o[b]);
#pragma unroll
    for (int b = 0; b < N; ++b) B1[ta * SI + b * SJ + tb] = o[b];
  }
  __syncthreads();
  if (ta < N && tb < N) {                           // thread (a, b): contract k -> c, write y
    double v[Q], o[N];
#pragma unroll
    for (int k = 0; k < Q; ++k) v[k] = B1[ta * SI + tb * SJ + k];
#pragma unroll
    for (int c = 0; c < N; ++c) o[c] = 0.0;
#pragma unroll
    for (int k = 0; k < Q; ++k)
#pragma unroll
      for (int c = 0; c < N; ++c) o[c] = fma(hxV<N, Q>[k * N + c], v[k], o[c]);
    double* ye = y + dof0 + (ta * N + tb) * N;
#pragma unroll
    for (int c = 0; c < N; ++c) ye[c] = o[c];
  }
  fence_proxy_async();   // generic accesses of this element before the next TMA writes
  __syncthreads();
  }  // element loop
}

// Upload the constant tables of one (N, Q) instantiation (from the plan's pool).
template <int N, int Q>
cudaError_t hex_fast_upload(const double* V, const double* D, const double* W, const double* dVend) {
  cudaError_t e;
  if ((e = cudaMemcpyToSymbol(hxV<N, Q>, V, sizeof(double) * Q * N)) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(hxD<N, Q>, D, sizeof(double) * Q * Q)) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(hxW<N, Q>, W, sizeof(double) * Q)) != cudaSuccess) return e;
  return cudaMemcpyToSymbol(hxDVE<N, Q>, dVend, sizeof(double) * 2 * N);
}

}  // namespace sipg
