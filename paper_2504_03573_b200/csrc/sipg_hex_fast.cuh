// Register-column hexahedron kernel (sm_100a, fp64): modified-modal basis on
// GLL points, affine elements.  One CTA of Q*Q threads per element; thread
// (j,k) owns the Q points (i, j, k) along axis 0 in registers, so the axis-0
// contractions of BwdTrans / PhysDeriv / PhysDeriv^T / IProduct are in-register
// and only the axis-1/2 contractions go through (bank-padded) shared memory.
// 1-D tables live in __constant__ memory per (N, Q) instantiation and are
// read as immediate operands of DFMA.
//
// Faces: conforming same-class neighbours and boundary faces take the batched
// fast path (all six faces' neighbour traces evaluated together from the
// neighbours' coefficients, flux computed by the thread owning each face point
// and added straight into its register point arrays — no scatter, no
// atomics).  Any other coupling (shared trace, p2p, orientation transfers,
// pointwise geometry) goes through generic_face().
#pragma once
#include "sipg_kernels.cuh"

namespace sipg {

template <int N, int Q> __constant__ double hxV[Q * N];     // psi_i(x_p), [p][i]
template <int N, int Q> __constant__ double hxD[Q * Q];     // collocation derivative
template <int N, int Q> __constant__ double hxW[Q];         // GLL weights
template <int N, int Q> __constant__ double hxDVE[2 * N];   // psi_i'(-1), psi_i'(+1)

template <int N, int Q>
struct HexFast {
  static constexpr int NT = Q * Q;
  static constexpr int SJ = Q + 1;            // padded row stride (bank spread)
  static constexpr int SI = Q * SJ;
  static constexpr int BUF = Q * SI;
  static constexpr int FSC = 12 * N * N + 12 * Q * N + 12 * Q * Q;   // fast-face scratch
  static constexpr int SCR = 4 * BUF > FSC ? 4 * BUF : FSC;            // B0..B3 as one array
  // generic-face scratch (dynamic smem): us (4 FP), fscr (4*4 FP + 4 QMAX^2 + nscr), fb (6*4*Q*Q)
  static constexpr int FP = QMAX * QMAX;
  static constexpr int GSZ = 4 * FP + 16 * FP + 4 * QMAX * QMAX + 2 * NMAX * NMAX + 3 * QMAX * NMAX + 6 * 4 * Q * Q;
};

// face f of a hex: fixed axis f>>1, side (f&1 ? +1 : -1), run axes ascending
__device__ __forceinline__ int hex_stride(int axis, int n) { return axis == 0 ? n * n : (axis == 1 ? n : 1); }

template <int N, int Q, bool GEN>
__global__ void __launch_bounds__(Q * Q)
k_hex(const DevPlan P, const int cls, const double* __restrict__ x, double* __restrict__ y) {
  using H = HexFast<N, Q>;
  constexpr int NT = H::NT, SJ = H::SJ, SI = H::SI, BUF = H::BUF;
  __shared__ double S[H::SCR];
  __shared__ double sW[Q];
  __shared__ FaceRec srec[6];
  __shared__ int sfast[6];            // 1 fast conforming, 2 boundary, 0 generic
  __shared__ int snbr[6];
  __shared__ int64_t snoff[6];
  extern __shared__ double gsm[];
  double* B0 = S;
  double* B1 = S + BUF;
  double* B2 = S + 2 * BUF;
  const int t = threadIdx.x;
  const int ta = t / Q, tb = t - (t / Q) * Q;
  const int* cd = P.cd + cls * CD_WORDS;
  const int iel = blockIdx.x;
  const int e = P.class_elems[cd[CD_ELEM_OFF] + iel];
  const double* xe = x + P.dof_off[e];
  const int rbase = cd[CD_REC_OFF] + iel * 6;

  // ---- records, weights, coefficients
  for (int i = t; i < 6 * 16; i += NT)
    reinterpret_cast<double*>(srec)[i] = __ldg(reinterpret_cast<const double*>(P.recs + rbase) + i);
  if (t < Q) sW[t] = hxW<N, Q>[t];
  for (int idx = t; idx < N * N * N; idx += NT) {
    const int a = idx / (N * N), r = idx - a * N * N, b = r / N, c = r - b * N;
    B0[a * SI + b * SJ + c] = __ldg(xe + idx);
  }
  __syncthreads();
  if (t < 6) {
    const FaceRec& r = srec[t];
    int kind = 0;
    if (r.type == FT_BOUNDARY && !(r.flags & F_SELF_PW)) {
      kind = 2;
    } else if (r.type == FT_DIRECT && (r.flags & F_OTHER_ID) && !(r.flags & (F_SELF_PW | F_OTHER_PW))) {
      const int* cdo = P.cd + P.elem_class[r.nbr] * CD_WORDS;
      const int fo = r.nbr_face;
      const int b0 = (fo >> 1) == 0 ? 1 : 0, b1 = (fo >> 1) == 2 ? 1 : 2;
      if (cdo[CD_SHAPE] == SHAPE_HEX && cdo[CD_N] == N && cdo[CD_Q0] == Q && r.go[b0] == 0.0 && r.go[b1] == 0.0)
        kind = 1;
    }
    sfast[t] = kind;
    snbr[t] = r.nbr;
    snoff[t] = r.nbr >= 0 ? P.dof_off[r.nbr] : 0;
  }

  // ---- BwdTrans: axis 2 (thread (a,b)), axis 1 (thread (a,k)), axis 0 (thread (j,k))
  if (ta < N && tb < N) {
    double v[N];
#pragma unroll
    for (int c = 0; c < N; ++c) v[c] = B0[ta * SI + tb * SJ + c];
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < N; ++c) acc = fma(hxV<N, Q>[k * N + c], v[c], acc);
      B1[ta * SI + tb * SJ + k] = acc;
    }
  }
  __syncthreads();
  if (ta < N) {
    double v[N];
#pragma unroll
    for (int b = 0; b < N; ++b) v[b] = B1[ta * SI + b * SJ + tb];
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < N; ++b) acc = fma(hxV<N, Q>[j * N + b], v[b], acc);
      B2[ta * SI + j * SJ + tb] = acc;
    }
  }
  __syncthreads();
  double u[Q], d0[Q], d1[Q], d2[Q];
  {
    double v[N];
#pragma unroll
    for (int a = 0; a < N; ++a) v[a] = B2[a * SI + ta * SJ + tb];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(hxV<N, Q>[i * N + a], v[a], acc);
      u[i] = acc;
    }
  }
  // ---- PhysDeriv: axis 0 in registers; axes 1, 2 through shared memory
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < Q; ++m) acc = fma(hxD<N, Q>[i * Q + m], u[m], acc);
    d0[i] = acc;
    B0[i * SI + ta * SJ + tb] = u[i];
  }
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
      double a1 = 0.0, a2 = 0.0;
#pragma unroll
      for (int m = 0; m < Q; ++m) {
        a1 = fma(hxD<N, Q>[r * Q + m], v[m], a1);
        a2 = fma(hxD<N, Q>[r * Q + m], w[m], a2);
      }
      B1[ta * SI + r * SJ + tb] = a1;
      B2[ta * SI + tb * SJ + r] = a2;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    d1[i] = B1[i * SI + ta * SJ + tb];
    d2[i] = B2[i * SI + ta * SJ + tb];
  }
  __syncthreads();   // S is face scratch from here on

  // ---- faces.  Fast path: neighbour (u, du_normal) on the shared face grid
  // straight from the neighbours' coefficients, all fast faces at once.
  // planes: NPu/NPd [f][i0][i1] (N*N each), stage 1 T[f][pl][p0][i1], stage 2 U[f][pl][p0][p1]
  double* NP = S;                              // 6*2*N*N
  double* T1 = NP + 12 * N * N;                // 6*2*Q*N
  double* U2 = T1 + 12 * Q * N;                // 6*2*Q*Q
  static_assert(12 * N * N + 12 * Q * N + 12 * Q * Q <= H::SCR, "face scratch");
  for (int it = t; it < 6 * N * N; it += NT) {
    const int f = it / (N * N), r = it - f * N * N;
    if (sfast[f] != 1) continue;
    const int i0 = r / N, i1 = r - i0 * N;
    const int fo = srec[f].nbr_face, ao = fo >> 1, so = fo & 1;
    const int b0 = ao == 0 ? 1 : 0, b1 = ao == 2 ? 1 : 2;
    const double* xo = x + snoff[f];
    const int base = i0 * hex_stride(b0, N) + i1 * hex_stride(b1, N);
    const int sa = hex_stride(ao, N);
    double pd = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double dv = so ? hxDVE<N, Q>[N + i] : hxDVE<N, Q>[i];
      pd = fma(dv, __ldg(xo + base + i * sa), pd);
    }
    NP[(2 * f) * N * N + r] = __ldg(xo + base + (so ? (N - 1) * sa : 0));   // modified-modal boundary mode
    NP[(2 * f + 1) * N * N + r] = pd;
  }
  __syncthreads();
  for (int it = t; it < 12 * N; it += NT) {      // stage 1: contract i0 -> p0, line over i0 at fixed i1
    const int fp = it / N, i1 = it - fp * N;
    if (sfast[fp >> 1] != 1) continue;
    double v[N];
#pragma unroll
    for (int i0 = 0; i0 < N; ++i0) v[i0] = NP[fp * N * N + i0 * N + i1];
#pragma unroll
    for (int p0 = 0; p0 < Q; ++p0) {
      double acc = 0.0;
#pragma unroll
      for (int i0 = 0; i0 < N; ++i0) acc = fma(hxV<N, Q>[p0 * N + i0], v[i0], acc);
      T1[fp * Q * N + p0 * N + i1] = acc;
    }
  }
  __syncthreads();
  for (int it = t; it < 12 * Q; it += NT) {      // stage 2: contract i1 -> p1
    const int fp = it / Q, p0 = it - fp * Q;
    if (sfast[fp >> 1] != 1) continue;
    double v[N];
#pragma unroll
    for (int i1 = 0; i1 < N; ++i1) v[i1] = T1[fp * Q * N + p0 * N + i1];
#pragma unroll
    for (int p1 = 0; p1 < Q; ++p1) {
      double acc = 0.0;
#pragma unroll
      for (int i1 = 0; i1 < N; ++i1) acc = fma(hxV<N, Q>[p1 * N + i1], v[i1], acc);
      U2[fp * Q * Q + p0 * Q + p1] = acc;
    }
  }
  // generic faces (dynamic shared memory; GEN instantiations only)
  double* gfb = gsm + 4 * H::FP + 16 * H::FP + 4 * QMAX * QMAX + 2 * NMAX * NMAX + 3 * QMAX * NMAX;
  if (GEN) {
    __syncthreads();
    for (int f = 0; f < 6; ++f) {
      if (sfast[f] != 0) continue;
      // own u, du_k on face f's grid (owners write), then the generic flux
      const int a = f >> 1, hi = f & 1;
      double* us = gsm;
      // point (p0, p1) of face f: a=0 -> (j,k); a=1 -> (i,k); a=2 -> (i,j)
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
      generic_face<SHAPE_HEX, N, Q>(P, srec[f], f, x, us, gfb + f * 4 * Q * Q, gsm + 4 * H::FP, t, NT);
      __syncthreads();
    }
  }
  __syncthreads();

  // ---- flux at the face points owned by this thread + volume metric, per point
  const double lam = P.lam;
  const double* eg = P.egeo + cd[CD_EGEO_OFF] + (int64_t)iel * cd[CD_EGEO_STRIDE];
  const double J = eg[0];
  const double K0 = eg[1], K1 = eg[2], K2 = eg[3], K3 = eg[4], K4 = eg[5], K5 = eg[6];
  const double wjk = sW[ta] * sW[tb];
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;     // face contributions to P0..P3
    const double ui = u[i], g0 = d0[i], g1 = d1[i], g2 = d2[i];
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      const int a = f >> 1, hi = f & 1;
      const int own = a == 0 ? (i == (hi ? Q - 1 : 0)) : (a == 1 ? (ta == (hi ? Q - 1 : 0)) : (tb == (hi ? Q - 1 : 0)));
      if (!own) continue;
      const int p0 = a == 0 ? ta : i, p1 = a == 2 ? ta : tb;
      const int kind = sfast[f];
      if (kind == 0) {
        if (GEN) {
          const double* fbf = gfb + f * 4 * Q * Q;
          const int p = p0 * Q + p1;
          c0 += fbf[p]; c1 += fbf[Q * Q + p]; c2 += fbf[2 * Q * Q + p]; c3 += fbf[3 * Q * Q + p];
        }
        continue;
      }
      const FaceRec& r = srec[f];
      const double swj = r.sJ * sW[p0] * sW[p1];
      const double gs = r.gs[0] * g0 + r.gs[1] * g1 + r.gs[2] * g2;
      double jump, avg;
      if (kind == 2) {
        jump = 2.0 * ui;
        avg = gs;
      } else {
        const int ao = r.nbr_face >> 1;
        const double uo = U2[(2 * f) * Q * Q + p0 * Q + p1];
        const double go = r.go[ao] * U2[(2 * f + 1) * Q * Q + p0 * Q + p1];
        jump = ui - uo;
        avg = 0.5 * (gs - go);
      }
      const double fv = (r.tau * jump - avg) * swj;
      const double fd = -0.5 * jump * swj;
      c0 += fv;
      c1 += fd * r.gs[0];
      c2 += fd * r.gs[1];
      c3 += fd * r.gs[2];
    }
    const double jw = J * hxW<N, Q>[i] * wjk;
    u[i] = lam * jw * ui + c0;
    d0[i] = jw * (K0 * g0 + K1 * g1 + K2 * g2) + c1;
    d1[i] = jw * (K1 * g0 + K3 * g1 + K4 * g2) + c2;
    d2[i] = jw * (K2 * g0 + K4 * g1 + K5 * g2) + c3;
  }
  __syncthreads();   // face scratch (S) is reused below

  // ---- R = P0 + D0^T P1 (registers) + D1^T P2 + D2^T P3 (shared memory)
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    B1[i * SI + ta * SJ + tb] = d1[i];
    B2[i * SI + ta * SJ + tb] = d2[i];
  }
#pragma unroll
  for (int i = 0; i < Q; ++i) {
    double acc = u[i];
#pragma unroll
    for (int m = 0; m < Q; ++m) acc = fma(hxD<N, Q>[m * Q + i], d0[m], acc);
    u[i] = acc;
  }
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
      double a1 = 0.0, a2 = 0.0;
#pragma unroll
      for (int m = 0; m < Q; ++m) {
        a1 = fma(hxD<N, Q>[m * Q + r], v[m], a1);
        a2 = fma(hxD<N, Q>[m * Q + r], w[m], a2);
      }
      B1[ta * SI + r * SJ + tb] = a1;
      B2[ta * SI + tb * SJ + r] = a2;
    }
  }
  __syncthreads();
  // ---- IProduct: axis 0 in registers (thread (j,k)), then axes 1 and 2
#pragma unroll
  for (int i = 0; i < Q; ++i) u[i] += B1[i * SI + ta * SJ + tb] + B2[i * SI + ta * SJ + tb];
#pragma unroll
  for (int a = 0; a < N; ++a) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < Q; ++i) acc = fma(hxV<N, Q>[i * N + a], u[i], acc);
    B0[a * SI + ta * SJ + tb] = acc;
  }
  __syncthreads();
  if (ta < N) {                                     // thread (a, k): contract j -> b
    double v[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) v[j] = B0[ta * SI + j * SJ + tb];
#pragma unroll
    for (int b = 0; b < N; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < Q; ++j) acc = fma(hxV<N, Q>[j * N + b], v[j], acc);
      B1[ta * SI + b * SJ + tb] = acc;
    }
  }
  __syncthreads();
  if (ta < N && tb < N) {                           // thread (a, b): contract k -> c, write y
    double v[Q];
#pragma unroll
    for (int k = 0; k < Q; ++k) v[k] = B1[ta * SI + tb * SJ + k];
    double* ye = y + P.dof_off[e] + (ta * N + tb) * N;
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < Q; ++k) acc = fma(hxV<N, Q>[k * N + c], v[k], acc);
      ye[c] = acc;
    }
  }
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
