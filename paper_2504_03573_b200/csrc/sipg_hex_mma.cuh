// Hexahedron kernel on the fp64 tensor cores (sm_100a DMMA, mma.sync m8n8k4 f64).
//
// Every 1-D sum-factorisation contraction of an element — BwdTrans (V), PhysDeriv
// (D), PhysDeriv^T (D^T) and IProduct (V^T), each along the three axes — is an
// (8 x 8) x (8 x 64) product: the 1-D matrix (zero-padded to 8 x 8, held as two
// A fragments per lane for the whole kernel) times the 64 lines of the element
// tensor (zero-padded to 8^3).  One DMMA.8x8x4 does 256 FMAs in one issue slot;
// the measured fp64 tensor rate on this B200 is 36.9 TFLOP/s against 34.1 for
// DFMA (profiles/r01_dmma_peak.log), with an 8x lower instruction count.
// The neighbour traces (boundary-mode and normal-derivative planes, V P V^T) use
// the same tiles.  Tensors live in shared memory as [i][j][k] with strides
// (SI, SJ) = (100, 12) doubles so that every B-fragment load and C store pattern
// is bank-conflict free.
//
// Persistent CTAs of 4 warps; TMA bulk copies on mbarriers stream in the next
// element's face records and coefficients and the current element's six
// neighbour blocks.  Modified-modal basis on GLL points, affine elements, Q <= 8.
#pragma once
#include "sipg_kernels.cuh"
#include "sipg_hex_fast.cuh"   // mbarrier / bulk-copy helpers

namespace sipg {

template <int N, int Q> __constant__ double hmV[64];     // V [p][i]   (p < Q, i < N), zero padded
template <int N, int Q> __constant__ double hmVt[64];    // V^T [i][p]
template <int N, int Q> __constant__ double hmD[64];     // D [q][m]
template <int N, int Q> __constant__ double hmDt[64];    // D^T [m][q]
template <int N, int Q> __constant__ double hmW[8];      // GLL weights, zero padded
template <int N, int Q> __constant__ double hmDVE[16];   // psi_i'(-1) [0..7], psi_i'(+1) [8..15]

__device__ __forceinline__ void dmma(double& c0, double& c1, const double a, const double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

struct AFrag { double a0, a1; };

constexpr int MSI = 100, MSJ = 12, MBUF = 800;     // padded [i][j][k] tensor

// index of element (m along axis AX, tile = first other axis, n = second other axis)
template <int AX>
__device__ __forceinline__ int tidx(int m, int tile, int n) {
  return AX == 0 ? m * MSI + tile * MSJ + n : (AX == 1 ? tile * MSI + m * MSJ + n : tile * MSI + n * MSJ + m);
}

// out (+)= M contracted along AX of in; this warp's tiles: tile0 .. tile0+NTL-1
template <int AX, bool ACC, int NTL>
__device__ __forceinline__ void mma_axis(const double* __restrict__ in, double* __restrict__ out, const AFrag A,
                                         const int lane, const int tile0) {
  const int kq = lane & 3, n = lane >> 2;
  const int r = lane >> 2, c = 2 * (lane & 3);
  double b0[NTL], b1[NTL], c0[NTL], c1[NTL];
#pragma unroll
  for (int tt = 0; tt < NTL; ++tt) {
    b0[tt] = in[tidx<AX>(kq, tile0 + tt, n)];
    b1[tt] = in[tidx<AX>(4 + kq, tile0 + tt, n)];
    c0[tt] = ACC ? out[tidx<AX>(r, tile0 + tt, c)] : 0.0;
    c1[tt] = ACC ? out[tidx<AX>(r, tile0 + tt, c + 1)] : 0.0;
  }
#pragma unroll
  for (int tt = 0; tt < NTL; ++tt) {
    dmma(c0[tt], c1[tt], A.a0, b0[tt]);
    dmma(c0[tt], c1[tt], A.a1, b1[tt]);
  }
#pragma unroll
  for (int tt = 0; tt < NTL; ++tt) {
    out[tidx<AX>(r, tile0 + tt, c)] = c0[tt];
    out[tidx<AX>(r, tile0 + tt, c + 1)] = c1[tt];
  }
}

template <int N, int Q>
struct HexMma {
  static constexpr int NT = 128;
  static constexpr int N3 = N * N * N;
  static constexpr int BLK = (N3 + 2 + 1) & ~1;
  static constexpr int PL = 96;                        // one 8 x 8 face plane, row stride 12
  // face scratch inside the neighbour region once the planes are built
  static constexpr int NBR0 = 6 * BLK;
  static constexpr int NBR1 = 12 * PL + 12 * 64;       // stage-1 tiles + (fv, fd) of 6 faces
  static constexpr int NBR = NBR0 > NBR1 ? NBR0 : NBR1;
  static constexpr int FP = QMAX * QMAX;
  static constexpr int GFB = 4 * FP + 16 * FP + 4 * QMAX * QMAX + 2 * NMAX * NMAX + 3 * QMAX * NMAX;
  static constexpr int GSZ = GFB + 6 * 4 * Q * Q;
  // dynamic shared memory (doubles): REC[2] | X[2] | NB | U G0 G1 G2 | PLANES | generic
  static constexpr int O_REC = 0;
  static constexpr int O_X = 192;
  static constexpr int O_NB = O_X + 2 * BLK;
  static constexpr int O_T = O_NB + NBR;
  static constexpr int O_PL = O_T + 4 * MBUF;
  static constexpr int O_G = O_PL + 12 * PL;
  static size_t smem_bytes(bool gen) { return sizeof(double) * (size_t)(O_G + (gen ? GSZ : 0)); }
};

template <int N, int Q, bool GEN>
__global__ void __launch_bounds__(128)
k_hex_mma(const DevPlan P, const int cls, const double* __restrict__ x, double* __restrict__ y) {
  using H = HexMma<N, Q>;
  constexpr int N3 = H::N3, QQ = Q * Q, PL = H::PL;
  static_assert(Q <= 8 && N <= Q, "single 8-tile DMMA kernel");
  extern __shared__ __align__(16) double dsm[];
  double* NB = dsm + H::O_NB;
  double* U = dsm + H::O_T;
  double* G0 = U + MBUF;
  double* G1 = G0 + MBUF;
  double* G2 = G1 + MBUF;
  double* PLN = dsm + H::O_PL;        // planes, later stage-2 outputs
  double* TT = NB;                    // stage-1 outputs (12 planes), after the planes are built
  double* FVD = NB + 12 * PL;         // (fv, fd) per face point [f][2][64]
  double* gsm = dsm + H::O_G;
  __shared__ double sM[4 * 64];
  __shared__ double sW[8];
  __shared__ double sDVE[16];
  __shared__ int sk[6];
  __shared__ int soff[8];
  __shared__ __align__(8) uint64_t mbar[3];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int* cd = P.cd + cls * CD_WORDS;
  const int count = cd[CD_COUNT];
  const int* elist = P.class_elems + cd[CD_ELEM_OFF];
  const double lam = P.lam;

  for (int i = t; i < 64; i += 128) {
    sM[i] = hmV<N, Q>[i];
    sM[64 + i] = hmVt<N, Q>[i];
    sM[128 + i] = hmD<N, Q>[i];
    sM[192 + i] = hmDt<N, Q>[i];
  }
  if (t < 8) sW[t] = hmW<N, Q>[t];
  if (t < 16) sDVE[t] = hmDVE<N, Q>[t];
  if (t == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&mbar[2], 1);
    fence_proxy_async();
  }
  __syncthreads();
  const int ar = lane >> 2, ac = lane & 3;
  const AFrag AV = {sM[ar * 8 + ac], sM[ar * 8 + 4 + ac]};
  const AFrag AVt = {sM[64 + ar * 8 + ac], sM[64 + ar * 8 + 4 + ac]};
  const AFrag AD = {sM[128 + ar * 8 + ac], sM[128 + ar * 8 + 4 + ac]};
  const AFrag ADt = {sM[192 + ar * 8 + ac], sM[192 + ar * 8 + 4 + ac]};

  auto issue_own = [&](int iel, int st) {
    const FaceRec* rsrc = P.recs + cd[CD_REC_OFF] + (int64_t)iel * 6;
    bulk_g2s(dsm + H::O_REC + st * 96, rsrc, 6 * sizeof(FaceRec), &mbar[st]);
    unsigned nb;
    soff[st] = bulk_block(dsm + H::O_X + st * H::BLK, x + P.dof_off[elist[iel]], N3, &mbar[st], &nb);
    mbar_expect_tx(&mbar[st], 6 * sizeof(FaceRec) + nb);
    cp_async_commit();
  };
  if (t == 0 && blockIdx.x < count) issue_own(blockIdx.x, 0);

  int kk = 0;
  for (int iel = blockIdx.x; iel < count; iel += gridDim.x, ++kk) {
    const int st = kk & 1;
    const bool more = iel + (int)gridDim.x < count;
    if (t == 0 && more) issue_own(iel + gridDim.x, st ^ 1);
    if (t == 0) {                        // head/tail doubles of this element (issued by thread 0)
      if (more) cp_async_wait<1>(); else cp_async_wait<0>();
    }
    mbar_wait(&mbar[st], (kk >> 1) & 1);
    __syncthreads();
    const FaceRec* srec = reinterpret_cast<const FaceRec*>(dsm + H::O_REC + st * 96);
    const double* X = dsm + H::O_X + st * H::BLK + soff[st];
    const int e = elist[iel];
    const int64_t dof0 = P.dof_off[e];
    if (t < 6) {
      const int fl = srec[t].flags, ty = srec[t].type;
      sk[t] = (ty == FT_DIRECT && (fl & F_FAST_HEX)) ? 1 : ((ty == FT_BOUNDARY && !(fl & F_SELF_PW)) ? 2 : 0);
    }
    if (t == 32) {   // neighbour blocks of this element (another warp than the prefetch issuer)
      unsigned total = 0;
#pragma unroll
      for (int f = 0; f < 6; ++f) {
        if (srec[f].type == FT_DIRECT && (srec[f].flags & F_FAST_HEX)) {
          unsigned nb;
          soff[2 + f] = bulk_block(NB + f * H::BLK, x + srec[f].nbr_dof, N3, &mbar[2], &nb);
          total += nb;
        }
      }
      mbar_expect_tx(&mbar[2], total);
      cp_async_commit();
    }

    // ---- BwdTrans.  Axis 2 straight from the raw coefficient block (zero padded on the fly)
    {
      const int kq = lane & 3, n = lane >> 2, r = lane >> 2, c = 2 * (lane & 3);
#pragma unroll
      for (int tt = 0; tt < 2; ++tt) {
        const int a = warp * 2 + tt;                 // line (a, b = n), contracted index m
        double c0 = 0.0, c1 = 0.0;
        const bool okl = a < N && n < N;
        const double b0 = (okl && kq < N) ? X[(a * N + n) * N + kq] : 0.0;
        const double b1 = (okl && 4 + kq < N) ? X[(a * N + n) * N + 4 + kq] : 0.0;
        dmma(c0, c1, AV.a0, b0);
        dmma(c0, c1, AV.a1, b1);
        G0[tidx<2>(r, a, c)] = c0;                   // t1[a][b][k]
        G0[tidx<2>(r, a, c + 1)] = c1;
      }
    }
    __syncthreads();
    mma_axis<1, false, 2>(G0, G1, AV, lane, warp * 2);   // t2[a][j][k]
    __syncthreads();
    mma_axis<0, false, 2>(G1, U, AV, lane, warp * 2);    // u[i][j][k]
    __syncthreads();
    // ---- PhysDeriv along the three axes
    mma_axis<0, false, 2>(U, G0, AD, lane, warp * 2);
    mma_axis<1, false, 2>(U, G1, AD, lane, warp * 2);
    mma_axis<2, false, 2>(U, G2, AD, lane, warp * 2);
    if (t == 32) cp_async_wait<0>();     // neighbour head/tail doubles (issued by thread 32)
    mbar_wait(&mbar[2], kk & 1);
    __syncthreads();

    // ---- fast faces: neighbour boundary-mode / normal-derivative planes (DFMA), then V P V^T (DMMA)
    if (t < 64) {
      const int i0 = t >> 3, i1 = t & 7;
#pragma unroll
      for (int f = 0; f < 6; ++f) {
        if (sk[f] != 1) continue;
        double pu = 0.0, pd = 0.0;
        if (i0 < N && i1 < N) {
          const int fo = srec[f].nbr_face, ao = fo >> 1;
          const int b0 = ao == 0 ? 1 : 0, b1 = ao == 2 ? 1 : 2;
          const double* cc = NB + f * H::BLK + soff[2 + f] + i0 * hex_stride(b0, N) + i1 * hex_stride(b1, N);
          const int sa = hex_stride(ao, N);
          const double* dv = sDVE + ((fo & 1) ? 8 : 0);
#pragma unroll
          for (int i = 0; i < N; ++i) pd = fma(dv[i], cc[i * sa], pd);
          pu = cc[(fo & 1) ? (N - 1) * sa : 0];
        }
        PLN[(2 * f) * PL + i0 * 12 + i1] = pu;
        PLN[(2 * f + 1) * PL + i0 * 12 + i1] = pd;
      }
    }
    __syncthreads();
    {
      const int kq = lane & 3, n = lane >> 2, r = lane >> 2, c = 2 * (lane & 3);
      // stage 1: T[p0][i1] = sum_i0 V[p0][i0] P[i0][i1]      (3 face-planes per warp)
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int fp = warp * 3 + q;
        if (sk[fp >> 1] != 1) continue;
        const double* pl = PLN + fp * PL;
        double c0 = 0.0, c1 = 0.0;
        dmma(c0, c1, AV.a0, pl[kq * 12 + n]);
        dmma(c0, c1, AV.a1, pl[(4 + kq) * 12 + n]);
        TT[fp * PL + r * 12 + c] = c0;
        TT[fp * PL + r * 12 + c + 1] = c1;
      }
      __syncwarp();
      // stage 2: U2[p0][p1] = sum_i1 V[p1][i1] T[p0][i1]    (same face-planes, same warp)
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int fp = warp * 3 + q;
        if (sk[fp >> 1] != 1) continue;
        const double* tt = TT + fp * PL;
        double c0 = 0.0, c1 = 0.0;
        dmma(c0, c1, AV.a0, tt[n * 12 + kq]);
        dmma(c0, c1, AV.a1, tt[n * 12 + 4 + kq]);
        PLN[fp * PL + c * 12 + r] = c0;               // U2[p0 = c][p1 = r]
        PLN[fp * PL + (c + 1) * 12 + r] = c1;
      }
    }
    // ---- generic faces (own u, du_k published, then generic_face)
    double* gfb = gsm + H::GFB;
    if (GEN) {
      __syncthreads();
      for (int f = 0; f < 6; ++f) {
        if (sk[f] != 0) continue;
        double* us = gsm;
        const int a = f >> 1, hi = f & 1;
        for (int p = t; p < QQ; p += 128) {
          const int p0 = p / Q, p1 = p - (p / Q) * Q;
          const int fix = hi ? Q - 1 : 0;
          const int v = a == 0 ? fix * MSI + p0 * MSJ + p1 : (a == 1 ? p0 * MSI + fix * MSJ + p1 : p0 * MSI + p1 * MSJ + fix);
          us[p] = U[v]; us[H::FP + p] = G0[v]; us[2 * H::FP + p] = G1[v]; us[3 * H::FP + p] = G2[v];
        }
        __syncthreads();
        generic_face<SHAPE_HEX, N, Q>(P, srec[f], f, x, us, gfb + f * 4 * QQ, gsm + 4 * H::FP, t, 128);
        __syncthreads();
      }
    }
    __syncthreads();
    // ---- flux at every face point of the fast / boundary faces: (fv, fd) -> FVD
    for (int it = t; it < 6 * 64; it += 128) {
      const int f = it >> 6, p = it & 63;
      const int kind = sk[f];
      const int p0 = p >> 3, p1 = p & 7;
      if (kind == 0 || p0 >= Q || p1 >= Q) continue;
      const FaceRec& rr = srec[f];
      const int a = f >> 1, fix = (f & 1) ? Q - 1 : 0;
      const int v = a == 0 ? fix * MSI + p0 * MSJ + p1 : (a == 1 ? p0 * MSI + fix * MSJ + p1 : p0 * MSI + p1 * MSJ + fix);
      const double swj = rr.sJ * sW[p0] * sW[p1];
      const double us = U[v];
      const double gs = rr.gs[0] * G0[v] + rr.gs[1] * G1[v] + rr.gs[2] * G2[v];
      double jump, avg;
      if (kind == 2) {
        jump = 2.0 * us;
        avg = gs;
      } else {
        jump = us - PLN[(2 * f) * PL + p0 * 12 + p1];
        avg = 0.5 * (gs - rr.go[rr.nbr_face >> 1] * PLN[(2 * f + 1) * PL + p0 * 12 + p1]);
      }
      FVD[f * 128 + p] = (rr.tau * jump - avg) * swj;
      FVD[f * 128 + 64 + p] = -0.5 * jump * swj;
    }
    __syncthreads();
    // ---- volume metric (in place): U -> lam jw u, G -> jw G G^T du
    {
      const double* eg = P.egeo + cd[CD_EGEO_OFF] + (int64_t)iel * cd[CD_EGEO_STRIDE];
      const double J = eg[0];
      const double K0 = eg[1], K1 = eg[2], K2 = eg[3], K3 = eg[4], K4 = eg[5], K5 = eg[6];
      const int j = t >> 4, kb = (t & 15) >> 3;   // 128 threads: (j, k-half, k) x 4 i-values
      const int k = t & 7;
      const double wjk = J * sW[j] * sW[k];
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const int i = kb * 4 + s;
        const int v = i * MSI + j * MSJ + k;
        const double jw = wjk * sW[i];
        const double g0 = G0[v], g1 = G1[v], g2 = G2[v];
        U[v] = lam * jw * U[v];
        G0[v] = jw * (K0 * g0 + K1 * g1 + K2 * g2);
        G1[v] = jw * (K1 * g0 + K3 * g1 + K4 * g2);
        G2[v] = jw * (K2 * g0 + K4 * g1 + K5 * g2);
      }
    }
    __syncthreads();
    // ---- lift: fold face fluxes into the point arrays, one face at a time (faces share edges)
    for (int f = 0; f < 6; ++f) {
      const int kind = sk[f];
      if (t < 64) {
        const int p0 = t >> 3, p1 = t & 7;
        if (p0 < Q && p1 < Q && (kind != 0 || GEN)) {
          const int a = f >> 1, fix = (f & 1) ? Q - 1 : 0;
          const int v = a == 0 ? fix * MSI + p0 * MSJ + p1 : (a == 1 ? p0 * MSI + fix * MSJ + p1 : p0 * MSI + p1 * MSJ + fix);
          if (kind != 0) {
            const double fv = FVD[f * 128 + t], fd = FVD[f * 128 + 64 + t];
            U[v] += fv;
            G0[v] = fma(fd, srec[f].gs[0], G0[v]);
            G1[v] = fma(fd, srec[f].gs[1], G1[v]);
            G2[v] = fma(fd, srec[f].gs[2], G2[v]);
          } else {
            const double* fbf = gfb + f * 4 * QQ;
            const int p = p0 * Q + p1;
            U[v] += fbf[p];
            G0[v] += fbf[QQ + p];
            G1[v] += fbf[2 * QQ + p];
            G2[v] += fbf[3 * QQ + p];
          }
        }
      }
      __syncthreads();
    }
    // ---- R = P0 + D^T along each axis (accumulated in U), then IProduct
    mma_axis<0, true, 2>(G0, U, ADt, lane, warp * 2);
    __syncthreads();
    mma_axis<1, true, 2>(G1, U, ADt, lane, warp * 2);
    __syncthreads();
    mma_axis<2, true, 2>(G2, U, ADt, lane, warp * 2);
    __syncthreads();
    mma_axis<0, false, 2>(U, G0, AVt, lane, warp * 2);   // [a][j][k]
    __syncthreads();
    mma_axis<1, false, 2>(G0, G1, AVt, lane, warp * 2);  // [a][b][k]
    __syncthreads();
    mma_axis<2, false, 2>(G1, G2, AVt, lane, warp * 2);  // [a][b][c]
    __syncthreads();
    for (int i = t; i < N3; i += 128) {
      const int a = i / (N * N), rm = i - a * N * N, b = rm / N, c = rm - b * N;
      y[dof0 + i] = G2[a * MSI + b * MSJ + c];
    }
    fence_proxy_async();
    __syncthreads();
  }
}

template <int N, int Q>
cudaError_t hex_mma_upload(const double* V, const double* D, const double* W, const double* dVend) {
  double v[64] = {0}, vt[64] = {0}, d[64] = {0}, dt[64] = {0}, w[8] = {0}, dve[16] = {0};
  for (int p = 0; p < Q; ++p)
    for (int i = 0; i < N; ++i) {
      v[p * 8 + i] = V[p * N + i];
      vt[i * 8 + p] = V[p * N + i];
    }
  for (int q = 0; q < Q; ++q)
    for (int m = 0; m < Q; ++m) {
      d[q * 8 + m] = D[q * Q + m];
      dt[m * 8 + q] = D[q * Q + m];
    }
  for (int p = 0; p < Q; ++p) w[p] = W[p];
  for (int i = 0; i < N; ++i) {
    dve[i] = dVend[i];
    dve[8 + i] = dVend[N + i];
  }
  cudaError_t e;
  if ((e = cudaMemcpyToSymbol(hmV<N, Q>, v, sizeof(v))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(hmVt<N, Q>, vt, sizeof(vt))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(hmD<N, Q>, d, sizeof(d))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(hmDt<N, Q>, dt, sizeof(dt))) != cudaSuccess) return e;
  if ((e = cudaMemcpyToSymbol(hmW<N, Q>, w, sizeof(w))) != cudaSuccess) return e;
  return cudaMemcpyToSymbol(hmDVE<N, Q>, dve, sizeof(dve));
}

}  // namespace sipg
