// Warp-per-element hexahedron kernel on the fp64 tensor cores (sm_100a DMMA).
//
// Each warp owns one element at a time (persistent: warps stride over the
// class's elements) and never synchronises with other warps: every 1-D
// contraction is 8 independent (8x8)x(8x8) DMMA tiles issued back to back by
// the warp (ILP 8), separated only by __syncwarp.  A warp's shared-memory slice
// holds the element tensor fields (u, du_0..2 -> P_0..3) as [i][j][k] with row
// stride 8, plane stride 68 and an XOR swizzle k ^ 4*((j>>1)&1), which makes
// the B-fragment loads of all three axes bank-conflict free at 544 doubles per
// field.  Face records, the element's coefficients (next element prefetched)
// and the six neighbours' coefficient blocks arrive by TMA bulk copies on
// per-warp mbarriers.  Faces: constant-metric boundary faces and F_FAST_HEX
// conforming faces (neighbour boundary-mode / normal-derivative planes -> V P V^T
// on DMMA).  Classes with other couplings use k_hex_mma / k_hex.
#pragma once
#include "sipg_kernels.cuh"
#include "sipg_hex_fast.cuh"
#include "sipg_hex_mma.cuh"

namespace sipg {

constexpr int WSI = 68;          // plane stride of a swizzled field
constexpr int WBUF = 8 * WSI;    // 544 doubles per field

__device__ __forceinline__ int wsw(int i, int j, int k) { return i * WSI + j * 8 + (k ^ ((j & 2) << 1)); }

template <int AX>
__device__ __forceinline__ int widx(int m, int tile, int n) {
  return AX == 0 ? wsw(m, tile, n) : (AX == 1 ? wsw(tile, m, n) : wsw(tile, n, m));
}

// whole-tensor contraction by one warp: out (+)= M along AX, 8 tiles
template <int AX, bool ACC>
__device__ __forceinline__ void w_axis(const double* __restrict__ in, double* __restrict__ out, const AFrag A,
                                       const int lane) {
  const int kq = lane & 3, n = lane >> 2;
  const int r = lane >> 2, c = 2 * (lane & 3);
  double b0[8], b1[8], c0[8], c1[8];
#pragma unroll
  for (int tt = 0; tt < 8; ++tt) {
    b0[tt] = in[widx<AX>(kq, tt, n)];
    b1[tt] = in[widx<AX>(4 + kq, tt, n)];
  }
#pragma unroll
  for (int tt = 0; tt < 8; ++tt) {
    c0[tt] = ACC ? out[widx<AX>(r, tt, c)] : 0.0;
    c1[tt] = ACC ? out[widx<AX>(r, tt, c + 1)] : 0.0;
  }
#pragma unroll
  for (int tt = 0; tt < 8; ++tt) dmma(c0[tt], c1[tt], A.a0, b0[tt]);
#pragma unroll
  for (int tt = 0; tt < 8; ++tt) dmma(c0[tt], c1[tt], A.a1, b1[tt]);
#pragma unroll
  for (int tt = 0; tt < 8; ++tt) {
    out[widx<AX>(r, tt, c)] = c0[tt];
    out[widx<AX>(r, tt, c + 1)] = c1[tt];
  }
  __syncwarp();
}

template <int N, int Q>
struct HexWarpSlice {
  static constexpr int N3 = N * N * N;
  static constexpr int BLK = (N3 + 2 + 1) & ~1;
  static constexpr int FBLK = BLK > 320 ? BLK : 320;
  static constexpr int SLICE = (192 + 2 * BLK + 6 * FBLK + 4 * WBUF + 3 * 96 + 1) & ~1;
  // warps per CTA: as many slices as fit in ~216 KB of shared memory, at most 8
  static constexpr int W0 = (216 * 1024) / (8 * SLICE);
  static constexpr int W = W0 > 8 ? 8 : (W0 < 1 ? 1 : W0);
};

template <int N, int Q, int W>
struct HexWarp {
  static constexpr int N3 = N * N * N;
  static constexpr int BLK = (N3 + 2 + 1) & ~1;
  static constexpr int FBLK = BLK > 320 ? BLK : 320;     // per face: TMA block, later 2 planes + (fv, fd)
  // per-warp slice (doubles): REC[2] | X[2] | NB[6] | U G0 G1 G2 | TT (3 planes)
  static constexpr int O_REC = 0;
  static constexpr int O_X = 192;
  static constexpr int O_NB = O_X + 2 * BLK;
  static constexpr int O_T = O_NB + 6 * FBLK;
  static constexpr int O_TT = O_T + 4 * WBUF;
  static constexpr int SLICE = (O_TT + 3 * 96 + 1) & ~1;
  static size_t smem_bytes() { return sizeof(double) * (size_t)SLICE * W; }
};

template <int N, int Q, int W>
__global__ void __launch_bounds__(32 * W)
k_hexw(const DevPlan P, const int cls, const double* __restrict__ x, double* __restrict__ y) {
  using H = HexWarp<N, Q, W>;
  constexpr int N3 = H::N3;
  static_assert(Q <= 8 && N <= Q, "single 8-tile DMMA kernel");
  extern __shared__ __align__(16) double dsm[];
  __shared__ double sM[4 * 64];
  __shared__ double sW[8];
  __shared__ double sDVE[16];
  __shared__ __align__(8) uint64_t mbar_all[W][3];
  __shared__ int soff_all[W][8];
  __shared__ int sk_all[W][6];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double* sl = dsm + warp * H::SLICE;
  double* NB = sl + H::O_NB;
  double* U = sl + H::O_T;
  double* G0 = U + WBUF;
  double* G1 = G0 + WBUF;
  double* G2 = G1 + WBUF;
  double* TT = sl + H::O_TT;
  uint64_t* mbar = mbar_all[warp];
  int* soff = soff_all[warp];
  int* sk = sk_all[warp];
  const int* cd = P.cd + cls * CD_WORDS;
  const int count = cd[CD_COUNT];
  const int* elist = P.class_elems + cd[CD_ELEM_OFF];
  const double lam = P.lam;
  const double* egeo = P.egeo + cd[CD_EGEO_OFF];
  const int estride = cd[CD_EGEO_STRIDE];

  for (int i = t; i < 64; i += 32 * W) {
    sM[i] = hmV<N, Q>[i];
    sM[64 + i] = hmVt<N, Q>[i];
    sM[128 + i] = hmD<N, Q>[i];
    sM[192 + i] = hmDt<N, Q>[i];
  }
  if (t < 8) sW[t] = hmW<N, Q>[t];
  if (t < 16) sDVE[t] = hmDVE<N, Q>[t];
  if (lane == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&mbar[2], 6);
    fence_proxy_async();
  }
  __syncthreads();     // the only CTA-wide barrier: tables + barrier init
  const int ar = lane >> 2, ac = lane & 3;
  const AFrag AV = {sM[ar * 8 + ac], sM[ar * 8 + 4 + ac]};
  const AFrag AVt = {sM[64 + ar * 8 + ac], sM[64 + ar * 8 + 4 + ac]};
  const AFrag AD = {sM[128 + ar * 8 + ac], sM[128 + ar * 8 + 4 + ac]};
  const AFrag ADt = {sM[192 + ar * 8 + ac], sM[192 + ar * 8 + 4 + ac]};

  const int gw = blockIdx.x * W + warp, nw = gridDim.x * W;
  auto issue_own = [&](int iel, int st) {     // lane 0
    const FaceRec* rsrc = P.recs + cd[CD_REC_OFF] + (int64_t)iel * 6;
    bulk_g2s(sl + H::O_REC + st * 96, rsrc, 6 * sizeof(FaceRec), &mbar[st]);
    unsigned nb;
    soff[st] = bulk_block(sl + H::O_X + st * H::BLK, x + P.dof_off[elist[iel]], N3, &mbar[st], &nb);
    mbar_expect_tx(&mbar[st], 6 * sizeof(FaceRec) + nb);
    cp_async_commit();
  };
  if (lane == 0 && gw < count) issue_own(gw, 0);

  int kk = 0;
  for (int iel = gw; iel < count; iel += nw, ++kk) {
    const int st = kk & 1;
    const bool more = iel + nw < count;
    if (lane == 0) {
      if (more) issue_own(iel + nw, st ^ 1);
      if (more) cp_async_wait<1>(); else cp_async_wait<0>();
    }
    mbar_wait(&mbar[st], (kk >> 1) & 1);
    __syncwarp();
    const FaceRec* srec = reinterpret_cast<const FaceRec*>(sl + H::O_REC + st * 96);
    const double* X = sl + H::O_X + st * H::BLK + soff[st];
    // element metric (prefetched into registers; used after the faces)
    const double* eg = egeo + (int64_t)iel * estride;
    const double J = __ldg(eg), K0 = __ldg(eg + 1), K1 = __ldg(eg + 2), K2 = __ldg(eg + 3);
    const double K3 = __ldg(eg + 4), K4 = __ldg(eg + 5), K5 = __ldg(eg + 6);
    const int64_t dof0 = P.dof_off[elist[iel]];
    if (lane < 6) {
      const FaceRec& r = srec[lane];
      const bool fast = r.type == FT_DIRECT && (r.flags & F_FAST_HEX);
      sk[lane] = (P.debug & 1) ? 0 : (fast ? 1 : ((r.type == FT_BOUNDARY && !(r.flags & F_SELF_PW)) ? 2 : 0));
    }
    if (lane >= 1 && lane <= 6) {     // one neighbour block per lane
      const int f = lane - 1;
      const FaceRec& r = srec[f];
      unsigned nb = 0;
      if (r.type == FT_DIRECT && (r.flags & F_FAST_HEX) && !(P.debug & 1))
        soff[2 + f] = bulk_block(NB + f * H::FBLK, x + r.nbr_dof, N3, &mbar[2], &nb);
      mbar_expect_tx(&mbar[2], nb);
      cp_async_commit();
    }

    // ---- BwdTrans: axis 2 from the raw block, then axes 1 and 0
    {
      const int kq = lane & 3, n = lane >> 2, r = lane >> 2, c = 2 * (lane & 3);
      double b0[8], b1[8], c0[8], c1[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const bool okl = a < N && n < N;
        b0[a] = (okl && kq < N) ? X[(a * N + n) * N + kq] : 0.0;
        b1[a] = (okl && 4 + kq < N) ? X[(a * N + n) * N + 4 + kq] : 0.0;
        c0[a] = 0.0;
        c1[a] = 0.0;
      }
#pragma unroll
      for (int a = 0; a < 8; ++a) dmma(c0[a], c1[a], AV.a0, b0[a]);
#pragma unroll
      for (int a = 0; a < 8; ++a) dmma(c0[a], c1[a], AV.a1, b1[a]);
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        G0[widx<2>(r, a, c)] = c0[a];
        G0[widx<2>(r, a, c + 1)] = c1[a];
      }
      __syncwarp();
    }
    w_axis<1, false>(G0, G1, AV, lane);
    w_axis<0, false>(G1, U, AV, lane);
    // ---- PhysDeriv
    w_axis<0, false>(U, G0, AD, lane);
    w_axis<1, false>(U, G1, AD, lane);
    w_axis<2, false>(U, G2, AD, lane);
    if (lane >= 1 && lane <= 6) cp_async_wait<0>();
    mbar_wait(&mbar[2], kk & 1);
    __syncwarp();

    // ---- neighbour planes (boundary mode, normal derivative) into each face's slot
#pragma unroll 1
    for (int f = 0; f < 6; ++f) {
      if (sk[f] != 1) continue;
      double* slot = NB + f * H::FBLK;
      const int fo = srec[f].nbr_face, ao = fo >> 1;
      const int b0 = ao == 0 ? 1 : 0, b1 = ao == 2 ? 1 : 2;
      const int sa = hex_stride(ao, N);
      const double* dv = sDVE + ((fo & 1) ? 8 : 0);
      double pu[2], pd[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e2 = lane + 32 * h, i0 = e2 >> 3, i1 = e2 & 7;
        pu[h] = 0.0;
        pd[h] = 0.0;
        if (i0 < N && i1 < N) {
          const double* cc = slot + soff[2 + f] + i0 * hex_stride(b0, N) + i1 * hex_stride(b1, N);
#pragma unroll
          for (int i = 0; i < N; ++i) pd[h] = fma(dv[i], cc[i * sa], pd[h]);
          pu[h] = cc[(fo & 1) ? (N - 1) * sa : 0];
        }
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e2 = lane + 32 * h, i0 = e2 >> 3, i1 = e2 & 7;
        slot[i0 * 12 + i1] = pu[h];
        slot[96 + i0 * 12 + i1] = pd[h];
      }
    }
    __syncwarp();
    // ---- V P V^T for the planes, 3 at a time through TT
    {
      const int kq = lane & 3, n = lane >> 2, r = lane >> 2, c = 2 * (lane & 3);
#pragma unroll 1
      for (int base = 0; base < 12; base += 3) {
        double c0[3], c1[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int fp = base + q, f = fp >> 1;
          c0[q] = 0.0;
          c1[q] = 0.0;
          if (sk[f] != 1) continue;
          const double* pl = NB + f * H::FBLK + (fp & 1) * 96;
          const double bb0 = pl[kq * 12 + n], bb1 = pl[(4 + kq) * 12 + n];
          dmma(c0[q], c1[q], AV.a0, bb0);
          dmma(c0[q], c1[q], AV.a1, bb1);
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          TT[q * 96 + r * 12 + c] = c0[q];
          TT[q * 96 + r * 12 + c + 1] = c1[q];
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int fp = base + q, f = fp >> 1;
          if (sk[f] != 1) continue;
          double d0 = 0.0, d1 = 0.0;
          const double* tt = TT + q * 96;
          dmma(d0, d1, AV.a0, tt[n * 12 + kq]);
          dmma(d0, d1, AV.a1, tt[n * 12 + 4 + kq]);
          double* pl = NB + f * H::FBLK + (fp & 1) * 96;
          pl[c * 12 + r] = d0;            // U2[p0 = c][p1 = r]
          pl[(c + 1) * 12 + r] = d1;
        }
        __syncwarp();
      }
    }
    // ---- flux at the face points: (fv, fd) into each face's slot
#pragma unroll 1
    for (int f = 0; f < 6; ++f) {
      const int kind = sk[f];
      if (kind == 0) continue;
      const FaceRec& rr = srec[f];
      const double* pl = NB + f * H::FBLK;
      double* fvd = NB + f * H::FBLK + 192;
      const int a = f >> 1, fix = (f & 1) ? Q - 1 : 0;
      const double gsa = rr.gs[0], gsb = rr.gs[1], gsc = rr.gs[2];
      const double goa = kind == 1 ? rr.go[rr.nbr_face >> 1] : 0.0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = lane + 32 * h, p0 = p >> 3, p1 = p & 7;
        if (p0 >= Q || p1 >= Q) continue;
        const int v = a == 0 ? wsw(fix, p0, p1) : (a == 1 ? wsw(p0, fix, p1) : wsw(p0, p1, fix));
        const double swj = rr.sJ * sW[p0] * sW[p1];
        const double us = U[v];
        const double gs = gsa * G0[v] + gsb * G1[v] + gsc * G2[v];
        double jump, avg;
        if (kind == 2) {
          jump = 2.0 * us;
          avg = gs;
        } else {
          jump = us - pl[p0 * 12 + p1];
          avg = 0.5 * (gs - goa * pl[96 + p0 * 12 + p1]);
        }
        fvd[p] = (rr.tau * jump - avg) * swj;
        fvd[64 + p] = -0.5 * jump * swj;
      }
    }
    __syncwarp();
    // ---- volume metric in place: U -> lam jw u, G -> jw G G^T du
#pragma unroll 4
    for (int s = 0; s < 16; ++s) {
      const int pidx = lane + 32 * s, i = pidx >> 6, j = (pidx >> 3) & 7, k = pidx & 7;
      const int v = wsw(i, j, k);
      const double jw = J * sW[i] * sW[j] * sW[k];
      const double g0 = G0[v], g1 = G1[v], g2 = G2[v];
      U[v] = lam * jw * U[v];
      G0[v] = jw * (K0 * g0 + K1 * g1 + K2 * g2);
      G1[v] = jw * (K1 * g0 + K3 * g1 + K4 * g2);
      G2[v] = jw * (K2 * g0 + K4 * g1 + K5 * g2);
    }
    __syncwarp();
    // ---- lift: fold the face fluxes (one face at a time: faces share edge points)
#pragma unroll 1
    for (int f = 0; f < 6; ++f) {
      if (sk[f] == 0) continue;
      const double* fvd = NB + f * H::FBLK + 192;
      const int a = f >> 1, fix = (f & 1) ? Q - 1 : 0;
      const double gsa = srec[f].gs[0], gsb = srec[f].gs[1], gsc = srec[f].gs[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = lane + 32 * h, p0 = p >> 3, p1 = p & 7;
        if (p0 >= Q || p1 >= Q) continue;
        const int v = a == 0 ? wsw(fix, p0, p1) : (a == 1 ? wsw(p0, fix, p1) : wsw(p0, p1, fix));
        const double fv = fvd[p], fd = fvd[64 + p];
        U[v] += fv;
        G0[v] = fma(fd, gsa, G0[v]);
        G1[v] = fma(fd, gsb, G1[v]);
        G2[v] = fma(fd, gsc, G2[v]);
      }
      __syncwarp();
    }
    // ---- R = P0 + D^T along each axis, then IProduct
    w_axis<0, true>(G0, U, ADt, lane);
    w_axis<1, true>(G1, U, ADt, lane);
    w_axis<2, true>(G2, U, ADt, lane);
    w_axis<0, false>(U, G0, AVt, lane);
    w_axis<1, false>(G0, G1, AVt, lane);
    w_axis<2, false>(G1, G2, AVt, lane);
    for (int i = lane; i < N3; i += 32) {
      const int a = i / (N * N), rm = i - a * N * N, b = rm / N, c = rm - b * N;
      y[dof0 + i] = G2[wsw(a, b, c)];
    }
    fence_proxy_async();
    __syncwarp();
  }
}

}  // namespace sipg
