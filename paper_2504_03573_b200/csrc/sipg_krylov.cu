// GPU-resident conjugate gradient around the SIP apply.
//
// Restates the reference's unpreconditioned CG (pkg/src/dgsipg/krylov.py:39-81) with the
// vectors resident in HBM: per iteration one sipg_apply, one fused dot (p.Ap), one fused
// update (x += a p, r -= a Ap, partial r.r) and one direction update (p = r + b p).  The
// scalars (rr, p.Ap, alpha, beta) never leave the device except the two the reference's
// control flow tests (p.Ap and the new r.r), read back through a pinned 32-byte buffer
// once per iteration.  Reductions use a fixed grid and a fixed combine order, so a solve
// is bitwise reproducible run to run.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <string>
#include "../../include/sipg.h"

extern void sipg_set_error(const std::string& s);   // sipg_capi.cu

namespace {

constexpr int RB = 592;    // reduction CTAs (4 per SM on 148 SMs), fixed for determinism
constexpr int RT = 256;

// scalar slots (device): 0/1 rr by iteration parity, 2 pap, 3 spare, 4 true residual^2
enum { S_RR0 = 0, S_RR1 = 1, S_PAP = 2, S_TRUE = 4, S_N = 8 };

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = 0.0;
  if (w == 0) {
    v = l < (RT / 32) ? sh[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  }
  return v;   // valid in thread 0
}

// part[b] = sum over the block's grid-stride slice of a[i] * b[i]
__global__ void __launch_bounds__(RT) k_dot(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                                            double* __restrict__ part) {
  __shared__ double sh[RT / 32];
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < n; i += (int64_t)RB * RT) v = fma(a[i], b[i], v);
  v = block_sum(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}

// part[b] = sum (b[i] - c[i])^2   (true residual of the final check)
__global__ void __launch_bounds__(RT) k_resid(const double* __restrict__ b, const double* __restrict__ c, int64_t n,
                                              double* __restrict__ part) {
  __shared__ double sh[RT / 32];
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < n; i += (int64_t)RB * RT) {
    const double d = b[i] - c[i];
    v = fma(d, d, v);
  }
  v = block_sum(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}

// s[slot] = sum of the RB partials (fixed order), optionally copied to a pinned host word
__global__ void __launch_bounds__(RT) k_final(const double* __restrict__ part, double* s, int slot) {
  __shared__ double sh[RT / 32];
  double v = 0.0;
  for (int i = threadIdx.x; i < RB; i += RT) v += part[i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) s[slot] = v;
}

// alpha = rr / pap (skipped when pap <= 0 or not finite: the reference returns x untouched);
// x += alpha p, r -= alpha Ap, part = partial sums of the new r.r
__global__ void __launch_bounds__(RT) k_cg_xr(double* __restrict__ x, double* __restrict__ r,
                                              const double* __restrict__ p, const double* __restrict__ ap,
                                              int64_t n, const double* s, int rr_slot, double* __restrict__ part) {
  __shared__ double sh[RT / 32];
  const double pap = s[S_PAP];
  const bool ok = pap > 0.0 && isfinite(pap);
  const double alpha = ok ? s[rr_slot] / pap : 0.0;
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < n; i += (int64_t)RB * RT) {
    double ri = r[i];
    if (ok) {
      x[i] = fma(alpha, p[i], x[i]);
      ri = fma(-alpha, ap[i], ri);
      r[i] = ri;
    }
    v = fma(ri, ri, v);
  }
  v = block_sum(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}

// p = r + beta p with beta = rr_new / rr_old
__global__ void __launch_bounds__(RT) k_cg_p(double* __restrict__ p, const double* __restrict__ r, int64_t n,
                                             const double* s, int old_slot, int new_slot) {
  const double beta = s[new_slot] / s[old_slot];
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < n; i += (int64_t)RB * RT) p[i] = fma(beta, p[i], r[i]);
}

__global__ void k_copy(double* __restrict__ d, const double* __restrict__ a, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < n; i += (int64_t)RB * RT) d[i] = a[i];
}

struct Ctx {
  cudaStream_t s;
  double* part;
  double* sc;         // device scalars
  double* host;       // pinned: host mirror of up to 8 scalars
};

int dot_into(Ctx& c, const double* a, const double* b, int64_t n, int slot) {
  k_dot<<<RB, RT, 0, c.s>>>(a, b, n, c.part);
  k_final<<<1, RT, 0, c.s>>>(c.part, c.sc, slot);
  return cudaGetLastError() == cudaSuccess ? 0 : SIPG_ERR_CUDA;
}

int fetch(Ctx& c) {
  if (cudaMemcpyAsync(c.host, c.sc, sizeof(double) * S_N, cudaMemcpyDeviceToHost, c.s) != cudaSuccess ||
      cudaStreamSynchronize(c.s) != cudaSuccess)
    return SIPG_ERR_CUDA;
  return 0;
}

}  // namespace

extern "C" int sipg__workspace(sipg_plan* p, size_t bytes, void** dev, double** host);   // sipg_capi.cu

extern "C" int sipg_cg(sipg_plan* plan, const double* b, double* x, int64_t n, double tol, int64_t maxiter,
                       sipg_solve_report* rep, void* stream) {
  if (!plan || !b || !x || !rep || n <= 0 || n != sipg_plan_n_dofs(plan)) {
    sipg_set_error("sipg_cg: bad argument (null pointer or n != plan n_dofs)");
    return SIPG_ERR_ARG;
  }
  memset(rep, 0, sizeof(*rep));
  Ctx c{(cudaStream_t)stream, nullptr, nullptr, nullptr};
  double *r = nullptr, *p = nullptr, *ap = nullptr;
  int rc = 0;
  auto cleanup = [&]() {};   // the workspace belongs to the plan (reused by the next solve)
  {
    // r, p, Ap, reduction partials, device scalars: one cached block (sipg__workspace)
    const size_t nn = ((size_t)n + 31) & ~(size_t)31;   // 256-byte aligned vectors
    void* ws = nullptr;
    if (sipg__workspace(plan, sizeof(double) * (3 * nn + RB + S_N + 8), &ws, &c.host) != 0) {
      sipg_set_error("sipg_cg: device allocation failed");
      return SIPG_ERR_CUDA;
    }
    r = static_cast<double*>(ws);
    p = r + nn;
    ap = p + nn;
    c.part = ap + nn;
    c.sc = c.part + RB;
  }
  // nb = ||b||; x = 0
  cudaMemsetAsync(x, 0, sizeof(double) * n, c.s);
  cudaMemsetAsync(c.sc, 0, sizeof(double) * S_N, c.s);
  if ((rc = dot_into(c, b, b, n, S_RR0)) || (rc = fetch(c))) {
    cleanup();
    sipg_set_error("sipg_cg: CUDA failure");
    return rc;
  }
  const double nb = sqrt(c.host[S_RR0]);
  if (nb == 0.0) {
    rep->converged = 1;
    cleanup();
    return 0;
  }
  if (maxiter <= 0) maxiter = 10 * n > 200 ? 10 * n : 200;
  // r = b, p = r
  k_copy<<<RB, RT, 0, c.s>>>(r, b, n);
  k_copy<<<RB, RT, 0, c.s>>>(p, b, n);
  double rr = c.host[S_RR0];
  double best = sqrt(rr) / nb;
  int stall = 0;
  for (int64_t it = 1; it <= maxiter; ++it) {
    const int old_slot = (it & 1) ? S_RR0 : S_RR1, new_slot = (it & 1) ? S_RR1 : S_RR0;
    if ((rc = sipg_apply(plan, p, ap, stream)) != 0) break;
    if ((rc = dot_into(c, p, ap, n, S_PAP)) != 0) break;
    k_cg_xr<<<RB, RT, 0, c.s>>>(x, r, p, ap, n, c.sc, old_slot, c.part);
    k_final<<<1, RT, 0, c.s>>>(c.part, c.sc, new_slot);
    if ((rc = fetch(c)) != 0) break;
    const double pap = c.host[S_PAP];
    if (!(pap > 0.0) || !isfinite(pap)) {
      *rep = {0, 1, it, sqrt(rr > 0.0 ? rr : 0.0) / nb};
      cleanup();
      return 0;
    }
    const double rr_new = c.host[new_slot];
    const double rel = sqrt(rr_new) / nb;
    if (rel <= tol) {
      // verify the true residual (the recurrence drifts on a non-symmetric operator)
      if ((rc = sipg_apply(plan, x, ap, stream)) != 0) break;
      k_resid<<<RB, RT, 0, c.s>>>(b, ap, n, c.part);
      k_final<<<1, RT, 0, c.s>>>(c.part, c.sc, S_TRUE);
      if ((rc = fetch(c)) != 0) break;
      const double true_rel = sqrt(c.host[S_TRUE]) / nb;
      if (true_rel <= 10.0 * tol)
        *rep = {1, 0, it, true_rel};
      else
        *rep = {0, 2, it, true_rel};
      cleanup();
      return 0;
    }
    if (rel < 0.999 * best) {
      best = rel;
      stall = 0;
    } else if (++stall >= 250) {
      *rep = {0, 3, it, rel};
      cleanup();
      return 0;
    }
    k_cg_p<<<RB, RT, 0, c.s>>>(p, r, n, c.sc, old_slot, new_slot);
    rr = rr_new;
  }
  if (rc) {
    cleanup();
    sipg_set_error("sipg_cg: CUDA failure during the solve");
    return rc;
  }
  *rep = {0, 4, maxiter, sqrt(rr) / nb};
  cleanup();
  return 0;
}
