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
#include <vector>
#include <algorithm>
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

extern "C" int sipg__workspace(sipg_plan* p, size_t bytes, size_t host_doubles, void** dev,
                               double** host);   // sipg_capi.cu

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
    if (sipg__workspace(plan, sizeof(double) * (3 * nn + RB + S_N + 8), 64, &ws, &c.host) != 0) {
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
  if (maxiter < 0) maxiter = 10 * n > 200 ? 10 * n : 200;   // reference: maxiter=None
  if (maxiter == 0) {                                          // no iteration: x = 0, r = b
    *rep = {0, 4, 0, 1.0};
    return 0;
  }
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

// ---------------------------------------------------------------------------------------------
// GPU-resident restarted GMRES (the reference's interface and stopping rules,
// pkg/src/dgsipg/krylov.py:84-141).  Design for the device rather than a restatement of the
// reference's modified Gram-Schmidt loop: the Arnoldi step orthogonalises the new vector against the
// whole basis with classical Gram-Schmidt applied twice (CGS2 — as stable as MGS in practice, and
// every pass is one batched multi-dot kernel plus one fused update kernel instead of k + 1 dependent
// dot / axpy pairs), and the k + 2 scalars of an iteration (both projection passes and the new norm)
// come back in one read: one host synchronisation per Arnoldi step.  The (m + 1) x m Hessenberg
// least-squares problem is tiny and stays on the host (Givens rotations).  Fixed grids and fixed
// combine orders keep a solve bitwise reproducible.
namespace {

constexpr int MB = 8;   // basis vectors per multi-dot pass

// part[j * RB + b] = block b's partial of V_j . w for j in [j0, j0 + nj), nj <= MB
__global__ void __launch_bounds__(RT) k_mdot(const double* __restrict__ V, int64_t ld, int j0, int nj,
                                             const double* __restrict__ w, int64_t n, double* __restrict__ part) {
  __shared__ double sh[RT / 32];
  double acc[MB];
#pragma unroll
  for (int j = 0; j < MB; ++j) acc[j] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < n; i += (int64_t)RB * RT) {
    const double wi = w[i];
#pragma unroll
    for (int j = 0; j < MB; ++j)
      if (j < nj) acc[j] = fma(V[(int64_t)(j0 + j) * ld + i], wi, acc[j]);
  }
#pragma unroll
  for (int j = 0; j < MB; ++j) {
    if (j >= nj) break;
    const double v = block_sum(acc[j], sh);
    if (threadIdx.x == 0) part[(int64_t)(j0 + j) * RB + blockIdx.x] = v;
    __syncthreads();
  }
}

// out[j] = sum of the RB partials of row j (one block per j, fixed order)
__global__ void __launch_bounds__(RT) k_final_rows(const double* __restrict__ part, double* __restrict__ out) {
  __shared__ double sh[RT / 32];
  double v = 0.0;
  for (int i = threadIdx.x; i < RB; i += RT) v += part[(int64_t)blockIdx.x * RB + i];
  v = block_sum(v, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = v;
}

// w -= sum_{j <= k} h[j] V_j ; part = partials of the new w.w
__global__ void __launch_bounds__(RT) k_gs_update(const double* __restrict__ V, int64_t ld, int k1,
                                                  const double* __restrict__ h, double* __restrict__ w, int64_t n,
                                                  double* __restrict__ part) {
  __shared__ double sh[RT / 32];
  __shared__ double hs[256];
  for (int j = threadIdx.x; j < k1; j += RT) hs[j] = h[j];
  __syncthreads();
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < n; i += (int64_t)RB * RT) {
    double wi = w[i];
    for (int j = 0; j < k1; ++j) wi = fma(-hs[j], V[(int64_t)j * ld + i], wi);
    w[i] = wi;
    v = fma(wi, wi, v);
  }
  v = block_sum(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}

__global__ void k_scale(double* __restrict__ d, const double* __restrict__ a, double s, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < n; i += (int64_t)RB * RT) d[i] = a[i] * s;
}

// x += sum_j y[j] V_j
__global__ void __launch_bounds__(RT) k_combine(double* __restrict__ x, const double* __restrict__ V, int64_t ld,
                                                const double* __restrict__ y, int k1, int64_t n) {
  __shared__ double ys[256];
  for (int j = threadIdx.x; j < k1; j += RT) ys[j] = y[j];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < n; i += (int64_t)RB * RT) {
    double xi = x[i];
    for (int j = 0; j < k1; ++j) xi = fma(ys[j], V[(int64_t)j * ld + i], xi);
    x[i] = xi;
  }
}

// r = b - Ar, part = partials of r.r
__global__ void __launch_bounds__(RT) k_resvec(double* __restrict__ r, const double* __restrict__ b, int64_t n,
                                               double* __restrict__ part) {
  __shared__ double sh[RT / 32];
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * RT + threadIdx.x; i < n; i += (int64_t)RB * RT) {
    const double d = b[i] - r[i];
    r[i] = d;
    v = fma(d, d, v);
  }
  v = block_sum(v, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = v;
}

// rows [0, k1) of V against w -> dst (device), all in one stream
void multidot(cudaStream_t s, const double* V, int64_t ld, int k1, const double* w, int64_t n, double* part,
              double* dst) {
  for (int j0 = 0; j0 < k1; j0 += MB) k_mdot<<<RB, RT, 0, s>>>(V, ld, j0, k1 - j0 < MB ? k1 - j0 : MB, w, n, part);
  k_final_rows<<<k1, RT, 0, s>>>(part, dst);
}

}  // namespace

extern "C" int sipg_gmres(sipg_plan* plan, const double* b, double* x, int64_t n, double tol, int32_t restart,
                          int64_t maxiter, sipg_solve_report* rep, void* stream) {
  if (!plan || !b || !x || !rep || n <= 0 || n != sipg_plan_n_dofs(plan)) {
    sipg_set_error("sipg_gmres: bad argument (null pointer or n != plan n_dofs)");
    return SIPG_ERR_ARG;
  }
  memset(rep, 0, sizeof(*rep));
  cudaStream_t s = (cudaStream_t)stream;
  if (maxiter < 0) maxiter = 20 * n > 400 ? 20 * n : 400;   // reference: maxiter=None
  int64_t m_cap = restart < 1 ? 1 : restart;
  if (m_cap > n) m_cap = n;
  if (m_cap > 255) {
    sipg_set_error("sipg_gmres: restart > 255 is not supported by the device solver");
    return SIPG_ERR_ARG;
  }
  const int M = (int)m_cap;
  const size_t nn = ((size_t)n + 31) & ~(size_t)31;
  // workspace: basis V (M + 1 vectors), w, partials (RB per row, M + 2 rows), device scalars
  const size_t nsc = 2 * (size_t)(M + 2) + 8;
  void* ws = nullptr;
  double* host = nullptr;
  if (sipg__workspace(plan, sizeof(double) * ((M + 2) * nn + (size_t)RB * (M + 2) + nsc), nsc, &ws, &host) != 0) {
    sipg_set_error("sipg_gmres: device allocation failed (basis of restart + 1 vectors)");
    return SIPG_ERR_CUDA;
  }
  double* V = static_cast<double*>(ws);
  double* w = V + (size_t)(M + 1) * nn;
  double* part = w + nn;
  double* sc = part + (size_t)RB * (M + 2);   // [0, M+1) pass-1 h, [M+1, 2M+2) pass-2 h, then norms
  double* h1 = sc;
  double* h2 = sc + (M + 1);
  double* nrm = sc + 2 * (M + 1);
  auto fetch_n = [&](int cnt) -> int {
    if (cudaMemcpyAsync(host, sc, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return SIPG_ERR_CUDA;
    return 0;
  };
  auto fail_cuda = [&](const char* what) {
    cudaStreamSynchronize(s);
    sipg_set_error(std::string("sipg_gmres: ") + what);
    return SIPG_ERR_CUDA;
  };
  // ||b||, x = 0
  cudaMemsetAsync(x, 0, sizeof(double) * n, s);
  k_dot<<<RB, RT, 0, s>>>(b, b, n, part);
  k_final<<<1, RT, 0, s>>>(part, nrm, 0);
  if (cudaGetLastError() != cudaSuccess || fetch_n((int)nsc)) return fail_cuda("CUDA failure");
  const double nb = sqrt(host[2 * (M + 1)]);
  if (nb == 0.0) {
    *rep = {1, 0, 0, 0.0};
    return 0;
  }
  // host Hessenberg (column-major (M + 1) x M), Givens rotations, rhs g
  std::vector<double> H((size_t)(M + 1) * M), cs(M), sn(M), g(M + 1), y(M);
  auto Hc = [&](int i, int k) -> double& { return H[(size_t)k * (M + 1) + i]; };
  int64_t total = 0;
  // r = b - A x (x = 0 on the first cycle: r = b) into V_0, beta = ||r||
  auto residual = [&](double* r_out, double& rel) -> int {
    int rc = sipg_apply(plan, x, r_out, stream);
    if (rc) return rc;
    k_resvec<<<RB, RT, 0, s>>>(r_out, b, n, part);
    k_final<<<1, RT, 0, s>>>(part, nrm, 0);
    if (cudaGetLastError() != cudaSuccess || fetch_n((int)nsc)) return SIPG_ERR_CUDA;
    rel = sqrt(host[2 * (M + 1)]) / nb;
    return 0;
  };
  while (total < maxiter) {
    double rel = 0.0;
    int rc = residual(V, rel);
    if (rc) return rc == SIPG_ERR_CUDA ? fail_cuda("CUDA failure (residual)") : rc;
    if (rel <= tol) {
      *rep = {1, 0, total, rel};
      return 0;
    }
    const double beta = rel * nb;
    const int m = (int)((maxiter - total) < M ? (maxiter - total) : M);
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    k_scale<<<RB, RT, 0, s>>>(V, V, 1.0 / beta, n);
    int kd = 0;
    for (int k = 0; k < m; ++k) {
      double* vk1 = V + (size_t)(k + 1) * nn;
      if ((rc = sipg_apply(plan, V + (size_t)k * nn, w, stream)) != 0) return rc;
      // CGS2: two projection passes against V_0..V_k, then the norm of what is left
      multidot(s, V, (int64_t)nn, k + 1, w, n, part, h1);
      k_gs_update<<<RB, RT, 0, s>>>(V, (int64_t)nn, k + 1, h1, w, n, part);
      multidot(s, V, (int64_t)nn, k + 1, w, n, part, h2);
      k_gs_update<<<RB, RT, 0, s>>>(V, (int64_t)nn, k + 1, h2, w, n, part);
      k_final<<<1, RT, 0, s>>>(part, nrm, 0);
      if (cudaGetLastError() != cudaSuccess || fetch_n((int)nsc)) return fail_cuda("CUDA failure (Arnoldi)");
      for (int i = 0; i <= k; ++i) Hc(i, k) = host[i] + host[(M + 1) + i];
      const double hk1 = sqrt(host[2 * (M + 1)]);
      Hc(k + 1, k) = hk1;
      // the next basis vector (left zero on breakdown, as the reference's basis row stays zero)
      if (hk1 > 1e-300)
        k_scale<<<RB, RT, 0, s>>>(vk1, w, 1.0 / hk1, n);
      else
        cudaMemsetAsync(vk1, 0, sizeof(double) * n, s);
      // previous rotations on the new column, then this column's rotation
      for (int i = 0; i < k; ++i) {
        const double a = Hc(i, k), c2 = Hc(i + 1, k);
        Hc(i, k) = cs[i] * a + sn[i] * c2;
        Hc(i + 1, k) = -sn[i] * a + cs[i] * c2;
      }
      const double den = hypot(Hc(k, k), Hc(k + 1, k));
      cs[k] = Hc(k, k) / den;
      sn[k] = Hc(k + 1, k) / den;
      Hc(k, k) = den;
      Hc(k + 1, k) = 0.0;
      g[k + 1] = -sn[k] * g[k];
      g[k] = cs[k] * g[k];
      kd = k + 1;
      ++total;
      if (fabs(g[k + 1]) / nb <= tol) break;
    }
    // back substitution on the rotated (upper triangular) Hessenberg, then x += V y
    for (int i = kd - 1; i >= 0; --i) {
      double v = g[i];
      for (int j = i + 1; j < kd; ++j) v -= Hc(i, j) * y[j];
      y[i] = v / Hc(i, i);
    }
    if (kd > 0) {
      for (int i = 0; i < kd; ++i) host[i] = y[i];
      if (cudaMemcpyAsync(sc, host, sizeof(double) * kd, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return fail_cuda("CUDA failure (update)");
      k_combine<<<RB, RT, 0, s>>>(x, V, (int64_t)nn, sc, kd, n);
    }
    if ((rc = residual(w, rel)) != 0) return rc == SIPG_ERR_CUDA ? fail_cuda("CUDA failure (residual)") : rc;
    if (rel <= tol) {
      *rep = {1, 0, total, rel};
      return 0;
    }
  }
  double rel = 0.0;
  const int rc = residual(w, rel);
  if (rc) return rc == SIPG_ERR_CUDA ? fail_cuda("CUDA failure (residual)") : rc;
  *rep = {0, 4, total, rel};
  return 0;
}
