"""Krylov solvers around the GPU apply.

Mirrors the reference's `dgsipg.krylov` interface (pkg/src/dgsipg/krylov.py):
`cg(apply_op, b, tol=1e-9, maxiter=None) -> (x, SolveReport)` and
`gmres(apply_op, b, tol=1e-9, restart=50, maxiter=None) -> (x, SolveReport)`,
with the same stopping rules and report fields.  `apply_op` must be this
package's `HelmholtzOperator` (the vectors stay in HBM; there is no CPU path):

* cg runs entirely in libsipg.so (`sipg_cg`, csrc/sipg_krylov.cu): one apply,
  one fused dot and one fused update per iteration, two scalars read back.
* probe_dense / asymmetry_norm / block_sparsity (reference krylov.py:144-183,
  the paper's symmetry study): the columns are sm_100a applies of device-resident unit vectors
  written straight into a device matrix; the two diagnostics are host post-processing of that
  matrix, as in the reference.
* gmres runs in libsipg.so too (`sipg_gmres`): the Arnoldi basis stays in HBM, each step
  is one apply, two batched Gram-Schmidt passes (multi-dot + fused update kernels) and one
  read of k + 2 scalars; the tiny Hessenberg least-squares problem is solved on the host.

`b` may be a numpy array (copied in, x copied out as numpy, like the reference)
or a CUDA float64 tensor (x returned as a CUDA tensor).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["SolveReport", "cg", "gmres", "REASONS", "probe_dense", "asymmetry_norm", "block_sparsity",
           "DEFAULT_PROBE_LIMIT"]

DEFAULT_PROBE_LIMIT = 20000     # reference krylov.py:24

REASONS = {0: "", 1: "indefinite direction", 2: "residual drift", 3: "stagnation", 4: "maxiter"}


@dataclass
class SolveReport:
    """Same fields and text as the reference's SolveReport (krylov.py:27-37)."""
    converged: bool
    iterations: int
    residual: float
    reason: str = ""

    def __str__(self) -> str:
        state = "converged" if self.converged else f"FAILED ({self.reason})"
        return f"{state} in {self.iterations} iterations, relres {self.residual:.3e}"


def _device_rhs(op, b):
    import torch
    from .sipg import HelmholtzOperator, _is_cuda_tensor
    if not isinstance(op, HelmholtzOperator):
        raise TypeError("the GPU solvers need a paper_2504_03573_b200 HelmholtzOperator as apply_op")
    if _is_cuda_tensor(b):
        if b.dtype != torch.float64 or b.shape != (op.n_dofs,):
            raise ValueError(f"expected a float64 vector of length {op.n_dofs}")
        return b.contiguous(), True
    b = np.ascontiguousarray(np.asarray(b, dtype=float))
    if b.shape != (op.n_dofs,):
        raise ValueError(f"expected a vector of length {op.n_dofs}")
    return torch.from_numpy(b).cuda(), False


def cg(apply_op, b, tol: float = 1e-9, maxiter: int | None = None):
    """Unpreconditioned CG on the GPU (reference krylov.py:39-81); returns (x, SolveReport)."""
    import torch
    bd, on_dev = _device_rhs(apply_op, b)
    x = torch.empty_like(bd)
    stream = torch.cuda.current_stream()
    rep = apply_op.native.cg(bd.data_ptr(), x.data_ptr(), int(bd.numel()), float(tol),
                             int(maxiter) if maxiter is not None else -1, stream.cuda_stream)
    out = SolveReport(bool(rep.converged), int(rep.iterations), float(rep.residual), REASONS[int(rep.reason)])
    return (x if on_dev else x.cpu().numpy()), out


def gmres(apply_op, b, tol: float = 1e-9, restart: int = 50, maxiter: int | None = None):
    """Restarted GMRES on the GPU (reference interface krylov.py:84-141; device solver sipg_gmres in
    csrc/sipg_krylov.cu: basis in HBM, twice-applied classical Gram-Schmidt as batched multi-dot
    kernels, one host read per Arnoldi step); returns (x, SolveReport)."""
    import torch
    bd, on_dev = _device_rhs(apply_op, b)
    x = torch.empty_like(bd)
    stream = torch.cuda.current_stream()
    rep = apply_op.native.gmres(bd.data_ptr(), x.data_ptr(), int(bd.numel()), float(tol), int(restart),
                                int(maxiter) if maxiter is not None else -1, stream.cuda_stream)
    out = SolveReport(bool(rep.converged), int(rep.iterations), float(rep.residual), REASONS[int(rep.reason)])
    return (x if on_dev else x.cpu().numpy()), out


def probe_dense(apply_op, n: int, limit: int = DEFAULT_PROBE_LIMIT) -> np.ndarray:
    """Assemble the operator column by column from unit-vector applications (reference
    krylov.py:144-156): every column is one device apply of e_j; returns a numpy (n, n) matrix."""
    import torch
    if n > limit:
        raise ValueError(f"probe size {n} exceeds the limit {limit}; use a smaller mesh")
    _device_rhs(apply_op, np.zeros(n))          # type / length checks of the reference call
    e = torch.zeros(n, dtype=torch.float64, device="cuda")
    at = torch.empty((n, n), dtype=torch.float64, device="cuda")   # row j = column j of A
    stream = torch.cuda.current_stream().cuda_stream
    for j in range(n):
        e[j] = 1.0
        apply_op.apply_into(e.data_ptr(), at[j].data_ptr(), stream)
        e[j] = 0.0
    return np.ascontiguousarray(at.cpu().numpy().T)


def asymmetry_norm(m) -> float:
    """||M - M^T||_1 / ||M||_1 with the max-absolute-column-sum norm (reference krylov.py:159-164)."""
    m = np.asarray(m)
    num = np.abs(m - m.T).sum(axis=0).max()
    den = np.abs(m).sum(axis=0).max()
    return float(num / den) if den else 0.0


def block_sparsity(m, offsets, tol: float = 1e-12) -> np.ndarray:
    """Element-block nonzero pattern of a probed matrix (reference krylov.py:167-183):
    (n_elem, n_elem) booleans, blocks with an entry above tol x the largest entry."""
    m = np.asarray(m)
    off = np.asarray(offsets)
    ne = len(off) - 1
    scale = np.abs(m).max()
    a = np.abs(m)
    # block maxima: reduce rows within element i, then columns within element j
    rows = np.maximum.reduceat(a, off[:-1], axis=0) if ne else np.zeros((0, a.shape[1]))
    blk = np.maximum.reduceat(rows, off[:-1], axis=1) if ne else np.zeros((0, 0))
    return blk > tol * scale
