"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restatement of the reference's matrix-free CG (pkg/src/dgsipg/krylov.py:39-81)
and restarted GMRES (krylov.py:84-141) over any `apply_op(x) -> y`, used by
tests/test_krylov.py as the checker of the GPU solvers.
"""
from __future__ import annotations

import numpy as np


def cg(apply_op, b, tol=1e-9, maxiter=None):
    """krylov.py:39-81: returns (x, converged, iterations, residual, reason)."""
    b = np.asarray(b, dtype=float)
    n = b.size
    nb = float(np.linalg.norm(b))                         # :43
    x = np.zeros(n)
    if nb == 0.0:
        return x, True, 0, 0.0, ""
    maxiter = max(10 * n, 200) if maxiter is None else maxiter   # :48-49
    r = b.copy()
    p = r.copy()
    rr = float(r @ r)
    best, stall = np.sqrt(rr) / nb, 0
    for it in range(1, maxiter + 1):
        ap = apply_op(p)                                  # :56
        pap = float(p @ ap)
        if pap <= 0.0 or not np.isfinite(pap):            # :58-60
            return x, False, it, np.sqrt(max(rr, 0.0)) / nb, "indefinite direction"
        alpha = rr / pap
        x = x + alpha * p
        r = r - alpha * ap
        rr_new = float(r @ r)
        rel = np.sqrt(rr_new) / nb
        if rel <= tol:                                    # :66-71
            true_rel = float(np.linalg.norm(b - apply_op(x))) / nb
            if true_rel <= 10.0 * tol:
                return x, True, it, true_rel, ""
            return x, False, it, true_rel, "residual drift"
        if rel < 0.999 * best:                            # :72-78
            best, stall = rel, 0
        else:
            stall += 1
            if stall >= 250:
                return x, False, it, rel, "stagnation"
        beta = rr_new / rr
        rr = rr_new
        p = r + beta * p
    return x, False, maxiter, np.sqrt(rr) / nb, "maxiter"


def gmres(apply_op, b, tol=1e-9, restart=50, maxiter=None):
    """The reference's restarted GMRES contract (krylov.py:84-141): restart cycles of at most
    `restart` Arnoldi steps; a cycle ends early when the least-squares residual drops to tol; the
    solve stops when the residual at a cycle start or the true residual after an update is <= tol,
    else after `maxiter` steps in total with reason "maxiter".  Restated with Householder-free
    numpy: modified Gram-Schmidt Arnoldi and the small least-squares problem by np.linalg.lstsq
    (the reference rotates with Givens; both minimise the same residual).
    Returns (x, converged, iterations, residual, reason)."""
    b = np.asarray(b, dtype=float)
    n = b.size
    nb = float(np.linalg.norm(b))
    x = np.zeros(n)
    if nb == 0.0:
        return x, True, 0, 0.0, ""
    maxiter = max(20 * n, 400) if maxiter is None else maxiter
    m_cap = max(1, min(restart, n))
    steps = 0
    while steps < maxiter:
        r = b - apply_op(x)
        beta = float(np.linalg.norm(r))
        if beta / nb <= tol:
            return x, True, steps, beta / nb, ""
        m = min(m_cap, maxiter - steps)
        basis = [r / beta]
        hess = np.zeros((m + 1, m))
        e1 = np.zeros(m + 1)
        e1[0] = beta
        y = np.zeros(0)
        for k in range(m):
            v = apply_op(basis[k])
            for i, qi in enumerate(basis):
                hess[i, k] = float(v @ qi)
                v = v - hess[i, k] * qi
            hess[k + 1, k] = float(np.linalg.norm(v))
            basis.append(v / hess[k + 1, k] if hess[k + 1, k] > 1e-300 else np.zeros(n))
            steps += 1
            y, *_ = np.linalg.lstsq(hess[:k + 2, :k + 1], e1[:k + 2], rcond=None)
            res = float(np.linalg.norm(e1[:k + 2] - hess[:k + 2, :k + 1] @ y))
            if res / nb <= tol:
                break
        x = x + np.stack(basis[:y.size], axis=1) @ y
        rel = float(np.linalg.norm(b - apply_op(x))) / nb
        if rel <= tol:
            return x, True, steps, rel, ""
    rel = float(np.linalg.norm(b - apply_op(x))) / nb
    return x, False, steps, rel, "maxiter"
