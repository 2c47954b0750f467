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
