"""ORACLE (test infrastructure only) — 1-D polynomial toolkit.

Restates reference pkg/src/dgsipg/polylib.py: Jacobi recurrences (76-107),
Golub-Welsch + one Newton step quadrature (110-180), barycentric Lagrange
interpolation (183-220), collocation differentiation (223-236) and the 1-D
basis families (285-340).
"""
from __future__ import annotations

import functools
import math

import numpy as np

GL = "gauss_legendre"
GRM = "gauss_radau_m"
GLL = "gauss_lobatto"

MODIFIED = "modified_modal"
ORTHO = "orthogonal"
LAGRANGE = "lagrange"


def exactness(kind: str, n: int) -> int:
    """polylib.py:39-43."""
    return {GL: 2 * n - 1, GRM: 2 * n - 2, GLL: 2 * n - 3}[kind]


def includes(kind: str, side: int) -> bool:
    """polylib.py:64-73: which endpoints a rule carries."""
    if side < 0:
        return kind in (GRM, GLL)
    return kind == GLL


def _jac(a: float, b: float, n: int, x: np.ndarray) -> np.ndarray:
    # three-term recurrence, polylib.py:95-107
    if n == 0:
        return np.ones_like(x)
    prev = np.ones_like(x)
    cur = 0.5 * ((a + b + 2.0) * x + (a - b))
    for k in range(2, n + 1):
        s = 2.0 * k + a + b
        den = 2.0 * k * (k + a + b) * (s - 2.0)
        c1 = (s - 1.0) * (a * a - b * b)
        c2 = (s - 1.0) * s * (s - 2.0)
        c3 = 2.0 * (k + a - 1.0) * (k + b - 1.0) * s
        prev, cur = cur, ((c1 + c2 * x) * cur - c3 * prev) / den
    return cur


def jacobi(a: float, b: float, n: int, x):
    """(P_n^{a,b}(x), d/dx P_n^{a,b}(x)) — polylib.py:76-92."""
    x = np.asarray(x, dtype=float)
    v = _jac(a, b, n, x)
    if n == 0:
        return v, np.zeros_like(x)
    return v, 0.5 * (n + a + b + 1.0) * _jac(a + 1.0, b + 1.0, n - 1, x)


def _gw_nodes(a: float, b: float, n: int) -> np.ndarray:
    # Golub-Welsch symmetric tridiagonal eigenproblem, polylib.py:110-132
    if n == 0:
        return np.zeros(0)
    k = np.arange(n, dtype=float)
    s = 2.0 * k + a + b
    diag = np.zeros(n)
    diag[0] = 0.0 if a + b == 0.0 else (b - a) / (a + b + 2.0)
    if n > 1:
        diag[1:] = (b * b - a * a) / (s[1:] * (s[1:] + 2.0))
    kk, ss = k[1:], s[1:]
    off = np.sqrt(4.0 * kk * (kk + a) * (kk + b) * (kk + a + b)
                  / (ss * ss * (ss + 1.0) * (ss - 1.0)))
    t = np.diag(diag) + np.diag(off, 1) + np.diag(off, -1)
    x = np.sort(np.linalg.eigvalsh(t))
    v, dv = jacobi(a, b, n, x)           # one Newton step, polylib.py:135-137
    return x - v / dv


@functools.lru_cache(maxsize=None)
def rule(kind: str, n: int):
    """(points, weights) — polylib.py:146-180."""
    if kind == GL:
        x = _gw_nodes(0.0, 0.0, n)
        _, dp = jacobi(0.0, 0.0, n, x)
        w = 2.0 / ((1.0 - x * x) * dp * dp)
    elif kind == GRM:
        if n == 1:
            x, w = np.array([-1.0]), np.array([2.0])
        else:
            x = np.concatenate(([-1.0], _gw_nodes(0.0, 1.0, n - 1)))
            p, _ = jacobi(0.0, 0.0, n - 1, x)
            w = (1.0 - x) / (n * n * p * p)
            w[0] = 2.0 / (n * n)
    elif kind == GLL:
        if n < 2:
            raise ValueError("GLL needs n >= 2")
        inner = _gw_nodes(1.0, 1.0, n - 2) if n > 2 else np.zeros(0)
        x = np.concatenate(([-1.0], inner, [1.0]))
        p, _ = jacobi(0.0, 0.0, n - 1, x)
        w = 2.0 / (n * (n - 1) * p * p)
    else:
        raise ValueError(kind)
    x.flags.writeable = False
    w.flags.writeable = False
    return x, w


def bary(src: np.ndarray) -> np.ndarray:
    d = src[:, None] - src[None, :]
    np.fill_diagonal(d, 1.0)
    return 1.0 / d.prod(axis=1)


def interp(src, dst) -> np.ndarray:
    """Lagrange interpolation matrix src -> dst (barycentric, exact hits one-hot)
    — polylib.py:200-220."""
    src = np.asarray(src, dtype=float)
    dst = np.atleast_1d(np.asarray(dst, dtype=float))
    lam = bary(src)
    out = np.zeros((dst.size, src.size))
    for r, y in enumerate(dst):
        d = y - src
        hit = np.flatnonzero(d == 0.0)
        if hit.size:
            out[r, hit[0]] = 1.0
        else:
            t = lam / d
            out[r] = t / t.sum()
    return out


def dmat(pts) -> np.ndarray:
    """Collocation differentiation matrix — polylib.py:223-236."""
    x = np.asarray(pts, dtype=float)
    lam = bary(x)
    n = x.size
    d = np.zeros((n, n))
    for i in range(n):
        dx = x[i] - x
        dx[i] = 1.0
        row = (lam / lam[i]) / dx
        row[i] = 0.0
        row[i] = -row.sum()
        d[i] = row
    return d


def modified(n: int, x):
    """Modified-modal family and derivative — polylib.py:285-302."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    v = np.empty((x.size, n))
    dv = np.empty((x.size, n))
    v[:, 0] = 0.5 * (1.0 - x)
    dv[:, 0] = -0.5
    v[:, n - 1] = 0.5 * (1.0 + x)
    dv[:, n - 1] = 0.5
    bub = 0.25 * (1.0 - x) * (1.0 + x)
    for i in range(1, n - 1):
        p, dp = jacobi(1.0, 1.0, i - 1, x)
        v[:, i] = bub * p
        dv[:, i] = -0.5 * x * p + bub * dp
    return v, dv


def orthonormal(n: int, x):
    """polylib.py:305-315."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    v = np.empty((x.size, n))
    dv = np.empty((x.size, n))
    for i in range(n):
        p, dp = jacobi(0.0, 0.0, i, x)
        v[:, i] = math.sqrt(i + 0.5) * p
        dv[:, i] = math.sqrt(i + 0.5) * dp
    return v, dv


def basis(kind: str, n: int, x, nodes=None):
    """(V, dV) of a 1-D family at x — polylib.py:318-340 (Lagrange: derivative
    by interpolating the collocation derivative, 318-325)."""
    if kind == MODIFIED:
        return modified(n, x)
    if kind == ORTHO:
        return orthonormal(n, x)
    if kind == LAGRANGE:
        v = interp(nodes, x)
        return v, v @ dmat(nodes)
    raise ValueError(kind)
