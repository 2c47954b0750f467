"""1-D quadrature rules, bases and interpolation operators (plan construction).

Host-side setup that tabulates the small per-class matrices the sm_100a kernels
consume (they are uploaded once per plan).  Names and enum values mirror the
reference's `dgsipg.polylib` (reference pkg/src/dgsipg/polylib.py:33-43,
239-242) so reference enums are accepted interchangeably (matched by `.value`).

Nodes: Golub-Welsch start, then Newton iterations on the defining Jacobi
polynomial until the update stalls (the reference does one fixed step,
polylib.py:135-137; tables agree to rounding).
"""
from __future__ import annotations

import enum
import functools
import math

import numpy as np

__all__ = ["QuadKind", "BasisKind", "QuadRule", "quad_rule", "jacobi_eval",
           "lagrange_interp_matrix", "diff_matrix", "eval_basis_1d"]


class QuadKind(enum.Enum):
    GAUSS_LEGENDRE = "gauss_legendre"
    GAUSS_RADAU_M = "gauss_radau_m"
    GAUSS_LOBATTO = "gauss_lobatto"


class BasisKind(enum.Enum):
    MODIFIED_MODAL = "modified_modal"
    ORTHOGONAL = "orthogonal"
    LAGRANGE = "lagrange"


def as_quad_kind(k) -> QuadKind:
    return k if isinstance(k, QuadKind) else QuadKind(getattr(k, "value", k))


def as_basis_kind(k) -> BasisKind:
    return k if isinstance(k, BasisKind) else BasisKind(getattr(k, "value", k))


class QuadRule:
    __slots__ = ("kind", "n", "points", "weights")

    def __init__(self, kind, n, points, weights):
        self.kind, self.n, self.points, self.weights = kind, n, points, weights

    @property
    def exactness(self) -> int:
        """Degree integrated exactly (reference polylib.py:39-43)."""
        return {QuadKind.GAUSS_LEGENDRE: 2 * self.n - 1,
                QuadKind.GAUSS_RADAU_M: 2 * self.n - 2,
                QuadKind.GAUSS_LOBATTO: 2 * self.n - 3}[self.kind]

    def includes_endpoint(self, side: int) -> bool:
        if side < 0:
            return self.kind in (QuadKind.GAUSS_RADAU_M, QuadKind.GAUSS_LOBATTO)
        return self.kind is QuadKind.GAUSS_LOBATTO


def jacobi_eval(alpha: float, beta: float, n: int, x):
    """P_n^{(alpha,beta)}(x) and its derivative by the three-term recurrence."""
    x = np.asarray(x, dtype=float)

    def p(a, b, m):
        if m == 0:
            return np.ones_like(x)
        lo, hi = np.ones_like(x), 0.5 * ((a + b + 2.0) * x + (a - b))
        for k in range(2, m + 1):
            s = 2.0 * k + a + b
            lo, hi = hi, (((s - 1.0) * (a * a - b * b) + (s - 1.0) * s * (s - 2.0) * x) * hi
                          - 2.0 * (k + a - 1.0) * (k + b - 1.0) * s * lo) / (2.0 * k * (k + a + b) * (s - 2.0))
        return hi

    v = p(alpha, beta, n)
    dv = np.zeros_like(x) if n == 0 else 0.5 * (n + alpha + beta + 1.0) * p(alpha + 1.0, beta + 1.0, n - 1)
    return v, dv


def _jacobi_roots(a: float, b: float, n: int) -> np.ndarray:
    if n == 0:
        return np.zeros(0)
    k = np.arange(n, dtype=float)
    s = 2.0 * k + a + b
    diag = np.where(k == 0, (b - a) / (a + b + 2.0) if a + b != 0.0 else 0.0,
                    (b * b - a * a) / np.where(k == 0, 1.0, s * (s + 2.0)))
    kk, ss = k[1:], s[1:]
    off = np.sqrt(4.0 * kk * (kk + a) * (kk + b) * (kk + a + b) / (ss * ss * (ss + 1.0) * (ss - 1.0)))
    x = np.sort(np.linalg.eigvalsh(np.diag(diag) + np.diag(off, 1) + np.diag(off, -1)))
    for _ in range(4):
        v, dv = jacobi_eval(a, b, n, x)
        step = v / dv
        x = x - step
        if np.max(np.abs(step)) < 1e-16:
            break
    return x


@functools.lru_cache(maxsize=None)
def quad_rule(kind, n: int) -> QuadRule:
    """n-point rule of the given kind on [-1, 1] (cached singleton)."""
    kind = as_quad_kind(kind)
    if kind is QuadKind.GAUSS_LEGENDRE:
        x = _jacobi_roots(0.0, 0.0, n)
        _, dp = jacobi_eval(0.0, 0.0, n, x)
        w = 2.0 / ((1.0 - x * x) * dp * dp)
    elif kind is QuadKind.GAUSS_RADAU_M:
        x = np.concatenate(([-1.0], _jacobi_roots(0.0, 1.0, n - 1)))
        pv, _ = jacobi_eval(0.0, 0.0, n - 1, x)
        w = (1.0 - x) / (n * n * pv * pv)
        w[0] = 2.0 / (n * n)
    else:
        if n < 2:
            raise ValueError("Gauss-Lobatto rules need n >= 2")
        x = np.concatenate(([-1.0], _jacobi_roots(1.0, 1.0, n - 2), [1.0]))
        pv, _ = jacobi_eval(0.0, 0.0, n - 1, x)
        w = 2.0 / (n * (n - 1) * pv * pv)
    x.flags.writeable = False
    w.flags.writeable = False
    return QuadRule(kind, n, x, w)


def lagrange_interp_matrix(src, dst) -> np.ndarray:
    """Rows: Lagrange cardinal functions of `src` at each `dst` point
    (barycentric form; a coincident point gives an exact one-hot row)."""
    src = np.asarray(src, dtype=float)
    dst = np.atleast_1d(np.asarray(dst, dtype=float))
    diff = src[:, None] - src[None, :]
    np.fill_diagonal(diff, 1.0)
    lam = 1.0 / diff.prod(axis=1)
    d = dst[:, None] - src[None, :]
    hit = d == 0.0
    safe = np.where(hit, 1.0, d)
    t = lam[None, :] / safe
    out = t / t.sum(axis=1, keepdims=True)
    rows = hit.any(axis=1)
    if rows.any():
        out[rows] = 0.0
        out[rows, np.argmax(hit[rows], axis=1)] = 1.0
    return out


def diff_matrix(points) -> np.ndarray:
    """Collocation derivative matrix D[i, j] = l_j'(x_i)."""
    x = np.asarray(points, dtype=float)
    diff = x[:, None] - x[None, :]
    np.fill_diagonal(diff, 1.0)
    lam = 1.0 / diff.prod(axis=1)
    d = (lam[None, :] / lam[:, None]) / diff
    np.fill_diagonal(d, 0.0)
    np.fill_diagonal(d, -d.sum(axis=1))
    return d


def eval_basis_1d(kind, n: int, x, nodes=None):
    """(V, dV) of a 1-D family at points x: modified modal
    ((1-x)/2, bubbles (1-x)(1+x)/4 P^{1,1}_{i-1}, (1+x)/2), orthonormal
    Legendre, or Lagrange on `nodes`."""
    kind = as_basis_kind(kind)
    x = np.atleast_1d(np.asarray(x, dtype=float))
    if kind is BasisKind.LAGRANGE:
        v = lagrange_interp_matrix(nodes, x)
        return v, v @ diff_matrix(nodes)
    v = np.empty((x.size, n))
    dv = np.empty((x.size, n))
    if kind is BasisKind.ORTHOGONAL:
        for i in range(n):
            p, dp = jacobi_eval(0.0, 0.0, i, x)
            v[:, i], dv[:, i] = math.sqrt(i + 0.5) * p, math.sqrt(i + 0.5) * dp
        return v, dv
    v[:, 0], dv[:, 0] = 0.5 * (1.0 - x), -0.5
    v[:, n - 1], dv[:, n - 1] = 0.5 * (1.0 + x), 0.5
    bub = 0.25 * (1.0 - x) * (1.0 + x)
    for i in range(1, n - 1):
        p, dp = jacobi_eval(1.0, 1.0, i - 1, x)
        v[:, i] = bub * p
        dv[:, i] = -0.5 * x * p + bub * dp
    return v, dv
