"""ORACLE (test infrastructure only) — reference elements and sum-factorised
kernels.

Restates reference pkg/src/dgsipg/stdregions.py: face topology (103-192),
triangle generalized-tensor tables (266-383), expansions (469-552), batched
BwdTrans / IProduct / IProductDeriv / PhysDeriv (566-674), face restriction
(850-889); and the dense face tables of trace.py:213-256.
Arrays carry a trailing element-batch axis W as in the reference.
"""
from __future__ import annotations

import functools
import math
from dataclasses import dataclass

import numpy as np

from . import polylib as pl

QUAD, TRI, HEX = "quad", "tri", "hex"
DIM = {QUAD: 2, TRI: 2, HEX: 3}


@dataclass(frozen=True)
class Face:
    """stdregions.py:103-133."""
    fixed: int
    side: int
    run: tuple
    center: tuple
    tangents: tuple
    ref_normal: tuple
    corners: tuple

    def to_ref(self, prm: np.ndarray) -> np.ndarray:
        return np.asarray(self.center) + prm @ np.asarray(self.tangents).reshape(len(self.run), -1)


_S = math.sqrt(0.5)
FACES = {  # stdregions.py:140-192
    QUAD: (
        Face(0, -1, (1,), (-1.0, 0.0), ((0.0, 1.0),), (-1.0, 0.0), (0, 3)),
        Face(0, +1, (1,), (1.0, 0.0), ((0.0, 1.0),), (1.0, 0.0), (1, 2)),
        Face(1, -1, (0,), (0.0, -1.0), ((1.0, 0.0),), (0.0, -1.0), (0, 1)),
        Face(1, +1, (0,), (0.0, 1.0), ((1.0, 0.0),), (0.0, 1.0), (3, 2)),
    ),
    TRI: (
        Face(1, -1, (0,), (0.0, -1.0), ((1.0, 0.0),), (0.0, -1.0), (0, 1)),
        Face(0, +1, (1,), (0.0, 0.0), ((-1.0, 1.0),), (_S, _S), (1, 2)),
        Face(0, -1, (1,), (-1.0, 0.0), ((0.0, 1.0),), (-1.0, 0.0), (0, 2)),
    ),
    HEX: (
        Face(0, -1, (1, 2), (-1.0, 0.0, 0.0), ((0.0, 1.0, 0.0), (0.0, 0.0, 1.0)), (-1.0, 0.0, 0.0), (0, 3, 4, 7)),
        Face(0, +1, (1, 2), (1.0, 0.0, 0.0), ((0.0, 1.0, 0.0), (0.0, 0.0, 1.0)), (1.0, 0.0, 0.0), (1, 2, 5, 6)),
        Face(1, -1, (0, 2), (0.0, -1.0, 0.0), ((1.0, 0.0, 0.0), (0.0, 0.0, 1.0)), (0.0, -1.0, 0.0), (0, 1, 4, 5)),
        Face(1, +1, (0, 2), (0.0, 1.0, 0.0), ((1.0, 0.0, 0.0), (0.0, 0.0, 1.0)), (0.0, 1.0, 0.0), (3, 2, 7, 6)),
        Face(2, -1, (0, 1), (0.0, 0.0, -1.0), ((1.0, 0.0, 0.0), (0.0, 1.0, 0.0)), (0.0, 0.0, -1.0), (0, 1, 3, 2)),
        Face(2, +1, (0, 1), (0.0, 0.0, 1.0), ((1.0, 0.0, 0.0), (0.0, 1.0, 0.0)), (0.0, 0.0, 1.0), (4, 5, 7, 6)),
    ),
}

DEFAULT_KINDS = {QUAD: (pl.GLL,) * 2, TRI: (pl.GL,) * 2, HEX: (pl.GLL,) * 3}


def tri_flat(n, i, j):
    """stdregions.py:282-283."""
    return sum(n - k for k in range(i)) + j


def tri_dir1(kind, n, z):
    """Direction-1 table, group columns [psi0, 1, psi_{n-1}, psi_1..psi_{n-2}]
    — stdregions.py:286-309 (modified modal) / orthogonal branch."""
    z = np.atleast_1d(np.asarray(z, dtype=float))
    if kind == pl.ORTHO:
        return pl.orthonormal(n, z)
    mm, dmm = pl.modified(n, z)
    a = np.empty((z.size, n + 1))
    da = np.empty_like(a)
    for g, c in enumerate([0, None, n - 1] + list(range(1, n - 1))):
        if c is None:
            a[:, g], da[:, g] = 1.0, 0.0
        else:
            a[:, g], da[:, g] = mm[:, c], dmm[:, c]
    return a, da


def tri_groups(kind, n, z):
    """Direction-2 tables per group: list of (modes, B, dB) — stdregions.py:312-383."""
    z = np.atleast_1d(np.asarray(z, dtype=float))
    out = []
    if kind == pl.ORTHO:
        for i in range(n):
            f = (0.5 * (1.0 - z)) ** i
            df = -0.5 * i * (0.5 * (1.0 - z)) ** (i - 1) if i > 0 else np.zeros_like(z)
            b = np.empty((z.size, n - i))
            db = np.empty_like(b)
            for j in range(n - i):
                sc = math.sqrt(i + j + 1.0)
                p, dp = pl.jacobi(2.0 * i + 1.0, 0.0, j, z)
                b[:, j] = sc * f * p
                db[:, j] = sc * (df * p + f * dp)
            out.append((np.array([tri_flat(n, i, j) for j in range(n - i)]), b, db))
        return out
    mm, dmm = pl.modified(n, z)
    j0 = [0] + list(range(2, n))
    cols = [0] + [j - 1 for j in j0[1:]]
    out.append((np.array([tri_flat(n, 0, j) for j in j0]), mm[:, cols], dmm[:, cols]))
    out.append((np.array([tri_flat(n, 0, 1)]), mm[:, [n - 1]], dmm[:, [n - 1]]))
    out.append((np.array([tri_flat(n, 1, j) for j in range(n - 1)]), mm[:, : n - 1], dmm[:, : n - 1]))
    for i in range(2, n):
        f = (0.5 * (1.0 - z)) ** i
        df = -0.5 * i * (0.5 * (1.0 - z)) ** (i - 1)
        hp = 0.5 * (1.0 + z)
        b = np.empty((z.size, n - i))
        db = np.empty_like(b)
        b[:, 0], db[:, 0] = f, df
        for j in range(1, n - i):
            p, dp = pl.jacobi(2.0 * i - 1.0, 1.0, j - 1, z)
            b[:, j] = f * hp * p
            db[:, j] = df * hp * p + f * (0.5 * p + hp * dp)
        out.append((np.array([tri_flat(n, i, j) for j in range(n - i)]), b, db))
    return out


class Expansion:
    """Reference-element discretisation — stdregions.py:390-552."""

    def __init__(self, shape, kind, n, nq, kinds):
        self.shape, self.kind, self.n = shape, kind, n
        self.dim = d = DIM[shape]
        self.nq = tuple(nq)
        self.kinds = tuple(kinds)
        self.rules = [pl.rule(k, q) for k, q in zip(self.kinds, self.nq)]
        self.pts = [r[0] for r in self.rules]
        self.faces = FACES[shape]
        g = np.meshgrid(*self.pts, indexing="ij")
        eta = np.stack([a.reshape(-1) for a in g], axis=-1)
        w = self.rules[0][1]
        for r in self.rules[1:]:
            w = np.multiply.outer(w, r[1])
        w = w.reshape(-1)
        self.n_phys = int(np.prod(self.nq))
        self.D = [pl.dmat(p) for p in self.pts]
        if shape == TRI:
            self.A, self.dA = tri_dir1(kind, n, self.pts[0])
            self.groups = tri_groups(kind, n, self.pts[1])
            self.n_coeffs = n * (n + 1) // 2
            xi = eta.copy()
            xi[:, 0] = 0.5 * (1.0 + eta[:, 0]) * (1.0 - eta[:, 1]) - 1.0
            self.ref_w = w * 0.5 * (1.0 - eta[:, 1])
            self.nodes = None
        else:
            self.nodes = [pl.rule(k, n)[0] if kind == pl.LAGRANGE else None for k in self.kinds]
            tabs = [pl.basis(kind, n, p, nd) for p, nd in zip(self.pts, self.nodes)]
            self.V = [t[0] for t in tabs]
            self.dV = [t[1] for t in tabs]
            self.n_coeffs = n ** d
            xi = eta
            self.ref_w = w
        self.eta, self.xi = eta, xi

    # --- identity: expansions are cached, so "same parameters" <=> "same object"
    @property
    def key(self):
        return (self.shape, self.kind, self.n, self.nq, self.kinds)

    def face_npts(self, f):
        return int(np.prod([self.nq[a] for a in self.faces[f].run], initial=1))

    def face_pts(self, f):
        return tuple(self.pts[a] for a in self.faces[f].run)

    def collapse_jac(self):
        """d eta / d xi at the volume points (tri) — stdregions.py:428-439."""
        if self.shape != TRI:
            return None
        e1, e2 = self.eta[:, 0], self.eta[:, 1]
        out = np.zeros((2, 2, self.n_phys))
        out[0, 0] = 2.0 / (1.0 - e2)
        out[0, 1] = (1.0 + e1) / (1.0 - e2)
        out[1, 1] = 1.0
        return out

    # --- sum-factorised kernels (stdregions.py:566-674) ------------------
    @staticmethod
    def _axis(mat, t, ax):
        return np.moveaxis(np.tensordot(mat, t, axes=(1, ax)), 0, ax)

    def bwd(self, c):
        w = c.shape[-1]
        if self.shape == TRI:
            t = np.empty((self.n + 1, self.nq[1], w))
            for g, (modes, b, _) in enumerate(self.groups):
                t[g] = b @ c[modes]
            u = np.tensordot(self.A, t, axes=(1, 0))
        else:
            u = c.reshape(*([self.n] * self.dim), w)
            for ax in range(self.dim):
                u = self._axis(self.V[ax], u, ax)
        return u.reshape(self.n_phys, w)

    def iprod(self, f):
        w = f.shape[-1]
        if self.shape == TRI:
            s = np.tensordot(self.A.T, f.reshape(self.nq[0], self.nq[1], w), axes=(1, 0))
            out = np.empty((self.n_coeffs, w))
            for g, (modes, b, _) in enumerate(self.groups):
                out[modes] = b.T @ s[g]
            return out
        t = f.reshape(*self.nq, w)
        for ax in range(self.dim):
            t = self._axis(self.V[ax].T, t, ax)
        return t.reshape(self.n_coeffs, w)

    def iprod_d(self, k, f):
        w = f.shape[-1]
        if self.shape == TRI:
            a = self.dA if k == 0 else self.A
            s = np.tensordot(a.T, f.reshape(self.nq[0], self.nq[1], w), axes=(1, 0))
            out = np.empty((self.n_coeffs, w))
            for g, (modes, b, db) in enumerate(self.groups):
                out[modes] = (b if k == 0 else db).T @ s[g]
            return out
        t = f.reshape(*self.nq, w)
        for ax in range(self.dim):
            t = self._axis((self.dV[ax] if ax == k else self.V[ax]).T, t, ax)
        return t.reshape(self.n_coeffs, w)

    def deriv(self, u):
        w = u.shape[-1]
        t = u.reshape(*self.nq, w)
        return np.stack([self._axis(self.D[ax], t, ax).reshape(self.n_phys, w)
                         for ax in range(self.dim)])

    # --- face restriction (stdregions.py:850-889) ------------------------
    def face_vals(self, f, phys):
        face = self.faces[f]
        w = phys.shape[-1]
        t = phys.reshape(*self.nq, w)
        kind, q = self.kinds[face.fixed], self.nq[face.fixed]
        if pl.includes(kind, face.side):
            out = np.take(t, 0 if face.side < 0 else q - 1, axis=face.fixed)
        else:
            row = pl.interp(self.pts[face.fixed], [float(face.side)])
            out = np.tensordot(row, t, axes=(1, face.fixed))[0]
        return out.reshape(-1, w)

    def face_vol_idx(self, f):
        face = self.faces[f]
        kind, q = self.kinds[face.fixed], self.nq[face.fixed]
        if not pl.includes(kind, face.side):
            return None
        idx = np.arange(self.n_phys).reshape(self.nq)
        return np.take(idx, 0 if face.side < 0 else q - 1, axis=face.fixed).reshape(-1)

    # --- dense face tables at arbitrary face parameters (trace.py:213-256)
    def face_table(self, f, prm, deriv=None):
        face = self.faces[f]
        prm = np.atleast_2d(np.asarray(prm, dtype=float))
        npts = prm.shape[0]
        if self.shape == TRI:
            n = self.n
            out = np.zeros((npts, self.n_coeffs))
            if face.fixed == 0:
                av, dav = tri_dir1(self.kind, n, [float(face.side)])
                arow = dav if deriv == 0 else av
                for g, (modes, b, db) in enumerate(tri_groups(self.kind, n, prm[:, 0])):
                    out[:, modes] = arow[0, g] * (db if deriv == 1 else b)
            else:
                a, da = tri_dir1(self.kind, n, prm[:, 0])
                arun = da if deriv == 0 else a
                for g, (modes, b, db) in enumerate(tri_groups(self.kind, n, [float(face.side)])):
                    out[:, modes] = arun[:, [g]] * (db if deriv == 1 else b)[0][None, :]
            return out
        pos = {ax: k for k, ax in enumerate(face.run)}
        m = None
        for ax in range(self.dim):
            x = np.array([float(face.side)]) if ax == face.fixed else prm[:, pos[ax]]
            v, dv = pl.basis(self.kind, self.n, x, self.nodes[ax])
            tab = dv if deriv == ax else v
            if ax == face.fixed:
                tab = np.broadcast_to(tab, (npts, self.n))
            m = tab if m is None else np.einsum("ti,tj->tij", m, tab).reshape(npts, -1)
        return m


@functools.lru_cache(maxsize=None)
def expansion(shape, kind, n, nq, kinds=None):
    """Cached expansion (one object per parameter set, stdregions.py:489-552)."""
    d = DIM[shape]
    nq = (nq,) * d if isinstance(nq, int) else tuple(nq)
    kinds = kinds or DEFAULT_KINDS[shape]
    kinds = (kinds,) * d if isinstance(kinds, str) else tuple(kinds)
    return Expansion(shape, kind, n, nq, kinds)
