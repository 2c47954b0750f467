"""Reference-element tables for the plan (host side, setup only).

Face topology of each shape (reference stdregions.py:140-192), the
generalized-tensor triangle tables (stdregions.py:266-383) and per-class 1-D
tables.  The sm_100a kernels consume these through the table pool built in
`plan.py`; nothing here runs per apply.
"""
from __future__ import annotations

import functools
import math
from dataclasses import dataclass

import numpy as np

from .polylib import BasisKind, QuadKind, as_basis_kind, as_quad_kind, eval_basis_1d, jacobi_eval, quad_rule

_S = math.sqrt(0.5)


@dataclass(frozen=True)
class FaceDef:
    fixed: int
    side: int
    run: tuple
    center: tuple
    tangents: tuple
    ref_normal: tuple


FACES = {
    "quad": (FaceDef(0, -1, (1,), (-1.0, 0.0), ((0.0, 1.0),), (-1.0, 0.0)),
             FaceDef(0, +1, (1,), (1.0, 0.0), ((0.0, 1.0),), (1.0, 0.0)),
             FaceDef(1, -1, (0,), (0.0, -1.0), ((1.0, 0.0),), (0.0, -1.0)),
             FaceDef(1, +1, (0,), (0.0, 1.0), ((1.0, 0.0),), (0.0, 1.0))),
    "tri": (FaceDef(1, -1, (0,), (0.0, -1.0), ((1.0, 0.0),), (0.0, -1.0)),
            FaceDef(0, +1, (1,), (0.0, 0.0), ((-1.0, 1.0),), (_S, _S)),
            FaceDef(0, -1, (1,), (-1.0, 0.0), ((0.0, 1.0),), (-1.0, 0.0))),
    "hex": tuple(FaceDef(a, s, tuple(b for b in range(3) if b != a),
                         tuple(float(s) if b == a else 0.0 for b in range(3)),
                         tuple(tuple(1.0 if c == b else 0.0 for c in range(3)) for b in range(3) if b != a),
                         tuple(float(s) if b == a else 0.0 for b in range(3)))
                 for a in range(3) for s in (-1, 1)),
}
DIM = {"quad": 2, "tri": 2, "hex": 3}
DEFAULT_RULES = {"quad": (QuadKind.GAUSS_LOBATTO,) * 2, "tri": (QuadKind.GAUSS_LEGENDRE,) * 2,
                 "hex": (QuadKind.GAUSS_LOBATTO,) * 3}


def tri_index(n: int, i: int, j: int) -> int:
    """Flat index of triangle mode (i, j), j <= n-1-i, lexicographic."""
    return i * n - i * (i - 1) // 2 + j


def tri_tables(kind, n: int, z1, z2):
    """Collapsed-coordinate triangle tables.

    Returns A, dA ((len z1, n+1) direction-1 functions per group), B, dB
    ((len z2, n_coeffs): column m holds the direction-2 function of mode m) and
    the group of each mode.  Modified modal groups: 0 = row i=0 without the
    collapsed-vertex mode, 1 = the vertex mode (0,1), 2 = row i=1, 2+i-1 = row
    i >= 2 (reference stdregions.py:286-383)."""
    kind = as_basis_kind(kind)
    z1 = np.atleast_1d(np.asarray(z1, dtype=float))
    z2 = np.atleast_1d(np.asarray(z2, dtype=float))
    nc = n * (n + 1) // 2
    B = np.zeros((z2.size, nc))
    dB = np.zeros((z2.size, nc))
    gid = np.zeros(nc, dtype=np.int64)
    if kind is BasisKind.ORTHOGONAL:
        A, dA = eval_basis_1d(BasisKind.ORTHOGONAL, n, z1)
        for i in range(n):
            f = (0.5 * (1.0 - z2)) ** i
            df = -0.5 * i * (0.5 * (1.0 - z2)) ** (i - 1) if i else np.zeros_like(z2)
            for j in range(n - i):
                m = tri_index(n, i, j)
                p, dp = jacobi_eval(2.0 * i + 1.0, 0.0, j, z2)
                s = math.sqrt(i + j + 1.0)
                B[:, m], dB[:, m], gid[m] = s * f * p, s * (df * p + f * dp), i
        return A, dA, B, dB, gid
    if kind is not BasisKind.MODIFIED_MODAL:
        raise ValueError("triangles support the modified modal and orthogonal bases")
    mm1, dmm1 = eval_basis_1d(BasisKind.MODIFIED_MODAL, n, z1)
    cols = [0, None, n - 1] + list(range(1, n - 1))
    A = np.empty((z1.size, n + 1))
    dA = np.empty_like(A)
    for g, c in enumerate(cols):
        A[:, g] = 1.0 if c is None else mm1[:, c]
        dA[:, g] = 0.0 if c is None else dmm1[:, c]
    mm, dmm = eval_basis_1d(BasisKind.MODIFIED_MODAL, n, z2)
    # row i = 0: (0,0) -> psi_0, (0,1) -> psi_{n-1} (vertex group), (0,j>=2) -> psi_{j-1}
    for j in range(n):
        m = tri_index(n, 0, j)
        c = 0 if j == 0 else (n - 1 if j == 1 else j - 1)
        B[:, m], dB[:, m], gid[m] = mm[:, c], dmm[:, c], (1 if j == 1 else 0)
    for j in range(n - 1):                     # row i = 1: psi_0 .. psi_{n-2}
        m = tri_index(n, 1, j)
        B[:, m], dB[:, m], gid[m] = mm[:, j], dmm[:, j], 2
    hp = 0.5 * (1.0 + z2)
    for i in range(2, n):
        f = (0.5 * (1.0 - z2)) ** i
        df = -0.5 * i * (0.5 * (1.0 - z2)) ** (i - 1)
        for j in range(n - i):
            m = tri_index(n, i, j)
            if j == 0:
                B[:, m], dB[:, m] = f, df
            else:
                p, dp = jacobi_eval(2.0 * i - 1.0, 1.0, j - 1, z2)
                B[:, m] = f * hp * p
                dB[:, m] = df * hp * p + f * (0.5 * p + hp * dp)
            gid[m] = i + 1
    return A, dA, B, dB, gid


@dataclass
class ClassTables:
    shape: str
    kind: BasisKind
    n: int
    nq: tuple
    rules: tuple
    n_coeffs: int
    n_phys: int
    ref_w: np.ndarray        # tensor weights (tri: with Duffy factor)
    xi: np.ndarray           # (n_phys, d) reference coords of the volume points
    eta: np.ndarray          # (n_phys, d) tensor coords
    axis: list               # tensor shapes: per-axis dict of 1-D tables
    tri: dict | None

    @property
    def dim(self):
        return DIM[self.shape]

    @property
    def faces(self):
        return FACES[self.shape]

    def face_npts(self, f):
        return int(np.prod([self.nq[a] for a in FACES[self.shape][f].run]))

    def face_pts(self, f):
        return tuple(self.rules[a].points for a in FACES[self.shape][f].run)

    def face_weights(self, f):
        w = np.ones(1)
        for a in FACES[self.shape][f].run:
            w = np.multiply.outer(w, self.rules[a].weights).reshape(-1)
        return w

    # reference Expansion field names (stdregions.py:391-412)
    @property
    def n_modes(self):
        return self.n

    @property
    def ref_weights(self):
        return self.ref_w

    @property
    def xi_phys(self):
        return self.xi

    @property
    def eta_phys(self):
        return self.eta

    def face_n_phys(self, face):
        f = face if isinstance(face, int) else self.faces.index(face)
        return self.face_npts(f)

    @property
    def key(self):
        return (self.shape, self.kind.value, self.n, self.nq, tuple(r.kind.value for r in self.rules))


@functools.lru_cache(maxsize=None)
def class_tables(shape: str, kind, n: int, nq: tuple, kinds: tuple) -> ClassTables:
    kind = as_basis_kind(kind)
    d = DIM[shape]
    if n < 2:
        raise ValueError("expansions need n_modes >= 2")
    rules = tuple(quad_rule(as_quad_kind(k), q) for k, q in zip(kinds, nq))
    if shape == "tri" and rules[1].kind is QuadKind.GAUSS_LOBATTO:
        raise ValueError("the triangle collapsed direction cannot carry an endpoint at eta2 = +1")
    g = np.meshgrid(*[r.points for r in rules], indexing="ij")
    eta = np.stack([a.reshape(-1) for a in g], axis=-1)
    w = rules[0].weights
    for r in rules[1:]:
        w = np.multiply.outer(w, r.weights)
    w = w.reshape(-1)
    axis = []
    for a, r in enumerate(rules):
        ends = np.array([-1.0, 1.0])
        L = np.vstack([_endpoint_row(r, -1), _endpoint_row(r, +1)])
        t = {"pts": r.points, "w": r.weights, "D": _dmat(r.points), "L": L,
             "gll": r.kind is QuadKind.GAUSS_LOBATTO}
        if shape != "tri":
            nodes = quad_rule(r.kind, n).points if kind is BasisKind.LAGRANGE else None
            t["V"], t["dV"] = eval_basis_1d(kind, n, r.points, nodes)
            t["Vend"], t["dVend"] = eval_basis_1d(kind, n, ends, nodes)
            t["nodes"] = nodes
        axis.append(t)
    tri = None
    if shape == "tri":
        A, dA, B, dB, gid = tri_tables(kind, n, rules[0].points, rules[1].points)
        Ae, dAe, Be, dBe, _ = tri_tables(kind, n, [-1.0, 1.0], [-1.0])
        order = np.argsort(gid, kind="stable")
        ng = A.shape[1]
        gstart = np.searchsorted(gid[order], np.arange(ng + 1))
        tri = {"A": A, "dA": dA, "B": B, "dB": dB, "gid": gid, "gmodes": order,
               "gstart": gstart, "Aend": Ae, "dAend": dAe, "Bm1": Be[0], "dBm1": dBe[0]}
        nc = n * (n + 1) // 2
        xi = eta.copy()
        xi[:, 0] = 0.5 * (1.0 + eta[:, 0]) * (1.0 - eta[:, 1]) - 1.0
        ref_w = w * 0.5 * (1.0 - eta[:, 1])
    else:
        nc = n ** d
        xi = eta
        ref_w = w
    return ClassTables(shape, kind, n, tuple(nq), rules, nc, int(np.prod(nq)), ref_w, xi, eta, axis, tri)


def _endpoint_row(rule, side):
    from .polylib import lagrange_interp_matrix
    return lagrange_interp_matrix(rule.points, np.array([float(side)]))[0]


def _dmat(pts):
    from .polylib import diff_matrix
    return diff_matrix(pts)


def face_basis(ct: ClassTables, f: int, prm: np.ndarray, deriv=None) -> np.ndarray:
    """Dense table of every mode (or its eta_deriv derivative) at face
    parameters prm (npts, d-1).  Setup/test helper (reference trace.py:213-256)."""
    face = FACES[ct.shape][f]
    prm = np.atleast_2d(prm)
    npts = prm.shape[0]
    if ct.shape == "tri":
        t = ct.tri
        if face.fixed == 0:
            A, dA, B, dB, gid = tri_tables(ct.kind, ct.n, [float(face.side)], prm[:, 0])
            arow = (dA if deriv == 0 else A)[0]
            return arow[gid][None, :] * (dB if deriv == 1 else B)
        A, dA, B, dB, gid = tri_tables(ct.kind, ct.n, prm[:, 0], [float(face.side)])
        arun = dA if deriv == 0 else A
        return arun[:, gid] * (dB if deriv == 1 else B)[0][None, :]
    pos = {ax: k for k, ax in enumerate(face.run)}
    m = np.ones((npts, 1))
    for ax in range(ct.dim):
        x = np.array([float(face.side)]) if ax == face.fixed else prm[:, pos[ax]]
        v, dv = eval_basis_1d(ct.kind, ct.n, x, ct.axis[ax].get("nodes"))
        tab = dv if deriv == ax else v
        tab = np.broadcast_to(tab, (npts, ct.n))
        m = np.einsum("ti,tj->tij", m, tab).reshape(npts, -1)
    return m
