"""ORACLE (test infrastructure only) — config 4: the SIP-Helmholtz apply on 3-D
hybrid hex / prism / tet meshes.

PARITY UNPINNED for prisms and tets: the reference has no prism or tet
expansion (reference stdregions.py:57-69 lists seg/quad/tri/hex only; mesh.py
rejects other 3-D shapes).  This module extends the
reference's algorithm to those shapes, following its own machinery:

* bases — the reference's modified-modal triangle is a "collapse" of the 1-D
  modified family: every 1-D function psi of degree d is multiplied by
  ((1-z)/2)^d [1, (1+z)/2 P^{2d-1,1}_{k-1}(z)] in the collapsed direction,
  plus the apex (1+z)/2 (reference stdregions.py:286-383, `tri_dir1` /
  `tri_groups`).  The tet applies the same collapse to the reference's
  triangle (degree of triangle mode (i, j) = max(i + j, 1)) plus the apex; the
  prism is the reference triangle times the 1-D modified family.  Both span
  the full polynomial space of the shape (tested);
* quadrature — Gauss-Legendre in collapsed directions with the Duffy factor
  folded into the weights (the reference's triangle reading of
  "Gauss-Jacobi", stdregions.py:481-524), GLL in the prism's tensor direction;
* operator — the reference's two-phase apply (sipg.py:558-602) with every
  interface on the shared-trace route (TracePhysEval + TraceIProduct,
  sipg.py:513-554, 653-677; the reference's `face_absorb="trace_iproduct"`
  mode, exact for these affine meshes).  Trace points follow the reference's
  shared rule patched per SURVEY §8c P2: GLL only when both sides are GLL
  (hex-hex), else Gauss-Legendre (collapsed Gauss-Legendre on triangular
  faces), max(q) points per direction, on the left side's face parameters; the
  other side's parameters come from the geometry (physical point -> reference
  coordinates).  A hex / prism quad face meeting the two triangles of a split
  cube couples to each triangle as its own shared trace (SURVEY a18's
  resolution), the triangle side being "left";
* tau = max(n_L, n_R)^2 / h with h = min over sides of volume / face area
  (reference sipg.py:351-360 with patch P1).  Jacobians enter as |det J|: a
  sorted-vertex tet or prism may be left-handed (the reference requires
  det J > 0, mesh.py:337-338, for its hex/quad-only meshes).

What pins it: on all-hex meshes this operator is checked against the
reference-pinned 2-D/hex oracle (`OracleOperator(face_absorb=
"trace_iproduct")`); prisms/tets are checked by property tests
(tests/test_hybrid3d_oracle.py): polynomial span, symmetry, A.0 = 0,
consistency on global linear fields, mass matrix.
"""
from __future__ import annotations

import functools
import math
from dataclasses import dataclass

import numpy as np

from . import polylib as pl
from .elements import FACES as _REF_FACES, tri_dir1, tri_groups

HEX, PRISM, TET = "hex", "prism", "tet"
SHAPES = (HEX, PRISM, TET)


# --- faces -----------------------------------------------------------------------------------
@dataclass(frozen=True)
class Face3:
    fixed: int            # eta axis held at `side`
    side: int
    run: tuple            # eta axes that parametrise the face (first = first face parameter)
    corners: tuple        # local vertex indices (matching key)
    ref_normal: tuple     # outward normal in xi space
    tri: bool             # triangular face (collapsed parameters)


_S2, _S3 = math.sqrt(0.5), math.sqrt(1.0 / 3.0)
FACES3 = {
    HEX: tuple(Face3(f.fixed, f.side, f.run, f.corners, f.ref_normal, False) for f in _REF_FACES["hex"]),
    PRISM: (
        Face3(2, -1, (0, 1), (0, 1, 2, 3), (0.0, 0.0, -1.0), False),
        Face3(1, -1, (0, 2), (0, 1, 4), (0.0, -1.0, 0.0), True),
        Face3(0, +1, (1, 2), (1, 2, 5, 4), (_S2, 0.0, _S2), False),
        Face3(1, +1, (0, 2), (3, 2, 5), (0.0, 1.0, 0.0), True),
        Face3(0, -1, (1, 2), (0, 3, 4, 5), (-1.0, 0.0, 0.0), False),
    ),
    TET: (
        Face3(2, -1, (0, 1), (0, 1, 2), (0.0, 0.0, -1.0), True),
        Face3(1, -1, (0, 2), (0, 1, 3), (0.0, -1.0, 0.0), True),
        Face3(0, +1, (1, 2), (1, 2, 3), (_S3, _S3, _S3), True),
        Face3(0, -1, (1, 2), (0, 2, 3), (-1.0, 0.0, 0.0), True),
    ),
}
N_VERTS = {HEX: 8, PRISM: 6, TET: 4}
AXIS_KINDS = {HEX: (pl.GLL,) * 3, PRISM: (pl.GL, pl.GLL, pl.GL), TET: (pl.GL,) * 3}


def n_coeffs(shape, n):
    return {HEX: n ** 3, PRISM: n * n * (n + 1) // 2, TET: n * (n + 1) * (n + 2) // 6}[shape]


# --- collapsed coordinates --------------------------------------------------------------------
def xi_of_eta(shape, eta):
    """Collapsed (eta) -> reference (xi) coordinates."""
    eta = np.asarray(eta, dtype=float)
    xi = eta.copy()
    if shape == PRISM:
        xi[..., 0] = 0.5 * (1.0 + eta[..., 0]) * (1.0 - eta[..., 2]) - 1.0
    elif shape == TET:
        xi[..., 0] = 0.25 * (1.0 + eta[..., 0]) * (1.0 - eta[..., 1]) * (1.0 - eta[..., 2]) - 1.0
        xi[..., 1] = 0.5 * (1.0 + eta[..., 1]) * (1.0 - eta[..., 2]) - 1.0
    return xi


def eta_of_xi(shape, xi):
    xi = np.asarray(xi, dtype=float)
    eta = xi.copy()
    if shape == PRISM:
        eta[..., 0] = 2.0 * (1.0 + xi[..., 0]) / (1.0 - xi[..., 2]) - 1.0
    elif shape == TET:
        eta[..., 1] = 2.0 * (1.0 + xi[..., 1]) / (1.0 - xi[..., 2]) - 1.0
        eta[..., 0] = 2.0 * (1.0 + xi[..., 0]) / (-xi[..., 1] - xi[..., 2]) - 1.0
    return eta


def deta_dxi(shape, eta):
    """Collapse chain d eta_k / d xi_j at points (npts, 3, 3) — the 3-D analogue of
    stdregions.py:428-439."""
    eta = np.atleast_2d(eta)
    out = np.zeros((eta.shape[0], 3, 3))
    out[:, 0, 0] = out[:, 1, 1] = out[:, 2, 2] = 1.0
    e0, e1, e2 = eta[:, 0], eta[:, 1], eta[:, 2]
    if shape == PRISM:
        out[:, 0, 0] = 2.0 / (1.0 - e2)
        out[:, 0, 2] = (1.0 + e0) / (1.0 - e2)
    elif shape == TET:
        a = 2.0 * (1.0 + e0) / ((1.0 - e1) * (1.0 - e2))
        out[:, 0, 0] = 4.0 / ((1.0 - e1) * (1.0 - e2))
        out[:, 0, 1] = a
        out[:, 0, 2] = a
        out[:, 1, 1] = 2.0 / (1.0 - e2)
        out[:, 1, 2] = (1.0 + e1) / (1.0 - e2)
    return out


def dxi_deta(shape, eta):
    """d xi_i / d eta_k at points (npts, 3, 3)."""
    eta = np.atleast_2d(eta)
    out = np.zeros((eta.shape[0], 3, 3))
    out[:, 0, 0] = out[:, 1, 1] = out[:, 2, 2] = 1.0
    e0, e1, e2 = eta[:, 0], eta[:, 1], eta[:, 2]
    if shape == PRISM:
        out[:, 0, 0] = 0.5 * (1.0 - e2)
        out[:, 0, 2] = -0.5 * (1.0 + e0)
    elif shape == TET:
        out[:, 0, 0] = 0.25 * (1.0 - e1) * (1.0 - e2)
        out[:, 0, 1] = -0.25 * (1.0 + e0) * (1.0 - e2)
        out[:, 0, 2] = -0.25 * (1.0 + e0) * (1.0 - e1)
        out[:, 1, 1] = 0.5 * (1.0 - e2)
        out[:, 1, 2] = -0.5 * (1.0 + e1)
    return out


def shape_funcs(shape, xi):
    """Vertex shape functions N (npts, nv) and dN/dxi (npts, nv, 3)."""
    xi = np.atleast_2d(xi)
    x0, x1, x2 = xi[:, 0], xi[:, 1], xi[:, 2]
    npts = xi.shape[0]
    if shape == TET:
        n = np.stack([-0.5 * (1.0 + x0 + x1 + x2), 0.5 * (1 + x0), 0.5 * (1 + x1), 0.5 * (1 + x2)], axis=1)
        dn = np.broadcast_to(np.array([[[-0.5, -0.5, -0.5], [0.5, 0, 0], [0, 0.5, 0], [0, 0, 0.5]]]), (npts, 4, 3))
        return n, np.ascontiguousarray(dn)
    if shape == PRISM:
        la, lb, lc = -0.5 * (x0 + x2), 0.5 * (1 + x0), 0.5 * (1 + x2)
        m0, m1 = 0.5 * (1 - x1), 0.5 * (1 + x1)
        n = np.stack([la * m0, lb * m0, lb * m1, la * m1, lc * m0, lc * m1], axis=1)
        dla, dlb, dlc = np.array([-0.5, 0, -0.5]), np.array([0.5, 0, 0]), np.array([0, 0, 0.5])
        dm0, dm1 = np.array([0, -0.5, 0]), np.array([0, 0.5, 0])
        dn = np.empty((npts, 6, 3))
        for v, (l, dl, m, dm) in enumerate([(la, dla, m0, dm0), (lb, dlb, m0, dm0), (lb, dlb, m1, dm1),
                                             (la, dla, m1, dm1), (lc, dlc, m0, dm0), (lc, dlc, m1, dm1)]):
            dn[:, v, :] = dl[None, :] * m[:, None] + l[:, None] * dm[None, :]
        return n, dn
    ref = np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                    [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], dtype=float)
    terms = 0.5 * (1.0 + xi[:, None, :] * ref[None, :, :])
    n = terms.prod(axis=2)
    dn = np.empty((npts, 8, 3))
    for j in range(3):
        others = [k for k in range(3) if k != j]
        dn[:, :, j] = 0.5 * ref[None, :, j] * terms[:, :, others].prod(axis=2)
    return n, dn


# --- bases -------------------------------------------------------------------------------------
def tri_modes(n):
    """Reference triangle modes (i, j) in tri_flat order (stdregions.py:282-283) and their degree."""
    modes = [(i, j) for i in range(n) for j in range(n - i)]
    return modes, [max(i + j, 1) for i, j in modes]


def tri_eval(n, a, b):
    """Reference modified-modal triangle at paired points (a, b): values and d/da, d/db
    (stdregions.py:286-383)."""
    a = np.atleast_1d(np.asarray(a, dtype=float))
    b = np.atleast_1d(np.asarray(b, dtype=float))
    A, dA = tri_dir1(pl.MODIFIED, n, a)
    nt = n * (n + 1) // 2
    T, Ta, Tb = (np.zeros((a.size, nt)) for _ in range(3))
    for g, (modes, B, dB) in enumerate(tri_groups(pl.MODIFIED, n, b)):
        T[:, modes] = A[:, [g]] * B
        Ta[:, modes] = dA[:, [g]] * B
        Tb[:, modes] = A[:, [g]] * dB
    return T, Ta, Tb


def collapse_fn(d, k, z):
    """C^d_k(z) = ((1-z)/2)^d [k = 0: 1; k >= 1: (1+z)/2 P^{2d-1,1}_{k-1}(z)] and derivative:
    the reference triangle's direction-2 functions (stdregions.py:360-383) for a base
    function of degree d."""
    z = np.asarray(z, dtype=float)
    f = (0.5 * (1.0 - z)) ** d
    df = -0.5 * d * (0.5 * (1.0 - z)) ** (d - 1)
    if k == 0:
        return f, df
    hp = 0.5 * (1.0 + z)
    p, dp = pl.jacobi(2.0 * d - 1.0, 1.0, k - 1, z)
    return f * hp * p, df * hp * p + f * (0.5 * p + hp * dp)


def tet_mode_list(n):
    """[(tri mode index, k)] in DoF order, then the apex (-1, 0)."""
    _, degs = tri_modes(n)
    out = [(m, k) for m, d in enumerate(degs) for k in range(n - d)]
    return out + [(-1, 0)]


def basis_eval(shape, n, eta):
    """Values (npts, nc) and eta-derivatives [3 x (npts, nc)] of the modified-modal basis."""
    eta = np.atleast_2d(np.asarray(eta, dtype=float))
    npts = eta.shape[0]
    nc = n_coeffs(shape, n)
    if shape == HEX:
        tabs = [pl.modified(n, eta[:, a]) for a in range(3)]
        out = []
        for der in (None, 0, 1, 2):
            m = None
            for a in range(3):
                t = tabs[a][1] if der == a else tabs[a][0]
                m = t if m is None else np.einsum("pi,pj->pij", m, t).reshape(npts, -1)
            out.append(m)
        return out[0], out[1:]
    if shape == PRISM:
        T, Ta, Tb = tri_eval(n, eta[:, 0], eta[:, 2])
        psi, dpsi = pl.modified(n, eta[:, 1])

        def outer(t, p):
            return np.einsum("pm,pl->pml", t, p).reshape(npts, nc)
        return outer(T, psi), [outer(Ta, psi), outer(T, dpsi), outer(Tb, psi)]
    T, Ta, Tb = tri_eval(n, eta[:, 0], eta[:, 1])
    _, degs = tri_modes(n)
    phi = np.zeros((npts, nc))
    d = [np.zeros((npts, nc)) for _ in range(3)]
    for col, (m, k) in enumerate(tet_mode_list(n)):
        if m < 0:
            phi[:, col] = 0.5 * (1.0 + eta[:, 2])
            d[2][:, col] = 0.5
            continue
        c, dc = collapse_fn(degs[m], k, eta[:, 2])
        phi[:, col] = T[:, m] * c
        d[0][:, col] = Ta[:, m] * c
        d[1][:, col] = Tb[:, m] * c
        d[2][:, col] = T[:, m] * dc
    return phi, d


def tensor_params(axes):
    g = np.meshgrid(*axes, indexing="ij")
    return np.stack([a.reshape(-1) for a in g], axis=-1)


class Expansion3:
    """A (shape, n_modes, n_quad) discretisation: volume rule, dense basis tables,
    collocation derivatives (the reference's BwdTrans / PhysDeriv / IProduct /
    IProductDeriv, stdregions.py:566-674, as dense products)."""

    def __init__(self, shape, n, q):
        self.shape, self.n, self.q = shape, n, q
        self.kinds = AXIS_KINDS[shape]
        self.rules = [pl.rule(k, q) for k in self.kinds]
        self.pts = [r[0] for r in self.rules]
        self.eta = tensor_params(self.pts)
        w = np.einsum("i,j,k->ijk", *[r[1] for r in self.rules]).reshape(-1)
        if shape == PRISM:
            w = w * 0.5 * (1.0 - self.eta[:, 2])
        elif shape == TET:
            w = w * 0.5 * (1.0 - self.eta[:, 1]) * (0.5 * (1.0 - self.eta[:, 2])) ** 2
        self.ref_w = w
        self.xi = xi_of_eta(shape, self.eta)
        self.n_phys = q ** 3
        self.n_coeffs = n_coeffs(shape, n)
        self.Phi, self.dPhi = basis_eval(shape, n, self.eta)
        self.D = [pl.dmat(p) for p in self.pts]
        self.chain = deta_dxi(shape, self.eta)
        self.faces = FACES3[shape]

    def bwd(self, c):
        return self.Phi @ c

    def deriv(self, u):
        w = u.shape[-1]
        t = u.reshape(self.q, self.q, self.q, w)
        return [np.moveaxis(np.tensordot(self.D[a], t, axes=(1, a)), 0, a).reshape(self.n_phys, w)
                for a in range(3)]

    def iprod(self, f):
        return self.Phi.T @ f

    def iprod_d(self, k, f):
        return self.dPhi[k].T @ f

    def face_grid(self, f):
        """Own face grid: parameters (npts, 2) and weights (npts,)."""
        face = self.faces[f]
        a, b = face.run
        prm = tensor_params([self.pts[a], self.pts[b]])
        w = np.multiply.outer(self.rules[a][1], self.rules[b][1]).reshape(-1)
        return prm, w


@functools.lru_cache(maxsize=None)
def expansion3(shape, n, q):
    return Expansion3(shape, n, q)


def face_to_eta(face, prm):
    prm = np.atleast_2d(prm)
    eta = np.empty((prm.shape[0], 3))
    eta[:, face.fixed] = float(face.side)
    eta[:, face.run[0]] = prm[:, 0]
    eta[:, face.run[1]] = prm[:, 1]
    return eta


# --- topology (dict-based: the check on the product's vectorised matcher) -----------------------
def build_couplings(shapes, elem_verts):
    """Interfaces of a 3-D hybrid mesh, as [(left (e, f), right (e, f) | None, kind)], kind in
    {"conform", "subface", "boundary"}, ordered by (left e, left f, right e, right f).
    conform: identical corner sets (left = lower element id); subface: a triangle
    (left) inside a quad face (right) of a split-cube neighbour; boundary: unmatched."""
    tri_of, quad_of = {}, {}
    for e, (s, vs) in enumerate(zip(shapes, elem_verts)):
        for f, face in enumerate(FACES3[s]):
            key = tuple(sorted(vs[c] for c in face.corners))
            (tri_of if face.tri else quad_of).setdefault(key, []).append((e, f))
    out = []
    covered = set()
    for table in (tri_of, quad_of):
        for key, sides in table.items():
            if len(sides) > 2:
                raise ValueError("face shared by more than two elements")
            if len(sides) == 2:
                a, b = sorted(sides)
                out.append((a, b, "conform"))
                covered.update(sides)
    for key, sides in quad_of.items():
        if len(sides) != 1:
            continue
        subs = [tri_of[t][0] for t in (tuple(sorted(c)) for c in _subsets3(key)) if t in tri_of and len(tri_of[t]) == 1]
        if subs:
            if len(subs) != 2:
                raise ValueError("quad face not covered by exactly two triangles")
            for t in subs:
                out.append((t, sides[0], "subface"))
                covered.add(t)
            covered.add(sides[0])
    for e, s in enumerate(shapes):
        for f in range(len(FACES3[s])):
            if (e, f) not in covered:
                out.append(((e, f), None, "boundary"))
    out.sort(key=lambda t: (t[0][0], t[0][1], -1 if t[1] is None else t[1][0], -1 if t[1] is None else t[1][1]))
    return out


def _subsets3(key):
    return [tuple(v for j, v in enumerate(key) if j != i) for i in range(4)]


# --- the operator --------------------------------------------------------------------------------
class HybridOracle3D:
    """y = (lambda M + L_SIP) x on a 3-D hybrid mesh: `shapes` (list of "hex"/"prism"/"tet"),
    `elem_verts` (list of vertex-id tuples in the shapes' local order), `vertices` (nv, 3),
    `n_modes`, `n_quad` per element.  Affine elements only (cube-split meshes)."""

    def __init__(self, shapes, elem_verts, vertices, n_modes, n_quad, lambda_=1.0, couplings=None):
        self.lam = float(lambda_)
        self.shapes = list(shapes)
        self.elem_verts = [tuple(int(v) for v in vs) for vs in elem_verts]
        self.X = np.asarray(vertices, dtype=float)
        self.nm = np.asarray(n_modes, dtype=int)
        self.nq = np.asarray(n_quad, dtype=int)
        nel = len(self.shapes)
        self.exps = [expansion3(self.shapes[e], int(self.nm[e]), int(self.nq[e])) for e in range(nel)]
        self.dof_off = np.zeros(nel + 1, dtype=np.int64)
        self.dof_off[1:] = np.cumsum([ex.n_coeffs for ex in self.exps])
        self.n_dofs = int(self.dof_off[-1])
        # affine maps: x = x0 + F (xi + 1)
        self.F = np.empty((nel, 3, 3))
        self.x0 = np.empty((nel, 3))
        for s in SHAPES:
            ids = np.array([e for e in range(nel) if self.shapes[e] == s], dtype=np.int64)
            if ids.size == 0:
                continue
            V = self.X[np.array([self.elem_verts[e] for e in ids])]            # (W, nv, 3)
            _, dn = shape_funcs(s, np.array([[-1.0, -1.0, -1.0]]))
            self.F[ids] = np.einsum("vj,evi->eij", dn[0], V)
            n0, _ = shape_funcs(s, np.array([[-1.0, -1.0, -1.0]]))
            self.x0[ids] = np.einsum("v,evi->ei", n0[0], V)
            # affine check at the opposite corner
            n1, dn1 = shape_funcs(s, np.array([[0.3, -0.2, 0.1]]) if s != TET else np.array([[-0.5, -0.4, -0.3]]))
            F1 = np.einsum("vj,evi->eij", dn1[0], V)
            if not np.allclose(F1, self.F[ids], atol=1e-12 * np.abs(self.F[ids]).max()):
                raise ValueError("non-affine element: the hybrid oracle supports affine elements only")
        self.detJ = np.abs(np.linalg.det(self.F))
        if np.any(self.detJ <= 0.0):
            raise ValueError("degenerate element")
        self.dxidx = np.linalg.inv(self.F)                                         # [e, j, m] = dxi_j/dx_m
        self.classes = {}
        for e in range(nel):
            self.classes.setdefault((self.shapes[e], int(self.nm[e]), int(self.nq[e])), []).append(e)
        self.vol = np.array([self.detJ[e] * self.exps[e].ref_w.sum() for e in range(nel)])
        self.couplings = couplings if couplings is not None else build_couplings(self.shapes, self.elem_verts)
        self._build_faces()

    # -- geometry helpers ------------------------------------------------------------------------
    def _face_frame(self, elems, face, eta, weights):
        """Normal (W, 3) [constant on affine faces, taken at point 0], swj (W, npts) for the
        faces `face` of elements `elems` at eta points of that face."""
        shape = self.shapes[int(elems[0])]
        J = dxi_deta(shape, eta)                                                   # (p, i, k)
        F = self.F[elems]                                                          # (W, i, j)
        ta = np.einsum("wij,pj->wpi", F, J[:, :, face.run[0]])
        tb = np.einsum("wij,pj->wpi", F, J[:, :, face.run[1]])
        cr = np.cross(ta, tb)
        surf = np.linalg.norm(cr, axis=2)
        nrm = cr[:, 0, :] / surf[:, :1]
        out_dir = np.einsum("wji,j->wi", self.dxidx[elems], np.asarray(face.ref_normal))
        sgn = np.where(np.einsum("wi,wi->w", nrm, out_dir) >= 0.0, 1.0, -1.0)
        return nrm * sgn[:, None], surf * weights[None, :]

    def _gn(self, elems, eta, nrm):
        """(G n)_k = sum_m (d eta_k/d x_m) n_m at points: (3, W, npts)."""
        shape = self.shapes[int(elems[0])]
        ch = deta_dxi(shape, eta)                                                  # (p, k, j)
        G = np.einsum("pkj,wjm->wpkm", ch, self.dxidx[elems])
        return np.einsum("wpkm,wm->kwp", G, nrm)

    def face_area(self, e, f):
        ex = self.exps[e]
        prm, w = ex.face_grid(f)
        eta = face_to_eta(ex.faces[f], prm)
        _, swj = self._face_frame(np.array([e]), ex.faces[f], eta, w)
        return float(swj.sum())

    # -- setup -----------------------------------------------------------------------------------
    def _build_faces(self):
        self.groups = []
        buckets = {}
        for (l, r, kind) in self.couplings:
            le, lf = l
            cl = (self.shapes[le], int(self.nm[le]), int(self.nq[le]))
            if r is None:
                buckets.setdefault(("b", cl, lf), []).append((l, r))
            else:
                re_, rf = r
                cr = (self.shapes[re_], int(self.nm[re_]), int(self.nq[re_]))
                buckets.setdefault((kind, cl, lf, cr, rf), []).append((l, r))
        for key, items in buckets.items():
            self.groups.append(self._group(key, items))

    def _tau(self, le, lf, re_=None, rf=None):
        h = self.vol[le] / self.face_area(le, lf)
        nmax = self.nm[le]
        if re_ is not None:
            h = min(h, self.vol[re_] / self.face_area(re_, rf))
            nmax = max(nmax, self.nm[re_])
        return float(nmax * nmax) / h

    def _group(self, key, items):
        el = np.array([l[0] for l, _ in items], dtype=np.int64)
        lf = items[0][0][1]
        exl = self.exps[int(el[0])]
        facel = exl.faces[lf]
        g = {"key": key, "el": el}
        if key[0] == "b":
            prm, w = exl.face_grid(lf)
            g["tau"] = np.array([self._tau(int(e), lf) for e in el])[:, None]
        else:
            er = np.array([r[0] for _, r in items], dtype=np.int64)
            rf = items[0][1][1]
            exr = self.exps[int(er[0])]
            qt = max(exl.q, exr.q)
            if facel.tri:
                kinds = (pl.GL, pl.GL)
            else:
                both_gll = all(exl.kinds[a] == pl.GLL for a in facel.run) and \
                    all(exr.kinds[a] == pl.GLL for a in exr.faces[rf].run)
                kinds = (pl.GLL, pl.GLL) if both_gll else (pl.GL, pl.GL)
            ra, rb = pl.rule(kinds[0], qt), pl.rule(kinds[1], qt)
            prm = tensor_params([ra[0], rb[0]])
            w = np.multiply.outer(ra[1], rb[1]).reshape(-1)
            g["tau"] = np.array([self._tau(int(a), lf, int(b), rf) for a, b in zip(el, er)])[:, None]
            g["er"] = er
            g["rf"] = rf
        eta_l = face_to_eta(facel, prm)
        nrm, swj = self._face_frame(el, facel, eta_l, w)
        g["swj"] = swj
        g["B_l"], g["D_l"] = basis_eval(exl.shape, exl.n, eta_l)
        g["gn_l"] = self._gn(el, eta_l, nrm)
        g["dofs_l"] = self.dof_off[el][:, None] + np.arange(exl.n_coeffs)[None, :]
        if key[0] == "b":
            return g
        # right side: map the trace points through the geometry, group identical parameter sets
        xi_l = xi_of_eta(exl.shape, eta_l)
        x = self.x0[el][:, None, :] + np.einsum("wij,pj->wpi", self.F[el], xi_l + 1.0)
        xi_r = np.einsum("wjm,wpm->wpj", self.dxidx[er], x - self.x0[er][:, None, :]) - 1.0
        eta_r = eta_of_xi(exr.shape, xi_r)
        facer = exr.faces[rf]
        if np.abs(eta_r[..., facer.fixed] - facer.side).max() > 1e-9:
            raise ValueError("trace points do not lie on the right face")
        eta_r[..., facer.fixed] = float(facer.side)
        keys = np.round(eta_r, 10).reshape(len(er), -1)
        _, first, inv = np.unique(keys, axis=0, return_index=True, return_inverse=True)
        g["variant"] = inv.reshape(-1)
        g["B_r"], g["D_r"] = [], []
        for i in first:
            B, D = basis_eval(exr.shape, exr.n, eta_r[i])
            g["B_r"].append(B)
            g["D_r"].append(D)
        gn_r = np.empty((3, len(er), prm.shape[0]))
        for v, i in enumerate(first):
            sel = g["variant"] == v
            gn_r[:, sel] = self._gn(er[sel], eta_r[i], -nrm[sel])
        g["gn_r"] = gn_r
        g["dofs_r"] = self.dof_off[er][:, None] + np.arange(exr.n_coeffs)[None, :]
        return g

    # -- apply -----------------------------------------------------------------------------------
    def lhs_eval(self, x):
        """The reference's lhs_eval (sipg.py:558-602) on the hybrid mesh."""
        x = np.asarray(x, dtype=float)
        if x.shape != (self.n_dofs,):
            raise ValueError(f"expected a vector of length {self.n_dofs}")
        out = np.zeros(self.n_dofs)
        for (s, n, q), ids in self.classes.items():
            ex = self.exps[ids[0]]
            ids = np.asarray(ids)
            dof = self.dof_off[ids][None, :] + np.arange(ex.n_coeffs)[:, None]
            jw = ex.ref_w[:, None] * self.detJ[ids][None, :]                          # (p, W)
            G = np.einsum("pkj,wjm->kmpw", ex.chain, self.dxidx[ids])              # (k, m, p, W)
            u = ex.bwd(x[dof])
            du = ex.deriv(u)
            dux = [sum(G[k, m] * du[k] for k in range(3)) for m in range(3)]
            acc = ex.iprod(u * (self.lam * jw))
            for k in range(3):
                acc = acc + ex.iprod_d(k, sum(G[k, m] * dux[m] for m in range(3)) * jw)
            out[dof] = acc
        for g in self.groups:
            xl = x[g["dofs_l"]]
            ul = xl @ g["B_l"].T
            gl = sum(g["gn_l"][k] * (xl @ g["D_l"][k].T) for k in range(3))
            if g["key"][0] == "b":
                self._absorb(out, g["dofs_l"], g["B_l"], g["D_l"], g["gn_l"], g["tau"], g["swj"], 2.0 * ul, gl)
                continue
            xr = x[g["dofs_r"]]
            ur = np.empty_like(ul)
            gr = np.empty_like(ul)
            for v in range(len(g["B_r"])):
                sel = g["variant"] == v
                ur[sel] = xr[sel] @ g["B_r"][v].T
                gr[sel] = sum(g["gn_r"][k][sel] * (xr[sel] @ g["D_r"][v][k].T) for k in range(3))
            j = ul - ur
            c = 0.5 * (gl - gr)
            self._absorb(out, g["dofs_l"], g["B_l"], g["D_l"], g["gn_l"], g["tau"], g["swj"], j, c)
            for v in range(len(g["B_r"])):
                sel = g["variant"] == v
                self._absorb(out, g["dofs_r"][sel], g["B_r"][v], g["D_r"][v], g["gn_r"][:, sel],
                             g["tau"][sel], g["swj"][sel], -j[sel], -c[sel])
        return out

    __call__ = lhs_eval

    @staticmethod
    def _absorb(out, dofs, B, D, gn, tau, swj, jump, avg):
        """sipg.py:663-677 (TraceIProduct branch)."""
        fv = (tau * jump - avg) * swj
        fd = -0.5 * jump * swj
        contrib = fv @ B
        for k in range(3):
            contrib += (fd * gn[k]) @ D[k]
        np.add.at(out, dofs, contrib)


# --- right-hand side and error (reference sipg.py:697-741, restated on the hybrid machinery) -----
def _rhs_l2_methods():
    def phys_points(self, e, ex):
        """Physical coordinates (3, n_pts) of an expansion's volume points in element e."""
        return (self.x0[e][:, None] + self.F[e] @ (ex.xi.T + 1.0))

    def rhs_assemble(self, case, bcs):
        """b = -(v, f) plus the Dirichlet lift of the mirror ghost state (sipg.py:697-718): volume
        IProduct of the forcing, and on boundary faces the absorb of jump = -2 g, average 0 with
        sign -1 (TraceIProduct branch)."""
        b = np.zeros(self.n_dofs)
        for (s, n, q), ids in self.classes.items():
            ex = self.exps[ids[0]]
            ids = np.asarray(ids)
            xs = np.stack([phys_points(self, e, ex) for e in ids], axis=-1)            # (3, p, W)
            f = case.forcing(xs)
            jw = ex.ref_w[:, None] * self.detJ[ids][None, :]
            dof = self.dof_off[ids][None, :] + np.arange(ex.n_coeffs)[:, None]
            b[dof] = -ex.iprod(f * jw)
        for g in self.groups:
            if g["key"][0] != "b":
                continue
            gfun = bcs["dirichlet"]
            el = g["el"]
            exl = self.exps[int(el[0])]
            prm, _ = exl.face_grid(g["key"][2])
            eta = face_to_eta(exl.faces[g["key"][2]], prm)
            xi = xi_of_eta(exl.shape, eta)
            gv = np.stack([gfun(self.x0[e][:, None] + self.F[e] @ (xi.T + 1.0)) for e in el])   # (W, nf)
            jump, avg, sign = -2.0 * gv, 0.0 * gv, -1.0
            fv = (g["tau"] * jump - avg) * g["swj"] * sign
            fd = (-0.5 * sign) * jump * g["swj"]
            contrib = fv @ g["B_l"]
            for k in range(3):
                contrib += (fd * g["gn_l"][k]) @ g["D_l"][k]
            np.add.at(b, g["dofs_l"], contrib)
        return b

    def l2_error(self, x, exact):
        """sqrt(sum_e int (u_h - u)^2 J) on rules with 2 extra points per direction (sipg.py:720-741)."""
        err2 = 0.0
        for (s, n, q), ids in self.classes.items():
            fine = expansion3(s, n, q + 2)
            ids = np.asarray(ids)
            dof = self.dof_off[ids][None, :] + np.arange(fine.n_coeffs)[:, None]
            uh = fine.bwd(np.asarray(x)[dof])
            xs = np.stack([phys_points(self, e, fine) for e in ids], axis=-1)
            diff = uh - exact(xs)
            err2 += float((diff * diff * fine.ref_w[:, None] * self.detJ[ids][None, :]).sum())
        return math.sqrt(err2)

    return rhs_assemble, l2_error


HybridOracle3D.rhs_assemble, HybridOracle3D.l2_error = _rhs_l2_methods()
