"""Plan builder for 3-D hybrid hex / prism / tet meshes (config 4).

Flattens a `mesh3d.HybridMesh3D` + `OrderMap` into the device plan of
`csrc/sipg_h3.cuh` (C-ABI `sipg_h3_plan_create`, include/sipg.h).  The
algorithm is the reference's shared-trace SIP apply (sipg.py:513-554,
653-693) extended to prisms and tets as restated in oracle/hybrid3d.py; this
module is an independent vectorised restatement (it never imports the oracle).

Layout (all element-major, element ids = mesh order = DoF order):
* classes (shape, n): one kernel launch each; q = n + 1 (the BASELINE rule).
* element geometry, 8 doubles: |det F|, S = (dxi/dx)(dxi/dx)^T (6, symmetric),
  pad — affine elements only.
* slots, 96 B (`SLOT`): one per (element, coupling it takes part in) — a
  subface quad carries two — sorted by (element, face): the face, boundary or
  interior, trace size nt, own-face-grid -> trace map (identity or a dense
  nt x q^2 matrix in the table pool), trace-weight table, tau, the constant
  surface Jacobian sJ (swj = sJ * wt[p], wt holding the collapsed-triangle
  Duffy factor), v = (dxi/dx) n (n = the left side's outward unit normal, -n on
  the right side, sipg.py:545), and the published-trace offsets of this slot and
  of its partner.
* published traces: per slot, (u, n.grad u) interleaved at the trace points (phase 1 writes them,
  phase 2 reads its own and its partner's).
"""
from __future__ import annotations

import math

import numpy as np

from .polylib import BasisKind, QuadKind, diff_matrix, eval_basis_1d, jacobi_eval, lagrange_interp_matrix, \
    quad_rule
from .stdregions import tri_tables

GL, GLL = QuadKind.GAUSS_LEGENDRE, QuadKind.GAUSS_LOBATTO
HEX, PRISM, TET = "hex", "prism", "tet"
SHAPE_ID = {HEX: 0, PRISM: 1, TET: 2}
AXIS_KINDS = {HEX: (GLL, GLL, GLL), PRISM: (GL, GLL, GL), TET: (GL, GL, GL)}

H3_ABI_VERSION = 1
# class descriptor words (int32[CD3_WORDS]) — csrc/sipg_h3.cuh
CD3_WORDS = 16
(CD3_SHAPE, CD3_N, CD3_Q, CD3_NC, CD3_COUNT, CD3_ELEM_OFF, CD3_T_PTS, CD3_T_D, CD3_T_W, CD3_T_E,
 CD3_T_A, CD3_T_B, CD3_T_C, CD3_ROLE, CD3_T_R, CD3_T_ED) = range(16)
NSMAX = {"hex": 12, "prism": 8, "tet": 4}     # slots per element (subface quads carry two)

SLOT = np.dtype([
    ("face", "<i4"), ("kind", "<i4"), ("nt", "<i4"), ("mkind", "<i4"),
    ("moff", "<i4"), ("moff2", "<i4"), ("nab", "<i4"), ("wtoff", "<i4"),
    ("elem", "<i4"), ("partner", "<i4"),
    ("pub_self", "<i8"), ("pub_other", "<i8"),
    ("tau", "<f8"), ("sJ", "<f8"), ("v", "<f8", (3,)),
])
assert SLOT.itemsize == 96
# trace maps (own face grid q x q -> trace points): 0 identity, 1 tensor X (n1 x q) then Y (n2 x q)
# with trace index r1 * n2 + r2 (or r2 * n1 + r1 when swapped; nab = n1 | n2 << 8 | swap << 16),
# 2 dense (nt x q^2, subface quad sides)
# 3 row (subface quad side): the trace's second axis (collapsed b) fixes the own axis `perp`
# (Y[pb] over it), the own axis `par` varies along each trace row (X[pb][pa] over it);
# nab = nta | ntb << 8 | perp << 16
MAP_ID, MAP_TENSOR, MAP_DENSE, MAP_ROW = 0, 1, 2, 3
EGEO_STRIDE = 8

# faces: (fixed eta axis, side, run axes, triangular, outward normal in xi) — oracle FACES3 order
_S2, _S3 = math.sqrt(0.5), math.sqrt(1.0 / 3.0)
FACES = {
    HEX: ((0, -1, (1, 2), False, (-1, 0, 0)), (0, 1, (1, 2), False, (1, 0, 0)),
          (1, -1, (0, 2), False, (0, -1, 0)), (1, 1, (0, 2), False, (0, 1, 0)),
          (2, -1, (0, 1), False, (0, 0, -1)), (2, 1, (0, 1), False, (0, 0, 1))),
    PRISM: ((2, -1, (0, 1), False, (0, 0, -1)), (1, -1, (0, 2), True, (0, -1, 0)),
            (0, 1, (1, 2), False, (_S2, 0, _S2)), (1, 1, (0, 2), True, (0, 1, 0)),
            (0, -1, (1, 2), False, (-1, 0, 0))),
    TET: ((2, -1, (0, 1), True, (0, 0, -1)), (1, -1, (0, 2), True, (0, -1, 0)),
          (0, 1, (1, 2), True, (_S3, _S3, _S3)), (0, -1, (1, 2), True, (-1, 0, 0))),
}
REF_VERTS = {
    HEX: np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                   [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], dtype=float),
    PRISM: np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1], [-1, -1, 1], [-1, 1, 1]], dtype=float),
    TET: np.array([[-1, -1, -1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], dtype=float),
}
# vertices spanning the xi axes from V0: x = V0 + F (xi + 1), F[:, a] = (V_axis[a] - V0) / 2
AXIS_VERTS = {HEX: (1, 3, 4), PRISM: (1, 3, 4), TET: (1, 2, 3)}


def n_coeffs(shape, n):
    return {HEX: n ** 3, PRISM: n * n * (n + 1) // 2, TET: n * (n + 1) * (n + 2) // 6}[shape]


def tri_degrees(n):
    return [max(i + j, 1) for i in range(n) for j in range(n - i)]


def collapse_rows(d, nk, z):
    """((1-z)/2)^d [1, (1+z)/2 P^{2d-1,1}_{k-1}(z)] for k < nk — the reference triangle's
    direction-2 family (stdregions.py:360-383) for a base function of degree d."""
    f = (0.5 * (1.0 - z)) ** d
    rows = [f]
    for k in range(1, nk):
        p, _ = jacobi_eval(2.0 * d - 1.0, 1.0, k - 1, z)
        rows.append(f * 0.5 * (1.0 + z) * p)
    return rows


def xi_of_eta(shape, eta):
    xi = eta.copy()
    if shape == PRISM:
        xi[..., 0] = 0.5 * (1.0 + eta[..., 0]) * (1.0 - eta[..., 2]) - 1.0
    elif shape == TET:
        xi[..., 0] = 0.25 * (1.0 + eta[..., 0]) * (1.0 - eta[..., 1]) * (1.0 - eta[..., 2]) - 1.0
        xi[..., 1] = 0.5 * (1.0 + eta[..., 1]) * (1.0 - eta[..., 2]) - 1.0
    return xi


def eta_of_xi(shape, xi):
    eta = xi.copy()
    if shape == PRISM:
        eta[..., 0] = 2.0 * (1.0 + xi[..., 0]) / (1.0 - xi[..., 2]) - 1.0
    elif shape == TET:
        eta[..., 1] = 2.0 * (1.0 + xi[..., 1]) / (1.0 - xi[..., 2]) - 1.0
        eta[..., 0] = 2.0 * (1.0 + xi[..., 0]) / (-xi[..., 1] - xi[..., 2]) - 1.0
    return eta


def dxi_deta(shape, eta):
    """d xi_i / d eta_k at one point (3, 3)."""
    e0, e1, e2 = eta
    J = np.eye(3)
    if shape == PRISM:
        J[0, 0], J[0, 2] = 0.5 * (1.0 - e2), -0.5 * (1.0 + e0)
    elif shape == TET:
        J[0, 0] = 0.25 * (1.0 - e1) * (1.0 - e2)
        J[0, 1] = -0.25 * (1.0 + e0) * (1.0 - e2)
        J[0, 2] = -0.25 * (1.0 + e0) * (1.0 - e1)
        J[1, 1], J[1, 2] = 0.5 * (1.0 - e2), -0.5 * (1.0 + e1)
    return J


def _face_cross_xi(shape, fixed, side, run):
    """d xi/d eta_run0 x d xi/d eta_run1 on the face at run0 = run1 = -1: constant on quads; on a
    collapsed triangle the product is this value times the Duffy factor (1 - eta_run1)/2."""
    eta = np.full(3, -1.0)
    eta[fixed] = side
    J = dxi_deta(shape, eta)
    return np.cross(J[:, run[0]], J[:, run[1]])


class ClassTables3:
    def __init__(self, shape, n, q):
        self.shape, self.n, self.q = shape, n, q
        kinds = AXIS_KINDS[shape]
        self.kinds = kinds
        self.rules = [quad_rule(k, q) for k in kinds]
        self.n_modes, self.nq, self.n_phys = n, (q, q, q), q ** 3
        self.pts = [r.points for r in self.rules]
        self.wts = [r.weights for r in self.rules]
        g = np.meshgrid(*self.pts, indexing="ij")
        eta = np.stack([a.reshape(-1) for a in g], axis=-1)
        w = np.einsum("i,j,k->ijk", *self.wts).reshape(-1)
        if shape == PRISM:
            w = w * 0.5 * (1.0 - eta[:, 2])
        elif shape == TET:
            w = w * 0.5 * (1.0 - eta[:, 1]) * (0.5 * (1.0 - eta[:, 2])) ** 2
        self.wref = w
        self.nc = n_coeffs(shape, n)
        self.n_coeffs, self.ref_weights, self.eta_phys = self.nc, w, eta
        self.xi_phys = xi_of_eta(shape, eta)
        E = [lagrange_interp_matrix(p, [sd])[0] for p in self.pts for sd in (-1.0, 1.0)]
        Dm = [diff_matrix(p) for p in self.pts]
        parts = {"pts": np.concatenate(self.pts),
                 # 1 / (1 - eta) for the collapse chain (used on the GL collapsed axes only)
                 "R": np.concatenate([np.where(p < 1.0, 1.0 / np.maximum(1.0 - p, 1e-300), 0.0) for p in self.pts]),
                 "ED": np.concatenate([E[2 * a + sd] @ Dm[a] for a in range(3) for sd in (0, 1)]),
                 "WA": np.concatenate(self.wts),
                 "D": np.concatenate([diff_matrix(p).reshape(-1) for p in self.pts]),
                 # volume weights w0[k0] * (w1 w2 Duffy)[k1, k2] (the Duffy factor depends on eta1, eta2)
                 "W": np.concatenate([self.wts[0], (w.reshape(q, q, q)[0] / self.wts[0][0]).reshape(-1)]),
                 "E": np.concatenate([lagrange_interp_matrix(p, [s])[0] for p in self.pts for s in (-1.0, 1.0)])}
        mm = BasisKind.MODIFIED_MODAL
        if shape == HEX:
            parts["A"] = eval_basis_1d(mm, n, self.pts[0])[0].reshape(-1)                # (Q, N)
        else:
            zb = self.pts[2] if shape == PRISM else self.pts[1]
            A, _, B, _, _ = tri_tables(mm, n, self.pts[0], zb)
            parts["A"] = A.reshape(-1)                                                  # (Q, N+1)
            rows = [B[:, m] for m in range(B.shape[1])]
            if shape == TET:
                rows.append(np.ones(q))                                                 # apex pseudo-mode
                C = []
                for d in tri_degrees(n):
                    C += collapse_rows(d, n - d, self.pts[2])
                C.append(0.5 * (1.0 + self.pts[2]))                                      # apex
                parts["C"] = np.concatenate(C)                                           # (NTET, Q)
            else:
                parts["C"] = eval_basis_1d(mm, n, self.pts[1])[0].reshape(-1)           # psi (Q, N)
            parts["B"] = np.concatenate(rows)
        self.parts = parts
        # face data: own grid weights (with the Duffy factor) and the xi-space cross product
        self.face_wt, self.face_cross = [], []
        for fixed, side, run, tri, _ in FACES[shape]:
            wt = np.multiply.outer(self.wts[run[0]], self.wts[run[1]])
            if tri:
                wt = wt * 0.5 * (1.0 - self.pts[run[1]])[None, :]
            self.face_wt.append(wt.reshape(-1))
            self.face_cross.append(_face_cross_xi(shape, fixed, side, run))


_CT_CACHE = {}


def _class_tables(shape, n):
    if (shape, n) not in _CT_CACHE:
        _CT_CACHE[(shape, n)] = ClassTables3(shape, n, n + 1)
    return _CT_CACHE[(shape, n)]


class Pool:
    """Deduplicating double pool."""

    def __init__(self):
        self.chunks, self.size, self.index = [], 0, {}

    def add(self, arr, key=None):
        arr = np.ascontiguousarray(arr, dtype=np.float64).reshape(-1)
        k = key if key is not None else arr.tobytes()
        if k in self.index:
            return self.index[k]
        off = self.size
        self.chunks.append(arr)
        self.size += arr.size
        self.index[k] = off
        return off

    def array(self):
        return np.concatenate(self.chunks) if self.chunks else np.zeros(1)


class Plan3DBuilder:
    """Vectorised flattening of a hybrid 3-D mesh into the h3 device plan."""
    is_h3 = True

    def __init__(self, mesh, order_map, *, lambda_=1.0, element_roles=None):
        self.mesh = mesh
        self.lam = float(lambda_)
        self.shapes = [el.shape.value for el in mesh.elements]
        self.nm = np.asarray(order_map.n_modes, dtype=np.int64)
        self.nq = np.asarray(order_map.n_quad, dtype=np.int64)
        if np.any(self.nq != self.nm + 1):
            raise ValueError("hybrid 3-D plans use n_quad = n_modes + 1 (the BASELINE rule)")
        if np.any(self.nm < 2) or np.any(self.nm > 7):
            raise ValueError("hybrid 3-D kernels are instantiated for 2 <= n_modes <= 7")
        self.roles = None if element_roles is None else np.asarray(element_roles, dtype=np.int64)

    def build(self):
        nel = len(self.shapes)
        sid = np.array([SHAPE_ID[s] for s in self.shapes], dtype=np.int64)
        self.sid = sid
        nc = np.array([n_coeffs(s, int(n)) for s, n in zip(self.shapes, self.nm)], dtype=np.int64)
        self.dof_off = np.zeros(nel + 1, dtype=np.int64)
        self.dof_off[1:] = np.cumsum(nc)
        self.n_dofs = int(self.dof_off[-1])
        self.pool = Pool()
        self._geometry()
        self._classes()
        self._slots()
        self.tables = self.pool.array()
        return self

    # -- geometry ---------------------------------------------------------------------------------
    def _geometry(self):
        X = np.asarray(self.mesh.vertices, dtype=float)
        nel = len(self.shapes)
        self.F = np.zeros((nel, 3, 3))
        self.x0 = np.zeros((nel, 3))
        for s in (HEX, PRISM, TET):
            ids = np.flatnonzero(self.sid == SHAPE_ID[s])
            if ids.size == 0:
                continue
            V = X[np.array([self.mesh.elements[e].verts for e in ids], dtype=np.int64)]   # (W, nv, 3)
            av = AXIS_VERTS[s]
            F = np.stack([(V[:, a] - V[:, 0]) * 0.5 for a in av], axis=2)                 # (W, 3, 3)
            pred = V[:, :1] + np.einsum("wij,vj->wvi", F, REF_VERTS[s] + 1.0)
            scale = np.abs(V).max() + 1.0
            if np.abs(pred - V).max() > 1e-12 * scale:
                raise ValueError("hybrid 3-D plans support affine elements only")
            self.F[ids] = F
            self.x0[ids] = V[:, 0]
        det = np.linalg.det(self.F)
        if np.any(np.abs(det) <= 0.0):
            raise ValueError("degenerate element")
        self.detJ = np.abs(det)
        self.dxidx = np.linalg.inv(self.F)                                                   # [e, j, m]
        S = np.einsum("ejm,ekm->ejk", self.dxidx, self.dxidx)
        eg = np.zeros((nel, EGEO_STRIDE))
        eg[:, 0] = self.detJ
        eg[:, 1:7] = S[:, [0, 0, 0, 1, 1, 2], [0, 1, 2, 1, 2, 2]]
        self.egeo = eg

    # -- classes / tables -------------------------------------------------------------------------
    def _classes(self):
        roles = np.zeros(len(self.shapes), dtype=np.int64) if self.roles is None else self.roles
        keys = sorted(set(zip(self.sid.tolist(), self.nm.tolist(), roles.tolist())))
        self.class_of = np.zeros(len(self.shapes), dtype=np.int64)
        cd = np.zeros((len(keys), CD3_WORDS), dtype=np.int32)
        elems, self.ct = [], []
        off = 0
        names = {v: k for k, v in SHAPE_ID.items()}
        for c, (s, n, role) in enumerate(keys):
            ids = np.flatnonzero((self.sid == s) & (self.nm == n) & (roles == role))
            self.class_of[ids] = c
            ct = _class_tables(names[s], n)
            self.ct.append(ct)
            cd[c, [CD3_SHAPE, CD3_N, CD3_Q, CD3_NC, CD3_COUNT, CD3_ELEM_OFF, CD3_ROLE]] = \
                [s, n, n + 1, ct.nc, ids.size, off, role]
            for w, name in ((CD3_T_PTS, "pts"), (CD3_T_D, "D"), (CD3_T_W, "W"), (CD3_T_E, "E"),
                            (CD3_T_A, "A"), (CD3_T_B, "B"), (CD3_T_C, "C"), (CD3_T_R, "R"), (CD3_T_ED, "ED")):
                cd[c, w] = self.pool.add(ct.parts[name]) if name in ct.parts else -1
            elems.append(ids)
            off += ids.size
        self.class_desc = cd
        self.class_elems = np.concatenate(elems).astype(np.int32)

    # -- faces ------------------------------------------------------------------------------------
    def _face_frame(self, elems, f):
        """Outward unit normal (W, 3) and constant surface Jacobian (W,) of local face f."""
        ct = self.ct[self.class_of[elems[0]]]
        cx = ct.face_cross[f]
        ref_n = np.asarray(FACES[ct.shape][f][4], dtype=float)
        inv = self.dxidx[elems]                                            # (W, j, m)
        dirn = np.einsum("wjm,j->wm", inv, cx)                              # F^{-T} c
        nlen = np.linalg.norm(dirn, axis=1)
        sJ = self.detJ[elems] * nlen
        nrm = dirn / nlen[:, None]
        out = np.einsum("wjm,j->wm", inv, ref_n)
        sgn = np.where(np.einsum("wm,wm->w", nrm, out) >= 0.0, 1.0, -1.0)
        return nrm * sgn[:, None], sJ

    def _slots(self):
        itf = self.mesh.interfaces
        nI = len(itf)
        le = np.array([t.left[0] for t in itf], dtype=np.int64)
        lf = np.array([t.left[1] for t in itf], dtype=np.int64)
        re_ = np.array([-1 if t.right is None else t.right[0] for t in itf], dtype=np.int64)
        rf = np.array([-1 if t.right is None else t.right[1] for t in itf], dtype=np.int64)
        kind = np.array([2 if t.right is None else (1 if t.tag == "subface" else 0) for t in itf], dtype=np.int64)
        vol = self.detJ * np.array([self.ct[c].wref.sum() for c in self.class_of])
        # per-side frames, by (class, face) buckets
        nL = np.zeros((nI, 3))
        sJL = np.zeros(nI)
        areaL = np.zeros(nI)
        areaR = np.ones(nI)
        for side_e, side_f, store in ((le, lf, True), (re_, rf, False)):
            ok = side_e >= 0
            cls = np.where(ok, self.class_of[np.maximum(side_e, 0)], -1)
            for c in np.unique(cls[ok]):
                for f in np.unique(side_f[ok & (cls == c)]):
                    sel = np.flatnonzero(ok & (cls == c) & (side_f == f))
                    nrm, sJ = self._face_frame(side_e[sel], int(f))
                    area = sJ * self.ct[c].face_wt[f].sum()
                    if store:
                        nL[sel], sJL[sel], areaL[sel] = nrm, sJ, area
                    else:
                        areaR[sel] = area
        h = vol[le] / areaL
        nmax = self.nm[le].copy()
        inter = re_ >= 0
        h[inter] = np.minimum(h[inter], vol[re_[inter]] / areaR[inter])
        nmax[inter] = np.maximum(nmax[inter], self.nm[re_[inter]])
        tau = nmax.astype(float) ** 2 / h
        # slots: left of every coupling, right of interior ones
        ns = nI + int(inter.sum())
        S = np.zeros(ns, dtype=SLOT)
        sl = np.arange(nI)
        sr = nI + np.arange(int(inter.sum()))
        ri = np.flatnonzero(inter)
        S["elem"][sl], S["face"][sl] = le, lf
        S["elem"][sr], S["face"][sr] = re_[ri], rf[ri]
        S["kind"][sl] = np.where(inter, 1, 0)
        S["kind"][sr] = 1
        S["tau"][sl], S["tau"][sr] = tau, tau[ri]
        S["sJ"][sl], S["sJ"][sr] = sJL, sJL[ri]
        S["v"][sl] = np.einsum("ejm,em->ej", self.dxidx[le], nL)
        S["v"][sr] = np.einsum("ejm,em->ej", self.dxidx[re_[ri]], -nL[ri])
        S["partner"][sl] = -1
        S["partner"][sl[ri]] = sr
        S["partner"][sr] = ri
        right_slot = np.full(nI, -1, dtype=np.int64)
        right_slot[ri] = sr
        # trace grids: the own face grid of the side with the larger q (ties and subfaces: the left /
        # triangle side), its weights and surface Jacobian; that side maps by the identity, the other
        # through the geometry (exact: every rule here integrates the face terms exactly, so the
        # choice only moves rounding, cf. sipg.py:513-554).  A lower-q triangle side of a subface
        # interpolates to the GL(q_quad) collapsed rule on its own triangle.
        clsL = self.class_of[le]
        clsR = np.where(inter, self.class_of[np.maximum(re_, 0)], -1)
        qL = self.nq[le]
        qR = np.where(inter, self.nq[np.maximum(re_, 0)], 0)
        owner_right = inter & (kind == 0) & (qR > qL)
        bkey = np.stack([kind, clsL, lf, clsR, rf, owner_right.astype(np.int64)], axis=1)
        ub, binv = np.unique(bkey, axis=0, return_inverse=True)
        binv = binv.reshape(-1)
        for b, (kd, cl, fl, cr, fr, orr) in enumerate(ub):
            sel = np.flatnonzero(binv == b)
            if kd == 2:
                ct = self.ct[cl]
                S["nt"][sel] = ct.q * ct.q
                S["wtoff"][sel] = self.pool.add(ct.face_wt[fl])
                S["mkind"][sel], S["moff"][sel], S["moff2"][sel] = MAP_ID, -1, -1
                continue
            # H: trace-grid owner, O: the other side
            if orr:
                eH, fH, cH, eO, fO, cO, sH, sO = re_[sel], fr, cr, le[sel], fl, cl, right_slot[sel], sel
            else:
                eH, fH, cH, eO, fO, cO, sH, sO = le[sel], fl, cl, re_[sel], fr, cr, sel, right_slot[sel]
            ctH, ctO = self.ct[cH], self.ct[cO]
            hfix, hside, hrun, htri, _ = FACES[ctH.shape][fH]
            if kd == 1 and ctO.q > ctH.q:      # subface, the quad side has the larger q
                r = quad_rule(GL, ctO.q)
                taxes = [r.points, r.points]
                wt = np.multiply.outer(r.weights, r.weights) * 0.5 * (1.0 - r.points)[None, :]
                self._set_tensor(S, sH, lagrange_interp_matrix(ctH.pts[hrun[0]], taxes[0]),
                                 lagrange_interp_matrix(ctH.pts[hrun[1]], taxes[1]), False, ctH.q)
            else:
                taxes = [ctH.pts[hrun[0]], ctH.pts[hrun[1]]]
                wt = ctH.face_wt[fH]
                S["mkind"][sH], S["moff"][sH], S["moff2"][sH] = MAP_ID, -1, -1
            wt = np.asarray(wt).reshape(-1)
            nt = wt.size
            wtoff = self.pool.add(wt)
            for idx in (sH, sO):
                S["nt"][idx] = nt
                S["wtoff"][idx] = wtoff
            # the owner's surface Jacobian (its face parameters carry the weights)
            _, sJH = self._face_frame(eH, int(fH))
            S["sJ"][sH] = S["sJ"][sO] = sJH
            # the other side's parameters of the trace points, through the geometry
            ofix, oside, orun, _, _ = FACES[ctO.shape][fO]
            g = np.meshgrid(*taxes, indexing="ij")
            eta_h = np.zeros((nt, 3))
            eta_h[:, hfix] = hside
            eta_h[:, hrun[0]] = g[0].reshape(-1)
            eta_h[:, hrun[1]] = g[1].reshape(-1)
            xi_h = xi_of_eta(ctH.shape, eta_h)
            x = self.x0[eH][:, None, :] + np.einsum("wij,pj->wpi", self.F[eH], xi_h + 1.0)
            xi_o = np.einsum("wjm,wpm->wpj", self.dxidx[eO], x - self.x0[eO][:, None, :]) - 1.0
            with np.errstate(divide="ignore", invalid="ignore"):
                eta_o = eta_of_xi(ctO.shape, xi_o)
            # the fixed coordinate is undefined on a collapsed edge that the face contains
            fx_ok = np.where(np.isfinite(eta_o[..., ofix]), eta_o[..., ofix], oside)
            if np.abs(fx_ok - oside).max() > 1e-9 or not np.all(np.isfinite(eta_o[..., list(orun)])):
                raise ValueError("trace points do not lie on the neighbour's face")
            prm = np.stack([eta_o[..., orun[0]], eta_o[..., orun[1]]], axis=-1)        # (W, nt, 2)
            keyr = np.round(prm.reshape(len(sel), -1), 11)
            _, first, vinv = np.unique(keyr, axis=0, return_index=True, return_inverse=True)
            vinv = vinv.reshape(-1)
            na, nb = taxes[0].size, taxes[1].size
            for v, i0 in enumerate(first):
                idx = sO[vinv == v]
                p = prm[i0].reshape(na, nb, 2)
                pa, pb = p[..., 0], p[..., 1]
                tol = 1e-12
                if np.ptp(pa, axis=1).max() < tol and np.ptp(pb, axis=0).max() < tol:
                    self._set_tensor(S, idx, lagrange_interp_matrix(ctO.pts[orun[0]], pa[:, 0]),
                                     lagrange_interp_matrix(ctO.pts[orun[1]], pb[0, :]), False, ctO.q)
                elif np.ptp(pa, axis=0).max() < tol and np.ptp(pb, axis=1).max() < tol:
                    # own axis 0 follows the trace's second index: r1 runs over trace axis b
                    self._set_tensor(S, idx, lagrange_interp_matrix(ctO.pts[orun[0]], pa[0, :]),
                                     lagrange_interp_matrix(ctO.pts[orun[1]], pb[:, 0]), True, ctO.q)
                elif np.ptp(pa, axis=0).max() < tol or np.ptp(pb, axis=0).max() < tol:
                    perp = 0 if np.ptp(pa, axis=0).max() < tol else 1
                    par = 1 - perp
                    pp = p[..., par]                                              # (na, nb)
                    X = np.stack([lagrange_interp_matrix(ctO.pts[orun[par]], pp[:, j]) for j in range(nb)])
                    Y = lagrange_interp_matrix(ctO.pts[orun[perp]], p[0, :, perp])
                    S["mkind"][idx] = MAP_ROW
                    S["moff"][idx] = self.pool.add(X)                              # (nb, na, q)
                    S["moff2"][idx] = self.pool.add(Y)                             # (nb, q)
                    S["nab"][idx] = na | (nb << 8) | (perp << 16)
                else:
                    Ma = lagrange_interp_matrix(ctO.pts[orun[0]], pa.reshape(-1))
                    Mb = lagrange_interp_matrix(ctO.pts[orun[1]], pb.reshape(-1))
                    S["mkind"][idx] = MAP_DENSE
                    S["moff"][idx] = self.pool.add(np.einsum("pa,pb->pab", Ma, Mb).reshape(nt, -1))
                    S["moff2"][idx] = -1
        # order by (element, face, coupling) and publish offsets
        order = np.lexsort((np.arange(ns), S["face"], S["elem"]))
        newpos = np.empty(ns, dtype=np.int64)
        newpos[order] = np.arange(ns)
        S = S[order]
        S["partner"] = np.where(S["partner"] >= 0, newpos[np.maximum(S["partner"], 0)], -1)
        # every slot publishes its own trace (the apply kernel reads its own and its partner's)
        pub = 2 * S["nt"].astype(np.int64)
        off = np.concatenate([[0], np.cumsum(pub)[:-1]])
        S["pub_self"] = off
        S["pub_other"] = np.where(S["partner"] >= 0, S["pub_self"][np.maximum(S["partner"], 0)], -1)
        self.n_pub = int(pub.sum())
        self.slots = S
        counts = np.bincount(S["elem"], minlength=len(self.shapes))
        lim = np.array([NSMAX[s] for s in self.shapes])
        if np.any(counts > lim):
            raise ValueError("an element couples to more faces than its kernel holds")
        self.slot_off = np.zeros(len(self.shapes) + 1, dtype=np.int64)
        self.slot_off[1:] = np.cumsum(counts)

    def _set_tensor(self, S, idx, X, Y, swap, q):
        """Trace map M[p(r1, r2), (ia, ib)] = X[r1, ia] Y[r2, ib]; p = r1 n2 + r2, or r2 n1 + r1 when
        swapped (the trace's first axis follows own axis 1)."""
        n1, n2 = X.shape[0], Y.shape[0]
        if not swap and n1 == q and n2 == q and np.abs(X - np.eye(q)).max() < 1e-12 and \
                np.abs(Y - np.eye(q)).max() < 1e-12:
            S["mkind"][idx], S["moff"][idx], S["moff2"][idx] = MAP_ID, -1, -1
            return
        S["mkind"][idx] = MAP_TENSOR
        S["moff"][idx] = self.pool.add(X)
        S["moff2"][idx] = self.pool.add(Y)
        S["nab"][idx] = n1 | (n2 << 8) | (int(swap) << 16)
