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
* published traces: per interior slot, (u, n.grad u) interleaved at the trace
  points (phase 1 writes them, phase 2 reads the partner's).
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
 CD3_T_A, CD3_T_B, CD3_T_C, CD3_ROLE) = range(14)

SLOT = np.dtype([
    ("face", "<i4"), ("kind", "<i4"), ("nt", "<i4"), ("mkind", "<i4"),
    ("moff", "<i4"), ("wtoff", "<i4"), ("elem", "<i4"), ("partner", "<i4"),
    ("pub_self", "<i8"), ("pub_other", "<i8"),
    ("tau", "<f8"), ("sJ", "<f8"), ("v", "<f8", (3,)), ("pad", "<f8"),
])
assert SLOT.itemsize == 96
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
        self.rules = [quad_rule(k, q) for k in kinds]
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
        parts = {"pts": np.concatenate(self.pts),
                 "D": np.concatenate([diff_matrix(p).reshape(-1) for p in self.pts]),
                 "W": w,
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
        keys = sorted(set(zip(self.sid.tolist(), self.nm.tolist())))
        self.class_of = np.zeros(len(self.shapes), dtype=np.int64)
        cd = np.zeros((len(keys), CD3_WORDS), dtype=np.int32)
        elems, self.ct = [], []
        off = 0
        names = {v: k for k, v in SHAPE_ID.items()}
        for c, (s, n) in enumerate(keys):
            ids = np.flatnonzero((self.sid == s) & (self.nm == n))
            self.class_of[ids] = c
            ct = ClassTables3(names[s], n, n + 1)
            self.ct.append(ct)
            cd[c, [CD3_SHAPE, CD3_N, CD3_Q, CD3_NC, CD3_COUNT, CD3_ELEM_OFF]] = [s, n, n + 1, ct.nc, ids.size, off]
            for w, name in ((CD3_T_PTS, "pts"), (CD3_T_D, "D"), (CD3_T_W, "W"), (CD3_T_E, "E"),
                            (CD3_T_A, "A"), (CD3_T_B, "B"), (CD3_T_C, "C")):
                cd[c, w] = self.pool.add(ct.parts[name]) if name in ct.parts else -1
            elems.append(ids)
            off += ids.size
        self.class_desc = cd
        self.class_elems = np.concatenate(elems).astype(np.int32)
        self.ct_of_elem = lambda e: self.ct[self.class_of[e]]

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
        # trace rules and maps, per bucket (kind, left class, left face, right class, right face)
        clsL = self.class_of[le]
        clsR = np.where(inter, self.class_of[np.maximum(re_, 0)], -1)
        bkey = np.stack([kind, clsL, lf, clsR, rf], axis=1)
        ub, binv = np.unique(bkey, axis=0, return_inverse=True)
        binv = binv.reshape(-1)
        for b, (kd, cl, fl, cr, fr) in enumerate(ub):
            sel = np.flatnonzero(binv == b)
            ctl = self.ct[cl]
            fixed, side, run, tri, _ = FACES[ctl.shape][fl]
            if kd == 2:
                taxes = [ctl.pts[run[0]], ctl.pts[run[1]]]
                wt = ctl.face_wt[fl]
            else:
                ctr = self.ct[cr]
                qt = max(ctl.q, ctr.q)
                both_gll = ctl.shape == HEX and ctr.shape == HEX
                kk = GLL if (both_gll and not tri) else GL
                r = quad_rule(kk, qt)
                taxes = [r.points, r.points]
                wt = np.multiply.outer(r.weights, r.weights)
                if tri:
                    wt = wt * 0.5 * (1.0 - r.points)[None, :]
                wt = wt.reshape(-1)
            nt = wt.size
            wtoff = self.pool.add(wt)
            S["nt"][sel] = nt
            S["wtoff"][sel] = wtoff
            if kd != 2:
                S["nt"][right_slot[sel]] = nt
                S["wtoff"][right_slot[sel]] = wtoff
            # left map: own grid -> trace grid (tensor)
            La = lagrange_interp_matrix(ctl.pts[run[0]], taxes[0])
            Lb = lagrange_interp_matrix(ctl.pts[run[1]], taxes[1])
            self._set_map(S, sel, np.kron(La, Lb), ctl.q)
            if kd == 2:
                continue
            # right map: trace points through the geometry into the right face parameters
            ctr = self.ct[cr]
            rfix, rside, rrun, _, _ = FACES[ctr.shape][fr]
            g = np.meshgrid(*taxes, indexing="ij")
            eta_l = np.zeros((nt, 3))
            eta_l[:, fixed] = side
            eta_l[:, run[0]] = g[0].reshape(-1)
            eta_l[:, run[1]] = g[1].reshape(-1)
            xi_l = xi_of_eta(ctl.shape, eta_l)
            eL, eR = le[sel], re_[sel]
            x = self.x0[eL][:, None, :] + np.einsum("wij,pj->wpi", self.F[eL], xi_l + 1.0)
            xi_r = np.einsum("wjm,wpm->wpj", self.dxidx[eR], x - self.x0[eR][:, None, :]) - 1.0
            eta_r = eta_of_xi(ctr.shape, xi_r)
            if np.abs(eta_r[..., rfix] - rside).max() > 1e-9:
                raise ValueError("trace points do not lie on the neighbour's face")
            prm = np.stack([eta_r[..., rrun[0]], eta_r[..., rrun[1]]], axis=-1)        # (W, nt, 2)
            keyr = np.round(prm.reshape(len(sel), -1), 11)
            uv, first, vinv = np.unique(keyr, axis=0, return_index=True, return_inverse=True)
            vinv = vinv.reshape(-1)
            for v, i0 in enumerate(first):
                p = prm[i0]
                Ma = lagrange_interp_matrix(ctr.pts[rrun[0]], p[:, 0])
                Mb = lagrange_interp_matrix(ctr.pts[rrun[1]], p[:, 1])
                M = np.einsum("pa,pb->pab", Ma, Mb).reshape(nt, -1)
                self._set_map(S, right_slot[sel[vinv == v]], M, ctr.q)
        # order by (element, face, coupling) and publish offsets
        order = np.lexsort((np.arange(ns), S["face"], S["elem"]))
        newpos = np.empty(ns, dtype=np.int64)
        newpos[order] = np.arange(ns)
        S = S[order]
        S["partner"] = np.where(S["partner"] >= 0, newpos[np.maximum(S["partner"], 0)], -1)
        pub = np.where(S["kind"] == 1, 2 * S["nt"].astype(np.int64), 0)
        off = np.concatenate([[0], np.cumsum(pub)[:-1]])
        S["pub_self"] = np.where(S["kind"] == 1, off, -1)
        S["pub_other"] = np.where(S["partner"] >= 0, S["pub_self"][np.maximum(S["partner"], 0)], -1)
        self.n_pub = int(pub.sum())
        self.slots = S
        counts = np.bincount(S["elem"], minlength=len(self.shapes))
        self.slot_off = np.zeros(len(self.shapes) + 1, dtype=np.int64)
        self.slot_off[1:] = np.cumsum(counts)

    def _set_map(self, S, idx, M, q):
        if M.shape == (q * q, q * q) and np.abs(M - np.eye(q * q)).max() < 1e-12:
            S["mkind"][idx] = 0
            S["moff"][idx] = -1
            return
        S["mkind"][idx] = 1
        S["moff"][idx] = self.pool.add(M)
