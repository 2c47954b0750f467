"""Plan builder: flattens a mesh + order map into the device-resident SoA plan
consumed by the sm_100a kernels (`csrc/`).

It restates the reference's operator setup (reference sipg.py:234-554) in a
vectorised form: expansions grouped into element classes (sipg.py:302-349),
geometric factors (mesh.py:331-432), DoF offsets (sipg.py:269-273), interface
strategy selection with the p2p certificate (sipg.py:371-420,
trace.py:84-106), transfers (trace.py:172-199), shared-trace rules and
geometry (sipg.py:513-554) and penalties (sipg.py:351-360).

Nothing here runs per apply.  The apply itself is one fused CUDA kernel per
element class: volume terms, neighbour-trace evaluation, SIP flux and lift
(see DESIGN.md).
"""
from __future__ import annotations

import numpy as np

from . import layout as L
from .mesh import as_shape

# k_hexp sizes its shared-trace scratch for neighbour orders <= own order + SF_RANGE
# (SIPG_SF_RANGE in csrc/sipg_hex_planes.cuh); farther neighbours take the generic face path
SF_RANGE = 3
from .polylib import (BasisKind, QuadKind, as_basis_kind, as_quad_kind, eval_basis_1d,
                      lagrange_interp_matrix, quad_rule)
from .stdregions import DEFAULT_RULES, DIM, FACES, class_tables

REF_VERTS = {
    "quad": np.array([[-1.0, -1.0], [1.0, -1.0], [1.0, 1.0], [-1.0, 1.0]]),
    "hex": np.array([[-1, -1, -1], [1, -1, -1], [1, 1, -1], [-1, 1, -1],
                     [-1, -1, 1], [1, -1, 1], [1, 1, 1], [-1, 1, 1]], dtype=float),
}
NSYM = {2: 3, 3: 6}
SYM_IDX = {2: [(0, 0), (0, 1), (1, 1)], 3: [(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]}


# --------------------------------------------------------------------------
# geometry (vectorised over a batch of elements of one shape)

def vertex_maps(shape, xi):
    """Vertex shape functions N (npts, nv) and gradients dN (npts, nv, d)."""
    xi = np.atleast_2d(xi)
    if shape == "tri":
        N = np.stack([-0.5 * (xi[:, 0] + xi[:, 1]), 0.5 * (1 + xi[:, 0]), 0.5 * (1 + xi[:, 1])], axis=1)
        dN = np.broadcast_to(np.array([[-0.5, -0.5], [0.5, 0.0], [0.0, 0.5]]), (xi.shape[0], 3, 2))
        return N, dN
    r = REF_VERTS[shape]
    fac = 0.5 * (1.0 + xi[:, None, :] * r[None, :, :])
    N = fac.prod(axis=2)
    d = r.shape[1]
    dN = np.stack([0.5 * r[None, :, j] * np.prod(np.delete(fac, j, axis=2), axis=2) for j in range(d)], axis=2)
    return N, dN


def _const_rows(a):
    """Per element: all points equal to point 0 within 1e-12 relative
    (reference mesh.py:325-328)."""
    ref = a[:, :1]
    scale = np.abs(ref).reshape(len(a), -1).max(axis=1) + 1.0
    return np.abs(a - ref).reshape(len(a), -1).max(axis=1) < 1e-12 * scale


def jacobians(shape, verts, xi):
    N, dN = vertex_maps(shape, xi)
    x = np.einsum("pv,evi->epi", N, verts)
    F = np.einsum("pvj,evi->epij", dN, verts)
    return x, F


def tri_chain(face_fixed, side, p):
    """d eta / d xi at triangle face parameters p (run-axis eta)."""
    if face_fixed == 0:
        e1, e2 = np.full_like(p, float(side)), p
    else:
        e1, e2 = p, np.full_like(p, -1.0)
    c = np.zeros((p.size, 2, 2))
    c[:, 0, 0] = 2.0 / (1.0 - e2)
    c[:, 0, 1] = (1.0 + e1) / (1.0 - e2)
    c[:, 1, 1] = 1.0
    return c


def gn_at(ct, f, inv, nrm, prm):
    """(G n)_k = sum_m (chain . dxi/dx)_km n_m at face points -> (nE, npts, d)."""
    gxn = np.einsum("epkm,epm->epk", inv, nrm)
    if ct.shape == "tri":
        face = FACES["tri"][f]
        ch = tri_chain(face.fixed, face.side, np.atleast_2d(prm)[:, 0])
        gxn = np.einsum("pkj,epj->epk", ch, gxn)
    return gxn


def tensor_params(axes):
    if not axes:
        return np.zeros((1, 0))
    g = np.meshgrid(*axes, indexing="ij")
    return np.stack([a.reshape(-1) for a in g], axis=-1)


def apply_code(code, p):
    """Left face parameters -> right parameters (reference orient.py:25-38)."""
    p = np.atleast_2d(p)
    if p.shape[1] == 1:
        return -p if code == 1 else p.copy()
    out = p[:, ::-1].copy() if (code >> 2) & 1 else p.copy()
    if (code >> 1) & 1:
        out[:, 0] = -out[:, 0]
    if code & 1:
        out[:, 1] = -out[:, 1]
    return out


def inverse_code(code, fd):
    if fd == 1:
        return code
    probe = np.array([[0.25, 0.625]])
    fwd = apply_code(code, probe)
    for c in range(8):
        if np.allclose(apply_code(c, fwd), probe):
            return c
    raise ValueError(code)


def axis_transfer(src_axes, dst_axes, code):
    """Tensor transfer src face grid -> dst grid through orientation `code` as
    per-destination-axis 1-D Lagrange matrices (reference trace.py:172-199):
    returns (mats, swap, identity)."""
    fd = len(dst_axes)
    if fd == 1:
        m = lagrange_interp_matrix(src_axes[0], -dst_axes[0] if code == 1 else dst_axes[0])
        ident = m.shape[0] == m.shape[1] and np.array_equal(m, np.eye(m.shape[0]))
        return [m], False, ident
    swap = bool((code >> 2) & 1)
    sign = [-1.0 if (code >> 1) & 1 else 1.0, -1.0 if code & 1 else 1.0]
    mats = []
    for k in range(2):
        s = (1 - k) if swap else k
        mats.append(lagrange_interp_matrix(src_axes[s], sign[s] * dst_axes[k]))
    ident = (not swap) and all(m.shape[0] == m.shape[1] and np.array_equal(m, np.eye(m.shape[0])) for m in mats)
    return mats, swap, ident


class _Pool:
    """Deduplicating float64 table pool."""

    def __init__(self):
        self.chunks, self.size, self.index = [], 0, {}

    def add(self, a) -> int:
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))
        key = a.tobytes()
        off = self.index.get(key)
        if off is None:
            off = self.size
            self.index[key] = off
            self.chunks.append(a)
            self.size += a.size
        return off

    def array(self):
        return np.concatenate(self.chunks) if self.chunks else np.zeros(1)


def certify(nl, ql, kl, nr, qr, kr, p_geom, deformed):
    """p2p symmetry certificate (reference trace.py:84-106)."""
    c1 = ql >= nr and qr >= nl
    req = (nl - 1) + (nr - 1) + (3 * p_geom if deformed else p_geom)
    act = min(quad_rule(kl, ql).exactness, quad_rule(kr, qr).exactness)
    return c1 and act >= req, c1, act >= req, req, act


def shared_rule(rl, rr, patched):
    """Shared-trace rule: max(q) points; kind of the higher side
    (reference trace.py:202-206), or Gauss-Legendre whenever a side is not
    GLL (patch P2, SURVEY §8c — the reference divides by zero at a
    collapsed vertex otherwise)."""
    q = max(rl.n, rr.n)
    if patched and not (rl.kind is QuadKind.GAUSS_LOBATTO and rr.kind is QuadKind.GAUSS_LOBATTO):
        return quad_rule(QuadKind.GAUSS_LEGENDRE, q)
    return quad_rule((rr if rr.n > rl.n else rl).kind, q)


def corner_params(d):
    g = np.meshgrid(*([np.array([-1.0, 1.0])] * d), indexing="ij")
    return np.stack([a.reshape(-1) for a in g], axis=-1)


class ElemGeo:
    """Geometry of all elements of one expansion.  Affine elements (F equal at
    every reference corner, hence everywhere, to the reference's 1e-12
    relative test, mesh.py:325-328) keep one F; the others carry per-point
    arrays at the volume points."""

    def __init__(self, ct, verts):
        self.ct = ct
        d = ct.dim
        _, Fc = jacobians(ct.shape, verts, corner_params(d) if ct.shape != "tri" else np.zeros((1, 2)))
        self.regular = _const_rows(Fc)
        self.verts = verts
        self.F0 = Fc[:, 0]
        self.J0 = np.linalg.det(self.F0)
        self.G0 = np.linalg.inv(self.F0)                  # dxi_k/dx_m
        nr = np.flatnonzero(~self.regular)
        self.nr = nr
        self.nr_pos = np.full(len(verts), -1, dtype=np.int64)
        self.nr_pos[nr] = np.arange(nr.size)
        if nr.size:
            _, F = jacobians(ct.shape, verts[nr], ct.xi)
            self.J = np.linalg.det(F)
            self.G = np.linalg.inv(F)
            if np.any(self.J <= 0.0):
                raise ValueError("element with a non-positive Jacobian")
        if np.any(self.J0 <= 0.0):
            raise ValueError("element with a non-positive Jacobian")
        w = ct.ref_w
        self.volume = self.J0 * w.sum()
        if nr.size:
            self.volume[nr] = (self.J * w[None, :]).sum(axis=1)

    def face(self, f, prm, weights, elems=None):
        """Face geometry at parameters prm for elements `elems` (indices into
        this group): swj (nE, np), normal (nE, np, d), inv (nE, np, d, d),
        F-constant flag, normal-constant flag.  Regular elements are evaluated
        once and broadcast."""
        ct = self.ct
        face = FACES[ct.shape][f]
        prm = np.atleast_2d(prm)
        npts = prm.shape[0]
        idx = np.arange(len(self.verts)) if elems is None else np.asarray(elems)
        nE, d = idx.size, ct.dim
        tang = np.asarray(face.tangents)
        F = np.broadcast_to(self.F0[idx][:, None], (nE, npts, d, d)).copy()
        nrm_mask = ~self.regular[idx]
        if nrm_mask.any():
            xi = np.asarray(face.center) + prm @ tang
            _, Fp = jacobians(ct.shape, self.verts[idx[nrm_mask]], xi)
            F[nrm_mask] = Fp
        tp = np.einsum("epij,kj->epki", F, tang)
        if d == 2:
            t = tp[:, :, 0, :]
            surf = np.linalg.norm(t, axis=2)
            nrm = np.stack([t[..., 1], -t[..., 0]], axis=2)
        else:
            nrm = np.cross(tp[:, :, 0, :], tp[:, :, 1, :])
            surf = np.linalg.norm(nrm, axis=2)
        nrm = nrm / surf[..., None]
        inv = np.broadcast_to(self.G0[idx][:, None], (nE, npts, d, d)).copy()
        if nrm_mask.any():
            inv[nrm_mask] = np.linalg.inv(F[nrm_mask])
        outward = np.einsum("epji,j->epi", inv, np.asarray(face.ref_normal))
        nrm = nrm * np.where(np.einsum("epi,epi->ep", nrm, outward) >= 0.0, 1.0, -1.0)[..., None]
        ncst = _const_rows(nrm)
        nrm = np.where(ncst[:, None, None], nrm[:, :1], nrm)
        icst = _const_rows(inv)
        inv = np.where(icst[:, None, None, None], inv[:, :1], inv)
        return surf * weights[None, :], nrm, inv, _const_rows(F), ncst


class PlanBuilder:
    """Builds the flattened plan.  Attributes after build():
    class_desc (n_cls, CD_WORDS) int32, class_elems int32, elem_class int32,
    elem_pos int32, dof_off int64, recs (FACE_REC), tables/egeo/fgeo float64,
    plus host-side maps (strategy per interface, certificates, trace slots)."""

    def __init__(self, mesh, order_map, *, basis_kind=BasisKind.LAGRANGE, rule_kinds=None,
                 lambda_=1.0, tau_constant=10.0, strategy="p2p", face_absorb="auto",
                 force_interp=False, p_geom=1, tau_rule="reference", shared_rule="patched",
                 element_roles=None):
        self.mesh = mesh
        self.dim = int(mesh.dim)
        # per-element launch role: 0 = computed first, 1 = computed after the halo
        # exchange (touches a ghost), 2 = ghost (never computed; neighbour data only)
        self.roles = None if element_roles is None else np.asarray(element_roles, dtype=np.int64)
        if self.dim not in (2, 3):
            raise ValueError("only 2D and 3D meshes are supported")
        self.kind = as_basis_kind(basis_kind)
        self.rule_kinds = rule_kinds
        self.lam, self.C = float(lambda_), float(tau_constant)
        self.strategy, self.face_absorb, self.force_interp = strategy, face_absorb, force_interp
        self.p_geom, self.tau_rule, self.shared_patched = p_geom, tau_rule, shared_rule == "patched"
        self.nm = np.asarray(order_map.n_modes, dtype=np.int64)
        self.nq = np.asarray(order_map.n_quad, dtype=np.int64)

    def _kinds(self, shape):
        rk = self.rule_kinds
        d = DIM[shape]
        if rk is None:
            return tuple(k.value for k in DEFAULT_RULES[shape])
        if isinstance(rk, (tuple, list)):
            return tuple(as_quad_kind(k).value for k in rk)
        return (as_quad_kind(rk).value,) * d

    # ------------------------------------------------------------------
    def build(self):
        mesh = self.mesh
        nel = len(mesh.elements)
        shapes = [as_shape(el.shape).value for el in mesh.elements]
        if any(s not in ("quad", "tri", "hex") for s in shapes):
            raise ValueError("supported shapes: quad, tri, hex")
        verts = np.asarray(mesh.vertices, dtype=float)
        # expansions: identity = parameters (reference sipg.py:262-266, 395)
        keys = {}
        self.exp_list = []
        self.exp_of = np.zeros(nel, dtype=np.int64)
        for e in range(nel):
            s = shapes[e]
            q = int(self.nq[e])
            k = (s, int(self.nm[e]), q)
            ei = keys.get(k)
            if ei is None:
                ei = keys[k] = len(self.exp_list)
                self.exp_list.append(class_tables(s, self.kind, k[1], (q,) * DIM[s], self._kinds(s)))
            self.exp_of[e] = ei
        self.ct = [self.exp_list[i] for i in self.exp_of]
        ncoef = np.array([c.n_coeffs for c in self.exp_list])[self.exp_of]
        self.dof_off = np.zeros(nel + 1, dtype=np.int64)
        self.dof_off[1:] = np.cumsum(ncoef)
        self.n_dofs = int(self.dof_off[-1])
        if self.n_dofs >= 2 ** 31:
            raise ValueError("plans are limited to 2^31 DoFs per GPU")
        nfp = np.array([[c.face_npts(f) for f in range(len(c.faces))] + [0] * (6 - len(c.faces))
                        for c in self.exp_list])[self.exp_of]
        nfc = np.array([len(c.faces) for c in self.exp_list])[self.exp_of]
        mask = np.arange(6)[None, :] < nfc[:, None]
        flat = nfp[mask]
        self.trace_slots = np.concatenate([[0], np.cumsum(flat)[:-1]]).astype(np.int64)
        # geometry per expansion group
        ev = np.full((nel, 8), -1, dtype=np.int64)
        for e, el in enumerate(mesh.elements):
            ev[e, :len(el.verts)] = el.verts
        self.exp_members = [np.flatnonzero(self.exp_of == i) for i in range(len(self.exp_list))]
        self.exp_pos = np.zeros(nel, dtype=np.int64)
        self.geo = []
        self.vol = np.zeros(nel)
        self.regular = np.zeros(nel, dtype=bool)
        # own-face geometry per (element, face): constants + pointwise where needed
        d = self.dim
        self.f_const = np.zeros((nel, 6), dtype=bool)
        self.f_ncst = np.zeros((nel, 6), dtype=bool)
        self.f_sJ = np.zeros((nel, 6))
        self.f_gxn = np.zeros((nel, 6, 3))
        self.f_area = np.ones((nel, 6))
        self.f_pw = {}                 # (e, f) -> (swj, gn (npts, d)) for non-constant faces
        for i, ids in enumerate(self.exp_members):
            c = self.exp_list[i]
            self.exp_pos[ids] = np.arange(ids.size)
            nv = {"quad": 4, "tri": 3, "hex": 8}[c.shape]
            g = ElemGeo(c, verts[ev[ids, :nv]])
            self.geo.append(g)
            self.vol[ids] = g.volume
            self.regular[ids] = g.regular
            for f in range(len(c.faces)):
                prm = tensor_params(c.face_pts(f))
                w = c.face_weights(f)
                swj, nrm, inv, fconst, ncst = g.face(f, prm, w)
                self.f_const[ids, f] = fconst
                self.f_ncst[ids, f] = ncst
                self.f_sJ[ids, f] = swj[:, 0] / w[0]
                self.f_gxn[ids, f, :d] = np.einsum("ekm,em->ek", inv[:, 0], nrm[:, 0])
                self.f_area[ids, f] = swj.sum(axis=1)
                for j in np.flatnonzero(~fconst):
                    gn = gn_at(c, f, inv[j:j + 1], nrm[j:j + 1], prm)[0]
                    self.f_pw[(int(ids[j]), f)] = (swj[j], gn)
        self._classes(nel)
        self._faces()
        return self

    # ------------------------------------------------------------------
    def _classes(self, nel):
        """Kernel classes: (expansion, geometry mode, launch role), first-appearance order."""
        geom = np.where(self.regular, L.GEOM_REGULAR, L.GEOM_POINTWISE)
        role = np.zeros(nel, dtype=np.int64) if self.roles is None else self.roles
        key = (self.exp_of * 2 + geom) * 3 + role
        _, first = np.unique(key, return_index=True)
        order = key[np.sort(first)]
        self.pool = _Pool()
        self.class_list = []
        desc, elems, egeo = [], [], []
        egeo_size = rec_off = 0
        self.elem_class = np.zeros(nel, dtype=np.int32)
        self.elem_pos = np.zeros(nel, dtype=np.int32)
        self.rec_base = np.zeros(nel, dtype=np.int64)
        for k in order:
            ei, gm, rl = int(k) // 6, (int(k) // 3) % 2, int(k) % 3
            ids = np.flatnonzero(key == k)
            c, g = self.exp_list[ei], self.geo[ei]
            ci = len(self.class_list)
            self.class_list.append((c, gm, ids))
            self.elem_class[ids] = ci
            self.elem_pos[ids] = np.arange(ids.size)
            nf = len(c.faces)
            self.rec_base[ids] = rec_off + np.arange(ids.size) * nf
            d = c.dim
            cd = np.zeros(L.CD_WORDS, dtype=np.int32)
            cd[L.CD_SHAPE] = L.SHAPE_ID[c.shape]
            cd[L.CD_N] = c.n
            cd[L.CD_Q0:L.CD_Q0 + d] = c.nq
            cd[L.CD_NC], cd[L.CD_NPHYS], cd[L.CD_NFACES] = c.n_coeffs, c.n_phys, nf
            cd[L.CD_GEOM], cd[L.CD_COUNT] = gm, ids.size
            cd[L.CD_ROLE] = rl
            cd[L.CD_ELEM_OFF] = sum(x.size for x in elems)
            cd[L.CD_REC_OFF] = rec_off
            rec_off += ids.size * nf
            cd[L.CD_GLLMASK] = sum(1 << a for a in range(d) if c.axis[a]["gll"])
            cd[L.CD_KIND] = ["modified_modal", "orthogonal", "lagrange"].index(c.kind.value)
            self._tables(c, cd)
            pos = self.exp_pos[ids]
            if gm == L.GEOM_REGULAR:
                G0 = g.G0[pos]
                S = np.einsum("ekm,ejm->ekj", G0, G0)
                blk = np.concatenate([g.J0[pos][:, None]] + [S[:, a, b][:, None] for a, b in SYM_IDX[d]],
                                     axis=1)
            else:
                rows = g.nr_pos[pos]
                G, J = g.G[rows], g.J[rows]
                jw = J * c.ref_w[None, :]
                if c.shape == "tri":
                    e1, e2 = c.eta[:, 0], c.eta[:, 1]
                    cj = np.zeros((c.n_phys, 2, 2))
                    cj[:, 0, 0] = 2.0 / (1.0 - e2)
                    cj[:, 0, 1] = (1.0 + e1) / (1.0 - e2)
                    cj[:, 1, 1] = 1.0
                    G = np.einsum("pkm,epmj->epkj", cj, G)
                K = np.einsum("epkm,epjm->epkj", G, G) * jw[:, :, None, None]
                blk = np.concatenate([jw[:, None, :]] + [K[:, None, :, a, b] for a, b in SYM_IDX[d]],
                                     axis=1).reshape(ids.size, -1)
            cd[L.CD_EGEO_OFF], cd[L.CD_EGEO_STRIDE] = egeo_size, blk.shape[1]
            egeo.append(blk.reshape(-1))
            egeo_size += blk.size
            desc.append(cd)
            elems.append(ids.astype(np.int32))
        self.class_desc = np.stack(desc)
        self.class_elems = np.concatenate(elems)
        self.egeo = np.concatenate(egeo)
        self.n_recs = rec_off

    def _tables(self, c, cd):
        P = self.pool
        if c.shape == "tri":
            t = c.tri
            cd[L.TR_A], cd[L.TR_DA] = P.add(t["A"]), P.add(t["dA"])
            cd[L.TR_D0], cd[L.TR_D1] = P.add(c.axis[0]["D"]), P.add(c.axis[1]["D"])
            cd[L.TR_W0], cd[L.TR_W1] = P.add(c.axis[0]["w"]), P.add(c.axis[1]["w"])
            cd[L.TR_B], cd[L.TR_DB] = P.add(t["B"]), P.add(t["dB"])
            cd[L.TR_GID] = P.add(t["gmodes"].astype(float))
            cd[L.TR_GSTART] = P.add(t["gstart"].astype(float))
            cd[L.TR_AEND], cd[L.TR_DAEND] = P.add(t["Aend"]), P.add(t["dAend"])
            cd[L.TR_BM1], cd[L.TR_DBM1] = P.add(t["Bm1"]), P.add(t["dBm1"])
            cd[L.TR_L0], cd[L.TR_L1] = P.add(c.axis[0]["L"]), P.add(c.axis[1]["L"])
            cd[L.TR_REFW] = P.add(c.ref_w)
            cd[L.TR_PTS0], cd[L.TR_PTS1] = P.add(c.axis[0]["pts"]), P.add(c.axis[1]["pts"])
            return
        for a in range(c.dim):
            t = c.axis[a]
            base = L.CD_TAX + 8 * a
            cd[base + L.TX_V], cd[base + L.TX_DV] = P.add(t["V"]), P.add(t["dV"])
            cd[base + L.TX_D], cd[base + L.TX_W] = P.add(t["D"]), P.add(t["w"])
            cd[base + L.TX_VEND], cd[base + L.TX_DVEND] = P.add(t["Vend"]), P.add(t["dVend"])
            cd[base + L.TX_LEND], cd[base + L.TX_PTS] = P.add(t["L"]), P.add(t["pts"])

    def rec_index(self, e, f):
        return self.rec_base[e] + f

    def _rule_block(self, rule):
        return self.pool.add(np.concatenate([rule.weights, rule.points]))

    def _tau(self, le, lf, re_=None, rf=None):
        """Penalty per interface, vectorised (reference sipg.py:351-360);
        tau_rule="baseline" is the BASELINE (P+1)^2/h override (patch P1)."""
        h = self.vol[le] / self.f_area[le, lf]
        nmax = self.nm[le]
        if re_ is not None:
            h = np.minimum(h, self.vol[re_] / self.f_area[re_, rf])
            nmax = np.maximum(nmax, self.nm[re_])
        if self.tau_rule == "baseline":
            return (nmax * nmax).astype(float) / h
        return self.C * np.maximum(nmax - 1, 1).astype(float) ** 2 / h

    # ------------------------------------------------------------------
    def _faces(self):
        mesh = self.mesh
        d = self.dim
        fd = d - 1
        nI = len(mesh.interfaces)
        LE = np.empty(nI, dtype=np.int64)
        LF = np.empty(nI, dtype=np.int64)
        RE = np.full(nI, -1, dtype=np.int64)
        RF = np.full(nI, -1, dtype=np.int64)
        CODE = np.zeros(nI, dtype=np.int64)
        for i, itf in enumerate(mesh.interfaces):
            LE[i], LF[i] = itf.left
            if itf.right is not None:
                RE[i], RF[i] = itf.right
            CODE[i] = itf.orientation
        recs = np.zeros(self.n_recs, dtype=L.FACE_REC)
        self._perm_buckets = []
        self._n_itf, self._bnd_itf = nI, RE < 0
        self.rec_ext = np.zeros((self.n_recs, 2), dtype=np.int64)
        self.rec_ext[:, 0] = -1
        self._rec_face = np.zeros(self.n_recs, dtype=np.int64)
        for ci, (c, gm, ids) in enumerate(self.class_list):
            nf = len(c.faces)
            base = self.rec_base[ids]
            for f in range(nf):
                self._rec_face[base + f] = f
        recs["nbr"] = -1
        recs["nbr_face"] = -1
        recs["nbr_rec"] = -1
        recs["geo"] = -1
        self._fgeo, self._fsize = [], 0
        self.recs = recs
        bnd = RE < 0
        # strategies (reference sipg.py:371-420)
        xl, xr = self.exp_of[LE], np.where(bnd, -1, self.exp_of[np.maximum(RE, 0)])
        conforming = (~bnd) & (xl == xr)
        strat = np.full(nI, -1, dtype=np.int64)       # 0 gather, 1 p2p, 2 shared
        strat[conforming] = 2 if self.face_absorb == "trace_iproduct" else 0
        nc = np.flatnonzero((~bnd) & ~conforming)
        deformed = ~(self.f_ncst[LE[nc], LF[nc]] & self.f_ncst[RE[nc], RF[nc]])
        self.certificates = []
        cert_cache = {}
        for t, i in enumerate(nc):
            cl, cr = self.exp_list[xl[i]], self.exp_list[xr[i]]
            al, ar = cl.faces[LF[i]].run[0], cr.faces[RF[i]].run[0]
            ck = (xl[i], al, xr[i], ar, bool(deformed[t]))
            cert = cert_cache.get(ck)
            if cert is None:
                cert = cert_cache[ck] = certify(cl.n, cl.nq[al], cl.rules[al].kind, cr.n, cr.nq[ar],
                                                cr.rules[ar].kind, self.p_geom, bool(deformed[t]))
            if self.face_absorb == "trace_iproduct" or self.strategy == "shared_trace":
                s = 2
            elif self.strategy == "p2p_forced":
                s = 1
            else:
                s = 1 if cert[0] else 2
            strat[i] = s
            self.certificates.append((int(i), cert, ["gather", "p2p", "shared"][s]))
        self.strategy_of = strat.astype(np.int8)
        # boundary faces
        bi = np.flatnonzero(bnd)
        if bi.size:
            r = self.rec_index(LE[bi], LF[bi])
            recs["type"][r] = L.FT_BOUNDARY
            recs["flags"][r] |= L.F_SELF_ID | L.F_OTHER_ID
            recs["tau"][r] = self._tau(LE[bi], LF[bi])
            self._own_geometry(r, LE[bi], LF[bi])
        # interior faces, bucketed like the reference's groups
        ii = np.flatnonzero(~bnd)
        if not ii.size:
            self._finish()
            return
        bkey = np.stack([xl[ii], LF[ii], xr[ii], RF[ii], CODE[ii], strat[ii]], axis=1)
        ukeys, inv = np.unique(bkey, axis=0, return_inverse=True)
        inv = inv.reshape(-1)
        order = np.argsort(inv, kind="stable")
        bounds = np.searchsorted(inv[order], np.arange(ukeys.shape[0] + 1))
        for b in range(ukeys.shape[0]):
            mem = ii[order[bounds[b]:bounds[b + 1]]]
            el, fl, er, fr, code, s = (int(v) for v in ukeys[b])
            le, re_ = LE[mem], RE[mem]
            rl, rr = self.rec_index(le, fl), self.rec_index(re_, fr)
            tau = self._tau(le, fl, re_, fr)
            recs["tau"][rl] = tau
            recs["tau"][rr] = tau
            recs["nbr"][rl], recs["nbr_face"][rl], recs["nbr_rec"][rl] = re_, fr, rr
            recs["nbr"][rr], recs["nbr_face"][rr], recs["nbr_rec"][rr] = le, fl, rl
            cl, cr = self.exp_list[el], self.exp_list[er]
            pts_l, pts_r = cl.face_pts(fl), cr.face_pts(fr)
            if s in (0, 1):
                self._perm_buckets.append((mem, self._transfer_perm(pts_r, pts_l, code, fd),
                                           self._transfer_perm(pts_l, pts_r, inverse_code(code, fd), fd)))
                for r, ee, ff_, eo, fo, src, dst, cc in (
                        (rl, le, fl, re_, fr, pts_r, pts_l, code),
                        (rr, re_, fr, le, fl, pts_l, pts_r, inverse_code(code, fd))):
                    recs["type"][r] = L.FT_DIRECT
                    recs["flags"][r] |= L.F_SELF_ID
                    self._own_geometry(r, ee, np.full(ee.size, ff_))
                    mats, swap, ident = axis_transfer(src, dst, cc)
                    if self.force_interp:
                        ident = False
                    recs["flags"][r] |= (L.F_OTHER_ID if ident else 0) | (L.F_OTHER_SWAP if swap else 0)
                    recs["to0"][r] = self.pool.add(mats[0])
                    recs["to1"][r] = self.pool.add(mats[1]) if len(mats) > 1 else -1
                    oc = self.f_const[eo, fo]
                    recs["go"][r, :d] = self.f_gxn[eo, fo, :d]
                    recs["flags"][r[~oc]] |= L.F_OTHER_PW
                    if (d == 3 and ident and el == er and cl.kind.value == "modified_modal"
                            and all(c_.axis[a]["gll"] for c_ in (cl,) for a in range(3))):
                        ao = fo // 2
                        tang = [b for b in range(3) if b != ao]
                        ok = (oc & self.f_const[ee, ff_] & (self.f_gxn[eo, fo, tang[0]] == 0.0)
                              & (self.f_gxn[eo, fo, tang[1]] == 0.0))
                        recs["flags"][r[ok]] |= L.F_FAST_HEX
                continue
            self._cur_mem = mem
            self._shared_bucket(cl, fl, cr, fr, code, le, re_, rl, rr)
        self._finish()

    def _transfer_perm(self, src, dst, code, fd):
        """Index permutation of the transfer src face grid -> dst grid, or None when it is a
        dense interpolation (the reference's one-hot test, trace.py:190-198), from this plan's
        own per-axis matrices; force_interp densifies every transfer (sipg.py:502-504)."""
        if self.force_interp:
            return None
        mats, swap, _ = axis_transfer(src, dst, code)
        if fd == 1:
            m = mats[0]
        else:
            a, b = (mats[1], mats[0]) if swap else (mats[0], mats[1])
            # M[(t0, t1), (i0, i1)]: no swap a[t0, i0] b[t1, i1]; swap a = mats[1][t1, i0], b = mats[0][t0, i1]
            if swap:
                m = np.einsum("yi,xj->xyij", a, b).reshape(b.shape[0] * a.shape[0], -1)
            else:
                m = np.einsum("xi,yj->xyij", a, b).reshape(a.shape[0] * b.shape[0], -1)
        if m.shape[0] != m.shape[1]:
            return None
        hits = np.isclose(m, 1.0, atol=1e-12)
        if np.all(hits.sum(axis=1) == 1) and np.allclose(m, hits.astype(float), atol=1e-12):
            return np.argmax(hits, axis=1)
        return None

    def transfer_perm_sha256(self) -> bytes:
        """SHA-256 over interfaces (ascending id) of [left perm, -1, right perm] for every interior
        interface (a side's own face grid -> the partner grid for gather / p2p, -> the shared trace
        grid for shared traces; empty for dense transfers) — the digest the golden
        fixtures record from the reference's Transfer.perm (tests/golden/make_golden.py maps_of)."""
        import hashlib
        rows = {}
        for mem, pl, pr in self._perm_buckets:
            a = np.zeros(0, np.int64) if pl is None else np.asarray(pl, np.int64)
            b = np.zeros(0, np.int64) if pr is None else np.asarray(pr, np.int64)
            row = np.concatenate([a, [-1], b]).astype(np.int64).tobytes()
            for i in mem:
                rows[int(i)] = row
        shared = np.int64(-1).tobytes()
        h = hashlib.sha256()
        for i in np.flatnonzero(~self._bnd_itf):
            h.update(np.int64(i).tobytes())
            h.update(rows.get(int(i), shared))
        return h.digest()

    def _own_geometry(self, r, e, f):
        """Self geometry on the own face grid for records r of faces (e, f)."""
        recs, d = self.recs, self.dim
        for c_idx in np.unique(self.exp_of[e]):
            sel = self.exp_of[e] == c_idx
            c = self.exp_list[c_idx]
            for ff in np.unique(f[sel]):
                s2 = sel & (f == ff)
                rr, ee = r[s2], e[s2]
                rules = [c.rules[a] for a in c.faces[ff].run]
                recs["nt0"][rr] = rules[0].n
                recs["nt1"][rr] = rules[1].n if len(rules) > 1 else 1
                recs["wt0"][rr] = self._rule_block(rules[0])
                recs["wt1"][rr] = self._rule_block(rules[1]) if len(rules) > 1 else -1
                recs["sJ"][rr] = self.f_sJ[ee, ff]
                recs["gs"][rr, :d] = self.f_gxn[ee, ff, :d]
                nc = ~self.f_const[ee, ff]
                for ri, ei in zip(rr[nc], ee[nc]):
                    swj, gn = self.f_pw[(int(ei), int(ff))]
                    recs["flags"][ri] |= L.F_SELF_PW
                    recs["geo"][ri] = self._add_fgeo(np.concatenate([swj, gn.T.reshape(-1)]))

    def _add_fgeo(self, blk):
        off = self._fsize
        self._fgeo.append(blk)
        self._fsize += blk.size
        return off

    def face_ids_of(self, r):
        """Local face index of (the first of) records r (all share it in a bucket)."""
        return int(self._rec_face[int(np.atleast_1d(r)[0])])

    def _shared_bucket(self, cl, fl, cr, fr, code, le, re_, rl, rr):
        """Shared trace (reference sipg.py:513-554): one grid (max q), one
        metric and one normal (left's; right uses -n)."""
        recs, d = self.recs, self.dim
        fd = d - 1
        swap = fd == 2 and bool((code >> 2) & 1)
        rules = []
        for k in range(fd):
            al = cl.faces[fl].run[k]
            ar = cr.faces[fr].run[(1 - k) if swap else k]
            rules.append(shared_rule(cl.rules[al], cr.rules[ar], self.shared_patched))
        t_axes = tuple(r_.points for r_ in rules)
        wt = np.ones(1)
        for r_ in rules:
            wt = np.multiply.outer(wt, r_.weights).reshape(-1)
        prm_t = tensor_params(t_axes)
        prm_tr = apply_code(code, prm_t)
        gl, gr = self.geo[self.exp_of[le[0]]], self.geo[self.exp_of[re_[0]]]
        swj, nl, invl, fcl, _ = gl.face(fl, prm_t, wt, self.exp_pos[le])
        _, _, invr, fcr, _ = gr.face(fr, prm_tr, np.ones(prm_t.shape[0]), self.exp_pos[re_])
        ml, swl, idl = axis_transfer(cl.face_pts(fl), t_axes, 0)
        mr, swr, idr = axis_transfer(cr.face_pts(fr), t_axes, code)
        self._perm_buckets.append((self._cur_mem, self._transfer_perm(cl.face_pts(fl), t_axes, 0, fd),
                                   self._transfer_perm(cr.face_pts(fr), t_axes, code, fd)))
        neg_r = fd == 1 and code == 1
        regular = fcl & fcr
        gxl = np.einsum("ekm,em->ek", invl[:, 0], nl[:, 0])
        gxr = np.einsum("ekm,em->ek", invr[:, 0], -nl[:, 0])
        wb = [self._rule_block(r_) for r_ in rules]
        for r, ms, sws, ids_, mo, swo, ido, negs, nego, gxs, gxo, self_is_left in (
                (rl, ml, swl, idl, mr, swr, idr, False, neg_r, gxl, gxr, True),
                (rr, mr, swr, idr, ml, swl, idl, neg_r, False, gxr, gxl, False)):
            recs["type"][r] = L.FT_SHARED
            fl_ = ((L.F_SELF_ID if ids_ else 0) | (L.F_SELF_SWAP if sws else 0) |
                   (L.F_OTHER_ID if ido else 0) | (L.F_OTHER_SWAP if swo else 0) |
                   (L.F_SELF_NEG if negs else 0) | (L.F_OTHER_NEG if nego else 0))
            recs["flags"][r] |= fl_
            recs["ts0"][r] = self.pool.add(ms[0])
            recs["ts1"][r] = self.pool.add(ms[1]) if fd > 1 else -1
            recs["to0"][r] = self.pool.add(mo[0])
            recs["to1"][r] = self.pool.add(mo[1]) if fd > 1 else -1
            recs["nt0"][r] = rules[0].n
            recs["nt1"][r] = rules[1].n if fd > 1 else 1
            recs["wt0"][r] = wb[0]
            recs["wt1"][r] = wb[1] if fd > 1 else -1
            recs["sJ"][r] = swj[:, 0] / wt[0]
            recs["gs"][r, :d] = gxs
            recs["go"][r, :d] = gxo
            # hex fast shared path: the other side's planes evaluated straight at the trace
            # points with E_k[t][i] = psi_i(other's parameter of t_k) (no axis swap here)
            c_o = cr if self_is_left else cl
            c_s = cl if self_is_left else cr
            if (d == 3 and not sws and not swo and c_o.kind.value == "modified_modal"
                    and c_s.kind.value == "modified_modal"
                    and all(c_.axis[a]["gll"] for c_ in (c_o, c_s) for a in range(3))
                    and c_o.n <= 9 and rules[0].n <= 11 and rules[1].n <= 11
                    and c_o.n <= c_s.n + SF_RANGE):
                code_o = code if self_is_left else 0
                sign = [-1.0 if (code_o >> 1) & 1 else 1.0, -1.0 if code_o & 1 else 1.0]
                E = [eval_basis_1d(c_o.kind, c_o.n, sign[k] * t_axes[k])[0] for k in range(2)]
                e0, e1 = self.pool.add(E[0]), self.pool.add(E[1])
                fs_ = self.face_ids_of(r)
                ok = regular.copy()
                a_s = FACES["hex"][fs_].fixed
                tang_s = [b for b in range(3) if b != a_s]
                f_o = fr if self_is_left else fl
                a_o = FACES["hex"][f_o].fixed
                tang_o = [b for b in range(3) if b != a_o]
                ok &= (gxs[:, tang_s[0]] == 0.0) & (gxs[:, tang_s[1]] == 0.0)
                ok &= (gxo[:, tang_o[0]] == 0.0) & (gxo[:, tang_o[1]] == 0.0)
                recs["flags"][r[ok]] |= L.F_FAST_SHARED
                self.rec_ext[r[ok], 1] = e0 | (e1 << 32)
            for j in np.flatnonzero(~regular):
                gn_l = gn_at(cl, fl, invl[j:j + 1], nl[j:j + 1], prm_t)[0]
                gn_r = gn_at(cr, fr, invr[j:j + 1], -nl[j:j + 1], prm_tr)[0]
                gs, go = (gn_l, gn_r) if self_is_left else (gn_r, gn_l)
                recs["flags"][r[j]] |= L.F_SELF_PW | L.F_OTHER_PW
                recs["geo"][r[j]] = self._add_fgeo(np.concatenate([swj[j], gs.T.reshape(-1), go.T.reshape(-1)]))

    def _finish(self):
        nb = self.recs["nbr"]
        self.recs["nbr_dof"] = np.where(nb >= 0, self.dof_off[np.maximum(nb, 0)], -1)
        # published face planes (hex): per element 6 faces x (boundary-mode plane, normal-
        # derivative plane), each N^2 doubles padded to even -> 16-byte aligned blocks
        # 2-D: per element, per face, (u, du/deta_0, du/deta_1) on the face's own q points
        nel = len(self.ct)
        is2d = self.dim == 2
        if is2d:
            qe = np.array([c.nq[0] for c in self.exp_list])[self.exp_of]
            nfe = np.array([len(c.faces) for c in self.exp_list])[self.exp_of]
            per_face = 3 * qe
            sizes = nfe * per_face
            sizes = (sizes + 1) & ~1
        else:
            nn = np.array([(c.n * c.n + 1) & ~1 if c.shape == "hex" else 0 for c in self.exp_list])[self.exp_of]
            per_face = 2 * nn
            sizes = 12 * nn
        self.plane_off = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
        self.plane_off[sizes == 0] = -1
        self.n_planes = int(sizes.sum())
        has = (nb >= 0)
        nbr = np.maximum(nb, 0)
        nfo = self.recs["nbr_face"].astype(np.int64)
        po = self.plane_off[nbr] + nfo * per_face[nbr]
        size_o = (qe if is2d else np.array([c.n for c in self.exp_list])[self.exp_of])[nbr].astype(np.int64)
        ok = has & (self.plane_off[nbr] >= 0)
        self.rec_ext[ok, 0] = po[ok] | (size_o[ok] << 48)
        self.fgeo = np.concatenate(self._fgeo) if self._fgeo else np.zeros(1)
        self.tables = self.pool.array()
