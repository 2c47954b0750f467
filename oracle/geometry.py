"""ORACLE (test infrastructure only) — geometry and orientation.

Restates reference pkg/src/dgsipg/mesh.py (vertex maps 110-148, element factors
325-357, face factors 360-432) vectorised over a batch of elements, and
pkg/src/dgsipg/orient.py (25-50) / trace.py (84-106, 172-206).
"""
from __future__ import annotations

import numpy as np

from . import polylib as pl
from .elements import TRI

REF_VERTS = {
    "quad": np.array([[-1.0, -1.0], [1.0, -1.0], [1.0, 1.0], [-1.0, 1.0]]),
    "hex": np.array([[-1.0, -1.0, -1.0], [1.0, -1.0, -1.0], [1.0, 1.0, -1.0], [-1.0, 1.0, -1.0],
                     [-1.0, -1.0, 1.0], [1.0, -1.0, 1.0], [1.0, 1.0, 1.0], [-1.0, 1.0, 1.0]]),
}


def shape_funcs(shape, xi):
    """(N (npts, nv), dN (npts, nv, d)) — mesh.py:110-136."""
    xi = np.atleast_2d(xi)
    npts = xi.shape[0]
    if shape == TRI:
        n = np.stack([-0.5 * (xi[:, 0] + xi[:, 1]), 0.5 * (1 + xi[:, 0]), 0.5 * (1 + xi[:, 1])], axis=1)
        dn = np.broadcast_to(np.array([[[-0.5, -0.5], [0.5, 0.0], [0.0, 0.5]]]), (npts, 3, 2))
        return n, np.ascontiguousarray(dn)
    ref = REF_VERTS[shape]
    d = ref.shape[1]
    terms = 0.5 * (1.0 + xi[:, None, :] * ref[None, :, :])
    n = terms.prod(axis=2)
    dn = np.empty((npts, ref.shape[0], d))
    for j in range(d):
        others = [k for k in range(d) if k != j]
        dn[:, :, j] = 0.5 * ref[None, :, j] * terms[:, :, others].prod(axis=2)
    return n, dn


def _is_const(a):
    """mesh.py:325-328 along the point axis (axis 1 of a batch array)."""
    ref = a[:, :1]
    scale = np.abs(ref).reshape(a.shape[0], -1).max(axis=1) + 1.0
    dev = np.abs(a - ref).reshape(a.shape[0], -1).max(axis=1)
    return dev < 1e-12 * scale


def element_factors(shape, verts, exp):
    """Batch of elements (verts (nE, nv, d)) — mesh.py:331-357.
    Returns dict with x, J, dxidx (nE, d, d, npts) [regular: point-0 value
    broadcast], jw, volume, regular."""
    n, dn = shape_funcs(shape, exp.xi)
    x = np.einsum("pv,evi->epi", n, verts)
    F = np.einsum("pvj,evi->epij", dn, verts)
    J = np.linalg.det(F)
    if np.any(J <= 0.0):
        raise ValueError("non-positive Jacobian")
    inv = np.linalg.inv(F)                       # inv[e,p,m,i] = dxi_m/dx_i
    jw = J * exp.ref_w[None, :]
    regular = _is_const(F)
    dxidx = np.where(regular[:, None, None, None], inv[:, :1], inv)   # (nE, p, d, d)
    return {"x": x, "jw": jw, "dxidx": np.ascontiguousarray(dxidx.transpose(0, 2, 3, 1)),
            "volume": jw.sum(axis=1), "regular": regular}


def face_factors(shape, verts, exp, f, prm, weights=None):
    """Face factors at face parameters prm (npts, d-1) for a batch — mesh.py:360-432.
    normal (nE, d, npts) and dxidx (nE, d, d, npts) carry the reference's
    per-factor compaction (point-0 value when constant)."""
    face = exp.faces[f]
    prm = np.atleast_2d(prm)
    npts = prm.shape[0]
    if weights is None:
        weights = np.ones(npts)
    xi = face.to_ref(prm)
    n, dn = shape_funcs(shape, xi)
    x = np.einsum("pv,evi->epi", n, verts)
    F = np.einsum("pvj,evi->epij", dn, verts)
    tang = np.asarray(face.tangents)
    tp = np.einsum("epij,kj->epki", F, tang)
    if exp.dim == 2:
        t = tp[:, :, 0, :]
        surf = np.linalg.norm(t, axis=2)
        nrm = np.stack([t[..., 1], -t[..., 0]], axis=2)
    else:
        nrm = np.cross(tp[:, :, 0, :], tp[:, :, 1, :])
        surf = np.linalg.norm(nrm, axis=2)
    nrm = nrm / surf[..., None]
    inv = np.linalg.inv(F)
    out_dir = np.einsum("epji,j->epi", inv, np.asarray(face.ref_normal))
    sgn = np.where(np.einsum("epi,epi->ep", nrm, out_dir) >= 0.0, 1.0, -1.0)
    nrm = nrm * sgn[..., None]
    jw = surf * weights[None, :]
    cn = _is_const(nrm)
    ci = _is_const(inv)
    nrm_c = np.where(cn[:, None, None], nrm[:, :1], nrm)
    inv_c = np.where(ci[:, None, None, None], inv[:, :1], inv)
    return {"normal": np.ascontiguousarray(nrm_c.transpose(0, 2, 1)),
            "n_const": cn,
            "swj": jw, "area": jw.sum(axis=1), "x": x,
            "dxidx": np.ascontiguousarray(inv_c.transpose(0, 2, 3, 1))}


def tri_face_chain(exp, f, prm):
    """d eta / d xi at face parameters (tri) — sipg.py:172-188."""
    if exp.shape != TRI:
        return None
    face = exp.faces[f]
    p = np.atleast_2d(prm)[:, 0]
    if face.fixed == 0:
        e1, e2 = np.full_like(p, float(face.side)), p
    else:
        e1, e2 = p, np.full_like(p, -1.0)
    out = np.zeros((2, 2, p.size))
    out[0, 0] = 2.0 / (1.0 - e2)
    out[0, 1] = (1.0 + e1) / (1.0 - e2)
    out[1, 1] = 1.0
    return out


def side_gn(exp, f, dxidx, normal, prm):
    """(G n)_k at face points for a batch: dxidx (nE,d,d,npts), normal (nE,d,npts)
    -> (d, nE, npts) — sipg.py:191-200."""
    chain = tri_face_chain(exp, f, prm)
    if chain is not None:
        dxidx = np.einsum("kmp,emjp->ekjp", chain, dxidx)
    return np.einsum("ekmp,emp->kep", dxidx, normal)


# --- orientation codes (orient.py) ----------------------------------------

def apply_code(code, p):
    """orient.py:25-38."""
    p = np.atleast_2d(np.asarray(p, dtype=float))
    d = p.shape[1]
    if d == 0:
        return p.copy()
    if d == 1:
        return -p if code == 1 else p.copy()
    out = p[:, ::-1].copy() if (code >> 2) & 1 else p.copy()
    if (code >> 1) & 1:
        out[:, 0] = -out[:, 0]
    if code & 1:
        out[:, 1] = -out[:, 1]
    return out


def inverse_code(code, fd):
    """orient.py:41-50."""
    if fd == 0:
        return 0
    probe = np.array([[0.25, 0.625]])[:, :fd]
    fwd = apply_code(code, probe)
    for c in range({1: 2, 2: 8}[fd]):
        if np.allclose(apply_code(c, fwd), probe):
            return c
    raise ValueError(code)


def tensor_params(axes):
    if not axes:
        return np.zeros((1, 0))
    g = np.meshgrid(*axes, indexing="ij")
    return np.stack([a.reshape(-1) for a in g], axis=-1)


class Transfer:
    """identity / permutation / dense — trace.py:137-162."""

    def __init__(self, perm=None, matrix=None, identity=False):
        self.perm, self.matrix, self.identity = perm, matrix, identity

    def apply(self, v):
        if self.identity:
            return v
        if self.perm is not None:
            return v[..., self.perm]
        return v @ self.matrix.T


def transfer(src_axes, dst_axes, code):
    """trace.py:172-199."""
    src_axes = tuple(np.atleast_1d(p) for p in src_axes)
    dst = tensor_params(tuple(np.atleast_1d(p) for p in dst_axes))
    mapped = apply_code(code, dst)
    mats = [pl.interp(src_axes[k], mapped[:, k]) for k in range(len(src_axes))]
    if not mats:
        m = np.ones((1, 1))
    else:
        m = mats[0]
        for k in range(1, len(mats)):
            m = np.einsum("ti,tj->tij", m, mats[k]).reshape(m.shape[0], -1)
    if m.shape[0] == m.shape[1]:
        hits = np.isclose(m, 1.0, atol=1e-12)
        if np.all(hits.sum(axis=1) == 1) and np.allclose(m, hits.astype(float), atol=1e-12):
            perm = np.argmax(hits, axis=1)
            return Transfer(perm=perm, identity=bool(np.all(perm == np.arange(perm.size))))
    return Transfer(matrix=m)


def densify(t):
    """sipg.py:748-754."""
    if t.matrix is not None:
        return t
    n = t.perm.size
    m = np.zeros((n, n))
    m[np.arange(n), t.perm] = 1.0
    return Transfer(matrix=m)


def certify(left, right, p_geom=1, deformed=False):
    """(n, q, kind) per side -> (symmetric, cond1, cond2, required, actual)
    — trace.py:84-106."""
    npl, nql, kl = left
    npr, nqr, kr = right
    c1 = nql >= npr and nqr >= npl
    req = (npl - 1) + (npr - 1) + (3 * p_geom if deformed else p_geom)
    act = min(pl.exactness(kl, nql), pl.exactness(kr, nqr))
    return (c1 and act >= req), c1, act >= req, req, act


def shared_rule(kind_l, q_l, kind_r, q_r, patched=True):
    """trace.py:202-206 (higher side's kind); patched (P2): GLL only when both
    sides are GLL, else Gauss-Legendre, max(q) points."""
    if patched and not (kind_l == pl.GLL and kind_r == pl.GLL):
        return pl.GL, max(q_l, q_r)
    kind = kind_r if q_r > q_l else kind_l
    return kind, max(q_l, q_r)
