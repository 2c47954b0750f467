"""`HelmholtzOperator.exps` / `.factors`: the reference's per-element setup objects
(reference sipg.py:262-267: `exps = [expansion(...) for e]`, `factors = geometric_factors(mesh,
exps)`, mesh.py:295-357 ElementFactors / FaceFactors / GeometricFactors).

They are not on the hot path (the device plan carries its own compact geometry); they are built
lazily on first access, vectorised per element class, with the reference's field names and
shapes: `J` (1,) or (n_phys,), `dxi_dx` (d, d, 1) or (d, d, n_phys), `jac_w`, `x` (d, n_phys),
`volume`, and per face `normal` (d, 1|n), `surf_jac` (1|n), `surf_jw`, `x`, `area`, `dxi_dx`.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .plan import ElemGeo, jacobians
from .stdregions import FACES

__all__ = ["FaceFactors", "ElementFactors", "GeometricFactors", "standard_factors", "hybrid_factors"]


@dataclass
class FaceFactors:
    normal: np.ndarray
    surf_jac: np.ndarray
    surf_jw: np.ndarray
    x: np.ndarray
    area: float
    dxi_dx: np.ndarray | None = None


@dataclass
class ElementFactors:
    regular: bool
    J: np.ndarray
    dxi_dx: np.ndarray
    jac_w: np.ndarray
    x: np.ndarray
    volume: float
    faces: list = field(default_factory=list)


@dataclass
class GeometricFactors:
    elements: list

    def __getitem__(self, e: int) -> ElementFactors:
        return self.elements[e]

    def __len__(self) -> int:
        return len(self.elements)


def _compact(a, const):
    """(n, ...) per-point array -> (1, ...) when constant (reference mesh.py:343-348)."""
    return a[:1] if const else a


def standard_factors(mesh, plan) -> GeometricFactors:
    """Quad / tri / hex plans (plan.PlanBuilder): one ElemGeo per expansion class."""
    verts_all = np.asarray(mesh.vertices, dtype=float)
    nel = len(plan.ct)
    out = [None] * nel
    exp_of = np.asarray(plan.exp_of)
    for c, ct in enumerate(plan.exp_list):
        ids = np.flatnonzero(exp_of == c)
        if ids.size == 0:
            continue
        V = verts_all[np.array([mesh.elements[e].verts for e in ids], dtype=np.int64)]
        geo = ElemGeo(ct, V)
        x, F = jacobians(ct.shape, V, ct.xi)
        J = np.linalg.det(F)
        inv = np.linalg.inv(F)                       # [e, p, m, i] = dxi_m / dx_i
        d = ct.dim
        face_data = []
        for f, fd in enumerate(FACES[ct.shape]):
            pts = ct.face_pts(f)
            g = np.meshgrid(*pts, indexing="ij")
            prm = np.stack([a.reshape(-1) for a in g], axis=-1)
            swj, nrm, finv, _, ncst = geo.face(f, prm, ct.face_weights(f))
            xi = np.asarray(fd.center) + prm @ np.asarray(fd.tangents)
            xf, _ = jacobians(ct.shape, V, xi)
            face_data.append((swj, nrm, finv, ncst, xf, ct.face_weights(f)))
        for k, e in enumerate(ids):
            reg = bool(geo.regular[k])
            faces = []
            for swj, nrm, finv, ncst, xf, w in face_data:
                sj = swj[k] / w
                sj_c = bool(np.abs(sj - sj[0]).max() < 1e-12 * (abs(sj[0]) + 1.0))
                faces.append(FaceFactors(
                    normal=np.ascontiguousarray(nrm[k].T if not ncst[k] else nrm[k][:1].T),
                    surf_jac=_compact(sj, sj_c), surf_jw=swj[k], x=np.ascontiguousarray(xf[k].T),
                    area=float(swj[k].sum()),
                    dxi_dx=np.ascontiguousarray(finv[k].transpose(1, 2, 0))))
            out[e] = ElementFactors(
                regular=reg, J=_compact(J[k], reg), dxi_dx=np.ascontiguousarray(_compact(inv[k], reg).transpose(1, 2, 0)),
                jac_w=J[k] * ct.ref_w, x=np.ascontiguousarray(x[k].T), volume=float(geo.volume[k]), faces=faces)
    return GeometricFactors(out)


def hybrid_factors(plan) -> GeometricFactors:
    """Config-4 hybrid plans (plan3d.Plan3DBuilder): affine elements, constant metric."""
    from .plan3d import FACES as FACES3, xi_of_eta
    nel = len(plan.shapes)
    out = [None] * nel
    for e in range(nel):
        ct = plan.ct[plan.class_of[e]]
        q = ct.q
        g = np.meshgrid(*ct.pts, indexing="ij")
        eta = np.stack([a.reshape(-1) for a in g], axis=-1)
        xi = xi_of_eta(ct.shape, eta)
        x = plan.x0[e][:, None] + plan.F[e] @ (xi.T + 1.0)
        faces = []
        for f, (fixed, side, run, tri, _) in enumerate(FACES3[ct.shape]):
            nrm, sJ = plan._face_frame(np.array([e]), f)
            gf = np.meshgrid(ct.pts[run[0]], ct.pts[run[1]], indexing="ij")
            et = np.zeros((q * q, 3))
            et[:, fixed] = side
            et[:, run[0]], et[:, run[1]] = gf[0].reshape(-1), gf[1].reshape(-1)
            xf = plan.x0[e][:, None] + plan.F[e] @ (xi_of_eta(ct.shape, et).T + 1.0)
            swj = sJ[0] * ct.face_wt[f]
            faces.append(FaceFactors(normal=nrm[0][:, None], surf_jac=np.array([sJ[0]]), surf_jw=swj, x=xf,
                                     area=float(swj.sum()), dxi_dx=plan.dxidx[e][:, :, None]))
        out[e] = ElementFactors(regular=True, J=np.array([plan.detJ[e]]), dxi_dx=plan.dxidx[e][:, :, None],
                                jac_w=plan.detJ[e] * ct.wref, x=x, volume=float(plan.detJ[e] * ct.wref.sum()),
                                faces=faces)
    return GeometricFactors(out)
