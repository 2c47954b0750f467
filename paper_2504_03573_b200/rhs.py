"""Right-hand side and L2 error on the GPU for the standard (quad / tri / hex) plans — SURVEY.md
§8f row f2, restating the reference's `HelmholtzOperator.rhs_assemble(case, bcs)` (sipg.py:697-718)
and `l2_error(x, exact)` (sipg.py:720-741):

* b = -(v, f): per expansion class one device GEMM  -Phi^T (jw * f), Phi the class's dense modal
  table at its volume points (mode order of the plan's DoF layout), jw = ref_w * det F per point
  (vertex maps, like the plan's geometry, plan.py `ElemGeo`);
* the Dirichlet lift: per boundary face (tag from the mesh's interface, KeyError when `bcs` lacks
  it, as the reference) the absorb of jump = -2 g, average 0 with sign -1 on the own face grid:
  fv = 2 tau g swj against the face trace table and fd = -g swj against (G n)_k times the
  eta-derivative tables (the reference's `_absorb`, sipg.py:663-677), batched per (class, face)
  as device GEMMs; tau is the plan's own penalty (plan.py `PlanBuilder._tau`);
* l2_error: u_h on rules with two extra points per direction of the same kinds (device GEMM per
  class) against `exact`, jw-weighted sum on the device.

The geometry and basis tables are set up in numpy on the host, as the plan is (setup work); the
products and reductions run on the GPU through torch (library GEMMs — this is not the hot path).
"""
from __future__ import annotations

import math

import numpy as np

from .mesh import element_vertex_array
from .plan import gn_at, jacobians, tensor_params
from .stdregions import FACES, class_tables, face_basis, tri_tables

NV = {"quad": 4, "tri": 3, "hex": 8}


def volume_basis(ct) -> np.ndarray:
    """Phi[point, mode] (n_phys x n_coeffs) of an expansion class at its volume points."""
    if ct.shape == "tri":
        A, _, B, _, gid = tri_tables(ct.kind, ct.n, ct.rules[0].points, ct.rules[1].points)
        out = A[:, None, gid] * B[None, :, :]
        return out.reshape(ct.n_phys, ct.n_coeffs)
    phi = np.ones((1, 1))
    for ax in range(ct.dim):
        V = ct.axis[ax]["V"]
        phi = np.einsum("pi,qj->pqij", phi, V).reshape(phi.shape[0] * V.shape[0], -1)
    return phi


def _fine(ct):
    return class_tables(ct.shape, ct.kind, ct.n, tuple(q + 2 for q in ct.nq),
                        tuple(r.kind.value for r in ct.rules))


def _volume(pb, i, ct, ids, verts, on_dev=False):
    """Physical points (d, p, W) as numpy (for the user's callbacks) and jw (p, W) on the device, of
    the class-i elements `ids` (vertex coords `verts` (W, nv, d)) at the volume points of `ct`.
    The vertex-map products run on the GPU; affine elements take the plan's constant Jacobian
    (ElemGeo.J0), the others det F per point (batched on the device)."""
    import torch
    from .plan import vertex_maps
    N, dN = vertex_maps(ct.shape, ct.xi)
    vd = _dev(verts)                                                          # (W, nv, d)
    x = torch.einsum("pv,evi->ipe", _dev(N), vd)
    g = pb.geo[i]
    pos = pb.exp_pos[ids]
    J = _dev(np.broadcast_to(g.J0[pos][None, :], (ct.n_phys, ids.size)))
    nr = np.flatnonzero(~g.regular[pos])
    if nr.size:
        F = torch.einsum("pvj,evi->epij", _dev(dN), vd[torch.from_numpy(nr).cuda()])
        J[:, torch.from_numpy(nr).cuda()] = torch.linalg.det(F).T
    return (x if on_dev else x.cpu().numpy()), J * _dev(ct.ref_w)[:, None]


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def rhs_assemble(op, case, bcs):
    """With device-capable callables (cases.py) the points stay on the GPU and the callables run
    there; otherwise they get host points like the reference's."""
    import torch
    from .cases import device_callable
    pb = op.plan
    mesh = op.mesh
    ev = element_vertex_array(mesh)
    X = np.asarray(mesh.vertices, dtype=float)
    on_dev = device_callable(case.forcing, mesh.dim)
    b = torch.zeros(pb.n_dofs, dtype=torch.float64, device="cuda")
    for i, ids in enumerate(pb.exp_members):
        if ids.size == 0:
            continue
        ct = pb.exp_list[i]
        xs, jw = _volume(pb, i, ct, ids, X[ev[ids, :NV[ct.shape]]], on_dev)
        f = case.forcing(xs) if on_dev else _dev(np.asarray(case.forcing(xs), dtype=float))
        contrib = -(_dev(volume_basis(ct)).T @ (f * jw))           # (nc, W)
        dof = pb.dof_off[ids][None, :] + np.arange(ct.n_coeffs)[:, None]
        b.index_copy_(0, torch.from_numpy(dof.reshape(-1)).cuda(), contrib.reshape(-1))
    # boundary faces grouped by (class, face, tag)
    bnd = [(itf.left[0], itf.left[1], itf.tag) for itf in mesh.interfaces if itf.right is None]
    groups = {}
    for e, f, tag in bnd:
        groups.setdefault((int(pb.exp_of[e]), int(f), tag), []).append(int(e))
    for (i, f, tag), el in groups.items():
        if tag not in bcs:
            raise KeyError(f"no boundary condition for tag {tag!r}")
        gfun = bcs[tag]
        el = np.asarray(el, dtype=np.int64)
        ct = pb.exp_list[i]
        face = FACES[ct.shape][f]
        prm = tensor_params(ct.face_pts(f))
        swj, nrm, inv, _, _ = pb.geo[i].face(f, prm, ct.face_weights(f), elems=pb.exp_pos[el])
        gn = gn_at(ct, f, inv, nrm, prm)                            # (W, p, d)
        xi = np.asarray(face.center) + prm @ np.asarray(face.tangents)
        if device_callable(gfun, mesh.dim):        # pointwise data: the whole group in one call
            from .plan import vertex_maps
            Nf, _ = vertex_maps(ct.shape, xi)
            xf = torch.einsum("pv,evi->ipe", _dev(Nf), _dev(X[ev[el, :NV[ct.shape]]]))   # (d, p, W)
            gv = gfun(xf).T                                                               # (W, p)
        else:                                      # the reference's pattern: one face at a time
            xf, _ = jacobians(ct.shape, X[ev[el, :NV[ct.shape]]], xi)   # (W, p, d)
            gv = _dev(np.stack([np.asarray(gfun(xf[w].T), dtype=float) for w in range(el.size)]))   # (W, p)
        tau = pb._tau(el, np.full(el.size, f))
        swj_d = _dev(swj)
        fv = 2.0 * _dev(tau)[:, None] * gv * swj_d
        fd = -gv * swj_d
        contrib = fv @ _dev(face_basis(ct, f, prm))
        for k in range(ct.dim):
            contrib += (fd * _dev(gn[:, :, k])) @ _dev(face_basis(ct, f, prm, deriv=k))
        dof = pb.dof_off[el][:, None] + np.arange(ct.n_coeffs)[None, :]
        b.index_add_(0, torch.from_numpy(dof.reshape(-1)).cuda(), contrib.reshape(-1))
    return b.cpu().numpy()


def l2_error(op, x, exact) -> float:
    import torch
    pb = op.plan
    mesh = op.mesh
    ev = element_vertex_array(mesh)
    X = np.asarray(mesh.vertices, dtype=float)
    from .cases import device_callable
    xd = x if (hasattr(x, "is_cuda") and x.is_cuda) else _dev(np.asarray(x, dtype=float))
    on_dev = device_callable(exact, mesh.dim)
    err2 = torch.zeros((), dtype=torch.float64, device="cuda")
    for i, ids in enumerate(pb.exp_members):
        if ids.size == 0:
            continue
        fine = _fine(pb.exp_list[i])
        xs, jw = _volume(pb, i, fine, ids, X[ev[ids, :NV[fine.shape]]], on_dev)
        dof = torch.from_numpy(pb.dof_off[ids][None, :] + np.arange(fine.n_coeffs)[:, None]).cuda()
        u = exact(xs) if on_dev else _dev(np.asarray(exact(xs), dtype=float))
        d = _dev(volume_basis(fine)) @ xd[dof] - u
        err2 += (d * d * jw).sum()
    return math.sqrt(float(err2))
