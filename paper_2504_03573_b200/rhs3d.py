"""Right-hand side and L2 error on the GPU for hybrid 3-D plans.

Restates the reference's `HelmholtzOperator.rhs_assemble(case, bcs)` (sipg.py:697-718) and
`l2_error(x, exact)` (sipg.py:720-741) on a `plan3d` plan:

* b = -(v, f): per element class one device GEMM  -Phi^T (jw * f)  with the class's dense
  modified-modal table Phi (q^3 x n_c, built from the plan's 1-D / collapsed tables — a plain
  library GEMM, cuBLAS through torch), f evaluated by the caller's `case.forcing` at the
  physical volume points (the reference evaluates it on the host too);
* the Dirichlet lift (sipg.py:707-717: absorb of jump = -2 g, average 0, sign -1 on the boundary
  faces) is the apply kernels themselves run on x = 0 with g as the boundary slots' own trace and
  0 as its normal derivative (sipg_h3_apply_traces): the boundary flux of u = g there is term for
  term the reference's lift;
* l2_error: u_h on rules with two extra points per direction (dense GEMM per class) against
  `exact` at the physical points, jw-weighted sum on the device.

The user callables see the reference's shapes: forcing / exact get x of shape (3, n_points, W),
the boundary data g gets (3, n_face_points).
"""
from __future__ import annotations

import math

import numpy as np

from .plan3d import FACES, CD3_COUNT, CD3_ELEM_OFF, ClassTables3, xi_of_eta


def _tri_groups(n, tet):
    gof = []
    for i in range(n):
        for j in range(n - i):
            gof.append(1 if (i == 0 and j == 1) else (0 if i == 0 else (2 if i == 1 else i + 1)))
    if tet:
        gof.append(1)
    mofr = []
    if tet:
        for m, (i, j) in enumerate((i, j) for i in range(n) for j in range(n - i)):
            mofr += [m] * (n - max(i + j, 1))
        mofr.append(len(gof) - 1)
    return np.array(gof), np.array(mofr, dtype=np.int64)


def dense_phi(ct: ClassTables3) -> np.ndarray:
    """Phi[(k0, k1, k2), mode] (q^3 x n_c) from the class's staged tables (the product of the
    BwdTrans stages that csrc/sipg_h3.cuh contracts one at a time)."""
    q, n = ct.q, ct.n
    P = ct.parts
    if ct.shape == "hex":
        V = P["A"].reshape(q, n)
        return np.einsum("ai,bj,ck->abcijk", V, V, V).reshape(q ** 3, n ** 3)
    gof, mofr = _tri_groups(n, ct.shape == "tet")
    A = P["A"].reshape(q, n + 1)
    B = P["B"].reshape(len(gof), q)
    if ct.shape == "prism":
        psi = P["C"].reshape(q, n)
        out = np.einsum("am,bl,mc->abcml", A[:, gof], psi, B)
        return out.reshape(q ** 3, len(gof) * n)
    C = P["C"].reshape(ct.nc, q)
    out = np.einsum("ar,br,rc->abcr", A[:, gof[mofr]], B[mofr].T, C)
    return out.reshape(q ** 3, ct.nc)


def _eta_grid(ct):
    g = np.meshgrid(*ct.pts, indexing="ij")
    return np.stack([a.reshape(-1) for a in g], axis=-1)


def _phys(pb, elems, xi):
    """Physical points (3, n_points, W) of reference points xi (n_points, 3) in elements `elems`."""
    x = pb.x0[elems][:, :, None] + np.einsum("eij,pj->eip", pb.F[elems], xi + 1.0)
    return np.ascontiguousarray(x.transpose(1, 2, 0))


def _classes(pb):
    for c, cd in enumerate(pb.class_desc):
        ids = pb.class_elems[cd[CD3_ELEM_OFF]:cd[CD3_ELEM_OFF] + cd[CD3_COUNT]].astype(np.int64)
        if ids.size:
            yield c, pb.ct[c], ids


def _geo_dev(op):
    """Element maps x = x0 + F (xi + 1) on the device (cached on the operator)."""
    import torch
    if getattr(op, "_geo_dev_cache", None) is None:
        op._geo_dev_cache = (torch.from_numpy(np.ascontiguousarray(op.plan.x0)).cuda(),
                             torch.from_numpy(np.ascontiguousarray(op.plan.F)).cuda())
    return op._geo_dev_cache


def _phys_dev(op, elems, xi):
    """Physical points (3, n_points, W) on the device."""
    import torch
    x0, F = _geo_dev(op)
    e = torch.from_numpy(np.asarray(elems, dtype=np.int64)).cuda()
    xr = torch.from_numpy(np.ascontiguousarray(xi + 1.0)).cuda()
    return (x0[e][:, :, None] + torch.einsum("eij,pj->eip", F[e], xr)).permute(1, 2, 0)


def rhs_assemble(op, case, bcs, tag: str = "dirichlet"):
    """b = -(v, f) + Dirichlet lift, a numpy vector (reference sipg.py:697-718).  With
    device-capable callables (cases.py) every step stays on the GPU; otherwise the callables get
    host points like the reference's."""
    import torch
    from .cases import device_callable
    pb = op.plan
    if tag not in bcs:
        raise KeyError(f"no boundary condition for tag {tag!r}")
    dev = torch.device("cuda")
    on_dev = device_callable(case.forcing, 3)
    b = torch.zeros(pb.n_dofs, dtype=torch.float64, device=dev)
    for c, ct, ids in _classes(pb):
        xi = xi_of_eta(ct.shape, _eta_grid(ct))
        if on_dev:
            f = case.forcing(_phys_dev(op, ids, xi))                                     # (p, W)
        else:
            f = torch.from_numpy(np.asarray(case.forcing(_phys(pb, ids, xi)), dtype=float)).to(dev)
        jw = torch.from_numpy(ct.wref[:, None] * pb.detJ[ids][None, :]).to(dev)
        phi = torch.from_numpy(dense_phi(ct)).to(dev)
        contrib = -(phi.T @ (f * jw))                                                    # (n_c, W)
        dof = torch.from_numpy((pb.dof_off[ids][None, :] + np.arange(ct.nc)[:, None]).reshape(-1)).to(dev)
        b.index_copy_(0, dof, contrib.reshape(-1))
    # boundary lift: the apply kernels on x = 0 with g as the boundary slots' own traces
    gfun = bcs[tag]
    g_dev = device_callable(gfun, 3)
    traces = np.zeros(max(op.native.trace_len, 1))
    tr = torch.zeros(max(op.native.trace_len, 1), dtype=torch.float64, device=dev) if g_dev else None
    S = pb.slots
    bnd = np.flatnonzero(S["kind"] == 0)
    for key in np.unique(np.stack([pb.class_of[S["elem"][bnd]], S["face"][bnd]], axis=1), axis=0):
        c, f = int(key[0]), int(key[1])
        sel = bnd[(pb.class_of[S["elem"][bnd]] == c) & (S["face"][bnd] == f)]
        ct = pb.ct[c]
        fixed, side, run, _, _ = FACES[ct.shape][f]
        g = np.meshgrid(ct.pts[run[0]], ct.pts[run[1]], indexing="ij")
        eta = np.zeros((g[0].size, 3))
        eta[:, fixed] = side
        eta[:, run[0]] = g[0].reshape(-1)
        eta[:, run[1]] = g[1].reshape(-1)
        off = S["pub_self"][sel][:, None] + 2 * np.arange(eta.shape[0])[None, :]
        if g_dev:      # pointwise data: all faces of the group in one call
            xs = _phys_dev(op, S["elem"][sel].astype(np.int64), xi_of_eta(ct.shape, eta))  # (3, nf, W)
            tr[torch.from_numpy(off.reshape(-1)).cuda()] = gfun(xs).T.reshape(-1)
        else:          # the reference's call pattern: one boundary face at a time, host points
            xs = _phys(pb, S["elem"][sel].astype(np.int64), xi_of_eta(ct.shape, eta))      # (3, nf, W)
            gv = np.stack([np.asarray(gfun(xs[:, :, w]), dtype=float) for w in range(len(sel))])   # (W, nf)
            traces[off] = gv
    if tr is None:
        tr = torch.from_numpy(traces).to(dev)
    x0 = torch.zeros(pb.n_dofs, dtype=torch.float64, device=dev)
    lift = torch.empty_like(x0)
    stream = torch.cuda.current_stream().cuda_stream
    op.native.apply_traces(x0.data_ptr(), tr.data_ptr(), lift.data_ptr(), stream)
    return (b + lift).cpu().numpy()


def l2_error(op, x, exact) -> float:
    """sqrt(sum_e int (u_h - u)^2 J) on rules with 2 extra points per direction (sipg.py:720-741)."""
    import torch
    pb = op.plan
    dev = torch.device("cuda")
    xd = torch.as_tensor(np.asarray(x, dtype=float)).to(dev) if not hasattr(x, "is_cuda") else x
    err2 = torch.zeros((), dtype=torch.float64, device=dev)
    from .cases import device_callable
    on_dev = device_callable(exact, 3)
    for c, ct, ids in _classes(pb):
        fine = ClassTables3(ct.shape, ct.n, ct.q + 2)
        xi = xi_of_eta(ct.shape, _eta_grid(fine))
        if on_dev:
            u = exact(_phys_dev(op, ids, xi))                                           # (p, W)
        else:
            u = torch.from_numpy(np.asarray(exact(_phys(pb, ids, xi)), dtype=float)).to(dev)
        dof = torch.from_numpy(pb.dof_off[ids][None, :] + np.arange(ct.nc)[:, None]).to(dev)
        uh = torch.from_numpy(dense_phi(fine)).to(dev) @ xd[dof]                        # (p, W)
        jw = torch.from_numpy(fine.wref[:, None] * pb.detJ[ids][None, :]).to(dev)
        d = uh - u
        err2 += (d * d * jw).sum()
    return math.sqrt(float(err2))
