"""Multi-GPU apply for config-4 hybrid hex / prism / tet meshes: one process per
GPU, x-slab partition (contiguous element ranges; cubes are generated x slowest), one ghost layer.

A rank's local problem is its slab plus the elements that share a coupling with it.  The local
couplings are the global ones with at least one owned side (ghost-ghost and ghost-boundary
couplings are dropped: ghosts are never applied; they only publish traces toward owned
elements).  Per apply (sipg_apply_role on an h3 plan with element roles):

  role 0: publish the owned elements' traces, apply the elements whose partners are all owned;
          meanwhile the ghost coefficient blocks arrive (NCCL batch_isend_irecv on NVLink);
  role 1: publish the ghosts' traces, apply the elements touching a ghost.

Every element runs the single-GPU arithmetic on the same inputs, so the owned part of y is
bit-identical to the one-GPU apply for any rank count.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .distributed import HaloExchange
from .mesh import Element, Interface, OrderMap
from .mesh3d import HybridMesh3D
from .plan3d import n_coeffs


def element_weights3d(mesh, order_map) -> np.ndarray:
    """Relative cost per element: q^4 n (sum-factorised, all shapes use q^3 points)."""
    n = np.asarray(order_map.n_modes, dtype=float)
    q = np.asarray(order_map.n_quad, dtype=float)
    return q ** 4 * n


def slab_ranges3d(mesh, order_map, world: int) -> list:
    w = element_weights3d(mesh, order_map)
    cw = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0] + [int(np.searchsorted(cw, cw[-1] * r / world)) for r in range(1, world)] + [len(w)]
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def dof_offsets3d(mesh, order_map) -> np.ndarray:
    nc = np.array([n_coeffs(el.shape.value, int(n)) for el, n in zip(mesh.elements, order_map.n_modes)])
    off = np.zeros(len(nc) + 1, dtype=np.int64)
    off[1:] = np.cumsum(nc)
    return off


@dataclass
class LocalProblem3D:
    """Same fields as partition.LocalProblem (HaloExchange reads dof_lo, owned_local_dofs, send,
    recv)."""
    rank: int
    mesh: HybridMesh3D
    order_map: OrderMap
    local_ids: np.ndarray
    owned_mask: np.ndarray
    roles: np.ndarray
    dof_lo: int
    dof_hi: int
    owned_local_dofs: slice
    recv: dict
    send: dict


def local_problem3d(mesh, order_map, ranges, rank: int) -> LocalProblem3D:
    lo, hi = ranges[rank]
    owner = np.empty(ranges[-1][1], dtype=np.int64)
    for r, (a, b) in enumerate(ranges):
        owner[a:b] = r
    itf = mesh.interfaces
    le = np.array([t.left[0] for t in itf], dtype=np.int64)
    re_ = np.array([-1 if t.right is None else t.right[0] for t in itf], dtype=np.int64)
    own_l = (le >= lo) & (le < hi)
    own_r = (re_ >= lo) & (re_ < hi)
    keep = own_l | own_r
    ghosts = np.unique(np.concatenate([re_[own_l & (re_ >= 0) & ~own_r], le[own_r & ~own_l]]))
    local_ids = np.union1d(np.arange(lo, hi), ghosts)
    owned_mask = (local_ids >= lo) & (local_ids < hi)
    lid = -np.ones(len(mesh.elements), dtype=np.int64)
    lid[local_ids] = np.arange(local_ids.size)
    used = np.unique(np.concatenate([np.asarray(mesh.elements[g].verts) for g in local_ids]))
    vmap = -np.ones(len(mesh.vertices), dtype=np.int64)
    vmap[used] = np.arange(used.size)
    els = [Element(mesh.elements[g].shape, tuple(int(vmap[v]) for v in mesh.elements[g].verts)) for g in local_ids]
    couplings = []
    for i in np.flatnonzero(keep):     # global order (left e, left f, right e, right f) maps monotonically
        t = itf[i]
        left = (int(lid[t.left[0]]), t.left[1])
        right = None if t.right is None else (int(lid[t.right[0]]), t.right[1])
        couplings.append(Interface(left, right, -1, t.tag))
    sub = HybridMesh3D(np.asarray(mesh.vertices)[used], els, couplings)
    om = OrderMap(np.asarray(order_map.n_modes)[local_ids], np.asarray(order_map.n_quad)[local_ids])
    goff = dof_offsets3d(mesh, order_map)
    loff = dof_offsets3d(sub, om)
    owned_local = np.flatnonzero(owned_mask)
    o_lo, o_hi = int(loff[owned_local[0]]), int(loff[owned_local[-1] + 1])
    recv = {}
    for li in np.flatnonzero(~owned_mask):
        g = int(local_ids[li])
        src = int(owner[g])
        a, b = recv.get(src, (np.zeros(0, np.int64), np.zeros(0, np.int64)))
        recv[src] = (np.concatenate([a, np.arange(loff[li], loff[li + 1])]),
                     np.concatenate([b, np.arange(goff[g], goff[g + 1])]))
    # what the other ranks need from us: our owned elements coupled to theirs
    send = {}
    inter = re_ >= 0
    for dst in range(len(ranges)):
        if dst == rank:
            continue
        dlo, dhi = ranges[dst]
        in_d_l = (le >= dlo) & (le < dhi)
        in_d_r = (re_ >= dlo) & (re_ < dhi)
        need = np.unique(np.concatenate([re_[inter & in_d_l & own_r], le[inter & in_d_r & own_l]]))
        if need.size:
            send[dst] = np.concatenate([np.arange(goff[g], goff[g + 1]) for g in need])
    # roles: 0 owned with owned partners only, 1 owned touching a ghost, 2 ghost
    roles = np.where(owned_mask, 0, 2)
    touch = np.unique(np.concatenate([le[own_l & inter & ~own_r], re_[own_r & ~own_l]]))
    roles[lid[touch]] = 1
    return LocalProblem3D(rank, sub, om, local_ids, owned_mask, roles, int(goff[lo]), int(goff[hi]),
                          slice(o_lo, o_hi), recv, send)


class DistributedHelmholtz3D:
    """Rank-local hybrid operator on (slab + ghost layer) with overlapped exchange."""

    def __init__(self, mesh, order_map, rank: int, world: int, dist, device="cuda", **op_kwargs):
        from .sipg import HelmholtzOperator
        self.ranges = slab_ranges3d(mesh, order_map, world)
        self.lp = local_problem3d(mesh, order_map, self.ranges, rank)
        self.op = HelmholtzOperator(self.lp.mesh, self.lp.order_map, element_roles=self.lp.roles, **op_kwargs)
        self.halo = HaloExchange(self.lp, device, dist)
        self.n_local = self.op.n_dofs
        self.owned = self.lp.owned_local_dofs

    def apply(self, x_local, y_local, stream_ptr: int = 0):
        self.halo.start(x_local)
        self.op.native.apply_role(0, x_local.data_ptr(), y_local.data_ptr(), stream_ptr)
        self.halo.finish()
        self.op.native.apply_role(1, x_local.data_ptr(), y_local.data_ptr(), stream_ptr)
