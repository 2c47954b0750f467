"""Slab partition of a config-4 plan with a trace-only halo.

The paper's distributed apply exchanges only trace data between partitions — no ghost elements.
The reference keeps the exchange point as an in-memory double buffer between its phase 1 (volume
work + trace publish, sipg.py:569-592, which writes u and n.grad u per face point, 585-592) and
phase 2 (interface flux, 607-651), sipg.py:565-567.  This build keeps exactly that split: the
publish kernels of every rank write (u, n.grad u) per trace point into the rank's published-trace
buffer, the partition-face slots' traces cross to the neighbour rank (NCCL send / recv inside
libsipg.so, sipg_comm_init), and the apply kernels read the partner traces from there.

`partition_plan` cuts the GLOBAL plan (built identically on every rank) rather than building a
plan from local geometry: every owned element keeps its global slot records (trace maps, penalty,
surface Jacobian, normal) bit for bit, the partner's trace is computed by the same kernel from the
same data on the other rank, so the owned part of y is bitwise identical to the one-GPU apply for
any rank count.

Layout of a rank's published-trace buffer (doubles):
  [ own slots that nobody else reads | send range to nbr 0 | send range to nbr 1 | ... |
    receive range from nbr 0 | receive range from nbr 1 | ... ]
A send range holds this rank's slots whose partner lives on that neighbour, ordered by global slot
id; the receiving rank lays out its receive range from the same rank in the order of those
partner slots' global ids — so a single contiguous ncclSend / ncclRecv pair per neighbour moves
the halo with no pack or unpack kernel, and the apply kernels read the received traces in place
(slot.pub_other points into the receive range).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .plan3d import CD3_COUNT, CD3_ELEM_OFF, CD3_ROLE, n_coeffs

__all__ = ["element_weights3d", "slab_ranges3d", "PartitionPlan", "partition_plan"]


def element_weights3d(shapes, n_modes) -> np.ndarray:
    """Relative cost of an element (all shapes carry q^3 points; sum-factorised ~ q^4 n)."""
    n = np.asarray(n_modes, dtype=float)
    return (n + 1.0) ** 4 * n


def slab_ranges3d(weights, world: int) -> list:
    """Contiguous element ranges [lo, hi) per rank with balanced weights.  Config-4 meshes number
    the cubes x slowest (mesh3d.generate_hybrid3d), so a range is an x-slab of cubes."""
    cw = np.concatenate([[0.0], np.cumsum(weights)])
    cuts = [0] + [int(np.searchsorted(cw, cw[-1] * r / world)) for r in range(1, world)] + [len(weights)]
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


@dataclass
class PartitionPlan:
    """A rank's device plan (the Plan3DBuilder attribute set NativePlan reads) plus its halo."""
    rank: int
    world: int
    lo: int
    hi: int
    dof_lo: int
    dof_hi: int
    lam: float
    class_desc: np.ndarray
    class_elems: np.ndarray
    dof_off: np.ndarray
    egeo: np.ndarray
    slot_off: np.ndarray
    slots: np.ndarray
    tables: np.ndarray
    n_pub: int
    n_dofs: int
    nbr: np.ndarray                 # neighbour ranks
    send_off: np.ndarray            # per neighbour, doubles of the published-trace buffer
    send_cnt: np.ndarray
    recv_off: np.ndarray
    recv_cnt: np.ndarray
    roles: np.ndarray               # per owned element: 0 interior, 1 boundary layer
    is_h3: bool = True
    extra: dict = field(default_factory=dict)

    @property
    def halo_doubles(self) -> int:
        return int(self.send_cnt.sum())


def partition_plan(pb, ranges, rank: int) -> PartitionPlan:
    """Rank `rank`'s part of the global hybrid plan `pb` (plan3d.Plan3DBuilder, built)."""
    lo, hi = ranges[rank]
    world = len(ranges)
    nel = len(pb.shapes)
    owner = np.empty(nel, dtype=np.int64)
    for r, (a, b) in enumerate(ranges):
        owner[a:b] = r
    S = pb.slots
    s0, s1 = int(pb.slot_off[lo]), int(pb.slot_off[hi])
    gids = np.arange(s0, s1)                          # global ids of the owned slots (sorted by element)
    L = S[s0:s1].copy()
    gp = S["partner"][s0:s1].astype(np.int64)         # global partner slot (-1 boundary)
    pown = np.where(gp >= 0, owner[S["elem"][np.maximum(gp, 0)]], rank)
    remote = (gp >= 0) & (pown != rank)
    L["elem"] = S["elem"][s0:s1] - lo
    L["partner"] = np.where((gp >= 0) & ~remote, gp - s0, -1)
    # roles: 1 = owns a slot whose partner lives on another rank
    roles = np.zeros(hi - lo, dtype=np.int64)
    roles[np.unique(L["elem"][remote])] = 1
    nbrs = np.unique(pown[remote])
    size = 2 * L["nt"].astype(np.int64)
    # published-trace layout: quiet slots, then per neighbour the send slots (global id order),
    # then per neighbour the receive ranges (partner global id order)
    pub = np.empty(s1 - s0, dtype=np.int64)
    quiet = np.flatnonzero(~remote)
    off = 0
    pub[quiet] = off + np.concatenate([[0], np.cumsum(size[quiet])[:-1]]) if quiet.size else 0
    off += int(size[quiet].sum())
    send_off, send_cnt = [], []
    for r in nbrs:
        sel = np.flatnonzero(remote & (pown == r))      # already ascending in global id
        send_off.append(off)
        pub[sel] = off + np.concatenate([[0], np.cumsum(size[sel])[:-1]])
        send_cnt.append(int(size[sel].sum()))
        off += send_cnt[-1]
    other = np.full(s1 - s0, -1, dtype=np.int64)
    recv_off, recv_cnt = [], []
    for r in nbrs:
        sel = np.flatnonzero(remote & (pown == r))
        sel = sel[np.argsort(gp[sel], kind="stable")]   # the sender's order: its global slot ids
        recv_off.append(off)
        other[sel] = off + np.concatenate([[0], np.cumsum(size[sel])[:-1]])
        recv_cnt.append(int(size[sel].sum()))
        off += recv_cnt[-1]
    L["pub_self"] = pub
    local_partner = L["partner"]
    other = np.where(local_partner >= 0, pub[np.maximum(local_partner, 0)], other)
    L["pub_other"] = np.where(gp >= 0, other, -1)
    # classes (shape, n, role), global class tables and constant-table layout reused
    gcls = pb.class_of[lo:hi]
    keys = sorted(set(zip(gcls.tolist(), roles.tolist())))
    cd = np.zeros((len(keys), pb.class_desc.shape[1]), dtype=np.int32)
    elems, eoff = [], 0
    for c, (g, role) in enumerate(keys):
        ids = np.flatnonzero((gcls == g) & (roles == role)).astype(np.int32)
        cd[c] = pb.class_desc[g]
        cd[c, CD3_COUNT], cd[c, CD3_ELEM_OFF], cd[c, CD3_ROLE] = ids.size, eoff, role
        elems.append(ids)
        eoff += ids.size
    dof = pb.dof_off[lo:hi + 1] - pb.dof_off[lo]
    return PartitionPlan(
        rank=rank, world=world, lo=lo, hi=hi, dof_lo=int(pb.dof_off[lo]), dof_hi=int(pb.dof_off[hi]), lam=pb.lam,
        class_desc=cd, class_elems=np.concatenate(elems) if elems else np.zeros(0, np.int32),
        dof_off=dof.astype(np.int64), egeo=pb.egeo[lo:hi], slot_off=(pb.slot_off[lo:hi + 1] - s0).astype(np.int64),
        slots=L, tables=pb.tables, n_pub=max(off, 1), n_dofs=int(dof[-1]),
        nbr=nbrs.astype(np.int32), send_off=np.asarray(send_off, np.int64), send_cnt=np.asarray(send_cnt, np.int64),
        recv_off=np.asarray(recv_off, np.int64), recv_cnt=np.asarray(recv_cnt, np.int64), roles=roles)
