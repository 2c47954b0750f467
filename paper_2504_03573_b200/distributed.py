"""Multi-GPU apply for the quad / tri / hex plans (configs 0-3b): one process per GPU, x-slab
partition of the configuration, ghost-layer halo exchange over torch.distributed (NCCL on NVLink /
NVSwitch between GPUs; gloo in the CPU tests), overlapped with the elements that do not touch a
ghost.  These plans' kernels evaluate a neighbour's trace from its coefficient block in registers
(k_hex) or from its published planes, so the halo they need is the ghost layer's coefficients —
2.7x the bytes of the paper's trace-only exchange, which config 4 implements (halo3d.py,
distributed3d.py).

Per apply:  pack/send owned boundary-layer coefficients to the slab
neighbours and receive the ghost layer (one P2P batch); meanwhile launch the
role-0 classes (elements with only local neighbours); wait on the exchange;
launch the role-1 classes (elements touching a ghost).  Every element is
computed by exactly one rank with the single-GPU arithmetic, so the gathered
result is bit-identical to the one-GPU apply.
"""
from __future__ import annotations

import numpy as np

from .partition import LocalProblem, local_problem, neighbours, slab_ranges


def element_roles(lp: LocalProblem) -> np.ndarray:
    roles = np.where(lp.owned_mask, 0, 2)
    roles[lp.boundary_elems] = 1
    return roles


class HaloExchange:
    """Ghost-layer exchange for one rank (torch tensors on the exchange device)."""

    def __init__(self, lp: LocalProblem, device, dist):
        import torch
        self.dist = dist
        self.lp = lp
        off = lp.owned_local_dofs.start - lp.dof_lo          # global owned dof -> local dof
        self.sends = []
        for dst, gdofs in sorted(lp.send.items()):
            ldofs = torch.as_tensor(gdofs + off, device=device)
            contiguous = bool(np.all(np.diff(gdofs) == 1))
            self.sends.append((dst, ldofs, contiguous, int(gdofs[0] + off), gdofs.size))
        self.recvs = []
        for src, (ldofs, _) in sorted(lp.recv.items()):
            contiguous = bool(np.all(np.diff(ldofs) == 1))
            self.recvs.append((src, torch.as_tensor(ldofs, device=device), contiguous, int(ldofs[0]), ldofs.size))

    def start(self, x_local):
        """Post sends of owned coefficients and receives into the ghost slots (receive / pack
        buffers of non-contiguous ranges are allocated once per x_local storage)."""
        import torch
        key = (x_local.data_ptr(), x_local.device)
        if getattr(self, "_key", None) != key:
            self._key = key
            self._sbuf = [None if c else torch.empty(n, dtype=x_local.dtype, device=x_local.device)
                          for _, _, c, _, n in self.sends]
            self._rbuf = [None if c else torch.empty(n, dtype=x_local.dtype, device=x_local.device)
                          for _, _, c, _, n in self.recvs]
        ops, self._unpack = [], []
        for (dst, idx, contig, start, n), sb in zip(self.sends, self._sbuf):
            if contig:
                buf = x_local[start:start + n]
            else:
                torch.index_select(x_local, 0, idx, out=sb)
                buf = sb
            ops.append(self.dist.P2POp(self.dist.isend, buf, dst))
        for (src, idx, contig, start, n), rb in zip(self.recvs, self._rbuf):
            buf = x_local[start:start + n] if contig else rb
            ops.append(self.dist.P2POp(self.dist.irecv, buf, src))
            if not contig:
                self._unpack.append((idx, buf))
        self._reqs = self.dist.batch_isend_irecv(ops) if ops else []
        self._x = x_local

    def finish(self):
        for r in self._reqs:
            r.wait()
        for idx, buf in self._unpack:
            self._x.index_copy_(0, idx, buf)


class DistributedHelmholtz:
    """Rank-local operator on (slab + ghost layer) with overlapped exchange."""

    def __init__(self, mesh, order_map, rank: int, world: int, dist, device="cuda", **op_kwargs):
        from .sipg import HelmholtzOperator
        self.ranges = slab_ranges(mesh, order_map, world)
        self.lp = local_problem(mesh, order_map, self.ranges, rank, neighbours(mesh))
        self.op = HelmholtzOperator(self.lp.mesh, self.lp.order_map, element_roles=element_roles(self.lp),
                                    **op_kwargs)
        self.halo = HaloExchange(self.lp, device, dist)
        self.n_local = self.op.n_dofs
        self.owned = self.lp.owned_local_dofs

    def apply(self, x_local, y_local, stream_ptr: int = 0):
        """x_local: owned part filled; ghost part is refreshed here.  y_local:
        owned part written (ghost part untouched)."""
        self.halo.start(x_local)
        self.op.native.apply_role(0, x_local.data_ptr(), y_local.data_ptr(), stream_ptr)
        self.halo.finish()
        self.op.native.apply_role(1, x_local.data_ptr(), y_local.data_ptr(), stream_ptr)
