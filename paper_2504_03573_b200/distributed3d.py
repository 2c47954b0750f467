"""Multi-GPU apply for config-4 hybrid hex / prism / tet meshes: one process per
GPU, x-slab partition of the configuration itself (strong scaling), trace-only halo.

Every rank builds the same global plan (plan3d.Plan3DBuilder, deterministic), keeps its slab of
elements (halo3d.partition_plan: the global slot records bit for bit, published-trace buffer laid
out with one contiguous send and one receive range per neighbour) and creates its device plan.
Rank 0 makes an NCCL unique id (sipg_nccl_unique_id), the process group broadcasts it, and every
rank builds its communicator inside libsipg.so (sipg_comm_init).  One apply (sipg_apply) is then:

  publish the boundary-layer elements' traces  ->  ncclSend / ncclRecv of the partition-face traces
  (u and n.grad u per trace point, the paper's two scalars) on a high-priority
  comm stream, while the interior elements publish and apply  ->  the boundary layer applies.

The owned part of y is bitwise identical to the one-GPU apply for any rank count (the same kernel
runs on the same data for every element and every trace; tests/test_partition3d.py).
"""
from __future__ import annotations

import numpy as np

from .halo3d import element_weights3d, partition_plan, slab_ranges3d

__all__ = ["DistributedHelmholtz3D", "partition_ranks"]


def partition_ranks(pb, world: int) -> list:
    """Slab ranges of a built global plan, balanced by the per-element cost."""
    return slab_ranges3d(element_weights3d(pb.shapes, pb.nm), world)


class DistributedHelmholtz3D:
    """Rank-local part of a config-4 operator.  `dist` is an initialised torch.distributed group
    (any backend: it only broadcasts the 128-byte NCCL id); `transport="none"` skips the
    communicator (the caller moves the halo itself, e.g. the loop-back tests)."""

    def __init__(self, mesh, order_map, rank: int, world: int, dist=None, *, lambda_: float = 1.0,
                 transport: str = "nccl", global_plan=None, **_unused):
        from . import _native
        from .plan3d import Plan3DBuilder
        self.rank, self.world = rank, world
        self.global_plan = global_plan if global_plan is not None else \
            Plan3DBuilder(mesh, order_map, lambda_=lambda_).build()
        self.ranges = partition_ranks(self.global_plan, world)
        self.part = partition_plan(self.global_plan, self.ranges, rank)
        self.native = _native.NativePlan(self.part)
        self.native.set_halo(self.part)
        self.n_dofs = self.part.n_dofs
        self.n_global = int(self.global_plan.n_dofs)
        self.dof_lo, self.dof_hi = self.part.dof_lo, self.part.dof_hi
        if transport == "nccl" and world > 1:
            uid = [_native.nccl_unique_id() if rank == 0 else None]
            if dist is not None:
                dist.broadcast_object_list(uid, src=0)
            self.native.comm_init(uid[0], rank, world)

    @property
    def plan(self):
        return self.part

    @property
    def halo_bytes(self) -> int:
        """Bytes this rank sends per apply (= bytes it receives, by symmetry of the couplings)."""
        return 8 * self.part.halo_doubles

    def apply(self, x_local, y_local, stream_ptr: int = 0):
        """y_local = (A x)[owned] from x_local = x[owned] (device tensors / pointers)."""
        xp = x_local if isinstance(x_local, int) else x_local.data_ptr()
        yp = y_local if isinstance(y_local, int) else y_local.data_ptr()
        self.native.apply_device(xp, yp, stream_ptr)
