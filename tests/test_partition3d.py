"""Config-4 x-slab decomposition: local problems (slab + ghost layer, roles), ghost exchange over
gloo (2 ranks, CPU) feeding a numpy emulation of the h3 kernels on each rank's local plan, checked
against the global oracle; (GPU) the role-split local apply equals the global apply."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_03573_b200.distributed3d import local_problem3d, slab_ranges3d
from paper_2504_03573_b200.partition import stack_box_config

ROOT = Path(__file__).resolve().parent.parent


def test_local_problem3d_maps():
    m, om, _ = stack_box_config("cfg4", 3, nx=3, seed=2)
    r = slab_ranges3d(m, om, 3)
    assert r[0][0] == 0 and r[-1][1] == m.n_elements
    lps = [local_problem3d(m, om, r, k) for k in range(3)]
    for a in range(3):
        for b in range(3):
            if a != b and b in lps[a].recv:
                assert np.array_equal(lps[a].recv[b][1], lps[b].send[a])
    for lp in lps:
        assert lp.owned_local_dofs.stop - lp.owned_local_dofs.start == lp.dof_hi - lp.dof_lo
        assert set(np.unique(lp.roles)) <= {0, 1, 2}
        assert np.all((lp.roles == 2) == ~lp.owned_mask)
        # every coupling of an owned element is present locally, ghosts only couple to owned ones
        for t in lp.mesh.interfaces:
            sides = [t.left[0]] + ([] if t.right is None else [t.right[0]])
            assert any(lp.owned_mask[s] for s in sides)


def _worker(rank, world, port, nx, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, str(ROOT / "tools"))
        from h3_emulate import emulate
        from oracle.hybrid3d import HybridOracle3D
        from paper_2504_03573_b200.distributed import HaloExchange
        from paper_2504_03573_b200.plan3d import Plan3DBuilder
        m, om, rng = stack_box_config("cfg4", world, nx=nx, seed=3)
        ref = HybridOracle3D(m.shapes, [el.verts for el in m.elements], m.vertices, om.n_modes, om.n_quad)
        x = rng.uniform(-1.0, 1.0, ref.n_dofs)
        r = slab_ranges3d(m, om, world)
        lp = local_problem3d(m, om, r, rank)
        pb = Plan3DBuilder(lp.mesh, lp.order_map, element_roles=lp.roles).build()
        xl = torch.zeros(pb.n_dofs, dtype=torch.float64)
        xl[lp.owned_local_dofs] = torch.from_numpy(x[lp.dof_lo:lp.dof_hi])
        hx = HaloExchange(lp, "cpu", dist)
        hx.start(xl)
        hx.finish()
        y_own = emulate(pb, xl.numpy())[lp.owned_local_dofs]
        parts = [None] * world
        dist.all_gather_object(parts, (lp.dof_lo, y_own))
        if rank == 0:
            y = np.zeros(ref.n_dofs)
            for lo, yy in parts:
                y[lo:lo + yy.size] = yy
            yr = ref(x)
            q.put(float(np.abs(y - yr).max() / np.abs(yr).max()))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_match_global():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 3, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs)
    err = q.get(timeout=5)
    assert err <= 1e-13, err


@pytest.mark.gpu
def test_gpu_role_split_matches_global():
    """Each rank of a 3-slab decomposition on one GPU: ghosts filled from the global vector, roles 0
    then 1 launched; the owned output equals the global apply (to rounding: the local plan's trace
    maps are rebuilt from the local geometry)."""
    from paper_2504_03573_b200.sipg import HelmholtzOperator
    kw = dict(basis_kind="modified_modal", tau_rule="baseline")
    m, om, rng = stack_box_config("cfg4", 3, nx=4, seed=5)
    glob = HelmholtzOperator(m, om, **kw)
    x = rng.uniform(-1.0, 1.0, glob.n_dofs)
    y_ref = glob.lhs_eval(x)
    r = slab_ranges3d(m, om, 3)
    for rank in range(3):
        lp = local_problem3d(m, om, r, rank)
        op = HelmholtzOperator(lp.mesh, lp.order_map, element_roles=lp.roles, **kw)
        xl = np.zeros(op.n_dofs)
        xl[lp.owned_local_dofs] = x[lp.dof_lo:lp.dof_hi]
        for src, (ldofs, gdofs) in lp.recv.items():
            xl[ldofs] = x[gdofs]
        xd = torch.from_numpy(xl).cuda()
        yd = torch.zeros_like(xd)
        s = torch.cuda.current_stream().cuda_stream
        op.native.apply_role(0, xd.data_ptr(), yd.data_ptr(), s)
        op.native.apply_role(1, xd.data_ptr(), yd.data_ptr(), s)
        y_own = yd.cpu().numpy()[lp.owned_local_dofs]
        yr = y_ref[lp.dof_lo:lp.dof_hi]
        assert np.abs(y_own - yr).max() <= 1e-13 * np.abs(y_ref).max()
