"""Config-4 x-slab partition with a trace-only halo (halo3d.py / distributed3d.py):
send / receive layouts that match across ranks, a 2-rank gloo run of the publish -> exchange ->
apply sequence on the numpy emulation of the h3 kernels (bitwise equal to the global emulation),
and (GPU) N-rank loop-back partitions on one GPU through the C-ABI (bitwise equal to the
one-GPU apply)."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_03573_b200 import configs
from paper_2504_03573_b200.distributed3d import partition_ranks
from paper_2504_03573_b200.halo3d import partition_plan
from paper_2504_03573_b200.plan3d import Plan3DBuilder


def _global(nx, seed):
    case = configs.build_case("cfg4", nx, seed)
    return case, Plan3DBuilder(case.mesh, case.order_map).build()


@pytest.mark.parametrize("world", [2, 3, 5])
def test_halo_layouts_match_across_ranks(world):
    case, pb = _global(4, 2)
    ranges = partition_ranks(pb, world)
    assert ranges[0][0] == 0 and ranges[-1][1] == len(pb.shapes)
    parts = [partition_plan(pb, ranges, r) for r in range(world)]
    owner = np.concatenate([np.full(hi - lo, r) for r, (lo, hi) in enumerate(ranges)])
    for p in parts:
        assert p.n_dofs == p.dof_hi - p.dof_lo
        assert p.slots["pub_self"].min() >= 0 and p.slots["pub_self"].max() < p.n_pub
        # every interior slot reads a partner trace of its own size; boundary slots read none
        kind = p.slots["kind"]
        assert np.all((p.slots["pub_other"] >= 0) == (kind == 1))
        for i, r in enumerate(p.nbr):
            q = parts[r]
            j = int(np.flatnonzero(q.nbr == p.rank)[0])
            assert p.send_cnt[i] == q.recv_cnt[j] and p.recv_cnt[i] == q.send_cnt[j]
        # published ranges do not overlap
        spans = sorted(zip(p.slots["pub_self"], 2 * p.slots["nt"]))
        assert all(a + n <= b for (a, n), (b, _) in zip(spans, spans[1:]))
        # boundary layer = elements with a partner on another rank
        for e in range(p.hi - p.lo):
            sl = p.slots[p.slot_off[e]:p.slot_off[e + 1]]
            gl = pb.slots[pb.slot_off[p.lo + e]:pb.slot_off[p.lo + e + 1]]
            far = [owner[pb.slots["elem"][g]] != p.rank for g in gl["partner"] if g >= 0]
            assert p.roles[e] == int(any(far))
            # slot records are the global ones bit for bit (apart from the local offsets)
            for f in ("face", "kind", "nt", "mkind", "moff", "moff2", "nab", "wtoff", "tau", "sJ", "v"):
                assert np.array_equal(sl[f], gl[f])
    assert sum(p.n_dofs for p in parts) == pb.n_dofs


def _emulated_rank(pb, part, x, exchange):
    from oracle.h3_emulate import emulate
    xl = x[part.dof_lo:part.dof_hi]
    pub = np.zeros(part.n_pub)
    emulate(part, xl, pub=pub, phases=(0,))
    exchange(part, pub)
    return emulate(part, xl, pub=pub, phases=(1,))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case, pb = _global(3, 3)
        x = case.draw_x(pb.n_dofs)
        part = partition_plan(pb, partition_ranks(pb, world), rank)

        def exchange(p, pub):
            # the transport of sipg_comm_init, over gloo: one send and one receive range per neighbour
            reqs = []
            for i, r in enumerate(p.nbr):
                out = torch.from_numpy(pub[p.send_off[i]:p.send_off[i] + p.send_cnt[i]].copy())
                reqs.append(dist.isend(out, int(r)))
            bufs = []
            for i, r in enumerate(p.nbr):
                b = torch.empty(int(p.recv_cnt[i]), dtype=torch.float64)
                reqs.append(dist.irecv(b, int(r)))
                bufs.append((i, b))
            for rq in reqs:
                rq.wait()
            for i, b in bufs:
                pub[p.recv_off[i]:p.recv_off[i] + p.recv_cnt[i]] = b.numpy()

        y_own = _emulated_rank(pb, part, x, exchange)
        parts = [None] * world
        dist.all_gather_object(parts, (part.dof_lo, y_own))
        if rank == 0:
            from oracle.h3_emulate import emulate
            y = np.zeros(pb.n_dofs)
            for lo, yy in parts:
                y[lo:lo + yy.size] = yy
            yg = emulate(pb, x)
            q.put((bool(np.array_equal(y, yg)), float(np.abs(y - yg).max())))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_trace_halo_bitwise():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    assert all(p.exitcode == 0 for p in procs)
    same, err = q.get(timeout=5)
    assert same, err


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 4])
def test_gpu_loopback_partition_bitwise(world):
    """N slab partitions on one GPU, exchanged by device copies (sipg_h3_halo_copy: the same send /
    receive ranges NCCL moves): the concatenated owned y is bitwise the one-GPU apply."""
    from paper_2504_03573_b200.distributed3d import DistributedHelmholtz3D
    from paper_2504_03573_b200.sipg import HelmholtzOperator
    case, pb = _global(6, 5)
    glob = HelmholtzOperator(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline")
    x = case.draw_x(glob.n_dofs)
    y_ref = glob.lhs_eval(x)
    ranks = [DistributedHelmholtz3D(case.mesh, case.order_map, r, world, transport="none", global_plan=pb)
             for r in range(world)]
    xs = [torch.from_numpy(x[d.dof_lo:d.dof_hi]).cuda() for d in ranks]
    ys = [torch.zeros_like(xx) for xx in xs]
    s = torch.cuda.current_stream().cuda_stream
    for d, xx, yy in zip(ranks, xs, ys):
        d.native.apply_role(0, xx.data_ptr(), yy.data_ptr(), s)      # publish all, interior applies
    for d in ranks:
        for src in ranks:
            if src is not d:
                d.native.halo_copy_from(src.native, s)
    for d, xx, yy in zip(ranks, xs, ys):
        d.native.apply_role(1, xx.data_ptr(), yy.data_ptr(), s)      # boundary layer
    y = np.concatenate([yy.cpu().numpy() for yy in ys])
    assert np.array_equal(y, y_ref)
    # halo = traces only: 2 doubles per trace point of every partition-face slot
    for d in ranks:
        sl = d.part.slots
        remote = (sl["kind"] == 1) & (sl["partner"] < 0)
        assert d.halo_bytes == 16 * int(sl["nt"][remote].sum())
