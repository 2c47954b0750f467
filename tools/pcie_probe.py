"""Instrumentation: PCIe H2D / D2H throughput alone, concurrent, and chunked (pinned host buffers)."""
import torch

n = 11239424
xh = torch.randn(n, dtype=torch.float64).pin_memory()
yh = torch.empty(n, dtype=torch.float64).pin_memory()
xd = torch.empty(n, dtype=torch.float64, device="cuda")
yd = torch.randn(n, dtype=torch.float64, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
main = torch.cuda.current_stream()


def run(h2d, d2h, K, dep):
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        sa.wait_stream(main)
        sb.wait_stream(main)
        cuts = [n * k // K for k in range(K + 1)]
        evs = []
        if h2d:
            with torch.cuda.stream(sa):
                for k in range(K):
                    xd[cuts[k]:cuts[k + 1]].copy_(xh[cuts[k]:cuts[k + 1]], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(sa)
                    evs.append(e)
        if d2h:
            with torch.cuda.stream(sb):
                for k in range(K):
                    if dep and h2d:
                        sb.wait_event(evs[min(k + 1, K - 1)])
                    yh[cuts[k]:cuts[k + 1]].copy_(yd[cuts[k]:cuts[k + 1]], non_blocking=True)
        main.wait_stream(sa)
        main.wait_stream(sb)
        b.record(main)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


def run_hop(K, interleave):
    sc = torch.cuda.Stream()
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        sa.wait_stream(main); sb.wait_stream(main); sc.wait_stream(main)
        cuts = [n * k // K for k in range(K + 1)]
        eh = [torch.cuda.Event() for _ in range(K)]
        ec = [torch.cuda.Event() for _ in range(K)]

        def h(k):
            with torch.cuda.stream(sa):
                xd[cuts[k]:cuts[k + 1]].copy_(xh[cuts[k]:cuts[k + 1]], non_blocking=True)
                eh[k].record(sa)

        def c(k):
            sc.wait_event(eh[k]); ec[k].record(sc)

        def d(j):
            sb.wait_event(ec[min(j + 1, K - 1)])
            with torch.cuda.stream(sb):
                yh[cuts[j]:cuts[j + 1]].copy_(yd[cuts[j]:cuts[j + 1]], non_blocking=True)
        if interleave:
            for k in range(K):
                h(k)
            for k in range(K):
                c(k)
                if k >= 1:
                    d(k - 1)
            d(K - 1)
        else:
            for k in range(K):
                h(k); c(k)
                if k >= 1:
                    d(k - 1)
            d(K - 1)
        main.wait_stream(sa); main.wait_stream(sb); main.wait_stream(sc)
        b.record(main)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


print(f"hop K=14 all-H-first {run_hop(14, True):.3f} interleaved-enqueue {run_hop(14, False):.3f} ms", flush=True)

for K in (1, 4, 14, 42):
    print(f"K={K:3d} h2d={run(1,0,K,0):.3f} d2h={run(0,1,K,0):.3f} both={run(1,1,K,0):.3f} "
          f"both_pipelined={run(1,1,K,1):.3f} ms", flush=True)

import os, sys  # noqa: E401,E402
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03573_b200 import configs  # noqa: E402
from paper_2504_03573_b200.plan import PlanBuilder  # noqa: E402
from paper_2504_03573_b200._native import NativePlan  # noqa: E402

case = configs.build_case("cfg3a", None, 0)
pb = PlanBuilder(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline").build()
plan = NativePlan(pb)


def lib(skip, stream):
    if skip:
        os.environ["SIPG_STREAM_NOCOMPUTE"] = "1"
    else:
        os.environ.pop("SIPG_STREAM_NOCOMPUTE", None)
    ts = []
    for _ in range(6):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.apply_host_ptr(xh.data_ptr(), yh.data_ptr(), stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts[1:])


side = torch.cuda.Stream()
print(f"lib K={plan.stream_chunks()} copies-only: default stream {lib(1, main):.3f} side stream {lib(1, side):.3f}; "
      f"with compute: default {lib(0, main):.3f} side {lib(0, side):.3f} ms", flush=True)

# H2D of the whole vector with / without the device apply running concurrently
xd2 = torch.empty(pb.n_dofs, dtype=torch.float64, device="cuda")
yd2 = torch.empty(pb.n_dofs, dtype=torch.float64, device="cuda")
xd2.copy_(xh)


def h2d_with_apply(n_apply):
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        sa.wait_stream(main)
        sb.wait_stream(main)
        with torch.cuda.stream(sa):
            xd.copy_(xh, non_blocking=True)
        for _ in range(n_apply):
            plan.apply_device(xd2.data_ptr(), yd2.data_ptr(), sb.cuda_stream)
        main.wait_stream(sa)
        main.wait_stream(sb)
        b.record(main)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)


print("H2D 90MB with 0/1/2/3 concurrent applies:", [round(h2d_with_apply(k), 3) for k in range(4)], flush=True)
