"""Instrumentation: sipg_apply_host time vs stream chunk size (env SIPG_STREAM_CHUNK_BYTES) on a config."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03573_b200 import configs  # noqa: E402
from paper_2504_03573_b200.plan import PlanBuilder  # noqa: E402
from paper_2504_03573_b200._native import NativePlan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3a"
case = configs.build_case(name, None, 0)
pb = PlanBuilder(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline").build()
n = pb.n_dofs
xp = torch.from_numpy(case.draw_x(n)).pin_memory()
yp = torch.empty(n, dtype=torch.float64).pin_memory()
s = torch.cuda.current_stream()
CHUNKS = os.environ.get("SWEEP_CHUNKS", "none,2,4,8,12").split(",")
for cb in [c if c == "none" else str(int(float(c) * (1 << 20))) for c in CHUNKS]:
    if cb == "none":
        os.environ["SIPG_NO_STREAM"] = "1"
    else:
        os.environ.pop("SIPG_NO_STREAM", None)
        os.environ["SIPG_STREAM_CHUNK_BYTES"] = cb
    plan = NativePlan(pb)
    ts = []
    for i in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        t0 = time.perf_counter()
        plan.apply_host_ptr(xp.data_ptr(), yp.data_ptr(), s.cuda_stream)
        t1 = time.perf_counter()
        b.record(s)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append((a.elapsed_time(b), (t1 - t0) * 1e3))
    ts = np.array(ts)
    print(f"{name} chunk={cb:>9} K={plan.stream_chunks():3d} launches={plan.host_launches_per_apply():4d} "
          f"event_ms={ts[:,0].mean():.3f} min={ts[:,0].min():.3f} wall_ms={ts[:,1].mean():.3f}", flush=True)
    del plan
