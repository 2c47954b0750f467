"""Instrumentation: median device-apply time of a config (CUDA events, L2 flushed between applies).
Usage: python tools/time_apply.py cfg3a [reps]; env knobs (SIPG_DEBUG, SIPG_HEX_FAST_KERNEL, ...) pass through."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03573_b200 import configs  # noqa: E402
from paper_2504_03573_b200.plan import PlanBuilder  # noqa: E402
from paper_2504_03573_b200._native import NativePlan  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["cfg3a"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for name in names:
    case = configs.build_case(name, None, 0)
    pb = PlanBuilder(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline").build()
    plan = NativePlan(pb)
    x = torch.from_numpy(case.draw_x(pb.n_dofs)).cuda()
    y = torch.empty_like(x)
    s = torch.cuda.current_stream()
    ts = []
    for i in range(reps + 3):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        plan.apply_device(x.data_ptr(), y.data_ptr(), s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SIPG_"))
    print(f"{name} {tag} median {np.median(ts):.4f} ms min {np.min(ts):.4f} GDoF/s {pb.n_dofs / np.median(ts) / 1e6:.2f}",
          flush=True)
