"""Instrumentation: per-class kernel time (apply_class, CUDA events, after one full apply so
published planes/traces are in place)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03573_b200 import configs  # noqa: E402
from paper_2504_03573_b200.plan import PlanBuilder  # noqa: E402
from paper_2504_03573_b200._native import NativePlan  # noqa: E402

KN = {0: "k_apply", 1: "k_hexw", 2: "k_hex_mma", 3: "k_hex_mma", 4: "k_hex", 5: "k_apply_w", 6: "k_hexp", 7: "k_hexp"}
for name in (sys.argv[1] if len(sys.argv) > 1 else "cfg3b").split(","):
    case = configs.build_case(name, None, 0)
    pb = PlanBuilder(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline").build()
    plan = NativePlan(pb)
    x = torch.from_numpy(case.draw_x(pb.n_dofs)).cuda()
    y = torch.empty_like(x)
    s = torch.cuda.current_stream()
    plan.apply_device(x.data_ptr(), y.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    tot = 0.0
    for c in range(pb.n_classes if hasattr(pb, "n_classes") else len(pb.class_desc)):
        info = plan.class_info(c)
        if info["count"] == 0:
            continue
        ts = []
        for i in range(8):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            plan.apply_class(c, x.data_ptr(), y.data_ptr(), s.cuda_stream)
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        t = float(np.median(ts[2:]))
        tot += t
        print(f"{name} class {c:3d} {KN.get(info['kernel'], info['kernel']):10s} shape={info['shape']} n={info['n']} "
              f"q={info['q']} geom={info['geom']} count={info['count']:6d} {t:.4f} ms "
              f"({t * 1e3 / info['count'] * 148:.2f} us/elem/SM)", flush=True)
    print(f"{name} sum of compute classes {tot:.4f} ms", flush=True)
