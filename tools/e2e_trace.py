"""Instrumentation: timeline of one streamed sipg_apply_host (SIPG_STREAM_TRACE)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03573_b200 import configs  # noqa: E402
from paper_2504_03573_b200.plan import PlanBuilder  # noqa: E402
from paper_2504_03573_b200._native import NativePlan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3a"
case = configs.build_case(name, None, 0)
pb = PlanBuilder(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline").build()
xp = torch.from_numpy(case.draw_x(pb.n_dofs)).pin_memory()
yp = torch.empty(pb.n_dofs, dtype=torch.float64).pin_memory()
plan = NativePlan(pb)
s = torch.cuda.current_stream()
for i in range(4):
    if i == 3:
        os.environ["SIPG_STREAM_TRACE"] = "1"
    plan.apply_host_ptr(xp.data_ptr(), yp.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
