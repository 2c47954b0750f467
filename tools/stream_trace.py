"""Timeline of the streamed host apply (SIPG_STREAM_TRACE=1: device timestamps after every chunk
copy (H), stage (C) and y copy (D), ms from the start), plus the plain e2e time.  usage:
SIPG_STREAM_TRACE=1 python tools/stream_trace.py [cfg4]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2504_03573_b200 import configs
from paper_2504_03573_b200.sipg import HelmholtzOperator

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
case = configs.build_case(name)
kw = dict(basis_kind="modified_modal", tau_rule="baseline")
op = HelmholtzOperator(case.mesh, case.order_map, **kw)
xp = torch.from_numpy(case.draw_x(op.n_dofs)).pin_memory()
yp = torch.empty(op.n_dofs, dtype=torch.float64).pin_memory()
print("chunks", op.native.stream_chunks(), "launches/host apply", op.native.host_launches_per_apply(), flush=True)
for i in range(4):
    t0 = time.perf_counter()
    op.native.apply_host_ptr(xp.data_ptr(), yp.data_ptr())
    print(f"host apply {1e3 * (time.perf_counter() - t0):.3f} ms", flush=True)
