"""Instrumentation: CG time per iteration vs apply time (cfg3a)."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_03573_b200 import configs, krylov
from paper_2504_03573_b200.sipg import HelmholtzOperator

for name, nx in (("cfg3a", 16), ("cfg3a", None), ("cfg3b", None)):
    case = configs.build_case(name, nx)
    op = HelmholtzOperator(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline")
    b = torch.from_numpy(case.draw_x(op.n_dofs)).cuda()
    for it in (5, 20, 50):
        torch.cuda.synchronize(); t = time.perf_counter()
        x, rep = krylov.cg(op, b, tol=0.0, maxiter=it)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(name, nx, op.n_dofs, "maxiter", it, rep, f"{dt*1e3:.1f} ms wall, {dt*1e3/max(rep.iterations,1):.3f} ms/it", flush=True)
    y = torch.empty_like(b)
    s = torch.cuda.current_stream().cuda_stream
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(20):
        op.apply_into(b.data_ptr(), y.data_ptr(), s)
    torch.cuda.synchronize(); print("apply", (time.perf_counter() - t) / 20 * 1e3, "ms", flush=True)
    p = torch.empty_like(b); p.copy_(b)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(20):
        op.apply_into(p.data_ptr(), y.data_ptr(), s)
    torch.cuda.synchronize(); print("apply copy", (time.perf_counter() - t) / 20 * 1e3, "ms", flush=True)
