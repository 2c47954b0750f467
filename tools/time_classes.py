"""Per-launch-unit device times (CUDA events, L2 flushed) and the whole-apply time of one config:
the quick measurement loop for kernel work.  usage: time_classes.py [cfg4] [reps]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2504_03573_b200 import configs
from paper_2504_03573_b200.sipg import HelmholtzOperator

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
case = configs.build_case(name)
kw = dict(basis_kind="modified_modal", tau_rule="baseline")
if name != "cfg4":
    kw["shared_rule"] = "patched"
op = HelmholtzOperator(case.mesh, case.order_map, **kw)
x = torch.from_numpy(case.draw_x(op.n_dofs)).cuda()
y = torch.empty_like(x)
s = torch.cuda.current_stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(3):
    op.apply_into(x.data_ptr(), y.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
for a, b in ev:
    flush.zero_()
    a.record(s)
    op.apply_into(x.data_ptr(), y.data_ptr(), s.cuda_stream)
    b.record(s)
torch.cuda.synchronize()
tot = np.array([a.elapsed_time(b) for a, b in ev])
n = op.native.n_classes
cls = np.zeros(n)
cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
for _ in range(3):
    flush.zero_()
    for c in range(n):
        cev[c][0].record(s)
        op.native.apply_class(c, x.data_ptr(), y.data_ptr(), s.cuda_stream)
        cev[c][1].record(s)
    torch.cuda.synchronize()
    cls += [a.elapsed_time(b) for a, b in cev]
cls /= 3
print(f"{name}: n_dofs={op.n_dofs} apply median {np.median(tot):.4f} ms min {tot.min():.4f} ms "
      f"({op.n_dofs / np.median(tot) / 1e6:.3f} GDoF/s); sum of units {cls.sum():.4f} ms")
for c in np.argsort(-cls):
    ci = op.native.class_info(int(c))
    print(f"  unit {c:3d} shape {ci['shape']} n {ci['n']} kind {ci['kernel']} count {ci['count']:7d}  {cls[c]:.4f} ms")
