"""Per-class timing diagnostic: full apply (with / without L2 flush) vs the element-class kernels
launched back to back and one at a time; the difference is the trace-publish kernels plus fork /
join.  Usage (GPU box): python tools/diag_classes.py cfg2 256"""
import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2504_03573_b200 import configs
from paper_2504_03573_b200.sipg import HelmholtzOperator
name = sys.argv[1]; nx = int(sys.argv[2])
case = configs.build_case(name, nx, 0)
op = HelmholtzOperator(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline", shared_rule="patched")
x = torch.from_numpy(case.draw_x(op.n_dofs)).cuda(); y = torch.empty_like(x)
s = torch.cuda.current_stream(); sp = s.cuda_stream
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
def t(fn, reps=20, fl=True):
    for _ in range(3): fn()
    ts = []
    for _ in range(reps):
        if fl: flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s); fn(); b.record(s); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts))
full = t(lambda: op.native.apply_device(x.data_ptr(), y.data_ptr(), sp))
nofl = t(lambda: op.native.apply_device(x.data_ptr(), y.data_ptr(), sp), fl=False)
def classes():
    for c in range(op.native.n_classes): op.native.apply_class(c, x.data_ptr(), y.data_ptr(), sp)
cls_only = t(classes)
per = []
for c in range(op.native.n_classes):
    per.append(t(lambda: op.native.apply_class(c, x.data_ptr(), y.data_ptr(), sp), reps=5))
print(f"{name} {os.environ.get('SIPG_CONCURRENT','default')}: full {full:.4f} ms, full no-flush {nofl:.4f}, classes back-to-back {cls_only:.4f}, sum of per-class {sum(per):.4f}, n_cls {op.native.n_classes}")
print(" ".join(f"{p:.3f}" for p in per))
