"""Small driver for ncu: build one config's operator and run a few applies."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2504_03573_b200 import configs
from paper_2504_03573_b200.sipg import HelmholtzOperator

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3a"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
case = configs.build_case(name)
op = HelmholtzOperator(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline")
x = torch.from_numpy(case.draw_x(op.n_dofs)).cuda()
y = torch.empty_like(x)
for _ in range(reps):
    op.apply_into(x.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", name, op.n_dofs)
