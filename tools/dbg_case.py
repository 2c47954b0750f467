import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2504_03573_b200 import configs
from paper_2504_03573_b200.sipg import HelmholtzOperator
name, nx, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
kw = dict(basis_kind="modified_modal", tau_rule="baseline")
if len(sys.argv) > 4:
    kw["face_absorb"] = sys.argv[4]
case = configs.build_case(name, nx, seed)
op = HelmholtzOperator(case.mesh, case.order_map, **kw)
for c in range(op.native.n_classes):
    print("class", c, op.native.class_info(c), flush=True)
x = case.draw_x(op.n_dofs)
t = time.time()
y = op.lhs_eval(x)
print("done", time.time() - t, np.abs(y).max(), flush=True)
from oracle import OracleOperator
ref = OracleOperator(case.mesh, case.order_map, **kw).lhs_eval(x)
print("err", np.abs(y - ref).max() / np.abs(ref).max())
