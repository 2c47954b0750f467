import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2504_03573_b200 import configs
from paper_2504_03573_b200.sipg import HelmholtzOperator
from oracle import OracleOperator
case = configs.build_case("cfg1", 10, 31)
kw = dict(basis_kind="modified_modal", tau_rule="baseline", shared_rule="patched")
ref = OracleOperator(case.mesh, case.order_map, **kw)
x = None
for env in ["none", "stream"]:
    if env == "stream":
        os.environ["SIPG_STREAM_CHUNK_BYTES"] = "4096"
    op = HelmholtzOperator(case.mesh, case.order_map, **kw)
    if x is None:
        x = case.draw_x(op.n_dofs); yr = ref.lhs_eval(x)
    yh = op.lhs_eval(x)
    yd = op.lhs_eval(torch.from_numpy(x).cuda()).cpu().numpy()
    def err(y):
        d = np.abs(y - yr) / np.abs(yr).max()
        bad = [e for e in range(len(op._dof_off) - 1) if d[op._dof_off[e]:op._dof_off[e+1]].max() > 1e-12]
        return f"{d.max():.2e} bad_elems={bad[:20]} n_bad={len(bad)}"
    print(env, "K", op.native.stream_chunks(), "host", err(yh), "dev", err(yd), flush=True)
