"""Measurement of the §8f rows built around the apply (f1 CG, f2 rhs / l2, f4 probe) on one B200.
Device times by CUDA events (CG, probe); rhs / l2 wall times include their host-side setup
(geometry, basis tables, user callbacks), like the reference's.  The oracle / reference CPU times
on a small case are printed beside them for scale (oracle = numpy restatement, 1 process).
Usage: python tools/time_next_rows.py > profiles/r01/next_rows.txt"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_03573_b200 import configs, krylov  # noqa: E402
from paper_2504_03573_b200.sipg import HelmholtzOperator  # noqa: E402

KW = dict(basis_kind="modified_modal", tau_rule="baseline")


def sin_case(d, k=2.0, lam=1.0):
    def ex(x):
        return np.prod([np.sin(k * x[i]) for i in range(d)], axis=0)
    return type("C", (), {"exact": staticmethod(ex), "forcing": staticmethod(lambda x: -(lam + d * k * k) * ex(x))})


def wall(f, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return float(np.median(ts)), r


def main():
    print("# f2 rhs_assemble / l2_error (GPU; wall time incl. host setup), f1 CG, f4 probe")
    for name, nx in (("cfg3a", None), ("cfg2", None), ("cfg4", None)):
        case = configs.build_case(name, nx)
        op = HelmholtzOperator(case.mesh, case.order_map, **KW)
        mc = sin_case(case.mesh.dim)
        t_rhs, b = wall(lambda: op.rhs_assemble(mc, {"dirichlet": mc.exact}))
        x = case.draw_x(op.n_dofs)
        t_l2, _ = wall(lambda: op.l2_error(x, mc.exact))
        print(f"{name}: n_dofs={op.n_dofs} rhs_assemble {t_rhs * 1e3:.1f} ms, l2_error {t_l2 * 1e3:.1f} ms", flush=True)
        # f1: CG iterations on the device (fixed count: maxiter, tol 0)
        bd = torch.from_numpy(b).cuda()
        it = 50
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        krylov.cg(op, bd, tol=0.0, maxiter=5)
        torch.cuda.synchronize()
        ev[0].record()
        _, rep = krylov.cg(op, bd, tol=0.0, maxiter=it)
        ev[1].record()
        torch.cuda.synchronize()
        ms_it = ev[0].elapsed_time(ev[1]) / max(rep.iterations, 1)
        xa, ya = torch.from_numpy(x).cuda(), torch.empty(op.n_dofs, dtype=torch.float64, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        for _ in range(3):
            op.apply_into(xa.data_ptr(), ya.data_ptr(), s)
        ev[0].record()
        for _ in range(20):
            op.apply_into(xa.data_ptr(), ya.data_ptr(), s)
        ev[1].record()
        torch.cuda.synchronize()
        ms_ap = ev[0].elapsed_time(ev[1]) / 20
        print(f"{name}: CG {rep.iterations} its ({rep.reason}) {ms_it:.3f} ms/iteration, apply {ms_ap:.3f} ms "
              f"(Krylov overhead {100 * (ms_it - ms_ap) / ms_it:.1f} %)", flush=True)
    # f4: probe of a small operator, device time per column
    case = configs.build_case("cfg1", 6, 3)
    op = HelmholtzOperator(case.mesh, case.order_map, **KW)
    t, m = wall(lambda: krylov.probe_dense(op, op.n_dofs), reps=2)
    print(f"cfg1 nx=6: probe_dense n={op.n_dofs}: {t * 1e3:.1f} ms ({t * 1e6 / op.n_dofs:.1f} us/column), "
          f"asymmetry {krylov.asymmetry_norm(m):.2e}", flush=True)
    # CPU scale: the oracle's restatement on a small case
    from oracle import OracleOperator
    case = configs.build_case("cfg3a", 4, 0)
    ref = OracleOperator(case.mesh, case.order_map, shared_rule="patched", **KW)
    op = HelmholtzOperator(case.mesh, case.order_map, **KW)
    mc = sin_case(3)
    t_o, b_o = wall(lambda: ref.rhs_assemble(mc, {"dirichlet": mc.exact}), reps=1)
    t_g, b_g = wall(lambda: op.rhs_assemble(mc, {"dirichlet": mc.exact}))
    print(f"cfg3a nx=4 (n_dofs={op.n_dofs}): rhs oracle CPU {t_o * 1e3:.1f} ms, GPU {t_g * 1e3:.1f} ms, "
          f"max rel diff {np.abs(b_o - b_g).max() / np.abs(b_o).max():.1e}", flush=True)


if __name__ == "__main__":
    main()
