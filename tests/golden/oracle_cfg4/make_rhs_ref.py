"""Reference fixture for the RHS / error restatement: runs the REAL reference
(`dgsipg`, this container only, patch P1 as in tests/golden/make_golden.py) on an all-hex mesh —
the shape the reference and the config-4 machinery share — and stores rhs_assemble(case, bcs) and
l2_error(x, exact) for the reference's own sinusoidal manufactured case.

Usage:  python tests/golden/oracle_cfg4/make_rhs_ref.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import make_golden as mg  # noqa: E402  (reference import + P1 operator)

OUT = HERE / "ref_rhs_hex.npz"


def main():
    mesh_m, sipg_m = mg.mesh_m, mg.sipg_m
    m = mesh_m.generate_box(3, 2, mesh_m.Shape.HEX, (0.0, 1.0))
    P = np.array([2, 3, 2, 3, 3, 2, 2, 3])
    om = mesh_m.OrderMap(P + 1, P + 2)
    op = mg.make_operator(m, om, patched=True)
    case = sipg_m.sinusoidal_case(2.0, 3, lambda_=1.0)
    b = op.rhs_assemble(case, {"dirichlet": case.exact})
    x = np.random.default_rng(5).uniform(-1.0, 1.0, op.n_dofs)
    err = op.l2_error(x, case.exact)
    verts = np.asarray(m.vertices)
    ev = np.array([list(el.verts) for el in m.elements])
    np.savez_compressed(OUT, P=P, b=b, x=x, err=err, k=2.0, verts=verts, elem_verts=ev)
    print(f"{OUT.name}: n_dofs={op.n_dofs} |b|={np.abs(b).max():.6g} err={err:.6g}")


if __name__ == "__main__":
    main()
