"""Reference fixtures for rhs_assemble / l2_error on the standard plans: runs
the REAL reference (`dgsipg`, this container only; patches P1/P2 as in make_golden.py unless the
case is "unpatched") on small meshes of configs 0-3 and stores b for the reference's sinusoidal and
Gaussian-pulse manufactured cases (reference sipg.py:88-121) plus l2_error of a random vector.
The GPU box only reads the committed npz files.

Usage:  python tests/golden/make_rhs_golden.py
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
import make_golden as mg  # noqa: E402

CASES = [
    # tag, config, nx, seed, patched
    ("rhs_cfg0_n3", "cfg0", 3, 31, True),
    ("rhs_cfg1_n4", "cfg1", 4, 32, True),
    ("rhs_cfg1_n4_unpatched", "cfg1", 4, 32, False),
    ("rhs_cfg2_n5", "cfg2", 5, 33, True),
    ("rhs_cfg3a_n2", "cfg3a", 2, 34, True),
    ("rhs_cfg3b_n2", "cfg3b", 2, 35, True),
]
K, A = 2.0, 0.35


def main():
    sipg_m = mg.sipg_m
    for tag, name, nx, seed, patched in CASES:
        m, om, rng = mg.build_case(name, nx, seed)
        op = mg.make_operator(m, om, patched=patched)
        sin = sipg_m.sinusoidal_case(K, m.dim, lambda_=1.0)
        pulse = sipg_m.gaussian_pulse_case(A, m.dim, lambda_=1.0)
        b_sin = op.rhs_assemble(sin, {"dirichlet": sin.exact})
        b_pulse = op.rhs_assemble(pulse, {"dirichlet": pulse.exact})
        x = rng.uniform(-1.0, 1.0, op.n_dofs)
        err = op.l2_error(x, sin.exact)
        np.savez_compressed(HERE / f"{tag}.npz", config=name, nx=nx, seed=seed, patched=int(patched),
                            k=K, a=A, b_sin=b_sin, b_pulse=b_pulse, x=x, err=err)
        print(f"{tag}: n_dofs={op.n_dofs} |b|={np.abs(b_sin).max():.6g} err={err:.6g}", flush=True)


if __name__ == "__main__":
    main()
