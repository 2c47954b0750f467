"""Config-4 fixtures from the CPU oracle (oracle/hybrid3d.py).

The reference has no prism / tet, so these are NOT reference
goldens: they freeze the property-tested oracle (tests/test_hybrid3d_oracle.py)
so that (a) the oracle cannot drift silently and (b) the GPU is checked at the
full BASELINE size (48^3 cubes, 25.2 M DoFs) through size-independent digests
(sampled entries, seeded projections, norms) without running the oracle there.

Usage:  python tests/golden/oracle_cfg4/make_cfg4.py [small|full|all]
"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[3]
sys.path.insert(0, str(ROOT))

from oracle.hybrid3d import HybridOracle3D  # noqa: E402
from paper_2504_03573_b200 import configs  # noqa: E402

OUT = Path(__file__).resolve().parent
SAMPLES = 4096


def checks_of(y, seed=1234):
    n = y.size
    idx = np.unique(np.linspace(0, n - 1, min(SAMPLES, n)).astype(np.int64))
    proj = np.random.default_rng(seed).uniform(-1.0, 1.0, (4, n)) @ y
    return {"sample_idx": idx, "sample_y": y[idx], "proj": proj, "ymax": np.abs(y).max(),
            "ynorm": np.linalg.norm(y)}


def run(tag, nx, seed, store_full):
    t0 = time.perf_counter()
    case = configs.build_case("cfg4", nx, seed)
    m = case.mesh
    op = HybridOracle3D(m.shapes, [el.verts for el in m.elements], m.vertices,
                        case.order_map.n_modes, case.order_map.n_quad)
    t1 = time.perf_counter()
    x = case.draw_x(op.n_dofs)
    y = op(x)
    t2 = time.perf_counter()
    rec = {"config": "cfg4", "nx": nx, "seed": seed, "n_dofs": op.n_dofs, "n_elements": m.n_elements,
           "setup_s": t1 - t0, "apply_s": t2 - t1, "dof_off": op.dof_off}
    rec.update(checks_of(y))
    if store_full:
        rec["x"], rec["y"] = x, y
    np.savez_compressed(OUT / f"{tag}.npz", **rec)
    print(f"{tag}: n_dofs={op.n_dofs} setup {t1 - t0:.1f}s apply {t2 - t1:.1f}s", flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "small"
    if which in ("small", "all"):
        run("cfg4_n3_s0", 3, 0, True)
        run("cfg4_n4_s7", 4, 7, True)
    if which in ("full", "all"):
        run("cfg4_full", 48, 0, False)
