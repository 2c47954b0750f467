import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: large CPU case")


def golden_files(full=False):
    out = []
    for p in sorted(GOLDEN.glob("*.npz")):
        if p.name.startswith("rhs_"):          # rhs_assemble / l2_error fixtures (test_gpu_rhs.py)
            continue
        with np.load(p) as g:
            has_y = "y" in g.files
        if has_y != full:
            out.append(p)
    return out


def load_golden(path):
    g = np.load(path)
    rec = {k: g[k] for k in g.files}
    rec["opts"] = {k[4:]: g[k].item() for k in g.files if k.startswith("opt_")}
    rec["name"] = Path(path).stem
    return rec


def golden_operator_kwargs(rec):
    patched = bool(rec["patched"])
    kw = dict(rec["opts"])
    kw["basis_kind"] = str(rec["basis"])
    kw["tau_rule"] = "baseline" if patched else "reference"
    kw["shared_rule"] = "patched" if patched else "reference"
    return kw


def rel_maxnorm(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max())
