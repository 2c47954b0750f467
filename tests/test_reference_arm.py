"""bench.py's reference arm (oracle/reference_arm.py): the unmodified reference package from
baseline/_ref (or /root/reference here), patched from outside like tests/golden/make_golden.py,
reproduces the committed golden y of cfg0 and times its own lhs_eval."""
import numpy as np
import pytest

from conftest import GOLDEN, load_golden


def _ref():
    from oracle import reference_arm
    pkg, path = reference_arm.load()
    if pkg is None:
        pytest.skip("reference package not installed (baseline/_ref)")
    return reference_arm, pkg


def test_reference_arm_reproduces_golden():
    ra, pkg = _ref()
    m, om, desc = ra.sample_case(pkg, "cfg0")
    g = load_golden(GOLDEN / "cfg0_full.npz")
    for w in (4, 64):
        op = ra._patched_operator(pkg)(m, om, w)
        assert op.n_dofs == g["x"].size
        assert np.array_equal(op.lhs_eval(g["x"]), g["y"])


def test_reference_arm_times_both_batch_widths():
    ra, pkg = _ref()
    r = ra.time_reference("cfg0", 2, 1)
    assert set(r["by_width"]) == {64, 4}
    for v in r["by_width"].values():
        assert v["n_dofs"] == 6400 and v["mean_s"] > 0.0
