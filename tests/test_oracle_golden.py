"""The CPU oracle is pinned to golden vectors produced by the real reference
(tests/golden/make_golden.py)."""
import numpy as np
import pytest

from conftest import golden_files, golden_operator_kwargs, load_golden, rel_maxnorm
from oracle import OracleOperator
from paper_2504_03573_b200 import configs

SMALL = golden_files(full=False)


@pytest.mark.parametrize("path", SMALL, ids=[p.stem for p in SMALL])
def test_oracle_matches_reference_golden(path):
    g = load_golden(path)
    case = configs.build_case(str(g["config"]), int(g["nx"]), int(g["seed"]))
    op = OracleOperator(case.mesh, case.order_map, **golden_operator_kwargs(g))
    assert np.array_equal(op.dof_off, g["dof_off"])
    x = case.draw_x(op.n_dofs)
    assert np.array_equal(x, g["x"]), "seeded input recipe drifted"
    y = op.lhs_eval(x)
    assert rel_maxnorm(y, g["y"]) <= 1e-14


def test_oracle_rejects_wrong_length():
    case = configs.build_case("cfg0", 2, 0)
    op = OracleOperator(case.mesh, case.order_map)
    with pytest.raises(ValueError):
        op.lhs_eval(np.zeros(op.n_dofs + 1))
