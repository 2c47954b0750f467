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


def test_rhs_fixtures_present_and_consistent():
    """The reference rhs / l2 fixtures (tests/golden/make_rhs_golden.py) carry what test_gpu_rhs.py
    needs, and their DoF counts match the plans this package builds for the same cases."""
    from conftest import GOLDEN
    from paper_2504_03573_b200 import configs
    from paper_2504_03573_b200.plan import PlanBuilder
    files = sorted(GOLDEN.glob("rhs_cfg*.npz"))
    assert len(files) >= 5
    for p in files:
        g = np.load(p)
        case = configs.build_case(str(g["config"]), int(g["nx"]), int(g["seed"]))
        pb = PlanBuilder(case.mesh, case.order_map, basis_kind="modified_modal").build()
        assert g["b_sin"].shape == g["b_pulse"].shape == g["x"].shape == (pb.n_dofs,)
        assert np.isfinite(g["b_sin"]).all() and float(g["err"]) > 0


def test_rhs_volume_basis_matches_oracle_expansion():
    """rhs.volume_basis (the dense class table of the GPU rhs / l2) equals the oracle's BwdTrans of
    unit coefficient vectors."""
    from oracle.elements import expansion
    from paper_2504_03573_b200.rhs import volume_basis
    from paper_2504_03573_b200.stdregions import DEFAULT_RULES, class_tables
    for shape, n, q in (("quad", 5, 6), ("tri", 4, 6), ("hex", 4, 5), ("tri", 7, 9)):
        kinds = tuple(k.value for k in DEFAULT_RULES[shape])
        ct = class_tables(shape, "modified_modal", n, (q,) * ct_dim(shape), kinds)
        ex = expansion(shape, "modified_modal", n, (q,) * ct_dim(shape), kinds)
        ref = ex.bwd(np.eye(ct.n_coeffs))
        assert np.abs(volume_basis(ct) - ref).max() <= 1e-13


def ct_dim(shape):
    return 3 if shape == "hex" else 2


@pytest.mark.parametrize("tag", ["rhs_cfg0_n3", "rhs_cfg1_n4", "rhs_cfg1_n4_unpatched", "rhs_cfg2_n5",
                                 "rhs_cfg3b_n2"])
def test_oracle_rhs_and_l2_match_reference(tag):
    """The oracle's restatement of rhs_assemble / l2_error (sipg.py:697-741) against the real
    reference's outputs (tests/golden/make_rhs_golden.py)."""
    from conftest import GOLDEN
    from oracle import OracleOperator
    from paper_2504_03573_b200 import configs
    g = np.load(GOLDEN / f"{tag}.npz")
    case = configs.build_case(str(g["config"]), int(g["nx"]), int(g["seed"]))
    patched = bool(g["patched"])
    ref = OracleOperator(case.mesh, case.order_map, basis_kind="modified_modal",
                         tau_rule="baseline" if patched else "reference",
                         shared_rule="patched" if patched else "reference")
    d, k, a = case.mesh.dim, float(g["k"]), float(g["a"])

    def s_ex(x):
        return np.prod([np.sin(k * x[i]) for i in range(d)], axis=0)

    def g_ex(x):
        return np.exp(-sum(x[i] ** 2 for i in range(d)) / (a * a))
    sin = type("C", (), {"exact": staticmethod(s_ex), "forcing": staticmethod(lambda x: -(1 + d * k * k) * s_ex(x))})
    pulse = type("C", (), {"exact": staticmethod(g_ex), "forcing": staticmethod(
        lambda x: (4.0 * sum(x[i] ** 2 for i in range(d)) / a ** 4 - 2.0 * d / (a * a) - 1.0) * g_ex(x))})
    assert rel_maxnorm(ref.rhs_assemble(sin, {"dirichlet": s_ex}), g["b_sin"]) <= 1e-13
    assert rel_maxnorm(ref.rhs_assemble(pulse, {"dirichlet": g_ex}), g["b_pulse"]) <= 1e-13
    assert abs(ref.l2_error(g["x"], s_ex) - float(g["err"])) <= 1e-13 * float(g["err"])
