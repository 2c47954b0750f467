"""SURVEY §8f row f2 on the standard plans: rhs_assemble / l2_error on the GPU against the REAL
reference's outputs (tests/golden/rhs_*.npz, made by tests/golden/make_rhs_golden.py) for the
reference's sinusoidal and Gaussian-pulse manufactured cases (sipg.py:88-121, restated here), on
configs 0-3 (conforming / perturbed p-nonconforming quads, hybrid quad / tri, hex), patched and
unpatched penalties. Bar: 1e-12 relative max-norm."""
import numpy as np
import pytest

from conftest import GOLDEN, rel_maxnorm

pytestmark = pytest.mark.gpu
FILES = sorted(GOLDEN.glob("rhs_cfg*.npz"))


def manufactured(d, k, a, lam=1.0):
    """(sinusoidal, pulse) cases as (exact, forcing) pairs."""
    def s_ex(x):
        return np.prod([np.sin(k * x[i]) for i in range(d)], axis=0)

    def g_ex(x):
        return np.exp(-sum(x[i] ** 2 for i in range(d)) / (a * a))
    sin = (s_ex, lambda x: -(lam + d * k * k) * s_ex(x))
    pulse = (g_ex, lambda x: (4.0 * sum(x[i] ** 2 for i in range(d)) / a ** 4 - 2.0 * d / (a * a) - lam) * g_ex(x))
    return [type("Case", (), {"exact": staticmethod(e), "forcing": staticmethod(f)}) for e, f in (sin, pulse)]


def _op(g):
    from paper_2504_03573_b200 import configs
    from paper_2504_03573_b200.sipg import HelmholtzOperator
    case = configs.build_case(str(g["config"]), int(g["nx"]), int(g["seed"]))
    patched = bool(g["patched"])
    return HelmholtzOperator(case.mesh, case.order_map, basis_kind="modified_modal",
                             tau_rule="baseline" if patched else "reference",
                             shared_rule="patched" if patched else "reference")


@pytest.mark.parametrize("path", FILES, ids=[p.stem for p in FILES])
def test_rhs_and_l2_match_reference(path):
    g = np.load(path)
    op = _op(g)
    sin, pulse = manufactured(op.mesh.dim, float(g["k"]), float(g["a"]))
    assert rel_maxnorm(op.rhs_assemble(sin, {"dirichlet": sin.exact}), g["b_sin"]) <= 1e-12
    assert rel_maxnorm(op.rhs_assemble(pulse, {"dirichlet": pulse.exact}), g["b_pulse"]) <= 1e-12
    err = float(g["err"])
    assert abs(op.l2_error(g["x"], sin.exact) - err) <= 1e-12 * err


def test_missing_boundary_tag_raises():
    g = np.load(FILES[0])
    op = _op(g)
    sin, _ = manufactured(op.mesh.dim, 2.0, 0.3)
    with pytest.raises(KeyError):
        op.rhs_assemble(sin, {"neumann": sin.exact})


def test_manufactured_solve_converges_2d():
    """rhs -> CG over the GPU apply -> l2_error, conforming quads: spectral in P."""
    from scipy.sparse.linalg import LinearOperator, cg
    from paper_2504_03573_b200.mesh import OrderMap, Shape, generate_box
    from paper_2504_03573_b200.sipg import HelmholtzOperator
    m = generate_box(2, 4, Shape.QUAD, (0.0, 1.0))
    sin, _ = manufactured(2, 2.0, 0.3)
    errs = []
    for P in (2, 4, 6):
        op = HelmholtzOperator(m, OrderMap(np.full(m.n_elements, P + 1), np.full(m.n_elements, P + 2)),
                               basis_kind="modified_modal", tau_rule="baseline")
        b = op.rhs_assemble(sin, {"dirichlet": sin.exact})
        x, info = cg(LinearOperator((op.n_dofs,) * 2, matvec=op.lhs_eval), b, rtol=1e-12, maxiter=20000)
        assert info == 0
        errs.append(op.l2_error(x, sin.exact))
    assert errs[1] < 0.05 * errs[0] and errs[2] < 0.05 * errs[1], errs


@pytest.mark.parametrize("name,nx,seed", [("cfg1", 6, 41), ("cfg2", 7, 42), ("cfg3b", 3, 43)])
def test_rhs_and_l2_match_oracle_seeded(name, nx, seed):
    """Seeded cases beyond the fixtures: GPU rhs / l2 against the oracle's restatement."""
    from oracle import OracleOperator
    from paper_2504_03573_b200 import configs
    from paper_2504_03573_b200.sipg import HelmholtzOperator
    case = configs.build_case(name, nx, seed)
    kw = dict(basis_kind="modified_modal", tau_rule="baseline", shared_rule="patched")
    op = HelmholtzOperator(case.mesh, case.order_map, **kw)
    ref = OracleOperator(case.mesh, case.order_map, **kw)
    sin, pulse = manufactured(case.mesh.dim, 2.5, 0.4)
    for mc in (sin, pulse):
        assert rel_maxnorm(op.rhs_assemble(mc, {"dirichlet": mc.exact}),
                           ref.rhs_assemble(mc, {"dirichlet": mc.exact})) <= 1e-12
    x = case.draw_x(op.n_dofs)
    e = ref.l2_error(x, pulse.exact)
    assert abs(op.l2_error(x, pulse.exact) - e) <= 1e-12 * e


@pytest.mark.parametrize("path", FILES[:4], ids=[p.stem for p in FILES[:4]])
def test_device_cases_match_reference(path):
    """The device-capable manufactured cases (cases.py) keep rhs / l2 on the GPU (points, callables,
    products); same reference fixtures, same bar."""
    from paper_2504_03573_b200.cases import gaussian_pulse_case, sinusoidal_case
    g = np.load(path)
    op = _op(g)
    d = op.mesh.dim
    sin, pulse = sinusoidal_case(float(g["k"]), d), gaussian_pulse_case(float(g["a"]), d)
    assert rel_maxnorm(op.rhs_assemble(sin, {"dirichlet": sin.exact}), g["b_sin"]) <= 1e-12
    assert rel_maxnorm(op.rhs_assemble(pulse, {"dirichlet": pulse.exact}), g["b_pulse"]) <= 1e-12
    err = float(g["err"])
    assert abs(op.l2_error(g["x"], sin.exact) - err) <= 1e-12 * err


def test_device_cases_hybrid3d_match_host_path():
    """Config 4: device callables and the reference-style host callables give the same rhs / l2."""
    from paper_2504_03573_b200 import configs
    from paper_2504_03573_b200.cases import sinusoidal_case
    from paper_2504_03573_b200.sipg import HelmholtzOperator
    case = configs.build_case("cfg4", 3, 2)
    op = HelmholtzOperator(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline")
    dev = sinusoidal_case(3.0, 3)
    host = manufactured(3, 3.0, 0.3)[0]
    b_dev = op.rhs_assemble(dev, {"dirichlet": dev.exact})
    b_host = op.rhs_assemble(host, {"dirichlet": host.exact})
    assert rel_maxnorm(b_dev, b_host) <= 1e-13
    x = case.draw_x(op.n_dofs)
    e_dev, e_host = op.l2_error(x, dev.exact), op.l2_error(x, host.exact)
    assert abs(e_dev - e_host) <= 1e-12 * e_host
