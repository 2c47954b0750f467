"""GPU parity: the sm_100a apply (through the C-ABI) against golden vectors of
the real reference and against the CPU oracle.  Bar: relative max-norm error
<= 1e-12 (BASELINE.json north_star)."""
import numpy as np
import pytest

from conftest import golden_files, golden_operator_kwargs, load_golden, rel_maxnorm

pytestmark = pytest.mark.gpu
TOL = 1e-12

SMALL = golden_files(full=False)
FULL = golden_files(full=True)


def _op(case, **kw):
    from paper_2504_03573_b200.sipg import HelmholtzOperator, HelmholtzParams
    return HelmholtzOperator(case.mesh, case.order_map, **kw)


@pytest.mark.parametrize("path", SMALL, ids=[p.stem for p in SMALL])
def test_gpu_matches_reference_golden(path):
    from paper_2504_03573_b200 import configs
    g = load_golden(path)
    case = configs.build_case(str(g["config"]), int(g["nx"]), int(g["seed"]))
    op = _op(case, **golden_operator_kwargs(g))
    x = case.draw_x(op.n_dofs)
    y = op.lhs_eval(x)
    err = rel_maxnorm(y, g["y"])
    print(f"{g['name']}: rel max-norm error {err:.3e}")
    assert err <= TOL


@pytest.mark.parametrize("name,nx,seed", [("cfg0", 5, 21), ("cfg1", 7, 22), ("cfg2", 7, 23),
                                          ("cfg3a", 2, 24), ("cfg3b", 3, 25)])
def test_gpu_matches_oracle_seeded(name, nx, seed):
    from oracle import OracleOperator
    from paper_2504_03573_b200 import configs
    case = configs.build_case(name, nx, seed)
    kw = dict(basis_kind="modified_modal", tau_rule="baseline", shared_rule="patched")
    op = _op(case, **kw)
    ref = OracleOperator(case.mesh, case.order_map, **kw)
    x = case.draw_x(op.n_dofs)
    assert rel_maxnorm(op.lhs_eval(x), ref.lhs_eval(x)) <= TOL


def test_gpu_torch_tensor_zero_copy():
    import torch
    from paper_2504_03573_b200 import configs
    case = configs.build_case("cfg3b", 2, 3)
    op = _op(case, basis_kind="modified_modal", tau_rule="baseline")
    x = case.draw_x(op.n_dofs)
    y_host = op.lhs_eval(x)
    y_dev = op.lhs_eval(torch.from_numpy(x).cuda())
    assert y_dev.is_cuda
    assert np.array_equal(y_dev.cpu().numpy(), y_host)


def test_gpu_linearity_and_zero():
    from paper_2504_03573_b200 import configs
    case = configs.build_case("cfg2", 5, 4)
    op = _op(case, basis_kind="modified_modal", tau_rule="baseline")
    rng = np.random.default_rng(0)
    a, b = rng.uniform(-1, 1, op.n_dofs), rng.uniform(-1, 1, op.n_dofs)
    assert np.abs(op.lhs_eval(np.zeros(op.n_dofs))).max() == 0.0
    lhs = op.lhs_eval(2.0 * a - 3.0 * b)
    rhs = 2.0 * op.lhs_eval(a) - 3.0 * op.lhs_eval(b)
    assert rel_maxnorm(lhs, rhs) <= 1e-13


def test_gpu_deterministic():
    from paper_2504_03573_b200 import configs
    case = configs.build_case("cfg3b", 3, 9)
    op = _op(case, basis_kind="modified_modal", tau_rule="baseline")
    x = case.draw_x(op.n_dofs)
    assert np.array_equal(op.lhs_eval(x), op.lhs_eval(x))


@pytest.mark.parametrize("path", FULL, ids=[p.stem for p in FULL])
def test_gpu_full_size_golden_samples(path):
    """BASELINE sizes: sampled entries + seeded projections of the reference y."""
    from paper_2504_03573_b200 import configs
    g = load_golden(path)
    case = configs.build_case(str(g["config"]), int(g["nx"]), int(g["seed"]))
    op = _op(case, **golden_operator_kwargs(g))
    x = case.draw_x(op.n_dofs)
    y = op.lhs_eval(x)
    ymax = float(g["ymax"])
    err = float(np.abs(y[g["sample_idx"]] - g["sample_y"]).max()) / ymax
    print(f"{g['name']}: n_dofs={op.n_dofs} sampled rel error {err:.3e}")
    assert err <= TOL
    assert abs(np.abs(y).max() - ymax) <= TOL * ymax
    proj = np.random.default_rng(1234).uniform(-1.0, 1.0, (4, op.n_dofs)) @ y
    scale = np.abs(np.random.default_rng(1234).uniform(-1.0, 1.0, (4, op.n_dofs))).sum(axis=1) * ymax
    assert np.all(np.abs(proj - g["proj"]) <= TOL * scale)


@pytest.mark.parametrize("name,nx,must_stream", [("cfg3a", 4, True), ("cfg3b", 4, True), ("cfg1", 10, True),
                                                 ("cfg0", 12, True), ("cfg2", 10, False)])
def test_gpu_streamed_host_apply(monkeypatch, name, nx, must_stream):
    """sipg_apply_host pipelines H2D / publish / compute / D2H by DoF chunk; every element runs the
    same kernel code as in sipg_apply, so the result is bit-identical to the device apply."""
    import torch
    from oracle import OracleOperator
    from paper_2504_03573_b200 import configs
    case = configs.build_case(name, nx, 31)
    kw = dict(basis_kind="modified_modal", tau_rule="baseline", shared_rule="patched")
    probe = _op(case, **kw)
    monkeypatch.setenv("SIPG_STREAM_CHUNK_BYTES", str(max(4096, probe.n_dofs * 8 // 5)))
    op = _op(case, **kw)
    k = op.native.stream_chunks()
    if must_stream:
        assert k >= 4
    x = case.draw_x(op.n_dofs)
    y_host = op.lhs_eval(x)
    y_dev = op.lhs_eval(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(y_host, y_dev)
    ref = OracleOperator(case.mesh, case.order_map, **kw)
    assert rel_maxnorm(y_host, ref.lhs_eval(x)) <= TOL
