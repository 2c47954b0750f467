"""GPU-resident Krylov solvers against the CPU restatement of the
reference's CG (oracle/krylov.py, reference krylov.py:39-81) over the oracle apply."""
import numpy as np
import pytest

from conftest import rel_maxnorm


def _case(name, nx, seed, basis="modified_modal", **kw):
    from paper_2504_03573_b200 import configs
    from paper_2504_03573_b200.sipg import HelmholtzOperator
    case = configs.build_case(name, nx, seed)
    # reference penalty (C = 10).  The 3-D modified-modal operators are SPD but so badly
    # conditioned (cond ~ 1e8 at P = 6) that the reference's CG stagnates on them; the 3-D
    # convergence cases use the reference's default LAGRANGE basis (generic kernels).
    args = dict(basis_kind=basis, tau_rule="reference", shared_rule="patched", **kw)
    return case, args, HelmholtzOperator(case.mesh, case.order_map, **args)


def test_oracle_cg_solves_dense_system():
    """The CPU restatement itself: CG on the probed oracle matrix matches a dense solve."""
    from oracle import OracleOperator
    from oracle.krylov import cg
    from paper_2504_03573_b200 import configs
    case = configs.build_case("cfg0", 3, 5)
    op = OracleOperator(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline")
    n = op.n_dofs
    a = np.stack([op.lhs_eval(np.eye(n)[j]) for j in range(n)], axis=1)
    b = np.random.default_rng(1).uniform(-1, 1, n)
    x, conv, it, res, why = cg(op.lhs_eval, b, tol=1e-12)
    assert conv and why == ""
    assert np.allclose(x, np.linalg.solve(a, b), rtol=1e-8, atol=1e-10)


@pytest.mark.gpu
@pytest.mark.parametrize("name,nx,seed,basis", [("cfg0", 6, 11, "modified_modal"), ("cfg1", 6, 12, "modified_modal"),
                                                ("cfg3a", 2, 13, "lagrange"), ("cfg3b", 2, 14, "lagrange")])
def test_gpu_cg_matches_oracle_cg(name, nx, seed, basis):
    from oracle import OracleOperator
    from oracle.krylov import cg as ocg
    from paper_2504_03573_b200.krylov import cg
    case, args, op = _case(name, nx, seed, basis)
    ref = OracleOperator(case.mesh, case.order_map, **args)
    b = case.draw_x(op.n_dofs)
    x, rep = cg(op, b, tol=1e-10)
    xo, conv, it, res, why = ocg(ref.lhs_eval, b, tol=1e-10)
    assert rep.converged and conv
    assert abs(rep.iterations - it) <= max(2, it // 50)
    assert rel_maxnorm(x, xo) <= 1e-7
    # the returned residual is the verified true residual
    assert np.linalg.norm(b - ref.lhs_eval(x)) / np.linalg.norm(b) <= 1e-9


@pytest.mark.gpu
def test_gpu_cg_reports_like_the_reference():
    """Zero right-hand side, maxiter, indefinite operator (lambda << 0): same reasons."""
    from oracle import OracleOperator
    from oracle.krylov import cg as ocg
    from paper_2504_03573_b200.krylov import cg
    from paper_2504_03573_b200.sipg import HelmholtzParams
    case, args, op = _case("cfg0", 4, 3)
    x, rep = cg(op, np.zeros(op.n_dofs))
    assert rep.converged and rep.iterations == 0 and not np.any(x)
    b = case.draw_x(op.n_dofs)
    x, rep = cg(op, b, tol=1e-14, maxiter=3)
    assert not rep.converged and rep.reason == "maxiter" and rep.iterations == 3
    assert str(rep).startswith("FAILED (maxiter) in 3 iterations")
    case, args, op = _case("cfg0", 4, 3, params=HelmholtzParams(lambda_=-2000.0))
    args.pop("params")
    ref = OracleOperator(case.mesh, case.order_map, lambda_=-2000.0, **args)
    x, rep = cg(op, b)
    xo, conv, it, res, why = ocg(ref.lhs_eval, b)
    assert not rep.converged and rep.reason == why == "indefinite direction"
    assert rep.iterations == it


@pytest.mark.gpu
def test_gpu_cg_stagnation_like_the_reference():
    """3-D modified-modal P = 6: the reference's CG stagnates (residual grows); so does ours."""
    from oracle import OracleOperator
    from oracle.krylov import cg as ocg
    from paper_2504_03573_b200.krylov import cg
    case, args, op = _case("cfg3a", 2, 13)
    ref = OracleOperator(case.mesh, case.order_map, **args)
    b = case.draw_x(op.n_dofs)
    x, rep = cg(op, b, tol=1e-10)
    xo, conv, it, res, why = ocg(ref.lhs_eval, b, tol=1e-10)
    assert not rep.converged and rep.reason == why == "stagnation" and rep.iterations == it


@pytest.mark.gpu
def test_gpu_cg_deterministic_and_torch_input():
    import torch
    from paper_2504_03573_b200.krylov import cg
    case, args, op = _case("cfg3b", 2, 21, "lagrange")
    b = case.draw_x(op.n_dofs)
    x1, r1 = cg(op, b, tol=1e-10)
    x2, r2 = cg(op, torch.from_numpy(b).cuda(), tol=1e-10)
    assert x2.is_cuda and r1.iterations == r2.iterations
    assert np.array_equal(x1, x2.cpu().numpy())


def test_oracle_gmres_solves_dense_system():
    from oracle import OracleOperator
    from oracle.krylov import gmres
    from paper_2504_03573_b200 import configs
    case = configs.build_case("cfg0", 3, 5)
    op = OracleOperator(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline")
    n = op.n_dofs
    a = np.stack([op.lhs_eval(np.eye(n)[j]) for j in range(n)], axis=1)
    b = np.random.default_rng(2).uniform(-1, 1, n)
    x, conv, it, res, why = gmres(op.lhs_eval, b, tol=1e-12, restart=n)
    assert conv and why == ""
    assert np.allclose(x, np.linalg.solve(a, b), rtol=1e-8, atol=1e-10)
    x, conv, it, res, why = gmres(op.lhs_eval, b, maxiter=0)
    assert not conv and it == 0 and why == "maxiter" and abs(res - 1.0) < 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("name,nx,seed,basis,restart,maxiter", [
    ("cfg0", 3, 8, "lagrange", 400, None), ("cfg1", 3, 9, "lagrange", 60, None),
    ("cfg1", 3, 9, "modified_modal", 30, 90), ("cfg4", 1, 4, "modified_modal", 200, 600)])
def test_gpu_gmres_matches_oracle_gmres(name, nx, seed, basis, restart, maxiter):
    """Device GMRES (sipg_gmres) against the CPU restatement of the reference's GMRES over the
    oracle apply: same stopping reason, iteration count within 2, same solution."""
    from oracle import OracleOperator
    from oracle.krylov import gmres as ogmres
    from paper_2504_03573_b200.krylov import gmres
    if name == "cfg4":
        from oracle.hybrid3d import HybridOracle3D
        from paper_2504_03573_b200 import configs
        from paper_2504_03573_b200.sipg import HelmholtzOperator
        case = configs.build_case(name, nx, seed)
        op = HelmholtzOperator(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline")
        m = case.mesh
        ref = HybridOracle3D(m.shapes, [el.verts for el in m.elements], m.vertices, case.order_map.n_modes,
                             case.order_map.n_quad)
    else:
        case, args, op = _case(name, nx, seed, basis)
        ref = OracleOperator(case.mesh, case.order_map, **args)
    b = case.draw_x(op.n_dofs)
    x, rep = gmres(op, b, tol=1e-10, restart=restart, maxiter=maxiter)
    xo, conv, it, res, why = ogmres(ref.lhs_eval, b, tol=1e-10, restart=restart, maxiter=maxiter)
    assert rep.converged == conv and rep.reason == why, (rep, why)
    if conv:
        assert abs(rep.iterations - it) <= 2
        assert rel_maxnorm(x, xo) <= 1e-7
        assert np.linalg.norm(b - ref.lhs_eval(x)) / np.linalg.norm(b) <= 1e-9
    else:      # restarted GMRES crawling on the ill-conditioned modal operator: same budget, same residual
        assert rep.iterations == it == maxiter
        assert abs(rep.residual - res) <= 1e-2 * res   # two orthogonalisations of an ill-conditioned basis


@pytest.mark.gpu
def test_gpu_solvers_maxiter_zero_and_zero_rhs():
    """maxiter=0 runs no iteration (reference krylov.py:54, 81, 97); b = 0 converges at once."""
    from paper_2504_03573_b200.krylov import cg, gmres
    case, args, op = _case("cfg0", 3, 8)
    b = case.draw_x(op.n_dofs)
    for solve in (cg, gmres):
        x, rep = solve(op, b, maxiter=0)
        assert not rep.converged and rep.iterations == 0 and rep.reason == "maxiter"
        assert abs(rep.residual - 1.0) < 1e-12 and not np.any(x)
        x, rep = solve(op, np.zeros(op.n_dofs))
        assert rep.converged and rep.iterations == 0 and not np.any(x)
    x, rep = gmres(op, b, tol=1e-14, restart=5, maxiter=7)
    assert not rep.converged and rep.reason == "maxiter" and rep.iterations == 7


@pytest.mark.gpu
def test_gpu_gmres_matches_cg_solution():
    from paper_2504_03573_b200.krylov import cg, gmres
    case, args, op = _case("cfg0", 3, 8, "lagrange")
    b = case.draw_x(op.n_dofs)
    xc, rc = cg(op, b, tol=1e-11)
    xg, rg = gmres(op, b, tol=1e-11, restart=op.n_dofs)   # full GMRES (the restarted one crawls here)
    assert rc.converged and rg.converged
    assert rel_maxnorm(xg, xc) <= 1e-7


def test_block_sparsity_and_asymmetry_match_reference_semantics():
    """reference krylov.py:159-183 restated as loops."""
    from paper_2504_03573_b200.krylov import asymmetry_norm, block_sparsity
    rng = np.random.default_rng(0)
    m = rng.standard_normal((12, 12))
    m[0:3, 5:8] = 0.0
    off = np.array([0, 3, 5, 8, 12])
    ref = np.zeros((4, 4), dtype=bool)
    for i in range(4):
        for j in range(4):
            ref[i, j] = np.abs(m[off[i]:off[i + 1], off[j]:off[j + 1]]).max() > 1e-12 * np.abs(m).max()
    assert np.array_equal(block_sparsity(m, off), ref)
    num = np.abs(m - m.T).sum(axis=0).max()
    assert asymmetry_norm(m) == float(num / np.abs(m).sum(axis=0).max())
    assert asymmetry_norm(np.zeros((3, 3))) == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("name,nx", [("cfg1", 2), ("cfg4", 1)])
def test_gpu_probe_dense_symmetric(name, nx):
    """Table-2 style symmetry probe (PAPER Table 2, reference krylov.py:144-164) on the GPU apply."""
    from paper_2504_03573_b200 import configs
    from paper_2504_03573_b200.krylov import asymmetry_norm, block_sparsity, probe_dense
    from paper_2504_03573_b200.sipg import HelmholtzOperator
    case = configs.build_case(name, nx, seed=3)
    kw = dict(basis_kind="modified_modal", tau_rule="baseline")
    if name != "cfg4":
        kw["shared_rule"] = "patched"
    op = HelmholtzOperator(case.mesh, case.order_map, **kw)
    A = probe_dense(op, op.n_dofs)
    x = case.draw_x(op.n_dofs)
    assert np.abs(A @ x - op(x)).max() <= 1e-12 * np.abs(A).sum(axis=1).max()
    assert asymmetry_norm(A) < 1e-12
    pat = block_sparsity(A, op._dof_off)
    assert np.all(np.diag(pat))
    with pytest.raises(ValueError):
        probe_dense(op, op.n_dofs, limit=op.n_dofs - 1)
