"""Config 4 (3-D hybrid hex / prism / tet): the CPU oracle (oracle/hybrid3d.py).

Parity for prisms/tets is UNPINNED by the reference (it has no such shapes,
SURVEY.md a18); the oracle is pinned instead by (1) bit-level agreement with the
reference-pinned hex oracle on all-hex meshes, and (2) properties of the exact
SIP operator: polynomial span of the bases, symmetry, positive definiteness,
Galerkin consistency on global polynomials (interior elements see -lap(u) only).
"""
import numpy as np
import pytest

from conftest import rel_maxnorm
from oracle import OracleOperator
from oracle import hybrid3d as h
from paper_2504_03573_b200 import configs
from paper_2504_03573_b200.mesh import OrderMap, Shape, generate_box
from paper_2504_03573_b200.mesh3d import generate_hybrid3d


def _ref_points(shape, rng, n):
    pts = []
    while len(pts) < n:
        xi = rng.uniform(-1, 1, 3)
        if shape == "tet" and xi.sum() > -1:
            continue
        if shape == "prism" and xi[0] + xi[2] > 0:
            continue
        pts.append(xi)
    return np.array(pts)


def _monomials(shape, n):
    P = n - 1
    r = range(n)
    if shape == "hex":
        return [(a, b, c) for a in r for b in r for c in r]
    if shape == "prism":
        return [(a, b, c) for a in r for b in r for c in r if a + c <= P]
    return [(a, b, c) for a in r for b in r for c in r if a + b + c <= P]


@pytest.mark.parametrize("shape", ["prism", "tet", "hex"])
@pytest.mark.parametrize("n", [2, 4, 7])
def test_basis_spans_the_shape_polynomials(shape, n):
    rng = np.random.default_rng(n)
    xi = _ref_points(shape, rng, 300)
    phi, _ = h.basis_eval(shape, n, h.eta_of_xi(shape, xi))
    mons = _monomials(shape, n)
    assert phi.shape[1] == len(mons) == h.n_coeffs(shape, n)
    M = np.stack([xi[:, 0] ** a * xi[:, 1] ** b * xi[:, 2] ** c for a, b, c in mons], axis=1)
    for A, B in ((M, phi), (phi, M)):      # each basis function is a polynomial, and they span
        res = B - A @ np.linalg.lstsq(A, B, rcond=None)[0]
        assert np.abs(res).max() < 1e-11


@pytest.mark.parametrize("shape", ["prism", "tet"])
def test_basis_derivatives_match_finite_differences(shape):
    rng = np.random.default_rng(0)
    eta = rng.uniform(-0.9, 0.9, (20, 3))
    _, d = h.basis_eval(shape, 5, eta)
    for k in range(3):
        e = np.zeros(3)
        e[k] = 1e-6
        fd = (h.basis_eval(shape, 5, eta + e)[0] - h.basis_eval(shape, 5, eta - e)[0]) / 2e-6
        assert np.abs(fd - d[k]).max() < 1e-7


def test_couplings_dict_matcher_equals_vectorised():
    m = generate_hybrid3d(4, np.random.default_rng(11))
    c_dict = h.build_couplings(m.shapes, [el.verts for el in m.elements])
    assert c_dict == m.couplings()
    kinds = {k for _, _, k in c_dict}
    assert kinds == {"conform", "subface", "boundary"}


def test_all_hex_matches_reference_pinned_oracle():
    m = generate_box(3, 3, Shape.HEX, (0.0, 1.0))
    rng = np.random.default_rng(3)
    P = rng.integers(2, 6, m.n_elements)
    ref = OracleOperator(m, OrderMap(P + 1, P + 2), basis_kind="modified_modal", tau_rule="baseline",
                         shared_rule="patched", face_absorb="trace_iproduct")
    hyb = h.HybridOracle3D(["hex"] * m.n_elements, [el.verts for el in m.elements], m.vertices, P + 1, P + 2)
    x = rng.uniform(-1, 1, ref.n_dofs)
    assert rel_maxnorm(hyb(x), ref(x)) <= 1e-14


def _oracle(case, lam=1.0):
    m = case.mesh
    return h.HybridOracle3D(m.shapes, [el.verts for el in m.elements], m.vertices,
                            case.order_map.n_modes, case.order_map.n_quad, lambda_=lam)


def test_symmetric_positive_definite():
    case = configs.build_case("cfg4", 2, seed=2)
    m = case.mesh
    P = np.random.default_rng(2).integers(1, 3, m.n_elements)
    op = h.HybridOracle3D(m.shapes, [el.verts for el in m.elements], m.vertices, P + 1, P + 2)
    A = np.stack([op(e) for e in np.eye(op.n_dofs)], axis=1)
    assert np.abs(A - A.T).max() <= 1e-13 * np.abs(A).max()
    assert np.linalg.eigvalsh(0.5 * (A + A.T)).min() > 0.0
    assert not np.any(op(np.zeros(op.n_dofs)))


@pytest.mark.parametrize("fun,lap", [
    (lambda x: 1 + 2 * x[:, 0] - 3 * x[:, 1] + 0.5 * x[:, 2], 0.0),
    (lambda x: x[:, 0] ** 2 + 2 * x[:, 1] * x[:, 2] - x[:, 2] ** 2 + x[:, 0], 0.0),
    (lambda x: x[:, 0] ** 2 + x[:, 1] ** 2 + 3 * x[:, 2] ** 2, 10.0),
])
def test_galerkin_consistency_on_global_polynomials(fun, lap):
    case = configs.build_case("cfg4", 4, seed=5)
    op = _oracle(case, lam=0.0)
    c = np.zeros(op.n_dofs)
    for e, ex in enumerate(op.exps):
        x = op.x0[e] + (ex.xi + 1.0) @ op.F[e].T
        c[op.dof_off[e]:op.dof_off[e + 1]] = np.linalg.lstsq(ex.Phi, fun(x), rcond=None)[0]
    y = op(c)
    bnd = {l[0] for l, r, _ in op.couplings if r is None}
    checked = 0
    for e, ex in enumerate(op.exps):
        if e in bnd:
            continue
        ip = ex.Phi.T @ (ex.ref_w * op.detJ[e])          # int phi_i
        assert np.abs(y[op.dof_off[e]:op.dof_off[e + 1]] + lap * ip).max() < 1e-11
        checked += 1
    assert checked > 50


def test_cfg4_recipe_counts():
    case = configs.build_case("cfg4", 6, seed=0)
    shapes = case.mesh.shapes
    cubes = 6 ** 3
    n_hex, n_pri, n_tet = shapes.count("hex"), shapes.count("prism"), shapes.count("tet")
    assert n_hex + n_pri // 2 + n_tet // 6 == cubes
    assert 0.25 < n_hex / cubes < 0.55 and 0.15 < n_tet / 6 / cubes < 0.45
    assert set(np.unique(case.order_map.n_modes)) == {4, 5, 6, 7}


FIX = sorted((__import__("pathlib").Path(__file__).resolve().parent / "golden" / "oracle_cfg4").glob("cfg4_n*.npz"))


@pytest.mark.parametrize("path", FIX, ids=[p.stem for p in FIX])
def test_oracle_matches_frozen_cfg4_fixtures(path):
    """tests/golden/oracle_cfg4 freezes the property-tested oracle (make_cfg4.py)."""
    g = np.load(path)
    case = configs.build_case("cfg4", int(g["nx"]), int(g["seed"]))
    op = _oracle(case)
    assert np.array_equal(op.dof_off, g["dof_off"])
    x = case.draw_x(op.n_dofs)
    assert np.array_equal(x, g["x"])
    assert rel_maxnorm(op(x), g["y"]) <= 1e-14


# ---- rhs_assemble / l2_error, pinned by the real reference on an all-hex mesh
def _sin_case(k, lam=1.0):
    """The reference's sinusoidal manufactured case (sipg.py:88-100), restated."""
    def exact(x):
        return np.sin(k * x[0]) * np.sin(k * x[1]) * np.sin(k * x[2])

    def forcing(x):
        return -(lam + 3 * k * k) * exact(x)
    return exact, forcing


def test_rhs_and_l2_match_reference_fixture():
    from pathlib import Path
    d = np.load(Path(__file__).resolve().parent / "golden" / "oracle_cfg4" / "ref_rhs_hex.npz")
    P = d["P"]
    ref = h.HybridOracle3D(["hex"] * len(P), d["elem_verts"], d["verts"], P + 1, P + 2)
    exact, forcing = _sin_case(float(d["k"]))
    case = type("Case", (), {"exact": staticmethod(exact), "forcing": staticmethod(forcing)})
    b = ref.rhs_assemble(case, {"dirichlet": exact})
    assert rel_maxnorm(b, d["b"]) <= 1e-13
    assert abs(ref.l2_error(d["x"], exact) - float(d["err"])) <= 1e-13 * float(d["err"])


@pytest.mark.parametrize("shape", ["hex", "prism", "tet"])
@pytest.mark.parametrize("n,dq", [(2, 1), (5, 1), (7, 3)])
def test_rhs3d_dense_phi_matches_oracle_basis(shape, n, dq):
    """The product's dense class table (built from the plan's staged BwdTrans tables) is the
    oracle's basis at the volume points."""
    from paper_2504_03573_b200.plan3d import ClassTables3
    from paper_2504_03573_b200.rhs3d import dense_phi
    ex = h.Expansion3(shape, n, n + dq)
    assert np.abs(dense_phi(ClassTables3(shape, n, n + dq)) - ex.Phi).max() <= 1e-14
