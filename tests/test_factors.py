"""`HelmholtzOperator.exps` / `.factors` (reference sipg.py:262-267, mesh.py:295-432) against the
real reference's setup objects (imported read-only in this container; skipped where it is absent)."""
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
mg = pytest.importorskip("make_golden") if Path("/root/reference/pkg/src").exists() else None
pytestmark = pytest.mark.skipif(mg is None, reason="reference not present")


@pytest.mark.parametrize("name,nx,seed", [("cfg1", 3, 3), ("cfg2", 3, 4), ("cfg3b", 2, 5)])
def test_factors_and_exps_match_reference(name, nx, seed):
    from paper_2504_03573_b200 import configs
    from paper_2504_03573_b200.factors import standard_factors
    from paper_2504_03573_b200.plan import PlanBuilder
    m, om, _ = mg.build_case(name, nx, seed)
    ref = mg.make_operator(m, om)
    case = configs.build_case(name, nx, seed)
    pb = PlanBuilder(case.mesh, case.order_map, basis_kind="modified_modal", tau_rule="baseline",
                     shared_rule="patched").build()
    f = standard_factors(case.mesh, pb)
    assert len(f) == len(ref.factors.elements)
    for e in range(len(f)):
        a, b = f[e], ref.factors[e]
        assert a.regular == b.regular
        for k in ("J", "dxi_dx", "jac_w", "x"):
            A, B = getattr(a, k), getattr(b, k)
            assert A.shape == B.shape, k
            assert np.abs(A - B).max() <= 1e-13 * (np.abs(B).max() + 1.0), k
        assert abs(a.volume - b.volume) <= 1e-14
        assert len(a.faces) == len(b.faces)
        for fa, fb in zip(a.faces, b.faces):
            for k in ("normal", "surf_jac", "surf_jw", "x"):
                A, B = getattr(fa, k), getattr(fb, k)
                assert A.shape == B.shape, (k, A.shape, B.shape)
                assert np.abs(A - B).max() <= 1e-13 * (np.abs(B).max() + 1.0), k
            assert abs(fa.area - fb.area) <= 1e-14
        ea, eb = pb.ct[e], ref.exps[e]
        assert (ea.n_modes, ea.n_coeffs, ea.n_phys, tuple(ea.nq)) == (eb.n_modes, eb.n_coeffs, eb.n_phys, tuple(eb.nq))
        assert np.abs(ea.ref_weights - eb.ref_weights).max() <= 1e-15
        assert np.abs(ea.xi_phys - eb.xi_phys).max() <= 1e-15
