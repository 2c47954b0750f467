"""Size-independent property at BASELINE sizes: the SIP operator is symmetric, so
a·(A b) = b·(A a) for any a, b (PAPER Table 2; reference krylov.py:159-164 measures the same
property column by column on small meshes).  Conforming gathers (cfg3a), shared traces (cfg3b,
cfg4) and certified point-to-point interpolation (cfg2: the certificate of trace.py:84-106 is
exactly the condition under which the p2p coupling is symmetric; the reference-pinned oracle gives
|a·Ab − b·Aa| / Σ|a·Ab| ≈ 1e-17 on cfg2 at 16², 32², 64²) all evaluate a symmetric discrete form, so
the GPU apply must be symmetric up to rounding.  Bar: |a·Ab − b·Aa| <= 1e-12 · Σ|a_i (Ab)_i|."""
import numpy as np
import pytest

from paper_2504_03573_b200 import configs
from paper_2504_03573_b200.sipg import HelmholtzOperator

pytestmark = pytest.mark.gpu
KW = dict(basis_kind="modified_modal", tau_rule="baseline", shared_rule="patched")


@pytest.mark.parametrize("name,nx", [("cfg3a", 32), ("cfg3b", 32), ("cfg4", 48), ("cfg1", 64), ("cfg2", 256)])
def test_full_size_bilinear_symmetry(name, nx):
    import torch
    case = configs.build_case(name, nx, 0)
    kw = dict(KW) if name != "cfg4" else dict(basis_kind="modified_modal", tau_rule="baseline")
    op = HelmholtzOperator(case.mesh, case.order_map, **kw)
    g = torch.Generator(device="cuda").manual_seed(7)
    a = torch.rand(op.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    b = torch.rand(op.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    ab, ba = op(b), op(a)
    lhs, rhs = float(torch.dot(a, ab)), float(torch.dot(b, ba))
    scale = float(torch.maximum((a * ab).abs().sum(), (b * ba).abs().sum()))
    print(f"{name}: n_dofs={op.n_dofs} |a.Ab - b.Aa| / scale = {abs(lhs - rhs) / scale:.3e}")
    assert abs(lhs - rhs) <= 1e-12 * scale
    # and A is not trivially zero / diagonal-free
    assert float(torch.dot(a, ba)) > 0.0
