"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's matrix-free SIP-Helmholtz apply
(`HelmholtzOperator.lhs_eval`, reference pkg/src/dgsipg/sipg.py:558-602) and of
the plan construction that feeds it.  Every function cites the reference
file:line it restates.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this package,
and only as the checker / the CPU baseline: the product
(`paper_2504_03573_b200`) never imports it and has no CPU fallback.

Parity pinning: `tests/test_oracle_golden.py` checks this oracle against golden
vectors produced by the real reference (tests/golden/make_golden.py).

Patches, selectable per operator:
  tau_rule="baseline"   P1: tau = max(n_L, n_R)^2 / h (BASELINE "(P+1)^2/h")
  tau_rule="reference"  tau = C max(n-1, 1)^2 / h (sipg.py:351-360)
  shared_rule="patched" P2: Gauss-Legendre max(q) trace rule when a side is not GLL
  shared_rule="reference"  rule of the higher side (trace.py:202-206)
"""

from .operator import OracleOperator  # noqa: F401
