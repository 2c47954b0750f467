"""Bit-exact maps against the reference: topology dump, DoF
offsets, trace slots, per-interface strategy, transfer permutations."""
import hashlib

import numpy as np
import pytest

from conftest import golden_files, golden_operator_kwargs, load_golden
from paper_2504_03573_b200 import configs
from paper_2504_03573_b200.plan import PlanBuilder

SMALL = golden_files(full=False)
FULL = golden_files(full=True)


def _plan(g):
    case = configs.build_case(str(g["config"]), int(g["nx"]), int(g["seed"]))
    kw = golden_operator_kwargs(g)
    return case, PlanBuilder(case.mesh, case.order_map, **kw).build()


@pytest.mark.parametrize("path", SMALL, ids=[p.stem for p in SMALL])
def test_maps_small(path):
    g = load_golden(path)
    case, pb = _plan(g)
    assert hashlib.sha256(case.mesh.dump().encode()).digest() == bytes(g["dump_sha256"])
    assert np.array_equal(pb.dof_off, g["dof_off"])
    assert np.array_equal(pb.trace_slots, g["trace_slots"])
    assert np.array_equal(pb.strategy_of, g["itf_strategy"])
    assert pb.transfer_perm_sha256() == bytes(g["perm_sha256"])


@pytest.mark.slow
@pytest.mark.parametrize("path", FULL, ids=lambda p: p.stem)
def test_maps_full(path):
    """BASELINE sizes (cfg1 64^2, cfg2 256^2, cfg3a / cfg3b 32^3): every map the reference run
    recorded, bit-exact."""
    g = load_golden(path)
    case, pb = _plan(g)
    assert hashlib.sha256(case.mesh.dump().encode()).digest() == bytes(g["dump_sha256"])
    assert np.array_equal(pb.dof_off, g["dof_off"])
    assert np.array_equal(pb.trace_slots, g["trace_slots"])
    key = "itf_strategy" if "itf_strategy" in g else "strategy"
    assert np.array_equal(pb.strategy_of, g[key])
    assert pb.transfer_perm_sha256() == bytes(g["perm_sha256"])
