"""Config-4 host logic without a GPU: the plan3d tables reproduce the oracle's bases, and a numpy
emulation of the kernels' algorithm (oracle/h3_emulate.py) on the flattened plan reproduces the
oracle apply — so a GPU mismatch can only be a kernel bug."""
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_maxnorm
from oracle import hybrid3d as h
from paper_2504_03573_b200 import configs
from paper_2504_03573_b200.plan3d import SLOT, Plan3DBuilder

from oracle.h3_emulate import emulate, phi_matrix  # noqa: E402


def _ref(case):
    m = case.mesh
    return h.HybridOracle3D(m.shapes, [el.verts for el in m.elements], m.vertices,
                            case.order_map.n_modes, case.order_map.n_quad)


@pytest.mark.parametrize("nx,seed", [(2, 0), (3, 5)])
def test_plan_emulation_matches_oracle(nx, seed):
    case = configs.build_case("cfg4", nx, seed=seed)
    pb = Plan3DBuilder(case.mesh, case.order_map).build()
    ref = _ref(case)
    assert np.array_equal(pb.dof_off, ref.dof_off)
    for c in range(pb.class_desc.shape[0]):
        e = pb.class_elems[pb.class_desc[c][5]]
        assert np.abs(phi_matrix(pb, c) - ref.exps[e].Phi).max() < 1e-14
    x = case.draw_x(pb.n_dofs)
    assert rel_maxnorm(emulate(pb, x), ref(x)) <= 1e-13


def test_plan_slots_are_consistent():
    case = configs.build_case("cfg4", 4, seed=1)
    pb = Plan3DBuilder(case.mesh, case.order_map).build()
    S = pb.slots
    assert S.dtype == SLOT and S.dtype.itemsize == 96
    inter = S["kind"] == 1
    p = S["partner"][inter]
    assert np.array_equal(S["partner"][p], np.flatnonzero(inter))          # partners are mutual
    assert np.array_equal(S["nt"][p], S["nt"][inter])
    assert np.array_equal(S["pub_other"][inter], S["pub_self"][p])
    assert np.allclose(S["v"][inter] @ np.zeros(3), 0)
    assert np.all(np.diff(S["elem"]) >= 0)
    n_sub = sum(1 for t in case.mesh.interfaces if t.tag == "subface")
    assert len(S) == len(case.mesh.interfaces) + int(inter.sum()) // 2
    assert n_sub > 0
    # identical tet-tet faces of equal order map by the identity on both sides
    shp = np.array(case.mesh.shapes)
    nm = case.order_map.n_modes
    tt = inter & (shp[S["elem"]] == "tet") & (shp[S["elem"][np.maximum(S["partner"], 0)]] == "tet") & \
        (nm[S["elem"]] == nm[S["elem"][np.maximum(S["partner"], 0)]])
    assert tt.sum() > 0 and np.all(S["mkind"][tt] == 0)
