"""Config 4's triangular faces pinned to the REAL reference's triangle expansion
(tests/golden/oracle_cfg4/tri_pin.npz, written by make_tri_pin.py from reference
stdregions.py:266-383 / 575-674 / 850-877).

Prisms and tets have no reference.  What can be pinned is every piece of them that the
reference does define:
* the basis on each triangular face: restricted to any tet face or prism triangle, the 3-D
  collapsed modified-modal basis must be exactly the reference triangle's basis in the face's
  collapsed coordinates — every non-vanishing restricted function equal to one reference triangle
  function, bijectively (measured: bit-identical, 0.0 difference, n_modes 2..7);
* the restriction operator: the endpoint rows the plan ships to the kernels (plan3d "E") equal the
  reference's `_endpoint_row`, and applying them to a field on the triangle grid reproduces the
  reference's `face_values_from_phys` on every triangle edge.
"""
import numpy as np
import pytest

from conftest import GOLDEN

PIN = GOLDEN / "oracle_cfg4" / "tri_pin.npz"


@pytest.mark.parametrize("n", range(2, 8))
def test_collapsed_faces_are_the_reference_triangle(n):
    from oracle.hybrid3d import FACES3, basis_eval, face_to_eta, tensor_params, tri_eval
    g = np.load(PIN)
    q = n + 1
    pts = g[f"gl_pts_q{q}"]
    T = g[f"tri_phi_n{n}"]
    prm = tensor_params([pts, pts])
    To, Ta, Tb = tri_eval(n, prm[:, 0], prm[:, 1])
    assert np.abs(To - T).max() <= 1e-15
    assert np.abs(Ta - g[f"tri_d0_n{n}"]).max() <= 1e-11 * np.abs(Ta).max()
    assert np.abs(Tb - g[f"tri_d1_n{n}"]).max() <= 1e-11 * np.abs(Tb).max()
    for shape, faces in (("tet", (0, 1, 2, 3)), ("prism", (1, 3))):
        for f in faces:
            phi, _ = basis_eval(shape, n, face_to_eta(FACES3[shape][f], prm))
            nz = np.abs(phi).max(axis=0) > 1e-13
            assert nz.sum() == T.shape[1], (shape, f)
            hits = []
            for c in phi[:, nz].T:
                d = np.abs(T - c[:, None]).max(axis=0)
                assert d.min() <= 1e-15, (shape, f)
                hits.append(int(d.argmin()))
            assert sorted(hits) == list(range(T.shape[1])), (shape, f)


@pytest.mark.parametrize("n", range(2, 8))
def test_face_restriction_rows_match_reference(n):
    from paper_2504_03573_b200.plan3d import ClassTables3
    g = np.load(PIN)
    q = n + 1
    ct = ClassTables3("tet", n, q)
    E = ct.parts["E"].reshape(3, 2, q)          # [axis][side][k]
    for a in range(3):
        assert np.abs(E[a, 0] - g[f"endrow_q{q}_m"]).max() <= 1e-14
        assert np.abs(E[a, 1] - g[f"endrow_q{q}_p"]).max() <= 1e-14
    # the triangle's edges: fixed axis 1 side -1, axis 0 side +1, axis 0 side -1 (stdregions.py:155-169)
    u = g[f"u_n{n}"].reshape(q, q)
    faces = {0: u @ E[1, 0], 1: E[0, 1] @ u, 2: E[0, 0] @ u}
    for f, vals in faces.items():
        ref = g[f"tri_face{f}_n{n}"]
        assert np.abs(vals - ref).max() <= 1e-14 * np.abs(ref).max()
