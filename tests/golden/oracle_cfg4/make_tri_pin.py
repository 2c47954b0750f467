"""Fixtures that pin config 4's triangular faces to the REAL reference's triangle expansion.

Config 4's prisms and tets have no reference, but every triangular face of them is,
by construction of oracle/hybrid3d.py, the reference's own modified-modal triangle in the face's
collapsed coordinates.  This script runs the reference (`/root/reference/pkg/src/dgsipg`, read-only)
and records, for n_modes = 2..7 with q = n + 1 Gauss-Legendre points per direction (the config-4
rule):

  tri_phi_n{n}   reference triangle basis at the collapsed q x q grid (bwd_trans of unit vectors,
                 stdregions.py:575-597 on the tables of stdregions.py:266-383), (q*q, n(n+1)/2)
  tri_d0_n{n}, tri_d1_n{n}   its collapsed-coordinate derivatives (phys_deriv, stdregions.py:658-674)
  tri_face{f}_n{n}           face_values_from_phys (stdregions.py:855-877) of a seeded random field
                             u_n{n} on the q x q grid, for the triangle's three edges
  u_n{n}                     that field
  endrow_q{q}_{m|p}          the endpoint rows of GL(q) at -1 / +1 (stdregions.py:850-852)

Usage: python tests/golden/oracle_cfg4/make_tri_pin.py   (writes tri_pin.npz next to this file)
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"


def main():
    sys.path.insert(0, REF)
    from dgsipg import polylib, stdregions as sr
    out = {}
    rng = np.random.default_rng(2024)
    for n in range(2, 8):
        q = n + 1
        exp = sr.expansion(sr.Shape.TRI, polylib.BasisKind.MODIFIED_MODAL, n, q)
        nc = exp.n_coeffs
        phi = sr.bwd_trans(exp, np.eye(nc))                     # (q*q, nc)
        d = sr.phys_deriv(exp, phi)
        out[f"tri_phi_n{n}"] = phi
        out[f"tri_d0_n{n}"] = d[0]
        out[f"tri_d1_n{n}"] = d[1]
        u = rng.uniform(-1.0, 1.0, q * q)
        out[f"u_n{n}"] = u
        for f in range(3):
            out[f"tri_face{f}_n{n}"] = sr.face_values_from_phys(exp, f, u)
        rule = polylib.quad_rule(polylib.QuadKind.GAUSS_LEGENDRE, q)
        out[f"endrow_q{q}_m"] = sr._endpoint_row(rule, -1)[0]
        out[f"endrow_q{q}_p"] = sr._endpoint_row(rule, 1)[0]
        out[f"gl_pts_q{q}"] = rule.points
    np.savez_compressed(Path(__file__).resolve().parent / "tri_pin.npz", **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
