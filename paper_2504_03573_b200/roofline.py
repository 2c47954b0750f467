"""Algorithmic bytes and flops of one apply, from a plan.

Bytes (primary, %HBM): read x + write y (16 B per DoF) + compact geometry:
  regular element  8 (d^2 + 1) + sum_faces 8 (d + 2)
  deformed element 8 (d^2 + 1) q^d + sum_faces 8 (d + 1) q^(d-1)
Flops (secondary, %fp64), sum-factorised lower bound per element:
  2 [2 BT + 2 d q^(d+1) + (2 d^2 + 1) q^d],
  BT = sum_{k=1..d} q^k n^(d-k+1) (tensor), q n(n+1)/2 + q^2 (n+1) (triangle).
Trace intermediates, tables and index maps are excluded.
"""
from __future__ import annotations

import numpy as np

from . import layout as L


def per_class(pb):
    rows = []
    for ci, (c, geom, ids) in enumerate(pb.class_list):
        d, n, q = c.dim, c.n, c.nq[0]
        nf = len(c.faces)
        if geom == L.GEOM_REGULAR:
            gb = 8 * (d * d + 1) + nf * 8 * (d + 2)
        else:
            gb = 8 * (d * d + 1) * q ** d + nf * 8 * (d + 1) * q ** (d - 1)
        if c.shape == "tri":
            bt = q * n * (n + 1) // 2 + q * q * (n + 1)
        else:
            bt = sum(q ** k * n ** (d - k + 1) for k in range(1, d + 1))
        fl = 2 * (2 * bt + 2 * d * q ** (d + 1) + (2 * d * d + 1) * q ** d)
        rows.append({"cls": ci, "shape": c.shape, "n": n, "q": q, "geom": int(geom), "count": int(ids.size),
                     "dofs": int(ids.size * c.n_coeffs),
                     "bytes": int(ids.size * (16 * c.n_coeffs + gb)), "flops": int(ids.size * fl)})
    return rows


def totals(pb):
    rows = per_class(pb)
    return sum(r["bytes"] for r in rows), sum(r["flops"] for r in rows)
