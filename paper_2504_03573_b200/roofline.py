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


def _per_class_h3(pb):
    """Hybrid 3-D plans (plan3d.py): one row per launch unit — the publish kernels (recomputed
    BwdTrans / traces: not part of the algorithmic count, 0 bytes / flops), the apply kernels, which
    carry the element's whole algorithmic count, then the per-class flux slot launches (face work,
    not part of the volume count either).  BwdTrans of the
    collapsed shapes, stage by stage: prism n_tri n q + n_tri q^2 + (n+1) q^3, tet
    n_c q + (n_tri+1) q^2 + (n+1) q^3."""
    from .plan3d import CD3_COUNT, CD3_N, CD3_NC, CD3_Q, CD3_SHAPE
    names = {0: "hex", 1: "prism", 2: "tet"}
    nfaces = {0: 6, 1: 5, 2: 4}
    rows = []
    for unit in ("pub", "apply", "flux"):
        for ci, cd in enumerate(pb.class_desc):
            s, n, q, nc, cnt = int(cd[CD3_SHAPE]), int(cd[CD3_N]), int(cd[CD3_Q]), int(cd[CD3_NC]), int(cd[CD3_COUNT])
            ntri = n * (n + 1) // 2
            if s == 0:
                bt = q * n ** 3 + q * q * n * n + q ** 3 * n
            elif s == 1:
                bt = ntri * n * q + ntri * q * q + (n + 1) * q ** 3
            else:
                bt = nc * q + (ntri + 1) * q * q + (n + 1) * q ** 3
            d = 3
            fl = 2 * (2 * bt + 2 * d * q ** (d + 1) + (2 * d * d + 1) * q ** d)
            gb = 8 * (d * d + 1) + nfaces[s] * 8 * (d + 2)
            a = unit == "apply"
            rows.append({"cls": ci, "shape": names[s], "n": n, "q": q, "geom": 0, "count": cnt,
                         "unit": unit, "dofs": cnt * nc if a else 0,
                         "bytes": cnt * (16 * nc + gb) if a else 0, "flops": cnt * fl if a else 0})
    return rows


def per_class(pb):
    if getattr(pb, "is_h3", False):
        return _per_class_h3(pb)
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
