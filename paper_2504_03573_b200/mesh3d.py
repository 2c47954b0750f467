"""Config-4 meshes: 3-D hybrid hex / prism / tet on a cube grid (plan input).

Not in the reference (it has no prism or tet); this is
the BASELINE.json config-4 recipe: the unit cube on an n^3 cube grid, each
cube (x slowest, then y, z; one rng.uniform() per cube in that order) kept as
one hex (u < 0.4), split into 2 prisms (u < 0.7) or into 6 tets.

Conformity: every split follows the Kuhn pattern — each split face is cut
along its diagonal from the lowest to the highest lattice vertex — so two split
cubes always meet conformingly (tri-tri).  Prisms are extruded along z and cut
by the plane x = y.  A hex (or a prism's full quad face) next to a split cube
meets two triangles: that is a "subface" coupling (each triangle couples to
half of the quad face, SURVEY a18's resolution).

Local vertex orders: hex as `generate_box` (reference mesh.py:196-225);
prism V0..V3 the quad at xi2 = -1, V4/V5 the top edge (oracle/hybrid3d.py
shape_funcs); tet = the Kuhn path (c, c+e_a, c+e_a+e_b, c+1).  Prism triangles
and tets list their vertices in increasing global id on every triangular face,
so both sides of a tri-tri interface share one collapsed parametrisation (the
trace grids coincide; no orientation codes are needed).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

from .mesh import Element, Interface, Shape

HEX, PRISM, TET = "hex", "prism", "tet"

# local faces: (corner local vertex ids, triangular?) — same order as oracle/hybrid3d.py FACES3
FACE_CORNERS3 = {
    HEX: (((0, 3, 4, 7), False), ((1, 2, 5, 6), False), ((0, 1, 4, 5), False), ((3, 2, 7, 6), False),
          ((0, 1, 3, 2), False), ((4, 5, 7, 6), False)),
    PRISM: (((0, 1, 2, 3), False), ((0, 1, 4), True), ((1, 2, 5, 4), False), ((3, 2, 5), True),
            ((0, 3, 4, 5), False)),
    TET: (((0, 1, 2), True), ((0, 1, 3), True), ((1, 2, 3), True), ((0, 2, 3), True)),
}
SHAPE_CODE = {HEX: 0, PRISM: 1, TET: 2}
P_HEX, P_PRISM = 0.4, 0.7


@dataclass
class HybridMesh3D:
    """Vertices, elements (Element(Shape, verts)) and couplings as `Interface`s with
    `orientation=-1` (the mapping between the two sides is geometric) and `tag` in
    {"conform", "subface", "dirichlet"}; boundary couplings have `right=None`."""
    vertices: np.ndarray
    elements: list
    interfaces: list
    dim: int = 3
    is_hybrid3d = True

    @property
    def n_elements(self) -> int:
        return len(self.elements)

    @property
    def shapes(self) -> list:
        return [el.shape.value for el in self.elements]

    def element_verts(self, e: int) -> np.ndarray:
        return self.vertices[list(self.elements[e].verts)]

    def centroid(self, e: int) -> np.ndarray:
        return self.element_verts(e).mean(axis=0)

    def couplings(self):
        """[(left, right|None, kind)] with kind "boundary" for boundary faces."""
        return [(f.left, f.right, "boundary" if f.right is None else f.tag) for f in self.interfaces]


def generate_hybrid3d(nx, rng: np.random.Generator, extent=(0.0, 1.0),
                      p_hex: float = P_HEX, p_prism: float = P_PRISM) -> HybridMesh3D:
    """`nx`: cubes per axis (int) or (nx, ny, nz); `extent`: (lo, hi) for every axis or one pair
    per axis (weak-scaling boxes are stacked along x, partition.stack_box_config)."""
    nxs = (int(nx),) * 3 if np.ndim(nx) == 0 else tuple(int(v) for v in nx)
    ext = (tuple(extent),) * 3 if np.ndim(extent) == 1 else tuple(tuple(e) for e in extent)
    axes = [np.linspace(lo, hi, n + 1) for (lo, hi), n in zip(ext, nxs)]
    g = np.meshgrid(*axes, indexing="ij")
    verts = np.stack([a.reshape(-1) for a in g], axis=-1)
    my, mz = nxs[1] + 1, nxs[2] + 1

    def vid(i, j, k):
        return (i * my + j) * mz + k
    els = []
    perms = list(itertools.permutations(range(3)))
    for i in range(nxs[0]):
        for j in range(nxs[1]):
            for k in range(nxs[2]):
                r = rng.uniform()
                c = [[[vid(i + a, j + b, k + cc) for cc in (0, 1)] for b in (0, 1)] for a in (0, 1)]
                if r < p_hex:
                    els.append(Element(Shape.HEX, (c[0][0][0], c[1][0][0], c[1][1][0], c[0][1][0],
                                                   c[0][0][1], c[1][0][1], c[1][1][1], c[0][1][1])))
                elif r < p_prism:
                    els.append(Element(Shape.PRISM, (c[0][0][0], c[1][0][0], c[1][0][1], c[0][0][1],
                                                     c[1][1][0], c[1][1][1])))
                    els.append(Element(Shape.PRISM, (c[0][0][0], c[0][1][0], c[0][1][1], c[0][0][1],
                                                     c[1][1][0], c[1][1][1])))
                else:
                    for p in perms:
                        path = [(0, 0, 0)]
                        for a in p:
                            s = list(path[-1])
                            s[a] = 1
                            path.append(tuple(s))
                        els.append(Element(Shape.TET, tuple(c[a][b][cc] for a, b, cc in path)))
    return HybridMesh3D(verts, els, build_couplings3d(els))


def _face_table(elements):
    """(e, f, is_tri, sorted corner keys padded with -1) for every local face."""
    rows_e, rows_f, tri, keys = [], [], [], []
    for e, el in enumerate(elements):
        for f, (cv, is_tri) in enumerate(FACE_CORNERS3[el.shape.value]):
            rows_e.append(e)
            rows_f.append(f)
            tri.append(is_tri)
            k = sorted(el.verts[v] for v in cv)
            keys.append(k + [-1] * (4 - len(k)))
    return (np.asarray(rows_e, dtype=np.int64), np.asarray(rows_f, dtype=np.int64),
            np.asarray(tri, dtype=bool), np.asarray(keys, dtype=np.int64))


def _pack3(k):
    return (k[..., 0] << 42) | (k[..., 1] << 21) | k[..., 2]


def build_couplings3d(elements) -> list:
    """Vectorised face matcher (the dict-based oracle/hybrid3d.build_couplings is its check):
    conform pairs (identical corner sets, left = lower element id), subface pairs (a lone
    triangle inside a lone quad face; triangle = left), boundary faces; ordered by
    (left e, left f, right e, right f)."""
    fe, ff, tri, keys = _face_table(elements)
    if keys.max() >= (1 << 21):
        raise ValueError("too many vertices for the packed face keys")
    n = fe.size
    order = np.lexsort(keys.T[::-1])
    ks = keys[order]
    same = np.all(ks[1:] == ks[:-1], axis=1)
    if np.any(same[1:] & same[:-1]):
        raise ValueError("a face is shared by more than two elements")
    first = np.flatnonzero(same)
    a, b = order[first], order[first + 1]
    a, b = np.minimum(a, b), np.maximum(a, b)      # face rows are (e, f)-ordered
    paired = np.zeros(n, dtype=bool)
    paired[a] = paired[b] = True
    la, ra, kind = [a], [b], [np.zeros(a.size, dtype=np.int64)]
    # subfaces: lone quads against lone triangles
    lq = np.flatnonzero(~paired & ~tri)
    lt = np.flatnonzero(~paired & tri)
    if lq.size and lt.size:
        tcode = _pack3(keys[lt, :3])
        o = np.argsort(tcode)
        tcode_s = tcode[o]
        qk = keys[lq]
        hits = []
        for drop in range(4):
            sub = np.delete(qk, drop, axis=1)
            code = _pack3(sub)
            pos = np.clip(np.searchsorted(tcode_s, code), 0, tcode_s.size - 1)
            ok = tcode_s[pos] == code
            hits.append(np.where(ok, lt[o[pos]], -1))
        hits = np.stack(hits, axis=1)
        nh = (hits >= 0).sum(axis=1)
        if np.any((nh != 0) & (nh != 2)):
            raise ValueError("a quad face is not covered by exactly two triangles")
        qi, slot = np.nonzero(hits >= 0)
        tl = hits[qi, slot]
        qr = lq[qi]
        la.append(tl)
        ra.append(qr)
        kind.append(np.ones(tl.size, dtype=np.int64))
        paired[tl] = paired[qr] = True
    la = np.concatenate(la)
    ra = np.concatenate(ra)
    kind = np.concatenate(kind)
    bnd = np.flatnonzero(~paired)
    la = np.concatenate([la, bnd])
    ra = np.concatenate([ra, np.full(bnd.size, -1, dtype=np.int64)])
    kind = np.concatenate([kind, np.full(bnd.size, 2, dtype=np.int64)])
    re_ = np.where(ra >= 0, fe[np.maximum(ra, 0)], -1)
    rf_ = np.where(ra >= 0, ff[np.maximum(ra, 0)], -1)
    o = np.lexsort((rf_, re_, ff[la], fe[la]))
    tags = ("conform", "subface", "dirichlet")
    out = []
    for i in o:
        left = (int(fe[la[i]]), int(ff[la[i]]))
        right = None if ra[i] < 0 else (int(re_[i]), int(rf_[i]))
        out.append(Interface(left, right, -1, tags[kind[i]]))
    return out
