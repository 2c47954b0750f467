"""Mesh topology, generators and order maps (plan inputs).

Mirrors the reference's `dgsipg.mesh` surface — `Element`, `Interface`,
`MeshTopology` (+ `dump`, reference mesh.py:38-103), `generate_box`
(mesh.py:160-226), `perturb_mesh` (268-289), `OrderMap` (447-465) — with a
vectorised face matcher in place of the reference's per-face dictionary scan
(mesh.py:234-265).  The produced numbering, interface order and orientation
codes are identical to the reference's (checked bit-exact against reference
`dump()` hashes in tests/test_maps.py).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

__all__ = ["Shape", "Element", "Interface", "MeshTopology", "OrderMap",
           "generate_box", "perturb_mesh", "build_topology", "generate_hybrid"]


class Shape(enum.Enum):
    SEG = "seg"
    QUAD = "quad"
    TRI = "tri"
    HEX = "hex"
    PRISM = "prism"   # config 4 only (mesh3d.py): not in the reference
    TET = "tet"

    @property
    def dim(self) -> int:
        return {"seg": 1, "quad": 2, "tri": 2, "hex": 3, "prism": 3, "tet": 3}[self.value]


def as_shape(s) -> Shape:
    return s if isinstance(s, Shape) else Shape(getattr(s, "value", s))


# corner vertices of each face in the element's vertex list, in face-parameter
# order (reference stdregions.py:140-192, Face.corner_verts)
FACE_CORNERS = {
    "quad": ((0, 3), (1, 2), (0, 1), (3, 2)),
    "tri": ((0, 1), (1, 2), (0, 2)),
    "hex": ((0, 3, 4, 7), (1, 2, 5, 6), (0, 1, 4, 5), (3, 2, 7, 6), (0, 1, 3, 2), (4, 5, 7, 6)),
}


@dataclass(frozen=True)
class Element:
    shape: Shape
    verts: tuple


@dataclass(frozen=True)
class Interface:
    left: tuple
    right: tuple | None
    orientation: int
    tag: str | None = None

    @property
    def is_boundary(self) -> bool:
        return self.right is None


@dataclass
class MeshTopology:
    dim: int
    vertices: np.ndarray
    elements: list
    interfaces: list

    @property
    def n_elements(self) -> int:
        return len(self.elements)

    def element_verts(self, e: int) -> np.ndarray:
        return self.vertices[list(self.elements[e].verts)]

    def centroid(self, e: int) -> np.ndarray:
        return self.element_verts(e).mean(axis=0)

    def interior(self):
        return [(i, f) for i, f in enumerate(self.interfaces) if not f.is_boundary]

    def boundary(self):
        return [(i, f) for i, f in enumerate(self.interfaces) if f.is_boundary]

    def dump(self) -> str:
        """Plain-text topology dump, same fields and formatting as the
        reference's MeshTopology.dump (mesh.py:82-103)."""
        out = ["vertex %d %s" % (i, " ".join("%.17g" % c for c in v))
               for i, v in enumerate(self.vertices)]
        out += ["element %d %s %s" % (i, as_shape(e.shape).value, " ".join(str(v) for v in e.verts))
                for i, e in enumerate(self.elements)]
        for i, f in enumerate(self.interfaces):
            r = f.right or (-1, -1)
            out.append("interface %d %d %d %d %d %d %s"
                       % (i, f.left[0], f.left[1], r[0], r[1], f.orientation, f.tag or "-"))
        return "\n".join(out) + "\n"


# --- orientation codes between two parametrisations of a shared face -------

_CORNER_PRM = {1: np.array([[-1.0], [1.0]]),
               2: np.array([[-1.0, -1.0], [1.0, -1.0], [-1.0, 1.0], [1.0, 1.0]])}


def _code_points(code: int, p: np.ndarray) -> np.ndarray:
    """Left face parameters -> right parameters of the same point: edges flip
    on code 1; quad faces: bit 2 swaps axes, bits 1/0 flip the first/second
    (reference orient.py:25-38)."""
    if p.shape[1] == 1:
        return -p if code == 1 else p.copy()
    out = p[:, ::-1].copy() if (code >> 2) & 1 else p.copy()
    if (code >> 1) & 1:
        out[:, 0] = -out[:, 0]
    if code & 1:
        out[:, 1] = -out[:, 1]
    return out


def _corner_maps(fd: int):
    prm = _CORNER_PRM[fd]
    maps = []
    for code in range({1: 2, 2: 8}[fd]):
        m = _code_points(code, prm)
        maps.append(np.array([int(np.argmin(np.abs(prm - r).sum(axis=1))) for r in m]))
    return maps


def _match_codes(lc: np.ndarray, rc: np.ndarray, fd: int, tol: float) -> np.ndarray:
    """First orientation code under which every left corner lands on the
    matching right corner (reference orient.py:75-95), vectorised over faces.
    lc, rc: (nF, ncorner, d) physical corner coordinates."""
    codes = np.full(lc.shape[0], -1, dtype=np.int64)
    for code, jmap in enumerate(_corner_maps(fd)):
        ok = np.all(np.abs(lc - rc[:, jmap, :]).max(axis=2) <= tol, axis=1)
        codes = np.where((codes < 0) & ok, code, codes)
    if np.any(codes < 0):
        raise ValueError("faces do not match geometrically under any orientation")
    return codes


def build_topology(dim: int, verts: np.ndarray, elements: list, tag: str = "dirichlet") -> MeshTopology:
    """Face matching by corner-vertex sets; interior interfaces ordered by
    (left, right), left = first occurrence; boundary faces appended in (e, f)
    order (reference mesh.py:234-265)."""
    verts = np.asarray(verts, dtype=float)
    ef, keys, ncorner = [], [], []
    for e, el in enumerate(elements):
        s = as_shape(el.shape).value
        for f, cv in enumerate(FACE_CORNERS[s]):
            ef.append((e, f))
            ncorner.append(len(cv))
            keys.append(tuple(sorted(el.verts[v] for v in cv)))
    nfaces = len(ef)
    width = max(ncorner)
    kk = np.full((nfaces, width), -1, dtype=np.int64)
    for i, k in enumerate(keys):
        kk[i, :len(k)] = k
    order = np.lexsort(kk.T[::-1])
    ks = kk[order]
    same = np.all(ks[1:] == ks[:-1], axis=1)
    if np.any(same[1:] & same[:-1]):
        raise ValueError("a face is shared by more than two elements")
    first = np.flatnonzero(same)
    li, ri = order[first], order[first + 1]
    swap = li > ri
    li, ri = np.where(swap, ri, li), np.where(swap, li, ri)
    paired = np.zeros(nfaces, dtype=bool)
    paired[li] = True
    paired[ri] = True
    ef_arr = np.asarray(ef, dtype=np.int64)
    scale = max(np.ptp(verts, axis=0).max(), 1.0)
    codes = np.zeros(li.size, dtype=np.int64)
    fd = dim - 1
    if fd > 0 and li.size:
        def corners(idx):
            out = np.empty((idx.size, width, dim))
            for t, i in enumerate(idx):
                e, f = ef[i]
                el = elements[e]
                cv = FACE_CORNERS[as_shape(el.shape).value][f]
                out[t] = verts[[el.verts[v] for v in cv]]
            return out
        codes = _match_codes(corners(li), corners(ri), fd, 1e-10 * scale)
    # interfaces sorted by (left, right); since face ids are (e, f)-ordered,
    # sorting by (li, ri) index is the same order
    o = np.lexsort((ri, li))
    interfaces = [Interface((int(ef_arr[a, 0]), int(ef_arr[a, 1])),
                            (int(ef_arr[b, 0]), int(ef_arr[b, 1])), int(c))
                  for a, b, c in zip(li[o], ri[o], codes[o])]
    for i in np.flatnonzero(~paired):
        interfaces.append(Interface((int(ef_arr[i, 0]), int(ef_arr[i, 1])), None, 0, tag))
    return MeshTopology(dim, verts, list(elements), interfaces)


def _grid_vertices(axes):
    g = np.meshgrid(*axes, indexing="ij")
    return np.stack([a.reshape(-1) for a in g], axis=-1)


def generate_box(dim: int, nx, shape, extent=None, taper: float = 0.0,
                 tag: str = "dirichlet") -> MeshTopology:
    """Structured box mesh, x slowest (reference mesh.py:160-226); TRI splits
    each cell along the low-low / high-high diagonal."""
    shape = as_shape(shape)
    if shape.dim != dim:
        raise ValueError(f"shape {shape.value} is not {dim}-dimensional")
    nxs = (nx,) * dim if isinstance(nx, (int, np.integer)) else tuple(nx)
    if len(nxs) != dim or any(n < 1 for n in nxs):
        raise ValueError("need one positive cell count per axis")
    if extent is None:
        extent = ((-1.0, 1.0),) * dim
    if np.ndim(extent) == 1:
        extent = (tuple(extent),) * dim
    axes = [np.linspace(lo, hi, n + 1) for (lo, hi), n in zip(extent, nxs)]
    verts = _grid_vertices(axes)
    if taper != 0.0:
        lo, hi = extent[-1]
        t = (verts[:, -1] - lo) / (hi - lo)
        verts = verts.copy()
        verts[:, 0] = verts[:, 0] * (1.0 + taper * t)
    shp = [n + 1 for n in nxs]
    els = []
    if dim == 1:
        els = [Element(Shape.SEG, (i, i + 1)) for i in range(nxs[0])]
    elif dim == 2:
        for i in range(nxs[0]):
            for j in range(nxs[1]):
                v00, v10 = i * shp[1] + j, (i + 1) * shp[1] + j
                v11, v01 = (i + 1) * shp[1] + j + 1, i * shp[1] + j + 1
                if shape is Shape.QUAD:
                    els.append(Element(Shape.QUAD, (v00, v10, v11, v01)))
                else:
                    els.append(Element(Shape.TRI, (v00, v10, v11)))
                    els.append(Element(Shape.TRI, (v00, v11, v01)))
    else:
        if shape is not Shape.HEX:
            raise ValueError("3D meshes support hexahedra only")

        def vid(i, j, k):
            return (i * shp[1] + j) * shp[2] + k
        for i in range(nxs[0]):
            for j in range(nxs[1]):
                for k in range(nxs[2]):
                    els.append(Element(Shape.HEX, (
                        vid(i, j, k), vid(i + 1, j, k), vid(i + 1, j + 1, k), vid(i, j + 1, k),
                        vid(i, j, k + 1), vid(i + 1, j, k + 1), vid(i + 1, j + 1, k + 1),
                        vid(i, j + 1, k + 1))))
    if dim == 1:
        raise ValueError("1D meshes are not supported by this build")
    return build_topology(dim, verts, els, tag)


def generate_hybrid(nx: int, rng: np.random.Generator, extent=(0.0, 1.0)) -> MeshTopology:
    """BASELINE config 2 mesh: [0,1]^2 on an nx x nx grid, each cell (x
    slowest) kept as a quad when rng.uniform() < 0.5, otherwise split into two
    counter-clockwise triangles, along the low-low/high-high diagonal when a
    second rng.uniform() < 0.5, else along the other diagonal."""
    lo, hi = extent
    axes = [np.linspace(lo, hi, nx + 1)] * 2
    verts = _grid_vertices(axes)
    els = []
    for i in range(nx):
        for j in range(nx):
            v00, v10 = i * (nx + 1) + j, (i + 1) * (nx + 1) + j
            v11, v01 = (i + 1) * (nx + 1) + j + 1, i * (nx + 1) + j + 1
            if rng.uniform() < 0.5:
                els.append(Element(Shape.QUAD, (v00, v10, v11, v01)))
            elif rng.uniform() < 0.5:
                els.append(Element(Shape.TRI, (v00, v10, v11)))
                els.append(Element(Shape.TRI, (v00, v11, v01)))
            else:
                els.append(Element(Shape.TRI, (v00, v10, v01)))
                els.append(Element(Shape.TRI, (v10, v11, v01)))
    return build_topology(2, verts, els, "dirichlet")


def element_vertex_array(mesh) -> np.ndarray:
    """(n_elements, max_nv) vertex ids, -1 padded."""
    nv = max(len(el.verts) for el in mesh.elements)
    out = np.full((len(mesh.elements), nv), -1, dtype=np.int64)
    for e, el in enumerate(mesh.elements):
        out[e, :len(el.verts)] = el.verts
    return out


def perturb_mesh(mesh, amplitude: float, seed: int = 0) -> MeshTopology:
    """Move interior vertices by uniform(-1,1) * amplitude * h per coordinate,
    h = smallest element extent; boundary vertices fixed (reference
    mesh.py:268-289, same generator draws)."""
    v = np.array(mesh.vertices, dtype=float, copy=True)
    lo, hi = v.min(axis=0), v.max(axis=0)
    scale = (hi - lo).max()
    on_bnd = np.zeros(len(v), dtype=bool)
    for d in range(mesh.dim):
        on_bnd |= np.abs(v[:, d] - lo[d]) < 1e-12 * scale
        on_bnd |= np.abs(v[:, d] - hi[d]) < 1e-12 * scale
    ev = element_vertex_array(mesh)
    h = np.inf
    for e in range(ev.shape[0]):
        ids = ev[e][ev[e] >= 0]
        h = min(h, np.ptp(mesh.vertices[ids], axis=0).min())
    rng = np.random.default_rng(seed)
    disp = rng.uniform(-1.0, 1.0, v.shape) * amplitude * h
    v[~on_bnd] += disp[~on_bnd]
    return MeshTopology(mesh.dim, v, mesh.elements, mesh.interfaces)


@dataclass
class OrderMap:
    """Per-element (n_modes, n_quad) (reference mesh.py:447-465)."""
    n_modes: np.ndarray
    n_quad: np.ndarray

    def pair(self, e: int):
        return int(self.n_modes[e]), int(self.n_quad[e])

    def levels(self):
        return sorted(set(zip(np.asarray(self.n_modes).tolist(), np.asarray(self.n_quad).tolist())))
