"""x-slab domain decomposition with a one-layer ghost halo.

Phase 1 of the apply is element-local and phase 2 only needs the neighbour's
face data (reference sipg.py:569-592 vs 607-651) — the paper's trace-only
exchange.  In this build a face's neighbour trace is
evaluated from the neighbour's coefficients inside the element kernel, so the
halo a rank needs is the coefficient blocks of the elements across its slab
faces (one layer).  Each rank's local problem is its slab plus that ghost
layer; only owned elements are computed, so every element's output is produced
by exactly one rank with the same arithmetic as on one GPU (bit-identical
results for any rank count).

Slabs are element ranges ordered by centroid x (for the generated boxes x is
the slowest index, so slabs are contiguous element and DoF ranges) and
balanced by the sum-factorised flop estimate of each element.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import Element, MeshTopology, OrderMap, as_shape, build_topology, element_vertex_array


def element_weights(mesh, order_map) -> np.ndarray:
    """Relative cost per element (sum-factorised flops ~ q^(d+1) n)."""
    d = mesh.dim
    n = np.asarray(order_map.n_modes, dtype=float)
    q = np.asarray(order_map.n_quad, dtype=float)
    return q ** (d + 1) * n


def slab_ranges(mesh, order_map, world: int) -> list:
    """Contiguous element ranges [lo, hi) per rank, split along the element
    order (x slowest for generated boxes) with balanced weights."""
    w = element_weights(mesh, order_map)
    cw = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cw, cw[-1] * r / world)))
    cuts.append(len(w))
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def owner_of(ranges) -> np.ndarray:
    n = ranges[-1][1]
    out = np.empty(n, dtype=np.int64)
    for r, (lo, hi) in enumerate(ranges):
        out[lo:hi] = r
    return out


@dataclass
class LocalProblem:
    """A rank's slab plus its ghost layer, as a self-contained mesh.

    local elements = `local_ids` (global ids, ascending); owned ones are
    `local_ids[owned_mask]`; x_local is laid out in local element order, so
    the owned DoFs form the contiguous global slice [dof_lo, dof_hi).
    """
    rank: int
    mesh: MeshTopology
    order_map: OrderMap
    local_ids: np.ndarray
    owned_mask: np.ndarray
    dof_lo: int
    dof_hi: int
    owned_local_dofs: slice          # owned slice of x_local
    recv: dict                       # src rank -> (local dof indices to fill, global dof indices)
    send: dict                       # dst rank -> global dof indices (of owned elements) to send
    boundary_elems: np.ndarray       # local ids of owned elements that touch a ghost


def _dof_offsets(order_map, mesh):
    nm = np.asarray(order_map.n_modes)
    shapes = [as_shape(el.shape).value for el in mesh.elements]
    nc = np.array([n * (n + 1) // 2 if s == "tri" else n ** mesh.dim for s, n in zip(shapes, nm)])
    off = np.zeros(len(nc) + 1, dtype=np.int64)
    off[1:] = np.cumsum(nc)
    return off


def neighbours(mesh) -> list:
    """Element adjacency from the interior interfaces."""
    nb = [[] for _ in range(len(mesh.elements))]
    for itf in mesh.interfaces:
        if itf.right is not None:
            a, b = itf.left[0], itf.right[0]
            nb[a].append(b)
            nb[b].append(a)
    return nb


def local_problem(mesh, order_map, ranges, rank: int, adjacency=None) -> LocalProblem:
    """Build rank `rank`'s local mesh (owned slab + one ghost layer)."""
    lo, hi = ranges[rank]
    owner = owner_of(ranges)
    adj = adjacency if adjacency is not None else neighbours(mesh)
    ghosts = sorted({b for a in range(lo, hi) for b in adj[a] if not (lo <= b < hi)})
    local_ids = np.array(sorted(set(range(lo, hi)) | set(ghosts)), dtype=np.int64)
    owned_mask = (local_ids >= lo) & (local_ids < hi)
    # sub-mesh: keep global vertex coordinates, renumber vertices densely
    ev = element_vertex_array(mesh)[local_ids]
    used = np.unique(ev[ev >= 0])
    vmap = -np.ones(len(mesh.vertices), dtype=np.int64)
    vmap[used] = np.arange(used.size)
    els = [Element(mesh.elements[g].shape, tuple(int(vmap[v]) for v in mesh.elements[g].verts)) for g in local_ids]
    sub = build_topology(mesh.dim, np.asarray(mesh.vertices)[used], els, "dirichlet")
    om = OrderMap(np.asarray(order_map.n_modes)[local_ids], np.asarray(order_map.n_quad)[local_ids])
    goff = _dof_offsets(order_map, mesh)
    loff = _dof_offsets(om, sub)
    owned_local = np.flatnonzero(owned_mask)
    assert np.all(np.diff(owned_local) == 1), "owned elements must be contiguous in local order"
    o_lo, o_hi = int(loff[owned_local[0]]), int(loff[owned_local[-1] + 1])
    recv = {}
    for li, g in enumerate(local_ids):
        if owned_mask[li]:
            continue
        src = int(owner[g])
        ldofs = np.arange(loff[li], loff[li + 1])
        gdofs = np.arange(goff[g], goff[g + 1])
        a, b = recv.get(src, (np.zeros(0, np.int64), np.zeros(0, np.int64)))
        recv[src] = (np.concatenate([a, ldofs]), np.concatenate([b, gdofs]))
    send = {}
    for dst in range(len(ranges)):
        if dst == rank:
            continue
        dlo, dhi = ranges[dst]
        need = sorted({b for a in range(dlo, dhi) for b in adj[a] if lo <= b < hi})
        if need:
            send[dst] = np.concatenate([np.arange(goff[g], goff[g + 1]) for g in need])
    lid = {int(g): i for i, g in enumerate(local_ids)}
    bnd = sorted({lid[a] for a in range(lo, hi) if any(not (lo <= b < hi) for b in adj[a])})
    return LocalProblem(rank, sub, om, local_ids, owned_mask, int(goff[lo]), int(goff[hi]),
                        slice(o_lo, o_hi), recv, send, np.asarray(bnd, dtype=np.int64))


def stack_box_config(name: str, world: int, nx=None, seed: int = 0):
    """Weak-scaling workload: `world` copies of a BASELINE config box stacked
    along x (x in [0, world]); seeded draws over the whole stacked mesh in the
    config's order (shape choices, degrees, x).  world = 1 is the config."""
    from . import configs
    from .mesh import Shape, generate_box, generate_hybrid, perturb_mesh
    nx = configs.DEFAULT_NX[name] if nx is None else int(nx)
    rng = np.random.default_rng(seed)
    if name in ("cfg3a", "cfg3b"):
        m = generate_box(3, (nx * world, nx, nx), Shape.HEX, ((0.0, float(world)), (0.0, 1.0), (0.0, 1.0)))
        P = np.full(m.n_elements, 6) if name == "cfg3a" else rng.integers(4, 8, m.n_elements)
    elif name in ("cfg0", "cfg1"):
        m = generate_box(2, (nx * world, nx), Shape.QUAD, ((0.0, float(world)), (0.0, 1.0)))
        if name == "cfg1":
            m = perturb_mesh(m, 0.2, seed=seed)
        P = np.full(m.n_elements, 4) if name == "cfg0" else rng.integers(3, 7, m.n_elements)
    elif name == "cfg2":
        if world != 1:
            raise ValueError("cfg2 weak scaling: use the square config per rank")
        m = generate_hybrid(nx, rng)
        P = rng.integers(2, 9, m.n_elements)
    elif name == "cfg4":
        from .mesh3d import generate_hybrid3d
        m = generate_hybrid3d((nx * world, nx, nx), rng, ((0.0, float(world)), (0.0, 1.0), (0.0, 1.0)))
        P = rng.integers(3, 7, m.n_elements)
    else:
        raise KeyError(name)
    om = OrderMap(np.asarray(P + 1, dtype=np.int64), np.asarray(P + 2, dtype=np.int64))
    return m, om, rng
