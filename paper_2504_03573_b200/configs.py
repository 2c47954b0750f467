"""The five BASELINE.json configurations as seeded synthetic recipes
(SURVEY.md §8d).  One generator `rng = default_rng(seed)` is drawn in this
order: (i) per-cell shape/diagonal choices (cfg2; cfg4: one
rng.uniform() per cube, mesh3d.py), (ii) per-element degrees
P = rng.integers(lo, hi + 1, n_elements), (iii) x = rng.uniform(-1, 1, N_dof)
in DoF order.  cfg1's vertex perturbation uses perturb_mesh's own generator
seeded with the same seed (reference mesh.py:286).  n_modes = P + 1,
n_quad = P + 2 (GLL on quads/hexes, Gauss-Legendre on triangles).

`nx` may be reduced for parity tests; the defaults are the BASELINE sizes.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import OrderMap, Shape, generate_box, generate_hybrid, perturb_mesh
from .mesh3d import generate_hybrid3d

DEFAULT_NX = {"cfg0": 16, "cfg1": 64, "cfg2": 256, "cfg3a": 32, "cfg3b": 32, "cfg4": 48}
DESCRIPTION = {
    "cfg0": "2D conforming quads 16x16, P=4",
    "cfg1": "2D p-nonconforming perturbed quads 64x64, P in {3..6}",
    "cfg2": "2D hybrid quad/tri 256x256, P in {2..8}",
    "cfg3a": "3D hex 32^3, P=6",
    "cfg3b": "3D hex 32^3, P in {4..7}",
    "cfg4": "3D hybrid hex/prism/tet 48^3 cubes, P in {3..6}",
}


@dataclass
class Case:
    name: str
    nx: int
    seed: int
    mesh: object
    order_map: OrderMap
    rng: np.random.Generator

    def draw_x(self, n_dofs: int) -> np.ndarray:
        return self.rng.uniform(-1.0, 1.0, n_dofs)


def build_case(name: str, nx: int | None = None, seed: int = 0) -> Case:
    nx = DEFAULT_NX[name] if nx is None else int(nx)
    rng = np.random.default_rng(seed)
    if name == "cfg0":
        m = generate_box(2, nx, Shape.QUAD, (0.0, 1.0))
        P = np.full(m.n_elements, 4)
    elif name == "cfg1":
        m = perturb_mesh(generate_box(2, nx, Shape.QUAD, (0.0, 1.0)), 0.2, seed=seed)
        P = rng.integers(3, 7, m.n_elements)
    elif name == "cfg2":
        m = generate_hybrid(nx, rng)
        P = rng.integers(2, 9, m.n_elements)
    elif name == "cfg3a":
        m = generate_box(3, nx, Shape.HEX, (0.0, 1.0))
        P = np.full(m.n_elements, 6)
    elif name == "cfg3b":
        m = generate_box(3, nx, Shape.HEX, (0.0, 1.0))
        P = rng.integers(4, 8, m.n_elements)
    elif name == "cfg4":
        m = generate_hybrid3d(nx, rng)
        P = rng.integers(3, 7, m.n_elements)
    else:
        raise KeyError(f"unknown config {name!r}")
    om = OrderMap(np.asarray(P + 1, dtype=np.int64), np.asarray(P + 2, dtype=np.int64))
    return Case(name, nx, seed, m, om, rng)
