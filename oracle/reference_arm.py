"""ORACLE / BENCH INFRASTRUCTURE ONLY — the reference's own CPU apply, timed for `bench.py --impl
reference` and the CPU baseline.  Never used by the product path.

The reference (`dgsipg`, pure Python + numpy) is installed unmodified into `baseline/_ref` by the
recipe in DESIGN.md (`pip install --no-index --no-build-isolation --no-deps --target baseline/_ref
<copy of /root/reference/pkg>`; git-ignored, travels to the GPU box).  The BASELINE configuration
needs two patches, applied here from outside the package exactly as tests/golden/make_golden.py
does: P1 tau = max(n_modes)^2 / h (subclass override of `_face_tau`, reference
sipg.py:351-360) and P2 the Gauss-Legendre shared-trace rule on faces touching a collapsed side
(name replacement of `dgsipg.sipg.shared_trace_rule`, sipg.py:515).  Config 4 has no reference
(no prism / tet): callers fall back to the oracle port there.
"""
from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
CANDIDATES = [ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")]


def load():
    """Import the installed reference package; None when it is absent."""
    for p in CANDIDATES:
        if (p / "dgsipg" / "sipg.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            import dgsipg.mesh
            import dgsipg.polylib
            import dgsipg.sipg
            import dgsipg.trace
            return dgsipg, p
    return None, None


def _patched_operator(pkg):
    sipg_m, polylib_m, trace_m = pkg.sipg, pkg.polylib, pkg.trace
    orig = trace_m.shared_trace_rule
    QK = polylib_m.QuadKind

    def shared_rule_p2(rl, rr):
        if rl.kind is QK.GAUSS_LOBATTO and rr.kind is QK.GAUSS_LOBATTO:
            return orig(rl, rr)
        return polylib_m.quad_rule(QK.GAUSS_LEGENDRE, max(rl.n, rr.n))

    class BaselineTau(sipg_m.HelmholtzOperator):
        def _face_tau(self, itf):
            le, lf = itf.left
            h = self.factors[le].volume / self.factors[le].faces[lf].area
            n = int(self.order_map.n_modes[le])
            if itf.right is not None:
                re_, rf = itf.right
                h = min(h, self.factors[re_].volume / self.factors[re_].faces[rf].area)
                n = max(n, int(self.order_map.n_modes[re_]))
            return float(n * n) / h

    def make(m, om, batch_width):
        sipg_m.shared_trace_rule = shared_rule_p2
        try:
            return BaselineTau(m, om, basis_kind=polylib_m.BasisKind.MODIFIED_MODAL, batch_width=batch_width)
        finally:
            sipg_m.shared_trace_rule = orig
    return make


def sample_case(pkg, name):
    """A bounded sample of config `name` built with the reference's own generators and the
    BASELINE recipe (seed 0): the full mesh for cfg0 / cfg1, a 64^2 cell grid for cfg2 (the full
    256^2 setup alone takes ~4 min in the reference), the first x-slab of 1/8 of the cube for
    cfg3a / cfg3b.  Returns (mesh, order_map, x, description)."""
    mesh_m, Shape = pkg.mesh, pkg.stdregions.Shape
    rng = np.random.default_rng(0)
    if name == "cfg0":
        m = mesh_m.generate_box(2, 16, Shape.QUAD, (0.0, 1.0))
        P = np.full(m.n_elements, 4)
        desc = "cfg0 full mesh (16^2 quads)"
    elif name == "cfg1":
        m = mesh_m.perturb_mesh(mesh_m.generate_box(2, 64, Shape.QUAD, (0.0, 1.0)), 0.2, seed=0)
        P = rng.integers(3, 7, m.n_elements)
        desc = "cfg1 full mesh (64^2 perturbed quads)"
    elif name == "cfg2":
        nx = 64
        axes = np.linspace(0.0, 1.0, nx + 1)
        g = np.meshgrid(axes, axes, indexing="ij")
        verts = np.stack([a.reshape(-1) for a in g], axis=-1)
        els = []
        for i in range(nx):
            for j in range(nx):
                v00, v10, v11, v01 = i * (nx + 1) + j, (i + 1) * (nx + 1) + j, (i + 1) * (nx + 1) + j + 1, \
                    i * (nx + 1) + j + 1
                if rng.uniform() < 0.5:
                    els.append(mesh_m.Element(Shape.QUAD, (v00, v10, v11, v01)))
                elif rng.uniform() < 0.5:
                    els += [mesh_m.Element(Shape.TRI, (v00, v10, v11)), mesh_m.Element(Shape.TRI, (v00, v11, v01))]
                else:
                    els += [mesh_m.Element(Shape.TRI, (v00, v10, v01)), mesh_m.Element(Shape.TRI, (v10, v11, v01))]
        m = mesh_m._build_topology(2, verts, els, "dirichlet")
        P = rng.integers(2, 9, m.n_elements)
        desc = "cfg2 recipe on a 64^2 cell grid (1/16 of the 256^2 cells)"
    elif name in ("cfg3a", "cfg3b"):
        m = mesh_m.generate_box(3, (4, 32, 32), Shape.HEX, ((0.0, 0.125), (0.0, 1.0), (0.0, 1.0)))
        P = np.full(m.n_elements, 6) if name == "cfg3a" else rng.integers(4, 8, 32 ** 3)[:m.n_elements]
        desc = f"{name} x-slab 4x32x32 (4096 of 32768 elements)"
    else:
        raise KeyError(name)
    om = mesh_m.OrderMap(np.asarray(P + 1, dtype=int), np.asarray(P + 2, dtype=int))
    return m, om, desc


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def time_reference(name, steps, warmup, batch_widths=(64, 4)):
    """Median / mean apply time of the patched reference on the sample, per batch width
    (64 = its fastest, bit-identical output; 4 = its default).  Returns dict or None."""
    pkg, path = load()
    if pkg is None:
        return None
    import dgsipg.stdregions  # noqa: F401
    m, om, desc = sample_case(pkg, name)
    make = _patched_operator(pkg)
    out = {"sample": desc, "path": str(path), "by_width": {}}
    for w in batch_widths:
        t0 = time.perf_counter()
        op = make(m, om, w)
        setup = time.perf_counter() - t0
        x = np.random.default_rng(0).uniform(-1.0, 1.0, op.n_dofs)
        for _ in range(warmup):
            op.lhs_eval(x)
        ts = []
        for _ in range(steps):
            t1 = time.perf_counter()
            op.lhs_eval(x)
            ts.append(time.perf_counter() - t1)
        out["by_width"][w] = {"n_dofs": op.n_dofs, "mean_s": float(np.mean(ts)), "setup_s": setup}
        steps = max(3, steps // 4)     # the slower widths: fewer steps, same sample
        warmup = 1
    return out


def threads() -> int:
    return int(os.environ.get("OPENBLAS_NUM_THREADS") or os.cpu_count() or 1)
