"""Generate golden vectors for the SIP-Helmholtz apply by running the REAL
reference (`/root/reference/pkg/src/dgsipg`, imported read-only) in this
container.  The fixtures it writes (`tests/golden/*.npz`) are committed; the GPU
box never reads /root/reference.

Patches applied to the reference (all outside /root/reference):
  P1  tau = max(n_modes_L, n_modes_R)^2 / h   (BASELINE "(P+1)^2/h"), by
      overriding HelmholtzOperator._face_tau (reference sipg.py:351-360);
  P2  shared-trace rule on faces touching a non-GLL (collapsed) side is
      Gauss-Legendre with max(q) points, by replacing the name
      `dgsipg.sipg.shared_trace_rule` (reference trace.py:202-206, imported at
      sipg.py:50 and used at sipg.py:515).
Cases marked "unpatched" use the reference exactly as shipped.

Usage:  python tests/golden/make_golden.py [small|full|all]
"""
from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent


def _import_reference():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import dgsipg  # noqa: F401
    from dgsipg import mesh, polylib, sipg, stdregions, trace
    return mesh, polylib, sipg, stdregions, trace


mesh_m, polylib_m, sipg_m, std_m, trace_m = _import_reference()
Shape = std_m.Shape
BasisKind = polylib_m.BasisKind
QuadKind = polylib_m.QuadKind

_orig_shared_rule = trace_m.shared_trace_rule


def _shared_rule_p2(rule_l, rule_r):
    # P2: Gauss-Legendre with max(q) when either side's rule is not GLL
    if rule_l.kind is QuadKind.GAUSS_LOBATTO and rule_r.kind is QuadKind.GAUSS_LOBATTO:
        return _orig_shared_rule(rule_l, rule_r)
    return polylib_m.quad_rule(QuadKind.GAUSS_LEGENDRE, max(rule_l.n, rule_r.n))


class BaselineTauOperator(sipg_m.HelmholtzOperator):
    """P1: tau = max(n_modes)^2 / h with the reference's own h."""

    def _face_tau(self, itf):
        le, lf = itf.left
        h = self.factors[le].volume / self.factors[le].faces[lf].area
        n = int(self.order_map.n_modes[le])
        if itf.right is not None:
            re_, rf = itf.right
            h = min(h, self.factors[re_].volume / self.factors[re_].faces[rf].area)
            n = max(n, int(self.order_map.n_modes[re_]))
        return float(n * n) / h


# ---------------------------------------------------------------------------
# config recipes (BASELINE.json configs), reference generators


def hybrid_mesh(nx, rng):
    """cfg2 mesh: per cell (x slowest) quad with p=0.5 else two triangles on a
    random diagonal; built with the reference's generic topology builder."""
    axes = [np.linspace(0.0, 1.0, nx + 1)] * 2
    g = np.meshgrid(*axes, indexing="ij")
    verts = np.stack([a.reshape(-1) for a in g], axis=-1)

    def vid(i, j):
        return i * (nx + 1) + j

    els = []
    for i in range(nx):
        for j in range(nx):
            v00, v10, v11, v01 = vid(i, j), vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)
            if rng.uniform() < 0.5:
                els.append(mesh_m.Element(Shape.QUAD, (v00, v10, v11, v01)))
            elif rng.uniform() < 0.5:
                els.append(mesh_m.Element(Shape.TRI, (v00, v10, v11)))
                els.append(mesh_m.Element(Shape.TRI, (v00, v11, v01)))
            else:
                els.append(mesh_m.Element(Shape.TRI, (v00, v10, v01)))
                els.append(mesh_m.Element(Shape.TRI, (v10, v11, v01)))
    return mesh_m._build_topology(2, verts, els, "dirichlet")


def build_case(name, nx, seed):
    rng = np.random.default_rng(seed)
    if name == "cfg0":
        m = mesh_m.generate_box(2, nx, Shape.QUAD, (0.0, 1.0))
        P = np.full(m.n_elements, 4)
    elif name == "cfg1":
        m = mesh_m.perturb_mesh(mesh_m.generate_box(2, nx, Shape.QUAD, (0.0, 1.0)), 0.2, seed=seed)
        P = rng.integers(3, 7, m.n_elements)
    elif name == "cfg2":
        m = hybrid_mesh(nx, rng)
        P = rng.integers(2, 9, m.n_elements)
    elif name == "cfg3a":
        m = mesh_m.generate_box(3, nx, Shape.HEX, (0.0, 1.0))
        P = np.full(m.n_elements, 6)
    elif name == "cfg3b":
        m = mesh_m.generate_box(3, nx, Shape.HEX, (0.0, 1.0))
        P = rng.integers(4, 8, m.n_elements)
    else:
        raise KeyError(name)
    om = mesh_m.OrderMap(np.asarray(P + 1, dtype=int), np.asarray(P + 2, dtype=int))
    return m, om, rng


def make_operator(m, om, patched=True, basis=BasisKind.MODIFIED_MODAL, **kw):
    if patched:
        sipg_m.shared_trace_rule = _shared_rule_p2
        cls = BaselineTauOperator
    else:
        sipg_m.shared_trace_rule = _orig_shared_rule
        cls = sipg_m.HelmholtzOperator
    try:
        op = cls(m, om, basis_kind=basis, batch_width=64, **kw)
    finally:
        sipg_m.shared_trace_rule = _orig_shared_rule
    return op


def maps_of(op, m):
    """Bit-exact maps: topology dump hash, dof offsets, trace slots,
    per-interface strategy (0 gather, 1 p2p, 2 shared, -1 boundary) and the
    transfer permutations of every interface (hashed in interface order)."""
    dump = m.dump()
    code = {"gather": 0, "p2p": 1, "shared": 2}
    strat = np.full(len(m.interfaces), -1, dtype=np.int8)
    iid_of = {itf.left: iid for iid, itf in enumerate(m.interfaces)}
    perms = {}
    for g in op.groups:
        if g.kind == "boundary":
            continue
        for r, el in enumerate(g.left.elems):
            iid = iid_of[(int(el), g.left.face_id)]
            s = g.strategy
            if s == "p2p" and g.left.exp is g.right.exp:
                s = "gather"
            strat[iid] = code[s]
            tl, tr = g.left.transfer, g.right.transfer
            pl = tl.perm if (tl is not None and tl.perm is not None) else np.zeros(0, int)
            pr = tr.perm if (tr is not None and tr.perm is not None) else np.zeros(0, int)
            perms[iid] = np.concatenate([pl, [-1], pr]).astype(np.int64)
    h = hashlib.sha256()
    for iid in sorted(perms):
        h.update(np.int64(iid).tobytes())
        h.update(perms[iid].tobytes())
    slots = np.array([op._slot[(e, f)][0] for e in range(m.n_elements)
                      for f in range(len(op.exps[e].faces))], dtype=np.int64)
    return {
        "dump_sha256": np.frombuffer(hashlib.sha256(dump.encode()).digest(), dtype=np.uint8),
        "dof_off": np.asarray(op._dof_off, dtype=np.int64),
        "trace_slots": slots,
        "itf_strategy": strat,
        "perm_sha256": np.frombuffer(h.digest(), dtype=np.uint8),
    }


SAMPLES = 4096


def checks_of(y, seed=1234):
    """Size-independent digests of y: sampled entries + seeded projections."""
    n = y.size
    idx = np.unique(np.linspace(0, n - 1, min(SAMPLES, n)).astype(np.int64))
    r = np.random.default_rng(seed)
    proj = r.uniform(-1.0, 1.0, (4, n)) @ y
    return {"sample_idx": idx, "sample_y": y[idx], "proj": proj,
            "ymax": np.abs(y).max(), "ynorm": np.linalg.norm(y)}


def run_case(tag, name, nx, seed, patched=True, store_full=True, basis=BasisKind.MODIFIED_MODAL,
             **kw):
    t0 = time.perf_counter()
    m, om, rng = build_case(name, nx, seed)
    op = make_operator(m, om, patched=patched, basis=basis, **kw)
    t1 = time.perf_counter()
    x = rng.uniform(-1.0, 1.0, op.n_dofs)
    y = op.lhs_eval(x)
    t2 = time.perf_counter()
    assert np.all(np.isfinite(y)), f"{tag}: non-finite output"
    rec = {"config": name, "nx": nx, "seed": seed, "patched": int(patched),
           "basis": basis.value, "n_dofs": op.n_dofs, "n_elements": m.n_elements,
           "setup_s": t1 - t0, "apply_s": t2 - t1}
    rec.update({"opt_" + k: v for k, v in kw.items()})
    rec.update(maps_of(op, m))
    rec.update(checks_of(y))
    if store_full:
        rec["x"] = x
        rec["y"] = y
    np.savez_compressed(OUT / f"{tag}.npz", **{k: np.asarray(v) for k, v in rec.items()})
    print(f"{tag}: n_dofs={op.n_dofs} setup={t1-t0:.1f}s apply={t2-t1:.3f}s "
          f"|y|inf={np.abs(y).max():.6g}", flush=True)


SMALL = [
    # tag, config, nx, seed, patched, extra kwargs
    ("cfg0_full", "cfg0", 16, 0, True, {}),
    ("cfg0_n4", "cfg0", 4, 1, True, {}),
    ("cfg1_n6", "cfg1", 6, 2, True, {}),
    ("cfg1_n6_unpatched", "cfg1", 6, 2, False, {}),
    ("cfg2_n6", "cfg2", 6, 3, True, {}),
    ("cfg2_n8", "cfg2", 8, 7, True, {}),
    ("cfg3a_n3", "cfg3a", 3, 4, True, {}),
    ("cfg3b_n3", "cfg3b", 3, 5, True, {}),
    ("cfg3b_n3_unpatched", "cfg3b", 3, 5, False, {}),
    ("cfg1_n5_shared", "cfg1", 5, 6, True, {"strategy": "shared_trace"}),
    ("cfg2_n5_shared", "cfg2", 5, 8, True, {"strategy": "shared_trace"}),
    ("cfg1_n5_traceip", "cfg1", 5, 9, True, {"face_absorb": "trace_iproduct"}),
    ("cfg3b_n2_traceip", "cfg3b", 2, 10, True, {"face_absorb": "trace_iproduct"}),
    ("cfg2_n5_p2pforced", "cfg2", 5, 11, True, {"strategy": "p2p_forced"}),
    ("cfg0_n3_forceinterp", "cfg0", 3, 12, True, {"force_interp": True}),
]

FULL = [
    ("cfg1_full", "cfg1", 64, 0, True, {}),
    ("cfg3a_full", "cfg3a", 32, 0, True, {}),
    ("cfg3b_full", "cfg3b", 32, 0, True, {}),
    ("cfg2_full", "cfg2", 256, 0, True, {}),
]


def main(which):
    if which in ("small", "all"):
        for tag, name, nx, seed, patched, kw in SMALL:
            run_case(tag, name, nx, seed, patched=patched, **kw)
        # reference defaults (LAGRANGE basis, tau_constant=10), unpatched
        run_case("quad_lagrange_default", "cfg1", 4, 13, patched=False,
                 basis=BasisKind.LAGRANGE)
        run_case("hex_lagrange_default", "cfg3b", 2, 14, patched=False,
                 basis=BasisKind.LAGRANGE)
    if which in ("full", "all"):
        for tag, name, nx, seed, patched, kw in FULL:
            run_case(tag, name, nx, seed, patched=patched, store_full=False, **kw)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "small")
