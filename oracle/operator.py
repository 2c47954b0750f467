"""ORACLE (test infrastructure only) — the SIP-Helmholtz operator apply.

Restates reference pkg/src/dgsipg/sipg.py: plan construction (234-554) and the
two-phase apply `lhs_eval` (558-602) with `_phase2` (607-651), `_trace_eval`
(653-661), `_absorb` (663-677) and `_final_sweep` (679-693).  Elements of one
expansion form one batch (the reference's batch_width only regroups columns;
its output is bit-identical for every width).
"""
from __future__ import annotations

import time

import numpy as np

from . import geometry as geo
from . import polylib as pl
from .elements import DIM, expansion


def _sv(x):
    return getattr(x, "value", x)


class _Side:
    pass


class OracleOperator:
    """y = (lambda M + L_SIP) x on a duck-typed mesh (dim, vertices, elements
    with .shape/.verts, interfaces with .left/.right/.orientation/.tag) and an
    order map (n_modes, n_quad arrays)."""

    def __init__(self, mesh, order_map, *, basis_kind="modified_modal", rule_kinds=None,
                 lambda_=1.0, tau_constant=10.0, strategy="p2p", face_absorb="auto",
                 force_interp=False, p_geom=1, tau_rule="baseline", shared_rule="patched"):
        if strategy not in ("p2p", "p2p_forced", "shared_trace"):
            raise ValueError(strategy)
        if face_absorb not in ("auto", "trace_iproduct"):
            raise ValueError(face_absorb)
        self.mesh, self.lam, self.C = mesh, float(lambda_), float(tau_constant)
        self.strategy, self.face_absorb, self.force_interp = strategy, face_absorb, force_interp
        self.p_geom, self.tau_rule, self.shared_patched = p_geom, tau_rule, shared_rule == "patched"
        self.dim = mesh.dim
        kind = _sv(basis_kind)
        rk = None if rule_kinds is None else (
            _sv(rule_kinds) if not isinstance(rule_kinds, (tuple, list))
            else tuple(_sv(k) for k in rule_kinds))
        nel = len(mesh.elements)
        self.nm = np.asarray(order_map.n_modes, dtype=int)
        self.nq = np.asarray(order_map.n_quad, dtype=int)
        self.shapes = [_sv(el.shape) for el in mesh.elements]
        self.exps = [expansion(self.shapes[e], kind, int(self.nm[e]), int(self.nq[e]), rk)
                     for e in range(nel)]
        verts = np.asarray(mesh.vertices, dtype=float)
        self.ev = [verts[list(el.verts)] for el in mesh.elements]
        # classes in first-appearance order (sipg.py:302-349)
        self.classes = {}
        for e, ex in enumerate(self.exps):
            self.classes.setdefault(id(ex), []).append(e)
        self.col = np.zeros(nel, dtype=int)
        self.cls_of = [None] * nel
        self.vol = np.zeros(nel)
        self.efac = {}
        self.ffac = {}
        for cid, ids in self.classes.items():
            ex = self.exps[ids[0]]
            vb = np.stack([self.ev[e] for e in ids])
            ef = geo.element_factors(ex.shape, vb, ex)
            self.efac[cid] = ef
            for c, e in enumerate(ids):
                self.col[e], self.cls_of[e] = c, cid
                self.vol[e] = ef["volume"][c]
            for f in range(len(ex.faces)):
                prm = geo.tensor_params(ex.face_pts(f))
                w = None
                if ex.faces[f].run:
                    w = ex.rules[ex.faces[f].run[0]][1]
                    for a in ex.faces[f].run[1:]:
                        w = np.multiply.outer(w, ex.rules[a][1]).reshape(-1)
                self.ffac[(cid, f)] = geo.face_factors(ex.shape, vb, ex, f, prm, w)
        self.dof_off = np.zeros(nel + 1, dtype=np.int64)
        for e in range(nel):
            self.dof_off[e + 1] = self.dof_off[e] + self.exps[e].n_coeffs
        self.n_dofs = int(self.dof_off[-1])
        # trace slots, per element per face contiguous (sipg.py:288-296)
        self.slot = {}
        off = 0
        for e, ex in enumerate(self.exps):
            for f in range(len(ex.faces)):
                self.slot[(e, f)] = off
                off += ex.face_npts(f)
        self.trace_len = off
        # volume metric per class (sipg.py:210-216, 327-333)
        self.G = {}
        for cid, ids in self.classes.items():
            ex = self.exps[ids[0]]
            dx = self.efac[cid]["dxidx"]                 # (W, d, d, p)
            cj = ex.collapse_jac()
            if cj is not None:
                dx = np.einsum("kmp,wmjp->wkjp", cj, dx)
            self.G[cid] = np.ascontiguousarray(dx.transpose(1, 2, 3, 0))   # (d, d, p, W)
        self._build_groups()
        self.timers = {"phase1": 0.0, "phase2": 0.0, "total": 0.0, "applies": 0}

    # -- setup -----------------------------------------------------------------
    def _fac(self, e, f):
        ff = self.ffac[(self.cls_of[e], f)]
        c = self.col[e]
        return {k: v[c] for k, v in ff.items()}

    def _tau(self, itf):
        """sipg.py:351-360; tau_rule="baseline" is patch P1."""
        le, lf = itf.left
        h = self.vol[le] / self._fac(le, lf)["area"]
        nmax, pmax = self.nm[le], self.nm[le] - 1
        if itf.right is not None:
            re_, rf = itf.right
            h = min(h, self.vol[re_] / self._fac(re_, rf)["area"])
            nmax, pmax = max(nmax, self.nm[re_]), max(pmax, self.nm[re_] - 1)
        if self.tau_rule == "baseline":
            return float(nmax * nmax) / h
        return self.C * max(pmax, 1) ** 2 / h

    def _own_side(self, exp, f, elems):
        """Side data on the element's own face grid (sipg.py:422-446, 475-481)."""
        s = _Side()
        s.exp, s.f, s.elems = exp, f, np.asarray(elems)
        prm = geo.tensor_params(exp.face_pts(f))
        facs = [self._fac(e, f) for e in elems]
        s.swj = np.stack([ff["swj"] for ff in facs])
        dx = np.stack([ff["dxidx"] for ff in facs])
        nrm = np.stack([np.broadcast_to(ff["normal"], (exp.dim, prm.shape[0])) for ff in facs])
        s.gn = geo.side_gn(exp, f, dx, nrm, prm)
        s.B = exp.face_table(f, prm)
        s.D = [exp.face_table(f, prm, k) for k in range(exp.dim)]
        s.dofs = np.stack([np.arange(self.dof_off[e], self.dof_off[e + 1]) for e in elems])
        s.buf = np.stack([np.arange(self.slot[(e, f)], self.slot[(e, f)] + exp.face_npts(f))
                          for e in elems])
        vi = exp.face_vol_idx(f)
        s.pv = None if (vi is None or self.face_absorb == "trace_iproduct") else vi
        s.transfer = None
        return s

    def _build_groups(self):
        """sipg.py:382-420 (+ boundary 458-473, interior 483-554)."""
        mesh = self.mesh
        buckets = {}
        self.strategy_of = {}
        self.certificates = []
        for iid, itf in enumerate(mesh.interfaces):
            le, lf = itf.left
            expl = self.exps[le]
            if itf.right is None:
                buckets.setdefault(("b", id(expl), lf, itf.tag), []).append(itf)
                continue
            re_, rf = itf.right
            expr = self.exps[re_]
            conforming = expl is expr
            if conforming:
                strat = "shared" if self.face_absorb == "trace_iproduct" else "gather"
            else:
                deformed = (not self._fac(le, lf)["n_const"]) or (not self._fac(re_, rf)["n_const"])
                al, ar = expl.faces[lf].run[0], expr.faces[rf].run[0]
                cert = geo.certify((expl.n, expl.nq[al], expl.kinds[al]),
                                   (expr.n, expr.nq[ar], expr.kinds[ar]), self.p_geom, deformed)
                if self.face_absorb == "trace_iproduct" or self.strategy == "shared_trace":
                    strat = "shared"
                elif self.strategy == "p2p_forced":
                    strat = "p2p"
                else:
                    strat = "p2p" if cert[0] else "shared"
                self.certificates.append((iid, cert, strat))
            self.strategy_of[iid] = strat
            key = ("i", id(expl), lf, id(expr), rf, itf.orientation,
                   "p2p" if strat == "gather" else strat)
            buckets.setdefault(key, []).append(itf)
        self.groups = []
        for key, items in buckets.items():
            if key[0] == "b":
                e0, f0 = items[0].left
                g = {"kind": "boundary", "tau": np.array([[self._tau(t)] for t in items]), "tag": key[3]}
                g["left"] = self._own_side(self.exps[e0], f0, [t.left[0] for t in items])
                self.groups.append(g)
            else:
                self.groups.append(self._interior(key[-1], items))

    def _interior(self, strat, items):
        it0 = items[0]
        (le0, lf), (re0, rf) = it0.left, it0.right
        expl, expr = self.exps[le0], self.exps[re0]
        code = it0.orientation
        el = [t.left[0] for t in items]
        er = [t.right[0] for t in items]
        g = {"kind": "interior", "strategy": strat,
             "tau": np.array([[self._tau(t)] for t in items])}
        pts_l, pts_r = expl.face_pts(lf), expr.face_pts(rf)
        fd = len(pts_l)
        left = self._own_side(expl, lf, el)
        right = self._own_side(expr, rf, er)
        if strat == "p2p":
            left.transfer = geo.transfer(pts_r, pts_l, code)
            right.transfer = geo.transfer(pts_l, pts_r, geo.inverse_code(code, fd))
            if self.force_interp:
                left.transfer = geo.densify(left.transfer)
                right.transfer = geo.densify(right.transfer)
            g["left"], g["right"] = left, right
            return g
        # shared trace: one grid, one metric, one normal (sipg.py:513-554)
        swap = fd == 2 and (code >> 2) & 1
        rules = []
        for k in range(fd):
            al = expl.faces[lf].run[k]
            ar = expr.faces[rf].run[(1 - k) if swap else k]
            rules.append(geo.shared_rule(expl.kinds[al], expl.nq[al], expr.kinds[ar], expr.nq[ar],
                                         self.shared_patched))
        t_axes = tuple(pl.rule(k, q)[0] for k, q in rules)
        wt = pl.rule(*rules[0])[1] if fd else np.ones(1)
        for r in rules[1:]:
            wt = np.multiply.outer(wt, pl.rule(*r)[1]).reshape(-1)
        prm_t = geo.tensor_params(t_axes)
        prm_tr = geo.apply_code(code, prm_t)
        left.B, left.D = expl.face_table(lf, prm_t), [expl.face_table(lf, prm_t, k) for k in range(expl.dim)]
        right.B, right.D = expr.face_table(rf, prm_tr), [expr.face_table(rf, prm_tr, k) for k in range(expr.dim)]
        vl = np.stack([self.ev[e] for e in el])
        vr = np.stack([self.ev[e] for e in er])
        ffl = geo.face_factors(expl.shape, vl, expl, lf, prm_t, wt)
        ffr = geo.face_factors(expr.shape, vr, expr, rf, prm_tr, None)
        n_sh = np.broadcast_to(ffl["normal"], (len(el), expl.dim, prm_t.shape[0]))
        left.swj = right.swj = ffl["swj"]
        left.gn = geo.side_gn(expl, lf, ffl["dxidx"], n_sh, prm_t)
        right.gn = geo.side_gn(expr, rf, ffr["dxidx"], -n_sh, prm_tr)
        left.pv = right.pv = None
        g["left"], g["right"] = left, right
        return g

    # -- apply -------------------------------------------------------------------
    def lhs_eval(self, x):
        """sipg.py:558-602."""
        x = np.asarray(x, dtype=float)
        if x.shape != (self.n_dofs,):
            raise ValueError(f"expected a vector of length {self.n_dofs}")
        t0 = time.perf_counter()
        out = np.zeros(self.n_dofs)
        bu = np.zeros(self.trace_len)
        bg = np.zeros(self.trace_len)
        lam = self.lam
        self._u = {}
        for cid, ids in self.classes.items():
            ex = self.exps[ids[0]]
            d = ex.dim
            ids_a = np.asarray(ids)
            dof_idx = (self.dof_off[ids_a][None, :] + np.arange(ex.n_coeffs)[:, None])
            G = self.G[cid]
            jw = self.efac[cid]["jw"].T                    # (n_phys, W)
            u = ex.bwd(x[dof_idx])
            du = ex.deriv(u)
            dux = [sum(G[k, m] * du[k] for k in range(d)) for m in range(d)]
            acc = ex.iprod(u * (lam * jw)) if lam != 0.0 else 0.0
            for k in range(d):
                flux = sum(G[k, m] * dux[m] for m in range(d)) * jw
                term = ex.iprod_d(k, flux)
                acc = term if isinstance(acc, float) else acc + term
            out[dof_idx] = acc
            for f in range(len(ex.faces)):
                nrm = self.ffac[(cid, f)]["normal"]        # (W, d, 1|nf)
                nf = ex.face_npts(f)
                nrm = np.broadcast_to(nrm, (len(ids), d, nf)).transpose(1, 2, 0)
                uf = ex.face_vals(f, u)
                gf = sum(nrm[m] * ex.face_vals(f, dux[m]) for m in range(d))
                slots = np.array([self.slot[(e, f)] for e in ids])[None, :] + np.arange(nf)[:, None]
                bu[slots] = uf
                bg[slots] = gf
        t1 = time.perf_counter()
        pacc = self._phase2(x, bu, bg, out)
        self._final_sweep(out, pacc)
        t2 = time.perf_counter()
        self.timers["phase1"] += t1 - t0
        self.timers["phase2"] += t2 - t1
        self.timers["total"] += t2 - t0
        self.timers["applies"] += 1
        return out

    __call__ = lhs_eval

    def _phase2(self, x, bu, bg, out):
        """sipg.py:607-651."""
        pacc = {cid: np.zeros((1 + self.dim, self.exps[ids[0]].n_phys, len(ids)))
                for cid, ids in self.classes.items()}
        for g in self.groups:
            L = g["left"]
            if g["kind"] == "boundary":
                self._absorb(L, g["tau"], 2.0 * bu[L.buf], bg[L.buf], out, pacc)
                continue
            R = g["right"]
            if g["strategy"] == "p2p":
                ul, gl, ur, gr = bu[L.buf], bg[L.buf], bu[R.buf], bg[R.buf]
                url, grl = L.transfer.apply(ur), L.transfer.apply(gr)
                self._absorb(L, g["tau"], ul - url, 0.5 * (gl - grl), out, pacc)
                ulr, glr = R.transfer.apply(ul), R.transfer.apply(gl)
                self._absorb(R, g["tau"], ur - ulr, 0.5 * (gr - glr), out, pacc)
            else:
                ult, glt = self._trace_eval(x, L)
                urt, grt = self._trace_eval(x, R)
                j = ult - urt
                c = 0.5 * (glt - grt)
                self._absorb(L, g["tau"], j, c, out, pacc)
                self._absorb(R, g["tau"], -j, -c, out, pacc)
        return pacc

    @staticmethod
    def _trace_eval(x, s):
        """sipg.py:653-661."""
        uh = x[s.dofs]
        u = uh @ s.B.T
        gn = s.gn[0] * (uh @ s.D[0].T)
        for k in range(1, s.exp.dim):
            gn += s.gn[k] * (uh @ s.D[k].T)
        return u, gn

    def _absorb(self, s, tau, jump, avg, out, pacc, sign=1.0):
        """sipg.py:663-677."""
        fv = (tau * jump - avg) * s.swj * sign
        fd = (-0.5 * sign) * jump * s.swj
        if s.pv is not None and pacc is not None:
            cls = self.cls_of[int(s.elems[0])]
            cols = self.col[s.elems]
            p = pacc[cls]
            p[0][s.pv[None, :], cols[:, None]] += fv
            for k in range(s.exp.dim):
                p[1 + k][s.pv[None, :], cols[:, None]] += fd * s.gn[k]
            return
        contrib = fv @ s.B
        for k in range(s.exp.dim):
            contrib += (fd * s.gn[k]) @ s.D[k]
        out[s.dofs] += contrib

    def _final_sweep(self, out, pacc):
        """sipg.py:679-693."""
        for cid, ids in self.classes.items():
            ex = self.exps[ids[0]]
            blk = pacc[cid]
            terms = ex.iprod(blk[0])
            for k in range(ex.dim):
                terms += ex.iprod_d(k, blk[1 + k])
            dof_idx = (self.dof_off[np.asarray(ids)][None, :] + np.arange(ex.n_coeffs)[:, None])
            out[dof_idx] += terms

    # -- right-hand side and error ----------------------------------------

    def rhs_assemble(self, case, bcs):
        """sipg.py:697-718: b = -(v, f) per class, then on every boundary group the absorb of the
        mirror ghost's jump = -2 g and average 0 with sign -1, straight into b (no final sweep)."""
        b = np.zeros(self.n_dofs)
        for cid, ids in self.classes.items():
            ex = self.exps[ids[0]]
            ids_a = np.asarray(ids)
            xs = self.efac[cid]["x"].transpose(2, 1, 0)               # (d, n_phys, W)
            dof_idx = self.dof_off[ids_a][None, :] + np.arange(ex.n_coeffs)[:, None]
            b[dof_idx] = -ex.iprod(case.forcing(xs) * self.efac[cid]["jw"].T)
        for g in self.groups:
            if g["kind"] != "boundary":
                continue
            if g["tag"] not in bcs:
                raise KeyError(f"no boundary condition for tag {g['tag']!r}")
            L = g["left"]
            xf = [self._fac(int(e), L.f)["x"] for e in L.elems]           # (nf, d) each
            gv = np.stack([bcs[g["tag"]](x.T) for x in xf])
            self._absorb(L, g["tau"], -2.0 * gv, 0.0 * gv, b, None, -1.0)
        return b

    def l2_error(self, x, exact):
        """sipg.py:720-741: per element on rules with 2 extra points per direction."""
        x = np.asarray(x, dtype=float)
        err2 = 0.0
        for cid, ids in self.classes.items():
            ex = self.exps[ids[0]]
            fine = expansion(ex.shape, ex.kind, ex.n, tuple(q + 2 for q in ex.nq), ex.kinds)
            ids_a = np.asarray(ids)
            ef = geo.element_factors(ex.shape, np.stack([self.ev[e] for e in ids]), fine)
            dof_idx = self.dof_off[ids_a][None, :] + np.arange(ex.n_coeffs)[:, None]
            diff = fine.bwd(x[dof_idx]) - exact(ef["x"].transpose(2, 1, 0))
            err2 += float((diff * diff * ef["jw"].T).sum())
        return float(np.sqrt(err2))
