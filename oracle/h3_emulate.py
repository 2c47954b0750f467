"""ORACLE (test infrastructure only) — CPU emulation of the config-4 kernels (csrc/sipg_h3.cuh) on a
flattened plan3d / halo3d plan: same stages, same tables, same published-trace layout, per element
in numpy.  Separates plan-builder bugs from kernel bugs, and lets the multi-rank trace-halo path run
on CPU (tests/test_partition3d.py: publish, exchange over gloo, apply)."""
import numpy as np

from paper_2504_03573_b200.plan3d import (CD3_ELEM_OFF, CD3_COUNT, CD3_N, CD3_NC, CD3_Q, CD3_SHAPE, CD3_T_A,
                                          CD3_T_B, CD3_T_C, CD3_T_D, CD3_T_E, CD3_T_PTS, CD3_T_W, FACES)

NAMES = {0: "hex", 1: "prism", 2: "tet"}


def chain(S, e0, e1, e2):
    c = dict(c00=1.0, c01=0.0, c02=0.0, c11=1.0, c12=0.0)
    if S == 1:
        c["c00"] = 2 / (1 - e2)
        c["c02"] = (1 + e0) / (1 - e2)
    elif S == 2:
        r2 = 1 / (1 - e2)
        r12 = r2 / (1 - e1)
        c.update(c00=4 * r12, c01=2 * (1 + e0) * r12, c02=2 * (1 + e0) * r12, c11=2 * r2, c12=(1 + e1) * r2)
    return c


def tri_groups(N, tet):
    gof = []
    for i in range(N):
        for j in range(N - i):
            gof.append(1 if (i == 0 and j == 1) else (0 if i == 0 else (2 if i == 1 else i + 1)))
    if tet:
        gof.append(1)
    coff, mofr = [], []
    if tet:
        r = 0
        m = 0
        for i in range(N):
            for j in range(N - i):
                d = max(i + j, 1)
                coff.append(r)
                mofr += [m] * (N - d)
                r += N - d
                m += 1
        coff.append(r)
        mofr.append(m)
        coff.append(r + 1)
    return np.array(gof), coff, np.array(mofr)


def slot_map(T, sl, Q):
    """Dense nt x q^2 matrix of a slot's trace map (None: identity)."""
    mk, nt = int(sl["mkind"]), int(sl["nt"])
    if mk == 0:
        return None
    if mk == 2:
        return T[sl["moff"]:sl["moff"] + nt * Q * Q].reshape(nt, Q * Q)
    nab = int(sl["nab"])
    n1, n2, swap = nab & 255, (nab >> 8) & 255, (nab >> 16) & 1
    if mk == 3:       # row map: M[(pa, pb), own(i_par, i_perp)] = X[pb, pa, i_par] Y[pb, i_perp]
        X = T[sl["moff"]:sl["moff"] + n2 * n1 * Q].reshape(n2, n1, Q)
        Y = T[sl["moff2"]:sl["moff2"] + n2 * Q].reshape(n2, Q)
        M4 = np.einsum("bai,bj->abij", X, Y)            # (pa, pb, i_par, i_perp)
        if swap == 0:                                    # perp = own axis 0
            M4 = M4.transpose(0, 1, 3, 2)
        return M4.reshape(nt, Q * Q)
    X = T[sl["moff"]:sl["moff"] + n1 * Q].reshape(n1, Q)
    Y = T[sl["moff2"]:sl["moff2"] + n2 * Q].reshape(n2, Q)
    M4 = np.einsum("ra,sb->rsab", X, Y)                  # (r1, r2, ia, ib)
    if swap:
        M4 = M4.transpose(1, 0, 2, 3)                    # p = r2 n1 + r1
    return M4.reshape(nt, Q * Q)


def phi_matrix(pb, c):
    """Dense Phi (Q^3 x NC) of class c from the staged tables (applying bwd to unit vectors)."""
    cd = pb.class_desc[c]
    S, N, Q, NC = cd[CD3_SHAPE], cd[CD3_N], cd[CD3_Q], cd[CD3_NC]
    T = pb.tables
    NG = N + 1
    if S == 0:
        V = T[cd[CD3_T_A]:cd[CD3_T_A] + Q * N].reshape(Q, N)
        return np.einsum("ai,bj,ck->abcijk", V, V, V).reshape(Q ** 3, N ** 3)
    gof, coff, mofr = tri_groups(N, S == 2)
    A = T[cd[CD3_T_A]:cd[CD3_T_A] + Q * NG].reshape(Q, NG)
    NPM = len(gof)
    B = T[cd[CD3_T_B]:cd[CD3_T_B] + NPM * Q].reshape(NPM, Q)
    out = np.zeros((Q, Q, Q, NC))
    if S == 1:
        psi = T[cd[CD3_T_C]:cd[CD3_T_C] + Q * N].reshape(Q, N)
        for m in range(NPM):
            for l in range(N):
                out[:, :, :, m * N + l] = np.einsum("a,b,c->abc", A[:, gof[m]], psi[:, l], B[m])
    else:
        C = T[cd[CD3_T_C]:cd[CD3_T_C] + NC * Q].reshape(NC, Q)
        for r in range(NC):
            m = mofr[r]
            out[:, :, :, r] = np.einsum("a,b,c->abc", A[:, gof[m]], B[m], C[r])
    return out.reshape(Q ** 3, NC)


def emulate(pb, x, skip_faces=False, skip_volume=False, pub=None, phases=(0, 1)):
    """Phase 0 publishes every element's slot traces into `pub`, phase 1 applies (y returned)."""
    y = np.zeros(pb.n_dofs)
    T = pb.tables
    if pub is None:
        pub = np.zeros(max(pb.n_pub, 1))
    S_ = pb.slots
    ctx = {}
    for c in range(pb.class_desc.shape[0]):
        cd = pb.class_desc[c]
        S, N, Q = cd[CD3_SHAPE], cd[CD3_N], cd[CD3_Q]
        Phi = phi_matrix(pb, c)
        pts = T[cd[CD3_T_PTS]:cd[CD3_T_PTS] + 3 * Q].reshape(3, Q)
        D = T[cd[CD3_T_D]:cd[CD3_T_D] + 3 * Q * Q].reshape(3, Q, Q)
        Wt = T[cd[CD3_T_W]:cd[CD3_T_W] + Q + Q * Q]
        Wr = np.multiply.outer(Wt[:Q], Wt[Q:]).reshape(-1)
        E = T[cd[CD3_T_E]:cd[CD3_T_E] + 6 * Q].reshape(3, 2, Q)
        ctx[c] = (S, N, Q, Phi, pts, D, Wr, E)

    def own_trace(c, e, u, du, sl):
        S, N, Q, Phi, pts, D, Wr, E = ctx[c]
        fx, sd, run, _, _ = FACES[NAMES[S]][sl["face"]]
        ra, rb = run
        Ek = E[fx, 1 if sd > 0 else 0]
        uf = np.tensordot(Ek, np.moveaxis(u, fx, 0), axes=(0, 0))          # remaining axes in order
        dfs = [np.tensordot(Ek, np.moveaxis(d, fx, 0), axes=(0, 0)) for d in du]
        # remaining axes order after moveaxis(fx -> 0): the other two in increasing order = (ra, rb)
        assert ra < rb
        gn = np.zeros((3, Q, Q))
        for ia in range(Q):
            for ib in range(Q):
                eta = [0.0] * 3
                eta[fx] = sd
                eta[ra] = pts[ra, ia]
                eta[rb] = pts[rb, ib]
                ch = chain(S, *eta)
                v = sl["v"]
                gn[0, ia, ib] = ch["c00"] * v[0] + ch["c01"] * v[1] + ch["c02"] * v[2]
                gn[1, ia, ib] = ch["c11"] * v[1] + ch["c12"] * v[2]
                gn[2, ia, ib] = v[2]
        gf = sum(gn[k] * dfs[k] for k in range(3))
        uf, gf = uf.reshape(-1), gf.reshape(-1)
        M = slot_map(T, sl, Q)
        if M is not None:
            return M @ uf, M @ gf, M, gn.reshape(3, -1), (fx, sd, ra, rb, Ek)
        return uf, gf, None, gn.reshape(3, -1), (fx, sd, ra, rb, Ek)

    def element_fields(c, e):
        S, N, Q, Phi, pts, D, Wr, E = ctx[c]
        u = (Phi @ x[pb.dof_off[e]:pb.dof_off[e + 1]]).reshape(Q, Q, Q)
        du = [np.moveaxis(np.tensordot(D[a], u, axes=(1, a)), 0, a) for a in range(3)]
        return u, du

    for phase in phases:
        for c in range(pb.class_desc.shape[0]):
            cd = pb.class_desc[c]
            S, N, Q, Phi, pts, D, Wr, E = ctx[c]
            for i in range(cd[CD3_COUNT]):
                e = pb.class_elems[cd[CD3_ELEM_OFF] + i]
                u, du = element_fields(c, e)
                W = np.zeros((4, Q, Q, Q))
                for si in range(pb.slot_off[e], pb.slot_off[e + 1]):
                    sl = S_[si]
                    if phase == 0:
                        if True:        # every slot publishes its own trace
                            ut, gt, *_ = own_trace(c, e, u, du, sl)
                            nt = sl["nt"]
                            pub[sl["pub_self"]:sl["pub_self"] + 2 * nt:2] = ut
                            pub[sl["pub_self"] + 1:sl["pub_self"] + 2 * nt:2] = gt
                        continue
                    if skip_faces:
                        continue
                    _, _, M, gn, (fx, sd, ra, rb, Ek) = own_trace(c, e, u, du, sl)
                    nt = sl["nt"]
                    ut = pub[sl["pub_self"]:sl["pub_self"] + 2 * nt:2]
                    gt = pub[sl["pub_self"] + 1:sl["pub_self"] + 2 * nt:2]
                    if sl["kind"]:
                        un = pub[sl["pub_other"]:sl["pub_other"] + 2 * nt:2]
                        gnb = pub[sl["pub_other"] + 1:sl["pub_other"] + 2 * nt:2]
                    else:
                        un, gnb = -ut, -gt
                    j = ut - un
                    cc = 0.5 * (gt - gnb)
                    w = sl["sJ"] * T[sl["wtoff"]:sl["wtoff"] + nt]
                    fv = (sl["tau"] * j - cc) * w
                    fd = -0.5 * j * w
                    if M is not None:
                        fv, fd = M.T @ fv, M.T @ fd
                    fvq, fdq = fv.reshape(Q, Q), fd.reshape(Q, Q)
                    add0 = np.multiply.outer(Ek, fvq)                                # (k, a, b)
                    W[0] += np.moveaxis(add0, 0, fx)
                    for k in range(3):
                        W[1 + k] += np.moveaxis(np.multiply.outer(Ek, gn[k].reshape(Q, Q) * fdq), 0, fx)
                if phase == 0:
                    continue
                if not skip_volume:
                    eg = pb.egeo[e]
                    Sm = np.array([[eg[1], eg[2], eg[3]], [eg[2], eg[4], eg[5]], [eg[3], eg[5], eg[6]]])
                    for k0 in range(Q):
                        for k1 in range(Q):
                            for k2 in range(Q):
                                ch = chain(S, pts[0, k0], pts[1, k1], pts[2, k2])
                                jw = eg[0] * Wr[(k0 * Q + k1) * Q + k2]
                                d0, d1, d2 = du[0][k0, k1, k2], du[1][k0, k1, k2], du[2][k0, k1, k2]
                                xv = np.array([ch["c00"] * d0, ch["c01"] * d0 + ch["c11"] * d1,
                                               ch["c02"] * d0 + ch["c12"] * d1 + d2])
                                f = Sm @ xv
                                W[0, k0, k1, k2] += pb.lam * jw * u[k0, k1, k2]
                                W[1, k0, k1, k2] += jw * (ch["c00"] * f[0] + ch["c01"] * f[1] + ch["c02"] * f[2])
                                W[2, k0, k1, k2] += jw * (ch["c11"] * f[1] + ch["c12"] * f[2])
                                W[3, k0, k1, k2] += jw * f[2]
                Tt = W[0].copy()
                for a in range(3):
                    Tt += np.moveaxis(np.tensordot(D[a].T, W[1 + a], axes=(1, a)), 0, a)
                y[pb.dof_off[e]:pb.dof_off[e + 1]] = Phi.T @ Tt.reshape(-1)
    return y
