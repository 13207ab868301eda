"""CPU emulator of liblq's execution plans (test infrastructure).

Executes the JSON plan exported by ``lq_plan_export_json`` with numpy, at the
level of the plan's semantics (tiles, register sub-blocks, folded affine
permutations, lowered ops, Pauli-group terms) -- not of the kernel's thread
mechanics.  Comparing it with the oracle tests the host planner on CPU at
any size the emulator handles; comparing the GPU with the oracle tests the
kernels.  Shares no code with oracle/ or with the CUDA sources.
"""
from __future__ import annotations

import math

import numpy as np

NOREG = 255
K_U1, K_D1, K_X, K_U2, K_D2, K_SWAP, K_QFT, K_SCALE, K_EXPV, K_G, K_DT, K_GG = range(12)
GG_YY = 1
GK_REAL, GK_IMAG, GK_HAD = range(3)
FK_YDIAG = 100
PASS_TILE, PASS_PAIR, PASS_DIAG = 0, 1, 2
MF_U2x2, MF_DIAG2, MF_U4x4, MF_DIAG4, MF_G = range(5)
PF_EXPV, PF_NO_STORE, PF_RELABEL = 2, 4, 8
QF_INVERSE, QF_REVERSED, QF_GENERAL, QF_SCALE = 1, 2, 8, 16
# lq_kind numbering
(LQ_H, LQ_X, LQ_Y, LQ_Z, LQ_S, LQ_SDG, LQ_T, LQ_TDG, LQ_RX, LQ_RY, LQ_RZ, LQ_CNOT, LQ_CZ, LQ_CP,
 LQ_SWAP, LQ_U1, LQ_U2, LQ_CRY, LQ_CCX, LQ_RXX, LQ_RYY, LQ_RZZ) = range(22)


def _gate2(kind, th, cst):
    c, s = math.cos(th / 2), math.sin(th / 2)
    r2 = 1 / math.sqrt(2)
    tab = {LQ_H: [[r2, r2], [r2, -r2]], LQ_X: [[0, 1], [1, 0]], LQ_Y: [[0, -1j], [1j, 0]],
           LQ_Z: [[1, 0], [0, -1]], LQ_S: [[1, 0], [0, 1j]], LQ_SDG: [[1, 0], [0, -1j]],
           LQ_T: [[1, 0], [0, (1 + 1j) * r2]], LQ_TDG: [[1, 0], [0, (1 - 1j) * r2]],
           LQ_RX: [[c, -1j * s], [-1j * s, c]], LQ_RY: [[c, -s], [s, c]],
           LQ_RZ: [[c - 1j * s, 0], [0, c + 1j * s]], LQ_CP: [[1, 0], [0, complex(math.cos(th), math.sin(th))]]}
    if kind == LQ_U1:
        return np.array(cst, np.complex128).reshape(2, 2)
    if kind == FK_YDIAG:
        return np.array([[1j, 0], [0, -1j]], np.complex128)
    return np.array(tab[kind], np.complex128)


def build_mats(plan, theta, shift=None):
    """Per-op matrices as the device builder computes them (one circuit)."""
    cst = np.array(plan["cst"], np.float64)
    cstc = cst[0::2] + 1j * cst[1::2] if cst.size else np.zeros(0, np.complex128)
    mats = np.zeros(max(plan["mat_size"], 1), np.complex128)
    fac = plan["factors"]

    def angle(f):
        kind, pidx, ang, c = f
        if pidx < 0:
            return ang
        a = theta[pidx]
        if shift is not None and pidx == shift[0]:
            a = a + shift[1]
        return a
    for out, fb, fe, form in plan["specs"]:
        if form in (MF_U2x2, MF_DIAG2):
            A = np.eye(2, dtype=np.complex128)
            for f in fac[fb:fe]:
                F = _gate2(f[0], angle(f), cstc[f[3]:f[3] + 4] if f[3] >= 0 else None)
                A = F @ A
            if form == MF_U2x2:
                mats[out:out + 4] = A.reshape(-1)
            else:
                mats[out:out + 3] = [A[0, 0], A[1, 1], A[1, 1] / A[0, 0]]
        elif form == MF_G:
            # the op's exact matrix; _apply_op expands (p, lambda, variant)
            f = fac[fb]
            if f[0] == LQ_H:
                mats[out:out + 2] = [0.7071067811865476j, 0]
            else:
                c, s = math.cos(angle(f) / 2), math.sin(angle(f) / 2)
                mats[out:out + 2] = [complex(s / c, c), 0] if abs(c) >= abs(s) else [complex(c / s, s), 1]
        else:
            f = fac[fb]
            th = angle(f)
            c, s = math.cos(th / 2), math.sin(th / 2)
            if form == MF_DIAG4:
                mats[out:out + 4] = [c - 1j * s, c + 1j * s, c + 1j * s, c - 1j * s]
            elif f[0] == LQ_U2:
                mats[out:out + 16] = cstc[f[3]:f[3] + 16]
            else:
                P = np.array([[0, 1], [1, 0]] if f[0] == LQ_RXX else [[0, -1j], [1j, 0]], np.complex128)
                mats[out:out + 16] = (c * np.eye(4) - 1j * s * np.kron(P, P)).reshape(-1)
    return mats, cstc


def _deposit(l, T):
    g = np.zeros_like(l, dtype=np.int64)
    for i, b in enumerate(T):
        g |= ((l >> i) & 1) << b
    return g


def _parity(x):
    x = np.asarray(x, np.uint64).copy()
    p = np.zeros(x.shape, np.int64)
    while np.any(x):
        p ^= (x & np.uint64(1)).astype(np.int64)
        x >>= np.uint64(1)
    return p


def _brev(x, n):
    r = np.zeros_like(x)
    for i in range(n):
        r |= ((x >> i) & 1) << (n - 1 - i)
    return r


def _logical(g, lpos):
    """Logical index bits of physical indices g under a pass's lpos map."""
    out = np.zeros_like(g)
    for p, l in enumerate(lpos):
        if l < 64:
            out |= ((g >> p) & 1) << l
    return out


def _apply_op(x, g, op, S, mats, cstc, n, et_all, et0, lpos=None):
    """One lowered op on a tile vector x (index = local l), g = global index."""
    typ = op["type"]
    lb = lambda r: 1 << S[r]
    if typ == K_DT:   # members (register position, table offset) in the plan constants
        L = np.arange(x.size, dtype=np.int64)
        for k in range(op["flags"]):
            m = cstc[op["mat"] + k]
            pos, off = int(m.real), int(m.imag)
            bit = (L >> S[pos]) & 1
            x *= np.where(bit == 1, mats[off + 1], mats[off])
        return 0.0
    M = mats[op["mat"]:op["mat"] + 16] if typ in (K_U1, K_D1, K_U2, K_D2, K_G, K_GG) else None
    if typ == K_GG:  # RXX / RYY: lambda * [[one, -i off] on 01<->10, -+i off on 00<->11]
        p, lam, alt = M[0].real, M[0].imag, M[1].real != 0
        one, off = (p, 1.0) if alt else (1.0, p)
        s3 = 1j * off if op["flags"] & GG_YY else -1j * off
        U = np.zeros((4, 4), np.complex128)
        for d in range(4):
            U[d, d] = one
        U[0, 3] = U[3, 0] = s3
        U[1, 2] = U[2, 1] = -1j * off
        M = lam * U.reshape(-1)
        typ = K_U2
    if typ == K_G:   # lambda * M (lq_internal.h GKind)
        p, lam, alt = M[0].real, M[0].imag, M[1].real != 0
        one, off = (p, 1.0) if alt else (1.0, p)
        gk = op["qj"]
        if gk == GK_REAL:
            M = lam * np.array([one, -off, off, one], np.complex128)
        elif gk == GK_IMAG:
            M = lam * np.array([one, -1j * off, -1j * off, one], np.complex128)
        else:
            M = lam * np.array([1, 1, 1, -1], np.complex128)
        typ = K_U1
    L = np.arange(x.size, dtype=np.int64)
    ok = np.ones(x.size, bool)
    for r in range(4):
        if (op["rcm"] >> r) & 1 and typ != K_EXPV:
            ok &= (L & lb(r)) != 0
    if op["cmask"]:
        ok &= (g & op["cmask"]) == op["cmask"]
    if typ in (K_U1, K_X):
        m = lb(op["r0"])
        l0 = L[((L & m) == 0) & ok]
        a, b = x[l0].copy(), x[l0 | m].copy()
        if typ == K_X:
            x[l0], x[l0 | m] = b, a
        else:
            x[l0] = M[0] * a + M[1] * b
            x[l0 | m] = M[2] * a + M[3] * b
    elif typ == K_D1:
        bit = ((L >> S[op["r0"]]) & 1) if op["r0"] != NOREG else ((g >> op["b0"]) & 1)
        x[ok] *= np.where(bit == 1, M[1], M[0])[ok]
    elif typ == K_D2:
        ba = ((L >> S[op["r0"]]) & 1) if op["r0"] != NOREG else ((g >> op["b0"]) & 1)
        bb = ((L >> S[op["r1"]]) & 1) if op["r1"] != NOREG else ((g >> op["b1"]) & 1)
        x[ok] *= M[2 * ba + bb][ok]
    elif typ in (K_U2, K_SWAP):
        m0, m1 = lb(op["r0"]), lb(op["r1"])
        l0 = L[((L & (m0 | m1)) == 0) & ok]
        v = [x[l0].copy(), x[l0 | m1].copy(), x[l0 | m0].copy(), x[l0 | m0 | m1].copy()]
        if typ == K_SWAP:
            x[l0 | m1], x[l0 | m0] = v[2], v[1]
        else:
            U = M.reshape(4, 4)
            for r, idx in enumerate([l0, l0 | m1, l0 | m0, l0 | m0 | m1]):
                x[idx] = U[r, 0] * v[0] + U[r, 1] * v[1] + U[r, 2] * v[2] + U[r, 3] * v[3]
    elif typ == K_QFT:
        m = lb(op["r0"])
        j = op["qj"]
        inv = bool(op["flags"] & QF_INVERSE)
        if op["flags"] & QF_GENERAL:
            lg = _logical(g, lpos)
        else:
            lg = _brev(g, n) if op["flags"] & QF_REVERSED else g
        l0 = L[(L & m) == 0]
        l1 = l0 | m
        Lt = (lg[l1] & ((1 << j) - 1)) if j > 0 else np.zeros(l1.size, np.int64)
        tw = np.exp((-1j if inv else 1j) * np.pi * Lt / float(1 << j))
        u, w = x[l0].copy(), x[l1].copy()
        if not inv:
            x[l0], x[l1] = u + w, (u - w) * tw
        else:
            y = w * tw
            x[l0], x[l1] = u + y, u - y
        if op["flags"] & QF_SCALE:
            x *= 1 / np.sqrt(2)
    elif typ == K_SCALE:
        x *= cstc[op["mat"]].real
    elif typ == K_EXPV:
        xl = 0
        for r in range(4):
            if (op["rcm"] >> r) & 1:
                xl |= lb(r)
        sphys = 0
        for r in range(4):
            if r < len(S):
                pass
        e = 0.0
        w = np.conj(x[L ^ xl]) * x
        for k in range(op["aux"]):
            c, znr, zreg, y = et_all[et0 + op["mat"] + k]
            zl = 0
            for r in range(4):
                if (zreg >> r) & 1:
                    zl |= lb(r)
            sign = 1 - 2 * ((_parity(g & int(znr)) + _parity(L & zl)) & 1)
            e += c * np.sum(sign * (w * (1j ** y)).real)
        return e
    return 0.0


def run(plan, psi, theta=None, shift=None, gofs=0):
    """Run the plan on the physical-layout state psi (modified in place).
    Returns the Pauli-sum value accumulated by the plan's K_EXPV ops plus the
    wide groups (direct).  For a shard of a distributed state psi holds the
    2^nl local amplitudes and gofs the shard's physical global bits (they
    enter the logic index only, as in the kernels)."""
    n, K = plan.get("nl", plan["n"]), plan["K"]
    mats, cstc = build_mats(plan, theta if theta is not None else np.zeros(0), shift)
    subs, kops, perms, pts = plan["subs"], plan["kops"], plan["perms"], plan["perm_terms"]
    et_all = plan["eterms"]
    E = 0.0
    for p in plan["passes"]:
        if p["kind"] != PASS_TILE:
            gidx = np.arange(psi.size, dtype=np.int64) | gofs
            for op in kops[p["op_begin"]:p["op_end"]]:
                # physical form: b0/b1 are bits, controls in cmask
                S_phys = [op["b0"], op["b1"], 0, 0]
                op2 = dict(op)
                if op["type"] in (K_U1, K_X, K_U2, K_SWAP, K_G, K_GG):
                    op2["r0"], op2["r1"] = 0, 1
                _apply_op(psi, gidx, op2 if op["type"] in (K_U1, K_X, K_U2, K_SWAP, K_G, K_GG) else op,
                          S_phys, mats, cstc, n, et_all, 0)
            continue
        T = p["T"]
        Kp = p["K"]
        tmask = 0
        for b in T:
            tmask |= 1 << b
        free = [b for b in range(n) if not (tmask >> b) & 1]
        L = np.arange(1 << Kp, dtype=np.int64)
        dep = _deposit(L, T)
        # relabelling out-of-place store: the pass writes a new array in the
        # next frame (physical bit b -> spos[b])
        oop = bool(p.get("oop", 0)) and not (p["flags"] & PF_NO_STORE)
        out = np.empty_like(psi) if oop else psi
        for tile in range(1 << (n - Kp)):
            tb = 0
            for i, b in enumerate(free):
                tb |= ((tile >> i) & 1) << b
            g = tb | dep
            x = psi[g].copy()
            tb |= gofs   # logic index of the tile (controls / phases on global bits)

            def apply_perm(x, pi):
                P = perms[p["perm_begin"] + pi]
                binv = 0
                for cm, vec in pts[P["term_begin"]:P["term_end"]]:
                    if (tb & cm) == cm:
                        binv ^= vec
                src = np.full(L.size, binv, np.int64)
                for i in range(Kp):
                    src ^= ((L >> i) & 1) * P["col"][i]
                return x[src]
            for sb in subs[p["sub_begin"]:p["sub_end"]]:
                if sb["perm"] >= 0:
                    x = apply_perm(x, sb["perm"])
                for op in kops[sb["op_begin"]:sb["op_end"]]:
                    E += _apply_op(x, g | gofs, op, sb["S"], mats, cstc, plan["n"], et_all, p["eterm_begin"],
                                   p.get("lpos"))
            if p["store_perm"] >= 0:
                x = apply_perm(x, p["store_perm"])
            if p["flags"] & PF_RELABEL:
                # no store exchange (lq_internal.h PassFlags): the thread that
                # holds local index l under the last sub-block's register
                # mapping stores it where the Sstore mapping puts the same
                # (thread, register) pair: register bit i moves from local bit
                # S_last[i] to Sstore[i], thread bit k from the k-th other bit
                # of one mapping to the k-th other bit of the other
                Rr = plan["Rr"]
                S_last = subs[p["sub_end"] - 1]["S"][:Rr]
                S_st = p["Sstore"][:Rr]
                o_last = [b for b in range(Kp) if b not in S_last]
                o_st = [b for b in range(Kp) if b not in S_st]
                dst = np.zeros_like(L)
                for a, b in list(zip(S_last, S_st)) + list(zip(o_last, o_st)):
                    dst |= ((L >> a) & 1) << b
                y = np.empty_like(x)
                y[dst] = x
                x = y
            if not (p["flags"] & PF_NO_STORE):
                if oop:
                    gs = np.zeros_like(g)
                    for b, sb in enumerate(p["spos"]):
                        gs |= ((g >> b) & 1) << sb
                    out[gs] = x
                else:
                    psi[g] = x
        if oop:
            psi[:] = out
    # wide groups (direct kernel)
    j = np.arange(psi.size, dtype=np.int64)
    for gi in plan["wide_groups"]:
        G = plan["groups"][gi]
        w = np.conj(psi[j ^ G["x"]]) * psi
        for c, z, y in G["terms"]:
            E += c * np.sum((1 - 2 * _parity((j | gofs) & int(z))) * (w * (1j ** y)).real)
    return E


def logical_state(plan_qmap, psi):
    """Reorder a physical-layout state into logical (MSB-first) order."""
    n = len(plan_qmap)
    x = np.arange(psi.size, dtype=np.int64)
    g = np.zeros_like(x)
    for q in range(n):
        g |= ((x >> (n - 1 - q)) & 1) << plan_qmap[q]
    return psi[g]
