"""TEST INFRASTRUCTURE ONLY (see gfors_oracle.h): plain dense-numpy TUReformulate of PAPER §2.4.1
(Theorem), written literally from the theorem's definitions.

Given the USER-form instance (gen.instances dict) and index sets J (equality rows, input order) and
I (columns), |J| = |I|, with B_J, d_J integral and B_JI invertible:

    s := B_JI^{-1} d_J,   S := -B_JI^{-1} B_{J,Ibar},   x_I = s + S x_Ibar
    Q' = S'Q_II S + S'Q_{I,Ibar} + Q_{I,Ibar}' S + Q_{Ibar,Ibar}
    c' = 2 S'Q_II s + 2 Q_{I,Ibar}' s + S'c_I + c_Ibar,    c0' = <s, Q_II s> + <c_I, s> (+ c0)
    A' = A_.I S + A_.Ibar,  b' = b - A_.I s  (reading A20: A_{.I}, not A_I)
    B' = B_{Jbar,I} S + B_{Jbar,Ibar},  d' = d_Jbar - B_{Jbar,I} s
    plus  S x_Ibar >= -s  and  S x_Ibar <= 1 - s   (x_I in [0,1])

Row order of the reduced instance (reading R24): the rows of the input other than J, in input order
and with their input senses, then for t = 0..|J|-1 the two box rows of t in the GE form
S_t x >= -s_t and -S_t x >= s_t - 1; a box row that every binary x satisfies (sum of its negative
coefficients >= rhs) is dropped.  Reduced variables: Ibar in ascending input order.
Shares nothing with the CUDA library.
"""
from __future__ import annotations

import numpy as np


def _dense_K(inst):
    m, n = inst["m"], inst["n"]
    K = np.zeros((m, n))
    for j in range(m):
        a, b = inst["k_rowptr"][j], inst["k_rowptr"][j + 1]
        K[j, inst["k_col"][a:b]] = inst["k_val"][a:b]
    return K


def _dense_Q(inst):
    n = inst["n"]
    Q = np.zeros((n, n))
    if inst.get("q_rowptr") is not None:
        for i in range(n):
            a, b = inst["q_rowptr"][i], inst["q_rowptr"][i + 1]
            Q[i, inst["q_col"][a:b]] = inst["q_val"][a:b]
    return Q


def _csr(M):
    ptr = np.zeros(M.shape[0] + 1, dtype=np.int64)
    cols, vals = [], []
    for j in range(M.shape[0]):
        nz = np.flatnonzero(M[j])
        cols.append(nz)
        vals.append(M[j, nz])
        ptr[j + 1] = ptr[j] + nz.size
    col = np.concatenate(cols).astype(np.int32) if cols else np.zeros(0, np.int32)
    val = np.concatenate(vals).astype(np.float64) if vals else np.zeros(0)
    return ptr, col, val


def _exact(M, what):
    R = np.rint(M)
    if not np.allclose(M, R, atol=1e-9):
        raise ValueError(f"TUReformulate: {what} is not integral (B_J not TU?)")
    return R + 0.0


def tu_reformulate(inst, J, I):
    """Returns (reduced user-form instance, lift) where lift(xbar) -> x (uint8, length n)."""
    n, m = inst["n"], inst["m"]
    J = np.asarray(J, dtype=np.int64)
    I = np.asarray(I, dtype=np.int64)
    if J.size != I.size or J.size == 0:
        raise ValueError("TUReformulate: |J| = |I| > 0 required")
    sense = np.asarray(inst["sense"])
    if np.any(sense[J] != 0):
        raise ValueError("TUReformulate: J must index equality rows")
    K = _dense_K(inst)
    r = np.asarray(inst["r"], dtype=np.float64)
    Q = _dense_Q(inst)
    c = np.asarray(inst["c"], dtype=np.float64)
    Ibar = np.setdiff1d(np.arange(n), I)          # ascending
    Jbar = np.setdiff1d(np.arange(m), J)          # ascending = input order
    B_J, d_J = K[J], r[J]
    if not (np.all(B_J == np.rint(B_J)) and np.all(d_J == np.rint(d_J))):
        raise ValueError("TUReformulate: B_J and d_J must be integral")
    B_JI = B_J[:, I]
    if abs(np.linalg.det(B_JI)) < 0.5:
        raise ValueError("TUReformulate: B_JI is singular")
    inv = np.linalg.inv(B_JI)
    s = _exact(inv @ d_J, "s")
    S = _exact(-inv @ B_J[:, Ibar], "S")
    # objective (theorem's Q', c', c0')
    Q_II, Q_IIb, Q_IbIb = Q[np.ix_(I, I)], Q[np.ix_(I, Ibar)], Q[np.ix_(Ibar, Ibar)]
    Qp = S.T @ Q_II @ S + S.T @ Q_IIb + Q_IIb.T @ S + Q_IbIb
    cp = 2.0 * S.T @ Q_II @ s + 2.0 * Q_IIb.T @ s + S.T @ c[I] + c[Ibar]
    c0p = float(s @ Q_II @ s + c[I] @ s + inst["c0"])
    # constraints other than J (GE, LE and EQ alike: row' = row_.I S + row_.Ibar, rhs' = rhs - row_.I s)
    Kb = K[Jbar]
    Kp = Kb[:, I] @ S + Kb[:, Ibar]
    rp = r[Jbar] - Kb[:, I] @ s
    sp = sense[Jbar].astype(np.int8)
    # box rows of x_I = s + S x_Ibar in [0, 1]
    box, box_r = [], []
    for t in range(I.size):
        for coef, rhs in ((S[t], -s[t]), (-S[t], s[t] - 1.0)):
            if np.minimum(coef, 0.0).sum() >= rhs:
                continue  # satisfied by every binary x
            box.append(coef)
            box_r.append(rhs)
    if box:
        Kp = np.vstack([Kp, np.array(box)])
        rp = np.concatenate([rp, np.array(box_r)])
        sp = np.concatenate([sp, np.ones(len(box), np.int8)])
    kptr, kcol, kval = _csr(Kp)
    red = dict(name=inst.get("name", "inst") + "_tu", n=int(Ibar.size), m=int(Kp.shape[0]), k_rowptr=kptr,
               k_col=kcol, k_val=kval, r=rp, sense=sp, c=cp, c0=c0p, maximize=inst["maximize"],
               q_rowptr=None, q_col=None, q_val=None)
    if np.any(Qp != 0):
        qptr, qcol, qval = _csr(Qp)
        red.update(q_rowptr=qptr, q_col=qcol, q_val=qval)

    def lift(xbar):
        xbar = np.asarray(xbar, dtype=np.float64)
        x = np.zeros(n)
        x[Ibar] = xbar
        x[I] = s + S @ xbar
        if np.any((x != 0) & (x != 1)):
            raise ValueError("TUReformulate: lifted x_I is not binary")
        return x.astype(np.uint8)

    return red, lift
