"""Test helpers: build user-form instances from dense arrays; brute force by enumeration."""
import numpy as np


def inst_from_dense(K_u, r, sense, c, Q=None, c0=0.0, maximize=False, name="dense"):
    K_u = np.asarray(K_u, dtype=np.float64).reshape(-1, len(c)) if len(K_u) else np.zeros((0, len(c)))
    n = len(c)
    m = K_u.shape[0]
    ptr = np.zeros(m + 1, dtype=np.int64)
    cols, vals = [], []
    for j in range(m):
        nz = np.nonzero(K_u[j])[0]
        cols.append(nz)
        vals.append(K_u[j, nz])
        ptr[j + 1] = ptr[j] + nz.size
    inst = dict(name=name, n=n, m=m, k_rowptr=ptr,
                k_col=(np.concatenate(cols) if m else np.zeros(0)).astype(np.int32),
                k_val=(np.concatenate(vals) if m else np.zeros(0)).astype(np.float64),
                r=np.asarray(r, dtype=np.float64), sense=np.asarray(sense, dtype=np.int8),
                q_rowptr=None, q_col=None, q_val=None, c=np.asarray(c, dtype=np.float64),
                c0=float(c0), maximize=bool(maximize))
    if Q is not None:
        Q = np.asarray(Q, dtype=np.float64)
        qptr = np.zeros(n + 1, dtype=np.int64)
        qc, qv = [], []
        for i in range(n):
            nz = np.nonzero(Q[i])[0]
            qc.append(nz)
            qv.append(Q[i, nz])
            qptr[i + 1] = qptr[i] + nz.size
        if qptr[-1] > 0:
            inst.update(q_rowptr=qptr, q_col=np.concatenate(qc).astype(np.int32),
                        q_val=np.concatenate(qv).astype(np.float64))
    return inst


def all_points(n):
    """All 2^n binary points as an (2^n, n) uint8 matrix; row l has x_i = bit i of l."""
    l = np.arange(2 ** n, dtype=np.int64)
    return ((l[:, None] >> np.arange(n)[None, :]) & 1).astype(np.uint8)


def exhaustive_bits(n):
    """Bit-sliced batch holding all 2^n points: lane l = integer whose bit i is x_i (n >= 6)."""
    nw = max(1, 2 ** n // 64)
    bits = np.zeros((n, nw), dtype=np.uint64)
    lanes = np.arange(64, dtype=np.uint64)
    for i in range(n):
        if i < 6:
            word = np.uint64(0)
            for b in range(64):
                if (b >> i) & 1:
                    word |= np.uint64(1) << np.uint64(b)
            bits[i, :] = word
        else:
            w = np.arange(nw, dtype=np.int64)
            bits[i, :] = np.where(((w >> (i - 6)) & 1) == 1, np.uint64(0xFFFFFFFFFFFFFFFF), np.uint64(0))
    del lanes
    return bits


def brute_force(inst):
    """Independent enumeration in the USER form with dense numpy algebra.
    Returns (z_opt in user sense, x_opt, feasible mask, z vector (user sense))."""
    from gen.instances import dense_K, dense_Q
    n = inst["n"]
    X = all_points(n).astype(np.float64)
    K = dense_K(inst)
    Q = dense_Q(inst)
    ax = X @ K.T
    r = inst["r"]
    s = inst["sense"]
    ok = np.ones(X.shape[0], dtype=bool)
    for j in range(inst["m"]):
        if s[j] == 1:
            ok &= ax[:, j] >= r[j] - 1e-9
        elif s[j] == -1:
            ok &= ax[:, j] <= r[j] + 1e-9
        else:
            ok &= np.abs(ax[:, j] - r[j]) <= 1e-9
    z = np.einsum("li,ij,lj->l", X, Q, X) + X @ inst["c"] + inst["c0"]
    if not ok.any():
        return None, None, ok, z
    if inst["maximize"]:
        zz = np.where(ok, z, -np.inf)
        l = int(np.argmax(zz))
    else:
        zz = np.where(ok, z, np.inf)
        l = int(np.argmin(zz))
    return z[l], X[l].astype(np.uint8), ok, z
