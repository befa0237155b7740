"""Seeded synthetic BIP instances shaped like the paper's workloads (PAPER §4).

This module holds NO arithmetic of the method: it only draws random problem data
(numpy ``Generator(PCG64(seed))``).  Both the CUDA path's tests/bench and the CPU
oracle consume its output.  Every instance is returned in USER form

    min/max  x'Qx + c'x + c0   s.t.  K_u x (>= | = | <=) r,   x in {0,1}^n

as a dict with CSR arrays:
    n, m, k_rowptr[int64 m+1], k_col[int32], k_val[float64], r[float64 m],
    sense[int8 m] (+1 GE, 0 EQ, -1 LE), q_rowptr/q_col/q_val (or None),
    c[float64 n], c0, maximize, name.
The recipes are listed in DESIGN.md §4 (input recipe).
"""
from __future__ import annotations

import numpy as np


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def _csr_from_rows(rows_cols, rows_vals, m):
    lens = np.array([len(c) for c in rows_cols], dtype=np.int64)
    ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    col = np.concatenate(rows_cols).astype(np.int32) if m else np.zeros(0, np.int32)
    val = np.concatenate(rows_vals).astype(np.float64) if m else np.zeros(0)
    return ptr, col, val


def _distinct_sorted_rows(rng, m, n, deg):
    """Row j gets deg[j] distinct uniform columns, sorted.  Vectorised with redraw of duplicates."""
    deg = np.asarray(deg, dtype=np.int64)
    ptr = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(deg, out=ptr[1:])
    nnz = int(ptr[-1])
    row = np.repeat(np.arange(m, dtype=np.int64), deg)
    col = rng.integers(0, n, size=nnz, dtype=np.int64)
    while True:
        key = row * n + col
        order = np.argsort(key, kind="stable")
        ks = key[order]
        dup = np.zeros(nnz, dtype=bool)
        dup[order[1:]] = ks[1:] == ks[:-1]
        nd = int(dup.sum())
        if nd == 0:
            break
        col[dup] = rng.integers(0, n, size=nd, dtype=np.int64)
    key = row * n + col
    order = np.argsort(key, kind="stable")
    return ptr, col[order].astype(np.int32)


def set_cover(m, n, dmin, dmax, seed, name="set_cover"):
    """min c'x s.t. sum_{i in S_j} x_i >= 1; |S_j| ~ U{dmin..dmax}; c ~ U{1..100}."""
    rng = _rng(seed)
    dmax = min(dmax, n)
    deg = rng.integers(dmin, dmax + 1, size=m)
    ptr, col = _distinct_sorted_rows(rng, m, n, deg)
    c = rng.integers(1, 101, size=n).astype(np.float64)
    return dict(name=name, n=n, m=m, k_rowptr=ptr, k_col=col, k_val=np.ones(col.shape[0]),
                r=np.ones(m), sense=np.ones(m, dtype=np.int8),
                q_rowptr=None, q_col=None, q_val=None, c=c, c0=0.0, maximize=False)


def max_independent_set(n, p, seed, weighted=False, name="mis"):
    """max sum w_i x_i s.t. x_i + x_j <= 1 for each edge of G(n,p) (BASELINE config 2)."""
    rng = _rng(seed)
    npairs = n * (n - 1) // 2
    target = int(rng.binomial(npairs, p))
    edges = np.zeros((0, 2), dtype=np.int64)
    while edges.shape[0] < target:
        need = target - edges.shape[0]
        a = rng.integers(0, n, size=2 * need + 16)
        b = rng.integers(0, n, size=2 * need + 16)
        keep = a != b
        e = np.stack([np.minimum(a, b), np.maximum(a, b)], 1)[keep]
        edges = np.unique(np.concatenate([edges, e]), axis=0)
    if edges.shape[0] > target:
        sel = np.sort(rng.choice(edges.shape[0], size=target, replace=False))
        edges = edges[sel]
    m = edges.shape[0]
    ptr = np.arange(0, 2 * m + 1, 2, dtype=np.int64)
    col = edges.reshape(-1).astype(np.int32)
    c = rng.integers(1, 101, size=n).astype(np.float64) if weighted else np.ones(n)
    return dict(name=name, n=n, m=m, k_rowptr=ptr, k_col=col, k_val=np.ones(2 * m),
                r=np.ones(m), sense=-np.ones(m, dtype=np.int8),
                q_rowptr=None, q_col=None, q_val=None, c=c, c0=0.0, maximize=True)


def multi_knapsack(n, m, density, seed, name="mkp"):
    """max v'x s.t. W x <= cap, W_ji ~ U{1..100} w.p. density, cap_j = floor(sum_i W_ji / 2)."""
    rng = _rng(seed)
    cols, vals = [], []
    for _ in range(m):
        mask = rng.random(n) < density
        cc = np.nonzero(mask)[0]
        if cc.size == 0:
            cc = np.array([rng.integers(0, n)])
        cols.append(cc)
        vals.append(rng.integers(1, 101, size=cc.size).astype(np.float64))
    ptr, col, val = _csr_from_rows(cols, vals, m)
    cap = np.array([np.floor(v.sum() / 2.0) for v in vals])
    v = rng.integers(1, 101, size=n).astype(np.float64)
    return dict(name=name, n=n, m=m, k_rowptr=ptr, k_col=col, k_val=val, r=cap,
                sense=-np.ones(m, dtype=np.int8), q_rowptr=None, q_col=None, q_val=None,
                c=v, c0=0.0, maximize=True)


def assignment_bqp(n_agents, n_slots, links, seed, name="bqp"):
    """min x'Qx + c'x, Q = Laplacian of a random graph (each variable links to `links` others),
    s.t. sum_b x_ab = 1 per agent (EQ), sum_a x_ab <= 1 per slot (LE); c ~ U{1..100}.
    Variables x_ab are indexed a*n_slots + b.  (PAPER L81 PSD Q; TU rows L819-821.)"""
    rng = _rng(seed)
    n = n_agents * n_slots
    rows_c, rows_v = [], []
    for a in range(n_agents):
        rows_c.append(a * n_slots + np.arange(n_slots))
        rows_v.append(np.ones(n_slots))
    for b in range(n_slots):
        rows_c.append(np.arange(n_agents) * n_slots + b)
        rows_v.append(np.ones(n_agents))
    m = n_agents + n_slots
    ptr, col, val = _csr_from_rows(rows_c, rows_v, m)
    sense = np.concatenate([np.zeros(n_agents, np.int8), -np.ones(n_slots, np.int8)])
    r = np.ones(m)
    # Laplacian of a random simple graph
    src = np.repeat(np.arange(n, dtype=np.int64), links)
    dst = rng.integers(0, n, size=src.shape[0])
    keep = src != dst
    e = np.stack([np.minimum(src, dst), np.maximum(src, dst)], 1)[keep]
    e = np.unique(e, axis=0)
    deg = np.bincount(e.reshape(-1), minlength=n).astype(np.float64)
    qi = np.concatenate([e[:, 0], e[:, 1], np.arange(n)])
    qj = np.concatenate([e[:, 1], e[:, 0], np.arange(n)])
    qv = np.concatenate([-np.ones(e.shape[0]), -np.ones(e.shape[0]), deg])
    nz = qv != 0
    qi, qj, qv = qi[nz], qj[nz], qv[nz]
    order = np.lexsort((qj, qi))
    qi, qj, qv = qi[order], qj[order], qv[order]
    qptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(qi, minlength=n), out=qptr[1:])
    c = rng.integers(1, 101, size=n).astype(np.float64)
    return dict(name=name, n=n, m=m, k_rowptr=ptr, k_col=col, k_val=val, r=r, sense=sense,
                q_rowptr=qptr, q_col=qj.astype(np.int32), q_val=qv, c=c, c0=0.0, maximize=False)


def random_general(n, m_ge, m_eq, deg, seed, vmax=5, real=False, with_q=False, name="general"):
    """Small mixed instance for parity edge cases: integer (or real) coefficients of both signs,
    GE/EQ/LE rows, optional symmetric indefinite Q.  Not a paper workload; a test family."""
    rng = _rng(seed)
    m = m_ge + m_eq
    degs = rng.integers(1, deg + 1, size=m)
    ptr, col = _distinct_sorted_rows(rng, m, n, np.minimum(degs, n))
    nnz = col.shape[0]
    if real:
        val = np.round(rng.uniform(-vmax, vmax, size=nnz), 3)
        val[val == 0] = 0.5
    else:
        val = rng.integers(1, vmax + 1, size=nnz) * rng.choice([-1.0, 1.0], size=nnz)
    # right-hand side from a random binary point so the instance is feasible
    x0 = (rng.random(n) < 0.5).astype(np.float64)
    row = np.repeat(np.arange(m), np.diff(ptr))
    ax = np.bincount(row, weights=val * x0[col], minlength=m)
    sense = np.concatenate([rng.choice([1, -1], size=m_ge).astype(np.int8), np.zeros(m_eq, np.int8)])
    slack = rng.integers(0, 3, size=m).astype(np.float64)
    r = np.where(sense == 1, ax - slack, np.where(sense == -1, ax + slack, ax))
    if real:
        r = np.round(r, 3)
    inst = dict(name=name, n=n, m=m, k_rowptr=ptr, k_col=col, k_val=val.astype(np.float64), r=r,
                sense=sense, q_rowptr=None, q_col=None, q_val=None,
                c=(np.round(rng.uniform(-20, 20, size=n), 2) if real else rng.integers(-20, 21, size=n).astype(np.float64)),
                c0=float(rng.integers(-5, 6)), maximize=False)
    if with_q:
        k = max(1, n)
        qi = rng.integers(0, n, size=k)
        qj = rng.integers(0, n, size=k)
        qv = rng.integers(-4, 5, size=k).astype(np.float64)
        if real:
            qv = np.round(rng.uniform(-2, 2, size=k), 2)
        Qd = np.zeros((n, n))
        for a, b, v in zip(qi, qj, qv):
            Qd[a, b] += v
            Qd[b, a] += v if a != b else 0.0
        inst.update(dense_to_csr_sym(Qd))
    return inst


def max_cut(n, density, seed, wmin=-8, wmax=10, name="maxcut"):
    """Max cut QP: max sum_{(i,j) in E} w_ij (x_i + x_j - 2 x_i x_j) over x in {0,1}^V,
    G(n, density) with integer weights w ~ U{wmin..wmax} (density 0.5, w in [-8, 10];
    integral reading, zero-weight edges dropped).  User form: maximize x'Qx + c'x with
    Q_ij = Q_ji = -w_ij (i != j; x'Qx = -2 sum w_ij x_i x_j) and c_i = sum_j w_ij; no constraints.
    Generated one row block at a time (upper triangle mirrored), so n = 20480 stays within a few GB."""
    rng = _rng(seed)
    Wup = np.zeros((n, n), dtype=np.int8)
    B = 1024
    for r0 in range(0, n, B):
        r1 = min(n, r0 + B)
        blk = rng.integers(wmin, wmax + 1, size=(r1 - r0, n), dtype=np.int16).astype(np.int8)
        keep = rng.random((r1 - r0, n), dtype=np.float32) < density
        blk[~keep] = 0
        ii = np.arange(r0, r1)[:, None]
        blk[np.arange(n)[None, :] <= ii] = 0  # strict upper triangle
        Wup[r0:r1] = blk
    inst = dict(name=name, n=n, m=0, k_rowptr=np.zeros(1, np.int64), k_col=np.zeros(0, np.int32),
                k_val=np.zeros(0), r=np.zeros(0), sense=np.zeros(0, np.int8), c0=0.0, maximize=True)
    deg = np.zeros(n, dtype=np.int64)
    qptr = np.zeros(n + 1, dtype=np.int64)
    cols, vals = [], []
    for r0 in range(0, n, B):
        r1 = min(n, r0 + B)
        rows = Wup[r0:r1].astype(np.int16) + Wup[:, r0:r1].T.astype(np.int16)  # symmetric W rows
        deg[r0:r1] = rows.sum(axis=1, dtype=np.int64)
        for k in range(r1 - r0):
            nz = np.flatnonzero(rows[k])
            cols.append(nz.astype(np.int32))
            vals.append(-rows[k, nz].astype(np.float64))
            qptr[r0 + k + 1] = qptr[r0 + k] + nz.size
    del Wup
    inst.update(q_rowptr=qptr, q_col=np.concatenate(cols), q_val=np.concatenate(vals), c=deg.astype(np.float64))
    return inst


def dense_laplacian(n, density, m, seed, name="dense_psd"):
    """Dense PSD test family for the dense-Q path: min x'Lx + c'x, L = Laplacian of G(n, density)
    (0/1 weights, so |L_ij| <= 127 for n <= 200), c ~ U{1..100}, m covering rows of 2..8 columns.
    Not a paper workload: the PSD (non-expansive) dense counterpart of the bqp family, on which the
    1000-iteration parity bar applies."""
    rng = _rng(seed)
    A = np.triu((rng.random((n, n)) < density).astype(np.int64), 1)
    A = A + A.T
    L = np.diag(A.sum(1)) - A
    inst = set_cover(m, n, 2, 8, seed + 1000, name)
    inst.update(dense_to_csr_sym(L.astype(np.float64)))
    inst["c"] = rng.integers(1, 101, size=n).astype(np.float64)
    return inst


def facility_location(nf, nc, seed, name="facility"):
    """Uncapacitated facility location: min f'x + sum_ij c_ij y_ij s.t.
    sum_i y_ij = 1 for every customer j (EQ), y_ij <= x_i (LE as y_ij - x_i <= 0).  Reading R24:
    c_ij ~ U{1..100}, f_i ~ U{1..100} * ceil(nc/nf).  Variables: x_i at i, y_ij at nf + j*nf + i.
    Rows: the nc customer rows first, then y_ij - x_i <= 0 in (j, i) order.  Also returns the TU
    index sets of the paper's reformulation: J = the customer rows, I = for each
    customer its cheapest y_ij (lowest i on ties) -> B_JI = identity."""
    rng = _rng(seed)
    f = (rng.integers(1, 101, size=nf) * -(-nc // nf)).astype(np.float64)
    cost = rng.integers(1, 101, size=(nc, nf)).astype(np.float64)
    n = nf + nf * nc
    y = lambda j, i: nf + j * nf + i  # noqa: E731
    rows_c, rows_v = [], []
    for j in range(nc):
        rows_c.append(np.array([y(j, i) for i in range(nf)]))
        rows_v.append(np.ones(nf))
    for j in range(nc):
        for i in range(nf):
            rows_c.append(np.array([i, y(j, i)]))
            rows_v.append(np.array([-1.0, 1.0]))
    m = nc + nf * nc
    ptr, col, val = _csr_from_rows(rows_c, rows_v, m)
    sense = np.concatenate([np.zeros(nc, np.int8), -np.ones(nf * nc, np.int8)])
    r = np.concatenate([np.ones(nc), np.zeros(nf * nc)])
    c = np.concatenate([f, cost.reshape(-1)])
    inst = dict(name=name, n=n, m=m, k_rowptr=ptr, k_col=col, k_val=val, r=r, sense=sense,
                q_rowptr=None, q_col=None, q_val=None, c=c, c0=0.0, maximize=False)
    inst["tu_rows"] = np.arange(nc, dtype=np.int64)
    inst["tu_cols"] = np.array([y(j, int(np.argmin(cost[j]))) for j in range(nc)], dtype=np.int32)
    return inst


def facility_location_slack(nf, nc, seed, name="facility_slack"):
    """The facility-location instance of facility_location (same costs) with every constraint an
    equality (reading R24, round 2; "when it eliminates all inequality constraints"):
    y_ij - x_i + s_ij = 0 with a binary slack s_ij (cost 0) replaces y_ij <= x_i, so the whole
    constraint matrix B (customer rows + linking rows) is TU and TUReformulate can remove every row.
    Variables: x_i at i, y_ij at nf + j*nf + i, s_ij at nf + nf*nc + j*nf + i.  Rows: the nc customer
    rows, then the linking rows in (j, i) order.  TU sets: J = all rows; I = for customer row j its
    cheapest y_ij (lowest i on ties), for linking row (j, i) the slack s_ij — B_JI is unit triangular
    (the linking row of the cheapest facility meets both y_{i*j} and s_{i*j}), not a permutation."""
    base = facility_location(nf, nc, seed)
    n0 = base["n"]
    ns = nf * nc
    rows_c, rows_v = [], []
    ptr, col, val = base["k_rowptr"], base["k_col"], base["k_val"]
    for j in range(nc):
        rows_c.append(col[ptr[j]:ptr[j + 1]]); rows_v.append(val[ptr[j]:ptr[j + 1]])
    for j in range(nc):
        for i in range(nf):
            rows_c.append(np.array([i, nf + j * nf + i, n0 + j * nf + i]))
            rows_v.append(np.array([-1.0, 1.0, 1.0]))
    m = nc + ns
    kp, kc, kv = _csr_from_rows(rows_c, rows_v, m)
    c = np.concatenate([base["c"], np.zeros(ns)])
    inst = dict(name=name, n=n0 + ns, m=m, k_rowptr=kp, k_col=kc, k_val=kv,
                r=np.concatenate([np.ones(nc), np.zeros(ns)]), sense=np.zeros(m, np.int8),
                q_rowptr=None, q_col=None, q_val=None, c=c, c0=0.0, maximize=False)
    inst["tu_rows"] = np.arange(m, dtype=np.int64)
    inst["tu_cols"] = np.concatenate([base["tu_cols"], n0 + np.arange(ns)]).astype(np.int32)
    return inst


def assignment3d(n, seed, name="assign3d"):
    """3D assignment (PAPER eq. assign3d): min c'x over x in {0,1}^(n^3), sum_{jk} x_ijk = 1,
    sum_{ik} x_ijk = 1, sum_{ij} x_ijk = 1; c_ijk ~ U{1..100} (reading R25).  Variable (i,j,k) at flat
    index i*n^2 + j*n + k; rows: the n i-rows, then the n j-rows, then the n k-rows (all EQ)."""
    rng = _rng(seed)
    N = n ** 3
    v = np.arange(N)
    I, J, K = v // (n * n), (v // n) % n, v % n
    rows_c = [np.flatnonzero(I == a) for a in range(n)] + [np.flatnonzero(J == a) for a in range(n)] + \
             [np.flatnonzero(K == a) for a in range(n)]
    ptr, col, val = _csr_from_rows(rows_c, [np.ones(len(r)) for r in rows_c], 3 * n)
    c = rng.integers(1, 101, size=N).astype(np.float64)
    return dict(name=name, n=N, m=3 * n, k_rowptr=ptr, k_col=col, k_val=val, r=np.ones(3 * n),
                sense=np.zeros(3 * n, np.int8), q_rowptr=None, q_col=None, q_val=None, c=c, c0=0.0,
                maximize=False, a3_n=n)


def cut_value(inst_edges_w, x):
    """Cut weight sum_{i<j} w_ij [x_i != x_j] from a dense symmetric weight matrix (test helper)."""
    x = np.asarray(x).astype(bool)
    W = inst_edges_w
    return float(W[np.ix_(x, ~x)].sum())


def dense_to_csr_sym(Qd):
    n = Qd.shape[0]
    qptr = np.zeros(n + 1, dtype=np.int64)
    cols, vals = [], []
    for i in range(n):
        nz = np.nonzero(Qd[i])[0]
        cols.append(nz)
        vals.append(Qd[i, nz])
        qptr[i + 1] = qptr[i] + nz.size
    return dict(q_rowptr=qptr, q_col=np.concatenate(cols).astype(np.int32),
                q_val=np.concatenate(vals).astype(np.float64))


def dense_K(inst):
    """Dense user-form K_u (for small test instances)."""
    K = np.zeros((inst["m"], inst["n"]))
    for j in range(inst["m"]):
        s, e = inst["k_rowptr"][j], inst["k_rowptr"][j + 1]
        K[j, inst["k_col"][s:e]] = inst["k_val"][s:e]
    return K


def dense_Q(inst):
    n = inst["n"]
    Q = np.zeros((n, n))
    if inst.get("q_rowptr") is not None:
        for i in range(n):
            s, e = inst["q_rowptr"][i], inst["q_rowptr"][i + 1]
            Q[i, inst["q_col"][s:e]] = inst["q_val"][s:e]
    return Q


# --------------------------------------------------------------------------------------------
# The five BASELINE.json configurations, plus scaled-down parity versions.
# --------------------------------------------------------------------------------------------
CONFIGS = {
    1: dict(desc="tiny set cover n=20, m=30", make=lambda s: set_cover(30, 20, 2, 5, s, "cfg1_setcover_20x30")),
    2: dict(desc="max independent set G(1e4, 1e-3)", make=lambda s: max_independent_set(10_000, 1e-3, s, name="cfg2_mis_10k")),
    3: dict(desc="multi-dim knapsack n=1e5, m=50, density 0.5",
            make=lambda s: multi_knapsack(100_000, 50, 0.5, s, "cfg3_mkp_100k_50")),
    4: dict(desc="BQP 400x500 assignment, Laplacian Q",
            make=lambda s: assignment_bqp(400, 500, 4, s, "cfg4_bqp_400x500")),
    5: dict(desc="set cover n=5e6, m=1e6, row degree U{2..98}",
            make=lambda s: set_cover(1_000_000, 5_000_000, 2, 98, s, "cfg5_setcover_5M_1M")),
    # next row f1: dense-Q workload, the paper's largest max-cut size
    6: dict(desc="max cut QP n=20480, density 0.5, w ~ U{-8..10} (dense Q, next row f1)",
            make=lambda s: max_cut(20_480, 0.5, s, name="cfg6_maxcut_20480")),
    # next row f2: the paper's facility-location TU workload at (nf, nc) = (512, 2048)
    7: dict(desc="facility location nf=512, nc=2048 (TU reformulation, next row f2)",
            make=lambda s: facility_location(512, 2048, s, name="cfg7_facility_512x2048")),
    # next row f3: 3D assignment n = 64 (262,144 binaries, 192 equality rows) for Alg. 4 sampling
    8: dict(desc="3D assignment n=64 (customised sampling, next row f3)",
            make=lambda s: assignment3d(64, s, name="cfg8_assign3d_64")),
}

SMALL = {
    "setcover": lambda s: set_cover(600, 2000, 2, 98, s, "small_setcover"),
    "mis": lambda s: max_independent_set(700, 0.01, s, name="small_mis"),
    "mkp": lambda s: multi_knapsack(3000, 6, 0.5, s, "small_mkp"),
    "bqp": lambda s: assignment_bqp(12, 15, 4, s, "small_bqp"),
    "general": lambda s: random_general(300, 80, 20, 12, s, with_q=True, name="small_general"),
    "real": lambda s: random_general(200, 60, 10, 10, s, real=True, with_q=True, name="small_real"),
    "maxcut": lambda s: max_cut(300, 0.5, s, name="small_maxcut"),
    "dense_psd": lambda s: dense_laplacian(200, 0.5, 40, s, name="small_dense_psd"),
    "facility": lambda s: facility_location(6, 24, s, name="small_facility"),
    "assign3d": lambda s: assignment3d(8, s, name="small_assign3d"),
}


def make_config(cfg: int, seed: int = 1):
    return CONFIGS[cfg]["make"](seed)


def p_vectors(n, seed, x_traj=None):
    """Sampling-only probability vectors: uniform, 90/10 mix of exact {0,1} and U(0,1)."""
    rng = _rng(seed)
    unif = rng.random(n)
    mix = np.where(rng.random(n) < 0.9, (rng.random(n) < 0.5).astype(np.float64), rng.random(n))
    out = {"unif": unif, "mix": mix}
    if x_traj is not None:
        out["traj"] = np.asarray(x_traj, dtype=np.float64)
    return out
