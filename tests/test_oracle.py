"""Pins of the CPU oracle against what the paper and mathematics fix (never against itself).

Each test names the passage it pins.  CPU only (runs under -m "not gpu").
"""
import json
import math
import os

import numpy as np
import pytest

from gen import instances as G
from oracle import oracle as O
from tests.util import all_points, brute_force, exhaustive_bits, inst_from_dense

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))


# ----------------------------------------------------------------------------- Philox / sampling
def test_philox_known_answers():
    """Random123 KAT (tests/golden/philox_kat.txt) pins the generator of reading R10."""
    for line in open(os.path.join(GOLD, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(t, 16) for t in line.split()]
        out = O.philox(v[0:4], v[4:6])
        assert [int(a) for a in out] == v[6:10]


def _planes(i, w, rnd, seed, q):
    out = O.philox([i, w, q, rnd], [seed & 0xFFFFFFFF, seed >> 32])
    p0 = int(out[0]) | (int(out[1]) << 32)
    p1 = int(out[2]) | (int(out[3]) << 32)
    return p0, p1


def test_sample_dyadic_thresholds_closed_form():
    """PAPER L753 Bernoulli(p_i) under the MSB-first plane contract: for p = 1/2 the sample is
    [u < 2^31] = NOT plane0; p = 1/4 -> NOT plane0 AND NOT plane1; p = 3/4 -> NOT(plane0 AND plane1)."""
    seed, rnd = 0x123456789ABCDEF, 7
    p = np.array([0.5, 0.25, 0.75, 0.0, 1.0])
    bits = O.sample(p, seed, rnd, 3, 2)
    M = (1 << 64) - 1
    for w in range(2):
        for i in range(5):
            p0, p1 = _planes(i, 3 + w, rnd, seed, 0)
            expect = [~p0 & M, ~p0 & ~p1 & M, ~(p0 & p1) & M, 0, M][i]
            assert int(bits[i, w]) == expect


def _uniform(i, w, rnd, seed, b):
    """u of (variable i, lane 64w+b) assembled from all 32 planes, plane 0 the MSB (App. B)."""
    u = 0
    for q in range(16):
        p0, p1 = _planes(i, w, rnd, seed, q)
        u = (u << 1) | ((p0 >> b) & 1)
        u = (u << 1) | ((p1 >> b) & 1)
    return u


def test_sample_non_dyadic_threshold_by_hand():
    """Bernoulli(p) = [u < ceil(p 2^32)] (reading R10) for NON-dyadic p, where the lazy
    MSB-first compare has to look past the first planes: every lane is recomputed from the 32 Philox
    planes (generator pinned by the KAT above) and compared with the integer threshold worked by hand.
    0.3 * 2^32 = 1288490188.8 -> T = 1288490189; 0.7 -> 3006477107.2 -> 3006477108; 1/3 ->
    1431655765.33 -> 1431655766; and p = 1288490189 / 2^32 (T exactly, no rounding) gives the same
    bits as 0.3."""
    seed, rnd, w0 = 0xDEADBEEF12345, 5, 2
    T = {0.3: 1288490189, 0.7: 3006477108, 1.0 / 3.0: 1431655766, 1288490189 / 2**32: 1288490189}
    ps = np.array(list(T))
    bits = O.sample(ps, seed, rnd, w0, 2)
    for i, p in enumerate(ps):
        assert math.ceil(p * 2**32) == T[p]
        for w in range(2):
            expect = 0
            for b in range(64):
                if _uniform(i, w0 + w, rnd, seed, b) < T[p]:
                    expect |= 1 << b
            assert int(bits[i, w]) == expect
    # equal thresholds -> equal decisions on the same stream (variable 0 at p = 0.3 and at T/2^32)
    same = O.sample(np.array([0.3]), seed, rnd, w0, 2)
    exact = O.sample(np.array([1288490189 / 2**32]), seed, rnd, w0, 2)
    assert np.array_equal(same, exact)


def test_sample_constant_and_statistics():
    """p = 0 -> zeros, p = 1 -> ones; column means within 4 sqrt(p(1-p)/k)."""
    p = np.array([0.0, 1.0, 0.5, 0.1, 0.9, 0.37])
    k_words = 160  # 10240 samples
    bits = O.sample(p, 2025, 3, 0, k_words)
    assert not bits[0].any()
    assert (bits[1] == np.uint64(0xFFFFFFFFFFFFFFFF)).all()
    k = 64 * k_words
    for i in range(2, 6):
        mean = sum(bin(int(w)).count("1") for w in bits[i]) / k
        assert abs(mean - p[i]) <= 4 * math.sqrt(p[i] * (1 - p[i]) / k)


def test_sample_rank_invariance():
    """Disjoint word ranges compose: words [0,4) == [0,2) ++ [2,4) (sharding contract)."""
    p = np.random.default_rng(0).random(50)
    full = O.sample(p, 5, 11, 0, 4)
    a = O.sample(p, 5, 11, 0, 2)
    b = O.sample(p, 5, 11, 2, 2)
    assert np.array_equal(full, np.concatenate([a, b], axis=1))


# ----------------------------------------------------------------------------- spectral norm / preprocess
def _csr(M):
    M = np.asarray(M, dtype=np.float64)
    ptr = [0]; col = []; val = []
    for row in M:
        nz = np.nonzero(row)[0]
        col += list(nz); val += list(row[nz]); ptr.append(len(col))
    return np.array(ptr), np.array(col, dtype=np.int32), np.array(val), M.shape


@pytest.mark.parametrize("ex", SPEC["spectral_norm"])
def test_spectral_norm_spec(ex):
    ptr, col, val, (r, c) = _csr(ex["M"])
    # power iteration stops at relative change 1e-7: accuracy 1e-6 relative
    assert abs(O.spectral_norm(ptr, col, val, r, c) - ex["expect"]) <= 1e-6 * max(1.0, ex["expect"])


def test_spectral_norm_random_and_null_start():
    """matches a dense singular-value solver to 1e-5; [[1,-1]] (all-ones start in the null
    space) is handled by the restart of reading R5 and gives sqrt(2)."""
    rng = np.random.default_rng(3)
    for t in range(5):
        M = rng.standard_normal((20, 20)) * (rng.random((20, 20)) < 0.3)
        ptr, col, val, (r, c) = _csr(M)
        est = O.spectral_norm(ptr, col, val, r, c, tol=1e-12, max_iter=5000)
        assert abs(est - np.linalg.norm(M, 2)) <= 1e-5 * np.linalg.norm(M, 2)
        assert est <= np.linalg.norm(M, 2) * (1 + 1e-12)  # never overestimates
    ptr, col, val, (r, c) = _csr([[1.0, -1.0]])
    assert abs(O.spectral_norm(ptr, col, val, r, c) - math.sqrt(2)) <= 1e-9


def test_preprocess_spec_examples():
    """SPEC L135-136 / PAPER L15-17."""
    ex = SPEC["preprocess"][0]
    # saddle K = -K_u -> user form K_u = -[[3,4]], r = 5
    inst = inst_from_dense(-np.array(ex["K_saddle"]), ex["r"], [1], [1.0, 1.0])
    o = O.Oracle(inst)
    rec = o.preprocess()
    K, r, _, _ = o.scaled_dense()
    assert np.allclose(K, ex["expect_K"], atol=1e-12) and np.allclose(r, ex["expect_r"], atol=1e-12)
    assert abs(rec["k_scale"] - ex["expect_k_scale"]) <= 1e-9
    ex = SPEC["preprocess"][1]
    o = O.Oracle(inst_from_dense([], [], [], ex["c"]))
    rec = o.preprocess()
    _, _, _, c = o.scaled_dense()
    assert np.allclose(c, ex["expect_c"]) and abs(rec["obj_scale"] - ex["expect_obj_scale"]) <= 1e-12


@pytest.mark.parametrize("fam", ["general", "bqp", "mis"])
def test_preprocess_invariants(fam):
    """after Preprocess ||K||_2 = 1 (+-1e-6); K = -D^{-1}K_u/kappa with
    D the row 2-norms; (Q,c) divided by ||Q||_2 + ||c||_2 (dense numpy references)."""
    inst = G.SMALL[fam](4)
    o = O.Oracle(inst)
    rec = o.preprocess(tol=1e-10, max_iter=5000)
    K, r, Qs, cs = o.scaled_dense()
    assert abs(np.linalg.norm(K, 2) - 1.0) <= 1e-6
    Ku = G.dense_K(inst)[o.row_perm()]
    sgn = np.where(inst["sense"][o.row_perm()] == -1, -1.0, 1.0)
    Ku = Ku * sgn[:, None]
    s = np.linalg.norm(Ku, axis=1)
    s[s == 0] = 1
    assert np.allclose(K, -Ku / s[:, None] / rec["k_scale"], rtol=1e-12, atol=1e-15)
    Q = G.dense_Q(inst) * (-1 if inst["maximize"] else 1)
    c = inst["c"] * (-1 if inst["maximize"] else 1)
    omega = (np.linalg.norm(Q, 2) if Q.any() else 0.0) + np.linalg.norm(c)
    assert abs(rec["obj_scale"] - omega) <= 1e-6 * omega
    assert np.allclose(Qs * rec["obj_scale"], Q, atol=1e-9) and np.allclose(cs * rec["obj_scale"], c)


def test_preprocess_preserves_feasible_set_and_argmin():
    """row scaling by positive numbers keeps the feasible set; objective scaling keeps argmin."""
    inst = G.random_general(10, 6, 2, 5, 7, with_q=True)
    o = O.Oracle(inst)
    rec = o.preprocess()
    K, r, Qs, cs = o.scaled_dense()
    _, _, ok, z = brute_force(inst)
    from tests.util import all_points
    X = all_points(10).astype(float)
    g = X @ K.T + r  # a GE row holds iff (Kx + r)_j <= 0, an EQ row iff = 0
    m1 = o.m1
    ok2 = (g[:, :m1] <= 1e-12).all(1) & (np.abs(g[:, m1:]) <= 1e-12).all(1)
    assert np.array_equal(ok, ok2)
    zs = np.einsum("li,ij,lj->l", X, Qs, X) + X @ cs
    assert np.allclose(zs * rec["obj_scale"] + inst["c0"], z, atol=1e-9)


# ----------------------------------------------------------------------------- UpdatePenalty
def test_rho_schedule_spec_and_invariants():
    """PAPER L28-31; SPEC L272-274 worked values; monotone and within [rho_min, rho_max]."""
    e = SPEC["update_penalty"]
    rho = O.rho_schedule(e["rho_min"], e["rho_max"], e["T"], e["p"], e["delta"], 1001)
    for t, v in e["expect"].items():
        assert abs(rho[int(t)] - v) <= 1e-12
    rng = np.random.default_rng(1)
    for _ in range(2000):
        rmin = 10 ** rng.uniform(-4, 0); rmax = rmin * 10 ** rng.uniform(0, 3)
        T = rng.uniform(1, 200); p = rng.uniform(0.2, 3); d = 10 ** rng.uniform(-8, -1)
        rho = O.rho_schedule(rmin, rmax, T, p, d, 50)
        assert (np.diff(rho) >= 0).all() and (rho >= rmin).all() and (rho <= rmax).all()
        t = np.arange(50)
        free = rmin * (1 + t / T) ** p
        prev = np.concatenate([[rmin], rho[:-1]])
        unclipped = (free >= prev + d) & (free <= rmax)
        assert np.allclose(rho[unclipped], free[unclipped], rtol=1e-14)


# ----------------------------------------------------------------------------- Alg. 2
@pytest.mark.parametrize("ex", SPEC["first_order_step"])
def test_step_spec_examples(ex):
    n = ex["n"]
    m = len(ex["K_u"])
    inst = inst_from_dense(ex["K_u"], ex["r"], [1] * m, ex["c"])
    o = O.Oracle(inst)
    o.preprocess()
    o.set_state(ex["x"], ex["xbar"], ex["y"])
    o.step(ex["rho"], ex["tau1"], ex["tau2"])
    x, xb, y = o.get_state()
    assert np.allclose(x, ex["expect_x"], atol=1e-15)
    if "expect_y" in ex:
        assert np.allclose(y, ex["expect_y"], atol=1e-15)


def _lagr(K, r, Q, c, rho, x, y):
    """L^(x;y) = <x,Qx> + <c,x> + <y,Kx+r> + rho<x,1-x>  (eq. saddle)."""
    return x @ Q @ x + c @ x + y @ (K @ x + r) + rho * x @ (1 - x)


@pytest.mark.parametrize("seed", [1, 2])
def test_step_gradients_vs_finite_differences(seed):
    """Alg. 2 lines 1-2 against central finite differences of L^:
    interior point + small tau1 -> (x - x+)/tau1 = grad_x L^(x, y+); (y+ - y)/tau2 = grad_y L^(xbar, y)."""
    inst = G.random_general(12, 6, 3, 6, seed, with_q=True)
    o = O.Oracle(inst)
    o.preprocess()
    K, r, Q, c = o.scaled_dense()
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.3, 0.7, 12); xb = rng.uniform(0.3, 0.7, 12); y = rng.uniform(5, 6, o.m)
    rho, t1, t2 = 0.37, 1e-4, 1e-4
    o.set_state(x, xb, y)
    o.step(rho, t1, t2)
    x1, _, y1 = o.get_state()
    h = 1e-5
    gx = np.array([(_lagr(K, r, Q, c, rho, x + h * e, y1) - _lagr(K, r, Q, c, rho, x - h * e, y1)) / (2 * h)
                   for e in np.eye(12)])
    gy = np.array([(_lagr(K, r, Q, c, rho, xb, y + h * e) - _lagr(K, r, Q, c, rho, xb, y - h * e)) / (2 * h)
                   for e in np.eye(o.m)])
    assert np.allclose((x - x1) / t1, gx, rtol=1e-6, atol=1e-6)
    assert np.allclose((y1 - y) / t2, gy, rtol=1e-6, atol=1e-6)
    _, xb1, _ = o.get_state()
    assert np.array_equal(xb1, 2 * x1 - x)


def test_projection_invariants():
    """Iterates stay in the box and inequality duals stay >= 0."""
    inst = G.SMALL["general"](2)
    o = O.Oracle(inst)
    o.preprocess()
    o.state_init()
    rho = O.rho_schedule(1e-3, 10, 100, 2, 1e-6, 100)
    for k in range(300):
        o.step(rho[k // 10] * 50, 0.99 ** 0.5, 0.99 ** 0.5)
        x, _, y = o.get_state()
        assert (x >= 0).all() and (x <= 1).all() and (y[: o.m1] >= 0).all()


def test_box_qp_closed_form():
    """Convex separable QP over the box: min q_i x_i^2 + c_i x_i on [0,1] has
    x*_i = clip(-c_i/(2 q_i), 0, 1); PDHG with rho = 0, no K, reaches it to 1e-4."""
    rng = np.random.default_rng(5)
    n = 30
    q = rng.uniform(1, 4, n); c = rng.uniform(-10, 3, n)
    inst = inst_from_dense([], [], [], c, Q=np.diag(q))
    o = O.Oracle(inst)
    o.preprocess()
    o.state_init()
    tau = math.sqrt(0.2)
    for _ in range(10000):
        o.step(0.0, tau, tau)
    x, _, _ = o.get_state()
    assert np.abs(x - np.clip(-c / (2 * q), 0, 1)).max() <= 1e-4


def test_lp_relaxation_vs_linprog():
    """Thm. 1 convex case: with Q = 0, rho = 0 the iterates approach an LP optimum;
    objective checked against scipy.optimize.linprog (HiGHS)."""
    from scipy.optimize import linprog
    inst = G.make_config(1, 3)
    o = O.Oracle(inst)
    rec = o.preprocess()
    o.state_init()
    tau = math.sqrt(0.25)
    for _ in range(20000):
        o.step(0.0, tau, tau)
    x, _, _ = o.get_state()
    K = G.dense_K(inst)
    lp = linprog(inst["c"], A_ub=-K, b_ub=-inst["r"], bounds=[(0, 1)] * inst["n"], method="highs")
    assert abs(inst["c"] @ x - lp.fun) <= 1e-3 * abs(lp.fun)
    ind = o.indicators(0.0, tau, tau)
    assert ind["primal_gap"] <= 1e-4


def test_tu_assignment_integral_vs_linear_sum_assignment():
    """TU instance with integral LP optimum: 6x6 assignment with Q = 0, rho = 0;
    round(x_k) equals scipy.optimize.linear_sum_assignment's unique optimum."""
    from scipy.optimize import linear_sum_assignment
    rng = np.random.default_rng(11)
    a = 6
    cost = rng.permutation(np.arange(1, a * a + 1)).astype(float).reshape(a, a) * 7 + rng.integers(0, 3, (a, a))
    n = a * a
    K = np.zeros((2 * a, n))
    for i in range(a):
        K[i, i * a:(i + 1) * a] = 1
        K[a + i, np.arange(a) * a + i] = 1
    inst = inst_from_dense(K, np.ones(2 * a), np.zeros(2 * a), cost.reshape(-1))
    o = O.Oracle(inst)
    o.preprocess()
    o.state_init()
    tau = math.sqrt(0.25)
    for _ in range(30000):
        o.step(0.0, tau, tau)
    x, _, _ = o.get_state()
    ri, ci = linear_sum_assignment(cost)
    X = np.zeros((a, a)); X[ri, ci] = 1
    assert np.array_equal((x >= 0.5).astype(float).reshape(a, a), X)


def test_indicators_closed_values():
    """binary x -> binary gap 0; x = 0.5*1, n = 4 -> 0.25.  Fixed point (rho = Q = c = 0,
    no K) -> s^x = 0."""
    o = O.Oracle(inst_from_dense([], [], [], [0.0] * 4))
    o.preprocess()
    o.set_state([0.5] * 4, [0.5] * 4, [])
    o.step(0.0, 0.5, 0.5)
    ind = o.indicators(0.0, 0.5, 0.5)
    assert abs(ind["binary_gap"] - 0.25) <= 1e-15 and ind["sx"] == 0.0
    o.set_state([0, 1, 1, 0], [0, 1, 1, 0], [])
    o.step(0.0, 0.5, 0.5)
    assert o.indicators(0.0, 0.5, 0.5)["binary_gap"] == 0.0


def test_indicators_match_definition_dense():
    """Thm. 2 residuals from their gradient definition with dense numpy algebra,
    and SPEC L220 primal gap."""
    inst = G.random_general(15, 5, 3, 6, 4, with_q=True)
    o = O.Oracle(inst)
    o.preprocess()
    K, r, Q, c = o.scaled_dense()
    rng = np.random.default_rng(2)
    x0 = rng.random(15); xb0 = rng.random(15); y0 = np.abs(rng.random(o.m))
    o.set_state(x0, xb0, y0)
    rho, t1, t2 = 0.2, 0.3, 0.4
    o.step(rho, t1, t2)
    x1, _, y1 = o.get_state()
    ind = o.indicators(rho, t1, t2)

    def gx(x, y):
        return c + rho + K.T @ y + 2 * Q @ x - 2 * rho * x  # eq:dy

    def gy(x):
        return K @ x + r
    sx = (x0 - x1) / t1 + gx(x1, y1) - gx(x0, y1)
    sy = (y0 - y1) / t2 - gy(x1) + gy(xb0)
    g = K @ x1 + r
    pg = max(np.maximum(g[: o.m1], 0).max(initial=0), np.abs(g[o.m1:]).max(initial=0))
    pg = np.maximum(g[: o.m1], 0).max(initial=0) + np.abs(g[o.m1:]).max(initial=0)
    assert abs(ind["sx"] - np.linalg.norm(sx)) <= 1e-10 * max(1, np.linalg.norm(sx))
    assert abs(ind["sy"] - np.linalg.norm(sy)) <= 1e-10 * max(1, np.linalg.norm(sy))
    assert abs(ind["primal_gap"] - pg) <= 1e-12
    assert abs(ind["binary_gap"] - (x1 @ (1 - x1)) / 15) <= 1e-15


# ----------------------------------------------------------------------------- EvalBest
def test_eval_spec_examples():
    e = SPEC["eval_best"]
    o = O.Oracle(inst_from_dense(e["K_u"], e["r"], [1], e["c"]))
    f, z = o.eval_point(np.array(e["batch"][0], dtype=np.uint8))
    assert f and z == e["expect_z"]
    f, _ = o.eval_point(np.array(e["infeasible"], dtype=np.uint8))
    assert not f
    for ex in SPEC["objective"]:
        o = O.Oracle(inst_from_dense([], [], [], ex["c"], Q=ex["Q"]))
        assert o.eval_point(np.array(ex["x"], dtype=np.uint8)) == (True, ex["expect"])
    k = SPEC["knapsack_n2"]
    inst = inst_from_dense([k["w"]], [k["W"]], [-1], k["v"], maximize=True)
    zb, xb, _, _ = brute_force(inst)
    assert zb == k["expect_value"] and list(xb) == k["expect_x"]
    o = O.Oracle(inst)
    f, z = o.eval_point(np.array(k["expect_x"], dtype=np.uint8))
    assert f and z == -k["expect_value"]  # canonical minimisation value


@pytest.mark.parametrize("fam,seed", [("cfg1", 1), ("cfg1", 2), ("general", 3), ("mis", 4), ("real", 5)])
def test_eval_exhaustive_equals_brute_force(fam, seed):
    """EvalBest on the exhaustive batch of all 2^n points equals enumeration with dense algebra
    (SURVEY §8(c) pin)."""
    if fam == "cfg1":
        inst = G.make_config(1, seed)
    elif fam == "general":
        inst = G.random_general(12, 8, 3, 6, seed, with_q=True)
    elif fam == "mis":
        inst = G.max_independent_set(14, 0.3, seed, weighted=True)
    else:
        inst = G.random_general(10, 6, 2, 5, seed, real=True, with_q=True)
    n = inst["n"]
    zb, xb, ok, zu = brute_force(inst)
    o = O.Oracle(inst)
    feas, z = o.eval(exhaustive_bits(n))
    assert np.array_equal(feas.astype(bool), ok)
    sign = -1.0 if inst["maximize"] else 1.0
    if o.integral:
        assert np.array_equal(z, sign * zu)
    else:
        assert np.allclose(z, sign * zu, rtol=1e-12, atol=1e-9)
    if zb is not None:
        assert abs(z[feas.astype(bool)].min() - sign * zb) <= 1e-9


@pytest.mark.parametrize("seed", [1, 2])
def test_maxcut_qp_equals_cut_definition(seed):
    """Max cut (next row f1): the oracle's EvalBest of the QP form on all 2^n points
    equals the cut weight sum_{i<j} w_ij [x_i != x_j] computed from the edge weights by definition,
    and its best lane is the maximum cut found by enumerating bipartitions directly."""
    n = 13
    inst = G.max_cut(n, 0.5, seed)
    Wd = -G.dense_Q(inst)  # user Q_ij = -w_ij
    assert np.all(np.diag(Wd) == 0) and np.array_equal(Wd, Wd.T)
    assert np.abs(Wd).max() <= 10 and Wd.min() >= -8
    o = O.Oracle(inst)
    feas, z = o.eval(exhaustive_bits(n))
    assert feas.all()
    pts = all_points(n).astype(bool)
    cuts = np.array([Wd[np.ix_(x, ~x)].sum() for x in pts])
    assert np.array_equal(-z, cuts)  # canonical minimisation value = -cut
    assert -z.min() == cuts.max()


def test_brute_force_vs_milp():
    """The enumeration helper itself agrees with scipy's MILP solver (HiGHS) on config 1."""
    from scipy.optimize import Bounds, LinearConstraint, milp
    for seed in (1, 2):
        inst = G.make_config(1, seed)
        zb, _, _, _ = brute_force(inst)
        K = G.dense_K(inst)
        res = milp(inst["c"], constraints=LinearConstraint(K, inst["r"], np.inf),
                   integrality=np.ones(inst["n"]), bounds=Bounds(0, 1))
        assert abs(res.fun - zb) <= 1e-9


def test_validation_errors():
    """bad CSR, explicit zeros, asymmetric Q, bad sense are input errors."""
    good = inst_from_dense([[1, 1]], [1], [1], [1.0, 2.0])
    bad = dict(good, k_col=np.array([1, 0], dtype=np.int32))
    with pytest.raises(ValueError):
        O.Oracle(bad)
    bad = dict(good, k_val=np.array([1.0, 0.0]))
    with pytest.raises(ValueError):
        O.Oracle(bad)
    bad = dict(good, sense=np.array([3], dtype=np.int8))
    with pytest.raises(ValueError):
        O.Oracle(bad)
    with pytest.raises(ValueError):
        O.Oracle(inst_from_dense([], [], [], [1.0, 1.0], Q=[[0, 1], [2, 0]]))


# ----------------------------------------------------------------------------- CheckHalt
def test_halt_semantics():
    """SPEC L281-283 (reading R9)."""
    h = O.HaltState(window=5)
    assert [h.push(0, 0, 0, False) for _ in range(5)] == [False] * 4 + [True]
    h = O.HaltState(window=5)
    res = [h.push(1, 1, 0.1 + 0.05 * (k % 2), False) for k in range(20)]
    assert not any(res)  # oscillating binary gap, above tolerance
    h = O.HaltState(window=5)
    res = [h.push(0.5, 0.5, 0.5, k == 3) for k in range(12)]
    assert res.index(True) == 8  # stalled from check 5, but needs 5 checks without improvement after k=3
    h = O.HaltState(window=5)
    assert not any(h.push(1 + k, 0, 0, False) for k in range(10))  # growing primal gap never stalls


# ----------------------------------------------------------------------------- Alg. 1 end to end
def test_run_quality_vs_brute_force():
    """SPEC L738 (#8): incumbent feasible, within 10% of the enumeration optimum in >= 80% of seeds."""
    good = 0
    seeds = range(1, 11)
    for s in seeds:
        inst = G.make_config(1, s)
        zb, _, _, _ = brute_force(inst)
        o = O.Oracle(inst)
        o.preprocess()
        res = o.run(max_iters=3000)
        assert res["has_incumbent"]
        z, x = o.best()
        f, zz = o.eval_point(x)
        assert f and zz == z
        good += z <= 1.1 * zb
    assert good >= 8


def test_run_deterministic():
    """SPEC L741 (#11): identical inputs -> bit-identical traces."""
    inst = G.SMALL["bqp"](3)
    outs = []
    for _ in range(2):
        o = O.Oracle(inst)
        o.preprocess()
        outs.append(o.run(max_iters=300, trace_max=100))
    assert np.array_equal(outs[0]["trace"], outs[1]["trace"])
    assert outs[0]["z_best"] == outs[1]["z_best"]


def _alg1_by_hand(inst, prm, alt=None):
    """Alg. 1 written out from the paper for a few blocks, using only primitives
    pinned elsewhere in this file (Alg. 2 step, sampler, EvalBest): ρ from the closed form of
    PAPER L28-31 with n advancing once per block (R7) and ρ_{-1} = ρ_min (R8); x_k sampled after the
    k-th step; round_id = (k/k_int - 1)·k_r + r (R19); best lane = min z, ties lowest index, replace
    iff strictly better (R11).  `alt` switches in one plausible orchestration mistake."""
    o = O.Oracle(inst)
    o.preprocess()
    o.state_init()
    tau = math.sqrt(prm["sigma"])
    kint, kr, W = prm["k_int"], prm["k_r"], prm["k_b"] // 64
    rho, prev = [], prm["rho_min"]
    for t in range(prm["max_iters"] + 2):
        v = min(max(prm["rho_min"] * (1 + t / prm["growth_T"]) ** prm["growth_p"], prev + prm["rho_delta"]), 10.0)
        rho.append(v)
        prev = v
    if alt == "rho_minus1_is_rho0":
        rho = [prm["rho_min"]] + rho[:-1]
    zb, found, trace = math.inf, (-1, -1, -1), []
    for k in range(1, prm["max_iters"] + 1):
        r = rho[k - 1] if alt == "rho_per_iteration" else rho[(k - 1) // kint]
        x_before = o.get_state()[0].copy()
        o.step(r, tau, tau)
        if k % kint:
            continue
        x = x_before if alt == "sample_x_k_minus_1" else o.get_state()[0]
        imp = 0
        for rr in range(kr):
            rid = (k // kint - 1) * kr + rr
            if alt == "round_id_plus_1":
                rid += kr
            if alt == "round_id_ignores_r":
                rid = k // kint - 1
            f, z = o.eval(O.sample(x, prm["seed"], rid, 0, W))
            zz = np.where(f == 1, z, np.inf)
            l = int(np.argmin(zz)) if alt != "ties_highest_index" else len(zz) - 1 - int(np.argmin(zz[::-1]))
            if f[l] and (zz[l] < zb or (alt == "non_strict" and zz[l] <= zb)):
                zb, found, imp = zz[l], (k, rid, l), 1
        trace.append((k, r, zb, imp))
    return found, zb, trace


_ALTS = ["rho_minus1_is_rho0", "rho_per_iteration", "sample_x_k_minus_1", "round_id_plus_1",
         "round_id_ignores_r", "ties_highest_index", "non_strict"]


@pytest.mark.parametrize("cfg_seed,seed", [(1, 1), (4, 1), (2, 2)])
def test_run_orchestration_matches_alg1_by_hand(cfg_seed, seed):
    """orc_run's orchestration = Alg. 1 written out (4 blocks, k_int = 3, k_r = 2): same incumbent
    (iteration, round, lane, z), same per-block ρ (trace column 1) and improvement flags.  The cases
    are chosen so that each plausible mistake in `_ALTS` changes the outcome in at least one of them
    (checked below), i.e. the pin is discriminating."""
    inst = G.make_config(1, cfg_seed)
    prm = dict(sigma=0.9, k_int=3, k_r=2, k_b=64, max_iters=12, seed=seed, rho_min=0.05, growth_T=1.0,
               growth_p=1.0, rho_delta=0.01)
    o = O.Oracle(inst)
    o.preprocess()
    res = o.run(trace_max=10, **prm)
    found, zb, trace = _alg1_by_hand(inst, prm)
    assert (res["found_iter"], res["found_round"], res["found_index"]) == found
    assert res["z_best"] == zb and res["rounds"] == 4 * 2 and res["iters"] == 12
    tr = res["trace"]
    assert [int(t[0]) for t in tr] == [t[0] for t in trace] == [3, 6, 9, 12]
    assert [t[1] for t in tr] == [t[1] for t in trace]          # ρ per block, bit-exact
    assert [t[1] for t in trace] == pytest.approx([0.06, 0.1, 0.15, 0.2], rel=1e-15)  # max(0.05(1+t), ρ_prev+δ), ρ_0 = ρ_min+δ
    assert [int(t[7]) for t in tr] == [t[3] for t in trace]
    assert [t[6] for t in tr] == [t[2] for t in trace]


def test_run_orchestration_pin_is_discriminating():
    """Every alternative orchestration in _ALTS gives a different incumbent or trace on at least one
    of the cases of test_run_orchestration_matches_alg1_by_hand."""
    prm0 = dict(sigma=0.9, k_int=3, k_r=2, k_b=64, max_iters=12, rho_min=0.05, growth_T=1.0, growth_p=1.0,
                rho_delta=0.01)
    caught = set()
    for cfg_seed, seed in [(1, 1), (4, 1), (2, 2)]:
        inst = G.make_config(1, cfg_seed)
        prm = dict(prm0, seed=seed)
        ref = _alg1_by_hand(inst, prm)
        for a in _ALTS:
            alt = _alg1_by_hand(inst, prm, a)
            if alt[0] != ref[0] or [t[1:] for t in alt[2]] != [t[1:] for t in ref[2]]:
                caught.add(a)
    assert caught == set(_ALTS)


def test_run_final_round_half_goes_to_one():
    """PAPER L391 EvalBest(round(x_k)) with the tie x = 0.5 -> 1 (R13): one free variable with zero
    gradient (c = 0, no rows: g = ρ - 2ρ·0.5 = 0 exactly) stays at x0 = 0.5; with max_iters < k_int no
    sampling round happens, so the only candidate is the rounded point, x = (1), found at the last
    iteration with round = index = -1."""
    inst = inst_from_dense([], [], [], c=[0.0])
    o = O.Oracle(inst)
    o.preprocess()
    res = o.run(max_iters=3, k_int=10)
    z, x = o.best()
    assert res["rounds"] == 0 and res["has_incumbent"]
    assert (res["found_iter"], res["found_round"], res["found_index"]) == (3, -1, -1)
    assert z == 0.0 and list(x) == [1]
    assert o.get_state()[0][0] == 0.5


def test_sample_subset_is_rows_of_full_sample():
    """The bounded-sample helper draws variable idx[k] from the same Philox stream as the full
    sampler (counter word c0 = the variable index, App. B), so it equals those rows of the full batch."""
    p = np.random.default_rng(4).random(300)
    idx = np.array([0, 7, 150, 299], dtype=np.int64)
    full = O.sample(p, 77, 3, 1, 2)
    sub = O.sample_subset(p[idx], idx, 77, 3, 1, 2)
    assert np.array_equal(sub, full[idx])


def test_row_scales_are_row_norms():
    """PAPER L15 (Preprocess K1): s_j = ||K_j||_2 of the user rows (numpy.linalg.norm of the dense
    rows, in the oracle's canonical GE-first row order); zero rows keep s_j = 1."""
    inst = G.SMALL["general"](2)
    o = O.Oracle(inst)
    o.preprocess()
    K = G.dense_K(inst)[o.row_perm()]
    want = np.linalg.norm(K, axis=1)
    want[want == 0] = 1.0
    assert np.allclose(o.row_scales(), want, rtol=1e-15, atol=0)
