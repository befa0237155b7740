"""Pins of the oracle's TUReformulate (oracle/tu.py; PAPER §2.4.1 Theorem L823-846)
against what the theorem fixes: the SPEC worked example, exactness by brute-force enumeration (the
optimal values of the original and of the reduced + lifted problem are equal), and objective /
feasibility consistency z'(xbar) = z(lift(xbar)) on every binary point.  CPU only."""
import numpy as np
import pytest

from gen import instances as G
from oracle import oracle as O
from oracle.tu import tu_reformulate
from tests.util import all_points, brute_force, exhaustive_bits, inst_from_dense


def test_spec_example():
    """B = [[1,1]], d = 1, c = (2,1), J = {0}, I = {0}: s = 1, S = (-1); reduced objective
    -x2 + 2; optimum x2 = 1, lifted x = (0,1), objective 1 = brute force of the original."""
    inst = inst_from_dense([[1.0, 1.0]], [1.0], [0], [2.0, 1.0])
    red, lift = tu_reformulate(inst, [0], [0])
    assert red["n"] == 1 and np.array_equal(red["c"], [-1.0]) and red["c0"] == 2.0
    assert red["m"] == 0  # both box rows (-x2 >= -1, x2 >= 0) hold for every binary x2: dropped (R24)
    assert np.array_equal(lift([1]), [0, 1]) and np.array_equal(lift([0]), [1, 0])
    zb, xb, _, _ = brute_force(inst)
    zr, xr, _, _ = brute_force(red)
    assert zb == zr == 1.0 and np.array_equal(lift(xr), xb)


def test_singular_and_nonintegral_rejected():
    inst = inst_from_dense([[1.0, 1.0], [1.0, 1.0]], [1.0, 1.0], [0, 0], [1.0, 1.0])
    with pytest.raises(ValueError):
        tu_reformulate(inst, [0, 1], [0, 1])
    inst = inst_from_dense([[1.0, 1.0]], [1.0], [1], [1.0, 1.0])
    with pytest.raises(ValueError):
        tu_reformulate(inst, [0], [0])  # J must be equality rows


def _random_tu_instance(seed):
    """Tiny instance with a certified TU block: disjoint +-1 equality rows (GUB rows; every column
    has at most one nonzero in B_J -> TU), plus random general rows and an indefinite Q."""
    rng = np.random.default_rng(seed)
    n = 11
    perm = rng.permutation(n)
    groups = [perm[:3], perm[3:6], perm[6:8]]
    K, r, sense = [], [], []
    J, I = [], []
    for g in groups:
        row = np.zeros(n)
        sg = rng.choice([-1.0, 1.0], size=g.size)
        row[g] = sg
        K.append(row); r.append(float(rng.integers(-1, 2))); sense.append(0)
        J.append(len(K) - 1); I.append(int(g[rng.integers(0, g.size)]))
    for _ in range(4):
        row = np.zeros(n)
        idx = rng.choice(n, size=4, replace=False)
        row[idx] = rng.integers(-3, 4, size=4)
        K.append(row); r.append(float(rng.integers(-2, 3))); sense.append(int(rng.choice([1, -1, 0])))
    Qd = rng.integers(-3, 4, size=(n, n)).astype(float)
    Qd = np.triu(Qd) + np.triu(Qd, 1).T
    order = rng.permutation(len(K))  # J rows anywhere in the input
    K = [K[k] for k in order]; r = [r[k] for k in order]; sense = [sense[k] for k in order]
    J = [int(np.flatnonzero(order == j)[0]) for j in J]
    inst = inst_from_dense(K, r, sense, rng.integers(-9, 10, size=n).astype(float), Q=Qd,
                           c0=float(rng.integers(-3, 4)), maximize=bool(seed % 2))
    return inst, J, I


@pytest.mark.parametrize("seed", range(12))
def test_exactness_by_enumeration(seed):
    """Theorem (PAPER): the reformulation is exact.  Brute force of the original equals brute
    force of the reduced problem, and for every binary xbar: xbar feasible for the reduced problem
    <=> lift(xbar) feasible for the original (x_I binary), with equal objectives."""
    inst, J, I = _random_tu_instance(seed)
    red, lift = tu_reformulate(inst, J, I)
    zb, _, okb, _ = brute_force(inst)
    zr, xr, okr, zur = brute_force(red)
    if zb is None:
        assert zr is None
        return
    assert zr == zb
    o = O.Oracle(inst)
    X = all_points(red["n"])
    for l in range(X.shape[0]):
        if not okr[l]:
            continue
        x = lift(X[l])
        f, z = o.eval_point(x)
        assert f and (-z if inst["maximize"] else z) == zur[l]
    # every feasible original point is the lift of a feasible reduced point (J rows fix x_I)
    assert okb.sum() == okr.sum()


def test_facility_location_exact_small():
    inst = G.facility_location(2, 5, 3)
    red, lift = tu_reformulate(inst, inst["tu_rows"], inst["tu_cols"])
    assert red["n"] == inst["n"] - 5
    assert np.all(red["sense"][: inst["m"] - 5] == -1)  # the y_ij <= x_i rows keep their sense
    zb, xb, _, _ = brute_force(inst)
    zr, xr, _, _ = brute_force(red)
    assert zb == zr
    f, z = O.Oracle(inst).eval_point(lift(xr))
    assert f and z == zb


def _interval_tu_instance(seed):
    """Tiny instance whose J rows are overlapping intervals (consecutive ones) over a column order:
    an interval matrix is TU, and with I_t = the first column of interval t (distinct starts) B_JI is
    unit triangular but NOT a permutation (later intervals cover earlier starts).  Plus random
    general rows and an indefinite Q."""
    rng = np.random.default_rng(100 + seed)
    n = 10
    order = rng.permutation(n)
    K, r, sense, J, I = [], [], [], [], []
    starts = [0, 2, 3]
    for t, a in enumerate(starts):
        b = a + int(rng.integers(3, 5))
        row = np.zeros(n)
        row[order[a:b]] = 1.0
        K.append(row); r.append(1.0); sense.append(0)
        J.append(len(K) - 1); I.append(int(order[a]))
    for _ in range(3):
        row = np.zeros(n)
        idx = rng.choice(n, size=4, replace=False)
        row[idx] = rng.integers(-3, 4, size=4)
        K.append(row); r.append(float(rng.integers(-2, 3))); sense.append(int(rng.choice([1, -1])))
    Qd = rng.integers(-2, 3, size=(n, n)).astype(float)
    Qd = np.triu(Qd) + np.triu(Qd, 1).T
    inst = inst_from_dense(K, r, sense, rng.integers(-9, 10, size=n).astype(float), Q=Qd,
                           c0=float(rng.integers(-3, 4)), maximize=bool(seed % 2))
    return inst, J, I


@pytest.mark.parametrize("seed", range(8))
def test_general_bji_exactness_by_enumeration(seed):
    """The theorem for a NON-permutation B_JI (the case the paper applies with an LU of
    B_JI): B_JI really is not a signed permutation here, and the reduced problem is exact — brute
    force optima equal, and every feasible reduced point lifts to a feasible original point with the
    same objective, one to one."""
    inst, J, I = _interval_tu_instance(seed)
    Kd = G.dense_K(inst)
    BJI = Kd[np.ix_(J, I)]
    assert np.count_nonzero(BJI) > len(J)  # not a permutation
    red, lift = tu_reformulate(inst, J, I)
    zb, _, okb, _ = brute_force(inst)
    zr, xr, okr, zur = brute_force(red)
    assert (zb is None) == (zr is None)
    if zb is None:
        return
    assert zr == zb
    o = O.Oracle(inst)
    X = all_points(red["n"])
    for l in np.flatnonzero(okr):
        f, z = o.eval_point(lift(X[l]))
        assert f and (-z if inst["maximize"] else z) == zur[l]
    assert okb.sum() == okr.sum()


def test_facility_location_slack_form_removes_every_row():
    """Reading R24 (round 2): with binary slacks the facility-location constraints are all equalities
    of a TU matrix; eliminating them (B_JI unit triangular) leaves only box rows, and the optimum is
    the facility-location optimum (brute force of the inequality form, nf = 2, nc = 3)."""
    fl = G.facility_location(2, 3, 5)
    sl = G.facility_location_slack(2, 3, 5)
    red, lift = tu_reformulate(sl, sl["tu_rows"], sl["tu_cols"])
    assert red["n"] == fl["n"] - 3          # x_i and the non-cheapest y_ij remain
    assert np.all(red["sense"] == 1)         # only the box rows of x_I = s + S x_Ibar are left
    zb, xb, _, _ = brute_force(fl)
    zr, xr, _, _ = brute_force(red)
    assert zr == zb
    x = lift(xr)
    f, z = O.Oracle(fl).eval_point(x[: fl["n"]])
    assert f and z == zb
