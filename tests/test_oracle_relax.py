"""Pins of the oracle's monotone relaxation and repair (reading R26;
next row f4).  CPU only."""
import numpy as np
import pytest

from gen import instances as G
from oracle import oracle as O
from tests.util import all_points


def _bits_from_points(X):
    """(lanes, n) 0/1 matrix -> bit-sliced (n, lanes/64) words"""
    lanes, n = X.shape
    W = (lanes + 63) // 64
    bits = np.zeros((n, W), dtype=np.uint64)
    for l in range(lanes):
        bits[:, l // 64] |= (X[l].astype(np.uint64) << np.uint64(l % 64))
    return bits


def _points(bits, lanes):
    return np.array([((bits[:, l // 64] >> np.uint64(l % 64)) & np.uint64(1)).astype(np.uint8) for l in range(lanes)])


def test_repair_spec_example():
    """3D assignment n = 2, a relaxed solution with one row doubly covered -> repair drops
    the costlier redundant triple and all equalities hold again."""
    inst = G.assignment3d(2, 1)
    c = np.full(8, 5.0)
    v = lambda i, j, k: 4 * i + 2 * j + k  # noqa: E731
    c[v(0, 1, 1)] = 9.0
    inst["c"] = c
    o = O.Oracle(inst)
    o.set_relax(1)
    x = np.zeros(8, dtype=np.uint8)
    x[[v(0, 0, 0), v(1, 1, 1), v(0, 1, 1)]] = 1
    out = _points(o.repair(_bits_from_points(np.tile(x, (64, 1)))), 1)[0]
    expect = np.zeros(8, dtype=np.uint8)
    expect[[v(0, 0, 0), v(1, 1, 1)]] = 1
    assert np.array_equal(out, expect)
    f, z = o.eval_point(out)
    assert f and z == 10.0


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_repair_minimal_monotone_cover(seed):
    """Repair only removes entries: a cover stays a cover (relaxed rows), no remaining entry can be
    removed (minimality), the cost never increases, and an uncovered row stays uncovered."""
    n = 4
    inst = G.assignment3d(n, seed)
    o = O.Oracle(inst)
    o.set_relax(1)
    rng = np.random.default_rng(seed)
    X = (rng.random((128, n ** 3)) < 0.12).astype(np.uint8)
    R = _points(o.repair(_bits_from_points(X)), 128)
    Ku = G.dense_K(inst)
    c = inst["c"]
    for x, y in zip(X, R):
        assert np.all(y <= x) and c @ y <= c @ x
        cov_x, cov_y = Ku @ x, Ku @ y
        assert np.array_equal(cov_x >= 1, cov_y >= 1)
        if np.all(cov_y >= 1):
            for i in np.flatnonzero(y):  # minimal: removing any entry uncovers a row
                assert np.any(cov_y - Ku[:, i] < 1)


def test_relax_is_the_ge_problem_for_pdhg():
    """The relaxation changes only the dual projection / primal gap of the equality rows: one PDHG
    step with relax = 1 equals a step on the same instance with those rows declared >= (rows in
    another order, so to rounding)."""
    inst = G.assignment3d(3, 5)
    o1 = O.Oracle(inst)
    o1.preprocess(tol=1e-14, max_iter=100000)
    o1.set_relax(1)
    ge = dict(inst)
    ge["sense"] = np.ones(inst["m"], dtype=np.int8)
    o2 = O.Oracle(ge)
    o2.preprocess(tol=1e-14, max_iter=100000)
    rng = np.random.default_rng(0)
    x = rng.random(27)
    y = rng.standard_normal(inst["m"]) * 0.1
    for o in (o1, o2):
        o.set_state(x, x, y)
        for _ in range(5):
            o.step(0.01, 0.9, 0.9)
    assert np.allclose(o1.get_state()[0], o2.get_state()[0], rtol=1e-12, atol=1e-14)
    assert np.allclose(o1.indicators(0.01, 0.9, 0.9)["primal_gap"], o2.indicators(0.01, 0.9, 0.9)["primal_gap"],
                       rtol=1e-12, atol=1e-14)


def test_relax_rejects_non_monotone():
    inst = G.random_general(10, 3, 2, 4, 1)
    o = O.Oracle(inst)
    with pytest.raises(RuntimeError):
        o.set_relax(1)


def test_relaxed_feasible_set_contains_original():
    """Upper closure: every feasible point of the original is feasible for the relaxed
    rows, and the relaxed optimum value is <= the original optimum (brute force, n = 2)."""
    inst = G.assignment3d(2, 7)
    Ku = G.dense_K(inst)
    P = all_points(8).astype(float)
    orig = np.all(P @ Ku.T == 1, axis=1)
    relx = np.all(P @ Ku.T >= 1, axis=1)
    assert np.all(relx[orig])
    c = inst["c"]
    assert (P[relx] @ c).min() <= (P[orig] @ c).min()


def test_repair_large_lane_is_minimal_cover():
    """SPEC L354 has no size cap: a lane holding all 21^3 = 9261 entries (more than the 8192 that
    round 1 skipped) is repaired to a minimal cover of the relaxed rows, a subset of the lane."""
    n = 21
    inst = G.assignment3d(n, 4)
    o = O.Oracle(inst)
    o.set_relax(1)
    bits = np.zeros((n ** 3, 1), dtype=np.uint64)
    bits[:, 0] = np.uint64(1)
    y = (o.repair(bits)[:, 0] & np.uint64(1)).astype(np.int64)
    Ku = G.dense_K(inst)
    cov = Ku @ y
    assert np.all(cov >= 1) and y.sum() < n ** 3
    for i in np.flatnonzero(y):
        assert np.any(cov - Ku[:, i] < 1)
